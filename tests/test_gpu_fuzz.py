"""Randomised parity sweep (1 B200): graphs of many shapes and sizes, every
engine, single- and multi-shard contexts, each label array compared with
the oracle.  The shapes mix what the hand-written cases cover one at a time:
sparse and dense random graphs, skewed (RMAT-like) endpoints, long paths in
random order, stars on the lowest and highest ids, duplicate edges and
self-loops, vertex counts around the word / summary / bitmap-floor
boundaries, and empty or single-edge graphs.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ENGINES = ["baseline-mj", "adaptive", "atomic", "baseline"]


def _graph(seed: int):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 2, 31, 33, 1000, 65535, 65536, 70001, 1 << 18, (1 << 20) - 1,
                        1 << 20, (1 << 20) + 17, 3_000_000]))
    m = int(rng.choice([0, 1, 5, n // 2 + 1, 2 * n, 8 * n, 16 * n]))
    m = min(m, 1 << 23)
    parts = []
    kinds = rng.choice(["er", "skew", "path", "star_lo", "star_hi", "dup"], size=3)
    for kind in kinds:
        k = max(1, m // 3) if m else 0
        if k == 0:
            continue
        if kind == "er":
            e = rng.integers(0, n, size=(k, 2))
        elif kind == "skew":
            # low ids far more likely (product of uniforms, RMAT-like skew)
            e = (n * rng.random((k, 2)) ** 3).astype(np.int64)
        elif kind == "path":
            perm = rng.permutation(n)
            idx = rng.integers(0, max(1, n - 1), size=k)
            e = np.stack([perm[idx], perm[np.minimum(idx + 1, n - 1)]], 1)
        elif kind == "star_lo":
            e = np.stack([np.zeros(k, np.int64), rng.integers(0, n, size=k)], 1)
        elif kind == "star_hi":
            e = np.stack([np.full(k, n - 1, np.int64), rng.integers(0, n, size=k)], 1)
        else:  # duplicates and self-loops of a small random set
            base = rng.integers(0, n, size=(max(1, k // 16), 2))
            e = base[rng.integers(0, base.shape[0], size=k)]
            loops = rng.random(k) < 0.25
            e[loops, 1] = e[loops, 0]
        flip = rng.random(e.shape[0]) < 0.5
        e[flip] = e[flip][:, ::-1]
        parts.append(e)
    e = np.concatenate(parts) if parts else np.zeros((0, 2), np.int64)
    e = e[rng.permutation(e.shape[0])] if e.shape[0] else e
    return n, e.astype(np.uint32)


@pytest.mark.parametrize("seed", range(120))
def test_random_graph_all_engines(ctx, capi, oracle, seed):
    n, e = _graph(seed)
    want = oracle.cc(n, e)
    comps = int(np.sum(want == np.arange(n, dtype=np.uint32)))
    g = ctx.graph_from_edges(e, n)
    for algo in ENGINES:
        lab, mx = ctx.cc(g, algo)
        assert np.array_equal(lab, want), (seed, n, e.shape[0], algo)
        assert mx["components"] == comps, (seed, algo)
    # the worklist engine with the star bitmap below its size floor too
    os.environ["HCC_S0B_MIN_LOG2"] = "16"
    try:
        lab, _ = ctx.cc(g, "baseline-mj")
        assert np.array_equal(lab, want), (seed, "bitmap floor 2^16")
    finally:
        os.environ.pop("HCC_S0B_MIN_LOG2", None)
    g.close()
    if n >= 2 and e.shape[0] >= 2:
        G = 2 + seed % 3
        mc = capi.Context(devices=[0] * G)
        gm = mc.graph_from_edges(e, n)
        for algo in ("baseline-mj", "adaptive"):
            lab, mx = mc.cc(gm, algo)
            assert np.array_equal(lab, want), (seed, n, e.shape[0], algo, G)
            assert mx["components"] == comps
        gm.close()
        mc.close()
