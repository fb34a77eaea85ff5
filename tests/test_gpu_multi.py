"""Multi-device contexts through the C-ABI (hcc_create_multi; north-star (5),
SURVEY.md §8e): edge-partitioned CC in one process, merged by a kernel that
reads the peers' exports in place (P2P; shards on one device read plain
device memory).  The build pool has one B200, so G shards share device 0:
the same code path as G GPUs, minus the NVLink hop.

Every case is bit-exact against the oracle (or, for RMAT-28, against the
streaming oracle's committed digest, tests/golden/big.json).
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BIG = json.loads((Path(__file__).parent / "golden" / "big.json").read_text())


@pytest.fixture(scope="module")
def multi(capi):
    ctxs = {}

    def get(G):
        if G not in ctxs:
            ctxs[G] = capi.Context(devices=[0] * G)
        return ctxs[G]
    yield get
    for c in ctxs.values():
        c.close()


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("spec", ["rmatx:scale=18,ef=16,seed=3", "erx:n=300000,m=900000,seed=2",
                                  "grid:257x300"])
def test_multi_ctx_exact(multi, oracle, G, spec):
    mc = multi(G)
    assert mc.shards == G
    g = mc.generate(spec)
    want = oracle.cc(g.n, g.edges())
    for algo in ("baseline-mj", "adaptive"):
        lab, mx = mc.cc(g, algo)
        assert np.array_equal(lab, want), (spec, G, algo)
        assert mx["components"] == int(np.sum(want == np.arange(g.n, dtype=np.uint32)))
    sm = mc.shard_metrics()
    assert len(sm) == G
    assert all(s["local_ms"] > 0 and s["merge_ms"] >= 0 for s in sm)
    g.close()


def test_multi_ctx_in_place_forest_and_verify(multi, oracle):
    mc = multi(4)
    g = mc.generate("rmatx:scale=17,ef=16,seed=9")
    want = oracle.cc(g.n, g.edges())
    f = mc.forest(g.n)
    _, mx = mc.cc(g, "baseline-mj", forest=f, labels=False)
    assert np.array_equal(f.snapshot().astype(np.uint32), want)
    assert mc.verify(g, f) == (0, 0)
    # repeated calls reuse the shard graphs and merge buffers
    for _ in range(3):
        lab, _ = mc.cc(g, "baseline-mj")
        assert np.array_equal(lab, want)
    f.close()
    g.close()


def test_multi_ctx_host_edges_io_and_stats(ctx, multi, oracle):
    """Graph entry points on a sharded graph: host upload (u32 / u64 / CSR),
    assign and async upload across shard boundaries, download, position-keyed
    checksum (shard sums add up) and whole-graph compute_stats."""
    mc = multi(3)
    e = oracle.gen_rmatx(15, 4, 0, 16 << 15)
    n = 1 << 15
    single = ctx.graph_from_edges(e, n)
    want = oracle.cc(n, e)
    for g in (mc.graph_from_edges(e, n), mc.graph_from_edges(e.astype(np.uint64), n)):
        assert g.m == e.shape[0] and g.n == n
        assert np.array_equal(g.edges(), e)
        assert np.array_equal(g.edges(1000, 70000), e[1000:71000])
        assert g.checksum() == single.checksum() == oracle.checksum_u32(e)
        assert g.stats() == single.stats()
        lab, _ = mc.cc(g, "baseline-mj")
        assert np.array_equal(lab, want)
        g.close()
    g = mc.graph_from_edges(e, n)
    e2 = oracle.gen_rmatx(15, 5, 0, 16 << 15)
    g.assign(e2)
    lab, _ = mc.cc(g, "baseline-mj")
    assert np.array_equal(lab, oracle.cc(n, e2))
    g.upload_async(e)
    lab, _ = mc.cc(g, "baseline-mj")
    assert np.array_equal(lab, want)
    g.close()
    # CSR: rows expanded in row order, then partitioned
    rng = np.random.default_rng(4)
    deg = rng.integers(0, 5, size=1000)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    col = rng.integers(0, 1000, size=int(rp[-1])).astype(np.uint32)
    g = mc.graph_from_csr(rp, col)
    ec = np.stack([np.repeat(np.arange(1000, dtype=np.uint32), deg), col], axis=1)
    assert np.array_equal(g.edges(), ec)
    lab, _ = mc.cc(g, "baseline-mj")
    assert np.array_equal(lab, oracle.cc(1000, ec))
    g.close()
    single.close()


def test_multi_ctx_pair_buffer_overflow(multi, oracle):
    """More exported pairs than the initial merge buffers hold (max(2^16,
    n/64)): the host sees the device count, grows the buffers and repeats
    the export + merge; labels stay exact."""
    mc = multi(2)
    n = 1 << 20
    v = np.arange(1, n // 2, dtype=np.uint32)
    e = np.stack([2 * v, 2 * v + 1], axis=1)  # 524 K components of 2, none with 0
    e = e[np.random.default_rng(1).permutation(e.shape[0])]
    g = mc.graph_from_edges(e, n)
    lab, _ = mc.cc(g, "baseline-mj")
    assert np.array_equal(lab, oracle.cc(n, e))
    assert max(s["pairs_exported"] for s in mc.shard_metrics()) > (1 << 16)
    g.close()


def test_multi_ctx_errors(capi, multi, ctx):
    mc = multi(2)
    g1 = ctx.generate("rmatx:scale=10,ef=4,seed=1")
    with pytest.raises(capi.HccError):  # a single-device graph on a multi context
        mc.cc(g1, "baseline-mj")
    g2 = mc.generate("rmatx:scale=10,ef=4,seed=1")
    with pytest.raises(capi.HccError):  # a sharded graph on a single context
        ctx.cc(g2, "baseline-mj")
    with pytest.raises(capi.HccError):
        capi.Context(devices=[0] * 65)
    with pytest.raises(capi.HccError):
        capi.Context(devices=[0, 99])
    g1.close()
    g2.close()


def _digest(lab: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(lab, dtype="<u4").tobytes()).hexdigest()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_rmat28_edge_partitioned_exact(capi, G):
    """BASELINE configs[4]: RMAT scale-28 (2^32 edges) edge-partitioned over G
    shards, bit-exact against the streaming oracle's digest."""
    gold = BIG["rmat28"]
    mc = capi.Context(devices=[0] * G)
    g = mc.generate(gold["spec"])
    assert g.m == 1 << 32
    assert g.checksum() == gold["edges_checksum"]
    lab, mx = mc.cc(g, "baseline-mj")
    assert mx["components"] == gold["components"]
    assert [int(lab[i]) for i in gold["sample_idx"]] == gold["sample_labels"]
    assert _digest(lab) == gold["labels_sha256"]
    g.close()
    mc.close()
