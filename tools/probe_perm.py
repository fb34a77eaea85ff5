"""Developer probe: RMAT-24 with vertex ids randomly permuted (hubs spread
over pi's lines) vs the natural ids, per-slot timeline.  Timing only."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_01178_b200 import capi  # noqa: E402


def run(ctx, g, tag, reps=5):
    best = None
    for _ in range(reps):
        _, mx = ctx.cc(g, "baseline-mj", labels=False)
        if best is None or mx["total_ms"] < best["total_ms"]:
            best = mx
            best["segs"] = ctx.segments()
    print(json.dumps(dict(kind="time", spec=tag, total_ms=best["total_ms"], segs=[
        (round(s["hook_ms"], 4), round(s["compress_ms"], 4), s["edges_in"], s["edges_out"])
        for s in best["segs"]])), flush=True)


def main():
    ctx = capi.Context(0)
    spec = sys.argv[1] if len(sys.argv) > 1 else "rmatx:scale=24,ef=16,seed=1"
    g = ctx.generate(spec)
    run(ctx, g, spec)
    e = g.edges()
    n = g.n
    g.close()
    perm = np.random.default_rng(7).permutation(n).astype(np.uint32)
    e2 = perm[e.reshape(-1).astype(np.int64)].reshape(e.shape).astype(np.uint32)
    g2 = ctx.graph_from_edges(e2, n)
    run(ctx, g2, spec + ":perm")
    # low 10 bits only: hubs stay in id order at 1024-vertex granularity
    lo = (np.arange(n, dtype=np.uint64) & ~np.uint64(1023)) | (
        np.random.default_rng(8).permutation(1024).astype(np.uint64)[np.arange(n) & 1023])
    e3 = lo.astype(np.uint32)[e.reshape(-1).astype(np.int64)].reshape(e.shape)
    g3 = ctx.graph_from_edges(e3, n)
    run(ctx, g3, spec + ":perm_low10")


if __name__ == "__main__":
    main()
