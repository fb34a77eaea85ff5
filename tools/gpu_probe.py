"""Developer probe: parity + timing sweep of the CUDA engines on one GPU.

Usage: python tools/gpu_probe.py [--quick] [--big]
Prints one JSON object per line.  Uses the oracle only as the checker.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402  (checker)
from paper_1612_01178_b200 import capi  # noqa: E402

FLAGS = {"default": 0, "full": capi.FLAG_FULL_PASSES, "hostloop": capi.FLAG_HOST_LOOP,
         "nograph": capi.FLAG_NO_GRAPH}


def emit(**kw):
    print(json.dumps(kw), flush=True)


def parity(ctx):
    cases = {
        "rmatx16": ctx.generate("rmatx:scale=16,ef=16,seed=1"),
        "grid256": ctx.generate("grid:256x256"),
        "erx16": ctx.generate("erx:n=65536,m=1048576,seed=1"),
    }
    e = O.gen_rmat(16, 16, 1)
    cases["rmat16_ref"] = ctx.graph_from_edges(e, 1 << 16)
    for name, g in cases.items():
        ed = g.edges()
        want = O.cc(g.n, ed)
        for algo in ["baseline-mj", "adaptive", "atomic", "baseline"]:
            for fl in (["hostloop", "default", "full"] if algo == "baseline-mj" else ["default"]):
                for mt in [0, 1] if g.m <= 1 << 20 else [0]:
                    if mt == 1 and algo == "baseline":
                        continue
                    t = time.time()
                    print(f"# start {name} {algo} {fl} mt={mt}", file=sys.stderr, flush=True)
                    lab, mx = ctx.cc(g, algo, segments=8, max_threads=mt, flags=FLAGS[fl])
                    ok = bool(np.array_equal(lab, want))
                    emit(kind="parity", case=name, algo=algo, flags=fl, max_threads=mt, ok=ok,
                         total_ms=mx["total_ms"], outer=mx["outer_iterations"],
                         comps=mx["components"], wall=time.time() - t)


def timing(ctx, spec, reps=5, check=True, variants=None):
    t = time.time()
    g = ctx.generate(spec)
    emit(kind="gen", spec=spec, n=g.n, m=g.m, wall=time.time() - t)
    want = None
    if check:
        t = time.time()
        want = O.cc(g.n, g.edges())
        emit(kind="oracle", spec=spec, wall=time.time() - t, comps=int(np.sum(want == np.arange(g.n, dtype=np.uint32))))
    variants = variants or [("baseline-mj", dict(first_pass_segments=s)) for s in (1, 2, 4, 8)] + [
        ("baseline-mj", dict(flags=capi.FLAG_FULL_PASSES)),
        ("adaptive", dict(segments=16)), ("atomic", {}), ("baseline", {})]
    for algo, kw in variants:
        best = None
        for r in range(reps):
            lab, mx = ctx.cc(g, algo, labels=(r == 0 and check), **kw)
            if r == 0 and check:
                ok = bool(np.array_equal(lab, want))
            if best is None or mx["total_ms"] < best["total_ms"]:
                best = mx
                best["segs"] = ctx.segments()
        m = g.m
        emit(kind="time", spec=spec, algo=algo, kw=kw, ok=ok if check else None,
             total_ms=best["total_ms"], hook_ms=best["hook_ms"], compress_ms=best["compress_ms"],
             gteps=m / best["total_ms"] / 1e6, alg_gbs=(16 * m + 12 * g.n) / best["total_ms"] / 1e6,
             outer=best["outer_iterations"], s=best["s"], edges_processed=best["edges_processed"],
             segs=[(round(s["hook_ms"], 4), round(s["compress_ms"], 4), s["edges_in"], s["edges_out"],
                    s["jump_steps"]) for s in best["segs"]][:24],
             timeline=[tuple(round(s[k], 4) for k in ("hook_start_ms", "hook_end_ms",
                                                      "compress_start_ms", "compress_end_ms"))
                       for s in best["segs"]][:24])
    g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--specs", default="")
    ap.add_argument("--segs", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--walks", default="")
    ap.add_argument("--envs", default="", help="';'-separated K=V settings, one sweep each")
    args = ap.parse_args()
    emit(kind="env", devices=capi.device_count())
    ctx = capi.Context(0)
    emit(kind="ctx", sms=ctx.sm_count)
    if not args.no_parity:
        parity(ctx)
    if args.quick:
        return
    if args.specs:
        import os
        segs = [int(x) for x in args.segs.split(",")]
        walks = args.walks.split(",") if args.walks else [None]
        envs = args.envs.split(";") if args.envs else [None]
        for spec in args.specs.split(";"):
            for w in walks:
                for ev in envs:
                    # each sweep point sets its variables and restores them after
                    saved = dict(os.environ)
                    try:
                        if w is not None:
                            os.environ["HCC_WALK"] = w
                            emit(kind="walk", walk=int(w))
                        if ev is not None:
                            for kv in ev.split(","):
                                k, v = kv.split("=", 1)
                                os.environ[k] = v
                            emit(kind="env", env=ev)
                        timing(ctx, spec, reps=args.reps,
                               variants=[("baseline-mj", dict(first_pass_segments=s)) for s in segs],
                               check=not args.no_check)
                    finally:
                        os.environ.clear()
                        os.environ.update(saved)
        return
    timing(ctx, "rmatx:scale=20,ef=16,seed=1")
    timing(ctx, "rmatx:scale=24,ef=16,seed=1")
    timing(ctx, "grid:4096x4096", variants=[("baseline-mj", dict(first_pass_segments=1)),
                                             ("baseline-mj", dict(first_pass_segments=2)),
                                             ("baseline-mj", dict(flags=capi.FLAG_FULL_PASSES)),
                                             ("adaptive", dict(segments=4))])
    timing(ctx, "erx:n=16777216,m=268435456,seed=1")
    if args.big:
        timing(ctx, "rmatx:scale=26,ef=16,seed=1", check=False, reps=3)


if __name__ == "__main__":
    main()
