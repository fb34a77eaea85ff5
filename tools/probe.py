"""Developer timing probe: one spec, one engine, per-record device timeline.

Usage: python tools/probe.py SPEC [--algo A] [--reps N] [--forest] [--segments S]
                                  [--flags F] [--devices 0,0] [--check]
Prints one JSON line per rep summary plus the per-record timeline of the
last rep (hook/compress spans from the device %globaltimer records).  The
L2 is flushed between reps (a 256 MiB write).  --check compares the labels
with the oracle (small graphs) or with tests/golden/big.json (named specs).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1612_01178_b200 import capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("--algo", default="baseline-mj")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--segments", type=int, default=0)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--forest", action="store_true")
    ap.add_argument("--devices", default="")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--timeline", action="store_true")
    ap.add_argument("--ipc", type=int, default=0,
                    help="1: open a world-1 peer arena; 2: also export + merge every rep")
    ap.add_argument("--ballast", type=int, default=0, help="GiB of extra device memory held")
    ap.add_argument("--smi", action="store_true", help="poll nvidia-smi like bench.py's sampler")
    ap.add_argument("--gloo", action="store_true", help="gloo barrier before every rep")
    ap.add_argument("--noflush", action="store_true", help="no L2 flush between reps")
    ap.add_argument("--thread", action="store_true", help="run each CC on a fresh host thread")
    ap.add_argument("--range", default="", help="first,count: one shard of the spec")
    ap.add_argument("--extractx", action="store_true", help="create a second context first")
    a = ap.parse_args()
    import torch
    devs = [int(x) for x in a.devices.split(",") if x]
    extra = capi.Context(0) if a.extractx else None
    ctx = capi.Context(devices=devs) if devs else capi.Context(0)
    if a.range:
        first, count = (int(x) for x in a.range.split(","))
        g = ctx.generate_range(a.spec, first, count)
    else:
        g = ctx.generate(a.spec)
    f = ctx.forest(g.n) if a.forest else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    ballast = torch.empty(a.ballast << 30, dtype=torch.uint8, device="cuda:0") if a.ballast else None
    if a.ipc:
        blob = ctx.peer_open(g.n, max(1 << 16, g.n // 64), 0, 1)
        ctx.peer_connect(blob)
    times = []
    mx = None
    if a.smi:
        from bench import ClockSampler
        sampler = ClockSampler(0)
        sampler.start()
    if a.gloo:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=0, world_size=1, init_method="tcp://127.0.0.1:29533")
    for i in range(a.reps + 2):
        if not a.noflush:
            flush.add_(1)
        torch.cuda.synchronize()
        if a.gloo:
            dist.barrier()
        if a.thread:
            import threading
            box = {}
            th = threading.Thread(target=lambda: box.update(
                r=ctx.cc(g, a.algo, segments=a.segments, flags=a.flags, forest=f, labels=False)))
            th.start()
            th.join()
            _, mx = box["r"]
        else:
            _, mx = ctx.cc(g, a.algo, segments=a.segments, flags=a.flags, forest=f, labels=False)
        if i >= 2:
            times.append(mx["total_ms"])
        if a.ipc == 2:
            ctx.peer_export(f)
            ctx.peer_merge(f)
    if a.smi:
        print(json.dumps(sampler.stop()))
    out = {"spec": a.spec, "algo": a.algo, "ms_mean": round(statistics.mean(times), 4),
           "ms_min": round(min(times), 4), "gteps": round(g.m / statistics.mean(times) / 1e6, 2),
           "s": mx["s"], "kernels": mx["kernels"], "components": mx["components"],
           "hook_ms": round(mx["hook_ms"], 4), "compress_ms": round(mx["compress_ms"], 4),
           "cas_attempts": mx["hook_traversal_steps"], "cas_failures": mx["cas_failures"],
           "wl_capacity": mx["wl_capacity"], "wl_reruns": mx["wl_reruns"]}
    if devs:
        out["shards"] = ctx.shard_metrics()
    if a.check:
        lab, _ = ctx.cc(g, a.algo, segments=a.segments, flags=a.flags)
        big = json.loads((ROOT / "tests" / "golden" / "big.json").read_text())
        gold = next((v for v in big.values() if v["spec"] == a.spec), None)
        if gold:
            out["exact"] = hashlib.sha256(lab.astype("<u4").tobytes()).hexdigest() == gold["labels_sha256"]
        else:
            import oracle as O
            out["exact"] = bool(np.array_equal(lab, O.cc(g.n, g.edges())))
    print(json.dumps(out), flush=True)
    if devs:
        out["shards"] = ctx.shard_metrics()
    if a.timeline and not devs:
        for r in ctx.segments():
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}),
                  flush=True)


if __name__ == "__main__":
    main()
