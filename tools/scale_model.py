"""Per-rank cost model of the edge-partitioned RMAT-28 run at N = 1, 2, 4, 8
GPUs, measured on ONE B200 (the pool has one GPU per call).

A multi-device context with N shards on device 0, run with HCC_MULTI_SERIAL=1:
each shard's local CC and each shard's merge (gather of the N-1 peers'
exports + re-hook) run alone on the GPU, i.e. exactly the work one rank of an
N-GPU run does, except that the peers' exports are read from local HBM
instead of over NVLink (32 MiB bitmap + the pairs per peer; at the measured
~770 GB/s per-direction peer bandwidth that adds (N-1) x 0.045 ms, included
below) and that there is no skew between ranks.

Predicted step time at N = max over shards of (local + merge + NVLink
correction); predicted GTEPS = m / that.  Writes one JSON line per N and the
whole table to profiles/r2_rmat28_scaling_model.json.

python tools/scale_model.py [--spec S] [--reps K] [--ns 1,2,4,8]
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["HCC_MULTI_SERIAL"] = "1"
from paper_1612_01178_b200 import capi  # noqa: E402

PEER_GBPS = 770.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spec", default="rmatx:scale=28,ef=16,seed=1")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ns", default="1,2,4,8")
    a = ap.parse_args()
    rows = []
    for N in [int(x) for x in a.ns.split(",")]:
        ctx = capi.Context(devices=[0] * N)
        g = ctx.generate(a.spec)
        steps = []
        for i in range(a.reps + 1):
            _, mx = ctx.cc(g, "baseline-mj", labels=False)
            sm = ctx.shard_metrics()
            if i:
                steps.append(sm)
        nwords = (g.n + 31) // 32
        per = []
        for r in range(N):
            loc = statistics.mean(s[r]["local_ms"] for s in steps)
            mer = statistics.mean(s[r]["merge_ms"] for s in steps)
            nvl = (N - 1) * (4 * nwords + 8 * steps[-1][r]["pairs_exported"]) / (PEER_GBPS * 1e9) * 1e3
            per.append({"shard": r, "local_ms": round(loc, 3), "merge_ms": round(mer, 3),
                        "nvlink_ms": round(nvl, 3), "records_merged": steps[-1][r]["records_merged"],
                        "rehook_passes": steps[-1][r]["rehook_passes"],
                        "roots_linked": steps[-1][r]["roots_linked"],
                        "pairs_exported": steps[-1][r]["pairs_exported"]})
        t = max(p["local_ms"] + p["merge_ms"] + p["nvlink_ms"] for p in per)
        row = {"n_gpus": N, "spec": a.spec, "m": g.m, "pred_ms_per_step": round(t, 3),
               "pred_gteps": round(g.m / (t * 1e-3) / 1e9, 2), "components": mx["components"],
               "shards": per}
        rows.append(row)
        print(json.dumps(row), flush=True)
        g.close()
        ctx.close()
    base = rows[0]["pred_ms_per_step"] if rows and rows[0]["n_gpus"] == 1 else None
    for r in rows:
        if base:
            r["pred_speedup_vs_1"] = round(base / r["pred_ms_per_step"], 3)
            r["pred_efficiency"] = round(base / r["pred_ms_per_step"] / r["n_gpus"], 3)
    out = ROOT / "profiles" / "r2_rmat28_scaling_model.json"
    out.write_text(json.dumps({"how": __doc__.strip().splitlines()[0], "peer_gbps": PEER_GBPS,
                               "rows": rows}, indent=1) + "\n")


if __name__ == "__main__":
    main()
