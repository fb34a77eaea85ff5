"""ncu target: one CC call on an N-shard multi-device context (all shards on
device 0, run one at a time: HCC_MULTI_SERIAL=1), eager launches.

python tools/ncu_target_multi.py SPEC N [runs]
"""
import os
import sys
from pathlib import Path

os.environ.setdefault("HCC_MULTI_SERIAL", "1")
os.environ.setdefault("HCC_LAUNCH", "eager")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_01178_b200 import capi  # noqa: E402

spec = sys.argv[1]
N = int(sys.argv[2])
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ctx = capi.Context(devices=[0] * N)
g = ctx.generate(spec)
for _ in range(runs):
    _, mx = ctx.cc(g, "baseline-mj", labels=False)
print(mx["total_ms"], [(round(s["local_ms"], 3), round(s["merge_ms"], 3), s["rehook_passes"])
                       for s in ctx.shard_metrics()])
