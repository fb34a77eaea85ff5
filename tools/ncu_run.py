"""Target process for ncu launch lists: generate SPEC, run ALGO REPS times
with eager launches (HCC_LAUNCH=eager: ncu does not enter conditional CUDA
graphs).  Usage: python tools/ncu_run.py SPEC ALGO [REPS] [SEGMENTS]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HCC_LAUNCH", "eager")
from paper_1612_01178_b200 import capi  # noqa: E402

spec, algo = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
seg = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ctx = capi.Context(0)
g = ctx.generate(spec)
for _ in range(reps):
    _, mx = ctx.cc(g, algo, segments=seg, labels=False)
print(mx["total_ms"], mx["components"], file=sys.stderr)
