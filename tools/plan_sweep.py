"""Developer probe: CC device time under plan overrides (HCC_PLAN ...).

python tools/plan_sweep.py <spec> [runs]   (reads the plan env as set by the
caller; prints the median and min total_ms over `runs` after 3 warm-ups and
checks that the component count does not change)
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_01178_b200 import capi  # noqa: E402

spec = sys.argv[1]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = capi.Context(0)
g = ctx.generate(spec)
ts, comps = [], set()
for i in range(3 + runs):
    _, mx = ctx.cc(g, "baseline-mj", labels=False)
    comps.add(mx["components"])
    if i >= 3:
        ts.append(mx["total_ms"])
print(json.dumps({"spec": spec, "median_ms": round(statistics.median(ts), 4),
                  "min_ms": round(min(ts), 4), "components": sorted(comps)}))
