"""Minimal single-run target for ncu: one CC call on a device-generated graph.

python tools/ncu_target.py [spec] [algo] [first_pass_segments] [runs]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_01178_b200 import capi  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "rmatx:scale=24,ef=16,seed=1"
algo = sys.argv[2] if len(sys.argv) > 2 else "baseline-mj"
segs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
# ncu: kernels launched eagerly (host-driven loop) so every launch is visible
flags = capi.FLAG_NO_GRAPH if (len(sys.argv) > 5 and sys.argv[5] == "nograph") else 0
ctx = capi.Context(0)
g = ctx.generate(spec)
for _ in range(runs):
    _, mx = ctx.cc(g, algo, first_pass_segments=segs, labels=False, flags=flags)
print({k: mx[k] for k in ("total_ms", "hook_ms", "compress_ms", "s", "outer_iterations", "components")})
for i, s in enumerate(ctx.segments()):
    print(i, s)
