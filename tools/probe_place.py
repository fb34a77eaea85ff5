"""Placement sensitivity: the same RMAT-28 CC into several forests allocated
at different points (before/after the edges, after ballast), one process."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_01178_b200 import capi  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "rmatx:scale=28,ef=16,seed=1"
ctx = capi.Context(0)
f_early = ctx.forest(1 << 28)
g = ctx.generate(spec)
forests = {"early": f_early, "late1": ctx.forest(g.n)}
ball = torch.empty(3 << 30, dtype=torch.uint8, device="cuda:0")
forests["late2"] = ctx.forest(g.n)
del ball
torch.cuda.empty_cache()
forests["late3"] = ctx.forest(g.n)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
for rnd in range(2):
    for name, f in forests.items():
        ts = []
        for i in range(4):
            flush.add_(1)
            torch.cuda.synchronize()
            _, mx = ctx.cc(g, "baseline-mj", forest=f, labels=False)
            if i:
                ts.append(mx["total_ms"])
        print(rnd, name, round(statistics.mean(ts), 3), flush=True)
