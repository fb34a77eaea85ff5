"""One rank of the CUDA-IPC merge test (tests/test_distributed.py launches it
under torch.distributed.run; several ranks may share one GPU).  Host
collectives over gloo; the payload moves only through CUDA IPC mappings."""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(spec: str, out: str, cap: int, reps: int) -> None:
    from paper_1612_01178_b200 import capi
    from paper_1612_01178_b200.distributed import PeerMerge, edge_range
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = capi.Context(int(os.environ.get("IPC_DEVICE", "0")))
    probe = ctx.generate_range(spec, 0, 0)
    n = probe.n
    probe.close()
    full = ctx.generate(spec)
    m = full.m
    full.close()
    first, count = edge_range(m, world, rank)
    g = ctx.generate_range(spec, first, count)
    f = ctx.forest(n)
    pm = PeerMerge(ctx, n, cap=cap or None)
    for _ in range(reps):
        ctx.cc(g, "baseline-mj", forest=f, labels=False)
        mx = pm.merge(f)
    lab = f.snapshot().astype(np.uint32)
    res = {"rank": rank, "sha": hashlib.sha256(lab.tobytes()).hexdigest(),
           "components": mx["components"], "reopens": pm.reopens}
    Path(f"{out}.{rank}").write_text(json.dumps(res))
    pm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
