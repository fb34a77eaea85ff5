import os, sys, time
sys.path.insert(0, '.')
import torch, torch.distributed as dist
os.environ.setdefault("RANK","0"); os.environ.setdefault("WORLD_SIZE","1")
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29561")
dist.init_process_group("nccl")
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
n = 1 << 24
bits = torch.randint(0, 1 << 30, ((n + 31) // 32,), dtype=torch.int32, device=dev)
pairs = torch.randint(0, n, (2957, 2), dtype=torch.int32, device=dev)
S = torch.cuda.synchronize
def tm(f, reps=20):
    f(); S()
    t = time.perf_counter()
    for _ in range(reps): f()
    S()
    return 1e6 * (time.perf_counter() - t) / reps
world = 1
g = torch.empty(world * bits.numel(), dtype=bits.dtype, device=dev)
print("allgather bits us", tm(lambda: dist.all_gather_into_tensor(g, bits)))
k = torch.tensor([pairs.shape[0]], dtype=torch.int64, device=dev)
sizes = torch.empty(world, dtype=torch.int64, device=dev)
print("allgather sizes us", tm(lambda: dist.all_gather_into_tensor(sizes, k)))
print("sizes.cpu us", tm(lambda: sizes.cpu().tolist()))
print("tensor create us", tm(lambda: torch.tensor([pairs.shape[0]], dtype=torch.int64, device=dev)))
allp = torch.empty(world * pairs.numel(), dtype=pairs.dtype, device=dev)
print("allgather pairs us", tm(lambda: dist.all_gather_into_tensor(allp, pairs.view(-1))))
from paper_1612_01178_b200.distributed import exchange
print("exchange() us", tm(lambda: exchange(bits, pairs)))
dist.destroy_process_group()
