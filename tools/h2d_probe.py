"""H2D bandwidth from pinned host memory: one copy, or split over k streams."""
import torch

N = 2 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    part = N // k
    for rep in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in streams:
            e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        if rep == 3:
            print(f"streams={k}: {N / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
