"""Pinned host-to-device copy bandwidth (the e2e roofline): one 512 MB copy and 16 x 32 MB copies."""
import torch

dev = torch.device("cuda")
for size_mb, reps in ((512, 8), (32, 64)):
    n = size_mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D pinned {size_mb} MB x{reps}: {n * reps / (ms * 1e-3) / 1e9:.1f} GB/s")
    e0.record()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"D2H pinned {size_mb} MB x{reps}: {n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
