"""Pinned host->device copy bandwidth (what bounds the C2 e2e number)."""
import time
import torch
for mb in (16, 80, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"H2D {mb} MB: {dt * 1e3:.3f} ms  {n / dt / 1e9:.1f} GB/s")
