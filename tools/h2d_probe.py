"""Pinned host->device copy bandwidth (what bounds the C2 e2e number):
single copies of several sizes, and an 80 MB copy split over 1/2/4 streams."""
import time
import torch
for mb in (8, 16, 40, 80, 160, 256):
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
n = 80 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 10
    print(f"80 MB over {ns} streams: {dt * 1e3:.3f} ms  {n / dt / 1e9:.1f} GB/s")
