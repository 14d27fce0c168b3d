"""Host-side overhead of one C1 lcs_subsequence call: wall time with the
automatic row cap (a cudaMemGetInfo per call) vs an explicit cap, and the
cost of cudaMemGetInfo itself."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1306_4627_b200 as wl
from paper_1306_4627_b200 import workloads

x, y = workloads.config_pair("c1")
for cap in (0, 1 << 32, 0, 1 << 32):
    for _ in range(3):
        wl.lcs_subsequence(x, y, wl.NO_BUDGET, row_cap=cap)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); wl.lcs_subsequence(x, y, wl.NO_BUDGET, row_cap=cap); ts.append(time.perf_counter() - t0)
    print(f"row_cap={cap}: median {np.median(ts)*1e3:.3f} ms, min {min(ts)*1e3:.3f} ms")
torch.cuda.init()
ts = []
for _ in range(50):
    t0 = time.perf_counter(); torch.cuda.mem_get_info(); ts.append(time.perf_counter() - t0)
print(f"cudaMemGetInfo: median {np.median(ts)*1e6:.1f} us")
xs = x[:2000]; ys = y[:2000]
ts = []
for _ in range(30):
    t0 = time.perf_counter(); wl.lcs_subsequence(xs, ys, wl.NO_BUDGET, row_cap=1 << 32); ts.append(time.perf_counter() - t0)
print(f"2000x2000 subsequence: median {np.median(ts)*1e3:.3f} ms (fixed overhead floor)")
ts = []
for _ in range(30):
    t0 = time.perf_counter(); wl.lcs_length(xs, ys, wl.NO_BUDGET); ts.append(time.perf_counter() - t0)
print(f"2000x2000 length: median {np.median(ts)*1e3:.3f} ms")
