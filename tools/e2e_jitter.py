"""Per-call wall times of lcs_subsequence (C1, C3): find the outliers that
the e2e averages sometimes show (Python GC off / on; host-thread sleep)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1306_4627_b200 as wl  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402

for gcoff in (False, True):
    if gcoff:
        gc.disable()
    for name, n in (("c1", 60), ("c3", 30)):
        x, y = workloads.config_pair(name)
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            wl.lcs_subsequence(x, y, wl.NO_BUDGET)
            ts.append((time.perf_counter() - t0) * 1e3)
        ts = ts[3:]
        ts.sort()
        print(f"gc_off={gcoff} {name}: min {ts[0]:.2f} median {ts[len(ts)//2]:.2f} "
              f"p90 {ts[int(len(ts)*0.9)]:.2f} max {ts[-1]:.2f}")
