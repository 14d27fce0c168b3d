"""lcs_subsequence wall time on C1 / C3 / 2000x2000 for the walk block size in
WLCS_WALK_ROWS (set by the caller), median of 15 calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1306_4627_b200 as wl
from paper_1306_4627_b200 import workloads
R = os.environ.get("WLCS_WALK_ROWS", "default")
for name in ("c1", "c3", "s2k"):
    if name == "s2k":
        x, y = workloads.config_pair("c1")
        x, y = x[:2000], y[:2000]
    else:
        x, y = workloads.config_pair(name)
    for _ in range(3):
        s = wl.lcs_subsequence(x, y, wl.NO_BUDGET)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); s2 = wl.lcs_subsequence(x, y, wl.NO_BUDGET); ts.append(time.perf_counter() - t0)
    assert s2 == s
    print(f"R={R} {name}: median {np.median(ts)*1e3:.3f} ms  min {min(ts)*1e3:.3f}  len {len(s)}")
