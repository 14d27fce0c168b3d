"""Cell-wavefront pair kernel: kernel time vs number of bands (rows) at a
fixed column count, to separate the per-step time from the hand-off lag."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1306_4627_b200 as wl  # noqa: E402

n = int(os.environ.get("N", 1 << 20))
rng = np.random.default_rng(1)
y = rng.choice(np.frombuffer(b"ACGT", np.uint8), n).tobytes()
wl._check(wl.lib.wlcs_set_timing(1))
for rows in [int(r) for r in os.environ.get("ROWS", "512,1024,2048,4096,16384,65536,262144,1048576").split(",")]:
    x = rng.choice(np.frombuffer(b"ACGT", np.uint8), rows).tobytes()
    best = 1e9
    for _ in range(2):
        wl.lcs_length(y, x, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT)  # rows = longer string
        km = ctypes.c_float()
        wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
        best = min(best, km.value)
    print(f"rows {rows:8d} cols {n}: {best:9.3f} ms  {rows * n / best / 1e6:9.1f} GCUPS")
