"""Per-band start/end times of the cell-wavefront pair kernel (experiment
build with WLCS_WAVE_TRACE): band durations and start lags."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1306_4627_b200 as wl  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
x, y = workloads.config_pair(name)
buf = (ctypes.c_ulonglong * (8192 * 3))()
n = ctypes.c_uint()
wl.lcs_length(x, y, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT)
wl.lib.wlcs_debug_wave_trace(buf, 8192, ctypes.byref(n))
wl.lcs_length(x, y, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT)
wl.lib.wlcs_debug_wave_trace(buf, 8192, ctypes.byref(n))
a = np.frombuffer(buf, dtype=np.uint64)[: n.value * 3].reshape(-1, 3).astype(np.int64)
order = np.argsort(a[:, 0])
b, t0, t1 = a[order, 0], a[order, 1], a[order, 2]
base = t0.min()
t0, t1 = (t0 - base) / 1e6, (t1 - base) / 1e6
dur = t1 - t0
print(f"{name}: {n.value} bands; span {t1.max():.2f} ms")
for k in [0, 1, 2, 10, 100, 500, 1000, len(b) - 1]:
    if k < len(b):
        print(f"band {b[k]:5d}: start {t0[k]:8.3f} end {t1[k]:8.3f} duration {dur[k]:8.3f} ms")
print(f"end gap median {np.median(np.diff(t1))*1e3:.2f} us; duration min/median/max "
      f"{dur.min():.2f}/{np.median(dur):.2f}/{dur.max():.2f} ms")
