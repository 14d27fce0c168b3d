"""Per-strip start/end times and placement (SM, warp slot -> sub-partition)
of the strip kernel on C4 / C5 (experiment build with WLCS_STRIP_TRACE):
does any strip share a sub-partition, and how long does each strip take?"""
import collections
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1306_4627_b200 as wl  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
x, y = workloads.config_pair(name)
wl.lcs_length(x, y, wl.NO_BUDGET)
buf = (ctypes.c_ulonglong * (8192 * 4))()
n = ctypes.c_uint()
wl.lib.wlcs_debug_strip_trace(buf, 8192, ctypes.byref(n))  # clear
wl.lcs_length(x, y, wl.NO_BUDGET)
wl.lib.wlcs_debug_strip_trace(buf, 8192, ctypes.byref(n))
a = np.frombuffer(buf, dtype=np.uint64)[: n.value * 4].reshape(-1, 4).astype(np.int64)
q, strip = a[:, 0] >> 32, a[:, 0] & 0xffffffff
smid, wid = a[:, 1] >> 32, a[:, 1] & 0xffffffff
t0 = a[:, 2] - a[:, 2].min()
t1 = a[:, 3] - a[:, 2].min()
dur = (t1 - t0) / 1e6
print(f"{name}: {n.value} strips, kernel span {t1.max()/1e6:.3f} ms")
occ = collections.Counter(zip(smid.tolist(), (wid % 4).tolist()))
print("strips per (SM, sub-partition) slot:", collections.Counter(occ.values()))
for qq in sorted(set(q.tolist())):
    m = q == qq
    order = np.argsort(strip[m])
    st, en, du = t0[m][order] / 1e6, t1[m][order] / 1e6, dur[m][order]
    print(f"problem {qq}: start of strip 0/1/10/100/last {st[0]:.3f} {st[1]:.3f} {st[min(10,len(st)-1)]:.3f} "
          f"{st[min(100,len(st)-1)]:.3f} {st[-1]:.3f} ms; end first/last {en[0]:.3f} {en[-1]:.3f}; "
          f"duration min/median/max {du.min():.3f}/{np.median(du):.3f}/{du.max():.3f}")
    gaps = np.diff(st)
    print(f"   start gap median {np.median(gaps)*1e3:.1f} us, max {gaps.max()*1e3:.1f} us")
shared = [k for k, v in occ.items() if v > 1]
print("shared slots:", len(shared))
