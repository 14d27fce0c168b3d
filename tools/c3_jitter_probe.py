"""Per-call wall time of lcs_subsequence on C3 (20 calls) with the walk's
phase times (WLCS_DEBUG_WALK) and the fill's CUDA-event time, to find where
an occasional slow call spends its time."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1306_4627_b200 as wl
from paper_1306_4627_b200 import workloads
x, y = workloads.config_pair(os.environ.get("CFG", "c3"))
wl._check(wl.lib.wlcs_set_timing(1))
km = ctypes.c_float()
for i in range(int(os.environ.get("N", "20"))):
    t0 = time.perf_counter()
    s = wl.lcs_subsequence(x, y, wl.NO_BUDGET)
    t = time.perf_counter() - t0
    wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
    print(f"call {i}: {t*1e3:.3f} ms (fill {km.value:.3f} ms) len {len(s)}", flush=True)
