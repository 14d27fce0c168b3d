"""Strip hand-off cost: one 4096-column slice run alone, as a producer
(publishing into an inbox), as a consumer of a complete inbox, and the two
as one 2-strip fill (tools/pair_probe.py)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1306_4627_b200 as wl

os.environ.setdefault("WLCS_PAIR_K", "4")
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
rng = np.random.default_rng(1)
x = rng.choice(np.frombuffer(b"ACGT", np.uint8), rows).tobytes()
y = rng.choice(np.frombuffer(b"ACGT", np.uint8), 8192).tobytes()
words = wl.colsplit_inbox_words(rows)
box = wl.device_alloc(4 * words)
wl._check(wl.lib.wlcs_set_timing(1))
km = ctypes.c_float()


def timed(f):
    best = 1e9
    for _ in range(3):
        f()
        wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
        best = min(best, km.value)
    return best


F = wl.COLSPLIT_FORWARD
t_solo = timed(lambda: wl.colsplit_fill(x, y, 0, 4096, F))
t_prod = timed(lambda: (wl.device_zero(box, 4 * words), wl.colsplit_fill(x, y, 0, 4096, F, out_fwd=box)))
t_cons = timed(lambda: wl.colsplit_fill(x, y, 4096, 8192, F, in_fwd=box))
print(f"rows/2={rows // 2}: solo {t_solo:.3f} ms  producer {t_prod:.3f} ms  consumer(inbox ready) {t_cons:.3f} ms")
