"""Times the single-pair fill on custom shapes (strip-kernel diagnostics).

usage: python tools/pair_probe.py ROWS COLS [REPS]
Prints fill-kernel ms, steps per strip and cycles per step at the clock given
by WLCS_PROBE_MHZ (default 1965)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1306_4627_b200 as wl

rows, cols = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rng = np.random.default_rng(1)
x = rng.choice(np.frombuffer(b"ACGT", np.uint8), rows).tobytes()
y = rng.choice(np.frombuffer(b"ACGT", np.uint8), cols).tobytes()
wl._check(wl.lib.wlcs_set_timing(1))
km = ctypes.c_float()
best = 1e30
for _ in range(reps):
    n = wl.lcs_length(x, y, wl.NO_BUDGET)
    wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
    best = min(best, km.value)
split = os.environ.get("WLCS_PAIR_SPLIT", "")
r = rows if os.environ.get("WLCS_PAIR_ROWS") == "1" else min(rows, cols)
steps = (r // (2 if split != "0" and r >= 2048 else 1) + 15) // 16
mhz = float(os.environ.get("WLCS_PROBE_MHZ", 1965))
print(f"rows={rows} cols={cols} lcs={n} fill_ms={best:.3f} steps/strip={steps} "
      f"cycles/step={best * 1e-3 * mhz * 1e6 / steps:.0f} GCUPS={rows * cols / best / 1e6:.0f}")
