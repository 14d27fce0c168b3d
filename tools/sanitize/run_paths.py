"""Small invocations of every device path, for compute-sanitizer runs
(tools/sanitize/*.sh): C1 length + exact traceback (full and banded), a
batch with first-pass and second-pass pairs, the column split played in one
launch, the device tile kernel and the cell-wavefront variant."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (checker)
import paper_1306_4627_b200 as wl  # noqa: E402

ref = oracle.Restatement()
x = ref.generate_random(10000, b"ACGT", 1)
y = ref.generate_random(10000, b"ACGT", 1 + 0x9E3779B97F4A7C15)
assert wl.lcs_length(x, y) == 6538
assert wl.lcs_subsequence(x[:3000], y[:3000]) == ref.subsequence(x[:3000], y[:3000])
assert wl.lcs_subsequence(x[:4000], y[:3000], wl.NO_BUDGET, row_cap=600_000) == \
    ref.subsequence_bitrows(x[:4000], y[:3000])
rng = np.random.default_rng(3)
a = np.arange(256, dtype=np.uint8)
prot = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", np.uint8)
xs = [prot[rng.integers(0, 20, int(rng.integers(1, 900)))].tobytes() for _ in range(300)]
ys = [prot[rng.integers(0, 20, int(rng.integers(1, 900)))].tobytes() for _ in range(300)]
xs += [a[rng.integers(0, 256, 1500)].tobytes() for _ in range(20)]
ys += [a[rng.integers(0, 256, 1300)].tobytes() for _ in range(20)]
xb, xo, yb, yo = wl.pack_pairs(xs, ys)
assert np.array_equal(wl.lcs_length_batch(xb, xo, yb, yo), ref.length_batch(xb, xo, yb, yo))
assert wl.colsplit_emulate(x[:2000], y, 2, 4) == ref.length_bitpar(x[:2000], y)
dp, back = wl.fill_tables(x[:200], y[:150])
wdp, wback = ref.fill_tables(x[:200], y[:150])
assert np.array_equal(dp, wdp) and np.array_equal(back, wback)
assert wl.lcs_length(x[:3000], y[:2000], variant=wl.VARIANT_WAVEFRONT) == ref.length_bitpar(x[:3000], y[:2000])
print("sanitize paths: ok")
