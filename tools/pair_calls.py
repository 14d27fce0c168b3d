"""Wall time of single-pair C-ABI calls (length / subsequence) per config,
median of N calls after warm-up: python tools/pair_calls.py [lib]."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# PKG_ROOT: import the package from another tree (A/B against an older commit)
sys.path.insert(0, os.environ.get("PKG_ROOT", ROOT))
if len(sys.argv) > 1:
    os.environ["WLCS_LIB_PATH"] = sys.argv[1]
import numpy as np  # noqa: E402
import paper_1306_4627_b200 as wl  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402


def med(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


tag = os.path.basename(sys.argv[1]) if len(sys.argv) > 1 else "lib"
only_len = os.environ.get("ONLY_LENGTH") == "1"
x, y = workloads.config_pair("c1")
if only_len:
    for c in ("c1", "c4", "c5"):
        x, y = workloads.config_pair(c)
        print(tag, c, "length ms %.3f" % med(lambda: wl.lcs_length(x, y, wl.NO_BUDGET), 3))
    sys.exit(0)
print(tag, "c1 length ms %.3f" % med(lambda: wl.lcs_length(x, y)),
      "c1 subseq ms %.3f" % med(lambda: wl.lcs_subsequence(x, y)),
      "c1 subseq banded(4MB) ms %.3f" % med(lambda: wl.lcs_subsequence(x, y, wl.NO_BUDGET, row_cap=4 << 20)))
x, y = workloads.config_pair("c3")
print(tag, "c3 subseq ms %.3f" % med(lambda: wl.lcs_subsequence(x, y, wl.NO_BUDGET), 3),
      "c3 banded(64MB) ms %.3f" % med(lambda: wl.lcs_subsequence(x, y, wl.NO_BUDGET, row_cap=64 << 20), 3))
for c in ("c4", "c5"):
    x, y = workloads.config_pair(c)
    print(tag, c, "length ms %.3f" % med(lambda: wl.lcs_length(x, y, wl.NO_BUDGET), 3))
