"""Check (i) of SURVEY.md 8(c) at full size: the C4 / C5 lengths from the
two-row lcs_cell loop (oracle/lcs_oracle.c: orc_length_cells_mt, the value
rule of cell.hpp:30-38 in the loop order of kernels_scalar.cpp:6-16, spread
over host threads by column strips).  They must equal check (ii), the 64-bit
Hyyro lengths in tests/golden/large_configs.json (make_large_golden.py); the
result is merged into that file as "lcs_length_cells".

usage: python tests/golden/make_large_golden_cells.py [threads]
(~1e12 cell updates per config: tens of minutes on 8 host threads)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402

threads = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
path = os.path.join(ROOT, "tests", "golden", "large_configs.json")
res = oracle.Restatement()
for name in ("c4", "c5"):
    x, y = workloads.config_pair(name)
    t0 = time.time()
    length = res.length_cells_mt(x, y, threads)
    sec = time.time() - t0
    with open(path) as f:
        golden = json.load(f)
    golden[name]["lcs_length_cells"] = length
    golden[name]["cells_oracle"] = "oracle/lcs_oracle.c orc_length_cells_mt (two-row lcs_cell loop)"
    golden[name]["cells_cpu_seconds"] = round(sec, 1)
    golden[name]["cells_threads"] = threads
    with open(path, "w") as f:
        json.dump(golden, f, indent=1)
    print(name, length, "bitpar", golden[name]["lcs_length"], f"{sec:.0f}s", flush=True)
    if length != golden[name]["lcs_length"]:
        sys.exit(f"{name}: two-row cell loop {length} != Hyyro {golden[name]['lcs_length']}")
