"""Golden lengths for the full-size single-pair configs C4 (1M x 1M DNA) and
C5 (2M x 500k Zipf bytes), computed on the CPU by the pinned restatement
oracle (64-bit Hyyro bit-parallel, oracle/lcs_oracle.c: orc_length_bitpar;
pinned against the compiled reference in tests/test_oracle.py).  The
reference itself cannot run these sizes (5 TB of tables).

usage: python tests/golden/make_large_golden.py  (about a minute per config)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402

out = {}
res = oracle.Restatement()
for name in ("c4", "c5"):
    x, y = workloads.config_pair(name)
    t0 = time.time()
    out[name] = {"m": len(x), "n": len(y), "lcs_length": res.length_bitpar(x, y),
                 "seed": 20130619, "generator": "paper_1306_4627_b200/workloads.py:config_pair",
                 "oracle": "oracle/lcs_oracle.c orc_length_bitpar", "cpu_seconds": round(time.time() - t0, 1)}
    print(name, out[name], flush=True)
with open(os.path.join(ROOT, "tests", "golden", "large_configs.json"), "w") as f:
    json.dump(out, f, indent=1)
