# walk block size (64 / 128 / 256 rows) on C1 / C3 / 2000^2 subsequences: per-phase times and e2e
for R in 64 128 256; do
  echo "== R=$R"
  WLCS_WALK_ROWS=$R WLCS_DEBUG_WALK=1 timeout 300 python -c "
import time, numpy as np
import paper_1306_4627_b200 as wl
from paper_1306_4627_b200 import workloads
for name in ('c1', 'c3'):
    x, y = workloads.config_pair(name)
    for _ in range(2): wl.lcs_subsequence(x, y, wl.NO_BUDGET)
" 2>&1 | grep "walk ms" | tail -2
  WLCS_WALK_ROWS=$R timeout 300 python tools/c1_host_probe.py 2>&1 | grep -E "row_cap=0|2000x2000 sub" | tail -2
  WLCS_WALK_ROWS=$R timeout 300 python bench.py --config c3 --steps 5 --warmup 2 > gpurun_out/c3w.json 2>&1
  python3 -c "import json;d=json.loads(open('gpurun_out/c3w.json').read().strip().splitlines()[-1]);print('c3', d.get('ms_per_step'), d.get('golden_match', d.get('reference_match')))" || tail -2 gpurun_out/c3w.json
done
