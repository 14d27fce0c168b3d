cat > /tmp/c1once.py <<'PY'
import paper_1306_4627_b200 as wl
from paper_1306_4627_b200 import workloads
x, y = workloads.config_pair(__import__("os").environ.get("CFG","c1"))
for _ in range(3):
    s = wl.lcs_subsequence(x, y, wl.NO_BUDGET)
print(len(s))
PY
CFG=${CFG:-c1} PYTHONPATH=. timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python /tmp/c1once.py > gpurun_out/c1_ncu.log 2>&1
tail -1 gpurun_out/c1_ncu.log
