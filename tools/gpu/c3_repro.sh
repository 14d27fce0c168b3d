# reproduce the occasional slow C3 subsequence calls: full GPU suite, then the
# per-call probe, then the bench twice (C1 / C3 blocks)
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/rep_tests.log 2>&1; tail -1 gpurun_out/rep_tests.log
ps -eo pid,ppid,pcpu,etime,cmd --sort=-pcpu | head -8
N=10 timeout 300 python tools/c3_jitter_probe.py 2>&1 | tail -10
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/rep_b$i.json 2>&1
python3 -c "
import json;d=json.loads(open('gpurun_out/rep_b$i.json').read().strip().splitlines()[-1])
for c in ('c1','c3'): print(c, d[c]['e2e']['ms_per_step'], d[c]['e2e']['ms_median'], d[c]['fill_ms'])"
done
ps -eo pid,ppid,pcpu,etime,cmd --sort=-pcpu | head -5
