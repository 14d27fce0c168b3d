python -m pytest tests/test_gpu_parity.py -q -x --durations=5 2>&1 | tail -8
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python3 -c "
import json;d=json.load(open('gpurun_out/b.json'));print('c2',d['ms_per_step'],d['value'],d['roofline']['kernel_ms'],d['roofline']['frac'],d['e2e']['value'])"; done
