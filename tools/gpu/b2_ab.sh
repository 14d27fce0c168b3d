timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in "WLCS_LIB_PATH=tools/exp/base.so" "WLCS_LIB_PATH=tools/exp/c2r.so"; do
env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
python3 -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('[$v]',d['ms_per_step'],d['roofline']['kernel_ms'],d['value'])"
done; done
