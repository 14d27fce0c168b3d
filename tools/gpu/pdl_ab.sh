set -u
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in "WLCS_LIB_PATH=tools/exp/base.so" "WLCS_LIB_PATH=tools/exp/fine.so"; do
env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
python3 -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('[$v]',d['ms_per_step'],d['roofline']['kernel_ms'],d['value'],d['e2e']['value'])"
done; done
for v in "WLCS_LIB_PATH=tools/exp/base.so" "WLCS_LIB_PATH=tools/exp/fine.so"; do for c in c1 c3; do
env $v timeout 300 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/ab.json 2>gpurun_out/ab.err
python3 -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('[$v] $c',d['ms_per_step'],d['value'])"
done; done
