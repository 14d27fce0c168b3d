# C2 headline A/B: bench line (device + e2e), launch list of the step.
set -u
mkdir -p gpurun_out/ab
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/c2.json 2> gpurun_out/ab/c2.err
python3 -c "
import json;d=json.loads(open('gpurun_out/ab/c2.json').read().strip().splitlines()[-1]);r=d['roofline'];print('value',d['value'],'ms',d['ms_per_step'],'kernel',r['kernel_ms'],'frac',r['frac'],'e2e',d['e2e']['value'])"
for c in c1 c3; do timeout 300 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/ab/$c.json 2>&1; python3 -c "
import json;d=json.loads(open('gpurun_out/ab/$c.json').read().strip().splitlines()[-1]);print('$c',d['value'],d['ms_per_step'],d['fill_kernel_ms'])"; done
