python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for i in 1 2; do for lib in tools/exp/prev.so ""; do for c in c4 c3 c5; do WLCS_LIB_PATH=$lib timeout 300 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/b.json 2>/dev/null; python3 -c "
import json;d=json.load(open('gpurun_out/b.json'));print('[$lib] $c',d['ms_per_step'],d.get('fill_kernel_ms'))"; done; done; done
