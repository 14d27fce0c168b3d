python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for g in 1 0; do WLCS_PAIR_GEN=$g WLCS_DEBUG_PAIR=1 timeout 300 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/k.json 2>gpurun_out/k.err; grep "wlcs pair" gpurun_out/k.err | head -1; python3 -c "
import json;d=json.load(open('gpurun_out/k.json'));print('gen=$g c5', d['ms_per_step'], d.get('fill_kernel_ms'), d['config'].get('lcs_length'))" 2>&1 | tail -1; done
for K in 1 2 4; do WLCS_PAIR_K=$K WLCS_DEBUG_PAIR=1 timeout 300 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/k.json 2>gpurun_out/k.err; grep "wlcs pair" gpurun_out/k.err | head -1; python3 -c "
import json;d=json.load(open('gpurun_out/k.json'));print('K=$K c5', d['ms_per_step'], d.get('fill_kernel_ms'))" 2>&1 | tail -1; done
