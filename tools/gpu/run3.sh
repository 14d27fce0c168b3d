for k in 1 2 4; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('c5 K $k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done
for k in 1 2; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('c3 K $k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done
for k in 1 2; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c1 --steps 2 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('c1 K $k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done
