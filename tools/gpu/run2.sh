# carry window sweep
for w in 8 16 32 16; do for k in 2 4; do WLCS_PAIR_WIN=$w WLCS_PAIR_K=$k timeout 300 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/b.json 2>&1; 
python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('win $w K $k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done; done
