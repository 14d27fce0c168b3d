python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for k in 1 2 4 8; do WLCS_PAIR_ROWS=1 WLCS_PAIR_SPLIT=0 WLCS_PAIR_K=$k python tools/pair_probe.py 1000000 $((32*32*k)); done
for k in 2 4 8; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/b.json 2>&1; 
python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('K $k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done
for c in c1 c3 c5; do timeout 300 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('$c',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done
