for k in 1 2 4 8; do WLCS_PAIR_ROWS=1 WLCS_PAIR_SPLIT=0 WLCS_PAIR_K=$k python tools/pair_probe.py 200000 $((1024*k)); WLCS_PAIR_ROWS=1 WLCS_PAIR_SPLIT=0 WLCS_PAIR_K=$k python tools/pair_probe.py 200000 $((1024*k*64)); done
for k in 2 4 8; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('c4 K$k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'])" 2>&1 | tail -1; done
for k in 1 2 4; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('c5 K$k',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'])" 2>&1 | tail -1; done
