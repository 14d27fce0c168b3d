for ca in 1 2; do
for st in 1 2 64; do WLCS_PAIR_CARRY_AHEAD=$ca WLCS_PAIR_ROWS=1 WLCS_PAIR_SPLIT=0 WLCS_PAIR_K=4 python tools/pair_probe.py 200000 $((4096*st)); done
WLCS_PAIR_CARRY_AHEAD=$ca timeout 300 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/b.json 2>&1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('c4 ca $ca',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1
done
