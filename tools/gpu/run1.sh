# parity tests + single-pair configs + K sweep on C4
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest.log
for c in c1 c3 c4 c5; do timeout 300 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
for k in 1 2 4 8; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/b_c4_k$k.json 2>&1; done
for k in 1 2 4; do WLCS_PAIR_K=$k timeout 300 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/b_c5_k$k.json 2>&1; done
cat gpurun_out/pytest.log
for f in gpurun_out/b_*.json; do python3 -c "
import json,sys;d=json.load(open('$f'));print('$f',d['ms_per_step'],d.get('fill_kernel_ms'),d['value'],d['config'].get('lcs_length'))" 2>&1 | tail -1; done
