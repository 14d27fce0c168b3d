# lanes skewed by 8 rows (HALF) vs 16: parity first, then C4/C5/C1 fills
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "pair or c1 or c4 or c5 or length or split or colsplit or strips or golden" 2>&1 | tail -2
for i in 1 2; do for h in 0 1; do for c in c4 c5; do
WLCS_LIB_PATH=tools/exp/half$h.so timeout 300 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/h.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/h.json').read().strip().splitlines()[-1]);print('$c half=$h', d['fill_kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/h.json
done; done; done
