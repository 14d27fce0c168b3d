timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "pair or c1 or c4 or c5 or length or split or colsplit or strips or golden or banded or subsequence" 2>&1 | tail -2
for i in 1 2; do for L in 32 0 28 24 20; do
WLCS_PAIR_LANES=$L timeout 300 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/ln.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/ln.json').read().strip().splitlines()[-1]);print('c5 lanes=$L', d['fill_kernel_ms'], d['ms_per_step'], d['config']['lcs_length'])" || tail -2 gpurun_out/ln.json
done; done
