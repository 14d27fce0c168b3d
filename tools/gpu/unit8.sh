# 8-row-unit strip kernel vs the 16-row one: parity subset, then C1/C4/C5 fills (A/B by env)
mkdir -p gpurun_out/u8
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "pair or c1 or c4 or c5 or length or split" 2>&1 | tail -3
for i in 1 2; do for U in 0 1; do for c in c1 c4 c5; do
WLCS_PAIR_UNIT8=$U timeout 300 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/u8/$c.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/u8/$c.json').read().strip().splitlines()[-1]);print('$c unit8=$U', d.get('fill_kernel_ms', d.get('fill_ms')), d['ms_per_step'], d.get('lcs_length'))" || tail -3 gpurun_out/u8/$c.json
done; done; done
