mkdir -p gpurun_out/c4k
for K in 2 4 8; do
WLCS_PAIR_K=$K timeout 300 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/c4k/c4.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/c4k/c4.json').read().strip().splitlines()[-1]);print('c4 K=$K', d['value'], d['ms_per_step'])"
WLCS_PAIR_K=$K timeout 300 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/c4k/c5.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/c4k/c5.json').read().strip().splitlines()[-1]);print('c5 K=$K', d['value'], d['ms_per_step'])"
done
