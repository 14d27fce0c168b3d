for i in 1 2; do for K in 0 1 2; do
WLCS_PAIR_K=$K timeout 300 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/c5k.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/c5k.json').read().strip().splitlines()[-1]);print('c5 K=$K', d['fill_kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/c5k.json
done; done
