for i in 1 2 3; do for K in 0 2; do
WLCS_PAIR_K=$K timeout 300 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/c3k.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/c3k.json').read().strip().splitlines()[-1]);print('c3 K=$K', d['fill_kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/c3k.json
done; done
