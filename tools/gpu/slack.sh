for i in 1 2; do for sl in 0 2 4; do for c in c3 c4 c5 c1; do
WLCS_LIB_PATH=tools/exp/slack$sl.so timeout 300 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/sl.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/sl.json').read().strip().splitlines()[-1]);print('$c slack=$sl', d['fill_kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/sl.json
done; done; done
