timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "wavefront" 2>&1 | tail -2
for i in 1 2; do for a in 0 1; do for c in c4 c1; do
WLCS_LIB_PATH=tools/exp/ah$a.so timeout 300 python bench.py --variant wavefront --config $c --steps 2 --warmup 2 > gpurun_out/ah.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/ah.json').read().strip().splitlines()[-1]);print('$c ahead=$a', d['fill_kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/ah.json
done; done; done
