for i in 1 2; do for w in 1 2 4; do for c in c4 c1; do
WLCS_LIB_PATH=tools/exp/pw$w.so timeout 300 python bench.py --variant wavefront --config $c --steps 2 --warmup 2 > gpurun_out/pw.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/pw.json').read().strip().splitlines()[-1]);print('$c warps=$w', d['fill_kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/pw.json
done; done; done
