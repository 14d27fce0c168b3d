mkdir -p gpurun_out/ws
for lib in paper_1306_4627_b200/_lib/libwavelcs_b200.so tools/exp/sl50.so tools/exp/sl500.so tools/exp/sl2000.so; do for c in c1 c4; do
WLCS_LIB_PATH=$lib timeout 300 python bench.py --variant wavefront --config $c --steps 2 --warmup 3 > gpurun_out/ws/$c.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/ws/$c.json').read().strip().splitlines()[-1]);print('$c $(basename $lib)', d['value'], d['ms_per_step'])"
done; done
