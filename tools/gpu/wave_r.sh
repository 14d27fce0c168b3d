# pair-kernel rows-per-lane sweep on C1 / C4 (WLCS_WAVE_PAIR_R), plus the C2 batch
mkdir -p gpurun_out/wr
timeout 300 python bench.py --variant wavefront --no-single-pairs --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wr/c2.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/wr/c2.json').read().strip().splitlines()[-1]);print('c2', d['value'], d['roofline']['kernel_ms'])"
for R in 4 8 16; do for c in c1 c4; do
WLCS_WAVE_PAIR_R=$R timeout 300 python bench.py --variant wavefront --config $c --steps 2 --warmup 3 > gpurun_out/wr/$c.json 2>&1
python3 -c "import json;d=json.loads(open('gpurun_out/wr/$c.json').read().strip().splitlines()[-1]);print('$c R=$R', d['value'], d['ms_per_step'])"
done; done
