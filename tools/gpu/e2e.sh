python tools/h2d_probe.py
for n in 1 2 4 8 16; do WLCS_BATCH_CHUNKS=$n timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e.json 2>gpurun_out/e.err; python3 -c "
import json;d=json.load(open('gpurun_out/e.json'));print('chunks $n', d['ms_per_step'], 'e2e', d['e2e']['value'])"; done
