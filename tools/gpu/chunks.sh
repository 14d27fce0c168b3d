for ch in 2 4 8 16; do
WLCS_BATCH_CHUNKS=$ch timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-single-pairs > gpurun_out/ch.json 2>gpurun_out/ch.err
python3 -c "
import json;d=json.load(open('gpurun_out/ch.json'));print('chunks $ch e2e', d['e2e'])" || tail -2 gpurun_out/ch.err
done
python tools/h2d_probe.py 2>&1 | tail -5
