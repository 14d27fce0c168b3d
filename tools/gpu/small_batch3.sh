# C2 per-GPU shard sizes of a strong-scaling run (65536 / N pairs) on one GPU with the default lane shapes
for p in 8192 16384 32768 65536; do
timeout 300 python bench.py --pairs $p --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-single-pairs > gpurun_out/sb.json 2>gpurun_out/sb.err
python3 -c "
import json;d=json.load(open('gpurun_out/sb.json'));print('pairs $p', d['ms_per_step'],d['roofline']['kernel_ms'],round(d['value']), d['roofline']['frac'])" || tail -2 gpurun_out/sb.err
done
