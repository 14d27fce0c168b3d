for p in 8192 16384 65536; do
timeout 300 python bench.py --pairs $p --steps 20 --warmup 5 --no-cpu-baseline --no-single-pairs > gpurun_out/sb.json 2>gpurun_out/sb.err
python3 -c "
import json;d=json.load(open('gpurun_out/sb.json'));print('pairs $p', d['ms_per_step'],d['roofline']['kernel_ms'],round(d['value']), 'e2e', d['e2e']['value'])" || tail -2 gpurun_out/sb.err
done
