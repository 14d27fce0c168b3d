# per-GPU shard sizes of an N-GPU strong-scaling run, kmax sweep (fused plan)
for p in 4096 8192 16384; do for k in 2 3 4 6 8; do
WLCS_BATCH_KMAX=$k timeout 300 python bench.py --pairs $p --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-single-pairs > gpurun_out/sb.json 2>gpurun_out/sb.err
python3 -c "
import json;d=json.load(open('gpurun_out/sb.json'));print('pairs $p kmax $k', d['ms_per_step'],d['roofline']['kernel_ms'],round(d['value']))" || tail -2 gpurun_out/sb.err
done; done
