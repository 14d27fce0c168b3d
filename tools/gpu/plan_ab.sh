# fused (cooperative) plan+scatter vs the two-kernel plan, C2 and small shards
for i in 1 2 3; do for f in 0 1; do for p in 65536 8192; do
WLCS_BATCH_TWO_KERNEL_PLAN=$f timeout 300 python bench.py --pairs $p --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-single-pairs > gpurun_out/pab.json 2>gpurun_out/pab.err
python3 -c "
import json;d=json.load(open('gpurun_out/pab.json'));print('two_kernel=$f pairs $p', d['ms_per_step'], d['roofline']['kernel_ms'], round(d['value']))" || tail -2 gpurun_out/pab.err
done; done; done
