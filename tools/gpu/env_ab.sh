# A/B of env settings (same library) on the C2 kernel: env_ab.sh "A=1 B=2" "A=3" ... (reps via R env)
R=${R:-2}
for i in $(seq $R); do for v in "$@"; do
env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-single-pairs > gpurun_out/envab.json 2>gpurun_out/envab.err
python3 -c "
import json;d=json.load(open('gpurun_out/envab.json'));print('[$v]', d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'])" || tail -3 gpurun_out/envab.err
done; done
