# A/B of env settings on the C2 kernel time, interleaved: ab.sh "ENV_A" "ENV_B" [reps]
A=$1; B=$2; R=${3:-3}
for i in $(seq $R); do for v in "$A" "$B"; do
env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
python3 -c "
import json;d=json.load(open('gpurun_out/ab.json'));print('[$v]',d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'])"
done; done
