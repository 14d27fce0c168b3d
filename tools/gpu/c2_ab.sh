# A/B of library builds on the C2 batch kernel, interleaved: c2_ab.sh "libA libB ..." [reps] [extra bench args]
L=$1; R=${2:-3}; shift 2; X="$@"
for i in $(seq $R); do for lib in $L; do
WLCS_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-single-pairs $X > gpurun_out/c2ab.json 2>gpurun_out/c2ab.err
python3 -c "
import json;d=json.load(open('gpurun_out/c2ab.json'));print('$(basename $lib)', d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/c2ab.err
done; done
