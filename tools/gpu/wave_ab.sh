# A/B of wavefront library builds: wave_ab.sh "libA libB" reps
L=$1; R=${2:-2}
mkdir -p gpurun_out/wab
for i in $(seq $R); do for lib in $L; do
WLCS_LIB_PATH=$lib timeout 300 python bench.py --variant wavefront --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-single-pairs > gpurun_out/wab/c2.json 2>gpurun_out/wab/c2.err
python3 -c "
import json;d=json.load(open('gpurun_out/wab/c2.json'));print('c2 $(basename $lib)', d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/wab/c2.err
WLCS_LIB_PATH=$lib timeout 300 python bench.py --variant wavefront --config c4 --steps 2 --warmup 3 > gpurun_out/wab/c4.json 2>gpurun_out/wab/c4.err
python3 -c "
import json;d=json.load(open('gpurun_out/wab/c4.json'));print('c4 $(basename $lib)', d['value'], d['ms_per_step'])" || tail -3 gpurun_out/wab/c4.err
done; done
