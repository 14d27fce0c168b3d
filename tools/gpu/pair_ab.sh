# A/B of library builds on the single-pair configs: pair_ab.sh "libA libB ..." [reps] [configs]
L=${1:-"paper_1306_4627_b200/_lib/libwavelcs_b200.so"}; R=${2:-2}; C=${3:-"c4 c5"}
for i in $(seq $R); do for c in $C; do for lib in $L; do
WLCS_LIB_PATH=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/pab.json 2>gpurun_out/pab.err
python3 -c "
import json;d=json.load(open('gpurun_out/pab.json'));print('$c', '$(basename $lib)', d['fill_kernel_ms'], d['ms_per_step'], d['config']['lcs_length'])" || tail -3 gpurun_out/pab.err
done; done; done
