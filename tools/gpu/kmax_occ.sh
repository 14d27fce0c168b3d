# kmax / mask budget (occupancy) sweep on the C2 batch kernel
for i in 1 2; do for cfg in "10 0" "7 19" "6 17" "8 22" "5 14"; do set -- $cfg
WLCS_BATCH_KMAX=$1 WLCS_BATCH_PM_KB=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-single-pairs > gpurun_out/ko.json 2>gpurun_out/ko.err
python3 -c "
import json;d=json.loads(open('gpurun_out/ko.json').read().strip().splitlines()[-1]);print('kmax $1 pmkb $2', d['roofline']['kernel_ms'], d['ms_per_step'])" || tail -2 gpurun_out/ko.err
done; done
