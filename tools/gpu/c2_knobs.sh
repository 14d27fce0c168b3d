# C2 batch kernel: mask-budget / lane-shape knob sweep (kernel ms), then one
# ncu --set full capture with source counters of the default configuration.
set -u
mkdir -p gpurun_out/knobs
for kv in "12 33" "8 22" "8 24" "10 33" "6 17" "4 12"; do
  set -- $kv
  WLCS_BATCH_KMAX=$1 WLCS_BATCH_PM_KB=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/knobs/k$1_pm$2.json 2>&1
  python3 -c "
import json;d=json.loads(open('gpurun_out/knobs/k$1_pm$2.json').read().strip().splitlines()[-1]);r=d['roofline'];print('kmax=$1 pm=$2', d['value'], r['kernel_ms'], r['frac'])"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_main -c 1 -f -o gpurun_out/knobs/c2main python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/knobs/ncu.log 2>&1
tail -2 gpurun_out/knobs/ncu.log
