# occupancy at fixed lane shapes: kmax=8 with 33 / 26 / 22 KB mask budgets (6 / 8 / 9 warps per SM)
for r in 1 2; do for kv in "8 33" "8 26" "8 22" "12 33" "10 33"; do
  set -- $kv
  WLCS_BATCH_KMAX=$1 WLCS_BATCH_PM_KB=$2 timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/o.json 2>&1
  python3 -c "
import json;d=json.loads(open('gpurun_out/o.json').read().strip().splitlines()[-1]);r=d['roofline'];print('kmax=$1 pm=$2', r['kernel_ms'], r['frac'])"
done; done
