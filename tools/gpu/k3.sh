for r in 1 2; do for v in "X=1" "WLCS_PAIR_K=3 WLCS_PAIR_K3=1"; do for c in c4 c5; do
env $v timeout 300 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/k3.json 2>gpurun_out/k3.err
python3 -c "
import json;d=json.loads(open('gpurun_out/k3.json').read().strip().splitlines()[-1]);print('[$v] $c',d['ms_per_step'],d['fill_kernel_ms'],d['config']['lcs_length'])" 2>&1 | tail -1
done; done; done
