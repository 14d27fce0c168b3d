# e2e of the C2 host batch: chunk count x tapered / equal chunks
for i in 1 2; do for cfg in "3 1" "2 1" "3 0" "2 0"; do set -- $cfg
WLCS_BATCH_CHUNKS=$1 WLCS_BATCH_TAPER=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-single-pairs > gpurun_out/tp.json 2>gpurun_out/tp.err
python3 -c "
import json;d=json.loads(open('gpurun_out/tp.json').read().strip().splitlines()[-1]);print('chunks $1 taper $2 e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'dev', d['value'])" || tail -2 gpurun_out/tp.err
done; done
