for K in 0 1 2 4 8; do
  for c in c5 c3 c1; do WLCS_PAIR_K=$K timeout 300 python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/k.json 2>/dev/null; python3 -c "
import json;d=json.load(open('gpurun_out/k.json'));print('K=$K $c', d['ms_per_step'], d.get('fill_kernel_ms'))" 2>&1 | tail -1; done
done
