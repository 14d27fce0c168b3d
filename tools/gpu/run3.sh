python -m pytest tests/test_gpu_parity.py -q -x -k "subsequence or golden or c1 or c3 or checkpoint" 2>&1 | tail -2
for c in c1 c3; do WLCS_DEBUG_WALK=1 timeout 300 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/b.json 2>gpurun_out/b.err; grep "wlcs walk" gpurun_out/b.err | head -1; python3 -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print('$c',d['ms_per_step'],d.get('fill_kernel_ms'),d['config'].get('lcs_length'))" 2>&1 | tail -1; done
