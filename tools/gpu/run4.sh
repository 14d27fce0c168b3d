for c in c1 c3; do WLCS_DEBUG_WALK=1 timeout 300 python bench.py --config $c --steps 2 --warmup 1 > gpurun_out/b.json 2>gpurun_out/b.err; echo "$c"; grep "wlcs walk" gpurun_out/b.err | tail -3; done
