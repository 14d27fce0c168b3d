set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json | head -c 3000
WLCS_LIB_PATH=tools/exp/trace.so timeout 300 python tools/trace_probe.py > gpurun_out/trace.txt 2>&1; echo "trace rc=$?"; cat gpurun_out/trace.txt
