# Round-2 check: GPU parity suite, the default bench line, the reference arm.
set -u
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err
echo "bench rc=$?" >> gpurun_out/r2/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2/ref.json 2> gpurun_out/r2/ref.err
echo "ref rc=$?" >> gpurun_out/r2/ref.err
tail -5 gpurun_out/r2/pytest_gpu.txt; tail -c 3000 gpurun_out/r2/bench.json; tail -3 gpurun_out/r2/bench.err; cat gpurun_out/r2/ref.json | head -c 600; tail -2 gpurun_out/r2/ref.err
