# Full check: GPU parity suite, smoke, the default bench line, the reference arm.
set -u
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/fin/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/fin/smoke.txt
timeout 600 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
echo "bench rc=$?" >> gpurun_out/fin/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin/ref.json 2> gpurun_out/fin/ref.err
echo "ref rc=$?" >> gpurun_out/fin/ref.err
tail -3 gpurun_out/fin/pytest_gpu.txt; tail -2 gpurun_out/fin/smoke.txt; tail -2 gpurun_out/fin/bench.err; tail -2 gpurun_out/fin/ref.err
