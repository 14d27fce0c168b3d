set -u
mkdir -p gpurun_out/r2
for t in test_core test_kernels test_parallel test_bench test_cli test_io; do
  echo "== $t"; timeout 600 tests/cpp/_ref/$t > gpurun_out/r2/$t.txt 2>&1; echo "rc=$?"; tail -3 gpurun_out/r2/$t.txt; grep -m5 ERROR gpurun_out/r2/$t.txt
done
cd gpurun_out/r2 && timeout 1500 ../../tests/cpp/_ref/acceptance > acceptance.txt 2>&1; echo "acceptance rc=$?"; cat acceptance.txt
