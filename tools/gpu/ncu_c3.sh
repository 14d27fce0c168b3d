# ncu --set full of the C3 STORE fill (pair_strip_kernel<K,1>)
set -u
mkdir -p gpurun_out/ncu_c3
B="python bench.py --config c3 --steps 1 --warmup 1"
timeout 300 $B > /dev/null 2>&1 || { echo bench failed; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair_strip -c 1 -f -o gpurun_out/ncu_c3/c3 $B > gpurun_out/ncu_c3/log 2>&1
tail -1 gpurun_out/ncu_c3/log
