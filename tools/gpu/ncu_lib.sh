# ncu --set full of the batch main kernel of a given library build: ncu_lib.sh <lib.so> <out>
set -u
lib=$1; out=$2
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-single-pairs"
WLCS_LIB_PATH=$lib timeout 300 $B > /dev/null 2>&1 || { echo "bench failed"; exit 1; }
WLCS_LIB_PATH=$lib timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_main -c 1 -f -o $out $B > gpurun_out/ncu_lib.log 2>&1
tail -1 gpurun_out/ncu_lib.log
