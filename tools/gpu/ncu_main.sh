# ncu --set full of the batch main kernel (one launch of the C2 bench)
set -u
out=${1:-gpurun_out/c2main_new}
mkdir -p $(dirname $out)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-single-pairs"
timeout 300 $B > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_main -c 1 -f -o $out $B > gpurun_out/ncu_main.log 2>&1
tail -1 gpurun_out/ncu_main.log
