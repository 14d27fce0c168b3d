# ncu --set full of the cell-wavefront kernels: batch (C2) and pair (C1)
set -u
mkdir -p gpurun_out/ncu_wave
B="python bench.py --variant wavefront --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-single-pairs"
P="python bench.py --variant wavefront --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $B > /dev/null 2>&1 || { echo batch bench failed; exit 1; }
timeout 300 $P > /dev/null 2>&1 || { echo pair bench failed; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wave_batch -c 1 -f -o gpurun_out/ncu_wave/batch $B > gpurun_out/ncu_wave/batch.log 2>&1
tail -1 gpurun_out/ncu_wave/batch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wave_pair -c 1 -f -o gpurun_out/ncu_wave/pair $P > gpurun_out/ncu_wave/pair.log 2>&1
tail -1 gpurun_out/ncu_wave/pair.log
