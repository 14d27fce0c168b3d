# single-pair strip kernel (C4): one ncu --set full capture after a plain run
timeout 300 python bench.py --config c4 --steps 1 --warmup 0 > gpurun_out/c4_plain.json 2>&1 || exit 1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pair_strip -c 1 -f -o gpurun_out/c4_strip python bench.py --config c4 --steps 1 --warmup 0 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
