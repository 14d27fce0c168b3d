timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_main -c 1 -f -o gpurun_out/c2main python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
tail -2 gpurun_out/ncu_c2.log
