export WLCS_PAIR_K=${WLCS_PAIR_K:-4}
timeout 300 python bench.py --config c4 --steps 1 --warmup 0 > gpurun_out/c4_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair_strip -c 1 -f -o gpurun_out/c4k${WLCS_PAIR_K}${TAG} python bench.py --config c4 --steps 1 --warmup 0 > gpurun_out/ncu_c4.log 2>&1
tail -5 gpurun_out/ncu_c4.log
