export WLCS_PAIR_ROWS=1 WLCS_PAIR_SPLIT=0 WLCS_PAIR_K=${K:-4}
timeout 120 python tools/pair_probe.py 1000000 $((1024*${K:-4})) 1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair_strip -c 1 -f -o gpurun_out/solo_k${K:-4} python tools/pair_probe.py 1000000 $((1024*${K:-4})) 1 > gpurun_out/ncu_solo.log 2>&1
tail -2 gpurun_out/ncu_solo.log
