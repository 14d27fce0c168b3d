python tools/handoff_probe.py 400000 || exit 1
ncu --set full --import-source on --clock-control none -k regex:pair_strip --launch-skip 6 -c 1 -f -o gpurun_out/consumer python tools/handoff_probe.py 400000 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:pair_strip --launch-skip 0 -c 1 -f -o gpurun_out/solo4 python tools/handoff_probe.py 400000 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
