timeout 300 python bench.py --config c3 --steps 1 --warmup 0 > gpurun_out/b.json 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair_walk -c 1 -f -o gpurun_out/walk python bench.py --config c3 --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/walk*
