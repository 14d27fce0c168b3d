python bench.py --config c1 --steps 2 --warmup 1 > gpurun_out/c1.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c1.csv
