python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c2.csv
