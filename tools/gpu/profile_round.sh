# Round-end measurement set: bench lines (C2 headline + reference arm + the
# single-pair configs + variants) and the ncu launch list of the headline
# command (ncu only after the same command exited 0 without it).
set -u
mkdir -p gpurun_out/prof
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/prof/pytest_gpu.txt
python bench.py > gpurun_out/prof/bench_c2.json 2> gpurun_out/prof/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err
python bench.py --variant wavefront --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c2_wavefront.json 2>&1
for c in c1 c3 c4 c5; do python bench.py --config $c --steps 3 --warmup 1 > gpurun_out/prof/bench_$c.json 2>&1; done
python bench.py --config c4 --colsplit --steps 3 --warmup 1 > gpurun_out/prof/bench_c4_colsplit.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/c2_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/prof/launches_c2.csv > gpurun_out/prof/launches_c2.txt 2>&1
cat gpurun_out/prof/pytest_gpu.txt gpurun_out/prof/launches_c2.txt
ls gpurun_out/prof/
