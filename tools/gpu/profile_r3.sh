# Measurement set after the round-2 (second session) batch changes: the full
# GPU suite, smoke, the default bench line (C2 + C1/C3/C4/C5 blocks), the
# reference arm, the launch list of a short bench, and ncu --set full of the
# batch main kernel (each ncu pass only after its plain run exited 0).
set -u
O=gpurun_out/${PROF_OUT:-prof3}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-single-pairs"
timeout 300 $B > $O/c2_short.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $B > /dev/null 2>&1
python tools/launches.py $O/launches_c2.csv > $O/launches_c2.txt 2>&1
M="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-single-pairs"
timeout 300 $M > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_main -c 1 -f -o $O/c2main $M > $O/ncu_c2.log 2>&1
ls -la $O; tail -12 $O/launches_c2.txt
