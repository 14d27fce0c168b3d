# Round-2 measurement set: the default bench line (C2 + c4/c5 blocks), the
# reference arm, the launch list of a short bench, and ncu --set full of the
# batch main kernel and of the C4 / C5 strip kernels (each only after its
# plain run exited 0).
set -u
O=gpurun_out/prof2
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-single-pairs"
timeout 300 $B > $O/c2_short.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $B > /dev/null 2>&1
python tools/launches.py $O/launches_c2.csv > $O/launches_c2.txt 2>&1
M="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-single-pairs"
timeout 300 $M > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_main -c 1 -f -o $O/c2main $M > $O/ncu_c2.log 2>&1
for c in c4 c5; do
  P="python bench.py --config $c --steps 1 --warmup 0"
  timeout 300 $P > $O/plain_$c.json 2>&1 && \
    timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pair_strip -c 1 -f -o $O/strip_$c $P > $O/ncu_$c.log 2>&1
done
ls -la $O; cat $O/launches_c2.txt | tail -12
