# one compute-sanitizer tool over tools/sanitize/run_paths.py: tool.sh memcheck|synccheck|racecheck|initcheck
set -u
t=$1
mkdir -p gpurun_out/sanitize
timeout 300 python tools/sanitize/run_paths.py > gpurun_out/sanitize/plain_$t.txt 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize/plain_$t.txt; exit 1; }
timeout 2400 compute-sanitizer --tool $t --error-exitcode 17 --print-limit 50 python tools/sanitize/run_paths.py > gpurun_out/sanitize/$t.txt 2>&1
echo "$t rc=$?"
tail -6 gpurun_out/sanitize/$t.txt
