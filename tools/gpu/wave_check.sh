# Cell-wavefront (DPX 16x2) variant: parity tests, C2 batch + C1/C4 pair benches.
set -u
mkdir -p gpurun_out/wave
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "wavefront" > gpurun_out/wave/pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/wave/pytest.txt
timeout 300 python bench.py --variant wavefront --no-single-pairs --steps 5 --warmup 3 > gpurun_out/wave/c2.json 2> gpurun_out/wave/c2.err
echo "c2 rc=$?" >> gpurun_out/wave/c2.err
timeout 300 python bench.py --variant wavefront --config c1 --steps 5 --warmup 3 > gpurun_out/wave/c1.json 2> gpurun_out/wave/c1.err
timeout 300 python bench.py --variant wavefront --config c4 --steps 3 --warmup 3 > gpurun_out/wave/c4.json 2> gpurun_out/wave/c4.err
tail -5 gpurun_out/wave/pytest.txt
for f in c2 c1 c4; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/wave/{f}.json").read().strip().splitlines()[-1])
    print(f, d.get("value"), d.get("unit"), "ms", d.get("ms_per_step"), "roof", json.dumps(d.get("roofline")))
except Exception as e:
    print(f, "ERR", e, open(f"gpurun_out/wave/{f}.err").read()[-800:])
PY
done
