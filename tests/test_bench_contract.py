"""bench.py's output contract (the driver parses its last JSON line).

* the reference arm (--impl reference) runs the compiled reference only: its
  process never maps this repository's product library (the perf anchor would
  be void otherwise), and its line carries impl / cpu_baseline / e2e with the
  same workload string as the B200 arm;
* (-m gpu) the B200 arm's line carries every key of the contract: roofline,
  e2e with its copy byte counts, clocks, gpu_launches.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(text):
    lines = [ln for ln in text.strip().splitlines() if ln.startswith("{")]
    assert lines, text[-2000:]
    return json.loads(lines[-1])


def test_reference_arm_line_and_isolation():
    probe = (
        "import runpy, sys\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT_SO_MAPPED=' + str('libwavelcs_b200' in maps))\n")
    r = subprocess.run([sys.executable, "-c", probe], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "PRODUCT_SO_MAPPED=False" in r.stdout, "the reference arm loaded the product library"
    line = last_json(r.stdout.split("PRODUCT_SO_MAPPED")[0])
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "GCUPS"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    assert line["config"]["workload"] == bench.C2_CONFIG["workload"]


@pytest.mark.gpu
def test_b200_arm_line_keys():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--no-single-pairs"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = last_json(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    roof = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in roof, key
    assert 0 < roof["frac"] < 1
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 70_000_000
    assert e2e["d2h_bytes_per_step"] == 4 * 65536
    assert line["gpu_launches"] > 0
    assert line["clocks"]["sm_mhz"] is not None
