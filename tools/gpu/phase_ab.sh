set -u
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
WLCS_LIB_PATH=tools/exp/trace.so python tools/trace_probe.py
bash tools/gpu/ab.sh "WLCS_LIB_PATH=tools/exp/base.so" "X=1" 3
