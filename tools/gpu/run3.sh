python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
bash tools/gpu/ab.sh "WLCS_LIB_PATH=tools/exp/prev.so" "WLCS_LIB_PATH=" 3
