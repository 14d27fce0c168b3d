timeout 300 python bench.py --config c4 --colsplit --steps 2 --warmup 1 2>&1 | tail -3
