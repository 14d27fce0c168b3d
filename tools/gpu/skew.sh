# Strip hand-off skew: fill time vs strip count at fixed rows (K=4: 4096
# columns per strip), and the C4 shape at K = 2/4/8.  Measured (round 1):
# 1 strip 3.41 ms, 2 strips 3.74 ms, 16 strips 3.91 ms at 200k rows (12.5k
# steps): ~38-41 steps of skew per strip; C4 K=4 12.6 ms vs K=2 22.6, K=8 19.6.
for s in 1 2 4 8 16; do
  WLCS_PAIR_K=4 WLCS_PAIR_SPLIT=0 WLCS_PAIR_ROWS=1 python tools/pair_probe.py 200000 $((4096 * s)) 3 | sed "s/^/strips=$s /"
done
for K in 2 4 8; do WLCS_PAIR_K=$K python tools/pair_probe.py 1000000 1000000 2 | sed "s/^/C4 K=$K /"; done
