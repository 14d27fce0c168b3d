"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    name = r[ki].split("(")[0].replace("wlcs::<unnamed>::", "")[:60]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
for name in sorted(tot, key=lambda n: -tot[n]):
    print(f"{name:60s} n={cnt[name]:3d}  avg={tot[name] / cnt[name] / 1000:9.2f} us")
