"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches, total,
mean and share of time per kernel (cold-cache, serialised: compare SHARES, not absolutes).
Usage: python tools/launch_summary.py launches.csv [header comment]"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) <= iv or r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void |\(.*$|unnamed>::|aos::|tfdp::", "", r[ik]).strip()
    v = float(r[iv]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[iu], 1.0)
    tot[name] += v
    cnt[name] += 1
all_us = sum(tot.values())
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print("kernel,launches,total_us,mean_us,share")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k},{cnt[k]},{tot[k]:.1f},{tot[k] / cnt[k]:.2f},{tot[k] / all_us:.3f}")
