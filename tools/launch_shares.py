"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count, total device time and share of the total."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) <= mv:
        continue
    name = r[kn].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    agg[name][0] += 1
    agg[name][1] += float(r[mv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[-48:]:48s} n={v[0]:5d} total={v[1] / 1e3:10.1f} us  mean={v[1] / v[0] / 1e3:9.2f} us  share={v[1] / tot:.3f}")
