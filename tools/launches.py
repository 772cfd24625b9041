"""Summarise an ncu launch list (gpu__time_duration per kernel) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in data:
    if len(r) > vi:
        agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    big = sorted(v)[len(v) // 4:]          # drop the small warm-up launches
    print(f"{k[:48]:48s} n={len(v):5d} total={sum(v)/1e6:8.3f} ms  mean={sum(v)/len(v)/1e3:8.2f} us"
          f"  upper-3/4 mean={sum(big)/len(big)/1e3:8.2f} us  share={sum(v)/tot:.3f}")
