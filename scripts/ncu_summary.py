"""Summarise an ncu --csv launch list: total / count / mean time per kernel name.
    python scripts/ncu_summary.py launches.csv [name-filter]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0.0, 0])
flt = sys.argv[2] if len(sys.argv) > 2 else None
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum" or (flt and flt not in r[ki]):
        continue
    k = r[ki].split("(")[0][:60]
    try:
        val = float(r[vi].replace(",", ""))
    except ValueError:  # "n/a": a launch ncu could not measure
        continue
    if val != val:  # "nan" (a launch ncu could not measure)
        continue
    agg[k][0] += val
    agg[k][1] += 1
tot = sum(v[0] for v in agg.values())
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}%  n={n:4d}  mean={t / n / 1e3:8.2f} us  {k}")
print(f"total {tot / 1e3:.1f} us")
