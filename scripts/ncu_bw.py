"""Per-kernel time and DRAM bandwidth from an ncu --csv launch list captured
with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
    python scripts/ncu_bw.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ii, ki, mi, vi = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
launch = defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    if unit is not None:
        v *= scale.get(r[unit], 1)
    launch[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki].split("(")[0][:56]
agg = defaultdict(lambda: [0.0, 0.0, 0])
for i, m in launch.items():
    a = agg[names[i]]
    a[0] += m.get("gpu__time_duration.sum", 0.0)
    a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a[2] += 1
tot = sum(v[0] for v in agg.values())
for k, (t, b, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{t / 1e3:9.1f} us {100 * t / tot:5.1f}%  n={n:4d}  mean={t / n / 1e3:7.2f} us  "
          f"{b / 1e6:9.1f} MB  {b / max(t, 1):7.1f} GB/s  {k}")
print(f"total {tot / 1e3:.1f} us, {sum(v[1] for v in agg.values()) / 1e9:.3f} GB")
