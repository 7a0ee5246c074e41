"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
count, total, mean per kernel name.  python tools/launch_summary.py FILE.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows:
    if len(r) > vi and r[0] != "ID" and r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        k = r[ki].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
        total += v
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:6d} {t/1e6:9.3f} ms {100*t/total:5.1f}% {t/c/1e3:9.1f} us  {k}")
