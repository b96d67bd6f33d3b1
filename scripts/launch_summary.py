"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) == len(hdr)]
if last:
    data = data[-last:]
agg = collections.OrderedDict()
for n, v in data:
    key = n.split("(")[0].replace("void ", "")[:70]
    agg.setdefault(key, []).append(v)
tot = sum(v for _, v in data)
print(f"{len(data)} launches, total {tot / 1e3:.1f} us")
for n, v in agg.items():
    print(f"{n:70s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:8.2f}us total={sum(v) / 1e3:9.1f}us "
          f"share={sum(v) / tot * 100:5.1f}%")
