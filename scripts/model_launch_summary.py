"""Per-role summary of an ncu launch list of scripts/model_launches.py."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/model_launches.csv")))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
by = collections.OrderedDict()
for d in data:
    by.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
seq = list(by.values())
gem = [s for s in seq if "gemv" in s["name"]]
step = [s for s in seq if "step_kernel" in s["name"]]
nl = len(step)
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
for l in range(nl):
    for j, n in enumerate(("qkv", "o", "w1", "w2")):
        s = gem[4 * l + j]
        t = tot[n]
        t[0] += 1
        t[1] += s["gpu__time_duration.sum"]
        t[2] += s["dram__bytes_read.sum"]
for n, (c, ns, b) in tot.items():
    print(f"{n:4s} x{c}: {ns / c / 1e3:6.1f} us, {b / c / 1e6:6.1f} MB, {b / ns:5.0f} GB/s")
lm = gem[-1]
print(f"lm  x1: {lm['gpu__time_duration.sum'] / 1e3:6.1f} us, {lm['dram__bytes_read.sum'] / 1e6:6.1f} MB, "
      f"{lm['dram__bytes_read.sum'] / lm['gpu__time_duration.sum']:5.0f} GB/s")
print(f"gemv total {sum(s['gpu__time_duration.sum'] for s in gem) / 1e3:.1f} us, "
      f"attention (step kernel) total {sum(s['gpu__time_duration.sum'] for s in step) / 1e3:.1f} us")
