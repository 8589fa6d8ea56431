"""Summarise an ncu launch list (gpu__time_duration per kernel) for the timed bench step."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
names = [r[idx["Kernel Name"]] for r in data]
t = [float(r[idx["Metric Value"]]) for r in data]
start = max(i for i, n in enumerate(names) if "dmma_peak" in n) + 1
agg = collections.OrderedDict()
for n, v in zip(names[start:], t[start:]):
    key = n.split("(")[0][:80]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for k, (c, v) in agg.items() if "at::" not in k)
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    tag = "" if "at::" not in k else "   [torch: drift, untimed]"
    print(f"{v/1e3:10.1f} us {100*v/tot:5.1f}% n={c:4d}  {k}{tag}")
print("total (ours) us", round(tot / 1e3, 1))
