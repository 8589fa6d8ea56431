"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum CSV log, over the last WSSR step
(from its energy_stats launch) and over the whole run; optionally the last N launches.
python tools/launch_table.py gpurun_out/launches.csv [last_n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
data = [(r[ii], r[ki], float(r[vi].replace(",", ""))) for r in rows[h + 1:] if len(r) > vi]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if last:
    for i, k, v in data[-last:]:
        print(f"{i:>5} {v / 1000:9.1f} us  {k[:90]}")
def totals(seq, title):
    tot = collections.defaultdict(lambda: [0.0, 0])
    for _, k, v in seq:
        if k.startswith("void at::") or "at::native" in k:
            continue
        key = k.split("(")[0][:80]
        tot[key][0] += v
        tot[key][1] += 1
    print(f"---- {title} ----")
    for k, (v, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
        print(f"{v / 1000:9.1f} us n={n:4d}  {k}")
    print(f"sum {sum(v for v, _ in tot.values()) / 1000:.1f} us")


starts = [i for i, (_, k, _) in enumerate(data) if "energy_stats" in k]
if starts:
    totals(data[starts[-1]:], "last step (cold caches, serialised: compare shares)")
tot = collections.defaultdict(lambda: [0.0, 0])
for _, k, v in []:
    if k.startswith("void at::") or "at::native" in k:
        continue
    key = k.split("(")[0][:80]
    tot[key][0] += v
    tot[key][1] += 1
totals(data, "whole run (ours)")
