"""Mean gpu__time_duration per kernel from an `ncu --csv --metrics gpu__time_duration.sum` log."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), len(hdr) - 1
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")[:60]
    try:
        agg.setdefault(name, []).append(float(r[vi]))
    except ValueError:
        pass
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v) / 1000:9.1f} us  {k}")
