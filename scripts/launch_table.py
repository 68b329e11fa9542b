"""Median duration per kernel name of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = {}
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        try:
            t = float(r[-1].replace(",", ""))
        except ValueError:
            continue
        agg.setdefault(name, []).append(t)
unit = rows[[i for i, r in enumerate(rows) if "Kernel Name" in r][0] + 1][-1] if h else ""
tot = 0.0
for n, v in agg.items():
    v = sorted(v)
    med = v[len(v) // 2] / (1000.0 if unit in ("ns", "nsecond") else 1.0)
    tot += med
    print("%-32s n=%3d median %8.1f us" % (n[:32], len(v), med))
print("sum of medians %.1f us" % tot)
