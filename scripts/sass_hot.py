"""Hot SASS lines of an ncu report (stall samples): python scripts/sass_hot.py rep.ncu-rep [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []), capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) >= len(h) - 1 and r[0].startswith("0x")]
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[S] or 0) for d in data) or 1
ti = sum(float(d["Instructions Executed"] or 0) for d in data)
print("stall samples %d, warp instructions %d" % (tot, ti))
for i in sorted(range(len(data)), key=lambda i: -float(data[i][S] or 0))[:n]:
    d = data[i]
    print("%5.1f%% %10s %s  %s" % (100 * float(d[S]) / tot, d["Instructions Executed"], d["Address"][-5:],
                                   d["Source"][:80]))
c = collections.Counter()
for d in data:
    t = d["Source"].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    c[op.split(".")[0]] += float(d["Instructions Executed"] or 0)
print(c.most_common(16))
