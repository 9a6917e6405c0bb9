"""Instructions executed per source line from `ncu --page source --csv` output.

    python tools/ncu_inst_summary.py gpurun_out/<tag>_source.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = defaultdict(lambda: [0.0, ""])
f = None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r:
        continue
    try:
        v = float(r[hdr["Instructions Executed"]])
    except Exception:
        continue
    a = agg[(f, r[0])]
    a[0] += v
    a[1] = r[1][:90]
tot = sum(a[0] for a in agg.values()) or 1
print("total warp instructions", tot)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a[0]/tot:6.1%} {k[0]}:{k[1]:>4} {a[1]}")
