"""Summarise `ncu --page source --csv --print-source cuda,sass` output by source line:
warp-stall samples (all), top stall reasons per line."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None; file = None
agg = defaultdict(lambda: [0.0, defaultdict(float), ""])
for r in rows:
    if r and r[0] == "File Path": file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; idx = {h: i for i, h in enumerate(r)}; continue
    if hdr is None or not r or r[0] in ("", "Function Name"): continue
    try: v = float(r[idx["Warp Stall Sampling (All Samples)"]])
    except Exception: continue
    key = (file, r[0])
    a = agg[key]; a[0] += v; a[2] = r[1][:100]
    for h, i in idx.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try: a[1][h] += float(r[i])
            except Exception: pass
tot = sum(a[0] for a in agg.values()) or 1
reasons = defaultdict(float)
for a in agg.values():
    for k, v in a[1].items(): reasons[k] += v
rt = sum(reasons.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {v/rt:.1%}" for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:8]))
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    rs = ", ".join(f"{k[6:]} {v/max(a[0],1):.0%}" for k, v in sorted(a[1].items(), key=lambda kv: -kv[1])[:3])
    print(f"{a[0]/tot:6.1%} {f}:{ln:>4} {a[2]:60s} | {rs}")
