"""Extract per-launch DRAM traffic / duration of ncu raw CSVs into
profiles/traffic.json under a config key (read by bench.py for the roofline's
`traffic` field).

    python tools/ncu_traffic.py cfg4 L0.CF path/to/raw.csv [L0.FC raw2.csv ...]
"""
import csv
import json
import os
import sys

PATH = "profiles/traffic.json"
cfg = sys.argv[1]
out = json.load(open(PATH)) if os.path.exists(PATH) else {}
sec = out.setdefault(cfg, {})
for name, path in zip(sys.argv[2::2], sys.argv[3::2]):
    rows = list(csv.reader(open(path)))
    hdr, vals = rows[0], rows[2]
    get = lambda k: float(vals[hdr.index(k)].replace(",", ""))  # noqa: E731
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rs = sc.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
    ws = sc.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)
    dunit = rows[1][hdr.index("gpu__time_duration.sum")]
    ds = {"ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3,
          "ms": 1e-3}.get(dunit, 1e-9)
    rec = {"dram_read_bytes": get("dram__bytes_read.sum") * rs,
           "dram_write_bytes": get("dram__bytes_write.sum") * ws,
           "duration_s": get("gpu__time_duration.sum") * ds,
           "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
           "source": os.path.relpath(path)}
    k = "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
    if k in hdr:
        rec["fp64_pipe_active_pct"] = get(k)
    rec["dram_gbs"] = (rec["dram_read_bytes"] + rec["dram_write_bytes"]) / rec["duration_s"] / 1e9
    sec[name] = rec
json.dump(out, open(PATH, "w"), indent=1)
print(json.dumps(sec, indent=1))
