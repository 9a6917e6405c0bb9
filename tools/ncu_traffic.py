"""Extract per-launch DRAM traffic / duration of an ncu raw CSV into profiles/traffic.json
(read by bench.py for the roofline's `traffic` field)."""
import csv, json, os, sys
out = {}
for name, path in zip(sys.argv[1::2], sys.argv[2::2]):
    rows = list(csv.reader(open(path)))
    hdr, vals = rows[0], rows[2]
    get = lambda k: float(vals[hdr.index(k)].replace(",", ""))
    unit = rows[1][hdr.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    wunit = rows[1][hdr.index("dram__bytes_write.sum")]
    wscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(wunit, 1)
    dunit = rows[1][hdr.index("gpu__time_duration.sum")]
    dscale = {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(dunit, 1e-9)
    out[name] = {"dram_read_bytes": get("dram__bytes_read.sum") * scale,
                 "dram_write_bytes": get("dram__bytes_write.sum") * wscale,
                 "duration_s": get("gpu__time_duration.sum") * dscale,
                 "source": os.path.relpath(path)}
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
