"""Per-kernel totals of an ncu launch list (``--metrics gpu__time_duration.sum
--csv``): tools/launch_summary.py launches.csv > launch_summary.txt"""
import csv
import sys
from collections import defaultdict


def main(path):
    tot, cnt = defaultdict(float), defaultdict(int)
    with open(path) as f:
        rows = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(rows):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        tot[name] += float(r["Metric Value"]) / 1e3
        cnt[name] += 1
    allt = sum(tot.values())
    print("ncu launch list of `python bench.py --steps 1 --warmup 1 --no-cpu-baseline` "
          "(cold-cache, serialised; all kernels of warm-up + timed + profiled solves)")
    print(f"{'kernel':60s} {'launches':>9s} {'total_us':>12s} {'share':>7s}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k[:60]:60s} {cnt[k]:9d} {tot[k]:12.1f} {tot[k] / allt:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
