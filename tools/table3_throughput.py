"""Throughput of the paper's Table 3 (experiments.iteration_table over the three
grids, m = 2/4/8/16, two-level + V-cycle, ERK3 at 0.85 c_max and SDIRK3 at c = 5:
48 solves) run sequentially vs concurrently (mgrit.solve_many, one stream per
solve).  Prints one JSON line; the counts must agree between the two runs."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2209_06916_b200 as P  # noqa: E402
from paper_2209_06916_b200 import experiments as E  # noqa: E402

grids = [(64, 256), (256, 1024), (1024, 4096)]
if len(sys.argv) > 1:
    grids = grids[:int(sys.argv[1])]
runs = {}
for mode in ("warm", "sequential", "concurrent"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    table = {}
    for fam, c in (("erk", 0.85 * P.cfl_limit(3)), ("sdirk", 5.0)):
        cells = E.iteration_table(fam, 3, c, grids, [2, 4, 8, 16], max_iters=40,
                                  concurrent=(mode == "concurrent"))
        table[fam] = [(x.n_x, x.n_t, x.m, x.iters_two_level, x.iters_v_cycle) for x in cells]
    torch.cuda.synchronize()
    runs[mode] = (time.perf_counter() - t0, table)
assert runs["sequential"][1] == runs["concurrent"][1]
print(json.dumps({"solves": 2 * 2 * 4 * len(grids), "grids": grids,
                  "sequential_s": runs["sequential"][0], "concurrent_s": runs["concurrent"][0],
                  "speedup": runs["sequential"][0] / runs["concurrent"][0],
                  "table": runs["concurrent"][1]}))
