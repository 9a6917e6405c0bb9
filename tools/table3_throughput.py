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

GRIDS = [(64, 256), (256, 1024), (1024, 4096)]
STREAMS = int(os.environ.get("T3_STREAMS", "8"))


def table(grids, mode):
    out = {}
    for fam, c in (("erk", 0.85 * P.cfl_limit(3)), ("sdirk", 5.0)):
        cells = E.iteration_table(fam, 3, c, grids, [2, 4, 8, 16], max_iters=40,
                                  concurrent=mode != "sequential",
                                  streams=1 if mode == "graphs_1stream" else STREAMS)
        out[fam] = [(x.n_x, x.n_t, x.m, x.iters_two_level, x.iters_v_cycle) for x in cells]
    return out


res = {"streams": STREAMS, "per_grid": []}
for grids in [[g] for g in GRIDS] + [GRIDS]:
    times = {}
    tabs = {}
    for mode in ("sequential", "graphs_1stream", "concurrent"):
        table(grids, mode)  # warm: plans, workspaces, module load
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tabs[mode] = table(grids, mode)
        torch.cuda.synchronize()
        times[mode] = time.perf_counter() - t0
    assert tabs["sequential"] == tabs["concurrent"] == tabs["graphs_1stream"]
    res["per_grid"].append({"grids": grids, "solves": 16 * len(grids),
                            "sequential_s": times["sequential"],
                            "graphs_1stream_s": times["graphs_1stream"],
                            "concurrent_s": times["concurrent"],
                            "speedup": times["sequential"] / times["concurrent"]})
res["table"] = tabs["concurrent"]
print(json.dumps(res))
