"""Parity + timing report of the BASELINE configs on the GPU.

    python tools/parity_report.py [cfg1 cfg2 ...] > gpurun_out/parity.json

For every config with a full-size residual history of the REAL reference in
tests/golden/histories.json (made by tests/golden/make_golden.py --full):
iteration count, converged flag, max_k |r_k - r_k^ref| / r_0^ref, and the
per-iteration relative deviation for the iterations with r_k / r_0 >= 1e-4
(SURVEY 8c's contract).  cfg5 (2^14 x 2^20, 137 GB iterate) runs at a reduced
n_t (the n_x = 16384 row length is exercised in full) and reports convergence
only: there is no reference history at that size.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2209_06916_b200 as P  # noqa: E402
from paper_2209_06916_b200.configs import CONFIGS  # noqa: E402

hist = json.load(open(os.path.join(ROOT, "tests", "golden", "histories.json")))
names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5@16384x16384"]
out = {}
for name in names:
    if "@" in name:
        base, size = name.split("@")
        nx, nt = (int(v) for v in size.split("x"))
        cf = CONFIGS[base].scaled(nx, nt)
    else:
        cf = CONFIGS[name]
    prob = cf.problem()
    cfg = P.MgritConfig(nu=1, cycle=cf.cycle, tol=1e-10, max_iters=30, rng_seed=0)
    solver = P.MgritSolver(prob, cfg)
    u_host = solver.initial_state()
    ud = torch.from_numpy(u_host).cuda()
    solver.solve(ud.clone())  # warm-up (plans, workspaces)
    u = ud.clone()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    rep = solver.solve(u)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    row = {"n_x": cf.n_x, "n_t": cf.n_t, "iterations": rep.iterations, "converged": rep.converged,
           "final_ratio": rep.residual_norms[-1] / rep.residual_norms[0],
           "time_to_tolerance_ms": ms, "dof_per_s": cf.n_x * cf.n_t / (ms / 1e3)}
    ref = hist.get(name)
    if ref is not None:
        r0 = ref["norms"][0]
        row["reference_iterations"] = ref["iterations"]
        row["reference_wall_s"] = ref.get("wall")
        row["max_abs_dev_over_r0"] = max(abs(a - b) / r0 for a, b in zip(rep.residual_norms, ref["norms"]))
        rel = [abs(a - b) / b for a, b in zip(rep.residual_norms, ref["norms"]) if b / r0 >= 1e-4]
        row["max_rel_dev_while_r_ge_1e-4_r0"] = max(rel) if rel else None
        row["same_iterations"] = rep.iterations == ref["iterations"]
    out[name] = row
    print(json.dumps({name: row}), file=sys.stderr, flush=True)
    del u, ud, solver
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
