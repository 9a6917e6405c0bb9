"""Parity + timing report on the GPU against the REAL reference's full-size runs.

    python tools/parity_report.py [case ...] > gpurun_out/parity.json

Cases are the fixtures of tests/golden/full (made by tests/golden/make_full.py
with the real reference: residual history, iteration count, final-iterate
samples; `<case>_reordered` = the oracle with reordered GMRES reductions, the
reference's own reduction-order envelope): cfg1-cfg4 at full size and the
cfg4 / cfg5 proxies.  Per case: iterations, max_k |r_k - r_k^ref| / r_0, the
relative deviation while r_k >= 1e-4 r_0, the final-iterate deviation (17
sampled rows, relative l2; every row's l2 norm, max relative) next to the same
figures of the envelope run, and the time to tolerance.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_06916_b200 as P  # noqa: E402
from paper_2209_06916_b200.configs import CONFIGS  # noqa: E402

FULL = os.path.join(ROOT, "tests", "golden", "full")
CASES = {"cfg1": ("cfg1", None, None), "cfg2": ("cfg2", None, None), "cfg3": ("cfg3", None, None),
         "cfg4": ("cfg4", None, None), "cfg4p": ("cfg4", 1024, 65536),
         "cfg5p": ("cfg5", 16384, 16384), "cfg5q": ("cfg5", 16384, 131072)}


def load(name):
    path = os.path.join(FULL, name + ".json")
    if not os.path.exists(path):
        return None, None
    return json.load(open(path)), np.load(os.path.join(FULL, name + "_final.npz"))


def final_dev(fa, fb):
    ds = np.linalg.norm(fa["samples"] - fb["samples"]) / np.linalg.norm(fb["samples"])
    dn = np.max(np.abs(fa["row_norms"] - fb["row_norms"]) / np.maximum(fb["row_norms"], 1e-300))
    return float(ds), float(dn)


out = {}
for name in sys.argv[1:] or list(CASES):
    ref, fref = load(name)
    if ref is None:
        continue
    base, n_x, n_t = CASES[name]
    cf = CONFIGS[base]
    if cf.cycle == "f_cycle":
        cf = cf.as_v_cycle()  # the reference has no F-cycle
    if n_x:
        cf = cf.scaled(n_x, n_t)
    prob = cf.problem()
    solver = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
    ud = torch.from_numpy(solver.initial_state()).cuda()
    solver.solve(ud.clone())  # warm-up (plans, workspaces)
    u = ud.clone()
    del ud
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    rep = solver.solve(u)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    un = u.cpu().numpy()
    del u
    mine = {"samples": un[fref["rows"]], "row_norms": np.sqrt(np.einsum("ij,ij->i", un, un))}
    del un
    r0 = ref["norms"][0]
    rel = [abs(a - b) / b for a, b in zip(rep.residual_norms, ref["norms"]) if b / r0 >= 1e-4]
    ds, dn = final_dev(mine, fref)
    row = {"n_x": cf.n_x, "n_t": cf.n_t, "cycle": cf.cycle, "iterations": rep.iterations,
           "reference_iterations": ref["iterations"], "converged": rep.converged,
           "final_ratio": rep.residual_norms[-1] / rep.residual_norms[0],
           "history_max_abs_dev_over_r0": max(abs(a - b) / r0
                                              for a, b in zip(rep.residual_norms, ref["norms"])),
           "history_max_rel_dev_while_r_ge_1e-4_r0": max(rel) if rel else None,
           "final_iterate_sampled_rows_rel_l2": ds, "final_iterate_row_norms_max_rel": dn,
           "time_to_tolerance_ms": ms, "dof_per_s": cf.n_x * cf.n_t / (ms / 1e3),
           "reference_wall_s": ref.get("wall")}
    env, fenv = load(name + "_reordered")
    if env is not None:
        es, en = final_dev(fenv, fref)
        row["envelope"] = {"iterations": env["iterations"],
                           "history_max_abs_dev_over_r0": max(abs(a - b) / r0 for a, b in
                                                              zip(env["norms"], ref["norms"])),
                           "final_iterate_sampled_rows_rel_l2": es,
                           "final_iterate_row_norms_max_rel": en}
    out[name] = row
    print(json.dumps({name: row}), file=sys.stderr, flush=True)
    del solver
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
