"""Full-size (and proxy-size) reference runs for the BASELINE parity tests.

Run in the build container, where the REAL reference (mgrit-advection 0.1.0)
is importable; the GPU box only reads the committed outputs:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_full.py CASE [--reordered]

CASE is a BASELINE config (cfg1..cfg4) or a proxy that keeps a config's level
structure at a smaller grid (``CASES`` below).  Without ``--reordered`` the real
reference solves it (mgrit.py:251-291; SDIRK with the staged fine stepper,
ERK5 with rolled sums) from the seeded iterate.  With
``--reordered`` the pinned numpy oracle solves it with blocked, reversed-order
GMRES reductions: the reference's self-noise envelope (SURVEY 0.6 / 8c /
Appendix A).

Writes ``tests/golden/full/CASE[_reordered].json`` (history, iterations, wall
time) and ``..._final.npz`` (final-iterate samples: 17 evenly spaced rows,
every row's l2 norm, the whole array's l2 norm and sum).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2209_06916_b200.configs import CONFIGS, seeded_u0  # noqa: E402

OUT = os.path.join(HERE, "full")

# name -> (config, n_x, n_t); proxies keep the config's scheme, m and level count
CASES = {
    "cfg1": ("cfg1", None, None),
    "cfg2": ("cfg2", None, None),
    "cfg3": ("cfg3", None, None),
    "cfg4": ("cfg4", None, None),
    # cfg4's five levels (its L3 operator, phi = 57 at cumulative factor 4096,
    # is active) on a 1024-point mesh
    "cfg4p": ("cfg4", 1024, 65536),
    # cfg5's 16384-point rows with cfg2's level count
    "cfg5p": ("cfg5", 16384, 16384),
    # cfg5's rows and six levels
    "cfg5q": ("cfg5", 16384, 131072),
}


def final_samples(u: np.ndarray) -> dict:
    n_t = u.shape[0] - 1
    rows = np.unique(np.linspace(0, n_t, 17).astype(np.int64))
    return dict(rows=rows, samples=u[rows].copy(), row_norms=np.sqrt(np.einsum("ij,ij->i", u, u)),
                total_norm=np.array(np.linalg.norm(u.ravel())), total_sum=np.array(u.sum()))


def run_reference(cf, n_x, n_t):
    sys.path.insert(0, "/root/reference/pkg/src")
    import mgrit_advection as R
    from mgrit_advection import circulant as RC
    from mgrit_advection import experiments as RE
    RC._ROLL_LIMIT = 64 if cf.p == 5 else RC._ROLL_LIMIT
    spec = R.DiscretizationSpec(cf.family, cf.p, cf.c, n_x, n_t)
    cyc = "v_cycle" if cf.cycle == "f_cycle" else cf.cycle
    prob = RE.build_problem(spec, cf.m, cyc, cf.coarse)
    steps = list(prob.steppers)
    if cf.family == "sdirk":
        steps[0] = R.mol_stepper(spec, mode="staged")
    prob = R.TimeGridProblem(steps, prob.m, n_t, seeded_u0(cf.u0, n_x))
    sol = R.MgritSolver(prob, R.MgritConfig(nu=1, cycle=cyc, tol=1e-10, max_iters=30, rng_seed=0))
    u = sol.initial_state()
    t0 = time.time()
    rep = sol.solve(u)
    return dict(norms=rep.residual_norms, iterations=rep.iterations, converged=rep.converged,
                wall=time.time() - t0, cycle=cyc), u


def run_reordered(cf, n_x, n_t):
    from oracle import mgrit_oracle as O
    O.ROLL_LIMIT = 64 if cf.p == 5 else 16
    cyc = "v_cycle" if cf.cycle == "f_cycle" else cf.cycle
    steps, fac, _ = O.build_hierarchy(cf.family, cf.p, cf.c, n_x, n_t, cf.m, cyc, cf.coarse,
                                      fine_mode="staged" if cf.family == "sdirk" else "assembled",
                                      reduction="reordered")
    out = O.Mgrit(steps, fac, n_t, seeded_u0(cf.u0, n_x), cycle=cyc).solve()
    return dict(norms=out["norms"], iterations=out["iterations"], converged=out["converged"],
                wall=out["wall"], cycle=cyc), out["u"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=sorted(CASES))
    ap.add_argument("--reordered", action="store_true")
    a = ap.parse_args()
    base, n_x, n_t = CASES[a.case]
    cf = CONFIGS[base]
    n_x, n_t = n_x or cf.n_x, n_t or cf.n_t
    rec, u = (run_reordered if a.reordered else run_reference)(cf, n_x, n_t)
    rec.update(config=base, n_x=n_x, n_t=n_t,
               source="oracle, reordered GMRES reductions" if a.reordered
               else "reference mgrit-advection 0.1.0")
    os.makedirs(OUT, exist_ok=True)
    name = a.case + ("_reordered" if a.reordered else "")
    np.savez_compressed(os.path.join(OUT, name + "_final.npz"), **final_samples(u))
    json.dump(rec, open(os.path.join(OUT, name + ".json"), "w"), indent=0)
    print(name, rec["iterations"], f"{rec['wall']:.1f}s", flush=True)


if __name__ == "__main__":
    main()
