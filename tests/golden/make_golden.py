"""Generate golden fixtures by running the REAL reference (mgrit-advection 0.1.0).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--full]

Writes (committed, small):
  setup.npz        assembled stencil offsets/weights of every level of several
                   hierarchies, corrected-op phi / SL / D weights, c_max, constants
  relax.npz        f_relax / c_relax / restrict outputs on seeded iterates
  gmres.npz        _gmres_batched outputs (X, res, iters) on seeded batches
  histories.json   residual histories + iteration counts of small solves, the
                   exact Table-3 cells at 64x256, and (--full) the BASELINE configs
  final_u.npz      final iterates of two small solves
The seeded u0 of the BASELINE configs come from paper_2209_06916_b200.configs
(this project's definitions; the reference only ships sin^4).
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
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import mgrit_advection as R  # noqa: E402
from mgrit_advection import circulant as RC  # noqa: E402
from mgrit_advection import experiments as RE  # noqa: E402
from mgrit_advection import stepping as RS  # noqa: E402

from paper_2209_06916_b200.configs import CONFIGS, seeded_u0  # noqa: E402

HIERARCHIES = [  # (family, p, c, n_x, n_t, m, cycle, kind)
    ("erk", 1, 0.85, 1024, 1024, 8, "two_level", "modified"),
    ("erk", 3, 0.85, 4096, 16384, 8, "v_cycle", "modified"),
    ("sdirk", 3, 4.0, 4096, 16384, 4, "v_cycle", "modified"),
    ("erk", 5, 0.85, 8192, 65536, 16, "v_cycle", "modified"),
    ("erk", 3, 1.3820, 256, 1024, 4, "v_cycle", "modified"),
    ("sdirk", 3, 5.0, 64, 256, 16, "two_level", "rediscretized"),
    ("erk", 2, 0.4, 128, 256, 4, "two_level", "plain_sl"),
    ("sdirk", 1, 0.8, 32, 64, 8, "two_level", "ideal"),
]


def setup_fixture():
    out = {}
    for i, (fam, p, c, nx, nt, m, cyc, kind) in enumerate(HIERARCHIES):
        prob = RE.build_problem(R.DiscretizationSpec(fam, p, c, nx, nt), m, cyc, kind)
        out[f"h{i}_factors"] = np.array(prob.m)
        for l, st in enumerate(prob.steppers):
            out[f"h{i}_l{l}_off"] = np.asarray(st.op.offsets)
            out[f"h{i}_l{l}_w"] = np.asarray(st.op.weights)
    for p in range(1, 6):
        out[f"cmax_{p}"] = np.array(R.cfl_limit(p))
        out[f"efd_{p}"] = np.array(R.error_constant_fd(p))
        out[f"erk_err_{p}"] = np.array(R.rk_error_constant(R.erk_tableau(p)))
        out[f"sdirk_err_{p}"] = np.array(R.rk_error_constant(R.sdirk_tableau(p)))
    for j, (p, c, m, level) in enumerate([(1, 0.4, 4, 1), (3, 0.85, 8, 3), (3, 4.0, 4, 7),
                                          (5, 0.85, 16, 4), (2, 0.7, 4, 2)]):
        fam = "erk" if c < 1 else "sdirk"
        spec = R.DiscretizationSpec(fam, p, c, 256, 64)
        st = R.modified_coarse_stepper(spec, m, level)
        out[f"phi_{j}"] = np.array(RS.phi_coefficient(p, c, m, level, R.error_constant_fd(p),
                                                      R.rk_error_constant(spec.tableau())))
        sl = R.sl_stepper(p, m ** level * c, 256)
        out[f"sl_{j}_off"], out[f"sl_{j}_w"] = sl.stepper.op.offsets, sl.stepper.op.weights
        D = RS.correction_operator(p, 256)
        out[f"D_{j}_off"], out[f"D_{j}_w"] = D.offsets, D.weights
        out[f"mod_{j}_off"], out[f"mod_{j}_w"] = st.op.offsets, st.op.weights
    for j, (fam, p, c) in enumerate([("sdirk", 3, 4.0), ("erk", 3, 0.85), ("sdirk", 5, 1.3)]):
        st = R.mol_stepper(R.DiscretizationSpec(fam, p, c, 256, 8), mode="staged")
        v = np.random.default_rng(40 + j).random((3, 256))
        out[f"staged_{j}_in"], out[f"staged_{j}_out"] = v, st.apply(v)
    np.savez_compressed(os.path.join(HERE, "setup.npz"), **out)


def relax_fixture():
    out = {}
    cases = [("erk", 1, 0.85, 1024, 64, 8), ("erk", 3, 0.85, 256, 64, 8),
             ("erk", 5, 0.85, 128, 64, 16), ("sdirk", 3, 4.0, 128, 32, 4)]
    for i, (fam, p, c, nx, nt, m) in enumerate(cases):
        prob = RE.build_problem(R.DiscretizationSpec(fam, p, c, nx, nt), m, "two_level")
        sol = R.MgritSolver(prob, R.MgritConfig(rng_seed=i))
        u, g = sol.initial_state(), sol.rhs()
        saved = RC._ROLL_LIMIT
        RC._ROLL_LIMIT = 64
        try:
            out[f"c{i}_u0"] = u.copy()
            R.f_relax(u, g, prob.steppers[0], m)
            out[f"c{i}_f"] = u.copy()
            R.c_relax(u, g, prob.steppers[0], m)
            out[f"c{i}_fc"] = u.copy()
            out[f"c{i}_r"] = R.restrict_residual(u, g, prob.steppers[0], m)
        finally:
            RC._ROLL_LIMIT = saved
    np.savez_compressed(os.path.join(HERE, "relax.npz"), **out)


def gmres_fixture():
    out = {}
    cases = [(3, 0.85, 256, 8, 8, 20), (3, 0.85, 256, 8, 512, 20), (5, 0.85, 128, 16, 256, 20),
             (1, 0.6, 64, 4, 16, 10)]
    for i, (p, c, nx, m, cum, cap) in enumerate(cases):
        spec = R.DiscretizationSpec("erk", p, c, nx, 64)
        e_fd, e_rk = R.error_constant_fd(p), R.rk_error_constant(spec.tableau())
        phi = RS.phi_coefficient(p, c, cum, 1, e_fd, e_rk)
        D = RS.correction_operator(p, nx)
        corr = RC.CirculantOperator.identity(nx) - D.scale(phi)
        B = np.random.default_rng(100 + i).standard_normal((6, nx))
        B[2] = 0.0  # zero right-hand side row
        X, res, its, brk = RC._gmres_batched(corr, B, 1e-2, cap)
        out[f"g{i}_off"], out[f"g{i}_w"] = corr.offsets, corr.weights
        out[f"g{i}_B"], out[f"g{i}_X"], out[f"g{i}_res"] = B, X, res
        out[f"g{i}_meta"] = np.array([its, int(brk), cap])
    np.savez_compressed(os.path.join(HERE, "gmres.npz"), **out)


def _solve(fam, p, c, nx, nt, m, cyc, kind="modified", u0=None, staged=False, roll64=False,
           seed=0, max_iters=30, nu=1):
    saved = RC._ROLL_LIMIT
    if roll64:
        RC._ROLL_LIMIT = 64
    try:
        spec = R.DiscretizationSpec(fam, p, c, nx, nt)
        prob = RE.build_problem(spec, m, cyc, kind)
        steps = list(prob.steppers)
        if staged:
            steps[0] = R.mol_stepper(spec, mode="staged")
        prob = R.TimeGridProblem(steps, prob.m, nt, prob.u0 if u0 is None else u0)
        cfg = R.MgritConfig(nu=nu, cycle=cyc, max_iters=max_iters, rng_seed=seed)
        sol = R.MgritSolver(prob, cfg)
        u = sol.initial_state()
        t0 = time.time()
        rep = sol.solve(u)
        return rep, u, time.time() - t0
    finally:
        RC._ROLL_LIMIT = saved


def history_fixture(full: bool):
    path = os.path.join(HERE, "histories.json")
    hist = json.load(open(path)) if os.path.exists(path) else {}
    small = {
        "erk1_tl_256x256": ("erk", 1, 0.85, 256, 256, 8, "two_level"),
        "erk3_v_256x1024": ("erk", 3, 0.85 * R.cfl_limit(3), 256, 1024, 8, "v_cycle"),
        "erk1_v_256x1024": ("erk", 1, 0.85, 256, 1024, 4, "v_cycle"),
        "sdirk3_v_256x1024_staged": ("sdirk", 3, 4.0, 256, 1024, 4, "v_cycle"),
        "sdirk3_tl_64x256_redisc": ("sdirk", 3, 5.0, 64, 256, 16, "two_level", "rediscretized"),
        "erk5_v_256x4096_roll64": ("erk", 5, 0.85, 256, 4096, 16, "v_cycle"),
    }
    finals = {}
    for name, args in small.items():
        kind = args[7] if len(args) > 7 else "modified"
        rep, u, wall = _solve(*args[:7], kind=kind, staged="staged" in name,
                              roll64="roll64" in name)
        hist[name] = dict(norms=rep.residual_norms, iterations=rep.iterations,
                          converged=rep.converged, wall=wall)
        if name in ("erk1_tl_256x256", "sdirk3_v_256x1024_staged"):
            finals[name] = u
    np.savez_compressed(os.path.join(HERE, "final_u.npz"), **finals)
    for fam, c in (("erk", 0.85 * R.cfl_limit(3)), ("sdirk", 5.0)):
        for m in (2, 4, 8, 16):
            for cyc in ("two_level", "v_cycle"):
                rep, _, wall = _solve(fam, 3, c, 64, 256, m, cyc, max_iters=40)
                hist[f"table3_{fam}_64x256_m{m}_{cyc}"] = dict(
                    norms=rep.residual_norms, iterations=rep.iterations,
                    converged=rep.converged, wall=wall)
    json.dump(hist, open(path, "w"), indent=0)
    if not full:
        return
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        if name in hist:
            continue
        cf = CONFIGS[name]
        rep, _, wall = _solve(cf.family, cf.p, cf.c, cf.n_x, cf.n_t, cf.m, cf.cycle,
                              u0=seeded_u0(cf.u0, cf.n_x), staged=cf.family == "sdirk",
                              roll64=cf.p == 5)
        hist[name] = dict(norms=rep.residual_norms, iterations=rep.iterations,
                          converged=rep.converged, wall=wall)
        json.dump(hist, open(path, "w"), indent=0)
        print(name, rep.iterations, f"{wall:.1f}s", flush=True)


def cli_fixture():
    """Reference CLI output (cli.py solve/iters) for the CLI parity tests."""
    from mgrit_advection import cli as RCLI
    runs = {
        "cli_solve_erk1_tl.csv": ["solve", "--family", "erk", "--p", "1", "--c", "0.85", "--grid",
                                  "64,256", "--m", "4", "--cycle", "two-level", "--threads", "1"],
        "cli_solve_sdirk3_v.csv": ["solve", "--family", "sdirk", "--p", "3", "--c", "4", "--grid",
                                   "64,256", "--m", "4", "--cycle", "v", "--threads", "1"],
        "cli_iters_erk3.csv": ["iters", "--family", "erk", "--p", "3", "--c-fraction", "0.85",
                               "--grid", "64,256", "--m", "4,8", "--threads", "1"],
    }
    for name, argv in runs.items():
        path = os.path.join(HERE, name)
        assert RCLI.main(argv + ["--out", path]) == 0


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--only-full", action="store_true")
    ap.add_argument("--cli", action="store_true")
    a = ap.parse_args()
    if a.cli:
        cli_fixture()
        raise SystemExit(0)
    if not a.only_full:
        setup_fixture()
        relax_fixture()
        gmres_fixture()
    history_fixture(a.full or a.only_full)
