"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bitwise where the reference's arithmetic is
reproducible (rolled-sum stencils in exact mode), tolerance-bounded where it
is not (FFT solves, GMRES reductions); every tolerance is written here."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O


def rng_rows(seed, rows, n):
    return np.random.default_rng(seed).random((rows, n))


# ------------------------------------------------------------ stencil apply

@pytest.mark.parametrize("p,c,n", [(1, 0.85, 1024), (3, 0.85, 4096), (3, 1.382, 256),
                                   (5, 0.85, 512), (2, 0.4, 64), (4, 0.5, 96), (1, 0.3, 17)])
def test_erk_stencil_apply_bitwise(p, c, n):
    spec = P.DiscretizationSpec("erk", p, c, n, 8)
    st = P.mol_stepper(spec)
    ost = O.mol_step("erk", p, c, n)
    v = rng_rows(p, 37, n)
    saved = O.ROLL_LIMIT
    O.ROLL_LIMIT = 64  # rolled sums for every tap count (ERK5 has 31 taps)
    try:
        ref = ost.apply(v)
    finally:
        O.ROLL_LIMIT = saved
    out = st.apply(v)
    assert np.array_equal(out, ref)


def test_user_circulant_apply_matches_dense():
    rng = np.random.default_rng(11)
    n = 32
    offs = np.arange(-14, 14)
    w = rng.standard_normal(len(offs)) * np.exp(-0.3 * np.abs(offs))
    op = P.CirculantOperator.from_arrays(n, offs, w)
    v = rng.standard_normal(n)
    np.testing.assert_allclose(op.apply(v), op.dense() @ v, atol=1e-12)


@pytest.mark.parametrize("n", [8, 17, 32, 100, 1024])
def test_shift_and_identity(n):
    v = np.arange(float(n))
    assert np.array_equal(P.CirculantOperator.identity(n).apply(v), v)
    assert np.array_equal(P.CirculantOperator.shift(n, -3).apply(v), np.roll(v, 3))


# ------------------------------------------------------------- f-relaxation

@pytest.mark.parametrize("p,c,n,nt,m", [(1, 0.85, 1024, 1024, 8), (3, 0.85, 4096, 256, 8),
                                        (5, 0.85, 512, 256, 16), (3, 1.382, 64, 64, 4),
                                        (3, 0.85, 16384, 64, 8),
                                        # fixed-geometry builds of the explicit kernel: 16 x 256
                                        # and 16 x 512 threads, 31-tap ERK5 stencils, many
                                        # intervals per CTA (4096 x 4096: 512 intervals / 296 CTAs)
                                        (5, 0.85, 4096, 64, 16), (5, 0.85, 8192, 64, 16),
                                        (3, 0.85, 8192, 64, 8), (1, 0.85, 8192, 32, 8),
                                        (3, 0.85, 4096, 4096, 8)])
def test_f_relax_bitwise(p, c, n, nt, m):
    spec = P.DiscretizationSpec("erk", p, c, n, nt)
    st = P.mol_stepper(spec)
    ost = O.mol_step("erk", p, c, n)
    u = O.initial_iterate(0, nt, n, O.sin4(n))
    g = np.zeros_like(u)
    g[0] = u[0]
    uo = u.copy()
    saved = O.ROLL_LIMIT
    O.ROLL_LIMIT = 64
    try:
        O.f_relax(uo, g, ost, m)
        ug = u.copy()
        P.f_relax(ug, g, st, m)
        assert np.array_equal(ug, uo)
        O.c_relax(uo, g, ost, m)
        P.c_relax(ug, g, st, m)
        assert np.array_equal(ug, uo)
        r_ref = O.restrict(uo, g, ost, m)
    finally:
        O.ROLL_LIMIT = saved
    r = P.restrict_residual(ug, g, st, m)
    assert np.array_equal(r, r_ref)
    nref = float(np.linalg.norm(r_ref.ravel()))
    assert abs(P.cpoint_residual_norm(ug, g, st, m) - nref) <= 1e-14 * nref


# ---------------------------------------------------- coarse / implicit ops

@pytest.mark.parametrize("fam,p,c,n,m,level", [("erk", 1, 0.85, 1024, 8, 1),
                                               ("sdirk", 3, 4.0, 512, 4, 1),
                                               ("sdirk", 3, 4.0, 512, 4, 5),
                                               ("erk", 3, 0.85, 256, 8, 2)])
def test_corrected_direct_apply(fam, p, c, n, m, level):
    spec = P.DiscretizationSpec(fam, p, c, n, 64)
    st = P.modified_coarse_stepper(spec, m, 1, solver="direct", cumulative_factor=m ** level)
    ost = O.corrected_coarse(fam, p, c, n, m, 1, "direct", cumulative=m ** level)
    v = rng_rows(3, 9, n)
    ref = ost.apply(v)  # assembled pruned stencil via FFT (reference path)
    out = st.apply(v)
    # exact SL + factorised banded solve vs pruned assembled FFT: rounding of
    # kappa(I - phi D) ~ 1 + 16|phi| times eps, plus the 1e-14 pruning
    phi = abs(st.phi)
    tol = 1e-13 * (1 + 16 * phi) + 1e-13
    assert np.max(np.abs(out - ref)) <= tol * np.max(np.abs(ref))


@pytest.mark.parametrize("n", [64, 1000, 4096])
def test_solve_direct_roundtrip(n):
    D = P.high_derivative_operator(2, 2, "symmetric", n)
    op = P.CirculantOperator.identity(n) - D.scale(0.36)
    v = np.random.default_rng(0).standard_normal(n)
    x = op.solve_direct(O.Circ(n, op.offsets, op.weights).apply(v))
    np.testing.assert_allclose(x, v, atol=1e-12)


def test_solve_direct_singular_raises():
    op = P.CirculantOperator(8, [(0, 1.0), (-1, -1.0)])
    with pytest.raises(P.SingularOperatorError):
        op.solve_direct(np.ones(8))


@pytest.mark.parametrize("fam,p,c,n", [("sdirk", 3, 4.0, 4096), ("sdirk", 1, 1.0, 64),
                                       ("sdirk", 2, 1.3, 256), ("sdirk", 5, 1.3, 128),
                                       ("erk", 3, 0.85, 256)])
def test_staged_rk_apply(fam, p, c, n):
    spec = P.DiscretizationSpec(fam, p, c, n, 8)
    st = P.mol_stepper(spec, mode="staged")
    ost = O.mol_step(fam, p, c, n, mode="staged")
    v = rng_rows(5, 6, n)
    ref = ost.apply(v)
    out = st.apply(v)
    if fam == "erk":
        assert np.array_equal(out, ref)
    else:
        np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13 * np.max(np.abs(ref)))


@pytest.mark.parametrize("p,c,n,m,cum", [(3, 0.85, 256, 8, 8), (3, 0.85, 4096, 8, 64),
                                         (5, 0.85, 1024, 16, 256), (1, 0.6, 64, 4, 16)])
def test_gmres_coarse_apply(p, c, n, m, cum):
    spec = P.DiscretizationSpec("erk", p, c, n, 64)
    cap = 10 if p == 1 else 20
    st = P.modified_coarse_stepper(spec, m, 1, solver="gmres", gmres_max_iters=cap,
                                   cumulative_factor=cum)
    ost = O.corrected_coarse("erk", p, c, n, m, 1, "gmres", cap=cap, cumulative=cum)
    v = rng_rows(7, 12, n)
    ref = ost.apply(v)
    out = st.apply(v)
    # same Krylov depth per row; MGS dot order differs (oracle self-noise ~1e-14)
    assert np.max(np.abs(out - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_solve_gmres_result():
    n = 64
    D = P.high_derivative_operator(2, 2, "symmetric", n)
    op = P.CirculantOperator.identity(n) - D.scale(0.36)
    b = O.Circ(n, op.offsets, op.weights).apply(np.random.default_rng(1).standard_normal(n))
    res = op.solve_gmres(b, rel_tol=1e-2, max_iters=10)
    xr, rr, it, _ = O.gmres_rows(O.Circ(n, op.offsets, op.weights), b[None, :], 1e-2, 10)
    assert res.iterations == it and res.converged
    assert abs(res.relative_residual - rr[0]) <= 1e-12
    np.testing.assert_allclose(res.x, xr[0], atol=1e-12)
    z = op.solve_gmres(np.zeros(8 * 4), rel_tol=1e-2, max_iters=5) if False else None


# ------------------------------------------------------------- full solves

def _compare(rep, ref, hist_tol, iters_equal=True):
    assert rep.converged == ref["converged"]
    if iters_equal:
        assert rep.iterations == ref["iterations"]
    r0 = ref["norms"][0]
    dev = max(abs(a - b) / r0 for a, b in zip(rep.residual_norms, ref["norms"]))
    assert dev <= hist_tol, dev
    return dev


@pytest.mark.parametrize("n_x,n_t", [(1024, 1024), (256, 256)])
def test_cfg1_two_level_history(n_x, n_t):
    spec = P.DiscretizationSpec("erk", 1, 0.85, n_x, n_t)
    prob = P.experiments.build_problem(spec, 8, "two_level")
    steps, fac, u0 = O.build_hierarchy("erk", 1, 0.85, n_x, n_t, 8, "two_level")
    u = O.initial_iterate(0, n_t, n_x, u0)
    ref = O.Mgrit(steps, fac, n_t, u0).solve(u.copy())
    ug = u.copy()
    rep = P.solve(prob, P.MgritConfig(), initial_iterate=ug)
    _compare(rep, ref, 1e-12)
    assert np.max(np.abs(ug - ref["u"])) <= 1e-12 * np.max(np.abs(ref["u"]))


def test_sdirk3_vcycle_history_vs_staged_oracle():
    n_x, n_t = 256, 1024
    spec = P.DiscretizationSpec("sdirk", 3, 4.0, n_x, n_t)
    prob = P.experiments.build_problem(spec, 4, "v_cycle")
    steps, fac, u0 = O.build_hierarchy("sdirk", 3, 4.0, n_x, n_t, 4, "v_cycle",
                                       fine_mode="staged")
    ref = O.Mgrit(steps, fac, n_t, u0, cycle="v_cycle").solve()
    u = O.initial_iterate(0, n_t, n_x, u0)
    rep = P.solve(prob, P.MgritConfig(cycle="v_cycle"), initial_iterate=u)
    _compare(rep, ref, 1e-12)
    assert np.linalg.norm(u - ref["u"]) <= 1e-12 * np.linalg.norm(ref["u"])


def oracle_envelope(fam, p, c, n_x, n_t, m, cycle):
    """The oracle against itself with reordered GMRES reductions:
    returns (reference run, max |dr_k|/r0, ||du||/||u||)."""
    runs = {}
    for red in ("reference", "reordered"):
        steps, fac, u0 = O.build_hierarchy(fam, p, c, n_x, n_t, m, cycle, reduction=red)
        runs[red] = O.Mgrit(steps, fac, n_t, u0, cycle=cycle).solve()
    a, b = runs["reference"], runs["reordered"]
    r0 = a["norms"][0]
    dh = max(abs(x - y) / r0 for x, y in zip(a["norms"], b["norms"]))
    du = np.linalg.norm(a["u"] - b["u"]) / np.linalg.norm(a["u"])
    return a, dh, du


@pytest.mark.parametrize("p,cf,m,n_x,n_t", [(3, 0.85, 8, 256, 1024), (1, 0.85, 4, 256, 1024),
                                            (3, None, 8, 256, 1024), (5, None, 16, 256, 4096),
                                            (3, None, 8, 16384, 512)])
def test_erk_vcycle_gmres_history(p, cf, m, n_x, n_t):
    """GMRES-corrected V-cycles: identical iteration count; history and final
    iterate within 10x the oracle's self-noise envelope (floors 1e-13 / 1e-12)."""
    c = cf * O.cfl_max(p) if cf is not None else 0.85
    spec = P.DiscretizationSpec("erk", p, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, "v_cycle")
    saved = O.ROLL_LIMIT
    O.ROLL_LIMIT = 64 if p == 5 else 16
    try:
        ref, dh, du = oracle_envelope("erk", p, c, n_x, n_t, m, "v_cycle")
    finally:
        O.ROLL_LIMIT = saved
    u = O.initial_iterate(0, n_t, n_x, prob.u0)
    rep = P.solve(prob, P.MgritConfig(cycle="v_cycle"), initial_iterate=u)
    _compare(rep, ref, max(10 * dh, 1e-13))
    err_u = np.linalg.norm(u - ref["u"]) / np.linalg.norm(ref["u"])
    assert err_u <= max(10 * du, 1e-12), (err_u, du)


def test_ideal_coarse_one_iteration():
    spec = P.DiscretizationSpec("sdirk", 1, 0.8, 32, 64)
    fine = P.mol_stepper(spec)
    prob = P.TimeGridProblem([fine, P.ideal_coarse_stepper(fine, 8)], [8], 64,
                             P.initial_condition(32))
    for nu in (0, 1):
        rep = P.solve(prob, P.MgritConfig(nu=nu, max_iters=5, rng_seed=7))
        assert rep.converged and rep.iterations == 1


def test_sequential_solve_matches_oracle():
    spec = P.DiscretizationSpec("erk", 3, 0.85, 128, 64)
    prob = P.experiments.build_problem(spec, 4, "two_level")
    steps, fac, u0 = O.build_hierarchy("erk", 3, 0.85, 128, 64, 4, "two_level")
    assert np.array_equal(P.sequential_solve(prob), O.sequential(steps, fac, 64, u0))


# ------------------------------------------- BASELINE configs at full size

import json
import os

_FULL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full")
# name -> (config, n_x, n_t): the BASELINE configs and proxies that keep a
# config's level structure on a smaller grid (tests/golden/make_full.py)
_CASES = {"cfg1": ("cfg1", None, None), "cfg2": ("cfg2", None, None),
          "cfg3": ("cfg3", None, None), "cfg4": ("cfg4", None, None),
          "cfg4p": ("cfg4", 1024, 65536), "cfg5p": ("cfg5", 16384, 16384),
          "cfg5q": ("cfg5", 16384, 131072)}
# reduction-order self-noise of the reference measured on reduced grids (SURVEY
# 0.6 / 8c), used when a case has no full-size calibration run
_REDUCED_ENVELOPE = {3: 1.1e-11, 5: 2.9e-8}


def _load(name):
    path = os.path.join(_FULL, name + ".json")
    if not os.path.exists(path):
        return None, None
    return json.load(open(path)), np.load(os.path.join(_FULL, name + "_final.npz"))


def _final_dev(fa, fb):
    """(sampled rows: ||a - b|| / ||b|| over 17 evenly spaced rows; every row's
    l2 norm: max relative difference)."""
    ds = np.linalg.norm(fa["samples"] - fb["samples"]) / np.linalg.norm(fb["samples"])
    dn = np.max(np.abs(fa["row_norms"] - fb["row_norms"]) / np.maximum(fb["row_norms"], 1e-300))
    return float(ds), float(dn)


@pytest.mark.parametrize("name", sorted(_CASES))
def test_full_size_against_reference(name):
    """BASELINE workloads at full size (and proxies) against residual histories
    AND final iterates of the REAL reference (tests/golden/make_full.py; SDIRK
    with the staged fine stepper, ERK5 with rolled sums).  Direct-corrected
    configs: identical iterations, |dr_k| <= 1e-12 r_0, final iterate within
    1e-12.  GMRES-corrected configs: identical iterations, history and final
    iterate within 10x the reference's own reduction-order envelope (the
    oracle with reordered GMRES reductions at the same size when that run
    exists, else the reduced-grid figure)."""
    import torch
    from paper_2209_06916_b200.configs import CONFIGS
    ref, fref = _load(name)
    if ref is None:
        pytest.skip(f"no reference run for {name} (tests/golden/make_full.py {name})")
    base, n_x, n_t = _CASES[name]
    cf = CONFIGS[base]
    if cf.cycle == "f_cycle":
        cf = cf.as_v_cycle()  # the reference has no F-cycle
    if n_x:
        cf = cf.scaled(n_x, n_t)
    prob = cf.problem()
    sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
    u = torch.from_numpy(sol.initial_state()).cuda()
    rep = sol.solve(u)
    un = u.cpu().numpy()
    del u
    mine = {"samples": un[fref["rows"]], "row_norms": np.sqrt(np.einsum("ij,ij->i", un, un))}
    assert rep.iterations == ref["iterations"] and rep.converged == ref["converged"]
    r0 = ref["norms"][0]
    dev = max(abs(a - b) / r0 for a, b in zip(rep.residual_norms, ref["norms"]))
    ds, dn = _final_dev(mine, fref)
    gmres = cf.family == "erk" and cf.cycle != "two_level"
    if not gmres:
        assert dev <= 1e-12, dev
        assert ds <= 1e-12 and dn <= 1e-12, (ds, dn)
        return
    env, fenv = _load(name + "_reordered")
    if env is not None:
        assert env["iterations"] == ref["iterations"]
        tol_h = max(abs(a - b) / r0 for a, b in zip(env["norms"], ref["norms"]))
        tol_s, tol_n = _final_dev(fenv, fref)
    else:
        tol_h, tol_s, tol_n = _REDUCED_ENVELOPE[cf.p], 1e-11, 1e-11
    assert dev <= 10 * max(tol_h, 1e-13), (dev, tol_h)
    assert ds <= 10 * max(tol_s, 1e-12), (ds, tol_s)
    assert dn <= 10 * max(tol_n, 1e-12), (dn, tol_n)


@pytest.mark.parametrize("fam,p,c,n_x,n_t,m,cyc,nu,max_sharded", [
    ("erk", 3, 0.85, 256, 1024, 8, "v_cycle", 1, None),
    ("erk", 3, 0.85, 256, 1024, 8, "v_cycle", 1, 1),
    ("sdirk", 3, 4.0, 128, 1024, 4, "v_cycle", 1, None),
    ("erk", 3, 0.85, 128, 1024, 4, "f_cycle", 2, None),
    ("erk", 1, 0.85, 128, 256, 4, "two_level", 0, None)])
def test_time_sharded_engine_single_rank_matches_solver(fam, p, c, n_x, n_t, m, cyc, nu,
                                                        max_sharded):
    """The NCCL time-sharded driver (GpuEngine, every level sharded) on one rank
    reproduces the single-GPU solver bit for bit (multi-rank logic:
    tests/test_distributed_gloo.py)."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2209_06916_b200.distributed import GpuEngine, ShardedMgritSolver
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
        prob = P.experiments.build_problem(spec, m, "v_cycle" if cyc == "f_cycle" else cyc)
        cfg = P.MgritConfig(cycle=cyc, nu=nu)
        u = O.initial_iterate(0, n_t, n_x, prob.u0)
        ref_u = u.copy()
        ref = P.solve(prob, cfg, initial_iterate=ref_u)
        ud = torch.from_numpy(u).cuda()
        sol = ShardedMgritSolver(prob, cfg, GpuEngine(prob, cfg), max_sharded=max_sharded)
        rep = sol.solve(ud)
        assert sol.ls == (1 if (max_sharded == 1 or cyc == "two_level") else len(prob.m))
        assert rep.iterations == ref.iterations
        assert np.array_equal(ud.cpu().numpy(), ref_u)
        # the partials are reduced by the single-GPU fixed-order tree (mgb_sum)
        assert rep.residual_norms == ref.residual_norms
    finally:
        dist.destroy_process_group()


# ------------------------------------------------ host-iterate upload (solve)

@pytest.mark.parametrize("fam,p,c,n_x,n_t,m,cyc", [("erk", 3, 0.85, 256, 1024, 8, "v_cycle"),
                                                   ("erk", 1, 0.85, 128, 256, 4, "two_level"),
                                                   ("sdirk", 3, 4.0, 128, 256, 4, "v_cycle")])
def test_host_iterate_upload_of_live_rows_only(fam, p, c, n_x, n_t, m, cyc, monkeypatch):
    """solve(initial_iterate=<host>) copies only the C-points and the rows before
    them; the skipped rows are poisoned with NaN and the solve must still equal
    (bitwise) the solve of the same iterate given as a CUDA tensor, and write
    the full final iterate back in place (mgrit.py:288-291)."""
    import torch
    from paper_2209_06916_b200 import mgrit as M
    monkeypatch.setattr(M, "POISON_SKIPPED_ROWS", True)
    prob = P.experiments.build_problem(P.DiscretizationSpec(fam, p, c, n_x, n_t), m, cyc, "modified")
    cfg = P.MgritConfig(cycle=cyc)
    u0 = P.MgritSolver(prob, cfg).initial_state()
    dev = torch.from_numpy(u0.copy()).cuda()
    r_dev = P.solve(prob, cfg, initial_iterate=dev)
    host_np = u0.copy()
    r_np = P.solve(prob, cfg, initial_iterate=host_np)
    host_t = torch.from_numpy(u0.copy()).pin_memory()
    r_t = P.solve(prob, cfg, initial_iterate=host_t)
    for r in (r_np, r_t):
        assert r.residual_norms == r_dev.residual_norms and r.iterations == r_dev.iterations
    ref = dev.cpu().numpy()
    assert np.array_equal(host_np, ref) and np.array_equal(host_t.numpy(), ref)
    assert not np.isnan(ref).any()
    # default solve (internal iterate) gives the same history
    assert P.solve(prob, cfg).residual_norms == r_dev.residual_norms


@pytest.mark.parametrize("nu", [0, 2])
def test_pinned_upload_overlap_any_nu(nu, monkeypatch):
    """The pinned-host solve overlaps the upload of the rows before the
    C-points with the first cycle (the initial residual runs just before the
    first CF pass); for every relaxation count it equals the device-iterate
    solve bitwise, with the skipped rows poisoned."""
    import torch
    from paper_2209_06916_b200 import mgrit as M
    monkeypatch.setattr(M, "POISON_SKIPPED_ROWS", True)
    prob = P.experiments.build_problem(P.DiscretizationSpec("erk", 3, 0.85, 256, 1024), 8,
                                       "v_cycle", "modified")
    cfg = P.MgritConfig(cycle="v_cycle", nu=nu)
    u0 = P.MgritSolver(prob, cfg).initial_state()
    dev = torch.from_numpy(u0.copy()).cuda()
    r_dev = P.solve(prob, cfg, initial_iterate=dev)
    host_t = torch.from_numpy(u0.copy()).pin_memory()
    r_t = P.solve(prob, cfg, initial_iterate=host_t)
    assert r_t.residual_norms == r_dev.residual_norms and r_t.iterations == r_dev.iterations
    assert np.array_equal(host_t.numpy(), dev.cpu().numpy())


_SINGLE_CTA_CHECK = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O
worst = 0.0
for p, c, n, m, cum in [(1, 0.6, 1024, 4, 16), (3, 0.85, 1024, 8, 64), (5, 0.85, 1024, 16, 256),
                        (3, 0.85, 4096, 8, 64), (5, 0.85, 4096, 16, 256)]:
    cap = 10 if p == 1 else 20
    spec = P.DiscretizationSpec("erk", p, c, n, 64)
    st = P.modified_coarse_stepper(spec, m, 1, solver="gmres", gmres_max_iters=cap,
                                   cumulative_factor=cum)
    ost = O.corrected_coarse("erk", p, c, n, m, 1, "gmres", cap=cap, cumulative=cum)
    v = np.random.default_rng(7).random((12, n))
    ref, out = ost.apply(v), st.apply(v)
    err = np.max(np.abs(out - ref)) / np.max(np.abs(ref))
    assert err <= 1e-11, (p, n, err)
    worst = max(worst, err)
print("ok", worst)
"""


@pytest.mark.parametrize("extra_env", [{}, {"MGB_SLG_NO_OCC2": "1"}])
def test_single_cta_gmres_every_stencil_width(extra_env):
    """The single-CTA GMRES kernel (forced with MGB_NO_CLUSTER; the default
    picks it for levels with many intervals) against the oracle for operator
    half-widths 1, 2, 3 (p = 1, 3, 5) at 4 and 16 points per thread -- the
    register/shuffle stencil path -- in both occupancy builds."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MGB_NO_CLUSTER="1", **extra_env)
    r = subprocess.run([sys.executable, "-c", _SINGLE_CTA_CHECK.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


# ------------------------------------- opening F-relaxation of iterations >= 2

@pytest.mark.parametrize("fam,p,c,n_x,n_t,m,cyc,nu", [
    ("erk", 3, 0.85, 256, 1024, 8, "v_cycle", 1), ("erk", 1, 0.85, 128, 256, 4, "two_level", 0),
    ("erk", 3, 0.85, 128, 1024, 4, "f_cycle", 2), ("sdirk", 3, 4.0, 512, 256, 4, "v_cycle", 1),
    ("erk", 5, 0.85, 4096, 256, 16, "two_level", 1), ("sdirk", 3, 4.0, 256, 256, 4, "two_level", 0),
    # F-cycles: the V-cycle after each level's F-cycle also starts from relaxed F-points
    # (GMRES-corrected coarse levels on the single-CTA and cluster kernels)
    ("erk", 3, 0.85, 256, 4096, 4, "f_cycle", 1), ("erk", 3, 0.85, 4096, 512, 8, "f_cycle", 1),
    ("sdirk", 3, 4.0, 512, 1024, 4, "f_cycle", 1),
    # single-interval coarse levels (n_t a power of m) and a 16-interval cluster level
    ("erk", 3, 0.85, 256, 512, 8, "v_cycle", 1), ("erk", 5, 0.85, 8192, 4096, 16, "v_cycle", 1),
    ("erk", 3, 0.85, 128, 256, 4, "v_cycle", 2), ("sdirk", 3, 4.0, 512, 256, 4, "v_cycle", 2)])
def test_elided_opening_f_relaxation_is_bitwise_the_full_pass(fam, p, c, n_x, n_t, m, cyc, nu,
                                                              monkeypatch):
    """Iterations >= 2 of solve() read the F-points the previous closing
    F-relaxation left instead of recomputing them (mgrit.py:231 vs :247), and the
    FR / CF passes of a coarse level skip its first interval (zero C-point: a
    repeat of the FC pass): same iterate and history, bit for bit, as the
    reference-style full passes."""
    from paper_2209_06916_b200 import mgrit as M
    spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, "v_cycle" if cyc == "f_cycle" else cyc)
    cfg = P.MgritConfig(cycle=cyc, nu=nu, max_iters=6)
    u_a = P.MgritSolver(prob, cfg).initial_state()
    u_b = u_a.copy()
    rep_a = P.solve(prob, cfg, initial_iterate=u_a)
    monkeypatch.setattr(M, "ELIDE_OPENING_F_RELAX", False)
    monkeypatch.setattr(M, "ELIDE_FIRST_INTERVAL", False)
    monkeypatch.setattr(M, "REUSE_CLOSING_STEP", False)
    rep_b = P.solve(prob, cfg, initial_iterate=u_b)
    assert rep_a.iterations == rep_b.iterations >= 2
    if fam == "erk" and cyc != "two_level" and n_x >= 1024:
        # GMRES-corrected coarse levels on cluster kernels: the FR / CF passes of a level run
        # on one interval fewer, and the launch plan picks the cluster size from the interval
        # count (e.g. 15 instead of 15 + 1 intervals), so those passes may reduce in another
        # order: the same solve up to GMRES rounding amplified by the capped coarse solves
        # (bit for bit with one kernel variant: tests/test_gpu_variants.py)
        np.testing.assert_allclose(rep_a.residual_norms, rep_b.residual_norms, rtol=1e-3)
        assert np.max(np.abs(u_a - u_b)) <= 1e-6 * np.max(np.abs(u_b))
        return
    assert rep_a.residual_norms == rep_b.residual_norms
    assert np.array_equal(u_a, u_b)
