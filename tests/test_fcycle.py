"""F-cycle (extension: BASELINE cfg5 names an F-cycle; the reference has only
two_level | v_cycle, mgrit.py:41-42, so parity is against the oracle's own
F-cycle restatement, which is unpinned by the reference).

CPU: the oracle F-cycle equals the V-cycle on two-level hierarchies and
converges at least as fast on deep ones.  GPU: the device F-cycle matches the
oracle F-cycle (direct-corrected: 1e-12 r0; GMRES-corrected: 10x the oracle's
reduction-order envelope) and equals the device V-cycle on two-level grids."""

import numpy as np
import pytest

from oracle import mgrit_oracle as O


def _oracle(fam, p, c, n_x, n_t, m, cycle, reduction="reference", fine_mode="assembled"):
    steps, fac, u0 = O.build_hierarchy(fam, p, c, n_x, n_t, m, cycle, reduction=reduction,
                                       fine_mode=fine_mode)
    return O.Mgrit(steps, fac, n_t, u0, cycle=cycle).solve()


def test_oracle_fcycle_equals_vcycle_two_level():
    a = _oracle("erk", 3, 0.85, 32, 8, 8, "v_cycle")
    b = _oracle("erk", 3, 0.85, 32, 8, 8, "f_cycle")
    assert a["norms"] == b["norms"] and np.array_equal(a["u"], b["u"])


@pytest.mark.parametrize("fam,p,c,m", [("erk", 3, 0.85, 4), ("sdirk", 3, 4.0, 4)])
def test_oracle_fcycle_converges_no_slower(fam, p, c, m):
    v = _oracle(fam, p, c, 32, 256, m, "v_cycle")
    f = _oracle(fam, p, c, 32, 256, m, "f_cycle")
    assert f["converged"] and f["iterations"] <= v["iterations"]


@pytest.mark.gpu
def test_gpu_fcycle_sdirk_direct_vs_oracle():
    import paper_2209_06916_b200 as P
    n_x, n_t = 128, 1024
    spec = P.DiscretizationSpec("sdirk", 3, 4.0, n_x, n_t)
    prob = P.experiments.build_problem(spec, 4, "f_cycle")
    ref = _oracle("sdirk", 3, 4.0, n_x, n_t, 4, "f_cycle", fine_mode="staged")
    rep = P.solve(prob, P.MgritConfig(cycle="f_cycle"))
    assert rep.iterations == ref["iterations"] and rep.converged == ref["converged"]
    r0 = ref["norms"][0]
    assert max(abs(a - b) / r0 for a, b in zip(rep.residual_norms, ref["norms"])) <= 1e-12


@pytest.mark.gpu
def test_gpu_fcycle_erk_gmres_vs_oracle_envelope():
    import paper_2209_06916_b200 as P
    n_x, n_t, m = 256, 1024, 8
    c = 0.85 * O.cfl_max(3)
    spec = P.DiscretizationSpec("erk", 3, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, "f_cycle")
    a = _oracle("erk", 3, c, n_x, n_t, m, "f_cycle")
    b = _oracle("erk", 3, c, n_x, n_t, m, "f_cycle", reduction="reordered")
    r0 = a["norms"][0]
    env = max(abs(x - y) / r0 for x, y in zip(a["norms"], b["norms"]))
    u = O.initial_iterate(0, n_t, n_x, prob.u0)
    rep = P.solve(prob, P.MgritConfig(cycle="f_cycle"), initial_iterate=u)
    assert rep.iterations == a["iterations"] and rep.converged
    dev = max(abs(x - y) / r0 for x, y in zip(rep.residual_norms, a["norms"]))
    assert dev <= max(10 * env, 1e-13), (dev, env)


@pytest.mark.gpu
def test_gpu_fcycle_equals_vcycle_two_level():
    import paper_2209_06916_b200 as P
    spec = P.DiscretizationSpec("erk", 3, 0.85, 128, 8)
    prob_v = P.experiments.build_problem(spec, 8, "v_cycle")
    prob_f = P.experiments.build_problem(spec, 8, "f_cycle")
    rv = P.solve(prob_v, P.MgritConfig(cycle="v_cycle", max_iters=5))
    rf = P.solve(prob_f, P.MgritConfig(cycle="f_cycle", max_iters=5))
    assert rv.residual_norms == rf.residual_norms
