"""Concurrent small solves (Table-3 / measured-point sweeps,
experiments.py:150-242): ``solve_many`` runs each solve's exact kernel
sequence on its own stream, so reports and iterates must be bitwise equal to
the sequential solves; the concurrent Table 3 must reproduce the reference's
exact counts (tests/golden/histories.json, made by the real reference)."""

import json
import os

import numpy as np
import pytest

import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import experiments as E

HERE = os.path.dirname(os.path.abspath(__file__))
HIST = json.load(open(os.path.join(HERE, "golden", "histories.json")))


def test_solve_many_empty():
    assert P.solve_many([]) == []


def _jobs():
    out = []
    for fam, p, c, nx, nt, m, cyc in [("erk", 1, 0.85, 128, 256, 8, "two_level"),
                                      ("erk", 3, 0.85, 64, 256, 4, "v_cycle"),
                                      ("sdirk", 3, 4.0, 96, 256, 4, "v_cycle"),
                                      ("erk", 3, 1.0, 256, 512, 8, "v_cycle"),
                                      ("erk", 1, 0.5, 64, 128, 2, "two_level")]:
        spec = P.DiscretizationSpec(fam, p, c, nx, nt)
        out.append((E.build_problem(spec, m, cyc, "modified"), P.MgritConfig(cycle=cyc)))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("streams", [None, 2])
def test_solve_many_bitwise_equals_sequential(streams):
    jobs = _jobs()
    seq_u = [np.random.default_rng(7 + i).random((pr.n_t + 1, pr.n_x)) for i, (pr, _) in enumerate(jobs)]
    for u, (pr, _) in zip(seq_u, jobs):
        u[0] = pr.u0
    par_u = [u.copy() for u in seq_u]
    seq = [P.solve(pr, cfg, initial_iterate=u) for (pr, cfg), u in zip(jobs, seq_u)]
    par = P.solve_many([(pr, cfg, u) for (pr, cfg), u in zip(jobs, par_u)], streams=streams)
    for a, b, ua, ub in zip(seq, par, seq_u, par_u):
        assert a.residual_norms == b.residual_norms
        assert (a.iterations, a.converged) == (b.iterations, b.converged)
        assert np.array_equal(ua, ub)


@pytest.mark.gpu
@pytest.mark.parametrize("fam", ["erk", "sdirk"])
def test_table3_concurrent_matches_reference_counts(fam):
    c = 0.85 * P.cfl_limit(3) if fam == "erk" else 5.0
    cells = E.iteration_table(fam, 3, c, [(64, 256)], [2, 4, 8, 16], max_iters=40,
                              concurrent=True)
    for cell in cells:
        for cyc, got in (("two_level", cell.report_two_level), ("v_cycle", cell.report_v_cycle)):
            ref = HIST[f"table3_{fam}_64x256_m{cell.m}_{cyc}"]
            assert got.iterations == ref["iterations"], (cell.m, cyc)
            assert got.converged == ref["converged"]


@pytest.mark.gpu
def test_measured_points_equal_measured_point():
    cs = [0.3, 0.6, 0.85]
    many = E.measured_points("erk", 3, "modified", cs, 4, 64, 256, cycle="v_cycle")
    for c, r in zip(cs, many):
        one = E.measured_point("erk", 3, "modified", c, 4, 64, 256, cycle="v_cycle")
        assert one.residual_norms == r.residual_norms and one.iterations == r.iterations
