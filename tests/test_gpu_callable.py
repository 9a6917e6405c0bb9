"""Stepper(apply_fn=<callable>) (reference stepping.py:276-295) on the device
path: the MGRIT passes run on the GPU around the user's one-step callable."""
import numpy as np
import pytest

import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import stepping


def _roll_callable(op):
    """out = sum_k w_k roll(u, -o_k) in the reference's tap order with torch
    (rounded product, then rounded sum: the rolled-sum arithmetic)."""
    import torch
    offs = [int(o) for o in op.offsets]
    wts = [float(w) for w in op.weights]

    def fn(u):
        out = torch.zeros_like(u)
        for o, w in zip(offs, wts):
            out += w * torch.roll(u, -o, dims=-1)
        return out
    return fn


def _with_callables(prob, wrap):
    steps = [stepping.Stepper(s.n_x, s.op, s.symbol, mode=s.mode, level=s.level,
                              dt_multiplier=s.dt_multiplier, apply_fn=wrap(s.op),
                              description="user callable") for s in prob.steppers]
    return P.TimeGridProblem(steps, prob.m, prob.n_t, prob.u0)


def test_callable_program_is_built_without_gpu():
    spec = P.DiscretizationSpec("erk", 1, 0.85, 64, 64)
    st = P.mol_stepper(spec)
    user = stepping.Stepper(64, st.op, st.symbol, apply_fn=lambda u: u)
    assert user.program.kind == "callable" and user.program.fn is not None
    assert user.program.repeated(3).repeat == 3
    assert callable(stepping.host_callable(lambda a: a))


@pytest.mark.gpu
@pytest.mark.parametrize("cycle,nu", [("two_level", 1), ("v_cycle", 1), ("v_cycle", 0), ("f_cycle", 2)])
def test_user_callable_steppers_match_stencil_kernels_bitwise(cycle, nu):
    """Plain-SL hierarchy (every level an explicit stencil): torch callables with
    the rolled-sum arithmetic give the kernels' residual history and iterate
    bit for bit."""
    spec = P.DiscretizationSpec("erk", 3, 0.85, 128, 256)
    base = P.experiments.build_problem(spec, 4, "v_cycle" if cycle == "f_cycle" else cycle, "plain_sl")
    cfg = P.MgritConfig(cycle=cycle, nu=nu, max_iters=6)
    ref_u = P.MgritSolver(base, cfg).initial_state()
    usr_u = ref_u.copy()
    ref = P.solve(base, cfg, initial_iterate=ref_u)
    usr = P.solve(_with_callables(base, _roll_callable), cfg, initial_iterate=usr_u)
    assert usr.iterations == ref.iterations
    assert np.array_equal(usr_u, ref_u)
    # per-interval partials are summed by torch instead of the kernel's fixed tree
    np.testing.assert_allclose(usr.residual_norms, ref.residual_norms, rtol=1e-13)


@pytest.mark.gpu
def test_host_callable_round_trip_and_primitives():
    """A numpy-only callable (the reference's contract) through host_callable;
    f_relax / c_relax / restriction / norm and Stepper.apply against the kernels."""
    spec = P.DiscretizationSpec("erk", 3, 0.85, 128, 64)
    st = P.mol_stepper(spec)

    def numpy_step(a):
        out = np.zeros_like(a)
        for o, w in zip(st.op.offsets, st.op.weights):
            out += w * np.roll(a, -int(o), axis=-1)
        return out

    user = stepping.Stepper(128, st.op, st.symbol, apply_fn=stepping.host_callable(numpy_step))
    rng = np.random.default_rng(5)
    u = rng.random((65, 128))
    g = rng.random((65, 128))
    assert np.array_equal(user.apply(u[:7]), st.apply(u[:7]))
    ua, ub = u.copy(), u.copy()
    P.f_relax(ua, g, user, 4)
    P.f_relax(ub, g, st, 4)
    assert np.array_equal(ua, ub)
    P.c_relax(ua, g, user, 4)
    P.c_relax(ub, g, st, 4)
    assert np.array_equal(ua, ub)
    assert np.array_equal(P.restrict_residual(ua, g, user, 4), P.restrict_residual(ub, g, st, 4))
    assert P.cpoint_residual_norm(ua, g, user, 4) == pytest.approx(
        P.cpoint_residual_norm(ub, g, st, 4), rel=1e-13)
