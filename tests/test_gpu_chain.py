"""The contiguous interval blocks of the fine explicit kernel (relax_win_kernel:
each CTA walks a block of intervals and, in FR / CF passes, hands the next
interval's start row over from the residual tail) with MANY intervals per CTA:
the grid is capped (MGB_MAX_GRID, a test knob) so every CTA chains several
intervals.  Everything is a rolled-sum stencil (ERK fine + uncorrected SL
coarse operators), so the GPU must equal the oracle BIT FOR BIT for nu = 0, 1,
2, and a pass split into two launches (the second with k_global0 > 0, as on a
time-sharded rank) must equal the single launch bit for bit."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O
from paper_2209_06916_b200.device import plan_for, ptr

# 1) whole solves, every nu
for nu in (0, 1, 2):
    for p, c, nx, nt, m, cyc in [(3, 0.5, 256, 4096, 4, "v_cycle"), (1, 0.85, 256, 2048, 8, "two_level")]:
        prob = P.experiments.build_problem(P.DiscretizationSpec("erk", p, c, nx, nt), m, cyc, "plain_sl")
        steps, fac, u0 = O.build_hierarchy("erk", p, c, nx, nt, m, cyc, kind="plain_sl")
        u = O.initial_iterate(0, nt, nx, u0)
        rep = P.solve(prob, P.MgritConfig(nu=nu, cycle=cyc, max_iters=4), initial_iterate=u)
        orc = O.Mgrit(steps, fac, nt, u0, nu=nu, cycle=cyc, max_iters=4).solve()
        assert rep.iterations == orc["iterations"], (nu, p)
        assert np.array_equal(u, orc["u"]), (nu, p, float(np.max(np.abs(u - orc["u"]))))

# 2) a pass split over two launches (second with k_global0 > 0) == one launch
nx, m, nI = 256, 4, 512
st = P.mol_stepper(P.DiscretizationSpec("erk", 3, 0.85, nx, nI * m))
plan = plan_for(st.program)
rng = np.random.default_rng(4)
u = torch.from_numpy(rng.random((nI * m + 1, nx))).cuda()
cb = torch.from_numpy(rng.random((nI + 1, nx))).cuda()
e = torch.from_numpy(rng.random((nI + 1, nx))).cuda()
g = torch.from_numpy(rng.random((nI * m + 1, nx))).cuda()
row = nx * 8
def run(k0, nb, outs):
    uu, tail, part = outs
    off = k0 * row
    # FR pass (chained: cref = c_src + stride)
    plan.relax(nb, m, m - 1, k_global0=k0, c_src=ptr(cb) + off, c_stride=nx, c_src0=ptr(u),
               tail=2, cref=ptr(cb) + off + row, cref_stride=nx, tail_out=ptr(tail) + off + row,
               tail_stride=nx, g=ptr(g) + k0 * m * row, partials=ptr(part) + k0 * 8)
    # CF pass (chained with the correction: cref_e = e + stride)
    plan.relax(nb, m, m - 1, k_global0=k0, c_src=ptr(cb) + off, c_stride=nx, c_src0=ptr(u),
               e=ptr(e) + off, e_stride=nx, c_out=ptr(uu) + k0 * m * row, c_out_stride=m * nx,
               c_last_out=ptr(uu) + (k0 + nb) * m * row, u=ptr(uu) + k0 * m * row, write_f=2,
               g=ptr(g) + k0 * m * row, tail=2, cref=ptr(cb) + off + row, cref_stride=nx,
               cref_e=ptr(e) + off + row, cref_e_stride=nx, partials=ptr(part) + nI * 8 + k0 * 8)
def fresh():
    return (u.clone(), torch.zeros((nI + 1, nx), dtype=torch.float64, device="cuda"),
            torch.zeros(2 * nI, dtype=torch.float64, device="cuda"))
one, two = fresh(), fresh()
run(0, nI, one)
run(0, 200, two)
run(200, nI - 200, two)
torch.cuda.synchronize()
for a, b in zip(one, two):
    assert torch.equal(a, b)
print("ok")
"""


@pytest.mark.parametrize("cap", ["7", "64", ""])
def test_chained_interval_blocks_bitwise(cap):
    env = dict(os.environ)
    if cap:
        env["MGB_MAX_GRID"] = cap
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]
