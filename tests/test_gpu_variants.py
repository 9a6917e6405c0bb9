"""Kernel variants that must agree bit for bit: the dedicated SDIRK kernel
(relax_rkd_kernel) and the dedicated SL + direct-solve kernel (relax_sld_kernel)
against the generic kernels they replace (MGB_NO_RKD=1 / MGB_NO_SLD=1, read
once per process: the generic runs are subprocesses)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import json, sys, hashlib
import numpy as np
sys.path.insert(0, %r)
import paper_2209_06916_b200 as P
out = {}
for fam, p, c, n_x, n_t, m, cyc in %r:
    spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, cyc)
    cfg = P.MgritConfig(cycle=cyc, max_iters=8)
    u = P.MgritSolver(prob, cfg).initial_state()
    rep = P.solve(prob, cfg, initial_iterate=u)
    out[f"{fam}{p}_{n_x}x{n_t}_{cyc}"] = {"norms": rep.residual_norms,
                                           "sha": hashlib.sha256(u.tobytes()).hexdigest()}
print(json.dumps(out))
"""

CASES = [("sdirk", 3, 4.0, 512, 256, 4, "v_cycle"), ("sdirk", 3, 4.0, 4096, 64, 4, "two_level"),
         ("sdirk", 2, 2.0, 1024, 128, 4, "v_cycle"), ("sdirk", 1, 3.0, 512, 64, 2, "two_level"),
         # direct-corrected coarse operators: ERK two-level (cfg1's scheme), SDIRK V-cycles whose
         # deep levels have slow-decaying factors (hierarchical scan)
         ("erk", 1, 0.85, 1024, 256, 8, "two_level"), ("erk", 3, 0.85, 512, 128, 4, "two_level"),
         ("sdirk", 3, 4.0, 1024, 1024, 4, "v_cycle")]


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", _CHILD % (ROOT, CASES)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.gpu
def test_dedicated_kernels_bitwise_equal_generic_kernels():
    new = _run({})
    old = _run({"MGB_NO_RKD": "1", "MGB_NO_SLD": "1"})
    assert new.keys() == old.keys()
    for k in new:
        assert new[k]["norms"] == old[k]["norms"], k
        assert new[k]["sha"] == old[k]["sha"], k


_ELIDE_CHILD = r"""
import json, sys, hashlib
import numpy as np
sys.path.insert(0, %r)
import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import mgrit as M
out = {}
for fam, p, c, n_x, n_t, m, cyc, nu in %r:
    spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, "v_cycle" if cyc == "f_cycle" else cyc)
    cfg = P.MgritConfig(cycle=cyc, nu=nu, max_iters=5)
    u0 = P.MgritSolver(prob, cfg).initial_state()
    row = {}
    for name, flags in (("elided", (True, True)), ("full", (False, False))):
        M.ELIDE_OPENING_F_RELAX, M.ELIDE_FIRST_INTERVAL = flags
        M.REUSE_CLOSING_STEP = flags[0]
        u = u0.copy()
        rep = P.solve(prob, cfg, initial_iterate=u)
        row[name] = [rep.residual_norms, hashlib.sha256(u.tobytes()).hexdigest()]
    out[f"{fam}{p}_{n_x}x{n_t}_{cyc}_{nu}"] = row
print(json.dumps(out))
"""

ELIDE_CASES = [("erk", 3, 0.85, 4096, 512, 8, "f_cycle", 1), ("erk", 5, 0.85, 8192, 4096, 16, "v_cycle", 1),
               ("erk", 3, 0.85, 4096, 2048, 8, "v_cycle", 2), ("erk", 3, 0.85, 1024, 4096, 4, "f_cycle", 1)]


@pytest.mark.gpu
def test_elisions_are_bitwise_with_one_gmres_kernel_variant():
    """The recomputation the solve loop skips (opening F-relaxation of iterations
    >= 2, first interval of the coarse levels' FR / CF passes) leaves every bit
    unchanged when the GMRES kernel variant does not depend on the interval
    count (MGB_NO_CLUSTER=1: single-CTA GMRES on every level); in-process the
    launch plan may pick another cluster size for n - 1 intervals
    (tests/test_gpu_parity.py compares that case to GMRES rounding)."""
    env = dict(os.environ, MGB_NO_CLUSTER="1")
    r = subprocess.run([sys.executable, "-c", _ELIDE_CHILD % (ROOT, ELIDE_CASES)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert len(res) == len(ELIDE_CASES)
    for k, row in res.items():
        assert row["elided"] == row["full"], k
