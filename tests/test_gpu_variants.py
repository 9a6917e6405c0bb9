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
