"""Elision A/B on one case: python tools/elide_diag.py fam p c n_x n_t m cycle nu"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import mgrit as M
fam, p, c, n_x, n_t, m, cyc, nu = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6]), sys.argv[7], int(sys.argv[8])
spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
prob = P.experiments.build_problem(spec, m, "v_cycle" if cyc == "f_cycle" else cyc)
cfg = P.MgritConfig(cycle=cyc, nu=nu, max_iters=6)
u0 = P.MgritSolver(prob, cfg).initial_state()
res = {}
for name, (a, b) in {"both": (True, True), "open_only": (True, False), "first_only": (False, True), "none": (False, False)}.items():
    M.ELIDE_OPENING_F_RELAX, M.ELIDE_FIRST_INTERVAL, M.REUSE_CLOSING_STEP = a, b, a
    u = u0.copy()
    rep = P.solve(prob, cfg, initial_iterate=u)
    res[name] = (np.array(rep.residual_norms), u)
ref = res["none"]
for k, (nrm, u) in res.items():
    print(k, "norm rel diff %.3e" % np.max(np.abs(nrm - ref[0]) / ref[0]), "iterate rel diff %.3e" % (np.max(np.abs(u - ref[1])) / np.max(np.abs(ref[1]))), "bitwise", np.array_equal(u, ref[1]))
