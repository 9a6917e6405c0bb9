"""F-cycle convergence with / without the elisions: python tools/fcycle_check.py n_x n_t"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import mgrit as M
from paper_2209_06916_b200.configs import CONFIGS
n_x, n_t = int(sys.argv[1]), int(sys.argv[2])
cf = CONFIGS["cfg5"].scaled(n_x, n_t)
prob = cf.problem()
for cyc in ("f_cycle", "v_cycle"):
    for flags in ((True, True), (False, False)):
        M.ELIDE_OPENING_F_RELAX, M.ELIDE_FIRST_INTERVAL = flags
        sol = P.MgritSolver(prob, P.MgritConfig(cycle=cyc, max_iters=20))
        u = torch.from_numpy(sol.initial_state()).cuda()
        rep = sol.solve(u)
        print(cyc, flags, rep.iterations, rep.converged, " ".join(f"{x:.3e}" for x in rep.residual_norms[:8]), "...", f"{rep.residual_norms[-1]:.3e}", flush=True)
        del u, sol
        torch.cuda.empty_cache()
