"""GMRES depth statistics per coarse level of a config (one FC pass per level)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200.configs import CONFIGS
from paper_2209_06916_b200.device import plan_for, ptr
cf = CONFIGS[sys.argv[1]]
prob = cf.problem()
sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
u = torch.from_numpy(sol.initial_state()).cuda()
sol.solve(u.clone())
for l in range(1, len(prob.m)):
    L = sol.levels[l]
    nI = L.n_int
    d = torch.zeros(nI, dtype=torch.int32, device="cuda"); r = torch.zeros(nI, dtype=torch.float64, device="cuda")
    e = sol.ucoarse[l]; g = sol.gcoarse[l]
    hist = []
    # replay single steps: depth of the step-j solve for every interval
    for j in range(1, L.m):
        L.plan.relax(nI, L.m, j, c_src=ptr(e), c_stride=L.m * cf.n_x, g=ptr(g), stats_depth=ptr(d), stats_res=ptr(r))
        torch.cuda.synchronize()
        hist.append(d.cpu().numpy().copy())
    h = np.concatenate(hist)
    print(f"level {l}: intervals {nI}, depth mean {h.mean():.1f} max {h.max()} hist {np.bincount(h, minlength=21).tolist()}")
