"""Run one relax pass of a BASELINE config between cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures exactly that kernel.

    python tools/ncu_target.py cfg2 L0.CF      # fine correction + F-relax + norm pass
    python tools/ncu_target.py cfg2 L3.FC      # deepest GMRES level
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200.configs import CONFIGS

name, target = sys.argv[1], sys.argv[2]
cf = CONFIGS[name]
prob = cf.problem()
sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
u = torch.from_numpy(sol.initial_state()).cuda()
sol.solve(u.clone())  # warm: plans, workspaces
torch.cuda.synchronize()
# replay one cycle, capture only the target pass
orig = sol._timed
def timed(nm, fn, *a, **k):
    if nm == target and not getattr(sol, "_done", False):
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        sol._done = True
        return out
    return fn(*a, **k)
sol.profile = []
sol._timed = timed
sol._cycle(0, u.data_ptr(), None, False, True)
torch.cuda.synchronize()
print("captured", target, getattr(sol, "_done", False))
