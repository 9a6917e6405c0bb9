"""Run one solve of a BASELINE config with the CUDA profiler enabled only around
the first launch of one pass (for `ncu --profile-from-start off -c 1`).

    python tools/ncu_target.py cfg2 L0.CF
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2209_06916_b200 as P  # noqa: E402
from paper_2209_06916_b200.configs import CONFIGS  # noqa: E402

cf = CONFIGS[sys.argv[1]]
target = sys.argv[2]
prob = cf.problem()
sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle, tol=1e-10, max_iters=30))
u0 = torch.from_numpy(sol.initial_state()).cuda()
sol.solve(u0.clone())  # warm-up: plans, workspaces, module load
torch.cuda.synchronize()
orig = sol._timed
done = [False]


def timed(name, fn, *a, **k):
    if name == target and not done[0]:
        done[0] = True
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return out
    return fn(*a, **k)


sol._timed = timed
rep = sol.solve(u0.clone())
torch.cuda.synchronize()
print(f"{cf.name} {target}: profiled={done[0]} iterations={rep.iterations}")
if not done[0]:
    sys.exit(1)
