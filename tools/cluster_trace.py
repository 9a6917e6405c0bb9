"""Phase breakdown of the cluster GMRES kernel (needs `make trace`, MGB_TRACE=1)."""
import ctypes, os, sys
os.environ["MGB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import _native
from paper_2209_06916_b200.configs import CONFIGS
cf = CONFIGS[sys.argv[1]]; target = sys.argv[2]
prob = cf.problem()
sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
u = torch.from_numpy(sol.initial_state()).cuda()
sol.solve(u.clone())
lib = _native.load()
buf = (ctypes.c_ulonglong * 16)()
mode = sys.argv[3] if len(sys.argv) > 3 else "cluster"
single = mode == "single"
fetch = {"single": lib.mgb_trace_fetch_gen if hasattr(lib, "mgb_trace_fetch_gen") else None,
         "rk": getattr(lib, "mgb_trace_fetch_rk", None),
         "c1": getattr(lib, "mgb_trace_fetch_c1", None)}.get(mode, lib.mgb_trace_fetch)
fetch(buf)
orig = sol._timed
def timed(nm, fn, *a, **k):
    out = fn(*a, **k)
    if nm == target:
        torch.cuda.synchronize(); fetch(buf)
        if mode == "rk":
            names = ["", "row write+syncs", "L stencil", "", "factor local pass", "sync1",
                     "warp-0 carry scan", "sync2", "carry fix-up", "", "", "", "", "", "", ""]
        elif single:
            names = ["beta", "op2 stencil", "vi load+dot", "block_sum", "axpy+norm dot", "norm sum",
                     "V store+givens", "sync", "backsub+x", "row write+syncs", "", "", "", "", "", ""]
        elif mode == "c1":
            names = ["wait bar2", "v_j", "Z_j", "u'", "Au'+dots", "syncthreads", "exchange",
                     "backsub+x", "SL+b dots", "b exchange", "S:total+coef", "S:norm,sqrt,div",
                     "wait bar1", "reorth pass", "", ""]
        else:
          names = ["beta+halo", "passA1", "passB1", "upd1+pub+pd2", "sum2", "corr+upd2+hn",
                 "V/Z+givens", "backsub+x", "SL apply", "row+barrier", "", "", "", "", "gmres total", "steps"]
        steps = buf[15]
        tot = sum(buf[i] for i in range(10))
        print(f"{nm}: arnoldi steps {steps}")
        for i in range(16):
            if buf[i] and i != 15:
                print(f"  {names[i]:14s} {buf[i]/1e3:10.1f} kcyc  per step {buf[i]/max(steps,1):8.0f}")
    return out
sol.profile = []
sol._timed = timed
sol._cycle(0, u.data_ptr(), None, False, True)
torch.cuda.synchronize()
