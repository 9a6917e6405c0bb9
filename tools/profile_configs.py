"""Per-pass GPU timing of the BASELINE configs (CUDA events per launch)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200.configs import CONFIGS

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4"]
for name in names:
    cf = CONFIGS[name]
    t0 = time.time()
    prob = cf.problem()
    cfg = P.MgritConfig(cycle=cf.cycle)
    sol = P.MgritSolver(prob, cfg)
    u_host = sol.initial_state()
    up = torch.from_numpy(u_host).cuda()
    u = up.clone()
    rep = sol.solve(u)  # warm
    u.copy_(up)
    torch.cuda.synchronize()
    rep = sol.solve(u)
    u.copy_(up)
    sol.profile = []
    rep2 = sol.solve(u)
    summ = sol.profile_summary()
    tot = sum(v[1] for v in summ.values())
    print(f"== {name}: iters {rep.iterations} conv {rep.converged} wall {rep.wall_time*1e3:.2f} ms "
          f"(profiled sum {tot:.2f} ms) setup+run {time.time()-t0:.1f}s levels {prob.m}")
    print("   norms:", " ".join(f"{x:.4e}" for x in rep.residual_norms))
    for k, (c, ms) in sorted(summ.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:10s} launches {c:4d}  total {ms:9.3f} ms  mean {ms/c*1e3:9.1f} us  share {ms/tot:6.1%}")
    del sol, u, up
    torch.cuda.empty_cache()
