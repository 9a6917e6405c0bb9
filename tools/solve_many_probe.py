"""Probe: sequential solve() vs solve_many() (streams 1/8, with/without CUDA graphs, L2 budget) on Table-3 ERK3 cells."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200 import experiments as E
c = 0.85 * P.cfl_limit(3)
for nx, nt in [(256, 1024), (1024, 4096)]:
    jobs = []
    for m in (2, 4, 8, 16):
        for cyc in ("two_level", "v_cycle"):
            spec = P.DiscretizationSpec("erk", 3, c, nx, nt)
            jobs.append((E.build_problem(spec, m, cyc, "modified"), P.MgritConfig(cycle=cyc, max_iters=40)))
    def seq():
        return [P.solve(pr, cf) for pr, cf in jobs]
    variants = {"seq": seq,
                "many_s1_nog": lambda: P.solve_many(jobs, streams=1, graphs=False),
                "many_s1_g": lambda: P.solve_many(jobs, streams=1, graphs=True),
                "many_s8_nog": lambda: P.solve_many(jobs, streams=8, graphs=False),
                "many_s8_g": lambda: P.solve_many(jobs, streams=8, graphs=True),
                "many_s8_g_bigL2": lambda: P.solve_many(jobs, streams=8, graphs=True, l2_budget=1e12)}
    for name, fn in variants.items():
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(nx, nt, name, f"{t*1e3:.1f} ms", sum(x.iterations for x in r), flush=True)
