"""Small solves that exercise the round-2 kernels (fixed-geometry explicit kernel,
dedicated SDIRK kernel, SL + direct-solve kernel) for compute-sanitizer:

    compute-sanitizer --tool racecheck python tools/sanitize_new_kernels.py
    compute-sanitizer --tool memcheck  python tools/sanitize_new_kernels.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_06916_b200 as P  # noqa: E402

CASES = [("erk", 3, 0.85, 4096, 32, 8, "two_level"),     # relax_win_kernel 16 x 256 + SLD coarse
         ("erk", 5, 0.85, 8192, 32, 16, "two_level"),    # relax_win_kernel 16 x 512, 31 taps
         ("sdirk", 3, 4.0, 512, 64, 4, "v_cycle"),       # relax_rkd_kernel + SLD (windowed + scan)
         ("erk", 1, 0.85, 1024, 64, 8, "two_level")]     # SLD sequential coarse solve
for fam, p, c, n_x, n_t, m, cyc in CASES:
    spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, cyc)
    rep = P.solve(prob, P.MgritConfig(cycle=cyc, max_iters=2))
    print(fam, p, n_x, n_t, cyc, rep.iterations, f"{rep.residual_norms[-1] / rep.residual_norms[0]:.3e}", flush=True)
