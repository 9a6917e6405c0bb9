"""Run-to-run repeatability of the round-2 kernels (a race shows up as a changed
bit): every case is solved REPS times from the same iterate and hashed.

    python tools/repeat_check.py [REPS]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_06916_b200 as P  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 20
CASES = [("erk", 3, 0.85, 4096, 512, 8, "v_cycle"), ("erk", 5, 0.85, 8192, 512, 16, "v_cycle"),
         ("sdirk", 3, 4.0, 4096, 256, 4, "v_cycle"), ("erk", 1, 0.85, 1024, 1024, 8, "two_level"),
         ("sdirk", 3, 4.0, 512, 1024, 4, "f_cycle"), ("erk", 3, 0.85, 16384, 256, 8, "v_cycle")]
bad = 0
for fam, p, c, n_x, n_t, m, cyc in CASES:
    spec = P.DiscretizationSpec(fam, p, c, n_x, n_t)
    prob = P.experiments.build_problem(spec, m, "v_cycle" if cyc == "f_cycle" else cyc)
    cfg = P.MgritConfig(cycle=cyc, max_iters=4)
    u0 = P.MgritSolver(prob, cfg).initial_state()
    seen = set()
    for _ in range(REPS):
        u = u0.copy()
        rep = P.solve(prob, cfg, initial_iterate=u)
        seen.add((hashlib.sha256(u.tobytes()).hexdigest(), tuple(rep.residual_norms)))
    print(fam, p, n_x, n_t, cyc, "distinct results:", len(seen), flush=True)
    bad += len(seen) != 1
print("REPEATABLE" if bad == 0 else f"{bad} cases changed between runs")
sys.exit(1 if bad else 0)
