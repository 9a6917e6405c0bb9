"""Full-size self-noise envelope of a GMRES-corrected BASELINE config:
run the oracle with REORDERED GMRES reductions (blocked, reversed dot products;
mgrit_oracle.gmres_rows(reduction="reordered")) and compare its residual
history with the real reference's (tests/golden/histories.json, made by
tests/golden/make_golden.py --full; the default-order oracle is pinned bit for
bit to the reference).  Writes tests/golden/envelopes.json.  CPU only, hours
for cfg4:  python tools/oracle_envelope_full.py cfg4"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import mgrit_oracle as O  # noqa: E402
from paper_2209_06916_b200.configs import CONFIGS, seeded_u0  # noqa: E402

name = sys.argv[1]
cf = CONFIGS[name]
O.ROLL_LIMIT = 64 if cf.p == 5 else 16
steps, fac, _ = O.build_hierarchy(cf.family, cf.p, cf.c, cf.n_x, cf.n_t, cf.m, cf.cycle, cf.coarse,
                                  fine_mode="staged" if cf.family == "sdirk" else "assembled",
                                  reduction="reordered")
t0 = time.perf_counter()
out = O.Mgrit(steps, fac, cf.n_t, seeded_u0(cf.u0, cf.n_x), cycle=cf.cycle).solve()
wall = time.perf_counter() - t0
ref = json.load(open(os.path.join(ROOT, "tests", "golden", "histories.json")))[name]
r0 = ref["norms"][0]
dev = max(abs(a - b) / r0 for a, b in zip(out["norms"], ref["norms"]))
path = os.path.join(ROOT, "tests", "golden", "envelopes.json")
env = json.load(open(path)) if os.path.exists(path) else {}
env[name] = {"iterations_reordered": out["iterations"], "iterations_reference": ref["iterations"],
             "max_abs_dev_over_r0": dev, "norms_reordered": out["norms"], "wall_s": wall}
json.dump(env, open(path, "w"), indent=0)
print(name, out["iterations"], ref["iterations"], f"{dev:.3e}", f"{wall:.0f}s")
