"""Apply every level's stepper of a config to a few rows, one launch at a time,
and compare against the oracle (locates failing kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_06916_b200 as P
from paper_2209_06916_b200.configs import CONFIGS
from oracle import mgrit_oracle as O
name = sys.argv[1]
rows_list = [int(x) for x in sys.argv[2:]] or [1, 4, 16]
cf = CONFIGS[name]
prob = cf.problem()
steps, fac, _ = O.build_hierarchy(cf.family, cf.p, cf.c, cf.n_x, cf.n_t, cf.m, cf.cycle)
for l, (st, ost) in enumerate(zip(prob.steppers, steps)):
    for rows in rows_list:
        v = np.random.default_rng(l).random((rows, cf.n_x))
        out = st.apply(v)
        torch.cuda.synchronize()
        ref = ost.apply(v)
        err = np.max(np.abs(out - ref)) / np.max(np.abs(ref))
        print(f"level {l} {st.program.kind:10s} rows {rows:3d} rel err {err:.2e}", flush=True)
