"""Repeat cluster-GMRES applies against the oracle to expose intermittent races.
    python tools/race_check.py N [n cum rows]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O
reps = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cum = int(sys.argv[3]) if len(sys.argv) > 3 else 64; rows = int(sys.argv[4]) if len(sys.argv) > 4 else 12
spec = P.DiscretizationSpec("erk", 3, 0.85, n, 64)
st = P.modified_coarse_stepper(spec, 8, 1, solver="gmres", gmres_max_iters=20, cumulative_factor=cum)
ost = O.corrected_coarse("erk", 3, 0.85, n, 8, 1, "gmres", cap=20, cumulative=cum)
v = np.random.default_rng(7).standard_normal((rows, n))
ref = ost.apply(v)
bad = 0
first = st.apply(v)
fresh = os.environ.get("FRESH") is not None
for r in range(reps):
    if fresh:
        st = P.modified_coarse_stepper(spec, 8, 1, solver="gmres", gmres_max_iters=20, cumulative_factor=cum)
    out = st.apply(v)
    dev = np.max(np.abs(out - ref)) / np.max(np.abs(ref))
    same = np.array_equal(out, first)
    if dev > 1e-11 or not same:
        bad += 1
        rowdev = np.max(np.abs(out - ref), axis=1) / np.max(np.abs(ref))
        print(f"rep {r}: dev {dev:.3e} bitwise-same-as-first {same} bad rows {np.nonzero(rowdev > 1e-11)[0].tolist()}", flush=True)
print(f"{bad} / {reps} bad")
