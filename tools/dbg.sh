cd $GRAFT_REPO_ROOT
for args in "3 0.85 256 8 8" "3 0.85 4096 8 64" "5 0.85 1024 16 256" "1 0.6 64 4 16"; do
  timeout 40 python - $args <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O
p, c, n, m, cum = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
spec = P.DiscretizationSpec("erk", p, c, n, 64)
cap = 10 if p == 1 else 20
st = P.modified_coarse_stepper(spec, m, 1, solver="gmres", gmres_max_iters=cap, cumulative_factor=cum)
ost = O.corrected_coarse("erk", p, c, n, m, 1, "gmres", cap=cap, cumulative=cum)
for rows in (1, 2, 12):
    v = np.random.default_rng(7).random((rows, n))
    out = st.apply(v); ref = ost.apply(v)
    print(sys.argv[1:], rows, np.max(np.abs(out - ref)) / np.max(np.abs(ref)), flush=True)
PY
  echo "rc=$?"
done
