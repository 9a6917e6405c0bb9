"""SDIRK3 fine-operator realisation vs the reference's staged FFT stepper
(stepping.py:355-380): per-mode gain difference of one step on the GPU and
the cfg3 final-iterate deviation from the reference's full-size run.

    python tools/sdirk_drift.py [solve]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2209_06916_b200 as P  # noqa: E402
from oracle import mgrit_oracle as O  # noqa: E402

n = 4096
spec = P.DiscretizationSpec("sdirk", 3, 4.0, n, 16384)
st = P.mol_stepper(spec, mode="staged")
ost = O.mol_step("sdirk", 3, 4.0, n, mode="staged")
x = -1.0 + 2.0 * np.arange(n) / n
rows = [np.ones(n)] + [np.sin(np.pi * k * x + 0.3 * k) for k in range(1, 9)]
V = np.stack(rows)
g, o = st.apply(V), ost.apply(V)
out = {"mode_gain_dev": []}
for k in range(V.shape[0]):
    # complex gain of mode k from the DFT of input and output
    kk = k
    fi, fg, fo = np.fft.rfft(V[k])[kk], np.fft.rfft(g[k])[kk], np.fft.rfft(o[k])[kk]
    out["mode_gain_dev"].append([kk, float(abs(fg / fi - fo / fi)), float(abs(fo / fi))])
out["max_abs_row_dev"] = float(np.max(np.abs(g - o)))
if len(sys.argv) > 1 and sys.argv[1] == "solve":
    import torch
    from paper_2209_06916_b200.configs import CONFIGS
    cf = CONFIGS["cfg3"]
    prob = cf.problem()
    sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
    u = torch.from_numpy(sol.initial_state()).cuda()
    rep = sol.solve(u)
    un = u.cpu().numpy()
    fr = np.load(os.path.join(ROOT, "tests", "golden", "full", "cfg3_final.npz"))
    smp = un[fr["rows"]]
    out["final_rows_rel"] = float(np.linalg.norm(smp - fr["samples"]) / np.linalg.norm(fr["samples"]))
    out["final_rows_rel_by_row"] = (np.linalg.norm(smp - fr["samples"], axis=1)
                                    / np.linalg.norm(fr["samples"], axis=1)).tolist()
    out["iterations"] = rep.iterations
print(json.dumps(out))
