"""GPU tests of the one-reduction cluster GMRES (csrc/mgb_cluster1.cuh) against
the oracle's restatement of circulant.py:262-332 (MGS GMRES): edge cases of the
stop rule and every launch variant (cluster sizes, occupancy builds, the
legacy two-reduction kernel).  Variants are forced through the library's
environment switches in a subprocess (they are read once per process)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2209_06916_b200 as P  # noqa: E402
from oracle import mgrit_oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rows(n, seed=11):
    rng = np.random.default_rng(seed)
    x = -1.0 + 2.0 * np.arange(n) / n
    return np.stack([
        np.zeros(n),                              # zero right-hand side: x = 0, depth 0
        np.full(n, 0.75),                         # constant: D kills it -> happy breakdown
        np.sin(np.pi * x) ** 4,                   # smooth
        rng.standard_normal(n),                   # rough: deep Krylov spaces (cap)
        np.cos(3 * np.pi * x) + 1e-3 * rng.standard_normal(n),
    ])


def _pair(p, c, n, m, cum):
    spec = P.DiscretizationSpec("erk", p, c, n, 64)
    cap = 10 if p == 1 else 20
    st = P.modified_coarse_stepper(spec, m, 1, solver="gmres", gmres_max_iters=cap,
                                   cumulative_factor=cum)
    ost = O.corrected_coarse("erk", p, c, n, m, 1, "gmres", cap=cap, cumulative=cum)
    return st, ost


@pytest.mark.parametrize("p,c,n,m,cum", [(3, 0.85, 4096, 8, 64), (3, 0.85, 4096, 8, 512),
                                         (5, 0.85, 8192, 16, 256), (3, 0.85, 512, 8, 8),
                                         (1, 0.6, 256, 4, 16)])
def test_gmres_edge_rows(p, c, n, m, cum):
    st, ost = _pair(p, c, n, m, cum)
    v = _rows(n)
    ref = ost.apply(v)
    out = st.apply(v)
    assert np.array_equal(out[0], np.zeros(n))
    scale = np.max(np.abs(ref), axis=1, keepdims=True)
    scale[scale == 0] = 1.0
    dev = np.max(np.abs(out - ref) / scale)
    assert dev <= 1e-11, dev


_VARIANT_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O
n, cum = int(sys.argv[2]), int(sys.argv[3])
spec = P.DiscretizationSpec("erk", 3, 0.85, n, 64)
st = P.modified_coarse_stepper(spec, 8, 1, solver="gmres", gmres_max_iters=20, cumulative_factor=cum)
ost = O.corrected_coarse("erk", 3, 0.85, n, 8, 1, "gmres", cap=20, cumulative=cum)
rng = np.random.default_rng(5)
v = np.concatenate([rng.standard_normal((3, n)), np.zeros((1, n)), np.ones((1, n))])
ref = ost.apply(v)
out = st.apply(v)
print(json.dumps({"dev": float(np.max(np.abs(out - ref)) / np.max(np.abs(ref)))}))
"""


@pytest.mark.parametrize("env", [{}, {"MGB_C1_C": "16"}, {"MGB_C1_C": "8"}, {"MGB_C1_C": "4"},
                                 {"MGB_C1_C": "8", "MGB_C1_NO_OCC2": "1"}, {"MGB_CL_CGS2": "1"},
                                 {"MGB_NO_CLUSTER": "1"}, {"MGB_C1_C": "2", "MGB_C1_WIDE": "1"}])
def test_gmres_launch_variants(env):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, ROOT, "4096", "64"], env=e,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    dev = json.loads(out.stdout.strip().splitlines()[-1])["dev"]
    assert dev <= 1e-11, (env, dev)


_DEPTH_SCRIPT = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2209_06916_b200 as P
from oracle import mgrit_oracle as O
from paper_2209_06916_b200.device import plan_for, ptr
out = []
for p, n, m, cum, rows in json.loads(sys.argv[2]):
    cap = 10 if p == 1 else 20
    spec = P.DiscretizationSpec("erk", p, 0.85, n, 64)
    st = P.modified_coarse_stepper(spec, m, 1, solver="gmres", gmres_max_iters=cap,
                                   cumulative_factor=cum)
    ost = O.corrected_coarse("erk", p, 0.85, n, m, 1, "gmres", cap=cap, cumulative=cum)
    rng = np.random.default_rng(cum)
    x = -1.0 + 2.0 * np.arange(n) / n
    v = np.stack([np.sin(np.pi * (x - 0.1 * k)) ** 4 + 1e-2 * rng.standard_normal(n)
                  if k % 2 else np.cumsum(rng.standard_normal(n)) / 50 for k in range(rows)])
    src = torch.from_numpy(v).cuda()
    dst = torch.empty_like(src)
    dep = torch.zeros(rows, dtype=torch.int32, device="cuda")
    res = torch.zeros(rows, dtype=torch.float64, device="cuda")
    plan_for(st.program).relax(rows, 1, 0, c_src=ptr(src), c_stride=n, tail=1, tail_out=ptr(dst),
                               tail_stride=n, stats_depth=ptr(dep), stats_res=ptr(res))
    torch.cuda.synchronize()
    stats = {}
    ref = O.gmres_rows(ost.info["corr"], ost.info["sl"].op.apply(v), 1e-2, cap, stats=stats)[0]
    g = dst.cpu().numpy()
    out.append(dict(case=[p, n, cum], depth_gpu=dep.cpu().numpy().tolist(),
                    depth_ref=stats["depth"].tolist(),
                    res_dev=float(np.max(np.abs(res.cpu().numpy() - stats["res"]))),
                    dev=float(np.max(np.abs(g - ref) / np.max(np.abs(ref), axis=1, keepdims=True)))))
print(json.dumps(out))
"""

# cap-depth rows on the deep, ill-conditioned coarse operators of cfg4 (p = 5,
# cumulative factor 4096, phi = 57: kappa ~ 3.7e3) and cfg5 (p = 3, cumulative
# factors 4096 and 32768 on 16384-point rows), where every row of a 16-interval
# level runs to the column cap: per-row Krylov depth, residual estimate and
# solution against the oracle's MGS GMRES (circulant.py:262-332).  The 2-CTA/SM
# build keeps 19 of cfg4's 20 basis rows in shared memory and the last one in
# its L2 workspace slot.
_DEEP = [[5, 8192, 16, 4096, 16], [5, 8192, 16, 256, 24], [3, 16384, 8, 4096, 16],
         [3, 16384, 8, 32768, 4]]


@pytest.mark.parametrize("env", [{}, {"MGB_C1_NO_OCC2": "1"}, {"MGB_C1_C": "8"},
                                 {"MGB_CL_CGS2": "1"}, {"MGB_NO_CLUSTER": "1"}])
def test_gmres_depths_on_deep_levels(env):
    e = dict(os.environ, **env)
    # the single-CTA and two-reduction kernels stop at 8192-point rows
    cases = [c for c in _DEEP if c[1] <= 8192 or not ({"MGB_CL_CGS2", "MGB_NO_CLUSTER"} & set(env))]
    r = subprocess.run([sys.executable, "-c", _DEPTH_SCRIPT, ROOT, json.dumps(cases)], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    for case in json.loads(r.stdout.strip().splitlines()[-1]):
        assert case["depth_gpu"] == case["depth_ref"], (env, case)
        assert case["res_dev"] <= 1e-10, (env, case)
        assert case["dev"] <= 1e-10, (env, case)
