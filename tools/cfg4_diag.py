"""cfg4 parity bisection on the GPU.

    python tools/cfg4_diag.py > gpurun_out/cfg4_diag.json

For each GMRES kernel variant (default launch choice; single-CTA MGS
everywhere, MGB_NO_CLUSTER=1; two-reduction CGS2 clusters, MGB_CL_CGS2=1) in
its own process:
  * fine ERK5 relaxation at n_x = 8192 (cfg4's row length) vs the oracle, bitwise;
  * the full cfg4 solve: residual history vs the real reference's
    (tests/golden/histories.json);
  * per-call GMRES on realistic inputs: after one MGRIT iteration, rows of each
    coarse level's error e_l go through the level-l stepper on the GPU (per-row
    Krylov depth and residual from mgb_relax_args.stats_*) and through the
    oracle (circulant.py:262-332 restated), compared row by row.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {"default": {}, "mgs_single_cta": {"MGB_NO_CLUSTER": "1"},
            "cgs2_cluster": {"MGB_CL_CGS2": "1"}}


def child(variant):
    import numpy as np
    import torch
    import paper_2209_06916_b200 as P
    from oracle import mgrit_oracle as O
    from paper_2209_06916_b200.configs import CONFIGS
    from paper_2209_06916_b200.device import plan_for, ptr
    out = {"variant": variant}
    # ---- fine ERK5 pass at n_x = 8192
    n, nt, m = 8192, 64, 16
    spec = P.DiscretizationSpec("erk", 5, 0.85, n, nt)
    st, ost = P.mol_stepper(spec), O.mol_step("erk", 5, 0.85, n)
    u = O.initial_iterate(0, nt, n, O.sin4(n))
    g = np.zeros_like(u)
    g[0] = u[0]
    O.ROLL_LIMIT = 64
    uo, ug = u.copy(), u.copy()
    O.f_relax(uo, g, ost, m)
    P.f_relax(ug, g, st, m)
    out["fine_f_relax_bitwise"] = bool(np.array_equal(uo, ug))
    out["fine_f_relax_maxdiff"] = float(np.max(np.abs(uo - ug)))
    O.c_relax(uo, g, ost, m)
    P.c_relax(ug, g, st, m)
    out["fine_c_relax_bitwise"] = bool(np.array_equal(uo, ug))
    out["fine_restrict_bitwise"] = bool(np.array_equal(O.restrict(uo, g, ost, m),
                                                       P.restrict_residual(ug, g, st, m)))
    # ---- full solve history
    cf = CONFIGS["cfg4"]
    prob = cf.problem()
    hist = json.load(open(os.path.join(ROOT, "tests", "golden", "histories.json")))["cfg4"]
    sol = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle))
    u0 = sol.initial_state()
    ud = torch.from_numpy(u0).cuda()
    rep = sol.solve(ud)
    r0 = hist["norms"][0]
    out["iterations"] = rep.iterations
    out["norms"] = rep.residual_norms
    out["dev_over_r0"] = [abs(a - b) / r0 for a, b in zip(rep.residual_norms, hist["norms"])]
    out["rel_dev"] = [abs(a - b) / b for a, b in zip(rep.residual_norms, hist["norms"])]
    del ud
    # ---- per-call GMRES after one iteration
    sol1 = P.MgritSolver(prob, P.MgritConfig(cycle=cf.cycle, max_iters=1))
    ud = torch.from_numpy(u0).cuda()
    sol1.solve(ud)
    del ud
    torch.cuda.empty_cache()
    calls = {}
    for lvl in range(1, len(prob.m)):
        e = sol1.ucoarse[lvl]
        npts = e.shape[0]
        idx = np.unique(np.linspace(1, npts - 1, min(24, npts - 1)).astype(np.int64))
        src = e[torch.from_numpy(idx).cuda()].contiguous()
        rows = src.shape[0]
        dst = torch.empty_like(src)
        dep = torch.zeros(rows, dtype=torch.int32, device="cuda")
        res = torch.zeros(rows, dtype=torch.float64, device="cuda")
        plan = plan_for(prob.steppers[lvl].program)
        plan.relax(rows, 1, 0, c_src=ptr(src), c_stride=n * 0 + cf.n_x, tail=1, tail_out=ptr(dst),
                   tail_stride=cf.n_x, stats_depth=ptr(dep), stats_res=ptr(res))
        torch.cuda.synchronize()
        s_np = src.cpu().numpy()
        ost = O.corrected_coarse("erk", 5, 0.85, cf.n_x, 16, 1, "gmres", cap=20,
                                 cumulative=16 ** lvl)
        rhs = ost.info["sl"].op.apply(s_np)
        stats = {}
        x = O.gmres_rows(ost.info["corr"], rhs, 1e-2, 20, stats=stats)[0]
        xg = dst.cpu().numpy()
        scale = np.maximum(np.max(np.abs(x), axis=1), 1e-300)
        calls[f"L{lvl}"] = {
            "phi": float(ost.info["phi"]), "rows": int(rows),
            "depth_gpu": dep.cpu().numpy().tolist(), "depth_oracle": stats["depth"].tolist(),
            "res_gpu": res.cpu().numpy().tolist(), "res_oracle": stats["res"].tolist(),
            "row_rel_err": (np.max(np.abs(xg - x), axis=1) / scale).tolist()}
    out["calls"] = calls
    print(json.dumps(out), flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(sys.argv[2])
        return
    names = sys.argv[1:] or list(VARIANTS)
    res = {}
    for name in names:
        env = dict(os.environ, **VARIANTS[name])
        r = subprocess.run([sys.executable, __file__, "--child", name], env=env,
                           capture_output=True, text=True, timeout=1200)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        res[name] = json.loads(line[-1]) if line else {"error": r.stderr[-3000:]}
        print(name, "done", file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
