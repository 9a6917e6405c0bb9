"""Phase breakdown of the e2e solve (bench.py's e2e leg) on cfg2: solver
construction, row upload, device solve, write-back; plus raw pinned
H2D/D2H bandwidth of the iterate.  Prints one JSON line."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_06916_b200 as P  # noqa: E402
from paper_2209_06916_b200.configs import CONFIGS  # noqa: E402


def main(cfg_name="cfg2", reps=4):
    cf = CONFIGS[cfg_name]
    prob = cf.problem()
    cfg = P.MgritConfig(nu=1, cycle=cf.cycle, tol=1e-10, max_iters=30, rng_seed=0)
    u_host = P.MgritSolver(prob, cfg).initial_state()
    host = torch.from_numpy(u_host).pin_memory()
    dev = torch.empty(host.shape, dtype=torch.float64, device="cuda")
    out = {}
    for name, fn in (("h2d_full", lambda: dev.copy_(host, non_blocking=True)),
                     ("d2h_full", lambda: host.copy_(dev, non_blocking=True))):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[name + "_GBps"] = host.numel() * 8 / min(ts) / 1e9
    rows = []
    for _ in range(reps):
        host.copy_(torch.from_numpy(u_host))
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        s = P.MgritSolver(prob, cfg)
        s._build()
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        ud, uh, _ = s._upload(host)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        rep = s.solve(ud)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        host.copy_(ud.reshape(host.shape))
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        rows.append(np.diff(t) * 1e3)
        assert rep.iterations == 11, rep.iterations
    rows = np.array(rows)
    out.update({k: float(np.median(rows[:, i])) for i, k in
                enumerate(("build_ms", "upload_ms", "solve_ms", "writeback_ms"))})
    out["total_ms"] = float(np.median(rows.sum(1)))
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:2])
