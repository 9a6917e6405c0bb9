"""Time-sharded MGRIT host logic on CPU (gloo, world_size 1 and 2) with a
numpy engine built on the oracle: the sharded iterate must equal the
single-process oracle iterate BIT FOR BIT, and the residual history must be
bitwise identical for 1 and 2 ranks (fixed-order norm reduction)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mgrit_oracle as O
from paper_2209_06916_b200.distributed import Engine, ShardedMgritSolver, block_of
from paper_2209_06916_b200.mgrit import MgritConfig

CASES = {
    "erk1_two_level": ("erk", 1, 0.85, 64, 128, 8, "two_level"),
    "erk3_v_cycle": ("erk", 3, 0.85, 64, 256, 4, "v_cycle"),
    "sdirk3_v_cycle": ("sdirk", 3, 4.0, 64, 256, 4, "v_cycle"),
}


class OracleEngine(Engine):
    """Rank-local level-0 passes restated with the numpy oracle (test only)."""

    def __init__(self, steps, factors, n_t, u0, cycle):
        self.steps, self.factors, self.n_t, self.u0, self.cycle = steps, factors, n_t, u0, cycle
        self.step, self.m, self.n = steps[0], factors[0], len(u0)

    def zeros(self, rows):
        return np.zeros((rows, self.n))

    def to_comm(self, a):
        return torch.from_numpy(a) if isinstance(a, np.ndarray) else a

    def from_comm(self, t, like):
        return t.numpy()

    def _fsweep(self, X):
        for _ in range(self.m - 1):
            X = self.step.apply(X) + 0.0  # upd + g, g = 0 on the fine level
        return X

    def initial_partials(self, u_loc, nb):
        m = self.m
        r = (0.0 + self.step.apply(u_loc[m - 1::m][:nb])) - u_loc[m::m][:nb]
        return np.array([float(np.dot(x, x)) for x in r])

    def fc(self, u_loc, cb, k0, nb):
        cb[1:] = self.step.apply(self._fsweep(u_loc[0:nb * self.m:self.m].copy())) + 0.0

    def fr(self, cb, g1, k0, nb):
        g1[:] = (0.0 + self.step.apply(self._fsweep(cb[:nb].copy()))) - cb[1:]

    def cf(self, u_loc, cb, e_loc, k0, nb):
        m = self.m
        c = cb[:nb].copy()
        start = 1 if k0 == 0 else 0
        c[start:] = cb[start:nb] + e_loc[start:nb]
        u_loc[0:nb * m:m] = c
        X = c
        for j in range(1, m):
            X = self.step.apply(X) + 0.0
            u_loc[j:nb * m:m] = X
        u_loc[nb * m] = cb[nb] + e_loc[nb]
        r = (0.0 + self.step.apply(X)) - (cb[1:] + e_loc[1:])
        return np.array([float(np.dot(x, x)) for x in r])

    def coarse_solve(self, gc):
        if self.cycle == "two_level" or len(self.factors) == 1:
            return O.forward_substitute(self.steps[1], gc)
        mg = O.Mgrit(self.steps, self.factors, self.n_t, self.u0, cycle=self.cycle)
        e = np.zeros_like(gc)
        mg.cycle_once(1, e, gc)
        return e


def _worker(rank, world, port, case, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fam, p, c, nx, nt, m, cyc = CASES[case]
    steps, fac, u0 = O.build_hierarchy(fam, p, c, nx, nt, m, cyc,
                                       fine_mode="staged" if fam == "sdirk" else "assembled")
    u = O.initial_iterate(0, nt, nx, u0)
    eng = OracleEngine(steps, fac, nt, u0, cyc)
    # a problem object only for metadata (m, n_t) -- the engine does the work
    prob = type("Prob", (), {"m": fac, "n_t": nt, "n_x": nx})()
    sol = ShardedMgritSolver(prob, MgritConfig(cycle=cyc), eng)
    r0, r1 = sol.local_rows()
    u_loc = u[r0:r1].copy()
    rep = sol.solve(u_loc)
    np.savez(os.path.join(outdir, f"{case}_{world}_{rank}.npz"), u=u_loc, r0=r0,
             norms=np.array(rep.residual_norms), iters=rep.iterations)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_matches_single_process_oracle(case):
    fam, p, c, nx, nt, m, cyc = CASES[case]
    steps, fac, u0 = O.build_hierarchy(fam, p, c, nx, nt, m, cyc,
                                       fine_mode="staged" if fam == "sdirk" else "assembled")
    ref = O.Mgrit(steps, fac, nt, u0, cycle=cyc).solve()
    with tempfile.TemporaryDirectory() as d:
        runs = {}
        for world in (1, 2):
            mp.spawn(_worker, args=(world, _free_port(), case, d), nprocs=world, join=True)
            parts = [np.load(os.path.join(d, f"{case}_{world}_{r}.npz")) for r in range(world)]
            u = ref["u"].copy() * np.nan
            for q in parts:
                r0 = int(q["r0"])
                u[r0:r0 + q["u"].shape[0]] = q["u"]
            runs[world] = (u, parts[0]["norms"], int(parts[0]["iters"]))
    for world, (u, norms, iters) in runs.items():
        assert iters == ref["iterations"]
        assert np.array_equal(u, ref["u"]), world            # bit-identical iterate
        np.testing.assert_allclose(norms, ref["norms"], rtol=1e-13, atol=0)
    assert np.array_equal(runs[1][1], runs[2][1])               # bitwise across rank counts


def test_initial_rows_match_one_shot_rng():
    from paper_2209_06916_b200.distributed import initial_rows
    u0 = O.sin4(32)
    full = O.initial_iterate(7, 64, 32, u0)
    for r0, r1 in ((0, 17), (17, 40), (40, 65)):
        assert np.array_equal(initial_rows(7, r0, r1, 32, u0), full[r0:r1])


def test_block_partition():
    assert block_of(2048, 8, 3) == (768, 1024)
    with pytest.raises(ValueError):
        block_of(10, 4, 0)
