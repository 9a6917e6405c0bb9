"""Time-sharded MGRIT over several GPUs (one process per GPU, torch.distributed).

The reference has no distribution (the paper used XBraid + MPI on
CPUs).  MGRIT itself is the time-parallel method, so the B200 build shards the
TIME axis:

* rank g owns the contiguous block of level-0 CF-intervals [k0, k1) and the
  iterate rows [k0*m, k1*m] (the last row is the next rank's first C-point, kept
  as a consistent ghost);
* per cycle the level-0 passes FC, FR, CF run rank-locally; the only data-path
  exchanges are
    - one boundary C-point row per cycle: the C-relaxation of rank g's last
      interval is rank g+1's first C-point (point-to-point, n_x * 8 bytes),
    - the injected coarse right-hand side gathered to rank 0 (n_int rows) and
      the coarse correction scattered back: levels >= 1 run on rank 0 (the
      BASELINE "coarsest level solved sequentially on one GPU"),
    - the residual-norm partials gathered in global interval order and summed
      in fixed order on rank 0 -> the history is bitwise identical for any
      number of ranks.
* every per-interval arithmetic operation is the single-GPU one, so the final
  iterate equals the single-GPU iterate bit for bit.

The driver is written against an engine interface (`Engine`); `GpuEngine`
launches the libmgrit_b200 kernels on local CUDA tensors (NCCL); tests plug a
numpy engine built on the CPU oracle (gloo) to check the host logic.
"""

from __future__ import annotations

import math
import time
from typing import List, Optional

import numpy as np

from .mgrit import MgritConfig, MgritSolver, SolveReport, TimeGridProblem

_F64 = 8


def block_of(n_int: int, world: int, rank: int):
    """Contiguous interval block [k0, k1) of ``rank`` (n_int divisible by world)."""
    if n_int % world:
        raise ValueError(f"{n_int} level-0 intervals do not split over {world} ranks")
    b = n_int // world
    return rank * b, (rank + 1) * b


class Engine:
    """Rank-local level-0 operations on local row blocks.

    Arrays are engine-native (torch CUDA tensors or numpy); ``u_loc`` holds rows
    [k0*m, k1*m], ``cb`` the C-point buffer (nb+1 rows), ``g1`` the coarse rhs
    rows of this block (nb rows, global C-points k0+1..k1).
    """

    def zeros(self, rows: int): raise NotImplementedError
    def to_comm(self, a): raise NotImplementedError       # array -> torch tensor for dist
    def from_comm(self, t, like): raise NotImplementedError
    def initial_partials(self, u_loc, nb: int): raise NotImplementedError
    def fc(self, u_loc, cb, k0: int, nb: int): raise NotImplementedError
    def fr(self, cb, g1, k0: int, nb: int): raise NotImplementedError
    def cf(self, u_loc, cb, e_loc, k0: int, nb: int): raise NotImplementedError  # -> partials
    def coarse_solve(self, g_coarse): raise NotImplementedError  # rank 0: e (n_int+1 rows)


class GpuEngine(Engine):
    """libmgrit_b200 kernels on this rank's CUDA device."""

    def __init__(self, problem: TimeGridProblem, config: MgritConfig):
        from .device import plan_for, require_cuda
        self.torch = require_cuda()
        self.problem, self.config = problem, config
        self.n = problem.n_x
        self.m = problem.m[0]
        self.plan = plan_for(problem.steppers[0].program)
        self._coarse = None

    def zeros(self, rows):
        return self.torch.zeros((rows, self.n), dtype=self.torch.float64, device="cuda")

    def to_comm(self, a):
        return a

    def from_comm(self, t, like):
        return t

    def _p(self, a, row=0):
        return a.data_ptr() + row * self.n * _F64

    def initial_partials(self, u_loc, nb):
        part = self.torch.empty(nb, dtype=self.torch.float64, device="cuda")
        m, n = self.m, self.n
        self.plan.relax(nb, m, 0, c_src=self._p(u_loc, m - 1), c_stride=m * n, tail=2,
                        cref=self._p(u_loc, m), cref_stride=m * n, partials=part.data_ptr())
        return part

    def fc(self, u_loc, cb, k0, nb):
        m, n = self.m, self.n
        self.plan.relax(nb, m, m - 1, k_global0=k0, c_src=self._p(u_loc), c_stride=m * n,
                        tail=1, tail_out=self._p(cb, 1), tail_stride=n)

    def fr(self, cb, g1, k0, nb):
        m, n = self.m, self.n
        self.plan.relax(nb, m, m - 1, k_global0=k0, c_src=self._p(cb), c_stride=n, tail=2,
                        cref=self._p(cb, 1), cref_stride=n, tail_out=self._p(g1), tail_stride=n)

    def cf(self, u_loc, cb, e_loc, k0, nb):
        m, n = self.m, self.n
        part = self.torch.empty(nb, dtype=self.torch.float64, device="cuda")
        self.plan.relax(nb, m, m - 1, k_global0=k0, c_src=self._p(cb), c_stride=n,
                        e=self._p(e_loc), e_stride=n, c_out=self._p(u_loc), c_out_stride=m * n,
                        c_last_out=self._p(u_loc, nb * m), u=self._p(u_loc), write_f=2, tail=2,
                        cref=self._p(cb, 1), cref_stride=n, cref_e=self._p(e_loc, 1),
                        cref_e_stride=n, partials=part.data_ptr())
        return part

    def coarse_solve(self, g_coarse):
        if self._coarse is None:
            self._coarse = MgritSolver(self.problem, self.config)
            self._coarse._build()
        s = self._coarse
        s.gcoarse[1].copy_(g_coarse)
        s._coarse_solve(1)
        return s.ucoarse[1]


class ShardedMgritSolver:
    """MGRIT with the time axis split over the ranks of ``group`` (nu >= 1)."""

    def __init__(self, problem: TimeGridProblem, config: MgritConfig, engine: Engine,
                 group=None):
        import torch.distributed as dist
        self.dist = dist
        self.problem, self.config, self.engine, self.group = problem, config, engine, group
        if config.nu < 1:
            raise ValueError("the sharded solver implements nu >= 1 (FCF)")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.m = problem.m[0]
        self.n_int = problem.n_t // self.m
        self.k0, self.k1 = block_of(self.n_int, self.world, self.rank)
        self.nb = self.k1 - self.k0

    def local_rows(self):
        """Global row range [r0, r1) of this rank's iterate block (incl. ghost)."""
        return self.k0 * self.m, self.k1 * self.m + 1

    def _global_sum(self, part) -> float:
        """Fixed-order sum of per-interval partials over all ranks (bitwise
        independent of the number of ranks)."""
        import torch
        eng, dist = self.engine, self.dist
        t = eng.to_comm(part)
        if self.world > 1:
            bufs = [torch.empty_like(t) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(t, bufs, dst=0, group=self.group)
            allp = torch.cat(bufs) if self.rank == 0 else None
        else:
            allp = t
        tot = torch.zeros(1, dtype=torch.float64, device=t.device)
        if self.rank == 0:
            tot[0] = _ordered_sum(allp)
        if self.world > 1:
            dist.broadcast(tot, src=0, group=self.group)
        return math.sqrt(float(tot.item()))

    def iterate(self, u_loc):
        """One FCF cycle on the local block (mgrit.py:225-247, sharded)."""
        import torch
        eng, dist, nb, k0 = self.engine, self.dist, self.nb, self.k0
        cb = eng.zeros(nb + 1)
        eng.fc(u_loc, cb, k0, nb)
        # boundary exchange: my C-relaxed last point is the next rank's cb[0]
        first = eng.to_comm(cb[0:1])
        if self.rank == 0:
            first.copy_(eng.to_comm(u_loc[0:1]))
        if self.world > 1:
            reqs = []
            if self.rank + 1 < self.world:
                reqs.append(dist.isend(eng.to_comm(cb[nb:nb + 1]).contiguous(), self.rank + 1,
                                       group=self.group))
            if self.rank > 0:
                recv = torch.empty_like(first)
                dist.recv(recv, self.rank - 1, group=self.group)
                first.copy_(recv)
            for r in reqs:
                r.wait()
        cb[0:1] = eng.from_comm(first, cb[0:1])
        g1 = eng.zeros(nb)
        eng.fr(cb, g1, k0, nb)
        # gather the coarse rhs on rank 0, solve levels >= 1 there, scatter e back
        gt = eng.to_comm(g1).contiguous()
        if self.world > 1:
            bufs = [torch.empty_like(gt) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(gt, bufs, dst=0, group=self.group)
        else:
            bufs = [gt]
        e_all = None
        if self.rank == 0:
            gc = torch.cat([torch.zeros_like(gt[0:1])] + bufs)
            e_all = eng.to_comm(eng.coarse_solve(eng.from_comm(gc, None))).contiguous()
        e_loc_t = torch.empty((nb + 1, gt.shape[1]), dtype=gt.dtype, device=gt.device)
        if self.world > 1:
            if self.rank == 0:
                reqs = [dist.isend(e_all[r * nb:(r + 1) * nb + 1].contiguous(), r, group=self.group)
                        for r in range(1, self.world)]
                e_loc_t.copy_(e_all[0:nb + 1])
                for q in reqs:
                    q.wait()
            else:
                dist.recv(e_loc_t, 0, group=self.group)
        else:
            e_loc_t.copy_(e_all[0:nb + 1])
        e_loc = eng.from_comm(e_loc_t, None)
        return eng.cf(u_loc, cb, e_loc, k0, nb)

    def solve(self, u_loc) -> SolveReport:
        """Run to the halting rule; every rank returns the same report."""
        cfg = self.config
        t0 = time.perf_counter()
        norms = [self._global_sum(self.engine.initial_partials(u_loc, self.nb))]
        it, converged = 0, False
        while it < cfg.max_iters:
            part = self.iterate(u_loc)
            it += 1
            norms.append(self._global_sum(part))
            if norms[0] > 0 and norms[-1] / norms[0] <= cfg.tol:
                converged = True
                break
        wall = time.perf_counter() - t0
        rho = norms[-1] / norms[-2] if len(norms) >= 2 and norms[-2] > 0 else 0.0
        return SolveReport(norms, it, float(rho), converged, wall)


def initial_rows(seed: int, r0: int, r1: int, n_x: int, u0) -> np.ndarray:
    """Rows [r0, r1) of the reference's random initial iterate (mgrit.py:206-211)
    without generating the others: PCG64 advanced by r0*n_x draws (bit-exact
    with the one-shot ``default_rng(seed).random((n_t+1, n_x))``)."""
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance(r0 * n_x)
    u = rng.random((r1 - r0, n_x))
    if r0 == 0:
        u[0] = u0
    return u


def _ordered_sum(t) -> float:
    """Sequential sum in interval order (host side, exact same order for any
    rank count)."""
    acc = 0.0
    for v in t.detach().cpu().numpy().tolist():
        acc += v
    return acc
