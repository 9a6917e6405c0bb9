"""Time-sharded MGRIT over several GPUs (one process per GPU, torch.distributed).

The reference has no distribution (the paper used XBraid + MPI on
CPUs).  MGRIT itself is the time-parallel method, so the B200 build shards the
TIME axis on every level that has enough intervals:

* level l is *sharded* when its interval count splits evenly over the ranks
  (and the block boundaries of level l-1 are level-l interval boundaries);
  rank g owns the contiguous block of level-l CF-intervals [k0_l, k0_l + nb_l)
  and the level-l points [k0_l m_l, (k0_l + nb_l) m_l] -- the last point is the
  next rank's first, kept as a consistent ghost that both ranks compute with
  identical arithmetic;
* the level-l passes FC, FR, CF run rank-locally; the FR residual of a rank's
  intervals is exactly the right-hand side of its level-(l+1) points, and the
  level-(l+1) correction of its points is what its CF needs, so consecutive
  sharded levels exchange nothing;
* the only data-path exchanges are
    - per FC pass and sharded level: the C-relaxation of rank g's last interval
      is rank g+1's first C-point (point-to-point, one row of n_x * 8 bytes),
    - at the first non-sharded level (too few intervals, or the coarsest): the
      right-hand side rows gathered to rank 0, which runs the rest of the cycle
      (the BASELINE "coarsest level solved sequentially on one GPU"), and the
      correction rows scattered back,
    - the level-0 residual-norm partials gathered in global interval order and
      summed in fixed order on rank 0 -> the history is bitwise identical for
      any number of ranks;
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


def sharded_levels(factors, n_t: int, world: int, cycle: str, min_block: int = 1) -> int:
    """Number of leading levels that are time-sharded over ``world`` ranks:
    level 0 always (its interval count must split evenly); level l >= 1 while it
    is not the coarsest level, the cycle recurses (not two-level) and its
    n_int_l intervals split into blocks of at least ``min_block`` intervals."""
    n_int = n_t // factors[0]
    if n_int % world:
        raise ValueError(f"{n_int} level-0 intervals do not split over {world} ranks")
    ls = 1
    if cycle == "two_level":
        return ls
    n_pts = n_int
    for l in range(1, len(factors)):
        if n_pts % factors[l]:
            break
        n_int_l = n_pts // factors[l]
        if n_int_l % world or n_int_l // world < min_block:
            break
        ls += 1
        n_pts = n_int_l
    return ls


class Engine:
    """Rank-local passes of one level on local blocks.

    Arrays are engine-native (torch CUDA tensors or numpy).  On level l a rank
    holds ``u`` (its nb*m+1 points, ghost last), ``g`` (same rows; None on level
    0), C-point buffers ``cb`` (nb+1 rows; row 0 = the left neighbour's last
    C-relaxed point), the next level's right-hand side ``gn`` and correction
    ``e`` (nb+1 rows each, point k0..k0+nb).  ``src`` is the C-point source of a
    pass: None = the C-points of ``u`` (zeros when ``u_zero``), else a cb.
    The global first interval (k0 == 0, local 0) always starts from point 0 of
    ``u`` (zero when ``u_zero``), as the single-GPU kernels do.
    """

    def zeros(self, rows: int): raise NotImplementedError
    def to_comm(self, a): raise NotImplementedError       # array -> torch tensor for dist
    def from_comm(self, t, like): raise NotImplementedError
    def initial_partials(self, u_loc, nb: int): raise NotImplementedError
    def fc(self, l, u, g, src, cb, k0, nb, u_zero): raise NotImplementedError
    def fr(self, l, u, g, src, gn, k0, nb, u_zero): raise NotImplementedError
    def cf(self, l, u, g, src, e, k0, nb, u_zero, want_norm): raise NotImplementedError
    def coarse_solve(self, level, g_full, kind): raise NotImplementedError  # rank 0
    def ordered_sum(self, allp): raise NotImplementedError  # rank 0: (1,) comm tensor


class GpuEngine(Engine):
    """libmgrit_b200 kernels on this rank's CUDA device."""

    def __init__(self, problem: TimeGridProblem, config: MgritConfig):
        from .device import plan_for, require_cuda
        self.torch = require_cuda()
        self.problem, self.config = problem, config
        self.n = problem.n_x
        self.m = list(problem.m)
        self.plans = [plan_for(problem.steppers[l].program) for l in range(len(self.m))]
        self.zero_row = self.torch.zeros(self.n, dtype=self.torch.float64, device="cuda")
        self._coarse = None
        #: set to a list to record (name, start_event, end_event) per launch
        self.profile = None

    def _relax(self, name, l, *args, **kw):
        if self.profile is None:
            return self.plans[l].relax(*args, **kw)
        ev = [self.torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        self.plans[l].relax(*args, **kw)
        ev[1].record()
        self.profile.append((name, ev[0], ev[1]))

    def profile_summary(self) -> dict:
        """{pass name: (launches, total ms)} of the recorded launches."""
        self.torch.cuda.synchronize()
        out = {}
        for name, s, e in self.profile or []:
            cnt, ms = out.get(name, (0, 0.0))
            out[name] = (cnt + 1, ms + s.elapsed_time(e))
        return out

    def ordered_sum(self, allp):
        """mgb_sum over the partials in global interval order: the single-GPU
        solver's fixed-order tree, so the history is bitwise the single-GPU one."""
        from .device import device_sum
        out = self.torch.empty(1, dtype=self.torch.float64, device="cuda")
        device_sum(allp.data_ptr(), allp.numel(), out.data_ptr())
        return out

    def zeros(self, rows):
        return self.torch.zeros((rows, self.n), dtype=self.torch.float64, device="cuda")

    def to_comm(self, a):
        return a

    def from_comm(self, t, like):
        return t

    def _p(self, a, row=0):
        return None if a is None else a.data_ptr() + row * self.n * _F64

    def initial_partials(self, u_loc, nb):
        part = self.torch.empty(nb, dtype=self.torch.float64, device="cuda")
        m, n = self.m[0], self.n
        self._relax("L0.R", 0, nb, m, 0, c_src=self._p(u_loc, m - 1), c_stride=m * n, tail=2,
                    cref=self._p(u_loc, m), cref_stride=m * n, partials=part.data_ptr())
        return part

    def _src(self, l, u, src, u_zero):
        m, n = self.m[l], self.n
        u0row = self.zero_row.data_ptr() if u_zero else self._p(u)
        if src is None:
            return (None if u_zero else self._p(u)), m * n, u0row
        return self._p(src), n, u0row

    #: iterations >= 2: the opening F-relaxation reads the stored last F-points
    #: (MgritSolver._cycle, mgrit.py module docstring)
    supports_f_relaxed = True

    def fc(self, l, u, g, src, cb, k0, nb, u_zero, f_relaxed=False):
        m, n = self.m[l], self.n
        if f_relaxed and src is None and not u_zero:
            self._relax(f"L{l}.FC", l, nb, m, 0, k_global0=k0, c_src=self._p(u, m - 1),
                        c_stride=m * n, tail=1, tail_out=self._p(cb, 1), tail_stride=n,
                        g=self._p(g))
            return
        c_src, stride, u0row = self._src(l, u, src, u_zero)
        self._relax(f"L{l}.FC", l, nb, m, m - 1, k_global0=k0, c_src=c_src, c_stride=stride,
                    c_src0=u0row, tail=1, tail_out=self._p(cb, 1), tail_stride=n,
                    g=self._p(g))

    def fr(self, l, u, g, src, gn, k0, nb, u_zero, f_relaxed=False):
        m, n = self.m[l], self.n
        c_src, stride, u0row = self._src(l, u, src, u_zero)
        if src is None:
            cref, cref_stride = ((self.zero_row.data_ptr(), 0) if u_zero
                                 else (self._p(u, m), m * n))
        else:
            cref, cref_stride = self._p(src, 1), n
        if f_relaxed and src is None and not u_zero:
            self._relax(f"L{l}.FR", l, nb, m, 0, k_global0=k0, c_src=self._p(u, m - 1),
                        c_stride=m * n, tail=2, cref=cref, cref_stride=cref_stride,
                        tail_out=self._p(gn, 1), tail_stride=n, g=self._p(g))
            return
        self._relax(f"L{l}.FR", l, nb, m, m - 1, k_global0=k0, c_src=c_src, c_stride=stride,
                    c_src0=u0row, tail=2, cref=cref, cref_stride=cref_stride,
                    tail_out=self._p(gn, 1), tail_stride=n, g=self._p(g))

    def cf(self, l, u, g, src, e, k0, nb, u_zero, want_norm):
        m, n = self.m[l], self.n
        c_src, stride, u0row = self._src(l, u, src, u_zero)
        fuse = want_norm and src is not None
        part = self.torch.empty(nb, dtype=self.torch.float64, device="cuda") if want_norm else None
        self._relax(f"L{l}.CF", l, nb, m, m - 1, k_global0=k0, c_src=c_src, c_stride=stride,
                    c_src0=u0row, e=self._p(e), e_stride=n, c_out=self._p(u),
                    c_out_stride=m * n, c_last_out=self._p(u, nb * m), u=self._p(u),
                    write_f=2, g=self._p(g), tail=2 if fuse else 0,
                    cref=(c_src + n * _F64) if fuse else None, cref_stride=n,
                    cref_e=self._p(e, 1), cref_e_stride=n,
                    partials=part.data_ptr() if fuse else None)
        if want_norm and not fuse:
            self._relax("L0.R", l, nb, m, 0, c_src=self._p(u, m - 1), c_stride=m * n, tail=2,
                        cref=self._p(u, m), cref_stride=m * n, g=self._p(g),
                        partials=part.data_ptr())
        return part

    def coarse_solve(self, level, g_full, kind):
        if self._coarse is None:
            self._coarse = MgritSolver(self.problem, self.config)
            self._coarse._build()
        s = self._coarse
        s.profile = self.profile
        s.gcoarse[level].copy_(g_full)
        s._coarse_solve(level, kind)
        s.profile = None
        return s.ucoarse[level]


class ShardedMgritSolver:
    """MGRIT with the time axis split over the ranks of ``group`` on every
    sharded level (``sharded_levels``; ``max_sharded`` caps it, 1 = level 0
    only)."""

    def __init__(self, problem: TimeGridProblem, config: MgritConfig, engine: Engine,
                 group=None, max_sharded: Optional[int] = None, min_block: int = 1):
        import torch.distributed as dist
        self.dist = dist
        self.problem, self.config, self.engine, self.group = problem, config, engine, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.factors = list(problem.m)
        self.m = self.factors[0]
        self.n_int = problem.n_t // self.m
        self.k0, self.k1 = block_of(self.n_int, self.world, self.rank)
        self.nb = self.k1 - self.k0
        ls = sharded_levels(self.factors, problem.n_t, self.world, config.cycle, min_block)
        if max_sharded is not None:
            ls = max(1, min(ls, int(max_sharded)))
        self.ls = ls
        # per sharded level: (k0_l, nb_l); level l's points are level l-1's C-points
        self.blocks = []
        n_int = self.n_int
        for l in range(ls):
            if l > 0:
                n_int //= self.factors[l]
            nb = n_int // self.world
            self.blocks.append((self.rank * nb, nb))
        self._bufs = None

    def local_rows(self):
        """Global row range [r0, r1) of this rank's iterate block (incl. ghost)."""
        return self.k0 * self.m, self.k1 * self.m + 1

    # ------------------------------------------------------------ buffers
    def _buffers(self):
        if self._bufs is not None:
            return self._bufs
        eng = self.engine
        nu = self.config.nu
        b = {"cb": [], "u": [None], "g": [None]}
        for l in range(self.ls):
            nb = self.blocks[l][1]
            b["cb"].append([eng.zeros(nb + 1) for _ in range(min(max(nu, 0), 2))])
            # level l+1 vectors on this rank: points k0_l .. k0_l + nb_l
            b["u"].append(eng.zeros(nb + 1))
            b["g"].append(eng.zeros(nb + 1))
        self._bufs = b
        return b

    # --------------------------------------------------------- exchanges
    def _pass_right(self, cb, nb):
        """cb[nb] (my last C-relaxed point) -> the right neighbour's cb[0]
        (non-blocking send and receive, both posted before either waits)."""
        import torch
        if self.world == 1:
            return
        eng, dist = self.engine, self.dist
        reqs = []
        recv = None
        if self.rank > 0:
            first = eng.to_comm(cb[0:1])
            recv = torch.empty_like(first)
            reqs.append(dist.irecv(recv, self.rank - 1, group=self.group))
        if self.rank + 1 < self.world:
            reqs.append(dist.isend(eng.to_comm(cb[nb:nb + 1]).contiguous(), self.rank + 1,
                                   group=self.group))
        for r in reqs:
            r.wait()
        if recv is not None:
            first.copy_(recv)
            cb[0:1] = eng.from_comm(first, cb[0:1])

    def _gather_solve_scatter(self, level, gn, nb, kind):
        """Rows 1..nb of every rank's gn -> rank 0 (row 0 = 0), which solves
        level ``level`` (and below) from e = 0; rows [k0, k0+nb] of e back."""
        import torch
        eng, dist = self.engine, self.dist
        gt = eng.to_comm(gn[1:nb + 1]).contiguous()
        if self.world > 1:
            bufs = [torch.empty_like(gt) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(gt, bufs, dst=0, group=self.group)
        else:
            bufs = [gt]
        e_all = None
        if self.rank == 0:
            gc = torch.cat([torch.zeros_like(gt[0:1])] + bufs)
            e_all = eng.to_comm(eng.coarse_solve(level, eng.from_comm(gc, None), kind)).contiguous()
        e_t = torch.empty((nb + 1, gt.shape[1]), dtype=gt.dtype, device=gt.device)
        if self.world > 1:
            if self.rank == 0:
                reqs = [dist.isend(e_all[r * nb:(r + 1) * nb + 1].contiguous(), r, group=self.group)
                        for r in range(1, self.world)]
                e_t.copy_(e_all[0:nb + 1])
                for q in reqs:
                    q.wait()
            else:
                dist.recv(e_t, 0, group=self.group)
        else:
            e_t.copy_(e_all[0:nb + 1])
        return eng.from_comm(e_t, None)

    # --------------------------------------------------------------- cycle
    def _cycle(self, l, u, g, u_zero, want_norm, kind, f_relaxed=False):
        """One cycle on sharded level l (mgrit.py:225-247, MgritSolver._cycle)."""
        from . import mgrit as _mg
        eng, cfg = self.engine, self.config
        k0, nb = self.blocks[l]
        bufs = self._buffers()
        src = None
        opt = ({"f_relaxed": True} if f_relaxed and not u_zero and _mg.ELIDE_OPENING_F_RELAX
               and getattr(eng, "supports_f_relaxed", False) else {})
        for i in range(cfg.nu):
            cb = bufs["cb"][l][i % 2]
            eng.fc(l, u, g, src, cb, k0, nb, u_zero, **(opt if i == 0 else {}))
            self._pass_right(cb, nb)
            src = cb
        gn, e = bufs["g"][l + 1], bufs["u"][l + 1]
        eng.fr(l, u, g, src, gn, k0, nb, u_zero, **(opt if cfg.nu == 0 else {}))
        e = self._coarse(l + 1, e, gn, nb, kind)
        return eng.cf(l, u, g, src, e, k0, nb, u_zero, want_norm)

    def _coarse(self, child, e, gn, nb, kind):
        """Correction on level ``child`` (MgritSolver._coarse_solve, sharded)."""
        if child >= self.ls:
            return self._gather_solve_scatter(child, gn, nb, kind)
        # from e = 0: the passes never read e (zero C-points), CF writes all of it
        if kind == "f_cycle":
            self._cycle(child, e, gn, True, False, "f_cycle")
            self._cycle(child, e, gn, False, False, "v_cycle", f_relaxed=True)
        else:
            self._cycle(child, e, gn, True, False, "v_cycle")
        return e

    def _global_sum(self, part) -> float:
        """Sum of the per-interval partials of all ranks: gathered in global
        interval order into one buffer on rank 0 and reduced there by the
        engine's fixed-order sum (GPU: the single-GPU solver's ``mgb_sum``
        tree), so the history is bitwise independent of the number of ranks."""
        import torch
        eng, dist = self.engine, self.dist
        t = eng.to_comm(part).contiguous()
        if self.world > 1:
            bufs = [torch.empty_like(t) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(t, bufs, dst=0, group=self.group)
            allp = torch.cat(bufs) if self.rank == 0 else None
        else:
            allp = t
        if self.rank == 0:
            tot = eng.ordered_sum(allp)
        else:
            tot = torch.zeros(1, dtype=torch.float64, device=t.device)
        if self.world > 1:
            dist.broadcast(tot, src=0, group=self.group)
        return math.sqrt(float(tot.item()))

    def iterate(self, u_loc, f_relaxed=False):
        """One cycle on the local block; returns the level-0 norm partials.
        ``f_relaxed``: the F-points are the F-relaxation of the C-points (the
        state the previous cycle left)."""
        return self._cycle(0, u_loc, None, False, True, self.config.cycle, f_relaxed)

    def solve(self, u_loc) -> SolveReport:
        """Run to the halting rule; every rank returns the same report."""
        cfg = self.config
        t0 = time.perf_counter()
        norms = [self._global_sum(self.engine.initial_partials(u_loc, self.nb))]
        it, converged = 0, False
        while it < cfg.max_iters:
            part = self.iterate(u_loc, f_relaxed=it > 0)
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

