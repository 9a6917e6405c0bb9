"""Linear MGRIT on the B200 (drop-in for mgrit.py of the reference).

Same API and semantics as the reference (mgrit.py:28-297): F(CF)^nu
relaxation, injection restriction, two-level or V-cycle, halting on
``norms[-1] / norms[0] <= tol``, divergence reported, ``initial_iterate``
mutated in place.  The iterate lives in HBM; every relaxation, restriction,
correction and norm runs in ``libmgrit_b200.so``.

Kernel schedule of one cycle on a level with nu = 1:

  FC   interval k: F-relax from C-point k (interior writes elided), then
       C-relax into the ping buffer cbuf[k+1]           (mgrit.py:231-233)
  FR   interval k: F-relax from cbuf[k], then the injected residual
       r_{k+1} = g + Phi u_{(k+1)m-1} - cbuf[k+1] -> coarse rhs  (:234-237)
  ...  coarse solve: recursive cycle or one-CTA forward substitution (:239-244)
  CF   interval k: u_C[k] = cbuf[k] + e[k], F-relax writing all F-points,
       then (fine level) the residual of the next norm      (:246-247, :270)

Skipping interior F-point writes in FC/FR is exact: only u_{km+m-1} is read
before the closing F-relaxation rewrites every F-point (verified
bitwise on the reference).

Opening F-relaxation of iterations >= 2 (fine level): the closing F-relaxation
of iteration k (CF pass, mgrit.py:247) leaves u_{km+j} = Phi^j u_{km}; the
opening F-relaxation of iteration k+1 (mgrit.py:231) recomputes exactly those
values from the same C-points with the same kernel, so the solve loop replaces
it by a read of the stored u_{km+m-1}: the first FC (nu = 0: FR) pass is then
one C-step (residual step) per interval instead of m steps.  Bitwise the same
iterate and history (``ELIDE_OPENING_F_RELAX = False`` runs the full pass;
tests/test_gpu_parity.py compares both).

Closing residual step = next opening C-relaxation (fine level, nu >= 1): the
fused norm of the CF pass evaluates r_{k+1} = (g + Phi u_{km+m-1}) - u_{(k+1)m}; its
first term is exactly the value c_relax (mgrit.py:148-149) computes at the start of
the next cycle from the same stored F-point.  The CF pass stores it (``z_out`` of
``mgb_relax_args``) and the next cycle starts from it: iterations >= 2 run the
fine level in exactly two sweeps (FR and CF).  ``REUSE_CLOSING_STEP = False``
recomputes it.

First interval of a coarse level (nu >= 1): the error at t = 0 is zero, so on
levels >= 1 interval 0 starts from the same zero C-point in the FC, FR and CF
passes of a cycle (mgrit.py:231-247): the FR pass recomputes the FC pass's
F-points and gets r_1 = (g + Phi u_{m-1}) - (Phi u_{m-1} + g) = 0 exactly, the
child level then returns e_1 = 0, and the CF pass recomputes the same F-points
once more.  The FC pass therefore writes its F-points, the FR / CF passes run on
intervals 1.. only and r_1 is set to zero -- on a single-interval level (cfg4's
level 3) two of the three passes disappear, and a 16-interval level (cfg4's
level 2) fits one wave of clusters.  Bitwise the same iterate and history
(``ELIDE_FIRST_INTERVAL = False`` recomputes).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _native
from .device import device_sum, is_tensor, plan_for, ptr, require_cuda, stream_handle, to_device

nat_load, nat_check = _native.load, _native.check
#: tests: fill the rows ``MgritSolver._upload`` does not copy with NaN
POISON_SKIPPED_ROWS = False
#: iterations >= 2 of ``solve`` read the F-points the previous closing F-relaxation left
#: instead of recomputing them (module docstring); False: recompute like the reference
ELIDE_OPENING_F_RELAX = True
#: fine level: the residual step that closes a cycle (the fused norm of the CF pass) computes
#: g + Phi u_{km+m-1}, which IS the C-relaxation the next cycle opens with: the CF pass stores
#: it and the next cycle skips its first FC pass altogether (module docstring); False: the
#: next cycle recomputes it with one C-step per interval
REUSE_CLOSING_STEP = True
#: coarse levels: the first interval starts from e_0 = 0 in every pass, so its FR and CF
#: work repeats the FC pass bit for bit (module docstring); False: recompute
ELIDE_FIRST_INTERVAL = True
from .stepping import Stepper

_F64 = 8


@dataclass
class MgritConfig:
    """F(CF)^nu pre-relaxation, cycle type, halting (mgrit.py:28-44)."""

    nu: int = 1
    cycle: str = "two_level"
    tol: float = 1e-10
    max_iters: int = 30
    rng_seed: int = 0

    def __post_init__(self):
        if self.nu < 0:
            raise ValueError(f"nu must be >= 0, got {self.nu}")
        # "f_cycle" is an extension (the reference has two_level | v_cycle,
        # mgrit.py:41-42; BASELINE cfg5 names an F-cycle)
        if self.cycle not in ("two_level", "v_cycle", "f_cycle"):
            raise ValueError(f"unknown cycle {self.cycle!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclass
class TimeGridProblem:
    """Per-level steppers, coarsening factors and u0 (mgrit.py:47-93)."""

    steppers: List[Stepper]
    m: List[int]
    n_t: int
    u0: np.ndarray

    def __post_init__(self):
        self.u0 = np.asarray(self.u0, dtype=float)
        if len(self.steppers) != len(self.m) + 1:
            raise ValueError("need one stepper per level: "
                             f"{len(self.steppers)} steppers, {len(self.m)} factors")
        n = self.n_t
        for lvl, mf in enumerate(self.m):
            if mf < 2:
                raise ValueError(f"coarsening factor must be >= 2, got {mf}")
            if n % mf != 0:
                raise ValueError(f"level {lvl} has {n} steps, not divisible by m = {mf}")
            n //= mf
        if n < 1:
            raise ValueError("coarsest level must keep at least one step")
        if any(s.n_x != len(self.u0) for s in self.steppers):
            raise ValueError("stepper mesh sizes must match the initial condition")

    @property
    def n_levels(self) -> int:
        return len(self.steppers)

    @property
    def n_x(self) -> int:
        return len(self.u0)

    def points_on_level(self, level: int) -> int:
        n = self.n_t
        for mf in self.m[:level]:
            n //= mf
        return n + 1


@dataclass
class SolveReport:
    """Residual history and effective convergence factor (mgrit.py:96-110)."""

    residual_norms: List[float]
    iterations: int
    effective_rho: float
    converged: bool
    wall_time: float = 0.0

    @property
    def total_reduction(self) -> float:
        if self.residual_norms[0] == 0.0:
            return 0.0
        return self.residual_norms[-1] / self.residual_norms[0]


def initial_condition(n_x: int) -> np.ndarray:
    """sin^4(pi x) on [-1, 1) (mgrit.py:294-297)."""
    x = -1.0 + 2.0 * np.arange(n_x) / n_x
    return np.sin(np.pi * x) ** 4


# ------------------------------------------------------- drop-in primitives

def _writeback(host, dev):
    """Copy the device result back into the caller's host array (numpy or a
    CPU tensor), preserving the reference's in-place mutation semantics."""
    if host is None:
        return
    if isinstance(host, np.ndarray):
        host[...] = dev.cpu().numpy().reshape(host.shape)
    else:
        host.copy_(dev.reshape(host.shape))


def f_relax(u, g, stepper: Stepper, m: int, pool=None, threads: int = 1) -> None:
    """F-relaxation in place (mgrit.py:132-142); numpy or CUDA tensors."""
    ud, uh = to_device(u)
    gd, _ = to_device(g) if g is not None else (None, None)
    n = ud.shape[-1]
    N = ud.shape[0]
    plan = plan_for(stepper.program)
    full, rem = (N - 1) // m, (N - 1) % m
    plan.relax(full, m, m - 1, c_src=ptr(ud), c_stride=m * n, u=ptr(ud), write_f=2, g=ptr(gd))
    if rem:
        off = full * m * n * _F64
        plan.relax(1, m, rem, c_src=ptr(ud) + off, c_stride=0, u=ptr(ud) + off, write_f=2,
                   g=None if gd is None else ptr(gd) + off)
    _writeback(uh, ud)


def c_relax(u, g, stepper: Stepper, m: int, pool=None, threads: int = 1) -> None:
    """C-relaxation in place (mgrit.py:145-149)."""
    ud, uh = to_device(u)
    gd, _ = to_device(g) if g is not None else (None, None)
    n = ud.shape[-1]
    cnt = (ud.shape[0] - 1) // m
    plan_for(stepper.program).relax(cnt, m, 0, c_src=ptr(ud) + (m - 1) * n * _F64,
                                    c_stride=m * n, tail=1, tail_out=ptr(ud) + m * n * _F64,
                                    tail_stride=m * n, g=ptr(gd))
    _writeback(uh, ud)


def _residual(ud, gd, stepper, m, out=None, partials=None):
    n = ud.shape[-1]
    cnt = (ud.shape[0] - 1) // m
    plan_for(stepper.program).relax(cnt, m, 0, c_src=ptr(ud) + (m - 1) * n * _F64,
                                    c_stride=m * n, tail=2, cref=ptr(ud) + m * n * _F64,
                                    cref_stride=m * n, tail_out=ptr(out),
                                    tail_stride=n, g=ptr(gd), partials=ptr(partials))
    return cnt


def restrict_residual(u, g, stepper: Stepper, m: int, pool=None, threads: int = 1):
    """Coarse-point residuals g_km + Phi u_{km-1} - u_km, k >= 1 (mgrit.py:152-161)."""
    torch = require_cuda()
    ud, uh = to_device(u)
    gd, _ = to_device(g) if g is not None else (None, None)
    cnt = (ud.shape[0] - 1) // m
    r = torch.empty((cnt, ud.shape[-1]), dtype=torch.float64, device=ud.device)
    _residual(ud, gd, stepper, m, out=r)
    return r.cpu().numpy() if uh is not None else r


def cpoint_residual_norm(u, g, stepper: Stepper, m: int, pool=None, threads: int = 1) -> float:
    """Global l2 norm of the C-point residuals (mgrit.py:164-166)."""
    torch = require_cuda()
    ud, _ = to_device(u)
    gd, _ = to_device(g) if g is not None else (None, None)
    cnt = (ud.shape[0] - 1) // m
    part = torch.empty(max(cnt, 1), dtype=torch.float64, device=ud.device)
    tot = torch.empty(1, dtype=torch.float64, device=ud.device)
    _residual(ud, gd, stepper, m, partials=part)
    device_sum(ptr(part), cnt, ptr(tot))
    return math.sqrt(float(tot.item()))


def _forward_substitute_dev(plan, out, g, n_pts: int, start=None):
    """u_0 = start (or g_0), u_k = Phi u_{k-1} + g_k on one CTA (mgrit.py:169-191)."""
    plan.relax(1, n_pts, n_pts - 1, c_src=start if start is not None else g, c_stride=0,
               c_out=out, c_out_stride=0, u=out, write_f=2, g=g)


def sequential_solve(problem: TimeGridProblem, level: int = 0, g=None):
    """Exact forward substitution on ``level`` (mgrit.py:169-183)."""
    torch = require_cuda()
    n_pts = problem.points_on_level(level)
    out = torch.empty((n_pts, problem.n_x), dtype=torch.float64, device="cuda")
    plan = plan_for(problem.steppers[level].program)
    if g is None:
        u0 = torch.from_numpy(np.ascontiguousarray(problem.u0)).to("cuda")
        _forward_substitute_dev(plan, ptr(out), None, n_pts, start=ptr(u0))
        torch.cuda.synchronize()
        return out.cpu().numpy()
    gd, gh = to_device(g)
    _forward_substitute_dev(plan, ptr(out), ptr(gd), n_pts)
    return out.cpu().numpy() if gh is not None else out


# ----------------------------------------------------------------- solver

class _Level:
    def __init__(self, torch, stepper: Stepper, m: int, n_pts: int, n_x: int, nu: int,
                 tag=None):
        self.plan = plan_for(stepper.program, tag)
        self.m = m
        self.n_pts = n_pts
        self.n_int = (n_pts - 1) // m
        shape = (self.n_int + 1, n_x)
        self.cbuf = [torch.empty(shape, dtype=torch.float64, device="cuda")
                     for _ in range(min(nu, 2))]


class MgritSolver:
    """Level hierarchy, HBM buffers and the GPU cycle (mgrit.py:194-285)."""

    def __init__(self, problem: TimeGridProblem, config: MgritConfig, threads: int = 1):
        self.problem = problem
        self.config = config
        self.threads = max(1, int(threads))
        self._built = False
        #: set to a list to record (name, start_event, end_event) per launch
        self.profile = None
        #: plan tag: solvers that run concurrently (solve_many) get private plans
        self.plan_tag = None
        #: REUSE_CLOSING_STEP needs per-cycle buffer swaps (not for CUDA-graph replays)
        self._use_z = True
        self._z_valid = False

    # ---------------------------------------------------------- buffers
    def _build(self):
        if self._built:
            return
        torch = require_cuda()
        pr, cfg = self.problem, self.config
        n_x = pr.n_x
        self._torch = torch
        nlev = len(pr.m)
        self.levels = [_Level(torch, pr.steppers[l], pr.m[l], pr.points_on_level(l), n_x,
                              cfg.nu, self.plan_tag) for l in range(nlev)]
        # coarse iterates e_l and right-hand sides g_l for levels 1..nlev
        self.ucoarse = [None]
        self.gcoarse = [None]
        for l in range(1, nlev + 1):
            npts = pr.points_on_level(l)
            self.ucoarse.append(torch.zeros((npts, n_x), dtype=torch.float64, device="cuda"))
            self.gcoarse.append(torch.zeros((npts, n_x), dtype=torch.float64, device="cuda"))
        self.plans = [plan_for(s.program, self.plan_tag) for s in pr.steppers]
        #: gcoarse[l][1] (r_1 of level l - 1) still holds its zeros (ELIDE_FIRST_INTERVAL)
        self._r1_zero = [True] * (nlev + 2)
        self.zero_row = torch.zeros(n_x, dtype=torch.float64, device="cuda")
        n0 = self.levels[0].n_int
        self.partials = torch.empty(max(n0, 1), dtype=torch.float64, device="cuda")
        self.sumbuf = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.sumbuf0 = torch.zeros(1, dtype=torch.float64, device="cuda")
        self._built = True

    # ---------------------------------------------------------- iteration
    def initial_state(self) -> np.ndarray:
        """U[0,1) iterate from default_rng(rng_seed), row 0 := u0 (mgrit.py:206-211)."""
        rng = np.random.default_rng(self.config.rng_seed)
        u = rng.random((self.problem.n_t + 1, self.problem.n_x))
        u[0] = self.problem.u0
        return u

    def rhs(self) -> np.ndarray:
        g = np.zeros((self.problem.n_t + 1, self.problem.n_x))
        g[0] = self.problem.u0
        return g

    def _timed(self, name: str, fn, *args, **kw):
        if self.profile is None:
            return fn(*args, **kw)
        torch = self._torch
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = fn(*args, **kw)
        e.record()
        self.profile.append((name, s, e))
        return out

    def profile_summary(self) -> dict:
        """{pass name: (launches, total ms)} of the recorded launches."""
        self._torch.cuda.synchronize()
        out = {}
        for name, s, e in self.profile or []:
            cnt, ms = out.get(name, (0, 0.0))
            out[name] = (cnt + 1, ms + s.elapsed_time(e))
        return out

    def _cycle(self, l: int, u: int, g: Optional[int], u_zero: bool, want_norm: bool,
               kind: Optional[str] = None, pre_cf=None, f_relaxed: bool = False) -> None:
        """One cycle on level ``l``.  ``f_relaxed``: the F-points of ``u`` are the
        F-relaxation of its C-points (the state a previous cycle's CF pass left),
        so the opening F-relaxation reads u_{km+m-1} instead of recomputing it."""
        cfg = self.config
        kind = kind or cfg.cycle
        L = self.levels[l]
        n = self.problem.n_x
        m, nI, plan = L.m, L.n_int, L.plan
        row = n * _F64
        zero = ptr(self.zero_row)
        u0row = zero if u_zero else u
        src, stride = (None if u_zero else u), m * n
        f_relaxed = f_relaxed and not u_zero and ELIDE_OPENING_F_RELAX
        # coarse levels: interval 0 repeats the FC pass in FR and CF (module docstring)
        skip0 = ELIDE_FIRST_INTERVAL and l >= 1 and cfg.nu >= 1
        k0 = 1 if skip0 else 0
        for i in range(cfg.nu):
            dst = L.cbuf[i % 2]
            if i == 0 and f_relaxed and l == 0 and self._z_valid:
                # the previous cycle's closing residual step left these C-relaxed values
                L.cbuf[0], L.zbuf = L.zbuf, L.cbuf[0]
                dst = L.cbuf[0]
                self._z_valid = False
            elif i == 0 and f_relaxed:  # C-step from the stored last F-point of every interval
                self._timed(f"L{l}.FC", plan.relax, nI, m, 0, c_src=u + (m - 1) * row,
                            c_stride=m * n, tail=1, tail_out=ptr(dst) + row, tail_stride=n, g=g)
            elif i == 0 and skip0 and u_zero:  # interval 0's F-points are final: written here
                self._timed(f"L{l}.FC", plan.relax, nI, m, m - 1, c_src=src, c_stride=stride,
                            c_src0=u0row, tail=1, tail_out=ptr(dst) + row, tail_stride=n, g=g,
                            u=u, write_f=2)
            else:
                self._timed(f"L{l}.FC", plan.relax, nI, m, m - 1, c_src=src, c_stride=stride,
                            c_src0=u0row, tail=1, tail_out=ptr(dst) + row, tail_stride=n, g=g)
            src, stride = ptr(dst), n
        gC = self.gcoarse[l + 1]
        uC = self.ucoarse[l + 1]
        if cfg.nu == 0:
            cref, cref_stride = (zero, 0) if u_zero else (u + m * row, m * n)
        else:
            cref, cref_stride = src + row, n
        g_k0 = None if g is None else g + k0 * m * row
        if cfg.nu == 0 and f_relaxed:  # residual step from the stored last F-points
            self._r1_zero[l + 1] = False
            self._timed(f"L{l}.FR", plan.relax, nI, m, 0, c_src=u + (m - 1) * row, c_stride=m * n,
                        tail=2, cref=cref, cref_stride=cref_stride,
                        tail_out=ptr(gC) + row, tail_stride=n, g=g)
        elif skip0:
            if not self._r1_zero[l + 1]:  # r_1 = 0 exactly: the row is zero from allocation on
                gC[1].zero_()             # unless a full FR pass of this solver wrote it
                self._r1_zero[l + 1] = True
            if nI > 1:
                self._timed(f"L{l}.FR", plan.relax, nI - 1, m, m - 1, k_global0=1,
                            c_src=src + stride * _F64, c_stride=stride, tail=2,
                            cref=cref + cref_stride * _F64, cref_stride=cref_stride,
                            tail_out=ptr(gC) + 2 * row, tail_stride=n, g=g_k0)
        else:
            self._r1_zero[l + 1] = False
            self._timed(f"L{l}.FR", plan.relax, nI, m, m - 1, c_src=src, c_stride=stride,
                        c_src0=u0row, tail=2, cref=cref, cref_stride=cref_stride,
                        tail_out=ptr(gC) + row, tail_stride=n, g=g)
        self._coarse_solve(l + 1, kind)
        if pre_cf is not None:  # last reader of the incoming F-points (solve's initial norm)
            pre_cf()
        fuse_norm = want_norm and cfg.nu > 0
        if cfg.nu == 0:
            c_src, c_stride = (None if u_zero else u), m * n
        else:
            c_src, c_stride = src, n
        if skip0:
            if nI > 1:
                self._timed(f"L{l}.CF", plan.relax, nI - 1, m, m - 1, k_global0=1,
                            c_src=c_src + c_stride * _F64, c_stride=c_stride,
                            e=ptr(uC) + row, e_stride=n, c_out=u + m * row, c_out_stride=m * n,
                            c_last_out=u + nI * m * row, u=u + m * row, write_f=2, g=g_k0)
            else:  # the level's last C-point: C-relaxed value + correction (mgrit.py:246)
                torch = self._torch
                torch.add(L.cbuf[(cfg.nu - 1) % 2][1], uC[1], out=self.ucoarse[l][m])
        else:
            zkw = {}
            if (l == 0 and fuse_norm and self._use_z and REUSE_CLOSING_STEP and ELIDE_OPENING_F_RELAX
                    and plan.prog.kind in ("stencil", "rk", "callable")):
                if getattr(L, "zbuf", None) is None:
                    L.zbuf = self._torch.empty_like(L.cbuf[0])
                zkw = dict(z_out=ptr(L.zbuf) + row, z_stride=n)
                self._z_valid = True
            self._timed(f"L{l}.CF", plan.relax, nI, m, m - 1, c_src=c_src, c_stride=c_stride,
                        c_src0=u0row, e=ptr(uC),
                        e_stride=n, c_out=u, c_out_stride=m * n, c_last_out=u + nI * m * row,
                        u=u, write_f=2, g=g,
                        tail=2 if fuse_norm else 0, cref=(c_src + row) if fuse_norm else None,
                        cref_stride=n, cref_e=ptr(uC) + row, cref_e_stride=n,
                        partials=ptr(self.partials) if fuse_norm else None, **zkw)
        if want_norm and not fuse_norm:
            self._timed("L0.R", self._residual_partials, u, g)

    def _coarse_solve(self, child: int, kind: Optional[str] = None) -> None:
        """Solve level ``child`` for e = ucoarse[child] given g = gcoarse[child]:
        forward substitution (two-level / coarsest) or a recursive cycle from
        e = 0 (mgrit.py:239-244).  F-cycle (extension): an F-cycle on the child
        from e = 0 followed by one V-cycle on the child from that result (the
        multigrid F-cycle: the W-cycle with its second recursive call replaced
        by a V-cycle); on two-level hierarchies it equals the V-cycle."""
        kind = kind or self.config.cycle
        uC, gC = self.ucoarse[child], self.gcoarse[child]
        if kind == "two_level" or child == len(self.levels):
            self._timed(f"L{child}.seq", _forward_substitute_dev, self.plans[child], ptr(uC),
                        ptr(gC), self.problem.points_on_level(child))
        elif kind == "f_cycle":
            self._cycle(child, ptr(uC), ptr(gC), True, False, "f_cycle")
            # the V-cycle starts from the F-cycle's result, whose F-points its CF pass relaxed
            self._cycle(child, ptr(uC), ptr(gC), False, False, "v_cycle", f_relaxed=True)
        else:
            self._cycle(child, ptr(uC), ptr(gC), True, False, "v_cycle")

    def _residual_partials(self, u: int, g: Optional[int]) -> None:
        L = self.levels[0]
        n = self.problem.n_x
        m = L.m
        L.plan.relax(L.n_int, m, 0, c_src=u + (m - 1) * n * _F64, c_stride=m * n, tail=2,
                     cref=u + m * n * _F64, cref_stride=m * n, g=g, partials=ptr(self.partials))

    def _norm(self, buf=None) -> float:
        buf = self.sumbuf if buf is None else buf
        self._timed("norm", device_sum, ptr(self.partials), self.levels[0].n_int, ptr(buf))
        return math.sqrt(float(buf.item()))

    def _initial_norm_deferred(self, ev):
        """pre_cf hook of the first cycle when the rows before the C-points are
        still in flight (``_upload(split=True)``): wait for them, then the
        initial residual partials and their sum into ``sumbuf0`` -- before the
        CF pass rewrites the F-points and reuses the partials buffer."""
        torch = self._torch
        torch.cuda.current_stream().wait_event(ev)
        self._timed("L0.R", self._residual_partials, ptr(self._u_dev), None)
        self._timed("norm", device_sum, ptr(self.partials), self.levels[0].n_int,
                    ptr(self.sumbuf0))

    def iterate(self, u, g=None):
        """One MGRIT cycle in place; returns the updated iterate (mgrit.py:218-223)."""
        self._build()
        ud, uh = to_device(u)
        gd = None
        if g is not None:
            gd, _ = to_device(g)
        self._cycle(0, ptr(ud), ptr(gd), False, False)
        if uh is not None:
            _writeback(uh, ud)
            return u
        return ud

    # -------------------------------------------------------------- solve
    def solve(self, u=None) -> SolveReport:
        """Run to the halting rule (mgrit.py:251-285); divergence is reported."""
        self._build()
        torch = self._torch
        cfg = self.config
        internal = u is None
        if internal:
            u = self.initial_state()
        ud, uh, pending = self._upload(u, split=True)
        up = ptr(ud)
        self._z_valid = False
        hook = None
        if pending is None:
            torch.cuda.synchronize()
            start = time.perf_counter()
            self._timed("L0.R", self._residual_partials, up, None)
            norms = [self._norm()]
        else:
            # the C-points have landed; the rows before them are still in
            # flight on the copy stream and are first read by the initial
            # residual, which runs inside the first cycle before its CF pass
            torch.cuda.current_stream().synchronize()
            start = time.perf_counter()
            self._u_dev = ud
            hook = lambda: self._initial_norm_deferred(pending)  # noqa: E731
            norms = []
        converged = False
        it = 0
        while it < cfg.max_iters:
            self._cycle(0, up, None, False, True, pre_cf=hook, f_relaxed=it > 0)
            it += 1
            if hook is not None:
                hook = None
                self._u_dev = None
                norms.append(math.sqrt(float(self.sumbuf0.item())))
            norms.append(self._norm())
            if norms[0] > 0 and norms[-1] / norms[0] <= cfg.tol:
                converged = True
                break
        torch.cuda.synchronize()
        wall = time.perf_counter() - start
        self.last_iterate = ud
        if uh is not None and not internal:  # in-place semantics for a caller's array
            _writeback(uh, ud)
        rho = norms[-1] / norms[-2] if len(norms) >= 2 and norms[-2] > 0 else 0.0
        return SolveReport(norms, it, float(rho), converged, wall)

    def _upload(self, u, split: bool = False):
        """Device copy of a host iterate for ``solve``: only the rows the solve
        reads before rewriting them -- the C-points u[km] and the rows
        u[km-1] before them (initial residual, mgrit.py:164-166 / 259-261; the
        first FC pass reads the C-points) -- travel, as two strided DMAs.  The
        first closing F-relaxation (mgrit.py:247; the fused CF pass) rewrites
        every F-point before any is read, so the other rows of the initial
        iterate cannot influence the result (tests/test_gpu_parity.py checks
        host and device inputs give bitwise identical solves, with the
        skipped rows poisoned).  CUDA tensors are used in place.

        Returns ``(device iterate, caller's array, pending)``.  With ``split``
        and a pinned host tensor the rows before the C-points travel on a
        side copy stream and ``pending`` is the CUDA event that marks their
        arrival (the caller makes its stream wait on it before the first
        read); otherwise ``pending`` is None and both copies are ordered on
        the current stream."""
        torch = self._torch
        pr = self.problem
        m = pr.m[0] if pr.m else 0
        self.last_upload_bytes = 0
        if is_tensor(u) and u.is_cuda:
            return to_device(u) + (None,)
        if m < 3:
            self.last_upload_bytes = 8 * (pr.n_t + 1) * pr.n_x
            return to_device(u) + (None,)
        shape = (pr.n_t + 1, pr.n_x)
        if is_tensor(u):
            if u.dtype != torch.float64:
                raise TypeError("device arrays must be float64")
            src = u.contiguous().reshape(shape)
        else:
            arr = np.asarray(u)
            if np.iscomplexobj(arr):
                raise NotImplementedError("complex arrays are not supported on the device path")
            src = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).reshape(shape))
        ud = torch.empty(shape, dtype=torch.float64, device="cuda")
        if POISON_SKIPPED_ROWS:
            ud.fill_(float("nan"))
        row = pr.n_x * _F64
        n_int = pr.n_t // m
        h, d = src.data_ptr(), ud.data_ptr()
        lib, stream = nat_load(), stream_handle()
        pinned = is_tensor(u) and u.is_pinned()
        pending = None
        nat_check(lib.mgb_copy_rows(d, m * row, h, m * row, row, n_int + 1, stream))
        if split and pinned:
            cur = torch.cuda.current_stream()
            side = getattr(self, "_copy_stream", None)
            if side is None:
                side = self._copy_stream = torch.cuda.Stream()
            side.wait_stream(cur)  # ud's allocation / poison fill come first
            nat_check(lib.mgb_copy_rows(d + (m - 1) * row, m * row, h + (m - 1) * row, m * row,
                                        row, n_int, ctypes.c_void_p(side.cuda_stream)))
            pending = torch.cuda.Event()
            pending.record(side)
        else:
            nat_check(lib.mgb_copy_rows(d + (m - 1) * row, m * row, h + (m - 1) * row, m * row,
                                        row, n_int, stream))
        self.last_upload_bytes = (2 * n_int + 1) * row
        if not pinned:
            torch.cuda.current_stream().synchronize()  # pageable source: keep it alive
        return ud, u, pending


def solve(problem: TimeGridProblem, config: MgritConfig, threads: int = 1,
          initial_iterate=None) -> SolveReport:
    """Run MGRIT to the halting rule on the GPU (mgrit.py:288-291)."""
    return MgritSolver(problem, config, threads).solve(initial_iterate)


def solve_many(jobs, streams: Optional[int] = 8, graphs: bool = True,
               l2_budget: Optional[float] = None) -> List[SolveReport]:
    """Many independent solves in flight at once (the Table-3 /
    measured-point sweeps, experiments.py:150-242, are lists of small solves).

    ``jobs``: sequence of ``(problem, config)`` or ``(problem, config,
    initial_iterate)``.  Up to ``streams`` solves are active at a time, each on
    its own CUDA stream (slot) with private device plans and buffers, running
    exactly the kernel sequence of ``solve``: every report (and iterate) is
    bitwise identical to the sequential one.  Optionally a job is admitted to a
    free slot only while the active iterates fit ``l2_budget`` bytes (always
    when no other solve is active); measured on B200, concurrency beats L2
    residency even for 1024 x 4096 Table-3 cells, so there is no budget by
    default.  The host drives the active
    solves in lock step: it enqueues one cycle (plus the norm and an
    asynchronous read-back of the squared norm) for every active solve, then
    reads the norms in order and applies each solve's halting rule
    (mgrit.py:262-274).  With ``graphs`` a solve's cycle + norm + read-back is
    captured once as a CUDA graph and replayed per iteration (one launch
    instead of ~15 host calls: small solves are launch-bound).  ``wall_time``
    of a report is the time from the start of the batch to that solve's
    halting decision."""
    jobs = [tuple(j) for j in jobs]
    if not jobs:
        return []
    torch = require_cuda()
    ns = max(1, min(int(streams or len(jobs)), len(jobs)))
    pool = [torch.cuda.Stream() for _ in range(ns)]
    host = torch.zeros(len(jobs), dtype=torch.float64, pin_memory=True)
    st = []
    for job in jobs:
        problem = job[0]
        st.append(dict(problem=problem, config=job[1], init=job[2] if len(job) > 2 else None,
                       bytes=8.0 * (problem.n_t + 1) * problem.n_x, norms=[], it=0,
                       converged=False, ev=torch.cuda.Event(), wall=0.0, graph=None))

    def enqueue(k, first, f_relaxed=True):
        d = st[k]
        sol = d["sol"]
        if first:
            sol._residual_partials(d["up"], None)
        else:
            sol._cycle(0, d["up"], None, False, True, f_relaxed=f_relaxed)
        device_sum(ptr(sol.partials), sol.levels[0].n_int, ptr(sol.sumbuf))
        host[k:k + 1].copy_(sol.sumbuf, non_blocking=True)

    def start_job(k, slot):
        d = st[k]
        sol = MgritSolver(d["problem"], d["config"])
        sol.plan_tag = ("slot", slot)
        sol._use_z = False  # graph replays use fixed buffers
        d.update(sol=sol, slot=slot, stream=pool[slot])
        with torch.cuda.stream(pool[slot]):
            sol._build()
            u = sol.initial_state() if d["init"] is None else d["init"]
            d["ud"], d["uh"] = to_device(u)
            d["up"] = ptr(d["ud"])
            plans = [L.plan for L in sol.levels] + sol.plans
            # user callables (device.CallablePlan) run arbitrary torch code: not captured
            if graphs and not any(getattr(pl.prog, "kind", "") == "callable" for pl in plans):
                for plan in plans:
                    plan.reserve()
                g = torch.cuda.CUDAGraph()
                g.capture_begin(capture_error_mode="thread_local")
                try:
                    enqueue(k, False)
                finally:
                    g.capture_end()
                d["graph"] = g
            enqueue(k, True)
            d["ev"].record(pool[slot])

    def next_cycle(k):
        d = st[k]
        with torch.cuda.stream(d["stream"]):
            if d["it"] == 1:  # the first cycle starts from an arbitrary iterate: full opening pass
                enqueue(k, False, f_relaxed=False)
            elif d["graph"] is not None:
                d["graph"].replay()
            else:
                enqueue(k, False)
            d["ev"].record(d["stream"])

    def finish(d):
        d["sol"].last_iterate = d["ud"]
        if d["uh"] is not None:
            with torch.cuda.stream(d["stream"]):
                _writeback(d["uh"], d["ud"])
        d["graph"] = None

    torch.cuda.synchronize()
    start = time.perf_counter()
    pending = list(range(len(st)))
    active, free = [], list(range(ns))
    while pending or active:
        load = sum(st[k]["bytes"] for k in active)
        while pending and free and (not active or l2_budget is None
                                    or load + st[pending[0]]["bytes"] <= l2_budget):
            k = pending.pop(0)
            start_job(k, free.pop(0))
            active.append(k)
            load += st[k]["bytes"]
        nxt = []
        for k in active:
            d = st[k]
            d["ev"].synchronize()
            n = d["norms"]
            n.append(math.sqrt(float(host[k])))
            cfg = d["config"]
            if len(n) > 1 and n[0] > 0 and n[-1] / n[0] <= cfg.tol:
                d["converged"] = True
            if d["converged"] or d["it"] >= cfg.max_iters:
                d["wall"] = time.perf_counter() - start
                finish(d)
                free.append(d["slot"])
                continue
            d["it"] += 1
            next_cycle(k)
            nxt.append(k)
        active = nxt
    torch.cuda.synchronize()
    out = []
    for d in st:
        n = d["norms"]
        rho = n[-1] / n[-2] if len(n) >= 2 and n[-2] > 0 else 0.0
        out.append(SolveReport(n, d["it"], float(rho), d["converged"], d["wall"]))
    return out
