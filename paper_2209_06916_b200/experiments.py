"""Hierarchy assembly and solver policy (drop-in for experiments.py:26-104, 190-242).

The study suites of the reference (error-constant tables, LFA sweeps,
validation rows) are analysis tooling outside the time-parallel hot path and
are not part of this package ("Out of scope").
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import mgrit, stepping
from .stepping import (ButcherTableau, DiscretizationSpec, Stepper, ideal_coarse_stepper,
                       modified_coarse_stepper, mol_stepper, plain_sl_coarse_stepper,
                       rediscretized_coarse_stepper)

#: GMRES policy for the implicit correction on multilevel explicit runs
GMRES_TOL = 1e-2
GMRES_MAX_ITERS = {1: 10}

COARSE_KINDS = ("modified", "rediscretized", "plain_sl", "ideal")


def gmres_cap(p: int) -> int:
    return GMRES_MAX_ITERS.get(p, 20)


def fine_stepper(spec: DiscretizationSpec, tab: Optional[ButcherTableau] = None) -> Stepper:
    if spec.family == "semi_lagrangian":
        return stepping.sl_stepper(spec.p, spec.c, spec.n_x).stepper
    return mol_stepper(spec, tab)


def coarse_stepper(kind: str, spec: DiscretizationSpec, m: int, level: int, fine: Stepper,
                   solver: str = "direct", tab: Optional[ButcherTableau] = None,
                   cumulative_factor: Optional[int] = None) -> Stepper:
    """experiments.py:44-66."""
    if kind == "modified":
        return modified_coarse_stepper(spec, m, level, solver=solver, gmres_tol=GMRES_TOL,
                                       gmres_max_iters=gmres_cap(spec.p), tab=tab,
                                       cumulative_factor=cumulative_factor)
    if kind == "rediscretized":
        if level != 1:
            raise ValueError("rediscretized coarse operators are two-level only")
        return rediscretized_coarse_stepper(spec, m, tab)
    if kind == "plain_sl":
        if cumulative_factor is not None:
            return stepping.sl_stepper(spec.p, cumulative_factor * spec.c, spec.n_x,
                                       level=level).stepper
        return plain_sl_coarse_stepper(spec, m, level)
    if kind == "ideal":
        if level != 1:
            raise ValueError("the ideal coarse operator is two-level only")
        return ideal_coarse_stepper(fine, m)
    raise ValueError(f"unknown coarse kind {kind!r}")


def level_factors(n_t: int, m, cycle: str, coarse_kind: str) -> List[int]:
    """Per-level coarsening factors (experiments.py:80-93)."""
    m_list = [m] if np.isscalar(m) else list(m)
    if cycle == "two_level" or coarse_kind in ("ideal", "rediscretized"):
        return m_list[:1]
    # v_cycle and (extension) f_cycle share the multilevel hierarchy
    factors: List[int] = []
    n = n_t
    while True:
        mf = m_list[min(len(factors), len(m_list) - 1)]
        if n % mf != 0 or n // mf < 1:
            break
        factors.append(mf)
        n //= mf
    return factors


def build_problem(spec: DiscretizationSpec, m, cycle: str, coarse_kind: str = "modified",
                  tab: Optional[ButcherTableau] = None,
                  u0: Optional[np.ndarray] = None) -> mgrit.TimeGridProblem:
    """Level hierarchy for one MGRIT run (experiments.py:69-104).

    GMRES corrections iff family=erk, cycle=v_cycle and kind=modified.
    ``u0`` (extension) overrides the sin^4 initial profile.
    """
    fine = fine_stepper(spec, tab)
    factors = level_factors(spec.n_t, m, cycle, coarse_kind)
    solver = "gmres" if (spec.family == "erk" and cycle in ("v_cycle", "f_cycle")
                         and coarse_kind == "modified") else "direct"
    steppers = [fine]
    cumulative = 1
    for level, mf in enumerate(factors, start=1):
        cumulative *= mf
        steppers.append(coarse_stepper(coarse_kind, spec, mf, level, fine, solver=solver,
                                       tab=tab, cumulative_factor=cumulative))
    if u0 is None:
        u0 = mgrit.initial_condition(spec.n_x)
    return mgrit.TimeGridProblem(steppers, factors, spec.n_t, u0)


def measured_point(family: str, p: int, coarse_kind: str, c: float, m: int, n_x: int,
                   n_t: int, config: Optional[mgrit.MgritConfig] = None,
                   cycle: str = "two_level", threads: int = 1) -> mgrit.SolveReport:
    """One GPU MGRIT run returning its report (experiments.py:190-201)."""
    config = config or mgrit.MgritConfig()
    if config.cycle != cycle:
        config = mgrit.MgritConfig(config.nu, cycle, config.tol, config.max_iters,
                                   config.rng_seed)
    spec = DiscretizationSpec(family, p, c, n_x, n_t)
    return mgrit.solve(build_problem(spec, m, cycle, coarse_kind), config, threads=threads)


@dataclass
class IterationCell:
    n_x: int
    n_t: int
    m: int
    iters_two_level: str
    iters_v_cycle: str
    report_two_level: mgrit.SolveReport = field(repr=False, default=None)
    report_v_cycle: mgrit.SolveReport = field(repr=False, default=None)


def iteration_table(family: str, p: int, c: float, grids: Sequence[tuple],
                    m_values: Sequence[int], coarse_kind: str = "modified", nu: int = 1,
                    max_iters: int = 40, rng_seed: int = 0,
                    threads: int = 1, concurrent: bool = False,
                    streams: Optional[int] = 8) -> List[IterationCell]:
    """Two-level and V-cycle iteration counts (experiments.py:221-242), on the GPU.

    ``concurrent=True`` (extension) runs every cell's solves at once through
    ``mgrit.solve_many`` (one CUDA stream per solve); the reports are bitwise
    identical to the sequential ones."""
    keys, jobs = [], []
    for n_x, n_t in grids:
        for m in m_values:
            spec = DiscretizationSpec(family, p, c, n_x, n_t)
            for cycle in ("two_level", "v_cycle"):
                cfg = mgrit.MgritConfig(nu=nu, cycle=cycle, tol=1e-10, max_iters=max_iters,
                                        rng_seed=rng_seed)
                keys.append((n_x, n_t, m, cycle))
                jobs.append((build_problem(spec, m, cycle, coarse_kind), cfg))
    if concurrent:
        reports = mgrit.solve_many(jobs, streams=streams)
    else:
        reports = [mgrit.solve(pr, cfg, threads=threads) for pr, cfg in jobs]
    by = dict(zip(keys, reports))
    fmt = lambda r: str(r.iterations) if r.converged else f">{max_iters}"
    cells = []
    for n_x, n_t in grids:
        for m in m_values:
            two, v = by[(n_x, n_t, m, "two_level")], by[(n_x, n_t, m, "v_cycle")]
            cells.append(IterationCell(n_x, n_t, m, fmt(two), fmt(v), two, v))
    return cells


def measured_points(family: str, p: int, coarse_kind: str, c_values: Sequence[float], m: int,
                    n_x: int, n_t: int, config: Optional[mgrit.MgritConfig] = None,
                    cycle: str = "two_level", streams: Optional[int] = 8) -> List[mgrit.SolveReport]:
    """``measured_point`` for many CFL numbers at once (the measured curve of
    experiments.py:150-201, lfa_sweep(measure_grid=...)), solved concurrently
    through ``mgrit.solve_many``; each report equals ``measured_point``'s."""
    config = config or mgrit.MgritConfig()
    if config.cycle != cycle:
        config = mgrit.MgritConfig(config.nu, cycle, config.tol, config.max_iters,
                                   config.rng_seed)
    jobs = [(build_problem(DiscretizationSpec(family, p, c, n_x, n_t), m, cycle, coarse_kind),
             config) for c in c_values]
    return mgrit.solve_many(jobs, streams=streams)
