"""Command line for the B200 hot path: ``python -m paper_2209_06916_b200 solve|iters``.

Mirrors the reference's ``mgrit-advection`` driver (cli.py:391-427) for the two
subcommands that run MGRIT solves -- ``solve`` (one run with its residual
history, cli.py:281-299) and ``iters`` (two-level / V-cycle iteration counts,
cli.py:253-264) -- with the same INI configuration sections and keys
(cli.py:38-71), the same command-line overrides, the same CSV text (``%.8e``
floats, ``#`` metadata carrying the resolved configuration, cli.py:154-188)
and the same exit codes (0 ok, 1 configuration error, 2 numerical
singularity).  ``constants``, ``sweep`` and ``validate`` are analysis tooling
outside the time-parallel hot path and exit with status 1.
Extension: ``--cycle f`` (F-cycle).
"""

from __future__ import annotations

import argparse
import configparser
import io
import os
import sys
from dataclasses import dataclass, field, fields
from typing import List, Optional, Sequence

from . import experiments, mgrit
from .errors import SingularOperatorError
from .stepping import DiscretizationSpec, cfl_limit

CYCLES = {"two-level": "two_level", "v": "v_cycle", "f": "f_cycle"}
OUT_OF_SCOPE = ("constants", "sweep", "validate")


class ConfigError(ValueError):
    pass


# section -> keys, in the reference's order (cli.py:60-67)
_SECTIONS = (
    ("discretization", ("family", "p", "c", "c_fraction", "coarse")),
    ("mgrit", ("m", "nu", "cycle", "max_iters", "tol", "seed")),
    ("lfa", ("lfa_samples", "lfa_excluded")),
    ("grid", ("n_x", "n_t")),
    ("sweep", ("c_min", "c_max", "c_points", "measure")),
    ("run", ("threads", "out")),
)
_STR_KEYS = ("family", "coarse", "cycle", "out")
_FLOAT_KEYS = ("tol", "c", "c_fraction", "c_min", "c_max")


@dataclass
class ExperimentConfig:
    family: str = "erk"
    p: int = 3
    c: float = 0.0
    c_fraction: float = 0.0
    coarse: str = "modified"
    m: List[int] = field(default_factory=lambda: [2])
    nu: int = 1
    cycle: str = "two_level"
    max_iters: int = 30
    tol: float = 1e-10
    seed: int = 0
    n_x: int = 256
    n_t: int = 1024
    lfa_samples: int = 2 ** 11
    lfa_excluded: int = -1
    c_min: float = 0.0
    c_max: float = 0.0
    c_points: int = 512
    measure: bool = False
    threads: int = 0
    out: str = ""

    def validate(self) -> "ExperimentConfig":
        checks = (
            (self.family in ("erk", "sdirk"), f"unknown family {self.family!r}"),
            (1 <= self.p <= 5, f"order p must be in 1..5, got {self.p}"),
            (self.coarse in experiments.COARSE_KINDS,
             f"unknown coarse operator kind {self.coarse!r}"),
            (not (self.family == "erk" and self.coarse == "rediscretized"),
             "rediscretized coarse operators are unavailable for explicit fine grids: at m "
             "times the step they exceed the stability limit and the coarse operator is "
             "unstable"),
            (all(v >= 2 for v in self.m), f"coarsening factors must be >= 2, got {self.m}"),
            (self.cycle in CYCLES.values(), f"unknown cycle {self.cycle!r}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)
        return self

    def resolve_c(self) -> float:
        """Absolute fine-grid CFL number (a fraction refers to c_max)."""
        if self.c_fraction > 0.0:
            return self.c_fraction * cfl_limit(self.p)
        if self.c > 0.0:
            return self.c
        raise ConfigError("set either c or c_fraction")

    def to_text(self) -> str:
        cp = configparser.ConfigParser()
        for section, keys in _SECTIONS:
            cp[section] = {k: (",".join(map(str, v)) if isinstance(v, list) else str(v))
                           for k in keys for v in (getattr(self, k),)}
        buf = io.StringIO()
        cp.write(buf)
        return buf.getvalue()

    @classmethod
    def from_text(cls, text: str) -> "ExperimentConfig":
        cp = configparser.ConfigParser()
        try:
            cp.read_string(text)
        except configparser.Error as exc:
            raise ConfigError(f"cannot parse config: {exc}") from exc
        allowed = dict(_SECTIONS)
        values = {}
        for section in cp.sections():
            if section not in allowed:
                raise ConfigError(f"unknown config section [{section}]")
            for key, raw in cp[section].items():
                if key not in allowed[section]:
                    raise ConfigError(f"unknown key {key!r} in [{section}]")
                values[key] = _parse_value(key, raw.strip())
        return cls(**values).validate()


def _parse_value(key: str, raw: str):
    if key == "m":
        return [int(tok) for tok in raw.split(",") if tok]
    if key in _STR_KEYS:
        return raw
    if key == "measure":
        return raw.lower() in ("1", "true", "yes", "on")
    return float(raw) if key in _FLOAT_KEYS else int(raw)


def _cell(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        if v != v:
            return "nan"
        if v in (float("inf"), float("-inf")):
            return "inf" if v > 0 else "-inf"
        return f"{v:.8e}"
    return str(v)


def emit_csv(path: Optional[str], header: Sequence[str], rows, metadata: Sequence[str]) -> str:
    """'#'-prefixed metadata, a header line, comma-separated rows."""
    text = "".join(f"# {line}\n" for line in metadata)
    text += ",".join(header) + "\n"
    text += "".join(",".join(_cell(v) for v in row) + "\n" for row in rows)
    if path:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return text


def _meta(config: ExperimentConfig, command: str) -> List[str]:
    return [f"command: {command}"] + [ln for ln in config.to_text().splitlines() if ln.strip()]


def run_solve(config: ExperimentConfig) -> int:
    spec = DiscretizationSpec(config.family, config.p, config.resolve_c(), config.n_x, config.n_t)
    m = config.m[0] if config.cycle == "two_level" else config.m
    problem = experiments.build_problem(spec, m, config.cycle, config.coarse)
    report = mgrit.solve(problem, mgrit.MgritConfig(nu=config.nu, cycle=config.cycle,
                                                    tol=config.tol, max_iters=config.max_iters,
                                                    rng_seed=config.seed),
                         threads=config.threads)
    meta = _meta(config, "solve") + [
        f"converged: {report.converged}",
        f"iterations: {report.iterations}",
        f"effective_rho: {report.effective_rho:.8e}",
        f"wall_time_seconds: {report.wall_time:.6f}",
        f"threads: {config.threads}",
    ]
    emit_csv(config.out or None, ("iteration", "residual_norm"),
             list(enumerate(report.residual_norms)), meta)
    return 0


def run_iters(config: ExperimentConfig) -> int:
    cells = experiments.iteration_table(config.family, config.p, config.resolve_c(),
                                        [(config.n_x, config.n_t)], config.m, config.coarse,
                                        nu=config.nu, max_iters=config.max_iters,
                                        rng_seed=config.seed, threads=config.threads)
    emit_csv(config.out or None, ("n_x", "n_t", "m", "iters_two_level", "iters_v_cycle"),
             [(c.n_x, c.n_t, c.m, c.iters_two_level, c.iters_v_cycle) for c in cells],
             _meta(config, "iters"))
    return 0


RUNNERS = {"solve": run_solve, "iters": run_iters}


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2209_06916_b200",
                                 description="MGRIT for 1-D linear advection on B200 GPUs")
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("constants", "sweep", "iters", "validate", "solve"):
        sp = sub.add_parser(name)
        sp.add_argument("--config")
        sp.add_argument("--out")
        sp.add_argument("--threads", type=int)
        sp.add_argument("--seed", type=int)
        sp.add_argument("--measure", action="store_true", default=None)
        sp.add_argument("--cycle", choices=sorted(CYCLES))
        sp.add_argument("--nu", type=int)
        sp.add_argument("--m")
        sp.add_argument("--grid")
        sp.add_argument("--family", choices=["erk", "sdirk"])
        sp.add_argument("--p", type=int)
        sp.add_argument("--c", type=float)
        sp.add_argument("--c-fraction", type=float)
        sp.add_argument("--coarse", choices=list(experiments.COARSE_KINDS))
        sp.add_argument("--c-range")
        sp.add_argument("--max-iters", type=int)
    return ap


def _override(config: ExperimentConfig, a) -> ExperimentConfig:
    simple = {"out": a.out, "threads": a.threads, "seed": a.seed, "nu": a.nu, "family": a.family,
              "p": a.p, "c": a.c, "c_fraction": a.c_fraction, "coarse": a.coarse,
              "max_iters": a.max_iters}
    for key, val in simple.items():
        if val is not None:
            setattr(config, key, val)
    if a.measure:
        config.measure = True
    if a.cycle is not None:
        config.cycle = CYCLES[a.cycle]
    if a.m is not None:
        config.m = [int(tok) for tok in a.m.split(",") if tok]
    if a.grid is not None:
        parts = a.grid.split(",")
        if len(parts) != 2 or not all(p.strip().lstrip("-").isdigit() for p in parts):
            raise ConfigError(f"--grid expects NX,NT, got {a.grid!r}")
        config.n_x, config.n_t = int(parts[0]), int(parts[1])
    if a.c_range is not None:
        parts = a.c_range.split(",")
        try:
            config.c_min, config.c_max, config.c_points = float(parts[0]), float(parts[1]), int(parts[2])
        except (ValueError, IndexError) as exc:
            raise ConfigError(f"--c-range expects CMIN,CMAX,NPOINTS, got {a.c_range!r}") from exc
    return config


def main(argv: Optional[Sequence[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.command in OUT_OF_SCOPE:
            raise ConfigError(f"'{args.command}' is analysis tooling outside the B200 hot path; "
                              "use the reference package (mgrit-advection) for it")
        if args.config:
            with open(args.config, "r", encoding="utf-8") as fh:
                config = ExperimentConfig.from_text(fh.read())
        else:
            config = ExperimentConfig()
        config = _override(config, args)
        if config.threads <= 0:
            config.threads = os.cpu_count() or 1
        config.validate()
        return RUNNERS[args.command](config)
    except ConfigError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 1
    except SingularOperatorError as exc:
        print(f"numerical singularity: {exc}", file=sys.stderr)
        return 2
