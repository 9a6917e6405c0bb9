"""The BASELINE.json configurations as concrete synthetic inputs.

u0 generators other than sin^4 are this project's own seeded definitions
(BASELINE.json names "seeded Fourier noise" and "sum of 8 sinusoids"; the
reference ships only sin^4, mgrit.py:294-297).  CFL numbers are read as the
absolute c (ERK5 diverges at 0.85 c_max).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .mgrit import initial_condition


def seeded_u0(kind: str, n_x: int) -> np.ndarray:
    x = -1.0 + 2.0 * np.arange(n_x) / n_x
    if kind == "sin4":
        return initial_condition(n_x)
    if kind == "sin4_noise":  # sin^4 + 1e-2 RMS-normalised Fourier noise, k <= 32
        rng = np.random.default_rng(2)
        a = rng.standard_normal(32)
        b = rng.standard_normal(32)
        k = np.arange(1, 33)
        noise = (np.cos(np.pi * np.multiply.outer(x, k)) @ a
                 + np.sin(np.pi * np.multiply.outer(x, k)) @ b)
        noise = 1e-2 * noise / math.sqrt(float(np.sum(a * a + b * b)) / 2.0)
        return initial_condition(n_x) + noise
    if kind == "sines8":  # (1/8) sum_k sin(pi k x + theta_k), random phases
        theta = np.random.default_rng(3).uniform(0.0, 2.0 * np.pi, 8)
        k = np.arange(1, 9)
        return np.sin(np.pi * np.multiply.outer(x, k) + theta[None, :]).sum(axis=1) / 8.0
    raise ValueError(f"unknown u0 kind {kind!r}")


@dataclass(frozen=True)
class BaselineConfig:
    name: str
    family: str
    p: int
    c: float
    n_x: int
    n_t: int
    m: int
    cycle: str
    coarse: str
    u0: str

    def spec(self):
        from .stepping import DiscretizationSpec
        return DiscretizationSpec(self.family, self.p, self.c, self.n_x, self.n_t)

    def problem(self):
        from .experiments import build_problem
        return build_problem(self.spec(), self.m, self.cycle, self.coarse,
                             u0=seeded_u0(self.u0, self.n_x))

    def as_v_cycle(self) -> "BaselineConfig":
        return BaselineConfig(self.name, self.family, self.p, self.c, self.n_x, self.n_t, self.m,
                              "v_cycle", self.coarse, self.u0)

    def scaled(self, n_x: int, n_t: int) -> "BaselineConfig":
        return BaselineConfig(self.name + f"@{n_x}x{n_t}", self.family, self.p, self.c, n_x,
                              n_t, self.m, self.cycle, self.coarse, self.u0)


CONFIGS = {
    "cfg1": BaselineConfig("cfg1", "erk", 1, 0.85, 1024, 1024, 8, "two_level", "modified", "sin4"),
    "cfg2": BaselineConfig("cfg2", "erk", 3, 0.85, 4096, 16384, 8, "v_cycle", "modified",
                           "sin4_noise"),
    "cfg3": BaselineConfig("cfg3", "sdirk", 3, 4.0, 4096, 16384, 4, "v_cycle", "modified",
                           "sines8"),
    "cfg4": BaselineConfig("cfg4", "erk", 5, 0.85, 8192, 65536, 16, "v_cycle", "modified", "sin4"),
    # BASELINE names a multilevel F-cycle for cfg5 (the reference has only
    # two-level and V-cycles, so its parity runs use the V-cycle: ``as_v_cycle``)
    "cfg5": BaselineConfig("cfg5", "erk", 3, 0.85, 16384, 1 << 20, 8, "f_cycle", "modified",
                           "sin4_noise"),
}
