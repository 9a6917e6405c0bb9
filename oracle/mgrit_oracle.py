"""CPU oracle for the MGRIT hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module is a numpy restatement of the reference package ``mgrit-advection``
0.1.0 (``/root/reference/pkg/src/mgrit_advection``).  It exists only so that
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl
reference`` legs of ``bench.py`` have a checker and a CPU baseline on the GPU
box, where ``/root/reference`` is absent.  The product package
``paper_2209_06916_b200`` never imports it.

Parity pin: every function below follows the reference's numpy operation order
(same reductions, same mul-then-add order, same FFT calls), and
``tests/test_oracle_golden.py`` checks it against fixtures produced by running
the real reference (``tests/golden/make_golden.py``): stencil weights bitwise,
f-relaxation bitwise, GMRES outputs and full residual histories.

References are ``file:line`` relative to ``/root/reference/pkg/src/mgrit_advection``.
"""

from __future__ import annotations

import math
import time
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, List, Optional, Sequence

import numpy as np

# circulant.py:18-26, stepping.py:26-35
PRUNE_TOL = 1e-15
SINGULAR_TOL = 1e-14
ROLL_LIMIT = 16          # settable: cfg4 parity runs use 64
STEPPER_PRUNE_TOL = 1e-14
STABILITY_TOL = 1e-6
DOMAIN_LENGTH = 2.0
GMRES_TOL = 1e-2         # experiments.py:26-27
GMRES_CAPS = {1: 10}     # experiments.py:28, 33-34


class OracleSingular(ArithmeticError):
    pass


# ============================================================== circulants

def canonical_stencil(n, offsets, weights):
    """circulant.py:29-44 -- reduce offsets to [-(n//2), n - n//2), merge in
    input order, prune |w| <= 1e-15, sort by offset."""
    merged = {}
    for off, w in zip(offsets, weights):
        k = int(off) % n
        if k >= n - n // 2:
            k -= n
        merged[k] = merged.get(k, 0.0) + w
    kept = sorted((k, w) for k, w in merged.items() if abs(w) > PRUNE_TOL)
    if not kept:
        kept = [(0, 0.0)]
    offs = np.array([k for k, _ in kept], dtype=np.int64)
    wts = np.array([w for _, w in kept])
    if np.iscomplexobj(wts) and np.max(np.abs(wts.imag)) == 0.0:
        wts = wts.real
    return offs, wts


class Circ:
    """Periodic stencil operator (circulant.py:47-240), immutable by convention."""

    def __init__(self, n, offsets, weights):
        self.n = int(n)
        self.offsets, self.weights = canonical_stencil(self.n, offsets, weights)
        self._eig = None

    # circulant.py:81-83
    @classmethod
    def identity(cls, n):
        return cls(n, [0], [1.0])

    # circulant.py:85-102
    @classmethod
    def from_symbol_values(cls, n, lam, prune=PRUNE_TOL):
        lam = np.asarray(lam, dtype=complex)
        row = np.fft.fft(lam) / n
        if np.max(np.abs(row.imag)) < 1e-12 * max(1.0, np.max(np.abs(row))):
            row = row.real
        keep = np.abs(row) > prune
        return cls(n, np.nonzero(keep)[0], row[keep])

    def is_real(self):
        return not np.iscomplexobj(self.weights)

    # circulant.py:113-124 (rolled path :119-123, FFT path :126-131)
    def apply(self, v):
        v = np.asarray(v)
        if v.shape[-1] != self.n:
            raise ValueError(f"length {v.shape[-1]} != n {self.n}")
        if len(self.offsets) <= ROLL_LIMIT:
            acc = np.zeros(v.shape, dtype=np.result_type(v, self.weights))
            for off, w in zip(self.offsets, self.weights):
                acc += w * np.roll(v, -int(off), axis=-1)
            return acc
        lam = self.eig()
        if self.is_real() and not np.iscomplexobj(v):
            return np.fft.irfft(np.fft.rfft(v, axis=-1) * lam[: self.n // 2 + 1],
                                n=self.n, axis=-1)
        return np.fft.ifft(np.fft.fft(v, axis=-1) * lam, axis=-1)

    # circulant.py:133-143
    def symbol(self, omega):
        om = np.asarray(omega, dtype=float)
        ph = np.exp(1j * np.multiply.outer(om, self.offsets.astype(float)))
        out = ph @ self.weights.astype(complex)
        return complex(out) if np.isscalar(omega) else out

    # circulant.py:145-154
    def eig(self):
        if self._eig is None:
            self._eig = self.symbol(2.0 * np.pi * np.arange(self.n) / self.n)
        return self._eig

    # circulant.py:168-173, 175-181, 183-184
    def compose(self, other):
        offs = (self.offsets[:, None] + other.offsets[None, :]).ravel()
        wts = (self.weights[:, None] * other.weights[None, :]).ravel()
        return Circ(self.n, offs, wts)

    def plus(self, other):
        offs = np.concatenate([self.offsets, other.offsets])
        wts = np.concatenate([
            self.weights.astype(np.result_type(self.weights, other.weights)),
            other.weights])
        return Circ(self.n, offs, wts)

    def scaled(self, s):
        return Circ(self.n, self.offsets, s * self.weights)

    def minus(self, other):
        return self.plus(other.scaled(-1.0))

    def power(self, m):
        out, base = Circ.identity(self.n), self
        while m:
            if m & 1:
                out = out.compose(base)
            base = base.compose(base) if m > 1 else base
            m >>= 1
        return out

    def dense(self):
        M = np.zeros((self.n, self.n), dtype=self.weights.dtype)
        for off, w in zip(self.offsets, self.weights):
            for i in range(self.n):
                M[i, (i + int(off)) % self.n] += w
        return M

    # circulant.py:222-238
    def solve_direct(self, b):
        b = np.asarray(b)
        lam = self.eig()
        bad = np.abs(lam) < SINGULAR_TOL
        if np.any(bad):
            raise OracleSingular(f"singular at mode {int(np.argmax(bad))}")
        if self.is_real() and not np.iscomplexobj(b):
            return np.fft.irfft(np.fft.rfft(b, axis=-1) / lam[: self.n // 2 + 1],
                                n=self.n, axis=-1)
        return np.fft.ifft(np.fft.fft(b, axis=-1) / lam, axis=-1)


def _dot_rows_reordered(a, b, block=256):
    """Blocked, reversed-order row dot products (SURVEY Appendix A self-noise)."""
    prod = a * b
    n = prod.shape[-1]
    out = np.zeros(prod.shape[0])
    for start in reversed(range(0, n, block)):
        out += prod[:, start:start + block][:, ::-1].sum(axis=-1)
    return out


def gmres_rows(op, B, tol, cap, reduction="reference", stats=None):
    """Per-row unrestarted GMRES(x0 = 0), circulant.py:262-332.

    ``reduction="reordered"`` swaps every dot product / norm for a blocked,
    reversed-order sum: the oracle's self-noise calibration run (SURVEY 0.6,
    8c).  Returns (X, relative residuals, columns used, breakdown flag);
    ``stats`` (a dict, optional) receives the per-row depth and residual.
    """
    if reduction == "reference":
        rowdot = lambda a, b: np.einsum("kn,kn->k", a, b)          # :297
        rownorm = lambda a: np.linalg.norm(a, axis=-1)              # :274, :300
    else:
        rowdot = _dot_rows_reordered
        rownorm = lambda a: np.sqrt(_dot_rows_reordered(a, a))
    K, n = B.shape
    cap = min(cap, n)
    beta = rownorm(B)
    live = beta > 0.0
    X = np.zeros_like(B)
    if not np.any(live):
        if stats is not None:
            stats.update(depth=np.zeros(K, dtype=int), res=np.zeros(K))
        return X, np.zeros(K), 0, False
    V = np.zeros((K, cap + 1, n))
    H = np.zeros((K, cap + 1, cap))
    cs = np.zeros((K, cap))
    sn = np.zeros((K, cap))
    g = np.zeros((K, cap + 1))
    g[:, 0] = beta
    V[live, 0] = B[live] / beta[live, None]
    res = np.where(live, 1.0, 0.0)
    active = live.copy()
    used = np.zeros(K, dtype=int)
    broke = False
    j = 0
    while j < cap and np.any(active):
        w = op.apply(V[:, j, :])
        for i in range(j + 1):                                       # MGS :295-299
            h = rowdot(w, V[:, i, :])
            H[:, i, j] = np.where(active, h, H[:, i, j])
            w -= np.where(active, h, 0.0)[:, None] * V[:, i, :]
        hn = rownorm(w)
        happy = active & (hn <= 1e-14 * beta)
        broke = broke or bool(np.any(happy))
        H[:, j + 1, j] = np.where(active, hn, 0.0)
        safe = np.where(hn > 0.0, hn, 1.0)
        V[:, j + 1, :] = np.where(active[:, None], w / safe[:, None], V[:, j + 1, :])
        for i in range(j):                                           # Givens :308-312
            t = cs[:, i] * H[:, i, j] + sn[:, i] * H[:, i + 1, j]
            H[:, i + 1, j] = -sn[:, i] * H[:, i, j] + cs[:, i] * H[:, i + 1, j]
            H[:, i, j] = t
        den = np.hypot(H[:, j, j], H[:, j + 1, j])                    # :313-319
        den = np.where(den > 0.0, den, 1.0)
        cs[:, j] = H[:, j, j] / den
        sn[:, j] = H[:, j + 1, j] / den
        H[:, j, j] = cs[:, j] * H[:, j, j] + sn[:, j] * H[:, j + 1, j]
        H[:, j + 1, j] = 0.0
        g[:, j + 1] = np.where(active, -sn[:, j] * g[:, j], g[:, j + 1])
        g[:, j] = np.where(active, cs[:, j] * g[:, j], g[:, j])
        res = np.where(active, np.abs(g[:, j + 1]) / np.where(beta > 0, beta, 1.0), res)
        used[active] = j + 1
        j += 1
        active = active & (res > tol) & ~happy
    for k in range(K):                                               # :326-331
        jk = int(used[k])
        if jk:
            y = np.linalg.solve(H[k, :jk, :jk], g[k, :jk])
            X[k] = y @ V[k, :jk, :]
    if stats is not None:
        stats.update(depth=used.copy(), res=res.copy())
    return X, res, j, broke


# ================================================================ stencils

def fd_weights(d, offsets, x0=0.0):
    """stencils.py:20-40: moment conditions sum_j w_j o_j^k = d^d/dz^d z^k at x0."""
    o = np.asarray(offsets, dtype=float)
    n = len(o)
    vand = np.vander(o, n, increasing=True).T
    rhs = np.zeros(n)
    for k in range(d, n):
        rhs[k] = (math.factorial(k) // math.factorial(k - d)) * x0 ** (k - d)
    return np.linalg.solve(vand, rhs)


def upwind_window(p):
    """stencils.py:73-78 -> (ell, r)."""
    ell = (p + 1) // 2 if p % 2 == 1 else p // 2 + 1
    return ell, p - ell


def interp_window(p, eps):
    """stencils.py:80-89."""
    if p % 2 == 1:
        return (p + 1) // 2, (p - 1) // 2
    return (p // 2 + 1, p // 2 - 1) if eps > 0.5 else (p // 2, p // 2)


def window_offsets(win):
    return np.arange(-win[0], win[1] + 1)


def upwind_op(p, n):
    """stencils.py:92-98."""
    win = upwind_window(p)
    return Circ(n, window_offsets(win), fd_weights(1, window_offsets(win), 0.0))


def fd_error_constant(p):
    """stencils.py:101-109."""
    ell, r = upwind_window(p)
    return (-1) ** r * math.factorial(ell) * math.factorial(r) / math.factorial(p + 1)


def high_derivative_op(d, s, bias, n):
    """stencils.py:112-138."""
    win = (d // 2, d // 2) if bias == "symmetric" else (d // 2 + 1, d - (d // 2 + 1))
    offs = window_offsets(win)
    return Circ(n, offs, fd_weights(d, offs, 0.0))


def interp_error_poly(p, win, z):
    """stencils.py:141-152."""
    acc = 1.0
    for j in range(-win[0], win[1] + 1):
        acc *= j + z
    return acc / math.factorial(p + 1)


def lagrange(win, eps):
    """stencils.py:155-162."""
    return fd_weights(0, window_offsets(win), -eps)


# ================================================================ tableaux

class Tableau:
    def __init__(self, A, b, kind, q, name):
        self.A = np.atleast_2d(np.asarray(A, dtype=float))
        self.b = np.asarray(b, dtype=float)
        self.kind, self.q, self.name = kind, q, name

    @property
    def stages(self):
        return len(self.b)

    def taylor(self, j):
        """stepping.py:79-85."""
        if j == 0:
            return 1.0
        return float(self.b @ np.linalg.matrix_power(self.A, j - 1) @ np.ones(self.stages))


def erk(q):
    """stepping.py:108-134."""
    if q == 1:
        return Tableau(np.zeros((1, 1)), [1.0], "explicit", 1, "ERK1")
    A = np.zeros((q if q < 5 else 6,) * 2)
    if q == 2:
        A[1, 0] = 1.0
        return Tableau(A, [0.5, 0.5], "explicit", 2, "ERK2")
    if q == 3:
        A[1, 0] = 0.5
        A[2, 0], A[2, 1] = -1.0, 2.0
        return Tableau(A, np.array([1, 4, 1]) / 6.0, "explicit", 3, "ERK3")
    if q == 4:
        A[1, 0] = A[2, 1] = 0.5
        A[3, 2] = 1.0
        return Tableau(A, np.array([1, 2, 2, 1]) / 6.0, "explicit", 4, "ERK4")
    if q == 5:
        A[1, 0] = 1 / 4
        A[2, 0], A[2, 1] = 1 / 8, 1 / 8
        A[3, 2] = 1 / 2
        A[4, 0], A[4, 1], A[4, 2], A[4, 3] = 3 / 16, -3 / 8, 3 / 8, 9 / 16
        A[5, 0], A[5, 1], A[5, 2], A[5, 3], A[5, 4] = -3 / 7, 8 / 7, 6 / 7, -12 / 7, 8 / 7
        return Tableau(A, np.array([7, 0, 32, 12, 32, 7]) / 90.0, "explicit", 5, "ERK5")
    raise ValueError(q)


def sdirk(q):
    """stepping.py:137-176 (SDIRK5 chain weights :88-105)."""
    if q == 1:
        return Tableau([[1.0]], [1.0], "sdirk", 1, "SDIRK1")
    if q == 2:
        g = 1.0 - 1.0 / math.sqrt(2.0)
        return Tableau([[g, 0.0], [1.0 - g, g]], [1.0 - g, g], "sdirk", 2, "SDIRK2")
    if q == 3:
        g = 0.435866521508458999416019
        b1 = -1.5 * g * g + 4.0 * g - 0.25
        b2 = 1.5 * g * g - 5.0 * g + 1.25
        return Tableau([[g, 0.0, 0.0], [(1.0 - g) / 2.0, g, 0.0], [b1, b2, g]],
                       [b1, b2, g], "sdirk", 3, "SDIRK3")
    if q == 4:
        A = np.array([[1 / 4, 0, 0, 0, 0], [1 / 2, 1 / 4, 0, 0, 0],
                      [17 / 50, -1 / 25, 1 / 4, 0, 0],
                      [371 / 1360, -137 / 2720, 15 / 544, 1 / 4, 0],
                      [25 / 24, -49 / 48, 125 / 16, -85 / 12, 1 / 4]])
        return Tableau(A, A[-1].copy(), "sdirk", 4, "SDIRK4")
    if q == 5:
        g = 4024571134387 / 14474071345096
        nodes = [g, 0.45, 0.65, 0.85, 1.0]
        s = len(nodes)
        A = np.diag([g] * s)
        for i in range(1, s):
            A[i, i - 1] = nodes[i] - g
        M = np.empty((s, s))
        v = np.ones(s)
        for j in range(s):
            M[:, j] = v
            v = A @ v
        b = np.linalg.solve(M.T, np.array([1.0 / math.factorial(j + 1) for j in range(s)]))
        return Tableau(A, b, "sdirk", 5, "SDIRK5")
    raise ValueError(q)


def tableau_for(family, q):
    return erk(q) if family == "erk" else sdirk(q)


def rk_error_constant(tab):
    """stepping.py:187-199 (order check elided: shipped tableaux only)."""
    return tab.taylor(tab.q + 1) - 1.0 / math.factorial(tab.q + 1)


def stability(tab, z):
    """stepping.py:202-219."""
    za = np.asarray(z, dtype=complex)
    flat = za.reshape(-1)
    s = tab.stages
    if tab.kind == "sdirk" and np.any(np.abs(1.0 - tab.A[0, 0] * flat) < 1e-14):
        raise OracleSingular("stability pole")
    M = np.eye(s)[None, :, :] - flat[:, None, None] * tab.A[None, :, :]
    st = np.linalg.solve(M, np.ones((len(flat), s, 1)))[:, :, 0]
    out = 1.0 + flat * (st @ tab.b)
    return complex(out[0]) if np.isscalar(z) else out.reshape(za.shape)


_CMAX = {}


def cfl_max(p, tab=None, n_samples=4096, tol=1e-6):
    """stepping.py:425-460 (bisection on max |R(-c L_p)| <= 1 + 1e-6)."""
    tab = tab or erk(p)
    key = (p, tab.A.tobytes(), tab.b.tobytes(), n_samples, tol)
    if key in _CMAX:
        return _CMAX[key]
    offs = window_offsets(upwind_window(p))
    w = fd_weights(1, offs, 0.0)
    om = -np.pi + 2.0 * np.pi * np.arange(n_samples) / n_samples
    Ls = np.exp(1j * np.outer(om, offs.astype(float))) @ w.astype(complex)
    ok = lambda c: np.max(np.abs(stability(tab, -c * Ls))) <= 1.0 + STABILITY_TOL
    lo, hi = 1e-8, 1.0
    while ok(hi):
        lo, hi = hi, 2.0 * hi
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if ok(mid) else (lo, mid)
    _CMAX[key] = 0.5 * (lo + hi)
    return _CMAX[key]


# ================================================================ steppers

class Step:
    """One-step map Phi with an assembled stencil and an optional apply closure
    (stepping.py:266-309)."""

    def __init__(self, n, op, symbol_fn, apply_fn=None, kind="assembled",
                 level=0, mult=1.0, info=None):
        self.n, self.op, self.symbol_fn, self.apply_fn = n, op, symbol_fn, apply_fn
        self.kind, self.level, self.mult = kind, level, mult
        self.info = info or {}

    def apply(self, u):
        if self.apply_fn is not None:
            return self.apply_fn(np.asarray(u))
        return self.op.apply(u)

    def symbol(self, om):
        return self.symbol_fn(np.asarray(om, dtype=float))


def _assemble(n, symbol_fn):
    """stepping.py:312-314."""
    return Circ.from_symbol_values(n, symbol_fn(2.0 * np.pi * np.arange(n) / n),
                                   STEPPER_PRUNE_TOL)


def mol_step(family, p, c, n, q=None, tab=None, mode="assembled"):
    """stepping.py:317-352 and the staged sweep :355-380."""
    tab = tab or tableau_for(family, q or p)
    L = upwind_op(p, n)
    sym = lambda om: stability(tab, -c * L.symbol(om))
    op = _assemble(n, sym)
    apply_fn = None
    info = {"tab": tab, "c": c, "L": L}
    if mode == "staged":
        cL = L.scaled(-c)
        M = None
        if tab.kind == "sdirk":
            M = Circ.identity(n).minus(cL.scaled(tab.A[0, 0]))
        info.update(cL=cL, stage_matrix=M)

        def apply_fn(u):
            z = []
            for i in range(tab.stages):
                rhs = u.copy()
                for j in range(i):
                    if tab.A[i, j] != 0.0:
                        rhs = rhs + tab.A[i, j] * z[j]
                z.append(cL.apply(rhs if M is None else M.solve_direct(rhs)))
            out = u.copy()
            for i in range(tab.stages):
                if tab.b[i] != 0.0:
                    out = out + tab.b[i] * z[i]
            return out
    return Step(n, op, sym, apply_fn, kind=mode, info=info)


def sl_step(p, mc, n, level=0):
    """stepping.py:390-419 -> (Step, eps, shift, window)."""
    k = int(math.floor(mc + 1e-13))
    eps = mc - k
    if eps < 1e-13:
        eps = 0.0
    win = interp_window(p, eps)
    w = lagrange(win, eps)
    offs = window_offsets(win) - k
    op = Circ(n, offs, w)
    offs_f = offs.astype(float)
    sym = lambda om: np.exp(1j * np.multiply.outer(om, offs_f)) @ w.astype(complex)
    return Step(n, op, sym, kind="assembled", level=level, mult=mc,
                info={"eps": eps, "shift": -k}), eps, -k, win


def phi_value(p, c, m, level, e_fd, e_rk):
    """stepping.py:465-492."""
    def sl_term(mc):
        k = int(math.floor(mc + 1e-13))
        eps = mc - k
        if eps < 1e-13:
            eps = 0.0
        return interp_error_poly(p, interp_window(p, eps), eps)

    phi = m * (c * e_fd + (-c) ** (p + 1) * e_rk) + (-1) ** (p + 1) * sl_term(m * c)
    for lvl in range(2, level + 1):
        phi = (-1) ** (p + 1) * (-m * sl_term(m ** (lvl - 1) * c)
                                 + sl_term(m ** lvl * c)) + m * phi
    return phi


def correction_D(p, n):
    """stepping.py:495-501."""
    if p % 2 == 1:
        return high_derivative_op(p + 1, 2, "symmetric", n)
    return high_derivative_op(p + 1, 1, "left_biased", n)


def corrected_coarse(family, p, c, n, m, level=1, solver="direct", tol=GMRES_TOL,
                     cap=20, q=None, tab=None, cumulative=None, reduction="reference"):
    """stepping.py:504-568."""
    tab = tab or tableau_for(family, q or p)
    e_fd, e_rk = fd_error_constant(p), rk_error_constant(tab)
    if cumulative is None:
        phi, mc = phi_value(p, c, m, level, e_fd, e_rk), m ** level * c
    else:
        phi, mc = phi_value(p, c, cumulative, 1, e_fd, e_rk), cumulative * c
    sl = sl_step(p, mc, n, level)[0]
    D = correction_D(p, n)
    corr = Circ.identity(n).minus(D.scaled(phi))
    if np.any(np.abs(corr.eig()) < 1e-14):
        raise OracleSingular("correction singular")
    sym = lambda om: sl.symbol(om) / (1.0 - phi * D.symbol(om))
    op = _assemble(n, sym)
    apply_fn = None
    if solver == "gmres":
        def apply_fn(u):
            rhs = sl.op.apply(u)
            x = gmres_rows(corr, rhs.reshape(-1, n), tol, cap, reduction)[0]
            return x.reshape(rhs.shape)
    return Step(n, op, sym, apply_fn, kind="implicit_correction", level=level,
                mult=mc, info={"phi": phi, "sl": sl, "D": D, "corr": corr,
                               "solver": solver, "tol": tol, "cap": cap})


def rediscretized_coarse(family, p, c, n, m, q=None, tab=None):
    """stepping.py:571-586 (explicit families rejected, :578-580)."""
    if family != "sdirk":
        raise ValueError("rediscretized coarse steppers require an sdirk family")
    st = mol_step(family, p, m * c, n, q=q, tab=tab)
    st.level, st.mult = 1, float(m)
    return st


def ideal_coarse(fine, m):
    """stepping.py:589-598."""
    sym = lambda om: fine.symbol(om) ** m
    return Step(fine.n, _assemble(fine.n, sym), sym, level=1, mult=float(m))


def build_hierarchy(family, p, c, n_x, n_t, m, cycle, kind="modified", q=None,
                    fine_mode="assembled", reduction="reference"):
    """experiments.py:37-104 -> (steppers, factors, u0)."""
    tab = tableau_for(family, q or p)
    fine = mol_step(family, p, c, n_x, tab=tab, mode=fine_mode)
    ms = [m] if np.isscalar(m) else list(m)
    if cycle == "two_level" or kind in ("ideal", "rediscretized"):
        factors = ms[:1]
    else:
        factors, rem = [], n_t
        while True:
            mf = ms[min(len(factors), len(ms) - 1)]
            if rem % mf != 0 or rem // mf < 1:
                break
            factors.append(mf)
            rem //= mf
    solver = "gmres" if (family == "erk" and cycle in ("v_cycle", "f_cycle") and kind == "modified") \
        else "direct"
    steps, cum = [fine], 1
    for level, mf in enumerate(factors, start=1):
        cum *= mf
        if kind == "modified":
            steps.append(corrected_coarse(family, p, c, n_x, mf, level, solver,
                                          GMRES_TOL, GMRES_CAPS.get(p, 20), tab=tab,
                                          cumulative=cum, reduction=reduction))
        elif kind == "rediscretized":
            steps.append(rediscretized_coarse(family, p, c, n_x, mf, tab=tab))
        elif kind == "plain_sl":
            steps.append(sl_step(p, cum * c, n_x, level)[0])
        elif kind == "ideal":
            steps.append(ideal_coarse(fine, mf))
        else:
            raise ValueError(kind)
    return steps, factors, sin4(n_x)


# ================================================================== MGRIT

def sin4(n):
    """mgrit.py:294-297."""
    x = -1.0 + 2.0 * np.arange(n) / n
    return np.sin(np.pi * x) ** 4


def initial_iterate(seed, n_t, n_x, u0):
    """mgrit.py:206-211."""
    u = np.random.default_rng(seed).random((n_t + 1, n_x))
    u[0] = u0
    return u


def _apply_rows(step, block, pool=None, threads=1):
    """mgrit.py:113-129 (thread chunking is bitwise neutral)."""
    if pool is None or threads <= 1 or block.shape[0] < 2 * threads:
        return step.apply(block)
    out = np.empty_like(block)

    def work(idx):
        out[idx] = step.apply(block[idx])

    list(pool.map(work, [c for c in np.array_split(np.arange(block.shape[0]), threads)
                         if len(c)]))
    return out


def f_relax(u, g, step, m, pool=None, threads=1):
    """mgrit.py:132-142."""
    for j in range(1, m):
        dst = u[j::m]
        dst[...] = _apply_rows(step, u[j - 1::m][: dst.shape[0]], pool, threads) + g[j::m]


def c_relax(u, g, step, m, pool=None, threads=1):
    """mgrit.py:145-149."""
    upd = _apply_rows(step, u[m - 1::m], pool, threads)
    u[m::m] = upd[: u[m::m].shape[0]] + g[m::m]


def restrict(u, g, step, m, pool=None, threads=1):
    """mgrit.py:152-161."""
    prop = _apply_rows(step, u[m - 1::m], pool, threads)
    nc = u[m::m].shape[0]
    return g[m::m] + prop[:nc] - u[m::m]


def cpoint_norm(u, g, step, m, pool=None, threads=1):
    """mgrit.py:164-166."""
    return float(np.linalg.norm(restrict(u, g, step, m, pool, threads).ravel()))


def forward_substitute(step, g):
    """mgrit.py:186-191."""
    u = np.empty_like(g)
    u[0] = g[0]
    for k in range(1, g.shape[0]):
        u[k] = step.apply(u[k - 1]) + g[k]
    return u


def sequential(steps, factors, n_t, u0, level=0, g=None):
    """mgrit.py:169-183."""
    n_pts = n_t
    for mf in factors[:level]:
        n_pts //= mf
    n_pts += 1
    u = np.empty((n_pts, len(u0)))
    u[0] = u0 if g is None else g[0]
    for k in range(1, n_pts):
        u[k] = steps[level].apply(u[k - 1]) + (0.0 if g is None else g[k])
    return u


class Mgrit:
    """mgrit.py:194-285: F(CF)^nu relaxation, injection, two-level / V-cycle."""

    def __init__(self, steps, factors, n_t, u0, nu=1, cycle="two_level", tol=1e-10,
                 max_iters=30, seed=0, threads=1):
        self.steps, self.factors, self.n_t = steps, list(factors), n_t
        self.u0 = np.asarray(u0, dtype=float)
        self.nu, self.cycle, self.tol, self.max_iters, self.seed = nu, cycle, tol, max_iters, seed
        self.threads = max(1, int(threads))
        self.pool = None
        self.levels_visited = []

    def initial_state(self):
        return initial_iterate(self.seed, self.n_t, len(self.u0), self.u0)

    def rhs(self):
        g = np.zeros((self.n_t + 1, len(self.u0)))
        g[0] = self.u0
        return g

    def cycle_once(self, level, u, g, kind=None):
        """One cycle on ``level`` (mgrit.py:225-247).  ``kind="f_cycle"`` is the
        builder's extension (no reference counterpart, parity unpinned by the
        reference): the coarse problem is solved by an F-cycle from e = 0
        followed by one V-cycle from that result."""
        kind = kind or self.cycle
        step, m = self.steps[level], self.factors[level]
        pool, thr = self.pool, self.threads
        f_relax(u, g, step, m, pool, thr)
        for _ in range(self.nu):
            c_relax(u, g, step, m, pool, thr)
            f_relax(u, g, step, m, pool, thr)
        r = restrict(u, g, step, m, pool, thr)
        gc = np.vstack([np.zeros((1, len(self.u0))), r])
        if kind == "two_level" or level + 1 == len(self.factors):
            e = forward_substitute(self.steps[level + 1], gc)
        elif kind == "f_cycle":
            e = np.zeros_like(gc)
            self.cycle_once(level + 1, e, gc, "f_cycle")
            self.cycle_once(level + 1, e, gc, "v_cycle")
        else:
            e = np.zeros_like(gc)
            self.cycle_once(level + 1, e, gc, "v_cycle")
        u[m::m] += e[1:]
        f_relax(u, g, step, m, pool, thr)

    def solve(self, u=None, max_iters=None):
        """Returns dict(norms, iterations, rho, converged, wall, u).

        ``max_iters`` overrides the cap (bounded CPU-baseline samples)."""
        g = self.rhs()
        if u is None:
            u = self.initial_state()
        cap = self.max_iters if max_iters is None else max_iters
        step, m = self.steps[0], self.factors[0]
        t0 = time.perf_counter()
        if self.threads > 1:
            self.pool = ThreadPoolExecutor(max_workers=self.threads)
        try:
            norms = [cpoint_norm(u, g, step, m, self.pool, self.threads)]
            converged, it = False, 0
            while it < cap:
                self.cycle_once(0, u, g)
                it += 1
                norms.append(cpoint_norm(u, g, step, m, self.pool, self.threads))
                if norms[0] > 0 and norms[-1] / norms[0] <= self.tol:
                    converged = True
                    break
        finally:
            if self.pool is not None:
                self.pool.shutdown()
                self.pool = None
        wall = time.perf_counter() - t0
        rho = norms[-1] / norms[-2] if len(norms) >= 2 and norms[-2] > 0 else 0.0
        return dict(norms=norms, iterations=it, rho=float(rho), converged=converged,
                    wall=wall, u=u)


# ============================================== BASELINE configs

def seeded_u0(kind, n_x):
    """Builder-defined seeded u0 generators."""
    x = -1.0 + 2.0 * np.arange(n_x) / n_x
    if kind == "sin4":
        return sin4(n_x)
    if kind == "sin4_noise":
        rng = np.random.default_rng(2)
        a = rng.standard_normal(32)
        b = rng.standard_normal(32)
        k = np.arange(1, 33)
        N = (np.cos(np.pi * np.multiply.outer(x, k)) @ a
             + np.sin(np.pi * np.multiply.outer(x, k)) @ b)
        N = 1e-2 * N / math.sqrt(float(np.sum(a * a + b * b)) / 2.0)
        return sin4(n_x) + N
    if kind == "sines8":
        th = np.random.default_rng(3).uniform(0.0, 2.0 * np.pi, 8)
        k = np.arange(1, 9)
        return np.sin(np.pi * np.multiply.outer(x, k) + th[None, :]).sum(axis=1) / 8.0
    raise ValueError(kind)
