"""Periodic constant-coefficient operators (drop-in for circulant.py).

``CirculantOperator`` keeps the reference's immutable stencil representation
and its host-side algebra (canonical form, symbols, composition) because the
steppers are *assembled* from it during setup.  Everything that touches data
-- ``apply``, ``solve_direct``, ``solve_gmres`` -- runs on the B200 through
``libmgrit_b200.so``:

* ``apply``        -> generic / register-window stencil kernel; exact mode
                      reproduces the reference's rolled sums bit for bit
                      (circulant.py:119-123) for any tap count;
* ``solve_direct`` -> factorised periodic banded solve (circulant.py:222-238
                      solves by FFT; same operator, different rounding);
* ``solve_gmres``  -> the batched GMRES kernel (circulant.py:240-332).
"""

from __future__ import annotations

from typing import NamedTuple, Sequence, Tuple

import numpy as np

from .errors import DimensionMismatchError, SingularOperatorError

#: merged weights with |w| <= PRUNE_TOL are dropped (circulant.py:18-19)
PRUNE_TOL = 1e-15
#: |symbol| below this is a singular mode (circulant.py:21-22)
SINGULAR_TOL = 1e-14


def _canonical(n_x: int, offsets, weights):
    """Balanced offsets in [-(n//2), n - n//2), duplicates merged in input
    order, pruned, sorted (circulant.py:29-44)."""
    merged = {}
    upper = n_x - n_x // 2
    for off, w in zip(offsets, weights):
        k = int(off) % n_x
        if k >= upper:
            k -= n_x
        merged[k] = merged.get(k, 0.0) + w
    pairs = sorted((k, w) for k, w in merged.items() if abs(w) > PRUNE_TOL) or [(0, 0.0)]
    offs = np.array([k for k, _ in pairs], dtype=np.int64)
    wts = np.array([w for _, w in pairs])
    if np.iscomplexobj(wts) and np.max(np.abs(wts.imag)) == 0.0:
        wts = wts.real
    return offs, wts


class CirculantOperator:
    """Immutable periodic stencil; data-touching methods run on the GPU."""

    __slots__ = ("n_x", "offsets", "weights", "_eig", "_prog")

    def __init__(self, n_x: int, stencil: Sequence[Tuple[int, float]]):
        if n_x < 1:
            raise ValueError(f"n_x must be positive, got {n_x}")
        offs, wts = _canonical(n_x, [o for o, _ in stencil], [w for _, w in stencil])
        object.__setattr__(self, "n_x", int(n_x))
        object.__setattr__(self, "offsets", offs)
        object.__setattr__(self, "weights", wts)
        object.__setattr__(self, "_eig", None)
        object.__setattr__(self, "_prog", None)
        offs.setflags(write=False)
        wts.setflags(write=False)

    def __setattr__(self, name, value):
        raise AttributeError("CirculantOperator is immutable")

    # ------------------------------------------------------------ builders
    @classmethod
    def from_arrays(cls, n_x: int, offsets, weights) -> "CirculantOperator":
        return cls(n_x, list(zip(offsets, weights)))

    @classmethod
    def identity(cls, n_x: int) -> "CirculantOperator":
        return cls(n_x, [(0, 1.0)])

    @classmethod
    def shift(cls, n_x: int, k: int) -> "CirculantOperator":
        return cls(n_x, [(k, 1.0)])

    @classmethod
    def from_eigenvalues(cls, n_x: int, eigenvalues, prune_tol: float = PRUNE_TOL):
        """Stencil with the given symbol values at 2 pi k / n_x (circulant.py:85-102)."""
        lam = np.asarray(eigenvalues, dtype=complex)
        if lam.shape != (n_x,):
            raise DimensionMismatchError(f"need {n_x} eigenvalues, got shape {lam.shape}")
        first_row = np.fft.fft(lam) / n_x
        if np.max(np.abs(first_row.imag)) < 1e-12 * max(1.0, np.max(np.abs(first_row))):
            first_row = first_row.real
        keep = np.abs(first_row) > prune_tol
        return cls.from_arrays(n_x, np.nonzero(keep)[0], first_row[keep])

    # ------------------------------------------------------------- algebra
    @property
    def bandwidth(self) -> int:
        return int(np.max(np.abs(self.offsets)))

    def is_real(self) -> bool:
        return not np.iscomplexobj(self.weights)

    def symbol(self, omega):
        """sum_j w_j exp(i j omega) (circulant.py:133-143)."""
        om = np.asarray(omega, dtype=float)
        phases = np.exp(1j * np.multiply.outer(om, self.offsets.astype(float)))
        val = phases @ self.weights.astype(complex)
        return complex(val) if np.isscalar(omega) else val

    def eigenvalues(self) -> np.ndarray:
        """Symbol on the mesh frequencies, cached (circulant.py:145-154)."""
        if self._eig is None:
            eig = self.symbol(2.0 * np.pi * np.arange(self.n_x) / self.n_x)
            eig.setflags(write=False)
            object.__setattr__(self, "_eig", eig)
        return self._eig

    def dense(self) -> np.ndarray:
        M = np.zeros((self.n_x, self.n_x), dtype=self.weights.dtype)
        cols = np.arange(self.n_x)
        for off, w in zip(self.offsets, self.weights):
            M[cols, (cols + int(off)) % self.n_x] += w
        return M

    def compose(self, other: "CirculantOperator") -> "CirculantOperator":
        self._check_same_mesh(other)
        return CirculantOperator.from_arrays(
            self.n_x, (self.offsets[:, None] + other.offsets[None, :]).ravel(),
            (self.weights[:, None] * other.weights[None, :]).ravel())

    def add(self, other: "CirculantOperator") -> "CirculantOperator":
        self._check_same_mesh(other)
        dt = np.result_type(self.weights, other.weights)
        return CirculantOperator.from_arrays(
            self.n_x, np.concatenate([self.offsets, other.offsets]),
            np.concatenate([self.weights.astype(dt), other.weights]))

    def scale(self, s) -> "CirculantOperator":
        return CirculantOperator.from_arrays(self.n_x, self.offsets, s * self.weights)

    def power(self, m: int) -> "CirculantOperator":
        if m < 0:
            raise ValueError(f"power requires m >= 0, got {m}")
        acc, base = CirculantOperator.identity(self.n_x), self
        while m:
            if m & 1:
                acc = acc.compose(base)
            base = base.compose(base) if m > 1 else base
            m >>= 1
        return acc

    def __matmul__(self, other):
        return self.compose(other) if isinstance(other, CirculantOperator) else self.apply(other)

    def __add__(self, other):
        return self.add(other)

    def __sub__(self, other):
        return self.add(other.scale(-1.0))

    def __mul__(self, s):
        return self.scale(s)

    __rmul__ = __mul__

    def __repr__(self):
        taps = ", ".join(f"({int(o)}, {w:+.6g})" for o, w in zip(self.offsets, self.weights))
        return f"CirculantOperator(n_x={self.n_x}, [{taps}])"

    def _check_same_mesh(self, other):
        if self.n_x != other.n_x:
            raise DimensionMismatchError(f"mesh sizes differ: {self.n_x} vs {other.n_x}")

    # ------------------------------------------------------- device paths
    def device_program(self, exact: bool = True):
        from .device import DeviceProgram
        return DeviceProgram("stencil", self.n_x, self.offsets, self.weights, exact=exact)

    def apply(self, v):
        """Batched matrix-vector product on the GPU; ``v`` has shape (..., n_x)
        (numpy in -> numpy out; CUDA tensor in -> CUDA tensor out)."""
        from .device import apply_program
        if getattr(v, "shape", np.shape(v))[-1] != self.n_x:
            raise DimensionMismatchError(f"vector length {np.shape(v)[-1]} != n_x {self.n_x}")
        if not self.is_real():
            raise NotImplementedError("complex stencils are not supported on the device path")
        return apply_program(self.device_program(), v)

    def _check_invertible(self):
        lam = self.eigenvalues()
        bad = np.abs(lam) < SINGULAR_TOL
        if np.any(bad):
            k = int(np.argmax(bad))
            raise SingularOperatorError(f"operator is singular: |symbol| < {SINGULAR_TOL} "
                                        f"at omega = 2*pi*{k}/{self.n_x}")

    def solve_direct(self, b):
        """Solve op @ x = b exactly (factorised periodic banded solve on the GPU)."""
        from .device import DeviceProgram, apply_program
        if np.shape(b)[-1] != self.n_x:
            raise DimensionMismatchError(f"rhs length {np.shape(b)[-1]} != n_x {self.n_x}")
        self._check_invertible()
        prog = DeviceProgram("sl_direct", self.n_x, np.array([0]), np.array([1.0]),
                             self.offsets, self.weights)
        return apply_program(prog, b)

    def solve_gmres(self, b, rel_tol: float = 1e-2, max_iters: int = 20) -> "GmresResult":
        """Unrestarted GMRES(x0 = 0) on one vector (circulant.py:240-259)."""
        from .device import DeviceProgram, plan_for, ptr, require_cuda, to_device
        if not 0.0 < rel_tol < 1.0:
            raise ValueError(f"rel_tol must be in (0, 1), got {rel_tol}")
        if np.ndim(b) != 1 or np.shape(b)[0] != self.n_x:
            raise DimensionMismatchError(f"rhs must be a vector of length {self.n_x}")
        torch = require_cuda()
        prog = DeviceProgram("sl_gmres", self.n_x, np.array([0]), np.array([1.0]),
                             self.offsets, self.weights, gmres_tol=rel_tol,
                             gmres_cap=min(int(max_iters), self.n_x))
        dev, host = to_device(b)
        src = dev.reshape(1, self.n_x)
        out = torch.empty_like(src)
        depth = torch.zeros(1, dtype=torch.int32, device="cuda")
        res = torch.zeros(1, dtype=torch.float64, device="cuda")
        plan_for(prog).relax(1, 1, 0, c_src=ptr(src), c_stride=self.n_x, tail=1,
                             tail_out=ptr(out), tail_stride=self.n_x,
                             stats_depth=ptr(depth), stats_res=ptr(res))
        its, r = int(depth.item()), float(res.item())
        x = out.reshape(-1)
        x = x.cpu().numpy() if host is not None else x
        cap = min(int(max_iters), self.n_x)
        return GmresResult(x, its, r, bool(r <= rel_tol), bool(its < cap and r > rel_tol))


class GmresResult(NamedTuple):
    x: np.ndarray
    iterations: int
    relative_residual: float
    converged: bool
    breakdown: bool
