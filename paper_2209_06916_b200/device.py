"""Device plumbing: PyTorch tensors as HBM buffers, device plans for steppers,
and thin launch wrappers around the C ABI (``include/mgrit_b200.h``).

PyTorch is only used for allocation, streams and host<->device copies; all
arithmetic of the hot path runs in ``libmgrit_b200.so``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _native as nat


def torch_mod():
    import torch
    return torch


def require_cuda():
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_06916_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    nat.load()
    return torch


def stream_handle():
    torch = torch_mod()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_device(arr):
    """Return (cuda float64 contiguous tensor, host numpy array or None)."""
    torch = require_cuda()
    if is_tensor(arr):
        t = arr
        if t.dtype != torch.float64:
            raise TypeError("device arrays must be float64")
        if not t.is_cuda:  # host tensor (ideally pinned): copied in, written back
            return t.to("cuda", non_blocking=t.is_pinned()).contiguous(), t
        if not t.is_contiguous():
            raise ValueError("device arrays must be contiguous")
        return t, None
    host = np.asarray(arr)
    if np.iscomplexobj(host):
        raise NotImplementedError("complex arrays are not supported on the device path")
    host64 = np.ascontiguousarray(host, dtype=np.float64)
    return torch.from_numpy(host64).to("cuda"), host


@dataclass
class DeviceProgram:
    """Structured description of a one-step map Phi for the device.

    kind: ``"stencil"`` (assembled stencil, circulant.py:113-124),
    ``"rk"`` (staged RK; SDIRK stage solves, stepping.py:355-380),
    ``"sl_direct"`` / ``"sl_gmres"`` (semi-Lagrangian step then the
    (I - phi D) correction solve, stepping.py:546-561).
    """

    kind: str
    n_x: int
    offsets: np.ndarray
    weights: np.ndarray
    offsets2: Optional[np.ndarray] = None
    weights2: Optional[np.ndarray] = None
    rk_a: Optional[np.ndarray] = None
    rk_b: Optional[np.ndarray] = None
    implicit: bool = False
    gmres_tol: float = 1e-2
    gmres_cap: int = 20
    repeat: int = 1
    exact: bool = True
    #: kind "callable": the user's ``Stepper(apply_fn=...)`` (stepping.py:276-295),
    #: called with a CUDA tensor of shape (rows, n_x), returning the same
    fn: Optional[object] = None

    def key(self):
        def b(a):
            return None if a is None else np.asarray(a).tobytes()
        return (self.kind, self.n_x, b(self.offsets), b(self.weights), b(self.offsets2),
                b(self.weights2), b(self.rk_a), b(self.rk_b), self.implicit,
                self.gmres_tol, self.gmres_cap, self.repeat, self.exact,
                None if self.fn is None else id(self.fn))

    def repeated(self, times: int) -> "DeviceProgram":
        return DeviceProgram(self.kind, self.n_x, self.offsets, self.weights, self.offsets2,
                             self.weights2, self.rk_a, self.rk_b, self.implicit,
                             self.gmres_tol, self.gmres_cap, self.repeat * int(times),
                             self.exact, self.fn)


_KIND = {"stencil": nat.MGB_STEP_STENCIL, "rk": nat.MGB_STEP_RK_STAGED,
         "sl_direct": nat.MGB_STEP_SL_DIRECT, "sl_gmres": nat.MGB_STEP_SL_GMRES}


def _arr(a, dtype):
    a = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64 if dtype == np.int64
                                               else ctypes.c_double))


class StepPlan:
    """Owns one ``mgb_step`` device plan (kernel choice, factor tables, params)."""

    def __init__(self, prog: DeviceProgram):
        require_cuda()
        lib = nat.load()
        if np.iscomplexobj(prog.weights) or (prog.weights2 is not None
                                             and np.iscomplexobj(prog.weights2)):
            raise NotImplementedError("complex stencils are not supported on the device path")
        keep = []
        off, poff = _arr(prog.offsets, np.int64)
        w, pw = _arr(prog.weights, np.float64)
        keep += [off, w]
        d = nat.StepDesc()
        d.kind = _KIND[prog.kind]
        d.n_x = prog.n_x
        d.exact = 1 if prog.exact else 0
        d.repeat = int(prog.repeat)
        d.n_taps = len(off)
        d.offsets, d.weights = poff, pw
        if prog.offsets2 is not None:
            off2, poff2 = _arr(prog.offsets2, np.int64)
            w2, pw2 = _arr(prog.weights2, np.float64)
            keep += [off2, w2]
            d.n_taps2, d.offsets2, d.weights2 = len(off2), poff2, pw2
        if prog.rk_a is not None:
            A, pA = _arr(prog.rk_a, np.float64)
            B, pB = _arr(prog.rk_b, np.float64)
            keep += [A, B]
            d.stages, d.rk_a, d.rk_b = len(B), pA, pB
            d.implicit = 1 if prog.implicit else 0
        d.gmres_tol = float(prog.gmres_tol)
        d.gmres_cap = int(prog.gmres_cap)
        h = ctypes.c_void_p()
        nat.check(lib.mgb_step_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.prog = prog
        thr, ppt, smem = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        nat.check(lib.mgb_step_layout(h, ctypes.byref(thr), ctypes.byref(ppt), ctypes.byref(smem)))
        self.threads, self.points_per_thread, self.smem = thr.value, ppt.value, smem.value

    @property
    def handle(self):
        return self._h

    def reserve(self, stream=None) -> None:
        """Allocate the plan's lazily created workspace now (before a CUDA-graph
        capture, which cannot allocate)."""
        nat.check(self._lib.mgb_step_reserve_workspace(
            self._h, stream if stream is not None else stream_handle()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.mgb_step_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    def relax(self, n_intervals: int, m: int, n_fsteps: int, *, k_global0: int = 0,
              c_src=None, c_stride: int = 0, c_src0=None, e=None, e_stride: int = 0,
              c_out=None, c_out_stride: int = 0, c_last_out=None, u=None, write_f: int = 0, g=None,
              tail: int = 0, tail_out=None, tail_stride: int = 0, cref=None,
              cref_stride: int = 0, cref_e=None, cref_e_stride: int = 0, partials=None,
              stats_depth=None, stats_res=None, z_out=None, z_stride: int = 0,
              stream=None) -> None:
        """Launch one interval relaxation (see ``mgb_relax_args``).  Pointer
        arguments are ints (device addresses) or None."""
        a = nat.RelaxArgs()
        a.n_intervals, a.k_global0, a.m, a.n_fsteps = n_intervals, k_global0, m, n_fsteps
        a.c_src, a.c_stride, a.c_src0 = c_src, c_stride, c_src0
        a.e, a.e_stride = e, e_stride
        a.c_out, a.c_out_stride, a.c_last_out = c_out, c_out_stride, c_last_out
        a.u, a.write_f, a.g, a.tail = u, write_f, g, tail
        a.tail_out, a.tail_stride = tail_out, tail_stride
        a.cref, a.cref_stride, a.cref_e, a.cref_e_stride = cref, cref_stride, cref_e, cref_e_stride
        a.partials, a.stats_depth, a.stats_res = partials, stats_depth, stats_res
        a.z_out, a.z_stride = z_out, z_stride
        nat.check(self._lib.mgb_relax(self._h, ctypes.byref(a),
                                      stream if stream is not None else stream_handle()))


class _RawRows:
    """Strided (rows, n_x) float64 view of raw device memory for torch
    (``__cuda_array_interface__``; no copy)."""

    def __init__(self, addr: int, rows: int, n_x: int, stride: int):
        self.__cuda_array_interface__ = {
            "shape": (rows, n_x), "typestr": "<f8", "data": (int(addr), False), "version": 3,
            "strides": (8 * (int(stride) if rows > 1 else n_x), 8)}


class CallablePlan:
    """Interval relaxation around a user one-step callable
    (``Stepper(apply_fn=...)``, stepping.py:276-295): the same pass semantics as
    ``mgb_relax_args`` with every interval advanced at once by ONE call of the
    callable on a ``(n_intervals, n_x)`` CUDA tensor per time step.  The
    arithmetic of the step is the user's; the row updates, the residual and
    the per-interval partial sums are torch device operations in the
    reference's order (mgrit.py:132-166, 246)."""

    threads = points_per_thread = smem = 0

    def __init__(self, prog: DeviceProgram):
        self._torch = require_cuda()
        self.prog = prog

    def reserve(self, stream=None) -> None:
        pass

    def _rows(self, addr, rows, stride):
        t = self._torch
        return t.as_tensor(_RawRows(addr, rows, self.prog.n_x, stride), device="cuda")

    def _step(self, y):
        for _ in range(max(1, int(self.prog.repeat))):
            y = self.prog.fn(y)
            if not (self._torch.is_tensor(y) and y.is_cuda and y.dtype == self._torch.float64):
                raise TypeError("apply_fn must map a float64 CUDA tensor (rows, n_x) to the same; "
                                "wrap numpy-only callables with stepping.host_callable")
        return y

    def relax(self, n_intervals: int, m: int, n_fsteps: int, *, k_global0: int = 0,
              c_src=None, c_stride: int = 0, c_src0=None, e=None, e_stride: int = 0,
              c_out=None, c_out_stride: int = 0, c_last_out=None, u=None, write_f: int = 0, g=None,
              tail: int = 0, tail_out=None, tail_stride: int = 0, cref=None,
              cref_stride: int = 0, cref_e=None, cref_e_stride: int = 0, partials=None,
              stats_depth=None, stats_res=None, z_out=None, z_stride: int = 0,
              stream=None) -> None:
        t = self._torch
        nI, n = int(n_intervals), self.prog.n_x
        if nI <= 0:
            return
        if c_src is not None:
            y = self._rows(c_src, nI, c_stride).clone()
        else:
            y = t.zeros((nI, n), dtype=t.float64, device="cuda")
        if c_src0 is not None and k_global0 == 0:
            y[0] = self._rows(c_src0, 1, n)[0]
        if e is not None:  # u[m::m] += e[1:] (mgrit.py:246): global intervals k >= 1
            k0 = 1 if k_global0 == 0 else 0
            if nI > k0:
                y[k0:] += self._rows(e + 8 * k0 * e_stride, nI - k0, e_stride)
        if c_out is not None:
            self._rows(c_out, nI, c_out_stride).copy_(y)
        for j in range(1, n_fsteps + 1):
            y = self._step(y)
            if g is not None:
                y = y + self._rows(g + 8 * j * n, nI, m * n)
            if write_f == 2 or (write_f == 1 and j == n_fsteps):
                self._rows(u + 8 * j * n, nI, m * n).copy_(y)
        if tail:
            z = self._step(y)
            if g is not None:
                z = self._rows(g + 8 * m * n, nI, m * n) + z
            if tail == 1:
                self._rows(tail_out, nI, tail_stride).copy_(z)
            else:
                if z_out is not None:
                    self._rows(z_out, nI, z_stride).copy_(z)
                cr = self._rows(cref, nI, cref_stride)
                if cref_e is not None:
                    cr = cr + self._rows(cref_e, nI, cref_e_stride)
                r = z - cr
                if tail_out is not None:
                    self._rows(tail_out, nI, tail_stride).copy_(r)
                if partials is not None:
                    t.as_tensor(_RawRows(partials, 1, nI, nI), device="cuda")[0].copy_((r * r).sum(dim=1))
        if c_last_out is not None:
            if c_src is not None:
                last = self._rows(c_src + 8 * nI * c_stride, 1, n)[0].clone()
            else:
                last = t.zeros(n, dtype=t.float64, device="cuda")
            if e is not None:
                last += self._rows(e + 8 * nI * e_stride, 1, n)[0]
            self._rows(c_last_out, 1, n)[0].copy_(last)


def device_sum(partials, n: int, out, stream=None) -> None:
    nat.check(nat.load().mgb_sum(ctypes.c_void_p(partials), n, ctypes.c_void_p(out),
                                 stream if stream is not None else stream_handle()))


_PLAN_CACHE: dict = {}


def plan_for(prog: DeviceProgram, tag=None) -> StepPlan:
    """Memoised device plan per (program, device, tag).  Plans own their GMRES
    workspaces, so solves that run concurrently on different CUDA streams pass
    distinct tags (``solve_many`` uses the stream) to get private plans."""
    torch = require_cuda()
    key = (torch.cuda.current_device(), tag, prog.key())
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = CallablePlan(prog) if prog.kind == "callable" else StepPlan(prog)
        _PLAN_CACHE[key] = plan
    return plan


def apply_program(prog: DeviceProgram, u):
    """Batched one-step apply out[..., :] = Phi u[..., :] on the device.

    Accepts numpy (returns numpy) or a CUDA tensor (returns a CUDA tensor)."""
    torch = require_cuda()
    dev, host = to_device(u)
    shape = tuple(dev.shape)
    if shape[-1] != prog.n_x:
        from .errors import DimensionMismatchError
        raise DimensionMismatchError(f"vector length {shape[-1]} != n_x {prog.n_x}")
    rows = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
    src = dev.reshape(rows, prog.n_x)
    out = torch.empty_like(src)
    plan = plan_for(prog)
    plan.relax(rows, 1, 0, c_src=ptr(src), c_stride=prog.n_x, tail=1,
               tail_out=ptr(out), tail_stride=prog.n_x)
    out = out.reshape(shape)
    if host is not None:
        return out.cpu().numpy()
    return out
