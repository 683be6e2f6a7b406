"""Python binding of the C ABI (include/fmm.h): ``Plan`` and ``direct``.

Argument marshalling only. Tensors must be CUDA float64; every step of the
mat-vec runs in libfmm.so kernels on the tensor's device and PyTorch's
current stream. PyTorch supplies device memory and the stream (north_star:
"PyTorch is used only for device memory, streams and process groups").
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N


def _exec(device: torch.device, stream=None, rank: int = 0, world: int = 1) -> N.FmmExec:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return N.FmmExec(device.index if device.index is not None else torch.cuda.current_device(),
                     C.c_void_p(stream.cuda_stream), rank, world)


def _dev_f64(t: torch.Tensor, name: str, shape_tail=()) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    if tuple(t.shape[1:]) != tuple(shape_tail):
        raise ValueError(f"{name} must have shape [n{''.join(f', {s}' for s in shape_tail)}]")
    return t.contiguous()


class Plan:
    """FMM plan: ``fmm_setup`` at construction (tree + interaction lists),
    ``matvec`` = ``fmm_matvec`` (precalculation vs application)."""

    def __init__(self, points: torch.Tensor, p: int, ncrit: int, theta: float, *, rank: int = 0,
                 world: int = 1, stream=None):
        points = _dev_f64(points, "points", (3,))
        self.device = points.device
        self.n = points.shape[0]
        self.p, self.ncrit, self.theta = p, ncrit, theta
        self.rank, self.world = rank, world
        self._stream = stream
        self._ex = _exec(self.device, stream, rank, world)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().fmm_setup(C.byref(h), C.c_void_p(points.data_ptr()), self.n, p, ncrit, float(theta),
                                      C.byref(self._ex)))
        self._h = h

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib().fmm_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def matvec(self, q: torch.Tensor, grad: bool = False, out=None):
        """phi (+ grad phi) in caller order; stream ordered (no host sync)."""
        q = _dev_f64(q, "q")
        if q.shape[0] != self.n:
            raise ValueError("q length differs from the plan's point count")
        if out is None:
            phi = torch.empty(self.n, dtype=torch.float64, device=self.device)
            g = torch.empty(self.n, 3, dtype=torch.float64, device=self.device) if grad else None
        else:
            phi, g = out
        N.check(N.lib().fmm_matvec(self._h, C.c_void_p(q.data_ptr()), self.n, C.c_void_p(phi.data_ptr()),
                                   C.c_void_p(g.data_ptr()) if g is not None else None))
        return (phi, g) if grad else phi

    def matvec_host(self, q: np.ndarray | torch.Tensor, grad: bool = False, out=None):
        """End-to-end call with HOST buffers (fmm_matvec_host): H2D, mat-vec, D2H, sync."""
        if isinstance(q, np.ndarray):
            q = torch.from_numpy(np.ascontiguousarray(q, dtype=np.float64))
        if q.is_cuda or q.dtype != torch.float64 or q.shape != (self.n,):
            raise ValueError("q must be a host float64 tensor/array of length n")
        if out is None:
            phi = torch.empty(self.n, dtype=torch.float64)
            g = torch.empty(self.n, 3, dtype=torch.float64) if grad else None
        else:
            phi, g = out
        N.check(N.lib().fmm_matvec_host(self._h, C.c_void_p(q.data_ptr()), self.n, C.c_void_p(phi.data_ptr()),
                                        C.c_void_p(g.data_ptr()) if g is not None else None))
        return (phi, g) if grad else phi

    def sync(self):
        N.check(N.lib().fmm_sync(self._h))

    def set_timing(self, on: bool = True):
        N.check(N.lib().fmm_set_timing(self._h, int(on)))

    def stats(self) -> dict:
        s = N.FmmStats()
        N.check(N.lib().fmm_stats(self._h, C.byref(s)))
        d = {k: getattr(s, k) for k, _ in N.FmmStats._fields_}
        d["t_setup_ms"] = list(s.t_setup_ms)
        d["t_matvec_ms"] = list(s.t_matvec_ms)
        return d

    _EXPORT = {
        "keys": (N.FMM_X_KEYS, np.uint64, None), "perm": (N.FMM_X_PERM, np.uint32, None),
        "level": (N.FMM_X_LEVEL, np.int32, None), "anchor": (N.FMM_X_ANCHOR, np.int32, 3),
        "begin": (N.FMM_X_BEGIN, np.int32, None), "end": (N.FMM_X_END, np.int32, None),
        "child": (N.FMM_X_CHILD, np.int32, None), "nchild": (N.FMM_X_NCHILD, np.int32, None),
        "parent": (N.FMM_X_PARENT, np.int32, None), "center": (N.FMM_X_CENTER, np.float64, 3),
        "p2p": (N.FMM_X_P2P, np.int32, 2), "m2l": (N.FMM_X_M2L, np.int32, 2),
        "M": (N.FMM_X_M, np.float64, "c"), "L": (N.FMM_X_L, np.float64, "c"), "geom": (N.FMM_X_GEOM, np.float64, None),
    }

    def export(self, what: str) -> np.ndarray:
        code, dt, shape = self._EXPORT[what]
        cnt = C.c_int64()
        N.check(N.lib().fmm_export(self._h, code, None, 0, C.byref(cnt)))
        a = np.empty(cnt.value, dtype=dt)
        N.check(N.lib().fmm_export(self._h, code, C.c_void_p(a.ctypes.data), cnt.value, C.byref(cnt)))
        if shape == "c":
            nc = (self.p + 1) * (self.p + 2) // 2
            return a.view(np.complex128).reshape(-1, nc)
        return a.reshape(-1, shape) if shape else a


def direct(src: torch.Tensor, q: torch.Tensor, tgt: torch.Tensor | None = None, grad: bool = False):
    """fmm_direct: O(n_src n_tgt) sum on the GPU (checking path, north_star)."""
    src = _dev_f64(src, "src", (3,))
    q = _dev_f64(q, "q")
    tgt = src if tgt is None else _dev_f64(tgt, "tgt", (3,))
    nt = tgt.shape[0]
    phi = torch.empty(nt, dtype=torch.float64, device=src.device)
    g = torch.empty(nt, 3, dtype=torch.float64, device=src.device) if grad else None
    ex = _exec(src.device)
    N.check(N.lib().fmm_direct(C.c_void_p(src.data_ptr()), C.c_void_p(q.data_ptr()), src.shape[0],
                               C.c_void_p(tgt.data_ptr()), nt, C.c_void_p(phi.data_ptr()),
                               C.c_void_p(g.data_ptr()) if g is not None else None, C.byref(ex)))
    return (phi, g) if grad else phi


def version() -> str:
    return N.lib().fmm_version().decode()
