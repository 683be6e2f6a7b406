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


def _exec(device: torch.device, stream=None, rank: int = 0, world: int = 1, nccl_id=None) -> N.FmmExec:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return N.FmmExec(device.index if device.index is not None else torch.cuda.current_device(),
                     C.c_void_p(stream.cuda_stream), rank, world,
                     C.cast(nccl_id, C.c_void_p) if nccl_id is not None else None)


def nccl_unique_id() -> bytes:
    """A new ncclUniqueId (fmm_nccl_unique_id): make it on one rank, send it to the others."""
    buf = C.create_string_buffer(128)
    N.check(N.lib().fmm_nccl_unique_id(buf))
    return buf.raw


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

    _dim = 3

    def __init__(self, points: torch.Tensor, p: int, ncrit: int, theta: float, *, rank: int = 0,
                 world: int = 1, stream=None, nccl_id: bytes | None = None):
        """nccl_id (world > 1): collective mode — ``points`` is this rank's slice, ``matvec``
        takes and returns this rank's slices (include/fmm.h fmm_exec.nccl_id)."""
        points = _dev_f64(points, "points", (self._dim,))
        self.device = points.device
        self.n = points.shape[0]
        self.p, self.ncrit, self.theta = p, ncrit, theta
        self.rank, self.world = rank, world
        self._stream = stream
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self._ex = _exec(self.device, stream, rank, world, self._nccl_id)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            setup = N.lib().fmm_setup if self._dim == 3 else N.lib().fmm_setup_2d
            N.check(setup(C.byref(h), C.c_void_p(points.data_ptr()), self.n, p, ncrit, float(theta), C.byref(self._ex)))
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
        d["bytes_by"] = dict(zip(N.BYTES_CATEGORIES, list(s.bytes_by)))
        return d

    # ---- multi-GPU LET exchange (fmm.h fmm_let_*); buffers are device float64 tensors
    def let_setup(self, caller_counts):
        cc = (C.c_int64 * len(caller_counts))(*[int(c) for c in caller_counts])
        N.check(N.lib().fmm_let_setup(self._h, cc))
        nc = (self.p + 1) * (self.p + 2) // 2
        self.let = {name: self._let_counts(code) for name, code in (
            ("q_send", N.FMM_LET_Q_SEND), ("q_recv", N.FMM_LET_Q_RECV), ("m_send", N.FMM_LET_M_SEND),
            ("m_recv", N.FMM_LET_M_RECV), ("phi_send", N.FMM_LET_PHI_SEND), ("phi_recv", N.FMM_LET_PHI_RECV))}
        sh = (C.c_int64 * 1)()
        N.check(N.lib().fmm_let_counts(self._h, N.FMM_LET_SHARED, sh))
        self.let["shared"] = int(sh[0])
        rb = (C.c_int64 * (self.world + 1))()
        N.check(N.lib().fmm_let_counts(self._h, N.FMM_LET_RANK_BEGIN, rb))
        self.let["rank_begin"] = list(rb)
        self.let["ncd"] = 2 * nc  # doubles per expansion
        return self.let

    def _let_counts(self, code):
        out = (C.c_int64 * self.world)()
        N.check(N.lib().fmm_let_counts(self._h, code, out))
        return list(out)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else None

    def let_pack_q(self, q_local, q_send):
        N.check(N.lib().fmm_let_pack_q(self._h, self._p(q_local), self._p(q_send)))

    def let_upward(self, q_recv, shared_send, m_send):
        N.check(N.lib().fmm_let_upward(self._h, self._p(q_recv), self._p(shared_send), self._p(m_send)))

    def let_finish(self, shared_recv, m_recv, phi_send, grad_send=None):
        N.check(N.lib().fmm_let_finish(self._h, self._p(shared_recv), self._p(m_recv), self._p(phi_send),
                                       self._p(grad_send)))

    def let_unpack(self, phi_recv, grad_recv, phi_local, grad_local=None):
        N.check(N.lib().fmm_let_unpack(self._h, self._p(phi_recv), self._p(grad_recv), self._p(phi_local),
                                       self._p(grad_local)))

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


class Plan2D(Plan):
    """NEXT-3: FMM plan for planar points [n, 2] and the 2D log kernel (``fmm_setup_2d``):
    ``matvec`` returns phi_i = -sum_j q_j log|x_i - x_j| (+ its gradient as [n, 3], z = 0)."""

    _dim = 2


def _dev_c128(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.complex128 or t.dim() != 1:
        raise TypeError(f"{name} must be a 1-D CUDA complex128 tensor")
    return t.contiguous()


class HelmholtzPlan(Plan):
    """NEXT-4: FMM plan for the 3D Helmholtz kernel exp(i kappa r) / r
    (``fmm_setup_helmholtz``, include/fmm_helmholtz.h); ``matvec`` maps complex128 charges to
    complex128 potentials, caller order. Single GPU."""

    def __init__(self, points: torch.Tensor, p: int, ncrit: int, theta: float, kappa: float, *, stream=None):
        points = _dev_f64(points, "points", (3,))
        self.device = points.device
        self.n = points.shape[0]
        self.p, self.ncrit, self.theta, self.kappa = p, ncrit, theta, float(kappa)
        self.rank, self.world = 0, 1
        self._stream = stream
        self._nccl_id = None
        self._ex = _exec(self.device, stream, 0, 1)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().fmm_setup_helmholtz(C.byref(h), C.c_void_p(points.data_ptr()), self.n, p, ncrit,
                                                float(theta), float(kappa), C.byref(self._ex)))
        self._h = h

    def matvec(self, q: torch.Tensor, out: torch.Tensor | None = None):
        q = _dev_c128(q, "q")
        if q.shape[0] != self.n:
            raise ValueError("q length differs from the plan's point count")
        phi = torch.empty(self.n, dtype=torch.complex128, device=self.device) if out is None else out
        N.check(N.lib().fmm_matvec_helmholtz(self._h, C.c_void_p(q.data_ptr()), self.n, C.c_void_p(phi.data_ptr())))
        return phi


def direct_helmholtz(src: torch.Tensor, q: torch.Tensor, kappa: float, tgt: torch.Tensor | None = None):
    """fmm_direct_helmholtz: O(n_src n_tgt) sum of q exp(i kappa r) / r on the GPU (checking path)."""
    src = _dev_f64(src, "src", (3,))
    q = _dev_c128(q, "q")
    tgt = src if tgt is None else _dev_f64(tgt, "tgt", (3,))
    phi = torch.empty(tgt.shape[0], dtype=torch.complex128, device=src.device)
    ex = _exec(src.device)
    N.check(N.lib().fmm_direct_helmholtz(C.c_void_p(src.data_ptr()), C.c_void_p(q.data_ptr()), src.shape[0],
                                         C.c_void_p(tgt.data_ptr()), tgt.shape[0], float(kappa),
                                         C.c_void_p(phi.data_ptr()), C.byref(ex)))
    return phi


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


def let_lists_host(n, world, me, caller_off, perm, cbeg, cend, leaves, p2p, m2l, what, p=4):
    """Host-only exchange-list builder (fmm_let_lists_host; no device work): numpy arrays in, one list out."""
    import numpy as _np

    def a(x, dt):
        return _np.ascontiguousarray(x, dtype=dt)

    co, pm = a(caller_off, _np.int64), a(perm, _np.uint32)
    cb, ce, lv = a(cbeg, _np.int32), a(cend, _np.int32), a(leaves, _np.int32)
    pt, ps = a(p2p[:, 0], _np.int32), a(p2p[:, 1], _np.int32)
    mt, ms = a(m2l[:, 0], _np.int32), a(m2l[:, 1], _np.int32)
    ptr = lambda x: C.c_void_p(x.ctypes.data)  # noqa: E731
    args = [int(n), int(world), int(me), int(p), ptr(co), ptr(pm), len(cb), ptr(cb), ptr(ce), len(lv), ptr(lv), len(pt),
            ptr(pt), ptr(ps), len(mt), ptr(mt), ptr(ms), int(what)]
    cnt = C.c_int64()
    N.check(N.lib().fmm_let_lists_host(*args, None, 0, C.byref(cnt)))
    out = _np.empty(cnt.value, dtype=_np.int64)
    N.check(N.lib().fmm_let_lists_host(*args, C.c_void_p(out.ctypes.data), cnt.value, C.byref(cnt)))
    return out


def version() -> str:
    return N.lib().fmm_version().decode()
