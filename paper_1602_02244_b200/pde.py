"""NEXT-2 / NEXT-4 solve: the FMM as a low-accuracy preconditioner in a Krylov solve (include/fmm_pde.h).

3D Laplace and Helmholtz on the [-1,1]^3 lattice with Dirichlet faces (§4.2):
the 7-point operator (minus kappa^2), the FMM volume-potential preconditioner with single-layer
boundary correction, flexible PCG (Laplace) and GMRES (Helmholtz) — all libfmm.so kernels; this
module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .fmm import _dev_f64, _exec


def spacing(n: int) -> float:
    return 2.0 / (n + 1)


def stencil_apply(u: torch.Tensor, n: int) -> torch.Tensor:
    """A u, A = -Delta_h (fmm_stencil_apply)."""
    u = _dev_f64(u, "u")
    if u.shape[0] != n ** 3:
        raise ValueError("u must have n^3 entries")
    out = torch.empty_like(u)
    N.check(N.lib().fmm_stencil_apply(n, C.c_void_p(u.data_ptr()), C.c_void_p(out.data_ptr()),
                                      C.c_void_p(torch.cuda.current_stream(u.device).cuda_stream)))
    return out


class FmmPreconditioner:
    """M r (fmm_precond_setup / fmm_precond_apply): FMM order p, ncrit, theta set its accuracy."""

    def __init__(self, n: int, p: int = 4, ncrit: int = 32, theta: float = 0.5, face_stride: int = 1,
                 boundary: bool = True, device=None):
        self.n = n
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._h = C.c_void_p()
        ex = _exec(self.device)
        N.check(N.lib().fmm_precond_setup(C.byref(self._h), n, face_stride, p, ncrit, float(theta), int(boundary),
                                          C.byref(ex)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib().fmm_precond_destroy(h)
            self._h = None

    def apply(self, r: torch.Tensor) -> torch.Tensor:
        r = _dev_f64(r, "r")
        if r.shape[0] != self.n ** 3:
            raise ValueError("r must have n^3 entries")
        z = torch.empty_like(r)
        N.check(N.lib().fmm_precond_apply(self._h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr())))
        return z

    def info(self) -> dict:
        npan, nb = C.c_int64(), C.c_int64()
        N.check(N.lib().fmm_precond_info(self._h, C.byref(npan), C.byref(nb)))
        return {"panels": npan.value, "bytes": nb.value}


def pcg(b: torch.Tensor, n: int, M: FmmPreconditioner | None = None, rtol: float = 1e-8, maxit: int = 500):
    """Flexible PCG for A x = b (fmm_pcg_solve). Returns (x, history list, info dict)."""
    b = _dev_f64(b, "b")
    if b.shape[0] != n ** 3:
        raise ValueError("b must have n^3 entries")
    x = torch.empty_like(b)
    hist = (C.c_double * (maxit + 1))()
    info = N.PcgInfo()
    stream = C.c_void_p(torch.cuda.current_stream(b.device).cuda_stream)
    N.check(N.lib().fmm_pcg_solve(n, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), M._h if M else None,
                                  float(rtol), int(maxit), hist, C.byref(info), stream))
    it = info.iterations
    return x, [hist[i] for i in range(it + 1)], {k: getattr(info, k) for k, _ in N.PcgInfo._fields_}


def _dev_c128(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.complex128:
        raise TypeError(f"{name} must be complex128")
    if t.dim() != 1:
        raise ValueError(f"{name} must have shape [n^3]")
    return t.contiguous()


def helmholtz_stencil_apply(u: torch.Tensor, n: int, kappa: float) -> torch.Tensor:
    """A u, A = -Delta_h - kappa^2 (fmm_helmholtz_stencil_apply); complex128 in and out."""
    u = _dev_c128(u, "u")
    if u.shape[0] != n ** 3:
        raise ValueError("u must have n^3 entries")
    out = torch.empty_like(u)
    N.check(N.lib().fmm_helmholtz_stencil_apply(n, float(kappa), C.c_void_p(u.data_ptr()), C.c_void_p(out.data_ptr()),
                                                C.c_void_p(torch.cuda.current_stream(u.device).cuda_stream)))
    return out


class HelmholtzPreconditioner:
    """M r (fmm_hprecond_setup / fmm_hprecond_apply): the Helmholtz FMM of order p (ncrit, theta) over
    the lattice and face panels, wave number kappa; complex128 vectors."""

    def __init__(self, n: int, kappa: float, p: int = 4, ncrit: int = 32, theta: float = 0.5, face_stride: int = 1,
                 boundary: bool = True, device=None):
        self.n, self.kappa = n, float(kappa)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._h = C.c_void_p()
        ex = _exec(self.device)
        N.check(N.lib().fmm_hprecond_setup(C.byref(self._h), n, face_stride, p, ncrit, float(theta), self.kappa,
                                           int(boundary), C.byref(ex)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib().fmm_hprecond_destroy(h)
            self._h = None

    def apply(self, r: torch.Tensor) -> torch.Tensor:
        r = _dev_c128(r, "r")
        if r.shape[0] != self.n ** 3:
            raise ValueError("r must have n^3 entries")
        z = torch.empty_like(r)
        N.check(N.lib().fmm_hprecond_apply(self._h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr())))
        return z

    def info(self) -> dict:
        npan, nb = C.c_int64(), C.c_int64()
        N.check(N.lib().fmm_hprecond_info(self._h, C.byref(npan), C.byref(nb)))
        return {"panels": npan.value, "bytes": nb.value}


def gmres(b: torch.Tensor, n: int, kappa: float, M: HelmholtzPreconditioner | None = None, rtol: float = 1e-8,
          maxit: int = 200):
    """Right-preconditioned GMRES for (-Delta_h - kappa^2) x = b (fmm_gmres_solve). Returns (x complex128,
    history list, info dict)."""
    b = _dev_c128(b, "b")
    if b.shape[0] != n ** 3:
        raise ValueError("b must have n^3 entries")
    x = torch.empty_like(b)
    hist = (C.c_double * (maxit + 1))()
    info = N.PcgInfo()
    stream = C.c_void_p(torch.cuda.current_stream(b.device).cuda_stream)
    N.check(N.lib().fmm_gmres_solve(n, float(kappa), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                                    M._h if M else None, float(rtol), int(maxit), hist, C.byref(info), stream))
    it = info.iterations
    return x, [hist[i] for i in range(it + 1)], {k: getattr(info, k) for k, _ in N.PcgInfo._fields_}
