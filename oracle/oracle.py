"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/liboracle.so`` (plain C, see fmm_oracle.c), the
independent CPU FMM that the CUDA path is checked against. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this module. It shares no code with
``paper_1602_02244_b200`` and never imports it.

Method: arXiv:1602.02244 (PAPER.md:22-24 multipole/local expansions,
PAPER.md:149-153 M2L, PAPER.md:166-168 dual tree traversal + MAC,
PAPER.md:191-196 direct/translation operators as diagonal/off-diagonal blocks);
formulas and algorithm per SURVEY.md §8(c) as adopted in DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "fmm_oracle.c")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, A3)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "fmm_oracle.h"))
    ):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        dp = C.POINTER(C.c_double)
        i64p = C.POINTER(C.c_int64)
        L.oracle_direct.argtypes = [dp, dp, C.c_int64, dp, C.c_int64, dp, dp, C.c_int]
        L.oracle_direct.restype = C.c_int
        for nm in ("oracle_harmonics_R", "oracle_harmonics_I"):
            getattr(L, nm).argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, dp]
            getattr(L, nm).restype = None
        L.oracle_p2m.argtypes = [dp, dp, C.c_int64, dp, C.c_int, dp]
        for nm in ("oracle_m2m", "oracle_m2l", "oracle_l2l"):
            getattr(L, nm).argtypes = [dp, dp, dp, C.c_int, dp]
        L.oracle_l2p.argtypes = [dp, dp, dp, C.c_int, dp, dp]
        L.oracle_m2p.argtypes = [dp, dp, dp, C.c_int, dp]
        L.oracle_plan_new.argtypes = [C.POINTER(C.c_void_p), dp, C.c_int64, C.c_int, C.c_int, C.c_double]
        L.oracle_plan_new.restype = C.c_int
        L.oracle_plan_free.argtypes = [C.c_void_p]
        L.oracle_plan_info.argtypes = [C.c_void_p, C.c_int]
        L.oracle_plan_info.restype = C.c_int64
        L.oracle_plan_geometry.argtypes = [C.c_void_p, dp, dp, dp]
        L.oracle_plan_keys.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), i64p]
        i32p = C.POINTER(C.c_int32)
        L.oracle_plan_cells.argtypes = [C.c_void_p, i32p, i32p, i64p, i64p, i64p, i32p, i64p, dp]
        L.oracle_plan_lists.argtypes = [C.c_void_p, i64p, i64p]
        L.oracle_plan_eval.argtypes = [C.c_void_p, dp, i64p, C.c_int64, dp, dp, C.c_int]
        L.oracle_plan_eval.restype = C.c_int
        L.oracle_plan_expansions.argtypes = [C.c_void_p, dp, dp]
        _lib = L
    return _lib


def _p(a, ct=C.c_double):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def ncoef(p: int) -> int:
    return (p + 1) * (p + 2) // 2


def cidx(n: int, m: int) -> int:
    return n * (n + 1) // 2 + m


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


def direct(src, q, tgt=None, grad=False, nthreads=0):
    """phi_i = sum_{j: r_ij>0} q_j / r_ij (+ grad phi), long-double accumulation (A16)."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    tgt = src if tgt is None else np.ascontiguousarray(tgt, dtype=np.float64)
    nt = tgt.shape[0]
    phi = np.zeros(nt)
    g = np.zeros((nt, 3)) if grad else None
    st = lib().oracle_direct(_p(src), _p(q), src.shape[0], _p(tgt), nt, _p(phi), _p(g), nthreads)
    if st:
        raise OracleError(st)
    return (phi, g) if grad else phi


def harmonics_R(v, p):
    out = np.zeros(ncoef(p), dtype=np.complex128)
    lib().oracle_harmonics_R(float(v[0]), float(v[1]), float(v[2]), p, _p(out.view(np.float64)))
    return out


def harmonics_I(v, p):
    out = np.zeros(ncoef(p), dtype=np.complex128)
    lib().oracle_harmonics_I(float(v[0]), float(v[1]), float(v[2]), p, _p(out.view(np.float64)))
    return out


def _c3(c):
    return np.ascontiguousarray(c, dtype=np.float64)


def p2m(xyz, q, c, p, M=None):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    M = np.zeros(ncoef(p), dtype=np.complex128) if M is None else M
    lib().oracle_p2m(_p(xyz), _p(q), xyz.shape[0], _p(_c3(c)), p, _p(M.view(np.float64)))
    return M


def m2m(Mc, c_child, c_parent, p, Mp=None):
    Mp = np.zeros(ncoef(p), dtype=np.complex128) if Mp is None else Mp
    Mc = np.ascontiguousarray(Mc, dtype=np.complex128)
    lib().oracle_m2m(_p(Mc.view(np.float64)), _p(_c3(c_child)), _p(_c3(c_parent)), p, _p(Mp.view(np.float64)))
    return Mp


def m2l(MB, cB, cA, p, LA=None):
    LA = np.zeros(ncoef(p), dtype=np.complex128) if LA is None else LA
    MB = np.ascontiguousarray(MB, dtype=np.complex128)
    lib().oracle_m2l(_p(MB.view(np.float64)), _p(_c3(cB)), _p(_c3(cA)), p, _p(LA.view(np.float64)))
    return LA


def l2l(Lp, c_parent, c_child, p, Lc=None):
    Lc = np.zeros(ncoef(p), dtype=np.complex128) if Lc is None else Lc
    Lp = np.ascontiguousarray(Lp, dtype=np.complex128)
    lib().oracle_l2l(_p(Lp.view(np.float64)), _p(_c3(c_parent)), _p(_c3(c_child)), p, _p(Lc.view(np.float64)))
    return Lc


def l2p(L, c, x, p, grad=False):
    L = np.ascontiguousarray(L, dtype=np.complex128)
    phi = np.zeros(1)
    g = np.zeros(3) if grad else None
    lib().oracle_l2p(_p(L.view(np.float64)), _p(_c3(c)), _p(_c3(x)), p, _p(phi), _p(g))
    return (phi[0], g) if grad else phi[0]


def m2p(M, c, x, p):
    M = np.ascontiguousarray(M, dtype=np.complex128)
    phi = np.zeros(1)
    lib().oracle_m2p(_p(M.view(np.float64)), _p(_c3(c)), _p(_c3(x)), p, _p(phi))
    return phi[0]


class Plan:
    """Oracle plan: A1–A7 at construction, A8–A15 in :meth:`eval`."""

    INFO = dict(n=0, ncells=1, nleaves=2, np2p=3, nm2l=4, exp=5, maxlevel=6, p=7, p2p_interactions=8)

    def __init__(self, xyz, p, ncrit, theta):
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.p = p
        h = C.c_void_p()
        st = lib().oracle_plan_new(C.byref(h), _p(self.xyz), self.xyz.shape[0], p, ncrit, float(theta))
        if st:
            raise OracleError(st)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().oracle_plan_free(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def info(self, name):
        return int(lib().oracle_plan_info(self._h, self.INFO[name]))

    @property
    def ncells(self):
        return self.info("ncells")

    def geometry(self):
        lo = np.zeros(3)
        S = np.zeros(1)
        sc = np.zeros(1)
        lib().oracle_plan_geometry(self._h, _p(lo), _p(S), _p(sc))
        return lo, S[0], sc[0]

    def keys(self):
        n = self.info("n")
        k = np.zeros(n, dtype=np.uint64)
        perm = np.zeros(n, dtype=np.int64)
        lib().oracle_plan_keys(self._h, _p(k, C.c_uint64), _p(perm, C.c_int64))
        return k, perm

    def cells(self):
        nc = self.ncells
        out = dict(
            level=np.zeros(nc, np.int32), anchor=np.zeros((nc, 3), np.int32), begin=np.zeros(nc, np.int64),
            end=np.zeros(nc, np.int64), child_first=np.zeros(nc, np.int64), nchild=np.zeros(nc, np.int32),
            parent=np.zeros(nc, np.int64), center=np.zeros((nc, 3)),
        )
        i32, i64 = C.c_int32, C.c_int64
        lib().oracle_plan_cells(
            self._h, _p(out["level"], i32), _p(out["anchor"], i32), _p(out["begin"], i64), _p(out["end"], i64),
            _p(out["child_first"], i64), _p(out["nchild"], i32), _p(out["parent"], i64), _p(out["center"]),
        )
        return out

    def lists(self):
        p2p = np.zeros((self.info("np2p"), 2), np.int64)
        m2l = np.zeros((self.info("nm2l"), 2), np.int64)
        lib().oracle_plan_lists(self._h, _p(p2p, C.c_int64), _p(m2l, C.c_int64))
        return p2p, m2l

    def eval(self, q, grad=False, targets=None, nthreads=0):
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = self.info("n")
        if targets is None:
            nt, tp = n, None
        else:
            targets = np.ascontiguousarray(targets, dtype=np.int64)
            nt, tp = targets.shape[0], targets
        phi = np.zeros(nt)
        g = np.zeros((nt, 3)) if grad else None
        st = lib().oracle_plan_eval(self._h, _p(q), _p(tp, C.c_int64), nt if tp is not None else 0,
                                    _p(phi), _p(g), nthreads)
        if st:
            raise OracleError(st)
        return (phi, g) if grad else phi

    def expansions(self):
        nc = self.ncells
        M = np.zeros((nc, ncoef(self.p)), np.complex128)
        L = np.zeros((nc, ncoef(self.p)), np.complex128)
        lib().oracle_plan_expansions(self._h, _p(M.view(np.float64)), _p(L.view(np.float64)))
        return M, L


def fmm(xyz, q, p, ncrit, theta, grad=False, targets=None, nthreads=0):
    """One-shot oracle FMM mat-vec."""
    return Plan(xyz, p, ncrit, theta).eval(q, grad=grad, targets=targets, nthreads=nthreads)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
