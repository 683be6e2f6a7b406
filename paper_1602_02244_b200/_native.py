"""ctypes declarations for libfmm.so (include/fmm.h). Argument marshalling only.

The CUDA library is mandatory: importing this module raises if libfmm.so is
missing or cannot be loaded. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfmm.so")

FMM_OK, FMM_ERR_USAGE, FMM_ERR_NUMERIC, FMM_ERR_CUDA, FMM_ERR_OOM, FMM_ERR_COMM = 0, 2, 3, 4, 5, 6

(FMM_X_KEYS, FMM_X_PERM, FMM_X_LEVEL, FMM_X_ANCHOR, FMM_X_BEGIN, FMM_X_END, FMM_X_CHILD, FMM_X_NCHILD,
 FMM_X_PARENT, FMM_X_CENTER, FMM_X_P2P, FMM_X_M2L, FMM_X_M, FMM_X_L, FMM_X_GEOM) = range(15)

(FMM_LET_Q_SEND, FMM_LET_Q_RECV, FMM_LET_M_SEND, FMM_LET_M_RECV, FMM_LET_PHI_SEND, FMM_LET_PHI_RECV, FMM_LET_SHARED,
 FMM_LET_RANK_BEGIN, FMM_LET_Q_SEND_ROWS, FMM_LET_Q_RECV_POS, FMM_LET_SHARED_CELLS, FMM_LET_M_SEND_CELLS,
 FMM_LET_M_RECV_CELLS, FMM_LET_PHI_SEND_IDX, FMM_LET_PHI_RECV_ROWS) = range(15)
EXPORTED = ("fmm_setup", "fmm_setup_2d", "fmm_matvec", "fmm_matvec_host", "fmm_sync", "fmm_direct", "fmm_stats",
            "fmm_set_timing", "fmm_export", "fmm_destroy", "fmm_last_error", "fmm_version", "fmm_let_setup",
            "fmm_let_counts", "fmm_let_pack_q", "fmm_let_upward", "fmm_let_finish", "fmm_let_unpack",
            "fmm_let_lists_host", "fmm_stencil_apply", "fmm_precond_setup", "fmm_precond_apply", "fmm_precond_info",
            "fmm_precond_destroy", "fmm_pcg_solve", "fmm_nccl_unique_id", "fmm_setup_helmholtz",
            "fmm_matvec_helmholtz", "fmm_direct_helmholtz", "fmm_helmholtz_stencil_apply", "fmm_hprecond_setup",
            "fmm_hprecond_apply", "fmm_hprecond_info", "fmm_hprecond_destroy", "fmm_gmres_solve")


class FmmExec(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("rank", C.c_int), ("world_size", C.c_int),
                ("nccl_id", C.c_void_p)]


class FmmStats(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("n_cells", C.c_int64), ("n_leaves", C.c_int64), ("n_p2p_pairs", C.c_int64),
        ("n_m2l_pairs", C.c_int64), ("n_p2p_interactions", C.c_int64), ("own_begin", C.c_int64),
        ("own_end", C.c_int64), ("p", C.c_int32), ("ncrit", C.c_int32), ("max_level", C.c_int32),
        ("exponent", C.c_int32), ("theta", C.c_double), ("t_setup_ms", C.c_double * 8),
        ("t_matvec_ms", C.c_double * 8), ("bytes_device", C.c_int64), ("m2l_variant", C.c_int32),
        ("near_mutual", C.c_int32), ("m2l_flops_per_pair", C.c_double), ("bytes_by", C.c_int64 * 8), ("launches_total", C.c_int64),
    ]
BYTES_CATEGORIES = ("particles", "tree", "lists", "expansions", "operators", "schedule", "let", "other")


class PcgInfo(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("relres", C.c_double),
                ("t_total_ms", C.c_double), ("t_precond_ms", C.c_double)]


class FmmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"fmm status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1602_02244_b200.build` "
                          "(the CUDA path has no fallback)")
    L = C.CDLL(LIB_PATH)
    missing = [s for s in EXPORTED if not hasattr(L, s)]
    if missing:
        raise ImportError(f"{LIB_PATH} lacks {missing}: rebuild it (python -m paper_1602_02244_b200.build)")
    vp, dp, i64 = C.c_void_p, C.c_void_p, C.c_int64
    L.fmm_nccl_unique_id.argtypes = [vp]
    L.fmm_setup_helmholtz.argtypes = [C.POINTER(C.c_void_p), dp, i64, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.POINTER(FmmExec)]
    L.fmm_matvec_helmholtz.argtypes = [vp, dp, i64, dp]
    L.fmm_direct_helmholtz.argtypes = [dp, dp, i64, dp, i64, C.c_double, dp, C.POINTER(FmmExec)]
    L.fmm_setup.argtypes = [C.POINTER(C.c_void_p), dp, i64, C.c_int, C.c_int, C.c_double, C.POINTER(FmmExec)]
    L.fmm_setup_2d.argtypes = [C.POINTER(C.c_void_p), dp, i64, C.c_int, C.c_int, C.c_double, C.POINTER(FmmExec)]
    L.fmm_matvec.argtypes = [vp, dp, i64, dp, dp]
    L.fmm_matvec_host.argtypes = [vp, dp, i64, dp, dp]
    L.fmm_sync.argtypes = [vp]
    L.fmm_direct.argtypes = [dp, dp, i64, dp, i64, dp, dp, C.POINTER(FmmExec)]
    L.fmm_stats.argtypes = [vp, C.POINTER(FmmStats)]
    L.fmm_set_timing.argtypes = [vp, C.c_int]
    L.fmm_export.argtypes = [vp, C.c_int, vp, i64, C.POINTER(C.c_int64)]
    L.fmm_destroy.argtypes = [vp]
    L.fmm_destroy.restype = None
    L.fmm_last_error.restype = C.c_char_p
    L.fmm_version.restype = C.c_char_p
    L.fmm_let_setup.argtypes = [vp, C.POINTER(C.c_int64)]
    L.fmm_let_counts.argtypes = [vp, C.c_int, C.POINTER(C.c_int64)]
    L.fmm_let_pack_q.argtypes = [vp, dp, dp]
    L.fmm_let_upward.argtypes = [vp, dp, dp, dp]
    L.fmm_let_finish.argtypes = [vp, dp, dp, dp, dp]
    L.fmm_let_unpack.argtypes = [vp, dp, dp, dp, dp]
    L.fmm_let_lists_host.argtypes = [i64, C.c_int, C.c_int, C.c_int, vp, vp, i64, vp, vp, i64, vp, i64, vp, vp, i64, vp, vp,
                                     C.c_int, vp, i64, C.POINTER(C.c_int64)]
    # include/fmm_pde.h (NEXT-2)
    L.fmm_stencil_apply.argtypes = [C.c_int, dp, dp, vp]
    L.fmm_precond_setup.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                    C.POINTER(FmmExec)]
    L.fmm_precond_apply.argtypes = [vp, dp, dp]
    L.fmm_precond_info.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.fmm_precond_destroy.argtypes = [vp]
    L.fmm_precond_destroy.restype = None
    L.fmm_pcg_solve.argtypes = [C.c_int, dp, dp, vp, C.c_double, C.c_int, C.POINTER(C.c_double),
                                C.POINTER(PcgInfo), vp]
    # include/fmm_pde.h, NEXT-4 solve (Helmholtz, GMRES)
    L.fmm_helmholtz_stencil_apply.argtypes = [C.c_int, C.c_double, dp, dp, vp]
    L.fmm_hprecond_setup.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_int, C.POINTER(FmmExec)]
    L.fmm_hprecond_apply.argtypes = [vp, dp, dp]
    L.fmm_hprecond_info.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.fmm_hprecond_destroy.argtypes = [vp]
    L.fmm_hprecond_destroy.restype = None
    L.fmm_gmres_solve.argtypes = [C.c_int, C.c_double, dp, dp, vp, C.c_double, C.c_int, C.POINTER(C.c_double),
                                  C.POINTER(PcgInfo), vp]
    for nm in ("fmm_helmholtz_stencil_apply", "fmm_hprecond_setup", "fmm_hprecond_apply", "fmm_hprecond_info",
               "fmm_gmres_solve"):
        getattr(L, nm).restype = C.c_int
    for nm in ("fmm_setup", "fmm_setup_2d", "fmm_matvec", "fmm_matvec_host", "fmm_sync", "fmm_direct", "fmm_stats",
               "fmm_set_timing", "fmm_export", "fmm_let_setup", "fmm_let_counts", "fmm_let_pack_q",
               "fmm_let_upward", "fmm_let_finish", "fmm_let_unpack", "fmm_let_lists_host", "fmm_nccl_unique_id",
               "fmm_setup_helmholtz", "fmm_matvec_helmholtz", "fmm_direct_helmholtz",
               "fmm_stencil_apply",
               "fmm_precond_setup", "fmm_precond_apply", "fmm_precond_info", "fmm_pcg_solve"):
        getattr(L, nm).restype = C.c_int
    _lib = L
    return L


def check(status: int):
    if status != FMM_OK:
        raise FmmError(status, lib().fmm_last_error().decode())
