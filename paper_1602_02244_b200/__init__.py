"""B200-native 3D Laplace FMM mat-vec (arXiv:1602.02244 hot path).

``Plan(points, p, ncrit, theta).matvec(q, grad=...)`` and ``direct(...)`` over
the C ABI of ``include/fmm.h`` (libfmm.so, hand-written CUDA for sm_100a).
"""
from ._native import FmmError, LIB_PATH  # noqa: F401
from .fmm import HelmholtzPlan, Plan, Plan2D, direct, direct_helmholtz, version  # noqa: F401
