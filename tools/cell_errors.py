"""Worst per-cell relative error of the GPU multipoles / local expansions against the oracle
(the stage gates of tests/test_gpu_parity.py), per M2L variant.

    python tools/cell_errors.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402

CASES = [("cube", 1000, 4, 32, 0.4), ("cube", 20000, 10, 64, 0.4), ("plummer", 30000, 8, 64, 0.5),
         ("sphere", 30000, 12, 128, 0.4), ("plummer", 5000, 3, 7, 0.3)]
for dist, n, p, ncrit, theta in CASES:
    x, q = F.make(dist, n)
    orc = O.Plan(x, p, ncrit, theta)
    orc.eval(q, nthreads=O.default_threads())
    M, L = orc.expansions()
    for v in ("4", "3"):
        os.environ["FMM_M2L_VARIANT"] = v
        pl = Plan(torch.from_numpy(x).cuda(), p, ncrit, theta)
        pl.matvec(torch.from_numpy(q).cuda())
        torch.cuda.synchronize()
        Mg, Lg = pl.export("M"), pl.export("L")
        em = np.linalg.norm(Mg - M, axis=1) / np.maximum(np.linalg.norm(M, axis=1), 1e-300)
        el = np.linalg.norm(Lg - L, axis=1) / np.maximum(np.linalg.norm(L, axis=1), 1e-300)
        k = int(np.argmax(el))
        print(f"{dist} n={n} p={p} v{v}: worst M {em.max():.2e}  worst L {el.max():.2e} (cell {k}, "
              f"{(el > 1e-12).sum()} cells > 1e-12 of {len(el)})", flush=True)
