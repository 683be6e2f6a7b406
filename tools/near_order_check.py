"""Accuracy of the near field's 1/r refinement order (build with -DFMM_NEAR_ORDER=2 or 3):
rel-L2 of the GPU mat-vec against the oracle on 10^4 sampled targets at full sizes, and timings.

    python tools/near_order_check.py c2 c3 c4
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

for name in sys.argv[1:]:
    cfg = F.CONFIGS[name]
    x, q = F.make_config(name)
    pl = Plan(torch.from_numpy(x).cuda(), cfg.p, cfg.ncrit, cfg.theta)
    qd = torch.from_numpy(q).cuda()
    out = pl.matvec(qd, grad=cfg.grad)
    torch.cuda.synchronize()
    pl.set_timing(True)
    ts = []
    for _ in range(5):
        pl.matvec(qd, grad=cfg.grad)
        ts.append(pl.stats()["t_matvec_ms"][:5])
    t = np.median(np.array(ts), axis=0)
    phi = (out[0] if cfg.grad else out).cpu().numpy()
    T = F.target_sample(cfg.n, 10_000)
    orc = O.Plan(x, cfg.p, cfg.ncrit, cfg.theta)
    res = orc.eval(q, grad=cfg.grad, targets=T, nthreads=O.default_threads())
    po = res[0] if cfg.grad else res
    e = O.rel_l2(phi[T], po)
    eg = O.rel_l2(out[1].cpu().numpy()[T], res[1]) if cfg.grad else float("nan")
    print(f"{name}: rel_l2(phi) {e:.2e}  rel_l2(grad) {eg:.2e}  near {t[2]:.3f} ms  total {t[4]:.3f} ms", flush=True)
