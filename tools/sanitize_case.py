"""Small mat-vecs for compute-sanitizer (racecheck / memcheck): configs[0] and a
configs[1]-recipe case at 20K points (p = 10, gradients), default kernels, plus the collective
(one-rank NCCL) path and small M2L v4 units.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402

for dist, n, p, ncrit, theta in (("cube", 1000, 4, 32, 0.4), ("cube", 20000, 10, 64, 0.4),
                                 ("plummer", 8000, 8, 32, 0.5)):
    x, q = F.make(dist, n)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    pl = Plan(xd, p, ncrit, theta)
    phi, g = pl.matvec(qd, grad=True)
    torch.cuda.synchronize()
    pl.sync()
    print(dist, n, p, "ok", float(phi.abs().max()), flush=True)
    if "--collective" in sys.argv:
        from paper_1602_02244_b200.fmm import nccl_unique_id

        pc = Plan(xd, p, ncrit, theta, world=1, nccl_id=nccl_unique_id())
        pc.matvec(qd)
        torch.cuda.synchronize()
        print("collective ok", flush=True)
