"""One plan + a few mat-vecs of a BASELINE config, for ncu captures of single kernels.

    FMM_M2L_VARIANT=4 python tools/prof_matvec.py c3 [reps] [--grad]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
cfg = F.CONFIGS[name]
x, q = F.make_config(name)
pl = Plan(torch.from_numpy(x).cuda(), cfg.p, cfg.ncrit, cfg.theta)
qd = torch.from_numpy(q).cuda()
for _ in range(reps):
    pl.matvec(qd, grad="--grad" in sys.argv or cfg.grad)
torch.cuda.synchronize()
pl.sync()
print("ok", pl.stats()["m2l_variant"])
