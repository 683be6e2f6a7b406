"""Setup (precalculation) of one BASELINE config: stage times of a few plans,
then (under ncu) one plan's kernels with their DRAM bytes — the setup's HBM roofline.

    python tools/prof_setup.py c3 [plans]
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
        --log-file gpurun_out/setup.csv python tools/prof_setup.py c3 1
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = F.CONFIGS[name]
x, _ = F.make_config(name)
xd = torch.from_numpy(x).cuda()
torch.cuda.synchronize()
for i in range(k):
    t0 = time.perf_counter()
    pl = Plan(xd, cfg.p, cfg.ncrit, cfg.theta)
    wall = (time.perf_counter() - t0) * 1e3
    st = pl.stats()
    ts = st["t_setup_ms"]
    print(f"{name} plan {i}: setup {ts[3]:.1f} ms (tree {ts[1]:.1f}, traversal {ts[2]:.1f}, operators+rest "
          f"{ts[3] - ts[1] - ts[2]:.1f}) wall {wall:.1f} ms", flush=True)
    del pl
