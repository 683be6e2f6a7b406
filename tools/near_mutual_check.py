"""Mutual (each unordered leaf pair once) vs directed P2P near field: stage timings and agreement.

    python tools/near_mutual_check.py [config ...]      (default: c3 c2 c4; potentials only)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402


def run(xd, qd, cfg, mutual, reps=7):
    os.environ["FMM_NEAR_MUTUAL"] = "1" if mutual else "0"
    pl = Plan(xd, cfg.p, cfg.ncrit, cfg.theta)
    out = pl.matvec(qd)
    torch.cuda.synchronize()
    pl.set_timing(True)
    ts = []
    for _ in range(reps):
        pl.matvec(qd)
        ts.append(pl.stats()["t_matvec_ms"][:5])
    pl.set_timing(False)
    st = pl.stats()
    return out, np.median(np.array(ts), axis=0), st


def main():
    for name in sys.argv[1:] or ["c3", "c2", "c4"]:
        cfg = F.CONFIGS[name]
        x, q = F.make_config(name)
        xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
        pm, tm, sm = run(xd, qd, cfg, True)
        pd, td, sd = run(xd, qd, cfg, False)
        rel = (torch.linalg.norm(pm - pd) / torch.linalg.norm(pd)).item()
        print(f"{name}: mutual={sm['near_mutual']} near {tm[2]:.3f} ms (directed {td[2]:.3f}) total {tm[4]:.3f} "
              f"(directed {td[4]:.3f}) relL2 {rel:.2e} mutual bytes {sm['bytes_by']['particles'] / 1e6:.0f} MB",
              flush=True)


if __name__ == "__main__":
    main()
