"""Quick GPU check of M2L v4 against v3 and the oracle, and per-stage timings.

    python tools/v4_check.py [config ...]      (default: c1 small cases, then c2, c3)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402


def run(x, q, p, ncrit, theta, variant, grad=False, reps=5):
    os.environ["FMM_M2L_VARIANT"] = str(variant)
    pl = Plan(torch.from_numpy(x).cuda(), p, ncrit, theta)
    qd = torch.from_numpy(q).cuda()
    out = pl.matvec(qd, grad=grad)
    torch.cuda.synchronize()
    pl.sync()
    pl.set_timing(True)
    ts = []
    for _ in range(reps):
        pl.matvec(qd, grad=grad)
        ts.append(pl.stats()["t_matvec_ms"][:5])
    pl.set_timing(False)
    st = pl.stats()
    phi = (out[0] if grad else out).cpu().numpy()
    return phi, np.median(np.array(ts), axis=0), st


def main():
    if "--time" in sys.argv:  # timings of the default variant only
        for name in [a for a in sys.argv[1:] if not a.startswith("--")]:
            cfg = F.CONFIGS[name]
            x, q = F.make_config(name)
            _, t, st = run(x, q, cfg.p, cfg.ncrit, cfg.theta, os.environ.get("FMM_M2L_VARIANT", 4))
            print(f"{name} [{os.environ.get('FMM_V4_WARPS', '-')}]: stages {np.round(t, 3)}", flush=True)
        return
    small = [("cube", 1000, 4, 32, 0.4), ("cube", 20000, 10, 64, 0.4), ("plummer", 30000, 8, 64, 0.5),
             ("sphere", 30000, 12, 128, 0.4), ("plummer", 5000, 3, 7, 0.3), ("cube", 4000, 2, 16, 0.5),
             ("cube", 4000, 7, 16, 0.5)]
    for dist, n, p, ncrit, theta in small:
        x, q = getattr(F, dist)(n)
        po = O.fmm(x, q, p, ncrit, theta)
        p4, t4, s4 = run(x, q, p, ncrit, theta, 4)
        p3, t3, _ = run(x, q, p, ncrit, theta, 3)
        print(f"{dist} n={n} p={p}: v4 variant={s4['m2l_variant']} relL2(v4,oracle)={O.rel_l2(p4, po):.2e} "
              f"relL2(v3,oracle)={O.rel_l2(p3, po):.2e}  m2l v4 {t4[1]:.3f} ms v3 {t3[1]:.3f} ms", flush=True)
    for name in sys.argv[1:] or ["c2", "c3"]:
        cfg = F.CONFIGS[name]
        x, q = F.make_config(name)
        p4, t4, s4 = run(x, q, cfg.p, cfg.ncrit, cfg.theta, 4)
        p3, t3, s3 = run(x, q, cfg.p, cfg.ncrit, cfg.theta, 3)
        print(f"{name}: relL2(v4, v3)={O.rel_l2(p4, p3):.2e}  v4 stages {np.round(t4, 3)}  v3 stages {np.round(t3, 3)}"
              f"  pairs {s4['n_m2l_pairs']}  v4 flops/pair {s4['m2l_flops_per_pair']:.0f} "
              f"-> {s4['m2l_flops_per_pair'] * s4['n_m2l_pairs'] / (t4[1] * 1e-3) / 1e12:.2f} TF", flush=True)


if __name__ == "__main__":
    main()
