"""Stage times of the mat-vec at low order p on the h = 2^-5 lattice (+ face panels), M2L v1/v2/v3."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np, torch
from pcg_bench import points
for p in (1, 2, 3, 4, 5, 6, 8):
    for v in ("1", "2", "3"):
        os.environ["FMM_M2L_VARIANT"] = v
        from paper_1602_02244_b200 import Plan
        xyz = torch.from_numpy(points(63, 2)).cuda()
        q = torch.from_numpy(np.random.default_rng(1).standard_normal(xyz.shape[0])).cuda()
        pl = Plan(xyz, p, 64, 0.5)
        pl.set_timing(True)
        ts = []
        for i in range(5):
            pl.matvec(q); torch.cuda.synchronize()
            ts.append(pl.stats()["t_matvec_ms"])
        st = pl.stats()
        t = [statistics.median(x[k] for x in ts[2:]) for k in range(5)]
        print(f"p={p} req v{v} -> v{st['m2l_variant']}: up {t[0]:.3f} m2l {t[1]:.3f} near {t[2]:.3f} down {t[3]:.3f} total {t[4]:.3f} pairs {st['n_m2l_pairs']}", flush=True)
