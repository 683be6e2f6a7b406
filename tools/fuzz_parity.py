"""Randomised parity sweep of the CUDA mat-vec against the oracle (3D and 2D): random
distribution, size, order, ncrit, theta, scale/offset of the coordinates, coincident points and
gradients. Prints one line per case and a summary; exits non-zero on any case above 1e-11.

    python tools/fuzz_parity.py [--cases 40] [--seed 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from oracle import fmm2d_oracle as D  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1602_02244_b200 import Plan, Plan2D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=40)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    worst = 0.0
    bad = 0
    for c in range(args.cases):
        dim = 2 if rng.random() < 0.25 else 3
        n = int(rng.integers(1, 30000))
        p = int(rng.integers(0, 17))
        ncrit = int(rng.integers(1, 200))
        theta = float(rng.uniform(0.05, 0.57))
        dist = rng.choice(["cube", "plummer", "sphere", "lattice"])
        x, q = F.make(str(dist), n, seed=int(rng.integers(1 << 30)))
        n = x.shape[0]
        scale = 10.0 ** rng.uniform(-6, 6)
        x = x * scale + rng.uniform(-1e3, 1e3, 3) * scale
        if rng.random() < 0.2 and n > 10:  # coincident points
            k = int(rng.integers(2, min(n, 300)))
            x[:k] = x[int(rng.integers(n))]
        grad = bool(rng.random() < 0.5)
        try:
            if dim == 3:
                pl = Plan(torch.from_numpy(x).cuda(), p, ncrit, theta)
                out = pl.matvec(torch.from_numpy(q).cuda(), grad=grad)
                res = O.fmm(x, q, p, ncrit, theta, grad=grad, nthreads=O.default_threads())
            else:
                xy = np.ascontiguousarray(x[:, :2])
                pl = Plan2D(torch.from_numpy(xy).cuda(), p, ncrit, theta)
                out = pl.matvec(torch.from_numpy(q).cuda(), grad=grad)
                res = D.fmm2d(xy, q, p, ncrit, theta, grad=grad)
            torch.cuda.synchronize()
            phi = (out[0] if grad else out).cpu().numpy()
            po = res[0] if grad else res
            e = O.rel_l2(phi, po)
            if grad:
                g = out[1].cpu().numpy()[:, :dim]
                e = max(e, O.rel_l2(g, res[1][:, :dim]))
            status = "ok" if e <= 1e-11 else "FAIL"
        except Exception as ex:  # report and continue
            e, status = float("nan"), f"ERROR {ex}"
        worst = max(worst, e) if e == e else worst
        bad += status != "ok"
        print(f"case {c:3d} {dim}D {dist:8s} n={n:6d} p={p:2d} ncrit={ncrit:3d} theta={theta:.3f} "
              f"scale={scale:.1e} grad={int(grad)} rel={e:.2e} {status}", flush=True)
    print(f"summary: {args.cases} cases, {bad} above 1e-11 or failed, worst {worst:.2e}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
