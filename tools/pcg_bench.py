"""NEXT-2 measurement: FMM-preconditioned CG for the 3D Dirichlet Laplace
equation on the [-1,1]^3 lattice (Fig 5 at h = 2^-5), one B200.

Per lattice size and FMM accuracy (order p; epsilon = the FMM's measured relative L2 error of
the volume potential against fmm_direct on the same points): setup time of the preconditioner,
Krylov iterations to rtol = 1e-8, solve time, time inside M, and unpreconditioned CG for
reference. Random right-hand side (numpy PCG64 seed 0). Prints a markdown table.

    python tools/pcg_bench.py [--ns 15 31 63] [--ps 1 2 4 8]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02244_b200 import Plan, direct, pde  # noqa: E402


def points(n, stride):
    h = 2.0 / (n + 1)
    c = -1.0 + (np.arange(n) + 1.0) * h
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    X = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    cf = -1.0 + (np.arange(0, n, stride) + 1.0) * h
    v, u = np.meshgrid(cf, cf, indexing="ij")
    F = []
    for axis in range(3):
        for side in (-1.0, 1.0):
            f = np.zeros((u.size, 3))
            o = [d for d in range(3) if d != axis]
            f[:, axis], f[:, o[0]], f[:, o[1]] = side, u.ravel(), v.ravel()
            F.append(f)
    return np.concatenate([X] + F, 0)


def fmm_eps(n, stride, p, ncrit, theta):
    xyz = torch.from_numpy(points(n, stride)).cuda()
    q = torch.from_numpy(np.random.default_rng(1).standard_normal(xyz.shape[0])).cuda()
    phi = Plan(xyz, p, ncrit, theta).matvec(q)
    ref = direct(xyz, q)
    torch.cuda.synchronize()
    return float(torch.linalg.norm(phi - ref) / torch.linalg.norm(ref))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", nargs="+", type=int, default=[15, 31, 63])
    ap.add_argument("--ps", nargs="+", type=int, default=[1, 2, 4, 8])
    ap.add_argument("--ncrit", type=int, default=64)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--rtol", type=float, default=1e-8)
    args = ap.parse_args()
    print("| h | n^3 | panels | M | epsilon (FMM rel. L2) | setup ms | iterations | solve ms | in M ms | ms / iteration |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for n in args.ns:
        stride = 1 if n < 32 else 2
        b = torch.from_numpy(np.random.default_rng(0).standard_normal(n ** 3)).cuda()
        x, hist, info = pde.pcg(b, n, None, rtol=args.rtol, maxit=5000)
        h = f"2^-{int(round(-np.log2(2.0 / (n + 1))))}"
        print(f"| {h} | {n ** 3} | - | identity | - | - | {info['iterations']} | {info['t_total_ms']:.1f} | - | "
              f"{info['t_total_ms'] / max(1, info['iterations']):.3f} |", flush=True)
        for p in args.ps:
            eps = fmm_eps(n, stride, p, args.ncrit, args.theta)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            M = pde.FmmPreconditioner(n, p=p, ncrit=args.ncrit, theta=args.theta, face_stride=stride)
            torch.cuda.synchronize()
            ts = (time.perf_counter() - t0) * 1e3
            x, hist, info = pde.pcg(b, n, M, rtol=args.rtol, maxit=500)
            mi = M.info()
            print(f"| {h} | {n ** 3} | {mi['panels']} | FMM p={p} | {eps:.1e} | {ts:.0f} | {info['iterations']} | "
                  f"{info['t_total_ms']:.1f} | {info['t_precond_ms']:.1f} | "
                  f"{info['t_total_ms'] / max(1, info['iterations']):.2f} |", flush=True)
            del M
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
