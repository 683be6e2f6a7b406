"""NEXT-4 solve measurement: Helmholtz-FMM-preconditioned GMRES for the 3D Dirichlet
Helmholtz equation -Delta u - kappa^2 u = f on the [-1,1]^3 lattice (Fig 6 at
h = 2^-5 and kappa = 7; convergence independent of the problem size), one B200.

Per lattice size and FMM accuracy (order p; epsilon = the Helmholtz FMM's measured relative L2 error
of the volume potential against fmm_direct_helmholtz on the same points): setup time of the
preconditioner (includes the complex Newton-Schulz inverse of the boundary matrix), GMRES iterations
to rtol, solve time, time inside M, and unpreconditioned GMRES for reference. Random real
right-hand side (numpy PCG64 seed 0). Prints a markdown table.

    python tools/gmres_bench.py [--ns 15 31 63] [--ps 1 2 4 8] [--kappa 7]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02244_b200 import HelmholtzPlan, direct_helmholtz, pde  # noqa: E402
from tools.pcg_bench import points  # noqa: E402


def fmm_eps(n, stride, p, ncrit, theta, kappa):
    xyz = torch.from_numpy(points(n, stride)).cuda()
    rng = np.random.default_rng(1)
    q = torch.from_numpy(rng.standard_normal(xyz.shape[0]) + 1j * rng.standard_normal(xyz.shape[0])).cuda()
    pl = HelmholtzPlan(xyz, p, ncrit, theta, kappa)
    phi = pl.matvec(q)
    ref = direct_helmholtz(xyz, q, kappa)
    torch.cuda.synchronize()
    return float(torch.linalg.norm(phi - ref) / torch.linalg.norm(ref))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", nargs="+", type=int, default=[15, 31, 63])
    ap.add_argument("--ps", nargs="+", type=int, default=[1, 2, 4, 8])
    ap.add_argument("--kappa", type=float, default=7.0)
    ap.add_argument("--ncrit", type=int, default=64)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--rtol", type=float, default=1e-6)
    args = ap.parse_args()
    k = args.kappa
    print(f"kappa = {k}, rtol = {args.rtol}, ncrit = {args.ncrit}, theta = {args.theta}\n")
    print("| h | n^3 | panels | M | epsilon (FMM rel. L2) | setup ms | iterations | solve ms | in M ms | ms / iteration |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for n in args.ns:
        stride = 1 if n < 32 else 2
        b = torch.from_numpy(np.random.default_rng(0).standard_normal(n ** 3).astype(np.complex128)).cuda()
        x, hist, info = pde.gmres(b, n, k, None, rtol=args.rtol, maxit=1500 if n < 40 else 600)
        h = f"2^-{int(round(-np.log2(2.0 / (n + 1))))}"
        conv = "" if info["converged"] else " (not converged)"
        print(f"| {h} | {n ** 3} | - | identity | - | - | {info['iterations']}{conv} | {info['t_total_ms']:.1f} | - | "
              f"{info['t_total_ms'] / max(1, info['iterations']):.3f} |", flush=True)
        del x
        torch.cuda.empty_cache()
        for p in args.ps:
            eps = fmm_eps(n, stride, p, args.ncrit, args.theta, k)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            M = pde.HelmholtzPreconditioner(n, k, p=p, ncrit=args.ncrit, theta=args.theta, face_stride=stride)
            torch.cuda.synchronize()
            ts = (time.perf_counter() - t0) * 1e3
            x, hist, info = pde.gmres(b, n, k, M, rtol=args.rtol, maxit=200)
            mi = M.info()
            conv = "" if info["converged"] else " (not converged)"
            print(f"| {h} | {n ** 3} | {mi['panels']} | FMM p={p} | {eps:.1e} | {ts:.0f} | {info['iterations']}{conv} | "
                  f"{info['t_total_ms']:.1f} | {info['t_precond_ms']:.1f} | "
                  f"{info['t_total_ms'] / max(1, info['iterations']):.2f} |", flush=True)
            del M, x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
