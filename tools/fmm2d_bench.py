"""NEXT-3 measurement: the 2D log-kernel mat-vec on one B200 (fmm_setup_2d). Uniform 2D lattice
(the paper's §4.1 geometry) and uniform random points; CUDA-event stage times.

    python tools/fmm2d_bench.py [--m 1000] [--ps 4 8 12]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_02244_b200 import Plan2D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1000)
    ap.add_argument("--ps", nargs="+", type=int, default=[4, 8, 12])
    ap.add_argument("--ncrit", type=int, default=64)
    ap.add_argument("--theta", type=float, default=0.5)
    args = ap.parse_args()
    m = args.m
    g1 = -1.0 + (np.arange(m) + 1.0) * (2.0 / (m + 1))
    lat = np.stack(np.meshgrid(g1, g1, indexing="ij"), -1).reshape(-1, 2)
    rnd = np.random.default_rng(0).random((m * m, 2)) * 2 - 1
    q = np.random.default_rng(1).uniform(-1, 1, m * m)
    qd = torch.from_numpy(q).cuda()
    print("| points | N | p | upward ms | M2L ms | downward ms | near ms | mat-vec ms | particles/s | M2L pairs | P2P interactions |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for name, xy in (("2D lattice", lat), ("uniform square", rnd)):
        for p in args.ps:
            pl = Plan2D(torch.from_numpy(xy).cuda(), p, args.ncrit, args.theta)
            pl.set_timing(True)
            ts = []
            for i in range(7):
                pl.matvec(qd)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(pl.stats()["t_matvec_ms"])
            t = [statistics.median(x[k] for x in ts) for k in range(5)]
            st = pl.stats()
            print(f"| {name} | {xy.shape[0]} | {p} | {t[0]:.3f} | {t[1]:.3f} | {t[3]:.3f} | {t[2]:.3f} | {t[4]:.3f} | "
                  f"{xy.shape[0] / (t[4] * 1e-3):.3g} | {st['n_m2l_pairs']} | {st['n_p2p_interactions']} |", flush=True)


if __name__ == "__main__":
    main()
