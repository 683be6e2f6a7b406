"""NEXT-4 measurement: the Helmholtz FMM mat-vec on the paper's lattice (63^3 interior nodes of
[-1,1]^3, h = 2^-5, kappa = 7) for several orders: setup and mat-vec time
(CUDA events), M2L classes, and the error against the direct sum on 2000 sampled nodes.

    python tools/helmholtz_bench.py [p ...]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1602_02244_b200 import HelmholtzPlan, direct_helmholtz  # noqa: E402

n1, kappa = 63, 7.0
g = -1 + (np.arange(n1) + 1) * (2.0 / (n1 + 1))
x = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
rng = np.random.default_rng(5)
q = rng.uniform(-1, 1, len(x)) + 1j * rng.uniform(-1, 1, len(x))
xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
T = np.sort(np.random.default_rng(12345).choice(len(x), 2000, replace=False))
ref = direct_helmholtz(xd, qd, kappa, xd[torch.from_numpy(T).cuda()]).cpu().numpy()
print(f"| p | setup (ms) | mat-vec (ms) | M2L pairs | M2L classes | rel-L2 vs direct (2000 nodes) |")
print("|---|---|---|---|---|---|")
for p in [int(a) for a in sys.argv[1:]] or [2, 4, 6, 8, 10]:
    t0 = time.perf_counter()
    pl = HelmholtzPlan(xd, p, 64, 0.4, kappa)
    torch.cuda.synchronize()
    ts = (time.perf_counter() - t0) * 1e3
    phi = pl.matvec(qd)
    torch.cuda.synchronize()
    tm = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pl.matvec(qd, out=phi)
        b.record()
        b.synchronize()
        tm.append(a.elapsed_time(b))
    st = pl.stats()
    err = np.linalg.norm(phi.cpu().numpy()[T] - ref) / np.linalg.norm(ref)
    print(f"| {p} | {ts:.0f} | {np.median(tm):.2f} | {st['n_m2l_pairs']} | - | {err:.2e} |", flush=True)
