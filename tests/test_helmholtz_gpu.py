"""NEXT-4 on the GPU: the Helmholtz FMM mat-vec (include/fmm_helmholtz.h, csrc/helmholtz.cu) through
the C ABI against the independent numpy oracle (oracle/helmholtz_oracle.py) on the same tree and
lists: rel-L2 <= 1e-11 (the north_star gate), the direct sum against the oracle's, reductions,
errors, and at the paper's lattice (63^3 nodes of [-1,1]^3, h = 2^-5, kappa = 7)
agreement with the direct sum at the truncation level."""
import numpy as np
import pytest

import fmm_inputs as F
from oracle import helmholtz_oracle as H

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    from paper_1602_02244_b200 import build

    build.build()
    return torch


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def charges(n, seed=1):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def test_direct_matches_oracle(torch_cuda):
    torch = torch_cuda
    from paper_1602_02244_b200 import direct_helmholtz

    x, _ = F.cube(1500, seed=3)
    t, _ = F.plummer(300, seed=4)
    q = charges(1500)
    for tgt in (None, t):
        g = direct_helmholtz(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda(), 7.0,
                             None if tgt is None else torch.from_numpy(tgt).cuda())
        assert rel(g.cpu().numpy(), H.direct(x, q, 7.0, tgt=tgt)) < 1e-13


CASES = [("cube", 1500, 4, 32, 0.4, 7.0), ("cube", 2000, 6, 48, 0.4, 7.0), ("plummer", 2000, 5, 24, 0.5, 3.0),
         ("sphere", 1500, 6, 40, 0.4, 12.0), ("cube", 1200, 2, 16, 0.5, 0.5), ("plummer", 800, 0, 8, 0.3, 7.0),
         ("lattice", 1728, 5, 32, 0.4, 7.0)]


@pytest.mark.parametrize("dist,n,p,ncrit,theta,kappa", CASES)
def test_fmm_matches_oracle(torch_cuda, dist, n, p, ncrit, theta, kappa):
    torch = torch_cuda
    from paper_1602_02244_b200 import HelmholtzPlan

    x, _ = F.make(dist, n)
    q = charges(n)
    pl = HelmholtzPlan(torch.from_numpy(x).cuda(), p, ncrit, theta, kappa)
    phi = pl.matvec(torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    pl.sync()
    ref = H.fmm_helmholtz(x, q, p, ncrit, theta, kappa)
    assert rel(phi.cpu().numpy(), ref) <= TOL
    st = pl.stats()
    assert st["m2l_variant"] == 5 and st["m2l_flops_per_pair"] == 8.0 * (p + 1) ** 4


def test_reductions_and_determinism(torch_cuda):
    torch = torch_cuda
    from paper_1602_02244_b200 import HelmholtzPlan

    x, _ = F.cube(700, seed=8)
    q = charges(700, 2)
    d = H.direct(x, q, 7.0)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    for ncrit, theta in ((16, 1e-6), (700, 0.4)):  # every pair P2P / a single leaf: the direct sum
        phi = HelmholtzPlan(xd, 4, ncrit, theta, 7.0).matvec(qd).cpu().numpy()
        assert rel(phi, d) < 1e-13
    pl = HelmholtzPlan(xd, 5, 16, 0.4, 7.0)
    a, b = pl.matvec(qd), pl.matvec(qd)
    assert torch.equal(a, b)


def test_usage_errors(torch_cuda):
    torch = torch_cuda
    from paper_1602_02244_b200 import FmmError, HelmholtzPlan, Plan

    x, q = F.cube(200)
    xd = torch.from_numpy(x).cuda()
    for args in ((4, 16, 0.4, 0.0), (11, 16, 0.4, 7.0), (4, 16, 0.4, float("nan"))):
        with pytest.raises(FmmError) as e:
            HelmholtzPlan(xd, *args)
        assert e.value.status == 2
    pl = HelmholtzPlan(xd, 4, 16, 0.4, 7.0)
    with pytest.raises(FmmError):  # a Helmholtz plan has no real-kernel mat-vec
        Plan.matvec(pl, torch.from_numpy(q).cuda())
    lap = Plan(xd, 4, 16, 0.4)
    with pytest.raises(FmmError):
        HelmholtzPlan.matvec(lap, torch.from_numpy(charges(200)).cuda())


def test_paper_lattice_against_direct(torch_cuda):
    """The paper's §4.2 geometry: the 63^3 interior nodes of [-1,1]^3 (h = 2^-5), kappa = 7; the FMM
    agrees with the O(N^2) sum (GPU) on 2000 sampled nodes at the truncation level, decreasing in p."""
    torch = torch_cuda
    from paper_1602_02244_b200 import HelmholtzPlan, direct_helmholtz

    n1 = 63
    g = -1 + (np.arange(n1) + 1) * (2.0 / (n1 + 1))
    x = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    q = charges(x.shape[0], 5)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    T = np.sort(np.random.default_rng(12345).choice(x.shape[0], 2000, replace=False))
    ref = direct_helmholtz(xd, qd, 7.0, xd[torch.from_numpy(T).cuda()]).cpu().numpy()
    errs = []
    for p in (4, 8):
        phi = HelmholtzPlan(xd, p, 64, 0.4, 7.0).matvec(qd).cpu().numpy()
        errs.append(rel(phi[T], ref))
    assert errs[1] < errs[0] / 10 and errs[1] < 1e-3  # measured 1.8e-2 (p = 4), 3.0e-4 (p = 8)
