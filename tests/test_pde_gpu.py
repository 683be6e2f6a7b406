"""NEXT-2 on the GPU (include/fmm_pde.h through the C ABI) against the oracle
(oracle/pde_oracle.py): the stencil bit-exactly, the FMM preconditioner to the mat-vec's
parity level, the flexible PCG iteration by iteration, and the paper's mesh-independence
claim at the paper's own size h = 2^-5."""
import numpy as np
import pytest

from oracle import pde_oracle as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("n", [1, 2, 9, 20])
def test_stencil_bit_exact(torch_cuda, n):
    from paper_1602_02244_b200 import pde

    u = np.random.default_rng(n).standard_normal(n ** 3)
    out = pde.stencil_apply(dev(torch_cuda, u), n).cpu().numpy()
    assert np.array_equal(out, P.stencil_apply(u, n))


@pytest.mark.parametrize("n,stride,p,boundary", [(7, 1, 4, True), (7, 1, 4, False), (15, 2, 6, True),
                                                 (16, 3, 3, True)])
def test_preconditioner_matches_oracle(torch_cuda, n, stride, p, boundary):
    from paper_1602_02244_b200 import pde

    r = np.random.default_rng(7).standard_normal(n ** 3)
    M = pde.FmmPreconditioner(n, p=p, ncrit=16, theta=0.5, face_stride=stride, boundary=boundary)
    z = M.apply(dev(torch_cuda, r)).cpu().numpy()
    Mo = P.FmmPrecond(n, stride, p, 16, 0.5, boundary=boundary)
    zo = Mo.apply(r)
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)
    info = M.info()
    assert info["panels"] == (6 * ((n + stride - 1) // stride) ** 2 if boundary else 0) and info["bytes"] > 0
    assert not M.apply(dev(torch_cuda, np.zeros(n ** 3))).cpu().numpy().any()


@pytest.mark.parametrize("n,use_m", [(7, True), (15, True), (15, False)])
def test_pcg_matches_oracle(torch_cuda, n, use_m):
    from paper_1602_02244_b200 import pde

    b = np.random.default_rng(0).standard_normal(n ** 3)
    M = pde.FmmPreconditioner(n, p=4, ncrit=32, theta=0.5) if use_m else None
    x, hist, info = pde.pcg(dev(torch_cuda, b), n, M, rtol=1e-8, maxit=400)
    Mo = P.FmmPrecond(n, 1, 4, 32, 0.5) if use_m else None
    xo, ho = P.pcg(lambda v: P.stencil_apply(v, n), b, Mo.apply if Mo else None, 1e-8, 400)
    assert info["converged"] == 1 and hist[-1] <= 1e-8
    assert abs(len(hist) - len(ho)) <= 1
    k = min(len(hist), len(ho)) - 1
    assert np.allclose(hist[:k], ho[:k], rtol=1e-6, atol=0)
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-7 * np.linalg.norm(xo)
    # deterministic: a second solve is bitwise identical
    x2, hist2, _ = pde.pcg(dev(torch_cuda, b), n, M, rtol=1e-8, maxit=400)
    assert torch_cuda.equal(x, x2) and hist == hist2


def test_mesh_independence_at_paper_size(torch_cuda):
    """h = 2^-5 (n = 63, 250,047 unknowns): the FMM-preconditioned iteration count
    stays within a few of its n = 15 count while unpreconditioned CG grows like 1/h."""
    from paper_1602_02244_b200 import pde

    its = {}
    for n, stride in ((15, 1), (31, 2), (63, 2)):
        b = dev(torch_cuda, np.random.default_rng(0).standard_normal(n ** 3))
        M = pde.FmmPreconditioner(n, p=4, ncrit=64, theta=0.5, face_stride=stride)
        _, h1, i1 = pde.pcg(b, n, M, rtol=1e-8, maxit=200)
        _, h0, i0 = pde.pcg(b, n, None, rtol=1e-8, maxit=2000)
        assert i1["converged"] and i0["converged"]
        its[n] = (i1["iterations"], i0["iterations"])
    assert max(v[0] for v in its.values()) - min(v[0] for v in its.values()) <= 3
    assert its[63][1] > 3 * its[15][1] and its[63][0] * 10 < its[63][1]


def test_usage_errors(torch_cuda):
    import ctypes

    from paper_1602_02244_b200 import _native as N

    L = N.lib()
    assert L.fmm_stencil_apply(0, None, None, None) == N.FMM_ERR_USAGE
    h = ctypes.c_void_p()
    ex = N.FmmExec(0, None, 0, 1)
    assert L.fmm_precond_setup(ctypes.byref(h), 7, 0, 4, 16, 0.5, 1, ctypes.byref(ex)) == N.FMM_ERR_USAGE
    assert L.fmm_precond_setup(ctypes.byref(h), 7, 1, 4, 16, 0.9, 1, ctypes.byref(ex)) == N.FMM_ERR_USAGE
    assert L.fmm_pcg_solve(7, None, None, None, 1e-8, 10, None, None, None) == N.FMM_ERR_USAGE
