"""NEXT-3 on the GPU: the 2D log-kernel mat-vec (fmm_setup_2d + fmm_matvec through the C ABI)
against the 2D oracle (oracle/fmm2d_oracle.py) on the same tree and lists: random, lattice
(PAPER.md:386), coincident and large-coordinate inputs (the 2^-e rescale of the logarithm),
gradients, determinism, errors."""
import ctypes

import numpy as np
import pytest

from oracle import fmm2d_oracle as D

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def run(torch, xy, q, p, ncrit, theta):
    from paper_1602_02244_b200 import Plan2D

    pl = Plan2D(torch.from_numpy(np.ascontiguousarray(xy)).cuda(), p, ncrit, theta)
    phi, g = pl.matvec(torch.from_numpy(np.ascontiguousarray(q)).cuda(), grad=True)
    torch.cuda.synchronize()
    return pl, phi.cpu().numpy(), g.cpu().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,p,ncrit,theta", [(20000, 4, 32, 0.5), (20000, 8, 64, 0.4), (8000, 12, 16, 0.5),
                                             (8000, 16, 40, 0.3), (5000, 0, 16, 0.5), (5000, 1, 8, 0.5)])
def test_matches_oracle(torch_cuda, n, p, ncrit, theta):
    rng = np.random.default_rng(p)
    xy = rng.random((n, 2)) * 2 - 1
    q = rng.uniform(-1, 1, n)
    _, phi, g = run(torch_cuda, xy, q, p, ncrit, theta)
    po, go = D.fmm2d(xy, q, p, ncrit, theta, grad=True)
    assert rel(phi, po) <= TOL and rel(g[:, :2], go) <= TOL
    assert not g[:, 2].any()


@pytest.mark.parametrize("case", ["lattice", "coincident", "large_coords", "clustered", "single", "two"])
def test_edge_cases(torch_cuda, case):
    rng = np.random.default_rng(9)
    p, ncrit, theta = 8, 16, 0.5
    if case == "lattice":  # the paper's §4.1 geometry: points on cell faces
        g1 = np.arange(120) / 119.0
        xy = np.stack(np.meshgrid(g1, g1, indexing="ij"), -1).reshape(-1, 2)
    elif case == "coincident":
        xy = rng.random((3000, 2))
        xy[100:400] = xy[7]
    elif case == "large_coords":  # normalisation exponent e > 0: log rescale path
        xy = rng.random((5000, 2)) * 3000.0 + 1e4
    elif case == "clustered":
        xy = np.r_[rng.normal(0, 1e-3, (3000, 2)), rng.random((3000, 2)) * 10]
    elif case == "single":
        xy = np.array([[0.3, 0.4]])
    else:
        xy = np.array([[0.0, 0.0], [3.0, 4.0]])
    q = rng.uniform(-1, 1, xy.shape[0])
    _, phi, g = run(torch_cuda, xy, q, p, ncrit, theta)
    po, go = D.fmm2d(xy, q, p, ncrit, theta, grad=True)
    assert np.isfinite(phi).all() and np.isfinite(g).all()
    if case in ("single",):
        assert phi.tolist() == [0.0]
        return
    assert rel(phi, po) <= TOL and rel(g[:, :2], go) <= TOL
    if case == "two":
        assert np.allclose(phi, [-q[1] * np.log(5.0), -q[0] * np.log(5.0)], rtol=1e-15)


def test_truncation_vs_direct_and_determinism(torch_cuda):
    rng = np.random.default_rng(1)
    xy = rng.random((4000, 2))
    q = rng.uniform(-1, 1, 4000)
    pd = D.direct2d(xy, q)
    errs = [rel(run(torch_cuda, xy, q, p, 32, 0.5)[1], pd) for p in (4, 8, 16)]
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-8
    pl, a, ga = run(torch_cuda, xy, q, 10, 32, 0.5)
    b, gb = pl.matvec(torch_cuda.from_numpy(q).cuda(), grad=True)
    assert np.array_equal(a, b.cpu().numpy()) and np.array_equal(ga, gb.cpu().numpy())
    st = pl.stats()
    assert st["m2l_variant"] == 0 and st["m2l_flops_per_pair"] == 8.0 * 11 ** 2


def test_usage(torch_cuda):
    from paper_1602_02244_b200 import _native as N

    L = N.lib()
    h = ctypes.c_void_p()
    ex = N.FmmExec(0, None, 0, 2)
    x = torch_cuda.zeros(10, 2, dtype=torch_cuda.float64, device="cuda")
    assert L.fmm_setup_2d(ctypes.byref(h), ctypes.c_void_p(x.data_ptr()), 10, 4, 8, 0.4,
                          ctypes.byref(ex)) == N.FMM_ERR_USAGE
    ex1 = N.FmmExec(0, None, 0, 1)
    assert L.fmm_setup_2d(ctypes.byref(h), None, 10, 4, 8, 0.4, ctypes.byref(ex1)) == N.FMM_ERR_USAGE


def test_near_log_accuracy(torch_cuda):
    """The near field's table-driven logarithm (fmm2d.cu log_tab) against numpy's log over
    distances 1e-12 .. 1e5 (every table entry and binade), and the subnormal-r^2 fallback."""
    rng = np.random.default_rng(12)
    worst = 0.0
    for r in np.r_[10.0 ** rng.uniform(-12, 5, 300), 2.0 ** np.arange(-30, 16) * (1 + 2.0 ** -52)]:
        th = rng.uniform(0, 2 * np.pi)
        xy = np.array([[0.0, 0.0], [r * np.cos(th), r * np.sin(th)]])
        q = np.array([0.7, -1.3])
        _, phi, g = run(torch_cuda, xy, q, 4, 8, 0.5)
        ref = 0.5 * np.log(xy[1, 0] ** 2 + xy[1, 1] ** 2)  # phi_0 = -q_1 log r
        err = abs(phi[0] / -q[1] - ref) / (1.0 + abs(ref))
        worst = max(worst, err)
    assert worst < 4e-16, worst
    # r^2 = 1e-310 is subnormal (about 44 significant bits, hence the looser bound)
    xy = np.array([[0.0, 0.0], [1e-155, 0.0], [1.0, 1.0]])
    q = np.array([1.0, 2.0, -1.0])
    _, phi, _ = run(torch_cuda, xy, q, 4, 8, 0.5)
    ref = -2.0 * np.log(1e-155) + 1.0 * 0.5 * np.log(2.0)
    assert abs(phi[0] - ref) <= 1e-13 * abs(ref), (phi[0], ref)
