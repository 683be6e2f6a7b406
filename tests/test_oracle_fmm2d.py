"""Pins of the 2D (log-kernel) oracle (oracle/fmm2d_oracle.py; NEXT-3): closed
forms, exact translation identities, series convergence against the direct sum, and the
gradient against finite differences."""
import numpy as np
import pytest

from oracle import fmm2d_oracle as D


def test_direct_closed_forms():
    xy = np.array([[0.0, 0.0], [3.0, 4.0]])
    q = np.array([2.0, -1.0])
    phi, g = D.direct2d(xy, q, grad=True)
    assert np.allclose(phi, [np.log(5.0), -2.0 * np.log(5.0)], rtol=1e-15)
    assert np.allclose(g[0], [-(-1.0) * (-3.0) / 25.0, -(-1.0) * (-4.0) / 25.0], rtol=1e-15)
    # coincident points contribute nothing (r = 0 skipped)
    assert D.direct2d(np.zeros((3, 2)), np.ones(3)).tolist() == [0.0, 0.0, 0.0]


def test_direct_gradient_is_derivative_of_potential():
    rng = np.random.default_rng(3)
    xy, q = rng.random((50, 2)), rng.uniform(-1, 1, 50)
    t = np.array([[0.31, 0.47]])
    _, g = D.direct2d(xy, q, tgt=t, grad=True)
    h = 1e-6
    fx = (D.direct2d(xy, q, tgt=t + [h, 0]) - D.direct2d(xy, q, tgt=t - [h, 0])) / (2 * h)
    fy = (D.direct2d(xy, q, tgt=t + [0, h]) - D.direct2d(xy, q, tgt=t - [0, h])) / (2 * h)
    assert np.allclose(g[0], [fx[0], fy[0]], rtol=1e-7)


def test_multipole_far_field_and_m2m_l2l_exact():
    rng = np.random.default_rng(4)
    p = 20
    src = 0.3 * (rng.random(40) - 0.5) + 1j * 0.3 * (rng.random(40) - 0.5)
    q = rng.uniform(-1, 1, 40)
    c = 0.02 + 0.01j
    a = D.p2m(src, q, c, p)
    assert abs(a[0] - q.sum()) < 1e-15
    far = np.array([3.0 + 1.0j, -2.0 - 2.5j])
    Phi = a[0] * np.log(far - c) + sum(a[k] * (far - c) ** (-k) for k in range(1, p + 1))
    ref = D.direct2d(np.c_[src.real, src.imag], q, tgt=np.c_[far.real, far.imag])
    assert np.allclose(-Phi.real, ref, rtol=1e-13, atol=0)
    # M2M is exact: shifting the child expansion equals the expansion about the new centre
    c2 = -0.1 + 0.05j
    assert np.allclose(D.m2m(a, c - c2, p), D.p2m(src, q, c2, p), rtol=0, atol=1e-13 * np.abs(a).max())
    # L2L is exact for a polynomial
    loc = rng.standard_normal(p + 1) + 1j * rng.standard_normal(p + 1)
    w = 0.05 - 0.02j
    zt = np.array([0.01 + 0.02j, -0.03j])
    lhs = D.l2p(D.l2l(loc, w, p), zt, c + w, p)
    rhs = D.l2p(loc, zt, c, p)
    assert np.allclose(lhs, rhs, rtol=1e-12)


@pytest.mark.parametrize("dist", [1.5, 3.0])
def test_m2l_converges_geometrically(dist):
    rng = np.random.default_rng(5)
    src = 0.25 * (rng.random(60) - 0.5) + 1j * 0.25 * (rng.random(60) - 0.5)
    q = rng.uniform(-1, 1, 60)
    cA = dist + 0.2j
    tgt = cA + 0.25 * (rng.random(30) - 0.5) + 1j * 0.25 * (rng.random(30) - 0.5)
    ref = D.direct2d(np.c_[src.real, src.imag], q, tgt=np.c_[tgt.real, tgt.imag])
    errs = []
    for p in (4, 8, 16):
        a = D.p2m(src, q, 0.0, p)
        c = D.m2l(a, 0.0 - cA, p)[0]
        errs.append(np.abs(D.l2p(c, tgt, cA, p) - ref).max() / np.abs(ref).max())
    ratio = 0.25 * np.sqrt(2) / (dist - 0.25 * np.sqrt(2))  # (r_A + r_B) / (|cA| - r) style bound
    assert errs[0] > errs[1] > errs[2] and errs[2] < 10 * ratio ** 16 + 1e-14


def test_fmm2d_matches_direct_and_converges():
    rng = np.random.default_rng(0)
    xy = rng.random((2000, 2)) * 3 - 1
    q = rng.uniform(-1, 1, 2000)
    pd, gd = D.direct2d(xy, q, grad=True)
    prev = 1.0
    for p in (4, 8, 16):
        pf, gf = D.fmm2d(xy, q, p, 32, 0.5, grad=True)
        e = np.linalg.norm(pf - pd) / np.linalg.norm(pd)
        eg = np.linalg.norm(gf - gd) / np.linalg.norm(gd)
        assert e < prev / 10 and eg < 50 * e
        prev = e
    assert prev < 1e-8
    pl = D.Plan2D(xy, 8, 32, 0.5)
    pl.eval(q)
    assert abs(pl.M[0, 0] - q.sum()) < 1e-12  # root monopole = total charge


def test_fmm2d_lattice_and_single_leaf():
    g1 = np.arange(20) / 19.0
    xy = np.stack(np.meshgrid(g1, g1, indexing="ij"), -1).reshape(-1, 2)  # points on cell faces
    q = np.random.default_rng(1).uniform(-1, 1, xy.shape[0])
    pf = D.fmm2d(xy, q, 16, 16, 0.5)
    assert np.linalg.norm(pf - D.direct2d(xy, q)) <= 1e-8 * np.linalg.norm(pf)
    # everything in one leaf: the FMM is the direct sum
    assert np.allclose(D.fmm2d(xy[:50], q[:50], 4, 64, 0.5), D.direct2d(xy[:50], q[:50]), rtol=1e-13)
