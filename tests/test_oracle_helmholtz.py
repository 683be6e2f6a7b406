"""Pins of the Helmholtz oracle (oracle/helmholtz_oracle.py, NEXT-4) against what the mathematics
fixes: closed forms of the spherical Bessel functions and harmonics, the Gaunt integral by
quadrature, the addition theorem and the three translation identities by direct evaluation,
reductions of the whole FMM to the direct sum, its convergence in p, linearity, and its
kappa -> 0 limit against the (pinned) Laplace oracle."""
import math

import numpy as np
import pytest

import fmm_inputs as F
from oracle import helmholtz_oracle as H
from oracle import oracle as O


def test_radial_closed_forms():
    x = np.array([0.3, 1.7, 5.2, 11.0])
    j = H.radial("j", 2, x)
    h = H.radial("h", 1, x)
    np.testing.assert_allclose(j[:, 0], np.sin(x) / x, rtol=1e-14)
    np.testing.assert_allclose(j[:, 1], np.sin(x) / x**2 - np.cos(x) / x, rtol=1e-13)
    np.testing.assert_allclose(j[:, 2], (3 / x**3 - 1 / x) * np.sin(x) - 3 * np.cos(x) / x**2, rtol=1e-12)
    np.testing.assert_allclose(h[:, 0], -1j * np.exp(1j * x) / x, rtol=1e-14)  # h_0 = -i e^{ix}/x
    np.testing.assert_allclose(h[:, 1], -(x + 1j) * np.exp(1j * x) / x**2, rtol=1e-13)


def test_harmonics_closed_forms_and_orthonormality():
    rng = np.random.default_rng(3)
    v = rng.standard_normal((5, 3))
    r = np.linalg.norm(v, axis=1)
    ct, st = v[:, 2] / r, np.sqrt(1 - (v[:, 2] / r) ** 2)
    eph = (v[:, 0] + 1j * v[:, 1]) / np.hypot(v[:, 0], v[:, 1])
    Y = H.Y(2, v)
    np.testing.assert_allclose(Y[:, H.idx(0, 0)], 1 / math.sqrt(4 * math.pi), rtol=1e-14)
    np.testing.assert_allclose(Y[:, H.idx(1, 0)], math.sqrt(3 / (4 * math.pi)) * ct, rtol=1e-13)
    np.testing.assert_allclose(Y[:, H.idx(1, 1)], -math.sqrt(3 / (8 * math.pi)) * st * eph, rtol=1e-13)  # CS phase
    for n in range(3):
        for m in range(1, n + 1):
            np.testing.assert_allclose(Y[:, H.idx(n, -m)], (-1) ** m * Y[:, H.idx(n, m)].conj(), rtol=1e-13)
    # orthonormality by Gauss-Legendre x trapezoid quadrature (exact for degree <= 2 * 6)
    t, w = np.polynomial.legendre.leggauss(10)
    ph = 2 * np.pi * np.arange(16) / 16
    pts = np.array([[math.sqrt(1 - a * a) * math.cos(b), math.sqrt(1 - a * a) * math.sin(b), a] for a in t for b in ph])
    wq = np.array([wa * 2 * np.pi / 16 for wa in w for _ in ph])
    Yq = H.Y(6, pts)
    G = (Yq.conj() * wq[:, None]).T @ Yq
    np.testing.assert_allclose(G, np.eye(49), atol=1e-13)


def test_gaunt_against_quadrature():
    t, w = np.polynomial.legendre.leggauss(16)
    ph = 2 * np.pi * np.arange(32) / 32
    pts = np.array([[math.sqrt(1 - a * a) * math.cos(b), math.sqrt(1 - a * a) * math.sin(b), a] for a in t for b in ph])
    wq = np.array([wa * 2 * np.pi / 32 for wa in w for _ in ph])
    Yq = H.Y(8, pts)
    for (l1, m1, l2, m2, l3, m3) in [(1, 0, 1, 0, 2, 0), (2, 1, 3, -2, 3, 1), (4, -3, 2, 2, 4, 1), (3, 0, 3, 0, 0, 0),
                                     (5, 2, 3, -1, 6, -1), (2, 1, 2, 1, 4, -2), (1, 1, 2, 0, 2, -1)]:
        q = (Yq[:, H.idx(l1, m1)] * Yq[:, H.idx(l2, m2)] * Yq[:, H.idx(l3, m3)] * wq).sum()
        assert abs(H.gaunt(l1, m1, l2, m2, l3, m3) - q.real) < 1e-14 and abs(q.imag) < 1e-14
    assert H.gaunt(1, 0, 1, 0, 1, 0) == 0.0  # parity
    assert H.wigner3j(1, 1, 0, 1, -1, 0) == pytest.approx(1 / math.sqrt(3))  # textbook value


@pytest.mark.parametrize("kappa", [0.5, 7.0, 20.0])
def test_addition_theorem(kappa):
    rng = np.random.default_rng(int(kappa * 10))
    for _ in range(5):
        y = rng.standard_normal(3) * 0.1
        x = rng.standard_normal(3) * 0.2 + np.array([0.7, 0.0, 0.0])
        d = np.linalg.norm(x - y)
        lhs = np.exp(1j * kappa * d) / d
        rhs = 4 * np.pi * 1j * kappa * (H.R(40, y[None], kappa).conj() * H.S(40, x[None], kappa)).sum()
        assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_translation_identities_converge():
    """(R|R), (S|R), (S|S) reproduce the translated functions; error falls with the truncation."""
    k = 7.0
    rng = np.random.default_rng(5)
    t, r = rng.standard_normal(3) * 0.1, rng.standard_normal(3) * 0.1
    errs = []
    for p in (6, 10):
        T = H.translation("RR", t, p, k)
        errs.append(np.abs(H.R(p, (r + t)[None], k)[0][:16] - (T.T @ H.R(p, r[None], k)[0])[:16]).max())
    assert errs[1] < 1e-13 and errs[1] < errs[0]
    t, r = np.array([0.5, 0.3, -0.2]), rng.standard_normal(3) * 0.05  # S -> R: |r| < |t|
    e = [np.abs(H.S(p, (r + t)[None], k)[0][:9] - (H.translation("SR", t, p, k).T @ H.R(p, r[None], k)[0])[:9]).max()
         / np.abs(H.S(p, (r + t)[None], k)[0][:9]).max() for p in (6, 10, 14)]
    assert e[0] > e[1] > e[2] and e[2] < 1e-9
    t, r = np.array([0.05, 0.03, -0.02]), np.array([0.4, -0.3, 0.2])  # S -> S: |r| > |t|
    e = [np.abs(H.S(p, (r + t)[None], k)[0][:9] - (H.translation("RR", t, p, k).T @ H.S(p, r[None], k)[0])[:9]).max()
         / np.abs(H.S(p, (r + t)[None], k)[0][:9]).max() for p in (6, 10, 14)]
    assert e[0] > e[1] > e[2] and e[2] < 1e-10


def test_fmm_reduces_to_direct():
    """theta -> 0 (every pair P2P) and N <= ncrit (one leaf) give the direct sum to rounding."""
    x, q = F.cube(600, seed=2)
    qc = q * (1 + 0.3j)
    d = H.direct(x, qc, 7.0)
    for ncrit, theta in ((16, 1e-6), (600, 0.4)):
        f = H.fmm_helmholtz(x, qc, 4, ncrit, theta, 7.0)
        assert np.linalg.norm(f - d) <= 1e-14 * np.linalg.norm(d)


def test_fmm_converges_in_p_and_is_linear():
    x, q = F.cube(1000)
    qc = q * (1 + 0.5j)
    k = 7.0
    d = H.direct(x, qc, k)
    errs = [np.linalg.norm(H.fmm_helmholtz(x, qc, p, 32, 0.4, k) - d) / np.linalg.norm(d) for p in (2, 4, 6)]
    assert errs[0] > 3 * errs[1] > 9 * errs[2] and errs[2] < 1e-4
    q2 = np.random.default_rng(9).uniform(-1, 1, 1000) * (0.2 - 1j)
    a = H.fmm_helmholtz(x, qc + 2 * q2, 3, 32, 0.4, k)
    b = H.fmm_helmholtz(x, qc, 3, 32, 0.4, k) + 2 * H.fmm_helmholtz(x, q2, 3, 32, 0.4, k)
    assert np.linalg.norm(a - b) <= 1e-14 * np.linalg.norm(a)


def test_fmm_low_frequency_limit_is_the_laplace_fmm():
    """kappa -> 0: exp(i kappa r)/r = 1/r + i kappa - kappa^2 r/2 + ...; the truncated spherical-wave
    series become the truncated solid-harmonic ones on the same tree and lists, so Re phi tends to
    the Laplace oracle's FMM (same p) and Im phi / kappa to sum_{j != i} q_j."""
    x, q = F.plummer(1500, seed=4)
    k = 1e-4
    f = H.fmm_helmholtz(x, q.astype(complex), 5, 24, 0.5, k)
    lap = O.fmm(x, q, 5, 24, 0.5)
    assert np.linalg.norm(f.real - lap) <= 1e-7 * np.linalg.norm(lap)
    far = q.sum() - q
    assert np.linalg.norm(f.imag / k - far) <= 1e-6 * np.linalg.norm(far)
