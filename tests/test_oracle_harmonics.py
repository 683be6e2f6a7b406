"""Pins for the oracle's solid harmonics and the expansion identities.

The paper names spherical-harmonic expansions but prints no
formulas; these tests pin the oracle's Cartesian recurrences to the Legendre
closed form (scipy.special.lpmv, a library routine independent of the
oracle) and to the addition theorems H1–H3 evaluated by brute force.
"""
import math

import numpy as np
import pytest
from scipy.special import lpmv

from oracle import oracle as O


def sph(v):
    x, y, z = v
    r = math.sqrt(x * x + y * y + z * z)
    return r, z / r, math.atan2(y, x)


def R_closed(v, n, m):
    """R_n^m = r^n P_n^m(cos t) e^{i m phi} / (n+m)!, CS phase, any |m| <= n."""
    r, ct, ph = sph(v)
    if m < 0:
        return (-1) ** (-m) * np.conj(R_closed(v, n, -m))
    return r**n * lpmv(m, n, ct) * np.exp(1j * m * ph) / math.factorial(n + m)


def I_closed(v, n, m):
    """I_n^m = (n-m)! P_n^m(cos t) e^{i m phi} / r^{n+1}."""
    r, ct, ph = sph(v)
    if m < 0:
        return (-1) ** (-m) * np.conj(I_closed(v, n, -m))
    return math.factorial(n - m) * lpmv(m, n, ct) * np.exp(1j * m * ph) / r ** (n + 1)


def full(A, n, m):
    """coefficient at any |m| <= n from m >= 0 storage (A_n^{-m} = (-1)^m conj A_n^m)."""
    if abs(m) > n:
        return 0.0
    v = A[O.cidx(n, abs(m))]
    return v if m >= 0 else (-1) ** (-m) * np.conj(v)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_harmonics_match_legendre_closed_form(seed):
    rng = np.random.default_rng(seed)
    p = 12
    for _ in range(20):
        v = rng.normal(size=3) * rng.uniform(0.2, 3.0)
        R = O.harmonics_R(v, p)
        Iv = O.harmonics_I(v, p)
        for n in range(p + 1):
            rc = np.array([R_closed(v, n, m) for m in range(n + 1)])
            ic = np.array([I_closed(v, n, m) for m in range(n + 1)])
            ro = np.array([R[O.cidx(n, m)] for m in range(n + 1)])
            io = np.array([Iv[O.cidx(n, m)] for m in range(n + 1)])
            # absolute error relative to the largest coefficient of that degree
            assert np.abs(ro - rc).max() <= 1e-13 * np.abs(rc).max()
            assert np.abs(io - ic).max() <= 1e-13 * np.abs(ic).max()


def test_low_degree_explicit_values():
    """R_1^0 = z, R_1^1 = -(x+iy)/2, I_0^0 = 1/r, I_1^0 = z/r^3 (hand computation)."""
    v = np.array([0.3, -0.7, 1.1])
    R = O.harmonics_R(v, 2)
    Iv = O.harmonics_I(v, 2)
    r = np.linalg.norm(v)
    assert R[0] == 1.0
    assert R[O.cidx(1, 0)] == v[2]
    assert abs(R[O.cidx(1, 1)] - (-(v[0] + 1j * v[1]) / 2)) < 1e-16
    assert abs(Iv[0] - 1 / r) < 4e-16 / r
    assert abs(Iv[O.cidx(1, 0)] - v[2] / r**3) < 1e-15 * abs(v[2]) / r**3
    # R_2^0 = (3 z^2 - r^2)/4 ; I_2^0 = (3 z^2 - r^2)/r^5
    assert abs(R[O.cidx(2, 0)] - (3 * v[2] ** 2 - r**2) / 4) < 1e-15
    assert abs(Iv[O.cidx(2, 0)] - (3 * v[2] ** 2 - r**2) / r**5) < 1e-14


def test_H1_multipole_expansion_of_inverse_distance():
    """(H1) 1/|x-y| = sum_n sum_m conj R_n^m(y) I_n^m(x), |y| < |x|."""
    rng = np.random.default_rng(5)
    P = 40
    for _ in range(10):
        x = rng.normal(size=3)
        x *= 2.0 / np.linalg.norm(x)
        y = rng.normal(size=3)
        y *= 0.5 / np.linalg.norm(y)
        R = O.harmonics_R(y, P)
        Iv = O.harmonics_I(x, P)
        s = sum(np.conj(full(R, n, m)) * full(Iv, n, m) for n in range(P + 1) for m in range(-n, n + 1))
        assert abs(s.imag) < 1e-14
        assert abs(s.real - 1 / np.linalg.norm(x - y)) < 1e-14


def test_H2_regular_addition_theorem():
    """(H2) R_j^k(a+b) = sum_{n<=j} sum_m R_n^m(b) R_{j-n}^{k-m}(a): a finite identity."""
    rng = np.random.default_rng(6)
    p = 8
    a, b = rng.normal(size=3), rng.normal(size=3)
    Ra, Rb, Rab = O.harmonics_R(a, p), O.harmonics_R(b, p), O.harmonics_R(a + b, p)
    for j in range(p + 1):
        for k in range(-j, j + 1):
            s = sum(full(Rb, n, m) * full(Ra, j - n, k - m) for n in range(j + 1) for m in range(-n, n + 1))
            assert abs(s - full(Rab, j, k)) < 1e-13 * max(1.0, abs(full(Rab, j, k)))


def test_H3_irregular_addition_theorem():
    """(H3) I_j^k(a+b) = sum_n sum_m (-1)^n conj R_n^m(a) I_{j+n}^{k+m}(b), |a| < |b|."""
    rng = np.random.default_rng(7)
    P = 45
    a = rng.normal(size=3)
    a *= 0.4 / np.linalg.norm(a)
    b = rng.normal(size=3)
    b *= 2.0 / np.linalg.norm(b)
    Ra = O.harmonics_R(a, P)
    Ib = O.harmonics_I(b, P + 4)
    Iab = O.harmonics_I(a + b, 4)
    for j in range(4):
        for k in range(-j, j + 1):
            s = sum((-1) ** n * np.conj(full(Ra, n, m)) * full(Ib, j + n, k + m)
                    for n in range(P + 1) for m in range(-n, n + 1) if abs(k + m) <= j + n)
            ref = full(Iab, j, k)
            assert abs(s - ref) < 1e-13 * max(1.0, abs(ref))
