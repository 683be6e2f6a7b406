"""Pins for the oracle's single translation operators.

Each pin is a fact other than the oracle's own formula: a conservation law,
an exactness identity (M2M/L2L are exact for truncated data), the classical
closed-form truncation bound of the multipole/local expansion of 1/r
(far field approximated by multipole/local expansions), the
exact field of a point charge, and rotational invariance of the truncated
operator ("rotation of spherical harmonics").
"""
import numpy as np
import pytest

from oracle import oracle as O


def rand_cloud(rng, n, c, rad):
    d = rng.normal(size=(n, 3))
    d *= (rad * rng.random(n) ** (1 / 3) / np.linalg.norm(d, axis=1))[:, None]
    return c + d


def test_p2m_monopole_dipole():
    """M_0^0 = sum q; M_1^0 = sum q (z - cz); M_1^1 = -1/2 sum q ((x-cx) - i (y-cy))."""
    rng = np.random.default_rng(0)
    c = np.array([0.1, -0.2, 0.3])
    x = rand_cloud(rng, 50, c, 0.5)
    q = rng.uniform(-1, 1, 50)
    M = O.p2m(x, q, c, 3)
    d = x - c
    assert abs(M[0] - q.sum()) < 1e-14
    assert abs(M[O.cidx(1, 0)] - (q * d[:, 2]).sum()) < 1e-14
    assert abs(M[O.cidx(1, 1)] - (-0.5 * (q * (d[:, 0] - 1j * d[:, 1])).sum())) < 1e-14


def test_m2m_is_exact():
    """M2M(P2M(child)) == P2M(child particles about the parent centre)."""
    rng = np.random.default_rng(1)
    p = 10
    cp = np.array([0.0, 0.0, 0.0])
    Mp = np.zeros(O.ncoef(p), complex)
    xs, qs = [], []
    for oct_ in range(8):
        cc = 0.25 * np.array([1 if oct_ & 4 else -1, 1 if oct_ & 2 else -1, 1 if oct_ & 1 else -1])
        x = cc + rng.uniform(-0.25, 0.25, (20, 3))
        q = rng.uniform(-1, 1, 20)
        O.m2m(O.p2m(x, q, cc, p), cc, cp, p, Mp)
        xs.append(x)
        qs.append(q)
    Md = O.p2m(np.vstack(xs), np.concatenate(qs), cp, p)
    assert np.abs(Mp - Md).max() <= 1e-14 * np.abs(Md).max()


def test_l2l_is_exact():
    """L2P(L, x) == L2P(L2L(L), x) for any L of degree <= p (a polynomial re-expansion)."""
    rng = np.random.default_rng(2)
    p = 10
    L = rng.normal(size=O.ncoef(p)) + 1j * rng.normal(size=O.ncoef(p))
    for n in range(p + 1):
        L[O.cidx(n, 0)] = L[O.cidx(n, 0)].real  # real field => m = 0 coefficients real
    c = np.array([0.5, 0.5, 0.5])
    cc = c + np.array([0.125, -0.125, 0.125])
    Lc = O.l2l(L, c, cc, p)
    for _ in range(10):
        x = cc + rng.uniform(-0.125, 0.125, 3)
        a, ga = O.l2p(L, c, x, p, grad=True)
        b, gb = O.l2p(Lc, cc, x, p, grad=True)
        assert abs(a - b) <= 1e-13 * max(1.0, abs(a))
        assert np.abs(ga - gb).max() <= 1e-12 * max(1.0, np.abs(ga).max())


@pytest.mark.parametrize("p", [2, 4, 8, 12])
def test_m2l_l2p_single_charge_truncation_bound(p):
    """Single charge at distance a from cB, target at distance b from cA,
    d = |cA - cB| > a + b:  |error| <= |q| / (d - a - b) * ((a + b) / d)^{p+1}."""
    rng = np.random.default_rng(p)
    for _ in range(60):
        cB = rng.normal(size=3)
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        d = rng.uniform(2.0, 4.0)
        cA = cB + d * u
        a, b = rng.uniform(0.1, 0.8, 2) * (d / 2.2)
        y = cB + a * _unit(rng)
        x = cA + b * _unit(rng)
        q = rng.uniform(-1, 1)
        M = O.p2m(y[None], np.array([q]), cB, p)
        L = O.m2l(M, cB, cA, p)
        phi = O.l2p(L, cA, x, p)
        exact = q / np.linalg.norm(x - y)
        bound = abs(q) / (d - a - b) * ((a + b) / d) ** (p + 1)
        assert abs(phi - exact) <= bound * (1 + 1e-9) + 1e-15


@pytest.mark.parametrize("p", [2, 6, 10])
def test_multipole_only_bound(p):
    """|q| / (r - a) * (a / r)^{p+1} bounds the truncated multipole expansion."""
    rng = np.random.default_rng(100 + p)
    for _ in range(60):
        c = rng.normal(size=3)
        a = rng.uniform(0.1, 1.0)
        y = c + a * _unit(rng)
        r = rng.uniform(1.2 * a, 4 * a)
        x = c + r * _unit(rng)
        q = rng.uniform(-1, 1)
        M = O.p2m(y[None], np.array([q]), c, p)
        phi = O.m2p(M, c, x, p)
        bound = abs(q) / (r - a) * (a / r) ** (p + 1)
        assert abs(phi - q / np.linalg.norm(x - y)) <= bound * (1 + 1e-9) + 1e-15


def test_gradient_matches_point_charge_field_and_finite_difference():
    """grad phi from L2P vs -q (x-y)/|x-y|^3 (closed form, within truncation) and vs a
    central finite difference of the L2P potential (<= 1e-9)."""
    rng = np.random.default_rng(9)
    p = 14
    cB, cA = np.zeros(3), np.array([3.0, 0.5, -0.5])
    y = cB + 0.3 * _unit(rng)
    x = cA + 0.3 * _unit(rng)
    q = 0.7
    L = O.m2l(O.p2m(y[None], np.array([q]), cB, p), cB, cA, p)
    phi, g = O.l2p(L, cA, x, p, grad=True)
    r = x - y
    gex = -q * r / np.linalg.norm(r) ** 3
    assert np.abs(g - gex).max() < 1e-8
    h = 1e-5
    fd = np.array([(O.l2p(L, cA, x + h * e, p) - O.l2p(L, cA, x - h * e, p)) / (2 * h) for e in np.eye(3)])
    assert np.abs(g - fd).max() < 1e-9


def test_m2l_is_rotation_invariant():
    """The truncated M2L+L2P operator is frame independent degree by degree
    (rotation of spherical harmonics): rotating the whole geometry
    leaves the potentials unchanged to rounding. A transposed or mis-signed
    index in M2L breaks this."""
    rng = np.random.default_rng(11)
    p = 8
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    cB, cA = np.zeros(3), np.array([2.0, 1.0, 0.5])
    ys = cB + rng.uniform(-0.4, 0.4, (10, 3))
    qs = rng.uniform(-1, 1, 10)
    xs = cA + rng.uniform(-0.4, 0.4, (5, 3))

    def pot(R):
        L = O.m2l(O.p2m(ys @ R.T, qs, R @ cB, p), R @ cB, R @ cA, p)
        return np.array([O.l2p(L, R @ cA, R @ x, p) for x in xs])

    a, b = pot(np.eye(3)), pot(Q)
    assert np.abs(a - b).max() <= 1e-14 * np.abs(a).max()


def _unit(rng):
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)
