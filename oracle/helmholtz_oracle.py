"""oracle/helmholtz_oracle.py — TEST INFRASTRUCTURE ONLY (NEXT-4).

The paper's second kernel (§1: "FMM and HSS for Laplace and Helmholtz kernels";
PAPER.md:444, 456-460, 473-479, §4.2: the Helmholtz equation on a [-1,1]^3 lattice with wave
number kappa = 7): the FMM mat-vec for the 3D Helmholtz kernel

    phi_i = sum_{j : |x_i - x_j| > 0} q_j exp(i kappa r_ij) / r_ij        (complex q, phi)

in plain numpy, on the tree and interaction lists of the Laplace oracle (oracle.py; the same
MAC, split rule and ncrit, R50). The paper prints no formulas; this follows the
classical spherical-wave calculus (R50-R55), written out here:

  Y_n^m      orthonormal spherical harmonics with the Condon-Shortley phase (scipy sph_harm_y),
             Y_n^{-m} = (-1)^m conj Y_n^m
  R_n^m(v) = j_n(kappa |v|) Y_n^m(v^),  S_n^m(v) = h_n(kappa |v|) Y_n^m(v^),  h_n = j_n + i y_n
  addition   exp(i kappa |x - y|) / |x - y| = 4 pi i kappa sum_{n,m} conj R_n^m(y) S_n^m(x),
             |y| < |x|
  multipole  phi(x) ~ sum_{n <= p, |m| <= n} M_n^m S_n^m(x - c)
  local      phi(x) ~ sum_{n <= p, |m| <= n} L_n^m R_n^m(x - c)
  P2M        M_n^m = 4 pi i kappa sum_j q_j conj R_n^m(y_j - c)
  translation coefficients (from the plane-wave expansion exp(i kappa k.r) = 4 pi sum i^n
             R_n^m(r) conj Y_n^m(k^)):
               (E|F)[(n',m'), (n,m)](t) = 4 pi sum_l i^(n' + l - n) E_l^(m - m')(t)
                                          * integral Y_n^m conj Y_n'^m' conj Y_l^(m - m') dOmega
             with E = R for (R|R) = (S|S) and E = S for (S|R); the integral is a Gaunt
             coefficient (Wigner 3j symbols, Racah's formula)
  M2M        M(c_p) = (S|S)(c_p - c_c) M(c_c)        (truncated at p on both sides)
  M2L        L(c_A) += (S|R)(c_A - c_B) M(c_B)
  L2L        L(c_c) += (R|R)(c_c - c_p) L(c_p)
  L2P        phi(x) += sum L_n^m R_n^m(x - c)
  P2P        phi_i += q_j exp(i kappa r) / r, r > 0
Index of (n, m): n^2 + n + m. Coordinates are physical (the Laplace oracle's normalised centres
times 2^e). Small sizes only (Python loops over cells, numpy per pair).
"""
from __future__ import annotations

import functools
import math
from fractions import Fraction

import numpy as np
from scipy.special import sph_harm_y, spherical_jn, spherical_yn

from . import oracle as O


def idx(n: int, m: int) -> int:
    return n * n + n + m


def ncoef(p: int) -> int:
    return (p + 1) * (p + 1)


def _sph(v):
    v = np.atleast_2d(np.asarray(v, dtype=np.float64))
    r = np.sqrt((v * v).sum(1))
    th = np.arccos(np.clip(np.where(r > 0, v[:, 2] / np.where(r > 0, r, 1.0), 1.0), -1.0, 1.0))
    ph = np.arctan2(v[:, 1], v[:, 0])
    return r, th, ph


def Y(nmax: int, v):
    """Y_n^m(v^) for n <= nmax, all m: [len(v), (nmax+1)^2] (v = 0 -> direction +z)."""
    _, th, ph = _sph(v)
    out = np.zeros((th.shape[0], ncoef(nmax)), complex)
    for n in range(nmax + 1):
        for m in range(-n, n + 1):
            out[:, idx(n, m)] = sph_harm_y(n, m, th, ph)
    return out


def radial(kind: str, nmax: int, x):
    """j_n(x) ('j') or h_n^(1)(x) ('h') for n <= nmax: [len(x), nmax + 1] (library routines)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = np.arange(nmax + 1)
    j = spherical_jn(n[None, :], x[:, None])
    if kind == "j":
        return j
    return j + 1j * spherical_yn(n[None, :], x[:, None])


def R(nmax: int, v, kappa: float):
    r, _, _ = _sph(v)
    rad = radial("j", nmax, kappa * r)
    ns = np.array([n for n in range(nmax + 1) for _ in range(2 * n + 1)])
    return rad[:, ns] * Y(nmax, v)


def S(nmax: int, v, kappa: float):
    r, _, _ = _sph(v)
    rad = radial("h", nmax, kappa * r)
    ns = np.array([n for n in range(nmax + 1) for _ in range(2 * n + 1)])
    return rad[:, ns] * Y(nmax, v)


@functools.lru_cache(maxsize=None)
def _fact(n: int) -> int:
    return math.factorial(n)


def wigner3j(j1, j2, j3, m1, m2, m3) -> float:
    """Racah's formula, exact rational arithmetic then one sqrt."""
    if m1 + m2 + m3 != 0 or abs(m1) > j1 or abs(m2) > j2 or abs(m3) > j3:
        return 0.0
    if j3 < abs(j1 - j2) or j3 > j1 + j2:
        return 0.0
    f = _fact
    tri = Fraction(f(j1 + j2 - j3) * f(j1 - j2 + j3) * f(-j1 + j2 + j3), f(j1 + j2 + j3 + 1))
    pre = tri * f(j1 + m1) * f(j1 - m1) * f(j2 + m2) * f(j2 - m2) * f(j3 + m3) * f(j3 - m3)
    s = Fraction(0)
    for k in range(max(0, j2 - j3 - m1, j1 - j3 + m2), min(j1 + j2 - j3, j1 - m1, j2 + m2) + 1):
        s += Fraction((-1) ** k, f(k) * f(j1 + j2 - j3 - k) * f(j1 - m1 - k) * f(j2 + m2 - k) *
                      f(j3 - j2 + m1 + k) * f(j3 - j1 - m2 + k))
    sign = -1.0 if (j1 - j2 - m3) % 2 else 1.0
    return sign * math.sqrt(float(pre)) * float(s)


def gaunt(l1, m1, l2, m2, l3, m3) -> float:
    """integral over the sphere of Y_l1^m1 Y_l2^m2 Y_l3^m3."""
    w0 = wigner3j(l1, l2, l3, 0, 0, 0)
    if w0 == 0.0:
        return 0.0
    return math.sqrt((2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1) / (4 * math.pi)) * w0 * wigner3j(l1, l2, l3, m1, m2, m3)


@functools.lru_cache(maxsize=None)
def _coupling(p: int):
    """C[(n',m'), (n,m), l] = 4 pi i^(n' + l - n) integral Y_n^m conj Y_n'^m' conj Y_l^(m-m'),
    and the (l, mu = m - m') index of every entry, for n, n' <= p, l <= 2p."""
    nc = ncoef(p)
    C = np.zeros((nc, nc, 2 * p + 1), complex)
    for n1 in range(p + 1):
        for m1 in range(-n1, n1 + 1):
            for n in range(p + 1):
                for m in range(-n, n + 1):
                    mu = m - m1
                    for l in range(abs(n - n1), n + n1 + 1):
                        if abs(mu) > l:
                            continue
                        # conj Y_a^b = (-1)^b Y_a^-b
                        g = (-1) ** ((m1 + mu) & 1) * gaunt(n, m, n1, -m1, l, -mu)
                        if g != 0.0:
                            C[idx(n1, m1), idx(n, m), l] = 4 * math.pi * (1j ** ((n1 + l - n) % 4)) * g
    mus = np.array([[m - m1 for n in range(p + 1) for m in range(-n, n + 1)]
                    for n1 in range(p + 1) for m1 in range(-n1, n1 + 1)])
    return C, mus


def translation(kind: str, t, p: int, kappa: float):
    """(R|R) ('RR', also (S|S)) or (S|R) ('SR') for the translation vector t: [(p+1)^2]^2."""
    C, mus = _coupling(p)
    E = (R if kind == "RR" else S)(2 * p, np.asarray(t, dtype=np.float64)[None, :], kappa)[0]
    ls = np.arange(2 * p + 1)
    # E_l^mu per (row, col, l); zero where |mu| > l (C is zero there too)
    Eg = np.zeros((mus.shape[0], mus.shape[1], 2 * p + 1), complex)
    for l in ls:
        ok = np.abs(mus) <= l
        Eg[:, :, l][ok] = E[l * l + l + mus[ok]]
    return (C * Eg).sum(2)


def direct(xyz, q, kappa, tgt=None):
    """Plain O(N M) sum of q_j exp(i kappa r) / r (pairs with r = 0 skipped)."""
    xyz = np.asarray(xyz, dtype=np.float64)
    t = xyz if tgt is None else np.asarray(tgt, dtype=np.float64)
    q = np.asarray(q, dtype=complex)
    out = np.zeros(t.shape[0], complex)
    for i in range(t.shape[0]):
        d = t[i] - xyz
        r = np.sqrt((d * d).sum(1))
        m = r > 0
        out[i] = (q[m] * np.exp(1j * kappa * r[m]) / r[m]).sum()
    return out


class PlanH:
    """Tree and lists from the Laplace oracle; Helmholtz expansions per the module docstring."""

    def __init__(self, xyz, p, ncrit, theta, kappa):
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.p, self.kappa = p, float(kappa)
        self.plan = O.Plan(self.xyz, p, ncrit, theta)
        s = 2.0 ** self.plan.info("exp")
        self.cells = self.plan.cells()
        self.ctr = self.cells["center"] * s
        _, self.perm = self.plan.keys()
        self.p2p, self.m2l_pairs = self.plan.lists()

    def eval(self, q):
        p, C, k = self.p, self.cells, self.kappa
        nc = C["level"].shape[0]
        x = self.xyz[self.perm]
        qs = np.asarray(q, dtype=complex)[self.perm]
        M = np.zeros((nc, ncoef(p)), complex)
        L = np.zeros((nc, ncoef(p)), complex)
        leaf = C["nchild"] == 0
        for c in np.nonzero(leaf)[0]:  # P2M
            b, e = C["begin"][c], C["end"][c]
            M[c] = 4 * np.pi * 1j * k * (qs[b:e, None] * R(p, x[b:e] - self.ctr[c], k).conj()).sum(0)
        for lev in range(C["level"].max() - 1, -1, -1):  # M2M
            for c in np.nonzero((C["level"] == lev) & ~leaf)[0]:
                for ch in range(C["child_first"][c], C["child_first"][c] + C["nchild"][c]):
                    M[c] += translation("RR", self.ctr[c] - self.ctr[ch], p, k) @ M[ch]
        for a, b in self.m2l_pairs:  # M2L
            L[a] += translation("SR", self.ctr[a] - self.ctr[b], p, k) @ M[b]
        for lev in range(C["level"].max()):  # L2L
            for c in np.nonzero((C["level"] == lev) & ~leaf)[0]:
                for ch in range(C["child_first"][c], C["child_first"][c] + C["nchild"][c]):
                    L[ch] += translation("RR", self.ctr[ch] - self.ctr[c], p, k) @ L[c]
        n = x.shape[0]
        phi = np.zeros(n, complex)
        for c in np.nonzero(leaf)[0]:  # L2P
            b, e = C["begin"][c], C["end"][c]
            phi[b:e] += (R(p, x[b:e] - self.ctr[c], k) * L[c][None, :]).sum(1)
        for a, bc in self.p2p:  # P2P
            ta, te = C["begin"][a], C["end"][a]
            sa, se = C["begin"][bc], C["end"][bc]
            d = x[ta:te, None, :] - x[None, sa:se, :]
            r = np.sqrt((d * d).sum(2))
            m = r > 0
            w = np.where(m, np.exp(1j * k * r) / np.where(m, r, 1.0), 0.0)
            phi[ta:te] += (w * qs[None, sa:se]).sum(1)
        out = np.zeros(n, complex)
        out[self.perm] = phi
        self.M, self.L = M, L
        return out


def fmm_helmholtz(xyz, q, p, ncrit, theta, kappa):
    return PlanH(xyz, p, ncrit, theta, kappa).eval(q)
