"""oracle/fmm2d_oracle.py — TEST INFRASTRUCTURE ONLY (NEXT-3).

The 2D half of the paper's §4.1 experiment ("2D and 3D Laplace equation on uniform lattices",
PAPER.md:386): the FMM mat-vec for the 2D Laplace (log) kernel,

    phi_i = - sum_{j : |x_i - x_j| > 0} q_j log |x_i - x_j|,   grad_i = grad_{x_i} phi_i,

in plain numpy, complex notation z = x + i y. The paper prints no 2D formulas; this follows
the classical 2D multipole calculus (R40-R44): with Phi(z) = sum_j q_j log(z - z_j)
and phi = -Re Phi,
    P2M   Phi ~ a_0 log(z - c) + sum_{k=1..p} a_k (z - c)^-k,  a_0 = sum q,  a_k = -sum q (z_j - c)^k / k
    M2M   (to c' with z0 = c - c')  b_l = -a_0 z0^l / l + sum_{k=1..l} a_k z0^(l-k) C(l-1, k-1)
    M2L   (to a local expansion about c' with z0 = c - c')
          c_0 = a_0 log(-z0) + sum_k a_k (-1)^k z0^-k
          c_l = -a_0 / (l z0^l) + z0^-l sum_k a_k z0^-k C(l+k-1, k-1) (-1)^k
    L2L   (to c'' with w = c'' - c')  d_l = sum_{k>=l} c_k C(k, l) w^(k-l)
    L2P   phi = -Re sum_l c_l (z - c)^l,  (d/dx, d/dy) phi = (-Re Phi', Im Phi')
on the tree and interaction lists of the 3D oracle (oracle.py) built for the points (x, y, 0):
an octree of planar points is a quadtree, and the 3D MAC with theta < 1/sqrt(3) implies the 2D
series converge (R41). Expansions live in physical coordinates (centres = the oracle's
normalised centres times 2^e), so no rescaling of the logarithm is involved.
"""
from __future__ import annotations

from math import comb

import numpy as np

from . import oracle as O


def direct2d(xy, q, tgt=None, grad=False):
    """Plain O(N M) sum (pairs with r = 0 skipped)."""
    xy = np.asarray(xy, dtype=np.float64)
    t = xy if tgt is None else np.asarray(tgt, dtype=np.float64)
    phi = np.zeros(t.shape[0])
    g = np.zeros((t.shape[0], 2))
    for i in range(t.shape[0]):
        d = t[i] - xy
        r2 = (d * d).sum(1)
        m = r2 > 0
        phi[i] = -(q[m] * 0.5 * np.log(r2[m])).sum()
        g[i] = -(q[m, None] * d[m] / r2[m, None]).sum(0)
    return (phi, g) if grad else phi


def p2m(z, q, c, p):
    a = np.zeros(p + 1, complex)
    a[0] = q.sum()
    w = z - c
    for k in range(1, p + 1):
        a[k] = -(q * w ** k).sum() / k
    return a


def m2m(a, z0, p):
    b = np.zeros(p + 1, complex)
    b[0] = a[0]
    for l in range(1, p + 1):
        s = -a[0] * z0 ** l / l
        for k in range(1, l + 1):
            s += a[k] * z0 ** (l - k) * comb(l - 1, k - 1)
        b[l] = s
    return b


def m2l_matrix(p):
    """B[l, k] = C(l+k-1, k-1) (-1)^k for l, k >= 1 (zero elsewhere)."""
    B = np.zeros((p + 1, p + 1))
    for l in range(1, p + 1):
        for k in range(1, p + 1):
            B[l, k] = comb(l + k - 1, k - 1) * (-1) ** k
    return B


def m2l(a, z0, p):
    """Vectorised over rows: a [n, p+1], z0 [n] -> local coefficients [n, p+1]."""
    a = np.atleast_2d(a)
    z0 = np.atleast_1d(z0)
    inv = 1.0 / z0
    k = np.arange(p + 1)
    ik = inv[:, None] ** k[None, :]  # z0^-k
    c = np.zeros_like(a)
    c[:, 0] = a[:, 0] * np.log(-z0) + (a[:, 1:] * ((-1.0) ** k[1:])[None, :] * ik[:, 1:]).sum(1)
    if p >= 1:
        l = k[1:]
        t = (a[:, 1:] * ik[:, 1:]) @ m2l_matrix(p)[1:, 1:].T  # sum_k a_k z0^-k B[l, k]
        c[:, 1:] = -a[:, :1] * ik[:, 1:] / l[None, :] + ik[:, 1:] * t
    return c


def l2l(c, w, p):
    d = np.zeros(p + 1, complex)
    for l in range(p + 1):
        d[l] = sum(c[k] * comb(k, l) * w ** (k - l) for k in range(l, p + 1))
    return d


def l2p(c, z, ctr, p, grad=False):
    w = z - ctr
    Phi = np.zeros_like(w)
    dPhi = np.zeros_like(w)
    for l in range(p + 1):
        Phi = Phi + c[l] * w ** l
        if l >= 1:
            dPhi = dPhi + l * c[l] * w ** (l - 1)
    phi = -Phi.real
    return (phi, np.c_[-dPhi.real, dPhi.imag]) if grad else phi


class Plan2D:
    """Tree and lists from the 3D oracle on (x, y, 0); 2D expansions per the module docstring."""

    def __init__(self, xy, p, ncrit, theta):
        self.xy = np.ascontiguousarray(xy, dtype=np.float64)
        self.p = p
        n = self.xy.shape[0]
        self.plan = O.Plan(np.c_[self.xy, np.zeros(n)], p, ncrit, theta)
        s = 2.0 ** self.plan.info("exp")
        self.cells = self.plan.cells()
        self.ctr = (self.cells["center"][:, 0] + 1j * self.cells["center"][:, 1]) * s
        _, self.perm = self.plan.keys()
        self.p2p, self.m2l_pairs = self.plan.lists()

    def eval(self, q, grad=False):
        p, C = self.p, self.cells
        nc = C["level"].shape[0]
        z = (self.xy[:, 0] + 1j * self.xy[:, 1])[self.perm]
        qs = np.asarray(q, dtype=np.float64)[self.perm]
        M = np.zeros((nc, p + 1), complex)
        L = np.zeros((nc, p + 1), complex)
        leaf = C["nchild"] == 0
        for c in np.nonzero(leaf)[0]:
            b, e = C["begin"][c], C["end"][c]
            M[c] = p2m(z[b:e], qs[b:e], self.ctr[c], p)
        for lev in range(C["level"].max() - 1, -1, -1):
            for c in np.nonzero((C["level"] == lev) & ~leaf)[0]:
                for ch in range(C["child_first"][c], C["child_first"][c] + C["nchild"][c]):
                    M[c] += m2m(M[ch], self.ctr[ch] - self.ctr[c], p)
        if self.m2l_pairs.shape[0]:
            A, B = self.m2l_pairs[:, 0], self.m2l_pairs[:, 1]
            np.add.at(L, A, m2l(M[B], self.ctr[B] - self.ctr[A], p))
        for lev in range(C["level"].max()):
            for c in np.nonzero((C["level"] == lev) & ~leaf)[0]:
                for ch in range(C["child_first"][c], C["child_first"][c] + C["nchild"][c]):
                    L[ch] += l2l(L[c], self.ctr[ch] - self.ctr[c], p)
        n = z.shape[0]
        phi = np.zeros(n)
        g = np.zeros((n, 2))
        for c in np.nonzero(leaf)[0]:
            b, e = C["begin"][c], C["end"][c]
            r = l2p(L[c], z[b:e], self.ctr[c], p, grad=True)
            phi[b:e] += r[0]
            g[b:e] += r[1]
        for A, Bc in self.p2p:
            ta, te = C["begin"][A], C["end"][A]
            sa, se = C["begin"][Bc], C["end"][Bc]
            d = z[ta:te, None] - z[None, sa:se]
            r2 = (d * d.conj()).real
            m = r2 > 0
            lg = np.where(m, 0.5 * np.log(np.where(m, r2, 1.0)), 0.0)
            phi[ta:te] -= (qs[None, sa:se] * lg).sum(1)
            w = np.where(m, qs[None, sa:se] / np.where(m, r2, 1.0), 0.0)
            g[ta:te, 0] -= (w * d.real).sum(1)
            g[ta:te, 1] -= (w * d.imag).sum(1)
        out_phi = np.zeros(n)
        out_g = np.zeros((n, 2))
        out_phi[self.perm] = phi
        out_g[self.perm] = g
        self.M, self.L = M, L
        return (out_phi, out_g) if grad else out_phi


def fmm2d(xy, q, p, ncrit, theta, grad=False):
    return Plan2D(xy, p, ncrit, theta).eval(q, grad=grad)
