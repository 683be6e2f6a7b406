"""oracle/pde_helmholtz_oracle.py — TEST INFRASTRUCTURE ONLY (NEXT-4 solve).

Plain numpy reference for the Helmholtz half of the paper's §4.2 experiment: "the Laplace
equation and Helmholtz equation on a 3D cubic lattice [-1,1]^3 [...] Dirichlet boundary
conditions at the faces of the domain. The preconditioners are used inside a Krylov subspace
solver."; Fig 6: "the Helmholtz equation on a [-1,1]^3 lattice with spacing
h = 2^-5 and wave number kappa = 7"; "the FMM preconditioner has a convergence
rate that is independent of the problem size, up to moderate wave numbers".
Only ``tests/`` and the measurement tools may import it; it shares no code with
``paper_1602_02244_b200``.

The paper gives no formulas for this experiment. The readings (R56-R60), the
Laplace ones of pde_oracle.py (R30-R36) carried over with the Helmholtz Green's function:
  * lattice and faces as pde_oracle.py (h = 2/(n+1), x-fastest index);
  * A = -Delta_h - kappa^2 I, the 7-point stencil with zero Dirichlet ghost values (the
    Helmholtz equation -Delta u - kappa^2 u = f);
  * G(x, y) = exp(i kappa |x - y|) / (4 pi |x - y|), the outgoing free-space Green's function
    of -Delta - kappa^2;
  * preconditioner M r:
      1. volume potential u_v(x_i) = sum_{j != i} h^3 G(x_i, x_j) r_j + c_self r_i, with the
         own-cell integral to second order in kappa h: c_self = h^2 C_cube / (4 pi)
         + i kappa h^3 / (4 pi)  (exp(i kappa r) / r = 1/r + i kappa + O(kappa^2 r)), the sum
         by the Helmholtz FMM oracle (helmholtz_oracle.py: p, ncrit, theta);
      2. single-layer densities on the face panels: S sigma = -u_v|faces, S_ij = a^2 G(y_i, y_j),
         S_ii = a C_panel / (4 pi) + i kappa a^2 / (4 pi) (own-panel integral, same order);
      3. M r = u_v + sum_j a^2 G(x_i, y_j) sigma_j at the lattice nodes (by the FMM);
  * Krylov: GMRES (A is real symmetric but indefinite for kappa = 7, the preconditioner is
    complex and non-Hermitian: CG does not apply), right preconditioned (A M u = b, x = M u),
    x0 = 0, no restart, Arnoldi by modified Gram-Schmidt, the least-squares problem by Givens
    rotations; stop when the GMRES residual estimate |g_{k+1}| / ||b|| <= rtol (equal to
    ||b - A x_k|| / ||b|| in exact arithmetic).
"""
from __future__ import annotations

import math

import numpy as np

from . import helmholtz_oracle as H
from .pde_oracle import C_CUBE, C_PANEL, face_nodes, lattice, spacing, stencil_apply


def helmholtz_stencil_apply(u, n: int, kappa: float) -> np.ndarray:
    """A u = -Delta_h u - kappa^2 u (u real or complex): the Laplace stencil on the real and
    imaginary parts, minus kappa^2 u."""
    u = np.asarray(u)
    if np.iscomplexobj(u):
        lap = stencil_apply(u.real, n) + 1j * stencil_apply(u.imag, n)
    else:
        lap = stencil_apply(u, n)
    return lap - kappa * kappa * u


def green(x, y, kappa: float):
    """G(x_i, y_j) = exp(i kappa r) / (4 pi r) as a dense [len(x), len(y)] matrix (r > 0 assumed)."""
    d = np.sqrt(((np.asarray(x)[:, None, :] - np.asarray(y)[None, :, :]) ** 2).sum(-1))
    return np.exp(1j * kappa * d) / (4.0 * math.pi * d)


def self_cell(h: float, kappa: float) -> complex:
    """c_self: the own-cell integral of G to second order in kappa h (reading R57)."""
    return h * h * C_CUBE / (4.0 * math.pi) + 1j * kappa * h ** 3 / (4.0 * math.pi)


def self_panel(a: float, kappa: float) -> complex:
    """S_ii: the own-panel integral of a^-2 ... times a^2, to second order in kappa a (R57)."""
    return a * C_PANEL / (4.0 * math.pi) + 1j * kappa * a * a / (4.0 * math.pi)


def boundary_matrix(Y, a: float, kappa: float) -> np.ndarray:
    """S_ij = a^2 G(y_i, y_j) (i != j), S_ii = self_panel(a, kappa)."""
    Y = np.asarray(Y)
    d = np.sqrt(((Y[:, None, :] - Y[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(d, 1.0)
    S = a * a * np.exp(1j * kappa * d) / (4.0 * math.pi * d)
    np.fill_diagonal(S, self_panel(a, kappa))
    return S


class HelmholtzPrecond:
    """M r of the module docstring; both potential sums by the Helmholtz FMM oracle on one plan
    over the lattice nodes followed by the face panel centres."""

    def __init__(self, n: int, stride: int, p: int, ncrit: int, theta: float, kappa: float, boundary: bool = True):
        self.n, self.h, self.kappa = n, spacing(n), float(kappa)
        self.X = lattice(n)
        self.Y, self.a = face_nodes(n, stride)
        self.boundary = boundary
        self.plan = H.PlanH(np.concatenate([self.X, self.Y], 0), p, ncrit, theta, kappa)
        self.S = boundary_matrix(self.Y, self.a, kappa) if boundary else None
        self.c_self = self_cell(self.h, kappa)

    def volume(self, r):
        N = self.n ** 3
        r = np.asarray(r, dtype=complex)
        q = np.zeros(N + self.Y.shape[0], complex)
        q[:N] = self.h ** 3 / (4.0 * math.pi) * r
        phi = self.plan.eval(q)
        return phi[:N] + self.c_self * r, phi[N:]

    def apply(self, r):
        N = self.n ** 3
        uv, uf = self.volume(r)
        if not self.boundary:
            return uv
        sigma = np.linalg.solve(self.S, -uf)
        q = np.zeros(N + self.Y.shape[0], complex)
        q[N:] = self.a * self.a / (4.0 * math.pi) * sigma
        return uv + self.plan.eval(q)[:N]


def dense_precond(n: int, stride: int, kappa: float, boundary: bool = True) -> np.ndarray:
    """The exact-sum preconditioner as a dense [N, N] matrix (no FMM): the limit of
    HelmholtzPrecond as p grows and theta shrinks (small n only)."""
    h = spacing(n)
    X = lattice(n)
    Y, a = face_nodes(n, stride)
    d = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(d, 1.0)
    V = h ** 3 * np.exp(1j * kappa * d) / (4.0 * math.pi * d)
    np.fill_diagonal(V, self_cell(h, kappa))
    if not boundary:
        return V
    Gyx = a * a * green(X, Y, kappa)          # [N, nf]: layer potential at the nodes (per sigma)
    Gfx = h ** 3 * green(Y, X, kappa)         # [nf, N]: volume potential at the panels (per r)
    S = boundary_matrix(Y, a, kappa)
    return V - Gyx @ np.linalg.solve(S, Gfx)


def gmres(apply_A, b, apply_M=None, rtol=1e-8, maxit=200):
    """Right-preconditioned GMRES of the module docstring. Returns x and the history of the
    residual estimates |g_{k+1}| / ||b|| (history[0] = 1)."""
    b = np.asarray(b, dtype=complex)
    M = apply_M if apply_M else (lambda v: v.copy())
    nb = float(np.linalg.norm(b))
    hist = [1.0]
    x = np.zeros_like(b)
    if nb == 0.0 or maxit == 0:
        return x, hist
    V = [b / nb]
    Hm = np.zeros((maxit + 1, maxit), complex)
    cs = np.zeros(maxit, complex)
    sn = np.zeros(maxit, complex)
    g = np.zeros(maxit + 1, complex)
    g[0] = nb
    k = 0
    for k in range(maxit):
        w = apply_A(M(V[k]))
        for j in range(k + 1):  # modified Gram-Schmidt
            Hm[j, k] = np.vdot(V[j], w)
            w = w - Hm[j, k] * V[j]
        Hm[k + 1, k] = np.linalg.norm(w)
        for j in range(k):  # previous rotations
            t = cs[j] * Hm[j, k] + sn[j] * Hm[j + 1, k]
            Hm[j + 1, k] = -np.conj(sn[j]) * Hm[j, k] + np.conj(cs[j]) * Hm[j + 1, k]
            Hm[j, k] = t
        # new rotation [[c, s], [-conj(s), conj(c)]] with c = conj(a) / rho, s = h / rho maps
        # (a, h) to (rho, 0), rho = sqrt(|a|^2 + h^2) (h = H[k+1, k] is real and >= 0)
        a, c = Hm[k, k], Hm[k + 1, k].real
        den = math.sqrt(abs(a) ** 2 + c * c)
        cs[k] = np.conj(a) / den if den > 0 else 1.0
        sn[k] = c / den if den > 0 else 0.0
        Hm[k, k] = cs[k] * a + sn[k] * c
        Hm[k + 1, k] = 0.0
        g[k + 1] = -np.conj(sn[k]) * g[k]
        g[k] = cs[k] * g[k]
        hist.append(abs(g[k + 1]) / nb)
        done = hist[-1] <= rtol or Hm[k, k] == 0.0
        if not done and c > 0.0:
            V.append(w / c)
        if done or c == 0.0:
            break
    m = k + 1
    y = np.linalg.solve(np.triu(Hm[:m, :m]), g[:m])
    u = sum(y[j] * V[j] for j in range(m))
    return M(u), hist
