"""oracle/pde_oracle.py — TEST INFRASTRUCTURE ONLY (NEXT-2).

Plain numpy reference for the second workload of arXiv:1602.02244: the FMM used as a
low-accuracy preconditioner inside a Krylov solve of the 3D Laplace equation on a
[-1,1]^3 lattice with Dirichlet conditions at the faces (§4.2; Fig 5,
PAPER.md:448-453; "viewing these methods as a preconditioner instead of a direct solver
significantly reduces the accuracy requirements"). Only ``tests/`` and
the measurement tools may import it; it shares no code with ``paper_1602_02244_b200``.

The paper gives no formulas for this experiment. The readings (R30-R36):
  * lattice: the n^3 interior nodes x = -1 + (i+1) h, h = 2/(n+1) (h = 2^-5 -> n = 63),
    x-fastest index i + n (j + n k);
  * A = -Delta_h, the 7-point stencil with zero Dirichlet ghost values;
  * preconditioner M r (SPEC.md:434-442 precond_fmm, Ibeid et al. in spirit):
      1. volume potential u_v(x_i) = sum_{j != i} h^3 G(x_i, x_j) r_j + c_self r_i,
         G = 1/(4 pi |x - y|), c_self = h^2 C_cube / (4 pi) the integral of G over the
         node's own cell (C_cube = int_{[-1/2,1/2]^3} dV / |x| = 3 ln(2 + sqrt 3) - pi/2),
         the sum by the FMM (same approximation as the mat-vec: p, ncrit, theta);
      2. single-layer densities on face panels: S sigma = -u_v|faces, S_ij = a^2 G(y_i, y_j),
         S_ii = a ln(1 + sqrt 2) / pi (the integral of G over the own square panel of side a);
      3. M r = u_v + sum_j a^2 G(x_i, y_j) sigma_j at the lattice nodes (by the FMM).
    Face panels: on each face the lattice's in-face coordinates with stride s (a = s h).
  * Krylov: flexible preconditioned CG (Polak-Ribiere beta), x0 = 0, stop at
    ||b - A x|| / ||b|| <= rtol (the FMM preconditioner is only approximately symmetric).
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as O

C_CUBE = 3.0 * math.log(2.0 + math.sqrt(3.0)) - math.pi / 2.0  # int over the unit cube of 1/|x|
C_PANEL = 4.0 * math.log(1.0 + math.sqrt(2.0))  # int over the unit square of 1/|x|


def spacing(n: int) -> float:
    return 2.0 / (n + 1)


def lattice(n: int) -> np.ndarray:
    """[n^3, 3] interior nodes, x fastest."""
    h = spacing(n)
    c = -1.0 + (np.arange(n) + 1.0) * h
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], 1)


def stencil_apply(u: np.ndarray, n: int) -> np.ndarray:
    """A u with A = -Delta_h (7-point, zero Dirichlet ghosts): (6 u_c - sum of the 6 neighbours) / h^2."""
    h = spacing(n)
    U = np.zeros((n + 2, n + 2, n + 2))
    U[1:-1, 1:-1, 1:-1] = np.asarray(u, dtype=np.float64).reshape(n, n, n)  # [k][j][i]
    c = U[1:-1, 1:-1, 1:-1]
    nb = (U[1:-1, 1:-1, :-2] + U[1:-1, 1:-1, 2:] + U[1:-1, :-2, 1:-1] + U[1:-1, 2:, 1:-1] + U[:-2, 1:-1, 1:-1]
          + U[2:, 1:-1, 1:-1])
    return ((6.0 * c - nb) / (h * h)).ravel()


def stencil_matrix(n: int) -> np.ndarray:
    """Dense A (small n only), column by column from stencil_apply."""
    N = n ** 3
    A = np.zeros((N, N))
    e = np.zeros(N)
    for j in range(N):
        e[j] = 1.0
        A[:, j] = stencil_apply(e, n)
        e[j] = 0.0
    return A


def face_nodes(n: int, stride: int) -> tuple[np.ndarray, float]:
    """Panel centres on the 6 faces (x = -1, x = +1, y = -1, y = +1, z = -1, z = +1), the two
    in-face coordinates being the lattice coordinates 0, s, 2s, ... (first fastest); panel side a = s h."""
    h = spacing(n)
    c = -1.0 + (np.arange(0, n, stride) + 1.0) * h
    v, u = np.meshgrid(c, c, indexing="ij")
    u, v = u.ravel(), v.ravel()
    out = []
    for axis in range(3):
        for side in (-1.0, 1.0):
            f = np.zeros((u.size, 3))
            others = [d for d in range(3) if d != axis]
            f[:, axis] = side
            f[:, others[0]] = u
            f[:, others[1]] = v
            out.append(f)
    return np.concatenate(out, 0), stride * h


def boundary_matrix(Y: np.ndarray, a: float) -> np.ndarray:
    """S_ij = a^2 / (4 pi |y_i - y_j|), S_ii = a C_PANEL / (4 pi) (own-panel integral)."""
    d = np.sqrt(((Y[:, None, :] - Y[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(d, 1.0)
    S = a * a / (4.0 * math.pi * d)
    np.fill_diagonal(S, a * C_PANEL / (4.0 * math.pi))
    return S


class FmmPrecond:
    """M r of the module docstring; the two potential sums by the oracle FMM on one plan over
    the lattice nodes followed by the face panel centres."""

    def __init__(self, n: int, stride: int, p: int, ncrit: int, theta: float, boundary: bool = True,
                 nthreads: int = 0):
        self.n, self.h = n, spacing(n)
        self.X = lattice(n)
        self.Y, self.a = face_nodes(n, stride)
        self.boundary = boundary
        self.nthreads = nthreads
        self.plan = O.Plan(np.concatenate([self.X, self.Y], 0), p, ncrit, theta)
        self.S = boundary_matrix(self.Y, self.a) if boundary else None
        self.c_self = self.h * self.h * C_CUBE / (4.0 * math.pi)

    def volume(self, r):
        N = self.n ** 3
        q = np.zeros(N + self.Y.shape[0])
        q[:N] = self.h ** 3 / (4.0 * math.pi) * np.asarray(r)
        phi = self.plan.eval(q, nthreads=self.nthreads)
        return phi[:N] + self.c_self * np.asarray(r), phi[N:]

    def apply(self, r):
        N = self.n ** 3
        uv, uf = self.volume(r)
        if not self.boundary:
            return uv
        sigma = np.linalg.solve(self.S, -uf)
        q = np.zeros(N + self.Y.shape[0])
        q[N:] = self.a * self.a / (4.0 * math.pi) * sigma
        phi = self.plan.eval(q, nthreads=self.nthreads)
        return uv + phi[:N]


def pcg(apply_A, b, apply_M=None, rtol=1e-8, maxit=500):
    """Flexible PCG: x0 = 0; beta = (r_new, z_new - z_old) / (r_old, z_old) (Polak-Ribiere).
    Returns x and the relative-residual history (history[0] = 1)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    nb = float(np.sqrt(b @ b))
    hist = [1.0]
    if nb == 0.0:
        return x, hist
    r = b.copy()
    z = apply_M(r) if apply_M else r.copy()
    d = z.copy()
    rz = float(r @ z)
    for _ in range(maxit):
        q = apply_A(d)
        alpha = rz / float(d @ q)
        x = x + alpha * d
        r = r - alpha * q
        hist.append(float(np.sqrt(r @ r)) / nb)
        if hist[-1] <= rtol:
            break
        zn = apply_M(r) if apply_M else r.copy()
        rzn = float(r @ zn)
        beta = (rzn - float(r @ z)) / rz
        d = zn + beta * d
        z, rz = zn, rzn
    return x, hist
