"""Pins of the Helmholtz PDE oracle (oracle/pde_helmholtz_oracle.py): the FMM as a preconditioner
for the 3D Helmholtz equation on a [-1,1]^3 lattice with Dirichlet faces, inside GMRES
(§4.2). Each pin checks the oracle against something other
than itself: quadrature of the Green's function, the discrete eigenfunctions, the kappa -> 0
limit against the pinned Laplace oracle, the exact-sum (dense) preconditioner, the radiating
solution reproduced by the single layer, dense linear algebra, and the paper's claim that the
FMM preconditioner's convergence does not depend on the problem size."""
import math

import numpy as np
import pytest

from oracle import pde_helmholtz_oracle as PH
from oracle import pde_oracle as P


def _cube_integral(f, h):
    """int over the cube of side h centred at 0 of f(r) dV, f smooth (Gauss-Legendre 24^3)."""
    t, w = np.polynomial.legendre.leggauss(24)
    x = 0.5 * h * t
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    W = np.einsum("i,j,k->ijk", w, w, w) * (0.5 * h) ** 3
    return (W * f(np.sqrt(X * X + Y * Y + Z * Z))).sum()


def _square_integral(f, a):
    t, w = np.polynomial.legendre.leggauss(32)
    x = 0.5 * a * t
    X, Y = np.meshgrid(x, x, indexing="ij")
    return (np.outer(w, w) * (0.5 * a) ** 2 * f(np.sqrt(X * X + Y * Y))).sum()


@pytest.mark.parametrize("h,kappa", [(2.0 / 64, 7.0), (0.25, 1.0), (0.1, 3.0)])
def test_self_integrals_to_second_order(h, kappa):
    """c_self and S_ii are the own-cell / own-panel integrals of G = exp(i kappa r) / (4 pi r) up to
    the third term of exp(i kappa r) / r = 1/r + i kappa - kappa^2 r / 2 + ...: the remainder
    matches that term (so both kept terms are right)."""
    # 1/r part exactly (pinned constants), the smooth rest by Gauss quadrature
    smooth = lambda r: (np.exp(1j * kappa * r) - 1.0) / np.where(r > 0, r, 1.0) / (4 * math.pi)  # noqa: E731
    exact = h * h * P.C_CUBE / (4 * math.pi) + _cube_integral(smooth, h)
    third = -kappa * kappa / 2 * _cube_integral(lambda r: r, h) / (4 * math.pi)
    rem = exact - PH.self_cell(h, kappa)
    assert abs(rem - third) <= 0.2 * abs(third)
    exact_p = h * P.C_PANEL / (4 * math.pi) + _square_integral(smooth, h)
    third_p = -kappa * kappa / 2 * _square_integral(lambda r: r, h) / (4 * math.pi)
    assert abs(exact_p - PH.self_panel(h, kappa) - third_p) <= 0.2 * abs(third_p)


def test_stencil_eigenfunction_and_kappa_zero():
    n, kappa = 9, 7.0
    h = P.spacing(n)
    X = P.lattice(n)
    u = np.prod(np.sin(math.pi * (X + 1) / 2), axis=1)
    lam = 3 * (2 - 2 * math.cos(math.pi * h / 2)) / h ** 2  # discrete Dirichlet eigenvalue of -Delta_h
    Au = PH.helmholtz_stencil_apply(u, n, kappa)
    assert np.abs(Au - (lam - kappa * kappa) * u).max() < 1e-11 * lam
    rng = np.random.default_rng(3)
    v = rng.standard_normal(n ** 3) + 1j * rng.standard_normal(n ** 3)
    assert np.array_equal(PH.helmholtz_stencil_apply(v, n, 0.0), P.stencil_apply(v.real, n) + 1j * P.stencil_apply(v.imag, n))
    # A - kappa^2 I is indefinite at kappa = 7, h = 1/5: CG does not apply (GMRES reading)
    ev = np.linalg.eigvalsh(P.stencil_matrix(5)) - kappa * kappa
    assert ev.min() < 0 < ev.max()


def test_dense_preconditioner_kappa_zero_is_laplace():
    """kappa -> 0: the exact-sum preconditioner equals the Laplace oracle's (pinned) FMM preconditioner
    up to that FMM's truncation."""
    n = 5
    rng = np.random.default_rng(4)
    r = rng.standard_normal(n ** 3)
    D = PH.dense_precond(n, 1, 0.0)
    assert np.abs(D.imag).max() == 0.0
    ML = P.FmmPrecond(n, 1, 12, 8, 0.3)
    zl = ML.apply(r)
    assert np.linalg.norm(D.real @ r - zl) <= 1e-7 * np.linalg.norm(zl)


def test_fmm_preconditioner_matches_exact_sums_and_is_linear():
    n, kappa = 5, 4.0
    rng = np.random.default_rng(5)
    r = rng.standard_normal(n ** 3) + 0.5j * rng.standard_normal(n ** 3)
    zd = PH.dense_precond(n, 1, kappa) @ r
    M = PH.HelmholtzPrecond(n, 1, 8, 16, 0.3, kappa)
    z = M.apply(r)
    assert np.linalg.norm(z - zd) <= 1e-4 * np.linalg.norm(zd)  # FMM truncation at p = 8
    z2 = M.apply(2.0 * r - 3.0j * r.conj())
    z3 = 2.0 * z - 3.0j * M.apply(r.conj())
    assert np.linalg.norm(z2 - z3) <= 1e-12 * np.linalg.norm(z3)
    assert not M.apply(np.zeros(n ** 3)).any()
    # volume part only: the same without the boundary correction
    Mv = PH.HelmholtzPrecond(n, 1, 8, 16, 0.3, kappa, boundary=False)
    zv = PH.dense_precond(n, 1, kappa, boundary=False) @ r
    assert np.linalg.norm(Mv.apply(r) - zv) <= 1e-4 * np.linalg.norm(zv)


def _layer_error(n, kappa):
    Y, a = P.face_nodes(n, 1)
    x0 = np.array([2.5, 0.3, -0.2])
    g = lambda Z: PH.green(Z, x0[None, :], kappa)[:, 0]  # noqa: E731
    sigma = np.linalg.solve(PH.boundary_matrix(Y, a, kappa), g(Y))
    X = P.lattice(n)
    inner = X[(np.abs(X) < 0.75).all(1)]
    us = (a * a * PH.green(inner, Y, kappa)) @ sigma
    return np.abs(us - g(inner)).max() / np.abs(g(inner)).max()


def test_single_layer_reproduces_radiating_field():
    """For g = G(., x0), x0 outside the cube (a solution of the Helmholtz equation inside), the
    single layer with S sigma = g|faces equals g inside, up to the panel discretisation. Below the
    first interior Dirichlet eigenvalue (kappa = 2 < sqrt(3) pi / 2) as accurate as the Laplace
    case; at kappa = 7 (2 % above the eigenvalue sqrt(19) pi / 2 = 6.85, where the single layer is
    singular) the error is larger but falls with the panel size."""
    assert _layer_error(15, 2.0) <= 0.02
    e7, e15 = _layer_error(7, 7.0), _layer_error(15, 7.0)
    assert e15 <= 0.2 and e15 < 0.3 * e7


def test_gmres_dense_systems():
    rng = np.random.default_rng(6)
    m = 40
    A = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)) + 4 * np.eye(m)
    b = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    x, hist = PH.gmres(lambda v: A @ v, b, None, 1e-12, 200)
    assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-10 * np.linalg.norm(x)
    assert hist[0] == 1.0 and hist[-1] <= 1e-12 and len(hist) - 1 <= m
    assert all(hist[k + 1] <= hist[k] * (1 + 1e-12) for k in range(len(hist) - 1))  # GMRES: non-increasing
    # the residual estimate is the true residual of the returned iterate
    x5, h5 = PH.gmres(lambda v: A @ v, b, None, 1e-30, 5)
    assert len(h5) == 6 and abs(np.linalg.norm(b - A @ x5) / np.linalg.norm(b) - h5[-1]) <= 1e-10
    # exact preconditioner: one iteration; right preconditioning returns x = M u
    Ai = np.linalg.inv(A)
    x1, h1 = PH.gmres(lambda v: A @ v, b, lambda v: Ai @ v, 1e-10, 10)
    assert len(h1) == 2 and np.linalg.norm(A @ x1 - b) <= 1e-10 * np.linalg.norm(b)
    x0, h0 = PH.gmres(lambda v: A @ v, np.zeros(m))
    assert not x0.any() and h0 == [1.0]


def test_preconditioned_gmres_mesh_independent():
    """with the (exact-sum) FMM preconditioner the GMRES iteration count does not
    grow with the problem size at fixed kappa; unpreconditioned GMRES needs O(1/h) iterations."""
    kappa = 4.0
    rng = np.random.default_rng(0)
    its, its0 = [], []
    for n in (7, 15):
        b = rng.standard_normal(n ** 3)
        A = lambda v, n=n: PH.helmholtz_stencil_apply(v, n, kappa)  # noqa: E731
        x0, h0 = PH.gmres(A, b, None, 1e-8, 1000)
        D = PH.dense_precond(n, 1, kappa)
        x, h1 = PH.gmres(A, b, lambda v: D @ v, 1e-8, 100)
        assert np.linalg.norm(x - x0) <= 1e-6 * np.linalg.norm(x0)
        its.append(len(h1) - 1)
        its0.append(len(h0) - 1)
    assert max(its) <= 12 and its[1] - its[0] <= 2
    assert its0[1] > 1.7 * its0[0] and its0[0] > 3 * its[0]
