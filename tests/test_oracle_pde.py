"""Pins of the NEXT-2 oracle (oracle/pde_oracle.py): the FMM as a low-accuracy preconditioner
for the 3D Laplace equation on a [-1,1]^3 lattice with Dirichlet faces (PAPER.md:439-471,
§4.2). Each pin checks the oracle against something other than itself: closed forms,
quadrature, dense linear algebra, the harmonic-reproduction property of the single layer,
and the paper's mesh-independence claim."""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import pde_oracle as P


def test_self_integrals_match_quadrature():
    # cube: div(x/|x|) = 2/|x| -> int_V 1/|x| = 1/2 sum_faces int (d/|x|) dA, d = 1/2
    face, _ = integrate.dblquad(lambda z, y: 0.5 / math.sqrt(0.25 + y * y + z * z), -0.5, 0.5, -0.5, 0.5,
                                epsabs=1e-13, epsrel=1e-13)
    assert abs(6 * 0.5 * face - P.C_CUBE) < 1e-11
    # square: div_2(x/|x|) = 1/|x| -> int_A 1/|x| = sum_edges int (d/|x|) ds, d = 1/2
    edge, _ = integrate.quad(lambda t: 0.5 / math.sqrt(0.25 + t * t), -0.5, 0.5, epsabs=1e-14, epsrel=1e-14)
    assert abs(4 * edge - P.C_PANEL) < 1e-12


def test_lattice_and_faces():
    X = P.lattice(3)
    assert X.shape == (27, 3) and np.allclose(X[1] - X[0], [0.5, 0, 0]) and np.allclose(X[3] - X[0], [0, 0.5, 0])
    assert np.allclose(X[0], [-0.5, -0.5, -0.5]) and np.allclose(X[-1], [0.5, 0.5, 0.5])
    Y, a = P.face_nodes(7, 2)
    assert Y.shape == (6 * 16, 3) and a == 0.5
    assert (np.abs(Y).max(1) == 1.0).all()  # every panel centre lies on a face
    assert len({tuple(r) for r in np.round(Y, 12)}) == Y.shape[0]  # distinct


def test_stencil_eigenfunction_and_unit_vector():
    n = 9
    h = P.spacing(n)
    X = P.lattice(n)
    u = np.prod(np.sin(math.pi * (X + 1) / 2), axis=1)
    lam = 3 * (2 - 2 * math.cos(math.pi * h / 2)) / h ** 2  # discrete Dirichlet eigenvalue
    assert np.abs(P.stencil_apply(u, n) - lam * u).max() < 1e-11 * lam
    e = np.zeros(n ** 3)
    c = (n // 2) * (1 + n + n * n)
    e[c] = 1.0
    Ae = P.stencil_apply(e, n) * h * h
    assert Ae[c] == 6.0 and sorted(Ae[np.nonzero(Ae)].tolist()) == [-1.0] * 6 + [6.0]


def test_stencil_symmetric_positive_definite():
    A = P.stencil_matrix(5)
    assert np.array_equal(A, A.T)
    assert np.linalg.eigvalsh(A).min() > 0


def test_pcg_identity_matches_dense_solve():
    n = 7
    rng = np.random.default_rng(1)
    b = rng.standard_normal(n ** 3)
    x, hist = P.pcg(lambda v: P.stencil_apply(v, n), b, None, 1e-12, 1000)
    xd = np.linalg.solve(P.stencil_matrix(n), b)
    assert np.linalg.norm(x - xd) <= 1e-10 * np.linalg.norm(xd)
    assert hist[0] == 1.0 and hist[-1] <= 1e-12 and len(hist) - 1 <= n ** 3
    x0, h0 = P.pcg(lambda v: P.stencil_apply(v, n), np.zeros(n ** 3))
    assert not x0.any() and h0 == [1.0]


def test_single_layer_reproduces_harmonic_function():
    """For harmonic g (source outside the cube) the single layer with S sigma = g|faces equals g
    inside (Dirichlet uniqueness), up to the panel discretisation: the boundary correction step."""
    n = 15
    Y, a = P.face_nodes(n, 1)
    x0 = np.array([2.5, 0.3, -0.2])
    g = lambda Z: 1.0 / np.linalg.norm(Z - x0, axis=1)  # noqa: E731
    sigma = np.linalg.solve(P.boundary_matrix(Y, a), g(Y))
    X = P.lattice(n)
    inner = X[(np.abs(X) < 0.75).all(1)]
    d = np.linalg.norm(inner[:, None, :] - Y[None, :, :], axis=2)
    us = (a * a / (4 * math.pi) / d) @ sigma
    assert np.abs(us - g(inner)).max() <= 0.02 * np.abs(g(inner)).max()


def test_fmm_preconditioner_approximates_inverse_and_is_linear():
    n = 7
    X = P.lattice(n)
    u = np.prod(np.sin(math.pi * (X + 1) / 2), axis=1) * np.exp(X[:, 0])
    M = P.FmmPrecond(n, 1, 6, 16, 0.5)
    z = M.apply(P.stencil_apply(u, n))
    assert np.linalg.norm(z - u) <= 0.08 * np.linalg.norm(u)  # discretisation-level error at h = 1/4
    rng = np.random.default_rng(2)
    r1, r2 = rng.standard_normal(n ** 3), rng.standard_normal(n ** 3)
    lhs = M.apply(2.0 * r1 - 3.0 * r2)
    rhs = 2.0 * M.apply(r1) - 3.0 * M.apply(r2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    assert not M.apply(np.zeros(n ** 3)).any()


@pytest.mark.parametrize("n,stride", [(7, 1), (15, 1)])
def test_fmm_preconditioned_cg_mesh_independent(n, stride):
    """the FMM preconditioner's convergence rate is independent of the problem
    size; unpreconditioned CG needs O(1/h) iterations."""
    rng = np.random.default_rng(0)
    b = rng.standard_normal(n ** 3)
    A = lambda v: P.stencil_apply(v, n)  # noqa: E731
    x0, h0 = P.pcg(A, b, None, 1e-8, 5000)
    M = P.FmmPrecond(n, stride, 4, 32, 0.5)
    x, h1 = P.pcg(A, b, M.apply, 1e-8, 200)
    assert len(h1) - 1 <= 12 < len(h0) - 1
    assert np.linalg.norm(x - x0) <= 1e-6 * np.linalg.norm(x0)
