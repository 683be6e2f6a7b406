"""Design check (numpy; not product code, not the oracle) for M2L v4: the per-pair rotation
form of the M2L translation with a FIXED rotation matrix (Wigner d at pi/2), so that the only
pair-dependent operators are diagonal z-rotations and the z-axis (Hankel) translation.

PAPER.md:151-153 (§2.2): "Rotating the multipole expansion so that the translation is along
the z-axis reduces the complexity from O(p^4) to O(p^3)". The rotation about y by beta is
written as P . Rz(beta) . P^-1 with P = Rx(-pi/2) fixed, so

    Lambda = A(Q)^T Z(rho) A(Q) M,   Q = Ry(-b) Rz(-a),  A(Ry(-b)) = A(P) A(Rz(-b)) A(P^-1)

where A(R) is the action of rotation R on one degree's coefficients (real 2n+1 representation),
A(Rz(.)) is a 2x2 rotation per order m and A(P) is a fixed sparse matrix (about half its
entries vanish). This script derives the real matrices numerically, checks the factorised
pipeline against the dense M2L formula of SURVEY §8(c) c.1, and prints the non-zero counts.

    python tools/proto_m2l_v4.py [p]
"""
import math
import sys

import numpy as np
from scipy.special import lpmv


def sph(v):
    x, y, z = v
    r = math.sqrt(x * x + y * y + z * z)
    return r, max(-1.0, min(1.0, z / r)), math.atan2(y, x)


def R_all(v, p):
    """regular solid harmonics R_n^m, all m in [-n, n]"""
    r, ct, ph = sph(v)
    out = {}
    for n in range(p + 1):
        for m in range(0, n + 1):
            val = r ** n * lpmv(m, n, ct) * np.exp(1j * m * ph) / math.factorial(n + m)
            out[(n, m)] = val
            out[(n, -m)] = (-1) ** m * np.conj(val)
    return out


def I_all(v, p):
    r, ct, ph = sph(v)
    out = {}
    for n in range(p + 1):
        for m in range(0, n + 1):
            val = math.factorial(n - m) * lpmv(m, n, ct) * np.exp(1j * m * ph) / r ** (n + 1)
            out[(n, m)] = val
            out[(n, -m)] = (-1) ** m * np.conj(val)
    return out


def rot_complex(Q, n, rng):
    """A with conj R_n^m(Q x) = sum_m' A[m, m'] conj R_n^m'(x) (indices m + n)."""
    k = 4 * (2 * n + 1)
    X = rng.standard_normal((k, 3))
    B = np.array([[np.conj(R_all(x, n)[(n, m)]) for m in range(-n, n + 1)] for x in X])
    Y = np.array([[np.conj(R_all(Q @ x, n)[(n, m)]) for m in range(-n, n + 1)] for x in X])
    A, *_ = np.linalg.lstsq(B, Y, rcond=None)
    return A.T  # Y = B A^T


def to_real(n, c):
    """real 2n+1 vector of a symmetric coefficient set c[m + n]: [Re c0, Re c1, Im c1, ...]"""
    r = np.zeros(2 * n + 1)
    r[0] = c[n].real
    for m in range(1, n + 1):
        r[2 * m - 1] = c[n + m].real
        r[2 * m] = c[n + m].imag
    return r


def from_real(n, r):
    c = np.zeros(2 * n + 1, complex)
    c[n] = r[0]
    for m in range(1, n + 1):
        v = r[2 * m - 1] + 1j * r[2 * m]
        c[n + m] = v
        c[n - m] = (-1) ** m * np.conj(v)
    return c


def real_op(n, f):
    """real matrix of a complex linear map f acting on symmetric coefficient vectors"""
    Mr = np.zeros((2 * n + 1, 2 * n + 1))
    for k in range(2 * n + 1):
        e = np.zeros(2 * n + 1)
        e[k] = 1.0
        Mr[:, k] = to_real(n, f(from_real(n, e)))
    return Mr


def Rx(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]])


def Ry(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


def Rz(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])


def main(p=6):
    rng = np.random.default_rng(1)
    P = Rx(-math.pi / 2)
    # check Ry(b) = P Rz(b) P^-1
    b = 0.7
    assert np.allclose(Ry(b), P @ Rz(b) @ P.T)
    worst = 0.0
    nnz = 0
    for trial in range(3):
        d = rng.standard_normal(3) * 3
        rho = np.linalg.norm(d)
        a = math.atan2(d[1], d[0])
        bb = math.acos(d[2] / rho)
        Q = Ry(-bb) @ Rz(-a)
        assert np.allclose(Q @ d, [0, 0, rho])
        # dense M2L on a random symmetric M: Lambda_j^k = sum (-1)^n M_n^m I_{j+n}^{k+m}(d)
        I = I_all(d, 2 * p)
        M = {n: from_real(n, rng.standard_normal(2 * n + 1)) for n in range(p + 1)}
        L = {}
        for j in range(p + 1):
            c = np.zeros(2 * j + 1, complex)
            for k in range(-j, j + 1):
                s = 0
                for n in range(p + 1):
                    for m in range(-n, n + 1):
                        s += (-1) ** n * M[n][m + n] * I[(j + n, k + m)]
                c[k + j] = s
            L[j] = c
        # factorised: M' = A(Q) M ; Lambda' = Z(rho) M' ; Lambda = A(Q)^T Lambda'
        Mp = {}
        for n in range(p + 1):
            A = rot_complex(Q, n, rng)
            Mp[n] = A @ M[n]
        Lp = {}
        for j in range(p + 1):
            c = np.zeros(2 * j + 1, complex)
            for k in range(-j, j + 1):
                m = -k
                s = 0
                for n in range(abs(m), p + 1):
                    s += (-1) ** n * Mp[n][m + n] * math.factorial(j + n) / rho ** (j + n + 1)
                c[k + j] = s
            Lp[j] = c
        for j in range(p + 1):
            A = rot_complex(Q, j, rng)
            Lj = A.T @ Lp[j]
            err = np.abs(Lj - L[j]).max() / max(1e-300, np.abs(L[j]).max())
            worst = max(worst, err)
    print(f"factorised A(Q)^T Z A(Q) vs dense: max rel err {worst:.2e}")
    # J-trick: A(Ry(t)) = A(P) A(Rz(t)) A(P^-1) (or reversed): check, and count non-zeros of A(P)
    for n in range(p + 1):
        t = 0.37
        ARy = rot_complex(Ry(t), n, rng)
        AP = rot_complex(P, n, rng)
        APi = rot_complex(P.T, n, rng)
        ARz = rot_complex(Rz(t), n, rng)
        e1 = np.abs(AP @ ARz @ APi - ARy).max()
        e2 = np.abs(APi @ ARz @ AP - ARy).max()
        rP = real_op(n, lambda c: AP @ c)
        rPi = real_op(n, lambda c: APi @ c)
        nz = int((np.abs(rP) > 1e-10).sum())
        nzi = int((np.abs(rPi) > 1e-10).sum())
        nnz += nz
        print(f"n={n}: |AP Rz APi - Ry|={e1:.1e} |APi Rz AP - Ry|={e2:.1e} nnz(A(P))={nz} nnz(A(P^-1))={nzi} "
              f"of {(2 * n + 1) ** 2}")
    print("total nnz A(P):", nnz)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 6)


def structure(p=6):
    """real matrices of the four fixed factors and their relations"""
    rng = np.random.default_rng(2)
    P = Rx(-math.pi / 2)
    for n in range(1, p + 1):
        AP = rot_complex(P, n, rng)
        APi = rot_complex(P.T, n, rng)
        F = real_op(n, lambda c: AP @ c)
        G = real_op(n, lambda c: APi @ c)
        Ft = real_op(n, lambda c: AP.T @ c)
        Gt = real_op(n, lambda c: APi.T @ c)
        F[np.abs(F) < 1e-12] = 0
        G[np.abs(G) < 1e-12] = 0
        Ft[np.abs(Ft) < 1e-12] = 0
        Gt[np.abs(Gt) < 1e-12] = 0
        def rel(X, Y):
            with np.errstate(divide="ignore", invalid="ignore"):
                r = np.where(Y != 0, X / Y, np.nan)
            return r
        print(f"n={n}")
        np.set_printoptions(precision=4, suppress=True, linewidth=200)
        if n <= 2:
            print("F\n", F, "\nG\n", G, "\nFt\n", Ft, "\nGt\n", Gt)
        print(" G/F ratios:", np.unique(np.round(rel(G, F)[~np.isnan(rel(G, F))], 6)))
        print(" Gt vs F^T:", np.unique(np.round(rel(Gt, F.T)[~np.isnan(rel(Gt, F.T))], 6)))
        print(" Ft vs G^T:", np.unique(np.round(rel(Ft, G.T)[~np.isnan(rel(Ft, G.T))], 6)))
        print(" Ft/F ratios:", np.unique(np.round(rel(Ft, F)[~np.isnan(rel(Ft, F))], 6)))


def zrot(n, x, t):
    """real repr of c^m -> e^{i m t} c^m"""
    y = x.copy()
    for m in range(1, n + 1):
        c, s = math.cos(m * t), math.sin(m * t)
        re, im = x[2 * m - 1], x[2 * m]
        y[2 * m - 1] = c * re - s * im
        y[2 * m] = s * re + c * im
    return y


def pipeline_check(p=6):
    rng = np.random.default_rng(3)
    P = Rx(-math.pi / 2)
    F, G, Ft, Gt = {}, {}, {}, {}
    for n in range(p + 1):
        AP = rot_complex(P, n, rng)
        APi = rot_complex(P.T, n, rng)
        F[n] = real_op(n, lambda c: AP @ c)
        G[n] = real_op(n, lambda c: APi @ c)
        Ft[n] = real_op(n, lambda c: AP.T @ c)
        Gt[n] = real_op(n, lambda c: APi.T @ c)
        for X in (F, G, Ft, Gt):
            X[n][np.abs(X[n]) < 1e-12] = 0
        # relations: G = sG * F ; Ft = W^-1 G^T W ; Gt = W^-1 F^T W with W = diag(1, 2, 2, ...)?
        w = np.array([1.0] + [2.0] * (2 * n))
        e1 = np.abs(Ft[n] - np.diag(1 / w) @ G[n].T @ np.diag(w)).max()
        e2 = np.abs(Gt[n] - np.diag(1 / w) @ F[n].T @ np.diag(w)).max()
        e1b = np.abs(Ft[n] - np.diag(w) @ G[n].T @ np.diag(1 / w)).max()
        print(f"n={n} Ft=W^-1 G^T W: {e1:.1e} (W G^T W^-1: {e1b:.1e})  Gt=W^-1 F^T W: {e2:.1e}")
    worst = 0
    for trial in range(4):
        d = rng.standard_normal(3) * 3
        rho = np.linalg.norm(d)
        a = math.atan2(d[1], d[0])
        b = math.acos(d[2] / rho)
        I = I_all(d, 2 * p)
        M = {n: from_real(n, rng.standard_normal(2 * n + 1)) for n in range(p + 1)}
        # dense
        Ld = {}
        for j in range(p + 1):
            c = np.zeros(2 * j + 1, complex)
            for k in range(-j, j + 1):
                c[k + j] = sum((-1) ** n * M[n][m + n] * I[(j + n, k + m)] for n in range(p + 1)
                               for m in range(-n, n + 1))
            Ld[j] = to_real(j, c)
        # pipeline
        W = {}
        for n in range(p + 1):
            x = to_real(n, M[n])
            x = zrot(n, x, a)
            x = G[n] @ x
            x = zrot(n, x, b)
            x = F[n] @ x
            W[n] = x
        for j in range(p + 1):
            y = np.zeros(2 * j + 1)
            for m in range(0, j + 1):
                for part in ((0,) if m == 0 else (0, 1)):
                    idx = 0 if m == 0 else 2 * m - 1 + part
                    s = 0.0
                    for n in range(m, p + 1):
                        wi = W[n][0 if m == 0 else 2 * m - 1 + part]
                        s += (-1) ** n * wi * math.factorial(j + n) / rho ** (j + n + 1)
                    # Lambda'_j^{-m} = s (complex); Lambda'_j^m = (-1)^m conj
                    y[idx] = (-1) ** m * (s if part == 0 else -s)
            y = Ft[j] @ y
            y = zrot(j, y, b)
            y = Gt[j] @ y
            y = zrot(j, y, a)
            err = np.abs(y - Ld[j]).max() / np.abs(Ld[j]).max()
            worst = max(worst, err)
    print(f"real pipeline vs dense: {worst:.2e}")
