"""Design check (numpy, not product code, not the oracle): the rotation factorisation of the
scaled class M2L operator used by M2L v3 (m2l_dmma.cu),

    T~(delta0) = Az(-alpha)^L  D^L(beta)  Z~(|delta0|)  D^M(beta)  Az(alpha)^M,

against the dense real operator that build_ops_kernel tabulates. Prints the max relative
difference over random classes; the CUDA build kernel follows the same steps.

    python tools/proto_m2l_rotation.py [p]
"""
import math
import sys

import numpy as np
from scipy.special import lpmv


def real_index(n, m, part):
    return n * n if m == 0 else n * n + 2 * m - 1 + part


def irregular(x, y, z, P):
    r = math.sqrt(x * x + y * y + z * z)
    th = math.acos(z / r)
    ph = math.atan2(y, x)
    I = {}
    for n in range(P + 1):
        for m in range(0, n + 1):
            v = math.factorial(n - m) * lpmv(m, n, math.cos(th)) * np.exp(1j * m * ph) / r ** (n + 1)
            I[(n, m)] = v
            I[(n, -m)] = (-1) ** m * np.conj(v)
    return I


def regular(v, p):
    x, y, z = v
    r = math.sqrt(x * x + y * y + z * z)
    th = math.acos(max(-1.0, min(1.0, z / r))) if r > 0 else 0.0
    ph = math.atan2(y, x)
    R = {}
    for n in range(p + 1):
        for m in range(0, n + 1):
            R[(n, m)] = r ** n * lpmv(m, n, math.cos(th)) * np.exp(1j * m * ph) / math.factorial(n + m)
    return R


def dense_op(d0, dl, p):
    """build_ops_kernel's T~ (NR x NR), d0 = canonical integer offset, dl = level_A - level_B."""
    NR = (p + 1) ** 2
    I = irregular(*d0, 2 * p)
    fA = 2.0 ** (-dl) if dl < 0 else 1.0
    fB = 2.0 ** dl if dl > 0 else 1.0
    T = np.zeros((NR, NR))
    for j in range(p + 1):
        for k in range(j + 1):
            for po in range(2 if k else 1):
                ro = real_index(j, k, po)
                for n in range(p + 1):
                    for m in range(n + 1):
                        for pi in range(2 if m else 1):
                            ri = real_index(n, m, pi)
                            U, V = I[(j + n, k + m)], I[(j + n, k - m)]
                            s = -1.0 if m & 1 else 1.0
                            if m == 0:
                                w = U.real if po == 0 else U.imag
                            elif pi == 0:
                                w = (U.real + s * V.real) if po == 0 else (U.imag + s * V.imag)
                            else:
                                w = -(U.imag - s * V.imag) if po == 0 else (U.real - s * V.real)
                            T[ro, ri] = (-1) ** n * fB ** n * fA ** (j + 1) * w
    return T


def gauss_legendre(k):
    return np.polynomial.legendre.leggauss(k)


def d_blocks(beta, p):
    """Re/Im blocks of the multipole-side rotation Q = Ry(-beta) by exact sphere quadrature
    in the scaled basis u = c_nm v, v = [Re R_n^m, -Im R_n^m]."""
    xs, ws = gauss_legendre(p + 1)
    nphi = 2 * p + 1
    cb, sb = math.cos(-beta), math.sin(-beta)
    Q = np.array([[cb, 0, sb], [0, 1, 0], [-sb, 0, cb]])
    pts, wts = [], []
    for x, w in zip(xs, ws):
        st = math.sqrt(1 - x * x)
        for t in range(nphi):
            ph = 2 * math.pi * t / nphi
            pts.append(np.array([st * math.cos(ph), st * math.sin(ph), x]))
            wts.append(w * 2 * math.pi / nphi)
    Rs = [regular(s, p) for s in pts]
    Rq = [regular(Q @ s, p) for s in pts]
    out = []
    for n in range(p + 1):
        def c(m):
            return math.sqrt(math.factorial(n + m) * math.factorial(n - m) / (2.0 if m == 0 else 1.0))

        norm = (2 * n + 1) / (2 * math.pi)
        Dre = np.zeros((n + 1, n + 1))
        Dim = np.zeros((n + 1, n + 1))  # row/col 0 unused (Im of m = 0)
        for a in range(n + 1):
            for b in range(n + 1):
                sre = sum(w * (c(a) * R1[(n, a)].real) * (c(b) * R0[(n, b)].real) for w, R0, R1 in zip(wts, Rs, Rq))
                Dre[a, b] = norm * sre * c(b) / c(a)
                if a and b:
                    sim = sum(w * (c(a) * R1[(n, a)].imag) * (c(b) * R0[(n, b)].imag) for w, R0, R1 in zip(wts, Rs, Rq))
                    Dim[a, b] = norm * sim * c(b) / c(a)
        out.append((Dre, Dim))
    return out


def factored_apply(X, d0, dl, p):
    NR = (p + 1) ** 2
    x0, y0, z0 = d0
    rho = math.sqrt(x0 * x0 + y0 * y0 + z0 * z0)
    alpha = math.atan2(y0, x0)
    beta = math.acos(z0 / rho)
    fA = 2.0 ** (-dl) if dl < 0 else 1.0
    fB = 2.0 ** dl if dl > 0 else 1.0
    D = d_blocks(beta, p)
    X = X.copy()
    # 1. forward azimuthal rotation (helpers): (re, im) *= e^{i m alpha}
    for n in range(p + 1):
        for m in range(1, n + 1):
            c, s = math.cos(m * alpha), math.sin(m * alpha)
            re, im = X[real_index(n, m, 0)].copy(), X[real_index(n, m, 1)].copy()
            X[real_index(n, m, 0)] = c * re - s * im
            X[real_index(n, m, 1)] = s * re + c * im
    # 2. d-rotation per degree (Re and Im blocks)
    Y = np.zeros_like(X)
    for n in range(p + 1):
        Dre, Dim = D[n]
        xr = np.array([X[real_index(n, m, 0)] for m in range(n + 1)])
        xi = np.array([X[real_index(n, m, 1)] if m else np.zeros(X.shape[1]) for m in range(n + 1)])
        yr, yi = Dre @ xr, Dim @ xi
        for m in range(n + 1):
            Y[real_index(n, m, 0)] = yr[m]
            if m:
                Y[real_index(n, m, 1)] = yi[m]
    # 3. z translation per order m (Re; Im with the opposite sign)
    Z2 = np.zeros_like(Y)
    for m in range(p + 1):
        Zm = np.array([[(-1) ** (n + m) * math.factorial(j + n) / rho ** (j + n + 1) * fA ** (j + 1) * fB ** n
                        for n in range(m, p + 1)] for j in range(m, p + 1)])
        xr = np.array([Y[real_index(n, m, 0)] for n in range(m, p + 1)])
        yr = Zm @ xr
        for jj, j in enumerate(range(m, p + 1)):
            Z2[real_index(j, m, 0)] = yr[jj]
        if m:
            xi = np.array([Y[real_index(n, m, 1)] for n in range(m, p + 1)])
            yi = -(Zm @ xi)
            for jj, j in enumerate(range(m, p + 1)):
                Z2[real_index(j, m, 1)] = yi[jj]
    # 4. back d-rotation: Re block E^-1 Dre^T E, Im block Dim^T
    W = np.zeros_like(Z2)
    for j in range(p + 1):
        Dre, Dim = D[j]
        E = np.diag([1.0] + [2.0] * j)
        Bre = np.linalg.inv(E) @ Dre.T @ E
        xr = np.array([Z2[real_index(j, k, 0)] for k in range(j + 1)])
        xi = np.array([Z2[real_index(j, k, 1)] if k else np.zeros(X.shape[1]) for k in range(j + 1)])
        yr, yi = Bre @ xr, Dim.T @ xi
        for k in range(j + 1):
            W[real_index(j, k, 0)] = yr[k]
            if k:
                W[real_index(j, k, 1)] = yi[k]
    # 5. back azimuthal rotation (helpers, in the accumulate)
    for j in range(p + 1):
        for k in range(1, j + 1):
            c, s = math.cos(k * alpha), math.sin(k * alpha)
            re, im = W[real_index(j, k, 0)].copy(), W[real_index(j, k, 1)].copy()
            W[real_index(j, k, 0)] = c * re - s * im
            W[real_index(j, k, 1)] = s * re + c * im
    return W


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    rng = np.random.default_rng(0)
    worst = 0.0
    for d0, dl in [((0, 1, 3), 0), ((2, 3, 1), 0), ((1, 4, 2), -1), ((0, 0, 5), 1), ((3, 3, 3), 0), ((0, 5, 0), 0),
                   ((1, 2, 0), -1)]:
        T = dense_op(d0, dl, p)
        X = rng.standard_normal(((p + 1) ** 2, 5))
        ref = T @ X
        got = factored_apply(X, d0, dl, p)
        err = np.abs(got - ref).max() / np.abs(ref).max()
        worst = max(worst, err)
        print(d0, dl, f"{err:.3e}")
    print("worst", worst)


if __name__ == "__main__":
    main()


def potential_check(p, d0, dl, nq=20, seed=1):
    """Physical check: charges in B, targets in A; compare potentials from dense and factored Y."""
    rng = np.random.default_rng(seed)
    fA = 2.0 ** (-dl) if dl < 0 else 1.0
    fB = 2.0 ** dl if dl > 0 else 1.0
    NR = (p + 1) ** 2
    cols = []
    for _ in range(3):
        s = rng.uniform(-fB, fB, (nq, 3))
        q = rng.uniform(-1, 1, nq)
        v = np.zeros(NR)
        for si, qi in zip(s, q):
            R = regular(si, p)
            for n in range(p + 1):
                for m in range(n + 1):
                    z = qi * np.conj(R[(n, m)]) / fB ** n
                    v[real_index(n, m, 0)] += z.real
                    if m:
                        v[real_index(n, m, 1)] += z.imag
        cols.append(v)
    X = np.array(cols).T
    Yd = dense_op(d0, dl, p) @ X
    Yf = factored_apply(X, d0, dl, p)
    worst = 0.0
    for x in rng.uniform(-fA, fA, (10, 3)):
        R = regular(x, p)
        for c in range(X.shape[1]):
            def phi(Y):
                tot = 0.0
                for n in range(p + 1):
                    for m in range(n + 1):
                        lre = Y[real_index(n, m, 0), c] / fA ** (n + 1)
                        lim = Y[real_index(n, m, 1), c] / fA ** (n + 1) if m else 0.0
                        w = 1.0 if m == 0 else 2.0
                        tot += w * (lre * R[(n, m)].real + lim * R[(n, m)].imag)
                return tot
            a, b = phi(Yf), phi(Yd)
            worst = max(worst, abs(a - b) / abs(b))
    return worst


if __name__ == "__main__" and len(sys.argv) > 2:
    p = int(sys.argv[1])
    for d0, dl in [((0, 1, 3), 0), ((0, 0, 5), 1), ((1, 4, 2), -1), ((3, 3, 3), 0)]:
        print("potential", d0, dl, f"{potential_check(p, d0, dl):.3e}")
