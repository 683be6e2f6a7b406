// harmonics.cuh — device solid harmonics (Condon–Shortley
// R_n^m = r^n P_n^m e^{i m phi} / (n+m)!, I_n^m = (n-m)! P_n^m e^{i m phi} / r^{n+1},
// m >= 0 storage, index n(n+1)/2 + m), by Cartesian recurrences.
#pragma once
#include "common.cuh"

namespace fmm {

// 1 / ((n + m)(n - m)) for the regular-harmonic column recurrence (n >= m + 2), in
// constant memory: the L2P loop indices are warp-uniform, so reads are broadcasts and
// the per-coefficient FP64 division disappears.
struct InvNM {
  double v[(kMaxP + 1) * (kMaxP + 1)];
};
constexpr InvNM make_inv_nm() {
  InvNM t{};
  for (int n = 0; n <= kMaxP; ++n)
    for (int m = 0; m <= kMaxP; ++m) t.v[n * (kMaxP + 1) + m] = (n > m) ? 1.0 / ((double)(n + m) * (double)(n - m)) : 0.0;
  return t;
}
static __constant__ InvNM c_inv_nm = make_inv_nm();
// -1 / (2m): the diagonal step R_m^m = -(x+iy)/(2m) R_{m-1}^{m-1}
struct HalfInv {
  double v[kMaxP + 1];
};
constexpr HalfInv make_half_inv() {
  HalfInv t{};
  for (int m = 1; m <= kMaxP; ++m) t.v[m] = -0.5 / m;
  return t;
}
static __constant__ HalfInv c_half_inv = make_half_inv();

// Column m (n = m..p) of the regular harmonics R_n^m(x,y,z) into R (m >= 0 storage);
// columns are independent, so a block computes all of them in parallel.
__device__ inline void regular_column(double x, double y, double z, int m, int p, double2* R) {
  const double r2 = x * x + y * y + z * z;
  double2 d = make_double2(1.0, 0.0);
  for (int k = 1; k <= m; ++k) {
    const double s = c_half_inv.v[k];
    d = cmul(d, make_double2(s * x, s * y));
  }
  R[cidx(m, m)] = d;
  if (m + 1 > p) return;
  double2 a = d, b = cscale(d, z);
  R[cidx(m + 1, m)] = b;
  for (int n = m + 2; n <= p; ++n) {
    const double inv = c_inv_nm.v[n * (kMaxP + 1) + m];
    const double2 c = make_double2(((2 * n - 1) * z * b.x - r2 * a.x) * inv, ((2 * n - 1) * z * b.y - r2 * a.y) * inv);
    R[cidx(n, m)] = c;
    a = b;
    b = c;
  }
}

// Regular harmonics R_n^m(x,y,z), n <= p, written by ONE thread into R.
__device__ inline void regular_harmonics(double x, double y, double z, int p, double2* R) {
  const double r2 = x * x + y * y + z * z;
  double2 diag = make_double2(1.0, 0.0);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) {
      const double s = -0.5 / m;  // R_m^m = -(x+iy)/(2m) R_{m-1}^{m-1}
      diag = cmul(diag, make_double2(s * x, s * y));
    }
    R[cidx(m, m)] = diag;
    if (m + 1 > p) continue;
    double2 a = diag, b = cscale(diag, z);  // R_m^m, R_{m+1}^m
    R[cidx(m + 1, m)] = b;
    for (int n = m + 2; n <= p; ++n) {
      const double inv = 1.0 / ((double)(n + m) * (double)(n - m));
      double2 c = make_double2(((2 * n - 1) * z * b.x - r2 * a.x) * inv, ((2 * n - 1) * z * b.y - r2 * a.y) * inv);
      R[cidx(n, m)] = c;
      a = b;
      b = c;
    }
  }
}

// Irregular harmonics I_n^m(x,y,z), n <= P, columns m distributed over `nthr` threads.
__device__ inline void irregular_harmonics_par(double x, double y, double z, int P, double2* I, int tid, int nthr) {
  const double r2 = x * x + y * y + z * z;
  const double inv_r2 = 1.0 / r2;
  const double inv_r = 1.0 / sqrt(r2);
  for (int m = tid; m <= P; m += nthr) {
    double2 d = make_double2(inv_r, 0.0);
    for (int k = 1; k <= m; ++k) {  // I_k^k = -(2k-1)(x+iy)/r^2 I_{k-1}^{k-1}
      const double s = -(2.0 * k - 1.0) * inv_r2;
      d = cmul(d, make_double2(s * x, s * y));
    }
    I[cidx(m, m)] = d;
    if (m + 1 > P) continue;
    double2 a = d, b = cscale(d, (2.0 * m + 1.0) * z * inv_r2);
    I[cidx(m + 1, m)] = b;
    for (int n = m + 2; n <= P; ++n) {
      const double c1 = (2.0 * n - 1.0) * z, c2 = (double)(n - 1) * (n - 1) - (double)m * m;
      double2 c = make_double2((c1 * b.x - c2 * a.x) * inv_r2, (c1 * b.y - c2 * a.y) * inv_r2);
      I[cidx(n, m)] = c;
      a = b;
      b = c;
    }
  }
}

// (j, k) of coefficient index t = j(j+1)/2 + k
__device__ __forceinline__ void decode_jk(int t, int& j, int& k) {
  j = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (cidx(j + 1, 0) <= t) ++j;
  while (cidx(j, 0) > t) --j;
  k = t - cidx(j, 0);
}

// L2P (+grad) for one target with the regular harmonics generated on the fly
// (two-term column recurrence, O(1) registers), using the m >= 0 symmetry:
//   phi   = sum_n sum_{m>=0} w_m Re(L_n^m conj R_n^m),  w_0 = 1, w_{m>0} = 2
//   L'_0  = sum_{n<p} sum_{m>=0} w_m Re(L_{n+1}^m conj R_n^m)
//   L'_1  = sum_{n<p} sum_{m>=0} [L_{n+1}^{m+1} conj R_n^m - [m>0] conj(L_{n+1}^{m-1}) R_n^m]
//   grad  = (-Re L'_1, -Im L'_1, L'_0)
// (the same quantities as the oracle's full-m sums, regrouped).
template <bool kGrad>
__device__ __forceinline__ void l2p_eval(const double2* __restrict__ Lc, int p, double x, double y, double z,
                                         double& phi, double3& g) {
  const double r2 = x * x + y * y + z * z;
  double2 diag = make_double2(1.0, 0.0);
  double f = 0.0, g0 = 0.0;
  double2 g1 = make_double2(0.0, 0.0);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) {
      const double s = c_half_inv.v[m];
      diag = cmul(diag, make_double2(s * x, s * y));
    }
    const double w = m == 0 ? 1.0 : 2.0;
    double2 a = make_double2(0, 0), b = diag;  // R_{n-1}^m, R_n^m
    for (int n = m; n <= p; ++n) {
      if (n == m + 1) {
        a = b;
        b = cscale(diag, z);
      } else if (n > m + 1) {
        const double inv = c_inv_nm.v[n * (kMaxP + 1) + m];
        double2 c = make_double2(((2 * n - 1) * z * b.x - r2 * a.x) * inv, ((2 * n - 1) * z * b.y - r2 * a.y) * inv);
        a = b;
        b = c;
      }
      const double2 l = Lc[cidx(n, m)];
      f += w * (l.x * b.x + l.y * b.y);
      if (kGrad && n < p) {
        const double2 l0 = Lc[cidx(n + 1, m)];
        g0 += w * (l0.x * b.x + l0.y * b.y);
        const double2 lp = Lc[cidx(n + 1, m + 1)];  // L_{n+1}^{m+1} conj R
        g1.x += lp.x * b.x + lp.y * b.y;
        g1.y += lp.y * b.x - lp.x * b.y;
        if (m > 0) {  // - conj(L_{n+1}^{m-1}) R
          const double2 lm = Lc[cidx(n + 1, m - 1)];
          g1.x -= lm.x * b.x + lm.y * b.y;
          g1.y -= lm.x * b.y - lm.y * b.x;
        }
      }
    }
  }
  phi += f;
  if (kGrad) {
    g.x -= g1.x;
    g.y -= g1.y;
    g.z += g0;
  }
}

}  // namespace fmm
