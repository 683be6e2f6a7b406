// harmonics.cuh — device solid harmonics (Condon–Shortley
// R_n^m = r^n P_n^m e^{i m phi} / (n+m)!, I_n^m = (n-m)! P_n^m e^{i m phi} / r^{n+1},
// m >= 0 storage, index n(n+1)/2 + m), by Cartesian recurrences.
#pragma once
#include "common.cuh"

namespace fmm {

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

}  // namespace fmm
