// helmholtz.cu — NEXT-4: the FMM mat-vec for the 3D Helmholtz kernel
// exp(i kappa r) / r (include/fmm_helmholtz.h).
//
// Same tree and interaction lists as the Laplace plan (the MAC and split rule of fmm_setup);
// spherical-wave expansions of order p (R50-R55), all orders m = -n..n, complex:
//   Y_n^m      orthonormal spherical harmonics, Condon-Shortley phase
//   R_n^m(v) = j_n(kappa |v|) Y_n^m(v^),   S_n^m(v) = h_n(kappa |v|) Y_n^m(v^),  h_n = j_n + i y_n
//   P2M   M_n^m = 4 pi i kappa sum_j q_j conj R_n^m(y_j - c)
//   M2M   M(c_p)  = (S|S)(c_p - c_c) M(c_c)       (S|S) = (R|R)
//   M2L   L(c_A) += (S|R)(c_A - c_B) M(c_B)
//   L2L   L(c_c) += (R|R)(c_c - c_p) L(c_p)
//   L2P   phi(x) += sum L_n^m R_n^m(x - c);   P2P  phi_i += q_j exp(i kappa r) / r, r > 0
//   (E|F)[(n',m'),(n,m)](t) = 4 pi sum_l i^(n'+l-n) E_l^(m-m')(t) Gaunt(Y_n^m, conj Y_n'^m', conj Y_l^(m-m'))
// The operators are not scale invariant (kappa times the cell size), so they are tabulated at
// setup on the host in long double: per child level and octant for M2M / L2L, per M2L class
// (target level, source level, integer offset). The mat-vec kernels apply them as dense complex
// matrix-vector products (the algebraic end of the paper's compute-memory axis);
// tables are stored transposed ([column][row]) so a thread per output coefficient reads coalesced.
// Coordinates: the plan's normalised frame times 2^e (physical), where kappa applies.
#include <algorithm>
#include <cmath>
#include <complex>
#include <array>
#include <map>
#include <tuple>
#include <mutex>
#include <vector>

#include "../../include/fmm_helmholtz.h"
#include "plan.h"

namespace fmm {
namespace {

using cld = std::complex<long double>;
constexpr int kMaxPH = 10;
constexpr long double kPiL = 3.14159265358979323846264338327950288L;

__host__ __device__ inline int hidx(int n, int m) { return n * n + n + m; }

// ------------------------------------------------------------------ host: special functions
long double lfact(int n) {
  static const std::vector<long double> f = [] {  // thread-safe one-time init
    std::vector<long double> t(200);
    t[0] = 1;
    for (int i = 1; i < 200; ++i) t[i] = t[i - 1] * i;
    return t;
  }();
  return f[n];
}

// Wigner 3j symbol (Racah's formula)
long double wigner3j(int j1, int j2, int j3, int m1, int m2, int m3) {
  if (m1 + m2 + m3 != 0 || std::abs(m1) > j1 || std::abs(m2) > j2 || std::abs(m3) > j3) return 0;
  if (j3 < std::abs(j1 - j2) || j3 > j1 + j2) return 0;
  const long double tri = lfact(j1 + j2 - j3) * lfact(j1 - j2 + j3) * lfact(-j1 + j2 + j3) / lfact(j1 + j2 + j3 + 1);
  const long double pre = std::sqrt(tri * lfact(j1 + m1) * lfact(j1 - m1) * lfact(j2 + m2) * lfact(j2 - m2) *
                                    lfact(j3 + m3) * lfact(j3 - m3));
  long double s = 0;
  const int k0 = std::max({0, j2 - j3 - m1, j1 - j3 + m2}), k1 = std::min({j1 + j2 - j3, j1 - m1, j2 + m2});
  for (int k = k0; k <= k1; ++k) {
    const long double d = lfact(k) * lfact(j1 + j2 - j3 - k) * lfact(j1 - m1 - k) * lfact(j2 + m2 - k) *
                          lfact(j3 - j2 + m1 + k) * lfact(j3 - j1 - m2 + k);
    s += ((k & 1) ? -1.0L : 1.0L) / d;
  }
  return (((j1 - j2 - m3) & 1) ? -1.0L : 1.0L) * pre * s;
}

long double gaunt(int l1, int m1, int l2, int m2, int l3, int m3) {  // integral Y Y Y
  const long double w0 = wigner3j(l1, l2, l3, 0, 0, 0);
  if (w0 == 0) return 0;
  return std::sqrt((2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1) / (4 * kPiL)) * w0 * wigner3j(l1, l2, l3, m1, m2, m3);
}

// spherical Bessel j_0..j_L (Miller's downward recurrence, normalised by j_0 or j_1) and, for
// 'h', y_0..y_L by the (stable) upward recurrence
void sph_bessel(int L, long double x, std::vector<long double>& j, std::vector<long double>* y) {
  j.assign(L + 1, 0);
  if (x == 0) {
    j[0] = 1;
  } else {
    const int N = L + 30 + (int)x;
    std::vector<long double> t(N + 2, 0);
    t[N + 1] = 0;
    t[N] = 1e-300L;
    for (int n = N; n >= 1; --n) {
      t[n - 1] = (2 * n + 1) / x * t[n] - t[n + 1];
      if (std::fabs(t[n - 1]) > 1e200L)  // rescale
        for (int k = n - 1; k <= N; ++k) t[k] *= 1e-200L;
    }
    const long double j0 = std::sin(x) / x, j1 = std::sin(x) / (x * x) - std::cos(x) / x;
    const long double s = std::fabs(j0) > std::fabs(j1) ? j0 / t[0] : j1 / t[1];
    for (int n = 0; n <= L; ++n) j[n] = t[n] * s;
  }
  if (y) {
    y->assign(L + 1, 0);
    (*y)[0] = -std::cos(x) / x;
    if (L >= 1) (*y)[1] = -std::cos(x) / (x * x) - std::sin(x) / x;
    for (int n = 1; n < L; ++n) (*y)[n + 1] = (2 * n + 1) / x * (*y)[n] - (*y)[n - 1];
  }
}

// orthonormal Y_l^mu(t^) for l <= L, all mu (Condon-Shortley), index hidx
std::vector<cld> sph_harm(int L, const long double t[3]) {
  const long double r = std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  const long double ct = r > 0 ? t[2] / r : 1, st = std::sqrt(std::max(0.0L, 1 - ct * ct));
  const long double rho = std::sqrt(t[0] * t[0] + t[1] * t[1]);
  const cld e1 = rho > 0 ? cld(t[0] / rho, t[1] / rho) : cld(1, 0);
  std::vector<cld> Y((L + 1) * (L + 1));
  long double pmm = 1 / std::sqrt(4 * kPiL);  // normalised P_m^m
  cld em(1, 0);
  for (int m = 0; m <= L; ++m) {
    if (m > 0) {
      pmm *= -std::sqrt((2 * m + 1) / (2.0L * m)) * st;
      em *= e1;
    }
    long double a = pmm, b = 0;
    for (int n = m; n <= L; ++n) {
      long double v;
      if (n == m) {
        v = pmm;
      } else if (n == m + 1) {
        v = std::sqrt(2.0L * m + 3) * ct * pmm;
        b = a;
        a = v;
      } else {
        const long double an = std::sqrt((4.0L * n * n - 1) / ((long double)n * n - (long double)m * m));
        const long double bn =
            std::sqrt(((long double)(n - 1) * (n - 1) - (long double)m * m) / (4.0L * (n - 1) * (n - 1) - 1));
        v = an * (ct * a - bn * b);
        b = a;
        a = v;
      }
      Y[hidx(n, m)] = v * em;
      if (m > 0) Y[hidx(n, -m)] = ((m & 1) ? -1.0L : 1.0L) * std::conj(v * em);
    }
  }
  return Y;
}

// coupling C[(n',m'), (n,m), l] = 4 pi i^(n'+l-n) integral Y_n^m conj Y_n'^m' conj Y_l^(m-m')
struct Coupling {
  int p = -1, nc = 0;
  std::vector<cld> c;  // [nc][nc][2p+1]
};
const Coupling& coupling(int p) {
  static Coupling C[kMaxPH + 1];
  static std::mutex table_mu;  // plans may be set up from several host threads
  std::lock_guard<std::mutex> lock(table_mu);
  Coupling& K = C[p];
  if (K.p == p) return K;
  K.nc = (p + 1) * (p + 1);
  K.c.assign((size_t)K.nc * K.nc * (2 * p + 1), cld(0));
  const cld ipow[4] = {cld(1, 0), cld(0, 1), cld(-1, 0), cld(0, -1)};
  for (int n1 = 0; n1 <= p; ++n1)
    for (int m1 = -n1; m1 <= n1; ++m1)
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          const int mu = m - m1;
          for (int l = std::abs(n - n1); l <= n + n1; ++l) {
            if (std::abs(mu) > l) continue;
            const long double g = (((m1 + mu) & 1) ? -1.0L : 1.0L) * gaunt(n, m, n1, -m1, l, -mu);
            if (g == 0) continue;
            K.c[((size_t)hidx(n1, m1) * K.nc + hidx(n, m)) * (2 * p + 1) + l] =
                4 * kPiL * ipow[((n1 + l - n) % 4 + 4) % 4] * g;
          }
        }
  K.p = p;  // complete
  return K;
}

// translation operator ('R': (R|R) = (S|S), 'S': (S|R)) for the physical vector t, written
// transposed as double2: out[(n,m) * nc + (n',m')]
void translation(char kind, const long double t[3], int p, long double kappa, double2* out) {
  const Coupling& K = coupling(p);
  const int L = 2 * p, nc = K.nc;
  const long double r = std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  std::vector<long double> j, y;
  sph_bessel(L, kappa * r, j, kind == 'S' ? &y : nullptr);
  const std::vector<cld> Yl = sph_harm(L, t);
  for (int n1 = 0; n1 <= p; ++n1)
    for (int m1 = -n1; m1 <= n1; ++m1)
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          const int mu = m - m1;
          cld s(0);
          const cld* c = &K.c[((size_t)hidx(n1, m1) * nc + hidx(n, m)) * (L + 1)];
          for (int l = std::abs(n - n1); l <= n + n1; ++l) {
            if (std::abs(mu) > l || c[l] == cld(0)) continue;
            const cld rad = kind == 'S' ? cld(j[l], y[l]) : cld(j[l], 0);
            s += c[l] * rad * Yl[hidx(l, mu)];
          }
          out[(size_t)hidx(n, m) * nc + hidx(n1, m1)] = make_double2((double)s.real(), (double)s.imag());
        }
}

// ------------------------------------------------------------------ device
__device__ __forceinline__ double2 cmadd(double2 acc, double2 a, double2 b) {  // acc + a b
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}

// spherical Bessel j_0..j_P(x) (Miller), x >= 0
template <int P>
__device__ void dev_sph_jn(double x, double (&j)[P + 1]) {
  if (x < 1e-300) {
    j[0] = 1.0;
#pragma unroll
    for (int n = 1; n <= P; ++n) j[n] = 0.0;
    return;
  }
  const int N = P + 24 + (int)x;
  double t1 = 0.0, t0 = 1e-200;  // t_{n+1}, t_n
  const double ix = 1.0 / x;
  for (int n = N; n > P; --n) {  // down to t_P
    const double tm = (2 * n + 1) * ix * t0 - t1;
    t1 = t0;
    t0 = tm;
    if (fabs(t0) > 1e150) {
      t0 *= 1e-150;
      t1 *= 1e-150;
    }
  }
  // t0 = t_P, t1 = t_{P+1}
  double tv[P + 1];
  tv[P] = t0;
#pragma unroll
  for (int n = P; n >= 1; --n) {
    const double tm = (2 * n + 1) * ix * tv[n] - (n == P ? t1 : tv[n + 1]);
    tv[n - 1] = tm;
  }
  double s, c;
  sincos(x, &s, &c);
  const double j0 = s * ix, j1 = s * ix * ix - c * ix;
  const double scale = (fabs(j0) > fabs(j1) || P == 0) ? j0 / tv[0] : j1 / tv[1 <= P ? 1 : 0];
#pragma unroll
  for (int n = 0; n <= P; ++n) j[n] = tv[n] * scale;
}

// R_n^m(v) for all (n, m), n <= P (j_n times orthonormal Y_n^m), handed to f(hidx(n, m), value)
template <int P, typename F>
__device__ __forceinline__ void dev_regular(double vx, double vy, double vz, double kappa, F&& f) {
  const double r2 = vx * vx + vy * vy + vz * vz, r = sqrt(r2);
  double jn[P + 1];
  dev_sph_jn<P>(kappa * r, jn);
  const double ct = r > 0 ? vz / r : 1.0, st = sqrt(fmax(0.0, 1.0 - ct * ct));
  const double rho = sqrt(vx * vx + vy * vy);
  const double2 e1 = rho > 0 ? make_double2(vx / rho, vy / rho) : make_double2(1.0, 0.0);
  double pmm = 0.28209479177387814;  // 1 / sqrt(4 pi)
  double2 em = make_double2(1.0, 0.0);
#pragma unroll
  for (int m = 0; m <= P; ++m) {
    if (m > 0) {
      pmm *= -sqrt((2 * m + 1) / (2.0 * m)) * st;
      em = make_double2(em.x * e1.x - em.y * e1.y, em.x * e1.y + em.y * e1.x);
    }
    double a = pmm, b = 0.0;
#pragma unroll
    for (int n = m; n <= P; ++n) {
      double v;
      if (n == m) {
        v = pmm;
      } else if (n == m + 1) {
        v = sqrt(2.0 * m + 3) * ct * pmm;
        b = a;
        a = v;
      } else {
        const double an = sqrt((4.0 * n * n - 1) / ((double)n * n - (double)m * m));
        const double bn = sqrt(((double)(n - 1) * (n - 1) - (double)m * m) / (4.0 * (n - 1) * (n - 1) - 1));
        v = an * (ct * a - bn * b);
        b = a;
        a = v;
      }
      const double w = v * jn[n];
      f(hidx(n, m), make_double2(w * em.x, w * em.y));
      if (m > 0) {
        const double sg = (m & 1) ? -1.0 : 1.0;  // Y_n^-m = (-1)^m conj Y_n^m
        f(hidx(n, -m), make_double2(sg * w * em.x, -sg * w * em.y));
      }
    }
  }
}

// charges in Morton order
__global__ void gather_qh_kernel(const double2* __restrict__ q, const uint32_t* __restrict__ perm, int64_t n,
                                 double2* __restrict__ qs, int32_t* __restrict__ flags) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (s < n) {
    const double2 v = q[perm[s]];
    bad = !isfinite(v.x) || !isfinite(v.y);
    qs[s] = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
}

// P2M: block per leaf; the block builds R(y_j - c) for one particle at a time in shared memory
template <int P>
__global__ void p2m_h_kernel(const int32_t* __restrict__ leaves, const int32_t* __restrict__ cbeg,
                             const int32_t* __restrict__ cend, const double4* __restrict__ center,
                             const double4* __restrict__ pos, const double2* __restrict__ qs, double phys,
                             double kappa, double2* __restrict__ M) {
  constexpr int NC = (P + 1) * (P + 1);
  __shared__ double2 Rs[NC];
  const int leaf = leaves[blockIdx.x];
  const double4 c = center[leaf];
  double2 acc[(NC + 63) / 64];
#pragma unroll
  for (int k = 0; k < (NC + 63) / 64; ++k) acc[k] = make_double2(0, 0);
  for (int j = cbeg[leaf]; j < cend[leaf]; ++j) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const double4 x = pos[j];
      dev_regular<P>((x.x - c.x) * phys, (x.y - c.y) * phys, (x.z - c.z) * phys, kappa,
                     [&](int i, double2 v) { Rs[i] = v; });
    }
    __syncthreads();
    const double2 q = qs[j];
#pragma unroll
    for (int k = 0; k < (NC + 63) / 64; ++k) {
      const int i = threadIdx.x + 64 * k;
      if (i < NC) {
        const double2 r = Rs[i];  // q conj(R)
        acc[k] = make_double2(acc[k].x + q.x * r.x + q.y * r.y, acc[k].y + q.y * r.x - q.x * r.y);
      }
    }
  }
  const double f = 4.0 * 3.14159265358979323846 * kappa;  // times i
#pragma unroll
  for (int k = 0; k < (NC + 63) / 64; ++k) {
    const int i = threadIdx.x + 64 * k;
    if (i < NC) M[(int64_t)leaf * NC + i] = make_double2(-f * acc[k].y, f * acc[k].x);
  }
}

// child octant from the anchors: child anchor = 2 parent anchor + (x, y, z) bits
__device__ __forceinline__ int octant(const int32_t* anchor, int c) {
  return ((anchor[3 * c] & 1) << 2) | ((anchor[3 * c + 1] & 1) << 1) | (anchor[3 * c + 2] & 1);
}

// M2M for the parents [lb, lb + n): M_p = sum_children T[level_c][oct] M_c
template <int P>
__global__ void m2m_h_kernel(int64_t lb, const int32_t* __restrict__ child, const int32_t* __restrict__ nchild,
                             const int32_t* __restrict__ level, const int32_t* __restrict__ anchor,
                             const double2* __restrict__ ops, double2* __restrict__ M) {
  constexpr int NC = (P + 1) * (P + 1);
  __shared__ double2 src[NC];
  const int cell = (int)(lb + blockIdx.x);
  const int nch = nchild[cell];
  if (nch == 0) return;  // leaf (P2M)
  double2 acc[(NC + 63) / 64];
#pragma unroll
  for (int k = 0; k < (NC + 63) / 64; ++k) acc[k] = make_double2(0, 0);
  for (int q = 0; q < nch; ++q) {
    const int c = child[cell] + q;
    __syncthreads();
    for (int i = threadIdx.x; i < NC; i += blockDim.x) src[i] = M[(int64_t)c * NC + i];
    __syncthreads();
    const double2* T = ops + ((size_t)(level[c] * 8 + octant(anchor, c)) * 2 + 0) * NC * NC;
    for (int jj = 0; jj < NC; ++jj) {
      const double2 s = src[jj];
#pragma unroll
      for (int k = 0; k < (NC + 63) / 64; ++k) {
        const int i = threadIdx.x + 64 * k;
        if (i < NC) acc[k] = cmadd(acc[k], T[(size_t)jj * NC + i], s);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < (NC + 63) / 64; ++k) {
    const int i = threadIdx.x + 64 * k;
    if (i < NC) M[(int64_t)cell * NC + i] = acc[k];
  }
}

// M2L: block per target cell; L_A = sum over its list of T[class] M_B (written, not added)
template <int P>
__global__ void m2l_h_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ srcs,
                             const int32_t* __restrict__ cls, const double2* __restrict__ ops,
                             const double2* __restrict__ M, double2* __restrict__ L) {
  constexpr int NC = (P + 1) * (P + 1);
  __shared__ double2 src[NC];
  const int t = blockIdx.x;
  double2 acc[(NC + 63) / 64];
#pragma unroll
  for (int k = 0; k < (NC + 63) / 64; ++k) acc[k] = make_double2(0, 0);
  for (int q = off[t]; q < off[t + 1]; ++q) {
    const int b = srcs[q];
    __syncthreads();
    for (int i = threadIdx.x; i < NC; i += blockDim.x) src[i] = M[(int64_t)b * NC + i];
    __syncthreads();
    const double2* T = ops + (size_t)cls[q] * NC * NC;
    for (int jj = 0; jj < NC; ++jj) {
      const double2 s = src[jj];
#pragma unroll
      for (int k = 0; k < (NC + 63) / 64; ++k) {
        const int i = threadIdx.x + 64 * k;
        if (i < NC) acc[k] = cmadd(acc[k], T[(size_t)jj * NC + i], s);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < (NC + 63) / 64; ++k) {
    const int i = threadIdx.x + 64 * k;
    if (i < NC) L[(int64_t)t * NC + i] = acc[k];
  }
}

// L2L for the children of the parents [lb, lb + n): L_c += T[level_c][oct] L_p
template <int P>
__global__ void l2l_h_kernel(int64_t lb, const int32_t* __restrict__ child, const int32_t* __restrict__ nchild,
                             const int32_t* __restrict__ level, const int32_t* __restrict__ anchor,
                             const double2* __restrict__ ops, double2* __restrict__ L) {
  constexpr int NC = (P + 1) * (P + 1);
  __shared__ double2 src[NC];
  const int cell = (int)(lb + blockIdx.x);
  const int nch = nchild[cell];
  if (nch == 0) return;
  for (int i = threadIdx.x; i < NC; i += blockDim.x) src[i] = L[(int64_t)cell * NC + i];
  __syncthreads();
  for (int q = 0; q < nch; ++q) {
    const int c = child[cell] + q;
    const double2* T = ops + ((size_t)(level[c] * 8 + octant(anchor, c)) * 2 + 1) * NC * NC;
#pragma unroll
    for (int k = 0; k < (NC + 63) / 64; ++k) {
      const int i = threadIdx.x + 64 * k;
      if (i >= NC) continue;
      double2 acc = L[(int64_t)c * NC + i];
      for (int jj = 0; jj < NC; ++jj) acc = cmadd(acc, T[(size_t)jj * NC + i], src[jj]);
      L[(int64_t)c * NC + i] = acc;
    }
  }
}

// L2P + P2P: warp per leaf, lane per target (looping over the leaf's targets); caller order out
template <int P>
__global__ void near_h_kernel(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ cbeg,
                              const int32_t* __restrict__ cend, const double4* __restrict__ center,
                              const double4* __restrict__ pos, const double2* __restrict__ qs,
                              const int32_t* __restrict__ off, const int32_t* __restrict__ srcl,
                              const double2* __restrict__ L, const uint32_t* __restrict__ perm, double phys,
                              double kappa, double2* __restrict__ phi) {
  constexpr int NC = (P + 1) * (P + 1);
  const int64_t li = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (li >= nleaves) return;
  const int lane = threadIdx.x & 31;
  const int leaf = leaves[li];
  const double4 c = center[leaf];
  const double2* Lc = L + (int64_t)leaf * NC;
  for (int t = cbeg[leaf] + lane; t < cend[leaf]; t += 32) {
    const double4 x = pos[t];
    double2 f = make_double2(0, 0);
    dev_regular<P>((x.x - c.x) * phys, (x.y - c.y) * phys, (x.z - c.z) * phys, kappa,
                   [&](int i, double2 v) { f = cmadd(f, Lc[i], v); });
    for (int k = off[leaf]; k < off[leaf + 1]; ++k) {
      const int s = srcl[k];
      for (int j = cbeg[s]; j < cend[s]; ++j) {
        const double4 y = pos[j];
        const double dx = (x.x - y.x) * phys, dy = (x.y - y.y) * phys, dz = (x.z - y.z) * phys;
        const double r2 = dx * dx + dy * dy + dz * dz;
        if (r2 > 0.0) {
          const double ir = rsqrt(r2), r = r2 * ir;
          double sn, cs;
          sincos(kappa * r, &sn, &cs);
          const double2 q = qs[j];
          const double2 g = make_double2(cs * ir, sn * ir);
          f = cmadd(f, g, q);
        }
      }
    }
    phi[perm[t]] = f;
  }
}

__global__ void direct_h_kernel(const double* __restrict__ src, const double2* __restrict__ q, int64_t ns,
                                const double* __restrict__ tgt, int64_t nt, double kappa, double2* __restrict__ phi) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const double tx = tgt[3 * t], ty = tgt[3 * t + 1], tz = tgt[3 * t + 2];
  double2 f = make_double2(0, 0);
  for (int64_t s = 0; s < ns; ++s) {
    const double dx = tx - src[3 * s], dy = ty - src[3 * s + 1], dz = tz - src[3 * s + 2];
    const double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 > 0.0) {
      const double r = sqrt(r2);
      double sn, cs;
      sincos(kappa * r, &sn, &cs);
      f = cmadd(f, make_double2(cs / r, sn / r), q[s]);
    }
  }
  phi[t] = f;
}

template <int P>
void launch_all(fmm_plan_s& Pl, const double* q, double* phi) {
  constexpr int NC = (P + 1) * (P + 1);
  auto& H = Pl.helm;
  cudaStream_t s = Pl.stream;
  const double phys = std::ldexp(1.0, Pl.e), kappa = Pl.kappa;
  gather_qh_kernel<<<cdiv(Pl.n, 256), 256, 0, s>>>((const double2*)q, Pl.perm, Pl.n, H.qs, Pl.flags);
  FMM_LAUNCHED("gather_qh_kernel");
  // leaves (all of them; leaf index sorted by position)
  p2m_h_kernel<P><<<(unsigned)Pl.nleaves, 64, 0, s>>>(Pl.leaves, Pl.cells.begin, Pl.cells.end, Pl.cells.center,
                                                      Pl.pos, H.qs, phys, kappa, H.M);
  FMM_LAUNCHED("p2m_h_kernel");
  for (int l = Pl.max_level - 1; l >= 0; --l) {
    const int64_t lb = Pl.level_begin[l], n = Pl.level_begin[l + 1] - lb;
    if (n <= 0) continue;
    m2m_h_kernel<P><<<(unsigned)n, 64, 0, s>>>(lb, Pl.cells.child, Pl.cells.nchild, Pl.cells.level, Pl.cells.anchor,
                                                H.shift_ops, H.M);
    FMM_LAUNCHED("m2m_h_kernel");
  }
  m2l_h_kernel<P><<<(unsigned)Pl.cells.n, 64, 0, s>>>(Pl.m2l.off, Pl.m2l.src, H.m2l_class, H.m2l_ops, H.M, H.L);
  FMM_LAUNCHED("m2l_h_kernel");
  for (int l = 0; l < Pl.max_level; ++l) {
    const int64_t lb = Pl.level_begin[l], n = Pl.level_begin[l + 1] - lb;
    if (n <= 0) continue;
    l2l_h_kernel<P><<<(unsigned)n, 64, 0, s>>>(lb, Pl.cells.child, Pl.cells.nchild, Pl.cells.level, Pl.cells.anchor,
                                                H.shift_ops, H.L);
    FMM_LAUNCHED("l2l_h_kernel");
  }
  near_h_kernel<P><<<cdiv(Pl.nleaves, 2), 64, 0, s>>>(Pl.leaves, Pl.nleaves, Pl.cells.begin, Pl.cells.end,
                                                      Pl.cells.center, Pl.pos, H.qs, Pl.p2p.off, Pl.p2p.src, H.L,
                                                      Pl.perm, phys, kappa, (double2*)phi);
  FMM_LAUNCHED("near_h_kernel");
  (void)NC;
}

}  // namespace

// tables for the plan's tree (host, long double), then device copies
void helmholtz_setup(fmm_plan_s& P) {
  if (P.p > kMaxPH) throw Error(FMM_ERR_USAGE, "fmm_setup_helmholtz: p must be in [0, 10]");
  auto& H = P.helm;
  const int p = P.p, NC = (p + 1) * (p + 1);
  const long double kappa = P.kappa, phys = std::ldexp(1.0L, P.e);
  const int64_t nc = P.cells.n;
  std::vector<int32_t> level(nc), anchor(3 * nc), mt(P.m2l.n), ms(P.m2l.n);
  FMM_CUDA(cudaMemcpyAsync(level.data(), P.cells.level.ptr, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaMemcpyAsync(anchor.data(), P.cells.anchor.ptr, sizeof(int32_t) * 3 * nc, cudaMemcpyDeviceToHost,
                           P.stream));
  if (P.m2l.n) {
    FMM_CUDA(cudaMemcpyAsync(mt.data(), P.m2l.tgt.ptr, sizeof(int32_t) * P.m2l.n, cudaMemcpyDeviceToHost, P.stream));
    FMM_CUDA(cudaMemcpyAsync(ms.data(), P.m2l.src.ptr, sizeof(int32_t) * P.m2l.n, cudaMemcpyDeviceToHost, P.stream));
  }
  FMM_CUDA(cudaStreamSynchronize(P.stream));
  // M2M / L2L: per child level and octant; child centre = parent centre + h_c (2 b - 1)
  const int nlev = P.max_level + 1;
  std::vector<double2> shift((size_t)nlev * 8 * 2 * NC * NC);
  for (int l = 1; l < nlev; ++l) {
    const long double hc = (long double)P.S / std::ldexp(1.0L, l + 1) * phys;
    for (int o = 0; o < 8; ++o) {
      const long double d[3] = {hc * (((o >> 2) & 1) ? 1 : -1), hc * (((o >> 1) & 1) ? 1 : -1),
                                hc * ((o & 1) ? 1 : -1)};
      const long double tm[3] = {-d[0], -d[1], -d[2]};  // M2M: c_p - c_c
      translation('R', tm, p, kappa, &shift[((size_t)(l * 8 + o) * 2 + 0) * NC * NC]);
      translation('R', d, p, kappa, &shift[((size_t)(l * 8 + o) * 2 + 1) * NC * NC]);  // L2L: c_c - c_p
    }
  }
  H.shift_ops.alloc((int64_t)shift.size());
  FMM_CUDA(cudaMemcpyAsync(H.shift_ops.ptr, shift.data(), sizeof(double2) * shift.size(), cudaMemcpyHostToDevice,
                           P.stream));
  // M2L classes: (target level, source level, integer offset of the centres); t = c_A - c_B
  std::map<std::tuple<int, int, int64_t, int64_t, int64_t>, int> cls;
  std::vector<int32_t> pc(P.m2l.n);
  std::vector<std::array<long double, 3>> tv;
  auto ictr = [&](int c, int a) {  // (2 anchor + 1) 2^(21 - level)
    return (2 * (int64_t)anchor[3 * c + a] + 1) << (21 - level[c]);
  };
  for (int64_t k = 0; k < P.m2l.n; ++k) {
    const int a = mt[k], b = ms[k];
    const int64_t dx = ictr(a, 0) - ictr(b, 0), dy = ictr(a, 1) - ictr(b, 1), dz = ictr(a, 2) - ictr(b, 2);
    const auto key = std::make_tuple(level[a], level[b], dx, dy, dz);
    auto it = cls.find(key);
    if (it == cls.end()) {
      it = cls.emplace(key, (int)tv.size()).first;
      const long double u = (long double)P.S / std::ldexp(1.0L, 22) * phys;  // integer centre unit
      tv.push_back({dx * u, dy * u, dz * u});
    }
    pc[k] = it->second;
  }
  H.nclass = (int64_t)tv.size();
  std::vector<double2> ops((size_t)std::max<int64_t>(1, H.nclass) * NC * NC);
  for (int64_t c = 0; c < H.nclass; ++c) translation('S', tv[c].data(), p, kappa, &ops[(size_t)c * NC * NC]);
  H.m2l_ops.alloc((int64_t)ops.size());
  FMM_CUDA(cudaMemcpyAsync(H.m2l_ops.ptr, ops.data(), sizeof(double2) * ops.size(), cudaMemcpyHostToDevice, P.stream));
  H.m2l_class.alloc(std::max<int64_t>(1, P.m2l.n));
  if (P.m2l.n)
    FMM_CUDA(cudaMemcpyAsync(H.m2l_class.ptr, pc.data(), sizeof(int32_t) * P.m2l.n, cudaMemcpyHostToDevice, P.stream));
  H.M.alloc(nc * NC);
  H.L.alloc(nc * NC);
  H.qs.alloc(P.n);
  FMM_CUDA(cudaStreamSynchronize(P.stream));
}

void helmholtz_matvec(fmm_plan_s& P, const double* q, double* phi) {
  switch (P.p) {
    case 0: launch_all<0>(P, q, phi); break;
    case 1: launch_all<1>(P, q, phi); break;
    case 2: launch_all<2>(P, q, phi); break;
    case 3: launch_all<3>(P, q, phi); break;
    case 4: launch_all<4>(P, q, phi); break;
    case 5: launch_all<5>(P, q, phi); break;
    case 6: launch_all<6>(P, q, phi); break;
    case 7: launch_all<7>(P, q, phi); break;
    case 8: launch_all<8>(P, q, phi); break;
    case 9: launch_all<9>(P, q, phi); break;
    case 10: launch_all<10>(P, q, phi); break;
    default: throw Error(FMM_ERR_USAGE, "helmholtz: p out of range");
  }
}

void helmholtz_direct(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt, double kappa,
                      double* phi, cudaStream_t s) {
  if (nt <= 0) return;
  direct_h_kernel<<<cdiv(nt, 128), 128, 0, s>>>(src, (const double2*)q, ns, tgt, nt, kappa, (double2*)phi);
  FMM_LAUNCHED("direct_h_kernel");
}

}  // namespace fmm
