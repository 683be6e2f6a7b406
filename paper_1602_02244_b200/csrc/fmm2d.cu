// fmm2d.cu — NEXT-3: the FMM mat-vec for the 2D Laplace (log) kernel, the
// 2D half of the paper's §4.1 experiment ("2D and 3D Laplace equation on uniform lattices",
// PAPER.md:386), on the same tree and interaction lists as the 3D path (planar points (x, y, 0):
// the octree is a quadtree; R40-R44):
//
//   phi_i = - sum_{j : r_ij > 0} q_j log r_ij,   grad_i = grad_{x_i} phi_i   (grad z = 0)
//
// Complex notation z = x + i y, Phi(z) = sum_j q_j log(z - z_j), phi = -Re Phi; classical 2D
// multipole calculus (oracle/fmm2d_oracle.py states every formula):
//   P2M  a_0 = sum q, a_k = -sum q (z_j - c)^k / k                 (warp per leaf)
//   M2M  b_l = -a_0 z0^l / l + sum_{k=1..l} a_k z0^(l-k) C(l-1,k-1)  (thread per (parent, l))
//   M2L  c_0 = a_0 log(-z0) + sum_k a_k (-1)^k z0^-k,
//        c_l = -a_0 / (l z0^l) + z0^-l sum_k a_k z0^-k C(l+k-1,k-1) (-1)^k  (warp per target, lane l)
//   L2L  d_l = sum_{k>=l} c_k C(k,l) w^(k-l)                          (thread per (child, l))
//   L2P + P2P  warp per target leaf, lane per target
// Expansions live in the plan's normalised frame u = x 2^-e (exact); the logarithm then needs
// phi = phi_u - e ln 2 (Q - Q0_i), Q = sum q (the root's a_0), Q0_i = the charge at r = 0 from
// x_i (itself and coincident points, which the sum skips); gradients scale by 2^-e.
// Every coefficient is produced by one thread in a fixed order: deterministic, no atomics.
#include <cmath>

#include "plan.h"

#ifndef FMM_2D_NEAR_THREADS
#define FMM_2D_NEAR_THREADS 256  // 32: 2.28 ms, 128: 1.88 ms, 256: 1.80 ms (1M lattice, p = 8)
#endif
#ifndef FMM_2D_M2L_THREADS
#define FMM_2D_M2L_THREADS 256
#endif

namespace fmm {
namespace {

constexpr int kMaxP2 = kMaxP;  // 2D expansions carry a_0 .. a_p (p <= 16)

struct Binom {
  double v[2 * kMaxP2 + 2][2 * kMaxP2 + 2];
};
constexpr Binom make_binom() {
  Binom b{};
  for (int n = 0; n < 2 * kMaxP2 + 2; ++n) {
    b.v[n][0] = 1.0;
    for (int k = 1; k <= n; ++k) b.v[n][k] = b.v[n - 1][k - 1] + (k <= n - 1 ? b.v[n - 1][k] : 0.0);
  }
  return b;
}
__constant__ Binom c_binom = make_binom();

__device__ __forceinline__ double2 cm(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cadd2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csc(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cinv(double2 a) {
  const double d = a.x * a.x + a.y * a.y;
  return make_double2(a.x / d, -a.y / d);
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

__global__ void expand_xy_kernel(const double* __restrict__ xy, int64_t n, double* __restrict__ xyz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    xyz[3 * i] = xy[2 * i];
    xyz[3 * i + 1] = xy[2 * i + 1];
    xyz[3 * i + 2] = 0.0;
  }
}

// P2M: warp per leaf, lane = particle (strided), per-lane partial sums then a fixed butterfly
template <int P>
__global__ void p2m2d_kernel(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ cbeg,
                             const int32_t* __restrict__ cend, const double4* __restrict__ center,
                             const double4* __restrict__ pos, int stride, double2* __restrict__ M) {
  const int lane = threadIdx.x & 31;
  const int64_t li = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (li >= nleaves) return;
  const int leaf = leaves[li];
  const double4 c = center[leaf];
  double2 acc[P + 1];
#pragma unroll
  for (int k = 0; k <= P; ++k) acc[k] = make_double2(0.0, 0.0);
  for (int i = cbeg[leaf] + lane; i < cend[leaf]; i += 32) {
    const double4 v = pos[i];
    const double2 w = make_double2(v.x - c.x, v.y - c.y);
    acc[0].x += v.w;
    double2 wk = w;
#pragma unroll
    for (int k = 1; k <= P; ++k) {
      acc[k] = cadd2(acc[k], csc(wk, -v.w / k));
      wk = cm(wk, w);
    }
  }
#pragma unroll
  for (int k = 0; k <= P; ++k)
    for (int o = 16; o; o >>= 1) {
      acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
      acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
    }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k <= P; ++k) M[(int64_t)leaf * stride + k] = acc[k];
}

// M2M for the parents of one level: thread per (parent, l), children in order
__global__ void m2m2d_kernel(int64_t lb, int64_t ncell, const int32_t* __restrict__ child,
                             const int32_t* __restrict__ nchild, const double4* __restrict__ center, int p, int stride,
                             double2* __restrict__ M) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ncell * (p + 1);
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = lb + t / (p + 1);
    const int l = (int)(t % (p + 1));
    const int c0 = child[cell];
    if (c0 < 0) continue;
    const double4 cp = center[cell];
    double2 s = make_double2(0.0, 0.0);
    for (int ch = c0; ch < c0 + nchild[cell]; ++ch) {
      const double4 cc = center[ch];
      const double2 z0 = make_double2(cc.x - cp.x, cc.y - cp.y);
      const double2* a = M + (int64_t)ch * stride;
      if (l == 0) {
        s = cadd2(s, a[0]);
        continue;
      }
      // -a_0 z0^l / l + sum_{k=1..l} a_k z0^(l-k) C(l-1, k-1), z0 powers built from k = l down
      double2 zp = make_double2(1.0, 0.0), t2 = make_double2(0.0, 0.0);
      for (int k = l; k >= 1; --k) {
        t2 = cadd2(t2, csc(cm(a[k], zp), c_binom.v[l - 1][k - 1]));
        zp = cm(zp, z0);
      }
      s = cadd2(s, cadd2(t2, csc(cm(a[0], zp), -1.0 / l)));
    }
    M[cell * stride + l] = s;
  }
}

// M2L: warp per target cell; lane k < p+1 owns output l = k; per source, lane k forms
// b_k = a_k z0^-k and broadcasts it; sources in list order
// warp per target cell; W = 16 (p <= 15): two source cells per pass, one per half-warp, lane l of
// a half computing order l; W = 32 (p = 16): one source cell per pass
template <int W>
__global__ void m2l2d_kernel(int64_t ncells, const int32_t* __restrict__ off, const int32_t* __restrict__ src,
                             const double4* __restrict__ center, const double2* __restrict__ M, int p, int stride,
                             double2* __restrict__ L) {
  // signed series coefficients, [k][l] so that the lanes (l) of one k read consecutive words:
  // l = 0: (-1)^k; l >= 1: C(l+k-1, k-1) (-1)^k
  __shared__ double coef[(kMaxP2 + 1) * (kMaxP2 + 1)];
  for (int t = threadIdx.x; t < (p + 1) * (p + 1); t += blockDim.x) {
    const int k = t / (p + 1), l = t % (p + 1);
    coef[t] = k == 0 ? 0.0 : (l == 0 ? 1.0 : c_binom.v[l + k - 1][k - 1]) * ((k & 1) ? -1.0 : 1.0);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, h = lane / W, lw = lane % W;
  const int64_t A = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (A >= ncells) return;
  const double4 ca = center[A];
  const int l = lw <= p ? lw : 0;
  double2 acc = make_double2(0.0, 0.0);
  const int e1 = off[A + 1];
  for (int e0 = off[A]; e0 < e1; e0 += 32 / W) {
    const bool valid = e0 + h < e1;
    const int B = src[valid ? e0 + h : e0];
    const double4 cb = center[B];
    const double2 z0 = make_double2(cb.x - ca.x, cb.y - ca.y);
    const double2 inv = cinv(z0);
    double2 ip = make_double2(1.0, 0.0);  // inv^l by repeated multiplication (l <= 16)
    for (int k = 0; k < l; ++k) ip = cm(ip, inv);
    const double a0 = M[(int64_t)B * stride].x;  // a_0 = total charge of B: real
    const double2 bk = lw <= p ? cm(M[(int64_t)B * stride + l], ip) : make_double2(0.0, 0.0);  // a_l z0^-l
    double2 s = make_double2(0.0, 0.0);
    for (int k = 1; k <= p; ++k) {
      const double2 b = shfl2(bk, h * W + k);
      const double cf = coef[k * (p + 1) + l];
      s.x = fma(b.x, cf, s.x);
      s.y = fma(b.y, cf, s.y);
    }
    double2 v;
    if (l == 0) {  // a_0 log(-z0): only its real part a_0 log|z0| reaches an output (R45)
      v = make_double2(fma(a0, 0.5 * log(z0.x * z0.x + z0.y * z0.y), s.x), s.y);
    } else {
      v = cm(ip, make_double2(s.x - a0 / l, s.y));
    }
    if (valid) acc = cadd2(acc, v);
  }
  for (int o = 16; o >= W; o >>= 1) acc = cadd2(acc, make_double2(__shfl_xor_sync(0xffffffffu, acc.x, o),
                                                                  __shfl_xor_sync(0xffffffffu, acc.y, o)));
  if (lane <= p) L[A * stride + lane] = acc;
}

// L2L for the children of one level: thread per (child slot, l); adds to the child's M2L result
__global__ void l2l2d_kernel(int64_t lb, int64_t ncell, const int32_t* __restrict__ child,
                             const int32_t* __restrict__ nchild, const double4* __restrict__ center, int p, int stride,
                             double2* __restrict__ L) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ncell * 8 * (p + 1);
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = lb + t / (8 * (p + 1));
    const int r = (int)(t % (8 * (p + 1))), slot = r / (p + 1), l = r % (p + 1);
    const int c0 = child[cell];
    if (c0 < 0 || slot >= nchild[cell]) continue;
    const int ch = c0 + slot;
    const double4 cp = center[cell], cc = center[ch];
    const double2 w = make_double2(cc.x - cp.x, cc.y - cp.y);
    const double2* c = L + cell * stride;
    double2 s = make_double2(0.0, 0.0), wp = make_double2(1.0, 0.0);
    for (int k = l; k <= p; ++k) {
      s = cadd2(s, csc(cm(c[k], wp), c_binom.v[k][l]));
      wp = cm(wp, w);
    }
    L[(int64_t)ch * stride + l] = cadd2(L[(int64_t)ch * stride + l], s);
  }
}

// ln(x) for a normal positive double, split as ln x = k ln 2 + lm: x = 2^k m, m in [1, 2); the
// top 7 bits of m pick a table entry c_j = 1 / (1 + (j + 1/2) / 128) with T_j = -ln c_j (shared
// memory), u = m c_j - 1 is one fma (|u| <= 2^-8) and lm = T_j + ln(1 + u) with the series to u^7
// (truncation u^8 / 8 <= 2^-67, below 2^-13 ulp of any |ln x| >= 2^-8 and of u itself when k = 0
// and m ~ 1). k is returned as a double (exponent bits re-biased by one add, no conversion) so the
// caller accumulates sum q k and sum q lm separately and multiplies by ln 2 once per target.
// Subnormal and tiny x (never met at the normalised frame's distances, kept exact anyway) take
// the library log with k = 0.
#ifndef FMM_2D_LOG_TABLE
#define FMM_2D_LOG_TABLE 1
#endif
#ifndef FMM_2D_NEAR_UNROLL  // source-loop unroll; 1M lattice p = 8 near: 1 1.79, 2 1.73, 4 1.68, 8 1.655 ms
#define FMM_2D_NEAR_UNROLL 4
#endif
#ifndef FMM_2D_NEAR_BRANCHLESS  // 1: r = 0 by selects; measured neutral (1.72 vs 1.68 / 1.84 vs 1.85 ms)
#define FMM_2D_NEAR_BRANCHLESS 0
#endif
#ifndef FMM_2D_NEAR_SPLIT  // 1: G lanes per target (below); measured slower, profiles/r1_fmm2d.md
#define FMM_2D_NEAR_SPLIT 0
#endif
#ifndef FMM_2D_LOG_RCP  // 1: c_j rebuilt from j (rcp.approx.f32), only T_j loaded: measured slower (1.92 vs 1.68 ms)
#define FMM_2D_LOG_RCP 0
#endif
__device__ __forceinline__ double recip_mid(int j) {  // ~ 256 / (257 + 2 j), the same bits in table and lookup
  const float n = __uint_as_float(0x4B000000u | (unsigned)(257 + 2 * j)) - 8388608.0f;  // exact
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(n));
  const unsigned fb = __float_as_uint(r) + (8u << 23);  // x 256
  return __longlong_as_double(((long long)fb << 29) + ((long long)(1023 - 127) << 52));
}
__device__ __forceinline__ double log_tab(double x, const double2* __restrict__ tab, double& kd) {
  const long long b = __double_as_longlong(x);
  const long long be = b >> 52;  // biased exponent (x > 0)
  if (be < 1023 - 1000) {
    kd = 0.0;
    return log(x);
  }
  kd = __longlong_as_double(0x4330000000000000LL | be) - (4503599627370496.0 + 1023.0);
#if FMM_2D_LOG_RCP
  const int jj = (int)((b >> 45) & 127);
  const double2 cj = make_double2(recip_mid(jj), reinterpret_cast<const double*>(tab)[jj]);  // T_j packed
#else
  const double2 cj = tab[(b >> 45) & 127];  // (c_j, T_j)
#endif
  const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double u = fma(m, cj.x, -1.0);
  double s = 1.0 / 7.0;
  s = fma(s, u, -1.0 / 6.0);
  s = fma(s, u, 0.2);
  s = fma(s, u, -0.25);
  s = fma(s, u, 1.0 / 3.0);
  s = fma(s, u, -0.5);
  return fma(s * u, u, u) + cj.y;
}

// L2P + P2P: warp per target leaf, lane per target; outputs in caller order (perm), with the
// 2^-e rescale of the logarithm and the gradient
template <bool GRAD>
__global__ void near2d_kernel(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ cbeg,
                              const int32_t* __restrict__ cend, const int32_t* __restrict__ poff,
                              const int32_t* __restrict__ psrc, const double4* __restrict__ center,
                              const double4* __restrict__ pos, const double2* __restrict__ L, const double2* __restrict__ M,
                              int p, int stride, double eln2, double sgrad, const uint32_t* __restrict__ perm,
                              double* __restrict__ phi, double* __restrict__ grad) {
  __shared__ double2 tab[128];
  for (int j = threadIdx.x; j < 128; j += blockDim.x) {
    const double c = 1.0 / (1.0 + (j + 0.5) / 128.0);
#if FMM_2D_LOG_RCP
    (void)c;
    reinterpret_cast<double*>(tab)[j] = -log(recip_mid(j));  // T_j, 1 KB dense
#else
    tab[j] = make_double2(c, -log(c));
#endif
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t li = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (li >= nleaves) return;
  const int A = leaves[li];
  const double4 c = center[A];
  const double2* loc = L + (int64_t)A * stride;
  const double Q = M[0].x;  // root a_0 = total charge
  // FMM_2D_NEAR_SPLIT: G lanes per target (G | 32), each taking every G-th source, G chosen to
  // minimise the lane passes per source ceil(nt G / 32) / G (a leaf of 40 targets: G = 4, 5 passes
  // over 1/4 of the sources instead of 2 over all of them). Measured slower (uniform square 1M:
  // near 2.63 vs 1.95 ms), so the shipped kernel is G = 1: lane per target, sources broadcast.
  const int b0 = cbeg[A], nt = cend[A] - b0;
#if FMM_2D_NEAR_SPLIT
  int G = 1;
  for (int g = 2; g <= 32; g *= 2)
    if (((nt * g + 31) >> 5) * G < ((nt * G + 31) >> 5) * g) G = g;
#else
  const int G = 1;
#endif
  const int npass = (nt * G + 31) >> 5;
  for (int pass = 0; pass < npass; ++pass) {
    const int k = pass * 32 + lane, ti = k / G, ph = k & (G - 1);
    const bool act = ti < nt;
    const int i = b0 + (act ? ti : nt - 1);
    const double4 t = pos[i];
    double f = 0.0, fk = 0.0, gx = 0.0, gy = 0.0, q0 = 0.0;  // phi = -(f + ln2 fk) / 2 + ...
    for (int e = poff[A]; act && e < poff[A + 1]; ++e) {
      const int B = psrc[e];
#if FMM_2D_NEAR_UNROLL == 2
#pragma unroll 2
#elif FMM_2D_NEAR_UNROLL == 4
#pragma unroll 4
#elif FMM_2D_NEAR_UNROLL == 8
#pragma unroll 8
#endif
      for (int j = cbeg[B] + ph; j < cend[B]; j += G) {
        const double4 s = pos[j];
        const double dx = t.x - s.x, dy = t.y - s.y;
        const double r2 = dx * dx + dy * dy;
#if FMM_2D_NEAR_BRANCHLESS && FMM_2D_LOG_TABLE
        // r = 0 (the target itself, coincident points) as a select, not a branch: the term is
        // evaluated at r^2 = 1 with charge 0 (an exact zero) and the charge goes to q0
        const bool nz = r2 > 0.0;
        const double qj = nz ? s.w : 0.0, r2s = nz ? r2 : 1.0;
        if (!nz) q0 += s.w;
        double kd;
        const double lm = log_tab(r2s, tab, kd);
        f = fma(qj, lm, f);
        fk = fma(qj, kd, fk);
        if (GRAD) {
          const double w = qj / r2s;
          gx -= w * dx;
          gy -= w * dy;
        }
#else
        if (r2 > 0.0) {
#if FMM_2D_LOG_TABLE
          double kd;
          const double lm = log_tab(r2, tab, kd);
          f = fma(s.w, lm, f);
          fk = fma(s.w, kd, fk);
#else
          f = fma(s.w, log(r2), f);
#endif
          if (GRAD) {
            const double w = s.w / r2;
            gx -= w * dx;
            gy -= w * dy;
          }
        } else {
          q0 += s.w;
        }
#endif
      }
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
      f += __shfl_xor_sync(0xffffffffu, f, off);
      fk += __shfl_xor_sync(0xffffffffu, fk, off);
      q0 += __shfl_xor_sync(0xffffffffu, q0, off);
      if (GRAD) {
        gx += __shfl_xor_sync(0xffffffffu, gx, off);
        gy += __shfl_xor_sync(0xffffffffu, gy, off);
      }
    }
    if (!act || ph != 0) continue;
    // L2P: Phi = sum c_l w^l, Phi' = sum l c_l w^(l-1) (Horner)
    const double2 w = make_double2(t.x - c.x, t.y - c.y);
    double2 Ph = loc[p], dPh = csc(loc[p], (double)p);
    for (int l = p - 1; l >= 0; --l) {
      Ph = cadd2(cm(Ph, w), loc[l]);
      if (l >= 1) dPh = cadd2(cm(dPh, w), csc(loc[l], (double)l));
    }
    if (p == 0) dPh = make_double2(0.0, 0.0);
    f = -0.5 * fma(fk, 6.93147180559945286227e-01, fma(fk, 2.31904681384629955842e-17, f)) - Ph.x;
    gx -= dPh.x;
    gy += dPh.y;
    const uint32_t o = perm[i];
    phi[o] = f - eln2 * (Q - q0);
    if (GRAD) {
      grad[3 * (int64_t)o] = gx * sgrad;
      grad[3 * (int64_t)o + 1] = gy * sgrad;
      grad[3 * (int64_t)o + 2] = 0.0;
    }
  }
}

template <int P>
void launch_p2m2d(fmm_plan_s& Pl, int stride) {
  const int64_t nl = Pl.nleaves;
  p2m2d_kernel<P><<<cdiv(nl * 32, 128), 128, 0, Pl.stream>>>(Pl.leaves, nl, Pl.cells.begin, Pl.cells.end,
                                                               Pl.cells.center, Pl.pos, stride, Pl.M);
  FMM_LAUNCHED("p2m2d_kernel");
}

unsigned grid2d(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)); }

}  // namespace

void expand_xy(const double* xy, int64_t n, double* xyz, cudaStream_t s) {
  expand_xy_kernel<<<grid2d(n), 256, 0, s>>>(xy, n, xyz);
  FMM_LAUNCHED("expand_xy_kernel");
}

void upward_2d(fmm_plan_s& P) {
  const int stride = P.nc;
  switch (P.p) {
    case 0: launch_p2m2d<0>(P, stride); break;
    case 1: launch_p2m2d<1>(P, stride); break;
    case 2: launch_p2m2d<2>(P, stride); break;
    case 3: launch_p2m2d<3>(P, stride); break;
    case 4: launch_p2m2d<4>(P, stride); break;
    case 5: launch_p2m2d<5>(P, stride); break;
    case 6: launch_p2m2d<6>(P, stride); break;
    case 7: launch_p2m2d<7>(P, stride); break;
    case 8: launch_p2m2d<8>(P, stride); break;
    case 9: launch_p2m2d<9>(P, stride); break;
    case 10: launch_p2m2d<10>(P, stride); break;
    case 11: launch_p2m2d<11>(P, stride); break;
    case 12: launch_p2m2d<12>(P, stride); break;
    case 13: launch_p2m2d<13>(P, stride); break;
    case 14: launch_p2m2d<14>(P, stride); break;
    case 15: launch_p2m2d<15>(P, stride); break;
    default: launch_p2m2d<16>(P, stride); break;
  }
  for (int l = P.max_level - 1; l >= 0; --l) {
    const int64_t lb = P.level_begin[l], nl = P.level_begin[l + 1] - lb;
    m2m2d_kernel<<<grid2d(nl * (P.p + 1)), 256, 0, P.stream>>>(lb, nl, P.cells.child, P.cells.nchild, P.cells.center,
                                                                P.p, stride, P.M);
    FMM_LAUNCHED("m2m2d_kernel");
  }
}

void m2l_2d(fmm_plan_s& P) {
  FMM_CUDA(cudaMemsetAsync(P.L.ptr, 0, P.L.bytes(), P.stream));
  auto m2l = P.p <= 15 ? m2l2d_kernel<16> : m2l2d_kernel<32>;
  m2l<<<cdiv(P.cells.n * 32, FMM_2D_M2L_THREADS), FMM_2D_M2L_THREADS, 0, P.stream>>>(P.cells.n, P.m2l.off, P.m2l.src, P.cells.center, P.M,
                                                                 P.p, P.nc, P.L);
  FMM_LAUNCHED("m2l2d_kernel");
}

void downward_2d(fmm_plan_s& P) {
  for (int l = 0; l < P.max_level; ++l) {
    const int64_t lb = P.level_begin[l], nl = P.level_begin[l + 1] - lb;
    l2l2d_kernel<<<grid2d(nl * 8 * (P.p + 1)), 256, 0, P.stream>>>(lb, nl, P.cells.child, P.cells.nchild,
                                                                    P.cells.center, P.p, P.nc, P.L);
    FMM_LAUNCHED("l2l2d_kernel");
  }
}

void near_2d(fmm_plan_s& P, double* phi, double* grad) {
  const double eln2 = P.e * 0.69314718055994530942;  // phi = phi_u - e ln2 (Q - Q0)
  const double sgrad = std::ldexp(1.0, -P.e);
  auto k = grad ? near2d_kernel<true> : near2d_kernel<false>;
  k<<<cdiv(P.nleaves * 32, FMM_2D_NEAR_THREADS), FMM_2D_NEAR_THREADS, 0, P.stream>>>(
      P.leaves, P.nleaves, P.cells.begin, P.cells.end, P.p2p.off, P.p2p.src, P.cells.center, P.pos, P.L, P.M, P.p,
      P.nc, eln2, sgrad, P.perm, phi, grad);
  FMM_LAUNCHED("near2d_kernel");
}

}  // namespace fmm
