// expansions.cu — matvec steps S7 (P2M), S8 (M2M), S9 (M2L), S10 (L2L) on
// spherical-harmonic expansions of order p (north_star (3), (4)).
//
// Paper: far field approximated "with multipole/local expansions"
// (PAPER.md:22-24); "a large part of the calculation time of FMM is spent on
// the translation of multipole expansions to local expansions";
// nested basis (M2M/L2L) is what makes the H^2 / FMM mat-vec O(N)
// (PAPER.md:266-269). Formulas: DESIGN.md §1.
//
// Every output coefficient is owned by one thread that accumulates its terms
// in a fixed order: no floating-point atomics, bitwise-deterministic results.
#include "harmonics.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kExpThreads = 128;  // >= ncoef(p) for p <= 14; two outputs per thread up to p = 21
constexpr int kM2MThreads = 256;  // M2M / L2L: items (child, coefficient)

// S7 P2M, warp per leaf: for each order m the column R_n^m (n = m..p) of every particle is
// generated in registers (diagonal product + two-term recurrence), q conj(R) accumulated per
// lane over the leaf's particles (lane = particle), then butterfly-reduced over the warp in
// a fixed order (deterministic); lane k writes coefficient (m + k, m).
constexpr int kP2MWarps = 4;
constexpr int kP2MCache = 2;  // particles per lane kept in registers (leaves of <= 64 particles)

// one particle's column m contribution: acc[k] += q conj(R_{m+k}^m), given d = R_m^m
template <int P>
__device__ __forceinline__ void p2m_column(double2 (&acc)[P + 1], int m, double2 d, double x, double y, double z,
                                           double q) {
  const double r2 = x * x + y * y + z * z;
  double2 a = d, bb = cscale(d, z);
  acc[0].x = fma(q, a.x, acc[0].x);
  acc[0].y = fma(-q, a.y, acc[0].y);
#pragma unroll
  for (int k = 1; k <= P; ++k) {
    if (m + k > P) break;
    if (k >= 2) {
      const int n = m + k;
      const double inv = c_inv_nm.v[n * (kMaxP + 1) + m];
      const double2 cc = make_double2(((2 * n - 1) * z * bb.x - r2 * a.x) * inv, ((2 * n - 1) * z * bb.y - r2 * a.y) * inv);
      a = bb;
      bb = cc;
    }
    acc[k].x = fma(q, bb.x, acc[k].x);
    acc[k].y = fma(-q, bb.y, acc[k].y);
  }
}

template <int P>
__global__ void __launch_bounds__(32 * kP2MWarps) p2m_warp_kernel(const int32_t* __restrict__ leaves, int64_t nleaves,
                                                                 const int32_t* __restrict__ cbeg,
                                                                 const int32_t* __restrict__ cend,
                                                                 const double4* __restrict__ center,
                                                                 const double4* __restrict__ pos, int nc,
                                                                 double2* __restrict__ M) {
  constexpr int kStride = 2 * (P + 1) + 1;  // odd stride: row writes and column reads conflict-free
  __shared__ double red[kP2MWarps][32 * kStride];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t li = (int64_t)blockIdx.x * kP2MWarps + w;
  if (li >= nleaves) return;  // warp-uniform; only __syncwarp below
  const int leaf = leaves[li];
  const int32_t b = cbeg[leaf], e = cend[leaf];
  const double4 c = center[leaf];
  double* Ml = (double*)(M + (int64_t)leaf * nc);
  double* rw = red[w];
  // the lane's first kP2MCache particles: relative coordinates, charge, running diagonal R_m^m
  double px[kP2MCache], py[kP2MCache], pz[kP2MCache], pq[kP2MCache];
  double2 dg[kP2MCache];
#pragma unroll
  for (int u = 0; u < kP2MCache; ++u) {
    const int32_t i = b + lane + 32 * u;
    const double4 v = i < e ? pos[i] : make_double4(c.x, c.y, c.z, 0.0);
    px[u] = v.x - c.x;
    py[u] = v.y - c.y;
    pz[u] = v.z - c.z;
    pq[u] = v.w;
    dg[u] = make_double2(1.0, 0.0);
  }
  for (int m = 0; m <= P; ++m) {
    const int len = P + 1 - m;  // column (n = m..p) of complex values
    double2 acc[P + 1];
#pragma unroll
    for (int k = 0; k <= P; ++k) acc[k] = make_double2(0.0, 0.0);
    if (m > 0) {
      const double s = c_half_inv.v[m];
#pragma unroll
      for (int u = 0; u < kP2MCache; ++u) dg[u] = cmul(dg[u], make_double2(s * px[u], s * py[u]));
    }
#pragma unroll
    for (int u = 0; u < kP2MCache; ++u) p2m_column<P>(acc, m, dg[u], px[u], py[u], pz[u], pq[u]);
    for (int32_t i = b + lane + 32 * kP2MCache; i < e; i += 32) {  // leaves larger than 32 kP2MCache
      const double4 v = pos[i];
      const double x = v.x - c.x, y = v.y - c.y, z = v.z - c.z;
      double2 d = make_double2(1.0, 0.0);
      for (int k = 1; k <= m; ++k) {
        const double s = c_half_inv.v[k];
        d = cmul(d, make_double2(s * x, s * y));
      }
      p2m_column<P>(acc, m, d, x, y, z, v.w);
    }
    // transpose through shared memory: lane t sums value t of the column over the 32 lanes
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      if (k >= len) break;
      rw[lane * kStride + 2 * k] = acc[k].x;
      rw[lane * kStride + 2 * k + 1] = acc[k].y;
    }
    __syncwarp();
    if (lane < 2 * len) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
      for (int r = 0; r < 32; r += 2) {
        s0 += rw[r * kStride + lane];
        s1 += rw[(r + 1) * kStride + lane];
      }
      Ml[2 * cidx(m + (lane >> 1), m) + (lane & 1)] = s0 + s1;
    }
    __syncwarp();
  }
}

template <int P>
void launch_p2m(fmm_plan_s& P_, const int32_t* leaves, int64_t nl, cudaStream_t s) {
  p2m_warp_kernel<P><<<cdiv(nl, kP2MWarps), 32 * kP2MWarps, 0, s>>>(leaves, nl, P_.cells.begin, P_.cells.end,
                                                                   P_.cells.center, P_.pos, P_.nc, P_.M);
  FMM_LAUNCHED("p2m_warp_kernel");
}

// M2M term for output (j, k): sum_{n<=j} sum_m conj R_n^m(c - c') M_{j-n}^{k-m}(c)
__device__ __forceinline__ double2 m2m_term(const double2* R, const double2* Mc, int j, int k) {
  double2 s = make_double2(0, 0);
  for (int n = 0; n <= j; ++n) {
    const int lo = max(-n, k - (j - n)), hi = min(n, k + (j - n));
    for (int m = lo; m <= hi; ++m) cfma(s, cconj(cget(R, n, m)), cget(Mc, j - n, k - m));
  }
  return s;
}

// S8 M2M for the internal cells of one level: one block per parent; the children's
// shift harmonics (item = (child, m)) and terms (item = (child, coefficient)) are
// computed in parallel, then each coefficient sums its children in digit order.
__global__ void m2m_kernel(int64_t lb, const int32_t* __restrict__ child, const int32_t* __restrict__ nchild,
                           const double4* __restrict__ center, int p, int nc, double2* __restrict__ M) {
  extern __shared__ double2 sh[];  // R[8][nc], Mc[8][nc], part[8][nc]
  double2* R = sh;
  double2* Mc = sh + 8 * nc;
  double2* part = sh + 16 * nc;
  const int64_t cell = lb + blockIdx.x;
  const int c0 = child[cell];
  if (c0 < 0) return;  // leaf: P2M already wrote M
  const int nch = nchild[cell];
  const double4 cp = center[cell];
  for (int t = threadIdx.x; t < nch * nc; t += blockDim.x) Mc[t] = M[(int64_t)c0 * nc + t];
  for (int it = threadIdx.x; it < nch * (p + 1); it += blockDim.x) {
    const int ch = it / (p + 1), m = it - ch * (p + 1);
    const double4 cc = center[c0 + ch];
    regular_column(cc.x - cp.x, cc.y - cp.y, cc.z - cp.z, m, p, R + ch * nc);
  }
  __syncthreads();
  for (int it = threadIdx.x; it < nch * nc; it += blockDim.x) {
    const int ch = it / nc, t = it - ch * nc;
    int j, k;
    decode_jk(t, j, k);
    part[it] = m2m_term(R + ch * nc, Mc + ch * nc, j, k);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    double2 a = make_double2(0, 0);
    for (int ch = 0; ch < nch; ++ch) a = cadd(a, part[ch * nc + t]);
    M[cell * nc + t] = a;
  }
}

// M2L term for output (j, k): sum_{n<=p} (-1)^n sum_{|m|<=n} M_n^m I_{j+n}^{k+m}(cB - cA)
__device__ __forceinline__ double2 m2l_term(const double2* Mb, const double2* I, int p, int j, int k) {
  double2 s = make_double2(0, 0);
  for (int n = 0; n <= p; ++n) {
    double2 sn = make_double2(0, 0);
    for (int m = -n; m <= n; ++m) cfma(sn, cget(Mb, n, m), cget(I, j + n, k + m));
    if (n & 1)
      s = make_double2(s.x - sn.x, s.y - sn.y);
    else
      s = cadd(s, sn);
  }
  return s;
}

// S9 M2L v1 (matrix-free, O(p^4) per pair): one block per target cell, owner computes.
__global__ void m2l_v1_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ src,
                              const double4* __restrict__ center, const double2* __restrict__ M, int p, int nc,
                              double2* __restrict__ L) {
  extern __shared__ double2 sh[];  // I[ncoef(2p)], Mb[nc]
  double2* I = sh;
  double2* Mb = sh + ncoef(2 * p);
  const int A = blockIdx.x;
  const double4 ca = center[A];
  const int t0 = threadIdx.x, t1 = threadIdx.x + kExpThreads;
  int j0 = 0, k0 = 0, j1 = 0, k1 = 0;
  if (t0 < nc) decode_jk(t0, j0, k0);
  if (t1 < nc) decode_jk(t1, j1, k1);
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  for (int q = off[A]; q < off[A + 1]; ++q) {
    const int B = src[q];
    const double4 cb = center[B];
    __syncthreads();
    for (int t = threadIdx.x; t < nc; t += blockDim.x) Mb[t] = M[(int64_t)B * nc + t];
    irregular_harmonics_par(cb.x - ca.x, cb.y - ca.y, cb.z - ca.z, 2 * p, I, threadIdx.x, blockDim.x);
    __syncthreads();
    if (t0 < nc) a0 = cadd(a0, m2l_term(Mb, I, p, j0, k0));
    if (t1 < nc) a1 = cadd(a1, m2l_term(Mb, I, p, j1, k1));
  }
  if (t0 < nc) L[(int64_t)A * nc + t0] = a0;
  if (t1 < nc) L[(int64_t)A * nc + t1] = a1;
}

// L2L term for output (j, k): sum_{n=j}^{p} sum_m L_n^m(c) conj R_{n-j}^{m-k}(c' - c)
__device__ __forceinline__ double2 l2l_term(const double2* Lp, const double2* R, int p, int j, int k) {
  double2 s = make_double2(0, 0);
  for (int n = j; n <= p; ++n) {
    const int lo = max(-n, k - (n - j)), hi = min(n, k + (n - j));
    for (int m = lo; m <= hi; ++m) cfma_conjb(s, cget(Lp, n, m), cget(R, n - j, m - k));
  }
  return s;
}

// S10 L2L for the children of one level's internal cells: one block per parent, shift
// harmonics column-parallel, item = (child, coefficient); each child coefficient is
// written by exactly one thread.
__global__ void l2l_kernel(int64_t lb, const int32_t* __restrict__ child, const int32_t* __restrict__ nchild,
                           const double4* __restrict__ center, int p, int nc, double2* __restrict__ L) {
  extern __shared__ double2 sh[];  // R[8][nc], Lp[nc]
  double2* R = sh;
  double2* Lp = sh + 8 * nc;
  const int64_t cell = lb + blockIdx.x;
  const int c0 = child[cell];
  if (c0 < 0) return;
  const int nch = nchild[cell];
  const double4 cp = center[cell];
  for (int t = threadIdx.x; t < nc; t += blockDim.x) Lp[t] = L[cell * nc + t];
  for (int it = threadIdx.x; it < nch * (p + 1); it += blockDim.x) {
    const int ch = it / (p + 1), m = it - ch * (p + 1);
    const double4 cc = center[c0 + ch];
    regular_column(cc.x - cp.x, cc.y - cp.y, cc.z - cp.z, m, p, R + ch * nc);
  }
  __syncthreads();
  for (int it = threadIdx.x; it < nch * nc; it += blockDim.x) {
    const int ch = it / nc, t = it - ch * nc;
    int j, k;
    decode_jk(t, j, k);
    double2* dst = L + (int64_t)(c0 + ch) * nc + t;
    *dst = cadd(*dst, l2l_term(Lp, R + ch * nc, p, j, k));
  }
}

}  // namespace

namespace {
void upward_impl(fmm_plan_s& P, int64_t leaf_b, int64_t leaf_e) {
  cudaStream_t s = P.stream;
  const int nc = P.nc;
  if (leaf_e > leaf_b) {
    const int64_t nl = leaf_e - leaf_b;
    const int32_t* lv = P.leaves.ptr + leaf_b;
    switch (P.p) {
      case 0: launch_p2m<0>(P, lv, nl, s); break;
      case 1: launch_p2m<1>(P, lv, nl, s); break;
      case 2: launch_p2m<2>(P, lv, nl, s); break;
      case 3: launch_p2m<3>(P, lv, nl, s); break;
      case 4: launch_p2m<4>(P, lv, nl, s); break;
      case 5: launch_p2m<5>(P, lv, nl, s); break;
      case 6: launch_p2m<6>(P, lv, nl, s); break;
      case 7: launch_p2m<7>(P, lv, nl, s); break;
      case 8: launch_p2m<8>(P, lv, nl, s); break;
      case 9: launch_p2m<9>(P, lv, nl, s); break;
      case 10: launch_p2m<10>(P, lv, nl, s); break;
      case 11: launch_p2m<11>(P, lv, nl, s); break;
      case 12: launch_p2m<12>(P, lv, nl, s); break;
      case 13: launch_p2m<13>(P, lv, nl, s); break;
      case 14: launch_p2m<14>(P, lv, nl, s); break;
      case 15: launch_p2m<15>(P, lv, nl, s); break;
      default: launch_p2m<16>(P, lv, nl, s); break;
    }
  }
  const size_t sh = sizeof(double2) * 24 * nc;
  static size_t configured = 0;
  if (sh > 48 * 1024 && sh > configured) {
    FMM_CUDA(cudaFuncSetAttribute(m2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    configured = sh;
  }
  for (int l = P.max_level - 1; l >= 0; --l) {
    const int64_t lb = P.level_begin[l], le = P.level_begin[l + 1];
    m2m_kernel<<<(unsigned)(le - lb), kM2MThreads, sh, s>>>(lb, P.cells.child, P.cells.nchild, P.cells.center, P.p,
                                                            nc, P.M);
    FMM_LAUNCHED("m2m_kernel");
  }
}
}  // namespace

void upward(fmm_plan_s& P) { upward_impl(P, 0, P.nleaves); }
void upward_own(fmm_plan_s& P) { upward_impl(P, P.own_leaf_begin, P.own_leaf_end); }

void m2l_pass(fmm_plan_s& P) {
  const int nc = P.nc;
  const size_t sh = sizeof(double2) * (ncoef(2 * P.p) + nc);
  m2l_v1_kernel<<<(unsigned)P.cells.n, kExpThreads, sh, P.stream>>>(P.m2l.off, P.m2l.src, P.cells.center, P.M,
                                                                     P.p, nc, P.L);
  FMM_LAUNCHED("m2l_v1_kernel");
}

void downward(fmm_plan_s& P) {
  const int nc = P.nc;
  const size_t sh = sizeof(double2) * 9 * nc;
  for (int l = 0; l < P.max_level; ++l) {
    const int64_t lb = P.level_begin[l], le = P.level_begin[l + 1];
    l2l_kernel<<<(unsigned)(le - lb), kM2MThreads, sh, P.stream>>>(lb, P.cells.child, P.cells.nchild, P.cells.center,
                                                                   P.p, nc, P.L);
    FMM_LAUNCHED("l2l_kernel");
  }
}

}  // namespace fmm
