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
constexpr int kP2MChunk = 32;     // particles whose harmonics are staged per round
constexpr int kM2MThreads = 256;  // M2M / L2L: items (child, coefficient)

// S7 P2M: M_n^m(c) = sum_i q_i conj R_n^m(x_i - c), one block per leaf; the harmonics
// of a chunk of particles are computed column-parallel (item = (particle, m)).
__global__ void p2m_kernel(const int32_t* __restrict__ leaves, const int32_t* __restrict__ cbeg,
                           const int32_t* __restrict__ cend, const double4* __restrict__ center,
                           const double4* __restrict__ pos, int p, int nc, double2* __restrict__ M) {
  extern __shared__ double2 shR[];  // [kP2MChunk][nc], rows hold q * conj(R)
  const int leaf = leaves[blockIdx.x];
  const int32_t b = cbeg[leaf], e = cend[leaf];
  const double4 c = center[leaf];
  const int t0 = threadIdx.x, t1 = threadIdx.x + kExpThreads;
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  for (int32_t s0 = b; s0 < e; s0 += kP2MChunk) {
    const int cnt = min(kP2MChunk, e - s0);
    for (int it = threadIdx.x; it < cnt * (p + 1); it += blockDim.x) {
      const int i = it / (p + 1), m = it - i * (p + 1);
      const double4 x = pos[s0 + i];
      double2* R = shR + i * nc;
      regular_column(x.x - c.x, x.y - c.y, x.z - c.z, m, p, R);
      for (int n = m; n <= p; ++n) {
        const double2 v = R[cidx(n, m)];
        R[cidx(n, m)] = make_double2(x.w * v.x, -x.w * v.y);
      }
    }
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      if (t0 < nc) a0 = cadd(a0, shR[k * nc + t0]);
      if (t1 < nc) a1 = cadd(a1, shR[k * nc + t1]);
    }
    __syncthreads();
  }
  if (t0 < nc) M[(int64_t)leaf * nc + t0] = a0;
  if (t1 < nc) M[(int64_t)leaf * nc + t1] = a1;
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
    const size_t sh = sizeof(double2) * kP2MChunk * nc;
    if (sh > 48 * 1024) FMM_CUDA(cudaFuncSetAttribute(p2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    p2m_kernel<<<(unsigned)(leaf_e - leaf_b), kExpThreads, sh, s>>>(
        P.leaves.ptr + leaf_b, P.cells.begin, P.cells.end, P.cells.center, P.pos, P.p, nc, P.M);
    FMM_LAUNCHED("p2m_kernel");
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
