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
#include <algorithm>
#include <utility>
#include <vector>

#include "harmonics.cuh"
#include "m2l_common.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kExpThreads = 128;  // >= ncoef(p) for p <= 14; two outputs per thread up to p = 21
constexpr int kM2MThreads = 256;  // M2M / L2L: items (child, coefficient)

// S7 P2M, warp per leaf: for each order m the column R_n^m (n = m..p) of every particle is
// generated in registers (diagonal product + two-term recurrence), q conj(R) accumulated per
// lane over the leaf's particles (lane = particle), then butterfly-reduced over the warp in
// a fixed order (deterministic); lane k writes coefficient (m + k, m).
#ifndef FMM_P2M_WARPS
#define FMM_P2M_WARPS 4
#endif
constexpr int kP2MWarps = FMM_P2M_WARPS;
#ifndef FMM_P2M_CACHE
#define FMM_P2M_CACHE 2
#endif
// particles per lane kept in registers (leaves of <= 32 kP2MCache particles; slots beyond the
// leaf are skipped warp-uniformly); larger leaves fall back to recomputing the diagonal per order
constexpr int kP2MCache = FMM_P2M_CACHE;

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
    for (int u = 0; u < kP2MCache; ++u)
      if (u == 0 || 32 * u < e - b) p2m_column<P>(acc, m, dg[u], px[u], py[u], pz[u], pq[u]);
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
    for (int t = lane; t < 2 * len; t += 32) {  // 2 len = 34 > 32 only for p = 16, m = 0
      double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
      for (int r = 0; r < 32; r += 2) {
        s0 += rw[r * kStride + t];
        s1 += rw[(r + 1) * kStride + t];
      }
      Ml[2 * cidx(m + (t >> 1), m) + (t & 1)] = s0 + s1;
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
// ---- S8 / S10 on the FP64 tensor cores (shift_variant 2). In scaled form the M2M and L2L
// shifts of a child at offset d = h_c u from its parent (u in {-1, 1}^3, h_c the child half
// side) are level-independent real matrices A(u) acting on (p+1)^2 real coefficients:
//   M2M: M_p{j} = h_c^j  sum conj R_n^m(u) M~_c{j-n},     M~_c = M_c h_c^{-deg}
//   L2L: L_c{j} = h_c^-j sum L~_p{n} conj R_{n-j}^{m-k}(u), L~_p = L_p h_c^{deg}
// and the eight octants are one operator A = A(+,+,+) conjugated by diagonal sign matrices,
// A(rho u) = S_rho A S_rho (the coordinate flips act on a coefficient (n, m, re/im) as
// x: (-1)^m conj, y: conj, z: (-1)^(n+m)). So one DMMA GEMM serves a whole
// level: a warp takes two parents, their 8 children are the 8 columns of an m8n8k4 tile,
// signs and powers of h_c are applied when the columns are gathered and in the epilogue.
// M2M sums the 8 signed columns of its parent (shuffle over the quad, fixed order); L2L adds
// each column to its child. Degree-blocked real layout => M2M is block lower triangular
// (output degree j reads degrees <= j), L2L block upper triangular; zero blocks are skipped.
#ifndef FMM_SHIFT_WARPS
#define FMM_SHIFT_WARPS 4
#endif
constexpr int kShiftWarps = FMM_SHIFT_WARPS;

__host__ __device__ constexpr int shift_isq(int r) {
  int n = 0;
  while ((n + 1) * (n + 1) <= r) ++n;
  return n;
}
__host__ __device__ constexpr int shift_nr(int p) { return (p + 1) * (p + 1); }
__host__ __device__ constexpr int shift_nmt(int p) { return (shift_nr(p) + 7) / 8; }
__host__ __device__ constexpr int shift_nks(int p) { return (shift_nr(p) + 3) / 4; }
// k-step range [lo, hi) of the non-zero blocks of row tile mt
__host__ __device__ constexpr int shift_lo(int p, bool l2l, int mt) {
  return l2l ? (shift_isq(8 * mt) * shift_isq(8 * mt)) / 4 : 0;
}
__host__ __device__ constexpr int shift_hi(int p, bool l2l, int mt) {
  return l2l ? shift_nks(p)
             : ((shift_isq(8 * mt + 7 < shift_nr(p) ? 8 * mt + 7 : shift_nr(p) - 1) + 1) *
                    (shift_isq(8 * mt + 7 < shift_nr(p) ? 8 * mt + 7 : shift_nr(p) - 1) + 1) +
                3) / 4;
}
// packed fragment offset (in k-steps) of row tile mt; shift_off(p, l2l, nmt) = total
__host__ __device__ constexpr int shift_off(int p, bool l2l, int mt) {
  int o = 0;
  for (int t = 0; t < mt; ++t) o += shift_hi(p, l2l, t) - shift_lo(p, l2l, t);
  return o;
}

// A(+,+,+) column by column: block per input real coefficient r, thread per output (j, k);
// written in packed DMMA fragment order (only the non-zero k-step blocks of each row tile)
template <bool L2L>
__global__ void build_shift_ops_kernel(int p, int nc, double* __restrict__ frag) {
  extern __shared__ double2 sh[];  // R[nc], E[nc]
  double2* R = sh;
  double2* E = sh + nc;
  const int r = blockIdx.x;
  for (int m = threadIdx.x; m <= p; m += blockDim.x) regular_column(1.0, 1.0, 1.0, m, p, R);
  for (int t = threadIdx.x; t < nc; t += blockDim.x) E[t] = make_double2(0, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    int n, m, part;
    m2l::real_decode(r, n, m, part);
    E[cidx(n, m)] = part ? make_double2(0, 1) : make_double2(1, 0);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    int j, k;
    decode_jk(t, j, k);
    const double2 s = L2L ? l2l_term(E, R, p, j, k) : m2m_term(R, E, j, k);
    for (int part = 0; part < (k > 0 ? 2 : 1); ++part) {
      const int row = m2l::real_index(j, k, part), mt = row >> 3, ks = r >> 2;
      const double v = part ? s.y : s.x;
      if (ks >= shift_lo(p, L2L, mt) && ks < shift_hi(p, L2L, mt))
        frag[((size_t)shift_off(p, L2L, mt) + ks - shift_lo(p, L2L, mt)) * 32 + (row & 7) * 4 + (r & 3)] = v;
      else if (v != 0.0)
        __trap();  // a non-zero outside the degree-triangular structure: the skip rule is wrong
    }
  }
}

// rinfo(r) = cidx(n, m) | part << 12 | n << 13 | flip mask (bit0 x, bit1 y, bit2 z) << 18
__device__ __forceinline__ uint32_t shift_rinfo(int r) {
  int n, m, part;
  m2l::real_decode(r, n, m, part);
  const uint32_t fx = (m & 1) ^ part, fy = part, fz = (n + m) & 1;
  return (uint32_t)cidx(n, m) | (uint32_t)part << 12 | (uint32_t)n << 13 | (fx | fy << 1 | fz << 2) << 18;
}
__device__ __forceinline__ double sgn(uint32_t info, int oct) {
  return (__popc((info >> 18) & oct) & 1) ? -1.0 : 1.0;
}
// DMMA without `volatile`: independent row tiles may be interleaved by the scheduler
__device__ __forceinline__ void dmma_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int PAR>
struct ShiftTask {
  int64_t (&cell)[PAR];
  int (&c0)[PAR];
  int (&nch)[PAR];
  int (&oA)[PAR];
  int (&oB)[PAR];
  double (&hp)[PAR];
  double (&hi)[PAR];
};

// one row tile: DMMA over its non-zero k-steps (compile-time range), then the epilogue
template <int P, bool L2L, int PAR, int MT>
__device__ __forceinline__ void shift_tile(const ShiftTask<PAR>& st, const double (&x)[PAR][shift_nks(P)],
                                           const double* fa, const uint32_t* rinfo, double2* E, int lane) {
  constexpr int NR = shift_nr(P), NC = (P + 1) * (P + 2) / 2;
  constexpr int LO = shift_lo(P, L2L, MT), HI = shift_hi(P, L2L, MT), OFF = shift_off(P, L2L, MT);
  const int c = lane >> 2, kq = lane & 3;
  const int row = 8 * MT + c;
  const uint32_t inf = row < NR ? rinfo[row] : 0u;
  const int ci = inf & 0xfff, part = (inf >> 12) & 1, n = (inf >> 13) & 31;
  double y0[PAR], y1[PAR], old0[PAR], old1[PAR];
#pragma unroll
  for (int q = 0; q < PAR; ++q) {
    y0[q] = y1[q] = 0.0;
    old0[q] = old1[q] = 0.0;
    if (L2L && row < NR) {  // the L2L epilogue adds to the children's M2L results: load them early
      if (2 * kq < st.nch[q]) old0[q] = ((const double*)(E + (int64_t)(st.c0[q] + 2 * kq) * NC))[2 * ci + part];
      if (2 * kq + 1 < st.nch[q])
        old1[q] = ((const double*)(E + (int64_t)(st.c0[q] + 2 * kq + 1) * NC))[2 * ci + part];
    }
  }
#pragma unroll
  for (int ks = LO; ks < HI; ++ks) {
    const double a = __ldg(fa + (OFF + ks - LO) * 32);
#pragma unroll
    for (int q = 0; q < PAR; ++q) dmma_nv(y0[q], y1[q], a, x[q][ks]);
  }
#pragma unroll
  for (int q = 0; q < PAR; ++q) {
    const double sc = __shfl_sync(0xffffffffu, L2L ? st.hi[q] : st.hp[q], n);
    if (!L2L) {
      double v = sgn(inf, st.oA[q]) * y0[q] + sgn(inf, st.oB[q]) * y1[q];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (kq == 0 && row < NR && st.nch[q] > 0) {
        double* d = (double*)(E + st.cell[q] * NC) + 2 * ci;
        d[part] = v * sc;
        if (row == n * n) d[1] = 0.0;  // Im M_n^0 = 0 (real charges): written, not left uninitialised
      }
    } else if (row < NR) {
      if (2 * kq < st.nch[q])
        ((double*)(E + (int64_t)(st.c0[q] + 2 * kq) * NC))[2 * ci + part] = old0[q] + sgn(inf, st.oA[q]) * y0[q] * sc;
      if (2 * kq + 1 < st.nch[q])
        ((double*)(E + (int64_t)(st.c0[q] + 2 * kq + 1) * NC))[2 * ci + part] = old1[q] + sgn(inf, st.oB[q]) * y1[q] * sc;
    }
  }
}

template <int P, bool L2L, int PAR, int... MT>
__device__ __forceinline__ void shift_tiles(std::integer_sequence<int, MT...>, const ShiftTask<PAR>& st,
                                            const double (&x)[PAR][shift_nks(P)], const double* fa,
                                            const uint32_t* rinfo, double2* E, int lane, int G, int grp) {
  ((MT % G == grp ? shift_tile<P, L2L, PAR, MT>(st, x, fa, rinfo, E, lane) : void()), ...);
}

// Warp per PAR parents; lane = (column c = lane / 4, k-quad kq = lane % 4). The B fragments
// (X[4 ks + kq][c] for every k-step) live in registers: gathered from the expansions with
// all loads in flight at once; A fragments are read through L1 (packed, compile-time offsets).
template <int P, bool L2L, int PAR>
__global__ void __launch_bounds__(32 * kShiftWarps) shift_dmma_kernel(
    int64_t lb, int64_t ncell, const int32_t* __restrict__ child, const int32_t* __restrict__ nchild,
    const double4* __restrict__ center, const double* __restrict__ frag, double2* __restrict__ E, int G) {
  constexpr int NR = shift_nr(P), NMT = shift_nmt(P), NKS = shift_nks(P), NC = (P + 1) * (P + 2) / 2;
  __shared__ uint32_t rinfo[4 * NKS];
  for (int r = threadIdx.x; r < 4 * NKS; r += blockDim.x) rinfo[r] = r < NR ? shift_rinfo(r) : 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = lane >> 2, kq = lane & 3;
  const int64_t ntask = (ncell + PAR - 1) / PAR * G;  // (parent group, row-tile group) pairs
  for (int64_t tg = (int64_t)blockIdx.x * kShiftWarps + w; tg < ntask; tg += (int64_t)gridDim.x * kShiftWarps) {
    const int64_t task = tg / G;
    const int grp = (int)(tg - task * G);
    double x[PAR][NKS];
    int64_t cell[PAR];
    int c0[PAR], nch[PAR], oA[PAR], oB[PAR];
    double hp[PAR], hi[PAR];  // lane n <= P holds h^n and h^-n (h = child half side)
#pragma unroll
    for (int q = 0; q < PAR; ++q) {
      cell[q] = lb + task * PAR + q;
      const bool ok = task * PAR + q < ncell;
      c0[q] = ok ? child[cell[q]] : -1;
      nch[q] = c0[q] >= 0 ? nchild[cell[q]] : 0;
      int o = 0;
      double h = 1.0;
      if (nch[q] > 0) {
        const double4 cp = center[cell[q]];
        const double4 cc = center[c0[q] + (c < nch[q] ? c : 0)];
        o = (cc.x < cp.x ? 1 : 0) | (cc.y < cp.y ? 2 : 0) | (cc.z < cp.z ? 4 : 0);
        h = cc.w;
      }
      oA[q] = __shfl_sync(0xffffffffu, o, 8 * kq);
      oB[q] = __shfl_sync(0xffffffffu, o, 8 * kq + 4);
      double v = 1.0;
      for (int i = 0; i < (lane <= P ? lane : 0); ++i) v *= h;
      hp[q] = v;
      hi[q] = 1.0 / v;
      const bool mine = c < nch[q];
      const double* src = (const double*)(E + (L2L ? cell[q] : (int64_t)(c0[q] + (mine ? c : 0))) * NC);
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const int k = 4 * ks + kq;
        const uint32_t inf = rinfo[k];
        const double sc = __shfl_sync(0xffffffffu, L2L ? hp[q] : hi[q], (inf >> 13) & 31);
        double v2 = 0.0;
        if (mine && k < NR) v2 = sgn(inf, o) * __ldg(src + 2 * (inf & 0xfff) + ((inf >> 12) & 1)) * sc;
        x[q][ks] = v2;
      }
    }
    ShiftTask<PAR> st{cell, c0, nch, oA, oB, hp, hi};
    shift_tiles<P, L2L, PAR>(std::make_integer_sequence<int, NMT>{}, st, x, frag + lane, rinfo, E, lane, G, grp);
  }
}

template <int P, bool L2L, int PAR>
void launch_shift_pp(fmm_plan_s& Pl, int64_t lb, int64_t ncell) {
  const int64_t npair = (ncell + PAR - 1) / PAR;
  // small (upper) levels: split the row tiles of a parent group over G warps
  int G = 1;
  while (2 * G <= shift_nmt(P) && npair * G * 2 <= 148 * 16) G *= 2;
  const int64_t blocks = std::min<int64_t>(cdiv(npair * G, kShiftWarps), 148 * 16);
  const double* frag = Pl.shift_ops.ptr + (L2L ? (size_t)shift_off(P, false, shift_nmt(P)) * 32 : 0);
  shift_dmma_kernel<P, L2L, PAR><<<(unsigned)blocks, 32 * kShiftWarps, 0, Pl.stream>>>(
      lb, ncell, Pl.cells.child, Pl.cells.nchild, Pl.cells.center, frag, L2L ? Pl.L : Pl.M, G);
  FMM_LAUNCHED(L2L ? "shift_dmma_kernel<L2L>" : "shift_dmma_kernel<M2M>");
}

template <int P, bool L2L>
void launch_shift_p(fmm_plan_s& Pl, int64_t lb, int64_t ncell) {
  static const int par = [] {
    const char* s = getenv("FMM_SHIFT_PAR");
    return s && s[0] == '1' ? 1 : 2;
  }();
  if constexpr (P <= 10) {
    if (par == 2) return launch_shift_pp<P, L2L, 2>(Pl, lb, ncell);
  }
  launch_shift_pp<P, L2L, 1>(Pl, lb, ncell);
}

template <bool L2L>
void launch_shift(fmm_plan_s& P, int64_t lb, int64_t ncell) {
  if (ncell <= 0) return;
  switch (P.p) {
    case 0: launch_shift_p<0, L2L>(P, lb, ncell); break;
    case 1: launch_shift_p<1, L2L>(P, lb, ncell); break;
    case 2: launch_shift_p<2, L2L>(P, lb, ncell); break;
    case 3: launch_shift_p<3, L2L>(P, lb, ncell); break;
    case 4: launch_shift_p<4, L2L>(P, lb, ncell); break;
    case 5: launch_shift_p<5, L2L>(P, lb, ncell); break;
    case 6: launch_shift_p<6, L2L>(P, lb, ncell); break;
    case 7: launch_shift_p<7, L2L>(P, lb, ncell); break;
    case 8: launch_shift_p<8, L2L>(P, lb, ncell); break;
    case 9: launch_shift_p<9, L2L>(P, lb, ncell); break;
    case 10: launch_shift_p<10, L2L>(P, lb, ncell); break;
    case 11: launch_shift_p<11, L2L>(P, lb, ncell); break;
    case 12: launch_shift_p<12, L2L>(P, lb, ncell); break;
    case 13: launch_shift_p<13, L2L>(P, lb, ncell); break;
    case 14: launch_shift_p<14, L2L>(P, lb, ncell); break;
    case 15: launch_shift_p<15, L2L>(P, lb, ncell); break;
    default: launch_shift_p<16, L2L>(P, lb, ncell); break;
  }
}

// level l's parents to shift: all cells of the level, or (multi-GPU, LET) those overlapping
// the owned range [let_level_lo[l], let_level_hi[l])
struct LevelRange {
  int64_t b, n;
};
LevelRange level_range(const fmm_plan_s& P, int l, bool own) {
  if (own && P.let_ready && (int)P.let_level_lo.size() > l)
    return {P.let_level_lo[l], P.let_level_hi[l] - P.let_level_lo[l]};
  return {P.level_begin[l], P.level_begin[l + 1] - P.level_begin[l]};
}

void upward_impl(fmm_plan_s& P, int64_t leaf_b, int64_t leaf_e, bool own = false) {
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
  if (P.shift_variant == 1) {
    const size_t sh = sizeof(double2) * 24 * nc;
    if (sh > 48 * 1024)  // per call: the opt-in is per device context (no process-wide cache)
      FMM_CUDA(cudaFuncSetAttribute(m2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    for (int l = P.max_level - 1; l >= 0; --l) {
      const LevelRange r = level_range(P, l, own);
      if (r.n <= 0) continue;
      m2m_kernel<<<(unsigned)r.n, kM2MThreads, sh, s>>>(r.b, P.cells.child, P.cells.nchild, P.cells.center, P.p, nc,
                                                        P.M);
      FMM_LAUNCHED("m2m_kernel");
    }
    return;
  }
  for (int l = P.max_level - 1; l >= 0; --l) {
    const LevelRange r = level_range(P, l, own);
    launch_shift<false>(P, r.b, r.n);
  }
}

void downward_impl(fmm_plan_s& P, bool own) {
  const int nc = P.nc;
  if (P.shift_variant == 1) {
    const size_t sh = sizeof(double2) * 9 * nc;
    for (int l = 0; l < P.max_level; ++l) {
      const LevelRange r = level_range(P, l, own);
      if (r.n <= 0) continue;
      l2l_kernel<<<(unsigned)r.n, kM2MThreads, sh, P.stream>>>(r.b, P.cells.child, P.cells.nchild, P.cells.center,
                                                               P.p, nc, P.L);
      FMM_LAUNCHED("l2l_kernel");
    }
    return;
  }
  for (int l = 0; l < P.max_level; ++l) {
    const LevelRange r = level_range(P, l, own);
    launch_shift<true>(P, r.b, r.n);
  }
}

}  // namespace

void upward(fmm_plan_s& P) { upward_impl(P, 0, P.nleaves); }
// multi-GPU (LET): P2M of this rank's leaves, M2M of the cells overlapping its range
void upward_own(fmm_plan_s& P) { upward_impl(P, P.own_leaf_begin, P.own_leaf_end, true); }

void m2l_pass(fmm_plan_s& P) {
  const int nc = P.nc;
  const size_t sh = sizeof(double2) * (ncoef(2 * P.p) + nc);
  m2l_v1_kernel<<<(unsigned)P.cells.n, kExpThreads, sh, P.stream>>>(P.m2l.off, P.m2l.src, P.cells.center, P.M,
                                                                     P.p, nc, P.L);
  FMM_LAUNCHED("m2l_v1_kernel");
}

void downward(fmm_plan_s& P) { downward_impl(P, false); }
// multi-GPU (LET): L2L of the cells overlapping this rank's range only
void downward_own(fmm_plan_s& P) { downward_impl(P, true); }

// the M2M and L2L operators A(+,+,+) in packed DMMA fragment order (shift_variant 2)
void shift_setup(fmm_plan_s& P) {
  if (P.shift_variant != 2) return;
  const int p = P.p;
  const size_t nm = (size_t)shift_off(p, false, shift_nmt(p)) * 32, nl = (size_t)shift_off(p, true, shift_nmt(p)) * 32;
  P.shift_ops.alloc((int64_t)(nm + nl));
  FMM_CUDA(cudaMemsetAsync(P.shift_ops.ptr, 0, sizeof(double) * (nm + nl), P.stream));
  const size_t sh = sizeof(double2) * 2 * P.nc;
  build_shift_ops_kernel<false><<<shift_nr(p), 128, sh, P.stream>>>(p, P.nc, P.shift_ops.ptr);
  FMM_LAUNCHED("build_shift_ops_kernel<M2M>");
  build_shift_ops_kernel<true><<<shift_nr(p), 128, sh, P.stream>>>(p, P.nc, P.shift_ops.ptr + nm);
  FMM_LAUNCHED("build_shift_ops_kernel<L2L>");
}

}  // namespace fmm
