// m2l_rot.cuh — the M2L v3 kernel (m2l_rot_kernel<P, SPLIT>) and its device helpers (m2l_rot.cu has
// the design notes, setup and launch). SPLIT: a tile's chunks are shared by `split` CTAs that write
// partial accumulators to global scratch, summed in a fixed order by rot_split_reduce_kernel. (An
// earlier form reduced through distributed shared memory in a thread-block cluster; merely having
// cluster kernels in the library slowed the p >= 11 path, which reads class data through L1, by
// 40-60 %: configs[4] M2L 437 -> 738 ms. No cluster features are used.)
#pragma once
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "harmonics.cuh"
#include "m2l_common.cuh"
#include "near_common.cuh"
#include "plan.h"

namespace fmm {
namespace m2l {

// "RI" layout of one expansion in the M2L v3 kernel (and of M~ rows): a Re plane
// (n, m >= 0) at n(n+1)/2 + m followed by an Im plane (n, m >= 1) at nc + n(n-1)/2 + m - 1;
// (p+1)^2 doubles; the rotation blocks read and write runs contiguous in m.
__host__ __device__ inline int ri_pos(int p, int n, int m, int part) {
  return part == 0 ? n * (n + 1) / 2 + m : (p + 1) * (p + 2) / 2 + n * (n - 1) / 2 + m - 1;
}
__host__ __device__ inline void ri_decode(int p, int q, int& n, int& m, int& part) {
  const int nc = (p + 1) * (p + 2) / 2;
  part = q >= nc;
  if (part) q -= nc;
  n = part;
  while ((part ? (n + 1) * n / 2 : (n + 1) * (n + 2) / 2) <= q) ++n;
  m = part ? q - n * (n - 1) / 2 + 1 : q - n * (n + 1) / 2;
}
// column base in a chunk buffer: stride S (= 4 mod 16 doubles) plus a +-4 swizzle on columns
// 4..7 of every 8, so B-fragment loads (8 columns x 4 rows) and C-fragment stores (8 rows x
// columns 2k+e) both hit 16 distinct 8-byte banks per half-warp on contiguous positions
__host__ __device__ inline int col_base(int c, int S) { return c * S + ((c & 4) ? ((c & 1) ? -4 : 4) : 0); }

constexpr int rot_xstride(int kpad) {
  int s = kpad + 8;  // room for the +-4 column swizzle
  while (s % 16 != 4) ++s;
  return s;
}
// chunk width (columns) of the v3 kernel and its shared-memory budget
#ifndef FMM_ROT_NC
#define FMM_ROT_NC 40
#endif
#ifndef FMM_ROT_NC_SMALLP
#define FMM_ROT_NC_SMALLP FMM_ROT_NC
#endif
#ifndef FMM_ROT_NC_HIGHP
#define FMM_ROT_NC_HIGHP 32
#endif
constexpr int rot_nc(int p) { return p <= 8 ? FMM_ROT_NC_SMALLP : (p <= 10 ? FMM_ROT_NC : FMM_ROT_NC_HIGHP); }
// class data staged into shared memory by TMA (p <= 10, where it fits beside the chunk buffers)
// or read by the MMA warps straight from L2 with one-item prefetch (larger p); measured at
// configs[2]: M2L 7.5 ms (shared) vs 8.4 ms (L2)
#ifndef FMM_ROT_SA_MAXP
#define FMM_ROT_SA_MAXP 10
#endif
constexpr bool rot_smem_a(int p) { return p <= FMM_ROT_SA_MAXP; }
#ifndef FMM_ROT_MMA
#define FMM_ROT_MMA 8
#endif
constexpr int kRotMMA = FMM_ROT_MMA;  // MMA warps of the v3 kernel
#ifndef FMM_ROT_ACC
#define FMM_ROT_ACC 7
#endif
#ifndef FMM_ROT_NEAR
#define FMM_ROT_NEAR 0
#endif
#ifndef FMM_ROT_REGS
#define FMM_ROT_REGS 0
#endif
// register rebalancing between the warp roles (setmaxnreg, per warpgroup): the prep and accumulate
// warps give registers to the MMA warps, which prefetch the next item's A fragments
constexpr int kRotRegsLow = 64, kRotRegsMMA = 136;
constexpr int kRotAcc = FMM_ROT_ACC;    // accumulate warps (p > 8)
// p <= 8 and p >= 11: 6 accumulate warps and prep batches of 4 (less contention for the MMA warps)
// (configs[3], p = 8: M2L 56.8 -> 55.4 ms; configs[4], p = 12: 423 -> 381 ms; p = 9, 10 take 7
// warps / batches of 6, which configs[2] prefers)
#ifndef FMM_ROT_HIGHP_SMALL
#define FMM_ROT_HIGHP_SMALL 1
#endif
#ifndef FMM_ROT_ACC_SMALL
#define FMM_ROT_ACC_SMALL 6
#endif
#ifndef FMM_ROT_PB_SMALL
#define FMM_ROT_PB_SMALL 4
#endif
constexpr int rot_acc_warps(int p) { return (p <= 8 || FMM_ROT_HIGHP_SMALL && p >= 11) ? FMM_ROT_ACC_SMALL : kRotAcc; }
#ifndef FMM_ROT_PB_BIG
#define FMM_ROT_PB_BIG 6
#endif
#ifndef FMM_ROT_PREP_W_BIG
#define FMM_ROT_PREP_W_BIG 4
#endif
#ifndef FMM_ROT_PREP_W_SMALL
#define FMM_ROT_PREP_W_SMALL 4
#endif
constexpr int rot_prep_warps(int p) { return (p <= 8 || FMM_ROT_HIGHP_SMALL && p >= 11) ? FMM_ROT_PREP_W_SMALL : FMM_ROT_PREP_W_BIG; }
constexpr int rot_prep_batch(int p) { return (p <= 8 || FMM_ROT_HIGHP_SMALL && p >= 11) ? FMM_ROT_PB_SMALL : FMM_ROT_PB_BIG; }
constexpr int kRotNear = FMM_ROT_NEAR;  // near-field (P2P) warps fused into the kernel
constexpr int rot_ksb(int p) { return p < 4 ? 2 : (p + 1 + 3) / 4; }  // k-steps of a big item (16 x 4 KSB), >= 2 (small items use 2)
// ints of one per-chunk descriptor: [ncol, nseg, class, 0 | srcs | meta | sslot | sbeg[NC + 1]]
constexpr int rot_desc_ints(int nc) { return (4 + 4 * nc + 1 + 3) & ~3; }

// ------------------------------------------------------------------------- items (host)
// A block: stage 0/2 = rotation of degree n, part (Re: m = 0..n, Im: m = 1..n); stage 1 =
// z translation of order m (n = m..p; Re and Im parts share the operator). An item packs
// blocks block-diagonally into slots 0..15 (big: 16 rows x 4 KSB k, one block of size > 8)
// or 0..7 (small: 8 x 8); slot s is both row s and k index s.
struct RotItem {
  int st, big, nparts, aoff;   // aoff: first double of its fragments in a class blob
  int slot[16];                // block code (stage 0/2: n | part << 5; stage 1: m) | local << 8, -1 empty
  int pos[2][16];              // RI position of each slot per part (stage 1: Re, Im), -1 none
};

}  // namespace m2l

namespace {
using namespace m2l;

struct RotArgs {
  M2LArgs a;
  const double* blobs;   // [nclass][blob] class data: azimuths | A fragments of every item
  const uint32_t* masks; // [2][NR] symmetry masks: 0 = multipole side (inverse map), 1 = local side
  const int32_t* sched;  // [3][NMMA][smax] item ids (-1 = end)
  const int32_t* ihdr;   // [nitems] big | nparts << 1 | aoff << 8
  const int32_t* ipos;   // [nitems][2][16] RI positions
  const int32_t* desc;   // [nchunks][rot_desc_ints(NC)] chunk descriptors
  int smax, nitems, blob;
  // fused near field (P2P on the FP64 pipe while the MMA warps use the DMMA pipe); p2p_phi null = off
  const int32_t *leaves, *cbeg, *cend, *p2p_off, *p2p_src;
  const double4* pos;
  int64_t nleaves;
  int* leaf_counter;
  double *p2p_phi, *p2p_grad;
  unsigned long long* prof;  // timing experiments (dbg & 256): per MMA warp cycles [wait X, stage 0..2, barriers]
  int split;                 // CTAs per tile: each takes a contiguous share of the tile's columns
  const int32_t* order;      // [ntiles] launch order of the tiles (decreasing work)
  double* scratch;           // split > 1: [ntiles][split][T][NR] partial accumulators
};

template <int P>
struct RGeo {
  static constexpr int NR = (P + 1) * (P + 1);
  static constexpr int KPAD = (NR + 3) & ~3;
  static constexpr int S = rot_xstride(KPAD);  // column stride (see col_base)
  static constexpr int NC = rot_nc(P);
  static constexpr int NT = NC / 8;
  static_assert(NC % 8 == 0, "chunk width must be a whole number of 8-column n-tiles");
  static constexpr int NMMA = kRotMMA, NPREP = rot_prep_warps(P), NACC = rot_acc_warps(P), NNEAR = kRotNear;
  static constexpr int KSB = rot_ksb(P);
  static constexpr int NCOEF = (P + 1) * (P + 2) / 2;
  static constexpr bool SA = rot_smem_a(P);
};

struct RotSmem {
  double *acc, *x0, *x1, *az;  // az: [2][2 (p + 1)] azimuths (cos, sin of m a) of the chunk's class
  double* ob;                  // SA: [2][blob] class data (azimuths first, so az = ob)
  uint64_t* bar;               // [2] X + class data of buffer b; [2 + j] descriptor buffer j (0..2)
  int32_t *desc;               // [3][rot_desc_ints(NC)] chunk descriptors (chunk i in i % 3)
  int32_t *dec, *pairtab, *sched, *ihdr, *ipos;
  int2* colt;                  // [2][NC] per buffer: (column base, 2 g) of each chunk column
  uint32_t *mmask, *lmask;     // [NR] symmetry masks (bit 2g: take re/im partner, 2g+1: negate)
  int* flag;                   // MMA warps done (near warps stop)
  int32_t* flat;               // [NMMA][3 smax] per-warp flattened item lists
};
template <int P>
__device__ __forceinline__ RotSmem rot_carve(double* sm, const RotArgs& r) {
  using G = RGeo<P>;
  RotSmem m;
  m.acc = sm;
  m.x0 = m.acc + (size_t)r.a.T * G::NR;
  m.x1 = m.x0 + G::NC * G::S;
  m.ob = m.x1 + G::NC * G::S;
  m.az = m.ob;
  uint64_t* b = (uint64_t*)(m.ob + (G::SA ? 2 * (size_t)r.blob : 4 * (size_t)(P + 1)));
  m.bar = b;
  m.desc = (int32_t*)(b + 6);  // 16-byte aligned (ob and bar sizes are multiples of 16)
  m.dec = m.desc + 3 * rot_desc_ints(G::NC);
  m.mmask = (uint32_t*)(m.dec + G::NR);
  m.lmask = m.mmask + G::NR;
  m.pairtab = (int32_t*)(m.lmask + G::NR);
  m.colt = (int2*)(((uintptr_t)(m.pairtab + G::NCOEF) + 7) & ~(uintptr_t)7);
  m.flag = (int*)(m.colt + 2 * G::NC);
  m.ihdr = m.flag + 2;
  m.ipos = m.ihdr + r.nitems;
  m.sched = m.ipos + 32 * r.nitems;
  m.flat = m.sched + 3 * G::NMMA * r.smax;
  return m;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// explicit shared-space loads: the carved pointers reach the item code as generic pointers, and
// generic loads (LD) of shared memory sit on the item's critical path (positions -> B -> DMMA)
// (read-only tables written before the kernel's first __syncthreads: free to schedule)
__device__ __forceinline__ int lds_i32(const int32_t* p) {
#ifdef FMM_NO_LDS
  return *p;
#endif
  int v;
  asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
// (class data rewritten per chunk by TMA: volatile keeps it after the chunk's barrier)
__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}


// One MMA item of shape MT x KS (k-steps), NT n-tiles (compile-time), in place: B streamed
// per k-step, results held in registers until every k-step was read.
template <int P, int MT, int KS, int NT>
__device__ __forceinline__ void rot_item_nt(const double (&a)[2][RGeo<P>::KSB], const int32_t* pos, int nparts,
                                            double sgn1, double* xc, int lane, int dbg) {
  using G = RGeo<P>;
  const int colb = lane >> 2, kl = lane & 3;
  const double* xb = xc + col_base(colb, G::S);
  for (int pp = 0; pp < nparts; ++pp) {
    const int32_t* ps = pos + 16 * pp;
    int qk[KS], qr[MT];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) qk[ks] = 4 * ks + kl < 16 ? lds_i32(ps + 4 * ks + kl) : -1;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) qr[mt] = lds_i32(ps + 8 * mt + colb);
    double c[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int t = 0; t < NT; ++t) c[mt][t][0] = c[mt][t][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int q = qk[ks];
      double b[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) b[t] = (q >= 0 && !(dbg & 64)) ? xb[8 * t * G::S + q] : 0.0;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma884(c[mt][t][0], c[mt][t][1], a[mt][ks], b[t]);
    }
    __syncwarp();  // every lane's B loads precede the in-place stores
    const double sgn = pp ? sgn1 : 1.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int q = qr[mt];
      if (q < 0 || (dbg & 32)) continue;
      double* y0 = xc + col_base(2 * kl, G::S) + q;
      double* y1 = xc + col_base(2 * kl + 1, G::S) + q;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        y0[8 * t * G::S] = sgn * c[mt][t][0];
        y1[8 * t * G::S] = sgn * c[mt][t][1];
      }
    }
    __syncwarp();
  }
}

// n-tile dispatch: one inlined instance per n-tile count 1..NT (counts above NT cannot occur:
// a chunk has at most NC = 8 NT columns), keeping the kernel's code small (I-cache)
template <int P, int MT, int KS, int N>
__device__ __forceinline__ void rot_item_dispatch(const double (&a)[2][RGeo<P>::KSB], const int32_t* pos, int nparts,
                                                  double sgn1, int ntiles, double* xc, int lane, int dbg) {
  if constexpr (N >= RGeo<P>::NT) {
    rot_item_nt<P, MT, KS, RGeo<P>::NT>(a, pos, nparts, sgn1, xc, lane, dbg);
  } else {
    if (ntiles <= N)
      rot_item_nt<P, MT, KS, N>(a, pos, nparts, sgn1, xc, lane, dbg);
    else
      rot_item_dispatch<P, MT, KS, N + 1>(a, pos, nparts, sgn1, ntiles, xc, lane, dbg);
  }
}
template <int P, int MT, int KS>
__device__ __forceinline__ void rot_item(const double (&a)[2][RGeo<P>::KSB], const int32_t* pos, int nparts,
                                         double sgn1, int ntiles, double* xc, int lane, int dbg) {
  static_assert(RGeo<P>::NT <= 8, "n-tile dispatch covers up to 8");
  rot_item_dispatch<P, MT, KS, 1>(a, pos, nparts, sgn1, ntiles, xc, lane, dbg);
}

// A fragments of an item (class data in global memory, L2 resident), fragment order
template <bool GLOBAL>
__device__ __forceinline__ double lda(const double* p) {
  if (GLOBAL) {  // volatile: issued where written (the one-item prefetch), not sunk to its use
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
  return lds_f64(p);
}
template <int P, bool GLOBAL>
__device__ __forceinline__ void load_a(const double* __restrict__ A, bool big, double (&a)[2][RGeo<P>::KSB], int lane) {
  constexpr int KSB = RGeo<P>::KSB;
  if (big) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int ks = 0; ks < KSB; ++ks) a[mt][ks] = lda<GLOBAL>(A + (mt * KSB + ks) * 32 + lane);
  } else {
    a[0][0] = lda<GLOBAL>(A + lane);
    a[0][1] = lda<GLOBAL>(A + 32 + lane);
  }
}

// Named barriers: 1/2 Xfull(b) prep -> MMA; 3/4 Yfull(b) MMA -> acc; 7/8 Xfree(b) acc -> prep;
// 5 MMA warps (between stages); 6 prep warps.
template <int P, bool SPLIT>
__global__ void __launch_bounds__(32 * (RGeo<P>::NMMA + RGeo<P>::NPREP + RGeo<P>::NACC + RGeo<P>::NNEAR), 1)
    m2l_rot_kernel(const RotArgs r, int dbg) {
  using G = RGeo<P>;
  constexpr int NR = G::NR, NC = G::NC, S = G::S, NCOEF = G::NCOEF;
  constexpr int nmma_t = 32 * G::NMMA, nprep_t = 32 * G::NPREP, nacc_t = 32 * G::NACC;
  const int BLOB = r.blob;
  extern __shared__ double sm[];
  const RotSmem m = rot_carve<P>(sm, r);
  const M2LArgs& a = r.a;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int tile = SPLIT ? r.order[blockIdx.x / r.split] : r.order[blockIdx.x];
  const int h_split = SPLIT ? (int)(blockIdx.x % r.split) : 0;
  // ---- shared tables
  for (int e = tid; e < a.T * NR; e += nthr) m.acc[e] = 0.0;
  for (int k = tid; k < NCOEF - (P + 1); k += nthr) {  // k-th (n, m >= 1) pair
    int n = 1, kk = k;
    while (kk >= n) kk -= n, ++n;
    m.pairtab[k] = n | ((kk + 1) << 16);
  }
  for (int e = tid; e < 3 * G::NMMA * r.smax; e += nthr) m.sched[e] = r.sched[e];
  for (int e = tid; e < r.nitems; e += nthr) m.ihdr[e] = r.ihdr[e];
  for (int e = tid; e < 32 * r.nitems; e += nthr) m.ipos[e] = r.ipos[e];
  for (int q = tid; q < NR; q += nthr) {
    int n, mm, part;
    ri_decode(P, q, n, mm, part);
    m.dec[q] = (cidx(n, mm) << 8) | (n << 1) | part;
    m.mmask[q] = r.masks[q];
    m.lmask[q] = r.masks[NR + q];
  }
  if (tid == 0) {
    *m.flag = 0;
    for (int j = 0; j < 5; ++j) mbar_init(m.bar + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int c_first = a.tile_chunk[tile], c_last = a.tile_chunk[tile + 1];
  if (SPLIT && r.split > 1) {  // this CTA's share: chunks whose first column falls in its part of the column range
    const int col0 = a.chunk_begin[c_first], col1 = a.chunk_begin[c_last];
    auto first_at = [&](int col) {  // first chunk in [c_first, c_last] starting at or after col
      int lo = c_first, hi = c_last;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a.chunk_begin[mid] < col) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    const int b0 = first_at(col0 + (int)((int64_t)(col1 - col0) * h_split / r.split));
    const int b1 = first_at(col0 + (int)((int64_t)(col1 - col0) * (h_split + 1) / r.split));
    c_first = b0;
    c_last = h_split + 1 == r.split ? c_last : b1;
  }
  __syncthreads();
  if (warp >= G::NMMA + G::NPREP + G::NACC) {
    // ================= near warps: P2P of own leaves (global leaf counter) until the MMA warps are done
    if (r.p2p_phi && !(dbg & 512)) {
      while (true) {
        if (*(volatile int*)m.flag) break;
        int li = 0;
        if (lane == 0) li = atomicAdd(r.leaf_counter, 1);
        li = __shfl_sync(0xffffffffu, li, 0);
        if (li >= r.nleaves) break;
        if (r.p2p_grad)
          near::p2p_leaf_global<true, 2>(r.cbeg, r.cend, r.p2p_off, r.p2p_src, r.pos, r.leaves[li], lane, r.p2p_phi,
                                         r.p2p_grad);
        else
          near::p2p_leaf_global<false, 2>(r.cbeg, r.cend, r.p2p_off, r.p2p_src, r.pos, r.leaves[li], lane,
                                          r.p2p_phi, nullptr);
      }
    }
  } else if (warp >= G::NMMA + G::NPREP) {
    if (FMM_ROT_REGS && G::NNEAR == 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRotRegsLow));
    // ================= accumulate warps: acc[slot][r] += (D^L_g Az_L Y)[r] for chunk i
    const int h = tid - nmma_t - nprep_t;
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      named_sync(3 + b, nmma_t + nacc_t);  // Yfull(i)
      if (!(dbg & 4)) {
        const double* __restrict__ y = b ? m.x1 : m.x0;
        const double* __restrict__ ob = G::SA ? m.ob + b * BLOB : m.az + b * 2 * (P + 1);
        const int32_t* __restrict__ dsc = m.desc + (i % 3) * rot_desc_ints(NC);
        const int ns = dsc[1];
        const int* __restrict__ ss = dsc + 4 + 2 * NC;
        const int* __restrict__ sb = dsc + 4 + 3 * NC;
        double* __restrict__ acc = m.acc;
        const int2* __restrict__ colt = m.colt + b * NC;
        // thread per (n, m) pair (and segment range): the rotated column value e^{i m a}(yr + i yi)
        // is formed once per column and feeds both the Re and the Im row
        constexpr int RG2 = nacc_t / NCOEF > 0 ? nacc_t / NCOEF : 1;
        for (int t = h; t < RG2 * NCOEF; t += nacc_t) {
          const int rg = t / NCOEF, rre = t - rg * NCOEF;
          const int s_lo = ns * rg / RG2, s_hi = ns * (rg + 1) / RG2;
          const int d = m.dec[rre], n = (d >> 1) & 0x7f;
          const int mm = rre - cidx(n, 0);
          const int rim = mm ? NCOEF + rre - n - 1 : rre;
          const double ca = mm ? ob[2 * mm] : 1.0, sa = mm ? ob[2 * mm + 1] : 0.0;
          const uint32_t mre = m.lmask[rre], mim = mm ? m.lmask[rim] : 0u;
          for (int sgi = s_lo; sgi < s_hi; ++sgi) {
            const int ce = sb[sgi + 1];
            double* ap = acc + ss[sgi] * NR;
            double vre = ap[rre], vim = mm ? ap[rim] : 0.0;
            for (int col = sb[sgi]; col < ce; ++col) {
              const int2 cg = colt[col];  // (column base, 2 g)
              const double yr = y[cg.x + rre], yi = y[cg.x + rim];
              const double ure = fma(ca, yr, -sa * yi), uim = fma(sa, yr, ca * yi);
              const int ire = (int)((mre >> cg.y) & 3), iim = (int)((mim >> cg.y) & 3) ^ 1;
              const double tre = (ire & 1) ? uim : ure, tim = (iim & 1) ? uim : ure;
              vre = (ire & 2) ? vre - tre : vre + tre;
              vim = (iim & 2) ? vim - tim : vim + tim;
            }
            ap[rre] = vre;
            if (mm) ap[rim] = vim;
          }
        }
      }
      named_arrive(7 + b, nacc_t + nprep_t);  // Xfree(i): buffer b may take chunk i + 2
    }
  } else if (warp >= G::NMMA) {
    if (FMM_ROT_REGS && G::NNEAR == 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRotRegsLow));
    // ================= prep warps: descriptors, TMA bulk copies, symmetry map + Az_M in place
    const int h = tid - nmma_t;
    constexpr int DI = rot_desc_ints(NC);
    auto issue_desc = [&](int ch, int j) {  // descriptor of chunk ch into buffer j (one lane)
      fence_proxy_async();
      mbar_arrive_tx(m.bar + 2 + j, DI * sizeof(int32_t));
      bulk_g2s(m.desc + j * DI, r.desc + (int64_t)ch * DI, DI * sizeof(int32_t), m.bar + 2 + j);
    };
    if (h == 0 && c_first < c_last) issue_desc(c_first, 0);
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1, j = i % 3;
      if (i >= 2) named_sync(7 + b, nacc_t + nprep_t);  // Xfree(i - 2): X buffer b, descriptor (i + 1) % 3
      if (h == 0 && ch + 1 < c_last) issue_desc(ch + 1, (i + 1) % 3);
      double* xb = b ? m.x1 : m.x0;
      double* ob = G::SA ? m.ob + b * BLOB : m.az + b * 2 * (P + 1);
      const int32_t* dsc = m.desc + j * DI;
      mbar_wait(m.bar + 2 + j, (unsigned)((i / 3) & 1));
      const int ncol = dsc[0], cls = dsc[2];
      if (h < 32 && !(dbg & 8)) {
        fence_proxy_async();  // earlier generic accesses of xb / ob before the async-proxy writes
        if (h == 0) {
          mbar_arrive_tx(m.bar + b, (unsigned)((ncol * G::KPAD + (G::SA ? BLOB : 0)) * sizeof(double)));
          if (G::SA) bulk_g2s(ob, r.blobs + (int64_t)cls * BLOB, BLOB * sizeof(double), m.bar + b);
        }
        __syncwarp();
        for (int c = h; c < ncol; c += 32)
          bulk_g2s(xb + col_base(c, S), a.Mt + (int64_t)dsc[4 + c] * G::KPAD, G::KPAD * sizeof(double), m.bar + b);
      }
      for (int c = h; c < ncol; c += nprep_t) m.colt[b * NC + c] = make_int2(col_base(c, S), 2 * (dsc[4 + NC + c] >> 8));
      if (!G::SA) {
        for (int e = h; e < 2 * (P + 1); e += nprep_t) ob[e] = __ldg(r.blobs + (int64_t)cls * BLOB + e);
        named_sync(6, nprep_t);  // azimuths visible to every prep thread
      }
      const int ncol8 = (ncol + 7) & ~7;  // padding columns of the last n-tile: zeros
      for (int e = h; e < (ncol8 - ncol) * G::KPAD; e += nprep_t)
        xb[col_base(ncol + e / G::KPAD, S) + e % G::KPAD] = 0.0;
      if (!(dbg & 8)) mbar_wait(m.bar + b, (unsigned)((i >> 1) & 1));
      if (!(dbg & 2)) {
        // X[col] <- Az_M (D^M_g)^-1 X[col]; item = (column, (n, m >= 1) pair), batches of
        // four items: all loads, then the arithmetic, then the stores (no smem aliasing stalls)
        constexpr int NP = NCOEF - (P + 1);  // pairs with m >= 1
        constexpr int kPB = rot_prep_batch(P);  // items per batch
        const int nit = ncol * NP;
        for (int it0 = h; it0 < nit; it0 += kPB * nprep_t) {
          double v0[kPB], v1[kPB], cs[kPB], sn[kPB];
          uint32_t f0[kPB], f1[kPB];
          int base[kPB], rre[kPB], rim[kPB];
#pragma unroll
          for (int u = 0; u < kPB; ++u) {
            const int it = it0 + u * nprep_t;
            const int itc = it < nit ? it : 0;
            const int col = itc / NP, k = itc - col * NP;
            const int pe = m.pairtab[k], n = pe & 0xffff, mm = pe >> 16;
            const int g2 = 2 * (dsc[4 + NC + col] >> 8);
            base[u] = it < nit ? col_base(col, S) : -1;
            rre[u] = cidx(n, mm);
            rim[u] = NCOEF + rre[u] - n - 1;
            f0[u] = m.mmask[rre[u]] >> g2;
            f1[u] = m.mmask[rim[u]] >> g2;
            v0[u] = xb[col_base(col, S) + rre[u]];
            v1[u] = xb[col_base(col, S) + rim[u]];
            cs[u] = ob[2 * mm];
            sn[u] = ob[2 * mm + 1];
          }
#pragma unroll
          for (int u = 0; u < kPB; ++u) {
            double u0 = (f0[u] & 1) ? v1[u] : v0[u], u1 = (f1[u] & 1) ? v0[u] : v1[u];
            u0 = (f0[u] & 2) ? -u0 : u0;
            u1 = (f1[u] & 2) ? -u1 : u1;
            v0[u] = cs[u] * u0 - sn[u] * u1;
            v1[u] = sn[u] * u0 + cs[u] * u1;
          }
#pragma unroll
          for (int u = 0; u < kPB; ++u)
            if (base[u] >= 0) {
              xb[base[u] + rre[u]] = v0[u];
              xb[base[u] + rim[u]] = v1[u];
            }
        }
        // m = 0 entries: sign only
        for (int it = h; it < ncol * (P + 1); it += nprep_t) {
          const int col = it / (P + 1), n = it - col * (P + 1), q = cidx(n, 0);
          const int g2 = 2 * (dsc[4 + NC + col] >> 8);
          if ((m.mmask[q] >> g2) & 2) xb[col_base(col, S) + q] = -xb[col_base(col, S) + q];
        }
      }
      named_arrive(1 + b, nprep_t + nmma_t);  // Xfull(i)
    }
  } else {
    if (FMM_ROT_REGS && G::NNEAR == 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRotRegsMMA));
    // ================= MMA warps: the three block-GEMM stages in place
    unsigned long long tw = 0, ts[3] = {0, 0, 0}, tb = 0, t0 = 0;
    const bool prof = (dbg & 256) && r.prof;
    // this warp's items of the three stages, flattened once into shared memory: id | stage << 16
    int32_t* fl = m.flat + warp * 3 * r.smax;
    int nflat = 0;
    if (lane == 0)
      for (int st = 0; st < 3; ++st)
        for (int k = 0; k < r.smax; ++k) {
          const int id = m.sched[(st * G::NMMA + warp) * r.smax + k];
          if (id < 0) break;
          fl[nflat++] = id | (st << 16);
        }
    nflat = __shfl_sync(0xffffffffu, nflat, 0);
    __syncwarp();
    auto flat = [&](int f) -> int { return lds_i32(fl + f); };
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      if (prof) t0 = clock64();
      named_sync(1 + b, nprep_t + nmma_t);  // Xfull(i)
      if (prof) tw += clock64() - t0;
      double* xc = b ? m.x1 : m.x0;
      const int32_t* dsc = m.desc + (i % 3) * rot_desc_ints(NC);
      const int ntiles = (dsc[0] + 7) >> 3;
      const double* gblob = G::SA ? m.ob + b * BLOB : r.blobs + (int64_t)dsc[2] * BLOB;
      double a[2][G::KSB], an[2][G::KSB];
      constexpr bool PF = !G::SA || FMM_ROT_REGS;  // prefetch the next item's A fragments
      int cur = nflat ? flat(0) : -1;
      if (PF && cur >= 0) {
        const int h0 = lds_i32(m.ihdr + (cur & 0xffff));
        load_a<P, !G::SA>(gblob + (h0 >> 8), h0 & 1, a, lane);
      }
      int st_now = 0;
      if (prof) t0 = clock64();
      for (int f = 0; f < nflat && !(dbg & 1); ++f) {
        const int id = cur & 0xffff, st = cur >> 16;
        const int nxt = f + 1 < nflat ? flat(f + 1) : -1;
        if (!PF)  // class data in shared memory, no registers to spare: load at the item
          load_a<P, false>(gblob + (lds_i32(m.ihdr + id) >> 8), lds_i32(m.ihdr + id) & 1, a, lane);
        else if (nxt >= 0)  // next item's fragments one item ahead
          load_a<P, !G::SA>(gblob + (lds_i32(m.ihdr + (nxt & 0xffff)) >> 8), lds_i32(m.ihdr + (nxt & 0xffff)) & 1, an,
                            lane);
        while (st_now < st) {  // stage barrier(s) before this item's stage
          if (prof) {
            const unsigned long long t1 = clock64();
            ts[st_now] += t1 - t0;
            t0 = t1;
          }
          if (!(dbg & 16)) named_sync(5, nmma_t);
          if (prof) {
            const unsigned long long t1 = clock64();
            tb += t1 - t0;
            t0 = t1;
          }
          ++st_now;
        }
        const int hd = lds_i32(m.ihdr + id);
        const int32_t* ps = m.ipos + 32 * id;
        const int nparts = (hd >> 1) & 3;
        const double sgn1 = st == 1 ? -1.0 : 1.0;  // z translation: Im = -Z Im
        if (hd & 1)
          rot_item<P, 2, G::KSB>(a, ps, nparts, sgn1, ntiles, xc, lane, dbg);
        else
          rot_item<P, 1, 2>(a, ps, nparts, sgn1, ntiles, xc, lane, dbg);
        if (PF)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int ks = 0; ks < G::KSB; ++ks) a[mt][ks] = an[mt][ks];
        cur = nxt;
      }
      while (st_now < 2) {  // remaining stage barriers (warps without items in later stages)
        if (prof) {
          const unsigned long long t1 = clock64();
          ts[st_now] += t1 - t0;
          t0 = t1;
        }
        if (!(dbg & 16)) named_sync(5, nmma_t);
        if (prof) {
          const unsigned long long t1 = clock64();
          tb += t1 - t0;
          t0 = t1;
        }
        ++st_now;
      }
      if (prof) ts[2] += clock64() - t0;
      named_arrive(3 + b, nmma_t + nacc_t);  // Yfull(i)
    }
    if (warp == 0 && lane == 0) *(volatile int*)m.flag = 1;  // near warps stop taking leaves
    if (prof && lane == 0) {
      unsigned long long* o = r.prof + 8 * warp;
      atomicAdd(o + 0, tw);
      atomicAdd(o + 1, ts[0]);
      atomicAdd(o + 2, ts[1]);
      atomicAdd(o + 3, ts[2]);
      atomicAdd(o + 4, tb);
      atomicAdd(o + 5, (unsigned long long)(c_last - c_first));
    }
  }
  __syncthreads();
  // write back L = L~ / h^{j+1} in complex m >= 0 storage; a split tile writes its raw partial
  // accumulators to scratch instead (rot_split_reduce_kernel sums them in rank order)
  if constexpr (SPLIT) {
    double* dst = r.scratch + ((int64_t)tile * r.split + h_split) * a.T * NR;
    for (int e = tid; e < a.T * NR; e += nthr) dst[e] = m.acc[e];
    return;
  }
  for (int e = tid; e < a.T * NR; e += nthr) {
    const int slot = e / NR, q = e - slot * NR;
    const int cell = a.tile_cells[tile * a.T + slot];
    if (cell < 0) continue;
    const int d = m.dec[q];
    const double v = m.acc[e] * a.hpow[a.level[cell] * (a.p + 2) + ((d >> 1) & 0x7f) + 1];
    ((double*)(a.L + (int64_t)cell * a.nc))[2 * (d >> 8) + (d & 1)] = v;
  }
}

// split tiles: L = (sum over the tile's split CTAs, in rank order, of their partials) / h^{j+1}
__global__ void rot_split_reduce_kernel(const double* __restrict__ scratch, int split, int64_t ntiles, int T, int NR,
                                        int P_, const int32_t* __restrict__ tile_cells, const int32_t* __restrict__ level,
                                        const double* __restrict__ hpow, int p, int nc, double2* __restrict__ L) {
  const int64_t tot = ntiles * T * NR;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = i / ((int64_t)T * NR);
    const int e = (int)(i - tile * T * NR);
    const int slot = e / NR, q = e - slot * NR;
    const int cell = tile_cells[tile * T + slot];
    if (cell < 0) continue;
    double s = 0.0;
    for (int k = 0; k < split; ++k) s += scratch[((tile * split + k) * T) * NR + e];
    int n, m, part;
    ri_decode(P_, q, n, m, part);
    ((double*)(L + (int64_t)cell * nc))[2 * cidx(n, m) + part] = s * hpow[level[cell] * (p + 2) + n + 1];
  }
}

}  // namespace
}  // namespace fmm
