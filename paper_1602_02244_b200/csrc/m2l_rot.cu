// m2l_rot.cu — S9 M2L v3 (default for p = 0..14): the translation-invariant class
// operators of v2 (m2l_dmma.cu) applied in rotation-factored form on FP64 tensor cores.
//
// Paper: M2L dominates; "Rotating the multipole expansion so that the
// translation is along the z-axis reduces the complexity from O(p^4) to O(p^3)"
// (the analytic end of the compute-memory axis); translation operators
// for boxes with the same relative positioning are identical and can be precomputed and
// stored; symmetry reduces the storage further.
//
// For a canonical class offset delta0 = rho (sin b cos a, sin b sin a, cos b) (finer half
// sides) the dense scaled operator factorises exactly (tools/proto_m2l_rotation.py checks
// it against build_ops_kernel's dense T~ to ~1e-14):
//
//   T~ = Az_L(a) . Dt(b) . Z~(rho) . D(b) . Az_M(a)
//
//   Az_M(a): (re, im) of M~_n^m  ->  e^{i m a} (re + i im)          (2x2 per (n, m))
//   D(b)   : per degree n, the rotation Ry(-b) on multipole coefficients; it does not mix
//            Re and Im: an (n+1)^2 Re block and an n^2 Im block, computed per class by an
//            exact sphere quadrature (Gauss-Legendre x trapezoid, exact to degree 2p)
//   Z~(rho): per order m the z-axis translation L~_j^m = (-1)^{n+m} (j+n)!/rho^{j+n+1}
//            fA^{j+1} fB^n M~_n^m on Re, the negative on Im ((p+1-m)^2 each)
//   Dt(b)  : per degree j, Re block E^-1 D_re^T E (E = diag(1, 2, 2, ...)), Im block D_im^T
//   Az_L(a): (re, im) of L~_j^k  ->  e^{i k a} (re + i im)
//
// Work per pair (p = 10): 3 x 891 useful MACs (1392 padded DMMA-MAC blocks of 8x8x4 per
// 64 columns) instead of the dense 121^2 = 14641 (3968 DMMAs per 64 columns).
//
// Kernel (one CTA per tile of T target cells, as v2): warp-specialised, 16 warps.
//  * 4 prep warps: load chunk i's metadata, stage its class data (A fragments, azimuths)
//    and its source multipoles M~_B (contiguous rows of Kpad doubles) into shared memory
//    with cp.async.bulk (TMA bulk copies, completion on an mbarrier), apply each column's
//    symmetry map and Az_M in place, signal the MMA warps;
//  * 8 MMA warps: the three block-GEMM stages D, Z~, Dt on DMMA (mma.sync m8n8k4 f64), each
//    IN PLACE in the chunk's shared-memory buffer. The small per-degree / per-order blocks
//    are packed block-diagonally into "items" of two fixed shapes (16 x 4 KSB, 8 x 8); an
//    item reads and writes only its own positions (all B fragments are read before the
//    first store), A fragments come pre-arranged in fragment order (one 256-byte load per
//    fragment), a named barrier separates the stages, items are spread over the warps by a
//    static LPT schedule built on the host;
//  * 4 accumulate warps: add chunk i's result (Az_L and the symmetry map applied on the fly)
//    into the tile's shared-memory accumulators in column order (deterministic, no atomics).
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "harmonics.cuh"
#include "m2l_common.cuh"
#include "near_common.cuh"
#include "plan.h"

namespace cg = cooperative_groups;

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
constexpr int rot_nc(int p) { return p <= 10 ? FMM_ROT_NC : 32; }
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
#define FMM_ROT_ACC 8
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
constexpr int kRotAcc = FMM_ROT_ACC;    // accumulate warps
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

// ------------------------------------------------------------------- setup: operators
__global__ void quad_points_kernel(const double* __restrict__ glx, int p, double2* __restrict__ Rs) {
  const int nphi = 2 * p + 1, np = (p + 1) * nphi, nc = ncoef(p);
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < np * (p + 1); it += gridDim.x * blockDim.x) {
    const int pt = it / (p + 1), m = it - pt * (p + 1);
    const int kx = pt / nphi, t = pt - kx * nphi;
    const double ct = glx[kx], st = sqrt(fmax(0.0, 1.0 - ct * ct));
    double sp, cp;
    sincospi(2.0 * t / nphi, &sp, &cp);
    regular_column(st * cp, st * sp, ct, m, p, Rs + (int64_t)pt * nc);
  }
}


constexpr int kRotBuildThreads = 256;
constexpr int kQuadBatch = 32;
constexpr int kMaxEntPerThread = 13;  // ceil(sum_n (n+1)^2 + n^2 at p = 16 / 256)

struct ItemDev {  // device copy of RotItem (setup only)
  int st, big, nparts, aoff;
  int slot[16];
};

// One CTA per class: azimuth table, rotation blocks by quadrature, then every item's A
// fragments in DMMA fragment order (A[8 mt + lane/4][4 ks + lane%4]).
__global__ void __launch_bounds__(kRotBuildThreads) build_rot_ops_kernel(
    const uint64_t* __restrict__ class_keys, int p, const double* __restrict__ glx, const double* __restrict__ glw,
    const double2* __restrict__ Rs, const ItemDev* __restrict__ items, int nitems, int blob,
    double* __restrict__ blobs) {
  extern __shared__ double2 sh[];  // Rq[kQuadBatch][nc], then D[nent] (doubles)
  const int nc = ncoef(p), nphi = 2 * p + 1, np = (p + 1) * nphi;
  double2* Rq = sh;
  double* Dtab = (double*)(sh + kQuadBatch * nc);
  const int cls = blockIdx.x, tid = threadIdx.x;
  const uint64_t key = class_keys[cls];
  const int dl = (int)((key >> 57) & 0x3f) - 32;
  const double x0 = (double)((key >> 38) & 0x7ffff), y0 = (double)((key >> 19) & 0x7ffff),
               z0 = (double)(key & 0x7ffff);
  const double rxy = sqrt(x0 * x0 + y0 * y0), rho = sqrt(x0 * x0 + y0 * y0 + z0 * z0);
  const double alpha = atan2(y0, x0), beta = atan2(rxy, z0);
  const double cb = cos(beta), sb = sin(beta);
  const double fA = dl < 0 ? ldexp(1.0, -dl) : 1.0, fB = dl > 0 ? ldexp(1.0, dl) : 1.0;
  double* out = blobs + (int64_t)cls * blob;
  if (tid <= p) {
    double s, c;
    sincos(tid * alpha, &s, &c);
    out[2 * tid] = c;
    out[2 * tid + 1] = s;
  }
  // entries e -> (n, part, a, b): per degree n the Re block (a, b in 0..n) then the Im
  // block (a, b in 1..n)
  int nent = 0;
  for (int n = 0; n <= p; ++n) nent += (n + 1) * (n + 1) + n * n;
  double acc[kMaxEntPerThread];
#pragma unroll
  for (int i = 0; i < kMaxEntPerThread; ++i) acc[i] = 0.0;
  for (int b0 = 0; b0 < np; b0 += kQuadBatch) {
    const int nb = min(kQuadBatch, np - b0);
    __syncthreads();
    for (int it = tid; it < nb * (p + 1); it += blockDim.x) {
      const int i = it / (p + 1), m = it - i * (p + 1);
      const int pt = b0 + i, kx = pt / nphi, t = pt - kx * nphi;
      const double ct = glx[kx], st = sqrt(fmax(0.0, 1.0 - ct * ct));
      double sp, cp;
      sincospi(2.0 * t / nphi, &sp, &cp);
      const double x = st * cp, y = st * sp, z = ct;
      regular_column(cb * x - sb * z, y, sb * x + cb * z, m, p, Rq + i * nc);  // Q = Ry(-beta)
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kMaxEntPerThread; ++q) {
      const int e = tid + q * kRotBuildThreads;
      if (e >= nent) continue;
      int n = 0, r = e;
      while (r >= (n + 1) * (n + 1) + n * n) {
        r -= (n + 1) * (n + 1) + n * n;
        ++n;
      }
      int part = 0, a, b;
      if (r < (n + 1) * (n + 1)) {
        a = r / (n + 1);
        b = r - a * (n + 1);
      } else {
        part = 1;
        r -= (n + 1) * (n + 1);
        a = 1 + r / n;
        b = 1 + r % n;
      }
      double s = 0.0;
      for (int i = 0; i < nb; ++i) {
        const int pt = b0 + i;
        const double w = glw[pt / nphi];
        const double2 u = Rq[i * nc + cidx(n, a)];
        const double2 v = Rs[(int64_t)pt * nc + cidx(n, b)];
        s = fma(w, part ? u.y * v.y : u.x * v.x, s);
      }
      acc[q] += s;
    }
  }
  // D[n][part][a][b] = (2n+1)/(2 pi) * c_{n,b}^2 * (2 pi / nphi) * sum, c^2 = (n+b)!(n-b)! (/2 at b = 0)
#pragma unroll
  for (int q = 0; q < kMaxEntPerThread; ++q) {
    const int e = tid + q * kRotBuildThreads;
    if (e >= nent) continue;
    int n = 0, r = e;
    while (r >= (n + 1) * (n + 1) + n * n) {
      r -= (n + 1) * (n + 1) + n * n;
      ++n;
    }
    const int b = r < (n + 1) * (n + 1) ? r % (n + 1) : 1 + (r - (n + 1) * (n + 1)) % n;
    double c2 = b == 0 ? 0.5 : 1.0;
    for (int k = 2; k <= n + b; ++k) c2 *= k;
    for (int k = 2; k <= n - b; ++k) c2 *= k;
    Dtab[e] = (2.0 * n + 1.0) / nphi * c2 * acc[q];
  }
  __syncthreads();
  // fragments of every item
  for (int it = 0; it < nitems; ++it) {
    const ItemDev& I = items[it];
    const int MT = I.big ? 2 : 1, KS = I.big ? rot_ksb(p) : 2;
    for (int e = tid; e < MT * KS * 32; e += blockDim.x) {
      const int lane = e & 31, fr = e >> 5, ks = fr % KS, mt = fr / KS;
      const int r = 8 * mt + (lane >> 2), k = 4 * ks + (lane & 3);
      const int sr = r < 16 ? I.slot[r] : -1, sk = k < 16 ? I.slot[k] : -1;
      double v = 0.0;
      if (sr >= 0 && sk >= 0 && (sr & 0xff) == (sk & 0xff)) {
        const int lr = sr >> 8, lk = sk >> 8;
        if (I.st == 1) {  // Z~_m[j][n]: j = m + lr, n = m + lk
          const int m = sr & 0x1f, j = m + lr, n = m + lk;
          double g = 1.0 / rho;  // (j+n)! / rho^{j+n+1}
          for (int l = 1; l <= j + n; ++l) g *= l / rho;
          for (int t = 0; t <= j; ++t) g *= fA;
          for (int t = 0; t < n; ++t) g *= fB;
          v = ((n + m) & 1) ? -g : g;
        } else {
          const int n = sr & 0x1f, part = (sr >> 5) & 1;
          const int mr = part ? lr + 1 : lr, mk = part ? lk + 1 : lk;
          const int a = I.st == 0 ? mr : mk, b = I.st == 0 ? mk : mr;  // stage 2: transposed
          int base = 0;
          for (int q = 0; q < n; ++q) base += (q + 1) * (q + 1) + q * q;
          v = part ? Dtab[base + (n + 1) * (n + 1) + (a - 1) * n + (b - 1)] : Dtab[base + a * (n + 1) + b];
          if (I.st == 2 && part == 0) v *= (mk == 0 ? 1.0 : 2.0) / (mr == 0 ? 1.0 : 2.0);  // E^-1 D^T E
        }
      }
      out[I.aoff + e] = v;
    }
  }
}

// ------------------------------------------------------------------- the mat-vec kernel
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
  int split;                 // CTAs (one cluster) per tile: each takes a contiguous share of the tile's columns
  const int32_t* order;      // [ntiles] launch order of the tiles (decreasing work)
};

template <int P>
struct RGeo {
  static constexpr int NR = (P + 1) * (P + 1);
  static constexpr int KPAD = (NR + 3) & ~3;
  static constexpr int S = rot_xstride(KPAD);  // column stride (see col_base)
  static constexpr int NC = rot_nc(P);
  static constexpr int NT = NC / 8;
  static constexpr int NMMA = kRotMMA, NPREP = 4, NACC = kRotAcc, NNEAR = kRotNear;
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
__device__ __forceinline__ int lds_i32(const int32_t* p) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
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

template <int P, int MT, int KS>
__device__ __forceinline__ void rot_item(const double (&a)[2][RGeo<P>::KSB], const int32_t* pos, int nparts,
                                         double sgn1, int ntiles, double* xc, int lane, int dbg) {
  static_assert(RGeo<P>::NT <= 8, "n-tile dispatch covers up to 8");
  switch (ntiles) {
    case 1: rot_item_nt<P, MT, KS, 1>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    case 2: rot_item_nt<P, MT, KS, 2>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    case 3: rot_item_nt<P, MT, KS, 3>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    case 4: rot_item_nt<P, MT, KS, (RGeo<P>::NT < 4 ? RGeo<P>::NT : 4)>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    case 5: rot_item_nt<P, MT, KS, (RGeo<P>::NT < 5 ? RGeo<P>::NT : 5)>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    case 6: rot_item_nt<P, MT, KS, (RGeo<P>::NT < 6 ? RGeo<P>::NT : 6)>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    case 7: rot_item_nt<P, MT, KS, (RGeo<P>::NT < 7 ? RGeo<P>::NT : 7)>(a, pos, nparts, sgn1, xc, lane, dbg); break;
    default: rot_item_nt<P, MT, KS, RGeo<P>::NT>(a, pos, nparts, sgn1, xc, lane, dbg); break;
  }
}

// A fragments of an item (class data in global memory, L2 resident), fragment order
template <bool GLOBAL>
__device__ __forceinline__ double lda(const double* p) {
  if (GLOBAL) return __ldg(p);
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
template <int P>
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
  const int tile = r.order[blockIdx.x / r.split], h_split = blockIdx.x % r.split;
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
  if (r.split > 1) {  // this CTA's share: chunks whose first column falls in its part of the column range
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
        const int* __restrict__ meta = dsc + 4 + NC;
        const int* __restrict__ ss = dsc + 4 + 2 * NC;
        const int* __restrict__ sb = dsc + 4 + 3 * NC;
        double* __restrict__ acc = m.acc;
        const int2* __restrict__ colt = m.colt + b * NC;
        constexpr int RG = nacc_t / NR > 0 ? nacc_t / NR : 1;  // threads per row (segment ranges)
        for (int t = h; t < RG * NR; t += nacc_t) {
          const int rg = t / NR, row = t - rg * NR;
          const int s_lo = ns * rg / RG, s_hi = ns * (rg + 1) / RG;
          const int d = m.dec[row], part = d & 1, n = (d >> 1) & 0x7f;
          const int mm = (d >> 8) - cidx(n, 0);
          const int rre = d >> 8, rim = mm ? NCOEF + rre - n - 1 : rre;
          const double ca = mm ? ob[2 * mm] : 1.0, sa = mm ? ob[2 * mm + 1] : 0.0;
          // column value = c0 yr + c1 yi: source part = part ^ (take partner), then Az_L,
          // then the sign; idx = mask bits ^ part = (source part) | (negate) << 1
          const uint32_t mask = m.lmask[row];
          // column value = k0 yr + k1 yi: source part = part ^ (take partner), then Az_L,
          // then the sign (idx = mask bits ^ part = source part | negate << 1)
          const double kr0 = ca, ki0 = -sa, kr1 = sa, ki1 = ca;
          for (int sgi = s_lo; sgi < s_hi; ++sgi) {
            const int ce = sb[sgi + 1];
            double* ap = acc + ss[sgi] * NR + row;
            double v = *ap;
            for (int col = sb[sgi]; col < ce; ++col) {
              const int2 cg = colt[col];  // (column base, 2 g)
              const int idx = (int)((mask >> cg.y) & 3) ^ part;
              const double yr = y[cg.x + rre], yi = y[cg.x + rim];
              double k0 = (idx & 1) ? kr1 : kr0, k1 = (idx & 1) ? ki1 : ki0;
              const double t = fma(k0, yr, k1 * yi);
              v = (idx & 2) ? v - t : v + t;
            }
            *ap = v;
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
        constexpr int kPB = 6;               // items per batch
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
  // write back L = L~ / h^{j+1} in complex m >= 0 storage; a split tile first sums the cluster's
  // partial accumulators (distributed shared memory, rank order: deterministic), each CTA a share
  const int e0 = a.T * NR * h_split / r.split, e1 = a.T * NR * (h_split + 1) / r.split;
  if (r.split > 1) cg::this_cluster().sync();
  for (int e = e0 + tid; e < e1; e += nthr) {
    const int slot = e / NR, q = e - slot * NR;
    const int cell = a.tile_cells[tile * a.T + slot];
    if (cell < 0) continue;
    double s = m.acc[e];
    if (r.split > 1) {
      s = 0.0;
      for (int k = 0; k < r.split; ++k) s += cg::this_cluster().map_shared_rank(m.acc, k)[e];
    }
    const int d = m.dec[q];
    const double v = s * a.hpow[a.level[cell] * (a.p + 2) + ((d >> 1) & 0x7f) + 1];
    ((double*)(a.L + (int64_t)cell * a.nc))[2 * (d >> 8) + (d & 1)] = v;
  }
  if (r.split > 1) cg::this_cluster().sync();  // no CTA leaves while its accumulators are read
}

// S9 pre-pass (v3): M~ rows in the RI layout, M~[c][q] = {Re,Im} M_n^m(c) h_c^{-n}, zero for q >= NR.
__global__ void mtilde_ri_kernel(const double2* __restrict__ M, const int32_t* __restrict__ level,
                                 const double* __restrict__ hpow, int64_t ncells, int p, int nc, int NR, int Kpad,
                                 double* __restrict__ Mt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ncells * Kpad) return;
  const int64_t c = e / Kpad;
  const int q = (int)(e - c * Kpad);
  double v = 0.0;
  if (q < NR) {
    const int part = q >= nc;
    const int ci = part ? q - nc + 1 : q;  // Im plane: (n, m >= 1) -> cidx(n, m) = q - nc + n + 1
    int n = 0;
    if (part) {
      while ((n + 1) * n / 2 <= q - nc) ++n;
    } else {
      while ((n + 1) * (n + 2) / 2 <= q) ++n;
    }
    const int cix = part ? ci + n : ci;
    const double2 z = M[c * nc + cix];
    v = (part ? z.y : z.x) * hpow[level[c] * (p + 2) + n];
  }
  Mt[e] = v;
}

// Gauss-Legendre nodes and weights on [-1, 1] (Newton on P_k, host, double)
void gauss_legendre(int k, std::vector<double>& x, std::vector<double>& w) {
  x.assign(k, 0.0);
  w.assign(k, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < k; ++i) {
    double z = std::cos(pi * (i + 0.75) / (k + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int j = 2; j <= k; ++j) {
        const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      if (k == 1) p1 = z, p0 = 1.0;
      dp = k * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-17) break;
    }
    double p0 = 1.0, p1 = z;
    for (int j = 2; j <= k; ++j) {
      const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
      p0 = p1;
      p1 = p2;
    }
    dp = k * (z * p1 - p0) / (z * z - 1.0);
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}


// Per-chunk descriptor (one contiguous 16-byte-aligned record, loaded by one TMA bulk copy):
// [ncol, nseg, class, 0 | srcs[NC] | meta[NC] | sslot[NC] | sbeg[NC + 1]] (sbeg relative to the chunk)
__global__ void chunk_desc_kernel(const int32_t* __restrict__ chunk_begin, const int32_t* __restrict__ chunk_class,
                                  const int32_t* __restrict__ chunk_seg, const int32_t* __restrict__ seg_begin,
                                  const int32_t* __restrict__ col_src, const int32_t* __restrict__ col_meta,
                                  int64_t nchunks, int NC, int32_t* __restrict__ desc) {
  const int64_t ch = blockIdx.x;
  if (ch >= nchunks) return;
  int32_t* d = desc + ch * rot_desc_ints(NC);
  const int cb = chunk_begin[ch], ncol = chunk_begin[ch + 1] - cb;
  const int s0 = chunk_seg[ch], ns = chunk_seg[ch + 1] - s0;
  for (int t = threadIdx.x; t < rot_desc_ints(NC); t += blockDim.x) {
    int v = 0;
    if (t == 0) v = ncol;
    else if (t == 1) v = ns;
    else if (t == 2) v = chunk_class[ch];
    else if (t >= 4 && t < 4 + NC) v = t - 4 < ncol ? col_src[cb + t - 4] : 0;
    else if (t >= 4 + NC && t < 4 + 2 * NC) v = t - 4 - NC < ncol ? col_meta[cb + t - 4 - NC] : 0;
    else if (t >= 4 + 2 * NC && t < 4 + 3 * NC) v = t - 4 - 2 * NC < ns ? (col_meta[seg_begin[s0 + t - 4 - 2 * NC]] & 0xff) : 0;
    else if (t >= 4 + 3 * NC && t <= 4 + 4 * NC) v = t - 4 - 3 * NC <= ns ? seg_begin[s0 + t - 4 - 3 * NC] - cb : 0;
    d[t] = v;
  }
}

// Pack the blocks of every stage into items (first-fit decreasing for the small ones).
std::vector<RotItem> build_items(int p, int& blob_frag) {
  std::vector<RotItem> items;
  int aoff = 2 * (p + 1);
  for (int st = 0; st < 3; ++st) {
    struct Blk {
      int size, code, n0, m0, kind;  // kind 0: D (n, part), 1: Z (m)
    };
    std::vector<Blk> blks;
    if (st == 1) {
      for (int m = 0; m <= p; ++m) blks.push_back({p + 1 - m, m, 0, m, 1});
    } else {
      for (int n = 0; n <= p; ++n) {
        blks.push_back({n + 1, n, n, 0, 0});
        if (n > 0) blks.push_back({n, n | (1 << 5), n, 1, 0});
      }
    }
    std::stable_sort(blks.begin(), blks.end(), [](const Blk& x, const Blk& y) { return x.size > y.size; });
    std::vector<RotItem> bins;
    std::vector<int> fill;
    for (const Blk& bk : blks) {
      int target = -1;
      if (bk.size <= 8)
        for (size_t i = 0; i < bins.size(); ++i)
          if (!bins[i].big && fill[i] + bk.size <= 8) {
            target = (int)i;
            break;
          }
      if (target < 0) {
        RotItem it{};
        it.st = st;
        it.big = bk.size > 8;
        it.nparts = st == 1 ? 2 : 1;
        for (int s = 0; s < 16; ++s) it.slot[s] = -1, it.pos[0][s] = it.pos[1][s] = -1;
        bins.push_back(it);
        fill.push_back(0);
        target = (int)bins.size() - 1;
      }
      RotItem& it = bins[target];
      for (int l = 0; l < bk.size; ++l) {
        const int s = fill[target] + l;
        it.slot[s] = bk.code | (l << 8);
        if (st == 1) {  // order m, degree n = m + l
          it.pos[0][s] = ri_pos(p, bk.m0 + l, bk.m0, 0);
          it.pos[1][s] = bk.m0 > 0 ? ri_pos(p, bk.m0 + l, bk.m0, 1) : -1;
        } else {  // degree n, order m = l (+1 for Im)
          const int part = (bk.code >> 5) & 1;
          it.pos[0][s] = ri_pos(p, bk.n0, l + part, part);
        }
      }
      fill[target] += bk.size;
    }
    for (RotItem& it : bins) {
      it.aoff = aoff;
      aoff += (it.big ? 2 * rot_ksb(p) : 2) * 32;
      items.push_back(it);
    }
  }
  blob_frag = (aoff + 1) & ~1;
  return items;
}

}  // namespace

bool m2l_rot_supported(int p) { return p >= 0 && p <= 14; }
int rot_chunk_width(int p) { return rot_nc(p); }
size_t rot_smem_bytes(int p, int T, int extra_ints) {
  const int NR = (p + 1) * (p + 1), KPAD = (NR + 3) & ~3, S = rot_xstride(KPAD), nc = ncoef(p), NC = rot_nc(p);
  int blob = 0;
  std::vector<RotItem> items = build_items(p, blob);
  const int ni = (int)items.size();
  return sizeof(double) * ((size_t)T * NR + 2 * (size_t)NC * S + (rot_smem_a(p) ? 2 * (size_t)blob : 4 * (size_t)(p + 1))) +
         sizeof(uint64_t) * 6 +
         sizeof(int32_t) * (3 * rot_desc_ints(NC) + 3 * NR + nc + 4 + 4 * NC + ni + 32 * ni + 6 * kRotMMA * extra_ints);
}

void m2l_rot_setup(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  cudaStream_t s = P.stream;
  const int p = P.p;
  if (D.nclass == 0 || D.ntiles == 0) return;
  int blob = 0;
  std::vector<RotItem> items = build_items(p, blob);
  const int ni = (int)items.size();
  // quadrature (exact to degree 2p on the sphere)
  std::vector<double> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  DevBuf<double> dgx, dgw;
  DevBuf<double2> Rs;
  dgx.alloc(p + 1);
  dgw.alloc(p + 1);
  FMM_CUDA(cudaMemcpyAsync(dgx.ptr, gx.data(), sizeof(double) * (p + 1), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemcpyAsync(dgw.ptr, gw.data(), sizeof(double) * (p + 1), cudaMemcpyHostToDevice, s));
  const int np = (p + 1) * (2 * p + 1);
  Rs.alloc((int64_t)np * ncoef(p));
  quad_points_kernel<<<cdiv(np * (p + 1), 128), 128, 0, s>>>(dgx, p, Rs);
  FMM_LAUNCHED("quad_points_kernel");
  D.rot_blob = blob;
  D.rot_ops.alloc(D.nclass * blob);
  {  // symmetry masks from the signed-permutation tables (m2l_dmma.cu), rows in RI order
    const int NR = (p + 1) * (p + 1);
    std::vector<int32_t> sym = build_symtab(p);
    std::vector<uint32_t> mk(2 * NR, 0);
    for (int which = 0; which < 2; ++which)
      for (int q = 0; q < NR; ++q) {
        int n, mm, part;
        ri_decode(p, q, n, mm, part);
        const int rr = real_index(n, mm, part);
        for (int g = 0; g < 16; ++g) {
          const int ent = sym[(g * 2 + which) * NR + rr];
          if ((ent & 0xffff) != rr) mk[which * NR + q] |= 1u << (2 * g);
          if (ent >> 16) mk[which * NR + q] |= 2u << (2 * g);
        }
      }
    D.rot_masks.alloc(2 * NR);
    FMM_CUDA(cudaMemcpyAsync(D.rot_masks.ptr, mk.data(), sizeof(uint32_t) * mk.size(), cudaMemcpyHostToDevice, s));
  }
  // item tables: device copy for the build kernel, headers and positions for the mat-vec
  std::vector<ItemDev> idev(ni);
  std::vector<int32_t> hdr(ni), pos(32 * ni);
  for (int i = 0; i < ni; ++i) {
    idev[i].st = items[i].st;
    idev[i].big = items[i].big;
    idev[i].nparts = items[i].nparts;
    idev[i].aoff = items[i].aoff;
    for (int k = 0; k < 16; ++k) idev[i].slot[k] = items[i].slot[k];
    hdr[i] = items[i].big | (items[i].nparts << 1) | (items[i].aoff << 8);
    for (int k = 0; k < 16; ++k) {
      pos[32 * i + k] = items[i].pos[0][k];
      pos[32 * i + 16 + k] = items[i].pos[1][k];
    }
  }
  DevBuf<ItemDev> ditems;
  ditems.alloc(ni);
  FMM_CUDA(cudaMemcpyAsync(ditems.ptr, idev.data(), sizeof(ItemDev) * ni, cudaMemcpyHostToDevice, s));
  D.rot_ihdr.alloc(ni);
  D.rot_ipos.alloc(32 * ni);
  FMM_CUDA(cudaMemcpyAsync(D.rot_ihdr.ptr, hdr.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemcpyAsync(D.rot_ipos.ptr, pos.data(), sizeof(int32_t) * 32 * ni, cudaMemcpyHostToDevice, s));
  D.rot_nitems = ni;
  int nent = 0;
  for (int n = 0; n <= p; ++n) nent += (n + 1) * (n + 1) + n * n;
  const size_t sh = sizeof(double2) * kQuadBatch * ncoef(p) + sizeof(double) * nent;
  static size_t configured = 0;
  if (sh > 48 * 1024 && sh > configured) {
    FMM_CUDA(cudaFuncSetAttribute(build_rot_ops_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    configured = sh;
  }
  build_rot_ops_kernel<<<(unsigned)D.nclass, kRotBuildThreads, sh, s>>>(D.class_keys, p, dgx, dgw, Rs, ditems, ni,
                                                                         blob, D.rot_ops);
  FMM_LAUNCHED("build_rot_ops_kernel");
  // static LPT schedule of each stage's items over the MMA warps
  const int nmma = kRotMMA;
  std::vector<std::vector<int>> lists(3 * nmma);
  for (int st = 0; st < 3; ++st) {
    std::vector<std::pair<int, int>> its;  // (cost, id)
    for (int i = 0; i < ni; ++i)
      if (items[i].st == st)
        its.push_back({(items[i].big ? 2 * rot_ksb(p) : 2) * items[i].nparts * 8 + 24 * items[i].nparts, i});
    std::stable_sort(its.begin(), its.end(), [](auto& x, auto& y) { return x.first > y.first; });
    std::vector<int> load(nmma, 0);
    for (auto& it : its) {
      const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[w] += it.first;
      lists[st * nmma + w].push_back(it.second);
    }
  }
  int smax = 1;
  for (auto& l : lists) smax = std::max<int>(smax, (int)l.size() + 1);
  std::vector<int32_t> sched(3 * nmma * smax, -1);
  for (int i = 0; i < 3 * nmma; ++i)
    for (size_t k = 0; k < lists[i].size(); ++k) sched[i * smax + k] = lists[i][k];
  D.rot_smax = smax;
  D.rot_sched.alloc((int64_t)sched.size());
  FMM_CUDA(cudaMemcpyAsync(D.rot_sched.ptr, sched.data(), sizeof(int32_t) * sched.size(), cudaMemcpyHostToDevice, s));
  D.rot_T = D.T;
  D.rot_desc.alloc(D.nchunks * rot_desc_ints(D.NC));
  chunk_desc_kernel<<<(unsigned)D.nchunks, 128, 0, s>>>(D.chunk_begin, D.chunk_class, D.chunk_seg, D.seg_begin,
                                                         D.col_src, D.col_meta, D.nchunks, D.NC, D.rot_desc);
  FMM_LAUNCHED("chunk_desc_kernel");
  {  // launch order of the tiles: decreasing estimated work (per chunk: fixed cost + its n-tiles), so the
     // hardware's in-order CTA dispatch balances the last waves like an LPT schedule
    std::vector<int32_t> tc(D.ntiles + 1), cb(D.nchunks + 1);
    FMM_CUDA(cudaMemcpyAsync(tc.data(), D.tile_chunk.ptr, sizeof(int32_t) * tc.size(), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(cb.data(), D.chunk_begin.ptr, sizeof(int32_t) * cb.size(), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    std::vector<std::pair<int64_t, int32_t>> w(D.ntiles);
    for (int64_t t = 0; t < D.ntiles; ++t) {
      int64_t c = 0;
      for (int32_t ch = tc[t]; ch < tc[t + 1]; ++ch) c += 3 + (cb[ch + 1] - cb[ch] + 7) / 8;
      w[t] = {-c, (int32_t)t};
    }
    std::sort(w.begin(), w.end());
    std::vector<int32_t> order(D.ntiles);
    for (int64_t t = 0; t < D.ntiles; ++t) order[t] = w[t].second;
    D.rot_order.alloc(D.ntiles);
    FMM_CUDA(cudaMemcpyAsync(D.rot_order.ptr, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice, s));
  }
  FMM_CUDA(cudaStreamSynchronize(s));
}

void m2l_rot_mtilde(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  const int64_t ne = P.cells.n * D.Kpad;
  mtilde_ri_kernel<<<cdiv(ne, 256), 256, 0, P.stream>>>(P.M, P.cells.level, D.hpow, P.cells.n, P.p, P.nc, D.NR, D.Kpad,
                                                        D.Mt);
  FMM_LAUNCHED("mtilde_ri_kernel");
}

void m2l_rot_launch(fmm_plan_s& P, const m2l::M2LArgs& a) {
  M2LDmma& D = P.m2l_dmma;
  RotArgs r;
  r.a = a;
  r.blobs = D.rot_ops;
  r.masks = D.rot_masks;
  r.sched = D.rot_sched;
  r.ihdr = D.rot_ihdr;
  r.ipos = D.rot_ipos;
  r.smax = D.rot_smax;
  r.nitems = D.rot_nitems;
  r.blob = D.rot_blob;
  r.desc = D.rot_desc;
  r.order = D.rot_order;
  r.p2p_phi = nullptr;
  r.p2p_grad = nullptr;
  if (P.near_fused_active) {
    r.leaves = P.leaves.ptr + P.own_leaf_begin;
    r.nleaves = P.own_leaf_end - P.own_leaf_begin;
    r.cbeg = P.cells.begin;
    r.cend = P.cells.end;
    r.p2p_off = P.p2p.off;
    r.p2p_src = P.p2p.src;
    r.pos = P.pos;
    r.leaf_counter = P.near_counter;
    r.p2p_phi = P.near_p2p_phi;
    r.p2p_grad = P.near_fused_grad ? P.near_p2p_grad.ptr : nullptr;
  }
  const char* dbgs = getenv("FMM_M2L_DEBUG");  // timing experiments only (most bits skip work: wrong results)
  const int dbg = dbgs ? atoi(dbgs) : 0;
  r.prof = nullptr;
  static DevBuf<unsigned long long> prof_buf;
  if (dbg & 256) {  // timing experiment: per-warp cycle breakdown printed to stderr after the launch
    if (!prof_buf.ptr) prof_buf.alloc(8 * 32);
    FMM_CUDA(cudaMemsetAsync(prof_buf.ptr, 0, 8 * 32 * sizeof(unsigned long long), P.stream));
    r.prof = prof_buf.ptr;
  }
  const size_t sh = rot_smem_bytes(P.p, a.T, D.rot_smax);
  void (*k)(const RotArgs, int) = nullptr;
  switch (P.p) {
    case 0: k = m2l_rot_kernel<0>; break;
    case 1: k = m2l_rot_kernel<1>; break;
    case 2: k = m2l_rot_kernel<2>; break;
    case 3: k = m2l_rot_kernel<3>; break;
    case 4: k = m2l_rot_kernel<4>; break;
    case 5: k = m2l_rot_kernel<5>; break;
    case 6: k = m2l_rot_kernel<6>; break;
    case 7: k = m2l_rot_kernel<7>; break;
    case 8: k = m2l_rot_kernel<8>; break;
    case 9: k = m2l_rot_kernel<9>; break;
    case 10: k = m2l_rot_kernel<10>; break;
    case 11: k = m2l_rot_kernel<11>; break;
    case 12: k = m2l_rot_kernel<12>; break;
    case 13: k = m2l_rot_kernel<13>; break;
    default: k = m2l_rot_kernel<14>; break;
  }
  static size_t configured[17] = {0};
  if (sh > 48 * 1024 && sh > configured[P.p]) {
    FMM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    configured[P.p] = sh;
  }
  // split small problems over clusters of CTAs so that the grid covers the SMs (configs[1]: 73 tiles)
  // (one CTA per SM: minimise waves / split, ties to the smaller split; configs[1] -> 2, [2] -> 1)
  int nsm = 148;
  FMM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P.device));
  int split = 1;
  double best = 1e300;
  for (int s = 1; s <= 4; s *= 2) {
    const double cost = (double)((D.ntiles * s + nsm - 1) / nsm) / s;
    if (cost < best - 1e-9) best = cost, split = s;
  }
  if (const char* s = getenv("FMM_M2L_SPLIT")) split = std::max(1, std::min(8, atoi(s)));
  r.split = split;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(D.ntiles * split));
  cfg.blockDim = dim3(32 * (kRotMMA + 4 + kRotAcc + kRotNear));
  cfg.dynamicSmemBytes = sh;
  cfg.stream = P.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = split;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FMM_CUDA(cudaLaunchKernelEx(&cfg, k, r, dbg));
  FMM_LAUNCHED("m2l_rot_kernel");
  if (dbg & 256) {
    unsigned long long h[8 * 32];
    FMM_CUDA(cudaMemcpyAsync(h, prof_buf.ptr, sizeof(h), cudaMemcpyDeviceToHost, P.stream));
    FMM_CUDA(cudaStreamSynchronize(P.stream));
    for (int w = 0; w < kRotMMA; ++w)
      fprintf(stderr, "m2l_rot prof warp %2d: waitX %.0f  st0 %.0f  st1 %.0f  st2 %.0f  barrier %.0f  (cycles per chunk)\n",
              w, (double)h[8 * w] / h[8 * w + 5], (double)h[8 * w + 1] / h[8 * w + 5], (double)h[8 * w + 2] / h[8 * w + 5],
              (double)h[8 * w + 3] / h[8 * w + 5], (double)h[8 * w + 4] / h[8 * w + 5]);
  }
}

}  // namespace fmm
