// m2l_rot.cu — S9 M2L v3 (default for p = 5..14): the translation-invariant class
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
// Kernel (one CTA per tile of T target cells, as v2): warp-specialised.
//  * helper warps: load chunk i+1's metadata, stage its source multipoles M~_B (contiguous
//    rows of Kpad doubles) into shared memory with cp.async.bulk (TMA bulk copies, one per
//    column, completion on an mbarrier), apply the column's symmetry map and Az_M in place,
//    signal the MMA warps; then add chunk i's result (Az_L and the symmetry map applied on
//    the fly) into the tile's shared-memory accumulators (deterministic column order);
//  * MMA warps: the three block-GEMM stages D, Z~, Dt on DMMA (mma.sync m8n8k4 f64), each
//    IN PLACE in the chunk's shared-memory buffer: an item = (block, part, half of the
//    columns) reads and writes only its own positions (all B fragments are loaded into
//    registers before the first store), a named barrier separates the stages; operator
//    A fragments are streamed from L2; items are spread over the warps by a static LPT
//    schedule built on the host.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "harmonics.cuh"
#include "m2l_common.cuh"
#include "plan.h"

namespace fmm {
namespace m2l {

// --------------------------------------------------------------------- operator layout
__host__ __device__ inline int frag_count(int R, int K) { return ((R + 7) / 8) * ((K + 3) / 4) * 32; }
// rows (= K) of block blk in stage st: stages 0/2 (rotations) degree n = blk -> n + 1;
// stage 1 (z translation) order m = blk -> p + 1 - m
__host__ __device__ inline int rot_block_rows(int p, int st, int blk) { return st == 1 ? p + 1 - blk : blk + 1; }
__host__ __device__ inline int rot_block_parts(int st, int blk) { return st == 1 ? 1 : (blk > 0 ? 2 : 1); }
// offset (doubles) of (st, blk, part) inside one class's operator set; total at (3, 0, 0)
__host__ __device__ inline int rot_block_offset(int p, int st, int blk, int part) {
  int off = 0;
  for (int s = 0; s < 3; ++s)
    for (int b = 0; b <= p; ++b)
      for (int pt = 0; pt < rot_block_parts(s, b); ++pt) {
        if (s == st && b == blk && pt == part) return off;
        const int R = rot_block_rows(p, s, b);
        off += frag_count(R, R);
      }
  return off;
}
__host__ __device__ inline int rot_ops_size(int p) { return rot_block_offset(p, 3, 0, 0); }

// position (real index) of row/column index r of block (st, blk, part); -1 = none (zero)
__host__ __device__ inline int rot_pos(int p, int st, int blk, int part, int r) {
  if (st == 1) {  // order m = blk, degree n = m + r
    if (r > p - blk) return -1;
    return real_index(blk + r, blk, part);
  }
  if (r > blk || (part == 1 && r == 0)) return -1;  // degree n = blk, order m = r
  return real_index(blk, r, part);
}

}  // namespace m2l

namespace {
using namespace m2l;

// ------------------------------------------------------------------- setup: operators
// Regular harmonics at the quadrature points s_i (shared by every class).
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

// One CTA per class: azimuth table, rotation blocks by quadrature, fragments of the three
// stages in DMMA A-fragment order (A[8 mt + lane/4][4 ks + lane%4]).
__global__ void __launch_bounds__(kRotBuildThreads) build_rot_ops_kernel(
    const uint64_t* __restrict__ class_keys, int p, const double* __restrict__ glx, const double* __restrict__ glw,
    const double2* __restrict__ Rs, double* __restrict__ ops, double2* __restrict__ az) {
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
  if (tid <= p) {
    double s, c;
    sincos(tid * alpha, &s, &c);
    az[(int64_t)cls * (p + 1) + tid] = make_double2(c, s);
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
  // fragments
  double* out = ops + (int64_t)cls * rot_ops_size(p);
  for (int st = 0; st < 3; ++st)
    for (int blk = 0; blk <= p; ++blk)
      for (int part = 0; part < rot_block_parts(st, blk); ++part) {
        const int R = rot_block_rows(p, st, blk), KS = (R + 3) / 4, MT = (R + 7) / 8;
        double* o = out + rot_block_offset(p, st, blk, part);
        int base = 0;  // start of degree blk in Dtab
        for (int n = 0; n < blk; ++n) base += (n + 1) * (n + 1) + n * n;
        for (int e = tid; e < MT * KS * 32; e += blockDim.x) {
          const int lane = e & 31, fr = e >> 5, ks = fr % KS, mt = fr / KS;
          const int r = 8 * mt + (lane >> 2), k = 4 * ks + (lane & 3);
          double v = 0.0;
          if (r < R && k < R) {
            if (st == 1) {  // Z~_m[i][k]: j = m + i, n = m + k
              const int m = blk, j = m + r, n = m + k;
              double g = 1.0 / rho;  // (j+n)! / rho^{j+n+1}
              for (int l = 1; l <= j + n; ++l) g *= l / rho;
              for (int t = 0; t <= j; ++t) g *= fA;
              for (int t = 0; t < n; ++t) g *= fB;
              v = ((n + m) & 1) ? -g : g;
            } else {
              const int n = blk;
              int rr = st == 0 ? r : k, kk = st == 0 ? k : r;  // stage 2: transpose
              if (part == 0) {
                v = Dtab[base + rr * (n + 1) + kk];
                if (st == 2) v *= (rr == 0 ? 1.0 : 2.0) / (kk == 0 ? 1.0 : 2.0);  // (E^-1 D^T E)[r][k] = D[k][r] E_k / E_r
              } else if (rr > 0 && kk > 0) {
                v = Dtab[base + (n + 1) * (n + 1) + (rr - 1) * n + (kk - 1)];
              }
            }
          }
          o[e] = v;
        }
      }
}

// ------------------------------------------------------------------- the mat-vec kernel
struct RotArgs {
  M2LArgs a;
  const double* rops;    // [nclass][rot_ops_size(p)]
  const double2* raz;    // [nclass][p + 1]
  const int32_t* sched;  // [3][nmma][smax] items (-1 = end)
  int smax, S;
};

constexpr int rot_xstride(int kpad) {
  int s = kpad + 1;
  while (s % 16 != 4) ++s;
  return s;
}
template <int P>
struct RGeo {
  static constexpr int NR = (P + 1) * (P + 1);
  static constexpr int KPAD = (NR + 3) & ~3;
  static constexpr int S = rot_xstride(KPAD);  // column stride; position KPAD is the zero slot
  static constexpr int ZERO = KPAD;
  static constexpr int NC = 2 * S * 64 * 8 > 140 * 1024 ? 32 : 64;  // as v2's chunk width rule
  static constexpr int NMMA = 8;
  static constexpr int MTMAX = (P + 1 + 7) / 8;
  static constexpr int KSMAX = (P + 1 + 3) / 4;
  static constexpr int NCOEF = (P + 1) * (P + 2) / 2;
};

struct RotSmem {
  double *acc, *x0, *x1;
  double2* azs;  // [2][P+1]
  int32_t *meta, *srcs, *sslot, *sbeg, *sym, *dec, *lmask, *lpoff, *pairtab, *sched, *ccls, *blkoff;
  uint64_t* bar;  // [2]
};
template <int P>
__device__ __forceinline__ RotSmem rot_carve(double* sm, const RotArgs& r) {
  using G = RGeo<P>;
  RotSmem m;
  m.acc = sm;
  m.x0 = m.acc + (size_t)r.a.T * G::NR;
  m.x1 = m.x0 + G::NC * G::S;
  m.azs = (double2*)(m.x1 + G::NC * G::S);
  uint64_t* b = (uint64_t*)(m.azs + 2 * (P + 1));
  m.bar = b;
  m.meta = (int32_t*)(b + 2);
  m.srcs = m.meta + 2 * G::NC;
  m.sslot = m.srcs + 2 * G::NC;
  m.sbeg = m.sslot + 2 * G::NC;
  m.sym = m.sbeg + 2 * (G::NC + 1);
  m.dec = m.sym + 32 * G::NR;
  m.lmask = m.dec + G::NR;
  m.lpoff = m.lmask + G::NR;
  m.pairtab = m.lpoff + G::NR;
  m.ccls = m.pairtab + G::NCOEF;
  m.sched = m.ccls + 2;
  m.blkoff = m.sched + 3 * G::NMMA * r.smax;  // [3][P+1][2]
  return m;
}
}  // namespace
size_t rot_smem_bytes(int p, int T, int smax) {
  const int NR = (p + 1) * (p + 1), KPAD = (NR + 3) & ~3, S = rot_xstride(KPAD), nc = ncoef(p);
  const int NC = 2 * S * 64 * 8 > 140 * 1024 ? 32 : 64;
  return sizeof(double) * ((size_t)T * NR + 2 * NC * (size_t)S) + sizeof(double2) * 2 * (p + 1) +
         sizeof(uint64_t) * 2 + sizeof(int32_t) * (8 * NC + 2 + 35 * NR + nc + 2 + 3 * 8 * smax + 6 * (p + 1));
}
int rot_chunk_width(int p) {
  const int NR = (p + 1) * (p + 1), KPAD = (NR + 3) & ~3, S = rot_xstride(KPAD);
  return 2 * S * 64 * 8 > 140 * 1024 ? 32 : 64;
}
namespace {

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

// One MMA item: block (st, blk), part(s), n-tiles cg, cg + 2, ... of the chunk; in place.
template <int P>
__device__ __forceinline__ void rot_item(const double* __restrict__ ops, const int32_t* blkoff, int st, int blk,
                                         int part, int cg, int ntiles, double* xc, int lane) {
  using G = RGeo<P>;
  const int R = rot_block_rows(P, st, blk), MT = (R + 7) / 8, KS = (R + 3) / 4;
  const int np = st == 1 ? (blk > 0 ? 2 : 1) : 1;  // stage 1: Re and Im with the same operator
  const double* A = ops + blkoff[(st * (P + 1) + blk) * 2 + (st == 1 ? 0 : part)] + lane;
  double a[G::MTMAX][G::KSMAX];
#pragma unroll
  for (int mt = 0; mt < G::MTMAX; ++mt)
#pragma unroll
    for (int ks = 0; ks < G::KSMAX; ++ks) a[mt][ks] = (mt < MT && ks < KS) ? __ldg(A + (mt * KS + ks) * 32) : 0.0;
  const int colb = lane >> 2, kl = lane & 3;
  for (int pp = 0; pp < np; ++pp) {
    const int pt = st == 1 ? pp : part;
    double b[G::KSMAX][4];
#pragma unroll
    for (int ks = 0; ks < G::KSMAX; ++ks) {
      int pos = ks < KS ? rot_pos(P, st, blk, pt, 4 * ks + kl) : -1;
      if (pos < 0) pos = G::ZERO;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int nt = cg + 2 * t;
        b[ks][t] = (nt < ntiles && ks < KS) ? xc[(8 * nt + colb) * G::S + pos] : 0.0;
      }
    }
    double c[G::MTMAX][4][2];
#pragma unroll
    for (int mt = 0; mt < G::MTMAX; ++mt)
#pragma unroll
      for (int t = 0; t < 4; ++t) c[mt][t][0] = c[mt][t][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < G::KSMAX; ++ks)
      if (ks < KS)
#pragma unroll
        for (int mt = 0; mt < G::MTMAX; ++mt)
          if (mt < MT)
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (cg + 2 * t < ntiles) dmma884(c[mt][t][0], c[mt][t][1], a[mt][ks], b[ks][t]);
    __syncwarp();  // every lane's B loads precede the in-place stores
    const double sgn = (st == 1 && pt == 1) ? -1.0 : 1.0;
#pragma unroll
    for (int mt = 0; mt < G::MTMAX; ++mt) {
      const int r = 8 * mt + (lane >> 2);
      const int pos = (mt < MT && r < R) ? rot_pos(P, st, blk, pt, r) : -1;
      if (pos < 0) continue;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int nt = cg + 2 * t;
        if (nt < ntiles) {
          const int col = 8 * nt + 2 * kl;
          xc[col * G::S + pos] = sgn * c[mt][t][0];
          xc[(col + 1) * G::S + pos] = sgn * c[mt][t][1];
        }
      }
    }
    __syncwarp();
  }
}

template <int P>
__global__ void __launch_bounds__(512, 1) m2l_rot_kernel(const RotArgs r, int nhelp) {
  using G = RGeo<P>;
  constexpr int NR = G::NR, NC = G::NC, S = G::S, NCOEF = G::NCOEF;
  extern __shared__ double sm[];
  const RotSmem m = rot_carve<P>(sm, r);
  const M2LArgs& a = r.a;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  constexpr int nmma_t = 32 * G::NMMA;
  const int nhelp_t = 32 * nhelp, nall = nmma_t + nhelp_t;
  // ---- shared tables
  for (int e = tid; e < a.T * NR; e += nthr) m.acc[e] = 0.0;
  for (int e = tid; e < 32 * NR; e += nthr) m.sym[e] = a.symtab[e];
  for (int q = tid; q < NCOEF; q += nthr) {
    int n = 0;
    while (cidx(n + 1, 0) <= q) ++n;
    m.pairtab[q] = (n * n) | ((q - cidx(n, 0)) << 16);
  }
  for (int e = tid; e < 3 * G::NMMA * r.smax; e += nthr) m.sched[e] = r.sched[e];
  for (int e = tid; e < 6 * (P + 1); e += nthr) {
    const int st = e / (2 * (P + 1)), blk = (e / 2) % (P + 1), pt = e & 1;
    m.blkoff[e] = pt < rot_block_parts(st, blk) ? rot_block_offset(P, st, blk, pt) : 0;
  }
  for (int e = tid; e < 2 * NC; e += nthr) {  // zero slots and padding rows of both buffers
    double* xb = (e < NC ? m.x0 : m.x1) + (e % NC) * S;
    for (int k = G::KPAD; k < S; ++k) xb[k] = 0.0;
  }
  for (int q = tid; q < NR; q += nthr) {
    int n, mm, part;
    real_decode(q, n, mm, part);
    m.dec[q] = (cidx(n, mm) << 8) | (n << 1) | part;
  }
  if (tid == 0) {
    mbar_init(m.bar, 1);
    mbar_init(m.bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int q = tid; q < NR; q += nthr) {
    int poff = 0;
    m.lmask[q] = (int32_t)ltrans_mask(m.sym, NR, q, poff);
    m.lpoff[q] = poff;
  }
  const int c_first = a.tile_chunk[tile], c_last = a.tile_chunk[tile + 1];
  __syncthreads();
  if (warp >= G::NMMA) {
    // ================= helper warps
    const int h = tid - nmma_t;
    // stage chunk ch into buffer b: metadata, class azimuths, TMA bulk copies, symmetry + Az_M
    auto prep = [&](int ch, int b, unsigned parity) {
      double* xb = b ? m.x1 : m.x0;
      load_meta_dev(a, ch, m.meta + b * NC, m.srcs + b * NC, m.sslot + b * NC, m.sbeg + b * (NC + 1), h, nhelp_t);
      const int cls = a.chunk_class[ch];
      if (h <= P) m.azs[b * (P + 1) + h] = r.raz[(int64_t)cls * (P + 1) + h];
      const int ncol = a.chunk_begin[ch + 1] - a.chunk_begin[ch];
      named_sync(6, nhelp_t);  // metadata visible to all helpers
      if (h < 32) {
        fence_proxy_async();  // earlier generic accesses of xb before the async-proxy writes
        if (h == 0) mbar_arrive_tx(m.bar + b, (unsigned)(ncol * G::KPAD * sizeof(double)));
        __syncwarp();
        for (int c = h; c < ncol; c += 32)
          bulk_g2s(xb + c * S, a.Mt + (int64_t)m.srcs[b * NC + c] * G::KPAD, G::KPAD * sizeof(double), m.bar + b);
      }
      // padding columns of the last n-tile: zeros
      const int ncol8 = (ncol + 7) & ~7;
      for (int e = h; e < (ncol8 - ncol) * G::KPAD; e += nhelp_t) xb[(ncol + e / G::KPAD) * S + e % G::KPAD] = 0.0;
      mbar_wait(m.bar + b, parity);
      // X[col] <- Az_M (D^M_g)^-1 X[col], item = (column, (n, m) pair)
      const double2* azb = m.azs + b * (P + 1);
      for (int it = h; it < ncol * NCOEF; it += nhelp_t) {
        const int col = it / NCOEF, q = it - col * NCOEF;
        const int pe = m.pairtab[q], n2 = pe & 0xffff, mm = pe >> 16;
        const int32_t* sy = m.sym + (m.meta[b * NC + col] >> 8) * 2 * NR;
        double* xcol = xb + col * S;
        if (mm == 0) {
          const int ent = sy[n2];
          const double v = xcol[ent & 0xffff];
          xcol[n2] = (ent >> 16) ? -v : v;
        } else {
          const int rre = n2 + 2 * mm - 1, rim = rre + 1;
          const int e0 = sy[rre], e1 = sy[rim];
          double u0 = xcol[e0 & 0xffff], u1 = xcol[e1 & 0xffff];
          u0 = (e0 >> 16) ? -u0 : u0;
          u1 = (e1 >> 16) ? -u1 : u1;
          const double2 cs = azb[mm];
          xcol[rre] = cs.x * u0 - cs.y * u1;
          xcol[rim] = cs.y * u0 + cs.x * u1;
        }
      }
    };
    // add chunk ch (buffer b) into the accumulators: acc[slot][r] += (D^L_g Az_L Y)[r]
    auto accumulate = [&](int ch, int b) {
      const double* y = b ? m.x1 : m.x0;
      const int ns = a.chunk_seg[ch + 1] - a.chunk_seg[ch];
      const int* meta = m.meta + b * NC;
      const int* sb = m.sbeg + b * (NC + 1);
      const int* ss = m.sslot + b * NC;
      const double2* azb = m.azs + b * (P + 1);
      const int RG = max(1, nhelp_t / NR);
      for (int t = h; t < RG * NR; t += nhelp_t) {
        const int rg = t / NR, row = t - rg * NR;
        const int d = m.dec[row], part = d & 1, n = (d >> 1) & 0x7f;
        const int mm = (d >> 8) - cidx(n, 0);
        const int rre = real_index(n, mm, 0), rim = mm ? rre + 1 : rre;
        const double2 cs = mm ? azb[mm] : make_double2(1.0, 0.0);
        const uint32_t mask = (uint32_t)m.lmask[row];
        // value for (take partner, negate) combinations: src part = part ^ partner
        const double ca = cs.x, sa = cs.y;
        const int s_lo = ns * rg / RG, s_hi = ns * (rg + 1) / RG;
        for (int sgi = s_lo; sgi < s_hi; ++sgi) {
          double* ap = m.acc + ss[sgi] * NR + row;
          double v = *ap;
          for (int col = sb[sgi]; col < sb[sgi + 1]; ++col) {
            const uint32_t mg = mask >> (2 * (meta[col] >> 8));
            const double yr = y[col * S + rre], yi = y[col * S + rim];
            const int src = part ^ (int)(mg & 1);
            double t0 = src == 0 ? fma(-sa, yi, ca * yr) : fma(ca, yi, sa * yr);
            if (mm == 0) t0 = yr;
            v += (mg & 2) ? -t0 : t0;
          }
          *ap = v;
        }
      }
    };
    if (c_first < c_last) {
      prep(c_first, 0, 0);
      named_arrive(1, nall);  // Xfull(0)
    }
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1, nb = b ^ 1;
      if (ch + 1 < c_last) {
        prep(ch + 1, nb, (unsigned)(((i + 1) >> 1) & 1));
        named_arrive(1 + nb, nall);  // Xfull(i+1)
      }
      named_sync(3 + b, nall);  // Yfull(i)
      accumulate(ch, b);
      named_sync(6, nhelp_t);  // helpers done with meta[b] / Y(i) before they are overwritten
    }
  } else {
    // ================= MMA warps
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      named_sync(1 + b, nall);  // Xfull(i)
      double* xc = b ? m.x1 : m.x0;
      const int cls = a.chunk_class[ch];
      const int ntiles = (a.chunk_begin[ch + 1] - a.chunk_begin[ch] + 7) >> 3;
      const double* ops = r.rops + (int64_t)cls * rot_ops_size(P);
      for (int st = 0; st < 3; ++st) {
        const int32_t* sl = m.sched + (st * G::NMMA + warp) * r.smax;
        for (int k = 0; k < r.smax; ++k) {
          const int item = sl[k];
          if (item < 0) break;
          rot_item<P>(ops, m.blkoff, st, item & 0x1f, (item >> 5) & 1, (item >> 6) & 1, ntiles, xc, lane);
        }
        if (st < 2) named_sync(5, nmma_t);  // stage st complete before st + 1 reads it
      }
      named_arrive(3 + b, nall);  // Yfull(i)
    }
  }
  __syncthreads();
  // write back L = L~ / h^{j+1} in complex m >= 0 storage
  for (int e = tid; e < a.T * NR; e += nthr) {
    const int slot = e / NR, q = e - slot * NR;
    const int cell = a.tile_cells[tile * a.T + slot];
    if (cell < 0) continue;
    const int d = m.dec[q];
    const double v = m.acc[e] * a.hpow[a.level[cell] * (a.p + 2) + ((d >> 1) & 0x7f) + 1];
    ((double*)(a.L + (int64_t)cell * a.nc))[2 * (d >> 8) + (d & 1)] = v;
  }
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

}  // namespace

bool m2l_rot_supported(int p) { return p >= 5 && p <= 14; }

void m2l_rot_setup(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  cudaStream_t s = P.stream;
  const int p = P.p;
  if (D.nclass == 0 || D.ntiles == 0) return;
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
  D.rot_ops.alloc(D.nclass * rot_ops_size(p));
  D.rot_az.alloc(D.nclass * (p + 1));
  int nent = 0;
  for (int n = 0; n <= p; ++n) nent += (n + 1) * (n + 1) + n * n;
  const size_t sh = sizeof(double2) * kQuadBatch * ncoef(p) + sizeof(double) * nent;
  static size_t configured = 0;
  if (sh > 48 * 1024 && sh > configured) {
    FMM_CUDA(cudaFuncSetAttribute(build_rot_ops_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    configured = sh;
  }
  build_rot_ops_kernel<<<(unsigned)D.nclass, kRotBuildThreads, sh, s>>>(D.class_keys, p, dgx, dgw, Rs, D.rot_ops,
                                                                         D.rot_az);
  FMM_LAUNCHED("build_rot_ops_kernel");
  // static LPT schedule of the items of each stage over the MMA warps (full 64-column chunk costs)
  const int nmma = 8;
  std::vector<std::vector<int>> lists(3 * nmma);
  for (int st = 0; st < 3; ++st) {
    std::vector<std::pair<int, int>> items;  // (cost, code)
    for (int blk = 0; blk <= p; ++blk) {
      const int R = rot_block_rows(p, st, blk), cost1 = ((R + 7) / 8) * ((R + 3) / 4) * 4;
      const int nparts = rot_block_parts(st, blk);
      for (int cg = 0; cg < 2; ++cg) {
        if (st == 1)
          items.push_back({cost1 * (blk > 0 ? 2 : 1), blk | (cg << 6)});
        else
          for (int pt = 0; pt < nparts; ++pt) items.push_back({cost1, blk | (pt << 5) | (cg << 6)});
      }
    }
    std::stable_sort(items.begin(), items.end(), [](auto& x, auto& y) { return x.first > y.first; });
    std::vector<int> load(nmma, 0);
    for (auto& it : items) {
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
  FMM_CUDA(cudaStreamSynchronize(s));
}

void m2l_rot_launch(fmm_plan_s& P, const m2l::M2LArgs& a) {
  M2LDmma& D = P.m2l_dmma;
  RotArgs r;
  r.a = a;
  r.rops = D.rot_ops;
  r.raz = D.rot_az;
  r.sched = D.rot_sched;
  r.smax = D.rot_smax;
  r.S = rot_xstride((a.NR + 3) & ~3);
  const size_t sh = rot_smem_bytes(P.p, a.T, D.rot_smax);
  const int nhelp = 8;
  void (*k)(const RotArgs, int) = nullptr;
  switch (P.p) {
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
  k<<<(unsigned)D.ntiles, 32 * (8 + nhelp), sh, P.stream>>>(r, nhelp);
  FMM_LAUNCHED("m2l_rot_kernel");
}

}  // namespace fmm
