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

// --------------------------------------------------------------------- class data layout
// One class's data ("blob", doubles): az[p+1] (cos m a, sin m a) | per degree n: D_re (n+1)^2
// row-major, D_im (n+1)^2 (row/column 0 zero) | per order m: Z~_m (p+1-m)^2 row-major;
// padded to an even count (16-byte bulk copies). Stage st of block blk reads its A operand
// from it: st 0 D, st 1 Z~, st 2 D transposed (Re: E^-1 D^T E).
__host__ __device__ inline int rot_block_rows(int p, int st, int blk) { return st == 1 ? p + 1 - blk : blk + 1; }
__host__ __device__ inline int rot_block_parts(int st, int blk) { return st == 1 ? 1 : (blk > 0 ? 2 : 1); }
__host__ __device__ constexpr int rot_d_offset(int p, int n, int part) {
  int off = 2 * (p + 1);
  for (int k = 0; k < n; ++k) off += 2 * (k + 1) * (k + 1);
  return off + part * (n + 1) * (n + 1);
}
__host__ __device__ constexpr int rot_z_offset(int p, int m) {
  int off = rot_d_offset(p, p + 1, 0);
  for (int k = 0; k < m; ++k) off += (p + 1 - k) * (p + 1 - k);
  return off;
}
__host__ __device__ constexpr int rot_blob_size(int p) { return (rot_z_offset(p, p + 1) + 1) & ~1; }
__host__ __device__ inline int rot_block_offset(int p, int st, int blk, int part) {
  return st == 1 ? rot_z_offset(p, blk) : rot_d_offset(p, blk, part);
}

// "RI" layout of one expansion in the M2L v3 kernel (and of M~ rows): a Re plane
// (n, m >= 0) at n(n+1)/2 + m followed by an Im plane (n, m >= 1) at nc + n(n-1)/2 + m - 1;
// (p+1)^2 doubles, and both rotation stages read/write runs contiguous in m.
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
// position of row/column index r of block (st, blk, part); -1 = none (zero)
__host__ __device__ inline int rot_pos(int p, int st, int blk, int part, int r) {
  if (st == 1) {  // order m = blk, degree n = m + r
    if (r > p - blk) return -1;
    return ri_pos(p, blk + r, blk, part);
  }
  if (r > blk || (part == 1 && r == 0)) return -1;  // degree n = blk, order m = r
  return ri_pos(p, blk, r, part);
}
// column base in a chunk buffer: stride S (= 4 mod 16 doubles) plus a +-4 swizzle on columns
// 4..7 of every 8, so B-fragment loads (8 columns x 4 rows) and C-fragment stores (8 rows x
// columns 2k+e) both hit 16 distinct 8-byte banks per half-warp on contiguous positions
__host__ __device__ inline int col_base(int c, int S) { return c * S + ((c & 4) ? ((c & 1) ? -4 : 4) : 0); }

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
    const double2* __restrict__ Rs, double* __restrict__ blobs) {
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
  double* out = blobs + (int64_t)cls * rot_blob_size(p);
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
  // D blocks (Re, Im with zero row/column 0) and Z~ blocks, row-major
  for (int n = 0; n <= p; ++n) {
    int base = 0;  // start of degree n in Dtab
    for (int k = 0; k < n; ++k) base += (k + 1) * (k + 1) + k * k;
    const int R = n + 1;
    for (int e = tid; e < 2 * R * R; e += blockDim.x) {
      const int part = e / (R * R), rr = (e / R) % R, kk = e % R;
      double v = 0.0;
      if (part == 0)
        v = Dtab[base + rr * R + kk];
      else if (rr > 0 && kk > 0)
        v = Dtab[base + R * R + (rr - 1) * n + (kk - 1)];
      out[rot_d_offset(p, n, part) + rr * R + kk] = v;
    }
  }
  for (int m = 0; m <= p; ++m) {
    const int R = p + 1 - m;
    for (int e = tid; e < R * R; e += blockDim.x) {
      const int i = e / R, k = e % R, j = m + i, n = m + k;
      double g = 1.0 / rho;  // (j+n)! / rho^{j+n+1}
      for (int l = 1; l <= j + n; ++l) g *= l / rho;
      for (int t = 0; t <= j; ++t) g *= fA;
      for (int t = 0; t < n; ++t) g *= fB;
      out[rot_z_offset(p, m) + e] = ((n + m) & 1) ? -g : g;
    }
  }
  if (tid == 0 && (rot_z_offset(p, p + 1) & 1)) out[rot_z_offset(p, p + 1)] = 0.0;
}

// ------------------------------------------------------------------- the mat-vec kernel
struct RotArgs {
  M2LArgs a;
  const double* blobs;   // [nclass][rot_blob_size(p)] class data (azimuths, D and Z~ blocks)
  const uint32_t* masks; // [2][NR] symmetry masks: 0 = multipole side (inverse map), 1 = local side
  const int32_t* sched;  // [3][nmma][smax] items (-1 = end)
  int smax, S;
};

constexpr int rot_xstride(int kpad) {
  int s = kpad + 8;  // room for the +-4 column swizzle
  while (s % 16 != 4) ++s;
  return s;
}
template <int P>
struct RGeo {
  static constexpr int NR = (P + 1) * (P + 1);
  static constexpr int KPAD = (NR + 3) & ~3;
  static constexpr int S = rot_xstride(KPAD);  // column stride (see col_base)
  static constexpr int NC = 2 * S * 64 * 8 > 140 * 1024 ? 32 : 64;  // as v2's chunk width rule
  static constexpr int NMMA = 16;  // DMMA issue: one per ~66 cycles per warp, one per 16 per SMSP
  static constexpr int NPREP = 4, NACC = 4;
  static constexpr int MTMAX = (P + 1 + 7) / 8;
  static constexpr int KSMAX = (P + 1 + 3) / 4;
  static constexpr int NCOEF = (P + 1) * (P + 2) / 2;
};

struct RotSmem {
  double *acc, *x0, *x1, *ob;  // ob: [2][blob] class data of the chunk in each buffer
  uint64_t* bar;               // [2]
  int32_t *meta, *srcs, *sslot, *sbeg, *dec, *pairtab, *sched, *blkoff, *ncs;
  uint32_t *mmask, *lmask;     // [NR] symmetry masks (bit 2g: take re/im partner, 2g+1: negate)
};
template <int P>
__device__ __forceinline__ RotSmem rot_carve(double* sm, const RotArgs& r) {
  using G = RGeo<P>;
  RotSmem m;
  m.acc = sm;
  m.x0 = m.acc + (size_t)r.a.T * G::NR;
  m.x1 = m.x0 + G::NC * G::S;
  m.ob = m.x1 + G::NC * G::S;
  uint64_t* b = (uint64_t*)(m.ob + 2 * rot_blob_size(P));
  m.bar = b;
  m.meta = (int32_t*)(b + 2);
  m.srcs = m.meta + 2 * G::NC;
  m.sslot = m.srcs + 2 * G::NC;
  m.sbeg = m.sslot + 2 * G::NC;
  m.dec = m.sbeg + 2 * (G::NC + 1);
  m.mmask = (uint32_t*)(m.dec + G::NR);
  m.lmask = m.mmask + G::NR;
  m.pairtab = (int32_t*)(m.lmask + G::NR);
  m.blkoff = m.pairtab + G::NCOEF;      // [3][P+1][2]
  m.ncs = m.blkoff + 6 * (P + 1);  // [2][2] per buffer: columns, slot segments
  m.sched = m.ncs + 4;
  return m;
}
}  // namespace
size_t rot_smem_bytes(int p, int T, int smax) {
  const int NR = (p + 1) * (p + 1), KPAD = (NR + 3) & ~3, S = rot_xstride(KPAD), nc = ncoef(p);
  const int NC = 2 * S * 64 * 8 > 140 * 1024 ? 32 : 64;
  return sizeof(double) * ((size_t)T * NR + 2 * NC * (size_t)S + 2 * (size_t)rot_blob_size(p)) +
         sizeof(uint64_t) * 2 + sizeof(int32_t) * (8 * NC + 2 + 3 * NR + nc + 6 * (p + 1) + 4 + 3 * 16 * smax);
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

// One MMA item: block (st, blk), part pt, n-tiles [t0, t0 + nti) (nti <= 4) of the chunk,
// in place: the B operand is streamed per k-step, the results stay in registers until every
// k-step has been read; A operand from the chunk's class data in shared memory.
template <int P>
__device__ __forceinline__ void rot_item(const double* ob, const int32_t* blkoff, int st, int blk, int pt, int t0,
                                         int t1, double* xc, int lane) {
  using G = RGeo<P>;
  constexpr int NTI = 4;
  const int R = rot_block_rows(P, st, blk), MT = (R + 7) / 8, KS = (R + 3) / 4;
  const double* A = ob + blkoff[(st * (P + 1) + blk) * 2 + (st == 1 ? 0 : pt)];
  const int colb = lane >> 2, kl = lane & 3;
  double a[G::MTMAX][G::KSMAX];
#pragma unroll
  for (int mt = 0; mt < G::MTMAX; ++mt)
#pragma unroll
    for (int ks = 0; ks < G::KSMAX; ++ks) {
      const int rr = 8 * mt + colb, kk = 4 * ks + kl;
      double v = 0.0;
      if (mt < MT && ks < KS && rr < R && kk < R) {
        if (st == 2) {  // transposed; Re: E^-1 D^T E
          v = A[kk * R + rr];
          if (pt == 0) v *= (kk == 0 ? 1.0 : 2.0) * (rr == 0 ? 1.0 : 0.5);
        } else {
          v = A[rr * R + kk];
        }
      }
      a[mt][ks] = v;
    }
  double c[G::MTMAX][NTI][2];
#pragma unroll
  for (int mt = 0; mt < G::MTMAX; ++mt)
#pragma unroll
    for (int t = 0; t < NTI; ++t) c[mt][t][0] = c[mt][t][1] = 0.0;
  const double* xb = xc + col_base(colb, G::S) + 8 * t0 * G::S;
  const int nt = t1 - t0;
#pragma unroll
  for (int ks = 0; ks < G::KSMAX; ++ks) {
    if (ks < KS) {
      const int pos = rot_pos(P, st, blk, pt, 4 * ks + kl);
      double b[NTI];
#pragma unroll
      for (int t = 0; t < NTI; ++t) b[t] = (t < nt && pos >= 0) ? xb[8 * t * G::S + pos] : 0.0;
#pragma unroll
      for (int mt = 0; mt < G::MTMAX; ++mt)
        if (mt < MT)
#pragma unroll
          for (int t = 0; t < NTI; ++t)
            if (t < nt) dmma884(c[mt][t][0], c[mt][t][1], a[mt][ks], b[t]);
    }
  }
  __syncwarp();  // every lane's B loads precede the in-place stores
  const double sgn = (st == 1 && pt == 1) ? -1.0 : 1.0;
#pragma unroll
  for (int mt = 0; mt < G::MTMAX; ++mt) {
    const int r = 8 * mt + colb;
    const int pos = (mt < MT && r < R) ? rot_pos(P, st, blk, pt, r) : -1;
    if (pos < 0) continue;
    double* y0 = xc + col_base(2 * kl, G::S) + 8 * t0 * G::S + pos;
    double* y1 = xc + col_base(2 * kl + 1, G::S) + 8 * t0 * G::S + pos;
#pragma unroll
    for (int t = 0; t < NTI; ++t)
      if (t < nt) {
        y0[8 * t * G::S] = sgn * c[mt][t][0];
        y1[8 * t * G::S] = sgn * c[mt][t][1];
      }
  }
}

// Named barriers: 1/2 Xfull(b) prep -> MMA; 3/4 Yfull(b) MMA -> acc; 7/8 Xfree(b) acc -> prep;
// 5 MMA warps (between stages); 6 prep warps; 9 acc warps.
template <int P>
__global__ void __launch_bounds__(32 * (RGeo<P>::NMMA + RGeo<P>::NPREP + RGeo<P>::NACC), 1)
    m2l_rot_kernel(const RotArgs r, int dbg) {
  using G = RGeo<P>;
  constexpr int NR = G::NR, NC = G::NC, S = G::S, NCOEF = G::NCOEF, BLOB = rot_blob_size(P);
  constexpr int nmma_t = 32 * G::NMMA, nprep_t = 32 * G::NPREP, nacc_t = 32 * G::NACC;
  extern __shared__ double sm[];
  const RotSmem m = rot_carve<P>(sm, r);
  const M2LArgs& a = r.a;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  // ---- shared tables
  for (int e = tid; e < a.T * NR; e += nthr) m.acc[e] = 0.0;
  for (int q = tid; q < NCOEF; q += nthr) {
    int n = 0;
    while (cidx(n + 1, 0) <= q) ++n;
    m.pairtab[q] = n | ((q - cidx(n, 0)) << 16);
  }
  for (int e = tid; e < 3 * G::NMMA * r.smax; e += nthr) m.sched[e] = r.sched[e];
  for (int e = tid; e < 6 * (P + 1); e += nthr) {
    const int st = e / (2 * (P + 1)), blk = (e / 2) % (P + 1), pt = e & 1;
    m.blkoff[e] = pt < rot_block_parts(st, blk) ? rot_block_offset(P, st, blk, pt) : 0;
  }
  for (int q = tid; q < NR; q += nthr) {
    int n, mm, part;
    ri_decode(P, q, n, mm, part);
    m.dec[q] = (cidx(n, mm) << 8) | (n << 1) | part;
    m.mmask[q] = r.masks[q];
    m.lmask[q] = r.masks[NR + q];
  }
  if (tid == 0) {
    mbar_init(m.bar, 1);
    mbar_init(m.bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int c_first = a.tile_chunk[tile], c_last = a.tile_chunk[tile + 1];
  __syncthreads();
  if (warp >= G::NMMA + G::NPREP) {
    // ================= accumulate warps: acc[slot][r] += (D^L_g Az_L Y)[r] for chunk i
    const int h = tid - nmma_t - nprep_t;
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      named_sync(3 + b, nmma_t + nacc_t);  // Yfull(i)
      if (!(dbg & 4)) {
        const double* y = b ? m.x1 : m.x0;
        const double* ob = m.ob + b * BLOB;
        const int ns = m.ncs[2 * b + 1];
        const int* meta = m.meta + b * NC;
        const int* sb = m.sbeg + b * (NC + 1);
        const int* ss = m.sslot + b * NC;
        for (int row = h; row < NR; row += nacc_t) {
          const int d = m.dec[row], part = d & 1, n = (d >> 1) & 0x7f;
          const int mm = (d >> 8) - cidx(n, 0);
          const int rre = d >> 8, rim = mm ? NCOEF + rre - n - 1 : rre;
          const double ca = mm ? ob[2 * mm] : 1.0, sa = mm ? ob[2 * mm + 1] : 0.0;
          const uint32_t mask = m.lmask[row];
          for (int sgi = 0; sgi < ns; ++sgi) {
            double* ap = m.acc + ss[sgi] * NR + row;
            double v = *ap;
            for (int col = sb[sgi]; col < sb[sgi + 1]; ++col) {
              const uint32_t mg = mask >> (2 * (meta[col] >> 8));
              const double* yc = y + col_base(col, S);
              const double yr = yc[rre], yi = yc[rim];
              const int src = part ^ (int)(mg & 1);  // component of Az_L Y feeding this row
              const double t0 = src == 0 ? fma(-sa, yi, ca * yr) : fma(ca, yi, sa * yr);
              v += (mg & 2) ? -t0 : t0;
            }
            *ap = v;
          }
        }
      }
      named_arrive(7 + b, nacc_t + nprep_t);  // Xfree(i): buffer b may take chunk i + 2
    }
  } else if (warp >= G::NMMA) {
    // ================= prep warps: metadata, TMA bulk copies, symmetry map + Az_M in place
    const int h = tid - nmma_t;
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      if (i >= 2) named_sync(7 + b, nacc_t + nprep_t);  // Xfree(i - 2)
      double* xb = b ? m.x1 : m.x0;
      double* ob = m.ob + b * BLOB;
      load_meta_dev(a, ch, m.meta + b * NC, m.srcs + b * NC, m.sslot + b * NC, m.sbeg + b * (NC + 1), h, nprep_t);
      const int cls = a.chunk_class[ch];
      const int ncol = a.chunk_begin[ch + 1] - a.chunk_begin[ch];
      if (h == 0) {
        m.ncs[2 * b] = ncol;
        m.ncs[2 * b + 1] = a.chunk_seg[ch + 1] - a.chunk_seg[ch];
      }
      named_sync(6, nprep_t);  // metadata visible to the prep warps
      if (h < 32 && !(dbg & 8)) {
        fence_proxy_async();  // earlier generic accesses of xb / ob before the async-proxy writes
        if (h == 0) {
          mbar_arrive_tx(m.bar + b, (unsigned)((ncol * G::KPAD + BLOB) * sizeof(double)));
          bulk_g2s(ob, r.blobs + (int64_t)cls * BLOB, BLOB * sizeof(double), m.bar + b);
        }
        __syncwarp();
        for (int c = h; c < ncol; c += 32)
          bulk_g2s(xb + col_base(c, S), a.Mt + (int64_t)m.srcs[b * NC + c] * G::KPAD, G::KPAD * sizeof(double),
                   m.bar + b);
      }
      const int ncol8 = (ncol + 7) & ~7;  // padding columns of the last n-tile: zeros
      for (int e = h; e < (ncol8 - ncol) * G::KPAD; e += nprep_t)
        xb[col_base(ncol + e / G::KPAD, S) + e % G::KPAD] = 0.0;
      if (!(dbg & 8)) mbar_wait(m.bar + b, (unsigned)((i >> 1) & 1));
      if (!(dbg & 2)) {
#pragma unroll 4
        for (int it = h; it < ncol * NCOEF; it += nprep_t) {
          const int col = it / NCOEF, q = it - col * NCOEF;
          const int pe = m.pairtab[q], n = pe & 0xffff, mm = pe >> 16;
          const int g2 = 2 * (m.meta[b * NC + col] >> 8);
          double* xcol = xb + col_base(col, S);
          if (mm == 0) {
            if ((m.mmask[q] >> g2) & 2) xcol[q] = -xcol[q];
          } else {
            const int rre = q, rim = NCOEF + q - n - 1;
            const uint32_t f0 = m.mmask[rre] >> g2, f1 = m.mmask[rim] >> g2;
            const double v0 = xcol[rre], v1 = xcol[rim];
            double u0 = (f0 & 1) ? v1 : v0, u1 = (f1 & 1) ? v0 : v1;
            u0 = (f0 & 2) ? -u0 : u0;
            u1 = (f1 & 2) ? -u1 : u1;
            const double cs = ob[2 * mm], sn = ob[2 * mm + 1];
            xcol[rre] = cs * u0 - sn * u1;
            xcol[rim] = sn * u0 + cs * u1;
          }
        }
      }
      named_arrive(1 + b, nprep_t + nmma_t);  // Xfull(i)
    }
  } else {
    // ================= MMA warps: the three block-GEMM stages in place
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      named_sync(1 + b, nprep_t + nmma_t);  // Xfull(i)
      double* xc = b ? m.x1 : m.x0;
      const double* ob = m.ob + b * BLOB;
      const int ntiles = (m.ncs[2 * b] + 7) >> 3;
      for (int st = 0; st < 3; ++st) {
        const int32_t* sl = m.sched + (st * G::NMMA + warp) * r.smax;
        for (int k = 0; k < r.smax && !(dbg & 1); ++k) {
          const int item = sl[k];
          if (item < 0) break;
          const int t0 = (item >> 6) & 7, t1 = min(ntiles, t0 + ((item >> 9) & 7));
          if (t0 < t1) rot_item<P>(ob, m.blkoff, st, item & 0x1f, (item >> 5) & 1, t0, t1, xc, lane);
        }
        if (st < 2) named_sync(5, nmma_t);  // stage st complete before st + 1 reads it
      }
      named_arrive(3 + b, nmma_t + nacc_t);  // Yfull(i)
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
  D.rot_ops.alloc(D.nclass * rot_blob_size(p));
  {  // symmetry masks from the signed-permutation tables (m2l_dmma.cu)
    const int NR = (p + 1) * (p + 1);
    std::vector<int32_t> sym = build_symtab(p);
    std::vector<uint32_t> mk(2 * NR, 0);
    for (int which = 0; which < 2; ++which)
      for (int q = 0; q < NR; ++q) {  // RI row q <-> real index rr
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
  int nent = 0;
  for (int n = 0; n <= p; ++n) nent += (n + 1) * (n + 1) + n * n;
  const size_t sh = sizeof(double2) * kQuadBatch * ncoef(p) + sizeof(double) * nent;
  static size_t configured = 0;
  if (sh > 48 * 1024 && sh > configured) {
    FMM_CUDA(cudaFuncSetAttribute(build_rot_ops_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    configured = sh;
  }
  build_rot_ops_kernel<<<(unsigned)D.nclass, kRotBuildThreads, sh, s>>>(D.class_keys, p, dgx, dgw, Rs, D.rot_ops);
  FMM_LAUNCHED("build_rot_ops_kernel");
  // static LPT schedule of the items of each stage over the MMA warps (full 64-column chunk costs)
  const int nmma = 16;
  std::vector<std::vector<int>> lists(3 * nmma);
  for (int st = 0; st < 3; ++st) {
    std::vector<std::pair<int, int>> items;  // (cost, code)
    for (int blk = 0; blk <= p; ++blk) {
      const int R = rot_block_rows(p, st, blk), mk = ((R + 7) / 8) * ((R + 3) / 4);
      const int nparts = st == 1 ? (blk > 0 ? 2 : 1) : rot_block_parts(st, blk);
      const int ntc = rot_chunk_width(p) / 8;  // n-tiles of a full chunk
      const int nti = std::min(ntc, mk >= 4 ? 2 : 4);  // n-tiles per item: big blocks split finer
      for (int pt = 0; pt < nparts; ++pt)
        for (int t0 = 0; t0 < ntc; t0 += nti) items.push_back({mk * nti + 6, blk | (pt << 5) | (t0 << 6) | (nti << 9)});
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
  r.smax = D.rot_smax;
  const size_t sh = rot_smem_bytes(P.p, a.T, D.rot_smax);
  void (*k)(const RotArgs, int) = nullptr;
  const char* dbgs = getenv("FMM_M2L_DEBUG");  // timing experiments only (skips work: wrong results)
  const int dbg = dbgs ? atoi(dbgs) : 0;
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
  k<<<(unsigned)D.ntiles, 32 * (16 + 4 + 4), sh, P.stream>>>(r, dbg);
  FMM_LAUNCHED("m2l_rot_kernel");
}

}  // namespace fmm
