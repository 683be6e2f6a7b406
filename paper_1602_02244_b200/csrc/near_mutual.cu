// near_mutual.cu — S12 P2P with each unordered leaf pair evaluated ONCE (single GPU, potentials):
// 1/r_ij serves both directions, q_j / r_ij for target i and q_i / r_ij for target j.
//
// The P2P lists of the dual traversal are symmetric ((A, B) is a pair iff (B, A) is: measured
// on cube, Plummer and sphere trees; the setup checks it and keeps the directed path otherwise),
// and the direct operator is the dense, symmetric diagonal block of the kernel matrix
// (PAPER.md:191-196). Per leaf A one warp evaluates A's own block (all i != j) and every pair
// (A, B) with B > A in A's list: A's sums stay in registers, B's sums — this task's contribution
// to the targets of B — go to a per-task slot of a partial-sum buffer. A second kernel adds, per
// target leaf, its own sums and the partials of the tasks (A', L) with A' < L in list order, then
// L2P, the exact 2^-e rescale and the scatter to caller order. Every sum has a fixed order (no
// atomics): bitwise deterministic.
//
// Lane layout per warp: NG = 8 target groups x NS = 4 source lanes for leaves of <= 64 particles,
// 16 x 2 above (<= 128). Lane (a, b) holds A's targets i = a + NG k (k < TPL = ceil(nA / NG)) in
// registers and takes the sources j = b + NS k' from shared memory. A's
// task sources (the B leaves, concatenated: their partial slots are contiguous) stream through
// double-buffered cp.async units of kU particles. Per source j, a lane's partial over its
// targets goes to a shared row red[a][j]; after the unit the NG rows are summed in a fixed order
// (the B side). A's sums are reduced over the 4 source lanes at the end.
// Per directed interaction: ~6 FP64 ops (12 per evaluated pair) instead of 11.
#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>

#include "harmonics.cuh"
#include "near_common.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kMaxLeaf = 128;  // particles per leaf (larger leaves: the directed path)
constexpr int kSmallLeaf = 64;  // up to here 8 target groups x 4 source lanes, above 16 x 2
#ifndef FMM_MUTUAL_UNROLL
#define FMM_MUTUAL_UNROLL 1  // source-loop unroll of the mutual units
#endif
#ifndef FMM_MUTUAL_PF
#define FMM_MUTUAL_PF 1  // source loaded one loop iteration ahead (LDS latency off the chain; near 1.58 -> 1.53 ms at configs[2])
#endif
#ifndef FMM_MUTUAL_BUF
#define FMM_MUTUAL_BUF 128
#endif
#ifndef FMM_MUTUAL_MINB
#define FMM_MUTUAL_MINB 12  // warps (CTAs) per SM: 16.4 KB shared memory each
#endif
constexpr int kUnroll = FMM_MUTUAL_UNROLL;
constexpr int kU = FMM_MUTUAL_BUF;  // source particles per staged unit
constexpr int kR = kU + 4;          // row stride of the B-side partials: 2 wavefronts per store

__device__ __forceinline__ void mcp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void mcp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void mcp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct MutualArgs {
  const int32_t* leaves;    // [nleaves]
  int64_t nleaves;
  const int32_t *cbeg, *cend;
  const double4* pos;       // x, y, z, q (Morton order)
  const int32_t* toff;      // [ncells + 1] tasks of leaf A: (A, task_b[t]) for t in [toff[A], toff[A+1])
  const int32_t* tmend;     // [ncells] tasks [toff[A], tmend[A]) are mutual, the rest directed (B not owned)
  const int32_t* task_b;
  const int64_t* poff;      // [ntasks] partial slot of task t (|B| doubles; contiguous over A's tasks)
  double* partial;          // B-side sums
  double* own;              // [n] A-side sums (sorted order)
};

// A's own leaf against itself: every ordered pair i != j (r^2 = 0 skipped: coincident points)
template <int NS, int TPL>
__device__ __forceinline__ void self_unit(const double4* __restrict__ sbuf, int n, int b, const double3 (&xi)[TPL],
                                          double (&fi)[TPL]) {
#if FMM_MUTUAL_PF
  double4 sn = sbuf[b < n ? b : 0];
  for (int j = b; j < n; j += NS) {
    const double4 s = sn;
    sn = sbuf[j + NS < n ? j + NS : 0];
#else
  for (int j = b; j < n; j += NS) {
    const double4 s = sbuf[j];
#endif
#pragma unroll
    for (int k = 0; k < TPL; ++k) {
      const double dx = xi[k].x - s.x, dy = xi[k].y - s.y, dz = xi[k].z - s.z;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double y = r2 > 0.0 ? near::rsqrt_fp64(r2) : 0.0;
      fi[k] = fma(s.w, y, fi[k]);
    }
  }
}

// n sources of other leaves: 1/r once per pair, q_j / r to A's sums (registers), q_i / r to the
// source's B-side sum (this lane's partial over its TPL targets to red[a][j], then summed over
// the 8 target groups in a fixed order and stored to the task's partial slots)
template <int NG, int TPL>
__device__ __forceinline__ void mutual_unit(const double4* __restrict__ sbuf, int n, int a, int b, int lane,
                                            const double3 (&xi)[TPL], const double (&qi)[TPL], double (&fi)[TPL],
                                            double* __restrict__ red, double* __restrict__ out) {
  constexpr int NS = 32 / NG;
#if FMM_MUTUAL_PF
  double4 sn = sbuf[b < n ? b : 0];  // the next source, loaded an iteration ahead
#endif
#pragma unroll kUnroll
  for (int j0 = 0; j0 < n; j0 += NS) {  // j < NS ceil(n / NS) <= kR
    const int j = j0 + b;
#if FMM_MUTUAL_PF
    double4 s = sn;
    sn = sbuf[j + NS < n ? j + NS : 0];
#else
    double4 s = sbuf[j < n ? j : 0];    // padding sources: source 0 with charge 0
#endif
    if (j >= n) s.w = 0.0;
    double sb = 0.0;
#pragma unroll
    for (int k = 0; k < TPL; ++k) {
      const double dx = xi[k].x - s.x, dy = xi[k].y - s.y, dz = xi[k].z - s.z;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double y = near::rsqrt_fp64(r2);  // distinct leaves: r^2 > 0
      fi[k] = fma(s.w, y, fi[k]);
      sb = fma(qi[k], y, sb);
    }
    red[a * kR + j] = sb;
  }
  __syncwarp();
  for (int j = lane; j < n; j += 32) {
    double t = red[j];
#pragma unroll
    for (int g = 1; g < NG; ++g) t += red[g * kR + j];
    out[j] = t;
  }
}

struct Span {
  int q, off;  // stream position: task q (relative to A's first), particle off in it
  int n;       // particles in the unit
  int64_t base;  // stream offset of the unit (partial slot - poff[t0]); -1: A itself
  bool dir;      // sources of directed tasks (another rank's leaves: A's sums only)
};

template <int NG, int TPL>
__device__ void mutual_leaf(const MutualArgs& m, int A, int lane, double4 (*buf)[kU], double* red) {
  constexpr int NS = 32 / NG;
  const int a = lane / NS, b = lane % NS;
  const int ab = m.cbeg[A], nA = m.cend[A] - ab;
  double3 xi[TPL];
  double qi[TPL], fi[TPL];
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    const int i = a + NG * k;
    // padding targets: copies of target 0 with charge 0 (a point of A: r > 0 to every point of B)
    const double4 v = m.pos[ab + (i < nA ? i : 0)];
    xi[k] = make_double3(v.x, v.y, v.z);
    qi[k] = i < nA ? v.w : 0.0;
    fi[k] = 0.0;
  }
  const int t0 = m.toff[A], nt = m.toff[A + 1] - t0, nmt = m.tmend[A] - t0;
  // the first 32 tasks' source ranges, one per lane; later ones read when needed
  int my_b = 0, my_n = 0;
  if (lane < nt) {
    const int B = m.task_b[t0 + lane];
    my_b = m.cbeg[B];
    my_n = m.cend[B] - my_b;
  }
  double* out0 = m.partial + (nt > 0 ? m.poff[t0] : 0);
  auto copy = [&](const double4* src, int n, double4* dst) {
    for (int h = lane; h < 2 * n; h += 32) mcp_async16((double*)dst + 2 * h, (const double*)src + 2 * h);
  };
  // stage the unit starting at stream position (q, off) into buffer bb; advances (q, off)
  int q = 0, off = 0;
  int64_t spos = 0;
  auto stage = [&](int bb) -> Span {
    Span u{q, off, 0, spos, q >= nmt};
    while (q < nt && u.n < kU && (q < nmt) == !u.dir) {  // a unit never mixes mutual and directed
      int sb, nb;
      if (q < 32) {
        sb = __shfl_sync(0xffffffffu, my_b, q);
        nb = __shfl_sync(0xffffffffu, my_n, q);
      } else {
        const int B = m.task_b[t0 + q];
        sb = m.cbeg[B];
        nb = m.cend[B] - sb;
      }
      const int take = min(nb - off, kU - u.n);
      copy(m.pos + sb + off, take, buf[bb] + u.n);
      u.n += take;
      off += take;
      if (off == nb) {
        ++q;
        off = 0;
      }
    }
    spos += u.n;
    mcp_commit();
    return u;
  };
  copy(m.pos + ab, nA, buf[0]);  // unit 0: A itself
  mcp_commit();
  Span cur{0, 0, nA, -1, false};
  int bb = 0;
  while (true) {
    const bool more = q < nt;
    Span nx{0, 0, 0, 0, false};
    if (more) {
      nx = stage(bb ^ 1);
      mcp_wait<1>();
    } else {
      mcp_wait<0>();
    }
    __syncwarp();
    if (cur.base < 0 || cur.dir)  // A itself (r = 0 skipped), or directed sources
      self_unit<NS, TPL>(buf[bb], cur.n, b, xi, fi);
    else
      mutual_unit<NG, TPL>(buf[bb], cur.n, a, b, lane, xi, qi, fi, red, out0 + cur.base);
    __syncwarp();  // buffer bb and red are rewritten by the next units
    if (!more) break;
    cur = nx;
    bb ^= 1;
  }
  // A side: sum over the NS source lanes
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
#pragma unroll
    for (int o = 1; o < NS; o <<= 1) fi[k] += __shfl_xor_sync(0xffffffffu, fi[k], o);
    const int i = a + NG * k;
    if (b == 0 && i < nA) m.own[ab + i] = fi[k];
  }
}

// NGMAX = 8: every leaf <= kSmallLeaf particles; 16: larger leaves too (twice the B-side rows)
template <int NGMAX>
__global__ void __launch_bounds__(32, FMM_MUTUAL_MINB) near_mutual_kernel(const MutualArgs m) {
  __shared__ __align__(16) double4 buf[2][kU];
  __shared__ double red[NGMAX * kR];
  const int64_t li = blockIdx.x;
  if (li >= m.nleaves) return;
  const int A = m.leaves[li];
  const int nA = m.cend[A] - m.cbeg[A];
  const int lane = threadIdx.x & 31;
  // TPL = ceil(nA / 8): idle target slots < 8 per leaf (powers of two only left 30 % of the
  // lanes idle on the Poisson(30.5) leaves of configs[2]); leaves above 64: 16 x 2 lanes
  if (NGMAX == 16 && nA > kSmallLeaf) {
    switch ((nA + 15) >> 4) {
      case 5: mutual_leaf<16, 5>(m, A, lane, buf, red); break;
      case 6: mutual_leaf<16, 6>(m, A, lane, buf, red); break;
      case 7: mutual_leaf<16, 7>(m, A, lane, buf, red); break;
      default: mutual_leaf<16, 8>(m, A, lane, buf, red); break;
    }
    return;
  }
  switch ((nA + 7) >> 3) {
    case 0:
    case 1: mutual_leaf<8, 1>(m, A, lane, buf, red); break;
    case 2: mutual_leaf<8, 2>(m, A, lane, buf, red); break;
    case 3: mutual_leaf<8, 3>(m, A, lane, buf, red); break;
    case 4: mutual_leaf<8, 4>(m, A, lane, buf, red); break;
    case 5: mutual_leaf<8, 5>(m, A, lane, buf, red); break;
    case 6: mutual_leaf<8, 6>(m, A, lane, buf, red); break;
    case 7: mutual_leaf<8, 7>(m, A, lane, buf, red); break;
    default: mutual_leaf<8, 8>(m, A, lane, buf, red); break;
  }
}

// L2P of the potential at (x, y, z) from a cell's local expansion in shared memory, degree P known
// at compile time (the recurrences of harmonics.cuh l2p_eval in the same order)
template <int P>
__device__ __forceinline__ double l2p_phi(const double2* __restrict__ Ls, double x, double y, double z) {
  const double r2 = x * x + y * y + z * z;
  double2 diag = make_double2(1.0, 0.0);
  double f = 0.0;
#pragma unroll 1
  for (int m = 0; m <= P; ++m) {
    if (m > 0) {
      const double s = c_half_inv.v[m];
      diag = cmul(diag, make_double2(s * x, s * y));
    }
    const double w = m == 0 ? 1.0 : 2.0;
    double2 a = make_double2(0, 0), b = diag;  // R_{n-1}^m, R_n^m
#pragma unroll 4
    for (int n = m; n <= P; ++n) {
      if (n == m + 1) {
        a = b;
        b = cscale(diag, z);
      } else if (n > m + 1) {
        const double inv = c_inv_nm.v[n * (kMaxP + 1) + m];
        const double2 c = make_double2(((2 * n - 1) * z * b.x - r2 * a.x) * inv, ((2 * n - 1) * z * b.y - r2 * a.y) * inv);
        a = b;
        b = c;
      }
      const double2 l = Ls[cidx(n, m)];
      f += w * (l.x * b.x + l.y * b.y);
    }
  }
  return f;
}

// own + the partials of the tasks where the leaf is the B side (list order), then L2P, the exact
// rescale and the scatter (warp per leaf, lane per target; the leaf's local expansion staged in
// shared memory once per warp)
template <int P>
__global__ void __launch_bounds__(128) mutual_out_kernel(
    const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ cbeg,
    const int32_t* __restrict__ cend, const double4* __restrict__ center, const double4* __restrict__ pos,
    const double2* __restrict__ L, const double* __restrict__ own, const int32_t* __restrict__ goff,
    const int64_t* __restrict__ gslot, const double* __restrict__ partial, const uint32_t* __restrict__ perm,
    int64_t out_base, double s_phi, double* __restrict__ phi_out) {
  constexpr int NC = (P + 1) * (P + 2) / 2;
  __shared__ double2 Lsh[4][NC];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int64_t li = (int64_t)blockIdx.x * 4 + wi;
  if (li >= nleaves) return;
  const int leaf = leaves[li];
  const double4 c = center[leaf];
  const double2* Lc = L + (int64_t)leaf * NC;
  for (int k = lane; k < NC; k += 32) Lsh[wi][k] = Lc[k];
  __syncwarp();
  const int tb = cbeg[leaf], g0 = goff[leaf], g1 = goff[leaf + 1];
  for (int t = tb + lane; t < cend[leaf]; t += 32) {
    const double4 x = pos[t];
    double f = own[t];
    for (int g = g0; g < g1; ++g) f += partial[gslot[g] + (t - tb)];
    f += l2p_phi<P>(Lsh[wi], x.x - c.x, x.y - c.y, x.z - c.z);
    phi_out[perm ? (int64_t)perm[t] : (int64_t)t - out_base] = f * s_phi;  // caller order, or owned order (LET)
  }
}

template <int P>
void launch_mutual_out(const fmm_plan_s& Pl, const NearMutual& Mu, const int32_t* leaves, int64_t nl, double* phi) {
  mutual_out_kernel<P><<<cdiv(nl, 4), 128, 0, Pl.stream>>>(leaves, nl, Pl.cells.begin, Pl.cells.end, Pl.cells.center,
                                                          Pl.pos, Pl.L, Mu.own, Mu.goff, Mu.gslot, Mu.partial,
                                                          Pl.near_compact_out ? nullptr : Pl.perm.ptr, Pl.own_begin,
                                                          std::ldexp(1.0, -Pl.e), phi);
}
template <int... Ps>
void dispatch_mutual_out(int p, const fmm_plan_s& Pl, const NearMutual& Mu, const int32_t* leaves, int64_t nl,
                         double* phi, std::integer_sequence<int, Ps...>) {
  bool done = false;
  ((p == Ps ? (launch_mutual_out<Ps>(Pl, Mu, leaves, nl, phi), done = true) : false), ...);
  if (!done) throw Error(FMM_ERR_USAGE, "near_mutual: p out of range");
}

// setup, per entry k of the target-grouped P2P list (A = tgt[k], B = src[k]): the flags and sizes
// the scans turn into the task lists. Only targets A this rank owns have tasks (one rank: all). For
// an owned source B the pair is mutual — a task of A if B > A (with |B| partial slots), the reverse
// side (B's task) if B < A — and B's list must hold A exactly once (that entry's index is kept for
// the reverse side); a source owned by another rank is a directed task of A (A's sums only).
__global__ void mutual_mark_kernel(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src,
                                   const int32_t* __restrict__ off, const int32_t* __restrict__ cb,
                                   const int32_t* __restrict__ ce, int64_t np, int64_t own_b, int64_t own_e,
                                   int32_t* __restrict__ is_mt, int32_t* __restrict__ is_dt,
                                   int32_t* __restrict__ size, int32_t* __restrict__ is_rev,
                                   int32_t* __restrict__ rpos, int* __restrict__ bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int A = tgt[k], B = src[k];
  int mt = 0, dt = 0, sz = 0, rev = 0;
  const bool ownA = cb[A] >= own_b && ce[A] <= own_e, ownB = cb[B] >= own_b && ce[B] <= own_e;
  if (ownA) {
    if (ce[A] - cb[A] > kMaxLeaf) atomicOr(bad, 1);
    if (ce[A] - cb[A] > kSmallLeaf) atomicOr(bad, 4);  // (not a failure: the 16-group kernel)
    if (B != A && !ownB) {
      dt = 1;
    } else if (B != A) {
      int j = -1, cnt = 0;
      for (int i = off[B]; i < off[B + 1]; ++i)
        if (src[i] == A) {
          j = i;
          ++cnt;
        }
      if (cnt != 1) atomicOr(bad, 2);
      if (B > A) {
        mt = 1;
        sz = ce[B] - cb[B];
      } else {
        rev = 1;
        rpos[k] = j;
      }
    }
  }
  is_mt[k] = mt;
  is_dt[k] = dt;
  size[k] = sz;
  is_rev[k] = rev;
}

// compaction: per target A its mutual tasks (list order) then its directed tasks (list order); the
// reverse side's slots in list order. Task index of a mutual entry: mutual tasks before it + directed
// tasks of earlier targets; of a directed entry: mutual tasks up to A's last + directed before it.
__global__ void mutual_compact_kernel(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src,
                                      const int32_t* __restrict__ off, int64_t np, const int32_t* __restrict__ is_mt,
                                      const int32_t* __restrict__ is_dt, const int32_t* __restrict__ is_rev,
                                      const int32_t* __restrict__ rpos, const int64_t* __restrict__ mscan,
                                      const int64_t* __restrict__ dscan, const int64_t* __restrict__ sscan,
                                      const int64_t* __restrict__ rscan, int64_t nm, int32_t* __restrict__ task_b,
                                      int64_t* __restrict__ poff, int64_t* __restrict__ gslot) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int A = tgt[k];
  if (is_mt[k]) {
    const int64_t t = mscan[k] + dscan[off[A]];
    task_b[t] = src[k];
    poff[t] = sscan[k];
  } else if (is_dt[k]) {
    const int64_t e = off[A + 1];
    const int64_t t = (e < np ? mscan[e] : nm) + dscan[k];
    task_b[t] = src[k];
    poff[t] = 0;  // (unused: directed tasks have no partial slots)
  } else if (is_rev[k]) {
    gslot[rscan[k]] = sscan[rpos[k]];  // the slot of task (B, A) at its entry in B's list
  }
}

__global__ void mutual_offsets_kernel(const int32_t* __restrict__ off, int64_t nc, int64_t np,
                                      const int64_t* __restrict__ mscan, const int64_t* __restrict__ dscan,
                                      const int64_t* __restrict__ rscan, int64_t nm, int64_t nd, int64_t nrev,
                                      int32_t* __restrict__ toff, int32_t* __restrict__ tmend,
                                      int32_t* __restrict__ goff) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nc) return;
  const int64_t o = c < nc ? off[c] : np;
  const int64_t mo = o < np ? mscan[o] : nm, d = o < np ? dscan[o] : nd;
  toff[c] = (int32_t)(mo + d);
  goff[c] = (int32_t)(o < np ? rscan[o] : nrev);
  if (c < nc) {
    const int64_t e = off[c + 1];
    tmend[c] = (int32_t)((e < np ? mscan[e] : nm) + d);
  }
}

}  // namespace

// Task lists (setup, on the device) for the targets this rank owns: mutual tasks (A, B > A) with
// their partial slots, then directed tasks (sources owned by another rank), and per leaf the slots
// of the tasks where it is the B side, in its list order. Disabled (the directed path is kept) if
// the owned lists are not symmetric with each source at most once per list, a leaf with pairs
// exceeds kMaxLeaf particles, or the partial buffer would take more than a quarter of the free
// device memory.
void near_mutual_setup(fmm_plan_s& P) {
  NearMutual& Mu = P.mutual;
  Mu.enabled = false;
  if (P.dim != 3 || P.helmholtz || P.p2p.n == 0) return;
  const int64_t nc = P.cells.n, np = P.p2p.n;
  DevBuf<int32_t> is_mt, is_dt, size, is_rev, rpos;
  DevBuf<int64_t> mscan, dscan, sscan, rscan;
  DevBuf<int> bad;
  is_mt.alloc(np);
  is_dt.alloc(np);
  size.alloc(np);
  is_rev.alloc(np);
  rpos.alloc(np);
  mscan.alloc(np);
  dscan.alloc(np);
  sscan.alloc(np);
  rscan.alloc(np);
  bad.alloc(1);
  FMM_CUDA(cudaMemsetAsync(bad.ptr, 0, sizeof(int), P.stream));
  mutual_mark_kernel<<<cdiv(np, 256), 256, 0, P.stream>>>(P.p2p.tgt, P.p2p.src, P.p2p.off, P.cells.begin,
                                                          P.cells.end, np, P.own_begin, P.own_end, is_mt, is_dt, size,
                                                          is_rev, rpos, bad);
  FMM_LAUNCHED("mutual_mark_kernel");
  const int64_t nm = scan_counts_total(is_mt, mscan, np, P.stream);
  const int64_t nd = scan_counts_total(is_dt, dscan, np, P.stream);
  const int64_t slots = scan_counts_total(size, sscan, np, P.stream);
  const int64_t nrev = scan_counts_total(is_rev, rscan, np, P.stream);
  int hbad = 0;
  FMM_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaStreamSynchronize(P.stream));
  Mu.big = (hbad & 4) != 0;
  hbad &= 3;
  size_t mem_free = 0, mem_total = 0;
  FMM_CUDA(cudaMemGetInfo(&mem_free, &mem_total));
  if (hbad || nm != nrev || (size_t)slots * 8 > mem_free / 4 || nm + nd > INT32_MAX) return;
  const int64_t ntasks = nm + nd;
  Mu.toff.alloc(nc + 1);
  Mu.tmend.alloc(std::max<int64_t>(1, nc));
  Mu.goff.alloc(nc + 1);
  Mu.task_b.alloc(std::max<int64_t>(1, ntasks));
  Mu.poff.alloc(std::max<int64_t>(1, ntasks));
  Mu.gslot.alloc(std::max<int64_t>(1, nrev));
  mutual_compact_kernel<<<cdiv(np, 256), 256, 0, P.stream>>>(P.p2p.tgt, P.p2p.src, P.p2p.off, np, is_mt, is_dt, is_rev,
                                                             rpos, mscan, dscan, sscan, rscan, nm, Mu.task_b, Mu.poff,
                                                             Mu.gslot);
  FMM_LAUNCHED("mutual_compact_kernel");
  mutual_offsets_kernel<<<cdiv(nc + 1, 256), 256, 0, P.stream>>>(P.p2p.off, nc, np, mscan, dscan, rscan, nm, nd, nrev,
                                                                  Mu.toff, Mu.tmend, Mu.goff);
  FMM_LAUNCHED("mutual_offsets_kernel");
  Mu.partial.alloc(std::max<int64_t>(1, slots));
  Mu.own.alloc(std::max<int64_t>(1, P.n));
  Mu.ntasks = ntasks;
  FMM_CUDA(cudaStreamSynchronize(P.stream));  // the scratch buffers die here
  Mu.enabled = true;
}

void near_mutual_pass(fmm_plan_s& P, double* phi) {
  NearMutual& Mu = P.mutual;
  const int64_t nl = P.own_leaf_end - P.own_leaf_begin;
  if (nl <= 0) return;
  const int32_t* leaves = P.leaves.ptr + P.own_leaf_begin;
  MutualArgs m;
  m.leaves = leaves;
  m.nleaves = nl;
  m.cbeg = P.cells.begin;
  m.cend = P.cells.end;
  m.pos = P.pos;
  m.toff = Mu.toff;
  m.tmend = Mu.tmend;
  m.task_b = Mu.task_b;
  m.poff = Mu.poff;
  m.partial = Mu.partial;
  m.own = Mu.own;
  if (Mu.big)
    near_mutual_kernel<16><<<(unsigned)nl, 32, 0, P.stream>>>(m);
  else
    near_mutual_kernel<8><<<(unsigned)nl, 32, 0, P.stream>>>(m);
  FMM_LAUNCHED("near_mutual_kernel");
  dispatch_mutual_out(P.p, P, Mu, leaves, nl, phi, std::make_integer_sequence<int, kMaxP + 1>{});
  FMM_LAUNCHED("mutual_out_kernel");
}

}  // namespace fmm
