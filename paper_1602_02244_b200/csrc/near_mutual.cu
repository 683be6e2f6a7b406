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
// Lane layout per warp: 8 target groups x 4 source lanes. Lane (a, b) holds A's targets
// i = a + 8k (k < TPL) in registers and takes the sources j = b + 4k' from shared memory. A's
// task sources (the B leaves, concatenated: their partial slots are contiguous) stream through
// double-buffered cp.async units of kU particles. Per source j, a lane's partial over its
// targets goes to a shared row red[a][j]; after the unit the 8 rows are summed in a fixed order
// (the B side). A's sums are reduced over the 4 source lanes at the end.
// Per directed interaction: ~6 FP64 ops (12 per evaluated pair) instead of 11.
#include <algorithm>
#include <cmath>
#include <vector>

#include "harmonics.cuh"
#include "near_common.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kMaxLeaf = 64;  // particles per leaf (larger leaves: the directed path)
#ifndef FMM_MUTUAL_BUF
#define FMM_MUTUAL_BUF 128
#endif
#ifndef FMM_MUTUAL_MINB
#define FMM_MUTUAL_MINB 12  // warps (CTAs) per SM: 16.4 KB shared memory each
#endif
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
  const int32_t* task_b;
  const int64_t* poff;      // [ntasks] partial slot of task t (|B| doubles; contiguous over A's tasks)
  double* partial;          // B-side sums
  double* own;              // [n] A-side sums (sorted order)
};

// A's own leaf against itself: every ordered pair i != j (r^2 = 0 skipped: coincident points)
template <int TPL>
__device__ __forceinline__ void self_unit(const double4* __restrict__ sbuf, int n, int b, const double3 (&xi)[TPL],
                                          double (&fi)[TPL]) {
  for (int j = b; j < n; j += 4) {
    const double4 s = sbuf[j];
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
template <int TPL>
__device__ __forceinline__ void mutual_unit(const double4* __restrict__ sbuf, int n, int a, int b, int lane,
                                            const double3 (&xi)[TPL], const double (&qi)[TPL], double (&fi)[TPL],
                                            double* __restrict__ red, double* __restrict__ out) {
  for (int j0 = 0; j0 < n; j0 += 4) {  // j < 4 ceil(n / 4) <= kR
    const int j = j0 + b;
    double4 s = sbuf[j < n ? j : 0];    // padding sources: source 0 with charge 0
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
    for (int g = 1; g < 8; ++g) t += red[g * kR + j];
    out[j] = t;
  }
}

struct Span {
  int q, off;  // stream position: task q (relative to A's first), particle off in it
  int n;       // particles in the unit
  int64_t base;  // stream offset of the unit (partial slot - poff[t0])
};

template <int TPL>
__device__ void mutual_leaf(const MutualArgs& m, int A, int lane, double4 (*buf)[kU], double* red) {
  const int a = lane >> 2, b = lane & 3;
  const int ab = m.cbeg[A], nA = m.cend[A] - ab;
  double3 xi[TPL];
  double qi[TPL], fi[TPL];
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    const int i = a + 8 * k;
    // padding targets: copies of target 0 with charge 0 (a point of A: r > 0 to every point of B)
    const double4 v = m.pos[ab + (i < nA ? i : 0)];
    xi[k] = make_double3(v.x, v.y, v.z);
    qi[k] = i < nA ? v.w : 0.0;
    fi[k] = 0.0;
  }
  const int t0 = m.toff[A], nt = m.toff[A + 1] - t0;
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
    Span u{q, off, 0, spos};
    while (q < nt && u.n < kU) {
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
  Span cur{0, 0, nA, -1};
  int bb = 0;
  while (true) {
    const bool more = q < nt;
    Span nx{0, 0, 0, 0};
    if (more) {
      nx = stage(bb ^ 1);
      mcp_wait<1>();
    } else {
      mcp_wait<0>();
    }
    __syncwarp();
    if (cur.base < 0)
      self_unit<TPL>(buf[bb], cur.n, b, xi, fi);
    else
      mutual_unit<TPL>(buf[bb], cur.n, a, b, lane, xi, qi, fi, red, out0 + cur.base);
    __syncwarp();  // buffer bb and red are rewritten by the next units
    if (!more) break;
    cur = nx;
    bb ^= 1;
  }
  // A side: sum over the 4 source lanes
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    fi[k] += __shfl_xor_sync(0xffffffffu, fi[k], 1);
    fi[k] += __shfl_xor_sync(0xffffffffu, fi[k], 2);
    const int i = a + 8 * k;
    if (b == 0 && i < nA) m.own[ab + i] = fi[k];
  }
}

__global__ void __launch_bounds__(32, FMM_MUTUAL_MINB) near_mutual_kernel(const MutualArgs m) {
  __shared__ __align__(16) double4 buf[2][kU];
  __shared__ double red[8 * kR];
  const int64_t li = blockIdx.x;
  if (li >= m.nleaves) return;
  const int A = m.leaves[li];
  const int nA = m.cend[A] - m.cbeg[A];
  const int lane = threadIdx.x & 31;
  if (nA <= 8)
    mutual_leaf<1>(m, A, lane, buf, red);
  else if (nA <= 16)
    mutual_leaf<2>(m, A, lane, buf, red);
  else if (nA <= 32)
    mutual_leaf<4>(m, A, lane, buf, red);
  else
    mutual_leaf<8>(m, A, lane, buf, red);
}

// own + the partials of the tasks where the leaf is the B side (list order), then L2P, the exact
// rescale and the scatter (warp per leaf, lane per target)
__global__ void __launch_bounds__(128) mutual_out_kernel(
    const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ cbeg,
    const int32_t* __restrict__ cend, const double4* __restrict__ center, const double4* __restrict__ pos,
    const double2* __restrict__ L, int p, int nc, const double* __restrict__ own, const int32_t* __restrict__ goff,
    const int64_t* __restrict__ gslot, const double* __restrict__ partial, const uint32_t* __restrict__ perm,
    double s_phi, double* __restrict__ phi_out) {
  const int lane = threadIdx.x & 31;
  const int64_t li = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (li >= nleaves) return;
  const int leaf = leaves[li];
  const double4 c = center[leaf];
  const double2* Lc = L + (int64_t)leaf * nc;
  const int tb = cbeg[leaf], g0 = goff[leaf], g1 = goff[leaf + 1];
  for (int t = tb + lane; t < cend[leaf]; t += 32) {
    const double4 x = pos[t];
    double f = own[t];
    for (int g = g0; g < g1; ++g) f += partial[gslot[g] + (t - tb)];
    double3 gr = make_double3(0, 0, 0);
    l2p_eval<false>(Lc, p, x.x - c.x, x.y - c.y, x.z - c.z, f, gr);
    phi_out[perm[t]] = f * s_phi;
  }
}

}  // namespace

// host lists (setup): tasks (A, B > A) in A's list order, partial slots, and per leaf the slots of
// the tasks where it is the B side. Disabled (directed path kept) if the lists are not symmetric, a
// leaf exceeds kMaxLeaf particles, or the partial buffer would exceed 2 GB.
void near_mutual_setup(fmm_plan_s& P) {
  NearMutual& Mu = P.mutual;
  Mu.enabled = false;
  if (P.world != 1 || P.dim != 3 || P.helmholtz || P.p2p.n == 0) return;
  const int64_t nc = P.cells.n, np = P.p2p.n;
  std::vector<int32_t> cb(nc), ce(nc), ps(np), off(nc + 1);
  FMM_CUDA(cudaMemcpyAsync(cb.data(), P.cells.begin.ptr, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaMemcpyAsync(ce.data(), P.cells.end.ptr, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaMemcpyAsync(ps.data(), P.p2p.src.ptr, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaMemcpyAsync(off.data(), P.p2p.off.ptr, sizeof(int32_t) * (nc + 1), cudaMemcpyDeviceToHost,
                           P.stream));
  FMM_CUDA(cudaStreamSynchronize(P.stream));
  for (int64_t c = 0; c < nc; ++c)
    if (ce[c] - cb[c] > kMaxLeaf && off[c + 1] > off[c]) return;
  // tasks: the pairs (A, B > A) of A's list, in list order; their keys (A, B) -> task index
  std::vector<int32_t> toff(nc + 1, 0), tb;
  std::vector<int64_t> poff;
  std::vector<std::pair<uint64_t, int64_t>> fwd;  // (A << 32 | B, task)
  std::vector<uint64_t> rev;                      // the pairs (L, A < L) as (A << 32 | L)
  int64_t slots = 0;
  for (int64_t A = 0; A < nc; ++A) {
    toff[A] = (int32_t)tb.size();
    for (int k = off[A]; k < off[A + 1]; ++k) {
      const int64_t B = ps[k];
      if (B > A) {
        fwd.emplace_back((uint64_t)A << 32 | (uint64_t)B, (int64_t)tb.size());
        tb.push_back((int32_t)B);
        poff.push_back(slots);
        slots += ce[B] - cb[B];
      } else if (B < A) {
        rev.push_back((uint64_t)B << 32 | (uint64_t)A);
      }
    }
  }
  toff[nc] = (int32_t)tb.size();
  if (slots * 8 > ((int64_t)2 << 30)) return;
  // symmetry: the two key sets are equal (each list holds a source at most once)
  std::vector<std::pair<uint64_t, int64_t>> fs = fwd;
  std::sort(fs.begin(), fs.end());
  std::vector<uint64_t> rs = rev;
  std::sort(rs.begin(), rs.end());
  if (fs.size() != rs.size()) return;
  for (size_t i = 0; i < fs.size(); ++i)
    if (fs[i].first != rs[i] || (i > 0 && fs[i].first == fs[i - 1].first)) return;
  // gather lists: for leaf L, the slots of the tasks (A, L) with A < L, in L's list order
  std::vector<int32_t> goff(nc + 1, 0);
  std::vector<int64_t> gslot;
  gslot.reserve(rev.size());
  size_t r = 0;
  for (int64_t L = 0; L < nc; ++L) {
    goff[L] = (int32_t)gslot.size();
    for (int k = off[L]; k < off[L + 1]; ++k) {
      if (ps[k] >= L) continue;
      const uint64_t key = rev[r++];
      const auto it = std::lower_bound(fs.begin(), fs.end(), std::make_pair(key, (int64_t)-1));
      gslot.push_back(poff[it->second]);
    }
  }
  goff[nc] = (int32_t)gslot.size();
  auto up32 = [&](DevBuf<int32_t>& d, const std::vector<int32_t>& h) {
    d.alloc(std::max<int64_t>(1, (int64_t)h.size()));
    if (!h.empty())
      FMM_CUDA(cudaMemcpyAsync(d.ptr, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice, P.stream));
  };
  auto up64 = [&](DevBuf<int64_t>& d, const std::vector<int64_t>& h) {
    d.alloc(std::max<int64_t>(1, (int64_t)h.size()));
    if (!h.empty())
      FMM_CUDA(cudaMemcpyAsync(d.ptr, h.data(), sizeof(int64_t) * h.size(), cudaMemcpyHostToDevice, P.stream));
  };
  up32(Mu.toff, toff);
  up32(Mu.task_b, tb);
  up64(Mu.poff, poff);
  up32(Mu.goff, goff);
  up64(Mu.gslot, gslot);
  Mu.partial.alloc(std::max<int64_t>(1, slots));
  Mu.own.alloc(std::max<int64_t>(1, P.n));
  Mu.ntasks = (int64_t)tb.size();
  FMM_CUDA(cudaStreamSynchronize(P.stream));  // host vectors die here
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
  m.task_b = Mu.task_b;
  m.poff = Mu.poff;
  m.partial = Mu.partial;
  m.own = Mu.own;
  near_mutual_kernel<<<(unsigned)nl, 32, 0, P.stream>>>(m);
  FMM_LAUNCHED("near_mutual_kernel");
  mutual_out_kernel<<<cdiv(nl, 4), 128, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end, P.cells.center,
                                                       P.pos, P.L, P.p, P.nc, Mu.own, Mu.goff, Mu.gslot, Mu.partial,
                                                       P.perm, std::ldexp(1.0, -P.e), phi);
  FMM_LAUNCHED("mutual_out_kernel");
}

}  // namespace fmm
