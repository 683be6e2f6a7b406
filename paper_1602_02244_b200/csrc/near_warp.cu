// near_warp.cu — S11 L2P(+grad), S12 P2P and S13 un-permute, v2: one WARP per target
// leaf (the direct operator is the dense diagonal block).
//
//  * lane layout per leaf: nt targets are covered by (32 / G) target groups of G lanes,
//    each lane holding TPL targets in registers (G in {1,2,4,8}, TPL <= 4), chosen per
//    leaf to minimise the idle slots (32 / G) * TPL - nt; the G lanes of a group split
//    the sources (every G-th one) and are reduced with a butterfly at the end, so every
//    lane of the group holds the full sums and the L2P evaluations are spread over them;
//  * sources: the leaf's P2P source leaves are Morton-contiguous runs of double4
//    (x, y, z, q); consecutive list entries are packed into staging units of up to
//    kBuf particles (the self leaf always alone, it alone needs the r^2 == 0 test),
//    copied into the warp's shared-memory buffer with cp.async (16 B pieces) and
//    double-buffered so the next unit streams in during compute; the lanes of a
//    group read distinct sources, the groups the same ones (shared-memory broadcast);
//  * 1/r: rsqrt.approx.f64 seed (MUFU) + one third-order correction
//    y1 = y0 (1 + e/2 + 3e^2/8), e = 1 - r^2 y0^2: relative error O(e^3) << 2^-53,
//    5 FP64 ops; r^2 == 0 (self term, coincident points) is tested only in the
//    self-leaf unit, since equal coordinates imply equal keys and the same leaf
//    (R2, R11).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "harmonics.cuh"
#include "near_common.cuh"
#include "plan.h"

namespace fmm {
namespace {
using namespace near;

#ifndef FMM_NEAR_WARPS
#define FMM_NEAR_WARPS 1
#endif
#ifndef FMM_NEAR_MINB_GRAD
#define FMM_NEAR_MINB_GRAD (12 / FMM_NEAR_WARPS)  // 12 warps per SM for the phi + grad kernel
#endif
#ifndef FMM_NEAR_BUF
#define FMM_NEAR_BUF 128
#endif
constexpr int kWarps = FMM_NEAR_WARPS;  // warps (target leaves) per CTA: 1 (20 CTAs per SM) beat 4 and 2
                                        // (configs[2] near 2.66 -> 2.59 ms, [3] 13.4 -> 11.9, [4] 254.5 -> 239.1)
constexpr int kBuf = FMM_NEAR_BUF;      // source particles per staging buffer
#ifndef FMM_NEAR_TPL_MAX
#define FMM_NEAR_TPL_MAX 4
#endif
constexpr int kMaxTPL = FMM_NEAR_TPL_MAX;  // targets per lane (measured: 8 is slower, register pressure)
template <bool kGrad>
constexpr int max_tpl() { return kMaxTPL; }
#ifndef FMM_NEAR_MINB
#define FMM_NEAR_MINB 20  // CTAs (1 warp each) per SM for the phi-only kernel (96 registers, no spills)
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// A staging unit: list entries [qa, qb) from particle `off` of entry qa (off > 0 only
// for a leaf larger than kBuf, which is then a unit of its own), n particles in total.
struct Unit {
  int qa, qb, off, n;
  bool self;
};

struct NearArgs {
  const int32_t* cbeg;
  const int32_t* cend;
  const double4* center;
  const double4* pos;
  const double2* L;
  const int32_t* off;
  const int32_t* src;
  const uint32_t* perm;
  int p, nc;
  double s_phi, s_grad;
  double* phi_out;
  double* grad_out;
  int max_tpl, max_g;  // layout limits (tuning; defaults max_tpl<kGrad>(), 8)
  int64_t out_base;    // perm == nullptr: results at (sorted position - out_base) (LET, owned order)
  bool p2p_only;       // write the P2P sums (sorted order, unscaled) and skip L2P (overlapped near field)
};

// Targets [t0, t0 + cnt) of `leaf` as (32 / G) groups x TPL targets per lane.
template <bool kGrad, int TPL>
__device__ void process_group(const NearArgs& a, int leaf, int t0, int cnt, int G, int lane, double4 (*buf)[kBuf]) {
  const int tl = lane / G, sg = lane - tl * G, ngrp = 32 / G;
  double3 xi[TPL];
  double f[TPL];
  double3 g[TPL];
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    const int t = tl + ngrp * k;
    const double4 v = t < cnt ? a.pos[t0 + t] : make_double4(0, 0, 0, 0);
    xi[k] = make_double3(v.x, v.y, v.z);
    f[k] = 0.0;
    g[k] = make_double3(0, 0, 0);
  }
  const int q0 = a.off[leaf], q1 = a.off[leaf + 1];
  // the first 32 list entries' source ranges, one per lane, loaded once (no dependent
  // global loads on the staging path); later entries are read when needed
  int my_sl = -1, my_b = 0, my_e = 0;
  if (q0 + lane < q1) {
    my_sl = a.src[q0 + lane];
    my_b = a.cbeg[my_sl];
    my_e = a.cend[my_sl];
  }
  // Build and issue (cp.async) the unit starting at (qa, off) into buffer b.
  auto stage = [&](int qa, int off, int b) -> Unit {
    Unit u{qa, qa, off, 0, false};
    double* dst = (double*)buf[b];
    for (int q = qa; q < q1; ++q) {
      int sl, sb0, se;
      if (q - q0 < 32) {
        sl = __shfl_sync(0xffffffffu, my_sl, q - q0);
        sb0 = __shfl_sync(0xffffffffu, my_b, q - q0);
        se = __shfl_sync(0xffffffffu, my_e, q - q0);
      } else {
        sl = a.src[q];
        sb0 = a.cbeg[sl];
        se = a.cend[sl];
      }
      const int sb = sb0 + (q == qa ? off : 0);
      const int sz = se - sb;
      const bool self = sl == leaf;
      if (q > qa && (self || sz > kBuf - u.n)) break;  // the unit is full / the self leaf goes alone
      const int n = min(kBuf - u.n, sz);
      const double* gsrc = (const double*)(a.pos + sb);
      for (int h = lane; h < 2 * n; h += 32) cp_async16(dst + 4 * u.n + 2 * h, gsrc + 2 * h);
      u.n += n;
      u.qb = q + 1;
      u.self = self;
      if (self || n < sz) {  // self leaf alone; an oversized leaf continues in the next unit
        if (n < sz) u.qb = q;
        break;
      }
    }
    cp_commit();
    return u;
  };
  auto next_of = [&](const Unit& u) -> int2 {  // (qa, off) after u
    if (u.qb == u.qa) return make_int2(u.qa, u.off + u.n);  // partial oversized leaf
    return make_int2(u.qb, 0);
  };
  int qa = q0, off = 0, b = 0;
  if (qa < q1) {
    Unit u = stage(qa, off, 0);
    while (true) {
      const int2 nx = next_of(u);
      Unit un{0, 0, 0, 0, false};
      const bool more = nx.x < q1;
      if (more) {
        un = stage(nx.x, nx.y, b ^ 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncwarp();
      if (u.self)
        interact<kGrad, true, TPL>(buf[b], u.n, sg, G, xi, f, g);
      else
        interact<kGrad, false, TPL>(buf[b], u.n, sg, G, xi, f, g);
      __syncwarp();  // buffer b is rewritten by the unit after next
      if (!more) break;
      u = un;
      b ^= 1;
    }
  }
  // butterfly over the G lanes of each group: every lane ends with the group's sums
  for (int o = 1; o < G; o <<= 1) {
#pragma unroll
    for (int k = 0; k < TPL; ++k) {
      f[k] += __shfl_xor_sync(0xffffffffu, f[k], o);
      if (kGrad) {
        g[k].x += __shfl_xor_sync(0xffffffffu, g[k].x, o);
        g[k].y += __shfl_xor_sync(0xffffffffu, g[k].y, o);
        g[k].z += __shfl_xor_sync(0xffffffffu, g[k].z, o);
      }
    }
  }
  // L2P + store: lane sg of a group evaluates its targets k = sg, sg + G, ...
  const double4 c = a.center[leaf];
  const double2* Lc = a.L + (int64_t)leaf * a.nc;
  for (int k0 = 0; k0 < TPL; k0 += G) {
    const int kk = k0 + sg;
    double3 x = make_double3(0, 0, 0), gg = make_double3(0, 0, 0);
    double ff = 0.0;
#pragma unroll
    for (int k = 0; k < TPL; ++k)
      if (k == kk) {
        x = xi[k];
        ff = f[k];
        gg = g[k];
      }
    const int t = tl + ngrp * kk;
    if (kk < TPL && t < cnt) {
      if (a.p2p_only) {  // P2P sums only (sorted order, unscaled): L2P later, in l2p_out_kernel
        a.phi_out[t0 + t] = ff;
        if (kGrad) {
          a.grad_out[3 * (t0 + t)] = gg.x;
          a.grad_out[3 * (t0 + t) + 1] = gg.y;
          a.grad_out[3 * (t0 + t) + 2] = gg.z;
        }
        continue;
      }
      l2p_eval<kGrad>(Lc, a.p, x.x - c.x, x.y - c.y, x.z - c.z, ff, gg);
      const int64_t o = a.perm ? (int64_t)a.perm[t0 + t] : (int64_t)(t0 + t) - a.out_base;
      a.phi_out[o] = ff * a.s_phi;
      if (kGrad) {
        a.grad_out[3 * o] = gg.x * a.s_grad;
        a.grad_out[3 * o + 1] = gg.y * a.s_grad;
        a.grad_out[3 * o + 2] = gg.z * a.s_grad;
      }
    }
  }
}

template <bool kGrad>
__device__ __forceinline__ void dispatch(const NearArgs& a, int leaf, int t0, int cnt, int G, int TPL, int lane,
                                         double4 (*buf)[kBuf]) {
  switch (TPL) {
    case 1: process_group<kGrad, 1>(a, leaf, t0, cnt, G, lane, buf); break;
    case 2: process_group<kGrad, 2>(a, leaf, t0, cnt, G, lane, buf); break;
    case 3: process_group<kGrad, 3>(a, leaf, t0, cnt, G, lane, buf); break;
    case 4: process_group<kGrad, 4>(a, leaf, t0, cnt, G, lane, buf); break;
#if FMM_NEAR_TPL_MAX >= 5
    case 5: process_group<kGrad, 5>(a, leaf, t0, cnt, G, lane, buf); break;
#endif
#if FMM_NEAR_TPL_MAX >= 6
    case 6: process_group<kGrad, 6>(a, leaf, t0, cnt, G, lane, buf); break;
#endif
  }
}

template <bool kGrad>
__global__ void __launch_bounds__(32 * kWarps, kGrad ? FMM_NEAR_MINB_GRAD : FMM_NEAR_MINB) near_warp_kernel(const int32_t* __restrict__ leaves, int64_t nleaves,
                                                                const NearArgs a) {
  __shared__ __align__(16) double4 buf[kWarps][2][kBuf];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t li = (int64_t)blockIdx.x * kWarps + warp;
  if (li >= nleaves) return;  // warp-uniform; no block-level barriers below
  const int leaf = leaves[li];
  const int tb = a.cbeg[leaf], te = a.cend[leaf];
  int G, TPL;
  choose_layout(te - tb, a.max_tpl, a.max_g, G, TPL);
  if (TPL > 0) {
    dispatch<kGrad>(a, leaf, tb, te - tb, G, TPL, lane, buf[warp]);
  } else {  // more than 32 * kMaxTPL targets: groups of 32 * kMaxTPL, one lane per target
    constexpr int T = max_tpl<kGrad>();
    for (int t0 = tb; t0 < te; t0 += 32 * T) process_group<kGrad, T>(a, leaf, t0, min(32 * T, te - t0), 1, lane, buf[warp]);
  }
}

// P2P of the leaves not yet taken by the near warps fused into the M2L kernel: warps pull
// leaf indices from the same counter; results (unscaled, sorted order) to phi / grad.
template <bool kGrad>
__global__ void __launch_bounds__(128) p2p_tail_kernel(const int32_t* __restrict__ leaves, int64_t nleaves,
                                                       int* __restrict__ counter, const int32_t* __restrict__ cbeg,
                                                       const int32_t* __restrict__ cend, const int32_t* __restrict__ off,
                                                       const int32_t* __restrict__ src, const double4* __restrict__ pos,
                                                       double* __restrict__ phi, double* __restrict__ grad) {
  const int lane = threadIdx.x & 31;
  while (true) {
    int li = 0;
    if (lane == 0) li = atomicAdd(counter, 1);
    li = __shfl_sync(0xffffffffu, li, 0);
    if (li >= nleaves) return;
    p2p_leaf_global<kGrad, 4>(cbeg, cend, off, src, pos, leaves[li], lane, phi, grad);
  }
}

// L2P (+grad) of every target of the leaves, added to the P2P results, exact 2^-e rescale,
// scatter to caller order (or owned order, perm == nullptr). Warp per leaf, lane per target.
template <bool kGrad>
__global__ void __launch_bounds__(128) l2p_out_kernel(const int32_t* __restrict__ leaves, int64_t nleaves,
                                                      const int32_t* __restrict__ cbeg, const int32_t* __restrict__ cend,
                                                      const double4* __restrict__ center,
                                                      const double4* __restrict__ pos, const double2* __restrict__ L,
                                                      int p, int nc, const double* __restrict__ p2p_phi,
                                                      const double* __restrict__ p2p_grad,
                                                      const uint32_t* __restrict__ perm, int64_t out_base, double s_phi,
                                                      double s_grad, double* __restrict__ phi_out,
                                                      double* __restrict__ grad_out) {
  const int lane = threadIdx.x & 31;
  const int64_t li = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (li >= nleaves) return;
  const int leaf = leaves[li];
  const double4 c = center[leaf];
  const double2* Lc = L + (int64_t)leaf * nc;
  for (int t = cbeg[leaf] + lane; t < cend[leaf]; t += 32) {
    const double4 x = pos[t];
    double f = p2p_phi[t];
    double3 g = kGrad ? make_double3(p2p_grad[3 * t], p2p_grad[3 * t + 1], p2p_grad[3 * t + 2]) : make_double3(0, 0, 0);
    l2p_eval<kGrad>(Lc, p, x.x - c.x, x.y - c.y, x.z - c.z, f, g);
    const int64_t o = perm ? (int64_t)perm[t] : (int64_t)t - out_base;
    phi_out[o] = f * s_phi;
    if (kGrad) {
      grad_out[3 * o] = g.x * s_grad;
      grad_out[3 * o + 1] = g.y * s_grad;
      grad_out[3 * o + 2] = g.z * s_grad;
    }
  }
}

}  // namespace

void near_fused_prepare(fmm_plan_s& P, bool grad) {
  if (P.near_p2p_phi.count < P.n) P.near_p2p_phi.alloc(P.n);
  if (grad && P.near_p2p_grad.count < 3 * P.n) P.near_p2p_grad.alloc(3 * P.n);
  if (!P.near_counter.ptr) P.near_counter.alloc(1);
  FMM_CUDA(cudaMemsetAsync(P.near_counter.ptr, 0, sizeof(int), P.stream));
}

void near_fused_finish(fmm_plan_s& P, double* phi, double* grad) {
  const int64_t nl = P.own_leaf_end - P.own_leaf_begin;
  if (nl <= 0) return;
  const int32_t* leaves = P.leaves.ptr + P.own_leaf_begin;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(nl, 4), 148 * 8);
  if (grad)
    p2p_tail_kernel<true><<<grid, 128, 0, P.stream>>>(leaves, nl, P.near_counter, P.cells.begin, P.cells.end,
                                                       P.p2p.off, P.p2p.src, P.pos, P.near_p2p_phi, P.near_p2p_grad);
  else
    p2p_tail_kernel<false><<<grid, 128, 0, P.stream>>>(leaves, nl, P.near_counter, P.cells.begin, P.cells.end,
                                                        P.p2p.off, P.p2p.src, P.pos, P.near_p2p_phi, nullptr);
  FMM_LAUNCHED("p2p_tail_kernel");
  const uint32_t* perm = P.near_compact_out ? nullptr : P.perm.ptr;
  const double s_phi = std::ldexp(1.0, -P.e), s_grad = std::ldexp(1.0, -2 * P.e);
  if (grad)
    l2p_out_kernel<true><<<cdiv(nl, 4), 128, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end, P.cells.center,
                                                            P.pos, P.L, P.p, P.nc, P.near_p2p_phi, P.near_p2p_grad,
                                                            perm, P.own_begin, s_phi, s_grad, phi, grad);
  else
    l2p_out_kernel<false><<<cdiv(nl, 4), 128, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end,
                                                             P.cells.center, P.pos, P.L, P.p, P.nc, P.near_p2p_phi,
                                                             nullptr, perm, P.own_begin, s_phi, s_grad, phi, nullptr);
  FMM_LAUNCHED("l2p_out_kernel");
}

namespace {
void near_launch(fmm_plan_s& P, double* phi, double* grad, bool p2p_only, cudaStream_t stream) {
  const int64_t nl = P.own_leaf_end - P.own_leaf_begin;
  if (nl <= 0) return;
  NearArgs a;
  a.p2p_only = p2p_only;
  a.cbeg = P.cells.begin;
  a.cend = P.cells.end;
  a.center = P.cells.center;
  a.pos = P.pos;
  a.L = P.L;
  a.off = P.p2p.off;
  a.src = P.p2p.src;
  a.perm = P.near_compact_out ? nullptr : P.perm.ptr;
  a.out_base = P.own_begin;
  if (p2p_only) {  // sorted order, unscaled
    a.perm = nullptr;
    a.out_base = 0;
  }
  a.p = P.p;
  a.nc = P.nc;
  a.s_phi = std::ldexp(1.0, -P.e);
  a.s_grad = std::ldexp(1.0, -2 * P.e);
  a.phi_out = phi;
  a.grad_out = grad;
  a.max_tpl = grad ? max_tpl<true>() : max_tpl<false>();
  // few sources per target (< 1,200 interactions per particle, e.g. configs[3] at 849): four
  // targets per lane loses to three (near 13.4 vs 14.6 ms); configs[1], [2], [4] (1,641 - 2,256)
  // keep four (configs[2] 2.66 vs 2.72 ms)
  if (P.n > 0 && P.n_p2p_interactions < 1200LL * P.n) a.max_tpl = std::min(a.max_tpl, 3);
  a.max_g = 8;
  if (const char* e = getenv("FMM_NEAR_MAXTPL")) a.max_tpl = std::max(1, std::min(a.max_tpl, atoi(e)));
  if (const char* e = getenv("FMM_NEAR_MAXG")) a.max_g = std::max(1, std::min(8, atoi(e)));
  const int32_t* leaves = P.leaves.ptr + P.own_leaf_begin;
  const unsigned grid = cdiv(nl, kWarps);
  if (grad)
    near_warp_kernel<true><<<grid, 32 * kWarps, 0, stream>>>(leaves, nl, a);
  else
    near_warp_kernel<false><<<grid, 32 * kWarps, 0, stream>>>(leaves, nl, a);
  FMM_LAUNCHED("near_warp_kernel");
}
}  // namespace

void near_pass_warp(fmm_plan_s& P, double* phi, double* grad) { near_launch(P, phi, grad, false, P.stream); }

// overlapped near field: the P2P sums on a second stream while the far field
// (upward, M2L, L2L) runs, then L2P + rescale + scatter to caller order once L is complete
void near_p2p_async(fmm_plan_s& P, bool grad, cudaStream_t stream) {
  if (P.near_p2p_phi.count < P.n) P.near_p2p_phi.alloc(P.n);
  if (grad && P.near_p2p_grad.count < 3 * P.n) P.near_p2p_grad.alloc(3 * P.n);
  near_launch(P, P.near_p2p_phi, grad ? P.near_p2p_grad.ptr : nullptr, true, stream);
}

void near_l2p_out(fmm_plan_s& P, double* phi, double* grad) {
  const int64_t nl = P.own_leaf_end - P.own_leaf_begin;
  if (nl <= 0) return;
  const int32_t* leaves = P.leaves.ptr + P.own_leaf_begin;
  const uint32_t* perm = P.near_compact_out ? nullptr : P.perm.ptr;
  const double s_phi = std::ldexp(1.0, -P.e), s_grad = std::ldexp(1.0, -2 * P.e);
  if (grad)
    l2p_out_kernel<true><<<cdiv(nl, 4), 128, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end, P.cells.center,
                                                            P.pos, P.L, P.p, P.nc, P.near_p2p_phi, P.near_p2p_grad,
                                                            perm, P.own_begin, s_phi, s_grad, phi, grad);
  else
    l2p_out_kernel<false><<<cdiv(nl, 4), 128, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end,
                                                             P.cells.center, P.pos, P.L, P.p, P.nc, P.near_p2p_phi,
                                                             nullptr, perm, P.own_begin, s_phi, s_grad, phi, nullptr);
  FMM_LAUNCHED("l2p_out_kernel");
}

}  // namespace fmm
