// near_warp.cu — S11 L2P(+grad), S12 P2P and S13 un-permute, v2: one WARP per target
// leaf (the direct operator is the dense diagonal block).
//
//  * targets: a leaf with nt <= 32 targets uses G = 32 / pow2ceil(nt) (<= 8) lanes per
//    target, each summing every G-th source, reduced with shuffles; larger leaves run
//    in groups of 64 targets with 2 targets per lane (register blocking);
//  * sources: the source leaves of the P2P list are Morton-contiguous runs of double4
//    (x, y, z, q); each is staged into the warp's shared-memory buffer with cp.async
//    (16 B copies), double-buffered so the next leaf streams in during compute;
//    all lanes of a target group read the same source -> shared-memory broadcast;
//  * 1/r: rsqrt.approx.f64 seed (MUFU) + one third-order correction
//    y1 = y0 (1 + e/2 + 3e^2/8), e = 1 - r^2 y0^2: relative error O(e^3) << 2^-53,
//    5 FP64 ops; r^2 == 0 (self term, coincident points) is tested only in the
//    self-leaf loop, since equal coordinates imply equal keys and the same leaf
//    (R2, R11).
#include <cmath>

#include "harmonics.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kWarps = 4;   // warps (target leaves) per CTA
constexpr int kBuf = 128;   // source particles per staging buffer

__device__ __forceinline__ double rsqrt_fp64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);     // 1 - x y^2
  const double c = e * fma(e, 0.375, 0.5);  // e/2 + 3 e^2/8
  return fma(y, c, y);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// a staging unit: up to kBuf particles of source leaf q (chunk `off` of it)
struct Unit {
  int q, off;
};

template <bool kGrad, bool kCheck, int TPL>
__device__ __forceinline__ void interact(const double4* __restrict__ sb, int ns, int sg, int G, const double3 (&xi)[TPL],
                                         double (&f)[TPL], double3 (&g)[TPL]) {
#pragma unroll 4
  for (int j = sg; j < ns; j += G) {
    const double4 s = sb[j];
#pragma unroll
    for (int k = 0; k < TPL; ++k) {
      const double dx = xi[k].x - s.x, dy = xi[k].y - s.y, dz = xi[k].z - s.z;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      double y = rsqrt_fp64(r2);
      if (kCheck) y = r2 > 0.0 ? y : 0.0;
      if (!kGrad) {
        f[k] = fma(s.w, y, f[k]);
      } else {
        const double qy = s.w * y;
        f[k] += qy;
        const double w = qy * y * y;
        g[k].x = fma(-w, dx, g[k].x);
        g[k].y = fma(-w, dy, g[k].y);
        g[k].z = fma(-w, dz, g[k].z);
      }
    }
  }
}

template <bool kGrad, int TPL>
__device__ void process_group(int leaf, int t0, int cnt, int lane, double4 (*buf)[kBuf],
                              const int32_t* __restrict__ cbeg, const int32_t* __restrict__ cend,
                              const double4* __restrict__ center, const double4* __restrict__ pos,
                              const double2* __restrict__ L, const int32_t* __restrict__ off,
                              const int32_t* __restrict__ src, const uint32_t* __restrict__ perm, int p, int nc,
                              double s_phi, double s_grad, double* __restrict__ phi_out,
                              double* __restrict__ grad_out) {
  // lanes per target (TPL == 1 only): largest power of two with G * cnt <= 32, at most 8
  int G = 1;
  if (TPL == 1) {
    while (G < 8 && 2 * G * cnt <= 32) G *= 2;
  }
  const int tl = lane / G, sg = lane - tl * G;
  double3 xi[TPL];
  double f[TPL];
  double3 g[TPL];
  bool act[TPL];
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    const int t = tl + 32 * k;
    act[k] = t < cnt;
    const double4 v = act[k] ? pos[t0 + t] : make_double4(0, 0, 0, 0);
    xi[k] = make_double3(v.x, v.y, v.z);
    f[k] = 0.0;
    g[k] = make_double3(0, 0, 0);
  }
  const int q0 = off[leaf], q1 = off[leaf + 1];
  // staging pipeline over units (source leaf q, chunk offset)
  auto stage = [&](Unit u, int b) {
    const int sl = src[u.q];
    const int sb = cbeg[sl] + u.off;
    const int n = min(kBuf, cend[sl] - sb);
    const double* gsrc = (const double*)(pos + sb);
    double* dst = (double*)buf[b];
    for (int h = lane; h < 2 * n; h += 32) cp_async16(dst + 2 * h, gsrc + 2 * h);
    cp_commit();
  };
  auto next = [&](Unit u) {
    const int sl = src[u.q];
    if (u.off + kBuf < cend[sl] - cbeg[sl]) return Unit{u.q, u.off + kBuf};
    return Unit{u.q + 1, 0};
  };
  if (q0 < q1) {
    Unit u{q0, 0};
    stage(u, 0);
    int b = 0;
    while (u.q < q1) {
      const Unit un = next(u);
      if (un.q < q1) {
        stage(un, b ^ 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncwarp();
      const int sl = src[u.q];
      const int ns = min(kBuf, cend[sl] - cbeg[sl] - u.off);
      if (sl == leaf)
        interact<kGrad, true, TPL>(buf[b], ns, sg, G, xi, f, g);
      else
        interact<kGrad, false, TPL>(buf[b], ns, sg, G, xi, f, g);
      __syncwarp();  // buffer b is rewritten two units later
      u = un;
      b ^= 1;
    }
  }
  // reduce the G partial sums of each target
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
  if (sg != 0) return;
  const double4 c = center[leaf];
  const double2* Lc = L + (int64_t)leaf * nc;
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    if (!act[k]) continue;
    l2p_eval<kGrad>(Lc, p, xi[k].x - c.x, xi[k].y - c.y, xi[k].z - c.z, f[k], g[k]);
    const int64_t o = perm[t0 + tl + 32 * k];
    phi_out[o] = f[k] * s_phi;
    if (kGrad) {
      grad_out[3 * o] = g[k].x * s_grad;
      grad_out[3 * o + 1] = g[k].y * s_grad;
      grad_out[3 * o + 2] = g[k].z * s_grad;
    }
  }
}

template <bool kGrad>
__global__ void __launch_bounds__(32 * kWarps) near_warp_kernel(
    const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ cbeg,
    const int32_t* __restrict__ cend, const double4* __restrict__ center, const double4* __restrict__ pos,
    const double2* __restrict__ L, const int32_t* __restrict__ off, const int32_t* __restrict__ src,
    const uint32_t* __restrict__ perm, int p, int nc, double s_phi, double s_grad, double* __restrict__ phi_out,
    double* __restrict__ grad_out) {
  __shared__ __align__(16) double4 buf[kWarps][2][kBuf];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t li = (int64_t)blockIdx.x * kWarps + warp;
  if (li >= nleaves) return;  // warp-uniform; no block-level barriers below
  const int leaf = leaves[li];
  const int tb = cbeg[leaf], te = cend[leaf];
  if (te - tb <= 32) {
    process_group<kGrad, 1>(leaf, tb, te - tb, lane, buf[warp], cbeg, cend, center, pos, L, off, src, perm, p, nc,
                            s_phi, s_grad, phi_out, grad_out);
  } else {
    for (int t0 = tb; t0 < te; t0 += 64)
      process_group<kGrad, 2>(leaf, t0, min(64, te - t0), lane, buf[warp], cbeg, cend, center, pos, L, off, src,
                              perm, p, nc, s_phi, s_grad, phi_out, grad_out);
  }
}

}  // namespace

void near_pass_warp(fmm_plan_s& P, double* phi, double* grad) {
  const int64_t nl = P.own_leaf_end - P.own_leaf_begin;
  if (nl <= 0) return;
  const double s_phi = std::ldexp(1.0, -P.e), s_grad = std::ldexp(1.0, -2 * P.e);
  const int32_t* leaves = P.leaves.ptr + P.own_leaf_begin;
  const unsigned grid = cdiv(nl, kWarps);
  if (grad)
    near_warp_kernel<true><<<grid, 32 * kWarps, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end,
                                                               P.cells.center, P.pos, P.L, P.p2p.off, P.p2p.src,
                                                               P.perm, P.p, P.nc, s_phi, s_grad, phi, grad);
  else
    near_warp_kernel<false><<<grid, 32 * kWarps, 0, P.stream>>>(leaves, nl, P.cells.begin, P.cells.end,
                                                                P.cells.center, P.pos, P.L, P.p2p.off, P.p2p.src,
                                                                P.perm, P.p, P.nc, s_phi, s_grad, phi, grad);
  FMM_LAUNCHED("near_warp_kernel");
}

}  // namespace fmm
