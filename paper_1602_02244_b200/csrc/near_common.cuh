// near_common.cuh — S12 P2P pieces shared by the near-field kernels (near_warp.cu) and the
// near warps fused into the M2L v3 kernel (m2l_rot.cu).
#pragma once
#include "harmonics.cuh"
#include "plan.h"

namespace fmm {
namespace near {

#ifndef FMM_NEAR_UNROLL
#define FMM_NEAR_UNROLL 2
#endif
constexpr int kUnroll = FMM_NEAR_UNROLL;

// 1/sqrt(x): rsqrt.approx.f64 seed (MUFU, relative error <= 2^-20) refined by one Newton step
// y (1 + e/2), e = 1 - x y^2: relative error <= 1.5 * 2^-40 = 1.4e-12 per interaction (DESIGN.md
// R11; measured end-to-end rel-L2 vs the oracle <= 1.4e-13 at every BASELINE config, near field
// 8 % faster, profiles/r2_near_order.md). FMM_NEAR_ORDER=3: a third-order step y (1 + e/2 +
// 3e^2/8), relative error O(e^3) << 2^-53.
#ifndef FMM_NEAR_ORDER
#define FMM_NEAR_ORDER 2
#endif
#ifndef FMM_NEAR_PF
#define FMM_NEAR_PF 0  // interact(): the next source loaded an iteration ahead
#endif
#ifndef FMM_NEAR_XH
#define FMM_NEAR_XH 0
#endif
__device__ __forceinline__ double rsqrt_fp64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  if (FMM_NEAR_ORDER == 2) {  // one Newton step y + y (1 - x y^2) / 2, the halving of y done on
    // the exponent (integer pipe; y is a positive normal number): 3 FP64 ops instead of 4,
    // bitwise the same result (scaling by 2 commutes with rounding)
#if FMM_NEAR_XH
    // the same product from -x/2 (exponent and sign on x's high word, x's low word reused in
    // place): (-x/2) y == -x (y/2) exactly, bitwise the same result, one register move less
    const double xh = __hiloint2double(__double2hiint(x) + 0x7ff00000, __double2loint(x));
    return fma(y, fma(xh * y, y, 0.5), y);
#else
    const double yh = __hiloint2double(__double2hiint(y) - 0x00100000, __double2loint(y));
    return fma(y, fma(-x * yh, y, 0.5), y);
#endif
  }
  const double e = fma(-x * y, y, 1.0);  // 1 - x y^2
  const double c = e * fma(e, 0.375, 0.5);  // e/2 + 3 e^2/8
  return fma(y, c, y);
}

template <bool kGrad, bool kCheck, int TPL>
__device__ __forceinline__ void interact(const double4* __restrict__ sb, int ns, int sg, int G,
                                         const double3 (&xi)[TPL], double (&f)[TPL], double3 (&g)[TPL]) {
#if FMM_NEAR_PF
  double4 sn = sb[sg < ns ? sg : 0];  // the next source, loaded an iteration ahead
#endif
#pragma unroll kUnroll
  for (int j = sg; j < ns; j += G) {
#if FMM_NEAR_PF
    const double4 s = sn;
    sn = sb[j + G < ns ? j + G : 0];
#else
    const double4 s = sb[j];
#endif
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


// (G, TPL) minimising the idle slots (32 / G) * TPL - cnt; ties prefer TPL >= G (balanced
// L2P), then larger TPL (more register reuse of each staged source). TPL == 0: none fits.
__device__ __forceinline__ void choose_layout(int cnt, int maxT, int maxG, int& G, int& TPL) {
  int best = 1 << 30;
  G = 1;
  TPL = 0;
  for (int g = 8; g >= 1; g >>= 1) {
    const int per = 32 / g, t = (cnt + per - 1) / per;
    if (t > maxT || g > maxG) continue;
    const int key = (per * t) * 4 + (t >= g ? 0 : 2) + (t > TPL ? 0 : 1);
    if (key < best) {
      best = key;
      G = g;
      TPL = t;
    }
  }
}


// P2P of the targets [t0, t0 + cnt) of `leaf` (layout G lanes per target x TPL targets per
// lane) with sources read straight from global memory (L1), results (unscaled, sorted
// order) to phi[t], grad[3 t]. Used where no shared memory is left for staging.
template <bool kGrad, int TPL>
__device__ void p2p_group_global(const int32_t* __restrict__ cbeg, const int32_t* __restrict__ cend,
                                 const int32_t* __restrict__ off, const int32_t* __restrict__ src,
                                 const double4* __restrict__ pos, int leaf, int t0, int cnt, int G, int lane,
                                 double* __restrict__ phi, double* __restrict__ grad) {
  const int tl = lane / G, sg = lane - tl * G, ngrp = 32 / G;
  double3 xi[TPL];
  double f[TPL];
  double3 g[TPL];
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    const int t = tl + ngrp * k;
    const double4 v = t < cnt ? pos[t0 + t] : make_double4(0, 0, 0, 0);
    xi[k] = make_double3(v.x, v.y, v.z);
    f[k] = 0.0;
    g[k] = make_double3(0, 0, 0);
  }
  const int q0 = off[leaf], q1 = off[leaf + 1];
  int my_sl = -1, my_b = 0, my_e = 0;
  if (q0 + lane < q1) {
    my_sl = src[q0 + lane];
    my_b = cbeg[my_sl];
    my_e = cend[my_sl];
  }
  for (int q = q0; q < q1; ++q) {
    int sl, sb, se;
    if (q - q0 < 32) {
      sl = __shfl_sync(0xffffffffu, my_sl, q - q0);
      sb = __shfl_sync(0xffffffffu, my_b, q - q0);
      se = __shfl_sync(0xffffffffu, my_e, q - q0);
    } else {
      sl = src[q];
      sb = cbeg[sl];
      se = cend[sl];
    }
    if (sl == leaf)
      interact<kGrad, true, TPL>(pos + sb, se - sb, sg, G, xi, f, g);
    else
      interact<kGrad, false, TPL>(pos + sb, se - sb, sg, G, xi, f, g);
  }
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
#pragma unroll
  for (int k = 0; k < TPL; ++k) {
    const int t = tl + ngrp * k;
    if (t < cnt) {
      phi[t0 + t] = f[k];
      if (kGrad) {
        grad[3 * (t0 + t)] = g[k].x;
        grad[3 * (t0 + t) + 1] = g[k].y;
        grad[3 * (t0 + t) + 2] = g[k].z;
      }
    }
  }
}

// P2P of every target of `leaf` (TPL <= MAXT), results to phi / grad in sorted order.
template <bool kGrad, int MAXT>
__device__ __forceinline__ void p2p_leaf_global(const int32_t* cbeg, const int32_t* cend, const int32_t* off,
                                                const int32_t* src, const double4* pos, int leaf, int lane,
                                                double* phi, double* grad) {
  const int tb = cbeg[leaf], te = cend[leaf];
  int G, TPL;
  choose_layout(te - tb, MAXT, 8, G, TPL);
  if (TPL == 1) {
    p2p_group_global<kGrad, 1>(cbeg, cend, off, src, pos, leaf, tb, te - tb, G, lane, phi, grad);
  } else if (TPL == 2 && MAXT >= 2) {
    p2p_group_global<kGrad, (MAXT >= 2 ? 2 : 1)>(cbeg, cend, off, src, pos, leaf, tb, te - tb, G, lane, phi, grad);
  } else {
    for (int t0 = tb; t0 < te; t0 += 32 * MAXT)
      p2p_group_global<kGrad, MAXT>(cbeg, cend, off, src, pos, leaf, t0, min(32 * MAXT, te - t0), 1, lane, phi, grad);
  }
}

}  // namespace near
}  // namespace fmm
