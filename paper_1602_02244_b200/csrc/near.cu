// near.cu — matvec steps S11 (L2P + gradient), S12 (P2P near field) and S13
// (un-permute to caller order), fused in one kernel per target leaf; plus the
// charge gather and the O(N^2) fmm_direct check kernel.
//
// Paper: "the dense diagonal blocks ... are simply storing the direct operator
// (Green's function) in FMM": P2P evaluates those blocks
// matrix-free. North_star (5): source leaves tiled through shared memory,
// double4 (x, y, z, q) vector loads, rsqrt-based accumulation.
#include <cmath>

#include "harmonics.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kNearThreads = 128;

__global__ void gather_charges_kernel(const double* __restrict__ q, const uint32_t* __restrict__ perm, int64_t n,
                                      double4* __restrict__ pos, int32_t* __restrict__ flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < n) {
    double v = q[perm[i]];
    bad = !isfinite(v);
    pos[i].w = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
}

// One block per target leaf (of this rank's range): L2P, then P2P over the
// leaf's source leaves staged through shared memory, then the exact 2^-e
// un-normalisation and the scatter back to caller order.
template <bool kGrad>
__global__ void __launch_bounds__(kNearThreads) near_kernel(
    const int32_t* __restrict__ leaves, const int32_t* __restrict__ cbeg, const int32_t* __restrict__ cend,
    const double4* __restrict__ center, const double4* __restrict__ pos, const double2* __restrict__ L,
    const int32_t* __restrict__ off, const int32_t* __restrict__ src, const uint32_t* __restrict__ perm, int p,
    int nc, double s_phi, double s_grad, double* __restrict__ phi_out, double* __restrict__ grad_out) {
  extern __shared__ double2 shL[];  // [nc]
  __shared__ double4 tile[kNearThreads];
  const int leaf = leaves[blockIdx.x];
  const int32_t tb = cbeg[leaf], te = cend[leaf];
  const double4 c = center[leaf];
  for (int t = threadIdx.x; t < nc; t += blockDim.x) shL[t] = L[(int64_t)leaf * nc + t];
  const int q0 = off[leaf], q1 = off[leaf + 1];
  __syncthreads();
  for (int32_t base = tb; base < te; base += kNearThreads) {
    const int32_t i = base + threadIdx.x;
    const bool active = i < te;
    const double4 xi = active ? pos[i] : make_double4(0, 0, 0, 0);
    double f = 0.0;
    double3 g = make_double3(0, 0, 0);
    if (active) l2p_eval<kGrad>(shL, p, xi.x - c.x, xi.y - c.y, xi.z - c.z, f, g);
    for (int q = q0; q < q1; ++q) {
      const int sl = src[q];
      const int32_t sb = cbeg[sl], se = cend[sl];
      for (int32_t s0 = sb; s0 < se; s0 += kNearThreads) {
        const int cnt = min(kNearThreads, se - s0);
        __syncthreads();
        if (threadIdx.x < cnt) tile[threadIdx.x] = pos[s0 + threadIdx.x];
        __syncthreads();
        if (active) {
          for (int k = 0; k < cnt; ++k) {
            const double4 sj = tile[k];
            const double dx = xi.x - sj.x, dy = xi.y - sj.y, dz = xi.z - sj.z;
            const double r2 = dx * dx + dy * dy + dz * dz;
            const double rinv = r2 > 0.0 ? rsqrt(r2) : 0.0;  // R2: r^2 == 0 contributes nothing
            const double qr = sj.w * rinv;
            f += qr;
            if (kGrad) {
              const double qr3 = qr * rinv * rinv;
              g.x -= qr3 * dx;
              g.y -= qr3 * dy;
              g.z -= qr3 * dz;
            }
          }
        }
      }
    }
    if (active) {
      const int64_t o = perm[i];
      phi_out[o] = f * s_phi;
      if (kGrad) {
        grad_out[3 * o] = g.x * s_grad;
        grad_out[3 * o + 1] = g.y * s_grad;
        grad_out[3 * o + 2] = g.z * s_grad;
      }
    }
  }
}

constexpr int kDirectThreads = 256;

template <bool kGrad>
__global__ void __launch_bounds__(kDirectThreads) direct_kernel(const double* __restrict__ src,
                                                               const double* __restrict__ q, int64_t ns,
                                                               const double* __restrict__ tgt, int64_t nt,
                                                               double* __restrict__ phi, double* __restrict__ grad) {
  __shared__ double4 tile[kDirectThreads];
  const int64_t i = (int64_t)blockIdx.x * kDirectThreads + threadIdx.x;
  const bool active = i < nt;
  double xi = 0, yi = 0, zi = 0;
  if (active) {
    xi = tgt[3 * i];
    yi = tgt[3 * i + 1];
    zi = tgt[3 * i + 2];
  }
  double f = 0, gx = 0, gy = 0, gz = 0;
  for (int64_t s0 = 0; s0 < ns; s0 += kDirectThreads) {
    const int cnt = (int)(ns - s0 < kDirectThreads ? ns - s0 : kDirectThreads);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int64_t j = s0 + threadIdx.x;
      tile[threadIdx.x] = make_double4(src[3 * j], src[3 * j + 1], src[3 * j + 2], q[j]);
    }
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      const double4 sj = tile[k];
      const double dx = xi - sj.x, dy = yi - sj.y, dz = zi - sj.z;
      const double r2 = dx * dx + dy * dy + dz * dz;
      const double rinv = r2 > 0.0 ? rsqrt(r2) : 0.0;
      const double qr = sj.w * rinv;
      f += qr;
      if (kGrad) {
        const double qr3 = qr * rinv * rinv;
        gx -= qr3 * dx;
        gy -= qr3 * dy;
        gz -= qr3 * dz;
      }
    }
  }
  if (active) {
    phi[i] = f;
    if (kGrad) {
      grad[3 * i] = gx;
      grad[3 * i + 1] = gy;
      grad[3 * i + 2] = gz;
    }
  }
}

}  // namespace

void gather_charges(fmm_plan_s& P, const double* q) {
  gather_charges_kernel<<<cdiv(P.n, 256), 256, 0, P.stream>>>(q, P.perm, P.n, P.pos, P.flags);
  FMM_LAUNCHED("gather_charges_kernel");
}

void near_pass(fmm_plan_s& P, const double*, double* phi, double* grad) {
  const int64_t nl = P.own_leaf_end - P.own_leaf_begin;
  if (nl <= 0) return;
  const double s_phi = std::ldexp(1.0, -P.e), s_grad = std::ldexp(1.0, -2 * P.e);
  const size_t sh = sizeof(double2) * P.nc;
  const int32_t* leaves = P.leaves.ptr + P.own_leaf_begin;
  if (grad) {
    near_kernel<true><<<(unsigned)nl, kNearThreads, sh, P.stream>>>(leaves, P.cells.begin, P.cells.end,
                                                                    P.cells.center, P.pos, P.L, P.p2p.off, P.p2p.src,
                                                                    P.perm, P.p, P.nc, s_phi, s_grad, phi, grad);
  } else {
    near_kernel<false><<<(unsigned)nl, kNearThreads, sh, P.stream>>>(leaves, P.cells.begin, P.cells.end,
                                                                     P.cells.center, P.pos, P.L, P.p2p.off,
                                                                     P.p2p.src, P.perm, P.p, P.nc, s_phi, s_grad,
                                                                     phi, grad);
  }
  FMM_LAUNCHED("near_kernel");
}

void launch_direct(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt, double* phi,
                   double* grad, cudaStream_t s) {
  if (nt <= 0) return;
  if (grad)
    direct_kernel<true><<<cdiv(nt, kDirectThreads), kDirectThreads, 0, s>>>(src, q, ns, tgt, nt, phi, grad);
  else
    direct_kernel<false><<<cdiv(nt, kDirectThreads), kDirectThreads, 0, s>>>(src, q, ns, tgt, nt, phi, grad);
  FMM_LAUNCHED("direct_kernel");
}

}  // namespace fmm
