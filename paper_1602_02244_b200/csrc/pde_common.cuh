// pde_common.cuh — pieces shared by the NEXT-2 Laplace solve (pde.cu) and the NEXT-4 Helmholtz solve
// (pde_helmholtz.cu): C-ABI error guard, the lattice + face-panel points, grid sizing.
#pragma once
#include <cublas_v2.h>

#include <algorithm>
#include <new>
#include <string>

#include "plan.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

struct Guard {
  template <typename F>
  static fmm_status run(F&& body) {
    try {
      body();
      return FMM_OK;
    } catch (const fmm::Error& e) {
      return fmm::set_error(e.status, e.what());
    } catch (const std::bad_alloc&) {
      return fmm::set_error(FMM_ERR_OOM, "host allocation failed");
    } catch (const std::exception& e) {
      return fmm::set_error(FMM_ERR_CUDA, e.what());
    }
  }
};

void usage(bool ok, const char* msg) {
  if (!ok) throw fmm::Error(FMM_ERR_USAGE, msg);
}

void check_blas(cublasStatus_t s, const char* what) {
  if (s == CUBLAS_STATUS_ALLOC_FAILED) throw fmm::Error(FMM_ERR_OOM, what);
  if (s != CUBLAS_STATUS_SUCCESS) throw fmm::Error(FMM_ERR_CUDA, std::string(what) + ": cuBLAS status " + std::to_string((int)s));
}

unsigned grid_for(int64_t n, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32));
}

// lattice nodes then face panel centres (axis 0..2, side -1 then +1; in-face u fastest)
__global__ void points_kernel(int n, int stride, int nfa, double h, double* __restrict__ xyz) {
  const int64_t N = (int64_t)n * n * n, nf = 6LL * nfa * nfa;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x) {
    double p[3];
    if (t < N) {
      const int i = (int)(t % n), j = (int)((t / n) % n), k = (int)(t / ((int64_t)n * n));
      p[0] = __dadd_rn(-1.0, __dmul_rn(i + 1.0, h));
      p[1] = __dadd_rn(-1.0, __dmul_rn(j + 1.0, h));
      p[2] = __dadd_rn(-1.0, __dmul_rn(k + 1.0, h));
    } else {
      const int64_t f = t - N;
      const int face = (int)(f / ((int64_t)nfa * nfa)), w = (int)(f % ((int64_t)nfa * nfa));
      const int axis = face >> 1, o0 = axis == 0 ? 1 : 0, o1 = axis == 2 ? 1 : 2;
      p[axis] = (face & 1) ? 1.0 : -1.0;
      p[o0] = __dadd_rn(-1.0, __dmul_rn((w % nfa) * stride + 1.0, h));
      p[o1] = __dadd_rn(-1.0, __dmul_rn((w / nfa) * stride + 1.0, h));
    }
    xyz[3 * t] = p[0];
    xyz[3 * t + 1] = p[1];
    xyz[3 * t + 2] = p[2];
  }
}

}  // namespace
