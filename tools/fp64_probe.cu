// tools/fp64_probe.cu — FP64 roofline denominator for bench.py (measurement
// infrastructure, not part of the FMM path). MEASURED_PEAKS.json holds only
// HBM and bf16, so the DFMA pipe rate is measured here: every thread runs
// kChains independent FMA chains (no dependency stalls), grid = a multiple
// of the SM count, timed with CUDA events by the caller.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int kChains = 16;

__global__ void __launch_bounds__(256) dfma_kernel(const double* __restrict__ seed, double* __restrict__ out,
                                                   int64_t iters) {
  double a[kChains];
  const double m = seed[0], c = seed[1];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = seed[2] + k * 1e-3 + threadIdx.x * 1e-7;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int fp64_probe_launch(int blocks, int threads, int64_t iters,
                                                                        const double* seed, double* out,
                                                                        void* stream) {
  dfma_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(seed, out, iters);
  return (int)cudaGetLastError();
}

// flops performed by one launch
extern "C" __attribute__((visibility("default"))) double fp64_probe_flops(int blocks, int threads, int64_t iters) {
  return 2.0 * kChains * (double)iters * (double)blocks * (double)threads;
}

// DMMA probe: mma.sync.aligned.m8n8k4.row.col.f64 (FP64 tensor path, legacy warp MMA).
namespace {
__global__ void __launch_bounds__(256) dmma_kernel(const double* __restrict__ seed, double* __restrict__ out,
                                                   int64_t iters) {
  double a = seed[0] + threadIdx.x * 1e-9, b = seed[1] - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int dmma_probe_launch(int blocks, int threads, int64_t iters,
                                                                        const double* seed, double* out,
                                                                        void* stream) {
  dmma_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(seed, out, iters);
  return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) double dmma_probe_flops(int blocks, int threads, int64_t iters) {
  return 2.0 * 8 * 8 * 4 * 8 * (double)iters * (double)blocks * (double)(threads / 32);
}
