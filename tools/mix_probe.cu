// mix_probe.cu — measurement only: do FP64 tensor-core DMMA (mma.sync m8n8k4 f64) and FP64 ALU
// DFMA share one execution pipe on B200, or do they overlap? Decides whether moving the fixed
// operator products of M2L v4 (F, G applied to 32 pairs at once = small GEMMs) onto DMMA can add
// throughput beside the DFMA work that stays (z-rotations, Hankel translation).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_probe tools/mix_probe.cu
//   tools/mix_probe     (TFLOP/s of DMMA only, DFMA only, both in the same warps, split warps)
#include <cstdio>
#include <cuda_runtime.h>

// KD DMMA chains and KF DFMA chains (8 independent accumulators each) per iteration, same warp
template <int KD, int KF>
__global__ void __launch_bounds__(512) mix(double* out, int iters, int dmma_warps) {
  double c0[8], c1[8], f[8][4];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c0[i] = c1[i] = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) f[i][k] = 1e-3 * (i + k);
  }
  const int w = threadIdx.x >> 5;
  const bool do_d = dmma_warps < 0 || w < dmma_warps, do_f = dmma_warps < 0 || w >= dmma_warps;
  for (int it = 0; it < iters; ++it) {
    if (do_d) {
#pragma unroll
      for (int r = 0; r < KD; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
    }
    if (do_f) {
#pragma unroll
      for (int r = 0; r < KF; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[i][k]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s += c0[i] + c1[i];
#pragma unroll
    for (int k = 0; k < 4; ++k) s += f[i][k];
  }
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int KD, int KF>
void run(const char* name, int warps, int dmma_warps, int iters) {
  double* o;
  cudaMalloc(&o, 4096 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<KD, KF><<<148, 32 * warps>>>(o, 10, dmma_warps);
  cudaEventRecord(e0);
  mix<KD, KF><<<148, 32 * warps>>>(o, iters, dmma_warps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double wd = dmma_warps < 0 ? warps : dmma_warps, wf = dmma_warps < 0 ? warps : warps - dmma_warps;
  // one m8n8k4 = 256 FMA = 512 flop per warp; one warp DFMA = 32 FMA = 64 flop
  const double fl_d = 148.0 * wd * KD * 8 * iters * 512, fl_f = 148.0 * wf * KF * 32 * iters * 64;
  printf("%-28s warps %2d: %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", name, warps, ms,
         fl_d / (ms * 1e-3) / 1e12, fl_f / (ms * 1e-3) / 1e12, (fl_d + fl_f) / (ms * 1e-3) / 1e12);
  cudaFree(o);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<1, 0>("DMMA only", w, -1, 20000);
    run<0, 1>("DFMA only (4x work/iter)", w, -1, 20000);
    run<1, 1>("both, same warps", w, -1, 20000);
    run<1, 2>("both, same warps, 2x DFMA", w, -1, 20000);
    run<1, 1>("split: half DMMA warps", w, w / 2, 20000);
  }
  return 0;
}
