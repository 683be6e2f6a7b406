// Microbenchmark (measurement only): DMMA.8x8x4 (mma.sync m8n8k4 f64) throughput and
// dependent-chain latency on one SM and on all SMs, vs warps per SM and independent
// accumulators per warp. Informs the M2L kernels' warp / accumulator counts.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void dmma_loop(double* out, int iters) {
  double c0[C], c1[C];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < C; ++i) c0[i] = c1[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c0[i] + c1[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int C>
void run(int blocks, int warps, int iters) {
  double* o;
  cudaMalloc(&o, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_loop<C><<<blocks, 32 * warps>>>(o, 10);
  cudaEventRecord(e0);
  dmma_loop<C><<<blocks, 32 * warps>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int dev;
  cudaGetDevice(&dev);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double n = (double)blocks * warps * C * iters;  // DMMAs
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("blocks %4d warps/blk %2d chains %2d: %.3f ms, %.2f TFLOP/s, %.2f cycles per DMMA per SMSP (per-SM view)\n",
         blocks, warps, C, ms, n * 512 / (ms * 1e-3) / 1e12,
         cycles / (n / (blocks < 148 ? blocks : 148) / 4));
  cudaFree(o);
}

int main1() {
  for (int w : {1, 2, 4, 8, 16}) {
    run<1>(1, w, 20000);
    run<2>(1, w, 20000);
    run<4>(1, w, 10000);
    run<8>(1, w, 5000);
  }
  run<8>(148, 8, 5000);
  run<8>(148, 16, 5000);
  run<4>(148, 16, 10000);
  return 0;
}

// GEMM-like pattern: MT x NT accumulators, operands from registers that change per k-step
template <int MT, int NT>
__global__ void dmma_gemm(double* out, const double* in, int iters) {
  double c[MT][NT][2];
  double a[MT], b[NT];
#pragma unroll
  for (int i = 0; i < MT; ++i) a[i] = in[threadIdx.x + 32 * i];
#pragma unroll
  for (int j = 0; j < NT; ++j) b[j] = in[threadIdx.x + 32 * (j + MT)];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1]) : "d"(a[i]), "d"(b[j]));
#pragma unroll
    for (int i = 0; i < MT; ++i) a[i] = a[i] * 1.0000001;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int MT, int NT>
void run_gemm(int warps, int iters) {
  double *o, *in;
  cudaMalloc(&o, 1024 * sizeof(double));
  cudaMalloc(&in, 4096 * sizeof(double));
  cudaMemset(in, 0, 4096 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_gemm<MT, NT><<<148, 32 * warps>>>(o, in, 10);
  cudaEventRecord(e0);
  dmma_gemm<MT, NT><<<148, 32 * warps>>>(o, in, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = 148.0 * warps * MT * NT * iters;
  printf("gemm MT %d NT %d warps/SM %2d: %.2f TFLOP/s (%.0f%% of 36.4)\n", MT, NT, warps, n * 512 / (ms * 1e-3) / 1e12,
         100 * n * 512 / (ms * 1e-3) / 1e12 / 36.4);
  cudaFree(o);
  cudaFree(in);
}

// B operands from shared memory every k-step (LDS.64 per n-tile), like the M2L kernels
template <int MT, int NT>
__global__ void dmma_gemm_smem(double* out, const double* in, int iters) {
  __shared__ double xs[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = in[i % 1024];
  __syncthreads();
  double c[MT][NT][2];
  double a[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) a[i] = in[threadIdx.x + 32 * i];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int xo = ((lane >> 2) * 132 + (lane & 3) + (w & 7) * 8) & 4095;
  for (int it = 0; it < iters; ++it) {
    double b[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) b[j] = xs[(xo + j * 8 * 132 + 4 * (it & 7)) & 4095];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1]) : "d"(a[i]), "d"(b[j]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int MT, int NT>
void run_gemm_smem(int warps, int iters) {
  double *o, *in;
  cudaMalloc(&o, 1024 * sizeof(double));
  cudaMalloc(&in, 4096 * sizeof(double));
  cudaMemset(in, 0, 4096 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_gemm_smem<MT, NT><<<148, 32 * warps>>>(o, in, 10);
  cudaEventRecord(e0);
  dmma_gemm_smem<MT, NT><<<148, 32 * warps>>>(o, in, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = 148.0 * warps * MT * NT * iters;
  printf("gemm_smemB MT %d NT %d warps/SM %2d: %.2f TFLOP/s (%.0f%% of 36.4)\n", MT, NT, warps,
         n * 512 / (ms * 1e-3) / 1e12, 100 * n * 512 / (ms * 1e-3) / 1e12 / 36.4);
  cudaFree(o);
  cudaFree(in);
}

int main2();
int main2() {
  run_gemm_smem<1, 5>(8, 4000);
  run_gemm_smem<2, 5>(8, 2000);
  run_gemm_smem<2, 8>(8, 2000);
  run_gemm_smem<1, 5>(16, 4000);
  run_gemm_smem<2, 5>(16, 2000);
  run_gemm<1, 5>(8, 4000);
  run_gemm<2, 5>(8, 2000);
  run_gemm<2, 8>(8, 2000);
  run_gemm<1, 5>(16, 4000);
  run_gemm<2, 4>(8, 2000);
  run_gemm<1, 2>(8, 8000);
  run_gemm<1, 1>(8, 8000);
  return 0;
}
int main() { main1(); return main2(); }
