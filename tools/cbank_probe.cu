// cbank_probe.cu — does a DFMA whose matrix operand is a __constant__ (constant-bank) double run
// at the FP64 pipe rate when the kernel streams through several KB of such constants? This decides
// the M2L v4 design (fixed rotation matrices d(pi/2) as constant-bank operands).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cbank_probe tools/cbank_probe.cu
//   tools/cbank_probe            (prints TFLOP/s per variant)
#include <cstdio>
#include <cuda_runtime.h>
#include <utility>

constexpr int B = 11;                // block edge (degree 10)
__constant__ double cJ[B * B * 16];  // up to 16 blocks = 15.5 KB

template <int K, int NV, int R = K>
__global__ void __launch_bounds__(256) probe_const(double* out, int iters) {
  double v[NV][B];
#pragma unroll
  for (int s = 0; s < NV; ++s)
#pragma unroll
    for (int j = 0; j < B; ++j) v[s][j] = 1e-3 * (threadIdx.x + j + s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int s = 0; s < NV; ++s) {
        double o[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
          o[i] = 0.0;
#pragma unroll
          for (int j = 0; j < B; ++j) o[i] = fma(cJ[(k % R) * B * B + i * B + j], v[s][j], o[i]);
        }
#pragma unroll
        for (int i = 0; i < B; ++i) v[s][i] = o[i];
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int s = 0; s < NV; ++s)
#pragma unroll
    for (int j = 0; j < B; ++j) t += v[s][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// register-only operands, code of K blocks: separates instruction-cache from constant-cache effects
template <int K>
__global__ void __launch_bounds__(256) probe_reg(double* out, int iters) {
  double v[B];
#pragma unroll
  for (int j = 0; j < B; ++j) v[j] = 1e-3 * (threadIdx.x + j);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double o[B];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        o[i] = 0.0;
#pragma unroll
        for (int j = 0; j < B; ++j) o[i] = fma(v[(3 * i + j + k) % B], v[j], o[i]);
      }
#pragma unroll
      for (int i = 0; i < B; ++i) v[i] = o[i] * 1e-2;
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < B; ++j) t += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// same with the matrix in shared memory (uniform-address broadcast loads)
template <int K, int NV>
__global__ void __launch_bounds__(256) probe_smem(double* out, int iters) {
  __shared__ double sJ[B * B * K];
  for (int e = threadIdx.x; e < B * B * K; e += blockDim.x) sJ[e] = cJ[e];
  __syncthreads();
  double v[NV][B];
#pragma unroll
  for (int s = 0; s < NV; ++s)
#pragma unroll
    for (int j = 0; j < B; ++j) v[s][j] = 1e-3 * (threadIdx.x + j + s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int s = 0; s < NV; ++s) {
        double o[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
          o[i] = 0.0;
#pragma unroll
          for (int j = 0; j < B; ++j) o[i] = fma(sJ[k * B * B + i * B + j], v[s][j], o[i]);
        }
#pragma unroll
        for (int i = 0; i < B; ++i) v[s][i] = o[i];
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int s = 0; s < NV; ++s)
#pragma unroll
    for (int j = 0; j < B; ++j) t += v[s][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <typename F>
double run(F kern, int K, int NV, int blocks, int threads, int iters, double* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, threads>>>(out, 2);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * B * B * K * NV * (double)iters * blocks * threads;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  double h[B * B * 16];
  for (int i = 0; i < B * B * 16; ++i) h[i] = (((i * 37) % 23) - 11) / 121.0;
  cudaMemcpyToSymbol(cJ, h, sizeof(h));
  double* out;
  cudaMalloc(&out, 148 * 64 * 256 * sizeof(double));
  const int iters = 400;
  for (int bpsm : {2, 4}) {
    const int blocks = 148 * bpsm, thr = 128;
    printf("blocks/SM %d x %d threads\n", bpsm, thr);
    printf("  const K=1  NV=1: %.2f TF\n", run(probe_const<1, 1>, 1, 1, blocks, thr, iters * 8, out));
    printf("  const K=4  NV=1: %.2f TF\n", run(probe_const<4, 1>, 4, 1, blocks, thr, iters * 2, out));
    printf("  const K=8  NV=1: %.2f TF\n", run(probe_const<8, 1>, 8, 1, blocks, thr, iters, out));
    printf("  const K=16 NV=1: %.2f TF\n", run(probe_const<16, 1>, 16, 1, blocks, thr, iters / 2, out));
    printf("  const K=8  NV=2: %.2f TF\n", run(probe_const<8, 2>, 8, 2, blocks, thr, iters / 2, out));
    printf("  reg K=4: %.2f TF\n", run(probe_reg<4>, 4, 1, blocks, thr, iters * 2, out));
    printf("  reg K=16: %.2f TF\n", run(probe_reg<16>, 16, 1, blocks, thr, iters / 2, out));
    printf("  reg K=32: %.2f TF\n", run(probe_reg<32>, 32, 1, blocks, thr, iters / 4, out));
    printf("  reg K=64: %.2f TF\n", run(probe_reg<64>, 64, 1, blocks, thr, iters / 8, out));
    printf("  smem  K=4  NV=1: %.2f TF\n", run(probe_smem<4, 1>, 4, 1, blocks, thr, iters * 2, out));
    printf("  smem  K=4  NV=2: %.2f TF\n", run(probe_smem<4, 2>, 4, 2, blocks, thr, iters, out));
  }
  return 0;
}
