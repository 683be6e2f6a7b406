// tools/icache_probe.cu — does straight-line FP64 code larger than the instruction caches still run at the
// DFMA pipe rate? (measurement infrastructure for profiles/r2_m2l_bound.md, not part of the FMM path)
// One CTA per SM, W warps; every thread runs a loop whose body is NI independent-chain DFMAs, fully
// unrolled (NI * 16 bytes of code), optionally with the warps of a CTA started NI/2 instructions apart.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 16;

template <int NI>
__device__ __forceinline__ void body(double (&a)[kChains], double m, double c) {
#pragma unroll
  for (int i = 0; i < NI; ++i) a[i % kChains] = fma(a[i % kChains], m, c);
}

template <int NI, bool SKEW>
__global__ void __launch_bounds__(256, 1) probe(const double* seed, double* out, int iters) {
  double a[kChains];
  const double m = seed[0], c = seed[1];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = seed[2] + k * 1e-3 + threadIdx.x * 1e-7;
  if (SKEW && (threadIdx.x >> 5) >= 4) body<NI / 2>(a, m, c);  // the second warp of each scheduler half a body ahead
  for (int it = 0; it < iters; ++it) body<NI>(a, m, c);
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}

template <int NI, bool SKEW>
void run(int warps, const double* seed, double* out) {
  const int iters = (1 << 22) / NI;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<NI, SKEW><<<148, 32 * warps>>>(seed, out, iters);
  cudaEventRecord(e0);
  probe<NI, SKEW><<<148, 32 * warps>>>(seed, out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * NI * (double)iters * 148 * 32 * warps;
  printf("body %6d DFMA (%4d KB) warps/SM %d skew %d: %7.3f ms  %6.2f TFLOP/s  %.3f of 37.2\n", NI, NI * 16 / 1024, warps,
         (int)SKEW, ms, fl / ms * 1e-9, fl / ms * 1e-9 / 37.225);
}

int main() {
  double hs[3] = {0.999999, 1e-9, 1.0}, *seed, *out;
  cudaMalloc(&seed, sizeof(hs));
  cudaMalloc(&out, 8);
  cudaMemcpy(seed, hs, sizeof(hs), cudaMemcpyHostToDevice);
  for (int w : {4, 8}) {
    run<256, false>(w, seed, out);
    run<1024, false>(w, seed, out);
    run<2048, false>(w, seed, out);
    run<4096, false>(w, seed, out);
    run<8192, false>(w, seed, out);
    run<16384, false>(w, seed, out);
  }
  run<2048, true>(8, seed, out);
  run<8192, true>(8, seed, out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
