// Measurement only: cycles per M2L v3 MMA item (big 16x12, small 8x8, 5 n-tiles) in isolation,
// 8 warps per SM, operands in shared memory as in m2l_rot.cu (no barriers, no other warps).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int S = 132;
__device__ __forceinline__ int col_base(int c) { return c * S + ((c & 4) ? ((c & 1) ? -4 : 4) : 0); }

template <int MT, int KS, int NT, int VAR>
__device__ __forceinline__ void item(const double* A, const int* ps, double* xc, int lane) {
  const int colb = lane >> 2, kl = lane & 3;
  double a[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[mt][ks] = A[(mt * KS + ks) * 32 + lane];
  int qk[KS], qr[MT];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) qk[ks] = ps[4 * ks + kl];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) qr[mt] = ps[8 * mt + colb];
  double c[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int t = 0; t < NT; ++t) c[mt][t][0] = c[mt][t][1] = 0.0;
  const double* xb = xc + col_base(colb);
  if (VAR == 0) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int q = qk[ks];
      double b[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) b[t] = q >= 0 ? xb[8 * t * S + q] : 0.0;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma884(c[mt][t][0], c[mt][t][1], a[mt][ks], b[t]);
    }
  } else {  // all B first (no predicate), then DMMAs
    double b[KS][NT];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int t = 0; t < NT; ++t) b[ks][t] = xb[8 * t * S + (qk[ks] & 127)];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma884(c[mt][t][0], c[mt][t][1], a[mt][ks], b[ks][t]);
  }
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int q = qr[mt];
    if (q < 0) continue;
    double* y0 = xc + col_base(2 * kl) + q;
    double* y1 = xc + col_base(2 * kl + 1) + q;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      y0[8 * t * S] = c[mt][t][0];
      y1[8 * t * S] = c[mt][t][1];
    }
  }
  __syncwarp();
}

template <int MT, int KS, int VAR>
__global__ void probe(int iters, unsigned long long* out) {
  extern __shared__ double sm[];
  double* X = sm;                 // 40 x S
  double* A = X + 40 * S + 64;    // fragments
  int* pos = (int*)(A + 8 * 192);
  for (int i = threadIdx.x; i < 40 * S + 64 + 8 * 192; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * 16; i += blockDim.x) pos[i] = (i % 16) < MT * 8 ? (i / 16) * 12 + (i % 16) : -1;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) item<MT, KS, 5, VAR>(A + w * 192, pos + w * 16, X, lane);
  const unsigned long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) out[w] = t1 - t0;
}

template <int MT, int KS, int VAR>
void run(const char* name) {
  unsigned long long* o;
  cudaMalloc(&o, 64 * sizeof(unsigned long long));
  const size_t sh = (40 * S + 64 + 8 * 192) * 8 + 8 * 16 * 4;
  cudaFuncSetAttribute(probe<MT, KS, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
  const int iters = 2000;
  probe<MT, KS, VAR><<<148, 256, sh>>>(iters, o);
  cudaDeviceSynchronize();
  unsigned long long h[8];
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  const double dmma = MT * KS * 5.0;
  printf("%s var %d: %.0f cycles per item (%.0f DMMA) -> %.1f cycles per DMMA per warp (pipe share 33)\n", name, VAR,
         (double)h[0] / iters, dmma, (double)h[0] / iters / dmma);
  cudaFree(o);
}

int main() {
  run<2, 3, 0>("big");
  run<1, 2, 0>("small");
  run<2, 3, 1>("big");
  run<1, 2, 1>("small");
  return 0;
}
