// Accuracy of rsqrt.approx.ftz.f64 (MUFU) and of one / two refinement orders, over
// r^2 in [2^-60, 2^60] (log-uniform) — the error bound DESIGN.md quotes for the near field.
#include <cstdio>
#include <cmath>
#include <cstdint>
__device__ double rs_raw(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__global__ void k(int n, double* out) {
  __shared__ double m[4][256];
  double e0 = 0, e1 = 0, e2 = 0;
  uint64_t s = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double u = (double)(s >> 11) * 0x1p-53;
    const double x = exp2(120.0 * u - 60.0);
    const double t = 1.0 / sqrt(x);  // correctly rounded-ish reference
    const double y = rs_raw(x);
    const double e = fma(-x * y, y, 1.0);
    const double y1 = fma(y, 0.5 * e, y);
    const double y2 = fma(y, e * fma(e, 0.375, 0.5), y);
    e0 = fmax(e0, fabs(y / t - 1)); e1 = fmax(e1, fabs(y1 / t - 1)); e2 = fmax(e2, fabs(y2 / t - 1));
  }
  m[0][threadIdx.x] = e0; m[1][threadIdx.x] = e1; m[2][threadIdx.x] = e2;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < 256; ++j) for (int q = 0; q < 3; ++q) m[q][0] = fmax(m[q][0], m[q][j]);
    for (int q = 0; q < 3; ++q) out[3 * blockIdx.x + q] = m[q][0];
  }
}
int main() {
  double* d; cudaMalloc(&d, 3 * 148 * sizeof(double));
  k<<<148, 256>>>(4096, d);
  double h[3 * 148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double e[3] = {0, 0, 0};
  for (int b = 0; b < 148; ++b) for (int q = 0; q < 3; ++q) e[q] = fmax(e[q], h[3 * b + q]);
  printf("max rel err: raw %.3e (2^%.1f)  1st-order %.3e (2^%.1f)  2nd-order %.3e (2^%.1f)\n", e[0], log2(e[0]), e[1],
         log2(e[1]), e[2], log2(e[2] > 0 ? e[2] : 1e-300));
  return 0;
}
