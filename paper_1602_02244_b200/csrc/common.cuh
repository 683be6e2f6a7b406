// common.cuh — internal helpers shared by the libfmm.so translation units.
// Nothing here is exported through the C ABI (include/fmm.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace fmm {

constexpr int kMaxLevel = 21;  // 63-bit Morton keys, 21 bits per axis (R4)
constexpr int kMaxP = 16;      // ABI limit on the expansion order (R24)

// Error carried from deep inside the implementation to the ABI layer.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) throw Error(5, std::string(what) + ": " + cudaGetErrorString(e));
  if (e != cudaSuccess) throw Error(4, std::string(what) + ": " + cudaGetErrorString(e));
}
#define FMM_CUDA(x) ::fmm::check_cuda((x), #x)
// process-wide count of kernel launches (every launch is followed by FMM_LAUNCHED); fmm_stats
// reports it so a caller can count the launches of a timed region exactly
inline std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}
#define FMM_LAUNCHED(name) (::fmm::launch_counter()++, ::fmm::check_cuda(cudaGetLastError(), name))

__host__ __device__ inline int ncoef(int p) { return (p + 1) * (p + 2) / 2; }
__host__ __device__ inline int cidx(int n, int m) { return n * (n + 1) / 2 + m; }

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
// acc += a * conj(b)
__device__ __forceinline__ void cfma_conjb(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.y, b.x, fma(-a.x, b.y, acc.y));
}

// A_n^m for any |m| <= n from m >= 0 storage: A_n^{-m} = (-1)^m conj(A_n^m)
__device__ __forceinline__ double2 cget(const double2* A, int n, int m) {
  if (m >= 0) return A[cidx(n, m)];
  double2 v = A[cidx(n, -m)];
  return (m & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
}

// ------------------------------------------------------------- scans (scan.cu)
// Exclusive prefix sum of n int64 values (in may alias out). Returns nothing;
// the total is out[n-1] + in[n-1] computed by the caller if needed.
void scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
// Exclusive scan of int32 counts into int64 offsets, and returns the total (synchronises).
int64_t scan_counts_total(const int32_t* counts, int64_t* offsets, int64_t n, cudaStream_t s);

// ------------------------------------------------------- radix sort (sort.cu)
// Stable LSD radix sort of (key, value) pairs on the low `bits` bits of key.
// keys/vals are sorted in place (tmp buffers allocated internally).
void radix_sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n, int bits, cudaStream_t s);

}  // namespace fmm
