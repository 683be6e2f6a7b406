// sort.cu — hand-written stable LSD radix sort of (uint64 key, uint32 value)
// pairs (north_star (1): "Morton-code octree build with a device radix sort").
//
// Per 8-bit digit pass: (1) per-tile digit histogram, (2) exclusive scan of
// the digit-major histogram [digit][tile] -> global scatter base per
// (digit, tile), (3) stable scatter: inside a tile items are ranked in index
// order with warp match (__match_any_sync) + per-warp digit counts, so equal
// digits keep their input order. Stability of every pass makes the whole LSD
// sort stable: equal keys stay in input-index order (R5).
// Passes whose digit is identical for every key are skipped (histogram check).
#include <utility>
#include <vector>

#include "common.cuh"

namespace fmm {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 8;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 2048 items per tile
constexpr int kRadix = 256;

__global__ void radix_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift, int ntiles,
                                  int64_t* __restrict__ hist) {
  __shared__ int cnt[kRadix];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int r = 0; r < kSortRounds; ++r) {
    int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 0xff], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void radix_scatter_kernel(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                     uint64_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n,
                                     int shift, int ntiles, const int64_t* __restrict__ offs) {
  __shared__ int64_t base[kRadix];
  __shared__ int run[kRadix];
  __shared__ int whist[kSortThreads / 32][kRadix];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  base[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
  run[tid] = 0;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int r = 0; r < kSortRounds; ++r) {
    for (int w = 0; w < kSortThreads / 32; ++w) whist[w][tid] = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * kSortTile + r * kSortThreads + tid;
    const bool valid = i < n;
    uint64_t key = valid ? kin[i] : 0;
    uint32_t val = valid ? vin[i] : 0;
    int d = valid ? (int)((key >> shift) & 0xff) : kRadix;  // invalid lanes form their own group
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & lt_mask);
    if (valid && rank == 0) whist[wid][d] = __popc(peers);
    __syncthreads();
    {  // exclusive prefix over warps for digit `tid`, on top of the running count
      int s = run[tid];
      for (int w = 0; w < kSortThreads / 32; ++w) {
        int t = whist[w][tid];
        whist[w][tid] = s;
        s += t;
      }
      run[tid] = s;
    }
    __syncthreads();
    if (valid) {
      int64_t pos = base[d] + whist[wid][d] + rank;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
  }
}

__global__ void digit_start_kernel(const int64_t* __restrict__ offs, int ntiles, int64_t* __restrict__ starts) {
  starts[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles];
}

}  // namespace

void radix_sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n, int bits, cudaStream_t s) {
  if (n <= 1 || bits <= 0) return;
  const int ntiles = (int)cdiv(n, kSortTile);
  const int64_t nh = (int64_t)kRadix * ntiles;
  uint64_t* k2 = nullptr;
  uint32_t* v2 = nullptr;
  int64_t* hist = nullptr;
  int64_t* starts = nullptr;
  FMM_CUDA(cudaMallocAsync(&k2, sizeof(uint64_t) * n, s));
  FMM_CUDA(cudaMallocAsync(&v2, sizeof(uint32_t) * n, s));
  FMM_CUDA(cudaMallocAsync(&hist, sizeof(int64_t) * nh, s));
  FMM_CUDA(cudaMallocAsync(&starts, sizeof(int64_t) * kRadix, s));
  // digit-skip check: one histogram per pass is read back (setup only)
  std::vector<int64_t> col(kRadix);
  uint64_t* ka = keys;
  uint32_t* va = vals;
  uint64_t* kb = k2;
  uint32_t* vb = v2;
  for (int shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<ntiles, kSortThreads, 0, s>>>(ka, n, shift, ntiles, hist);
    FMM_LAUNCHED("radix_hist_kernel");
    scan_exclusive_i64(hist, hist, nh, s);
    // skip the pass if one digit holds all n keys (setup only: one small read-back)
    digit_start_kernel<<<1, kRadix, 0, s>>>(hist, ntiles, starts);
    FMM_LAUNCHED("digit_start_kernel");
    FMM_CUDA(cudaMemcpyAsync(col.data(), starts, sizeof(int64_t) * kRadix, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    bool trivial = false;
    for (int d = 0; d < kRadix; ++d) trivial |= ((d + 1 < kRadix ? col[d + 1] : n) - col[d]) == n;
    if (trivial) continue;
    radix_scatter_kernel<<<ntiles, kSortThreads, 0, s>>>(ka, va, kb, vb, n, shift, ntiles, hist);
    FMM_LAUNCHED("radix_scatter_kernel");
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    FMM_CUDA(cudaMemcpyAsync(keys, ka, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(vals, va, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
  }
  FMM_CUDA(cudaFreeAsync(k2, s));
  FMM_CUDA(cudaFreeAsync(v2, s));
  FMM_CUDA(cudaFreeAsync(hist, s));
  FMM_CUDA(cudaFreeAsync(starts, s));
}

}  // namespace fmm
