// scan.cu — device exclusive prefix sums (setup path: tree levels, traversal
// compaction, radix-sort digit offsets). Three-phase: per-block scan ->
// recursive scan of block totals -> add. Integer, deterministic.
#include "common.cuh"

namespace fmm {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;  // per thread
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename Tin>
__global__ void scan_tile_kernel(const Tin* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                                 int64_t* __restrict__ block_sums) {
  __shared__ int64_t warp_tot[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    v[k] = i < n ? (int64_t)in[i] : 0;
    sum += v[k];
  }
  // inclusive warp scan of thread sums
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = wi - w;  // exclusive
    if (lane == kScanThreads / 32 - 1 && block_sums) block_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  int64_t run = warp_tot[wid] + inc - sum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
}

__global__ void scan_add_kernel(int64_t* __restrict__ out, int64_t n, const int64_t* __restrict__ block_off) {
  int64_t i = (int64_t)blockIdx.x * kScanTile + threadIdx.x;
  int64_t add = block_off[blockIdx.x];
  for (int k = 0; k < kScanItems; ++k, i += kScanThreads)
    if (i < n) out[i] += add;
}

template <typename Tin>
void scan_impl(const Tin* in, int64_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  unsigned nb = cdiv(n, kScanTile);
  if (nb == 1) {
    scan_tile_kernel<Tin><<<1, kScanThreads, 0, s>>>(in, out, n, nullptr);
    FMM_LAUNCHED("scan_tile_kernel");
    return;
  }
  int64_t* sums = nullptr;
  FMM_CUDA(cudaMallocAsync(&sums, sizeof(int64_t) * nb, s));
  scan_tile_kernel<Tin><<<nb, kScanThreads, 0, s>>>(in, out, n, sums);
  FMM_LAUNCHED("scan_tile_kernel");
  scan_impl<int64_t>(sums, sums, nb, s);
  scan_add_kernel<<<nb, kScanThreads, 0, s>>>(out, n, sums);
  FMM_LAUNCHED("scan_add_kernel");
  FMM_CUDA(cudaFreeAsync(sums, s));
}

}  // namespace

void scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  scan_impl<int64_t>(in, out, n, s);
}

int64_t scan_counts_total(const int32_t* counts, int64_t* offsets, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  scan_impl<int32_t>(counts, offsets, n, s);
  int64_t last_off = 0;
  int32_t last_cnt = 0;
  FMM_CUDA(cudaMemcpyAsync(&last_off, offsets + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaMemcpyAsync(&last_cnt, counts + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  return last_off + last_cnt;
}

}  // namespace fmm
