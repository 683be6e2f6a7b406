// tree.cu — setup steps S1–S4: bounding cube with the exact
// 2^-e normalisation, quantisation + 63-bit Morton keys, device radix sort,
// Morton-ordered particles, adaptive octree built level by level.
//
// Paper: "hierarchically decomposed far field"; mapping
// 3-D to 1-D locality is the Morton order. Readings R2–R8
// in DESIGN.md fix every float -> integer decision so that the tree is a pure
// function of integers: IEEE __dsub_rn / __dmul_rn, no FMA contraction.
#include <cmath>
#include <vector>

#include "plan.h"

namespace fmm {
namespace {

constexpr int kBBoxThreads = 256;

__global__ void bbox_partial_kernel(const double* __restrict__ xyz, int64_t n, double* __restrict__ part,
                                    int32_t* __restrict__ bad) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int nonfinite = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double v = xyz[3 * i + k];
      if (!isfinite(v)) nonfinite = 1;
      mn[k] = fmin(mn[k], v);
      mx[k] = fmax(mx[k], v);
    }
  }
  __shared__ double sh[6][kBBoxThreads];
  for (int k = 0; k < 3; ++k) {
    sh[k][threadIdx.x] = mn[k];
    sh[3 + k][threadIdx.x] = mx[k];
  }
  if (__syncthreads_or(nonfinite) && threadIdx.x == 0) atomicOr(bad, 1);
  for (int s = kBBoxThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 3; ++k) {
        sh[k][threadIdx.x] = fmin(sh[k][threadIdx.x], sh[k][threadIdx.x + s]);
        sh[3 + k][threadIdx.x] = fmax(sh[3 + k][threadIdx.x], sh[3 + k][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[(int64_t)blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void bbox_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  // one thread per component; min for 0..2, max for 3..5 (order-independent => deterministic)
  int k = threadIdx.x;
  if (k >= 6) return;
  double v = part[k];
  for (int b = 1; b < nb; ++b) v = k < 3 ? fmin(v, part[6 * b + k]) : fmax(v, part[6 * b + k]);
  out[k] = v;
}

// bit b of v -> bit 3b
__device__ __forceinline__ uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

// R3/R4: t = x' - lo (IEEE), u = t * scale (IEEE), k = clamp(floor(u), 0, 2^21 - 1);
// key bit 3b+2 = bit b of kx, 3b+1 of ky, 3b of kz.
__global__ void morton_kernel(const double* __restrict__ xyz, int64_t n, double inv2e, double lox, double loy,
                              double loz, double scale, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo[3] = {lox, loy, loz};
  uint64_t k[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double x = __dmul_rn(xyz[3 * i + a], inv2e);  // exact power-of-two scaling
    double t = __dsub_rn(x, lo[a]);
    double u = __dmul_rn(t, scale);
    double f = floor(u);
    f = f < 0.0 ? 0.0 : (f > 2097151.0 ? 2097151.0 : f);
    k[a] = (uint64_t)f;
  }
  keys[i] = (spread3(k[0]) << 2) | (spread3(k[1]) << 1) | spread3(k[2]);
  idx[i] = (uint32_t)i;
}

__global__ void gather_positions_kernel(const double* __restrict__ xyz, const uint32_t* __restrict__ perm,
                                        int64_t n, double inv2e, double4* __restrict__ pos) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t j = perm[i];
  pos[i] = make_double4(__dmul_rn(xyz[3 * j], inv2e), __dmul_rn(xyz[3 * j + 1], inv2e),
                        __dmul_rn(xyz[3 * j + 2], inv2e), 0.0);
}

__device__ __forceinline__ int digit_at(uint64_t key, int shift) { return (int)((key >> shift) & 7u); }

// first index in [b, e) whose child digit is >= d (digits are monotone inside a cell)
__device__ __forceinline__ int32_t lower_digit(const uint64_t* __restrict__ keys, int32_t b, int32_t e, int shift,
                                               int d) {
  while (b < e) {
    int32_t mid = b + ((e - b) >> 1);
    if (digit_at(keys[mid], shift) < d)
      b = mid + 1;
    else
      e = mid;
  }
  return b;
}

// R8/R9: a cell splits iff count > ncrit and level < 21; empty children are not created.
__global__ void count_children_kernel(const uint64_t* __restrict__ keys, const int32_t* __restrict__ cbeg,
                                      const int32_t* __restrict__ cend, int64_t lb, int64_t le, int level, int ncrit,
                                      int32_t* __restrict__ nch) {
  int64_t c = lb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= le) return;
  int32_t b = cbeg[c], e = cend[c];
  int cnt = 0;
  if (e - b > ncrit && level < kMaxLevel) {
    const int shift = 3 * (kMaxLevel - level - 1);
    int32_t prev = b;
    for (int d = 1; d <= 8; ++d) {
      int32_t nxt = d < 8 ? lower_digit(keys, prev, e, shift, d) : e;
      cnt += nxt > prev;
      prev = nxt;
    }
  }
  nch[c - lb] = cnt;
}

__global__ void emit_children_kernel(const uint64_t* __restrict__ keys, int64_t lb, int64_t le, int level,
                                     const int32_t* __restrict__ nch, const int64_t* __restrict__ off,
                                     int32_t* __restrict__ clevel, int32_t* __restrict__ cbeg,
                                     int32_t* __restrict__ cend, int32_t* __restrict__ cchild,
                                     int32_t* __restrict__ cnchild, int32_t* __restrict__ cparent,
                                     int32_t* __restrict__ canchor) {
  int64_t c = lb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= le) return;
  int k = nch[c - lb];
  cnchild[c] = k;
  if (k == 0) {
    cchild[c] = -1;
    return;
  }
  const int64_t first = le + off[c - lb];
  cchild[c] = (int32_t)first;
  const int shift = 3 * (kMaxLevel - level - 1);
  const int32_t b = cbeg[c], e = cend[c];
  const int32_t ax = canchor[3 * c], ay = canchor[3 * c + 1], az = canchor[3 * c + 2];
  int32_t prev = b;
  int64_t w = first;
  for (int d = 0; d < 8; ++d) {
    int32_t nxt = d < 7 ? lower_digit(keys, prev, e, shift, d + 1) : e;
    if (nxt > prev) {
      clevel[w] = level + 1;
      cbeg[w] = prev;
      cend[w] = nxt;
      cchild[w] = -1;
      cnchild[w] = 0;
      cparent[w] = (int32_t)c;
      canchor[3 * w] = 2 * ax + ((d >> 2) & 1);
      canchor[3 * w + 1] = 2 * ay + ((d >> 1) & 1);
      canchor[3 * w + 2] = 2 * az + (d & 1);
      ++w;
    }
    prev = nxt;
  }
}

// R6: c = lo + (2a+1) * (S / 2^{l+1}) with one IEEE multiply and one IEEE add; h = S / 2^{l+1}.
__global__ void centers_kernel(const int32_t* __restrict__ clevel, const int32_t* __restrict__ canchor, int64_t nc,
                               double lox, double loy, double loz, double S, double4* __restrict__ center) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double h = ldexp(S, -(clevel[c] + 1));
  double x = __dadd_rn(lox, __dmul_rn((double)(2 * canchor[3 * c] + 1), h));
  double y = __dadd_rn(loy, __dmul_rn((double)(2 * canchor[3 * c + 1] + 1), h));
  double z = __dadd_rn(loz, __dmul_rn((double)(2 * canchor[3 * c + 2] + 1), h));
  center[c] = make_double4(x, y, z, h);
}

__global__ void leaf_flag_kernel(const int32_t* __restrict__ cchild, int64_t nc, int32_t* __restrict__ flag) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) flag[c] = cchild[c] < 0;
}

__global__ void compact_kernel(const int32_t* __restrict__ flag, const int64_t* __restrict__ off, int64_t nc,
                               int32_t* __restrict__ out) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc && flag[c]) out[off[c]] = (int32_t)c;
}

__global__ void root_kernel(int64_t n, int32_t* clevel, int32_t* cbeg, int32_t* cend, int32_t* cchild,
                            int32_t* cnchild, int32_t* cparent, int32_t* canchor) {
  clevel[0] = 0;
  cbeg[0] = 0;
  cend[0] = (int32_t)n;
  cchild[0] = -1;
  cnchild[0] = 0;
  cparent[0] = -1;
  canchor[0] = canchor[1] = canchor[2] = 0;
}

}  // namespace

void Cells::reserve(int64_t c, cudaStream_t s) {
  if (c <= cap) return;
  int64_t nc = cap ? cap : 1024;
  while (nc < c) nc *= 2;
  level.grow(nc, n, s);
  begin.grow(nc, n, s);
  end.grow(nc, n, s);
  child.grow(nc, n, s);
  nchild.grow(nc, n, s);
  parent.grow(nc, n, s);
  anchor.grow(3 * nc, 3 * n, s);
  cap = nc;
}

void build_tree(fmm_plan_s& P, const double* xyz) {
  cudaStream_t s = P.stream;
  const int64_t n = P.n;
  // ---- S1: bounding cube (+ non-finite check)
  const int nb = (int)std::min<int64_t>(cdiv(n, kBBoxThreads * 8), 2 * 148 * 4);
  DevBuf<double> part, box;
  part.alloc(6 * (int64_t)nb);
  box.alloc(6);
  P.flags.alloc(4);
  FMM_CUDA(cudaMemsetAsync(P.flags, 0, 4 * sizeof(int32_t), s));
  bbox_partial_kernel<<<nb, kBBoxThreads, 0, s>>>(xyz, n, part, P.flags);
  FMM_LAUNCHED("bbox_partial_kernel");
  bbox_final_kernel<<<1, 32, 0, s>>>(part, nb, box);
  FMM_LAUNCHED("bbox_final_kernel");
  double hb[6];
  int32_t bad = 0;
  FMM_CUDA(cudaMemcpyAsync(hb, box, sizeof(hb), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaMemcpyAsync(&bad, P.flags, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  if (bad) throw Error(FMM_ERR_USAGE, "fmm_setup: non-finite coordinate");
  FMM_CUDA(cudaMemsetAsync(P.flags, 0, 4 * sizeof(int32_t), s));

  // R2: root cube = min corner, side = max extent; exact 2^-e normalisation, S in [1, 2)
  double S = 0;
  for (int k = 0; k < 3; ++k) S = std::max(S, hb[3 + k] - hb[k]);
  if (S == 0) S = 1;
  int ex = 0;
  std::frexp(S, &ex);
  P.e = ex - 1;
  for (int k = 0; k < 3; ++k) P.lo[k] = std::ldexp(hb[k], -P.e);
  P.S = std::ldexp(S, -P.e);
  P.scale = 2097152.0 / P.S;
  const double inv2e = std::ldexp(1.0, -P.e);

  // ---- S1/S2: keys and stable radix sort (ties keep input order)
  P.keys.alloc(n);
  P.perm.alloc(n);
  morton_kernel<<<cdiv(n, 256), 256, 0, s>>>(xyz, n, inv2e, P.lo[0], P.lo[1], P.lo[2], P.scale, P.keys, P.perm);
  FMM_LAUNCHED("morton_kernel");
  radix_sort_pairs(P.keys, P.perm, n, 63, s);

  // ---- S3: particles in Morton order, normalised frame
  P.pos.alloc(n);
  gather_positions_kernel<<<cdiv(n, 256), 256, 0, s>>>(xyz, P.perm, n, inv2e, P.pos);
  FMM_LAUNCHED("gather_positions_kernel");

  // ---- S4: adaptive octree, breadth first
  Cells& C = P.cells;
  C.n = 0;
  C.reserve(std::max<int64_t>(1024, 2 * n / std::max(1, P.ncrit) + 64), s);
  root_kernel<<<1, 1, 0, s>>>(n, C.level, C.begin, C.end, C.child, C.nchild, C.parent, C.anchor);
  FMM_LAUNCHED("root_kernel");
  C.n = 1;
  P.level_begin.assign(1, 0);
  DevBuf<int32_t> nch;
  DevBuf<int64_t> off;
  int64_t lb = 0, le = 1;
  int level = 0;
  for (;;) {
    const int64_t m = le - lb;
    if (nch.count < m) {
      nch.alloc(m);
      off.alloc(m);
    }
    count_children_kernel<<<cdiv(m, 128), 128, 0, s>>>(P.keys, C.begin, C.end, lb, le, level, P.ncrit, nch);
    FMM_LAUNCHED("count_children_kernel");
    const int64_t total = scan_counts_total(nch, off, m, s);
    C.reserve(le + total, s);
    emit_children_kernel<<<cdiv(m, 128), 128, 0, s>>>(P.keys, lb, le, level, nch, off, C.level, C.begin, C.end,
                                                      C.child, C.nchild, C.parent, C.anchor);
    FMM_LAUNCHED("emit_children_kernel");
    P.level_begin.push_back(le);
    if (total == 0) break;
    C.n = le + total;
    lb = le;
    le = C.n;
    ++level;
  }
  C.n = le;
  P.max_level = level;
  C.center.alloc(C.n);
  centers_kernel<<<cdiv(C.n, 256), 256, 0, s>>>(C.level, C.anchor, C.n, P.lo[0], P.lo[1], P.lo[2], P.S, C.center);
  FMM_LAUNCHED("centers_kernel");

  // leaf list (ascending cell index)
  DevBuf<int32_t> flag;
  DevBuf<int64_t> loff;
  flag.alloc(C.n);
  loff.alloc(C.n);
  leaf_flag_kernel<<<cdiv(C.n, 256), 256, 0, s>>>(C.child, C.n, flag);
  FMM_LAUNCHED("leaf_flag_kernel");
  P.nleaves = scan_counts_total(flag, loff, C.n, s);
  P.leaves.alloc(P.nleaves);
  compact_kernel<<<cdiv(C.n, 256), 256, 0, s>>>(flag, loff, C.n, P.leaves);
  FMM_LAUNCHED("compact_kernel");
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fmm
