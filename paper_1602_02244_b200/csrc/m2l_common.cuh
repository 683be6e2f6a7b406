// m2l_common.cuh — helpers shared by the M2L class-operator kernels (m2l_dmma.cu: v2 dense
// operators, m2l_rot.cu: v3 rotation-factored operators).
#pragma once
#include <vector>

#include "plan.h"

namespace fmm {
namespace m2l {

// real (p+1)^2 basis: (n,0) -> n^2, (n,m,re) -> n^2+2m-1, (n,m,im) -> n^2+2m
__host__ __device__ inline int real_count(int p) { return (p + 1) * (p + 1); }

// real index -> (n, m, part)
__host__ __device__ inline void real_decode(int r, int& n, int& m, int& part) {
  n = 0;
  while ((n + 1) * (n + 1) <= r) ++n;
  const int t = r - n * n;
  m = (t + 1) >> 1;
  part = t > 0 ? ((t + 1) & 1) : 0;
}
__host__ __device__ inline int real_index(int n, int m, int part) { return m == 0 ? n * n : n * n + 2 * m - 1 + part; }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}


struct M2LArgs {
  const double* ops;
  const int32_t* col_src;
  const int32_t* col_meta;
  const int32_t* chunk_begin;
  const int32_t* chunk_class;
  const int32_t* chunk_seg;  // [nchunks + 1] first slot segment of each chunk
  const int32_t* seg_begin;  // [nseg + 1] first column of each segment (global index)
  const int32_t* tile_chunk;
  const int32_t* tile_cells;
  const int32_t* symtab;  // [16][2][NR]
  const double* hpow;     // [22][p+2]
  const int32_t* level;
  const double* Mt;       // [ncells][Kpad] scaled real-form multipoles
  double2* L;
  int p, nc, NR, NRpad, Kpad, nks, nmt, T, NC, ystride;
};

// per-row output transform for all 16 g: bit 2g = take the re/im partner row, bit 2g+1 = negate
__device__ __forceinline__ uint32_t ltrans_mask(const int32_t* sym, int NR, int r, int& partner_off) {
  uint32_t mask = 0;
  partner_off = 0;
  for (int g = 0; g < 16; ++g) {
    const int ent = sym[(g * 2 + 1) * NR + r];
    const int src = ent & 0xffff;
    if (src != r) {
      partner_off = src - r;
      mask |= 1u << (2 * g);
    }
    if (ent >> 16) mask |= 2u << (2 * g);
  }
  return mask;
}

// chunk metadata (columns + slot segments) into buffer slot b
__device__ __forceinline__ void load_meta_dev(const M2LArgs& a, int ch, int32_t* meta, int32_t* srcs, int32_t* sslot,
                                              int32_t* sbeg, int t0, int nt) {
  const int cb = a.chunk_begin[ch], ncol = a.chunk_begin[ch + 1] - cb;
  const int s0 = a.chunk_seg[ch], ns = a.chunk_seg[ch + 1] - s0;
  for (int t = t0; t < a.NC; t += nt) {
    meta[t] = t < ncol ? a.col_meta[cb + t] : 0;
    srcs[t] = t < ncol ? a.col_src[cb + t] : 0;
    if (t < ns) sslot[t] = a.col_meta[a.seg_begin[s0 + t]] & 0xff;
  }
  for (int t = t0; t <= ns; t += nt) sbeg[t] = a.seg_begin[s0 + t] - cb;
}

// Host: signed-permutation tables of the 16 axis flips / x-y swap on multipole (which = 0,
// inverse map) and local (which = 1) real coefficients; [16][2][NR], bits 0..15 source
// index, bit 16 negative sign (m2l_dmma.cu).
std::vector<int32_t> build_symtab(int p);

}  // namespace m2l
}  // namespace fmm
