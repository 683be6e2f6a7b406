// traverse.cu — setup step S5: dual tree traversal with the multipole
// acceptance criterion (§2.2: "dual tree traversal along
// with the multipole acceptance criterion to construct optimal interaction
// lists"), emitting the P2P (near, "dense diagonal blocks") and M2L
// ("off-diagonal blocks") lists.
//
// GPU formulation: level-synchronous frontier of (target A, source B) cell
// pairs. Each round classifies every pair (integer MAC R10/R11, split rule
// R12), then compacts the three outputs with exclusive scans, so the emitted
// order is deterministic. The pair SET equals the recursive formulation's
// (same decision per pair); only the order differs. Lists are then grouped by
// target with the stable radix sort.
#include <algorithm>

#include "plan.h"

namespace fmm {
namespace {

struct PairAction {
  int m2l, p2p, nsplit;
  bool split_a;
};

__device__ __forceinline__ PairAction classify(int A, int B, const int32_t* __restrict__ level,
                                               const int32_t* __restrict__ anchor, const int32_t* __restrict__ child,
                                               const int32_t* __restrict__ nchild, double theta2) {
  const int la = level[A], lb = level[B];
  const int64_t ha = (int64_t)1 << (kMaxLevel - la), hb = (int64_t)1 << (kMaxLevel - lb);
  int64_t d2 = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    int64_t ca = (2 * (int64_t)anchor[3 * A + k] + 1) * ha;
    int64_t cb = (2 * (int64_t)anchor[3 * B + k] + 1) * hb;
    d2 += (ca - cb) * (ca - cb);
  }
  const int64_t r = ha + hb;
  PairAction act{0, 0, 0, false};
  // R10/R11: accept iff (theta*theta) * D^2 > (H_A + H_B)^2, two IEEE multiplies then compare
  if (__dmul_rn(theta2, (double)d2) > (double)(r * r)) {
    act.m2l = 1;
    return act;
  }
  const bool leaf_a = child[A] < 0, leaf_b = child[B] < 0;
  if (leaf_a && leaf_b) {
    act.p2p = 1;
    return act;
  }
  // R12: split the target if the source is a leaf, or the target is not a leaf and not deeper
  act.split_a = leaf_b || (!leaf_a && la <= lb);
  act.nsplit = act.split_a ? nchild[A] : nchild[B];
  return act;
}

__global__ void classify_kernel(const int2* __restrict__ fr, int64_t nf, const int32_t* __restrict__ level,
                                const int32_t* __restrict__ anchor, const int32_t* __restrict__ child,
                                const int32_t* __restrict__ nchild, double theta2, int32_t* __restrict__ cm,
                                int32_t* __restrict__ cp, int32_t* __restrict__ cn) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  int2 pr = fr[i];
  PairAction a = classify(pr.x, pr.y, level, anchor, child, nchild, theta2);
  cm[i] = a.m2l;
  cp[i] = a.p2p;
  cn[i] = a.nsplit;
}

__global__ void emit_kernel(const int2* __restrict__ fr, int64_t nf, const int32_t* __restrict__ level,
                            const int32_t* __restrict__ anchor, const int32_t* __restrict__ child,
                            const int32_t* __restrict__ nchild, double theta2, const int64_t* __restrict__ om,
                            const int64_t* __restrict__ op, const int64_t* __restrict__ on, int64_t base_m,
                            int64_t base_p, int32_t* __restrict__ m_tgt, int32_t* __restrict__ m_src,
                            int32_t* __restrict__ p_tgt, int32_t* __restrict__ p_src, int2* __restrict__ next) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  int2 pr = fr[i];
  PairAction a = classify(pr.x, pr.y, level, anchor, child, nchild, theta2);
  if (a.m2l) {
    m_tgt[base_m + om[i]] = pr.x;
    m_src[base_m + om[i]] = pr.y;
  } else if (a.p2p) {
    p_tgt[base_p + op[i]] = pr.x;
    p_src[base_p + op[i]] = pr.y;
  } else {
    int64_t w = on[i];
    if (a.split_a) {
      int c0 = child[pr.x];
      for (int k = 0; k < a.nsplit; ++k) next[w + k] = make_int2(c0 + k, pr.y);
    } else {
      int c0 = child[pr.y];
      for (int k = 0; k < a.nsplit; ++k) next[w + k] = make_int2(pr.x, c0 + k);
    }
  }
}

__global__ void widen_kernel(const int32_t* __restrict__ t, int64_t n, uint64_t* __restrict__ k) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) k[i] = (uint64_t)(uint32_t)t[i];
}

__global__ void narrow_kernel(const uint64_t* __restrict__ k, const uint32_t* __restrict__ v, int64_t n,
                              int32_t* __restrict__ t, int32_t* __restrict__ s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    t[i] = (int32_t)k[i];
    s[i] = (int32_t)v[i];
  }
}

// off[c] = first pair index with target >= c, for c in [0, ncells]; tgt sorted ascending
__global__ void offsets_kernel(const int32_t* __restrict__ tgt, int64_t n, int64_t ncells, int32_t* __restrict__ off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  int64_t lo = i == 0 ? 0 : (int64_t)tgt[i - 1] + 1;
  int64_t hi = i == n ? ncells : (int64_t)tgt[i];
  for (int64_t c = lo; c <= hi; ++c) off[c] = (int32_t)i;
}

__global__ void p2p_work_kernel(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src, int64_t n,
                                const int32_t* __restrict__ cb, const int32_t* __restrict__ ce,
                                unsigned long long* __restrict__ total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long w = 0;
  if (i < n) w = (unsigned long long)(ce[tgt[i]] - cb[tgt[i]]) * (unsigned long long)(ce[src[i]] - cb[src[i]]);
  for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(total, w);
}

void group_by_target(PairList& L, int64_t ncells, cudaStream_t s) {
  const int64_t n = L.n;
  L.off.alloc(ncells + 1);
  if (n > 0) {
    DevBuf<uint64_t> k;
    DevBuf<uint32_t> v;
    k.alloc(n);
    v.alloc(n);
    widen_kernel<<<cdiv(n, 256), 256, 0, s>>>(L.tgt, n, k);
    FMM_LAUNCHED("widen_kernel");
    FMM_CUDA(cudaMemcpyAsync(v.ptr, L.src.ptr, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    int bits = 1;
    while (((int64_t)1 << bits) < ncells) ++bits;
    radix_sort_pairs(k, v, n, bits, s);
    narrow_kernel<<<cdiv(n, 256), 256, 0, s>>>(k, v, n, L.tgt, L.src);
    FMM_LAUNCHED("narrow_kernel");
  }
  offsets_kernel<<<cdiv(n + 1, 256), 256, 0, s>>>(L.tgt, n, ncells, L.off);
  FMM_LAUNCHED("offsets_kernel");
}

}  // namespace

void traverse(fmm_plan_s& P) {
  cudaStream_t s = P.stream;
  const Cells& C = P.cells;
  DevBuf<int2> fr, nx;
  DevBuf<int32_t> cm, cp, cn;
  DevBuf<int64_t> om, op, on;
  fr.alloc(1);
  const int2 root = make_int2(0, 0);
  FMM_CUDA(cudaMemcpyAsync(fr.ptr, &root, sizeof(int2), cudaMemcpyHostToDevice, s));
  int64_t nf = 1;
  P.m2l.n = P.p2p.n = 0;
  int64_t cap_m = std::max<int64_t>(1024, 64 * C.n), cap_p = std::max<int64_t>(1024, 32 * P.nleaves);
  P.m2l.tgt.alloc(cap_m);
  P.m2l.src.alloc(cap_m);
  P.p2p.tgt.alloc(cap_p);
  P.p2p.src.alloc(cap_p);
  while (nf > 0) {
    if (cm.count < nf) {
      int64_t c = std::max<int64_t>(nf, 2 * cm.count);
      cm.alloc(c);
      cp.alloc(c);
      cn.alloc(c);
      om.alloc(c);
      op.alloc(c);
      on.alloc(c);
    }
    classify_kernel<<<cdiv(nf, 256), 256, 0, s>>>(fr, nf, C.level, C.anchor, C.child, C.nchild, P.theta2, cm, cp,
                                                  cn);
    FMM_LAUNCHED("classify_kernel");
    const int64_t tm = scan_counts_total(cm, om, nf, s);
    const int64_t tp = scan_counts_total(cp, op, nf, s);
    const int64_t tn = scan_counts_total(cn, on, nf, s);
    if (P.m2l.n + tm > P.m2l.tgt.count) {
      int64_t c = std::max(P.m2l.n + tm, 2 * P.m2l.tgt.count);
      P.m2l.tgt.grow(c, P.m2l.n, s);
      P.m2l.src.grow(c, P.m2l.n, s);
    }
    if (P.p2p.n + tp > P.p2p.tgt.count) {
      int64_t c = std::max(P.p2p.n + tp, 2 * P.p2p.tgt.count);
      P.p2p.tgt.grow(c, P.p2p.n, s);
      P.p2p.src.grow(c, P.p2p.n, s);
    }
    if (nx.count < tn) nx.alloc(std::max<int64_t>(tn, 2 * nx.count));
    emit_kernel<<<cdiv(nf, 256), 256, 0, s>>>(fr, nf, C.level, C.anchor, C.child, C.nchild, P.theta2, om, op, on,
                                              P.m2l.n, P.p2p.n, P.m2l.tgt, P.m2l.src, P.p2p.tgt, P.p2p.src, nx);
    FMM_LAUNCHED("emit_kernel");
    P.m2l.n += tm;
    P.p2p.n += tp;
    std::swap(fr, nx);
    nf = tn;
  }
  group_by_target(P.m2l, C.n, s);
  group_by_target(P.p2p, C.n, s);
  // near-field work (interactions incl. self terms), for stats and the roofline
  DevBuf<unsigned long long> tot;
  tot.alloc(1);
  FMM_CUDA(cudaMemsetAsync(tot.ptr, 0, sizeof(unsigned long long), s));
  if (P.p2p.n > 0) {
    p2p_work_kernel<<<cdiv(P.p2p.n, 256), 256, 0, s>>>(P.p2p.tgt, P.p2p.src, P.p2p.n, C.begin, C.end, tot);
    FMM_LAUNCHED("p2p_work_kernel");
  }
  unsigned long long h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, tot.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  P.n_p2p_interactions = (int64_t)h;
}

}  // namespace fmm
