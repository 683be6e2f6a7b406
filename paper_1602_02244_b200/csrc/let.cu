// let.cu — S14 multi-GPU mat-vec with a local-essential-tree (LET) exchange
// (north_star: "partitioned across the 8xB200 box by Morton-ordered domain
// decomposition, with a local-essential-tree exchange (boundary multipoles plus
// halo particles) over NCCL/NVLink").
//
// Every rank holds the same global tree and interaction lists (built by fmm_setup
// from the all-gathered points), so the approximation is the single-GPU one
// (reading R12). Rank r owns the Morton particle range [B_r, B_{r+1}) cut at leaf
// boundaries. Per mat-vec (the caller moves the buffers with its collectives):
//   1. q: each rank sends every charge of its caller slice to the owner of the
//      particle and to every rank whose near field needs it (halo leaves);
//   2. upward pass on the owned particles only: P2M of own leaves, M2M of the cells
//      overlapping the range (their children outside it read as zero, so a cell
//      straddling several ranks holds this rank's PARTIAL multipole, by linearity
//      of M2M);
//   3. shared (straddling) cells: all partials are all-gathered and summed in
//      rank order (deterministic); boundary multipoles: each rank sends the
//      complete multipoles of its own cells that are M2L sources of another
//      rank's targets;
//   4. M2L for the targets overlapping the range (a rank-local pair list), L2L of
//      the cells overlapping it, near field of own leaves (halo charges received in
//      step 1), results in owned Morton order;
//   5. results are routed back to the callers' slices.
// Index lists are built on the host at fmm_let_setup from the global tree; the
// moves are gathers/scatters on the device. let_lists() is plain host code with
// no CUDA calls (tested on CPU against a brute-force model, tests/test_let.py).
#include <algorithm>
#include <cstring>
#include <vector>

#include "plan.h"

namespace fmm {

// ----------------------------------------------------------------------------- host
// Owner range cuts, cost-weighted (the Plummer tree is strongly non-uniform, so
// equal particle counts are not equal work). Each target cell's work is spread evenly over its
// particles: 11 flop per P2P interaction of a target leaf, kM2LCost per M2L pair of a target
// cell (the pairs of an ancestor are shared by the leaves below it), plus a per-particle term
// for P2M / L2P. Rank r's range starts at the first leaf boundary where the running weight
// reaches r / world of the total, so ranges are contiguous in Morton order and never split a
// leaf (one 3-D -> 1-D ordering serves locality and partitioning).
std::vector<int64_t> let_cuts(int64_t n, int world, int p, const int32_t* cbeg, const int32_t* cend, int64_t nleaves,
                              const int32_t* leaves /*sorted by begin*/, int64_t np2p, const int32_t* p2p_tgt,
                              const int32_t* p2p_src, int64_t nm2l, const int32_t* m2l_tgt) {
  std::vector<double> dens(n + 1, 0.0);  // difference array of per-particle cost density
  auto spread = [&](int32_t c, double w) {
    const int64_t a = cbeg[c], b = cend[c];
    if (b <= a) return;
    dens[a] += w / (double)(b - a);
    dens[b] -= w / (double)(b - a);
  };
  const double m2l_cost = 6.0 * (p + 1.0) * (p + 1.0) * (p + 1.0);  // executed flops of one rotation-form pair
  for (int64_t k = 0; k < np2p; ++k)
    spread(p2p_tgt[k], 11.0 * (double)(cend[p2p_tgt[k]] - cbeg[p2p_tgt[k]]) * (cend[p2p_src[k]] - cbeg[p2p_src[k]]));
  for (int64_t k = 0; k < nm2l; ++k) spread(m2l_tgt[k], m2l_cost);
  const double per_particle = 18.0 * (p + 1.0) * (p + 2.0) / 2.0;  // P2M + L2P
  std::vector<double> leafw(nleaves + 1, 0.0);  // prefix sums of leaf weights in Morton order
  double run = 0.0;
  int64_t pos = 0;
  double acc = 0.0;
  for (int64_t i = 0; i < nleaves; ++i) {
    const int64_t a = cbeg[leaves[i]], b = cend[leaves[i]];
    double w = 0.0;
    for (; pos < a; ++pos) run += dens[pos];
    for (; pos < b; ++pos) {
      run += dens[pos];
      w += run + per_particle;
    }
    acc += w;
    leafw[i + 1] = acc;
  }
  std::vector<int64_t> B(world + 1);
  for (int r = 0; r <= world; ++r) {
    const double target = acc * r / world;
    const int64_t i = std::lower_bound(leafw.begin(), leafw.end(), target) - leafw.begin();  // first prefix >= target
    B[r] = i < nleaves ? cbeg[leaves[i]] : n;
  }
  B[0] = 0;
  B[world] = n;
  for (int r = 1; r <= world; ++r) B[r] = std::max(B[r], B[r - 1]);
  return B;
}

namespace {
int find_rank(const std::vector<int64_t>& off, int64_t x) {  // off[r] <= x < off[r+1]
  return (int)(std::upper_bound(off.begin(), off.end(), x) - off.begin()) - 1;
}
}  // namespace

// All index lists of rank `me` (host arrays in, host vectors out). See fmm.h fmm_let_*.
void let_lists(int64_t n, int world, int me, int p, const int64_t* caller_off /*[world+1]*/, const uint32_t* perm,
               int64_t ncells, const int32_t* cbeg, const int32_t* cend, int64_t nleaves,
               const int32_t* leaves /*sorted by begin*/, int64_t np2p, const int32_t* p2p_tgt,
               const int32_t* p2p_src, int64_t nm2l, const int32_t* m2l_tgt, const int32_t* m2l_src,
               LetLists& out) {
  const std::vector<int64_t> B =
      let_cuts(n, world, p, cbeg, cend, nleaves, leaves, np2p, p2p_tgt, p2p_src, nm2l, m2l_tgt);
  const std::vector<int64_t> C(caller_off, caller_off + world + 1);
  out.world = world;
  out.rank_begin = B;
  auto owner = [&](int64_t s) { return find_rank(B, s); };
  auto caller = [&](int64_t s) { return find_rank(C, (int64_t)perm[s]); };
  // ---- halo leaves of every rank: P2P sources outside the range of the target's owner
  std::vector<std::vector<int32_t>> halo(world);
  for (int64_t k = 0; k < np2p; ++k) {
    const int t = p2p_tgt[k], s = p2p_src[k];
    const int d = owner(cbeg[t]);
    if (owner(cbeg[s]) != d) halo[d].push_back(s);
  }
  for (auto& h : halo) {
    std::sort(h.begin(), h.end(), [&](int a, int b) { return cbeg[a] < cbeg[b]; });
    h.erase(std::unique(h.begin(), h.end()), h.end());
  }
  // positions needed by rank d: its range and its halo leaves, ascending
  auto needed = [&](int d, std::vector<int64_t>& pos) {
    pos.clear();
    size_t hi = 0;
    int64_t s = B[d];
    // merge the owned range with the halo ranges (all disjoint from it)
    while (true) {
      const int64_t hb = hi < halo[d].size() ? cbeg[halo[d][hi]] : INT64_MAX;
      if (s < B[d + 1] && s < hb) {
        pos.push_back(s++);
      } else if (hi < halo[d].size()) {
        for (int64_t x = cbeg[halo[d][hi]]; x < cend[halo[d][hi]]; ++x) pos.push_back(x);
        ++hi;
      } else {
        break;
      }
    }
  };
  // ---- q: send (my caller rows -> each d), receive (positions from each r)
  out.q_send.assign(world, 0);
  out.q_recv.assign(world, 0);
  out.q_send_rows.clear();
  out.q_recv_pos.clear();
  std::vector<int64_t> pos;
  for (int d = 0; d < world; ++d) {
    needed(d, pos);
    for (int64_t s : pos)
      if (caller(s) == me) {
        out.q_send_rows.push_back((int64_t)perm[s] - C[me]);
        ++out.q_send[d];
      }
  }
  needed(me, pos);
  for (int r = 0; r < world; ++r)
    for (int64_t s : pos)
      if (caller(s) == r) {
        out.q_recv_pos.push_back(s);
        ++out.q_recv[r];
      }
  // ---- shared cells (straddling at least two ranges), cell order
  out.shared.clear();
  std::vector<char> is_shared(ncells, 0);
  for (int64_t c = 0; c < ncells; ++c)
    if (cend[c] > cbeg[c] && owner(cbeg[c]) != owner(cend[c] - 1)) {
      out.shared.push_back((int32_t)c);
      is_shared[c] = 1;
    }
  // ---- boundary multipoles: (cell owner r) -> (rank d whose targets use it), unique, cell order
  std::vector<std::vector<int32_t>> need_from(world);  // me receives from r
  std::vector<std::vector<int32_t>> send_to(world);    // me sends to d
  for (int64_t k = 0; k < nm2l; ++k) {
    const int t = m2l_tgt[k], s = m2l_src[k];
    if (is_shared[s]) continue;
    const int os = owner(cbeg[s]);
    const int d0 = owner(cbeg[t]), d1 = owner(cend[t] - 1);
    for (int d = d0; d <= d1; ++d) {
      if (d == os) continue;
      if (d == me) need_from[os].push_back(s);
      if (os == me) send_to[d].push_back(s);
    }
  }
  out.m_send.assign(world, 0);
  out.m_recv.assign(world, 0);
  out.m_send_cells.clear();
  out.m_recv_cells.clear();
  for (int r = 0; r < world; ++r) {
    auto& a = send_to[r];
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    out.m_send[r] = (int64_t)a.size();
    out.m_send_cells.insert(out.m_send_cells.end(), a.begin(), a.end());
    auto& b = need_from[r];
    std::sort(b.begin(), b.end());
    b.erase(std::unique(b.begin(), b.end()), b.end());
    out.m_recv[r] = (int64_t)b.size();
    out.m_recv_cells.insert(out.m_recv_cells.end(), b.begin(), b.end());
  }
  // ---- results: my owned positions -> their caller rank; positions whose caller is me, by owner
  out.phi_send.assign(world, 0);
  out.phi_recv.assign(world, 0);
  out.phi_send_idx.clear();
  out.phi_recv_rows.clear();
  for (int r = 0; r < world; ++r)
    for (int64_t s = B[me]; s < B[me + 1]; ++s)
      if (caller(s) == r) {
        out.phi_send_idx.push_back(s - B[me]);
        ++out.phi_send[r];
      }
  for (int d = 0; d < world; ++d)
    for (int64_t s = B[d]; s < B[d + 1]; ++s)
      if (caller(s) == me) {
        out.phi_recv_rows.push_back((int64_t)perm[s] - C[me]);
        ++out.phi_recv[d];
      }
}

// ----------------------------------------------------------------------------- device
namespace {

__global__ void gather_rows_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                                   int width, double* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * width) return;
  const int64_t k = e / width;
  dst[e] = src[idx[k] * width + (e - k * width)];
}

__global__ void scatter_rows_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                                    int width, double* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * width) return;
  const int64_t k = e / width;
  dst[idx[k] * width + (e - k * width)] = src[e];
}

// received charges into pos[].w of their (Morton) positions; non-finite flagged
__global__ void scatter_q_kernel(const double* __restrict__ q, const int64_t* __restrict__ pos_idx, int64_t n,
                                 double4* __restrict__ pos, int32_t* __restrict__ flags) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (k < n) {
    const double v = q[k];
    bad = !isfinite(v);
    pos[pos_idx[k]].w = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
}

// M[shared c] = sum over ranks r (in rank order) of the partials recv[r][k]
__global__ void sum_shared_kernel(const double* __restrict__ recv, const int32_t* __restrict__ cells, int64_t ns,
                                  int world, int ncd, double* __restrict__ M) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ns * ncd) return;
  const int64_t k = e / ncd;
  double v = 0.0;
  for (int r = 0; r < world; ++r) v += recv[((int64_t)r * ns + k) * ncd + (e - k * ncd)];
  M[(int64_t)cells[k] * ncd + (e - k * ncd)] = v;
}

__global__ void zero_cells_kernel(const int32_t* __restrict__ cells, int64_t n, int ncd, double* __restrict__ M) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * ncd) return;
  const int64_t k = e / ncd;
  M[(int64_t)cells[k] * ncd + (e - k * ncd)] = 0.0;
}

template <typename T>
void upload(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.alloc((int64_t)h.size());
  if (!h.empty()) FMM_CUDA(cudaMemcpyAsync(d.ptr, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
}

}  // namespace

// host copies of the tree and lists the partition and the exchange lists are built from
void let_host_copy(fmm_plan_s& P) {
  LetHost& H = P.let_host;
  if (H.valid) return;
  cudaStream_t s = P.stream;
  const int64_t nc = P.cells.n;
  H.perm.resize(P.n);
  H.cb.resize(nc);
  H.ce.resize(nc);
  H.child.resize(nc);
  H.nchild.resize(nc);
  H.lv.resize(P.nleaves);
  H.pt.resize(P.p2p.n);
  H.ps.resize(P.p2p.n);
  H.mt.resize(P.m2l.n);
  H.ms.resize(P.m2l.n);
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) FMM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  };
  d2h(H.perm.data(), P.perm.ptr, sizeof(uint32_t) * P.n);
  d2h(H.cb.data(), P.cells.begin.ptr, sizeof(int32_t) * nc);
  d2h(H.ce.data(), P.cells.end.ptr, sizeof(int32_t) * nc);
  d2h(H.child.data(), P.cells.child.ptr, sizeof(int32_t) * nc);
  d2h(H.nchild.data(), P.cells.nchild.ptr, sizeof(int32_t) * nc);
  d2h(H.lv.data(), P.leaves.ptr, sizeof(int32_t) * P.nleaves);
  d2h(H.pt.data(), P.p2p.tgt.ptr, sizeof(int32_t) * P.p2p.n);
  d2h(H.ps.data(), P.p2p.src.ptr, sizeof(int32_t) * P.p2p.n);
  d2h(H.mt.data(), P.m2l.tgt.ptr, sizeof(int32_t) * P.m2l.n);
  d2h(H.ms.data(), P.m2l.src.ptr, sizeof(int32_t) * P.m2l.n);
  FMM_CUDA(cudaStreamSynchronize(s));
  H.valid = true;
}

// this rank's Morton range (cost-weighted cut at leaf boundaries, let_cuts)
void let_partition(fmm_plan_s& P) {
  let_host_copy(P);
  const LetHost& H = P.let_host;
  const std::vector<int64_t> B = let_cuts(P.n, P.world, P.p, H.cb.data(), H.ce.data(), P.nleaves, H.lv.data(), P.p2p.n,
                                          H.pt.data(), H.ps.data(), P.m2l.n, H.mt.data());
  P.own_begin = B[P.rank];
  P.own_end = B[P.rank + 1];
  P.own_leaf_begin = std::lower_bound(H.lv.begin(), H.lv.end(), P.own_begin,
                                      [&](int32_t l, int64_t v) { return H.cb[l] < v; }) - H.lv.begin();
  P.own_leaf_end = std::lower_bound(H.lv.begin(), H.lv.end(), P.own_end,
                                    [&](int32_t l, int64_t v) { return H.cb[l] < v; }) - H.lv.begin();
}

void let_setup(fmm_plan_s& P, const int64_t* caller_counts) {
  cudaStream_t s = P.stream;
  std::vector<int64_t> C(P.world + 1, 0);
  for (int r = 0; r < P.world; ++r) {
    if (caller_counts[r] < 0) throw Error(FMM_ERR_USAGE, "fmm_let_setup: negative caller count");
    C[r + 1] = C[r] + caller_counts[r];
  }
  if (C[P.world] != P.n) throw Error(FMM_ERR_USAGE, "fmm_let_setup: caller counts do not sum to n");
  let_host_copy(P);
  const LetHost& H = P.let_host;
  const int64_t nc = P.cells.n;
  LetLists& L = P.let;
  let_lists(P.n, P.world, P.rank, P.p, C.data(), H.perm.data(), nc, H.cb.data(), H.ce.data(), P.nleaves,
            H.lv.data(), P.p2p.n, H.pt.data(), H.ps.data(), P.m2l.n, H.mt.data(), H.ms.data(), L);
  // this rank's range must be the one let_partition picked (same cut rule)
  if (L.rank_begin[P.rank] != P.own_begin || L.rank_begin[P.rank + 1] != P.own_end)
    throw Error(FMM_ERR_CUDA, "fmm_let_setup: owner range mismatch");
  upload(P.let_dev.q_send_rows, L.q_send_rows, s);
  upload(P.let_dev.q_recv_pos, L.q_recv_pos, s);
  std::vector<int64_t> sh(L.shared.begin(), L.shared.end()), msend(L.m_send_cells.begin(), L.m_send_cells.end()),
      mrecv(L.m_recv_cells.begin(), L.m_recv_cells.end());
  upload(P.let_dev.shared, sh, s);
  upload(P.let_dev.m_send_cells, msend, s);
  upload(P.let_dev.m_recv_cells, mrecv, s);
  upload(P.let_dev.phi_send_idx, L.phi_send_idx, s);
  upload(P.let_dev.phi_recv_rows, L.phi_recv_rows, s);
  std::vector<int32_t> sh32(L.shared.begin(), L.shared.end());
  upload(P.let_dev.shared32, sh32, s);
  P.let_dev.phi_own.alloc(std::max<int64_t>(1, P.own_end - P.own_begin));
  P.let_dev.grad_own.alloc(std::max<int64_t>(1, 3 * (P.own_end - P.own_begin)));
  // ---- the rank-local passes (only what this rank's targets need):
  // per level, the cells overlapping the owned range (contiguous: cells of a level are in
  // Morton order); children of those that lie outside it, and shared cells that lie outside
  // it, hold zero multipoles (M2M inputs, this rank's partials); M2L pairs whose target
  // overlaps the range
  const int64_t ob = P.own_begin, oe = P.own_end;
  auto overlaps = [&](int64_t c) { return H.ce[c] > ob && H.cb[c] < oe && H.ce[c] > H.cb[c]; };
  P.let_level_lo.assign(P.max_level + 1, 0);
  P.let_level_hi.assign(P.max_level + 1, 0);
  std::vector<int32_t> zero;
  for (int l = 0; l <= P.max_level; ++l) {
    int64_t lo = P.level_begin[l + 1], hi = P.level_begin[l];
    for (int64_t c = P.level_begin[l]; c < P.level_begin[l + 1]; ++c)
      if (overlaps(c)) {
        lo = std::min(lo, c);
        hi = std::max(hi, c + 1);
      }
    if (hi <= lo) lo = hi = P.level_begin[l];
    P.let_level_lo[l] = lo;
    P.let_level_hi[l] = hi;
    for (int64_t c = lo; c < hi; ++c)
      for (int k = 0; k < H.nchild[c]; ++k)
        if (!overlaps(H.child[c] + k)) zero.push_back(H.child[c] + k);
  }
  for (int32_t c : L.shared)  // a straddling cell away from this range: this rank's partial is 0
    if (!overlaps(c)) zero.push_back(c);
  upload(P.let_dev.zero_cells, zero, s);
  std::vector<int32_t> ot, os;
  for (int64_t k = 0; k < P.m2l.n; ++k)
    if (overlaps(H.mt[k])) {
      ot.push_back(H.mt[k]);
      os.push_back(H.ms[k]);
    }
  upload(P.let_dev.m2l_tgt, ot, s);
  upload(P.let_dev.m2l_src, os, s);
  if (P.m2l_variant == 4) m2l_v4_resize(P, (int64_t)ot.size());
  P.let_ready = true;
  P.let_host = LetHost{};  // the host copies are no longer needed
  FMM_CUDA(cudaStreamSynchronize(s));
}

namespace {
void gather(const double* src, const DevBuf<int64_t>& idx, int width, double* dst, cudaStream_t s) {
  const int64_t n = idx.count;
  if (n == 0) return;
  gather_rows_kernel<<<cdiv(n * width, 256), 256, 0, s>>>(src, idx.ptr, n, width, dst);
  FMM_LAUNCHED("gather_rows_kernel");
}
void scatter(const double* src, const DevBuf<int64_t>& idx, int width, double* dst, cudaStream_t s) {
  const int64_t n = idx.count;
  if (n == 0) return;
  scatter_rows_kernel<<<cdiv(n * width, 256), 256, 0, s>>>(src, idx.ptr, n, width, dst);
  FMM_LAUNCHED("scatter_rows_kernel");
}
}  // namespace

void let_pack_q(fmm_plan_s& P, const double* q_local, double* send) {
  gather(q_local, P.let_dev.q_send_rows, 1, send, P.stream);
}

void let_upward(fmm_plan_s& P, const double* q_recv, double* shared_send, double* m_send) {
  cudaStream_t s = P.stream;
  const int64_t n = P.let_dev.q_recv_pos.count;
  if (n > 0) {
    scatter_q_kernel<<<cdiv(n, 256), 256, 0, s>>>(q_recv, P.let_dev.q_recv_pos.ptr, n, P.pos, P.flags);
    FMM_LAUNCHED("scatter_q_kernel");
  }
  const int64_t nz = P.let_dev.zero_cells.count;  // children outside the range of cells inside it
  if (nz > 0) {
    zero_cells_kernel<<<cdiv(nz * 2 * P.nc, 256), 256, 0, s>>>(P.let_dev.zero_cells.ptr, nz, 2 * P.nc,
                                                                (double*)P.M.ptr);
    FMM_LAUNCHED("zero_cells_kernel");
  }
  upward_own(P);
  gather((const double*)P.M.ptr, P.let_dev.shared, 2 * P.nc, shared_send, s);
  gather((const double*)P.M.ptr, P.let_dev.m_send_cells, 2 * P.nc, m_send, s);
}

void let_exchange_in(fmm_plan_s& P, const double* shared_recv, const double* m_recv) {
  cudaStream_t s = P.stream;
  const int64_t ns = P.let_dev.shared32.count, ncd = 2 * P.nc;
  if (ns > 0) {
    sum_shared_kernel<<<cdiv(ns * ncd, 256), 256, 0, s>>>(shared_recv, P.let_dev.shared32.ptr, ns, P.world, (int)ncd,
                                                           (double*)P.M.ptr);
    FMM_LAUNCHED("sum_shared_kernel");
  }
  scatter(m_recv, P.let_dev.m_recv_cells, (int)ncd, (double*)P.M.ptr, s);
}

void let_pack_phi(fmm_plan_s& P, double* phi_send, double* grad_send) {
  gather(P.let_dev.phi_own.ptr, P.let_dev.phi_send_idx, 1, phi_send, P.stream);
  if (grad_send) gather(P.let_dev.grad_own.ptr, P.let_dev.phi_send_idx, 3, grad_send, P.stream);
}

void let_unpack(fmm_plan_s& P, const double* phi_recv, const double* grad_recv, double* phi, double* grad) {
  scatter(phi_recv, P.let_dev.phi_recv_rows, 1, phi, P.stream);
  if (grad && grad_recv) scatter(grad_recv, P.let_dev.phi_recv_rows, 3, grad, P.stream);
}

}  // namespace fmm
