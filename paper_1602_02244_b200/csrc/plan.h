// plan.h — the internal state behind the opaque fmm_plan of include/fmm.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

#include "../../include/fmm.h"
#include "common.cuh"

namespace fmm {

// Owning device buffer (cudaMalloc / cudaFree), byte accounting in the plan.
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  int64_t count = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count) { o.ptr = nullptr; o.count = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(ptr, o.ptr);
    std::swap(count, o.count);
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    count = 0;
  }
  void alloc(int64_t n) {
    release();
    if (n > 0) FMM_CUDA(cudaMalloc(&ptr, sizeof(T) * n));
    count = n;
  }
  // grow to at least n elements keeping the first `keep` elements
  void grow(int64_t n, int64_t keep, cudaStream_t s) {
    if (n <= count) return;
    T* np = nullptr;
    FMM_CUDA(cudaMalloc(&np, sizeof(T) * n));
    if (ptr && keep > 0) FMM_CUDA(cudaMemcpyAsync(np, ptr, sizeof(T) * keep, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    if (ptr) cudaFree(ptr);
    ptr = np;
    count = n;
  }
  int64_t bytes() const { return count * (int64_t)sizeof(T); }
  operator T*() const { return ptr; }
};

// Cells in breadth-first (level, Morton) order: level_begin[l] .. level_begin[l+1].
struct Cells {
  DevBuf<int32_t> level, begin, end, child, nchild, parent;
  DevBuf<int32_t> anchor;  // [3 * n]
  DevBuf<double4> center;  // x, y, z, half side h (normalised frame)
  int64_t n = 0, cap = 0;
  void reserve(int64_t c, cudaStream_t s);
};

// Pair list grouped by target: src[off[t] .. off[t+1]) are the sources of cell t.
struct PairList {
  DevBuf<int32_t> tgt, src;  // [npairs]
  DevBuf<int32_t> off;       // [ncells + 1]
  int64_t n = 0;
};

// M2L v2 state (m2l_dmma.cu): canonical operator classes, tiles, chunks.
struct M2LDmma {
  int NR = 0, NRpad = 0, nmt = 0, Kpad = 0, nks = 0, NC = 0, T = 0, ystride = 0;
  bool use_ws = false;  // warp-specialised DMMA kernel
  int nhelp = 0;        // its helper warps
  int64_t nclass = 0, ntiles = 0, nchunks = 0, npairs = 0, nseg = 0;
  DevBuf<int32_t> chunk_seg;   // [nchunks + 1] first slot segment of each chunk
  DevBuf<int32_t> seg_begin;   // [nseg + 1] first column of each slot segment
  DevBuf<double> Mt;           // [ncells][Kpad] scaled real-form multipoles (per matvec)
  DevBuf<double> ops;          // [nclass][nmt][nks][32] A fragments
  DevBuf<int32_t> col_src;     // [npairs] source cell per GEMM column
  DevBuf<int32_t> col_meta;    // [npairs] slot | g << 8
  DevBuf<int32_t> chunk_begin; // [nchunks + 1]
  DevBuf<int32_t> chunk_class; // [nchunks]
  DevBuf<int32_t> tile_chunk;  // [ntiles + 1]
  DevBuf<int32_t> tile_cells;  // [ntiles * T], -1 padding
  DevBuf<int32_t> symtab;      // [16][2][NR]
  DevBuf<double> hpow;         // [22][p + 2]
  DevBuf<uint64_t> class_keys; // [nclass] canonical (level difference, offset) keys
  // M2L v3 (m2l_rot.cu): rotation-factored class operators
  DevBuf<double> rot_ops;      // [nclass][rot_blob_size(p)] azimuths, D and Z~ blocks per class
  DevBuf<uint32_t> rot_masks;  // [2][NR] symmetry masks (multipole side, local side)
  DevBuf<int32_t> rot_sched;   // [3][8][rot_smax] MMA-warp item lists
  DevBuf<int32_t> rot_ihdr;    // [nitems] item headers (shape, parts, fragment offset)
  DevBuf<int32_t> rot_ipos;    // [nitems][2][16] item slot positions
  DevBuf<int32_t> rot_desc;    // [nchunks][desc ints] per-chunk descriptors (TMA-loaded)
  DevBuf<int32_t> rot_order;   // [ntiles] launch order of the tiles (decreasing estimated work)
  DevBuf<double> rot_scratch;  // split tiles: [ntiles][split][T][NR] partial accumulators
  int rot_smax = 0, rot_T = 0, rot_nitems = 0, rot_blob = 0;
  int64_t bytes() const {
    return ops.bytes() + col_src.bytes() + col_meta.bytes() + chunk_begin.bytes() + chunk_class.bytes() +
           tile_chunk.bytes() + tile_cells.bytes() + symtab.bytes() + hpow.bytes() + chunk_seg.bytes() +
           seg_begin.bytes() + Mt.bytes() + class_keys.bytes() + rot_ops.bytes() + rot_masks.bytes() +
           rot_sched.bytes() + rot_ihdr.bytes() + rot_ipos.bytes() + rot_desc.bytes() + rot_order.bytes() + rot_scratch.bytes();
  }
};

// M2L v4 state (m2l_v4.cu): work units over the target-grouped pair list, scaled multipoles
struct M2L4 {
  DevBuf<double> Mt;        // [ncells][(p+1)^2] (-1)^n M_n / h^n, degree-major real layout
  DevBuf<double> part;      // [nunits][2][(p+1)^2] partial sums of targets crossing unit boundaries
  DevBuf<double> ihalf;     // [ncells] inverse half sides
  int64_t nunits = 0;       // > 0 if there are M2L pairs (units of chunks of 32 pairs, sized at launch)
  int warps_per_sm = 0;     // 0 = as many as shared memory / registers allow (FMM_V4_WARPS)
  int unit_chunks = 0;      // 0 = balanced at setup (FMM_V4_UNIT_CHUNKS: tests)
  int uchunks = 0, wpc = 1, grid = 1;  // launch geometry (setup)
  size_t smem = 0;
  int64_t bytes() const { return Mt.bytes() + part.bytes() + ihalf.bytes(); }
};

// mutual near field (near_mutual.cu): each unordered leaf pair evaluated once, single GPU, potentials
struct NearMutual {
  bool enabled = false;
  bool big = false;  // a leaf with pairs has more than 64 particles (16 target groups x 2 source lanes)
  DevBuf<int32_t> toff, task_b;  // tasks (A, B > A) grouped by A: [ncells + 1], [ntasks]
  DevBuf<int32_t> tmend;         // [ncells] end of A's mutual tasks (then directed: B on another rank)
  DevBuf<int64_t> poff;          // [ntasks] B-side partial slot
  DevBuf<int32_t> goff;          // [ncells + 1] per leaf, its B-side slots (gslot) in list order
  DevBuf<int64_t> gslot;
  DevBuf<double> partial, own;   // [sum of |B| over tasks], [n] (sorted order)
  int64_t ntasks = 0;
  int64_t bytes() const {
    return toff.bytes() + tmend.bytes() + task_b.bytes() + poff.bytes() + goff.bytes() + gslot.bytes() + partial.bytes() + own.bytes();
  }
};

// Helmholtz plan state (helmholtz.cu, NEXT-4)
struct HelmState {
  DevBuf<double2> qs;         // [n] charges in Morton order
  DevBuf<double2> M, L;       // [ncells][(p+1)^2] spherical-wave expansions
  DevBuf<double2> shift_ops;  // [levels][8][2][(p+1)^2]^2 (S|S) for M2M, (R|R) for L2L, transposed
  DevBuf<double2> m2l_ops;    // [nclass][(p+1)^2]^2 (S|R), transposed
  DevBuf<int32_t> m2l_class;  // [npairs] class of every M2L pair
  int64_t nclass = 0;
  int64_t bytes() const {
    return qs.bytes() + M.bytes() + L.bytes() + shift_ops.bytes() + m2l_ops.bytes() + m2l_class.bytes();
  }
};

// LET exchange lists of one rank (let.cu); counts per peer rank, index lists concatenated in rank order.
struct LetLists {
  int world = 1;
  std::vector<int64_t> rank_begin;                   // [world + 1] owner ranges (Morton positions)
  std::vector<int64_t> q_send, q_recv;               // charges: my caller rows -> d, positions from r
  std::vector<int64_t> q_send_rows, q_recv_pos;
  std::vector<int32_t> shared;                       // straddling cells (all-gathered partials)
  std::vector<int64_t> m_send, m_recv;               // boundary multipoles (cells)
  std::vector<int32_t> m_send_cells, m_recv_cells;
  std::vector<int64_t> phi_send, phi_recv;           // results: owned index -> caller rows
  std::vector<int64_t> phi_send_idx, phi_recv_rows;
};
struct LetDev {
  DevBuf<int64_t> q_send_rows, q_recv_pos, shared, m_send_cells, m_recv_cells, phi_send_idx, phi_recv_rows;
  DevBuf<int32_t> shared32;
  DevBuf<double> phi_own, grad_own;  // owned results in Morton order
  DevBuf<int32_t> zero_cells;        // children outside the owned range of cells overlapping it (M = 0)
  DevBuf<int32_t> m2l_tgt, m2l_src;  // M2L pairs whose target overlaps the owned range (grouped by target)
  // collective mode (fmm_exec.nccl_id): the exchange buffers fmm_matvec moves with NCCL
  DevBuf<double> q_send, q_recv, shared_send, shared_recv, m_send, m_recv, phi_send, phi_recv, grad_send, grad_recv;
  int64_t bytes() const {
    return q_send_rows.bytes() + q_recv_pos.bytes() + shared.bytes() + m_send_cells.bytes() + m_recv_cells.bytes() +
           phi_send_idx.bytes() + phi_recv_rows.bytes() + shared32.bytes() + phi_own.bytes() + grad_own.bytes() +
           zero_cells.bytes() + m2l_tgt.bytes() + m2l_src.bytes() + q_send.bytes() + q_recv.bytes() +
           shared_send.bytes() + shared_recv.bytes() + m_send.bytes() + m_recv.bytes() + phi_send.bytes() +
           phi_recv.bytes() + grad_send.bytes() + grad_recv.bytes();
  }
};
// host copies of the tree and lists while the partition and the exchange lists are built (setup)
struct LetHost {
  bool valid = false;
  std::vector<uint32_t> perm;
  std::vector<int32_t> cb, ce, child, nchild, lv, pt, ps, mt, ms;
};

}  // namespace fmm

struct fmm_plan_s {
  // execution context
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  int dim = 3;  // 2: planar points (x, y, 0) with the 2D log kernel (fmm2d.cu, fmm_setup_2d)
  bool helmholtz = false;  // exp(i kappa r) / r kernel (helmholtz.cu, fmm_setup_helmholtz)
  double kappa = 0;
  fmm::HelmState helm;
  bool poisoned = false;
  bool timing = false;
  bool debug_skip_l2l = false;

  // problem
  int64_t n = 0;
  int p = 0, ncrit = 0, nc = 0;
  double theta = 0, theta2 = 0;
  int e = 0;               // exact normalisation: coordinates are multiplied by 2^-e
  double lo[3] = {0, 0, 0};
  double S = 1, scale = 1; // normalised cube side and 2^21 / S

  // particles in Morton order
  fmm::DevBuf<uint64_t> keys;
  fmm::DevBuf<uint32_t> perm;  // sorted position -> input index
  fmm::DevBuf<double4> pos;    // x, y, z (normalised), q (filled per matvec)

  // tree
  fmm::Cells cells;
  std::vector<int64_t> level_begin;  // host, size max_level + 2
  int max_level = 0;
  int64_t nleaves = 0;
  fmm::DevBuf<int32_t> leaves;       // indices of leaf cells (ascending)

  // interaction lists (dual tree traversal)
  fmm::PairList p2p, m2l;
  int64_t n_p2p_interactions = 0;
  fmm::M2LDmma m2l_dmma;
  fmm::M2L4 m2l4;
  int m2l_variant = 4;  // 1 = matrix-free O(p^4) per pair (v1), 2 = dense DMMA operator classes (v2),
                        // 3 = rotation-factored DMMA operator classes (v3, p <= 14; else v2),
                        // 4 = per-pair rotation on DFMA with a fixed constant-bank operator
                        //     (2 <= p <= 12; else v3)
  int near_variant = 2; // 1 = block per leaf, thread per target (v1), 2 = warp per leaf (v2)
  fmm::NearMutual mutual;  // v2 potentials-only, single GPU: symmetric leaf pairs once (FMM_NEAR_MUTUAL)

  // this rank's targets (Morton range of sorted positions) and its leaves
  int64_t own_begin = 0, own_end = 0;
  int64_t own_leaf_begin = 0, own_leaf_end = 0;  // range in `leaves`

  // expansions [ncells][nc] complex (m >= 0), normalised frame
  fmm::DevBuf<double2> M, L;
  // M2M / L2L operators A(+,+,+) in DMMA fragment order, [2][nmt][nks][32] (expansions.cu shift_setup)
  fmm::DevBuf<double> shift_ops;
  int shift_variant = 2;  // 1 = block per parent, thread per coefficient; 2 = DMMA (FMM_SHIFT_VARIANT)

  // device status word: bit 0 = non-finite charge seen
  fmm::DevBuf<int32_t> flags;
  fmm::DevBuf<double> host_stage_q, host_stage_phi, host_stage_grad;  // fmm_matvec_host buffers

  // multi-GPU LET exchange (let.cu)
  fmm::LetLists let;
  fmm::LetDev let_dev;
  fmm::LetHost let_host;
  std::vector<int64_t> let_level_lo, let_level_hi;  // per level: cells overlapping the owned range
  bool let_ready = false;
  // collective mode (world > 1 with fmm_exec.nccl_id): callers pass local slices, libfmm moves
  // the LET buffers with NCCL (comm.cu)
  void* nccl_comm = nullptr;  // ncclComm_t
  bool collective = false;
  int64_t n_local = 0;
  std::vector<int64_t> caller_counts;
  bool near_compact_out = false;  // near field writes owned results in Morton order (LET)
  // near field fused into the M2L v3 kernel (P2P by extra warps, then tail + L2P kernels)
  bool fuse_near = false;  // FMM_FUSE_NEAR=1: measured slower (profiles/r1_v3.md)
  fmm::DevBuf<double> near_p2p_phi, near_p2p_grad;  // P2P results in sorted order (unscaled)
  fmm::DevBuf<int> near_counter;                    // next own leaf to take
  bool near_fused_active = false, near_fused_grad = false;  // set for the current mat-vec
  // near field overlapped with the far field (P2P on a second stream, L2P after L2L)
  bool overlap_near = false;
  cudaStream_t stream2 = nullptr, stream3 = nullptr;  // far field (high priority), P2P (low)
  cudaEvent_t ev_q = nullptr, ev_up = nullptr, ev_p2p = nullptr, ev_far = nullptr;

  double t_setup[8] = {0};
  double t_matvec[8] = {0};
  cudaEvent_t ev[8] = {nullptr};

  int64_t bytes() const;
};

namespace fmm {
// records msg as fmm_last_error() and returns status (api.cu)
fmm_status set_error(int status, const std::string& msg);
// 2D log-kernel mat-vec stages (fmm2d.cu)
void expand_xy(const double* xy, int64_t n, double* xyz, cudaStream_t s);
void upward_2d(fmm_plan_s& P);
void m2l_2d(fmm_plan_s& P);
void downward_2d(fmm_plan_s& P);
void near_2d(fmm_plan_s& P, double* phi, double* grad);
// setup stages (tree.cu, traverse.cu)
void build_tree(fmm_plan_s& P, const double* xyz);
void traverse(fmm_plan_s& P);
// matvec stages (expansions.cu, near.cu)
void upward(fmm_plan_s& P);
void upward_own(fmm_plan_s& P);  // P2M of this rank's leaves only, then M2M (LET)
void m2l_pass(fmm_plan_s& P);
void m2l_dmma_setup(fmm_plan_s& P);
void m2l_dmma_pass(fmm_plan_s& P);
bool m2l_rot_supported(int p);
bool m2l_v4_supported(int p);
void m2l_v4_setup(fmm_plan_s& P);
void m2l_v4_pass(fmm_plan_s& P);
void m2l_rot_setup(fmm_plan_s& P);
size_t rot_smem_bytes(int p, int T, int smax);
int rot_chunk_width(int p);
void downward(fmm_plan_s& P);
void shift_setup(fmm_plan_s& P);  // M2M / L2L term tables
void near_pass(fmm_plan_s& P, const double* q_unused, double* phi, double* grad);
void near_pass_warp(fmm_plan_s& P, double* phi, double* grad);
void near_mutual_setup(fmm_plan_s& P);
void near_mutual_pass(fmm_plan_s& P, double* phi);
void helmholtz_setup(fmm_plan_s& P);
void helmholtz_matvec(fmm_plan_s& P, const double* q, double* phi);
void helmholtz_direct(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt, double kappa,
                      double* phi, cudaStream_t s);
void near_p2p_async(fmm_plan_s& P, bool grad, cudaStream_t stream);
void near_l2p_out(fmm_plan_s& P, double* phi, double* grad);
void near_fused_prepare(fmm_plan_s& P, bool grad);
void near_fused_finish(fmm_plan_s& P, double* phi, double* grad);
void gather_charges(fmm_plan_s& P, const double* q);
std::vector<int64_t> let_cuts(int64_t n, int world, int p, const int32_t* cbeg, const int32_t* cend, int64_t nleaves,
                              const int32_t* leaves, int64_t np2p, const int32_t* p2p_tgt, const int32_t* p2p_src,
                              int64_t nm2l, const int32_t* m2l_tgt);
void let_host_copy(fmm_plan_s& P);
void let_partition(fmm_plan_s& P);
void m2l_v4_resize(fmm_plan_s& P, int64_t npairs);
void downward_own(fmm_plan_s& P);
// NCCL (comm.cu)
void comm_unique_id(void* out);
void comm_init(fmm_plan_s& P, const void* id);
void comm_destroy(fmm_plan_s& P);
std::vector<int64_t> comm_gather_counts(fmm_plan_s& P, int64_t n_local);
void comm_gather_points(fmm_plan_s& P, const double* xyz_local, const std::vector<int64_t>& counts, DevBuf<double>& xyz);
void comm_exchange(fmm_plan_s& P, const double* send, const std::vector<int64_t>& scount, double* recv,
                   const std::vector<int64_t>& rcount, int width);
void comm_allgather(fmm_plan_s& P, const double* send, int64_t count, double* recv);
void let_lists(int64_t n, int world, int me, int p, const int64_t* caller_off, const uint32_t* perm, int64_t ncells,
               const int32_t* cbeg, const int32_t* cend, int64_t nleaves, const int32_t* leaves, int64_t np2p,
               const int32_t* p2p_tgt, const int32_t* p2p_src, int64_t nm2l, const int32_t* m2l_tgt,
               const int32_t* m2l_src, LetLists& out);
void let_setup(fmm_plan_s& P, const int64_t* caller_counts);
void let_pack_q(fmm_plan_s& P, const double* q_local, double* send);
void let_upward(fmm_plan_s& P, const double* q_recv, double* shared_send, double* m_send);
void let_exchange_in(fmm_plan_s& P, const double* shared_recv, const double* m_recv);
void let_pack_phi(fmm_plan_s& P, double* phi_send, double* grad_send);
void let_unpack(fmm_plan_s& P, const double* phi_recv, const double* grad_recv, double* phi, double* grad);
void launch_direct(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt,
                   double* phi, double* grad, cudaStream_t s);
}  // namespace fmm
