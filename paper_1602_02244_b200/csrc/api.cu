// api.cu — the C ABI of include/fmm.h: argument validation, plan lifecycle,
// stage orchestration on the caller's stream, error mapping. Every exported
// function catches all exceptions and returns an fmm_status (never aborts).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/fmm_helmholtz.h"
#include "plan.h"

namespace {

int ncoef_host(int p) { return (p + 1) * (p + 2) / 2; }

thread_local std::string g_last_error;

fmm_status fail(int status, const std::string& msg) {
  g_last_error = msg;
  return (fmm_status)status;
}

template <typename F>
fmm_status guarded(fmm_plan_s* P, F&& body) {
  try {
    body();
    return FMM_OK;
  } catch (const fmm::Error& e) {
    if (P && e.status != FMM_ERR_USAGE && e.status != FMM_ERR_NUMERIC) P->poisoned = true;
    return fail(e.status, e.what());
  } catch (const std::bad_alloc&) {
    if (P) P->poisoned = true;
    return fail(FMM_ERR_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    if (P) P->poisoned = true;
    return fail(FMM_ERR_CUDA, e.what());
  }
}

void usage(bool ok, const char* msg) {
  if (!ok) throw fmm::Error(FMM_ERR_USAGE, msg);
}
}  // namespace

namespace fmm {
fmm_status set_error(int status, const std::string& msg) { return fail(status, msg); }
}  // namespace fmm

namespace {

// leaves sorted by their first particle (Morton order of the particle ranges)
__global__ void leaf_keys_kernel(const int32_t* __restrict__ leaves, const int32_t* __restrict__ cbeg, int64_t nl,
                                 uint64_t* __restrict__ k, uint32_t* __restrict__ v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nl) {
    k[i] = (uint64_t)(uint32_t)cbeg[leaves[i]];
    v[i] = (uint32_t)leaves[i];
  }
}

__global__ void leaf_store_kernel(const uint32_t* __restrict__ v, int64_t nl, int32_t* __restrict__ leaves) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nl) leaves[i] = (int32_t)v[i];
}

void order_leaves_by_position(fmm_plan_s& P) {
  const int64_t nl = P.nleaves;
  if (nl <= 1) return;
  fmm::DevBuf<uint64_t> k;
  fmm::DevBuf<uint32_t> v;
  k.alloc(nl);
  v.alloc(nl);
  leaf_keys_kernel<<<fmm::cdiv(nl, 256), 256, 0, P.stream>>>(P.leaves, P.cells.begin, nl, k, v);
  FMM_LAUNCHED("leaf_keys_kernel");
  int bits = 1;
  while (((int64_t)1 << bits) < P.n) ++bits;
  fmm::radix_sort_pairs(k, v, nl, bits, P.stream);
  leaf_store_kernel<<<fmm::cdiv(nl, 256), 256, 0, P.stream>>>(v, nl, P.leaves);
  FMM_LAUNCHED("leaf_store_kernel");
}

// This rank's targets: a contiguous range of leaves in Morton order with about 1 / world of
// the estimated work (cut at leaf boundaries).
void choose_own_range(fmm_plan_s& P) {
  if (P.world == 1) {
    P.own_leaf_begin = 0;
    P.own_leaf_end = P.nleaves;
    P.own_begin = 0;
    P.own_end = P.n;
    return;
  }
  fmm::let_partition(P);  // cost-weighted cut at leaf boundaries (let.cu let_cuts)
}

struct Timer {
  fmm_plan_s& P;
  bool on;
  explicit Timer(fmm_plan_s& p, bool enable) : P(p), on(enable) {
    if (on && !P.ev[0])
      for (auto& e : P.ev) FMM_CUDA(cudaEventCreate(&e));
  }
  void mark(int i) {
    if (on) FMM_CUDA(cudaEventRecord(P.ev[i], P.stream));
  }
  float between(int a, int b) {
    float ms = 0;
    FMM_CUDA(cudaEventElapsedTime(&ms, P.ev[a], P.ev[b]));
    return ms;
  }
};

void run_matvec(fmm_plan_s& P, const double* q, double* phi, double* grad) {
  Timer T(P, P.timing);
  T.mark(0);
  fmm::gather_charges(P, q);
  if (P.dim == 2) {  // 2D log kernel (fmm2d.cu)
    fmm::upward_2d(P);
    T.mark(1);
    fmm::m2l_2d(P);
    T.mark(2);
    fmm::downward_2d(P);
    T.mark(3);
    fmm::near_2d(P, phi, grad);
    T.mark(4);
    if (T.on) {
      FMM_CUDA(cudaEventSynchronize(P.ev[4]));
      P.t_matvec[FMM_T_UPWARD] = T.between(0, 1);
      P.t_matvec[FMM_T_M2L] = T.between(1, 2);
      P.t_matvec[FMM_T_DOWNWARD] = T.between(2, 3);
      P.t_matvec[FMM_T_NEAR] = T.between(3, 4);
      P.t_matvec[FMM_T_MATVEC_TOTAL] = T.between(0, 4);
    }
    return;
  }
  if (P.overlap_near && P.near_variant == 2 && !P.fuse_near) {
    // near field overlapped with the far field: the P2P sums need only the
    // charges, the far field (M2L, L2L) only the multipoles. After the upward pass both are
    // released together, the far field on a high-priority stream (its persistent M2L CTAs are
    // placed first, one per SM) and the P2P on a low-priority one filling the SMs' remaining
    // room; L2P + rescale + scatter on the caller's stream once both are done.
    cudaStream_t sF = P.stream2, sN = P.stream3, s0 = P.stream;
    FMM_CUDA(cudaEventRecord(P.ev_q, s0));
    FMM_CUDA(cudaStreamWaitEvent(sF, P.ev_q, 0));
    P.stream = sF;  // the far-field stages enqueue on P.stream
    fmm::upward(P);
    FMM_CUDA(cudaEventRecord(P.ev_up, sF));
    FMM_CUDA(cudaStreamWaitEvent(sN, P.ev_up, 0));
    P.stream = sN;
    fmm::near_p2p_async(P, grad != nullptr, sN);
    FMM_CUDA(cudaEventRecord(P.ev_p2p, sN));
    P.stream = sF;
    if (T.on) FMM_CUDA(cudaEventRecord(P.ev[1], sF));
    if (P.m2l_variant == 4)
      fmm::m2l_v4_pass(P);
    else if (P.m2l_variant >= 2)
      fmm::m2l_dmma_pass(P);
    else
      fmm::m2l_pass(P);
    if (T.on) FMM_CUDA(cudaEventRecord(P.ev[2], sF));
    fmm::downward(P);
    FMM_CUDA(cudaEventRecord(P.ev_far, sF));
    P.stream = s0;
    FMM_CUDA(cudaStreamWaitEvent(s0, P.ev_far, 0));
    FMM_CUDA(cudaStreamWaitEvent(s0, P.ev_p2p, 0));
    T.mark(3);
    fmm::near_l2p_out(P, phi, grad);
    T.mark(4);
    if (T.on) {  // (M2L concurrent with the P2P; NEAR = the L2P tail; UPWARD = up to the M2L start)
      FMM_CUDA(cudaEventSynchronize(P.ev[4]));
      P.t_matvec[FMM_T_UPWARD] = T.between(0, 1);
      P.t_matvec[FMM_T_M2L] = T.between(1, 2);
      P.t_matvec[FMM_T_DOWNWARD] = T.between(2, 3);
      P.t_matvec[FMM_T_NEAR] = T.between(3, 4);
      P.t_matvec[FMM_T_MATVEC_TOTAL] = T.between(0, 4);
    }
    return;
  }
  fmm::upward(P);
  // near field fused into the M2L v3 kernel (P2P warps on the FP64 pipe)
  P.near_fused_active = P.fuse_near && P.m2l_variant == 3 && P.near_variant == 2 && P.m2l_dmma.ntiles > 0;
  P.near_fused_grad = grad != nullptr;
  if (P.near_fused_active) fmm::near_fused_prepare(P, grad != nullptr);
  T.mark(1);
  if (P.m2l_variant == 4)
    fmm::m2l_v4_pass(P);
  else if (P.m2l_variant >= 2)
    fmm::m2l_dmma_pass(P);
  else
    fmm::m2l_pass(P);
  T.mark(2);
  if (!P.debug_skip_l2l) fmm::downward(P);
  T.mark(3);
  if (P.world > 1) {
    FMM_CUDA(cudaMemsetAsync(phi, 0, sizeof(double) * P.n, P.stream));
    if (grad) FMM_CUDA(cudaMemsetAsync(grad, 0, sizeof(double) * 3 * P.n, P.stream));
  }
  if (P.near_fused_active)
    fmm::near_fused_finish(P, phi, grad);
  else if (P.near_variant == 2 && P.mutual.enabled && !grad)
    fmm::near_mutual_pass(P, phi);
  else if (P.near_variant == 2)
    fmm::near_pass_warp(P, phi, grad);
  else
    fmm::near_pass(P, q, phi, grad);
  P.near_fused_active = false;
  T.mark(4);
  if (T.on) {
    FMM_CUDA(cudaEventSynchronize(P.ev[4]));
    P.t_matvec[FMM_T_UPWARD] = T.between(0, 1);
    P.t_matvec[FMM_T_M2L] = T.between(1, 2);
    P.t_matvec[FMM_T_DOWNWARD] = T.between(2, 3);
    P.t_matvec[FMM_T_NEAR] = T.between(3, 4);
    P.t_matvec[FMM_T_MATVEC_TOTAL] = T.between(0, 4);
  }
}

void check_flags(fmm_plan_s& P) {
  int32_t f = 0;
  FMM_CUDA(cudaMemcpyAsync(&f, P.flags.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaStreamSynchronize(P.stream));
  if (f) {
    FMM_CUDA(cudaMemsetAsync(P.flags.ptr, 0, sizeof(int32_t), P.stream));
    throw fmm::Error(FMM_ERR_NUMERIC, "fmm_matvec: non-finite charge");
  }
}

// multi-GPU (LET) steps 4-5 on this rank: exchanged multipoles in, M2L of the targets overlapping
// the range, L2L, near field of own leaves, results packed for their callers
void let_finish_impl(fmm_plan_s& P, const double* shared_recv, const double* m_recv, double* phi_send,
                     double* grad_send) {
  Timer T(P, P.timing);
  T.mark(1);
  fmm::let_exchange_in(P, shared_recv, m_recv);
  P.near_fused_active = P.fuse_near && P.m2l_variant == 3 && P.near_variant == 2 && P.m2l_dmma.ntiles > 0;
  P.near_fused_grad = grad_send != nullptr;
  if (P.near_fused_active) fmm::near_fused_prepare(P, grad_send != nullptr);
  if (P.m2l_variant == 4)
    fmm::m2l_v4_pass(P);
  else if (P.m2l_variant >= 2)
    fmm::m2l_dmma_pass(P);
  else
    fmm::m2l_pass(P);
  T.mark(2);
  fmm::downward_own(P);
  T.mark(3);
  P.near_compact_out = true;
  if (P.near_fused_active)
    fmm::near_fused_finish(P, P.let_dev.phi_own.ptr, grad_send ? P.let_dev.grad_own.ptr : nullptr);
  else if (P.mutual.enabled && !grad_send)
    fmm::near_mutual_pass(P, P.let_dev.phi_own.ptr);
  else
    fmm::near_pass_warp(P, P.let_dev.phi_own.ptr, grad_send ? P.let_dev.grad_own.ptr : nullptr);
  P.near_compact_out = false;
  P.near_fused_active = false;
  fmm::let_pack_phi(P, phi_send, grad_send);
  T.mark(4);
  if (T.on) {
    FMM_CUDA(cudaEventSynchronize(P.ev[4]));
    P.t_matvec[FMM_T_M2L] = T.between(1, 2);
    P.t_matvec[FMM_T_DOWNWARD] = T.between(2, 3);
    P.t_matvec[FMM_T_NEAR] = T.between(3, 4);
  }
}

// collective mode (world > 1, fmm_exec.nccl_id): the whole LET protocol on the plan's stream,
// the buffers moved by NCCL (comm.cu); q / phi / grad are this rank's caller slices
void run_matvec_collective(fmm_plan_s& P, const double* q, double* phi, double* grad) {
  fmm::LetLists& L = P.let;
  fmm::LetDev& D = P.let_dev;
  const int ncd = 2 * P.nc;
  Timer T(P, P.timing);
  T.mark(0);
  fmm::let_pack_q(P, q, D.q_send.ptr);
  fmm::comm_exchange(P, D.q_send.ptr, L.q_send, D.q_recv.ptr, L.q_recv, 1);
  fmm::let_upward(P, D.q_recv.ptr, D.shared_send.ptr, D.m_send.ptr);
  fmm::comm_allgather(P, D.shared_send.ptr, (int64_t)L.shared.size() * ncd, D.shared_recv.ptr);
  fmm::comm_exchange(P, D.m_send.ptr, L.m_send, D.m_recv.ptr, L.m_recv, ncd);
  T.mark(1);
  const float t_up = T.on ? (FMM_CUDA(cudaEventSynchronize(P.ev[1])), T.between(0, 1)) : 0.f;
  let_finish_impl(P, D.shared_recv.ptr, D.m_recv.ptr, D.phi_send.ptr, grad ? D.grad_send.ptr : nullptr);
  T.mark(5);
  fmm::comm_exchange(P, D.phi_send.ptr, L.phi_send, D.phi_recv.ptr, L.phi_recv, 1);
  if (grad) fmm::comm_exchange(P, D.grad_send.ptr, L.phi_send, D.grad_recv.ptr, L.phi_recv, 3);
  fmm::let_unpack(P, D.phi_recv.ptr, grad ? D.grad_recv.ptr : nullptr, phi, grad);
  T.mark(6);
  if (T.on) {
    FMM_CUDA(cudaEventSynchronize(P.ev[6]));
    P.t_matvec[FMM_T_UPWARD] = t_up;  // q exchange + upward pass + multipole exchange
    P.t_matvec[FMM_T_MATVEC_TOTAL] = T.between(0, 6);
  }
}

void alloc_exchange_buffers(fmm_plan_s& P) {
  fmm::LetLists& L = P.let;
  fmm::LetDev& D = P.let_dev;
  auto sum = [](const std::vector<int64_t>& v) {
    int64_t s = 0;
    for (int64_t x : v) s += x;
    return std::max<int64_t>(1, s);
  };
  const int64_t ncd = 2 * P.nc, ns = (int64_t)L.shared.size();
  D.q_send.alloc(sum(L.q_send));
  D.q_recv.alloc(sum(L.q_recv));
  D.shared_send.alloc(std::max<int64_t>(1, ns * ncd));
  D.shared_recv.alloc(std::max<int64_t>(1, ns * ncd * P.world));
  D.m_send.alloc(sum(L.m_send) * ncd);
  D.m_recv.alloc(sum(L.m_recv) * ncd);
  D.phi_send.alloc(sum(L.phi_send));
  D.phi_recv.alloc(sum(L.phi_recv));
  D.grad_send.alloc(3 * sum(L.phi_send));
  D.grad_recv.alloc(3 * sum(L.phi_recv));
}

}  // namespace

int64_t fmm_plan_s::bytes() const {
  int64_t b = keys.bytes() + perm.bytes() + pos.bytes() + leaves.bytes() + M.bytes() + L.bytes() + flags.bytes();
  b += cells.level.bytes() + cells.begin.bytes() + cells.end.bytes() + cells.child.bytes() + cells.nchild.bytes() +
       cells.parent.bytes() + cells.anchor.bytes() + cells.center.bytes();
  b += p2p.tgt.bytes() + p2p.src.bytes() + p2p.off.bytes() + m2l.tgt.bytes() + m2l.src.bytes() + m2l.off.bytes();
  b += host_stage_q.bytes() + host_stage_phi.bytes() + host_stage_grad.bytes();
  b += m2l_dmma.bytes() + m2l4.bytes() + helm.bytes() + mutual.bytes();
  b += shift_ops.bytes();
  b += let_dev.bytes();
  return b;
}

extern "C" {

}  // extern "C"

namespace {
// streams, events and the NCCL communicator of a plan, then the plan (device buffers: DevBuf)
void release_plan(fmm_plan_s* P) {
  for (cudaStream_t st : {P->stream2, P->stream3})
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t e : {P->ev_q, P->ev_up, P->ev_p2p, P->ev_far})
    if (e) cudaEventDestroy(e);
  try {
    fmm::comm_destroy(*P);
  } catch (...) {
  }
  delete P;
}

fmm_status setup_impl(fmm_plan* out, const double* xyz, int64_t n, int p, int ncrit, double theta,
                      const fmm_exec* ex, int dim, double kappa = 0.0) {
  if (!out) return fail(FMM_ERR_USAGE, "fmm_setup: out is NULL");
  *out = nullptr;
  fmm_plan_s* P = nullptr;
  fmm_status st = guarded(nullptr, [&] {
    usage(ex != nullptr, "fmm_setup: ex is NULL");
    const bool collective = ex->nccl_id != nullptr;  // (world_size 1 too: a one-rank communicator)
    usage(xyz != nullptr || (collective && n == 0), "fmm_setup: xyz is NULL");
    usage(collective ? (n >= 0 && n < ((int64_t)1 << 31) - 1) : (n >= 1 && n < ((int64_t)1 << 31) - 1),
          "fmm_setup: n must be in [1, 2^31 - 2] (collective mode: this rank's slice, >= 0)");
    usage(p >= 0 && p <= fmm::kMaxP, "fmm_setup: p must be in [0, 16]");
    usage(ncrit >= 1, "fmm_setup: ncrit must be >= 1");
    usage(theta > 0.0 && theta * theta * 3.0 < 1.0, "fmm_setup: theta must be in (0, 1/sqrt(3))");
    usage(ex->world_size >= 1 && ex->rank >= 0 && ex->rank < ex->world_size, "fmm_setup: bad rank / world_size");
    FMM_CUDA(cudaSetDevice(ex->device));
    P = new fmm_plan_s();
    P->device = ex->device;
    P->stream = (cudaStream_t)ex->stream;
    P->rank = ex->rank;
    P->world = ex->world_size;
    P->n = n;
    P->p = p;
    P->ncrit = ncrit;
    P->nc = fmm::ncoef(p);
    P->theta = theta;
    P->theta2 = theta * theta;
    P->dim = dim;
    usage(dim == 3 || ex->world_size == 1, "fmm_setup_2d: single-GPU only");
    fmm::DevBuf<double> xyz_global;
    if (collective) {  // every rank's slice -> the global point set (NCCL, comm.cu)
      P->collective = true;
      P->n_local = n;
      fmm::comm_init(*P, ex->nccl_id);
      P->caller_counts = fmm::comm_gather_counts(*P, n);
      int64_t N = 0;
      for (int64_t c : P->caller_counts) N += c;
      usage(N >= 1 && N < ((int64_t)1 << 31) - 1, "fmm_setup: global n must be in [1, 2^31 - 2]");
      fmm::comm_gather_points(*P, xyz, P->caller_counts, xyz_global);
      xyz = xyz_global.ptr;
      P->n = N;
    }
    cudaEvent_t e0, e1, e2, e3;
    FMM_CUDA(cudaEventCreate(&e0));
    FMM_CUDA(cudaEventCreate(&e1));
    FMM_CUDA(cudaEventCreate(&e2));
    FMM_CUDA(cudaEventCreate(&e3));
    FMM_CUDA(cudaEventRecord(e0, P->stream));
    fmm::build_tree(*P, xyz);
    FMM_CUDA(cudaEventRecord(e1, P->stream));
    fmm::traverse(*P);
    FMM_CUDA(cudaEventRecord(e2, P->stream));
    order_leaves_by_position(*P);
    choose_own_range(*P);
    const char* v = getenv("FMM_M2L_VARIANT");
    if (v && v[0] >= '1' && v[0] <= '4') P->m2l_variant = v[0] - '0';
    if (P->m2l_variant == 4 && !fmm::m2l_v4_supported(p)) P->m2l_variant = 3;
    const char* nv = getenv("FMM_NEAR_VARIANT");
    if (nv && nv[0] == '1') P->near_variant = 1;
    const char* sv = getenv("FMM_SHIFT_VARIANT");
    if (sv && sv[0] == '1') P->shift_variant = 1;
#ifdef FMM_DEV  // development builds only (work-skipping / experimental paths)
    const char* fz = getenv("FMM_FUSE_NEAR");  // experiment: P2P warps inside the M2L v3 kernel (slower)
    P->fuse_near = fz && fz[0] == '1';
    const char* dbg = getenv("FMM_DEBUG_SKIP_L2L");  // export M2L-only local expansions
    P->debug_skip_l2l = dbg && dbg[0] == '1';
#endif
    const char* ov = getenv("FMM_OVERLAP_NEAR");
    P->overlap_near = dim == 3 && P->world == 1 && !collective && ov && ov[0] == '1';
    if (P->overlap_near) {
      int lo = 0, hi = 0;
      FMM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // (lo: least, hi: greatest priority)
      FMM_CUDA(cudaStreamCreateWithPriority(&P->stream2, cudaStreamNonBlocking, hi));
      FMM_CUDA(cudaStreamCreateWithPriority(&P->stream3, cudaStreamNonBlocking, lo));
      for (cudaEvent_t* e : {&P->ev_q, &P->ev_up, &P->ev_p2p, &P->ev_far})
        FMM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    if (kappa > 0.0) {  // Helmholtz (NEXT-4): its own level / class tables (helmholtz.cu)
      usage(P->world == 1 && !collective, "fmm_setup_helmholtz: single GPU only");
      P->helmholtz = true;
      P->kappa = kappa;
      P->m2l_variant = 5;
      fmm::helmholtz_setup(*P);
    } else if (dim == 3) {  // 3D translation operators (the 2D kernels are matrix-free)
      if (P->m2l_variant == 4)
        fmm::m2l_v4_setup(*P);
      else if (P->m2l_variant >= 2)
        fmm::m2l_dmma_setup(*P);
      fmm::shift_setup(*P);
      const char* mu = getenv("FMM_NEAR_MUTUAL");  // 0: directed P2P for potentials too
      if (P->near_variant == 2 && !(mu && mu[0] == '0'))  // (world > 1: mutual among this rank's leaves)
        fmm::near_mutual_setup(*P);
    }
    P->M.alloc(P->cells.n * P->nc);
    if (collective) {  // exchange lists and buffers of this rank (let.cu)
      fmm::let_setup(*P, P->caller_counts.data());
      alloc_exchange_buffers(*P);
    }
    P->L.alloc(P->cells.n * P->nc);
    const char* poison = getenv("FMM_DEBUG_POISON");  // test hook: NaN-fill expansions so unwritten
    if (poison && poison[0] == '1') {                 // coefficients surface in the results
      FMM_CUDA(cudaMemsetAsync(P->M.ptr, 0xff, P->M.bytes(), P->stream));
      FMM_CUDA(cudaMemsetAsync(P->L.ptr, 0xff, P->L.bytes(), P->stream));
    }
    FMM_CUDA(cudaEventRecord(e3, P->stream));
    FMM_CUDA(cudaEventSynchronize(e3));
    float a = 0, b = 0, c = 0;
    FMM_CUDA(cudaEventElapsedTime(&a, e0, e1));
    FMM_CUDA(cudaEventElapsedTime(&b, e1, e2));
    FMM_CUDA(cudaEventElapsedTime(&c, e0, e3));
    P->t_setup[FMM_T_TREE] = a;
    P->t_setup[FMM_T_TRAVERSE] = b;
    P->t_setup[FMM_T_SETUP_TOTAL] = c;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaEventDestroy(e3);
  });
  if (st != FMM_OK) {
    if (P) release_plan(P);
    return st;
  }
  *out = P;
  return FMM_OK;
}
}  // namespace

extern "C" {

fmm_status fmm_setup(fmm_plan* out, const double* xyz, int64_t n, int p, int ncrit, double theta,
                     const fmm_exec* ex) {
  return setup_impl(out, xyz, n, p, ncrit, theta, ex, 3);
}

fmm_status fmm_setup_2d(fmm_plan* out, const double* xy, int64_t n, int p, int ncrit, double theta,
                        const fmm_exec* ex) {
  if (!out) return fail(FMM_ERR_USAGE, "fmm_setup_2d: out is NULL");
  *out = nullptr;
  fmm::DevBuf<double> xyz;
  const fmm_status st = guarded(nullptr, [&] {
    usage(ex != nullptr && xy != nullptr, "fmm_setup_2d: ex / xy is NULL");
    usage(n >= 1 && n < ((int64_t)1 << 31) - 1, "fmm_setup_2d: n must be in [1, 2^31 - 2]");
    FMM_CUDA(cudaSetDevice(ex->device));
    xyz.alloc(3 * n);
    fmm::expand_xy(xy, n, xyz, (cudaStream_t)ex->stream);
  });
  if (st != FMM_OK) return st;
  return setup_impl(out, xyz, n, p, ncrit, theta, ex, 2);
}

fmm_status fmm_setup_helmholtz(fmm_plan* out, const double* xyz, int64_t n, int p, int ncrit, double theta,
                               double kappa, const fmm_exec* ex) {
  if (!out) return fail(FMM_ERR_USAGE, "fmm_setup_helmholtz: out is NULL");
  *out = nullptr;
  if (!(kappa > 0.0) || !std::isfinite(kappa)) return fail(FMM_ERR_USAGE, "fmm_setup_helmholtz: kappa must be > 0");
  if (p < 0 || p > 10) return fail(FMM_ERR_USAGE, "fmm_setup_helmholtz: p must be in [0, 10]");
  if (ex && (ex->world_size != 1 || ex->nccl_id)) return fail(FMM_ERR_USAGE, "fmm_setup_helmholtz: single GPU only");
  return setup_impl(out, xyz, n, p, ncrit, theta, ex, 3, kappa);
}

fmm_status fmm_matvec_helmholtz(fmm_plan P, const double* q, int64_t n, double* phi) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_matvec_helmholtz: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_matvec_helmholtz: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    usage(P->helmholtz, "fmm_matvec_helmholtz: not a Helmholtz plan (fmm_setup_helmholtz)");
    usage(n == P->n, "fmm_matvec_helmholtz: n differs from the setup n");
    usage(q != nullptr && phi != nullptr, "fmm_matvec_helmholtz: q / phi is NULL");
    FMM_CUDA(cudaSetDevice(P->device));
    Timer T(*P, P->timing);
    T.mark(0);
    fmm::helmholtz_matvec(*P, q, phi);
    T.mark(4);
    if (T.on) {
      FMM_CUDA(cudaEventSynchronize(P->ev[4]));
      P->t_matvec[FMM_T_MATVEC_TOTAL] = T.between(0, 4);
    }
  });
}

fmm_status fmm_direct_helmholtz(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt,
                                double kappa, double* phi, const fmm_exec* ex) {
  return guarded(nullptr, [&] {
    usage(ex != nullptr, "fmm_direct_helmholtz: ex is NULL");
    usage(ns >= 0 && nt >= 0, "fmm_direct_helmholtz: negative size");
    usage(ns == 0 || (src && q), "fmm_direct_helmholtz: src / q is NULL");
    usage(nt == 0 || (tgt && phi), "fmm_direct_helmholtz: tgt / phi is NULL");
    usage(std::isfinite(kappa), "fmm_direct_helmholtz: kappa must be finite");
    FMM_CUDA(cudaSetDevice(ex->device));
    fmm::helmholtz_direct(src, q, ns, tgt, nt, kappa, phi, (cudaStream_t)ex->stream);
  });
}

fmm_status fmm_matvec(fmm_plan P, const double* q, int64_t n, double* phi, double* grad) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_matvec: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_matvec: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    usage(!P->helmholtz, "fmm_matvec: a Helmholtz plan takes fmm_matvec_helmholtz");
    if (P->collective) {  // this rank's caller slice in and out; collective over the world
      usage(n == P->n_local, "fmm_matvec: n differs from this rank's setup slice");
      usage(n == 0 || (q != nullptr && phi != nullptr), "fmm_matvec: q / phi is NULL");
      FMM_CUDA(cudaSetDevice(P->device));
      run_matvec_collective(*P, q, phi, grad);
      return;
    }
    usage(n == P->n, "fmm_matvec: n differs from the setup n");
    usage(q != nullptr && phi != nullptr, "fmm_matvec: q / phi is NULL");
    FMM_CUDA(cudaSetDevice(P->device));
    run_matvec(*P, q, phi, grad);
  });
}

fmm_status fmm_matvec_host(fmm_plan P, const double* q_host, int64_t n, double* phi_host, double* grad_host) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_matvec_host: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_matvec_host: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    usage(!P->helmholtz, "fmm_matvec_host: a Helmholtz plan takes fmm_matvec_helmholtz");
    const int64_t nn = P->collective ? P->n_local : P->n;
    usage(n == nn, "fmm_matvec_host: n differs from the setup n (collective mode: this rank's slice)");
    usage(n == 0 || (q_host != nullptr && phi_host != nullptr), "fmm_matvec_host: q / phi is NULL");
    FMM_CUDA(cudaSetDevice(P->device));
    if (P->host_stage_q.count < std::max<int64_t>(n, 1)) P->host_stage_q.alloc(std::max<int64_t>(n, 1));
    if (P->host_stage_phi.count < std::max<int64_t>(n, 1)) P->host_stage_phi.alloc(std::max<int64_t>(n, 1));
    if (grad_host && P->host_stage_grad.count < 3 * n) P->host_stage_grad.alloc(3 * n);
    if (n > 0)
      FMM_CUDA(cudaMemcpyAsync(P->host_stage_q.ptr, q_host, sizeof(double) * n, cudaMemcpyHostToDevice, P->stream));
    double* dg = grad_host ? P->host_stage_grad.ptr : nullptr;
    if (P->collective)
      run_matvec_collective(*P, P->host_stage_q.ptr, P->host_stage_phi.ptr, dg);
    else
      run_matvec(*P, P->host_stage_q.ptr, P->host_stage_phi.ptr, dg);
    if (n > 0)
      FMM_CUDA(cudaMemcpyAsync(phi_host, P->host_stage_phi.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost,
                               P->stream));
    if (grad_host && n > 0)
      FMM_CUDA(cudaMemcpyAsync(grad_host, dg, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, P->stream));
    check_flags(*P);
  });
}

fmm_status fmm_sync(fmm_plan P) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_sync: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_sync: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    FMM_CUDA(cudaSetDevice(P->device));
    FMM_CUDA(cudaGetLastError());
    check_flags(*P);
  });
}

fmm_status fmm_direct(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt, double* phi,
                      double* grad, const fmm_exec* ex) {
  return guarded(nullptr, [&] {
    usage(ex != nullptr, "fmm_direct: ex is NULL");
    usage(ns >= 0 && nt >= 0, "fmm_direct: negative size");
    usage(ns == 0 || (src && q), "fmm_direct: src / q is NULL");
    usage(nt == 0 || (tgt && phi), "fmm_direct: tgt / phi is NULL");
    FMM_CUDA(cudaSetDevice(ex->device));
    fmm::launch_direct(src, q, ns, tgt, nt, phi, grad, (cudaStream_t)ex->stream);
  });
}

fmm_status fmm_stats(fmm_plan P, fmm_stats_t* out) {
  if (!P || !out) return fail(FMM_ERR_USAGE, "fmm_stats: NULL argument");
  std::memset(out, 0, sizeof(*out));
  out->n = P->n;
  out->n_cells = P->cells.n;
  out->n_leaves = P->nleaves;
  out->n_p2p_pairs = P->p2p.n;
  out->n_m2l_pairs = P->m2l.n;
  out->n_p2p_interactions = P->n_p2p_interactions;
  out->own_begin = P->own_begin;
  out->own_end = P->own_end;
  out->p = P->p;
  out->ncrit = P->ncrit;
  out->max_level = P->max_level;
  out->exponent = P->e;
  out->theta = P->theta;
  for (int i = 0; i < 8; ++i) {
    out->t_setup_ms[i] = P->t_setup[i];
    out->t_matvec_ms[i] = P->t_matvec[i];
  }
  out->bytes_device = P->bytes();
  out->launches_total = fmm::launch_counter().load();
  {
    const fmm::M2LDmma& D = P->m2l_dmma;
    const fmm::Cells& c = P->cells;
    int64_t* b = out->bytes_by;
    for (int k = 0; k < 8; ++k) b[k] = 0;
    b[FMM_B_PARTICLES] = P->keys.bytes() + P->perm.bytes() + P->pos.bytes() + P->helm.qs.bytes() + P->host_stage_q.bytes() +
                         P->host_stage_phi.bytes() + P->host_stage_grad.bytes() + P->mutual.partial.bytes() +
                         P->mutual.own.bytes();
    b[FMM_B_TREE] = c.level.bytes() + c.begin.bytes() + c.end.bytes() + c.child.bytes() + c.nchild.bytes() +
                    c.parent.bytes() + c.anchor.bytes() + c.center.bytes() + P->leaves.bytes() + P->m2l4.ihalf.bytes();
    b[FMM_B_LISTS] = P->p2p.tgt.bytes() + P->p2p.src.bytes() + P->p2p.off.bytes() + P->m2l.tgt.bytes() +
                     P->m2l.src.bytes() + P->m2l.off.bytes() + P->mutual.toff.bytes() + P->mutual.tmend.bytes() + P->mutual.task_b.bytes() +
                     P->mutual.poff.bytes() + P->mutual.goff.bytes() + P->mutual.gslot.bytes();
    b[FMM_B_EXPANSIONS] = P->M.bytes() + P->L.bytes() + D.Mt.bytes() + P->m2l4.Mt.bytes() + P->helm.M.bytes() +
                          P->helm.L.bytes();
    b[FMM_B_OPERATORS] = D.ops.bytes() + D.rot_ops.bytes() + D.hpow.bytes() + D.symtab.bytes() +
                         D.rot_masks.bytes() + D.class_keys.bytes() + P->shift_ops.bytes() + P->helm.shift_ops.bytes() +
                         P->helm.m2l_ops.bytes();
    b[FMM_B_SCHEDULE] = D.col_src.bytes() + D.col_meta.bytes() + D.chunk_begin.bytes() + D.chunk_class.bytes() +
                        D.tile_chunk.bytes() + D.tile_cells.bytes() + D.chunk_seg.bytes() + D.seg_begin.bytes() +
                        D.rot_sched.bytes() + D.rot_ihdr.bytes() + D.rot_ipos.bytes() + D.rot_desc.bytes() +
                        D.rot_order.bytes() + D.rot_scratch.bytes() + P->m2l4.part.bytes() + P->helm.m2l_class.bytes();
    b[FMM_B_LET] = P->let_dev.bytes();
    int64_t s = 0;
    for (int k = 0; k < 7; ++k) s += b[k];
    b[FMM_B_OTHER] = out->bytes_device - s;
  }
  out->m2l_variant = P->m2l_variant;
  out->near_mutual = P->mutual.enabled ? 1 : 0;
  {
    const double p1 = P->p + 1;
    if (P->helmholtz) {  // dense complex (S|R) class operator: 8 flop per complex MAC
      out->m2l_flops_per_pair = 8.0 * p1 * p1 * p1 * p1;
    } else if (P->dim == 2) {  // 2D log kernel: one complex multiply-add per (l, k) pair
      out->m2l_variant = 0;
      out->m2l_flops_per_pair = 8.0 * p1 * p1;
    } else if (P->m2l_variant == 4) {  // per degree 2 (n^2+n+1) fixed-operator MACs + 2 zrot (4 n), twice;
      double f = 0, z = 0;              // per order the Hankel (p+1-m)^2 (Re) + (Im, m > 0)
      for (int n = 0; n <= P->p; ++n) f += 2.0 * (2.0 * (n * n + n + 1) + 4.0 * n);
      for (int m = 0; m <= P->p; ++m) z += (m ? 2.0 : 1.0) * (p1 - m) * (p1 - m);
      out->m2l_flops_per_pair = 2.0 * (f + z);
    } else if (P->m2l_variant == 3) {  // sum_n (n+1)^2 + n^2 per rotation stage, sum_m (p+1-m)^2 (Re) + (Im, m > 0)
      double rot = 0, z = 0;
      for (int n = 0; n <= P->p; ++n) rot += (n + 1.0) * (n + 1.0) + (double)n * n;
      for (int m = 0; m <= P->p; ++m) z += (m ? 2.0 : 1.0) * (p1 - m) * (p1 - m);
      const double az = 2.0 * 6.0 * (ncoef_host(P->p) - p1);  // two 2x2 rotations per (n, m >= 1) pair
      out->m2l_flops_per_pair = 2.0 * (2.0 * rot + z) + az;
    } else {
      out->m2l_flops_per_pair = 2.0 * p1 * p1 * p1 * p1;
    }
  }
  return FMM_OK;
}

fmm_status fmm_set_timing(fmm_plan P, int enable) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_set_timing: plan is NULL");
  P->timing = enable != 0;
  return FMM_OK;
}

fmm_status fmm_export(fmm_plan P, int what, void* dst, int64_t capacity, int64_t* count) {
  if (!P || !count) return fail(FMM_ERR_USAGE, "fmm_export: NULL argument");
  return guarded(P, [&] {
    const void* src = nullptr;
    int64_t cnt = 0, esz = 0;
    std::vector<double> geom;
    const int64_t nc = P->cells.n;
    switch (what) {
      case FMM_X_KEYS: src = P->keys.ptr; cnt = P->n; esz = 8; break;
      case FMM_X_PERM: src = P->perm.ptr; cnt = P->n; esz = 4; break;
      case FMM_X_LEVEL: src = P->cells.level.ptr; cnt = nc; esz = 4; break;
      case FMM_X_ANCHOR: src = P->cells.anchor.ptr; cnt = 3 * nc; esz = 4; break;
      case FMM_X_BEGIN: src = P->cells.begin.ptr; cnt = nc; esz = 4; break;
      case FMM_X_END: src = P->cells.end.ptr; cnt = nc; esz = 4; break;
      case FMM_X_CHILD: src = P->cells.child.ptr; cnt = nc; esz = 4; break;
      case FMM_X_NCHILD: src = P->cells.nchild.ptr; cnt = nc; esz = 4; break;
      case FMM_X_PARENT: src = P->cells.parent.ptr; cnt = nc; esz = 4; break;
      case FMM_X_CENTER: src = nullptr; cnt = 3 * nc; esz = 8; break;
      case FMM_X_P2P: src = nullptr; cnt = 2 * P->p2p.n; esz = 4; break;
      case FMM_X_M2L: src = nullptr; cnt = 2 * P->m2l.n; esz = 4; break;
      case FMM_X_M: src = P->M.ptr; cnt = 2 * nc * P->nc; esz = 8; break;
      case FMM_X_L: src = P->L.ptr; cnt = 2 * nc * P->nc; esz = 8; break;
      case FMM_X_GEOM:
        geom = {P->lo[0], P->lo[1], P->lo[2], P->S, P->scale};
        cnt = 5;
        esz = 8;
        break;
      default: usage(false, "fmm_export: unknown array");
    }
    *count = cnt;
    if (!dst) return;
    usage(capacity >= cnt, "fmm_export: capacity too small");
    FMM_CUDA(cudaSetDevice(P->device));
    FMM_CUDA(cudaStreamSynchronize(P->stream));
    if (what == FMM_X_GEOM) {
      std::memcpy(dst, geom.data(), sizeof(double) * 5);
    } else if (what == FMM_X_CENTER) {
      std::vector<double4> c(nc);
      FMM_CUDA(cudaMemcpy(c.data(), P->cells.center.ptr, sizeof(double4) * nc, cudaMemcpyDeviceToHost));
      double* d = (double*)dst;
      for (int64_t i = 0; i < nc; ++i) {
        d[3 * i] = c[i].x;
        d[3 * i + 1] = c[i].y;
        d[3 * i + 2] = c[i].z;
      }
    } else if (what == FMM_X_P2P || what == FMM_X_M2L) {
      const fmm::PairList& L = what == FMM_X_P2P ? P->p2p : P->m2l;
      std::vector<int32_t> t(L.n), s(L.n);
      if (L.n) {
        FMM_CUDA(cudaMemcpy(t.data(), L.tgt.ptr, sizeof(int32_t) * L.n, cudaMemcpyDeviceToHost));
        FMM_CUDA(cudaMemcpy(s.data(), L.src.ptr, sizeof(int32_t) * L.n, cudaMemcpyDeviceToHost));
      }
      int32_t* d = (int32_t*)dst;
      for (int64_t i = 0; i < L.n; ++i) {
        d[2 * i] = t[i];
        d[2 * i + 1] = s[i];
      }
    } else if (cnt > 0) {
      FMM_CUDA(cudaMemcpy(dst, src, esz * cnt, cudaMemcpyDeviceToHost));
    }
  });
}

fmm_status fmm_let_setup(fmm_plan P, const int64_t* caller_counts) {
  if (!P || !caller_counts) return fail(FMM_ERR_USAGE, "fmm_let_setup: NULL argument");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_let_setup: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    usage(P->world > 1, "fmm_let_setup: world_size must be > 1");
    usage(!P->collective, "fmm_let_setup: a collective (nccl_id) plan runs the exchange itself");
    FMM_CUDA(cudaSetDevice(P->device));
    fmm::let_setup(*P, caller_counts);
  });
}

namespace {
const std::vector<int64_t>* let_vec(const fmm::LetLists& L, int what) {
  switch (what) {
    case FMM_LET_Q_SEND: return &L.q_send;
    case FMM_LET_Q_RECV: return &L.q_recv;
    case FMM_LET_M_SEND: return &L.m_send;
    case FMM_LET_M_RECV: return &L.m_recv;
    case FMM_LET_PHI_SEND: return &L.phi_send;
    case FMM_LET_PHI_RECV: return &L.phi_recv;
    case FMM_LET_RANK_BEGIN: return &L.rank_begin;
    case FMM_LET_Q_SEND_ROWS: return &L.q_send_rows;
    case FMM_LET_Q_RECV_POS: return &L.q_recv_pos;
    case FMM_LET_PHI_SEND_IDX: return &L.phi_send_idx;
    case FMM_LET_PHI_RECV_ROWS: return &L.phi_recv_rows;
    default: return nullptr;
  }
}
void let_require(fmm_plan_s* P) { usage(P->let_ready, "fmm_let_*: call fmm_let_setup first"); }
}  // namespace

fmm_status fmm_let_counts(fmm_plan P, int what, int64_t* out) {
  if (!P || !out) return fail(FMM_ERR_USAGE, "fmm_let_counts: NULL argument");
  return guarded(P, [&] {
    let_require(P);
    if (what == FMM_LET_SHARED) {
      out[0] = (int64_t)P->let.shared.size();
      return;
    }
    usage(what >= FMM_LET_Q_SEND && what <= FMM_LET_RANK_BEGIN, "fmm_let_counts: unknown what");
    const std::vector<int64_t>* v = let_vec(P->let, what);
    std::copy(v->begin(), v->end(), out);
  });
}

fmm_status fmm_let_pack_q(fmm_plan P, const double* q_local, double* q_send) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_let_pack_q: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_let_pack_q: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    let_require(P);
    usage(P->let.q_send_rows.empty() || (q_local && q_send), "fmm_let_pack_q: NULL buffer");
    FMM_CUDA(cudaSetDevice(P->device));
    fmm::let_pack_q(*P, q_local, q_send);
  });
}

fmm_status fmm_let_upward(fmm_plan P, const double* q_recv, double* shared_send, double* m_send) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_let_upward: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_let_upward: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    let_require(P);
    usage((P->let.q_recv_pos.empty() || q_recv) && (P->let.shared.empty() || shared_send) &&
              (P->let.m_send_cells.empty() || m_send),
          "fmm_let_upward: NULL buffer");
    FMM_CUDA(cudaSetDevice(P->device));
    Timer T(*P, P->timing);
    T.mark(0);
    fmm::let_upward(*P, q_recv, shared_send, m_send);
    T.mark(1);
    if (T.on) {
      FMM_CUDA(cudaEventSynchronize(P->ev[1]));
      P->t_matvec[FMM_T_UPWARD] = T.between(0, 1);
    }
  });
}

fmm_status fmm_let_finish(fmm_plan P, const double* shared_recv, const double* m_recv, double* phi_send,
                          double* grad_send) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_let_finish: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_let_finish: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    let_require(P);
    usage((P->let.shared.empty() || shared_recv) && (P->let.m_recv_cells.empty() || m_recv) &&
              (P->let.phi_send_idx.empty() || phi_send),
          "fmm_let_finish: NULL buffer");
    FMM_CUDA(cudaSetDevice(P->device));
    let_finish_impl(*P, shared_recv, m_recv, phi_send, grad_send);
  });
}

fmm_status fmm_let_unpack(fmm_plan P, const double* phi_recv, const double* grad_recv, double* phi_local,
                          double* grad_local) {
  if (!P) return fail(FMM_ERR_USAGE, "fmm_let_unpack: plan is NULL");
  if (P->poisoned) return fail(FMM_ERR_USAGE, "fmm_let_unpack: plan is poisoned by an earlier error");
  return guarded(P, [&] {
    let_require(P);
    usage(P->let.phi_recv_rows.empty() || (phi_recv && phi_local), "fmm_let_unpack: NULL buffer");
    FMM_CUDA(cudaSetDevice(P->device));
    fmm::let_unpack(*P, phi_recv, grad_recv, phi_local, grad_local);
  });
}

fmm_status fmm_let_lists_host(int64_t n, int world, int me, int p, const int64_t* caller_off, const uint32_t* perm,
                              int64_t ncells, const int32_t* cbeg, const int32_t* cend, int64_t nleaves,
                              const int32_t* leaves, int64_t np2p, const int32_t* p2p_tgt, const int32_t* p2p_src,
                              int64_t nm2l, const int32_t* m2l_tgt, const int32_t* m2l_src, int what, int64_t* dst,
                              int64_t capacity, int64_t* count) {
  return guarded(nullptr, [&] {
    usage(count != nullptr && world >= 1 && me >= 0 && me < world && n >= 1 && p >= 0 && p <= fmm::kMaxP,
          "fmm_let_lists_host: bad arguments");
    usage(caller_off && perm && cbeg && cend && leaves, "fmm_let_lists_host: NULL array");
    fmm::LetLists L;
    fmm::let_lists(n, world, me, p, caller_off, perm, ncells, cbeg, cend, nleaves, leaves, np2p, p2p_tgt, p2p_src, nm2l,
                   m2l_tgt, m2l_src, L);
    std::vector<int64_t> tmp;
    const std::vector<int64_t>* v = let_vec(L, what);
    if (what == FMM_LET_SHARED) {
      tmp = {(int64_t)L.shared.size()};
      v = &tmp;
    } else if (what == FMM_LET_SHARED_CELLS || what == FMM_LET_M_SEND_CELLS || what == FMM_LET_M_RECV_CELLS) {
      const std::vector<int32_t>& c = what == FMM_LET_SHARED_CELLS ? L.shared
                                     : what == FMM_LET_M_SEND_CELLS ? L.m_send_cells
                                                                    : L.m_recv_cells;
      tmp.assign(c.begin(), c.end());
      v = &tmp;
    }
    usage(v != nullptr, "fmm_let_lists_host: unknown what");
    *count = (int64_t)v->size();
    if (!dst) return;
    usage(capacity >= *count, "fmm_let_lists_host: capacity too small");
    std::copy(v->begin(), v->end(), dst);
  });
}

void fmm_destroy(fmm_plan P) {
  if (!P) return;
  cudaSetDevice(P->device);
  cudaStreamSynchronize(P->stream);
  for (auto& e : P->ev)
    if (e) cudaEventDestroy(e);
  release_plan(P);
}

const char* fmm_last_error(void) { return g_last_error.c_str(); }

const char* fmm_version(void) { return "fmm-b200 0.1 (sm_100a, fp64)"; }

}  // extern "C"
