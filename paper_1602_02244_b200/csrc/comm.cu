// comm.cu — NCCL inside libfmm for the multi-GPU mat-vec (S14; north_star: "a local-essential-
// tree exchange (boundary multipoles plus halo particles) over NCCL/NVLink").
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): a single-GPU user never needs it, and in a
// process that already holds NCCL (PyTorch's) the loader returns that same library. The caller
// passes a 128-byte ncclUniqueId in fmm_exec.nccl_id (rank 0 makes it with fmm_nccl_unique_id and
// broadcasts it by any means — the Python layer uses its torch.distributed group); every
// collective below is enqueued on the plan's stream.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"

namespace fmm {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f && a.error.empty()) a.error = std::string("libnccl lacks ") + n;
      return f;
    };
    a.getUniqueId = (decltype(a.getUniqueId))sym("ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))sym("ncclCommInitRank");
    a.commDestroy = (decltype(a.commDestroy))sym("ncclCommDestroy");
    a.allGather = (decltype(a.allGather))sym("ncclAllGather");
    a.send = (decltype(a.send))sym("ncclSend");
    a.recv = (decltype(a.recv))sym("ncclRecv");
    a.groupStart = (decltype(a.groupStart))sym("ncclGroupStart");
    a.groupEnd = (decltype(a.groupEnd))sym("ncclGroupEnd");
    a.errorString = (decltype(a.errorString))sym("ncclGetErrorString");
  });
  if (!a.error.empty()) throw Error(FMM_ERR_COMM, a.error);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(FMM_ERR_COMM, std::string(what) + ": " + (api().errorString ? api().errorString(r) : "NCCL error"));
}

__global__ void pack_points_kernel(const double* __restrict__ recv, const int64_t* __restrict__ off, int world,
                                   int64_t maxc, double* __restrict__ xyz) {
  // recv: [world][maxc][3] (rank r's rows first); xyz: [N][3] in rank order
  const int64_t N = off[world];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / 3;
    int r = 0;
    while (off[r + 1] <= row) ++r;
    xyz[i] = recv[(r * maxc + (row - off[r])) * 3 + (i - row * 3)];
  }
}

}  // namespace

void comm_unique_id(void* out) {
  ncclUniqueId id;
  check(api().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void comm_init(fmm_plan_s& P, const void* id) {
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  check(api().commInitRank(&c, P.world, uid, P.rank), "ncclCommInitRank");
  P.nccl_comm = c;
}

void comm_destroy(fmm_plan_s& P) {
  if (P.nccl_comm) api().commDestroy((ncclComm_t)P.nccl_comm);
  P.nccl_comm = nullptr;
}

// every rank's local count, in rank order (synchronises: the sizes shape the setup)
std::vector<int64_t> comm_gather_counts(fmm_plan_s& P, int64_t n_local) {
  DevBuf<int64_t> d;
  d.alloc(P.world + 1);
  FMM_CUDA(cudaMemcpyAsync(d.ptr + P.world, &n_local, sizeof(int64_t), cudaMemcpyHostToDevice, P.stream));
  check(api().allGather(d.ptr + P.world, d.ptr, 1, ncclInt64, (ncclComm_t)P.nccl_comm, P.stream), "ncclAllGather");
  std::vector<int64_t> h(P.world);
  FMM_CUDA(cudaMemcpyAsync(h.data(), d.ptr, sizeof(int64_t) * P.world, cudaMemcpyDeviceToHost, P.stream));
  FMM_CUDA(cudaStreamSynchronize(P.stream));
  return h;
}

// the global point set [N][3] (rank order) from every rank's slice
void comm_gather_points(fmm_plan_s& P, const double* xyz_local, const std::vector<int64_t>& counts,
                        DevBuf<double>& xyz) {
  int64_t maxc = 1, N = 0;
  std::vector<int64_t> off(P.world + 1, 0);
  for (int r = 0; r < P.world; ++r) {
    maxc = std::max(maxc, counts[r]);
    off[r + 1] = off[r] + counts[r];
  }
  N = off[P.world];
  DevBuf<double> send, recv;
  DevBuf<int64_t> doff;
  send.alloc(3 * maxc);
  recv.alloc(3 * maxc * P.world);
  doff.alloc(P.world + 1);
  FMM_CUDA(cudaMemsetAsync(send.ptr, 0, sizeof(double) * 3 * maxc, P.stream));
  if (counts[P.rank] > 0)
    FMM_CUDA(cudaMemcpyAsync(send.ptr, xyz_local, sizeof(double) * 3 * counts[P.rank], cudaMemcpyDeviceToDevice,
                             P.stream));
  check(api().allGather(send.ptr, recv.ptr, 3 * maxc, ncclDouble, (ncclComm_t)P.nccl_comm, P.stream),
        "ncclAllGather");
  FMM_CUDA(cudaMemcpyAsync(doff.ptr, off.data(), sizeof(int64_t) * (P.world + 1), cudaMemcpyHostToDevice, P.stream));
  xyz.alloc(3 * N);
  pack_points_kernel<<<cdiv(3 * N, 256 * 8), 256, 0, P.stream>>>(recv.ptr, doff.ptr, P.world, maxc, xyz.ptr);
  FMM_LAUNCHED("pack_points_kernel");
  FMM_CUDA(cudaStreamSynchronize(P.stream));
}

// uneven all-to-all of rows of `width` doubles: grouped point-to-point (the LET's irregular
// pattern), the self part as a device copy
void comm_exchange(fmm_plan_s& P, const double* send, const std::vector<int64_t>& scount, double* recv,
                   const std::vector<int64_t>& rcount, int width) {
  const NcclApi& a = api();
  std::vector<int64_t> so(P.world + 1, 0), ro(P.world + 1, 0);
  for (int r = 0; r < P.world; ++r) {
    so[r + 1] = so[r] + scount[r] * width;
    ro[r + 1] = ro[r] + rcount[r] * width;
  }
  if (scount[P.rank] != rcount[P.rank]) throw Error(FMM_ERR_COMM, "LET exchange: self counts differ (internal)");
  if (scount[P.rank] > 0)
    FMM_CUDA(cudaMemcpyAsync(recv + ro[P.rank], send + so[P.rank], sizeof(double) * scount[P.rank] * width,
                             cudaMemcpyDeviceToDevice, P.stream));
  check(a.groupStart(), "ncclGroupStart");
  for (int r = 0; r < P.world; ++r) {
    if (r == P.rank) continue;
    if (scount[r] > 0)
      check(a.send(send + so[r], (size_t)(scount[r] * width), ncclDouble, r, (ncclComm_t)P.nccl_comm, P.stream),
            "ncclSend");
    if (rcount[r] > 0)
      check(a.recv(recv + ro[r], (size_t)(rcount[r] * width), ncclDouble, r, (ncclComm_t)P.nccl_comm, P.stream),
            "ncclRecv");
  }
  check(a.groupEnd(), "ncclGroupEnd");
}

void comm_allgather(fmm_plan_s& P, const double* send, int64_t count, double* recv) {
  if (count == 0) return;
  check(api().allGather(send, recv, (size_t)count, ncclDouble, (ncclComm_t)P.nccl_comm, P.stream), "ncclAllGather");
}

}  // namespace fmm

extern "C" FMM_API fmm_status fmm_nccl_unique_id(void* out) {
  if (!out) return fmm::set_error(FMM_ERR_USAGE, "fmm_nccl_unique_id: out is NULL");
  try {
    fmm::comm_unique_id(out);
    return FMM_OK;
  } catch (const fmm::Error& e) {
    return fmm::set_error(e.status, e.what());
  }
}
