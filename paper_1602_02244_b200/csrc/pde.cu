// pde.cu — NEXT-2 (include/fmm_pde.h): the FMM mat-vec as a low-accuracy preconditioner in a
// Krylov solve of the 3D Dirichlet Laplace equation on the [-1,1]^3 lattice (PAPER.md:439-471,
// §4.2). Stencil, vector kernels, the boundary-correction operators and the flexible PCG
// driver; the two potential sums of every preconditioner application are fmm_matvec calls on
// one plan over the lattice nodes and the face panels. Readings: fmm_pde.h, DESIGN.md §3.
//
// Determinism: every reduction (dot products, the S^-1 GEMV) sums in a fixed order, so a
// solve is bitwise reproducible on one device, like the mat-vec.
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <utility>
#include <vector>

#include "fmm_pde.h"
#include "pde_common.cuh"
#include "plan.h"

namespace {

constexpr int kDotBlocks = 592;  // fixed grid of the two-pass dot product (4 x 148 SMs)
constexpr int kDotThreads = 256;

// A u = (6 u_c - (((((u_x- + u_x+) + u_y-) + u_y+) + u_z-) + u_z+)) / h^2, zero ghosts
__global__ void stencil_kernel(int n, double h2, const double* __restrict__ u, double* __restrict__ out) {
  const int64_t N = (int64_t)n * n * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % n), j = (int)((t / n) % n), k = (int)(t / ((int64_t)n * n));
    const int64_t sn = n, sn2 = (int64_t)n * n;
    const double xm = i > 0 ? u[t - 1] : 0.0, xp = i + 1 < n ? u[t + 1] : 0.0;
    const double ym = j > 0 ? u[t - sn] : 0.0, yp = j + 1 < n ? u[t + sn] : 0.0;
    const double zm = k > 0 ? u[t - sn2] : 0.0, zp = k + 1 < n ? u[t + sn2] : 0.0;
    const double nb = ((((xm + xp) + ym) + yp) + zm) + zp;
    out[t] = __ddiv_rn(__dsub_rn(__dmul_rn(6.0, u[t]), nb), h2);  // no contraction: the oracle's rounding
  }
}

// S_ij = a^2 / (4 pi |y_i - y_j|), S_ii = a C_panel / (4 pi), column-major (= row-major: symmetric)
__global__ void boundary_matrix_kernel(int nf, const double* __restrict__ Y, double a, double* __restrict__ S) {
  const double cpanel = 4.0 * log(1.0 + sqrt(2.0));
  const int64_t tot = (int64_t)nf * nf;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % nf), j = (int)(t / nf);
    double v;
    if (i == j) {
      v = a * cpanel / (4.0 * kPi);
    } else {
      const double dx = Y[3 * i] - Y[3 * j], dy = Y[3 * i + 1] - Y[3 * j + 1], dz = Y[3 * i + 2] - Y[3 * j + 2];
      const double d = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      v = a * a / (4.0 * kPi * d);
    }
    S[t] = v;
  }
}

__global__ void scaled_identity_kernel(int nf, double s, double* __restrict__ X) {
  const int64_t tot = (int64_t)nf * nf;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x)
    X[t] = (t % nf == t / nf) ? s : 0.0;
}

// per-row absolute sums (row r of a column-major symmetric matrix = its column r)
__global__ void rowsum_kernel(int nf, const double* __restrict__ S, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nf) return;
  double s = 0.0;
  for (int c = lane; c < nf; c += 32) s += fabs(S[(int64_t)r * nf + c]);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

// out = y . w (fixed-order two-pass reduction); partial[b] = block b's sum over its strided range
__global__ void dot_partial_kernel(int64_t n, const double* __restrict__ y, const double* __restrict__ w,
                                   const double* __restrict__ w2, double* __restrict__ part) {
  __shared__ double s1[kDotThreads], s2[kDotThreads];
  double a = 0.0, b = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    a = fma(y[t], w[t], a);
    if (w2) b = fma(y[t], w2[t], b);
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1[0];
    part[gridDim.x + blockIdx.x] = s2[0];
  }
}
__global__ void dot_final_kernel(int nb, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double s1[kDotThreads], s2[kDotThreads];
  double a = 0.0, b = 0.0;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    a += part[t];
    b += part[nb + t];
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s1[0];
    out[1] = s2[0];
  }
}

// sum of squares of R (Frobenius^2), same two-pass scheme
__global__ void sumsq_partial_kernel(int64_t n, const double* __restrict__ R, double* __restrict__ part) {
  __shared__ double s1[kDotThreads];
  double a = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    a = fma(R[t], R[t], a);
  s1[threadIdx.x] = a;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) s1[threadIdx.x] += s1[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1[0];
    part[gridDim.x + blockIdx.x] = 0.0;
  }
}

// sigma = Sinv b: warp per row, lanes over columns, fixed-order butterfly (Sinv symmetric)
__global__ void gemv_kernel(int nf, const double* __restrict__ A, const double* __restrict__ b,
                            double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nf) return;
  const double* row = A + (int64_t)r * nf;
  double s = 0.0;
  for (int c = lane; c < nf; c += 32) s = fma(row[c], b[c], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

// q = [c r ; 0]
__global__ void volume_charges_kernel(int64_t N, int64_t nf, double c, const double* __restrict__ r,
                                      double* __restrict__ q) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x)
    q[t] = t < N ? c * r[t] : 0.0;
}
// z = phi[:N] + c_self r; bf = -phi[N:]
__global__ void volume_split_kernel(int64_t N, int64_t nf, double c_self, const double* __restrict__ phi,
                                    const double* __restrict__ r, double* __restrict__ z, double* __restrict__ bf) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < N)
      z[t] = phi[t] + c_self * r[t];
    else if (bf)
      bf[t - N] = -phi[t];
  }
}
// q = [0 ; c sigma]
__global__ void layer_charges_kernel(int64_t N, int64_t nf, double c, const double* __restrict__ sigma,
                                     double* __restrict__ q) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x)
    q[t] = t < N ? 0.0 : c * sigma[t - N];
}
__global__ void add_kernel(int64_t N, const double* __restrict__ a, double* __restrict__ z) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    z[t] += a[t];
}
// x += alpha d; r -= alpha q
__global__ void cg_update_kernel(int64_t N, double alpha, const double* __restrict__ d, const double* __restrict__ q,
                                 double* __restrict__ x, double* __restrict__ r) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    x[t] = fma(alpha, d[t], x[t]);
    r[t] = fma(-alpha, q[t], r[t]);
  }
}
// d = z + beta d
__global__ void cg_direction_kernel(int64_t N, double beta, const double* __restrict__ z, double* __restrict__ d) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    d[t] = fma(beta, d[t], z[t]);
}

// fixed-order dot products (y.w, y.w2) read back to the host (synchronises s)
struct Dot {
  fmm::DevBuf<double> part, out;
  double* host = nullptr;
  Dot() {
    part.alloc(2 * kDotBlocks);
    out.alloc(2);
    FMM_CUDA(cudaMallocHost(&host, 2 * sizeof(double)));
  }
  ~Dot() {
    if (host) cudaFreeHost(host);
  }
  std::pair<double, double> operator()(int64_t n, const double* y, const double* w, const double* w2,
                                       cudaStream_t s) {
    dot_partial_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, y, w, w2, part);
    FMM_LAUNCHED("dot_partial_kernel");
    dot_final_kernel<<<1, kDotThreads, 0, s>>>(kDotBlocks, part, out);
    FMM_LAUNCHED("dot_final_kernel");
    FMM_CUDA(cudaMemcpyAsync(host, out.ptr, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    return {host[0], host[1]};
  }
  double sumsq(int64_t n, const double* R, cudaStream_t s) {
    sumsq_partial_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, R, part);
    FMM_LAUNCHED("sumsq_partial_kernel");
    dot_final_kernel<<<1, kDotThreads, 0, s>>>(kDotBlocks, part, out);
    FMM_LAUNCHED("dot_final_kernel");
    FMM_CUDA(cudaMemcpyAsync(host, out.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    return host[0];
  }
};

void stencil(int n, const double* u, double* out, cudaStream_t s) {
  const double h = 2.0 / (n + 1);
  const int64_t N = (int64_t)n * n * n;
  stencil_kernel<<<grid_for(N), 256, 0, s>>>(n, h * h, u, out);
  FMM_LAUNCHED("stencil_kernel");
}

}  // namespace

struct fmm_precond_s {
  int n = 0, stride = 1, nfa = 0;
  int64_t N = 0, nf = 0;
  double h = 0, a = 0, c_self = 0;
  bool boundary = true;
  int device = 0;
  cudaStream_t stream = nullptr;
  fmm_plan plan = nullptr;
  fmm::DevBuf<double> xyz, q, phi, Sinv, bf, sigma;
  ~fmm_precond_s() {
    if (plan) fmm_destroy(plan);
  }
  int64_t bytes() const {
    return xyz.bytes() + q.bytes() + phi.bytes() + Sinv.bytes() + bf.bytes() + sigma.bytes();
  }

  // S^-1 by the Newton-Schulz iteration X <- X (2I - S X) (X0 = I / ||S||_inf, S SPD), DGEMMs by cuBLAS
  void invert_boundary(const double* S) {
    const int m = (int)nf;
    const int64_t mm = (int64_t)m * m;
    cublasHandle_t hb = nullptr;
    check_blas(cublasCreate(&hb), "cublasCreate");
    struct HG {
      cublasHandle_t h;
      ~HG() { cublasDestroy(h); }
    } hg{hb};
    check_blas(cublasSetStream(hb, stream), "cublasSetStream");
    fmm::DevBuf<double> X2, R, rs;
    Sinv.alloc(mm);
    X2.alloc(mm);
    R.alloc(mm);
    rs.alloc(m);
    rowsum_kernel<<<(m + 7) / 8, 256, 0, stream>>>(m, S, rs);
    FMM_LAUNCHED("rowsum_kernel");
    std::vector<double> hrs(m);
    FMM_CUDA(cudaMemcpyAsync(hrs.data(), rs.ptr, sizeof(double) * m, cudaMemcpyDeviceToHost, stream));
    FMM_CUDA(cudaStreamSynchronize(stream));
    const double snorm = *std::max_element(hrs.begin(), hrs.end());
    scaled_identity_kernel<<<grid_for(mm), 256, 0, stream>>>(m, 1.0 / snorm, Sinv);
    FMM_LAUNCHED("scaled_identity_kernel");
    Dot dot;
    const double one = 1.0, mone = -1.0;
    bool ok = false;
    for (int it = 0; it < 200; ++it) {
      // R = I - S X
      scaled_identity_kernel<<<grid_for(mm), 256, 0, stream>>>(m, 1.0, R);
      FMM_LAUNCHED("scaled_identity_kernel");
      check_blas(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &mone, S, m, Sinv.ptr, m, &one, R.ptr, m),
                 "cublasDgemm");
      const double fro = std::sqrt(dot.sumsq(mm, R, stream));
      if (!std::isfinite(fro)) break;
      if (fro <= 1e-13 * std::sqrt((double)m)) {
        ok = true;
        break;
      }
      // X <- X + X R
      FMM_CUDA(cudaMemcpyAsync(X2.ptr, Sinv.ptr, sizeof(double) * mm, cudaMemcpyDeviceToDevice, stream));
      check_blas(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, Sinv.ptr, m, R.ptr, m, &one, X2.ptr, m),
                 "cublasDgemm");
      std::swap(Sinv, X2);
    }
    if (!ok) throw fmm::Error(FMM_ERR_NUMERIC, "fmm_precond_setup: Newton-Schulz inverse of S did not converge");
  }

  void apply(const double* r, double* z) {
    const int64_t T = N + nf;
    volume_charges_kernel<<<grid_for(T), 256, 0, stream>>>(N, nf, h * h * h / (4.0 * kPi), r, q);
    FMM_LAUNCHED("volume_charges_kernel");
    fmm_status st = fmm_matvec(plan, q, T, phi, nullptr);
    if (st != FMM_OK) throw fmm::Error(st, fmm_last_error());
    volume_split_kernel<<<grid_for(T), 256, 0, stream>>>(N, nf, c_self, phi, r, z, boundary ? bf.ptr : nullptr);
    FMM_LAUNCHED("volume_split_kernel");
    if (!boundary) return;
    gemv_kernel<<<(unsigned)((nf + 7) / 8), 256, 0, stream>>>((int)nf, Sinv, bf, sigma);
    FMM_LAUNCHED("gemv_kernel");
    layer_charges_kernel<<<grid_for(T), 256, 0, stream>>>(N, nf, a * a / (4.0 * kPi), sigma, q);
    FMM_LAUNCHED("layer_charges_kernel");
    st = fmm_matvec(plan, q, T, phi, nullptr);
    if (st != FMM_OK) throw fmm::Error(st, fmm_last_error());
    add_kernel<<<grid_for(N), 256, 0, stream>>>(N, phi, z);
    FMM_LAUNCHED("add_kernel");
  }
};

extern "C" {

fmm_status fmm_stencil_apply(int n, const double* u, double* out, void* stream) {
  return Guard::run([&] {
    usage(n >= 1 && (int64_t)n * n * n < ((int64_t)1 << 31), "fmm_stencil_apply: n must be in [1, 1290]");
    usage(u && out && u != out, "fmm_stencil_apply: u / out NULL or aliased");
    stencil(n, u, out, (cudaStream_t)stream);
  });
}

fmm_status fmm_precond_setup(fmm_precond* out, int n, int face_stride, int p, int ncrit, double theta, int boundary,
                             const fmm_exec* ex) {
  fmm_precond_s* P = nullptr;
  const fmm_status st = Guard::run([&] {
    usage(out != nullptr && ex != nullptr, "fmm_precond_setup: out / ex is NULL");
    *out = nullptr;
    usage(n >= 1 && (int64_t)n * n * n < ((int64_t)1 << 30), "fmm_precond_setup: n must be in [1, 1023]");
    usage(face_stride >= 1, "fmm_precond_setup: face_stride must be >= 1");
    usage(ex->world_size == 1, "fmm_precond_setup: single-GPU only");
    FMM_CUDA(cudaSetDevice(ex->device));
    P = new fmm_precond_s();
    P->n = n;
    P->stride = face_stride;
    P->nfa = (n + face_stride - 1) / face_stride;
    P->N = (int64_t)n * n * n;
    P->nf = 6LL * P->nfa * P->nfa;
    P->h = 2.0 / (n + 1);
    P->a = face_stride * P->h;
    P->c_self = P->h * P->h * (3.0 * std::log(2.0 + std::sqrt(3.0)) - kPi / 2.0) / (4.0 * kPi);
    P->boundary = boundary != 0;
    P->device = ex->device;
    P->stream = (cudaStream_t)ex->stream;
    const int64_t T = P->N + P->nf;
    P->xyz.alloc(3 * T);
    points_kernel<<<grid_for(T), 256, 0, P->stream>>>(n, face_stride, P->nfa, P->h, P->xyz);
    FMM_LAUNCHED("points_kernel");
    fmm_status s = fmm_setup(&P->plan, P->xyz, T, p, ncrit, theta, ex);
    if (s != FMM_OK) throw fmm::Error(s, fmm_last_error());
    P->q.alloc(T);
    P->phi.alloc(T);
    if (P->boundary) {
      P->bf.alloc(P->nf);
      P->sigma.alloc(P->nf);
      fmm::DevBuf<double> S;
      S.alloc(P->nf * P->nf);
      boundary_matrix_kernel<<<grid_for(P->nf * P->nf), 256, 0, P->stream>>>((int)P->nf, P->xyz.ptr + 3 * P->N, P->a,
                                                                              S);
      FMM_LAUNCHED("boundary_matrix_kernel");
      P->invert_boundary(S);
    }
    FMM_CUDA(cudaStreamSynchronize(P->stream));
    *out = P;
  });
  if (st != FMM_OK) delete P;
  return st;
}

fmm_status fmm_precond_apply(fmm_precond P, const double* r, double* z) {
  return Guard::run([&] {
    usage(P != nullptr && r && z && r != z, "fmm_precond_apply: NULL or aliased argument");
    FMM_CUDA(cudaSetDevice(P->device));
    P->apply(r, z);
  });
}

fmm_status fmm_precond_info(fmm_precond P, int64_t* n_panels, int64_t* bytes) {
  return Guard::run([&] {
    usage(P != nullptr, "fmm_precond_info: NULL");
    if (n_panels) *n_panels = P->boundary ? P->nf : 0;
    if (bytes) {
      fmm_stats_t s;
      fmm_status st = fmm_stats(P->plan, &s);
      if (st != FMM_OK) throw fmm::Error(st, fmm_last_error());
      *bytes = P->bytes() + s.bytes_device;
    }
  });
}

void fmm_precond_destroy(fmm_precond P) { delete P; }

fmm_status fmm_pcg_solve(int n, const double* b, double* x, fmm_precond M, double rtol, int maxit, double* hist,
                         fmm_pcg_info* info, void* stream) {
  return Guard::run([&] {
    usage(n >= 1 && (int64_t)n * n * n < ((int64_t)1 << 31), "fmm_pcg_solve: bad n");
    usage(b && x && b != x, "fmm_pcg_solve: b / x NULL or aliased");
    usage(rtol > 0.0 && maxit >= 0, "fmm_pcg_solve: rtol must be > 0 and maxit >= 0");
    usage(!M || M->n == n, "fmm_pcg_solve: preconditioner set up for another n");
    cudaStream_t s = M ? M->stream : (cudaStream_t)stream;
    const int64_t N = (int64_t)n * n * n;
    fmm::DevBuf<double> r, z, zo, d, q;
    r.alloc(N);
    z.alloc(N);
    zo.alloc(N);
    d.alloc(N);
    q.alloc(N);
    cudaEvent_t e0, e1, p0, p1;
    FMM_CUDA(cudaEventCreate(&e0));
    FMM_CUDA(cudaEventCreate(&e1));
    FMM_CUDA(cudaEventCreate(&p0));
    FMM_CUDA(cudaEventCreate(&p1));
    struct EG {
      cudaEvent_t a, b, c, d;
      ~EG() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaEventDestroy(c);
        cudaEventDestroy(d);
      }
    } eg{e0, e1, p0, p1};
    double t_pre = 0.0;
    auto precond = [&](const double* rr, double* zz) {
      if (!M) {
        FMM_CUDA(cudaMemcpyAsync(zz, rr, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
        return;
      }
      FMM_CUDA(cudaEventRecord(p0, s));
      M->apply(rr, zz);
      FMM_CUDA(cudaEventRecord(p1, s));
      FMM_CUDA(cudaEventSynchronize(p1));
      float ms = 0.f;
      FMM_CUDA(cudaEventElapsedTime(&ms, p0, p1));
      t_pre += ms;
    };
    Dot dot;
    FMM_CUDA(cudaEventRecord(e0, s));
    FMM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, s));
    FMM_CUDA(cudaMemcpyAsync(r.ptr, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    const double nb = std::sqrt(dot(N, b, b, nullptr, s).first);
    if (hist) hist[0] = 1.0;
    int it = 0;
    double rel = nb == 0.0 ? 0.0 : 1.0;
    if (nb > 0.0 && maxit > 0) {
      precond(r, z);
      FMM_CUDA(cudaMemcpyAsync(d.ptr, z.ptr, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
      double rz = dot(N, r, z, nullptr, s).first;
      while (it < maxit) {
        stencil(n, d, q, s);
        const double dq = dot(N, d, q, nullptr, s).first;
        if (!(dq > 0.0) || !std::isfinite(dq) || !std::isfinite(rz))
          throw fmm::Error(FMM_ERR_NUMERIC, "fmm_pcg_solve: breakdown (d^T A d <= 0 or non-finite)");
        const double alpha = rz / dq;
        cg_update_kernel<<<grid_for(N), 256, 0, s>>>(N, alpha, d, q, x, r);
        FMM_LAUNCHED("cg_update_kernel");
        ++it;
        rel = std::sqrt(dot(N, r, r, nullptr, s).first) / nb;
        if (hist) hist[it] = rel;
        if (rel <= rtol) break;
        std::swap(z, zo);
        precond(r, z);
        const auto rzz = dot(N, r, z, zo, s);  // (r, z_new), (r, z_old)
        const double beta = (rzz.first - rzz.second) / rz;
        cg_direction_kernel<<<grid_for(N), 256, 0, s>>>(N, beta, z, d);
        FMM_LAUNCHED("cg_direction_kernel");
        rz = rzz.first;
      }
    }
    FMM_CUDA(cudaEventRecord(e1, s));
    FMM_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FMM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (info) {
      info->iterations = it;
      info->converged = rel <= rtol;
      info->relres = rel;
      info->t_total_ms = ms;
      info->t_precond_ms = t_pre;
    }
  });
}

}  // extern "C"
