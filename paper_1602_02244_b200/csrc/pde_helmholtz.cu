// pde_helmholtz.cu — NEXT-4 solve (include/fmm_pde.h, second half): the Helmholtz FMM mat-vec of
// include/fmm_helmholtz.h as the preconditioner inside GMRES for -Delta_h u - kappa^2 u = f on the
// [-1,1]^3 lattice with Dirichlet faces ("the Laplace equation and Helmholtz equation on a 3D
// cubic lattice [-1,1]^3 [...] The preconditioners are used inside a Krylov subspace solver",
// PAPER.md:443-446; Fig 6: kappa = 7, h = 2^-5). Stencil, the complex
// boundary-correction operators and the GMRES driver; the two potential sums of every
// preconditioner application are fmm_matvec_helmholtz calls on one plan over the lattice nodes and
// the face panels. Readings: fmm_pde.h, DESIGN.md §3 (R56-R60).
//
// Complex vectors are double2 (re, im). Determinism: every reduction (norms, the Gram-Schmidt
// inner products, the S^-1 GEMV, the basis combinations) sums in a fixed order, so a solve is
// bitwise reproducible on one device.
#include <cublas_v2.h>

#include <cmath>
#include <complex>
#include <utility>
#include <vector>

#include "fmm_helmholtz.h"
#include "fmm_pde.h"
#include "pde_common.cuh"
#include "plan.h"

namespace {

constexpr int kRedBlocks = 296;  // fixed grid of the two-pass reductions (2 x 148 SMs)
constexpr int kRedThreads = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// out = lap(u) - kappa^2 u per component, lap = (6 u_c - (((((u_x- + u_x+) + u_y-) + u_y+) + u_z-) + u_z+)) / h^2
// (the oracle's rounding: no contraction)
__global__ void helm_stencil_kernel(int n, double h2, double k2, const double2* __restrict__ u,
                                    double2* __restrict__ out) {
  const int64_t N = (int64_t)n * n * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % n), j = (int)((t / n) % n), k = (int)(t / ((int64_t)n * n));
    const int64_t sn = n, sn2 = (int64_t)n * n;
    const double2 z = make_double2(0.0, 0.0);
    const double2 xm = i > 0 ? u[t - 1] : z, xp = i + 1 < n ? u[t + 1] : z;
    const double2 ym = j > 0 ? u[t - sn] : z, yp = j + 1 < n ? u[t + sn] : z;
    const double2 zm = k > 0 ? u[t - sn2] : z, zp = k + 1 < n ? u[t + sn2] : z;
    const double2 c = u[t];
    const double nbx = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(xm.x, xp.x), ym.x), yp.x), zm.x), zp.x);
    const double nby = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(xm.y, xp.y), ym.y), yp.y), zm.y), zp.y);
    const double lx = __ddiv_rn(__dsub_rn(__dmul_rn(6.0, c.x), nbx), h2);
    const double ly = __ddiv_rn(__dsub_rn(__dmul_rn(6.0, c.y), nby), h2);
    out[t] = make_double2(__dsub_rn(lx, __dmul_rn(k2, c.x)), __dsub_rn(ly, __dmul_rn(k2, c.y)));
  }
}

// S_ij = a^2 exp(i kappa d) / (4 pi d), S_ii = a C_panel / (4 pi) + i kappa a^2 / (4 pi); column-major
// (complex symmetric: S^T = S)
__global__ void helm_boundary_matrix_kernel(int nf, const double* __restrict__ Y, double a, double kappa,
                                            double2* __restrict__ S) {
  const double cpanel = 4.0 * log(1.0 + sqrt(2.0));
  const int64_t tot = (int64_t)nf * nf;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % nf), j = (int)(t / nf);
    double2 v;
    if (i == j) {
      v = make_double2(a * cpanel / (4.0 * kPi), kappa * a * a / (4.0 * kPi));
    } else {
      const double dx = Y[3 * i] - Y[3 * j], dy = Y[3 * i + 1] - Y[3 * j + 1], dz = Y[3 * i + 2] - Y[3 * j + 2];
      const double d = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      double s, c;
      sincos(kappa * d, &s, &c);
      const double f = a * a / (4.0 * kPi * d);
      v = make_double2(f * c, f * s);
    }
    S[t] = v;
  }
}

// X = s conj(S) (the Newton-Schulz start S^H / (||S||_1 ||S||_inf); S symmetric) or X = s I (S NULL)
__global__ void helm_start_kernel(int nf, double s, const double2* __restrict__ S, double2* __restrict__ X) {
  const int64_t tot = (int64_t)nf * nf;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    if (S)
      X[t] = make_double2(s * S[t].x, -s * S[t].y);
    else
      X[t] = make_double2((t % nf == t / nf) ? s : 0.0, 0.0);
  }
}

// per-row sums of |S_rc| (row r of a column-major symmetric matrix = its column r)
__global__ void helm_rowsum_kernel(int nf, const double2* __restrict__ S, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nf) return;
  double s = 0.0;
  for (int c = lane; c < nf; c += 32) {
    const double2 v = S[(int64_t)r * nf + c];
    s += sqrt(v.x * v.x + v.y * v.y);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

// fixed-order two-pass reductions. Pass 1, block (b, j): over its strided range of vector j,
// conj(V_j) . w (complex) or |w|^2 (V NULL: one vector); pass 2: one block per j sums the
// kRedBlocks partials.
__global__ void multidot_partial_kernel(int64_t N, const double2* __restrict__ V, int64_t ldv,
                                        const double2* __restrict__ w, double2* __restrict__ part) {
  __shared__ double sx[kRedThreads], sy[kRedThreads];
  const int j = blockIdx.y;
  const double2* v = V ? V + (int64_t)j * ldv : nullptr;
  double ax = 0.0, ay = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const double2 b = w[t];
    if (v) {
      const double2 a = v[t];
      ax = fma(a.x, b.x, fma(a.y, b.y, ax));
      ay = fma(a.x, b.y, fma(-a.y, b.x, ay));
    } else {
      ax = fma(b.x, b.x, fma(b.y, b.y, ax));
    }
  }
  sx[threadIdx.x] = ax;
  sy[threadIdx.x] = ay;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sx[threadIdx.x] += sx[threadIdx.x + o];
      sy[threadIdx.x] += sy[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)j * gridDim.x + blockIdx.x] = make_double2(sx[0], sy[0]);
}
__global__ void multidot_final_kernel(int nb, const double2* __restrict__ part, double2* __restrict__ out) {
  __shared__ double sx[kRedThreads], sy[kRedThreads];
  const int j = blockIdx.x;
  double ax = 0.0, ay = 0.0;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    ax += part[(int64_t)j * nb + t].x;
    ay += part[(int64_t)j * nb + t].y;
  }
  sx[threadIdx.x] = ax;
  sy[threadIdx.x] = ay;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sx[threadIdx.x] += sx[threadIdx.x + o];
      sy[threadIdx.x] += sy[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = make_double2(sx[0], sy[0]);
}

// out = w_in - sum_{j < k} c_j V_j, or out = sum_{j < k} c_j V_j (w_in NULL): fixed order in j (out may be w_in)
__global__ void combine_kernel(int64_t N, int k, const double2* __restrict__ V, int64_t ldv,
                               const double2* __restrict__ c, const double2* w_in, double2* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int j = 0; j < k; ++j) {
      const double2 v = V[(int64_t)j * ldv + t], cj = c[j];
      s.x = fma(cj.x, v.x, fma(-cj.y, v.y, s.x));
      s.y = fma(cj.x, v.y, fma(cj.y, v.x, s.y));
    }
    out[t] = w_in ? make_double2(w_in[t].x - s.x, w_in[t].y - s.y) : s;
  }
}

// out = w / sqrt(nrm2->x) (the next Arnoldi vector) or w * s (nrm2 NULL)
__global__ void scale_kernel(int64_t N, const double2* __restrict__ nrm2, double s, const double2* __restrict__ w,
                             double2* __restrict__ out) {
  const double f = nrm2 ? 1.0 / sqrt(nrm2->x) : s;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = make_double2(w[t].x * f, w[t].y * f);
}

// sigma = Sinv b: warp per row, lanes over columns, fixed-order butterfly (Sinv symmetric)
__global__ void helm_gemv_kernel(int nf, const double2* __restrict__ A, const double2* __restrict__ b,
                                 double2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nf) return;
  const double2* row = A + (int64_t)r * nf;
  double sx = 0.0, sy = 0.0;
  for (int c = lane; c < nf; c += 32) {
    const double2 a = row[c], v = b[c];
    sx = fma(a.x, v.x, fma(-a.y, v.y, sx));
    sy = fma(a.x, v.y, fma(a.y, v.x, sy));
  }
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
  }
  if (lane == 0) out[r] = make_double2(sx, sy);
}

// q = [c r ; 0] (c real)
__global__ void helm_volume_charges_kernel(int64_t N, int64_t nf, double c, const double2* __restrict__ r,
                                           double2* __restrict__ q) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x)
    q[t] = t < N ? make_double2(c * r[t].x, c * r[t].y) : make_double2(0.0, 0.0);
}
// z = phi[:N] + c_self r; bf = -phi[N:]
__global__ void helm_volume_split_kernel(int64_t N, int64_t nf, double2 c_self, const double2* __restrict__ phi,
                                         const double2* __restrict__ r, double2* __restrict__ z,
                                         double2* __restrict__ bf) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < N) {
      const double2 s = cmul(c_self, r[t]);
      z[t] = make_double2(phi[t].x + s.x, phi[t].y + s.y);
    } else if (bf) {
      bf[t - N] = make_double2(-phi[t].x, -phi[t].y);
    }
  }
}
// q = [0 ; c sigma]
__global__ void helm_layer_charges_kernel(int64_t N, int64_t nf, double c, const double2* __restrict__ sigma,
                                          double2* __restrict__ q) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N + nf; t += (int64_t)gridDim.x * blockDim.x)
    q[t] = t < N ? make_double2(0.0, 0.0) : make_double2(c * sigma[t - N].x, c * sigma[t - N].y);
}
__global__ void helm_add_kernel(int64_t N, const double2* __restrict__ a, double2* __restrict__ z) {  // a != z
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    z[t] = make_double2(z[t].x + a[t].x, z[t].y + a[t].y);
}

void helm_stencil(int n, double kappa, const double2* u, double2* out, cudaStream_t s) {
  const double h = 2.0 / (n + 1);
  const int64_t N = (int64_t)n * n * n;
  helm_stencil_kernel<<<grid_for(N), 256, 0, s>>>(n, h * h, kappa * kappa, u, out);
  FMM_LAUNCHED("helm_stencil_kernel");
}

// k fixed-order inner products conj(V_j) . w (j < k) into out[0..k) (device); V NULL: |w|^2 into out[0].x
void multidot(int64_t N, int k, const double2* V, int64_t ldv, const double2* w, double2* part, double2* out,
              cudaStream_t s) {
  multidot_partial_kernel<<<dim3(kRedBlocks, k), kRedThreads, 0, s>>>(N, V, ldv, w, part);
  FMM_LAUNCHED("multidot_partial_kernel");
  multidot_final_kernel<<<k, kRedThreads, 0, s>>>(kRedBlocks, part, out);
  FMM_LAUNCHED("multidot_final_kernel");
}

}  // namespace

struct fmm_hprecond_s {
  int n = 0, stride = 1, nfa = 0;
  int64_t N = 0, nf = 0;
  double h = 0, a = 0, kappa = 0;
  double2 c_self{0, 0};
  bool boundary = true;
  int device = 0;
  cudaStream_t stream = nullptr;
  fmm_plan plan = nullptr;
  fmm::DevBuf<double> xyz;
  fmm::DevBuf<double2> q, phi, Sinv, bf, sigma;
  ~fmm_hprecond_s() {
    if (plan) fmm_destroy(plan);
  }
  int64_t bytes() const {
    return xyz.bytes() + q.bytes() + phi.bytes() + Sinv.bytes() + bf.bytes() + sigma.bytes();
  }

  // S^-1 by the Newton-Schulz iteration X <- X + X (I - S X), X0 = S^H / ||S||_inf^2 (S symmetric:
  // ||S||_1 = ||S||_inf; then ||I - S X0||_2 < 1 for any non-singular S), ZGEMMs by cuBLAS
  void invert_boundary(const double2* S) {
    const int m = (int)nf;
    const int64_t mm = (int64_t)m * m;
    cublasHandle_t hb = nullptr;
    check_blas(cublasCreate(&hb), "cublasCreate");
    struct HG {
      cublasHandle_t h;
      ~HG() { cublasDestroy(h); }
    } hg{hb};
    check_blas(cublasSetStream(hb, stream), "cublasSetStream");
    fmm::DevBuf<double2> X2, R, part, out;
    fmm::DevBuf<double> rs;
    Sinv.alloc(mm);
    X2.alloc(mm);
    R.alloc(mm);
    rs.alloc(m);
    part.alloc(kRedBlocks);
    out.alloc(1);
    helm_rowsum_kernel<<<(m + 7) / 8, 256, 0, stream>>>(m, S, rs);
    FMM_LAUNCHED("helm_rowsum_kernel");
    std::vector<double> hrs(m);
    FMM_CUDA(cudaMemcpyAsync(hrs.data(), rs.ptr, sizeof(double) * m, cudaMemcpyDeviceToHost, stream));
    FMM_CUDA(cudaStreamSynchronize(stream));
    const double snorm = *std::max_element(hrs.begin(), hrs.end());
    helm_start_kernel<<<grid_for(mm), 256, 0, stream>>>(m, 1.0 / (snorm * snorm), S, Sinv);
    FMM_LAUNCHED("helm_start_kernel");
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), mone = make_cuDoubleComplex(-1.0, 0.0);
    bool ok = false;
    double2 fro2{0, 0};
    for (int it = 0; it < 400; ++it) {
      // R = I - S X
      helm_start_kernel<<<grid_for(mm), 256, 0, stream>>>(m, 1.0, nullptr, R);
      FMM_LAUNCHED("helm_start_kernel");
      check_blas(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &mone, (const cuDoubleComplex*)S, m,
                             (const cuDoubleComplex*)Sinv.ptr, m, &one, (cuDoubleComplex*)R.ptr, m),
                 "cublasZgemm");
      multidot(mm, 1, nullptr, 0, R, part, out, stream);
      FMM_CUDA(cudaMemcpyAsync(&fro2, out.ptr, sizeof(double2), cudaMemcpyDeviceToHost, stream));
      FMM_CUDA(cudaStreamSynchronize(stream));
      const double fro = std::sqrt(fro2.x);
      if (!std::isfinite(fro)) break;
      if (fro <= 1e-13 * std::sqrt((double)m)) {
        ok = true;
        break;
      }
      // X <- X + X R
      FMM_CUDA(cudaMemcpyAsync(X2.ptr, Sinv.ptr, sizeof(double2) * mm, cudaMemcpyDeviceToDevice, stream));
      check_blas(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, (const cuDoubleComplex*)Sinv.ptr, m,
                             (const cuDoubleComplex*)R.ptr, m, &one, (cuDoubleComplex*)X2.ptr, m),
                 "cublasZgemm");
      std::swap(Sinv, X2);
    }
    if (!ok) throw fmm::Error(FMM_ERR_NUMERIC, "fmm_hprecond_setup: Newton-Schulz inverse of S did not converge");
  }

  void apply(const double2* r, double2* z) {
    const int64_t T = N + nf;
    helm_volume_charges_kernel<<<grid_for(T), 256, 0, stream>>>(N, nf, h * h * h / (4.0 * kPi), r, q);
    FMM_LAUNCHED("helm_volume_charges_kernel");
    fmm_status st = fmm_matvec_helmholtz(plan, (const double*)q.ptr, T, (double*)phi.ptr);
    if (st != FMM_OK) throw fmm::Error(st, fmm_last_error());
    helm_volume_split_kernel<<<grid_for(T), 256, 0, stream>>>(N, nf, c_self, phi, r, z, boundary ? bf.ptr : nullptr);
    FMM_LAUNCHED("helm_volume_split_kernel");
    if (!boundary) return;
    helm_gemv_kernel<<<(unsigned)((nf + 7) / 8), 256, 0, stream>>>((int)nf, Sinv, bf, sigma);
    FMM_LAUNCHED("helm_gemv_kernel");
    helm_layer_charges_kernel<<<grid_for(T), 256, 0, stream>>>(N, nf, a * a / (4.0 * kPi), sigma, q);
    FMM_LAUNCHED("helm_layer_charges_kernel");
    st = fmm_matvec_helmholtz(plan, (const double*)q.ptr, T, (double*)phi.ptr);
    if (st != FMM_OK) throw fmm::Error(st, fmm_last_error());
    helm_add_kernel<<<grid_for(N), 256, 0, stream>>>(N, phi, z);
    FMM_LAUNCHED("helm_add_kernel");
  }
};

extern "C" {

fmm_status fmm_helmholtz_stencil_apply(int n, double kappa, const double* u, double* out, void* stream) {
  return Guard::run([&] {
    usage(n >= 1 && (int64_t)n * n * n < ((int64_t)1 << 30), "fmm_helmholtz_stencil_apply: n must be in [1, 1023]");
    usage(std::isfinite(kappa), "fmm_helmholtz_stencil_apply: kappa must be finite");
    usage(u && out && u != out, "fmm_helmholtz_stencil_apply: u / out NULL or aliased");
    helm_stencil(n, kappa, (const double2*)u, (double2*)out, (cudaStream_t)stream);
  });
}

fmm_status fmm_hprecond_setup(fmm_hprecond* out, int n, int face_stride, int p, int ncrit, double theta,
                              double kappa, int boundary, const fmm_exec* ex) {
  fmm_hprecond_s* P = nullptr;
  const fmm_status st = Guard::run([&] {
    usage(out != nullptr && ex != nullptr, "fmm_hprecond_setup: out / ex is NULL");
    *out = nullptr;
    usage(n >= 1 && (int64_t)n * n * n < ((int64_t)1 << 30), "fmm_hprecond_setup: n must be in [1, 1023]");
    usage(face_stride >= 1, "fmm_hprecond_setup: face_stride must be >= 1");
    usage(kappa > 0.0 && std::isfinite(kappa), "fmm_hprecond_setup: kappa must be > 0 and finite");
    usage(ex->world_size == 1, "fmm_hprecond_setup: single-GPU only");
    FMM_CUDA(cudaSetDevice(ex->device));
    P = new fmm_hprecond_s();
    P->n = n;
    P->stride = face_stride;
    P->nfa = (n + face_stride - 1) / face_stride;
    P->N = (int64_t)n * n * n;
    P->nf = 6LL * P->nfa * P->nfa;
    P->h = 2.0 / (n + 1);
    P->a = face_stride * P->h;
    P->kappa = kappa;
    P->c_self = make_double2(P->h * P->h * (3.0 * std::log(2.0 + std::sqrt(3.0)) - kPi / 2.0) / (4.0 * kPi),
                             kappa * P->h * P->h * P->h / (4.0 * kPi));
    P->boundary = boundary != 0;
    P->device = ex->device;
    P->stream = (cudaStream_t)ex->stream;
    const int64_t T = P->N + P->nf;
    P->xyz.alloc(3 * T);
    points_kernel<<<grid_for(T), 256, 0, P->stream>>>(n, face_stride, P->nfa, P->h, P->xyz);
    FMM_LAUNCHED("points_kernel");
    fmm_status s = fmm_setup_helmholtz(&P->plan, P->xyz, T, p, ncrit, theta, kappa, ex);
    if (s != FMM_OK) throw fmm::Error(s, fmm_last_error());
    P->q.alloc(T);
    P->phi.alloc(T);
    if (P->boundary) {
      P->bf.alloc(P->nf);
      P->sigma.alloc(P->nf);
      fmm::DevBuf<double2> S;
      S.alloc(P->nf * P->nf);
      helm_boundary_matrix_kernel<<<grid_for(P->nf * P->nf), 256, 0, P->stream>>>((int)P->nf, P->xyz.ptr + 3 * P->N,
                                                                                   P->a, kappa, S);
      FMM_LAUNCHED("helm_boundary_matrix_kernel");
      P->invert_boundary(S);
    }
    FMM_CUDA(cudaStreamSynchronize(P->stream));
    *out = P;
  });
  if (st != FMM_OK) delete P;
  return st;
}

fmm_status fmm_hprecond_apply(fmm_hprecond P, const double* r, double* z) {
  return Guard::run([&] {
    usage(P != nullptr && r && z && r != z, "fmm_hprecond_apply: NULL or aliased argument");
    FMM_CUDA(cudaSetDevice(P->device));
    P->apply((const double2*)r, (double2*)z);
  });
}

fmm_status fmm_hprecond_info(fmm_hprecond P, int64_t* n_panels, int64_t* bytes) {
  return Guard::run([&] {
    usage(P != nullptr, "fmm_hprecond_info: NULL");
    if (n_panels) *n_panels = P->boundary ? P->nf : 0;
    if (bytes) {
      fmm_stats_t s;
      fmm_status st = fmm_stats(P->plan, &s);
      if (st != FMM_OK) throw fmm::Error(st, fmm_last_error());
      *bytes = P->bytes() + s.bytes_device;
    }
  });
}

void fmm_hprecond_destroy(fmm_hprecond P) { delete P; }

fmm_status fmm_gmres_solve(int n, double kappa, const double* b_, double* x_, fmm_hprecond M, double rtol, int maxit,
                           double* hist, fmm_pcg_info* info, void* stream) {
  return Guard::run([&] {
    usage(n >= 1 && (int64_t)n * n * n < ((int64_t)1 << 30), "fmm_gmres_solve: bad n");
    usage(std::isfinite(kappa), "fmm_gmres_solve: kappa must be finite");
    usage(b_ && x_ && b_ != x_, "fmm_gmres_solve: b / x NULL or aliased");
    usage(rtol > 0.0 && maxit >= 0, "fmm_gmres_solve: rtol must be > 0 and maxit >= 0");
    usage(!M || (M->n == n && M->kappa == kappa), "fmm_gmres_solve: preconditioner set up for another n / kappa");
    const double2* b = (const double2*)b_;
    double2* x = (double2*)x_;
    cudaStream_t s = M ? M->stream : (cudaStream_t)stream;
    const int64_t N = (int64_t)n * n * n;
    fmm::DevBuf<double2> V, w, t, part, hd, nd;
    V.alloc((int64_t)(maxit + 1) * N);
    w.alloc(N);
    t.alloc(N);
    part.alloc((int64_t)kRedBlocks * (maxit + 1));
    hd.alloc(2 * (int64_t)(maxit + 1));  // two Gram-Schmidt passes
    nd.alloc(1);
    double2* hh = nullptr;  // pinned: [2 (maxit + 1)] passes, then the norm
    FMM_CUDA(cudaMallocHost(&hh, sizeof(double2) * (2 * (maxit + 1) + 1)));
    cudaEvent_t e0, e1, p0, p1;
    FMM_CUDA(cudaEventCreate(&e0));
    FMM_CUDA(cudaEventCreate(&e1));
    FMM_CUDA(cudaEventCreate(&p0));
    FMM_CUDA(cudaEventCreate(&p1));
    struct EG {
      cudaEvent_t a, b, c, d;
      double2* h;
      ~EG() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaEventDestroy(c);
        cudaEventDestroy(d);
        cudaFreeHost(h);
      }
    } eg{e0, e1, p0, p1, hh};
    double t_pre = 0.0;
    auto precond = [&](const double2* rr, double2* zz) {
      if (!M) {
        FMM_CUDA(cudaMemcpyAsync(zz, rr, sizeof(double2) * N, cudaMemcpyDeviceToDevice, s));
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
    using cd = std::complex<double>;
    FMM_CUDA(cudaEventRecord(e0, s));
    FMM_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * N, s));
    multidot(N, 1, nullptr, 0, b, part, nd, s);
    FMM_CUDA(cudaMemcpyAsync(hh, nd.ptr, sizeof(double2), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    const double nb = std::sqrt(hh[0].x);
    if (!std::isfinite(nb)) throw fmm::Error(FMM_ERR_NUMERIC, "fmm_gmres_solve: non-finite right-hand side");
    if (hist) hist[0] = 1.0;
    int it = 0;
    double rel = nb == 0.0 ? 0.0 : 1.0;
    if (nb > 0.0 && maxit > 0) {
      // Hessenberg columns (rotated), Givens rotations, the rotated right-hand side g
      std::vector<std::vector<cd>> H;
      std::vector<cd> cs, sn, g(maxit + 1, cd(0.0));
      g[0] = nb;
      scale_kernel<<<grid_for(N), 256, 0, s>>>(N, nullptr, 1.0 / nb, b, V);
      FMM_LAUNCHED("scale_kernel");
      for (int k = 0; k < maxit; ++k) {
        double2* vk = V.ptr + (int64_t)k * N;
        precond(vk, t);
        helm_stencil(n, kappa, t, w, s);
        // classical Gram-Schmidt, twice (one host read per Arnoldi step)
        multidot(N, k + 1, V, N, w, part, hd, s);
        combine_kernel<<<grid_for(N), 256, 0, s>>>(N, k + 1, V, N, hd, w, w);
        FMM_LAUNCHED("combine_kernel");
        multidot(N, k + 1, V, N, w, part, hd.ptr + (k + 1), s);
        combine_kernel<<<grid_for(N), 256, 0, s>>>(N, k + 1, V, N, hd.ptr + (k + 1), w, w);
        FMM_LAUNCHED("combine_kernel");
        multidot(N, 1, nullptr, 0, w, part, nd, s);
        FMM_CUDA(cudaMemcpyAsync(hh, hd.ptr, sizeof(double2) * 2 * (k + 1), cudaMemcpyDeviceToHost, s));
        FMM_CUDA(cudaMemcpyAsync(hh + 2 * (maxit + 1), nd.ptr, sizeof(double2), cudaMemcpyDeviceToHost, s));
        FMM_CUDA(cudaStreamSynchronize(s));
        std::vector<cd> col(k + 2);
        for (int j = 0; j <= k; ++j) col[j] = cd(hh[j].x, hh[j].y) + cd(hh[k + 1 + j].x, hh[k + 1 + j].y);
        const double hn = std::sqrt(hh[2 * (maxit + 1)].x);
        col[k + 1] = hn;
        for (const cd& c : col)
          if (!std::isfinite(c.real()) || !std::isfinite(c.imag()))
            throw fmm::Error(FMM_ERR_NUMERIC, "fmm_gmres_solve: non-finite Arnoldi coefficients");
        for (int j = 0; j < k; ++j) {  // previous rotations
          const cd tj = cs[j] * col[j] + sn[j] * col[j + 1];
          col[j + 1] = -std::conj(sn[j]) * col[j] + std::conj(cs[j]) * col[j + 1];
          col[j] = tj;
        }
        // new rotation [[c, s], [-conj(s), conj(c)]], c = conj(a) / rho, s = h / rho: (a, h) -> (rho, 0)
        const cd a = col[k];
        const double rho = std::sqrt(std::norm(a) + hn * hn);
        cs.push_back(rho > 0 ? std::conj(a) / rho : cd(1.0));
        sn.push_back(rho > 0 ? cd(hn / rho) : cd(0.0));
        col[k] = cs[k] * a + sn[k] * hn;
        col[k + 1] = 0.0;
        g[k + 1] = -std::conj(sn[k]) * g[k];
        g[k] = cs[k] * g[k];
        H.push_back(col);
        ++it;
        rel = std::abs(g[k + 1]) / nb;
        if (hist) hist[it] = rel;
        if (rel <= rtol || col[k] == 0.0 || hn == 0.0) break;
        scale_kernel<<<grid_for(N), 256, 0, s>>>(N, nd.ptr, 0.0, w, V.ptr + (int64_t)(k + 1) * N);
        FMM_LAUNCHED("scale_kernel");
      }
      // y = R^-1 g (back substitution), u = sum_j y_j V_j, x = M u
      const int m = it;
      std::vector<cd> y(m);
      for (int i = m - 1; i >= 0; --i) {
        cd sacc = g[i];
        for (int j = i + 1; j < m; ++j) sacc -= H[j][i] * y[j];
        y[i] = sacc / H[i][i];
      }
      for (int j = 0; j < m; ++j) hh[j] = make_double2(y[j].real(), y[j].imag());
      FMM_CUDA(cudaMemcpyAsync(hd.ptr, hh, sizeof(double2) * m, cudaMemcpyHostToDevice, s));
      combine_kernel<<<grid_for(N), 256, 0, s>>>(N, m, V, N, hd, nullptr, t);
      FMM_LAUNCHED("combine_kernel");
      if (M)
        precond(t, x);
      else
        FMM_CUDA(cudaMemcpyAsync(x, t.ptr, sizeof(double2) * N, cudaMemcpyDeviceToDevice, s));
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
