/*
 * include/fmm_pde.h — NEXT-2: the FMM mat-vec of fmm.h used as a
 * low-accuracy preconditioner inside a Krylov solve (libfmm.so, same conventions and
 * error handling as fmm.h: device pointers, caller-owned buffers, fmm_last_error()).
 *
 * The paper: "If we are to use the FMM as a matrix-free O(N) preconditioner [...] for
 * the Laplace equation [...] on a 3D cubic lattice [-1,1]^3 [...] we impose Dirichlet
 * boundary conditions at the faces of the domain. The preconditioners are used inside a
 * Krylov subspace solver." (§4.2; Fig 5 at h = 2^-5);
 * "viewing these methods as a preconditioner instead of a direct solver significantly
 * reduces the accuracy requirements"; the FMM preconditioner's
 * convergence rate is independent of the problem size.
 *
 * Readings (R30-R36; the paper prints no formulas for this experiment):
 *   lattice   the n^3 interior nodes x = -1 + (i+1) h, h = 2 / (n+1) (h = 2^-5 <=> n = 63),
 *             vectors indexed i + n (j + n k) (x fastest);
 *   operator  A = -Delta_h, 7-point stencil, zero Dirichlet ghost values;
 *   M r       u_v = h^3 G * r (FMM over the lattice, G = 1/(4 pi r), own-cell integral
 *             h^2 (3 ln(2+sqrt 3) - pi/2) / (4 pi) on the diagonal), then single-layer
 *             densities on square face panels of side a = stride h solving S sigma = -u_v|faces
 *             (S_ij = a^2 G(y_i, y_j), S_ii = a ln(1+sqrt 2)/pi; S^-1 formed once at setup),
 *             M r = u_v + a^2 G * sigma at the lattice nodes (FMM again);
 *   Krylov    flexible preconditioned CG (Polak-Ribiere beta), x0 = 0,
 *             stop when ||b - A x|| / ||b|| <= rtol.
 */
#ifndef FMM_PDE_H
#define FMM_PDE_H
#include "fmm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* out = A u on the n^3 lattice (n >= 1). u, out: device [n^3] doubles, distinct buffers.
 * Stream ordered on `stream`. USAGE for n < 1 or n^3 >= 2^31 or NULL pointers. */
FMM_API fmm_status fmm_stencil_apply(int n, const double* u, double* out, void* stream);

typedef struct fmm_precond_s* fmm_precond; /* opaque */

/* Precalculation of M: lattice + face-panel points, one FMM plan over both (order p, ncrit,
 * theta: the accuracy knob "epsilon" of Fig 5), the boundary matrix S and its inverse.
 *   n            lattice nodes per axis (>= 1)
 *   face_stride  panel stride s >= 1 in lattice spacings (6 ceil(n/s)^2 panels)
 *   boundary     0 = volume potential only (no boundary correction), 1 = full M
 * Synchronises ex->stream. Errors: USAGE (bad sizes / FMM arguments, see fmm_setup),
 * NUMERIC (the inverse of S did not converge), CUDA, OOM. */
FMM_API fmm_status fmm_precond_setup(fmm_precond* out, int n, int face_stride, int p, int ncrit, double theta,
                                     int boundary, const fmm_exec* ex);

/* z = M r. r, z: device [n^3] doubles, distinct buffers. Stream ordered (ex->stream of setup). */
FMM_API fmm_status fmm_precond_apply(fmm_precond P, const double* r, double* z);

/* Panel count and the device memory owned by M (bytes). Either pointer may be NULL. */
FMM_API fmm_status fmm_precond_info(fmm_precond P, int64_t* n_panels, int64_t* bytes);

FMM_API void fmm_precond_destroy(fmm_precond P);

typedef struct {
  int32_t iterations;  /* Krylov iterations performed */
  int32_t converged;   /* 1 if relres <= rtol */
  double relres;       /* final ||b - A x|| / ||b|| (recurrence residual) */
  double t_total_ms;   /* CUDA-event time of the whole solve */
  double t_precond_ms; /* of which inside M applications */
} fmm_pcg_info;

/* Solve A x = b by flexible PCG with M (NULL = identity). b, x: device [n^3]; hist: host
 * [maxit + 1] relative residuals (history[0] = 1) or NULL; info may be NULL. Synchronous
 * (reads one scalar per dot product). M must have been set up for the same n.
 * Errors: USAGE (n, rtol <= 0, maxit < 0, size mismatch with M), NUMERIC (breakdown:
 * p^T A p <= 0 or non-finite), CUDA. */
FMM_API fmm_status fmm_pcg_solve(int n, const double* b, double* x, fmm_precond M, double rtol, int maxit,
                                 double* hist, fmm_pcg_info* info, void* stream);

/*
 * NEXT-4 solve: the Helmholtz equation -Delta u - kappa^2 u = f on the same
 * lattice with Dirichlet faces, the Helmholtz FMM of include/fmm_helmholtz.h as the preconditioner
 * inside GMRES ("the Laplace equation and Helmholtz equation on a 3D cubic lattice [-1,1]^3 [...]
 * The preconditioners are used inside a Krylov subspace solver"; Fig 6, kappa = 7
 * at h = 2^-5). Readings (R56-R60), those above with:
 *   operator  A = -Delta_h - kappa^2 I (real symmetric, indefinite for kappa = 7);
 *   G         exp(i kappa r) / (4 pi r); own-cell integral c_self = h^2 C_cube / (4 pi)
 *             + i kappa h^3 / (4 pi), own-panel S_ii = a C_panel / (4 pi) + i kappa a^2 / (4 pi);
 *             S complex symmetric, S^-1 by complex Newton-Schulz (cuBLAS ZGEMM) at setup;
 *   Krylov    GMRES, right preconditioned (x = M u), x0 = 0, no restart, Arnoldi by classical
 *             Gram-Schmidt with one re-orthogonalisation, Givens rotations; stop when the residual
 *             estimate |g_{k+1}| / ||b|| <= rtol.
 * Complex vectors are interleaved (re, im) doubles: [n^3][2] (a torch complex128 tensor).
 */
typedef struct fmm_hprecond_s* fmm_hprecond; /* opaque */

/* out = (-Delta_h - kappa^2) u on the n^3 lattice; u, out: device [n^3][2], distinct. Stream
 * ordered on `stream`. USAGE for n < 1, n^3 >= 2^30, non-finite kappa, NULL/aliased pointers. */
FMM_API fmm_status fmm_helmholtz_stencil_apply(int n, double kappa, const double* u, double* out, void* stream);

/* Precalculation of the Helmholtz M (as fmm_precond_setup; kappa > 0 finite; p <= 10 as
 * fmm_setup_helmholtz). Synchronises ex->stream. Errors: USAGE, NUMERIC (Newton-Schulz did not
 * converge: S singular or too ill-conditioned, e.g. kappa^2 at an interior Dirichlet eigenvalue),
 * CUDA, OOM. */
FMM_API fmm_status fmm_hprecond_setup(fmm_hprecond* out, int n, int face_stride, int p, int ncrit, double theta,
                                      double kappa, int boundary, const fmm_exec* ex);

/* z = M r; r, z: device [n^3][2] complex, distinct. Stream ordered (ex->stream of setup). */
FMM_API fmm_status fmm_hprecond_apply(fmm_hprecond P, const double* r, double* z);

/* Panel count and the device memory owned by M (bytes). Either pointer may be NULL. */
FMM_API fmm_status fmm_hprecond_info(fmm_hprecond P, int64_t* n_panels, int64_t* bytes);

FMM_API void fmm_hprecond_destroy(fmm_hprecond P);

/* Solve (-Delta_h - kappa^2) x = b by GMRES with M (NULL = identity). b, x: device [n^3][2]
 * complex; hist: host [maxit + 1] residual estimates (history[0] = 1) or NULL; info may be NULL
 * (t_precond_ms: time inside M). Synchronous (one host read per Gram-Schmidt pass). Device
 * memory: (maxit + 1) n^3 complex basis vectors. M must have been set up for the same n and
 * kappa. Errors: USAGE (n, kappa, rtol <= 0, maxit < 0, mismatch with M), NUMERIC (non-finite
 * values), CUDA, OOM. */
FMM_API fmm_status fmm_gmres_solve(int n, double kappa, const double* b, double* x, fmm_hprecond M, double rtol,
                                   int maxit, double* hist, fmm_pcg_info* info, void* stream);

#ifdef __cplusplus
}
#endif
#endif
