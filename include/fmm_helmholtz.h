/*
 * include/fmm_helmholtz.h — NEXT-4: the FMM mat-vec for the 3D Helmholtz kernel,
 * the paper's second kernel ("a comparison between FMM and HSS for Laplace and Helmholtz
 * kernels", §1; the Helmholtz equation on a [-1,1]^3 lattice with wave number
 * kappa = 7, §4.2):
 *
 *   phi_i = sum_{j : |x_i - x_j| > 0} q_j exp(i kappa |x_i - x_j|) / |x_i - x_j|
 *
 * complex charges and potentials (interleaved re, im doubles), fp64. The plan's tree and
 * interaction lists are the Laplace plan's (same MAC, split rule, ncrit: fmm_setup's reading);
 * the expansions are spherical-wave series of order p (degrees 0..p, all orders, (p+1)^2 complex
 * coefficients): multipole sum M_n^m h_n(kappa r) Y_n^m, local sum L_n^m j_n(kappa r) Y_n^m, with
 * the (S|S), (S|R), (R|R) translation operators of the addition theorem (R50-R55).
 * The operators depend on the level (kappa times the cell size), so they are tabulated per level
 * (M2M, L2L: 8 octant offsets) and per M2L class (target level, level difference, integer offset)
 * at setup. Low frequency: meant for kappa times the root cube side up to a few tens.
 * Same conventions as include/fmm.h (device pointers on ex->device, caller order, stream ordered,
 * fmm_status codes, fmm_last_error, fmm_destroy, fmm_stats); single GPU (ex->world_size == 1).
 */
#ifndef FMM_HELMHOLTZ_H
#define FMM_HELMHOLTZ_H
#include "fmm.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * fmm_setup_helmholtz — precalculation: tree and lists (as fmm_setup) plus the level and class
 * translation tables for wave number kappa.
 *   xyz   : device [n][3] fp64 (copied)      n : >= 1
 *   p     : expansion order, 0 <= p <= 10     ncrit >= 1, 0 < theta < 1/sqrt(3)
 *   kappa : wave number, > 0 and finite
 * Errors: FMM_ERR_USAGE (ranges, NULL, non-finite coordinate, world_size != 1), FMM_ERR_OOM,
 * FMM_ERR_CUDA.
 */
FMM_API fmm_status fmm_setup_helmholtz(fmm_plan* out, const double* xyz, int64_t n, int p, int ncrit, double theta,
                                       double kappa, const fmm_exec* ex);

/*
 * fmm_matvec_helmholtz — phi = G q on the plan's stream.
 *   q   : device [n][2] fp64 (re, im) complex charges, caller order
 *   phi : device [n][2] fp64 (re, im) complex potentials, caller order
 * n must equal the setup n. FMM_ERR_USAGE for a plan not made by fmm_setup_helmholtz.
 */
FMM_API fmm_status fmm_matvec_helmholtz(fmm_plan plan, const double* q, int64_t n, double* phi);

/*
 * fmm_direct_helmholtz — O(n_src n_tgt) direct sum for checking: phi_t = sum_{s : r > 0}
 * q_s exp(i kappa r_ts) / r_ts. src/tgt [n][3], q/phi [n][2] (re, im), device, stream ordered.
 */
FMM_API fmm_status fmm_direct_helmholtz(const double* src_xyz, const double* q, int64_t n_src, const double* tgt_xyz,
                                        int64_t n_tgt, double kappa, double* phi, const fmm_exec* ex);

#ifdef __cplusplus
}
#endif
#endif /* FMM_HELMHOLTZ_H */
