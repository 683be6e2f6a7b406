/*
 * oracle/fmm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, independent CPU implementation of the 3D Laplace FMM mat-vec
 * (arXiv:1602.02244, Yokota/Ibeid/Keyes) used as the parity oracle for the
 * CUDA path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product
 * path (paper_1602_02244_b200/) never links, imports or calls it.
 *
 * Conventions: SURVEY.md §8(c) and DESIGN.md "Readings". Kernel 1/r (no 4π),
 * "order p" = degrees 0..p, Condon–Shortley solid harmonics, integer MAC,
 * split-the-larger traversal. All pointers are HOST pointers.
 *
 * Coefficient layout: complex, m >= 0 only, index n(n+1)/2 + m,
 * (p+1)(p+2)/2 complex doubles per expansion (interleaved re, im).
 */
#ifndef FMM_ORACLE_H
#define FMM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status: 0 ok, 2 usage error, 3 numeric error, 5 out of memory */

/* O(N_s N_t) direct sum, long-double accumulation. grad nullable. */
int oracle_direct(const double* src_xyz, const double* q, int64_t n_src,
                  const double* tgt_xyz, int64_t n_tgt,
                  double* phi, double* grad, int nthreads);

/* Solid harmonics R_n^m(x,y,z), I_n^m(x,y,z), n<=p, m>=0 (c.1). out: (p+1)(p+2)/2 complex. */
void oracle_harmonics_R(double x, double y, double z, int p, double* out);
void oracle_harmonics_I(double x, double y, double z, int p, double* out);

/* Single operators on one expansion (c.1), for pins. Outputs accumulate (+=). */
void oracle_p2m(const double* xyz, const double* q, int64_t n, const double* c, int p, double* M);
void oracle_m2m(const double* Mc, const double* c_child, const double* c_parent, int p, double* Mp);
void oracle_m2l(const double* MB, const double* cB, const double* cA, int p, double* LA);
void oracle_l2l(const double* Lp, const double* c_parent, const double* c_child, int p, double* Lc);
void oracle_l2p(const double* L, const double* c, const double* x, int p, double* phi, double* grad3);
void oracle_m2p(const double* M, const double* c, const double* x, int p, double* phi);

/* Plan: A1–A7 (validate, root cube, quantize, Morton, sort, tree, traversal). */
typedef struct oracle_plan_s* oracle_plan;
int  oracle_plan_new(oracle_plan* out, const double* xyz, int64_t n, int p, int ncrit, double theta);
void oracle_plan_free(oracle_plan plan);

enum {
  ORACLE_INFO_N = 0, ORACLE_INFO_NCELLS = 1, ORACLE_INFO_NLEAVES = 2, ORACLE_INFO_NP2P = 3,
  ORACLE_INFO_NM2L = 4, ORACLE_INFO_EXP = 5, ORACLE_INFO_MAXLEVEL = 6, ORACLE_INFO_P = 7,
  ORACLE_INFO_NP2P_INTERACTIONS = 8
};
int64_t oracle_plan_info(oracle_plan plan, int which);
/* root cube after the exact 2^-e normalisation: lo[3], S, scale */
void oracle_plan_geometry(oracle_plan plan, double* lo3, double* S, double* scale);
/* sorted keys [n], perm [n] (sorted position -> input index) */
void oracle_plan_keys(oracle_plan plan, uint64_t* keys, int64_t* perm);
/* cells in BFS (level, Morton) order; any pointer may be NULL */
void oracle_plan_cells(oracle_plan plan, int32_t* level, int32_t* anchor3, int64_t* begin,
                       int64_t* end, int64_t* child_first, int32_t* nchild, int64_t* parent,
                       double* center3);
/* lists in emission (recursive DFS) order: pairs [n][2] = (target cell, source cell) */
void oracle_plan_lists(oracle_plan plan, int64_t* p2p, int64_t* m2l);

/* A8–A15. targets == NULL: all N outputs in input order. Otherwise the sampled-target
 * mode A15: outputs for targets[0..n_tgt) (input indices) in that order. grad nullable. */
int oracle_plan_eval(oracle_plan plan, const double* q, const int64_t* targets, int64_t n_tgt,
                     double* phi, double* grad, int nthreads);
/* after a full (targets == NULL) eval: M and L of every cell, [ncells][(p+1)(p+2)/2] complex,
 * in the normalised (2^-e scaled) frame. */
void oracle_plan_expansions(oracle_plan plan, double* M, double* L);

#ifdef __cplusplus
}
#endif
#endif
