/*
 * include/fmm.h — C ABI of the B200-native 3D Laplace FMM mat-vec (libfmm.so).
 *
 * The operation (arXiv:1602.02244, Yokota/Ibeid/Keyes):
 *   phi_i = sum_{j : |x_i - x_j| > 0} q_j / |x_i - x_j|          (kernel 1/r, no 4*pi)
 *   grad_i = grad_{x_i} phi(x_i) = - sum_j q_j (x_i - x_j) / |x_i - x_j|^3
 * evaluated as the analytic, matrix-free H^2 mat-vec of the fast multipole
 * method: "a matrix-free H^2-matrix-vector product" (§1), whose
 * far field is "approximated with multipole/local expansions" over a
 * "hierarchically decomposed" domain, with interaction lists
 * from a "dual tree traversal along with the multipole acceptance criterion"
 * (§2.2). The direct operator (P2P) is the dense diagonal
 * block, the translation operators the off-diagonal blocks.
 * The paper times "the compression/precalculation and application of the
 * matrix-vector multiplication" separately (§4.1): hence the
 * split fmm_setup (precalculation: tree + lists) / fmm_matvec (application).
 * It asks for "a common interface between the hierarchical structure and
 * inner kernels" (§5): this header is that interface.
 *
 * Readings the paper leaves open (after SURVEY §8(c)):
 *   - "order p" = solid-harmonic degrees 0..p ((p+1)^2 real coefficients);
 *   - adaptive octree on 63-bit Morton keys (21 bits/axis), a cell splits iff
 *     it holds more than ncrit points and its level is < 21;
 *   - MAC: a cell pair (A,B) is translated by M2L iff theta^2 * D^2 > (H_A+H_B)^2,
 *     D = distance of the cell centres, H = half side (integer-exact), valid
 *     theta in (0, 1/sqrt(3)); split the larger cell, target on ties.
 *
 * Conventions for every call:
 *   - All array pointers are DEVICE pointers on ex->device unless the name ends
 *     in _host. Coordinates are [n][3] row-major doubles, charges / potentials
 *     [n] doubles, gradients [n][3] row-major doubles, all fp64, caller order.
 *   - The caller owns every buffer it passes; no caller pointer is retained
 *     after a call returns. The plan owns all internal device memory.
 *   - Work is enqueued on ex->stream (a cudaStream_t; NULL = legacy default).
 *     fmm_setup synchronises that stream (list sizes are data dependent);
 *     fmm_matvec and fmm_direct are stream ordered and return after enqueue
 *     (the caller synchronises before reading results); fmm_matvec_host is
 *     synchronous.
 *   - Results are in the caller's input order and are bitwise deterministic for
 *     identical inputs on the same device (no floating-point atomics).
 *   - Calls on one plan must be serialised. Tree, lists and tables are immutable
 *     after setup; expansion scratch is reused by every matvec.
 *   - Errors: every call returns an fmm_status; the library never aborts or
 *     exits. fmm_last_error() returns a thread-local message for the last
 *     non-OK status. After any status other than FMM_OK / FMM_ERR_USAGE /
 *     FMM_ERR_NUMERIC the plan is poisoned and only fmm_destroy is valid.
 */
#ifndef FMM_H
#define FMM_H
#include <stdint.h>

#if defined(__GNUC__)
#define FMM_API __attribute__((visibility("default")))
#else
#define FMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FMM_OK = 0,
  FMM_ERR_USAGE = 2,   /* bad argument: sizes, ranges, NULL, non-finite coordinate */
  FMM_ERR_NUMERIC = 3, /* non-finite charge or result */
  FMM_ERR_CUDA = 4,    /* CUDA launch / runtime error (plan poisoned) */
  FMM_ERR_OOM = 5,     /* device or host allocation failure (plan poisoned) */
  FMM_ERR_COMM = 6     /* multi-GPU exchange error (plan poisoned) */
} fmm_status;

typedef struct fmm_plan_s* fmm_plan; /* opaque */

/* Execution context. */
typedef struct {
  int device;     /* CUDA ordinal this process drives */
  void* stream;   /* cudaStream_t; NULL = legacy default stream */
  int rank;       /* 0 .. world_size-1 (multi-GPU: one process per GPU) */
  int world_size; /* 1 = single GPU */
  const void* nccl_id; /* a 128-byte ncclUniqueId, the same on every rank (rank 0 makes it with
                          fmm_nccl_unique_id and broadcasts it by any means), or NULL. Non-NULL:
                          "collective mode" — fmm_setup and fmm_matvec are COLLECTIVE over the
                          ranks and take and return each rank's own slice of the points /
                          charges / results (the library redistributes by Morton order and
                          moves the local-essential-tree exchange with NCCL on `stream`,
                          DESIGN.md §5); world_size 1 is allowed (a one-rank communicator: the
                          same code path). NULL with world_size > 1: the legacy mode below
                          (global points, caller-moved exchange, fmm_let_*). */
} fmm_exec;

/* Filled by fmm_stats. Times are CUDA-event milliseconds of the last call. */
enum {
  FMM_T_SORT = 0, FMM_T_TREE = 1, FMM_T_TRAVERSE = 2, FMM_T_SETUP_TOTAL = 3,
  FMM_T_UPWARD = 0, FMM_T_M2L = 1, FMM_T_NEAR = 2, FMM_T_DOWNWARD = 3, FMM_T_MATVEC_TOTAL = 4
};
typedef struct {
  int64_t n, n_cells, n_leaves, n_p2p_pairs, n_m2l_pairs, n_p2p_interactions;
  int64_t own_begin, own_end; /* this rank's target range in Morton order */
  int32_t p, ncrit, max_level, exponent; /* exponent e of the exact 2^-e normalisation */
  double theta;
  double t_setup_ms[8];  /* FMM_T_SORT .. FMM_T_SETUP_TOTAL */
  double t_matvec_ms[8]; /* FMM_T_UPWARD .. FMM_T_MATVEC_TOTAL (0 unless timing enabled) */
  int64_t bytes_device;  /* device memory owned by the plan */
  int m2l_variant;       /* M2L formulation in use: 1 matrix-free O(p^4) per pair, 2 dense class
                            operators on DMMA, 3 rotation-factored class operators on DMMA,
                            4 per-pair rotation on DFMA with one fixed operator (default,
                            2 <= p <= 12); 0 for a 2D (log-kernel) plan (complex series) */
  int near_mutual;       /* 1: potentials-only mat-vecs evaluate each unordered P2P leaf pair once
                            (single GPU, symmetric lists, leaves <= 64 particles; FMM_NEAR_MUTUAL=0
                            disables), 0: directed P2P */
  double m2l_flops_per_pair; /* flops per M2L pair of that formulation as executed (v4: the four
                                fixed-operator products, four z-rotations and the Hankel
                                translation; v3: the three block stages + the two azimuthal
                                rotations; v1/v2: 2(p+1)^4; 2D: 8(p+1)^2) */
  int64_t bytes_by[8];       /* bytes_device by category, FMM_B_* (the FMM side of PAPER.md
                                Fig 4, "strictly O(N) storage") */
  int64_t launches_total;    /* kernels launched by libfmm in this process so far (all plans,
                                setup included): differences count a region's launches */
} fmm_stats_t;
enum {
  FMM_B_PARTICLES = 0,  /* keys, permutation, positions + charges, host-call staging, mutual near-field sums */
  FMM_B_TREE = 1,       /* cell arrays, leaf index */
  FMM_B_LISTS = 2,      /* P2P and M2L interaction lists (+ the mutual near field's task lists) */
  FMM_B_EXPANSIONS = 3, /* M and L, plus the M2L kernels' scaled multipole rows */
  FMM_B_OPERATORS = 4,  /* precomputed translation operators: M2L class tables, M2M/L2L */
  FMM_B_SCHEDULE = 5,   /* M2L column / chunk / tile schedules and descriptors */
  FMM_B_LET = 6,        /* multi-GPU exchange lists and buffers */
  FMM_B_OTHER = 7
};

/*
 * fmm_setup — precalculation: bounding cube, Morton keys,
 * device radix sort, adaptive octree, dual tree traversal -> P2P and M2L lists.
 *   out   : receives the new plan (NULL on error)
 *   xyz   : device [n][3] fp64 point coordinates (copied; may be freed after return)
 *   n     : number of points, >= 1. Collective mode (nccl_id set): this
 *           rank's slice, >= 0 (the global count, the sum over ranks, >= 1); the plan is the
 *           single global tree and lists on every rank, the rank's targets a contiguous
 *           Morton range cut at leaf boundaries by estimated work. Legacy multi-GPU mode
 *           (nccl_id NULL): the GLOBAL point set on every rank.
 *   p     : expansion order, 0 <= p <= 16
 *   ncrit : maximum leaf population, >= 1
 *   theta : MAC parameter, 0 < theta < 1/sqrt(3)
 *   ex    : execution context (non-NULL)
 * Errors: FMM_ERR_USAGE for any argument outside the ranges above or a
 * non-finite coordinate; FMM_ERR_OOM; FMM_ERR_CUDA.
 */
FMM_API fmm_status fmm_setup(fmm_plan* out, const double* xyz, int64_t n, int p, int ncrit, double theta,
                     const fmm_exec* ex);

/*
 * fmm_setup_2d — NEXT-3: the same precalculation for PLANAR points and the 2D Laplace (log)
 * kernel, the 2D half of the paper's §4.1 experiment ("2D and 3D Laplace equation on uniform
 * lattices"). A plan made here makes fmm_matvec / fmm_matvec_host compute
 *   phi_i = - sum_{j : |x_i - x_j| > 0} q_j log |x_i - x_j|,   grad_i = grad_{x_i} phi_i
 * with grad written as [n][3] (third component 0). The tree and lists are those of the points
 * (x, y, 0) (the octree of planar points is a quadtree); expansions are complex Laurent /
 * Taylor series of order p (R40-R44).
 *   xy : device [n][2] fp64 coordinates (copied). Other arguments as fmm_setup; single GPU
 *        only (ex->world_size == 1, else FMM_ERR_USAGE).
 */
FMM_API fmm_status fmm_setup_2d(fmm_plan* out, const double* xy, int64_t n, int p, int ncrit, double theta,
                                const fmm_exec* ex);

/*
 * fmm_matvec — application: phi (+ grad) for charges q, on ex->stream.
 *   q    : device [n] fp64 charges, caller order
 *   n    : must equal the setup n (FMM_ERR_USAGE otherwise)
 *   phi  : device [n] fp64 output, caller order
 *   grad : device [n][3] fp64 output or NULL
 * Collective mode (nccl_id set): q, phi, grad are THIS RANK's slices (n =
 * the rank's setup n); the call is collective over the ranks, stream ordered, no host sync
 * (exchange sizes are fixed at setup): the charges go to their owners and halo ranks, the
 * boundary multipoles to the ranks whose targets need them, the results back to the caller
 * slices, all with NCCL on the plan's stream.
 * Legacy multi-GPU mode (nccl_id NULL): q is global and only the entries of targets owned by
 * this rank (Morton range [own_begin, own_end) of fmm_stats) are written, the others set to 0,
 * so a sum over ranks (reduce-scatter) assembles the global result exactly.
 * Non-finite charges give FMM_ERR_NUMERIC, detected on the device and reported
 * by the NEXT fmm_matvec / fmm_sync call on the plan (the call is stream ordered).
 */
FMM_API fmm_status fmm_matvec(fmm_plan plan, const double* q, int64_t n, double* phi, double* grad);

/*
 * fmm_matvec_host — the same with HOST buffers (pinned or pageable): copies q
 * host->device, runs fmm_matvec, copies phi (+grad) device->host, synchronises.
 * This is the end-to-end entry point a host application calls.
 */
FMM_API fmm_status fmm_matvec_host(fmm_plan plan, const double* q_host, int64_t n, double* phi_host,
                           double* grad_host);

/* fmm_sync — synchronise the plan's stream and report deferred device errors. */
FMM_API fmm_status fmm_sync(fmm_plan plan);

/*
 * fmm_direct — O(n_src * n_tgt) direct sum for checking (north_star):
 *   phi_t = sum_{s : r > 0} q_s / r_ts, grad_t = -sum_s q_s (x_t - x_s) / r_ts^3.
 * All pointers device, [n][3] / [n] fp64; grad may be NULL; n_src, n_tgt >= 0.
 * Stream ordered on ex->stream.
 */
FMM_API fmm_status fmm_direct(const double* src_xyz, const double* q, int64_t n_src, const double* tgt_xyz,
                      int64_t n_tgt, double* phi, double* grad, const fmm_exec* ex);

/* fmm_stats — counts and timings of the plan (host struct). */
FMM_API fmm_status fmm_stats(fmm_plan plan, fmm_stats_t* out);

/* fmm_set_timing — enable (1) / disable (0) per-stage CUDA-event timing in fmm_matvec. */
FMM_API fmm_status fmm_set_timing(fmm_plan plan, int enable);

/*
 * fmm_export — copy an internal array of the plan to a HOST buffer, for stage
 * tests against the oracle. `what` selects the array; `capacity` is the size of
 * `dst` in elements; *count receives the element count (call with dst = NULL to
 * query it). Arrays (element type):
 *   FMM_X_KEYS     uint64  [n]          sorted Morton keys
 *   FMM_X_PERM     uint32  [n]          sorted position -> input index
 *   FMM_X_LEVEL    int32   [ncells]     cells in breadth-first (level, Morton) order
 *   FMM_X_ANCHOR   int32   [ncells][3]
 *   FMM_X_BEGIN    int32   [ncells]     particle range [begin, end) in sorted order
 *   FMM_X_END      int32   [ncells]
 *   FMM_X_CHILD    int32   [ncells]     first child, -1 for a leaf
 *   FMM_X_NCHILD   int32   [ncells]
 *   FMM_X_PARENT   int32   [ncells]     -1 for the root
 *   FMM_X_CENTER   double  [ncells][3]  centres in the 2^-e normalised frame
 *   FMM_X_P2P      int32   [n_p2p][2]   (target leaf, source leaf), grouped by target
 *   FMM_X_M2L      int32   [n_m2l][2]   (target cell, source cell), grouped by target
 *   FMM_X_M        double  [ncells][(p+1)(p+2)/2][2]  multipoles of the last matvec
 *   FMM_X_L        double  [ncells][(p+1)(p+2)/2][2]  local expansions of the last matvec
 *   FMM_X_GEOM     double  [5]          lo_x, lo_y, lo_z, S, scale (normalised frame)
 * Expansions: complex coefficients for m >= 0, index n(n+1)/2 + m, normalised frame.
 */
typedef enum {
  FMM_X_KEYS = 0, FMM_X_PERM, FMM_X_LEVEL, FMM_X_ANCHOR, FMM_X_BEGIN, FMM_X_END, FMM_X_CHILD,
  FMM_X_NCHILD, FMM_X_PARENT, FMM_X_CENTER, FMM_X_P2P, FMM_X_M2L, FMM_X_M, FMM_X_L, FMM_X_GEOM
} fmm_array;
FMM_API fmm_status fmm_export(fmm_plan plan, int what, void* dst, int64_t capacity, int64_t* count);

/*
 * Multi-GPU mat-vec with a local-essential-tree exchange (world_size > 1;
 * north_star "Morton-ordered domain decomposition, with a local-essential-tree
 * exchange (boundary multipoles plus halo particles) over NCCL/NVLink";
 * DESIGN.md §5). Every rank calls fmm_setup with the GLOBAL points (same tree
 * and lists on every rank) and owns the Morton particle range
 * [rank_begin[r], rank_begin[r+1]) cut at leaf boundaries. The library builds
 * the exchange lists and packs/unpacks device buffers; the CALLER moves them
 * with its collectives (torch.distributed over NCCL), in this order:
 *   fmm_let_pack_q   (q_local [caller slice]      -> q_send)       all-to-all-v (Q)
 *   fmm_let_upward   (q_recv                      -> shared_send, m_send)
 *                    all-gather of shared_send (SHARED), all-to-all-v (M)
 *   fmm_let_finish   (shared_recv, m_recv         -> phi_send [, grad_send])
 *                    all-to-all-v (PHI)
 *   fmm_let_unpack   (phi_recv [, grad_recv]      -> phi_local [, grad_local])
 * Buffer sizes (doubles) from fmm_let_counts, per peer rank, in rank order:
 *   Q: counts; M: counts x 2 nc (nc = (p+1)(p+2)/2 complex coefficients);
 *   SHARED: count x 2 nc (send), world x count x 2 nc (receive, rank-major);
 *   PHI: counts (x 3 for gradients).
 * All pointers are device buffers on ex->device, stream ordered. The upward
 * pass runs only on the owned particles; straddling cells' partial multipoles
 * are summed in rank order, so results are deterministic and equal the
 * single-GPU mat-vec up to summation order.
 */
typedef enum {
  FMM_LET_Q_SEND = 0, FMM_LET_Q_RECV, FMM_LET_M_SEND, FMM_LET_M_RECV, FMM_LET_PHI_SEND, FMM_LET_PHI_RECV,
  FMM_LET_SHARED,     /* [1]: number of shared (straddling) cells */
  FMM_LET_RANK_BEGIN, /* [world + 1]: owner ranges */
  /* index lists (fmm_let_lists_host only) */
  FMM_LET_Q_SEND_ROWS, FMM_LET_Q_RECV_POS, FMM_LET_SHARED_CELLS, FMM_LET_M_SEND_CELLS, FMM_LET_M_RECV_CELLS,
  FMM_LET_PHI_SEND_IDX, FMM_LET_PHI_RECV_ROWS
} fmm_let_what;
/* caller_counts_host: [world] rows of the caller slice of every rank (sum = n). */
FMM_API fmm_status fmm_let_setup(fmm_plan plan, const int64_t* caller_counts_host);
/* counts_host: [world] (SHARED: [1], RANK_BEGIN: [world + 1]) host int64 */
FMM_API fmm_status fmm_let_counts(fmm_plan plan, int what, int64_t* counts_host);
FMM_API fmm_status fmm_let_pack_q(fmm_plan plan, const double* q_local, double* q_send);
FMM_API fmm_status fmm_let_upward(fmm_plan plan, const double* q_recv, double* shared_send, double* m_send);
FMM_API fmm_status fmm_let_finish(fmm_plan plan, const double* shared_recv, const double* m_recv, double* phi_send,
                                  double* grad_send);
FMM_API fmm_status fmm_let_unpack(fmm_plan plan, const double* phi_recv, const double* grad_recv, double* phi_local,
                                  double* grad_local);
/*
 * fmm_let_lists_host — the exchange lists of rank `me` from HOST copies of a tree
 * (no device work; the same host code fmm_let_setup runs). what = one of
 * fmm_let_what; dst NULL queries *count. Arrays as in fmm_export; caller_off
 * [world + 1] prefix sums of the caller counts; leaves sorted by first particle;
 * p the expansion order (it weights the owner cuts).
 */
FMM_API fmm_status fmm_let_lists_host(int64_t n, int world, int me, int p, const int64_t* caller_off, const uint32_t* perm,
                                      int64_t ncells, const int32_t* cbeg, const int32_t* cend, int64_t nleaves,
                                      const int32_t* leaves, int64_t np2p, const int32_t* p2p_tgt,
                                      const int32_t* p2p_src, int64_t nm2l, const int32_t* m2l_tgt,
                                      const int32_t* m2l_src, int what, int64_t* dst, int64_t capacity,
                                      int64_t* count);

/*
 * fmm_nccl_unique_id — a new ncclUniqueId (128 bytes written to out, host memory) for the
 * collective mode; call on ONE rank and send the bytes to the others. Loads NCCL
 * (libnccl.so.2) on first use; FMM_ERR_COMM if it is unavailable.
 */
FMM_API fmm_status fmm_nccl_unique_id(void* out);

/* fmm_destroy — free the plan (NULL is a no-op). */
FMM_API void fmm_destroy(fmm_plan plan);

/* fmm_last_error — thread-local message for the last non-OK status ("" if none). */
FMM_API const char* fmm_last_error(void);

/* fmm_version — library version string. */
FMM_API const char* fmm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FMM_H */
