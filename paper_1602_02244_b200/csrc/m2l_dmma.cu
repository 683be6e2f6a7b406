// m2l_dmma.cu — S9 M2L v2: precomputed translation-invariant operators applied
// as dense FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) contractions.
//
// Paper: "The translation operators can be stored as matrices that operate on
// the vector of expansion coefficients [...] BLAS can be used";
// "Precomputing these translation matrices and storing them is a typical
// optimization"; "translation operators for boxes with the
// same relative positioning are identical" -> O(1) storage per level
// (PAPER.md:199-206); "making use of the translational invariance and
// rotational symmetry of the interaction list one can reduce the amount of
// storage even further [...] blocking techniques for better cache
// utilization". North_star (4): DMMA only where the
// translations are cast as dense precomputed-operator contractions.
//
// Formulation (DESIGN.md §2 K10):
//  * scaled coefficients M~_n^m = M_n^m / h_B^n, L~_j^k = L_j^k h_A^{j+1} make
//    the operator depend only on the class (dl = level_A - level_B, integer
//    offset delta in units of the finer half side):
//      L~_j^k += sum (-1)^n (h_B/h_f)^n (h_A/h_f)^{j+1} I_{j+n}^{k+m}(delta) M~_n^m
//  * the 16 orthogonal maps G = flips(x,y,z) o swap(x,y) act on solid-harmonic
//    coefficients as signed re/im permutations, so T(G delta0) = D^L_G T(delta0)
//    (D^M_G)^{-1}: only canonical offsets delta0 = (min(|dx|,|dy|),
//    max(|dx|,|dy|), |dz|) get an operator (C3: 62 classes, ~1 MB);
//  * real basis of (p+1)^2 components: (n,0) -> n^2, (n,m,re) -> n^2+2m-1,
//    (n,m,im) -> n^2+2m;
//  * work: one CTA per tile of T target cells, accumulators in shared memory;
//    the tile's pairs sorted by (class, target, g) form runs; each run chunk of
//    <= NC columns is one GEMM Y = T~ X on DMMA (operator fragments streamed
//    from L2, X gathered with the D^M inverse applied), Y staged in shared
//    memory and added to the accumulators by one thread per (row, slot
//    parity) in column order: deterministic, no atomics.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "harmonics.cuh"
#include "m2l_common.cuh"
#include "plan.h"

namespace fmm {
namespace m2l {
std::vector<int32_t> build_symtab(int p);
}
void m2l_rot_launch(fmm_plan_s& P, const m2l::M2LArgs& a);
void m2l_rot_mtilde(fmm_plan_s& P);
namespace {
using namespace m2l;

constexpr int kNC = 64;  // max columns per chunk (8 n-tiles of 8)

// ------------------------------------------------------------- symmetry tables (host)
// A 2x2 signed permutation acting on (re, im).
struct M2 {
  int a, b, c, d;  // [[a, b], [c, d]]
};
M2 mul(M2 x, M2 y) {
  return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}
M2 phase(int e) {  // multiply by i^e
  e &= 3;
  const int c = e == 0 ? 1 : (e == 2 ? -1 : 0), s = e == 1 ? 1 : (e == 3 ? -1 : 0);
  return {c, -s, s, c};
}
const M2 kConj = {1, 0, 0, -1};
const M2 kId = {1, 0, 0, 1};

// coefficient map of one elementary orthogonal map on (n, m) (DESIGN.md §2 K10):
// op 0 = swap(x,y): multipole (-i)^m conj, local i^m conj; 1 = flip x: (-1)^m conj;
// 2 = flip y: conj; 3 = flip z: (-1)^{n+m}.
M2 elementary(int op, int n, int m, bool local) {
  switch (op) {
    case 0: return mul(phase(local ? m : 3 * m), kConj);
    case 1: return mul(phase(2 * m), kConj);
    case 2: return kConj;
    default: return phase(2 * (n + m));
  }
}

// D_G for g = sw | sx<<1 | sy<<2 | sz<<3, G = Fz^sz Fy^sy Fx^sx P^sw (P first)
M2 dmap(int g, int n, int m, bool local) {
  M2 D = kId;
  if (g & 1) D = mul(elementary(0, n, m, local), D);
  if (g & 2) D = mul(elementary(1, n, m, local), D);
  if (g & 4) D = mul(elementary(2, n, m, local), D);
  if (g & 8) D = mul(elementary(3, n, m, local), D);
  return D;
}

// ------------------------------------------------------------- setup kernels
__device__ __forceinline__ void pair_class(int A, int B, const int32_t* __restrict__ level,
                                           const int32_t* __restrict__ anchor, uint64_t& key, int& g) {
  const int la = level[A], lb = level[B];
  const int lf = max(la, lb);
  int64_t d[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int64_t ca = (2 * (int64_t)anchor[3 * A + k] + 1) << (kMaxLevel - la);
    const int64_t cb = (2 * (int64_t)anchor[3 * B + k] + 1) << (kMaxLevel - lb);
    d[k] = (cb - ca) >> (kMaxLevel - lf);  // exact: both are multiples of the finer half side
  }
  const int64_t ax = d[0] < 0 ? -d[0] : d[0], ay = d[1] < 0 ? -d[1] : d[1], az = d[2] < 0 ? -d[2] : d[2];
  const int sw = ax > ay;
  const uint64_t x0 = sw ? ay : ax, y0 = sw ? ax : ay;
  g = sw | ((d[0] < 0) << 1) | ((d[1] < 0) << 2) | ((d[2] < 0) << 3);
  // dl + 32 (6 bits) | x0 | y0 | z0 (19 bits each); offsets >= 2^19 are flagged by an all-ones key
  const uint64_t lim = (1ull << 19) - 1;
  key = (x0 > lim || y0 > lim || (uint64_t)az > lim)
            ? ~0ull >> 1
            : ((uint64_t)(la - lb + 32) << 57) | (x0 << 38) | (y0 << 19) | (uint64_t)az;
}

__global__ void class_key_kernel(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src, int64_t n,
                                 const int32_t* __restrict__ level, const int32_t* __restrict__ anchor,
                                 uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t key;
  int g;
  pair_class(tgt[i], src[i], level, anchor, key, g);
  keys[i] = key;
  idx[i] = (uint32_t)i;
}

__global__ void diff_flag_kernel(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// class id of every pair (scatter back through the sort permutation) + unique key list
__global__ void class_assign_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                    const int32_t* __restrict__ flag, const int64_t* __restrict__ off, int64_t n,
                                    int32_t* __restrict__ pair_class_id, uint64_t* __restrict__ class_keys) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t c = off[i] + flag[i] - 1;  // inclusive scan - 1
  pair_class_id[idx[i]] = (int32_t)c;
  if (flag[i]) class_keys[c] = keys[i];
}

// Operator of one canonical class in DMMA A-fragment order:
// ops[((cls * nmt + mt) * nks + ks) * 32 + lane] = T~[8 mt + lane/4][4 ks + lane%4].
__global__ void build_ops_kernel(const uint64_t* __restrict__ class_keys, int p, int nmt, int nks,
                                 double* __restrict__ ops) {
  extern __shared__ double2 shI[];  // I_n^m(delta0), n <= 2p
  const int cls = blockIdx.x;
  const uint64_t key = class_keys[cls];
  const int dl = (int)((key >> 57) & 0x3f) - 32;
  const double x0 = (double)((key >> 38) & 0x7ffff), y0 = (double)((key >> 19) & 0x7ffff),
               z0 = (double)(key & 0x7ffff);
  irregular_harmonics_par(x0, y0, z0, 2 * p, shI, threadIdx.x, blockDim.x);
  __syncthreads();
  const double fA = dl < 0 ? ldexp(1.0, -dl) : 1.0;  // h_A / h_f
  const double fB = dl > 0 ? ldexp(1.0, dl) : 1.0;   // h_B / h_f
  const int NR = real_count(p);
  const int64_t total = (int64_t)nmt * nks * 32;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int lane = (int)(e & 31);
    const int ks = (int)((e >> 5) % nks);
    const int mt = (int)((e >> 5) / nks);
    const int ro = 8 * mt + (lane >> 2), ri = 4 * ks + (lane & 3);
    double v = 0.0;
    if (ro < NR && ri < NR) {
      int j, k, po, n, m, pi;
      real_decode(ro, j, k, po);
      real_decode(ri, n, m, pi);
      // U = I_{j+n}^{k+m}, V = I_{j+n}^{k-m}
      const double2 U = cget(shI, j + n, k + m);
      const double2 V = cget(shI, j + n, k - m);
      const double s = (m & 1) ? -1.0 : 1.0;
      double w;
      if (m == 0) {
        w = po == 0 ? U.x : U.y;
      } else if (pi == 0) {  // d/d(Re M): U + sV
        w = po == 0 ? U.x + s * V.x : U.y + s * V.y;
      } else {  // d/d(Im M): i (U - sV)
        w = po == 0 ? -(U.y - s * V.y) : U.x - s * V.x;
      }
      double sc = (n & 1) ? -1.0 : 1.0;
      for (int t = 0; t < n; ++t) sc *= fB;
      for (int t = 0; t <= j; ++t) sc *= fA;
      v = sc * w;
    }
    ops[(int64_t)cls * total + e] = v;
  }
}

__global__ void target_flag_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ cbeg,
                                   const int32_t* __restrict__ cend, int64_t nc, int64_t own_b, int64_t own_e,
                                   int32_t* __restrict__ flag) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) flag[c] = (off[c + 1] > off[c] && cbeg[c] < own_e && cend[c] > own_b) ? 1 : 0;
}

__global__ void target_pos_kernel(const int32_t* __restrict__ flag, const int64_t* __restrict__ off, int64_t nc,
                                  int32_t* __restrict__ pos, int32_t* __restrict__ tcells) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  if (flag[c]) {
    pos[c] = (int32_t)off[c];
    tcells[off[c]] = (int32_t)c;
  } else {
    pos[c] = -1;
  }
}

// composite sort key (tile, class, slot, g); pairs of non-owned targets sort last
__global__ void tile_key_kernel(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src, int64_t n,
                                const int32_t* __restrict__ level, const int32_t* __restrict__ anchor,
                                const int32_t* __restrict__ pos, const int32_t* __restrict__ pcls, int T,
                                uint64_t* __restrict__ keys, uint32_t* __restrict__ idx, int32_t* __restrict__ own) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t ckey;
  int g;
  pair_class(tgt[i], src[i], level, anchor, ckey, g);
  const int ps = pos[tgt[i]];
  uint64_t k = ~0ull >> 1;
  if (ps >= 0) {
    const uint64_t tile = (uint64_t)(ps / T), slot = (uint64_t)(ps % T);
    k = (tile << 35) | ((uint64_t)pcls[i] << 11) | (slot << 4) | (uint64_t)g;
  }
  keys[i] = k;
  idx[i] = (uint32_t)i;
  own[i] = ps >= 0;
}

__global__ void columns_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx, int64_t n,
                               const int32_t* __restrict__ src, int32_t* __restrict__ col_src,
                               int32_t* __restrict__ col_meta, int32_t* __restrict__ run_flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  col_src[i] = src[idx[i]];
  col_meta[i] = (int32_t)(((k >> 4) & 0x7f) | ((k & 0xf) << 8));
  run_flag[i] = (i == 0 || (keys[i - 1] >> 11) != (k >> 11)) ? 1 : 0;
}

__global__ void run_start_kernel(const int32_t* __restrict__ run_flag, const int64_t* __restrict__ run_off,
                                 int64_t n, int32_t* __restrict__ run_start) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && run_flag[i]) run_start[run_off[i]] = (int32_t)i;
}

__global__ void chunk_flag_kernel(const int32_t* __restrict__ run_flag, const int64_t* __restrict__ run_off,
                                  const int32_t* __restrict__ run_start, int64_t n, int nc_max,
                                  int32_t* __restrict__ cflag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = run_off[i] + run_flag[i] - 1;
  cflag[i] = ((i - run_start[r]) % nc_max) == 0 ? 1 : 0;
}

__global__ void chunk_emit_kernel(const uint64_t* __restrict__ keys, const int32_t* __restrict__ cflag,
                                  const int64_t* __restrict__ coff, int64_t n, int32_t* __restrict__ chunk_begin,
                                  int32_t* __restrict__ chunk_class, int32_t* __restrict__ chunk_tile) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !cflag[i]) return;
  const int64_t c = coff[i];
  chunk_begin[c] = (int32_t)i;
  chunk_class[c] = (int32_t)((keys[i] >> 11) & 0xffffff);
  chunk_tile[c] = (int32_t)(keys[i] >> 35);
}

// tile_chunk[t] = first chunk of tile >= t  (chunk_tile ascending)
__global__ void tile_chunk_kernel(const int32_t* __restrict__ chunk_tile, int64_t nchunks, int64_t ntiles,
                                  int32_t* __restrict__ tile_chunk) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nchunks) return;
  const int64_t lo = i == 0 ? 0 : (int64_t)chunk_tile[i - 1] + 1;
  const int64_t hi = i == nchunks ? ntiles : (int64_t)chunk_tile[i];
  for (int64_t t = lo; t <= hi; ++t) tile_chunk[t] = (int32_t)i;
}

// h_l^{-n} for n = 0..p+1 and every level (normalised frame, h_l = S / 2^{l+1})
__global__ void hpow_kernel(double S, int p, double* __restrict__ tab) {
  const int l = threadIdx.x;
  if (l > kMaxLevel) return;
  const double ih = 1.0 / ldexp(S, -(l + 1));
  double v = 1.0;
  for (int n = 0; n <= p + 1; ++n) {
    tab[l * (p + 2) + n] = v;
    v *= ih;
  }
}

// ------------------------------------------------------------- the mat-vec kernel

// S9 pre-pass: M~ rows in the real basis, M~[c][r] = {Re,Im} M_n^m(c) h_c^{-n}, zero for r >= NR.
__global__ void mtilde_kernel(const double2* __restrict__ M, const int32_t* __restrict__ level,
                              const double* __restrict__ hpow, int64_t ncells, int p, int nc, int NR, int Kpad,
                              double* __restrict__ Mt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ncells * Kpad) return;
  const int64_t c = e / Kpad;
  const int r = (int)(e - c * Kpad);
  double v = 0.0;
  if (r < NR) {
    int n, m, part;
    real_decode(r, n, m, part);
    const double2 z = M[c * nc + cidx(n, m)];
    v = (part ? z.y : z.x) * hpow[level[c] * (p + 2) + n];
  }
  Mt[e] = v;
}

// ---------------------------------------------------------------------------------------
// Shared-memory layout of one chunk: X[col][k] (and later Y[col][row]) with a column stride
// S = xstride, S % 16 == 4 doubles, so the DMMA B-fragment loads (8 columns x 4 rows per warp),
// the column-wise gather stores and the staged-Y stores are all bank-conflict free.

// C[2][NT] = A(two m-tiles, fragments streamed from L2, 3 k-steps of prefetch) x X(NT n-tiles)
template <int NT>
__device__ __forceinline__ void gemm_chunk(double (&c)[2][8][2], const double* __restrict__ A0, int nks,
                                           const double* __restrict__ xc, int S, int lane) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  const double* A1 = A0 + (int64_t)nks * 32;
  constexpr int D = 3;
  double ra0[D], ra1[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    ra0[d] = d < nks ? __ldg(A0 + d * 32) : 0.0;
    ra1[d] = d < nks ? __ldg(A1 + d * 32) : 0.0;
  }
  const double* bx = xc + (lane >> 2) * S + (lane & 3);
  for (int ks = 0; ks < nks; ks += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (ks + d < nks) {
        const double a0 = ra0[d], a1 = ra1[d];
        if (ks + d + D < nks) {
          ra0[d] = __ldg(A0 + (ks + d + D) * 32);
          ra1[d] = __ldg(A1 + (ks + d + D) * 32);
        }
        double bv[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) bv[j] = bx[j * 8 * S + 4 * (ks + d)];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          dmma884(c[0][j][0], c[0][j][1], a0, bv[j]);
          dmma884(c[1][j][0], c[1][j][1], a1, bv[j]);
        }
      }
    }
  }
}

__device__ __forceinline__ void gemm_dispatch(int nta, double (&c)[2][8][2], const double* A0, int nks,
                                              const double* xc, int S, int lane) {
  switch (nta) {
    case 1: gemm_chunk<1>(c, A0, nks, xc, S, lane); break;
    case 2: gemm_chunk<2>(c, A0, nks, xc, S, lane); break;
    case 3: gemm_chunk<3>(c, A0, nks, xc, S, lane); break;
    case 4: gemm_chunk<4>(c, A0, nks, xc, S, lane); break;
    case 5: gemm_chunk<5>(c, A0, nks, xc, S, lane); break;
    case 6: gemm_chunk<6>(c, A0, nks, xc, S, lane); break;
    case 7: gemm_chunk<7>(c, A0, nks, xc, S, lane); break;
    default: gemm_chunk<8>(c, A0, nks, xc, S, lane); break;
  }
}

// Y[col][row] over the consumed X buffer (rows < NR only)
__device__ __forceinline__ void stage_y(const double (&c)[2][8][2], double* xc, int S, int NR, int nta, int warp,
                                        int lane) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int row = 16 * warp + 8 * i + (lane >> 2);
      const int col = 8 * j + 2 * (lane & 3);
      if (j < nta && row < NR) {
        xc[col * S + row] = c[i][j][0];
        xc[(col + 1) * S + row] = c[i][j][1];
      }
    }
}

// X[col][k] = (D^M_g)^{-1} M~_B[k] for the chunk's columns; one warp per column, 4 columns
// in flight per warp; zero for k in [NR, Kpad) and for columns in [ncol, 8 * ceil(ncol / 8)).
template <int U, int Q>  // U columns in flight per warp, Q * 32 >= Kpad rows
__device__ __forceinline__ void gather_cols(double* xb, int ncol, const int32_t* meta, const int32_t* srcs,
                                            const int32_t* sym, const double* __restrict__ Mt, int NR, int Kpad,
                                            int S, int w, int nw, int lane) {
  const int ncol8 = (ncol + 7) & ~7;
  for (int c0 = w * U; c0 < ncol8; c0 += nw * U) {
    double v[U][Q];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int col = c0 + u;
      const bool live = col < ncol;
      const int B = live ? srcs[col] : 0;
      const int32_t* sm_ = sym + (live ? (meta[col] >> 8) : 0) * 2 * NR;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int k = lane + 32 * q;
        v[u][q] = 0.0;
        if (live && k < NR) {
          const int ent = sm_[k];
          const double x = __ldg(Mt + (int64_t)B * Kpad + (ent & 0xffff));
          v[u][q] = (ent >> 16) ? -x : x;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int col = c0 + u;
      if (col < ncol8) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int k = lane + 32 * q;
          if (k < Kpad) xb[col * S + k] = v[u][q];
        }
      }
    }
  }
}

// acc[slot][r] += sum over the chunk's columns of (D^L_g Y)[r], segments [s_lo, s_hi) of this thread
__device__ __forceinline__ void accumulate_rows(double* acc, const double* y, int S, int NR, int r, uint32_t mask,
                                                int poff, const int32_t* meta, const int32_t* sb,
                                                const int32_t* ss, int s_lo, int s_hi) {
  for (int sgi = s_lo; sgi < s_hi; ++sgi) {
    double* ap = acc + ss[sgi] * NR + r;
    double v = *ap;
    const int cb = sb[sgi], ce = sb[sgi + 1];
    int col = cb;
    for (; col + 2 <= ce; col += 2) {
      const int g0 = meta[col] >> 8, g1 = meta[col + 1] >> 8;
      const double y00 = y[col * S + r], y01 = y[col * S + r + poff];
      const double y10 = y[(col + 1) * S + r], y11 = y[(col + 1) * S + r + poff];
      const uint32_t m0 = mask >> (2 * g0), m1 = mask >> (2 * g1);
      double t0 = (m0 & 1) ? y01 : y00, t1 = (m1 & 1) ? y11 : y10;
      v += (m0 & 2) ? -t0 : t0;
      v += (m1 & 2) ? -t1 : t1;
    }
    if (col < ce) {
      const int g0 = meta[col] >> 8;
      const uint32_t m0 = mask >> (2 * g0);
      const double t0 = (m0 & 1) ? y[col * S + r + poff] : y[col * S + r];
      v += (m0 & 2) ? -t0 : t0;
    }
    *ap = v;
  }
}

__device__ __forceinline__ void writeback(const M2LArgs& a, const double* acc, const int32_t* dec, int tile, int tid,
                                          int nthr) {
  const int NR = a.NR;
  for (int e = tid; e < a.T * NR; e += nthr) {
    const int slot = e / NR, r = e - slot * NR;
    const int cell = a.tile_cells[tile * a.T + slot];
    if (cell < 0) continue;
    const int d = dec[r];
    const double v = acc[e] * a.hpow[a.level[cell] * (a.p + 2) + ((d >> 1) & 0x7f) + 1];
    ((double*)(a.L + (int64_t)cell * a.nc))[2 * (d >> 8) + (d & 1)] = v;
  }
}

// shared-memory carve-up common to both kernels
struct Smem {
  double *acc, *x0, *x1;
  int32_t *meta, *srcs, *sslot, *sbeg, *sym, *dec, *lmask, *lpoff;
};
__device__ __forceinline__ Smem carve(double* sm, const M2LArgs& a) {
  Smem m;
  const int xsz = a.NC * a.ystride;
  m.acc = sm;
  m.x0 = m.acc + (size_t)a.T * a.NR;
  m.x1 = m.x0 + xsz;
  m.meta = (int32_t*)(m.x1 + xsz);  // [2][NC]
  m.srcs = m.meta + 2 * a.NC;       // [2][NC]
  m.sslot = m.srcs + 2 * a.NC;      // [2][NC]
  m.sbeg = m.sslot + 2 * a.NC;      // [2][NC + 1]
  m.sym = m.sbeg + 2 * (a.NC + 1);  // [16][2][NR]
  m.dec = m.sym + 32 * a.NR;        // [NR]
  m.lmask = m.dec + a.NR;           // [NR] output-transform bits per row (ltrans_mask)
  m.lpoff = m.lmask + a.NR;         // [NR] re/im partner offset per row
  return m;
}
__device__ __forceinline__ void init_smem(const M2LArgs& a, const Smem& m, int tid, int nthr) {
  for (int e = tid; e < a.T * a.NR; e += nthr) m.acc[e] = 0.0;
  for (int e = tid; e < 32 * a.NR; e += nthr) m.sym[e] = a.symtab[e];
  for (int r = tid; r < a.NR; r += nthr) {
    int n, mm, part;
    real_decode(r, n, mm, part);
    m.dec[r] = (cidx(n, mm) << 8) | (n << 1) | part;
  }
  __syncthreads();  // sym complete
  for (int r = tid; r < a.NR; r += nthr) {
    int poff = 0;
    m.lmask[r] = (int32_t)ltrans_mask(m.sym, a.NR, r, poff);
    m.lpoff[r] = poff;
  }
}

// all (row group, row) items of one chunk's accumulate, spread over nt threads starting at t0
__device__ __forceinline__ void accumulate_chunk(const Smem& m, const double* y, int S, int NR, int ns,
                                                 const int32_t* meta, const int32_t* sb, const int32_t* ss, int t0,
                                                 int nt) {
  const int RG = max(1, nt / NR);
  for (int t = t0; t < RG * NR; t += nt) {
    const int rg = t / NR, r = t - rg * NR;
    accumulate_rows(m.acc, y, S, NR, r, (uint32_t)m.lmask[r], m.lpoff[r], meta, sb, ss, ns * rg / RG,
                    ns * (rg + 1) / RG);
  }
}

// Plain variant (all warps take every phase in turn): used where the warp-specialised one
// does not fit (p <= 4: fewer than two rows of helpers; p >= 14: too many MMA warps).
__global__ void __launch_bounds__(640, 1) m2l_dmma_kernel(const M2LArgs a) {
  extern __shared__ double sm[];
  const Smem m = carve(sm, a);
  const int NR = a.NR, NC = a.NC, S = a.ystride;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
  const int tile = blockIdx.x;
  init_smem(a, m, tid, nthr);
  __syncthreads();
  for (int ch = a.tile_chunk[tile]; ch < a.tile_chunk[tile + 1]; ++ch) {
    const int cls = a.chunk_class[ch];
    const int ncol = a.chunk_begin[ch + 1] - a.chunk_begin[ch];
    __syncthreads();
    load_meta_dev(a, ch, m.meta, m.srcs, m.sslot, m.sbeg, tid, nthr);
    __syncthreads();
    gather_cols<2, 10>(m.x0, ncol, m.meta, m.srcs, m.sym, a.Mt, NR, a.Kpad, S, warp, nwarp, lane);
    __syncthreads();
    const int nta = (ncol + 7) >> 3;
    double c[2][8][2];
    if (2 * warp < a.nmt) {
      const double* A0 = a.ops + (((int64_t)cls * a.nmt + 2 * warp) * a.nks) * 32 + lane;
      gemm_dispatch(nta, c, A0, a.nks, m.x0, S, lane);
    }
    __syncthreads();
    if (2 * warp < a.nmt) stage_y(c, m.x0, S, NR, nta, warp, lane);
    __syncthreads();
    accumulate_chunk(m, m.x0, S, NR, a.chunk_seg[ch + 1] - a.chunk_seg[ch], m.meta, m.sbeg, m.sslot, tid, nthr);
  }
  __syncthreads();
  writeback(a, m.acc, m.dec, tile, tid, nthr);
}

// ---------------------------------------------------------------------------------------
// Warp-specialised variant: nmma = nmt/2 MMA warps run only the DMMA GEMMs; nhelp helper
// warps gather the next chunk's X and add the previous chunk's Y into the accumulators.
// Handshake with named barriers (ids alternate by chunk parity):
//   Xfull(i):  helpers bar.arrive after storing X(i);  MMA bar.sync before GEMM(i)
//   Yfull(i):  MMA bar.arrive after staging Y(i);      helpers bar.sync before adding Y(i)
// Y(i) is staged over X[i % 2] (consumed by GEMM(i)); helpers overwrite X[i % 2] with
// X(i+2) only after adding Y(i), so two X buffers suffice.
__global__ void __launch_bounds__(512, 1) m2l_ws_kernel(const M2LArgs a, int nmma, int nhelp, int dbg) {
  extern __shared__ double sm[];
  const Smem m = carve(sm, a);
  const int NR = a.NR, NC = a.NC, S = a.ystride;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int nmma_t = 32 * nmma, nhelp_t = 32 * nhelp, nall = nmma_t + nhelp_t;
  init_smem(a, m, tid, nthr);
  const int c_first = a.tile_chunk[tile], c_last = a.tile_chunk[tile + 1];
  __syncthreads();
  if (warp >= nmma) {
    // ================= helper warps
    const int h = tid - nmma_t, hw = warp - nmma;
    auto prep = [&](int ch, int b) {
      load_meta_dev(a, ch, m.meta + b * NC, m.srcs + b * NC, m.sslot + b * NC, m.sbeg + b * (NC + 1), h, nhelp_t);
      named_sync(6, nhelp_t);  // metadata visible to all helpers
      if (!(dbg & 1))
        gather_cols<4, 8>(b ? m.x1 : m.x0, a.chunk_begin[ch + 1] - a.chunk_begin[ch], m.meta + b * NC,
                          m.srcs + b * NC, m.sym, a.Mt, NR, a.Kpad, S, hw, nhelp, lane);
    };
    if (c_first < c_last) {
      prep(c_first, 0);
      named_arrive(1, nall);  // Xfull(0)
    }
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1, nb = b ^ 1;
      if (ch + 1 < c_last) {
        prep(ch + 1, nb);
        named_arrive(1 + nb, nall);  // Xfull(i+1)
      }
      named_sync(3 + b, nall);  // Yfull(i)
      if (!(dbg & 2))
        accumulate_chunk(m, b ? m.x1 : m.x0, S, NR, a.chunk_seg[ch + 1] - a.chunk_seg[ch], m.meta + b * NC,
                         m.sbeg + b * (NC + 1), m.sslot + b * NC, h, nhelp_t);
      named_sync(6, nhelp_t);  // helpers done with meta[b] / Y(i) before they are overwritten
    }
  } else {
    // ================= MMA warps
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      named_sync(1 + b, nall);  // Xfull(i)
      double* xc = b ? m.x1 : m.x0;
      const int cls = a.chunk_class[ch];
      const int nta = (a.chunk_begin[ch + 1] - a.chunk_begin[ch] + 7) >> 3;
      double c[2][8][2];
      const double* A0 = a.ops + (((int64_t)cls * a.nmt + 2 * warp) * a.nks) * 32 + lane;
      gemm_dispatch(nta, c, A0, a.nks, xc, S, lane);
      named_sync(5, nmma_t);  // all MMA warps done reading X[b]
      stage_y(c, xc, S, NR, nta, warp, lane);
      named_arrive(3 + b, nall);  // Yfull(i)
    }
  }
  __syncthreads();
  writeback(a, m.acc, m.dec, tile, tid, nthr);
}

// ---------------------------------------------------------------------------------------
// Compile-time-p version of the warp-specialised kernel (p = 5..14): all strides and loop
// bounds are constants, so the DMMA loop unrolls with immediate shared-memory offsets.
constexpr int ct_xstride(int kpad) {
  int s = kpad;
  while (s % 16 != 4) ++s;
  return s;
}
template <int P>
struct Geo {
  static constexpr int NR = (P + 1) * (P + 1);
  static constexpr int KPAD = (NR + 3) & ~3;
  static constexpr int NKS = KPAD / 4;
  static constexpr int NRPAD = (NR + 15) & ~15;
  static constexpr int NMT = NRPAD / 8;
  // m-tiles per MMA warp: one warp issues at most one DMMA per ~66 cycles (tools/dmma_probe.cu),
  // so the DMMA pipe (one per 16 cycles per SMSP) needs >= 16 issuing warps per SM
  static constexpr int MTW = 2;  // (one m-tile per warp with 16 MMA warps measured no faster)
  static constexpr int NMMA = NMT / MTW;
  static constexpr int NHELP = MTW == 1 ? 8 : (2 * ((NR + 31) / 32) < 16 - NMMA ? 2 * ((NR + 31) / 32) : 16 - NMMA);
  static constexpr int THREADS = 32 * (NMMA + NHELP);
  static constexpr int S = ct_xstride(KPAD);
  static constexpr int NC = 2 * S * 64 * 8 > 140 * 1024 ? 32 : 64;
  static constexpr int Q = (KPAD + 31) / 32;
};

template <int MTW, int NT, int S, int NKS>
__device__ __forceinline__ void gemm_ct(double (&c)[MTW][8][2], const double* __restrict__ A0,
                                        const double* __restrict__ xc, int lane) {
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  constexpr int D = 4;
  double ra[MTW][D];
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int d = 0; d < D; ++d) ra[i][d] = d < NKS ? __ldg(A0 + (i * NKS + d) * 32) : 0.0;
  const double* bx = xc + (lane >> 2) * S + (lane & 3);
#pragma unroll
  for (int ks = 0; ks < NKS; ++ks) {
    double av[MTW];
#pragma unroll
    for (int i = 0; i < MTW; ++i) {
      av[i] = ra[i][ks % D];
      if (ks + D < NKS) ra[i][ks % D] = __ldg(A0 + (i * NKS + ks + D) * 32);
    }
    double bv[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) bv[j] = bx[j * 8 * S + 4 * ks];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int i = 0; i < MTW; ++i) dmma884(c[i][j][0], c[i][j][1], av[i], bv[j]);
  }
}

template <int MTW, int S, int NKS>
__device__ __forceinline__ void gemm_ct_dispatch(int nta, double (&c)[MTW][8][2], const double* A0, const double* xc,
                                                 int lane) {
  switch (nta) {
    case 1: gemm_ct<MTW, 1, S, NKS>(c, A0, xc, lane); break;
    case 2: gemm_ct<MTW, 2, S, NKS>(c, A0, xc, lane); break;
    case 3: gemm_ct<MTW, 3, S, NKS>(c, A0, xc, lane); break;
    case 4: gemm_ct<MTW, 4, S, NKS>(c, A0, xc, lane); break;
    case 5: gemm_ct<MTW, 5, S, NKS>(c, A0, xc, lane); break;
    case 6: gemm_ct<MTW, 6, S, NKS>(c, A0, xc, lane); break;
    case 7: gemm_ct<MTW, 7, S, NKS>(c, A0, xc, lane); break;
    default: gemm_ct<MTW, 8, S, NKS>(c, A0, xc, lane); break;
  }
}

// Y[col][row] over the consumed X buffer, MTW m-tiles per warp (rows < NR only)
template <int MTW>
__device__ __forceinline__ void stage_y_ct(const double (&c)[MTW][8][2], double* xc, int S, int NR, int nta, int warp,
                                           int lane) {
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int row = 8 * (MTW * warp + i) + (lane >> 2);
      const int col = 8 * j + 2 * (lane & 3);
      if (j < nta && row < NR) {
        xc[col * S + row] = c[i][j][0];
        xc[(col + 1) * S + row] = c[i][j][1];
      }
    }
}

template <int P>
__global__ void __launch_bounds__(Geo<P>::THREADS, 1) m2l_ws_ct_kernel(const M2LArgs a, int nhelp) {
  using G = Geo<P>;
  constexpr int NR = G::NR, NC = G::NC, S = G::S;
  extern __shared__ double sm[];
  const Smem m = carve(sm, a);
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  constexpr int nmma_t = 32 * G::NMMA;
  const int nhelp_t = 32 * nhelp, nall = nmma_t + nhelp_t;
  init_smem(a, m, tid, nthr);
  const int c_first = a.tile_chunk[tile], c_last = a.tile_chunk[tile + 1];
  __syncthreads();
  if (warp >= G::NMMA) {
    const int h = tid - nmma_t, hw = warp - G::NMMA;
    auto prep = [&](int ch, int b) {
      load_meta_dev(a, ch, m.meta + b * NC, m.srcs + b * NC, m.sslot + b * NC, m.sbeg + b * (NC + 1), h, nhelp_t);
      named_sync(6, nhelp_t);
      gather_cols<4, G::Q>(b ? m.x1 : m.x0, a.chunk_begin[ch + 1] - a.chunk_begin[ch], m.meta + b * NC,
                           m.srcs + b * NC, m.sym, a.Mt, NR, G::KPAD, S, hw, nhelp, lane);
    };
    if (c_first < c_last) {
      prep(c_first, 0);
      named_arrive(1, nall);
    }
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1, nb = b ^ 1;
      if (ch + 1 < c_last) {
        prep(ch + 1, nb);
        named_arrive(1 + nb, nall);
      }
      named_sync(3 + b, nall);
      accumulate_chunk(m, b ? m.x1 : m.x0, S, NR, a.chunk_seg[ch + 1] - a.chunk_seg[ch], m.meta + b * NC,
                       m.sbeg + b * (NC + 1), m.sslot + b * NC, h, nhelp_t);
      named_sync(6, nhelp_t);
    }
  } else {
    for (int ch = c_first; ch < c_last; ++ch) {
      const int i = ch - c_first, b = i & 1;
      named_sync(1 + b, nall);
      double* xc = b ? m.x1 : m.x0;
      const int cls = a.chunk_class[ch];
      const int nta = (a.chunk_begin[ch + 1] - a.chunk_begin[ch] + 7) >> 3;
      double c[G::MTW][8][2];
      const double* A0 = a.ops + (((int64_t)cls * G::NMT + G::MTW * warp) * G::NKS) * 32 + lane;
      gemm_ct_dispatch<G::MTW, S, G::NKS>(nta, c, A0, xc, lane);
      named_sync(5, nmma_t);
      stage_y_ct<G::MTW>(c, xc, S, NR, nta, warp, lane);
      named_arrive(3 + b, nall);
    }
  }
  __syncthreads();
  writeback(a, m.acc, m.dec, tile, tid, nthr);
}

// segment flags: a new slot segment starts at a chunk start or where the slot changes
__global__ void seg_flag_kernel(const int32_t* __restrict__ col_meta, const int32_t* __restrict__ cflag, int64_t n,
                                int32_t* __restrict__ sflag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) sflag[i] = (cflag[i] || (col_meta[i] & 0xff) != (col_meta[i - 1] & 0xff)) ? 1 : 0;
}

__global__ void seg_emit_kernel(const int32_t* __restrict__ sflag, const int64_t* __restrict__ soff,
                                const int32_t* __restrict__ cflag, const int64_t* __restrict__ coff, int64_t n,
                                int32_t* __restrict__ seg_begin, int32_t* __restrict__ chunk_seg) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (sflag[i]) seg_begin[soff[i]] = (int32_t)i;
  if (cflag[i]) chunk_seg[coff[i]] = (int32_t)soff[i];
}

}  // namespace

namespace m2l {
// packed entry: bits 0..15 source real index, bit 16 = negative sign
std::vector<int32_t> build_symtab(int p) {
  const int NR = real_count(p);
  std::vector<int32_t> t(16 * 2 * NR);
  for (int g = 0; g < 16; ++g)
    for (int which = 0; which < 2; ++which) {  // 0: X = (D^M)^{-1} M, 1: L += D^L Y
      for (int n = 0; n <= p; ++n)
        for (int m = 0; m <= n; ++m) {
          M2 D = dmap(g, n, m, which == 1);
          if (which == 0) D = {D.a, D.c, D.b, D.d};  // inverse of a signed permutation = transpose
          // out = D * in on (re, im); m == 0 keeps only re (the map is diagonal there)
          for (int po = 0; po < (m == 0 ? 1 : 2); ++po) {
            const int c0 = po == 0 ? D.a : D.c, c1 = po == 0 ? D.b : D.d;
            int src_part = c0 != 0 ? 0 : 1;
            int sgn = c0 != 0 ? c0 : c1;
            if (m == 0) src_part = 0, sgn = D.a;
            const int ro = real_index(n, m, po), rs = real_index(n, m, src_part);
            t[(g * 2 + which) * NR + ro] = rs | (sgn < 0 ? (1 << 16) : 0);
          }
        }
    }
  return t;
}

}  // namespace m2l

size_t m2l_smem_bytes(const M2LDmma& D) {
  return ((size_t)D.T * D.NR + 2 * (size_t)D.ystride * D.NC) * sizeof(double) +
         (8 * D.NC + 2 + 35 * D.NR) * sizeof(int32_t);
}

void m2l_dmma_setup(fmm_plan_s& P) {
  cudaStream_t s = P.stream;
  M2LDmma& D = P.m2l_dmma;
  const Cells& C = P.cells;
  const int p = P.p;
  D.NR = real_count(p);
  D.NRpad = (D.NR + 15) / 16 * 16;
  D.nmt = D.NRpad / 8;
  D.Kpad = (D.NR + 3) / 4 * 4;
  D.nks = D.Kpad / 4;
  D.NC = kNC;
  D.ystride = D.Kpad;  // column stride S of X[col][k] / Y[col][row]: S >= Kpad, S % 16 == 4
  while (D.ystride % 16 != 4) ++D.ystride;
  if (2 * (size_t)D.ystride * D.NC * sizeof(double) > 140 * 1024) D.NC = kNC / 2;  // large p: 32-column chunks
  D.T = 64;
  while (D.T > 8 && m2l_smem_bytes(D) > 220 * 1024) D.T /= 2;
  if (P.m2l_variant == 3 && !m2l_rot_supported(p)) P.m2l_variant = 2;
  if (P.m2l_variant == 3) {  // v3 chunk width and tile size (shared-memory budget), else v2
    D.T = 128;  // as many targets per tile as shared memory allows (p <= 8: 128; configs[3] M2L -2 %)
    if (const char* t = getenv("FMM_M2L_T")) D.T = std::max(8, std::min(256, atoi(t)));  // experiments
    while (D.T > 16 && rot_smem_bytes(p, D.T, 8) > 225 * 1024) D.T /= 2;
    if (rot_smem_bytes(p, D.T, 8) > 225 * 1024)
      P.m2l_variant = 2, D.T = 64;
    else
      D.NC = rot_chunk_width(p);
  }
  if (P.m2l_variant == 2)
    while (D.T > 8 && m2l_smem_bytes(D) > 220 * 1024) D.T /= 2;
  // warp-specialised kernel: nmt/2 MMA warps + ceil(NR/32) helper warps, <= 512 threads
  D.nhelp = std::min(2 * ((D.NR + 31) / 32), 16 - D.nmt / 2);
  D.use_ws = D.nhelp >= 1 && D.NR > 32 && D.Kpad <= 256 && getenv("FMM_M2L_NO_WS") == nullptr;
  int64_t n = P.m2l.n;
  D.npairs = 0;
  D.ntiles = 0;
  D.nchunks = 0;
  D.nclass = 0;
  if (n == 0) return;

  // ---- own target cells (cells with M2L sources intersecting this rank's particles)
  DevBuf<int32_t> flag, pos;
  DevBuf<int64_t> off;
  flag.alloc(C.n);
  off.alloc(C.n);
  pos.alloc(C.n);
  target_flag_kernel<<<cdiv(C.n, 256), 256, 0, s>>>(P.m2l.off, C.begin, C.end, C.n, P.own_begin, P.own_end, flag);
  FMM_LAUNCHED("target_flag_kernel");
  const int64_t ntc = scan_counts_total(flag, off, C.n, s);
  if (P.m2l_variant == 3 && !getenv("FMM_M2L_T")) {
    // small problems: narrower tiles until there are two CTA waves (one CTA per SM); configs[1]
    // (4,681 cells) M2L 1.10 -> 0.84 ms with T = 16 (wider tiles are more efficient per pair:
    // configs[2] is fastest at T = 64, configs[3] at T = 128)
    int nsm = 148;
    FMM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P.device));
    while (D.T > 16 && (ntc + D.T - 1) / D.T < 2LL * nsm) D.T /= 2;
  }
  D.ntiles = (ntc + D.T - 1) / D.T;
  D.tile_cells.alloc(std::max<int64_t>(1, D.ntiles * D.T));
  FMM_CUDA(cudaMemsetAsync(D.tile_cells.ptr, 0xff, sizeof(int32_t) * D.tile_cells.count, s));
  target_pos_kernel<<<cdiv(C.n, 256), 256, 0, s>>>(flag, off, C.n, pos, D.tile_cells);
  FMM_LAUNCHED("target_pos_kernel");

  // ---- canonical classes
  DevBuf<uint64_t> keys;
  DevBuf<uint32_t> idx;
  DevBuf<int32_t> pflag, pcls;
  DevBuf<int64_t> poff;
  keys.alloc(n);
  idx.alloc(n);
  pflag.alloc(n);
  poff.alloc(n);
  pcls.alloc(n);
  class_key_kernel<<<cdiv(n, 256), 256, 0, s>>>(P.m2l.tgt, P.m2l.src, n, C.level, C.anchor, keys, idx);
  FMM_LAUNCHED("class_key_kernel");
  radix_sort_pairs(keys, idx, n, 63, s);
  {  // an all-ones key (offset beyond 2^19 finer half sides) sorts last
    uint64_t last = 0;
    FMM_CUDA(cudaMemcpyAsync(&last, keys.ptr + n - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    if (last == (~0ull >> 1)) throw Error(FMM_ERR_USAGE, "m2l: cell offset beyond 2^19 finer half sides");
  }
  diff_flag_kernel<<<cdiv(n, 256), 256, 0, s>>>(keys, n, pflag);
  FMM_LAUNCHED("diff_flag_kernel");
  D.nclass = scan_counts_total(pflag, poff, n, s);
  D.class_keys.alloc(D.nclass);
  DevBuf<uint64_t>& ckeys = D.class_keys;
  class_assign_kernel<<<cdiv(n, 256), 256, 0, s>>>(keys, idx, pflag, poff, n, pcls, ckeys);
  FMM_LAUNCHED("class_assign_kernel");
  if (D.nclass >= (1 << 24)) throw Error(FMM_ERR_USAGE, "m2l: too many operator classes");
  if (D.ntiles >= (1 << 28)) throw Error(FMM_ERR_USAGE, "m2l: too many tiles");

  // ---- operators (fragment order) and per-level scale table
  if (P.m2l_variant == 2) {
    const int64_t opsz = (int64_t)D.nmt * D.nks * 32;
    D.ops.alloc(D.nclass * opsz);
    build_ops_kernel<<<(unsigned)D.nclass, 256, sizeof(double2) * ncoef(2 * p), s>>>(ckeys, p, D.nmt, D.nks, D.ops);
    FMM_LAUNCHED("build_ops_kernel");
  }
  D.hpow.alloc((kMaxLevel + 1) * (p + 2));
  hpow_kernel<<<1, 32, 0, s>>>(P.S, p, D.hpow);
  FMM_LAUNCHED("hpow_kernel");
  std::vector<int32_t> sym = build_symtab(p);
  D.symtab.alloc((int64_t)sym.size());
  FMM_CUDA(cudaMemcpyAsync(D.symtab.ptr, sym.data(), sizeof(int32_t) * sym.size(), cudaMemcpyHostToDevice, s));

  // ---- sort pairs by (tile, class, slot, g) and cut runs into chunks of <= NC columns
  tile_key_kernel<<<cdiv(n, 256), 256, 0, s>>>(P.m2l.tgt, P.m2l.src, n, C.level, C.anchor, pos, pcls, D.T, keys,
                                               idx, pflag);
  FMM_LAUNCHED("tile_key_kernel");
  const int64_t n_all = n;
  n = scan_counts_total(pflag, poff, n_all, s);  // owned pairs; the others sort last
  radix_sort_pairs(keys, idx, n_all, 63, s);
  D.npairs = n;
  if (n == 0) {
    D.ntiles = 0;
    return;
  }
  D.col_src.alloc(n);
  D.col_meta.alloc(n);
  columns_kernel<<<cdiv(n, 256), 256, 0, s>>>(keys, idx, n, P.m2l.src, D.col_src, D.col_meta, pflag);
  FMM_LAUNCHED("columns_kernel");
  DevBuf<int64_t> roff;
  roff.alloc(n);
  const int64_t nruns = scan_counts_total(pflag, roff, n, s);
  DevBuf<int32_t> rstart, cflag;
  rstart.alloc(nruns);
  cflag.alloc(n);
  run_start_kernel<<<cdiv(n, 256), 256, 0, s>>>(pflag, roff, n, rstart);
  FMM_LAUNCHED("run_start_kernel");
  chunk_flag_kernel<<<cdiv(n, 256), 256, 0, s>>>(pflag, roff, rstart, n, D.NC, cflag);
  FMM_LAUNCHED("chunk_flag_kernel");
  DevBuf<int64_t> coff;
  coff.alloc(n);
  D.nchunks = scan_counts_total(cflag, coff, n, s);
  D.chunk_begin.alloc(D.nchunks + 1);
  D.chunk_class.alloc(D.nchunks);
  DevBuf<int32_t> ctile;
  ctile.alloc(D.nchunks);
  chunk_emit_kernel<<<cdiv(n, 256), 256, 0, s>>>(keys, cflag, coff, n, D.chunk_begin, D.chunk_class, ctile);
  FMM_LAUNCHED("chunk_emit_kernel");
  const int32_t nn = (int32_t)n;
  FMM_CUDA(cudaMemcpyAsync(D.chunk_begin.ptr + D.nchunks, &nn, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  // slot segments (runs of equal target slot inside a chunk) for the accumulate pass
  {
    DevBuf<int32_t> sflag;
    DevBuf<int64_t> soff;
    sflag.alloc(n);
    soff.alloc(n);
    seg_flag_kernel<<<cdiv(n, 256), 256, 0, s>>>(D.col_meta, cflag, n, sflag);
    FMM_LAUNCHED("seg_flag_kernel");
    D.nseg = scan_counts_total(sflag, soff, n, s);
    D.seg_begin.alloc(D.nseg + 1);
    D.chunk_seg.alloc(D.nchunks + 1);
    seg_emit_kernel<<<cdiv(n, 256), 256, 0, s>>>(sflag, soff, cflag, coff, n, D.seg_begin, D.chunk_seg);
    FMM_LAUNCHED("seg_emit_kernel");
    const int32_t ns32 = (int32_t)D.nseg;
    FMM_CUDA(cudaMemcpyAsync(D.seg_begin.ptr + D.nseg, &nn, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(D.chunk_seg.ptr + D.nchunks, &ns32, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  D.Mt.alloc(C.n * D.Kpad);
  D.tile_chunk.alloc(D.ntiles + 1);
  tile_chunk_kernel<<<cdiv(D.nchunks + 1, 256), 256, 0, s>>>(ctile, D.nchunks, D.ntiles, D.tile_chunk);
  FMM_LAUNCHED("tile_chunk_kernel");
  FMM_CUDA(cudaStreamSynchronize(s));
  if (P.m2l_variant == 3) m2l_rot_setup(P);
}

void m2l_dmma_pass(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  FMM_CUDA(cudaMemsetAsync(P.L.ptr, 0, sizeof(double2) * P.L.count, P.stream));
  if (D.ntiles == 0) return;
  const int64_t ne = P.cells.n * D.Kpad;
  if (P.m2l_variant == 3) {
    m2l_rot_mtilde(P);
  } else {
    mtilde_kernel<<<cdiv(ne, 256), 256, 0, P.stream>>>(P.M, P.cells.level, D.hpow, P.cells.n, P.p, P.nc, D.NR, D.Kpad,
                                                       D.Mt);
    FMM_LAUNCHED("mtilde_kernel");
  }
  M2LArgs a;
  a.ops = D.ops;
  a.col_src = D.col_src;
  a.col_meta = D.col_meta;
  a.chunk_begin = D.chunk_begin;
  a.chunk_class = D.chunk_class;
  a.chunk_seg = D.chunk_seg;
  a.seg_begin = D.seg_begin;
  a.tile_chunk = D.tile_chunk;
  a.tile_cells = D.tile_cells;
  a.symtab = D.symtab;
  a.hpow = D.hpow;
  a.level = P.cells.level;
  a.Mt = D.Mt;
  a.L = P.L;
  a.p = P.p;
  a.nc = P.nc;
  a.NR = D.NR;
  a.NRpad = D.NRpad;
  a.Kpad = D.Kpad;
  a.nks = D.nks;
  a.nmt = D.nmt;
  a.T = D.T;
  a.NC = D.NC;
  a.ystride = D.ystride;
  if (P.m2l_variant == 3) {
    m2l_rot_launch(P, a);
    return;
  }
  const size_t sh = m2l_smem_bytes(D);
  const int threads = 32 * (D.nmt / 2);
  const int nmma = D.nmt / 2, nhelp = D.nhelp;
  if (D.use_ws && P.p >= 5 && P.p <= 14 && getenv("FMM_M2L_NO_CT") == nullptr) {
    void (*k)(const M2LArgs, int) = nullptr;
    int thr = 0, nh = 0;
    switch (P.p) {
      case 5: k = m2l_ws_ct_kernel<5>, thr = Geo<5>::THREADS, nh = Geo<5>::NHELP; break;
      case 6: k = m2l_ws_ct_kernel<6>, thr = Geo<6>::THREADS, nh = Geo<6>::NHELP; break;
      case 7: k = m2l_ws_ct_kernel<7>, thr = Geo<7>::THREADS, nh = Geo<7>::NHELP; break;
      case 8: k = m2l_ws_ct_kernel<8>, thr = Geo<8>::THREADS, nh = Geo<8>::NHELP; break;
      case 9: k = m2l_ws_ct_kernel<9>, thr = Geo<9>::THREADS, nh = Geo<9>::NHELP; break;
      case 10: k = m2l_ws_ct_kernel<10>, thr = Geo<10>::THREADS, nh = Geo<10>::NHELP; break;
      case 11: k = m2l_ws_ct_kernel<11>, thr = Geo<11>::THREADS, nh = Geo<11>::NHELP; break;
      case 12: k = m2l_ws_ct_kernel<12>, thr = Geo<12>::THREADS, nh = Geo<12>::NHELP; break;
      case 13: k = m2l_ws_ct_kernel<13>, thr = Geo<13>::THREADS, nh = Geo<13>::NHELP; break;
      default: k = m2l_ws_ct_kernel<14>, thr = Geo<14>::THREADS, nh = Geo<14>::NHELP; break;
    }
    if (sh > 48 * 1024)  // per launch: the opt-in is per device context
      FMM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    k<<<(unsigned)D.ntiles, thr, sh, P.stream>>>(a, nh);
    FMM_LAUNCHED("m2l_ws_ct_kernel");
    return;
  }
  if (D.use_ws) {
    if (sh > 48 * 1024)  // per launch: the opt-in is per device context
      FMM_CUDA(cudaFuncSetAttribute(m2l_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
#ifdef FMM_DEV  // development builds only: timing experiments (skips work: wrong results)
    const char* dbgs = getenv("FMM_M2L_DEBUG");
    const int dbg = dbgs ? atoi(dbgs) : 0;
#else
    const int dbg = 0;
#endif
    m2l_ws_kernel<<<(unsigned)D.ntiles, 32 * (nmma + nhelp), sh, P.stream>>>(a, nmma, nhelp, dbg);
    FMM_LAUNCHED("m2l_ws_kernel");
    return;
  }
  if (sh > 48 * 1024)  // per launch: the opt-in is per device context
    FMM_CUDA(cudaFuncSetAttribute(m2l_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  m2l_dmma_kernel<<<(unsigned)D.ntiles, threads, sh, P.stream>>>(a);
  FMM_LAUNCHED("m2l_dmma_kernel");
}

}  // namespace fmm
