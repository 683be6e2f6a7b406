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
#include <vector>

#include "harmonics.cuh"
#include "plan.h"

namespace fmm {
namespace {

constexpr int kNC = 64;  // max columns per chunk (8 n-tiles of 8)

__host__ __device__ inline int real_count(int p) { return (p + 1) * (p + 1); }

// real index -> (n, m, part)
__host__ __device__ inline void real_decode(int r, int& n, int& m, int& part) {
  n = 0;
  while ((n + 1) * (n + 1) <= r) ++n;
  const int t = r - n * n;
  m = (t + 1) >> 1;
  part = t > 0 ? ((t + 1) & 1) : 0;
}
__host__ __device__ inline int real_index(int n, int m, int part) { return m == 0 ? n * n : n * n + 2 * m - 1 + part; }

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
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct M2LArgs {
  const double* ops;
  const int32_t* col_src;
  const int32_t* col_meta;
  const int32_t* chunk_begin;
  const int32_t* chunk_class;
  const int32_t* tile_chunk;
  const int32_t* tile_cells;
  const int32_t* symtab;  // [16][2][NR]
  const double* hpow;     // [22][p+2]
  const int32_t* level;
  const double2* M;
  double2* L;
  int p, nc, NR, NRpad, Kpad, nks, nmt, T, NC, ystride;
};

// one CTA per tile; blockDim = 32 * nmt / 2 (each warp owns two 8-row m-tiles)
__global__ void __launch_bounds__(640, 1) m2l_dmma_kernel(const M2LArgs a) {
  extern __shared__ double sm[];
  const int NR = a.NR, T = a.T, NC = a.NC;
  double* acc = sm;                                                       // [T][NR]
  double* xy = acc + (size_t)T * NR;                                      // X frags / Y staging
  int32_t* meta = (int32_t*)(xy + (size_t)max(a.Kpad * NC, NC * a.ystride));  // [NC] slot | g << 8
  int32_t* srcs = meta + NC;                                              // [NC]
  int32_t* sym = srcs + NC;                                               // [16][2][NR]
  int32_t* dec = sym + 32 * NR;                                           // [NR] cidx << 8 | n << 1 | part
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
  const int tile = blockIdx.x;
  for (int e = tid; e < T * NR; e += nthr) acc[e] = 0.0;
  for (int e = tid; e < 32 * NR; e += nthr) sym[e] = a.symtab[e];
  for (int r = tid; r < NR; r += nthr) {
    int n, m, part;
    real_decode(r, n, m, part);
    dec[r] = (cidx(n, m) << 8) | (n << 1) | part;
  }
  const int ntn = NC / 8;
  const int c_first = a.tile_chunk[tile], c_last = a.tile_chunk[tile + 1];
  for (int ch = c_first; ch < c_last; ++ch) {
    const int cls = a.chunk_class[ch];
    const int cb = a.chunk_begin[ch];
    const int ncol = a.chunk_begin[ch + 1] - cb;
    __syncthreads();  // previous chunk's accumulate pass is done with xy / meta
    for (int t = tid; t < NC; t += nthr) {  // blockDim may be < NC (p <= 3: one warp)
      meta[t] = t < ncol ? a.col_meta[cb + t] : 0;
      srcs[t] = t < ncol ? a.col_src[cb + t] : 0;
    }
    __syncthreads();
    // ---- gather X~ (scaled, canonical frame) into B-fragment order: one warp per column
    for (int col = warp; col < NC; col += nwarp) {
      double* xcol = xy + (col >> 3) * 32 + (col & 7) * 4;
      if (col < ncol) {
        const int B = srcs[col];
        const int32_t* symM = sym + (meta[col] >> 8) * 2 * NR;
        const double* hp = a.hpow + a.level[B] * (a.p + 2);
        const double* Mb = (const double*)(a.M + (int64_t)B * a.nc);
        for (int k = lane; k < a.Kpad; k += 32) {
          double v = 0.0;
          if (k < NR) {
            const int ent = symM[k];
            const int d = dec[ent & 0xffff];
            v = Mb[2 * (d >> 8) + (d & 1)] * hp[(d >> 1) & 0x7f];
            if (ent >> 16) v = -v;
          }
          xcol[(k >> 2) * ntn * 32 + (k & 3)] = v;
        }
      } else {
        for (int k = lane; k < a.Kpad; k += 32) xcol[(k >> 2) * ntn * 32 + (k & 3)] = 0.0;
      }
    }
    __syncthreads();
    // ---- GEMM on DMMA: warp owns m-tiles 2w, 2w+1 and all n-tiles
    double c[2][8][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    const int nta = (ncol + 7) >> 3;
    const double* A0 = a.ops + (((int64_t)cls * a.nmt + 2 * warp) * a.nks) * 32 + lane;
    const double* A1 = A0 + (int64_t)a.nks * 32;
    double an0 = __ldg(A0), an1 = __ldg(A1);
    for (int ks = 0; ks < a.nks; ++ks) {
      const double a0 = an0, a1 = an1;
      if (ks + 1 < a.nks) {  // prefetch next k-step's operator fragments
        an0 = __ldg(A0 + (ks + 1) * 32);
        an1 = __ldg(A1 + (ks + 1) * 32);
      }
      const double* bx = xy + (ks * ntn) * 32 + lane;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nta) {
          const double b = bx[j * 32];
          dmma884(c[0][j][0], c[0][j][1], a0, b);
          dmma884(c[1][j][0], c[1][j][1], a1, b);
        }
      }
    }
    __syncthreads();  // everyone is done reading X
    // ---- stage Y[col][row]
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nta) {
          const int row = 16 * warp + 8 * i + (lane >> 2);
          const int col = 8 * j + 2 * (lane & 3);
          xy[col * a.ystride + row] = c[i][j][0];
          xy[(col + 1) * a.ystride + row] = c[i][j][1];
        }
      }
    __syncthreads();
    // ---- accumulate: thread (row r, slot parity q) walks the columns in order
    for (int t = tid; t < 2 * a.NRpad; t += nthr) {
      const int r = t % a.NRpad, q = t / a.NRpad;
      if (r >= NR) continue;
      double* accr = acc + r;
      for (int col = 0; col < ncol; ++col) {
        const int mt_ = meta[col];
        const int slot = mt_ & 0xff;
        if ((slot & 1) != q) continue;
        const int ent = sym[((mt_ >> 8) * 2 + 1) * NR + r];
        const double y = xy[col * a.ystride + (ent & 0xffff)];
        accr[slot * NR] += (ent >> 16) ? -y : y;
      }
    }
  }
  __syncthreads();
  // ---- write back L = L~ h_A^{-(j+1)} for the tile's targets (L was zeroed)
  for (int e = tid; e < T * NR; e += nthr) {
    const int slot = e / NR, r = e - slot * NR;
    const int cell = a.tile_cells[tile * T + slot];
    if (cell < 0) continue;
    const int d = dec[r];
    const double v = acc[e] * a.hpow[a.level[cell] * (a.p + 2) + ((d >> 1) & 0x7f) + 1];
    ((double*)(a.L + (int64_t)cell * a.nc))[2 * (d >> 8) + (d & 1)] = v;
  }
}

}  // namespace

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
  D.T = 64;
  while (D.T > 16 && ((size_t)D.T * D.NR + (size_t)std::max(D.Kpad * D.NC, D.NC * (D.NRpad + 2))) * 8 + 8 * D.NC +
                             132 * D.NR > 200 * 1024)
    D.T /= 2;
  D.ystride = D.NRpad + 2;
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
  DevBuf<uint64_t> ckeys;
  ckeys.alloc(D.nclass);
  class_assign_kernel<<<cdiv(n, 256), 256, 0, s>>>(keys, idx, pflag, poff, n, pcls, ckeys);
  FMM_LAUNCHED("class_assign_kernel");
  if (D.nclass >= (1 << 24)) throw Error(FMM_ERR_USAGE, "m2l: too many operator classes");
  if (D.ntiles >= (1 << 28)) throw Error(FMM_ERR_USAGE, "m2l: too many tiles");

  // ---- operators (fragment order) and per-level scale table
  const int64_t opsz = (int64_t)D.nmt * D.nks * 32;
  D.ops.alloc(D.nclass * opsz);
  build_ops_kernel<<<(unsigned)D.nclass, 256, sizeof(double2) * ncoef(2 * p), s>>>(ckeys, p, D.nmt, D.nks, D.ops);
  FMM_LAUNCHED("build_ops_kernel");
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
  D.tile_chunk.alloc(D.ntiles + 1);
  tile_chunk_kernel<<<cdiv(D.nchunks + 1, 256), 256, 0, s>>>(ctile, D.nchunks, D.ntiles, D.tile_chunk);
  FMM_LAUNCHED("tile_chunk_kernel");
  FMM_CUDA(cudaStreamSynchronize(s));
}

void m2l_dmma_pass(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  FMM_CUDA(cudaMemsetAsync(P.L.ptr, 0, sizeof(double2) * P.L.count, P.stream));
  if (D.ntiles == 0) return;
  M2LArgs a;
  a.ops = D.ops;
  a.col_src = D.col_src;
  a.col_meta = D.col_meta;
  a.chunk_begin = D.chunk_begin;
  a.chunk_class = D.chunk_class;
  a.tile_chunk = D.tile_chunk;
  a.tile_cells = D.tile_cells;
  a.symtab = D.symtab;
  a.hpow = D.hpow;
  a.level = P.cells.level;
  a.M = P.M;
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
  const size_t sh = ((size_t)D.T * D.NR + (size_t)std::max(D.Kpad * D.NC, D.NC * D.ystride)) * sizeof(double) +
                    (2 * D.NC + 33 * D.NR) * sizeof(int32_t);
  static size_t configured = 0;
  if (sh > 48 * 1024 && sh > configured) {
    FMM_CUDA(cudaFuncSetAttribute(m2l_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    configured = sh;
  }
  const int threads = 32 * (D.nmt / 2 + (D.nmt & 1));
  m2l_dmma_kernel<<<(unsigned)D.ntiles, threads, sh, P.stream>>>(a);
  FMM_LAUNCHED("m2l_dmma_kernel");
}

}  // namespace fmm
