// m2l_rot.cu — S9 M2L v3 (default for p = 0..14): the translation-invariant class
// operators of v2 (m2l_dmma.cu) applied in rotation-factored form on FP64 tensor cores.
//
// Paper: M2L dominates; "Rotating the multipole expansion so that the
// translation is along the z-axis reduces the complexity from O(p^4) to O(p^3)"
// (the analytic end of the compute-memory axis); translation operators
// for boxes with the same relative positioning are identical and can be precomputed and
// stored; symmetry reduces the storage further.
//
// For a canonical class offset delta0 = rho (sin b cos a, sin b sin a, cos b) (finer half
// sides) the dense scaled operator factorises exactly (tools/proto_m2l_rotation.py checks
// it against build_ops_kernel's dense T~ to ~1e-14):
//
//   T~ = Az_L(a) . Dt(b) . Z~(rho) . D(b) . Az_M(a)
//
//   Az_M(a): (re, im) of M~_n^m  ->  e^{i m a} (re + i im)          (2x2 per (n, m))
//   D(b)   : per degree n, the rotation Ry(-b) on multipole coefficients; it does not mix
//            Re and Im: an (n+1)^2 Re block and an n^2 Im block, computed per class by an
//            exact sphere quadrature (Gauss-Legendre x trapezoid, exact to degree 2p)
//   Z~(rho): per order m the z-axis translation L~_j^m = (-1)^{n+m} (j+n)!/rho^{j+n+1}
//            fA^{j+1} fB^n M~_n^m on Re, the negative on Im ((p+1-m)^2 each)
//   Dt(b)  : per degree j, Re block E^-1 D_re^T E (E = diag(1, 2, 2, ...)), Im block D_im^T
//   Az_L(a): (re, im) of L~_j^k  ->  e^{i k a} (re + i im)
//
// Work per pair (p = 10): 3 x 891 useful MACs (1392 padded DMMA-MAC blocks of 8x8x4 per
// 64 columns) instead of the dense 121^2 = 14641 (3968 DMMAs per 64 columns).
//
// Kernel (one CTA per tile of T target cells, as v2): warp-specialised, 16 warps.
//  * 4 prep warps: load chunk i's metadata, stage its class data (A fragments, azimuths)
//    and its source multipoles M~_B (contiguous rows of Kpad doubles) into shared memory
//    with cp.async.bulk (TMA bulk copies, completion on an mbarrier), apply each column's
//    symmetry map and Az_M in place, signal the MMA warps;
//  * 8 MMA warps: the three block-GEMM stages D, Z~, Dt on DMMA (mma.sync m8n8k4 f64), each
//    IN PLACE in the chunk's shared-memory buffer. The small per-degree / per-order blocks
//    are packed block-diagonally into "items" of two fixed shapes (16 x 4 KSB, 8 x 8); an
//    item reads and writes only its own positions (all B fragments are read before the
//    first store), A fragments come pre-arranged in fragment order (one 256-byte load per
//    fragment), a named barrier separates the stages, items are spread over the warps by a
//    static LPT schedule built on the host;
//  * 4 accumulate warps: add chunk i's result (Az_L and the symmetry map applied on the fly)
//    into the tile's shared-memory accumulators in column order (deterministic, no atomics).
#include "m2l_rot.cuh"

namespace fmm {
namespace {
using namespace m2l;

// ------------------------------------------------------------------- setup: operators
__global__ void quad_points_kernel(const double* __restrict__ glx, int p, double2* __restrict__ Rs) {
  const int nphi = 2 * p + 1, np = (p + 1) * nphi, nc = ncoef(p);
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < np * (p + 1); it += gridDim.x * blockDim.x) {
    const int pt = it / (p + 1), m = it - pt * (p + 1);
    const int kx = pt / nphi, t = pt - kx * nphi;
    const double ct = glx[kx], st = sqrt(fmax(0.0, 1.0 - ct * ct));
    double sp, cp;
    sincospi(2.0 * t / nphi, &sp, &cp);
    regular_column(st * cp, st * sp, ct, m, p, Rs + (int64_t)pt * nc);
  }
}


constexpr int kRotBuildThreads = 256;
constexpr int kQuadBatch = 32;
constexpr int kMaxEntPerThread = 13;  // ceil(sum_n (n+1)^2 + n^2 at p = 16 / 256)

struct ItemDev {  // device copy of RotItem (setup only)
  int st, big, nparts, aoff;
  int slot[16];
};

// One CTA per class: azimuth table, rotation blocks by quadrature, then every item's A
// fragments in DMMA fragment order (A[8 mt + lane/4][4 ks + lane%4]).
__global__ void __launch_bounds__(kRotBuildThreads) build_rot_ops_kernel(
    const uint64_t* __restrict__ class_keys, int p, const double* __restrict__ glx, const double* __restrict__ glw,
    const double2* __restrict__ Rs, const ItemDev* __restrict__ items, int nitems, int blob,
    double* __restrict__ blobs) {
  extern __shared__ double2 sh[];  // Rq[kQuadBatch][nc], then D[nent] (doubles)
  const int nc = ncoef(p), nphi = 2 * p + 1, np = (p + 1) * nphi;
  double2* Rq = sh;
  double* Dtab = (double*)(sh + kQuadBatch * nc);
  const int cls = blockIdx.x, tid = threadIdx.x;
  const uint64_t key = class_keys[cls];
  const int dl = (int)((key >> 57) & 0x3f) - 32;
  const double x0 = (double)((key >> 38) & 0x7ffff), y0 = (double)((key >> 19) & 0x7ffff),
               z0 = (double)(key & 0x7ffff);
  const double rxy = sqrt(x0 * x0 + y0 * y0), rho = sqrt(x0 * x0 + y0 * y0 + z0 * z0);
  const double alpha = atan2(y0, x0), beta = atan2(rxy, z0);
  const double cb = cos(beta), sb = sin(beta);
  const double fA = dl < 0 ? ldexp(1.0, -dl) : 1.0, fB = dl > 0 ? ldexp(1.0, dl) : 1.0;
  double* out = blobs + (int64_t)cls * blob;
  if (tid <= p) {
    double s, c;
    sincos(tid * alpha, &s, &c);
    out[2 * tid] = c;
    out[2 * tid + 1] = s;
  }
  // entries e -> (n, part, a, b): per degree n the Re block (a, b in 0..n) then the Im
  // block (a, b in 1..n)
  int nent = 0;
  for (int n = 0; n <= p; ++n) nent += (n + 1) * (n + 1) + n * n;
  double acc[kMaxEntPerThread];
#pragma unroll
  for (int i = 0; i < kMaxEntPerThread; ++i) acc[i] = 0.0;
  for (int b0 = 0; b0 < np; b0 += kQuadBatch) {
    const int nb = min(kQuadBatch, np - b0);
    __syncthreads();
    for (int it = tid; it < nb * (p + 1); it += blockDim.x) {
      const int i = it / (p + 1), m = it - i * (p + 1);
      const int pt = b0 + i, kx = pt / nphi, t = pt - kx * nphi;
      const double ct = glx[kx], st = sqrt(fmax(0.0, 1.0 - ct * ct));
      double sp, cp;
      sincospi(2.0 * t / nphi, &sp, &cp);
      const double x = st * cp, y = st * sp, z = ct;
      regular_column(cb * x - sb * z, y, sb * x + cb * z, m, p, Rq + i * nc);  // Q = Ry(-beta)
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kMaxEntPerThread; ++q) {
      const int e = tid + q * kRotBuildThreads;
      if (e >= nent) continue;
      int n = 0, r = e;
      while (r >= (n + 1) * (n + 1) + n * n) {
        r -= (n + 1) * (n + 1) + n * n;
        ++n;
      }
      int part = 0, a, b;
      if (r < (n + 1) * (n + 1)) {
        a = r / (n + 1);
        b = r - a * (n + 1);
      } else {
        part = 1;
        r -= (n + 1) * (n + 1);
        a = 1 + r / n;
        b = 1 + r % n;
      }
      double s = 0.0;
      for (int i = 0; i < nb; ++i) {
        const int pt = b0 + i;
        const double w = glw[pt / nphi];
        const double2 u = Rq[i * nc + cidx(n, a)];
        const double2 v = Rs[(int64_t)pt * nc + cidx(n, b)];
        s = fma(w, part ? u.y * v.y : u.x * v.x, s);
      }
      acc[q] += s;
    }
  }
  // D[n][part][a][b] = (2n+1)/(2 pi) * c_{n,b}^2 * (2 pi / nphi) * sum, c^2 = (n+b)!(n-b)! (/2 at b = 0)
#pragma unroll
  for (int q = 0; q < kMaxEntPerThread; ++q) {
    const int e = tid + q * kRotBuildThreads;
    if (e >= nent) continue;
    int n = 0, r = e;
    while (r >= (n + 1) * (n + 1) + n * n) {
      r -= (n + 1) * (n + 1) + n * n;
      ++n;
    }
    const int b = r < (n + 1) * (n + 1) ? r % (n + 1) : 1 + (r - (n + 1) * (n + 1)) % n;
    double c2 = b == 0 ? 0.5 : 1.0;
    for (int k = 2; k <= n + b; ++k) c2 *= k;
    for (int k = 2; k <= n - b; ++k) c2 *= k;
    Dtab[e] = (2.0 * n + 1.0) / nphi * c2 * acc[q];
  }
  __syncthreads();
  // fragments of every item
  for (int it = 0; it < nitems; ++it) {
    const ItemDev& I = items[it];
    const int MT = I.big ? 2 : 1, KS = I.big ? rot_ksb(p) : 2;
    for (int e = tid; e < MT * KS * 32; e += blockDim.x) {
      const int lane = e & 31, fr = e >> 5, ks = fr % KS, mt = fr / KS;
      const int r = 8 * mt + (lane >> 2), k = 4 * ks + (lane & 3);
      const int sr = r < 16 ? I.slot[r] : -1, sk = k < 16 ? I.slot[k] : -1;
      double v = 0.0;
      if (sr >= 0 && sk >= 0 && (sr & 0xff) == (sk & 0xff)) {
        const int lr = sr >> 8, lk = sk >> 8;
        if (I.st == 1) {  // Z~_m[j][n]: j = m + lr, n = m + lk
          const int m = sr & 0x1f, j = m + lr, n = m + lk;
          double g = 1.0 / rho;  // (j+n)! / rho^{j+n+1}
          for (int l = 1; l <= j + n; ++l) g *= l / rho;
          for (int t = 0; t <= j; ++t) g *= fA;
          for (int t = 0; t < n; ++t) g *= fB;
          v = ((n + m) & 1) ? -g : g;
        } else {
          const int n = sr & 0x1f, part = (sr >> 5) & 1;
          const int mr = part ? lr + 1 : lr, mk = part ? lk + 1 : lk;
          const int a = I.st == 0 ? mr : mk, b = I.st == 0 ? mk : mr;  // stage 2: transposed
          int base = 0;
          for (int q = 0; q < n; ++q) base += (q + 1) * (q + 1) + q * q;
          v = part ? Dtab[base + (n + 1) * (n + 1) + (a - 1) * n + (b - 1)] : Dtab[base + a * (n + 1) + b];
          if (I.st == 2 && part == 0) v *= (mk == 0 ? 1.0 : 2.0) / (mr == 0 ? 1.0 : 2.0);  // E^-1 D^T E
        }
      }
      out[I.aoff + e] = v;
    }
  }
}

// ------------------------------------------------------------------- the mat-vec kernel
// S9 pre-pass (v3): M~ rows in the RI layout, M~[c][q] = {Re,Im} M_n^m(c) h_c^{-n}, zero for q >= NR.
__global__ void mtilde_ri_kernel(const double2* __restrict__ M, const int32_t* __restrict__ level,
                                 const double* __restrict__ hpow, int64_t ncells, int p, int nc, int NR, int Kpad,
                                 double* __restrict__ Mt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ncells * Kpad) return;
  const int64_t c = e / Kpad;
  const int q = (int)(e - c * Kpad);
  double v = 0.0;
  if (q < NR) {
    const int part = q >= nc;
    const int ci = part ? q - nc + 1 : q;  // Im plane: (n, m >= 1) -> cidx(n, m) = q - nc + n + 1
    int n = 0;
    if (part) {
      while ((n + 1) * n / 2 <= q - nc) ++n;
    } else {
      while ((n + 1) * (n + 2) / 2 <= q) ++n;
    }
    const int cix = part ? ci + n : ci;
    const double2 z = M[c * nc + cix];
    v = (part ? z.y : z.x) * hpow[level[c] * (p + 2) + n];
  }
  Mt[e] = v;
}

// Gauss-Legendre nodes and weights on [-1, 1] (Newton on P_k, host, double)
void gauss_legendre(int k, std::vector<double>& x, std::vector<double>& w) {
  x.assign(k, 0.0);
  w.assign(k, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < k; ++i) {
    double z = std::cos(pi * (i + 0.75) / (k + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int j = 2; j <= k; ++j) {
        const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      if (k == 1) p1 = z, p0 = 1.0;
      dp = k * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-17) break;
    }
    double p0 = 1.0, p1 = z;
    for (int j = 2; j <= k; ++j) {
      const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
      p0 = p1;
      p1 = p2;
    }
    dp = k * (z * p1 - p0) / (z * z - 1.0);
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}


// Per-chunk descriptor (one contiguous 16-byte-aligned record, loaded by one TMA bulk copy):
// [ncol, nseg, class, 0 | srcs[NC] | meta[NC] | sslot[NC] | sbeg[NC + 1]] (sbeg relative to the chunk)
__global__ void chunk_desc_kernel(const int32_t* __restrict__ chunk_begin, const int32_t* __restrict__ chunk_class,
                                  const int32_t* __restrict__ chunk_seg, const int32_t* __restrict__ seg_begin,
                                  const int32_t* __restrict__ col_src, const int32_t* __restrict__ col_meta,
                                  int64_t nchunks, int NC, int32_t* __restrict__ desc) {
  const int64_t ch = blockIdx.x;
  if (ch >= nchunks) return;
  int32_t* d = desc + ch * rot_desc_ints(NC);
  const int cb = chunk_begin[ch], ncol = chunk_begin[ch + 1] - cb;
  const int s0 = chunk_seg[ch], ns = chunk_seg[ch + 1] - s0;
  for (int t = threadIdx.x; t < rot_desc_ints(NC); t += blockDim.x) {
    int v = 0;
    if (t == 0) v = ncol;
    else if (t == 1) v = ns;
    else if (t == 2) v = chunk_class[ch];
    else if (t >= 4 && t < 4 + NC) v = t - 4 < ncol ? col_src[cb + t - 4] : 0;
    else if (t >= 4 + NC && t < 4 + 2 * NC) v = t - 4 - NC < ncol ? col_meta[cb + t - 4 - NC] : 0;
    else if (t >= 4 + 2 * NC && t < 4 + 3 * NC) v = t - 4 - 2 * NC < ns ? (col_meta[seg_begin[s0 + t - 4 - 2 * NC]] & 0xff) : 0;
    else if (t >= 4 + 3 * NC && t <= 4 + 4 * NC) v = t - 4 - 3 * NC <= ns ? seg_begin[s0 + t - 4 - 3 * NC] - cb : 0;
    d[t] = v;
  }
}

// Pack the blocks of every stage into items (first-fit decreasing for the small ones).
std::vector<RotItem> build_items(int p, int& blob_frag) {
  std::vector<RotItem> items;
  int aoff = 2 * (p + 1);
  for (int st = 0; st < 3; ++st) {
    struct Blk {
      int size, code, n0, m0, kind;  // kind 0: D (n, part), 1: Z (m)
    };
    std::vector<Blk> blks;
    if (st == 1) {
      for (int m = 0; m <= p; ++m) blks.push_back({p + 1 - m, m, 0, m, 1});
    } else {
      for (int n = 0; n <= p; ++n) {
        blks.push_back({n + 1, n, n, 0, 0});
        if (n > 0) blks.push_back({n, n | (1 << 5), n, 1, 0});
      }
    }
    std::stable_sort(blks.begin(), blks.end(), [](const Blk& x, const Blk& y) { return x.size > y.size; });
    std::vector<RotItem> bins;
    std::vector<int> fill;
    for (const Blk& bk : blks) {
      int target = -1;
      if (bk.size <= 8)
        for (size_t i = 0; i < bins.size(); ++i)
          if (!bins[i].big && fill[i] + bk.size <= 8) {
            target = (int)i;
            break;
          }
      if (target < 0) {
        RotItem it{};
        it.st = st;
        it.big = bk.size > 8;
        it.nparts = st == 1 ? 2 : 1;
        for (int s = 0; s < 16; ++s) it.slot[s] = -1, it.pos[0][s] = it.pos[1][s] = -1;
        bins.push_back(it);
        fill.push_back(0);
        target = (int)bins.size() - 1;
      }
      RotItem& it = bins[target];
      for (int l = 0; l < bk.size; ++l) {
        const int s = fill[target] + l;
        it.slot[s] = bk.code | (l << 8);
        if (st == 1) {  // order m, degree n = m + l
          it.pos[0][s] = ri_pos(p, bk.m0 + l, bk.m0, 0);
          it.pos[1][s] = bk.m0 > 0 ? ri_pos(p, bk.m0 + l, bk.m0, 1) : -1;
        } else {  // degree n, order m = l (+1 for Im)
          const int part = (bk.code >> 5) & 1;
          it.pos[0][s] = ri_pos(p, bk.n0, l + part, part);
        }
      }
      fill[target] += bk.size;
    }
    for (RotItem& it : bins) {
      it.aoff = aoff;
      aoff += (it.big ? 2 * rot_ksb(p) : 2) * 32;
      items.push_back(it);
    }
  }
  blob_frag = (aoff + 1) & ~1;
  return items;
}

}  // namespace

bool m2l_rot_supported(int p) { return p >= 0 && p <= 14; }
int rot_chunk_width(int p) { return rot_nc(p); }
size_t rot_smem_bytes(int p, int T, int extra_ints) {
  const int NR = (p + 1) * (p + 1), KPAD = (NR + 3) & ~3, S = rot_xstride(KPAD), nc = ncoef(p), NC = rot_nc(p);
  int blob = 0;
  std::vector<RotItem> items = build_items(p, blob);
  const int ni = (int)items.size();
  return sizeof(double) * ((size_t)T * NR + 2 * (size_t)NC * S + (rot_smem_a(p) ? 2 * (size_t)blob : 4 * (size_t)(p + 1))) +
         sizeof(uint64_t) * 6 +
         sizeof(int32_t) * (3 * rot_desc_ints(NC) + 3 * NR + nc + 4 + 4 * NC + ni + 32 * ni + 6 * kRotMMA * extra_ints);
}

void m2l_rot_setup(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  cudaStream_t s = P.stream;
  const int p = P.p;
  if (D.nclass == 0 || D.ntiles == 0) return;
  int blob = 0;
  std::vector<RotItem> items = build_items(p, blob);
  const int ni = (int)items.size();
  // quadrature (exact to degree 2p on the sphere)
  std::vector<double> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  DevBuf<double> dgx, dgw;
  DevBuf<double2> Rs;
  dgx.alloc(p + 1);
  dgw.alloc(p + 1);
  FMM_CUDA(cudaMemcpyAsync(dgx.ptr, gx.data(), sizeof(double) * (p + 1), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemcpyAsync(dgw.ptr, gw.data(), sizeof(double) * (p + 1), cudaMemcpyHostToDevice, s));
  const int np = (p + 1) * (2 * p + 1);
  Rs.alloc((int64_t)np * ncoef(p));
  quad_points_kernel<<<cdiv(np * (p + 1), 128), 128, 0, s>>>(dgx, p, Rs);
  FMM_LAUNCHED("quad_points_kernel");
  D.rot_blob = blob;
  D.rot_ops.alloc(D.nclass * blob);
  {  // symmetry masks from the signed-permutation tables (m2l_dmma.cu), rows in RI order
    const int NR = (p + 1) * (p + 1);
    std::vector<int32_t> sym = build_symtab(p);
    std::vector<uint32_t> mk(2 * NR, 0);
    for (int which = 0; which < 2; ++which)
      for (int q = 0; q < NR; ++q) {
        int n, mm, part;
        ri_decode(p, q, n, mm, part);
        const int rr = real_index(n, mm, part);
        for (int g = 0; g < 16; ++g) {
          const int ent = sym[(g * 2 + which) * NR + rr];
          if ((ent & 0xffff) != rr) mk[which * NR + q] |= 1u << (2 * g);
          if (ent >> 16) mk[which * NR + q] |= 2u << (2 * g);
        }
      }
    D.rot_masks.alloc(2 * NR);
    FMM_CUDA(cudaMemcpyAsync(D.rot_masks.ptr, mk.data(), sizeof(uint32_t) * mk.size(), cudaMemcpyHostToDevice, s));
  }
  // item tables: device copy for the build kernel, headers and positions for the mat-vec
  std::vector<ItemDev> idev(ni);
  std::vector<int32_t> hdr(ni), pos(32 * ni);
  for (int i = 0; i < ni; ++i) {
    idev[i].st = items[i].st;
    idev[i].big = items[i].big;
    idev[i].nparts = items[i].nparts;
    idev[i].aoff = items[i].aoff;
    for (int k = 0; k < 16; ++k) idev[i].slot[k] = items[i].slot[k];
    hdr[i] = items[i].big | (items[i].nparts << 1) | (items[i].aoff << 8);
    for (int k = 0; k < 16; ++k) {
      pos[32 * i + k] = items[i].pos[0][k];
      pos[32 * i + 16 + k] = items[i].pos[1][k];
    }
  }
  DevBuf<ItemDev> ditems;
  ditems.alloc(ni);
  FMM_CUDA(cudaMemcpyAsync(ditems.ptr, idev.data(), sizeof(ItemDev) * ni, cudaMemcpyHostToDevice, s));
  D.rot_ihdr.alloc(ni);
  D.rot_ipos.alloc(32 * ni);
  FMM_CUDA(cudaMemcpyAsync(D.rot_ihdr.ptr, hdr.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemcpyAsync(D.rot_ipos.ptr, pos.data(), sizeof(int32_t) * 32 * ni, cudaMemcpyHostToDevice, s));
  D.rot_nitems = ni;
  int nent = 0;
  for (int n = 0; n <= p; ++n) nent += (n + 1) * (n + 1) + n * n;
  const size_t sh = sizeof(double2) * kQuadBatch * ncoef(p) + sizeof(double) * nent;
  if (sh > 48 * 1024)  // per call: the opt-in is per device context (no process-wide cache)
    FMM_CUDA(cudaFuncSetAttribute(build_rot_ops_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  build_rot_ops_kernel<<<(unsigned)D.nclass, kRotBuildThreads, sh, s>>>(D.class_keys, p, dgx, dgw, Rs, ditems, ni,
                                                                         blob, D.rot_ops);
  FMM_LAUNCHED("build_rot_ops_kernel");
  // static LPT schedule of each stage's items over the MMA warps
  const int nmma = kRotMMA;
  std::vector<std::vector<int>> lists(3 * nmma);
  for (int st = 0; st < 3; ++st) {
    std::vector<std::pair<int, int>> its;  // (cost, id)
    for (int i = 0; i < ni; ++i)
      if (items[i].st == st)
        its.push_back({(items[i].big ? 2 * rot_ksb(p) : 2) * items[i].nparts * 8 + 24 * items[i].nparts, i});
    std::stable_sort(its.begin(), its.end(), [](auto& x, auto& y) { return x.first > y.first; });
    std::vector<int> load(nmma, 0);
    for (auto& it : its) {
      const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[w] += it.first;
      lists[st * nmma + w].push_back(it.second);
    }
  }
  int smax = 1;
  for (auto& l : lists) smax = std::max<int>(smax, (int)l.size() + 1);
  std::vector<int32_t> sched(3 * nmma * smax, -1);
  for (int i = 0; i < 3 * nmma; ++i)
    for (size_t k = 0; k < lists[i].size(); ++k) sched[i * smax + k] = lists[i][k];
  D.rot_smax = smax;
  D.rot_sched.alloc((int64_t)sched.size());
  FMM_CUDA(cudaMemcpyAsync(D.rot_sched.ptr, sched.data(), sizeof(int32_t) * sched.size(), cudaMemcpyHostToDevice, s));
  D.rot_T = D.T;
  D.rot_desc.alloc(D.nchunks * rot_desc_ints(D.NC));
  chunk_desc_kernel<<<(unsigned)D.nchunks, 128, 0, s>>>(D.chunk_begin, D.chunk_class, D.chunk_seg, D.seg_begin,
                                                         D.col_src, D.col_meta, D.nchunks, D.NC, D.rot_desc);
  FMM_LAUNCHED("chunk_desc_kernel");
  // launch order of the tiles: with few waves (<= 8 per SM) decreasing estimated work (per chunk: fixed
  // cost + its n-tiles), so the hardware's in-order CTA dispatch balances the last waves like an LPT
  // schedule; with many waves the Morton order (L2 reuse of neighbouring tiles' sources and class data
  // wins: configs[4] 463 ms Morton vs 771 ms LPT)
  int nsm = 148;
  FMM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P.device));
  if (D.ntiles <= 8LL * nsm) {
    std::vector<int32_t> tc(D.ntiles + 1), cb(D.nchunks + 1);
    FMM_CUDA(cudaMemcpyAsync(tc.data(), D.tile_chunk.ptr, sizeof(int32_t) * tc.size(), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(cb.data(), D.chunk_begin.ptr, sizeof(int32_t) * cb.size(), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    std::vector<std::pair<int64_t, int32_t>> w(D.ntiles);
    for (int64_t t = 0; t < D.ntiles; ++t) {
      int64_t c = 0;
      for (int32_t ch = tc[t]; ch < tc[t + 1]; ++ch) c += 3 + (cb[ch + 1] - cb[ch] + 7) / 8;
      w[t] = {-c, (int32_t)t};
    }
    std::sort(w.begin(), w.end());
    std::vector<int32_t> order(D.ntiles);
    for (int64_t t = 0; t < D.ntiles; ++t) order[t] = w[t].second;
    D.rot_order.alloc(D.ntiles);
    FMM_CUDA(cudaMemcpyAsync(D.rot_order.ptr, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice, s));
  } else {
    std::vector<int32_t> order(D.ntiles);
    for (int64_t t = 0; t < D.ntiles; ++t) order[t] = (int32_t)t;
    D.rot_order.alloc(D.ntiles);
    FMM_CUDA(cudaMemcpyAsync(D.rot_order.ptr, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice, s));
  }
  FMM_CUDA(cudaStreamSynchronize(s));
}

void m2l_rot_mtilde(fmm_plan_s& P) {
  M2LDmma& D = P.m2l_dmma;
  const int64_t ne = P.cells.n * D.Kpad;
  mtilde_ri_kernel<<<cdiv(ne, 256), 256, 0, P.stream>>>(P.M, P.cells.level, D.hpow, P.cells.n, P.p, P.nc, D.NR, D.Kpad,
                                                        D.Mt);
  FMM_LAUNCHED("mtilde_ri_kernel");
}

void m2l_rot_launch(fmm_plan_s& P, const m2l::M2LArgs& a) {
  M2LDmma& D = P.m2l_dmma;
  RotArgs r;
  r.a = a;
  r.blobs = D.rot_ops;
  r.masks = D.rot_masks;
  r.sched = D.rot_sched;
  r.ihdr = D.rot_ihdr;
  r.ipos = D.rot_ipos;
  r.smax = D.rot_smax;
  r.nitems = D.rot_nitems;
  r.blob = D.rot_blob;
  r.desc = D.rot_desc;
  r.order = D.rot_order;
  r.p2p_phi = nullptr;
  r.p2p_grad = nullptr;
  if (P.near_fused_active) {
    r.leaves = P.leaves.ptr + P.own_leaf_begin;
    r.nleaves = P.own_leaf_end - P.own_leaf_begin;
    r.cbeg = P.cells.begin;
    r.cend = P.cells.end;
    r.p2p_off = P.p2p.off;
    r.p2p_src = P.p2p.src;
    r.pos = P.pos;
    r.leaf_counter = P.near_counter;
    r.p2p_phi = P.near_p2p_phi;
    r.p2p_grad = P.near_fused_grad ? P.near_p2p_grad.ptr : nullptr;
  }
#ifdef FMM_DEV  // development builds only: timing experiments (most bits skip work: wrong results)
  const char* dbgs = getenv("FMM_M2L_DEBUG");
  const int dbg = dbgs ? atoi(dbgs) : 0;
#else
  const int dbg = 0;
#endif
  r.prof = nullptr;
#ifdef FMM_DEV
  DevBuf<unsigned long long> prof_buf;  // timing experiment: per-warp cycle breakdown printed to stderr
  if (dbg & 256) {
    prof_buf.alloc(8 * 32);
    FMM_CUDA(cudaMemsetAsync(prof_buf.ptr, 0, 8 * 32 * sizeof(unsigned long long), P.stream));
    r.prof = prof_buf.ptr;
  }
#endif
  const size_t sh = rot_smem_bytes(P.p, a.T, D.rot_smax);
  // split small problems' tiles over several CTAs so that the grid covers the SMs (configs[1]: 73 tiles)
  // (one CTA per SM: minimise waves / split, ties to the smaller split; configs[1] -> 2, [2] -> 1)
  int nsm = 148;
  FMM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P.device));
  int split = 1;
  double best = 1e300;
  for (int s = 1; s <= 4; s *= 2) {
    const double cost = (double)((D.ntiles * s + nsm - 1) / nsm) / s;
    if (cost < best - 1e-9) best = cost, split = s;
  }
  if (const char* s = getenv("FMM_M2L_SPLIT")) split = std::max(1, std::min(8, atoi(s)));
  void (*k)(const RotArgs, int) = nullptr;
#define FMM_ROT_CASE(PP) \
  case PP: k = split > 1 ? m2l_rot_kernel<PP, true> : m2l_rot_kernel<PP, false>; break;
  switch (P.p) {
    FMM_ROT_CASE(0) FMM_ROT_CASE(1) FMM_ROT_CASE(2) FMM_ROT_CASE(3) FMM_ROT_CASE(4) FMM_ROT_CASE(5)
    FMM_ROT_CASE(6) FMM_ROT_CASE(7) FMM_ROT_CASE(8) FMM_ROT_CASE(9) FMM_ROT_CASE(10) FMM_ROT_CASE(11)
    FMM_ROT_CASE(12) FMM_ROT_CASE(13)
    default: k = split > 1 ? m2l_rot_kernel<14, true> : m2l_rot_kernel<14, false>; break;
  }
#undef FMM_ROT_CASE
  r.scratch = nullptr;
  if (split > 1) {
    const int64_t need = D.ntiles * split * (int64_t)a.T * D.NR;
    if (D.rot_scratch.count < need) D.rot_scratch.alloc(need);
    r.scratch = D.rot_scratch.ptr;
  }
  if (sh > 48 * 1024)  // per launch: the opt-in is per device context (no process-wide cache)
    FMM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  r.split = split;
  const dim3 grid((unsigned)(D.ntiles * split)), block(32 * (kRotMMA + rot_prep_warps(P.p) + rot_acc_warps(P.p) + kRotNear));
  k<<<grid, block, sh, P.stream>>>(r, dbg);
  FMM_LAUNCHED("m2l_rot_kernel");
  if (split > 1) {
    const int64_t tot = D.ntiles * (int64_t)a.T * D.NR;
    rot_split_reduce_kernel<<<cdiv(tot, 256), 256, 0, P.stream>>>(D.rot_scratch, split, D.ntiles, a.T, D.NR, P.p,
                                                                  a.tile_cells, a.level, a.hpow, P.p, P.nc, a.L);
    FMM_LAUNCHED("rot_split_reduce_kernel");
  }
#ifdef FMM_DEV
  if (dbg & 256) {
    unsigned long long h[8 * 32];
    FMM_CUDA(cudaMemcpyAsync(h, prof_buf.ptr, sizeof(h), cudaMemcpyDeviceToHost, P.stream));
    FMM_CUDA(cudaStreamSynchronize(P.stream));
    for (int w = 0; w < kRotMMA; ++w)
      fprintf(stderr, "m2l_rot prof warp %2d: waitX %.0f  st0 %.0f  st1 %.0f  st2 %.0f  barrier %.0f  (cycles per chunk)\n",
              w, (double)h[8 * w] / h[8 * w + 5], (double)h[8 * w + 1] / h[8 * w + 5], (double)h[8 * w + 2] / h[8 * w + 5],
              (double)h[8 * w + 3] / h[8 * w + 5], (double)h[8 * w + 4] / h[8 * w + 5]);
  }
#endif
}

}  // namespace fmm
