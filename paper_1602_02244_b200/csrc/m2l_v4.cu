// m2l_v4.cu — S9 M2L v4 (default for 2 <= p <= 12): the rotation ("point-and-shoot") form of
// every M2L translation, one pair per lane, on the FP64 pipe (DFMA), with the only fixed
// operator in constant memory.
//
// Paper: M2L dominates the FMM's run time (§2.2); "Rotating the multipole
// expansion so that the translation is along the z-axis reduces the complexity from O(p^4)
// to O(p^3)". This is the analytic, matrix-free end of the paper's
// compute-memory axis: nothing per class is stored, every pair's operator is
// formed on the fly from its own geometry.
//
// Factorisation (tools/proto_m2l_v4.py checks every step against the dense formula of
// SURVEY §8(c) c.1, Lambda_j^k = sum_{n,m} (-1)^n M_n^m I_{j+n}^{k+m}(c_B - c_A)):
//   d = c_B - c_A = rho (sin b cos a, sin b sin a, cos b),   Q = Ry(-b) Rz(-a),  Q d = rho z
//   Lambda = A(Q)^T Z(rho) A(Q) M,   A(R) = action of rotation R on one degree's coefficients
//   A(Ry(-b)) = A(P) A(Rz(-b)) A(P^-1),  P = Rx(-pi/2) fixed (Ry(t) = P Rz(t) P^-1)
// In the real 2n+1 representation of a degree ([Re c0, Re c1, Im c1, Re c2, ...]):
//   A(Rz(-t))        : (re, im) of order m -> e^{i m t} (re + i im)      ("zrot(t)", 4 flops)
//   F  = A(P)        : fixed sparse real matrix, n^2 + n + 1 non-zeros (c_F4, host-computed)
//   G  = A(P^-1)     : G_ik = (-1)^{m_i + m_k} F_ik  (P^-1 = Rz(pi) P Rz(pi))
//   local side       : A(Q)^T = W^-1 zrot(a) F^T zrot(b) G^T W,  W = diag(1, 2, 2, ...)
//   Z(rho)           : per order m the Hankel matrix (j+n)! / rho^{j+n+1} (z-axis translation)
// so one pair is, per degree n:  zrot(a) -> G -> zrot(b) -> F  (multipole side),
// per order m: Hankel (z translation), per degree j: G^T -> zrot(b) -> F^T -> zrot(a) (local
// side), about 3.7K FP64 instructions at p = 10 — against 29K flops for the dense operator.
// F's entries are the same for every pair, so they are constant-bank operands of the DFMAs
// (uniform across the warp whatever the pairs; tools/cbank_probe.cu: ~32 TFLOP/s for a 4 KB
// constant working set, p = 10 uses 3.6 KB).
//
// Scaled coefficients (as v2/v3): M~_n = (-1)^n M_n / h_B^n (the (-1)^n of the formula folded
// in), Lambda~_j = Lambda_j h_A^{j+1}; distances in units of the target half side h_A, so the
// Hankel entries are k!/u^{k+1} (u = rho / h_A) and the source side carries r^n, r = h_B / h_A
// (an exact power of two).
//
// Kernel: one warp = one worker; lane = one pair. The pair list is grouped by target (S5);
// "units" are kUnitChunks runs ("chunks") of 32 consecutive pairs, dealt round-robin to the warps
// (every unit is the same work). Per chunk:
//   1. the 32 source rows M~_B are copied into the warp's shared-memory buffer (one row per
//      lane, coalesced 8-byte cp.async);
//   2. each lane transforms its row IN PLACE (degree-major layout; stage 1 per degree, stage
//      2 per order, stage 3 per degree): registers hold one degree or one order at a time;
//   3. the warp sums the rows of lanes with the same target (segmented, in lane order) into
//      per-lane running accumulators (lane k owns coefficients k, k+32, ...) — a target whose
//      pairs continue into the next chunk keeps its accumulator; a finished target is
//      written to L once. A target crossing a unit boundary leaves partial sums per unit, which a
//      small fix-up kernel adds in unit order. Fixed order everywhere: bitwise deterministic, no
//      atomics.
#include <cmath>
#include <algorithm>
#include <complex>
#include <utility>
#include <vector>

#include "plan.h"

#ifndef FMM_V4_CIMM
#define FMM_V4_CIMM 1  // pair code as a called function: fixed-operator entries at immediate addresses (LDCU.128)
#endif

namespace fmm {
namespace m2l4 {

constexpr int kMinP = 2, kMaxP4 = 12;  // orders served by v4 (others: v3 / v2)
constexpr int kUnitChunks = 4;         // chunks of 32 pairs per work unit (balanced at setup); 16 -> 4:
                                       // a CTA's warps on adjacent targets share source rows in L1
                                       // (configs[2] M2L 2.96 -> 2.78 ms, configs[3] 20.9 -> 19.8 ms)
#ifndef FMM_V4_MAXW
#define FMM_V4_MAXW 8  // register cap of the launch bounds: 8 -> 255 registers, 12 -> 168
#endif
constexpr int kMaxWarpsPerCta = FMM_V4_MAXW;  // M2L v4 CTA: up to this many one-warp workers


__host__ __device__ constexpr int nnzF(int n) { return n * n + n + 1; }
__host__ __device__ constexpr int offF(int n) {
  int s = 0;
  for (int k = 0; k < n; ++k) s += nnzF(k);
  return s;
}
constexpr int kFTotal = offF(kMaxP + 1);  // 1649 doubles (13 KB) for n = 0..16
__host__ __device__ constexpr int ridx(int m, int part) { return m == 0 ? 0 : 2 * m - 1 + part; }

// Does F_n have a (structurally) non-zero entry in row (m, pi), column (mp, pj)? Given the row
// order m and the column order mp, there is at most one: F = Rz(-pi/2) d(-pi/2) Rz(pi/2) has
// complex entries i^{m - mp} d_{m mp}(pi/2); folding m < 0 (real potential) keeps only Re
// inputs when n + m is even and only Im inputs when n + m is odd, the output part follows the
// parity of m - mp (+1 for Im inputs), and d_{m mp}(pi/2) vanishes for m = 0, n + mp odd and
// for mp = 0, n + m odd. The host build below checks this pattern against the full matrix.
__host__ __device__ constexpr bool f_entry(int n, int m, int mp, int& pi, int& pj) {
  pj = ((n + m) & 1) ? 1 : 0;
  if (mp == 0 && pj == 1) return false;
  if (m == 0 && ((n + mp) & 1)) return false;
  if (mp == 0 && ((n + m) & 1)) return false;
  pi = ((m - mp + pj) & 1) ? 1 : 0;
  if (m == 0 && pi == 1) return false;
  return true;
}
constexpr int count_pattern(int n) {
  int c = 0;
  for (int m = 0; m <= n; ++m)
    for (int mp = 0; mp <= n; ++mp) {
      int pi = 0, pj = 0;
      if (f_entry(n, m, mp, pi, pj)) ++c;
    }
  return c;
}
static_assert(count_pattern(0) == nnzF(0) && count_pattern(5) == nnzF(5) && count_pattern(10) == nnzF(10) &&
                  count_pattern(16) == nnzF(16),
              "F pattern count");

}  // namespace m2l4

namespace {
using namespace m2l4;

}  // namespace
}  // namespace fmm
// the fixed operator F (non-zeros of every degree), addressed by name from inline PTX
extern "C" {
__constant__ double fmm_c_F4[fmm::m2l4::kFTotal];
}
namespace fmm {
namespace {
using namespace m2l4;

// ------------------------------------------------------------------ host: the fixed operator
using cld = std::complex<long double>;

// R_n^m(x) for m >= 0, n <= p (Cartesian recurrences of SURVEY §8(c) c.1), long double
void host_regular(long double x, long double y, long double z, int p, std::vector<cld>& R) {
  R.assign((p + 1) * (p + 2) / 2, cld(0));
  const long double r2 = x * x + y * y + z * z;
  cld d(1);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) d = d * cld(-x / (2 * m), -y / (2 * m));
    R[cidx(m, m)] = d;
    if (m + 1 > p) continue;
    cld a = d, b = d * z;
    R[cidx(m + 1, m)] = b;
    for (int n = m + 2; n <= p; ++n) {
      const cld c = ((long double)(2 * n - 1) * z * b - r2 * a) / (long double)((n + m) * (n - m));
      R[cidx(n, m)] = c;
      a = b;
      b = c;
    }
  }
}
cld host_Rget(const std::vector<cld>& R, int n, int m) {
  if (m >= 0) return R[cidx(n, m)];
  const cld v = std::conj(R[cidx(n, -m)]);
  return (m & 1) ? -v : v;
}

// Gauss-Legendre nodes / weights on [-1, 1] (Newton on P_K), long double
void gauss_legendre(int K, std::vector<long double>& t, std::vector<long double>& w) {
  t.resize(K);
  w.resize(K);
  const long double pi = 3.14159265358979323846264338327950288L;
  for (int i = 0; i < K; ++i) {
    long double x = std::cos(pi * (i + 0.75L) / (K + 0.5L)), dp = 0;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1, p1 = x;
      for (int k = 2; k <= K; ++k) {
        const long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = K * (x * p1 - p0) / (x * x - 1);
      const long double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
    t[i] = x;
    w[i] = 2 / ((1 - x * x) * dp * dp);
  }
}

// Real (2n+1)^2 matrices of A(Rx(sgn * pi/2)) for n = 0..kMaxP, by exact sphere quadrature:
// A_{m m'} = (2n+1)(n+m')!(n-m')!/(4 pi) * integral conj R_n^m(Rx x) R_n^m'(x) dOmega
// (orthogonality of the harmonics), then folded to the real representation.
std::vector<std::vector<double>> rotation_real(int sgn) {
  const int p = kMaxP, K = p + 2, L = 2 * p + 4;
  std::vector<long double> gt, gw;
  gauss_legendre(K, gt, gw);
  const long double pi = 3.14159265358979323846264338327950288L;
  // complex A[n][(m+n)*(2n+1) + (m'+n)]
  std::vector<std::vector<cld>> A(p + 1);
  for (int n = 0; n <= p; ++n) A[n].assign((2 * n + 1) * (2 * n + 1), cld(0));
  std::vector<cld> R0, R1;
  for (int i = 0; i < K; ++i)
    for (int l = 0; l < L; ++l) {
      const long double st = std::sqrt(1 - gt[i] * gt[i]), ph = 2 * pi * l / L;
      const long double x = st * std::cos(ph), y = st * std::sin(ph), z = gt[i];
      const long double wq = gw[i] * 2 * pi / L;
      host_regular(x, y, z, p, R0);
      // Rx(-pi/2): (x, y, z) -> (x, z, -y); Rx(+pi/2): (x, y, z) -> (x, -z, y)
      if (sgn < 0)
        host_regular(x, z, -y, p, R1);
      else
        host_regular(x, -z, y, p, R1);
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          const cld a = std::conj(host_Rget(R1, n, m)) * wq;
          for (int mp = -n; mp <= n; ++mp) A[n][(m + n) * (2 * n + 1) + (mp + n)] += a * host_Rget(R0, n, mp);
        }
    }
  std::vector<std::vector<double>> F(p + 1);
  for (int n = 0; n <= p; ++n) {
    const int D = 2 * n + 1;
    for (int mp = -n; mp <= n; ++mp) {
      long double f = (2 * n + 1) / (4 * pi);
      for (int k = 2; k <= n + mp; ++k) f *= k;
      for (int k = 2; k <= n - mp; ++k) f *= k;
      for (int m = -n; m <= n; ++m) A[n][(m + n) * D + (mp + n)] *= f;
    }
    F[n].assign(D * D, 0.0);
    for (int k = 0; k < D; ++k) {  // column k: basis vector e_k of the real representation
      const int mk = (k + 1) / 2, pk = k == 0 ? 0 : ((k + 1) & 1);
      std::vector<cld> c(D, cld(0));
      const cld v = pk ? cld(0, 1) : cld(1, 0);
      c[n + mk] = v;
      if (mk > 0) c[n - mk] = (mk & 1) ? -std::conj(v) : std::conj(v);
      for (int m = 0; m <= n; ++m) {
        cld o(0);
        for (int mp = -n; mp <= n; ++mp) o += A[n][(m + n) * D + (mp + n)] * c[mp + n];
        F[n][ridx(m, 0) * D + k] = (double)o.real();
        if (m > 0) F[n][ridx(m, 1) * D + k] = (double)o.imag();
      }
    }
  }
  return F;
}

// Packed non-zeros of F in the kernels' enumeration order (m, mp), after checking the pattern
// and the sign relation G = (-1)^{m + m'} F against the separately computed A(P^-1).
std::vector<double> build_f_table() {
  const auto F = rotation_real(-1), G = rotation_real(+1);
  std::vector<double> out;
  out.reserve(kFTotal);
  for (int n = 0; n <= kMaxP; ++n) {
    const int D = 2 * n + 1;
    double mx = 0;
    for (double v : F[n]) mx = std::fmax(mx, std::fabs(v));
    std::vector<char> used(D * D, 0);
    for (int m = 0; m <= n; ++m)
      for (int mp = 0; mp <= n; ++mp) {
        int pi = 0, pj = 0;
        if (!f_entry(n, m, mp, pi, pj)) continue;
        const int r = ridx(m, pi), k = ridx(mp, pj);
        out.push_back(F[n][r * D + k]);
        used[r * D + k] = 1;
      }
    for (int r = 0; r < D; ++r)
      for (int k = 0; k < D; ++k) {
        const int mr = (r + 1) / 2, mk = (k + 1) / 2;
        const double g = ((mr + mk) & 1) ? -F[n][r * D + k] : F[n][r * D + k];
        if (std::fabs(G[n][r * D + k] - g) > 1e-13 * mx)
          throw Error(FMM_ERR_NUMERIC, "m2l v4: A(P^-1) != sign-flipped A(P) (internal)");
        if (!used[r * D + k] && std::fabs(F[n][r * D + k]) > 1e-13 * mx)
          throw Error(FMM_ERR_NUMERIC, "m2l v4: rotation pattern mismatch (internal)");
      }
  }
  if ((int)out.size() != kFTotal) throw Error(FMM_ERR_NUMERIC, "m2l v4: table size (internal)");
  return out;
}

// ------------------------------------------------------------------ device: one pair's stages
// F_N's non-zeros in enumeration order (compile time): output index r, input index k, G's sign
struct FEnt {
  int r, k, mrow, prow, mcol, pcol;
  bool gneg;
};
template <int N>
struct FTab {
  FEnt e[nnzF(N)];
};
template <int N>
constexpr FTab<N> make_ftab() {
  FTab<N> t{};
  int i = 0;
  for (int m = 0; m <= N; ++m)
    for (int mp = 0; mp <= N; ++mp) {
      int pi = 0, pj = 0;
      if (!f_entry(N, m, mp, pi, pj)) continue;
      t.e[i++] = FEnt{ridx(m, pi), ridx(mp, pj), m, pi, mp, pj, ((m + mp) & 1) != 0};
    }
  return t;
}
template <int N>
struct FTabOf {
  static constexpr FTab<N> value = make_ftab<N>();
};

// sign of a stage-3 input element (Re of order m: (-1)^m, Im: -(-1)^m: the Hankel output's sign)
__host__ __device__ constexpr bool sx_neg(int m, int part) { return part == 0 ? (m & 1) : !(m & 1); }

// y += F x (T: y += F^T x); SG: G's signs (-1)^{m + mp}; SX: stage-3 input signs
template <int N, bool T, bool SG, bool SX, int I>
__device__ __forceinline__ void fstep(const double (&x)[2 * N + 1], double (&y)[2 * N + 1], int z) {
  constexpr FEnt E = FTabOf<N>::value.e[I];
  constexpr bool neg = (SG && E.gneg) != (SX && (T ? sx_neg(E.mrow, E.prow) : sx_neg(E.mcol, E.pcol)));
#if FMM_V4_CIMM
  // immediate constant-bank address behind a volatile asm: not hoisted out of the pair loop by
  // the compiler, folded by ptxas into the DFMA's c[0x3][imm] operand (no load instruction)
  const double f = fmm_c_F4[offF(N) + I];
  (void)z;
#else
  const double f = fmm_c_F4[offF(N) + I + 2 * z];  // (2 z: 16-byte aligned, LDCU.128 pairs)
#endif
  const double c = neg ? -f : f;
  if constexpr (!T)
    y[E.r] = fma(c, x[E.k], y[E.r]);
  else
    y[E.k] = fma(c, x[E.r], y[E.k]);
}
template <int N, bool T, bool SG, bool SX, int... I>
__device__ __forceinline__ void apply_seq(const double (&x)[2 * N + 1], double (&y)[2 * N + 1],
                                          int z, std::integer_sequence<int, I...>) {
  (fstep<N, T, SG, SX, I>(x, y, z), ...);
}
// z: a run-time zero the compiler cannot see (zmask = 0), different per call site and per chunk
// and warp-uniform: the constants are loaded (LDCU, uniform datapath) right where they are used,
// never held in registers across pairs or shared between the stages
// FMM_V4_ORDER = 1 (default; configs[2] M2L 3.00 -> 2.96 ms): the entries in output-interleaved order (for y = F x sorted by input column,
// for y = F^T x by row), so consecutive FMAs go to different accumulators (the table of constants
// is unchanged: an entry keeps its index I; each accumulator sums in the same order as before, so the
// results are bitwise the same)
#ifndef FMM_V4_S2ORDER
#define FMM_V4_S2ORDER 0  // stage 2 (Hankel) FMAs output-interleaved (measured neutral)
#endif
#ifndef FMM_V4_ORDER
#define FMM_V4_ORDER 1
#endif
template <int N, bool T>
struct FOrder {
  int v[nnzF(N)];
};
template <int N, bool T>
constexpr FOrder<N, T> make_forder() {
  FOrder<N, T> o{};
  int j = 0;
  // output index of entry I is e.r (F) or e.k (F^T); its input index the other one
  for (int in = 0; in < 2 * N + 1; ++in)
    for (int I = 0; I < nnzF(N); ++I) {
      const FEnt e = FTabOf<N>::value.e[I];
      if ((T ? e.r : e.k) == in) o.v[j++] = I;
    }
  return o;
}
template <int N, bool T>
struct FOrderOf {
  static constexpr FOrder<N, T> value = make_forder<N, T>();
};
template <int N, bool T, bool SG, bool SX, int... J>
__device__ __forceinline__ void apply_perm(const double (&x)[2 * N + 1], double (&y)[2 * N + 1], int z,
                                           std::integer_sequence<int, J...>) {
  (fstep<N, T, SG, SX, FOrderOf<N, T>::value.v[J]>(x, y, z), ...);
}
template <int N, bool T, bool SG, bool SX>
__device__ __forceinline__ void apply_fixed(const double (&x)[2 * N + 1], double (&y)[2 * N + 1], int z) {
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) y[i] = 0.0;
#if FMM_V4_ORDER
  apply_perm<N, T, SG, SX>(x, y, z, std::make_integer_sequence<int, nnzF(N)>{});
#else
  apply_seq<N, T, SG, SX>(x, y, z, std::make_integer_sequence<int, nnzF(N)>{});
#endif
}

// (re, im) of order m -> e^{i m t} (re + i im), m = 1..N; cs[m] = (cos mt, sin mt)
template <int N>
__device__ __forceinline__ void zrot(double (&x)[2 * N + 1], const double2* cs) {
#pragma unroll
  for (int m = 1; m <= N; ++m) {
    const double re = x[2 * m - 1], im = x[2 * m];
    x[2 * m - 1] = fma(cs[m].x, re, -cs[m].y * im);
    x[2 * m] = fma(cs[m].y, re, cs[m].x * im);
  }
}

// stage 1 (multipole side) of degree N, in place in the lane's row w (degree-major)
template <int N>
__device__ __forceinline__ void stage1(double* w, double rn, const double2* ca, const double2* cb, int z0, int z1) {
  double x[2 * N + 1], t[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = w[N * N + i] * rn;
  zrot<N>(x, ca);
  apply_fixed<N, false, true, false>(x, t, z0);
  zrot<N>(t, cb);
  apply_fixed<N, false, false, false>(t, x, z1);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = x[i];
}

// stage 2: z-axis translation of order M, part PART (Hankel h[j + n]); m = 0 rows halved
// (the W / V bookkeeping of the local side: V = diag(2, 1, ...), A(Q)^T = V X V^-1)
template <int P, int M, int PART>
__device__ __forceinline__ void stage2(double* w, const double* h) {
  constexpr int L = P + 1 - M;
  double a[L], y[L];
#pragma unroll
  for (int i = 0; i < L; ++i) a[i] = w[(M + i) * (M + i) + ridx(M, PART)];
#if FMM_V4_S2ORDER
  // n outer, j inner: consecutive FMAs to different outputs (each output sums over n in the same
  // order as below: bitwise the same)
#pragma unroll
  for (int j = 0; j < L; ++j) y[j] = 0.0;
#pragma unroll
  for (int n = 0; n < L; ++n)
#pragma unroll
    for (int j = 0; j < L; ++j) y[j] = fma(h[2 * M + j + n], a[n], y[j]);
  if (M == 0) {
#pragma unroll
    for (int j = 0; j < L; ++j) y[j] *= 0.5;
  }
#else
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s = 0.0;
#pragma unroll
    for (int n = 0; n < L; ++n) s = fma(h[2 * M + j + n], a[n], s);
    y[j] = M == 0 ? 0.5 * s : s;
  }
#endif
#pragma unroll
  for (int i = 0; i < L; ++i) w[(M + i) * (M + i) + ridx(M, PART)] = y[i];
}

// stage 3 (local side) of degree N, in place
template <int N>
__device__ __forceinline__ void stage3(double* w, const double2* ca, const double2* cb, int z0, int z1) {
  double x[2 * N + 1], t[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = w[N * N + i];
  apply_fixed<N, true, true, true>(x, t, z0);
  zrot<N>(t, cb);
  apply_fixed<N, true, false, false>(t, x, z1);
  zrot<N>(x, ca);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = x[i];
}

// (the empty asm with a memory clobber keeps the compiler from hoisting the next degree's
// shared-memory loads above this degree's stores: one degree / order live at a time)
__device__ __forceinline__ void order_fence() { asm volatile("" ::: "memory"); }
// blocks smaller than this many degrees are not fenced (the compiler may overlap them: more ILP
// where one degree / order alone has little)
#ifndef FMM_V4_STAGE_SYNC
#define FMM_V4_STAGE_SYNC 3  // CTA barriers between the stages: 0 none, 1 after stages 1 and 2, 2 after stage 1 only,
                             // 3 after stage 2 only (with no chunk-end barrier; configs[2] M2L: 0 -> 3.85 ms, the warps
                             // fetch the 112 KB of unrolled code apart; 1 2.64, 2 2.71, 3 2.64; configs[3] 20.7 / 18.3 / 18.4 / 18.1)
#endif
#ifndef FMM_V4_CHUNK_SYNC
#define FMM_V4_CHUNK_SYNC 0  // CTA barrier at the end of every chunk too (configs[2] M2L 2.64 ms without, 2.79 with;
                             // configs[3] 18.3 vs 19.8 ms: the warps' copy + segmented-sum imbalance waited on)
#endif
#ifndef FMM_V4_FENCE_MIN
#define FMM_V4_FENCE_MIN 0
#endif
#ifndef FMM_V4_COPY_ALIGNED
#define FMM_V4_COPY_ALIGNED 0  // cp.async instructions on 256-byte-aligned shared-memory windows (5 per row instead of
                                // 4): measured slower (configs[2] M2L 2.63 -> 2.71 ms); the copy's 480 wavefronts per
                                // chunk (242 ideal) are not a line-alignment effect
#endif
#ifndef FMM_V4_REFILL
#define FMM_V4_REFILL 0  // rows refilled with the next chunk's sources inside the segmented sum (measured: configs[2]
                         // M2L 2.63 -> 2.63 ms, configs[3] 18.1 -> 19.7 ms: the copy's latency was not the cost; kept off)
#endif
#ifndef FMM_V4_SKEW
#define FMM_V4_SKEW 0  // k > 0 (with FMM_V4_STAGE_SYNC=0): the chunk's one CTA barrier is taken by warps 0-3 after degree
                       // P - k of stage 1 and by the other warps at the end of stage 1, so the two warps of a scheduler
                       // run k degree steps apart (one's shared-memory bursts under the other's FP64 bursts) while
                       // both stay inside the instruction cache's window
#endif
#ifndef FMM_V4_GROUPS
#define FMM_V4_GROUPS 1  // the CTA's warps in this many barrier groups (contiguous warps: one warp of each group per
                         // scheduler), each in step on its own named barrier: one group's copy / segmented-sum
                         // phases under another's FP64 phases, at the price of that many instruction streams
#endif
#ifndef FMM_V4_SKEW_NS
#define FMM_V4_SKEW_NS 0  // group g starts g * this many ns late
#endif

// the stage barrier of the calling warp's group
__device__ __forceinline__ void stage_barrier() {
#if FMM_V4_GROUPS > 1
  const int nw = blockDim.x >> 5, g = (int)(threadIdx.x >> 5) * FMM_V4_GROUPS / nw;
  const int lo = (g * nw + FMM_V4_GROUPS - 1) / FMM_V4_GROUPS, hi = ((g + 1) * nw + FMM_V4_GROUPS - 1) / FMM_V4_GROUPS;
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(32 * (hi - lo)) : "memory");
#else
  __syncthreads();
#endif
}

template <int P, int N = 0>
__device__ __forceinline__ void stage1_all(double* w, double r, double rn, const double2* ca, const double2* cb,
                                           const int (&z)[4]) {
  stage1<N>(w, rn, ca, cb, z[0], z[1]);
  if constexpr (N >= FMM_V4_FENCE_MIN) order_fence();
#if FMM_V4_SKEW
  if constexpr (N == (P > FMM_V4_SKEW ? P - FMM_V4_SKEW : 0)) {
    if (threadIdx.x < 128) asm volatile("bar.sync 0;" ::: "memory");
  }
  if constexpr (N == P) {
    if (threadIdx.x >= 128) asm volatile("bar.sync 0;" ::: "memory");
  }
#endif
  if constexpr (N < P) stage1_all<P, N + 1>(w, r, rn * r, ca, cb, z);
}
template <int P, int M = 0>
__device__ __forceinline__ void stage2_all(double* w, const double* h) {
  stage2<P, M, 0>(w, h);
  if constexpr (P - M >= FMM_V4_FENCE_MIN) order_fence();
  if constexpr (M > 0) stage2<P, M, 1>(w, h);
  if constexpr (P - M >= FMM_V4_FENCE_MIN) order_fence();
  if constexpr (M < P) stage2_all<P, M + 1>(w, h);
}
#ifndef FMM_V4_PIPE
#define FMM_V4_PIPE 0  // software pipelining of the lane's shared-memory loads: the next step's inputs are loaded
                       // before this step's FMAs (bit 0: stage 1, bit 1: stage 2, bit 2: stage 3); same arithmetic
#endif
#ifndef FMM_V4_PIPE_MAX
#define FMM_V4_PIPE_MAX 8  // stages 1 / 3: highest degree whose inputs are loaded a step ahead (registers)
#endif

// stage 2 with the next (order, part)'s column loaded a step ahead
template <int P, int M, int PART>
__device__ __forceinline__ void stage2_pipe(double* w, const double* h, const double (&a)[P + 1 - M]) {
  constexpr int L = P + 1 - M;
  constexpr bool last = M == P && (PART == 1 || M == 0);
  constexpr int MN = (PART == 0 && M > 0) ? M : M + 1, PN = (PART == 0 && M > 0) ? 1 : 0;
  double an[last ? 1 : P + 1 - MN];
  if constexpr (!last) {
#pragma unroll
    for (int i = 0; i < P + 1 - MN; ++i) an[i] = w[(MN + i) * (MN + i) + ridx(MN, PN)];
  }
  double y[L];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s = 0.0;
#pragma unroll
    for (int n = 0; n < L; ++n) s = fma(h[2 * M + j + n], a[n], s);
    y[j] = M == 0 ? 0.5 * s : s;
  }
#pragma unroll
  for (int i = 0; i < L; ++i) w[(M + i) * (M + i) + ridx(M, PART)] = y[i];
  order_fence();
  if constexpr (!last) stage2_pipe<P, MN, PN>(w, h, an);
}
template <int P>
__device__ __forceinline__ void stage2_piped(double* w, const double* h) {
  double a0[P + 1];
#pragma unroll
  for (int i = 0; i < P + 1; ++i) a0[i] = w[i * i];
  stage2_pipe<P, 0, 0>(w, h, a0);
}

// stages 1 / 3 with the next degree's inputs loaded a step ahead (degrees <= FMM_V4_PIPE_MAX)
template <int P, int N>
__device__ __forceinline__ void stage1_pipe(double* w, double r, double rn, const double2* ca, const double2* cb,
                                            const int (&z)[4], const double (&xin)[2 * N + 1]) {
  constexpr bool pre = N < P && N + 1 <= FMM_V4_PIPE_MAX;
  double xn[N < P ? 2 * N + 3 : 1];
  if constexpr (pre) {
#pragma unroll
    for (int i = 0; i < 2 * N + 3; ++i) xn[i] = w[(N + 1) * (N + 1) + i];
  }
  double x[2 * N + 1], t[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = xin[i] * rn;
  zrot<N>(x, ca);
  apply_fixed<N, false, true, false>(x, t, z[0]);
  zrot<N>(t, cb);
  apply_fixed<N, false, false, false>(t, x, z[1]);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = x[i];
  order_fence();
  if constexpr (N < P) {
    if constexpr (!pre) {
#pragma unroll
      for (int i = 0; i < 2 * N + 3; ++i) xn[i] = w[(N + 1) * (N + 1) + i];
    }
    stage1_pipe<P, N + 1>(w, r, rn * r, ca, cb, z, xn);
  }
}
template <int P, int N>
__device__ __forceinline__ void stage3_pipe(double* w, const double2* ca, const double2* cb, const int (&z)[4],
                                            const double (&xin)[2 * N + 1]) {
  constexpr bool pre = N < P && N + 1 <= FMM_V4_PIPE_MAX;
  double xn[N < P ? 2 * N + 3 : 1];
  if constexpr (pre) {
#pragma unroll
    for (int i = 0; i < 2 * N + 3; ++i) xn[i] = w[(N + 1) * (N + 1) + i];
  }
  double x[2 * N + 1], t[2 * N + 1];
  apply_fixed<N, true, true, true>(xin, t, z[2]);
  zrot<N>(t, cb);
  apply_fixed<N, true, false, false>(t, x, z[3]);
  zrot<N>(x, ca);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = x[i];
  order_fence();
  if constexpr (N < P) {
    if constexpr (!pre) {
#pragma unroll
      for (int i = 0; i < 2 * N + 3; ++i) xn[i] = w[(N + 1) * (N + 1) + i];
    }
    stage3_pipe<P, N + 1>(w, ca, cb, z, xn);
  }
}

template <int P, int N = 0>
__device__ __forceinline__ void stage3_all(double* w, const double2* ca, const double2* cb, const int (&z)[4]) {
  stage3<N>(w, ca, cb, z[2], z[3]);
  if constexpr (N >= FMM_V4_FENCE_MIN) order_fence();
  if constexpr (N < P) stage3_all<P, N + 1>(w, ca, cb, z);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 1/sqrt(x) to full double precision: MUFU seed (rsqrt.approx.ftz.f64, ~2^-20; x is a squared
// distance >= 1 in target half sides, never subnormal), a Newton step and a third-order step
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x * y, y, 1.0);
  return fma(y, fma(0.375, e, 0.5) * e, y);
}

struct V4Args {
  const int32_t* tgt;      // [npairs] grouped by target
  const int32_t* src;
  int64_t npairs, nunits;  // units: uchunks chunks of 32 pairs of the flat list
  int uchunks;
 const double4* center;   // cells: x, y, z, h
  const double* ihalf;     // [ncells] 1 / h
  const int32_t* level;
  const double* Mt;        // [ncells][NR] (-1)^n M_n / h^n, degree-major real
  double2* L;              // [ncells][nc]
  double* part;            // [nunits][2][NR] partial sums of targets crossing unit boundaries
  int zmask;               // 0 (see apply_fixed)
};

template <int P>
struct V4Geo {
  static constexpr int NR = (P + 1) * (P + 1);
  static constexpr int NRS = NR | 1;  // odd row stride: lane-private 8-byte accesses conflict-free
  static constexpr int KPL = (NR + 31) / 32;
};

#ifndef FMM_V4_REP
#define FMM_V4_REP 0  // one code body for both fixed-operator applications of a stage, run twice over the row:
                      // G = S F S with S = diag((-1)^m) = the z-rotation by pi, folded into the angles, so
                      //   stage 1 = T(b + pi) T(a + pi),           T(t) = F zrot(t)
                      //   stage 3 = S U(a + pi) U(b + pi) K,       U(t) = zrot(t) F^T, K = conjugation (the sign of
                      // stage 2's Im outputs), S applied once per target in write_target; r^n moves to stage 2's
                      // input. 31 % fewer unique instructions per pair for two more passes over the row in shared
                      // memory; parity-tested, measured slower (configs[2] M2L 2.62 -> 3.14 ms, configs[3] 18.1 ->
                      // 20.8 ms: the added shared-memory wavefronts cost their full time, profiles/r2_m2l_bound.md); off.
#endif
#ifndef FMM_V4_REP_MINP
#define FMM_V4_REP_MINP 11  // orders from this one up use the shared-body form: at p = 12 the pair function is 140 KB and
                            // the kernel waits on instructions (no_instruction 2.9 warps per issue, FP64 pipe 24 %):
                            // configs[4] M2L 227 -> 216 ms (202 ms with the passes per degree group)
#endif
template <int P>
constexpr bool use_rep = FMM_V4_REP != 0 || P >= FMM_V4_REP_MINP;
// Lambda = V Lambda~ / h^{j+1} (V: m = 0 entries x 2) of target t from the per-lane sums (lane k
// owns real coefficients q = k + 32 c), into the complex (n, m >= 0) layout of L
template <int P>
__device__ __forceinline__ void write_target(const V4Args& a, int t, const double (&acc)[V4Geo<P>::KPL], int lane) {
  constexpr int NR = V4Geo<P>::NR;
  const double ih = a.ihalf[t];
  double* Lc = (double*)(a.L + (int64_t)t * ((P + 1) * (P + 2) / 2));
#pragma unroll
  for (int c = 0; c < V4Geo<P>::KPL; ++c) {
    const int q = lane + 32 * c;
    if (q >= NR) continue;
    int j = 0;
    while ((j + 1) * (j + 1) <= q) ++j;
    const int r = q - j * j, m = (r + 1) >> 1, part = r > 0 ? ((r + 1) & 1) : 0;
    double s = m == 0 ? 2.0 * ih : ih;
    if constexpr (use_rep<P>) {
      if (m & 1) s = -s;  // the deferred S = diag((-1)^m) of stage 3 (shared-body form)
    }
    for (int k = 0; k < j; ++k) s *= ih;
    Lc[2 * cidx(j, m) + part] = acc[c] * s;
  }
}

// a finished segment of target t in unit u: written to L if the target lies inside the unit,
// else its partial sum goes to part[u][0] (target began in an earlier unit) or part[u][1]
template <int P>
__device__ __forceinline__ void finish_segment(const V4Args& a, int64_t u, int t, bool from_prev, bool to_next,
                                            const double (&acc)[V4Geo<P>::KPL], int lane) {
  constexpr int NR = V4Geo<P>::NR;
  if (!from_prev && !to_next) {
    write_target<P>(a, t, acc, lane);
    return;
  }
  double* d = a.part + (u * 2 + (from_prev ? 0 : 1)) * NR;
#pragma unroll
  for (int c = 0; c < V4Geo<P>::KPL; ++c)
    if (lane + 32 * c < NR) d[lane + 32 * c] = acc[c];
}

template <int N>
__device__ __forceinline__ void body1(double* w, const double2* cs) {
  double x[2 * N + 1], t[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = w[N * N + i];
  zrot<N>(x, cs);
  apply_fixed<N, false, false, false>(x, t, 0);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = t[i];
}
template <int N>
__device__ __forceinline__ void body3(double* w, const double2* cs) {
  double x[2 * N + 1], t[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = w[N * N + i];
  apply_fixed<N, true, false, false>(x, t, 0);
  zrot<N>(t, cs);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = t[i];
}
template <int P, int N = 0>
__device__ __forceinline__ void body1_all(double* w, const double2* cs) {
  body1<N>(w, cs);
  order_fence();
  if constexpr (N < P) body1_all<P, N + 1>(w, cs);
}
template <int P, int N = 0>
__device__ __forceinline__ void body3_all(double* w, const double2* cs) {
  body3<N>(w, cs);
  order_fence();
  if constexpr (N < P) body3_all<P, N + 1>(w, cs);
}
// stage 2 with the source scaling r^n on its input and conjugated (negated Im) output
template <int P, int M, int PART>
__device__ __forceinline__ void stage2r(double* w, const double* h, const double* rp) {
  constexpr int L = P + 1 - M;
  double a[L], y[L];
#pragma unroll
  for (int i = 0; i < L; ++i) a[i] = w[(M + i) * (M + i) + ridx(M, PART)] * rp[M + i];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s = 0.0;
#pragma unroll
    for (int n = 0; n < L; ++n) s = PART ? fma(-h[2 * M + j + n], a[n], s) : fma(h[2 * M + j + n], a[n], s);
    y[j] = M == 0 ? 0.5 * s : s;
  }
#pragma unroll
  for (int i = 0; i < L; ++i) w[(M + i) * (M + i) + ridx(M, PART)] = y[i];
}
template <int P, int M = 0>
__device__ __forceinline__ void stage2r_all(double* w, const double* h, const double* rp) {
  stage2r<P, M, 0>(w, h, rp);
  order_fence();
  if constexpr (M > 0) stage2r<P, M, 1>(w, h, rp);
  order_fence();
  if constexpr (M < P) stage2r_all<P, M + 1>(w, h, rp);
}
template <int P>
__device__ __forceinline__ void phasors(double2 (&cs)[P + 1], double2 e) {
  cs[0] = make_double2(1.0, 0.0);
  cs[1] = e;
#pragma unroll
  for (int m = 2; m <= P; ++m)
    cs[m] = make_double2(fma(cs[m - 1].x, e.x, -cs[m - 1].y * e.y), fma(cs[m - 1].x, e.y, cs[m - 1].y * e.x));
}
// one pass of a stage over the row: called twice (two call sites, one copy of the code; not a loop — inside
// a loop the compiler would hoist the fixed operator's constants into registers and spill them)
template <int P>
__device__ __noinline__ void pass1(double* w, double2 e) {
  double2 cs[P + 1];
  phasors<P>(cs, e);
  body1_all<P>(w, cs);
}
template <int P>
__device__ __noinline__ void pass3(double* w, double2 e) {
  double2 cs[P + 1];
  phasors<P>(cs, e);
  body3_all<P>(w, cs);
}
template <int P>
__device__ __noinline__ void pass2(double* w, double r, double iu) {
  double h[2 * P + 1], rp[P + 1];  // Hankel entries k! / u^{k+1}; r^n
  h[0] = iu;
#pragma unroll
  for (int k = 1; k <= 2 * P; ++k) h[k] = h[k - 1] * (k * iu);
  rp[0] = 1.0;
#pragma unroll
  for (int n = 1; n <= P; ++n) rp[n] = rp[n - 1] * r;
  stage2r_all<P>(w, h, rp);
}
#ifndef FMM_V4_REP_S2SPLIT
#define FMM_V4_REP_S2SPLIT 1  // stage 2 of the orders m >= 1 as one function called for the Re and then the Im parts (the
                              // same Hankel products one coefficient further along the row; the conjugation K as the
                              // sign of r^n): its code is fetched once (configs[4] M2L 201.9 -> 190.4 ms)
#endif
// stage 2 of order M >= 1 for one part: wp = w + part (the part's coefficient of degree n sits at n^2 + 2M - 1 + part)
template <int P, int M>
__device__ __forceinline__ void stage2p(double* wp, const double* h, const double* rp) {
  constexpr int L = P + 1 - M;
  double a[L], y[L];
#pragma unroll
  for (int i = 0; i < L; ++i) a[i] = wp[(M + i) * (M + i) + 2 * M - 1] * rp[M + i];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double t = 0.0;
#pragma unroll
    for (int n = 0; n < L; ++n) t = fma(h[2 * M + j + n], a[n], t);
    y[j] = t;
  }
#pragma unroll
  for (int i = 0; i < L; ++i) wp[(M + i) * (M + i) + 2 * M - 1] = y[i];
}
template <int P, int M = 1>
__device__ __forceinline__ void stage2p_all(double* wp, const double* h, const double* rp) {
  stage2p<P, M>(wp, h, rp);
  order_fence();
  if constexpr (M < P) stage2p_all<P, M + 1>(wp, h, rp);
}
template <int P>
__device__ __noinline__ void pass2g(double* wp, double r, double iu, double sgn) {
  double h[2 * P + 1], rp[P + 1];  // Hankel entries k! / u^{k+1}; sgn r^n
  h[0] = iu;
#pragma unroll
  for (int k = 1; k <= 2 * P; ++k) h[k] = h[k - 1] * (k * iu);
  rp[0] = sgn;
#pragma unroll
  for (int n = 1; n <= P; ++n) rp[n] = rp[n - 1] * r;
  stage2p_all<P>(wp, h, rp);
}
template <int P>
__device__ __noinline__ void pass2m0(double* w, double r, double iu) {
  double h[2 * P + 1], rp[P + 1];
  h[0] = iu;
#pragma unroll
  for (int k = 1; k <= 2 * P; ++k) h[k] = h[k - 1] * (k * iu);
  rp[0] = 1.0;
#pragma unroll
  for (int n = 1; n <= P; ++n) rp[n] = rp[n - 1] * r;
  stage2r<P, 0, 0>(w, h, rp);
}
#ifndef FMM_V4_REP_GROUPS
#define FMM_V4_REP_GROUPS 1  // the two passes of a stage taken per group of degrees (a stage acts on each degree alone):
                             // a group's code (<= ~14 KB) is still in the 32 KB L1.5 instruction cache for its second
                             // call, where a whole-stage pass (34 KB at p = 12) has evicted itself (configs[4] M2L
                             // 216.1 -> 202.0 ms)
#endif
template <int P, int N0, int N1, int N = N0>
__device__ __forceinline__ void body1_range(double* w, const double2* cs) {
  body1<N>(w, cs);
  order_fence();
  if constexpr (N < N1) body1_range<P, N0, N1, N + 1>(w, cs);
}
template <int P, int N0, int N1, int N = N0>
__device__ __forceinline__ void body3_range(double* w, const double2* cs) {
  body3<N>(w, cs);
  order_fence();
  if constexpr (N < N1) body3_range<P, N0, N1, N + 1>(w, cs);
}
template <int P, int N0, int N1>
__device__ __noinline__ void pass1g(double* w, double2 e) {
  double2 cs[N1 + 1];
  phasors<N1>(cs, e);
  body1_range<P, N0, N1>(w, cs);
}
template <int P, int N0, int N1>
__device__ __noinline__ void pass3g(double* w, double2 e) {
  double2 cs[N1 + 1];
  phasors<N1>(cs, e);
  body3_range<P, N0, N1>(w, cs);
}
template <int P>
__device__ __forceinline__ void pair_transform_rep(double* w, double r, double2 e1, double2 e2, double iu) {
  const double2 ea = make_double2(-e1.x, -e1.y), eb = make_double2(-e2.x, -e2.y);  // angles a + pi, b + pi
  constexpr bool grouped = FMM_V4_REP_GROUPS != 0 && P >= 8;
  constexpr int G1 = P - 4, G2 = P - 2;  // degree groups [0, G1], (G1, G2], (G2, P]: about equal code
  if constexpr (grouped) {
    pass1g<P, 0, G1>(w, ea);
    pass1g<P, 0, G1>(w, eb);
    pass1g<P, G1 + 1, G2>(w, ea);
    pass1g<P, G1 + 1, G2>(w, eb);
    pass1g<P, G2 + 1, P>(w, ea);
    pass1g<P, G2 + 1, P>(w, eb);
  } else {
    pass1<P>(w, ea);
    pass1<P>(w, eb);
  }
#if FMM_V4_REP_S2SPLIT
  pass2m0<P>(w, r, iu);
  pass2g<P>(w, r, iu, 1.0);
  pass2g<P>(w + 1, r, iu, -1.0);
#else
  pass2<P>(w, r, iu);
#endif
#if FMM_V4_STAGE_SYNC == 1 || FMM_V4_STAGE_SYNC == 3
  stage_barrier();
#endif
  if constexpr (grouped) {
    pass3g<P, 0, G1>(w, eb);
    pass3g<P, 0, G1>(w, ea);
    pass3g<P, G1 + 1, G2>(w, eb);
    pass3g<P, G1 + 1, G2>(w, ea);
    pass3g<P, G2 + 1, P>(w, eb);
    pass3g<P, G2 + 1, P>(w, ea);
  } else {
    pass3<P>(w, eb);
    pass3<P>(w, ea);
  }
}
#ifndef FMM_V4_TMEM
#define FMM_V4_TMEM 0  // the lane-private hand-offs stage 1 -> 2 -> 3 through tensor memory (32x32b tcgen05.st / ld:
                       // thread i <-> TMEM lane i, the row as 2 NR 32-bit columns) instead of shared memory:
                       // 4 of the 8 passes over the row leave the shared-memory pipe (orders p <= 10, <= 8 warps).
                       // 1: one double per access (x2); 2: degree blocks as x4..x32 pieces, stage 2's Re / Im as x4.
                       // Parity green (127 GPU tests each); measured slower: configs[2] M2L 2.63 -> 2.73 (1) / 2.85 ms
                       // (2), configs[3] 18.1 -> 18.7 / 18.1 ms: tensor-memory reads cost at least the shared-memory
                       // wavefronts they replace (profiles/r2_m2l_bound.md); off.
#endif
template <int P>
constexpr bool use_tmem = FMM_V4_TMEM != 0 && P <= 10 && !use_rep<P>;
__shared__ uint32_t tm_base_s;  // the CTA's tensor-memory allocation (written by tcgen05.alloc)
// the calling warp's region, from warp-uniform values only (a uniform-register address for LDTM / STTM)
__device__ __forceinline__ uint32_t tm_warp_base() {
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  return tm_base_s + ((warp & 3u) << 21) + (warp >> 2) * 256u;
}

__device__ __forceinline__ void tm_st(uint32_t addr, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(__double2loint(v)),
               "r"(__double2hiint(v))
               : "memory");
}
__device__ __forceinline__ void tm_ld(uint32_t addr, int& lo, int& hi) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(addr) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// the loaded halves are defined only after tm_wait_ld: this keeps their uses behind it
__device__ __forceinline__ double tm_value(int lo, int hi) {
  asm volatile("" : "+r"(lo), "+r"(hi));
  return __hiloint2double(hi, lo);
}

// K consecutive 32-bit columns of the calling thread's TMEM lane (K a power of two)
template <int K>
__device__ __forceinline__ void tm_ldk(uint32_t addr, int* r);
template <int K>
__device__ __forceinline__ void tm_stk(uint32_t addr, const int* r);
template <>
__device__ __forceinline__ void tm_ldk<2>(uint32_t addr, int* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr) : "memory");
}
template <>
__device__ __forceinline__ void tm_stk<2>(uint32_t addr, const int* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(r[0]), "r"(r[1]) : "memory");
}
template <>
__device__ __forceinline__ void tm_ldk<4>(uint32_t addr, int* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr) : "memory");
}
template <>
__device__ __forceinline__ void tm_stk<4>(uint32_t addr, const int* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}
template <>
__device__ __forceinline__ void tm_ldk<8>(uint32_t addr, int* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(addr) : "memory");
}
template <>
__device__ __forceinline__ void tm_stk<8>(uint32_t addr, const int* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
template <>
__device__ __forceinline__ void tm_ldk<16>(uint32_t addr, int* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(addr) : "memory");
}
template <>
__device__ __forceinline__ void tm_stk<16>(uint32_t addr, const int* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
template <>
__device__ __forceinline__ void tm_ldk<32>(uint32_t addr, int* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(addr) : "memory");
}
template <>
__device__ __forceinline__ void tm_stk<32>(uint32_t addr, const int* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}

constexpr int pow2_le(int c) { return c >= 32 ? 32 : c >= 16 ? 16 : c >= 8 ? 8 : c >= 4 ? 4 : 2; }
// C columns (even) from / to column offset OFF of the block at addr, in power-of-two pieces
template <int C, int OFF = 0>
__device__ __forceinline__ void tm_ld_block(uint32_t addr, int* r) {
  constexpr int K = pow2_le(C);
  tm_ldk<K>(addr + OFF, r + OFF);
  if constexpr (C > K) tm_ld_block<C - K, OFF + K>(addr, r);
}
template <int C, int OFF = 0>
__device__ __forceinline__ void tm_st_block(uint32_t addr, const int* r) {
  constexpr int K = pow2_le(C);
  tm_stk<K>(addr + OFF, r + OFF);
  if constexpr (C > K) tm_st_block<C - K, OFF + K>(addr, r);
}
template <int N>
__device__ __forceinline__ void stage1_t(const double* w, uint32_t tm, double rn, const double2* ca, const double2* cb) {
  double x[2 * N + 1], t[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = w[N * N + i] * rn;
  zrot<N>(x, ca);
  apply_fixed<N, false, true, false>(x, t, 0);
  zrot<N>(t, cb);
  apply_fixed<N, false, false, false>(t, x, 0);
#if FMM_V4_TMEM >= 2
  int rr[2 * (2 * N + 1)];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) {
    rr[2 * i] = __double2loint(x[i]);
    rr[2 * i + 1] = __double2hiint(x[i]);
  }
  tm_st_block<2 * (2 * N + 1)>(tm + 2 * N * N, rr);
#else
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) tm_st(tm + 2 * (N * N + i), x[i]);
#endif
}
template <int P, int M, int PART>
__device__ __forceinline__ void stage2_t(uint32_t tm, const double* h) {
  constexpr int L = P + 1 - M;
  int lo[L], hi[L];
  double a[L], y[L];
#pragma unroll
  for (int i = 0; i < L; ++i) tm_ld(tm + 2 * ((M + i) * (M + i) + ridx(M, PART)), lo[i], hi[i]);
  tm_wait_ld();
#pragma unroll
  for (int i = 0; i < L; ++i) a[i] = tm_value(lo[i], hi[i]);
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s = 0.0;
#pragma unroll
    for (int n = 0; n < L; ++n) s = fma(h[2 * M + j + n], a[n], s);
    y[j] = M == 0 ? 0.5 * s : s;
  }
#pragma unroll
  for (int i = 0; i < L; ++i) tm_st(tm + 2 * ((M + i) * (M + i) + ridx(M, PART)), y[i]);
}
// stage 2 of order M >= 1, Re and Im together (adjacent in the row: one x4 access per degree)
template <int P, int M>
__device__ __forceinline__ void stage2_t4(uint32_t tm, const double* h) {
  constexpr int L = P + 1 - M;
  int rr[L][4];
  double ar[L], ai[L];
#pragma unroll
  for (int i = 0; i < L; ++i) tm_ldk<4>(tm + 2 * ((M + i) * (M + i) + 2 * M - 1), rr[i]);
  tm_wait_ld();
#pragma unroll
  for (int i = 0; i < L; ++i) {
    ar[i] = tm_value(rr[i][0], rr[i][1]);
    ai[i] = tm_value(rr[i][2], rr[i][3]);
  }
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int n = 0; n < L; ++n) sr = fma(h[2 * M + j + n], ar[n], sr);
#pragma unroll
    for (int n = 0; n < L; ++n) si = fma(h[2 * M + j + n], ai[n], si);
    rr[j][0] = __double2loint(sr);
    rr[j][1] = __double2hiint(sr);
    rr[j][2] = __double2loint(si);
    rr[j][3] = __double2hiint(si);
  }
#pragma unroll
  for (int i = 0; i < L; ++i) tm_stk<4>(tm + 2 * ((M + i) * (M + i) + 2 * M - 1), rr[i]);
}
template <int N>
__device__ __forceinline__ void stage3_t(double* w, uint32_t tm, const double2* ca, const double2* cb) {
  double x[2 * N + 1], t[2 * N + 1];
#if FMM_V4_TMEM >= 2
  int rr[2 * (2 * N + 1)];
  tm_ld_block<2 * (2 * N + 1)>(tm + 2 * N * N, rr);
  tm_wait_ld();
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = tm_value(rr[2 * i], rr[2 * i + 1]);
#else
  int lo[2 * N + 1], hi[2 * N + 1];
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) tm_ld(tm + 2 * (N * N + i), lo[i], hi[i]);
  tm_wait_ld();
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) x[i] = tm_value(lo[i], hi[i]);
#endif
  apply_fixed<N, true, true, true>(x, t, 0);
  zrot<N>(t, cb);
  apply_fixed<N, true, false, false>(t, x, 0);
  zrot<N>(x, ca);
#pragma unroll
  for (int i = 0; i < 2 * N + 1; ++i) w[N * N + i] = x[i];
}
template <int P, int N = 0>
__device__ __forceinline__ void stage1_t_all(const double* w, uint32_t tm, double r, double rn, const double2* ca,
                                             const double2* cb) {
  stage1_t<N>(w, tm, rn, ca, cb);
  order_fence();
  if constexpr (N < P) stage1_t_all<P, N + 1>(w, tm, r, rn * r, ca, cb);
}
template <int P, int M = 0>
__device__ __forceinline__ void stage2_t_all(uint32_t tm, const double* h) {
#if FMM_V4_TMEM >= 2
  if constexpr (M == 0)
    stage2_t<P, 0, 0>(tm, h);
  else
    stage2_t4<P, M>(tm, h);
#else
  stage2_t<P, M, 0>(tm, h);
  if constexpr (M > 0) stage2_t<P, M, 1>(tm, h);
#endif
  if constexpr (M < P) stage2_t_all<P, M + 1>(tm, h);
}
template <int P, int N = 0>
__device__ __forceinline__ void stage3_t_all(double* w, uint32_t tm, const double2* ca, const double2* cb) {
  stage3_t<N>(w, tm, ca, cb);
  order_fence();
  if constexpr (N < P) stage3_t_all<P, N + 1>(w, tm, ca, cb);
}
template <int P>
__device__ __noinline__ void pair_transform_tmem(double* w, double r, double2 e1, double2 e2, double iu) {
  const uint32_t tm = tm_warp_base();
  double2 ca[P + 1], cb[P + 1];
  ca[0] = cb[0] = make_double2(1.0, 0.0);
  ca[1] = e1;
  cb[1] = e2;
#pragma unroll
  for (int m = 2; m <= P; ++m) {
    ca[m] = make_double2(fma(ca[m - 1].x, e1.x, -ca[m - 1].y * e1.y), fma(ca[m - 1].x, e1.y, ca[m - 1].y * e1.x));
    cb[m] = make_double2(fma(cb[m - 1].x, e2.x, -cb[m - 1].y * e2.y), fma(cb[m - 1].x, e2.y, cb[m - 1].y * e2.x));
  }
  stage1_t_all<P>(w, tm, r, 1.0, ca, cb);
  tm_wait_st();
  double h[2 * P + 1];  // Hankel entries k! / u^{k+1}
  h[0] = iu;
#pragma unroll
  for (int k = 1; k <= 2 * P; ++k) h[k] = h[k - 1] * (k * iu);
  stage2_t_all<P>(tm, h);
  tm_wait_st();
#if FMM_V4_STAGE_SYNC == 1 || FMM_V4_STAGE_SYNC == 3
  stage_barrier();
#endif
  stage3_t_all<P>(w, tm, ca, cb);
}

#if FMM_V4_CIMM
// one pair's rotation-translation-rotation, in place in the lane's row w. Not inlined: the fixed
// operator's constant-bank entries are then DFMA operands at immediate addresses (no load
// instruction) that the compiler cannot hoist out of the chunk loop into registers.
template <int P>
__device__ __noinline__ void pair_transform(double* w, double r, double2 e1, double2 e2, double iu) {
  double2 ca[P + 1], cb[P + 1];
  ca[0] = cb[0] = make_double2(1.0, 0.0);
  ca[1] = e1;
  cb[1] = e2;
#pragma unroll
  for (int m = 2; m <= P; ++m) {
    ca[m] = make_double2(fma(ca[m - 1].x, e1.x, -ca[m - 1].y * e1.y), fma(ca[m - 1].x, e1.y, ca[m - 1].y * e1.x));
    cb[m] = make_double2(fma(cb[m - 1].x, e2.x, -cb[m - 1].y * e2.y), fma(cb[m - 1].x, e2.y, cb[m - 1].y * e2.x));
  }
  const int z[4] = {0, 0, 0, 0};
#if FMM_V4_PIPE & 1
  {
    const double x0[1] = {w[0]};
    stage1_pipe<P, 0>(w, r, 1.0, ca, cb, z, x0);
  }
#else
  stage1_all<P>(w, r, 1.0, ca, cb, z);
#endif
#if FMM_V4_STAGE_SYNC == 1 || FMM_V4_STAGE_SYNC == 2
  stage_barrier();
#endif
  double h[2 * P + 1];  // Hankel entries k! / u^{k+1}
  h[0] = iu;
#pragma unroll
  for (int k = 1; k <= 2 * P; ++k) h[k] = h[k - 1] * (k * iu);
#if FMM_V4_PIPE & 2
  stage2_piped<P>(w, h);
#else
  stage2_all<P>(w, h);
#endif
#if FMM_V4_STAGE_SYNC == 1 || FMM_V4_STAGE_SYNC == 3
  stage_barrier();
#endif
#if FMM_V4_PIPE & 4
  {
    const double x0[1] = {w[0]};
    stage3_pipe<P, 0>(w, ca, cb, z, x0);
  }
#else
  stage3_all<P>(w, ca, cb, z);
#endif
}
#endif

template <int P>
__global__ void __launch_bounds__(32 * kMaxWarpsPerCta, 1) m2l_v4_kernel(const V4Args a) {
  using G = V4Geo<P>;
  constexpr int NR = G::NR, NRS = G::NRS, KPL = G::KPL;
  const int64_t UP = 32 * (int64_t)a.uchunks;
  extern __shared__ __align__(256) double sm4[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* const wb = sm4 + (size_t)warp * 32 * NRS;
  double* const w = wb + lane * NRS;
  // tensor memory: all 512 columns of the SM (one CTA per SM); warp k owns lanes 32 (k % 4) .. + 31 (the only
  // ones it can address) and columns 256 (k / 4) .. + 2 NR - 1
  if constexpr (use_tmem<P>) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&tm_base_s))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // static round-robin over equal-work units; every warp of the CTA runs the same number of
  // units and chunks (a barrier after each stage keeps the warps on the same instructions:
  // the unrolled code is larger than the instruction cache, so warps in step share its fetches)
  const int64_t per_round = (int64_t)gridDim.x * nw;
#if FMM_V4_GROUPS > 1 && FMM_V4_SKEW_NS > 0
  for (int k = warp * FMM_V4_GROUPS / nw; k > 0; --k) __nanosleep(FMM_V4_SKEW_NS);
#endif
  const int rounds = (int)((a.nunits + per_round - 1) / per_round);
#if FMM_V4_REFILL
  // FMM_V4_REFILL: a row of the warp's buffer is refilled with the NEXT chunk's source row (of this unit or of
  // the warp's next unit) as soon as the segmented sum has read it, so the copies' issue and L2 latency run
  // under the sum and the next chunk's geometry instead of after them (same sums in the same order).
  auto chunk_range = [&](int it, int ich, int64_t& base, int& nact) {
    const int64_t u = ((int64_t)it * gridDim.x + blockIdx.x) * nw + warp;
    const int64_t u0 = min(u * UP, a.npairs), u1 = min(u0 + UP, a.npairs);
    base = u0 + 32 * ich;
    nact = (int)max((int64_t)0, min((int64_t)32, u1 - base));
  };
  int64_t base_n = 0;
  int nact_n = 0, tg_next = -1, sr_next = 0;
  auto copy_row = [&](int l) {  // row l of the next chunk (l warp-uniform, < nact_n)
    const int s = __shfl_sync(0xffffffffu, sr_next, l);
    const double* g = a.Mt + (int64_t)s * NR;
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int q = lane + 32 * c;
      if (q < NR) cp_async8(wb + l * NRS + q, g + q);
    }
  };
  if (rounds > 0) {
    chunk_range(0, 0, base_n, nact_n);
    tg_next = lane < nact_n ? a.tgt[base_n + lane] : -1;
    sr_next = lane < nact_n ? a.src[base_n + lane] : 0;
#pragma unroll 8
    for (int l = 0; l < nact_n; ++l) copy_row(l);
  }
#endif
  for (int it = 0; it < rounds; ++it) {
    const int64_t u = ((int64_t)it * gridDim.x + blockIdx.x) * nw + warp;  // may be >= nunits: idle
    const int64_t u0 = min(u * UP, a.npairs), u1 = min(u0 + UP, a.npairs);
    const int tprev = u0 > 0 && u0 < a.npairs ? a.tgt[u0 - 1] : -1;  // target continued from the previous unit
    const int tnext = u1 < a.npairs ? a.tgt[u1] : -1;               // target continued in the next unit
    int cur = -1;
    double acc[KPL];
#pragma unroll
    for (int c = 0; c < KPL; ++c) acc[c] = 0.0;
#if !FMM_V4_REFILL
    // the chunk's (target, source) pairs, loaded one chunk ahead (their latency off the critical path)
    int tg_next = lane < u1 - u0 ? a.tgt[u0 + lane] : -1, sr_next = lane < u1 - u0 ? a.src[u0 + lane] : 0;
#endif
    for (int ich = 0; ich < a.uchunks; ++ich) {
#if FMM_V4_REFILL
      const int nact = nact_n;
      const bool act = lane < nact;
      const int tg = tg_next, sr = sr_next;
      if (it + 1 < rounds || ich + 1 < a.uchunks) {
        const bool same = ich + 1 < a.uchunks;
        chunk_range(same ? it : it + 1, same ? ich + 1 : 0, base_n, nact_n);
      } else {
        nact_n = 0;
      }
      tg_next = lane < nact_n ? a.tgt[base_n + lane] : -1;
      sr_next = lane < nact_n ? a.src[base_n + lane] : 0;
#else
      const int64_t base = u0 + 32 * ich;
      const int nact = (int)max((int64_t)0, min((int64_t)32, u1 - base));
      const bool act = lane < nact;
      const int tg = tg_next, sr = sr_next;
      {
        const int64_t nb = base + 32 + lane;
        tg_next = nb < u1 ? a.tgt[nb] : -1;
        sr_next = nb < u1 ? a.src[nb] : 0;
      }
      // 1. source rows into the lanes' buffers (coalesced: row by row)
#if FMM_V4_COPY_ALIGNED
      // every cp.async instruction writes one 256-byte-aligned window of shared memory (two wavefronts):
      // the rows start at odd 8-byte offsets, so a row is KPL + 1 windows with the ends masked
#pragma unroll 8
      for (int l = 0; l < nact; ++l) {
        const int s = __shfl_sync(0xffffffffu, sr, l);
        const int off = l * NRS, q0 = lane - (off & 31);  // the lane's coefficient in the row's first window
        const double* g = a.Mt + (int64_t)s * NR;
        double* d = wb + off;
#pragma unroll
        for (int c = 0; c <= KPL; ++c) {
          const int q = q0 + 32 * c;
          if (q >= 0 && q < NR) cp_async8(d + q, g + q);
        }
      }
#else
#pragma unroll 8
      for (int l = 0; l < nact; ++l) {
        const int s = __shfl_sync(0xffffffffu, sr, l);
        const double* g = a.Mt + (int64_t)s * NR;
#pragma unroll
        for (int c = 0; c < KPL; ++c) {
          const int q = lane + 32 * c;
          if (q < NR) cp_async8(wb + l * NRS + q, g + q);
        }
      }
#endif
#endif
      // geometry of the lane's pair (overlaps the copies)
      // (inactive lanes of a ragged chunk run the same code on the chunk's first pair and their
      // own stale rows — no divergence, results unused: the stages stay warp-uniform)
      double2 e1, e2;
#if !FMM_V4_CIMM
      double2 ca[P + 1], cb[P + 1];
#endif
      double r = 1.0, iu = 0.0;
      // (no IEEE division or sqrt here: their slow-path subroutine calls would force every
      // loop-carried value out of the uniform registers; rsqrt is inline)
      {
        int tgi = __shfl_sync(0xffffffffu, tg, act ? lane : 0), sri = __shfl_sync(0xffffffffu, sr, act ? lane : 0);
        if (nact == 0) tgi = sri = 0;  // idle chunk: any valid cell (results unused)
        const double4 A = a.center[tgi], B = a.center[sri];
        const double ih = a.ihalf[tgi];
        const double dx = (B.x - A.x) * ih, dy = (B.y - A.y) * ih, dz = (B.z - A.z) * ih;
        const double rxy2 = dx * dx + dy * dy, u2 = rxy2 + dz * dz;
        iu = rsqrt_nr(u2);
        if (rxy2 > 0.0) {
          const double ir = rsqrt_nr(rxy2);
          e1 = make_double2(dx * ir, dy * ir);
          e2 = make_double2(dz * iu, rxy2 * ir * iu);
        } else {
          e1 = make_double2(1.0, 0.0);
          e2 = make_double2(dz * iu, 0.0);
        }
        r = __hiloint2double((1023 + a.level[tgi] - a.level[sri]) << 20, 0);  // h_B / h_A = 2^{l_A - l_B}
      }
#if FMM_V4_CIMM
      cp_async_wait_all();
      __syncwarp();
      if constexpr (use_rep<P>)
        pair_transform_rep<P>(w, r, e1, e2, iu);
      else if constexpr (use_tmem<P>)
        pair_transform_tmem<P>(w, r, e1, e2, iu);
      else
        pair_transform<P>(w, r, e1, e2, iu);
#else
      ca[0] = cb[0] = make_double2(1.0, 0.0);
      ca[1] = e1;
      cb[1] = e2;
#pragma unroll
      for (int m = 2; m <= P; ++m) {
        ca[m] = make_double2(fma(ca[m - 1].x, e1.x, -ca[m - 1].y * e1.y), fma(ca[m - 1].x, e1.y, ca[m - 1].y * e1.x));
        cb[m] = make_double2(fma(cb[m - 1].x, e2.x, -cb[m - 1].y * e2.y), fma(cb[m - 1].x, e2.y, cb[m - 1].y * e2.x));
      }
      cp_async_wait_all();
      __syncwarp();
      // 2. the pair's rotation-translation-rotation, in place
      {
        int z[4];
        int zc;
        asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(zc));  // re-read per chunk: uniform (S2UR), opaque
#pragma unroll
        for (int k = 0; k < 4; ++k) z[k] = (zc * (k + 1)) & a.zmask;
        stage1_all<P>(w, r, 1.0, ca, cb, z);
#if FMM_V4_STAGE_SYNC
        __syncthreads();
#endif
        double h[2 * P + 1];  // Hankel entries k! / u^{k+1}
        h[0] = iu;
#pragma unroll
        for (int k = 1; k <= 2 * P; ++k) h[k] = h[k - 1] * (k * iu);
        stage2_all<P>(w, h);
#if FMM_V4_STAGE_SYNC
        __syncthreads();
#endif
        stage3_all<P>(w, ca, cb, z);
      }
#endif
      __syncwarp();
      // 3. segmented sum over lanes with the same target: segments (runs of one target in the
      // target-grouped list) from a ballot; within a segment four interleaved partial sums
      // (rows s0+k, s0+k+4, ...) combined as (p0 + p1) + (p2 + p3): a fixed order, four
      // independent add chains per coefficient instead of one
      {
        const int prev_tg = __shfl_up_sync(0xffffffffu, tg, 1);
        unsigned starts = __ballot_sync(0xffffffffu, act && (lane == 0 || tg != prev_tg));
        while (starts) {
          const int s0 = __ffs(starts) - 1;
          starts &= starts - 1;
          const int s1 = starts ? __ffs(starts) - 1 : nact;
          const int t = __shfl_sync(0xffffffffu, tg, s0);
          if (t != cur) {
            if (cur >= 0) finish_segment<P>(a, u, cur, cur == tprev, false, acc, lane);
            cur = t;
#pragma unroll
            for (int c = 0; c < KPL; ++c) acc[c] = 0.0;
          }
#if FMM_V4_REFILL
          double ps[KPL][4];
#pragma unroll
          for (int c = 0; c < KPL; ++c) ps[c][0] = ps[c][1] = ps[c][2] = ps[c][3] = 0.0;
          int l = s0;
          for (; l + 3 < s1; l += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int c = 0; c < KPL; ++c)
                if (lane + 32 * c < NR) ps[c][j] += wb[(l + j) * NRS + lane + 32 * c];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (l + j < nact_n) copy_row(l + j);
          }
          for (; l < s1; ++l) {
#pragma unroll
            for (int c = 0; c < KPL; ++c)
              if (lane + 32 * c < NR) ps[c][0] += wb[l * NRS + lane + 32 * c];
            if (l < nact_n) copy_row(l);
          }
#pragma unroll
          for (int c = 0; c < KPL; ++c) acc[c] += (ps[c][0] + ps[c][1]) + (ps[c][2] + ps[c][3]);
#else
#pragma unroll
          for (int c = 0; c < KPL; ++c) {
            const int k = lane + 32 * c;
            if (k >= NR) continue;
            double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
            int l = s0;
            for (; l + 3 < s1; l += 4) {
              p0 += wb[l * NRS + k];
              p1 += wb[(l + 1) * NRS + k];
              p2 += wb[(l + 2) * NRS + k];
              p3 += wb[(l + 3) * NRS + k];
            }
            for (; l < s1; ++l) p0 += wb[l * NRS + k];
            acc[c] += (p0 + p1) + (p2 + p3);
          }
#endif
        }
#if FMM_V4_REFILL
        for (int l = nact; l < nact_n; ++l) copy_row(l);  // rows the finished chunk did not use
#endif
      }
#if FMM_V4_CHUNK_SYNC
      __syncthreads();
#else
      __syncwarp();
#endif
    }
    if (cur >= 0) finish_segment<P>(a, u, cur, cur == tprev, cur == tnext, acc, lane);
  }
  if constexpr (use_tmem<P>) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base_s) : "memory");
  }
}

// Targets crossing unit boundaries: one warp per unit whose last target continues into the next
// unit and began in this one; partial sums added in unit order (deterministic), then written.
template <int P>
__global__ void m2l_v4_fixup_kernel(const V4Args a) {
  using G = V4Geo<P>;
  constexpr int NR = G::NR, KPL = G::KPL;
  const int64_t UP = 32 * (int64_t)a.uchunks;
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u >= a.nunits) return;
  const int64_t u0 = u * UP, u1 = min(u0 + UP, a.npairs);
  if (u1 >= a.npairs) return;
  const int t = a.tgt[u1 - 1];
  if (a.tgt[u1] != t) return;                 // last target ends inside this unit
  if (u0 > 0 && a.tgt[u0 - 1] == t) return;   // began in an earlier unit: handled there
  double acc[KPL];
#pragma unroll
  for (int c = 0; c < KPL; ++c) acc[c] = lane + 32 * c < NR ? a.part[(u * 2 + 1) * NR + lane + 32 * c] : 0.0;
  for (int64_t v = u + 1; v < a.nunits; ++v) {
#pragma unroll
    for (int c = 0; c < KPL; ++c)
      if (lane + 32 * c < NR) acc[c] += a.part[(v * 2) * NR + lane + 32 * c];
    const int64_t v1 = min((v + 1) * UP, a.npairs);
    if (v1 >= a.npairs || a.tgt[v1] != t) break;  // t ends in unit v
  }
  write_target<P>(a, t, acc, lane);
}

// M~[c][q] = (-1)^n {Re, Im} M_n^m(c) / h_c^n, degree-major real layout q = n^2 + ridx(m, part)
__global__ void m2l4_mtilde_kernel(const double2* __restrict__ M, const double4* __restrict__ center, int64_t ncells,
                                   int p, int nc, int NR, double* __restrict__ Mt, double* __restrict__ ihalf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells * NR) return;
  const int64_t c = i / NR;
  const int q = (int)(i - c * NR);
  if (q == 0) ihalf[c] = 1.0 / center[c].w;
  int n = 0;
  while ((n + 1) * (n + 1) <= q) ++n;
  const int t = q - n * n, m = (t + 1) >> 1, part = t > 0 ? ((t + 1) & 1) : 0;
  const double2 v = M[c * nc + cidx(n, m)];
  const double ih = 1.0 / center[c].w;
  double s = (n & 1) ? -1.0 : 1.0;
  for (int k = 0; k < n; ++k) s *= ih;
  Mt[i] = (part ? v.y : v.x) * s;
}

// launch geometry (setup): warps per CTA from shared memory and registers, units sized so every
// warp gets the same number of units (as close to kUnitChunks chunks as that allows)
template <int P>
void size_v4(fmm_plan_s& P_, int64_t npairs) {
  using G = V4Geo<P>;
  M2L4& V = P_.m2l4;
  const size_t sh = (size_t)32 * G::NRS * sizeof(double);
  int nsm = 148;
  FMM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P_.device));
  cudaFuncAttributes fa;
  FMM_CUDA(cudaFuncGetAttributes(&fa, m2l_v4_kernel<P>));
  const size_t dyn_max = (size_t)227 * 1024 - fa.sharedSizeBytes;  // (static: the tensor-memory base, if used)
  FMM_CUDA(cudaFuncSetAttribute(m2l_v4_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max));
  const int by_smem = (int)(dyn_max / sh), by_regs = 65536 / (32 * std::max(1, fa.numRegs));
  const int fit = std::max(1, std::min({by_smem, by_regs, kMaxWarpsPerCta}));
  V.wpc = std::max(1, std::min(V.warps_per_sm > 0 ? V.warps_per_sm : fit, fit));
  V.smem = sh * V.wpc;
  const int64_t nchunks = (npairs + 31) / 32, warps = (int64_t)nsm * V.wpc;
  V.uchunks = V.unit_chunks;
  if (V.uchunks <= 0) {
    const int64_t rounds = std::max<int64_t>(1, (nchunks + warps * kUnitChunks - 1) / (warps * kUnitChunks));
    V.uchunks = (int)std::max<int64_t>(1, (nchunks + rounds * warps - 1) / (rounds * warps));
  }
  V.nunits = (nchunks + V.uchunks - 1) / V.uchunks;
  V.grid = (int)std::max<int64_t>(1, std::min<int64_t>(nsm, (V.nunits + V.wpc - 1) / V.wpc));
  V.part.alloc(V.nunits * 2 * G::NR);
}

template <int P>
void launch_v4(fmm_plan_s& P_, const V4Args& a) {
  const M2L4& V = P_.m2l4;
  m2l_v4_kernel<P><<<(unsigned)V.grid, 32 * V.wpc, V.smem, P_.stream>>>(a);
  FMM_LAUNCHED("m2l_v4_kernel");
  if (a.nunits > 1) {
    m2l_v4_fixup_kernel<P><<<cdiv(a.nunits, 4), 128, 0, P_.stream>>>(a);
    FMM_LAUNCHED("m2l_v4_fixup_kernel");
  }
}

template <int P>
void dispatch_v4(fmm_plan_s& P_, const V4Args* a, int64_t npairs) {  // a == nullptr: size at setup
  if (a)
    launch_v4<P>(P_, *a);
  else
    size_v4<P>(P_, npairs);
}

void v4_switch(fmm_plan_s& P, const V4Args* a, int64_t npairs = 0) {
  switch (P.p) {
#ifdef FMM_V4_ONLY  // development builds: one instantiation (compile time)
    case FMM_V4_ONLY: dispatch_v4<FMM_V4_ONLY>(P, a, npairs); break;
#else
    case 2: dispatch_v4<2>(P, a, npairs); break;
    case 3: dispatch_v4<3>(P, a, npairs); break;
    case 4: dispatch_v4<4>(P, a, npairs); break;
    case 5: dispatch_v4<5>(P, a, npairs); break;
    case 6: dispatch_v4<6>(P, a, npairs); break;
    case 7: dispatch_v4<7>(P, a, npairs); break;
    case 8: dispatch_v4<8>(P, a, npairs); break;
    case 9: dispatch_v4<9>(P, a, npairs); break;
    case 10: dispatch_v4<10>(P, a, npairs); break;
    case 11: dispatch_v4<11>(P, a, npairs); break;
    case 12: dispatch_v4<12>(P, a, npairs); break;
#endif
    default: throw Error(FMM_ERR_USAGE, "m2l v4: order out of range");
  }
}

}  // namespace

bool m2l_v4_supported(int p) { return p >= kMinP && p <= kMaxP4; }

void m2l_v4_setup(fmm_plan_s& P) {
  static const std::vector<double> table = build_f_table();  // host copy, same for every plan (thread-safe init)
  FMM_CUDA(cudaMemcpyToSymbolAsync(fmm_c_F4, table.data(), sizeof(double) * kFTotal, 0, cudaMemcpyHostToDevice,
                                   P.stream));
  M2L4& V = P.m2l4;
  const int NR = (P.p + 1) * (P.p + 1);
  V.Mt.alloc(P.cells.n * NR);
  V.ihalf.alloc(P.cells.n);
  const char* w = getenv("FMM_V4_WARPS");
  V.warps_per_sm = w ? atoi(w) : 0;
  const char* uc = getenv("FMM_V4_UNIT_CHUNKS");  // tests: small units cross many targets
  V.unit_chunks = uc ? atoi(uc) : 0;
  V.nunits = 0;
  if (P.m2l.n > 0) v4_switch(P, nullptr, P.m2l.n);
  FMM_CUDA(cudaStreamSynchronize(P.stream));
}

// multi-GPU (LET): units over the rank-local pair list (targets overlapping the owned range)
void m2l_v4_resize(fmm_plan_s& P, int64_t npairs) {
  P.m2l4.nunits = 0;
  if (npairs > 0) v4_switch(P, nullptr, npairs);
}

void m2l_v4_pass(fmm_plan_s& P) {
  M2L4& V = P.m2l4;
  FMM_CUDA(cudaMemsetAsync(P.L.ptr, 0, sizeof(double2) * P.L.count, P.stream));
  if (V.nunits == 0) return;
  const int NR = (P.p + 1) * (P.p + 1);
  const int64_t ne = P.cells.n * NR;
  m2l4_mtilde_kernel<<<cdiv(ne, 256), 256, 0, P.stream>>>(P.M, P.cells.center, P.cells.n, P.p, P.nc, NR, V.Mt,
                                                           V.ihalf);
  FMM_LAUNCHED("m2l4_mtilde_kernel");
  V4Args a;
  const bool own = P.let_ready;  // LET: the pairs of targets overlapping the owned range
  a.tgt = own ? P.let_dev.m2l_tgt.ptr : P.m2l.tgt.ptr;
  a.src = own ? P.let_dev.m2l_src.ptr : P.m2l.src.ptr;
  a.npairs = own ? P.let_dev.m2l_tgt.count : P.m2l.n;
  a.nunits = V.nunits;
  a.uchunks = V.uchunks;
  a.center = P.cells.center;
  a.ihalf = V.ihalf;
  a.level = P.cells.level;
  a.Mt = V.Mt;
  a.L = P.L;
  a.part = V.part;
  a.zmask = 0;
  v4_switch(P, &a);
}

}  // namespace fmm
