/*
 * oracle/fmm_oracle.c — TEST INFRASTRUCTURE ONLY (see fmm_oracle.h).
 *
 * A plain, slow, obviously-correct CPU FMM for the 3D Laplace kernel 1/r,
 * written from arXiv:1602.02244 and the readings fixed in DESIGN.md (which
 * adopts SURVEY.md §8(c)). Nothing here is shared with the CUDA path.
 *
 * Paper passages followed (PAPER.md line numbers):
 *   - far field approximated by multipole/local expansions over a
 *     hierarchically decomposed domain: PAPER.md:22-24 (§1);
 *   - M2L translation of spherical-harmonic expansions is the dominant step:
 *     PAPER.md:149-153 (§2.2 "Fast Translation Operators");
 *   - parent boxes as coarser sources, dual tree traversal + multipole
 *     acceptance criterion builds the interaction lists: PAPER.md:161-168;
 *   - direct operator = dense diagonal blocks, translation operators =
 *     off-diagonal blocks: PAPER.md:191-196;
 *   - 3-D -> 1-D locality (Morton) ordering: PAPER.md:328-334 (§3.1).
 * The paper prints no formulas; the harmonics, recurrences and operator
 * formulas are SURVEY.md §8(c) c.1 and the algorithm is §8(c) c.2 A1–A16.
 *
 * Compiled with -O2 -ffp-contract=off -fno-fast-math (A3: no FMA contraction
 * in the quantisation or the MAC).
 */
#include "fmm_oracle.h"

#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define MAXLEVEL 21

/* ---------------------------------------------------------------- helpers */

static inline int64_t cidx(int n, int m) { return (int64_t)n * (n + 1) / 2 + m; } /* m >= 0 */
static inline int ncoef(int p) { return (p + 1) * (p + 2) / 2; }

/* A_n^m for any |m| <= n from m >= 0 storage: A_n^{-m} = (-1)^m conj(A_n^m)  (c.1) */
static cplx getc(const cplx* A, int n, int m) {
  if (m >= 0) return A[cidx(n, m)];
  cplx v = conj(A[cidx(n, -m)]);
  return ((-m) & 1) ? -v : v;
}

/* ------------------------------------------------------ solid harmonics (c.1) */

/* Regular solid harmonic R_n^m = r^n P_n^m(cos t) e^{i m phi} / (n+m)!, by the
 * Cartesian recurrences of SURVEY §8(c) c.1 (CS phase). */
static void harm_R(double x, double y, double z, int p, cplx* R) {
  double r2 = x * x + y * y + z * z;
  cplx w = x + I * y;
  R[0] = 1.0;
  for (int m = 0; m <= p; ++m) {
    if (m > 0) R[cidx(m, m)] = -w / (2.0 * m) * R[cidx(m - 1, m - 1)];
    if (m + 1 <= p) R[cidx(m + 1, m)] = z * R[cidx(m, m)];
    for (int n = m + 2; n <= p; ++n)
      R[cidx(n, m)] = ((2.0 * n - 1.0) * z * R[cidx(n - 1, m)] - r2 * R[cidx(n - 2, m)]) /
                      ((double)(n + m) * (double)(n - m));
  }
}

/* Irregular solid harmonic I_n^m = (n-m)! P_n^m(cos t) e^{i m phi} / r^{n+1}. */
static void harm_I(double x, double y, double z, int p, cplx* Iv) {
  double r2 = x * x + y * y + z * z;
  double inv_r2 = 1.0 / r2;
  cplx w = x + I * y;
  Iv[0] = 1.0 / sqrt(r2);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) Iv[cidx(m, m)] = -(2.0 * m - 1.0) * w * inv_r2 * Iv[cidx(m - 1, m - 1)];
    if (m + 1 <= p) Iv[cidx(m + 1, m)] = (2.0 * m + 1.0) * z * inv_r2 * Iv[cidx(m, m)];
    for (int n = m + 2; n <= p; ++n)
      Iv[cidx(n, m)] = ((2.0 * n - 1.0) * z * Iv[cidx(n - 1, m)] -
                        ((double)(n - 1) * (n - 1) - (double)m * m) * Iv[cidx(n - 2, m)]) *
                       inv_r2;
  }
}

void oracle_harmonics_R(double x, double y, double z, int p, double* out) {
  harm_R(x, y, z, p, (cplx*)out);
}
void oracle_harmonics_I(double x, double y, double z, int p, double* out) {
  harm_I(x, y, z, p, (cplx*)out);
}

/* ------------------------------------------------------- operators (c.1) */

/* P2M: M_n^m(c) += sum_i q_i conj R_n^m(x_i - c) */
static void p2m(const double* xyz, const double* q, int64_t n, const double* c, int p, cplx* M,
                cplx* R) {
  for (int64_t i = 0; i < n; ++i) {
    harm_R(xyz[3 * i] - c[0], xyz[3 * i + 1] - c[1], xyz[3 * i + 2] - c[2], p, R);
    for (int nn = 0; nn <= p; ++nn)
      for (int m = 0; m <= nn; ++m) M[cidx(nn, m)] += q[i] * conj(R[cidx(nn, m)]);
  }
}

/* M2M (child c -> parent c'): M_j^k(c') += sum_{n=0}^{j} sum_{|m|<=n}
 *   conj R_n^m(c - c') M_{j-n}^{k-m}(c),   terms with |k-m| > j-n vanish. */
static void m2m(const cplx* Mc, const double* cc, const double* cp, int p, cplx* Mp, cplx* R) {
  harm_R(cc[0] - cp[0], cc[1] - cp[1], cc[2] - cp[2], p, R);
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k <= j; ++k) {
      cplx s = 0;
      for (int n = 0; n <= j; ++n)
        for (int m = -n; m <= n; ++m) {
          if (abs(k - m) > j - n) continue;
          s += conj(getc(R, n, m)) * getc(Mc, j - n, k - m);
        }
      Mp[cidx(j, k)] += s;
    }
}

/* M2L (source B -> target A): L_j^k(cA) += sum_{n=0}^{p} sum_{|m|<=n}
 *   (-1)^n M_n^m(cB) I_{j+n}^{k+m}(cB - cA).   Needs I up to degree 2p. */
static void m2l(const cplx* MB, const double* cB, const double* cA, int p, cplx* LA, cplx* Iw) {
  harm_I(cB[0] - cA[0], cB[1] - cA[1], cB[2] - cA[2], 2 * p, Iw);
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k <= j; ++k) {
      cplx s = 0;
      for (int n = 0; n <= p; ++n) {
        cplx sn = 0;
        for (int m = -n; m <= n; ++m) sn += getc(MB, n, m) * getc(Iw, j + n, k + m);
        s += (n & 1) ? -sn : sn;
      }
      LA[cidx(j, k)] += s;
    }
}

/* L2L (parent c -> child c'): L_j^k(c') += sum_{n=j}^{p} sum_{|m|<=n}
 *   L_n^m(c) conj R_{n-j}^{m-k}(c' - c),   terms with |m-k| > n-j vanish. */
static void l2l(const cplx* Lp, const double* cp, const double* cc, int p, cplx* Lc, cplx* R) {
  harm_R(cc[0] - cp[0], cc[1] - cp[1], cc[2] - cp[2], p, R);
  for (int j = 0; j <= p; ++j)
    for (int k = 0; k <= j; ++k) {
      cplx s = 0;
      for (int n = j; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          if (abs(m - k) > n - j) continue;
          s += getc(Lp, n, m) * conj(getc(R, n - j, m - k));
        }
      Lc[cidx(j, k)] += s;
    }
}

/* L2P: phi(x) = Re sum_{n<=p} sum_{|m|<=n} L_n^m conj R_n^m(x - c).
 * Gradient: for k in {0,1}, L'_k = sum_{n=1}^{p} sum_m L_n^m conj R_{n-1}^{m-k}(x - c);
 *   grad phi = (-Re L'_1, -Im L'_1, Re L'_0). */
static void l2p(const cplx* L, const double* c, const double* x, int p, double* phi,
                double* grad, cplx* R) {
  harm_R(x[0] - c[0], x[1] - c[1], x[2] - c[2], p, R);
  cplx s = 0;
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m) s += getc(L, n, m) * conj(getc(R, n, m));
  *phi += creal(s);
  if (grad) {
    cplx g[2] = {0, 0};
    for (int k = 0; k <= 1; ++k)
      for (int n = 1; n <= p; ++n)
        for (int m = -n; m <= n; ++m) {
          if (abs(m - k) > n - 1) continue;
          g[k] += getc(L, n, m) * conj(getc(R, n - 1, m - k));
        }
    grad[0] += -creal(g[1]);
    grad[1] += -cimag(g[1]);
    grad[2] += creal(g[0]);
  }
}

/* M2P (multipole evaluated at a point), for the multipole-only bound pin. */
void oracle_m2p(const double* M, const double* c, const double* x, int p, double* phi) {
  cplx* Iw = malloc(sizeof(cplx) * ncoef(p));
  harm_I(x[0] - c[0], x[1] - c[1], x[2] - c[2], p, Iw);
  cplx s = 0;
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m) s += getc((const cplx*)M, n, m) * getc(Iw, n, m);
  *phi += creal(s);
  free(Iw);
}

void oracle_p2m(const double* xyz, const double* q, int64_t n, const double* c, int p, double* M) {
  cplx* R = malloc(sizeof(cplx) * ncoef(p));
  p2m(xyz, q, n, c, p, (cplx*)M, R);
  free(R);
}
void oracle_m2m(const double* Mc, const double* cc, const double* cp, int p, double* Mp) {
  cplx* R = malloc(sizeof(cplx) * ncoef(p));
  m2m((const cplx*)Mc, cc, cp, p, (cplx*)Mp, R);
  free(R);
}
void oracle_m2l(const double* MB, const double* cB, const double* cA, int p, double* LA) {
  cplx* Iw = malloc(sizeof(cplx) * ncoef(2 * p));
  m2l((const cplx*)MB, cB, cA, p, (cplx*)LA, Iw);
  free(Iw);
}
void oracle_l2l(const double* Lp, const double* cp, const double* cc, int p, double* Lc) {
  cplx* R = malloc(sizeof(cplx) * ncoef(p));
  l2l((const cplx*)Lp, cp, cc, p, (cplx*)Lc, R);
  free(R);
}
void oracle_l2p(const double* L, const double* c, const double* x, int p, double* phi,
                double* grad3) {
  cplx* R = malloc(sizeof(cplx) * ncoef(p));
  l2p((const cplx*)L, c, x, p, phi, grad3, R);
  free(R);
}

/* -------------------------------------------------- direct sum (A16, P1) */

int oracle_direct(const double* src, const double* q, int64_t ns, const double* tgt, int64_t nt,
                  double* phi, double* grad, int nthreads) {
  if (ns < 0 || nt < 0 || (ns > 0 && (!src || !q)) || (nt > 0 && (!tgt || !phi))) return 2;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t i = 0; i < nt; ++i) {
    long double s = 0, gx = 0, gy = 0, gz = 0;
    for (int64_t j = 0; j < ns; ++j) {
      long double dx = (long double)tgt[3 * i] - src[3 * j];
      long double dy = (long double)tgt[3 * i + 1] - src[3 * j + 1];
      long double dz = (long double)tgt[3 * i + 2] - src[3 * j + 2];
      long double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0) continue; /* Q2: coincident points / self term contribute nothing */
      long double r = sqrtl(r2);
      s += q[j] / r;
      long double w = q[j] / (r2 * r);
      gx -= w * dx;
      gy -= w * dy;
      gz -= w * dz;
    }
    phi[i] = (double)s;
    if (grad) {
      grad[3 * i] = (double)gx;
      grad[3 * i + 1] = (double)gy;
      grad[3 * i + 2] = (double)gz;
    }
  }
  return 0;
}

/* ------------------------------------------------------------ the plan */

typedef struct {
  int32_t level, anchor[3];
  int64_t begin, end;       /* particle range in sorted order */
  int64_t child_first;      /* index of first child, -1 for a leaf */
  int32_t nchild;
  int64_t parent;           /* -1 for the root */
  int64_t C[3], H;          /* integer geometry, units of S / 2^22 (A6) */
  double c[3];              /* float centre (A6) */
} cell_t;

typedef struct {
  int64_t* a;
  int64_t n, cap;
} pairvec; /* flat (target, source) pairs */

static int pv_push(pairvec* v, int64_t t, int64_t s) {
  if (v->n == v->cap) {
    int64_t nc = v->cap ? 2 * v->cap : 1024;
    int64_t* na = realloc(v->a, sizeof(int64_t) * 2 * nc);
    if (!na) return 5;
    v->a = na;
    v->cap = nc;
  }
  v->a[2 * v->n] = t;
  v->a[2 * v->n + 1] = s;
  v->n++;
  return 0;
}

struct oracle_plan_s {
  int64_t n;
  int p, ncrit, e;
  double theta;
  double lo[3], S, scale;
  double* xs;       /* scaled coordinates in sorted order [n][3] */
  uint64_t* keys;   /* sorted keys */
  int64_t* perm;    /* sorted position -> input index */
  cell_t* cells;
  int64_t ncells, nleaves;
  int maxlevel;
  pairvec p2p, m2l;
  cplx *M, *L;      /* expansions of the last full eval */
};

typedef struct {
  uint64_t key;
  int64_t idx;
} keyidx;

static int cmp_keyidx(const void* a, const void* b) {
  const keyidx* x = a;
  const keyidx* y = b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx); /* A5: ties by input index (stable) */
}

/* A4: key = sum_b bit_b(kx) 2^{3b+2} + bit_b(ky) 2^{3b+1} + bit_b(kz) 2^{3b} */
static uint64_t morton_key(uint32_t kx, uint32_t ky, uint32_t kz) {
  uint64_t key = 0;
  for (int b = 0; b < MAXLEVEL; ++b) {
    key |= (uint64_t)((kx >> b) & 1u) << (3 * b + 2);
    key |= (uint64_t)((ky >> b) & 1u) << (3 * b + 1);
    key |= (uint64_t)((kz >> b) & 1u) << (3 * b);
  }
  return key;
}

static int is_leaf(const cell_t* c) { return c->child_first < 0; }

/* A7: Interact(A, B) — recursive dual tree traversal with the integer MAC.
 * `want` (nullable) restricts the descent on the target side to cells that
 * contain a sampled target (A15). */
static int interact(struct oracle_plan_s* P, int64_t A, int64_t B, const char* want,
                    pairvec* p2p, pairvec* m2l) {
  const cell_t* a = &P->cells[A];
  const cell_t* b = &P->cells[B];
  int64_t d2 = 0;
  for (int k = 0; k < 3; ++k) {
    int64_t d = a->C[k] - b->C[k];
    d2 += d * d;
  }
  int64_t rr = a->H + b->H;
  int64_t r2 = rr * rr;
  double tt = P->theta * P->theta;
  double lhs = tt * (double)d2; /* two IEEE multiplies, then compare (A7.2) */
  if (lhs > (double)r2) return pv_push(m2l, A, B);
  if (is_leaf(a) && is_leaf(b)) return pv_push(p2p, A, B);
  if (is_leaf(b) || (!is_leaf(a) && a->level <= b->level)) {
    for (int i = 0; i < a->nchild; ++i) {
      int64_t ch = a->child_first + i;
      if (want && !want[ch]) continue;
      int st = interact(P, ch, B, want, p2p, m2l);
      if (st) return st;
    }
  } else {
    for (int i = 0; i < b->nchild; ++i) {
      int st = interact(P, A, b->child_first + i, want, p2p, m2l);
      if (st) return st;
    }
  }
  return 0;
}

int oracle_plan_new(oracle_plan* out, const double* xyz, int64_t n, int p, int ncrit,
                    double theta) {
  /* A1: validate */
  if (!out) return 2;
  *out = NULL;
  if (n < 1 || !xyz || p < 0 || p > 16 || ncrit < 1) return 2;
  if (!(theta > 0.0) || !(theta * theta * 3.0 < 1.0)) return 2; /* theta in (0, 1/sqrt3) */
  for (int64_t i = 0; i < 3 * n; ++i)
    if (!isfinite(xyz[i])) return 2;

  struct oracle_plan_s* P = calloc(1, sizeof(*P));
  if (!P) return 5;
  P->n = n;
  P->p = p;
  P->ncrit = ncrit;
  P->theta = theta;

  /* A2: root cube, then exact 2^-e normalisation so that S in [1, 2) */
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) lo[k] = hi[k] = xyz[k];
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      if (xyz[3 * i + k] < lo[k]) lo[k] = xyz[3 * i + k];
      if (xyz[3 * i + k] > hi[k]) hi[k] = xyz[3 * i + k];
    }
  double S = 0;
  for (int k = 0; k < 3; ++k)
    if (hi[k] - lo[k] > S) S = hi[k] - lo[k];
  if (S == 0) S = 1;
  int ex;
  frexp(S, &ex); /* S = f 2^ex, f in [0.5, 1)  =>  floor(log2 S) = ex - 1 */
  P->e = ex - 1;
  for (int k = 0; k < 3; ++k) P->lo[k] = ldexp(lo[k], -P->e);
  P->S = ldexp(S, -P->e);
  P->scale = 2097152.0 / P->S; /* 2^21 / S, one IEEE division */

  /* A3–A5: quantise, Morton key, stable sort */
  keyidx* ki = malloc(sizeof(keyidx) * n);
  if (!ki) {
    free(P);
    return 5;
  }
  for (int64_t i = 0; i < n; ++i) {
    uint32_t kq[3];
    for (int k = 0; k < 3; ++k) {
      double x = ldexp(xyz[3 * i + k], -P->e);
      double t = x - P->lo[k];
      double u = t * P->scale;
      double f = floor(u);
      if (f < 0) f = 0;
      if (f > 2097151.0) f = 2097151.0;
      kq[k] = (uint32_t)f;
    }
    ki[i].key = morton_key(kq[0], kq[1], kq[2]);
    ki[i].idx = i;
  }
  qsort(ki, n, sizeof(keyidx), cmp_keyidx);
  P->keys = malloc(sizeof(uint64_t) * n);
  P->perm = malloc(sizeof(int64_t) * n);
  P->xs = malloc(sizeof(double) * 3 * n);
  for (int64_t i = 0; i < n; ++i) {
    P->keys[i] = ki[i].key;
    P->perm[i] = ki[i].idx;
    for (int k = 0; k < 3; ++k) P->xs[3 * i + k] = ldexp(xyz[3 * ki[i].idx + k], -P->e);
  }
  free(ki);

  /* A6: adaptive octree, breadth first (level, then Morton order) */
  int64_t cap = 1024;
  P->cells = malloc(sizeof(cell_t) * cap);
  P->ncells = 1;
  cell_t* root = &P->cells[0];
  memset(root, 0, sizeof(*root));
  root->begin = 0;
  root->end = n;
  root->child_first = -1;
  root->parent = -1;
  for (int64_t ci = 0; ci < P->ncells; ++ci) {
    cell_t* c = &P->cells[ci];
    int l = c->level;
    c->H = (int64_t)1 << (MAXLEVEL - l);
    for (int k = 0; k < 3; ++k) {
      c->C[k] = (2 * (int64_t)c->anchor[k] + 1) * c->H;
      c->c[k] = P->lo[k] + (double)(2 * (int64_t)c->anchor[k] + 1) * ldexp(P->S, -(l + 1));
    }
    if (l > P->maxlevel) P->maxlevel = l;
    if (c->end - c->begin > ncrit && l < MAXLEVEL) {
      int shift = 3 * (MAXLEVEL - l - 1);
      int64_t i = c->begin;
      c->child_first = P->ncells;
      c->nchild = 0;
      for (int d = 0; d < 8; ++d) {
        int64_t j = i;
        while (j < c->end && (int)((P->keys[j] >> shift) & 7u) == d) ++j;
        if (j == i) continue; /* empty children are not created */
        if (P->ncells == cap) {
          cap *= 2;
          cell_t* nc = realloc(P->cells, sizeof(cell_t) * cap);
          if (!nc) {
            oracle_plan_free(P);
            return 5;
          }
          P->cells = nc;
          c = &P->cells[ci];
        }
        cell_t* ch = &P->cells[P->ncells++];
        memset(ch, 0, sizeof(*ch));
        ch->level = l + 1;
        ch->anchor[0] = 2 * c->anchor[0] + ((d >> 2) & 1);
        ch->anchor[1] = 2 * c->anchor[1] + ((d >> 1) & 1);
        ch->anchor[2] = 2 * c->anchor[2] + (d & 1);
        ch->begin = i;
        ch->end = j;
        ch->child_first = -1;
        ch->parent = ci;
        c->nchild++;
        i = j;
      }
    } else {
      c->child_first = -1;
      P->nleaves++;
    }
  }

  /* A7: traversal from (root, root) */
  int st = interact(P, 0, 0, NULL, &P->p2p, &P->m2l);
  if (st) {
    oracle_plan_free(P);
    return st;
  }
  *out = P;
  return 0;
}

void oracle_plan_free(oracle_plan P) {
  if (!P) return;
  free(P->xs);
  free(P->keys);
  free(P->perm);
  free(P->cells);
  free(P->p2p.a);
  free(P->m2l.a);
  free(P->M);
  free(P->L);
  free(P);
}

int64_t oracle_plan_info(oracle_plan P, int which) {
  switch (which) {
    case ORACLE_INFO_N: return P->n;
    case ORACLE_INFO_NCELLS: return P->ncells;
    case ORACLE_INFO_NLEAVES: return P->nleaves;
    case ORACLE_INFO_NP2P: return P->p2p.n;
    case ORACLE_INFO_NM2L: return P->m2l.n;
    case ORACLE_INFO_EXP: return P->e;
    case ORACLE_INFO_MAXLEVEL: return P->maxlevel;
    case ORACLE_INFO_P: return P->p;
    case ORACLE_INFO_NP2P_INTERACTIONS: {
      int64_t s = 0;
      for (int64_t i = 0; i < P->p2p.n; ++i) {
        const cell_t* a = &P->cells[P->p2p.a[2 * i]];
        const cell_t* b = &P->cells[P->p2p.a[2 * i + 1]];
        s += (a->end - a->begin) * (b->end - b->begin);
      }
      return s;
    }
  }
  return -1;
}

void oracle_plan_geometry(oracle_plan P, double* lo3, double* S, double* scale) {
  if (lo3)
    for (int k = 0; k < 3; ++k) lo3[k] = P->lo[k];
  if (S) *S = P->S;
  if (scale) *scale = P->scale;
}

void oracle_plan_keys(oracle_plan P, uint64_t* keys, int64_t* perm) {
  if (keys) memcpy(keys, P->keys, sizeof(uint64_t) * P->n);
  if (perm) memcpy(perm, P->perm, sizeof(int64_t) * P->n);
}

void oracle_plan_cells(oracle_plan P, int32_t* level, int32_t* anchor3, int64_t* begin,
                       int64_t* end, int64_t* child_first, int32_t* nchild, int64_t* parent,
                       double* center3) {
  for (int64_t i = 0; i < P->ncells; ++i) {
    const cell_t* c = &P->cells[i];
    if (level) level[i] = c->level;
    if (anchor3)
      for (int k = 0; k < 3; ++k) anchor3[3 * i + k] = c->anchor[k];
    if (begin) begin[i] = c->begin;
    if (end) end[i] = c->end;
    if (child_first) child_first[i] = c->child_first;
    if (nchild) nchild[i] = c->nchild;
    if (parent) parent[i] = c->parent;
    if (center3)
      for (int k = 0; k < 3; ++k) center3[3 * i + k] = c->c[k];
  }
}

void oracle_plan_lists(oracle_plan P, int64_t* p2p, int64_t* m2l) {
  if (p2p) memcpy(p2p, P->p2p.a, sizeof(int64_t) * 2 * P->p2p.n);
  if (m2l) memcpy(m2l, P->m2l.a, sizeof(int64_t) * 2 * P->m2l.n);
}

void oracle_plan_expansions(oracle_plan P, double* M, double* L) {
  int64_t nc = (int64_t)P->ncells * ncoef(P->p);
  if (M && P->M) memcpy(M, P->M, sizeof(cplx) * nc);
  if (L && P->L) memcpy(L, P->L, sizeof(cplx) * nc);
}

/* CSR grouping of a pair list by target, keeping list order within a target. */
static void group_by_target(const pairvec* v, int64_t ncells, int64_t** off_out,
                            int64_t** src_out) {
  int64_t* off = calloc(ncells + 1, sizeof(int64_t));
  int64_t* src = malloc(sizeof(int64_t) * (v->n > 0 ? v->n : 1));
  for (int64_t i = 0; i < v->n; ++i) off[v->a[2 * i] + 1]++;
  for (int64_t c = 0; c < ncells; ++c) off[c + 1] += off[c];
  int64_t* fill = malloc(sizeof(int64_t) * (ncells + 1));
  memcpy(fill, off, sizeof(int64_t) * (ncells + 1));
  for (int64_t i = 0; i < v->n; ++i) src[fill[v->a[2 * i]]++] = v->a[2 * i + 1];
  free(fill);
  *off_out = off;
  *src_out = src;
}

/* A8–A15 */
int oracle_plan_eval(oracle_plan P, const double* q, const int64_t* targets, int64_t nt,
                     double* phi, double* grad, int nthreads) {
  const int64_t n = P->n;
  const int p = P->p;
  const int nc = ncoef(p);
  if (!q || !phi) return 2;
  if (targets && nt < 0) return 2;
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(q[i])) return 3;
  for (int64_t t = 0; targets && t < nt; ++t)
    if (targets[t] < 0 || targets[t] >= n) return 2;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif

  double* qs = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) qs[i] = q[P->perm[i]];

  /* A15: sampled targets, mapped to sorted positions; flag cells containing one */
  char* want = NULL;
  char* pwant = NULL;
  int64_t* inv = NULL;
  if (targets) {
    inv = malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; ++i) inv[P->perm[i]] = i;
    pwant = calloc(n, 1);
    for (int64_t t = 0; t < nt; ++t) pwant[inv[targets[t]]] = 1;
    int64_t* pre = malloc(sizeof(int64_t) * (n + 1));
    pre[0] = 0;
    for (int64_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + pwant[i];
    want = calloc(P->ncells, 1);
    for (int64_t c = 0; c < P->ncells; ++c)
      want[c] = pre[P->cells[c].end] - pre[P->cells[c].begin] > 0;
    free(pre);
  }

  cplx* M = calloc((size_t)P->ncells * nc, sizeof(cplx));
  cplx* L = calloc((size_t)P->ncells * nc, sizeof(cplx));
  if (!M || !L) {
    free(M);
    free(L);
    free(qs);
    free(want);
    free(pwant);
    free(inv);
    return 5;
  }

  /* A8: P2M for every leaf */
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
    cplx* R = malloc(sizeof(cplx) * nc);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
    for (int64_t c = 0; c < P->ncells; ++c) {
      const cell_t* cl = &P->cells[c];
      if (!is_leaf(cl)) continue;
      p2m(P->xs + 3 * cl->begin, qs + cl->begin, cl->end - cl->begin, cl->c, p, M + c * nc, R);
    }
    free(R);
  }

  /* A9: M2M, children before parents (reverse breadth-first order is a post-order
   * for this dependency), one level at a time, children in digit order */
  for (int lev = P->maxlevel - 1; lev >= 0; --lev) {
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
      cplx* R = malloc(sizeof(cplx) * nc);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
      for (int64_t c = 0; c < P->ncells; ++c) {
        const cell_t* cl = &P->cells[c];
        if (cl->level != lev || is_leaf(cl)) continue;
        for (int i = 0; i < cl->nchild; ++i) {
          int64_t ch = cl->child_first + i;
          m2m(M + ch * nc, P->cells[ch].c, cl->c, p, M + c * nc, R);
        }
      }
      free(R);
    }
  }

  /* A7 (restricted, A15) or the plan's full lists */
  pairvec sp2p = {0}, sm2l = {0};
  const pairvec* lp2p = &P->p2p;
  const pairvec* lm2l = &P->m2l;
  if (targets) {
    if (nt > 0) {
      int st = interact(P, 0, 0, want, &sp2p, &sm2l);
      if (st) return st;
    }
    lp2p = &sp2p;
    lm2l = &sm2l;
  }

  /* A10: M2L, grouped by target cell (list order kept within a target) */
  int64_t *moff, *msrc;
  group_by_target(lm2l, P->ncells, &moff, &msrc);
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
    cplx* Iw = malloc(sizeof(cplx) * ncoef(2 * p));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
    for (int64_t A = 0; A < P->ncells; ++A)
      for (int64_t k = moff[A]; k < moff[A + 1]; ++k) {
        int64_t B = msrc[k];
        m2l(M + B * nc, P->cells[B].c, P->cells[A].c, p, L + A * nc, Iw);
      }
    free(Iw);
  }
  free(moff);
  free(msrc);

  /* A11: L2L, parents before children (breadth-first order) */
  for (int lev = 1; lev <= P->maxlevel; ++lev) {
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
      cplx* R = malloc(sizeof(cplx) * nc);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
      for (int64_t c = 0; c < P->ncells; ++c) {
        const cell_t* cl = &P->cells[c];
        if (cl->level != lev || (want && !want[c])) continue;
        l2l(L + cl->parent * nc, P->cells[cl->parent].c, cl->c, p, L + c * nc, R);
      }
      free(R);
    }
  }

  /* A12, A13: L2P (+grad) and P2P, per target leaf, into sorted-order buffers */
  double* phis = calloc(n, sizeof(double));
  double* grads = grad ? calloc(3 * n, sizeof(double)) : NULL;
  int64_t *poff, *psrc;
  group_by_target(lp2p, P->ncells, &poff, &psrc);
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
    cplx* R = malloc(sizeof(cplx) * nc);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
    for (int64_t A = 0; A < P->ncells; ++A) {
      const cell_t* a = &P->cells[A];
      if (!is_leaf(a) || (want && !want[A])) continue;
      for (int64_t i = a->begin; i < a->end; ++i) {
        if (pwant && !pwant[i]) continue;
        const double* xi = P->xs + 3 * i;
        double f = 0, g[3] = {0, 0, 0};
        l2p(L + A * nc, a->c, xi, p, &f, grad ? g : NULL, R);
        for (int64_t k = poff[A]; k < poff[A + 1]; ++k) {
          const cell_t* b = &P->cells[psrc[k]];
          for (int64_t j = b->begin; j < b->end; ++j) {
            double dx = xi[0] - P->xs[3 * j];
            double dy = xi[1] - P->xs[3 * j + 1];
            double dz = xi[2] - P->xs[3 * j + 2];
            double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 == 0.0) continue; /* Q2 */
            double r = sqrt(r2);
            f += qs[j] / r;
            double w = qs[j] / (r2 * r);
            g[0] -= w * dx;
            g[1] -= w * dy;
            g[2] -= w * dz;
          }
        }
        phis[i] = f;
        if (grads)
          for (int k = 0; k < 3; ++k) grads[3 * i + k] = g[k];
      }
    }
    free(R);
  }
  free(poff);
  free(psrc);

  /* A14 (+A2.4): undo the 2^-e normalisation exactly and return to input order */
  if (!targets) {
    for (int64_t i = 0; i < n; ++i) {
      int64_t o = P->perm[i];
      phi[o] = ldexp(phis[i], -P->e);
      if (grad)
        for (int k = 0; k < 3; ++k) grad[3 * o + k] = ldexp(grads[3 * i + k], -2 * P->e);
    }
    free(P->M);
    free(P->L);
    P->M = M;
    P->L = L;
  } else {
    for (int64_t t = 0; t < nt; ++t) {
      int64_t i = inv[targets[t]];
      phi[t] = ldexp(phis[i], -P->e);
      if (grad)
        for (int k = 0; k < 3; ++k) grad[3 * t + k] = ldexp(grads[3 * i + k], -2 * P->e);
    }
    free(M);
    free(L);
  }
  free(sp2p.a);
  free(sm2l.a);
  free(phis);
  free(grads);
  free(qs);
  free(want);
  free(pwant);
  free(inv);
  return 0;
}
