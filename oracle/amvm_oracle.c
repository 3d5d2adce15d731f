/*
 * amvm_oracle.c — CPU restatement of the reference AMVM path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker: tests/, the smoke()
 * of __graft_entry__.py and the cpu_baseline / --impl reference leg of
 * bench.py may load it; the product path (paper_2508_13437_b200 +
 * libamvm.so) never does.
 *
 * It restates, function by function, the Python reference
 * /root/reference/pkg/src/dmmv/{core,operators,localsearch,controller}.py in
 * plain sequential C with the reference's A layout (row-major m x n), and
 * reproduces the numpy arithmetic the reference relies on:
 *   - numpy Generator(PCG64): next64/next32 half-word buffer, random(),
 *     Lemire-32 bounded ints, choice(n, size, replace=False) (Floyd + hash
 *     set + Fisher-Yates, and the tail-shuffle path), choice(k, p=...)
 *     (sequential cumsum, /cdf[-1], searchsorted right);
 *   - numpy pairwise summation (8-accumulator blocks of <=128, halving with
 *     n2 -= n2 % 8) for 1-d .sum();
 *   - sequential axis-0 sums, sequential cumsum;
 *   - np.linalg.norm == sqrt(ddot) in the OpenBLAS 0.3.30 SkylakeX kernel
 *     order (verified bitwise against numpy on the dev host);
 *   - unfused DMUL/DADD for every residual update (compile with
 *     -ffp-contract=off).
 * Known, documented deviation from the reference:
 *   - exp() is libm's, numpy uses its own SIMD exp (<= 1 ulp apart);
 * and one more emulation:
 *   - A @ x (refresh, core.py:175, and compute_residual, core.py:196) is
 *     emulated in the single-threaded OpenBLAS 0.3.30 dgemv_t order
 *     (verified bitwise against numpy on the dev host).
 * Parity of this oracle with the reference is pinned by tests/golden/
 * (fixtures produced by running the reference itself, make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/amvm.h"

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ RNG */
/* numpy/random/src/pcg64: 128-bit LCG, XSL-RR output, advance-then-output */
typedef struct {
  u128 s, inc;
  int has32;
  uint32_t u32;
} pcg_t;

static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static void pcg_load(pcg_t *g, const amvm_pcg64 *st) {
  g->s = (((u128)st->state_hi) << 64) | st->state_lo;
  g->inc = (((u128)st->inc_hi) << 64) | st->inc_lo;
  g->has32 = (int)st->has_uint32;
  g->u32 = st->uinteger;
}
static void pcg_store(const pcg_t *g, amvm_pcg64 *st) {
  st->state_hi = (uint64_t)(g->s >> 64);
  st->state_lo = (uint64_t)g->s;
  st->inc_hi = (uint64_t)(g->inc >> 64);
  st->inc_lo = (uint64_t)g->inc;
  st->has_uint32 = (uint32_t)g->has32;
  st->uinteger = g->u32;
}
static uint64_t pcg_next64(pcg_t *g) {
  g->s = g->s * PCG_MULT + g->inc;
  uint64_t hi = (uint64_t)(g->s >> 64), lo = (uint64_t)g->s;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
static uint32_t pcg_next32(pcg_t *g) {
  if (g->has32) {
    g->has32 = 0;
    return g->u32;
  }
  uint64_t v = pcg_next64(g);
  g->has32 = 1;
  g->u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}
/* Generator.random(): 53-bit double */
static double pcg_random(pcg_t *g) {
  return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}
/* random_bounded_uint64(off=0, rng, use_masked=0) for rng <= 0xFFFFFFFF:
 * Lemire's method on next_uint32 (rng is the inclusive maximum). */
static uint64_t pcg_bounded(pcg_t *g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return pcg_next32(g);
  uint32_t ex = (uint32_t)rng + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * ex;
  uint32_t left = (uint32_t)m;
  if (left < ex) {
    uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % ex;
    while (left < thr) {
      m = (uint64_t)pcg_next32(g) * ex;
      left = (uint32_t)m;
    }
  }
  return m >> 32;
}
/* Generator.choice(pop, size=r, replace=False) index stream (no p). */
static void choice_noreplace(pcg_t *g, int64_t pop, int64_t r, int64_t *out) {
  if (pop > 10000 && r > pop / 50) { /* tail-shuffle path */
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)pop);
    for (int64_t i = 0; i < pop; i++) idx[i] = i;
    int64_t first = pop - r > 1 ? pop - r : 1;
    for (int64_t i = pop - 1; i >= first; i--) {
      int64_t j = (int64_t)pcg_bounded(g, (uint64_t)i);
      int64_t t = idx[i];
      idx[i] = idx[j];
      idx[j] = t;
    }
    memcpy(out, idx + (pop - r), sizeof(int64_t) * (size_t)r);
    free(idx);
    return;
  }
  uint64_t mask = (uint64_t)(1.2 * (double)r);
  mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
  mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
  uint64_t *hs = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(mask + 1));
  for (uint64_t k = 0; k <= mask; k++) hs[k] = ~(uint64_t)0;
  for (int64_t j = pop - r; j < pop; j++) {
    uint64_t val = pcg_bounded(g, (uint64_t)j);
    uint64_t loc = val & mask;
    while (hs[loc] != ~(uint64_t)0 && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == ~(uint64_t)0) {
      hs[loc] = val;
      out[j - pop + r] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != ~(uint64_t)0) loc = (loc + 1) & mask;
      hs[loc] = (uint64_t)j;
      out[j - pop + r] = j;
    }
  }
  free(hs);
  for (int64_t i = r - 1; i >= 1; i--) {
    int64_t j = (int64_t)pcg_bounded(g, (uint64_t)i);
    int64_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
}

/* ------------------------------------------------------- numpy arithmetic */
/* numpy pairwise_sum (umath loops), as used by 1-d ndarray.sum() */
static double pw_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; k++) r[k] = a[k];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
  }
}

/* x.dot(x) in the OpenBLAS 0.3.30 SkylakeX ddot order (ddot.c driver +
 * ddot_microk_skylakex-2.c): 4 x 8-lane FMA accumulators over n & ~31, fold
 * to 4 x 4 lanes, 4 x 4-lane FMA over the remaining 16-block, lanes combined
 * ((a0+a1)+a2)+a3, halves [0]+[2],[1]+[3], then h0+h1; the n - (n & -16)
 * tail through a scalar FMA loop. */
static double ddot_skx(const double *x, int64_t n) {
  int64_t n1 = n & -16;
  double dot = 0.0;
  if (n1) {
    double a[4][8] = {{0}};
    int64_t n32 = n1 & ~(int64_t)31, i = 0;
    for (; i < n32; i += 32)
      for (int q = 0; q < 4; q++)
        for (int l = 0; l < 8; l++) {
          double v = x[i + 8 * q + l];
          a[q][l] = fma(v, v, a[q][l]);
        }
    double acc[4][4];
    for (int q = 0; q < 4; q++)
      for (int l = 0; l < 4; l++) acc[q][l] = a[q][l] + a[q][l + 4];
    for (; i < n1; i += 16)
      for (int q = 0; q < 4; q++)
        for (int l = 0; l < 4; l++) {
          double v = x[i + 4 * q + l];
          acc[q][l] = fma(v, v, acc[q][l]);
        }
    double s[4];
    for (int l = 0; l < 4; l++) s[l] = ((acc[0][l] + acc[1][l]) + acc[2][l]) + acc[3][l];
    dot = (s[0] + s[2]) + (s[1] + s[3]);
  }
  for (int64_t i = n1; i < n; i++) dot = fma(x[i], x[i], dot);
  return dot;
}

/* x.dot(y) for two vectors, same SkylakeX ddot order (tail: fma(y, x, dot)) */
static double ddot_xy(const double *x, const double *y, int64_t n) {
  int64_t n1 = n & -16;
  double dot = 0.0;
  if (n1) {
    double a[4][8] = {{0}};
    int64_t n32 = n1 & ~(int64_t)31, i = 0;
    for (; i < n32; i += 32)
      for (int q = 0; q < 4; q++)
        for (int l = 0; l < 8; l++) a[q][l] = fma(x[i + 8 * q + l], y[i + 8 * q + l], a[q][l]);
    double acc[4][4];
    for (int q = 0; q < 4; q++)
      for (int l = 0; l < 4; l++) acc[q][l] = a[q][l] + a[q][l + 4];
    for (; i < n1; i += 16)
      for (int q = 0; q < 4; q++)
        for (int l = 0; l < 4; l++) acc[q][l] = fma(x[i + 4 * q + l], y[i + 4 * q + l], acc[q][l]);
    double s[4];
    for (int l = 0; l < 4; l++) s[l] = ((acc[0][l] + acc[1][l]) + acc[2][l]) + acc[3][l];
    dot = (s[0] + s[2]) + (s[1] + s[3]);
  }
  for (int64_t i = n1; i < n; i++) dot = fma(y[i], x[i], dot);
  return dot;
}

/* One output of OpenBLAS 0.3.30 dgemv_t (kernel/x86_64/dgemv_t_4.c, Haswell
 * micro-kernels, used for SkylakeX), i.e. one row of numpy's A @ x for a
 * C-contiguous A: the first K & -4 elements in blocks of NBMAX = 2048, each
 * block reduced by the kernel `kind` (4: 4x4 = 4-lane FMA accumulator,
 * lanes (0+2)+(1+3); 2: 4x2 = 2-lane mul+add, lane0+lane1; 1: 4x1 = two
 * 2-lane mul+add accumulators over {4k,4k+1},{4k+2,4k+3}) and added to y;
 * then the K & 3 leftover with the compiler-contracted scalar code. */
static double gemv_row(const double *a, const double *x, int64_t K, int kind) {
  int64_t m1 = K & -4, p = 0;
  double y = 0.0;
  while (p < m1) {
    int64_t nb = m1 - p < 2048 ? m1 - p : 2048;
    double t;
    if (kind == 4) {
      double l[4] = {0, 0, 0, 0};
      for (int64_t i = p; i < p + nb; i += 4)
        for (int q = 0; q < 4; q++) l[q] = fma(a[i + q], x[i + q], l[q]);
      t = (l[0] + l[2]) + (l[1] + l[3]);
    } else if (kind == 2) {
      double l[2] = {0, 0};
      for (int64_t i = p; i < p + nb; i += 2) {
        l[0] = l[0] + a[i] * x[i];
        l[1] = l[1] + a[i + 1] * x[i + 1];
      }
      t = l[0] + l[1];
    } else {
      double u[2] = {0, 0}, v[2] = {0, 0};
      for (int64_t i = p; i < p + nb; i += 4) {
        u[0] = u[0] + a[i] * x[i];
        u[1] = u[1] + a[i + 1] * x[i + 1];
        v[0] = v[0] + a[i + 2] * x[i + 2];
        v[1] = v[1] + a[i + 3] * x[i + 3];
      }
      t = (u[0] + v[0]) + (u[1] + v[1]);
    }
    y = y + t;
    p += nb;
  }
  switch (K & 3) {
    case 1: y = fma(a[m1], x[m1], y); break;
    case 2: y = y + fma(a[m1], x[m1], a[m1 + 1] * x[m1 + 1]); break;
    case 3: y = y + fma(a[m1 + 2], x[m1 + 2], fma(a[m1], x[m1], a[m1 + 1] * x[m1 + 1])); break;
  }
  return y;
}

/* numpy `A @ x` (A row-major m x K) with single-threaded OpenBLAS 0.3.30:
 * m == 1 goes through ddot; otherwise dgemv_t groups the m outputs as
 * 4x4 kernels, then one 4x2 and/or one 4x1 for the m & 3 leftover. */
static void gemv_numpy(const double *A, int64_t m, int64_t K, const double *x, double *y) {
  if (m == 1) {
    y[0] = ddot_xy(A, x, K);
    return;
  }
  int64_t g4 = m & ~(int64_t)3;
  for (int64_t i = 0; i < m; i++) {
    int kind = i < g4 ? 4 : ((m & 2) && i < g4 + 2) ? 2 : 1;
    y[i] = gemv_row(A + i * K, x, K, kind);
  }
}

/* Generator.choice(k, p=p): cdf = p.cumsum(); cdf /= cdf[-1];
 * searchsorted(cdf, random(), 'right').  `p` scratch of length k. */
static int64_t choice_p(pcg_t *g, const double *p, int64_t k, double *cdf) {
  double acc = 0.0;
  for (int64_t i = 0; i < k; i++) {
    acc += p[i];
    cdf[i] = acc;
  }
  double last = cdf[k - 1];
  for (int64_t i = 0; i < k; i++) cdf[i] = cdf[i] / last;
  double u = pcg_random(g);
  int64_t lo = 0, hi = k;
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (u < cdf[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

/* ----------------------------------------------------------- problem/state */
typedef struct {
  int64_t m, n, nlev;
  const double *A; /* row-major m x n (reference layout, core.py:84) */
  const double *At; /* optional column-major copy (n x m) or NULL: column
                       scans read it instead of striding A (same values,
                       same arithmetic order: speed only, for full-size
                       goldens) */
  const double *b, *lv;
} oprob;

/* column j of A as (pointer, stride): element i at c[i * st] */
static const double *acol(const oprob *P, int64_t j, int64_t *st) {
  if (P->At) { *st = 1; return P->At + j * P->m; }
  *st = P->n;
  return P->A + j;
}

typedef struct {
  int32_t *idx;
  double *r;
  double obj;
  int32_t cnt;
} osol;

static double max_abs(const double *r, int64_t m) {
  double t = 0.0;
  for (int64_t i = 0; i < m; i++) {
    double v = fabs(r[i]);
    if (v > t) t = v;
  }
  return t;
}

/* Solution.refresh core.py:173-177: A @ levels[idx] - b in numpy's
 * (OpenBLAS dgemv) order, then max|s|. */
static void sol_refresh(const oprob *P, osol *S) {
  double *x = (double *)malloc(sizeof(double) * (size_t)P->n);
  for (int64_t j = 0; j < P->n; j++) x[j] = P->lv[S->idx[j]];
  gemv_numpy(P->A, P->m, P->n, x, S->r);
  for (int64_t i = 0; i < P->m; i++) S->r[i] = S->r[i] - P->b[i];
  free(x);
  S->obj = max_abs(S->r, P->m);
  S->cnt = 0;
}

/* _bump core.py:200-205 */
static void bump(const oprob *P, const amvm_params *prm, osol *S) {
  S->cnt += 1;
  if (S->cnt >= prm->refresh_period) sol_refresh(P, S);
  else S->obj = max_abs(S->r, P->m);
}

/* apply_shift core.py:208-225 */
static void apply_shift(const oprob *P, const amvm_params *prm, osol *S, int64_t j, int32_t nl) {
  int32_t old = S->idx[j];
  if (nl == old) return;
  double d = P->lv[nl] - P->lv[old];
  int64_t st;
  const double *cj = acol(P, j, &st);
  for (int64_t i = 0; i < P->m; i++) S->r[i] = S->r[i] + d * cj[i * st];
  S->idx[j] = nl;
  bump(P, prm, S);
}

/* apply_swap core.py:228-245 */
static void apply_swap(const oprob *P, const amvm_params *prm, osol *S, int64_t i, int64_t j) {
  double xi = P->lv[S->idx[i]], xj = P->lv[S->idx[j]];
  double dl = xi - xj;
  int64_t st;
  const double *ci = acol(P, i, &st), *cj = acol(P, j, &st);
  for (int64_t k = 0; k < P->m; k++) S->r[k] = S->r[k] + dl * (cj[k * st] - ci[k * st]);
  int32_t t = S->idx[i];
  S->idx[i] = S->idx[j];
  S->idx[j] = t;
  bump(P, prm, S);
}

/* two_nearest core.py:62-72: first two of a stable argsort of |lv - v| */
static void two_nearest(const double *lv, int64_t nlev, double v, int32_t *c1, int32_t *c2) {
  int32_t a = 0;
  for (int32_t k = 1; k < nlev; k++)
    if (fabs(lv[k] - v) < fabs(lv[a] - v)) a = k;
  int32_t b = -1;
  for (int32_t k = 0; k < nlev; k++) {
    if (k == a) continue;
    if (b < 0 || fabs(lv[k] - v) < fabs(lv[b] - v)) b = k;
  }
  *c1 = a;
  *c2 = b;
}

/* ------------------------------------------------------------ local search */
typedef struct { int64_t moves_ref, moves_raw; } ocount;

/* one_opt localsearch.py:59-88 */
static void one_opt(const oprob *P, const amvm_params *prm, osol *S, ocount *C) {
  const double *lv = P->lv;
  for (int sw = 0; sw < prm->one_opt_max_sweeps; sw++) {
    int changed = 0;
    for (int64_t j = 0; j < P->n; j++) {
      int32_t k = S->idx[j];
      int32_t best_level = -1;
      double best_t = S->obj;
      for (int c = k - 1; c <= k + 1; c += 2) {
        if (c < 0 || c >= P->nlev) continue;
        double d = lv[c] - lv[k];
        double t = 0.0;
        int64_t st;
        const double *cj = acol(P, j, &st);
        for (int64_t i = 0; i < P->m; i++) {
          double v = fabs(S->r[i] + d * cj[i * st]);
          if (v > t) t = v;
        }
        if (C) { C->moves_ref++; C->moves_raw++; }
        if (t < best_t) {
          best_t = t;
          best_level = c;
        }
      }
      if (best_level >= 0) {
        apply_shift(P, prm, S, j, best_level);
        changed = 1;
      }
    }
    if (!changed) break;
  }
}

typedef struct { int32_t i, j; double delta; } ocand;

static int cmp_cand(const void *a, const void *b) {
  const ocand *x = (const ocand *)a, *y = (const ocand *)b;
  if (x->delta != y->delta) return x->delta > y->delta ? -1 : 1;
  if (x->i != y->i) return x->i < y->i ? -1 : 1;
  return (x->j > y->j) - (x->j < y->j);
}

typedef struct { double key; int64_t row; } orow;
static int cmp_row(const void *a, const void *b) {
  const orow *x = (const orow *)a, *y = (const orow *)b;
  if (x->key != y->key) return x->key > y->key ? -1 : 1;
  return (x->row > y->row) - (x->row < y->row);
}

/* find_candidates localsearch.py:128-169.  Survivors of the interval filter
 * over the top-k_eps rows, ordered (-delta, i, j), truncated.  The filter is
 * an AND over rows, so testing each pair against every row equals the
 * reference's row-by-row compression.  Returns the count; *out malloc'd. */
static int64_t find_candidates(const oprob *P, const amvm_params *prm, const osol *S, ocand **out) {
  *out = NULL;
  double t = S->obj;
  int64_t m = P->m, n = P->n;
  int64_t k = prm->k_eps < m ? prm->k_eps : m;
  orow *rows = (orow *)malloc(sizeof(orow) * (size_t)m);
  for (int64_t i = 0; i < m; i++) { rows[i].key = fabs(S->r[i]); rows[i].row = i; }
  qsort(rows, (size_t)m, sizeof(orow), cmp_row);
  int64_t nr = 0;
  int64_t *rk = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k ? k : 1));
  double *eps = (double *)malloc(sizeof(double) * (size_t)(k ? k : 1));
  int *pos = (int *)malloc(sizeof(int) * (size_t)(k ? k : 1));
  for (int64_t q = 0; q < k; q++) {
    double sk = S->r[rows[q].row];
    if (sk == 0.0) continue;
    rk[nr] = rows[q].row;
    eps[nr] = t - fabs(sk);
    pos[nr] = sk > 0;
    nr++;
  }
  free(rows);
  int64_t cap = 1024, cnt = 0;
  ocand *c = (ocand *)malloc(sizeof(ocand) * (size_t)cap);
  for (int64_t i = 0; i < n; i++) {
    double xi = P->lv[S->idx[i]];
    for (int64_t j = 0; j < n; j++) {
      double xj = P->lv[S->idx[j]];
      if (!(xi > xj)) continue;
      double delta = xi - xj;
      int alive = 1;
      for (int64_t q = 0; q < nr && alive; q++) {
        const double *row = P->A + rk[q] * n;
        double da = row[j] - row[i];
        double bound = eps[q] / delta;
        alive = pos[q] ? (da < bound) : (da > -bound);
      }
      if (!alive) continue;
      if (cnt == cap) { cap *= 2; c = (ocand *)realloc(c, sizeof(ocand) * (size_t)cap); }
      c[cnt].i = (int32_t)i; c[cnt].j = (int32_t)j; c[cnt].delta = delta;
      cnt++;
    }
  }
  free(rk); free(eps); free(pos);
  qsort(c, (size_t)cnt, sizeof(ocand), cmp_cand);
  if (prm->max_candidates > 0 && cnt > prm->max_candidates) cnt = prm->max_candidates;
  *out = c;
  return cnt;
}

/* best_swap + _evaluate_chunk localsearch.py:181-246 (l2_tiebreak is off on
 * the solve path, controller.py:65-68): min t', ties to lexicographic (i,j). */
static int best_swap(const oprob *P, const amvm_params *prm, const osol *S, int32_t *bi,
                     int32_t *bj, double *bd, double *bt, ocount *C) {
  if (S->obj <= 0) return 0;
  ocand *c;
  int64_t cnt = find_candidates(P, prm, S, &c);
  int found = 0;
  double best = 0;
  for (int64_t q = 0; q < cnt; q++) {
    double tn = 0.0;
    int64_t st;
    const double *ci = acol(P, c[q].i, &st), *cj = acol(P, c[q].j, &st);
    for (int64_t k = 0; k < P->m; k++) {
      double v = fabs(S->r[k] + c[q].delta * (cj[k * st] - ci[k * st]));
      if (v > tn) tn = v;
    }
    if (C) { C->moves_ref++; C->moves_raw++; }
    if (!(tn < S->obj)) continue;
    if (!found || tn < best || (tn == best && (c[q].i < *bi || (c[q].i == *bi && c[q].j < *bj)))) {
      found = 1; best = tn; *bi = c[q].i; *bj = c[q].j; *bd = c[q].delta;
    }
  }
  free(c);
  *bt = best;
  return found;
}

/* local_search localsearch.py:249-269 */
static void local_search(const oprob *P, const amvm_params *prm, osol *S, ocount *C) {
  one_opt(P, prm, S, C);
  for (int rd = 0; rd < prm->ls_max_rounds; rd++) {
    int32_t i, j;
    double d, t;
    if (!best_swap(P, prm, S, &i, &j, &d, &t, C)) break;
    apply_swap(P, prm, S, i, j);
    one_opt(P, prm, S, C);
  }
}

/* ---------------------------------------------------------------- operators */
/* impact_scores operators.py:54-74 */
static void impact_scores(const oprob *P, const osol *S, double alpha, double *d) {
  int64_t m = P->m, n = P->n;
  double t = S->obj;
  if (m <= 0) return;
  double *abs_s = (double *)malloc(sizeof(double) * (size_t)m);
  for (int64_t k = 0; k < m; k++) abs_s[k] = fabs(S->r[k]);
  for (int64_t j = 0; j < n; j++) d[j] = 0.0;
  double na = -alpha;
  for (int64_t k = 0; k < m; k++) {
    double num = na * (t - abs_s[k]);
    const double *row = P->A + k * n;
    for (int64_t j = 0; j < n; j++) {
      double a = fabs(row[j]);
      if (a > 0) d[j] = d[j] + abs_s[k] * exp(num / a);
    }
  }
  double total = pw_sum(abs_s, m);
  for (int64_t j = 0; j < n; j++) d[j] = d[j] / total;
  free(abs_s);
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* random_destroy operators.py:34-39 -> ascending removed[] */
static void random_destroy(pcg_t *g, int64_t n, int64_t r, int64_t *removed) {
  choice_noreplace(g, n, r, removed);
  qsort(removed, (size_t)r, sizeof(int64_t), cmp_i64);
}

/* worst_remove_destroy operators.py:77-105 -> ascending removed[] */
static void worst_destroy(const oprob *P, const osol *S, int64_t r, double alpha, pcg_t *g,
                          int64_t *removed) {
  int64_t n = P->n;
  if (S->obj <= 0) { random_destroy(g, n, r, removed); return; }
  double *d = (double *)malloc(sizeof(double) * (size_t)n);
  double *p = (double *)malloc(sizeof(double) * (size_t)n);
  double *cdf = (double *)malloc(sizeof(double) * (size_t)n);
  impact_scores(P, S, alpha, d);
  if (pw_sum(d, n) <= 0) {
    free(d); free(p); free(cdf);
    random_destroy(g, n, r, removed);
    return;
  }
  int64_t np_ = 0;
  for (int64_t q = 0; q < r; q++) {
    double total = pw_sum(d, n);
    if (total <= 0) {
      /* mass exhausted: rng.choice(setdiff1d(arange(n), picked), r-np, False) */
      char *used = (char *)calloc((size_t)n, 1);
      for (int64_t k = 0; k < np_; k++) used[removed[k]] = 1;
      int64_t *rest = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
      int64_t nrest = 0;
      for (int64_t k = 0; k < n; k++) if (!used[k]) rest[nrest++] = k;
      int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(r - np_));
      choice_noreplace(g, nrest, r - np_, fill);
      for (int64_t k = 0; k < r - np_; k++) removed[np_ + k] = rest[fill[k]];
      np_ = r;
      free(used); free(rest); free(fill);
      break;
    }
    for (int64_t k = 0; k < n; k++) p[k] = d[k] / total;
    int64_t k = choice_p(g, p, n, cdf);
    removed[np_++] = k;
    d[k] = 0.0;
  }
  free(d); free(p); free(cdf);
  qsort(removed, (size_t)r, sizeof(int64_t), cmp_i64);
}

/* random_repair operators.py:108-117 */
static void random_repair(const oprob *P, const amvm_params *prm, osol *S, const int64_t *removed,
                          const int32_t *saved, int64_t r, pcg_t *g) {
  for (int64_t q = 0; q < r; q++) {
    int32_t c1, c2;
    two_nearest(P->lv, P->nlev, P->lv[saved[q]], &c1, &c2);
    uint64_t coin = pcg_bounded(g, 1);
    apply_shift(P, prm, S, removed[q], coin ? c2 : c1);
  }
}

/* greedy_repair operators.py:120-138: the exact in-place sequence */
static void greedy_repair(const oprob *P, const amvm_params *prm, osol *S, const int64_t *removed,
                          const int32_t *saved, int64_t r, ocount *C) {
  for (int64_t q = 0; q < r; q++) {
    int64_t j = removed[q];
    int32_t c1, c2;
    two_nearest(P->lv, P->nlev, P->lv[saved[q]], &c1, &c2);
    apply_shift(P, prm, S, j, c1);
    double t1 = S->obj;
    apply_shift(P, prm, S, j, c2);
    double t2 = S->obj;
    if (C) { C->moves_ref += 2; C->moves_raw += 2; }
    if (t1 < t2 || (t1 == t2 && P->lv[c1] < P->lv[c2])) apply_shift(P, prm, S, j, c1);
  }
}

/* --------------------------------------------------------------- controller */
/* accept controller.py:168-183 */
static int accept(const amvm_params *prm, const osol *cur, const osol *cand, int64_t m) {
  if (cand->obj < cur->obj) return 1;
  if (prm->l2_tiebreak && cand->obj <= cur->obj + prm->accept_tie_tol &&
      sqrt(ddot_skx(cand->r, m)) < sqrt(ddot_skx(cur->r, m)))
    return 1;
  return 0;
}

typedef struct {
  double w[4], sc[4];
  int64_t seg[4], life[4], it;
} obank;

/* select_operators controller.py:88-90 */
static int select_pair(const obank *B, pcg_t *g) {
  double p[4], cdf[4];
  double s = pw_sum(B->w, 4);
  for (int k = 0; k < 4; k++) p[k] = B->w[k] / s;
  return (int)choice_p(g, p, 4, cdf);
}

/* update_weights controller.py:99-131; outcome 0 new best .. 3 rejected */
static void update_weights(obank *B, const amvm_params *prm, int pair, int outcome) {
  double pts = outcome == 0 ? prm->sigma1 : outcome == 1 ? prm->sigma2 : outcome == 2 ? prm->sigma3 : 0.0;
  B->sc[pair] += pts;
  B->seg[pair] += 1;
  B->life[pair] += 1;
  B->it += 1;
  if (B->it % prm->n_segment == 0) {
    double keep = 1 - prm->decay;
    for (int k = 0; k < 4; k++) {
      double nrm = B->seg[k] > 0 ? B->sc[k] / (double)B->seg[k] : 0.0;
      double w = prm->decay * B->w[k] + keep * nrm;
      B->w[k] = w < prm->weight_floor ? prm->weight_floor : w;
      B->sc[k] = 0.0;
      B->seg[k] = 0;
    }
  }
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void sol_copy(osol *dst, const osol *src, int64_t m, int64_t n) {
  memcpy(dst->idx, src->idx, sizeof(int32_t) * (size_t)n);
  memcpy(dst->r, src->r, sizeof(double) * (size_t)m);
  dst->obj = src->obj;
  dst->cnt = src->cnt;
}

typedef struct {
  const oprob *P;
  const amvm_params *prm;
} octx;

/* solve controller.py:211-286 for one instance.  Returns iterations. */
static int32_t solve_one(const oprob *P, const amvm_params *prm, osol *cur0, pcg_t *g, osol *best_out,
                         int64_t *op_uses, double *tr_cur, double *tr_best, uint8_t *tr_pair,
                         uint8_t *tr_acc, ocount *C) {
  int64_t m = P->m, n = P->n, r = prm->r;
  double started = now_s();
  osol bufs[2];
  for (int k = 0; k < 2; k++) {
    bufs[k].idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    bufs[k].r = (double *)malloc(sizeof(double) * (size_t)m);
  }
  osol *cur = &bufs[0], *cand = &bufs[1];
  sol_copy(cur, cur0, m, n);
  sol_copy(best_out, cur, m, n);
  obank B;
  for (int k = 0; k < 4; k++) { B.w[k] = 1.0; B.sc[k] = 0.0; B.seg[k] = 0; B.life[k] = 0; }
  B.it = 0;
  int64_t *removed = (int64_t *)malloc(sizeof(int64_t) * (size_t)r);
  int32_t *saved = (int32_t *)malloc(sizeof(int32_t) * (size_t)r);
  int32_t it = 0;
  while (it < prm->max_iters) {
    if (best_out->obj == 0.0) break;
    if (prm->time_limit_s >= 0 && now_s() - started > prm->time_limit_s) break;
    it++;
    int pair = select_pair(&B, g);
    sol_copy(cand, cur, m, n);
    if (pair < 2) random_destroy(g, n, r, removed);
    else worst_destroy(P, cand, r, prm->alpha, g, removed);
    for (int64_t q = 0; q < r; q++) saved[q] = cand->idx[removed[q]];
    if ((pair & 1) == 0) random_repair(P, prm, cand, removed, saved, r, g);
    else greedy_repair(P, prm, cand, removed, saved, r, C);
    local_search(P, prm, cand, C);
    int acc = accept(prm, cur, cand, m);
    int outcome;
    if (acc && cand->obj < best_out->obj) outcome = 0;
    else if (acc && cand->obj < cur->obj) outcome = 1;
    else if (acc) outcome = 2;
    else outcome = 3;
    if (acc) {
      osol *t = cur; cur = cand; cand = t;
      if (cur->obj < best_out->obj) sol_copy(best_out, cur, m, n);
    }
    update_weights(&B, prm, pair, outcome);
    if (tr_cur) {
      tr_cur[it - 1] = cur->obj;
      tr_best[it - 1] = best_out->obj;
      tr_pair[it - 1] = (uint8_t)pair;
      tr_acc[it - 1] = (uint8_t)acc;
    }
  }
  for (int k = 0; k < 4; k++) op_uses[k] = B.life[k];
  for (int k = 0; k < 2; k++) { free(bufs[k].idx); free(bufs[k].r); }
  free(removed); free(saved);
  return it;
}

/* ================================================================ C-ABI */
/* orc_problem mirrors amvm_problem but with A ROW-MAJOR on the HOST.      */
typedef struct {
  int64_t m, n, nlev, count;
  const double *A;      /* m x n row-major */
  const double *B;      /* count x m */
  const double *levels; /* count x nlev */
  const double *At;     /* optional n x m column-major copy of A, or NULL */
} orc_problem;

static void mk_prob(const orc_problem *p, int64_t k, oprob *P) {
  P->m = p->m; P->n = p->n; P->nlev = p->nlev; P->A = p->A; P->At = p->At;
  P->b = p->B + k * p->m;
  P->lv = p->levels + k * p->nlev;
}
static void mk_sol(const amvm_solution *s, int64_t k, int64_t m, int64_t n, osol *S) {
  S->idx = s->idx + k * n;
  S->r = s->residual + k * m;
  S->obj = s->objective[k];
  S->cnt = s->updates[k];
}
static void put_sol(const osol *S, amvm_solution *s, int64_t k) {
  s->objective[k] = S->obj;
  s->updates[k] = S->cnt;
}

typedef struct {
  const orc_problem *prob;
  const amvm_params *prm;
  const amvm_solution *start;
  amvm_pcg64 *rng;
  amvm_result *res;
  int64_t next;
  pthread_mutex_t mu;
} orc_batch;

static void solve_instance(orc_batch *B, int64_t k) {
  const orc_problem *pp = B->prob;
  int64_t m = pp->m, n = pp->n, T = B->prm->max_iters;
  oprob P;
  mk_prob(pp, k, &P);
  osol s0, best;
  mk_sol(B->start, k, m, n, &s0);
  best.idx = B->res->best.idx + k * n;
  best.r = B->res->best.residual + k * m;
  pcg_t g;
  pcg_load(&g, &B->rng[k]);
  ocount C = {0, 0};
  amvm_result *R = B->res;
  int32_t it = solve_one(&P, B->prm, &s0, &g, &best, R->operator_uses + 4 * k,
                         R->trace_current_t ? R->trace_current_t + k * T : NULL,
                         R->trace_best_t ? R->trace_best_t + k * T : NULL,
                         R->trace_pair ? R->trace_pair + k * T : NULL,
                         R->trace_accepted ? R->trace_accepted + k * T : NULL, &C);
  put_sol(&best, &R->best, k);
  R->iterations[k] = it;
  R->initial_objective[k] = s0.obj;
  if (R->moves_scored) { R->moves_scored[2 * k] = C.moves_ref; R->moves_scored[2 * k + 1] = C.moves_raw; }
  pcg_store(&g, &B->rng[k]);
}

static void *batch_worker(void *arg) {
  orc_batch *B = (orc_batch *)arg;
  for (;;) {
    pthread_mutex_lock(&B->mu);
    int64_t k = B->next++;
    pthread_mutex_unlock(&B->mu);
    if (k >= B->prob->count) break;
    solve_instance(B, k);
  }
  return NULL;
}

/* Host counterpart of amvm_solve (all pointers HOST).  threads <= 1 runs
 * the instances sequentially on the calling thread. */
int orc_solve(const orc_problem *prob, const amvm_params *prm, const amvm_solution *start,
              amvm_pcg64 *rng, amvm_result *res, int threads) {
  if (!prob || !prm || !start || !rng || !res) return AMVM_ERR_INVALID;
  orc_batch B;
  memset(&B, 0, sizeof(B));
  B.prob = prob; B.prm = prm; B.start = start; B.rng = rng; B.res = res;
  pthread_mutex_init(&B.mu, NULL);
  if (threads <= 1 || prob->count <= 1) {
    batch_worker(&B);
  } else {
    int nt = threads < prob->count ? threads : (int)prob->count;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nt);
    for (int t = 0; t < nt; t++) pthread_create(&th[t], NULL, batch_worker, &B);
    for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&B.mu);
  return AMVM_OK;
}

int orc_one_opt(const orc_problem *prob, const amvm_params *prm, amvm_solution *sol) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  one_opt(&P, prm, &S, NULL);
  put_sol(&S, sol, 0);
  return AMVM_OK;
}

int orc_local_search(const orc_problem *prob, const amvm_params *prm, amvm_solution *sol) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  local_search(&P, prm, &S, NULL);
  put_sol(&S, sol, 0);
  return AMVM_OK;
}

int orc_find_candidates(const orc_problem *prob, const amvm_params *prm, const amvm_solution *sol,
                        int32_t *oi, int32_t *oj, double *od, int32_t *count, int32_t cap) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  if (S.obj <= 0) return AMVM_ERR_INVALID;
  ocand *c;
  int64_t cnt = find_candidates(&P, prm, &S, &c);
  if (cnt > cap) cnt = cap;
  for (int64_t q = 0; q < cnt; q++) { oi[q] = c[q].i; oj[q] = c[q].j; od[q] = c[q].delta; }
  *count = (int32_t)cnt;
  free(c);
  return AMVM_OK;
}

int orc_best_swap(const orc_problem *prob, const amvm_params *prm, const amvm_solution *sol, double *out4) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  int32_t i = -1, j = -1;
  double d = 0, t = 0;
  if (!best_swap(&P, prm, &S, &i, &j, &d, &t, NULL)) { i = -1; j = -1; d = 0; t = 0; }
  out4[0] = i; out4[1] = j; out4[2] = d; out4[3] = t;
  return AMVM_OK;
}

int orc_impact_scores(const orc_problem *prob, const amvm_params *prm, const amvm_solution *sol, double *d) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  if (S.obj <= 0 || prm->alpha < 0) return AMVM_ERR_INVALID;
  impact_scores(&P, &S, prm->alpha, d);
  return AMVM_OK;
}

int orc_destroy(const orc_problem *prob, const amvm_params *prm, int kind, const amvm_solution *sol,
                amvm_pcg64 *rng, int32_t *removed) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  int64_t r = prm->r;
  if (r < 1 || r > prob->n) return AMVM_ERR_INVALID;
  pcg_t g;
  pcg_load(&g, rng);
  int64_t *rem = (int64_t *)malloc(sizeof(int64_t) * (size_t)r);
  if (kind == 0) random_destroy(&g, prob->n, r, rem);
  else worst_destroy(&P, &S, r, prm->alpha, &g, rem);
  for (int64_t q = 0; q < r; q++) removed[q] = (int32_t)rem[q];
  free(rem);
  pcg_store(&g, rng);
  return AMVM_OK;
}

int orc_repair(const orc_problem *prob, const amvm_params *prm, int kind, amvm_solution *sol,
               amvm_pcg64 *rng, const int32_t *removed, const int32_t *saved, int32_t r) {
  oprob P; osol S;
  mk_prob(prob, 0, &P);
  mk_sol(sol, 0, prob->m, prob->n, &S);
  if (prob->nlev < 2) return AMVM_ERR_INVALID;
  int64_t *rem = (int64_t *)malloc(sizeof(int64_t) * (size_t)(r > 0 ? r : 1));
  for (int32_t q = 0; q < r; q++) rem[q] = removed[q];
  pcg_t g;
  pcg_load(&g, rng);
  if (kind == 0) random_repair(&P, prm, &S, rem, saved, r, &g);
  else greedy_repair(&P, prm, &S, rem, saved, r, NULL);
  pcg_store(&g, rng);
  put_sol(&S, sol, 0);
  free(rem);
  return AMVM_OK;
}

/* Exposed numpy-arithmetic helpers (so the CPU tests can pin them). */
double orc_pairwise_sum(const double *a, int64_t n) { return pw_sum(a, n); }
double orc_norm(const double *x, int64_t n) { return sqrt(ddot_skx(x, n)); }
double orc_random(amvm_pcg64 *st) {
  pcg_t g; pcg_load(&g, st);
  double v = pcg_random(&g);
  pcg_store(&g, st);
  return v;
}
int64_t orc_bounded(amvm_pcg64 *st, int64_t rng_max) {
  pcg_t g; pcg_load(&g, st);
  int64_t v = (int64_t)pcg_bounded(&g, (uint64_t)rng_max);
  pcg_store(&g, st);
  return v;
}
void orc_choice_noreplace(amvm_pcg64 *st, int64_t pop, int64_t r, int64_t *out) {
  pcg_t g; pcg_load(&g, st);
  choice_noreplace(&g, pop, r, out);
  pcg_store(&g, st);
}
int64_t orc_choice_p(amvm_pcg64 *st, const double *p, int64_t k) {
  pcg_t g; pcg_load(&g, st);
  double *cdf = (double *)malloc(sizeof(double) * (size_t)k);
  int64_t v = choice_p(&g, p, k, cdf);
  free(cdf);
  pcg_store(&g, st);
  return v;
}

void orc_gemv(const double *A, int64_t m, int64_t K, const double *x, double *y) {
  gemv_numpy(A, m, K, x, y);
}
