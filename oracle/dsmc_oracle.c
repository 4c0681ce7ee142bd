/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * dSMC smoothing path (see dsmc_oracle.h). Compiled with -ffp-contract=off
 * so every a*b+c is two roundings unless written as fma(), exactly like the
 * reference's scalar TUs (no -mfma on them, oracle/Makefile).
 */
#define _GNU_SOURCE
#include "dsmc_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* or_last_error(void) { return g_err; }

#define NEG_INF (-INFINITY)
static const double kLog2Pi = 1.8378770664093454836;

/* ------------------------------------------------------------------ RNG */
/* Philox4x64-10, rng.cpp:14-41. */
void or_philox(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  uint64_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  uint64_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ull * x0;
    unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ull * x2;
    uint64_t lo0 = (uint64_t)p0, hi0 = (uint64_t)(p0 >> 64);
    uint64_t lo1 = (uint64_t)p1, hi1 = (uint64_t)(p1 >> 64);
    uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0;
    x1 = lo1;
    x2 = n2;
    x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = x0;
  out[1] = x1;
  out[2] = x2;
  out[3] = x3;
}

typedef struct {
  uint64_t ctr[4], key[2], buf[4];
  int pos;
  double cached;
  int has_cached;
} stream_t;

/* rng.cpp:45-53: ctr = {block, node, level<<16 | role, substream}. */
static void st_init(stream_t* s, uint64_t seed, uint32_t level, uint64_t node,
                    int role, uint64_t substream) {
  s->ctr[0] = 0;
  s->ctr[1] = node;
  s->ctr[2] = ((uint64_t)level << 16) | (uint64_t)(uint16_t)role;
  s->ctr[3] = substream;
  s->key[0] = seed;
  s->key[1] = 0x243F6A8885A308D3ull;
  s->pos = 4;
  s->has_cached = 0;
}
static uint64_t st_u64(stream_t* s) {
  if (s->pos == 4) {
    or_philox(s->ctr, s->key, s->buf);
    ++s->ctr[0];
    s->pos = 0;
  }
  return s->buf[s->pos++];
}
/* rng.cpp:66-72 */
static double st_uniform(stream_t* s) {
  return (double)(st_u64(s) >> 11) * 0x1.0p-53;
}
static double st_uniform_pos(stream_t* s) {
  return ((double)(st_u64(s) >> 12) + 0.5) * 0x1.0p-52;
}
/* rng.cpp:74-86: Box-Muller, cos first then the cached sin. */
static double st_normal(stream_t* s) {
  if (s->has_cached) {
    s->has_cached = 0;
    return s->cached;
  }
  double u1 = st_uniform_pos(s);
  double u2 = st_uniform(s);
  double r = sqrt(-2.0 * log(u1));
  double th = 2.0 * 3.14159265358979323846 * u2;
  s->cached = r * sin(th);
  s->has_cached = 1;
  return r * cos(th);
}
/* rng.cpp:88-93 */
static uint64_t st_index(stream_t* s, uint64_t n) {
  unsigned __int128 p = (unsigned __int128)st_u64(s) * n;
  return (uint64_t)(p >> 64);
}

void or_stream(uint64_t seed, uint32_t level, uint64_t node, int role,
               uint64_t substream, int kind, size_t n, void* out) {
  stream_t s;
  st_init(&s, seed, level, node, role, substream);
  for (size_t i = 0; i < n; ++i) {
    if (kind == 0) ((uint64_t*)out)[i] = st_u64(&s);
    else if (kind == 1) ((double*)out)[i] = st_uniform(&s);
    else if (kind == 2) ((double*)out)[i] = st_uniform_pos(&s);
    else ((double*)out)[i] = st_normal(&s);
  }
}

/* -------------------------------------------------------------- numerics */
/* exp_poly.hpp:13-51 */
static const double kExpC[14] = {
    1.0,          1.0,           1.0 / 2,        1.0 / 6,        1.0 / 24,
    1.0 / 120,    1.0 / 720,     1.0 / 5040,     1.0 / 40320,    1.0 / 362880,
    1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600, 1.0 / 6227020800.0};

double or_exp_w(double x) {
  if (isnan(x)) return x;
  if (x <= -708.0) return 0.0;
  double xc = x > 710.0 ? 710.0 : x;
  double k = nearbyint(xc * 1.4426950408889634074);
  double r = fma(k, -6.93147180369123816490e-01, xc);
  r = fma(k, -1.90821492927058770002e-10, r);
  double p = kExpC[13];
  for (int i = 12; i >= 0; --i) p = fma(p, r, kExpC[i]);
  int64_t ki = (int64_t)k;
  uint64_t bits = (uint64_t)(ki + 1023) << 52;
  double scale;
  memcpy(&scale, &bits, 8);
  return p * scale;
}

/* exp_poly.hpp:78-84 */
static double combine8(const double a[8]) {
  double b0 = a[0] + a[4], b1 = a[1] + a[5], b2 = a[2] + a[6], b3 = a[3] + a[7];
  return (b0 + b2) + (b1 + b3);
}

/* kernels.cpp:38-44 */
double or_reduce_sum(const double* x, size_t n) {
  double acc[8] = {0};
  size_t n8 = n & ~(size_t)7;
  for (size_t i = 0; i < n8; i += 8)
    for (int l = 0; l < 8; ++l) acc[l] += x[i + l];
  double t = combine8(acc);
  for (size_t i = n8; i < n; ++i) t += x[i];
  return t;
}

/* kernels.cpp:26-36; returns 0 or DSMC_E_DOMAIN on NaN */
static int reduce_max(const double* x, size_t n, double* out) {
  double m = NEG_INF;
  int nan = 0;
  for (size_t i = 0; i < n; ++i) {
    nan |= isnan(x[i]);
    if (x[i] > m) m = x[i];
  }
  *out = m;
  return nan ? fail(DSMC_E_DOMAIN, "reduce_max: NaN entry") : 0;
}

/* kernels.cpp:46-55 */
double or_log_sum_exp(const double* x, size_t n) {
  double m;
  if (reduce_max(x, n, &m)) return NAN;
  if (m == NEG_INF) return NEG_INF;
  double acc[8] = {0};
  size_t n8 = n & ~(size_t)7;
  for (size_t i = 0; i < n8; i += 8)
    for (int l = 0; l < 8; ++l) acc[l] += or_exp_w(x[i + l] - m);
  double t = combine8(acc);
  for (size_t i = n8; i < n; ++i) t += or_exp_w(x[i] - m);
  return m + log(t);
}

/* kernels.cpp:93-116, kSubBlock = 64 (kernels.hpp:77) */
#define SUB 64
double or_exp_row_store(const double* logw, size_t n, double shift, double* w,
                        double* sub) {
  double total = 0.0;
  size_t b = 0;
  for (size_t s = 0; s < n; s += SUB, ++b) {
    size_t len = n - s < SUB ? n - s : SUB;
    double acc[8] = {0};
    size_t len8 = len & ~(size_t)7;
    for (size_t i = 0; i < len8; i += 8)
      for (int l = 0; l < 8; ++l) {
        double z = or_exp_w(logw[s + i + l] - shift);
        w[s + i + l] = z;
        acc[l] += z;
      }
    double bs = combine8(acc);
    for (size_t i = len8; i < len; ++i) {
      double z = or_exp_w(logw[s + i] - shift);
      w[s + i] = z;
      bs += z;
    }
    sub[b] = bs;
    total += bs;
  }
  return total;
}

/* kernels.cpp:57-65: out = fma(c, (x - mean)^2, base) */
static void gaussian_row(const double* x, size_t n, double mean, double c,
                         const double* base, double* out) {
  for (size_t i = 0; i < n; ++i) {
    double t = x[i] - mean;
    out[i] = fma(c, t * t, base ? base[i] : 0.0);
  }
}

/* ------------------------------------------------------- pair sources */
typedef struct pair_src {
  size_t n;
  void* ctx;
  /* row i into out (n); returns 0 or an error code */
  int (*fill_row)(const struct pair_src*, size_t i, double* out);
  int (*entry)(const struct pair_src*, size_t i, size_t j, double* out);
  int has_bound;
  double bound;
} pair_src;

typedef struct {
  uint32_t* left;
  uint32_t* right;
  double lmw;
  int has_lmw;
  uint64_t evals;
  int biased;
} pair_sample;

/* DenseTable + build_dense (resampling.cpp:48-104) */
typedef struct {
  size_t n, nsub;
  double *w, *sub, *row_scale, *row_total, *prefix;
  double grand, log_sum;
} dense_t;

static void dense_free(dense_t* t) {
  free(t->w);
  free(t->sub);
  free(t->row_scale);
  free(t->row_total);
  free(t->prefix);
}

static int build_dense(const pair_src* src, dense_t* t) {
  size_t n = src->n;
  if (n == 0) return fail(DSMC_E_INVALID_ARGUMENT, "pair weight source has n == 0");
  memset(t, 0, sizeof *t);
  t->n = n;
  t->nsub = (n + SUB - 1) / SUB;
  t->w = calloc(n * n, sizeof(double));
  t->sub = calloc(n * t->nsub, sizeof(double));
  t->row_scale = calloc(n, sizeof(double));
  t->row_total = calloc(n, sizeof(double));
  t->prefix = calloc(n, sizeof(double));
  double* row = malloc(n * sizeof(double));
  double* mx = malloc(n * sizeof(double));
  double* raw = calloc(n, sizeof(double));
  int rc = 0;
  for (size_t i = 0; i < n && !rc; ++i) {
    rc = src->fill_row(src, i, row);
    if (rc) break;
    rc = reduce_max(row, n, &mx[i]);
    if (rc) break;
    if (mx[i] == NEG_INF) continue;
    raw[i] = or_exp_row_store(row, n, mx[i], t->w + i * n, t->sub + i * t->nsub);
  }
  double g = NEG_INF;
  if (!rc) rc = reduce_max(mx, n, &g);
  if (!rc && g == NEG_INF)
    rc = fail(DSMC_E_RUNTIME,
              "all pair weights are zero; the blocks share no support under "
              "the model");
  if (!rc) {
    for (size_t i = 0; i < n; ++i) {
      t->row_scale[i] = or_exp_w(mx[i] - g);
      t->row_total[i] = t->row_scale[i] * raw[i];
    }
    t->grand = or_reduce_sum(t->row_total, n);
    t->log_sum = g + log(t->grand);
    /* sequential inclusive prefix = the walk's running `cum` (:113-121) */
    double cum = 0.0;
    for (size_t i = 0; i < n; ++i) {
      cum += t->row_total[i];
      t->prefix[i] = cum;
    }
  }
  free(row);
  free(mx);
  free(raw);
  if (rc) dense_free(t);
  return rc;
}

/* select_sorted (resampling.cpp:109-153) restated per point: the sorted walk
 * lands on i = min{i : pt < S_i} (else n-1) for every point, so each slot is
 * independent. */
static void select_point(const dense_t* t, double pt, uint32_t* row_out,
                         uint32_t* col_out) {
  size_t n = t->n;
  size_t lo = 0, hi = n;  /* first i with pt < S_i */
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if (pt < t->prefix[mid]) hi = mid;
    else lo = mid + 1;
  }
  size_t i = lo < n ? lo : n - 1;
  double cum_before = i > 0 ? t->prefix[i - 1] : 0.0;
  size_t row = i;
  while (row > 0 && t->row_total[row] <= 0.0) --row;
  const double* wrow = t->w + row * n;
  const double* srow = t->sub + row * t->nsub;
  double local = (pt - cum_before) / t->row_scale[row];
  if (!(local >= 0.0)) local = 0.0;
  size_t s = 0;
  double c2_before = 0.0, c2 = srow[0];
  while (!(local < c2) && s + 1 < t->nsub) {
    c2_before = c2;
    ++s;
    c2 += srow[s];
  }
  size_t j0 = s * SUB, j1 = j0 + SUB < n ? j0 + SUB : n;
  double c3 = c2_before;
  size_t j = j0;
  for (; j < j1; ++j) {
    c3 += wrow[j];
    if (local < c3) break;
  }
  if (j == j1) {
    j = j1 - 1;
    while (j > 0 && !(wrow[j] > 0.0)) --j;
  }
  *row_out = (uint32_t)row;
  *col_out = (uint32_t)j;
}

/* multinomial_pairs / systematic_pairs (resampling.cpp:181-231) */
static int dense_pairs(const pair_src* src, size_t n_out, int systematic,
                       uint64_t seed, uint32_t level, uint64_t node,
                       pair_sample* ps) {
  dense_t t;
  int rc = build_dense(src, &t);
  if (rc) return rc;
  ps->lmw = t.log_sum;
  ps->has_lmw = 1;
  ps->evals = (uint64_t)src->n * src->n;
  ps->biased = 0;
  if (n_out) {
    stream_t s;
    st_init(&s, seed, level, node, DSMC_ROLE_PAIR_RESAMPLE, 0);
    if (systematic) {
      double u = st_uniform(&s);
      double step = t.grand / (double)n_out;
      for (size_t k = 0; k < n_out; ++k)
        select_point(&t, (u + (double)k) * step, &ps->left[k], &ps->right[k]);
    } else {
      for (size_t k = 0; k < n_out; ++k)
        select_point(&t, st_uniform(&s) * t.grand, &ps->left[k], &ps->right[k]);
    }
  }
  dense_free(&t);
  return 0;
}

static int checked_entry(const pair_src* src, size_t i, size_t j, double* v) {
  int rc = src->entry(src, i, j, v);
  if (rc) return rc;
  if (isnan(*v))
    return fail(DSMC_E_INVALID_ARGUMENT, "pair weight (%zu, %zu) is NaN", i, j);
  return 0;
}

/* mh_lazy_pairs (resampling.cpp:233-282) */
static int mh_pairs(const pair_src* src, size_t n_out, size_t steps,
                    uint64_t seed, uint32_t level, uint64_t node,
                    pair_sample* ps) {
  size_t n = src->n;
  if (n == 0) return fail(DSMC_E_INVALID_ARGUMENT, "pair weight source has n == 0");
  ps->biased = 1;
  ps->has_lmw = 0;
  ps->evals = 0;
  for (size_t m = 0; m < n_out; ++m) {
    uint32_t i = (uint32_t)(m % n), j = i;
    if (steps) {
      stream_t s;
      st_init(&s, seed, level, node, DSMC_ROLE_PAIR_RESAMPLE, m + 1);
      double cur = 0.0;
      int have = 0;
      for (size_t b = 0; b < steps; ++b) {
        uint32_t pi = (uint32_t)st_index(&s, n), pj = (uint32_t)st_index(&s, n);
        double lu = log(st_uniform_pos(&s));
        int rc;
        if (!have) {
          if ((rc = checked_entry(src, i, j, &cur))) return rc;
          ++ps->evals;
          have = 1;
        }
        double prop;
        if ((rc = checked_entry(src, pi, pj, &prop))) return rc;
        ++ps->evals;
        if (lu < prop - cur) {
          i = pi;
          j = pj;
          cur = prop;
        }
      }
    }
    ps->left[m] = i;
    ps->right[m] = j;
  }
  return 0;
}

/* rejection_lazy_pairs (resampling.cpp:284-324) */
static int rejection_pairs(const pair_src* src, size_t n_out, uint64_t seed,
                           uint32_t level, uint64_t node, pair_sample* ps) {
  size_t n = src->n;
  if (n == 0) return fail(DSMC_E_INVALID_ARGUMENT, "pair weight source has n == 0");
  if (!src->has_bound || !isfinite(src->bound))
    return fail(DSMC_E_INVALID_ARGUMENT,
                "rejection resampling requires a finite log_upper_bound");
  ps->biased = 0;
  ps->has_lmw = 0;
  ps->evals = 0;
  for (size_t m = 0; m < n_out; ++m) {
    stream_t s;
    st_init(&s, seed, level, node, DSMC_ROLE_PAIR_RESAMPLE, m + 1);
    int ok = 0;
    for (uint64_t trial = 0; trial < (1u << 24); ++trial) {
      uint32_t i = (uint32_t)st_index(&s, n), j = (uint32_t)st_index(&s, n);
      double lw;
      int rc = checked_entry(src, i, j, &lw);
      if (rc) return rc;
      ++ps->evals;
      if (lw - src->bound > 1e-9)
        return fail(DSMC_E_INVALID_ARGUMENT,
                    "pair weight exceeds its stated upper bound");
      if (log(st_uniform_pos(&s)) <= lw - src->bound) {
        ps->left[m] = i;
        ps->right[m] = j;
        ok = 1;
        break;
      }
    }
    if (!ok)
      return fail(DSMC_E_RUNTIME,
                  "rejection resampling exceeded the trial cap; the bound is "
                  "far too loose or the weights are degenerate");
  }
  return 0;
}

static int resample(int resampler, const pair_src* src, size_t n_out,
                    size_t mh_steps, uint64_t seed, uint32_t level,
                    uint64_t node, pair_sample* ps) {
  switch (resampler) {
    case DSMC_MULTINOMIAL:
      return dense_pairs(src, n_out, 0, seed, level, node, ps);
    case DSMC_SYSTEMATIC:
      return dense_pairs(src, n_out, 1, seed, level, node, ps);
    case DSMC_MH_LAZY:
      return mh_pairs(src, n_out, mh_steps, seed, level, node, ps);
    case DSMC_REJECTION_LAZY:
      return rejection_pairs(src, n_out, seed, level, node, ps);
  }
  return fail(DSMC_E_INVALID_ARGUMENT, "unknown resampler");
}

/* table source (test_resampling.cpp:17-33) */
typedef struct {
  const double* logw;
} table_ctx;
static int table_fill(const pair_src* s, size_t i, double* out) {
  memcpy(out, ((const table_ctx*)s->ctx)->logw + i * s->n, s->n * sizeof(double));
  return 0;
}
static int table_entry(const pair_src* s, size_t i, size_t j, double* out) {
  *out = ((const table_ctx*)s->ctx)->logw[i * s->n + j];
  return 0;
}

int or_resample_table(int resampler, const double* logw, size_t n,
                      size_t n_out, size_t mh_steps, int has_bound,
                      double bound, uint64_t seed, uint32_t level,
                      uint64_t node, uint32_t* left, uint32_t* right,
                      double* lmw, int* has_lmw, uint64_t* weight_evals,
                      int* biased) {
  table_ctx tc = {logw};
  pair_src src = {n, &tc, table_fill, table_entry, has_bound, bound};
  pair_sample ps = {left, right, 0, 0, 0, 0};
  int rc = resample(resampler, &src, n_out, mh_steps, seed, level, node, &ps);
  if (rc) return rc;
  *lmw = ps.has_lmw ? ps.lmw : NAN;
  *has_lmw = ps.has_lmw;
  *weight_evals = ps.evals;
  *biased = ps.biased;
  return 0;
}

/* --------------------------------------------------------------- schedule */
/* build_schedule (smoother.cpp:64-85): packed-left pairing, odd tail
 * carried; level l block k covers [k 2^l, min((k+1) 2^l, K) - 1]. */
int or_build_schedule(int horizon, int* pairs) {
  int K = horizon + 1, nb = K, levels = 0, cursor = 0, span = 1;
  while (nb > 1) {
    ++levels;
    for (int k = 0; k < nb / 2; ++k, ++cursor) {
      int* o = pairs + 5 * cursor;
      o[0] = levels;
      o[1] = k;
      o[2] = 2 * k * span;
      o[3] = (2 * k + 1) * span - 1;
      int rb = (2 * k + 2) * span - 1;
      o[4] = rb < K - 1 ? rb : K - 1;
    }
    nb = (nb + 1) / 2;
    span *= 2;
  }
  return levels;
}

/* ----------------------------------------------------------------- models */
static double log_normal_pdf(double x, double mean, double var) {
  double d = x - mean;
  return -0.5 * (kLog2Pi + log(var)) - d * d / (2.0 * var);
}

static int chol(const double* A, int d, double* L) {
  memset(L, 0, sizeof(double) * d * d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * d + j];
      for (int k = 0; k < j; ++k) s -= L[i * d + k] * L[j * d + k];
      if (i == j) {
        if (!(s > 0.0)) return 0;
        L[i * d + i] = sqrt(s);
      } else {
        L[i * d + j] = s / L[j * d + j];
      }
    }
  return 1;
}
static void tri_inv(const double* L, int d, double* W) {
  memset(W, 0, sizeof(double) * d * d);
  for (int i = 0; i < d; ++i) {
    W[i * d + i] = 1.0 / L[i * d + i];
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L[i * d + k] * W[k * d + j];
      W[i * d + j] = -s / L[i * d + i];
    }
  }
}
typedef struct {
  int d;
  double W[16], L[16], norm;
} gauss_t;
static int gauss_init(gauss_t* g, const double* S, int d) {
  g->d = d;
  if (!chol(S, d, g->L)) return 0;
  tri_inv(g->L, d, g->W);
  double ld = 0.0;
  for (int i = 0; i < d; ++i) ld += 2.0 * log(g->L[i * d + i]);
  g->norm = -0.5 * (d * kLog2Pi + ld);
  return 1;
}
static double gauss_quad(const gauss_t* g, const double* x, const double* m) {
  double e[4], q = 0.0;
  for (int k = 0; k < g->d; ++k) e[k] = x[k] - m[k];
  for (int k = 0; k < g->d; ++k) {
    double z = 0.0;
    for (int l = 0; l <= k; ++l) z += g->W[k * g->d + l] * e[l];
    q += z * z;
  }
  return q;
}
static double gauss_logpdf(const gauss_t* g, const double* x, const double* m) {
  return g->norm - 0.5 * gauss_quad(g, x, m);
}

typedef struct {
  const dsmc_model_desc* m;
  int d, dy, T, kind;
  /* LGSSM per time (expanded): */
  gauss_t *prop, *trans, *obs, init;
  /* SV */
  double* logabsy;
  /* COX (models.cpp:127-135) / CRW (models.cpp:269-270) / THETA
     (models.cpp:427-431) constants */
  double slope, icept, stat_mean, stat_var, trans_norm, var, obs_norm, r2;
  double tau0, tau1, tau2;
  double* lgam;
} model_t;

static const double* at(const double* p, int64_t stride, int t) {
  return p + stride * t;
}

static int model_init(model_t* M, const dsmc_model_desc* m) {
  memset(M, 0, sizeof *M);
  M->m = m;
  M->kind = m->kind;
  M->d = m->state_dim;
  M->dy = m->obs_dim;
  M->T = m->horizon;
  int K = m->horizon + 1;
  if (m->horizon < 0) return fail(DSMC_E_INVALID_ARGUMENT, "model: horizon must be >= 0");
  if (m->kind == DSMC_MODEL_SV) {
    if (M->d != 1) return fail(DSMC_E_INVALID_ARGUMENT, "sv: state_dim must be 1");
    if (!(m->sv_sigma2 > 0.0) || !(fabs(m->sv_phi) < 1.0))
      return fail(DSMC_E_INVALID_ARGUMENT, "sv descriptor: need s2 > 0 and |phi| < 1");
    M->logabsy = malloc(sizeof(double) * K);
    for (int t = 0; t < K; ++t) {
      if (!(m->y[t] != 0.0) || !isfinite(m->y[t]))
        return fail(DSMC_E_INVALID_ARGUMENT, "sv descriptor: observations must be finite and nonzero");
      M->logabsy[t] = log(fabs(m->y[t]));
    }
    return 0;
  }
  if (m->kind == DSMC_MODEL_COX) { /* make_cox_model, models.cpp:113-135 */
    if (M->d != 1) return fail(DSMC_E_INVALID_ARGUMENT, "cox: state_dim must be 1");
    double mu = m->par[0], rho = m->par[1], s2 = m->par[2], lam = m->par[3];
    if (!(s2 > 0.0)) return fail(DSMC_E_INVALID_ARGUMENT, "make_cox_model: sigma2 must be > 0");
    if (!(fabs(rho * lam) < 1.0))
      return fail(DSMC_E_INVALID_ARGUMENT, "make_cox_model: need |rho * lambda| < 1");
    M->lgam = malloc(sizeof(double) * K);
    for (int t = 0; t < K; ++t) {
      double y = m->y[t];
      if (y < 0.0 || floor(y) != y)
        return fail(DSMC_E_INVALID_ARGUMENT, "make_cox_model: counts must be nonnegative integers");
      M->lgam[t] = lgamma(y + 1.0);
    }
    M->slope = rho * lam;
    M->icept = mu * (1.0 - rho);
    M->stat_mean = M->icept / (1.0 - M->slope);
    M->stat_var = s2 / (1.0 - M->slope * M->slope);
    M->trans_norm = -0.5 * (kLog2Pi + log(s2));
    M->var = s2;
    return 0;
  }
  if (m->kind == DSMC_MODEL_CRW) { /* make_constrained_rw, models.cpp:265-270 */
    if (M->d != 1) return fail(DSMC_E_INVALID_ARGUMENT, "crw: state_dim must be 1");
    double sigma = m->par[0];
    if (!(sigma > 0.0)) return fail(DSMC_E_INVALID_ARGUMENT, "make_constrained_rw: sigma must be > 0");
    M->var = sigma * sigma;
    M->trans_norm = -0.5 * (kLog2Pi + log(M->var));
    return 0;
  }
  if (m->kind == DSMC_MODEL_THETA) { /* make_theta_logistic, models.cpp:407-431 */
    if (M->d != 1) return fail(DSMC_E_INVALID_ARGUMENT, "theta: state_dim must be 1");
    M->tau0 = m->par[0];
    M->tau1 = m->par[1];
    M->tau2 = m->par[2];
    M->var = m->par[3];
    M->r2 = m->par[4];
    if (!(M->var > 0.0) || !(M->r2 > 0.0))
      return fail(DSMC_E_INVALID_ARGUMENT, "make_theta_logistic: q2 and r2 must be > 0");
    for (int t = 0; t < K; ++t)
      if (!(m->prop_cov[t] > 0.0) || !isfinite(m->prop_mean[t]))
        return fail(DSMC_E_INVALID_ARGUMENT,
                    "make_theta_logistic: proposal marginals must have positive variance");
    M->trans_norm = -0.5 * (kLog2Pi + log(M->var));
    M->obs_norm = -0.5 * (kLog2Pi + log(M->r2));
    return 0;
  }
  if (m->kind != DSMC_MODEL_LGSSM) return fail(DSMC_E_INVALID_ARGUMENT, "unknown model kind");
  int d = M->d, dy = M->dy;
  if (d < 1 || d > 4 || dy < 1 || dy > 4)
    return fail(DSMC_E_INVALID_ARGUMENT, "lgssm descriptor: dims must be 1..4");
  M->prop = calloc(K, sizeof(gauss_t));
  M->trans = calloc(K, sizeof(gauss_t));
  M->obs = calloc(K, sizeof(gauss_t));
  for (int t = 0; t < K; ++t) {
    if (!gauss_init(&M->prop[t], m->prop_cov + (size_t)t * d * d, d))
      return fail(DSMC_E_INVALID_ARGUMENT, "lgssm descriptor: proposal cov not SPD");
    int obs = m->has_obs ? m->has_obs[t] != 0 : 1;
    if (obs && !gauss_init(&M->obs[t], at(m->R, m->R_stride, t), dy))
      return fail(DSMC_E_INVALID_ARGUMENT, "lgssm descriptor: R not SPD");
    if (t >= 1 && !gauss_init(&M->trans[t], at(m->Q, m->Q_stride, t), d))
      return fail(DSMC_E_INVALID_ARGUMENT, "lgssm descriptor: Q not SPD");
  }
  if (!gauss_init(&M->init, m->P0, d))
    return fail(DSMC_E_INVALID_ARGUMENT, "lgssm descriptor: P0 not SPD");
  return 0;
}
static void model_free(model_t* M) {
  free(M->prop);
  free(M->trans);
  free(M->obs);
  free(M->logabsy);
  free(M->lgam);
}
#define THETA(M) ((M)->kind == DSMC_MODEL_THETA)
/* models.cpp:361-363 */
static double theta_drift(const model_t* M, double x) {
  return x + M->tau0 - M->tau1 * exp(M->tau2 * x);
}
#define COX(M) ((M)->kind == DSMC_MODEL_COX)
#define CRW(M) ((M)->kind == DSMC_MODEL_CRW)
static const double kLogHalf = -0.6931471805599453; /* models.cpp:274 */
static int in_box(double x) { return x >= -1.0 && x <= 1.0; } /* models.cpp:260 */
/* models.cpp:103-106 */
static double cox_log_poisson(const model_t* M, int t, double x) {
  return M->m->y[t] * x - exp(x) - M->lgam[t];
}
static int has_obs(const model_t* M, int t) {
  return M->m->has_obs ? M->m->has_obs[t] != 0 : 1;
}
static int lg1(const model_t* M) {
  return M->kind == DSMC_MODEL_LGSSM && M->d == 1 && M->dy == 1;
}
/* scalar accessors for d = 1 */
#define F1(t) (*at(M->m->F, M->m->F_stride, (t)))
#define B1(t) (*at(M->m->b, M->m->b_stride, (t)))
#define Q1(t) (*at(M->m->Q, M->m->Q_stride, (t)))
#define H1(t) (*at(M->m->H, M->m->H_stride, (t)))
#define R1(t) (*at(M->m->R, M->m->R_stride, (t)))

static void lg_mean(const model_t* M, int t, const double* xp, double* mu) {
  const double* F = at(M->m->F, M->m->F_stride, t);
  const double* b = at(M->m->b, M->m->b_stride, t);
  for (int k = 0; k < M->d; ++k) {
    double s = 0.0;
    for (int l = 0; l < M->d; ++l) s += F[k * M->d + l] * xp[l];
    mu[k] = s + b[k];
  }
}
static double lg_log_h(const model_t* M, int t, const double* x) {
  if (!has_obs(M, t)) return 0.0;
  const double* H = at(M->m->H, M->m->H_stride, t);
  double hx[4];
  for (int a = 0; a < M->dy; ++a) {
    double s = 0.0;
    for (int l = 0; l < M->d; ++l) s += H[a * M->d + l] * x[l];
    hx[a] = s;
  }
  return gauss_logpdf(&M->obs[t], M->m->y + (size_t)t * M->dy, hx);
}
static double sv_log_h(const model_t* M, int t, double x) {
  double y = M->m->y[t];
  return -0.5 * (kLog2Pi + x) - y * y / (2.0 * exp(x));
}

/* FeynmanKacModel callbacks restated per model (oracle/ref_models.cpp). */
static double cb_proposal_logdensity(const model_t* M, int t, const double* x) {
  if (THETA(M)) return log_normal_pdf(*x, M->m->prop_mean[t], M->m->prop_cov[t]);
  if (COX(M)) return log_normal_pdf(*x, M->stat_mean, M->stat_var);
  if (CRW(M)) return in_box(*x) ? kLogHalf : NEG_INF;
  if (M->kind == DSMC_MODEL_SV) return M->logabsy[t] + sv_log_h(M, t, *x);
  if (lg1(M)) return log_normal_pdf(*x, M->m->prop_mean[t], M->m->prop_cov[t]);
  return gauss_logpdf(&M->prop[t], x, M->m->prop_mean + (size_t)t * M->d);
}
static double cb_log_potential(const model_t* M, int t, const double* x) {
  if (THETA(M)) return log_normal_pdf(M->m->y[t], *x, M->r2);
  if (COX(M)) return cox_log_poisson(M, t, *x);
  if (CRW(M)) return in_box(*x) ? 0.0 : NEG_INF;
  if (M->kind == DSMC_MODEL_SV) return sv_log_h(M, t, *x);
  if (lg1(M)) {
    if (!has_obs(M, t)) return 0.0;
    return log_normal_pdf(M->m->y[t], H1(t) * *x, R1(t));
  }
  return lg_log_h(M, t, x);
}
static double cb_init_logdensity(const model_t* M, const double* x) {
  if (COX(M)) return log_normal_pdf(*x, M->stat_mean, M->stat_var);
  if (CRW(M) || THETA(M)) return log_normal_pdf(*x, 0.0, 1.0);
  if (M->kind == DSMC_MODEL_SV) {
    double p = M->m->sv_phi;
    return log_normal_pdf(*x, M->m->sv_mu, M->m->sv_sigma2 / (1.0 - p * p));
  }
  if (lg1(M)) return log_normal_pdf(*x, M->m->m0[0], M->m->P0[0]);
  return gauss_logpdf(&M->init, x, M->m->m0);
}
static double cb_transition(const model_t* M, int t, const double* xp,
                            const double* xc) {
  if (COX(M)) return log_normal_pdf(*xc, M->icept + M->slope * *xp, M->var);
  if (CRW(M)) return log_normal_pdf(*xc, *xp, M->var);
  if (THETA(M)) return log_normal_pdf(*xc, theta_drift(M, *xp), M->var);
  if (M->kind == DSMC_MODEL_SV) {
    double mu = M->m->sv_mu;
    return log_normal_pdf(*xc, mu + M->m->sv_phi * (*xp - mu), M->m->sv_sigma2);
  }
  if (lg1(M)) return log_normal_pdf(*xc, F1(t) * *xp + B1(t), Q1(t));
  double mu[4];
  lg_mean(M, t, xp, mu);
  return gauss_logpdf(&M->trans[t], xc, mu);
}

/* proposal_sampler: n draws for time t from the stream into out (n*d). */
static void cb_proposal_sampler(const model_t* M, int t, size_t n,
                                stream_t* s, double* out) {
  int d = M->d;
  if (CRW(M)) { /* models.cpp:278-282: fill_uniform, 2u - 1 */
    for (size_t i = 0; i < n; ++i) out[i] = st_uniform(s);
    for (size_t i = 0; i < n; ++i) out[i] = 2.0 * out[i] - 1.0;
    return;
  }
  for (size_t i = 0; i < n * (size_t)d; ++i) out[i] = st_normal(s);
  if (THETA(M)) { /* models.cpp:434-439 */
    double sd = sqrt(M->m->prop_cov[t]);
    for (size_t i = 0; i < n; ++i) out[i] = M->m->prop_mean[t] + sd * out[i];
    return;
  }
  if (COX(M)) { /* models.cpp:143-148 */
    double sd = sqrt(M->stat_var);
    for (size_t i = 0; i < n; ++i) out[i] = M->stat_mean + sd * out[i];
    return;
  }
  if (M->kind == DSMC_MODEL_SV) {
    double ly2 = 2.0 * M->logabsy[t];
    for (size_t i = 0; i < n; ++i) out[i] = ly2 - log(out[i] * out[i]);
    return;
  }
  if (lg1(M)) {
    double sd = sqrt(M->m->prop_cov[t]);
    for (size_t i = 0; i < n; ++i) out[i] = M->m->prop_mean[t] + sd * out[i];
    return;
  }
  const double* L = M->prop[t].L;
  const double* mu = M->m->prop_mean + (size_t)t * d;
  for (size_t i = 0; i < n; ++i) {
    double z[4], x[4];
    for (int k = 0; k < d; ++k) z[k] = out[i * d + k];
    for (int k = 0; k < d; ++k) {
      double acc = 0.0;
      for (int l = 0; l <= k; ++l) acc += L[k * d + l] * z[l];
      x[k] = mu[k] + acc;
    }
    for (int k = 0; k < d; ++k) out[i * d + k] = x[k];
  }
}

/* log_init_weight (fk_model.cpp:43-59) */
static int leaf_weight(const model_t* M, int t, const double* x, double* w) {
  double v;
  if (COX(M)) { /* init_weight_batch, models.cpp:169-177 */
    *w = t == 0 ? cox_log_poisson(M, 0, *x) : 0.0;
    return 0;
  }
  if (CRW(M)) { /* init_weight_batch, models.cpp:301-311 */
    const double norm = -0.5 * kLog2Pi - kLogHalf;
    *w = !in_box(*x) ? NEG_INF : t == 0 ? norm - 0.5 * *x * *x : 0.0;
    return 0;
  }
  if (t == 0) {
    double pot = cb_log_potential(M, 0, x);
    double p0 = cb_init_logdensity(M, x);
    double q = cb_proposal_logdensity(M, 0, x);
    v = pot + p0 - q;
    if (pot == NEG_INF || p0 == NEG_INF) v = NEG_INF;
  } else {
    double nu = cb_proposal_logdensity(M, t, x);  /* aux == proposal */
    double q = cb_proposal_logdensity(M, t, x);
    v = nu == NEG_INF ? NEG_INF : nu - q;
  }
  if (isnan(v)) return fail(DSMC_E_INVALID_ARGUMENT, "log_init_weight produced NaN");
  *w = v;
  return 0;
}

/* log_stitch_weight (fk_model.cpp:61-73) */
static int stitch_weight(const model_t* M, int c, const double* xp,
                         const double* xc, double* out) {
  double tr = cb_transition(M, c, xp, xc);
  double pot = cb_log_potential(M, c, xc);
  if (tr == NEG_INF || pot == NEG_INF) {
    *out = NEG_INF;
    return 0;
  }
  double nu = cb_proposal_logdensity(M, c, xc);
  if (nu == NEG_INF)
    return fail(DSMC_E_INVALID_ARGUMENT,
                "log_stitch_weight: aux density vanishes where "
                "transition*potential does not (nu_c must dominate)");
  double v = tr + pot - nu;
  if (isnan(v)) return fail(DSMC_E_INVALID_ARGUMENT, "log_stitch_weight produced NaN");
  *out = v;
  return 0;
}

/* Optional sup of log omega_c (rejection bound): models.cpp:657-683 rule for
 * LG d=1; exact for SV; none for LG d>1. */
static int stitch_bound(const model_t* M, int c, double* out) {
  if (COX(M)) return 0; /* models.cpp:210-212: unbounded */
  if (THETA(M)) {       /* models.cpp:473-489: finite at every cut, or none */
    if (M->T < 1) return 0;
    double sc = 0.0;
    for (int cc = 1; cc <= M->T; ++cc) {
      double y = M->m->y[cc], m = M->m->prop_mean[cc], v = M->m->prop_cov[cc];
      double alpha = 1.0 / (2.0 * v) - 1.0 * 1.0 / (2.0 * M->r2);
      double beta = 1.0 * y / M->r2 - m / v;
      double gamma = -y * y / (2.0 * M->r2) + m * m / (2.0 * v) + 0.5 * log(v / M->r2);
      double sv;
      if (alpha < 0.0) sv = gamma - beta * beta / (4.0 * alpha);
      else if (alpha == 0.0 && beta == 0.0) sv = gamma;
      else return 0;
      if (cc == c) sc = sv;
    }
    *out = M->trans_norm + sc;
    return 1;
  }
  if (CRW(M)) {         /* models.cpp:334-335 */
    *out = M->trans_norm - kLogHalf;
    return 1;
  }
  if (M->kind == DSMC_MODEL_SV) {
    *out = -0.5 * (kLog2Pi + log(M->m->sv_sigma2)) - M->logabsy[c];
    return 1;
  }
  if (!lg1(M) || M->T < 1) return 0;
  for (int cc = 1; cc <= M->T; ++cc) {
    if (!has_obs(M, cc) || F1(cc) == 0.0) return 0;
  }
  double y = M->m->y[c], h = H1(c), r2 = R1(c);
  double m = M->m->prop_mean[c], v = M->m->prop_cov[c];
  double alpha = 1.0 / (2.0 * v) - h * h / (2.0 * r2);
  double beta = h * y / r2 - m / v;
  double gamma = -y * y / (2.0 * r2) + m * m / (2.0 * v) + 0.5 * log(v / r2);
  double s;
  if (alpha < 0.0) s = gamma - beta * beta / (4.0 * alpha);
  else if (alpha == 0.0 && beta == 0.0) s = gamma;
  else return 0;
  /* the model exposes a bound only if every cut has a finite one */
  for (int cc = 1; cc <= M->T; ++cc) {
    double yy = M->m->y[cc], hh = H1(cc), rr = R1(cc);
    double mm = M->m->prop_mean[cc], vv = M->m->prop_cov[cc];
    double al = 1.0 / (2.0 * vv) - hh * hh / (2.0 * rr);
    double be = hh * yy / rr - mm / vv;
    if (!(al < 0.0) && !(al == 0.0 && be == 0.0)) return 0;
  }
  *out = -0.5 * (kLog2Pi + log(Q1(c))) + s;
  return 1;
}

/* ------------------------------------------------------- combine source */
typedef struct {
  const model_t* M;
  int c;
  size_t n;
  const double *xl, *xr;     /* gathered boundary slabs (n*d) */
  const double *lw_l, *lw_r; /* NULL when that side is uniform */
  double* base;              /* column base (stitch_row_factory) */
  double* wcol;              /* d > 1: whitened columns, one slab per coordinate */
  int d;
} comb_ctx;

/* stitch_row_factory per model: column base bound once per combine. */
static void comb_prepare(comb_ctx* cc) {
  const model_t* M = cc->M;
  int c = cc->c;
  size_t n = cc->n;
  cc->base = malloc(sizeof(double) * n);
  if (COX(M)) { /* models.cpp:182-187 */
    for (size_t j = 0; j < n; ++j)
      cc->base[j] = cox_log_poisson(M, c, cc->xr[j]) -
                    log_normal_pdf(cc->xr[j], M->stat_mean, M->stat_var) + M->trans_norm;
  } else if (CRW(M)) { /* models.cpp:313-315 */
    for (size_t j = 0; j < n; ++j)
      cc->base[j] = in_box(cc->xr[j]) ? M->trans_norm - kLogHalf : NEG_INF;
  } else if (THETA(M)) { /* models.cpp:450-458 */
    double var = M->m->prop_cov[c];
    gaussian_row(cc->xr, n, M->m->y[c], -1.0 / (2.0 * M->r2), NULL, cc->base);
    gaussian_row(cc->xr, n, M->m->prop_mean[c], 1.0 / (2.0 * var), cc->base, cc->base);
    double sh = M->obs_norm + 0.5 * (kLog2Pi + log(var)) + M->trans_norm;
    for (size_t j = 0; j < n; ++j) cc->base[j] += sh;
  } else if (M->kind == DSMC_MODEL_SV) {
    double b = -0.5 * (kLog2Pi + log(M->m->sv_sigma2)) - M->logabsy[c];
    for (size_t j = 0; j < n; ++j) cc->base[j] = b;
  } else if (lg1(M)) { /* models.cpp:611-627 */
    double qvar = Q1(c), var = M->m->prop_cov[c];
    double trans_norm = -0.5 * (kLog2Pi + log(qvar));
    double shift = trans_norm + 0.5 * (kLog2Pi + log(var));
    if (has_obs(M, c)) {
      double h = H1(c), r = R1(c);
      gaussian_row(cc->xr, n, M->m->y[c] / h, -h * h / (2.0 * r), NULL, cc->base);
      shift += -0.5 * (kLog2Pi + log(r));
    } else {
      for (size_t j = 0; j < n; ++j) cc->base[j] = 0.0;
    }
    gaussian_row(cc->xr, n, M->m->prop_mean[c], 1.0 / (2.0 * var), cc->base,
                 cc->base);
    for (size_t j = 0; j < n; ++j) cc->base[j] += shift;
  } else {
    const double* pm = M->m->prop_mean + (size_t)c * M->d;
    const gauss_t* tr = &M->trans[c];
    int d = M->d;
    cc->wcol = malloc(sizeof(double) * n * d);
    for (size_t j = 0; j < n; ++j) {
      const double* x = cc->xr + j * d;
      cc->base[j] = tr->norm + lg_log_h(M, c, x) - gauss_logpdf(&M->prop[c], x, pm);
      for (int k = 0; k < d; ++k) {
        double z = 0.0;
        for (int l = 0; l <= k; ++l) z += tr->W[k * d + l] * x[l];
        cc->wcol[(size_t)k * n + j] = z;
      }
    }
  }
}

/* make_pair_source fill_row (smoother.cpp:153-161) */
static int comb_fill(const pair_src* s, size_t i, double* out) {
  const comb_ctx* cc = s->ctx;
  const model_t* M = cc->M;
  size_t n = cc->n;
  int c = cc->c;
  if (COX(M)) { /* models.cpp:188-191 */
    gaussian_row(cc->xr, n, M->icept + M->slope * cc->xl[i], -1.0 / (2.0 * M->var), cc->base,
                 out);
  } else if (CRW(M)) { /* models.cpp:316-319 */
    gaussian_row(cc->xr, n, cc->xl[i], -1.0 / (2.0 * M->var), cc->base, out);
  } else if (THETA(M)) { /* models.cpp:459-462 */
    gaussian_row(cc->xr, n, theta_drift(M, cc->xl[i]), -1.0 / (2.0 * M->var), cc->base, out);
  } else if (M->kind == DSMC_MODEL_SV) {
    double mu = M->m->sv_mu;
    double mean = mu + M->m->sv_phi * (cc->xl[i] - mu);
    gaussian_row(cc->xr, n, mean, -1.0 / (2.0 * M->m->sv_sigma2), cc->base, out);
  } else if (lg1(M)) {
    gaussian_row(cc->xr, n, F1(c) * cc->xl[i] + B1(c), -1.0 / (2.0 * Q1(c)),
                 cc->base, out);
  } else {
    /* d chained gaussian_row passes over the whitened columns
       (oracle/ref_models.cpp lgssm_nd) */
    double mu[4];
    int d = M->d;
    lg_mean(M, c, cc->xl + i * d, mu);
    const gauss_t* tr = &M->trans[c];
    const double* src = cc->base;
    for (int k = 0; k < d; ++k) {
      double v = 0.0;
      for (int l = 0; l <= k; ++l) v += tr->W[k * d + l] * mu[l];
      gaussian_row(cc->wcol + (size_t)k * n, n, v, -0.5, src, out);
      src = out;
    }
  }
  double sl = cc->lw_l ? cc->lw_l[i] : 0.0;
  if (cc->lw_r) {
    for (size_t j = 0; j < n; ++j) out[j] = (out[j] + sl) + cc->lw_r[j];
  } else if (sl != 0.0) {
    for (size_t j = 0; j < n; ++j) out[j] += sl;
  }
  return 0;
}
/* make_pair_source log_weight_at (smoother.cpp:163-169) */
static int comb_entry(const pair_src* s, size_t i, size_t j, double* out) {
  const comb_ctx* cc = s->ctx;
  int d = cc->d;
  double v;
  int rc = stitch_weight(cc->M, cc->c, cc->xl + i * d, cc->xr + j * d, &v);
  if (rc) return rc;
  if (cc->lw_l) v += cc->lw_l[i];
  if (cc->lw_r) v += cc->lw_r[j];
  *out = v;
  return 0;
}

/* ---------------------------------------------------------------- leaves */
typedef struct {
  double* x;  /* n*d */
  double* lw; /* n, normalized */
  double lnc;
  int uniform;
} leaf_t;

/* make_leaf (smoother.cpp:98-130) / conditional_leaf (conditional.cpp:52-87)
 * with optional injected raw states / log-weights. */
static int make_leaf(const model_t* M, int t, size_t n, uint64_t seed,
                     const double* star, uint32_t sweep,
                     const double* inj_x, const double* inj_lw, leaf_t* L) {
  int d = M->d;
  L->x = malloc(sizeof(double) * n * d);
  L->lw = malloc(sizeof(double) * n);
  if (inj_x) {
    memcpy(L->x, inj_x, sizeof(double) * n * d);
    if (star) memcpy(L->x, star, sizeof(double) * d);
  } else if (star) {
    memcpy(L->x, star, sizeof(double) * d);
    stream_t s;
    st_init(&s, seed, 0, (uint64_t)(uint32_t)t | ((uint64_t)sweep << 32),
            DSMC_ROLE_LEAF_PROPOSAL, 0);
    cb_proposal_sampler(M, t, n - 1, &s, L->x + d);
  } else {
    stream_t s;
    st_init(&s, seed, 0, (uint64_t)t, DSMC_ROLE_LEAF_PROPOSAL, 0);
    cb_proposal_sampler(M, t, n, &s, L->x);
  }
  if (inj_lw && !star) {
    memcpy(L->lw, inj_lw, sizeof(double) * n);
  } else {
    for (size_t i = 0; i < n; ++i) {
      int rc = leaf_weight(M, t, L->x + i * d, &L->lw[i]);
      if (rc) return rc;
    }
  }
  if (star && L->lw[0] == NEG_INF)
    return fail(DSMC_E_INVALID_ARGUMENT,
                "conditional_leaf: the reference path has zero weight at time %d", t);
  double lse = or_log_sum_exp(L->lw, n);
  if (isnan(lse)) return DSMC_E_DOMAIN;
  if (lse == NEG_INF)
    return fail(DSMC_E_RUNTIME, "leaf %d: every proposal draw has zero weight", t);
  double lo = L->lw[0], hi = L->lw[0];
  for (size_t p = 1; p < n; ++p) {
    if (L->lw[p] < lo) lo = L->lw[p];
    if (L->lw[p] > hi) hi = L->lw[p];
  }
  for (size_t p = 0; p < n; ++p) L->lw[p] += -lse;
  L->uniform = lo == hi;
  L->lnc = lse - log((double)n);
  return 0;
}

/* ------------------------------------------------- tree with composition */
typedef struct {
  int a, b;
  uint32_t *first, *last; /* into leaf a / leaf b particles */
  double lnc;
  int has_lnc, biased;
  uint64_t evals;
} block_t;

typedef struct {
  uint32_t *l, *r; /* per combine, n each */
} comb_rec;

static uint32_t* iota_u32(size_t n) {
  uint32_t* v = malloc(sizeof(uint32_t) * n);
  for (size_t i = 0; i < n; ++i) v[i] = (uint32_t)i;
  return v;
}

/* Shared driver for smoothing and conditional sweeps. */
static int run_tree(const model_t* M, size_t n, int resampler, size_t mh_steps,
                    uint64_t seed, int conditional, uint32_t sweep,
                    const double* star, const double* inj_x,
                    const double* inj_lw, leaf_t* leaves, comb_rec* combs,
                    double* comb_lmw, block_t* root_out, int* levels_out) {
  int T = M->T, K = T + 1, d = M->d;
  int rc = 0;
  for (int t = 0; t < K && !rc; ++t)
    rc = make_leaf(M, t, n, seed, star ? star + (size_t)t * d : NULL, sweep,
                   inj_x ? inj_x + (size_t)t * n * d : NULL,
                   inj_lw ? inj_lw + (size_t)t * n : NULL, &leaves[t]);
  if (rc) return rc;
  block_t* cur = malloc(sizeof(block_t) * K);
  for (int t = 0; t < K; ++t) {
    cur[t].a = cur[t].b = t;
    cur[t].first = iota_u32(n);
    cur[t].last = iota_u32(n);
    cur[t].lnc = leaves[t].lnc;
    cur[t].has_lnc = 1;
    cur[t].biased = 0;
    cur[t].evals = 0;
  }
  int nb = K, level = 0, cursor = 0;
  double* xl = malloc(sizeof(double) * n * d);
  double* xr = malloc(sizeof(double) * n * d);
  size_t n_out = conditional ? n - 1 : n;
  uint32_t* pl = malloc(sizeof(uint32_t) * n);
  uint32_t* pr = malloc(sizeof(uint32_t) * n);
  while (nb > 1 && !rc) {
    ++level;
    int np = nb / 2;
    for (int k = 0; k < np && !rc; ++k) {
      block_t *L = &cur[2 * k], *R = &cur[2 * k + 1];
      int c = R->a;
      const leaf_t *LL = &leaves[c - 1], *RL = &leaves[c];
      for (size_t i = 0; i < n; ++i) {
        memcpy(xl + i * d, LL->x + (size_t)L->last[i] * d, sizeof(double) * d);
        memcpy(xr + i * d, RL->x + (size_t)R->first[i] * d, sizeof(double) * d);
      }
      /* a side's weights enter only while it is a non-uniform leaf */
      int l_leaf = L->a == L->b, r_leaf = R->a == R->b;
      comb_ctx cc = {M, c, n, xl, xr,
                     (l_leaf && !LL->uniform) ? LL->lw : NULL,
                     (r_leaf && !RL->uniform) ? RL->lw : NULL, NULL, NULL, d};
      comb_prepare(&cc);
      pair_src src = {n, &cc, comb_fill, comb_entry, 0, 0.0};
      double bnd;
      if (stitch_bound(M, c, &bnd)) {
        double mx;
        if (cc.lw_l) { reduce_max(cc.lw_l, n, &mx); bnd += mx; }
        if (cc.lw_r) { reduce_max(cc.lw_r, n, &mx); bnd += mx; }
        src.has_bound = 1;
        src.bound = bnd;
      }
      double logn = log((double)n);
      double shift = ((l_leaf && LL->uniform) || !l_leaf ? -logn : 0.0) +
                     ((r_leaf && RL->uniform) || !r_leaf ? -logn : 0.0);
      uint64_t node = conditional ? ((uint64_t)(uint32_t)k | ((uint64_t)sweep << 32))
                                  : (uint64_t)k;
      if (conditional) {
        if (resampler != DSMC_MULTINOMIAL && resampler != DSMC_REJECTION_LAZY) {
          rc = fail(DSMC_E_INVALID_ARGUMENT,
                    "conditional sweeps need exchangeable unbiased slot draws: "
                    "use the multinomial or rejection-lazy resampler");
          free(cc.base);
          free(cc.wcol);
          break;
        }
        double w00;
        rc = comb_entry(&src, 0, 0, &w00);
        if (!rc && !isfinite(w00))
          rc = fail(DSMC_E_INVALID_ARGUMENT,
                    "conditional_combine: the reference pair has zero stitch "
                    "weight at cut %d", c);
        if (rc) { free(cc.base); free(cc.wcol); break; }
      }
      pair_sample ps = {pl + (conditional ? 1 : 0), pr + (conditional ? 1 : 0), 0, 0, 0, 0};
      rc = resample(resampler, &src, n_out, mh_steps, seed, (uint32_t)level,
                    node, &ps);
      free(cc.base);
      free(cc.wcol);
      if (rc) {
        if (rc == DSMC_E_RUNTIME) {
          char msg[512];
          snprintf(msg, sizeof msg, "%s", g_err);
          fail(rc, "%scombine at cut %d (times %d..%d): %s",
               conditional ? "conditional " : "", c, L->a, R->b, msg);
        }
        break;
      }
      if (conditional) {
        pl[0] = 0;
        pr[0] = 0;
      }
      memcpy(combs[cursor + k].l, pl, sizeof(uint32_t) * n);
      memcpy(combs[cursor + k].r, pr, sizeof(uint32_t) * n);
      comb_lmw[cursor + k] = ps.has_lmw ? ps.lmw : NAN;
      /* combine_blocks (smoother.cpp:203-223): ancestor maps, not paths */
      block_t nbk;
      nbk.a = L->a;
      nbk.b = R->b;
      nbk.first = malloc(sizeof(uint32_t) * n);
      nbk.last = malloc(sizeof(uint32_t) * n);
      for (size_t q = 0; q < n; ++q) {
        nbk.first[q] = L->first[pl[q]];
        nbk.last[q] = R->last[pr[q]];
      }
      nbk.biased = L->biased || R->biased || ps.biased;
      nbk.evals = L->evals + R->evals + ps.evals + (conditional ? 1 : 0);
      nbk.has_lnc = L->has_lnc && R->has_lnc && ps.has_lmw;
      nbk.lnc = nbk.has_lnc ? L->lnc + R->lnc + ps.lmw + shift : NAN;
      free(L->first);
      free(L->last);
      free(R->first);
      free(R->last);
      cur[k] = nbk;
    }
    if (rc) break;
    if (nb % 2) cur[np] = cur[nb - 1];
    cursor += np;
    nb = (nb + 1) / 2;
  }
  free(xl);
  free(xr);
  free(pl);
  free(pr);
  if (!rc) {
    *root_out = cur[0];
    *levels_out = level;
  } else {
    for (int i = 0; i < nb; ++i) {
      /* best effort cleanup of live blocks */
    }
  }
  free(cur);
  return rc;
}

/* Top-down composition: sigma_t[q] = leaf particle of root slot q at t. */
static void compose_down(int K, size_t n, const comb_rec* combs,
                         uint32_t* sigma /* K*n */) {
  /* level block counts */
  int nlev = 0;
  int nbs[64];
  nbs[0] = K;
  while (nbs[nlev] > 1) {
    nbs[nlev + 1] = (nbs[nlev] + 1) / 2;
    ++nlev;
  }
  int cursor[64];
  cursor[1] = 0;
  for (int l = 1; l < nlev; ++l) cursor[l + 1] = cursor[l] + nbs[l - 1] / 2;
  uint32_t* maps = malloc(sizeof(uint32_t) * n * (size_t)K);
  uint32_t* next = malloc(sizeof(uint32_t) * n * (size_t)K);
  for (size_t q = 0; q < n; ++q) maps[q] = (uint32_t)q;
  for (int l = nlev; l >= 1; --l) {
    int nparent = nbs[l], nchild = nbs[l - 1];
    for (int k = 0; k < nparent; ++k) {
      const uint32_t* M = maps + (size_t)k * n;
      if (2 * k + 1 < nchild) {
        const comb_rec* cr = &combs[cursor[l] + k];
        for (size_t q = 0; q < n; ++q) {
          next[(size_t)(2 * k) * n + q] = cr->l[M[q]];
          next[(size_t)(2 * k + 1) * n + q] = cr->r[M[q]];
        }
      } else {
        memcpy(next + (size_t)(2 * k) * n, M, sizeof(uint32_t) * n);
      }
    }
    uint32_t* tmp = maps;
    maps = next;
    next = tmp;
  }
  memcpy(sigma, maps, sizeof(uint32_t) * n * (size_t)K);
  free(maps);
  free(next);
}

int or_smooth(const dsmc_model_desc* model, const dsmc_smooth_opts* opts,
              dsmc_smooth_out* out) {
  model_t M;
  int rc = model_init(&M, model);
  if (rc) return rc;
  size_t n = opts->n_particles;
  if (n == 0) { model_free(&M); return fail(DSMC_E_INVALID_ARGUMENT, "make_leaf: n must be >= 1"); }
  int K = M.T + 1, d = M.d, T = M.T;
  leaf_t* leaves = calloc(K, sizeof(leaf_t));
  comb_rec* combs = calloc(T > 0 ? T : 1, sizeof(comb_rec));
  for (int c = 0; c < T; ++c) {
    combs[c].l = malloc(sizeof(uint32_t) * n);
    combs[c].r = malloc(sizeof(uint32_t) * n);
  }
  double* lmw = calloc(T > 0 ? T : 1, sizeof(double));
  block_t root;
  int levels = 0;
  rc = run_tree(&M, n, opts->resampler, opts->mh_steps, opts->seed, 0, 0, NULL,
                opts->inject_states, opts->inject_logw, leaves, combs, lmw,
                &root, &levels);
  if (!rc) {
    uint32_t* sigma = malloc(sizeof(uint32_t) * n * K);
    compose_down(K, n, combs, sigma);
    if (out->paths)
      for (int t = 0; t < K; ++t)
        for (size_t q = 0; q < n; ++q)
          memcpy(out->paths + ((size_t)t * n + q) * d,
                 leaves[t].x + (size_t)sigma[(size_t)t * n + q] * d,
                 sizeof(double) * d);
    if (out->mean || out->cov) {
      for (int t = 0; t < K; ++t) {
        double mu[4] = {0};
        for (size_t q = 0; q < n; ++q)
          for (int k = 0; k < d; ++k)
            mu[k] += leaves[t].x[(size_t)sigma[(size_t)t * n + q] * d + k];
        for (int k = 0; k < d; ++k) mu[k] /= (double)n;
        if (out->mean) memcpy(out->mean + (size_t)t * d, mu, sizeof(double) * d);
        if (out->cov) {
          double* C = out->cov + (size_t)t * d * d;
          memset(C, 0, sizeof(double) * d * d);
          for (size_t q = 0; q < n; ++q) {
            const double* x = leaves[t].x + (size_t)sigma[(size_t)t * n + q] * d;
            for (int a = 0; a < d; ++a)
              for (int b = 0; b < d; ++b) C[a * d + b] += (x[a] - mu[a]) * (x[b] - mu[b]);
          }
          for (int a = 0; a < d * d; ++a) C[a] /= (double)n;
        }
      }
    }
    if (out->pair_left)
      for (int c = 0; c < T; ++c) {
        memcpy(out->pair_left + (size_t)c * n, combs[c].l, sizeof(uint32_t) * n);
        memcpy(out->pair_right + (size_t)c * n, combs[c].r, sizeof(uint32_t) * n);
      }
    if (out->log_mean_weight) memcpy(out->log_mean_weight, lmw, sizeof(double) * T);
    if (out->leaf_states)
      for (int t = 0; t < K; ++t)
        memcpy(out->leaf_states + (size_t)t * n * d, leaves[t].x, sizeof(double) * n * d);
    out->log_norm_const = root.lnc;
    out->has_log_norm_const = root.has_lnc;
    out->levels = levels;
    out->weight_evals = root.evals;
    out->biased = root.biased;
    out->wall_time_ms = 0.0;
    free(sigma);
    free(root.first);
    free(root.last);
  }
  for (int t = 0; t < K; ++t) {
    free(leaves[t].x);
    free(leaves[t].lw);
  }
  for (int c = 0; c < T; ++c) {
    free(combs[c].l);
    free(combs[c].r);
  }
  free(leaves);
  free(combs);
  free(lmw);
  model_free(&M);
  return rc;
}

int or_conditional(const dsmc_model_desc* model, const double* ref,
                   size_t n, int resampler, uint64_t seed, uint32_t sweep,
                   const double* inject_states, const double* inject_logw,
                   double* out_path, double* log_norm_const, int* has_lnc,
                   uint64_t* weight_evals) {
  (void)inject_logw;
  if (resampler != DSMC_MULTINOMIAL && resampler != DSMC_REJECTION_LAZY)
    return fail(DSMC_E_INVALID_ARGUMENT,
                "conditional sweeps need exchangeable unbiased slot draws: use "
                "the multinomial or rejection-lazy resampler");
  if (n < 2) return fail(DSMC_E_INVALID_ARGUMENT, "conditional_leaf: need n >= 2 slots");
  model_t M;
  int rc = model_init(&M, model);
  if (rc) return rc;
  int K = M.T + 1, d = M.d, T = M.T;
  leaf_t* leaves = calloc(K, sizeof(leaf_t));
  comb_rec* combs = calloc(T > 0 ? T : 1, sizeof(comb_rec));
  for (int c = 0; c < T; ++c) {
    combs[c].l = malloc(sizeof(uint32_t) * n);
    combs[c].r = malloc(sizeof(uint32_t) * n);
  }
  double* lmw = calloc(T > 0 ? T : 1, sizeof(double));
  block_t root;
  int levels = 0;
  rc = run_tree(&M, n, resampler, 0, seed, 1, sweep, ref, inject_states, NULL,
                leaves, combs, lmw, &root, &levels);
  if (!rc) {
    /* star selection (conditional.cpp:195-199, 35-48) */
    stream_t s;
    st_init(&s, seed, (uint32_t)(levels + 1), sweep, DSMC_ROLE_STAR_SELECT, 0);
    size_t chosen;
    if (T == 0 && !leaves[0].uniform) {
      double u = st_uniform(&s), cum = 0.0;
      size_t last_live = 0;
      chosen = n;
      for (size_t p = 0; p < n; ++p) {
        double w = or_exp_w(leaves[0].lw[p]);
        if (w > 0.0) last_live = p;
        cum += w;
        if (u < cum) { chosen = p; break; }
      }
      if (chosen == n) chosen = last_live;
    } else {
      chosen = (size_t)st_index(&s, n);
    }
    uint32_t* sigma = malloc(sizeof(uint32_t) * n * K);
    compose_down(K, n, combs, sigma);
    for (int t = 0; t < K; ++t)
      memcpy(out_path + (size_t)t * d,
             leaves[t].x + (size_t)sigma[(size_t)t * n + chosen] * d,
             sizeof(double) * d);
    *log_norm_const = root.lnc;
    *has_lnc = root.has_lnc;
    *weight_evals = root.evals;
    free(sigma);
    free(root.first);
    free(root.last);
  }
  for (int t = 0; t < K; ++t) {
    free(leaves[t].x);
    free(leaves[t].lw);
  }
  for (int c = 0; c < T; ++c) {
    free(combs[c].l);
    free(combs[c].r);
  }
  free(leaves);
  free(combs);
  free(lmw);
  model_free(&M);
  return rc;
}

/* ------------------------------------------------------------ SV Gibbs */
/* gamma_draw (pgibbs.cpp:80-102) */
static double gamma_draw_s(double shape, double rate, stream_t* s) {
  double boost = 1.0;
  if (shape < 1.0) {
    boost = pow(st_uniform_pos(s), 1.0 / shape);
    shape += 1.0;
  }
  double d = shape - 1.0 / 3.0;
  double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = st_normal(s);
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    double u = st_uniform_pos(s);
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return boost * d * v / rate;
  }
}

double or_gamma_draw(double shape, double rate, uint64_t seed, uint32_t level,
                     uint64_t node, int role) {
  stream_t s;
  st_init(&s, seed, level, node, role, 0);
  return gamma_draw_s(shape, rate, &s);
}

/* Log-likelihood of the path under AR(1) (mu, phi, s2), stationary start. */
static double sv_path_loglik(const double* x, int T, double mu, double phi,
                             double s2) {
  double v0 = s2 / (1.0 - phi * phi);
  double ll = log_normal_pdf(x[0], mu, v0);
  for (int t = 1; t <= T; ++t) ll += log_normal_pdf(x[t], mu + phi * (x[t - 1] - mu), s2);
  return ll;
}

/* SV ParamKernel: sigma2 | rest (inverse gamma), mu | rest (normal), RWM on
 * phi (flat prior on (-1, 1)). Draw order is part of the contract. */
int or_sv_param_update(const double* x, int T, const dsmc_sv_prior* pr,
                       uint64_t seed, uint32_t sweep, double* theta,
                       int* accepted_phi) {
  stream_t s;
  st_init(&s, seed, 0, sweep, DSMC_ROLE_GIBBS_PARAM, 0);
  double mu = theta[0], phi = theta[1], s2 = theta[2];
  /* sigma2 */
  double ss = (1.0 - phi * phi) * (x[0] - mu) * (x[0] - mu);
  for (int t = 1; t <= T; ++t) {
    double e = x[t] - mu - phi * (x[t - 1] - mu);
    ss += e * e;
  }
  double prec = gamma_draw_s(pr->s2_shape + 0.5 * (double)(T + 1),
                             pr->s2_rate + 0.5 * ss, &s);
  s2 = 1.0 / prec;
  /* mu */
  double p = 1.0 / pr->mu_var + (1.0 - phi * phi) / s2 +
             (double)T * (1.0 - phi) * (1.0 - phi) / s2;
  double acc = 0.0;
  for (int t = 1; t <= T; ++t) acc += x[t] - phi * x[t - 1];
  double h = pr->mu_mean / pr->mu_var + (1.0 - phi * phi) * x[0] / s2 +
             (1.0 - phi) * acc / s2;
  mu = h / p + sqrt(1.0 / p) * st_normal(&s);
  /* phi */
  double prop = phi + pr->phi_step * st_normal(&s);
  double lu = log(st_uniform_pos(&s));
  int acc_phi = 0;
  if (fabs(prop) < 1.0) {
    double dl = sv_path_loglik(x, T, mu, prop, s2) - sv_path_loglik(x, T, mu, phi, s2);
    if (lu < dl) {
      phi = prop;
      acc_phi = 1;
    }
  }
  theta[0] = mu;
  theta[1] = phi;
  theta[2] = s2;
  if (accepted_phi) *accepted_phi = acc_phi;
  return 0;
}

/* ------------------------------------------------------------------------
 * Kalman filter + RTS smoother of a DSMC_MODEL_LGSSM descriptor (host FP64),
 * restating kalman_smooth (kalman.cpp:78-138): predicted covariance
 * symmetrised, Joseph-form update, RTS gain by solving against the predicted
 * covariance, symmetrisation after every step, the jitter-escalating
 * Cholesky of robust_llt (kalman.cpp:15-26) and log_gaussian (:28-36). Used
 * by bench.py's reference arm to build the RTS-marginal proposals without
 * loading the product library. */
#define KMAXD 8
static void km_sym(double* P, int d) {
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < i; ++j) {
      double v = (P[i * d + j] + P[j * d + i]) * 0.5;
      P[i * d + j] = P[j * d + i] = v;
    }
}
/* robust_llt: symmetrise, then up to 4 Cholesky attempts with jitter
   scale * 10^(attempt - 12), scale = max(trace / n, 1e-300) */
static int km_llt(const double* A, int d, double* L) {
  double P[KMAXD * KMAXD];
  memcpy(P, A, sizeof(double) * d * d);
  km_sym(P, d);
  double tr = 0.0;
  for (int i = 0; i < d; ++i) tr += P[i * d + i];
  double scale = tr / d > 1e-300 ? tr / d : 1e-300;
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (chol(P, d, L)) return 1;
    for (int i = 0; i < d; ++i) P[i * d + i] += scale * pow(10.0, attempt - 12);
  }
  return 0;
}
/* X := A^{-1} B for A = L L' (B: d x m, row-major) */
static void km_solve(const double* L, int d, const double* B, int m, double* X) {
  for (int c = 0; c < m; ++c) {
    double z[KMAXD];
    for (int i = 0; i < d; ++i) {
      double s = B[i * m + c];
      for (int k = 0; k < i; ++k) s -= L[i * d + k] * z[k];
      z[i] = s / L[i * d + i];
    }
    for (int i = d - 1; i >= 0; --i) {
      double s = z[i];
      for (int k = i + 1; k < d; ++k) s -= L[k * d + i] * X[k * m + c];
      X[i * m + c] = s / L[i * d + i];
    }
  }
}
/* C (n x m) = A (n x k) * B (k x m), optional transposes of the stored arrays */
static void km_mul(const double* A, int ta, const double* B, int tb, int n, int k, int m,
                   double* C) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int q = 0; q < k; ++q)
        s += (ta ? A[q * n + i] : A[i * k + q]) * (tb ? B[j * k + q] : B[q * m + j]);
      C[i * m + j] = s;
    }
}

int or_kalman_smooth(const dsmc_model_desc* m, double* sm, double* sc, double* loglik) {
  if (!m || m->kind != DSMC_MODEL_LGSSM)
    return fail(DSMC_E_INVALID_ARGUMENT, "kalman_smooth: LGSSM descriptor required");
  const int d = m->state_dim, dy = m->obs_dim, T = m->horizon, K = T + 1;
  if (d < 1 || d > KMAXD || dy < 1 || dy > KMAXD)
    return fail(DSMC_E_INVALID_ARGUMENT, "kalman_smooth: dims must be 1..8");
  const size_t dd = (size_t)d * d;
  double* pm = malloc(sizeof(double) * K * d);
  double* pc = malloc(sizeof(double) * K * dd);
  double* fm = malloc(sizeof(double) * K * d);
  double* fc = malloc(sizeof(double) * K * dd);
  double ll = 0.0;
  int rc = 0;
  for (int t = 0; t <= T && !rc; ++t) {
    double* Pp = pc + t * dd;
    if (t == 0) {
      memcpy(pm, m->m0, sizeof(double) * d);
      memcpy(Pp, m->P0, sizeof(double) * dd);
    } else {
      const double* F = at(m->F, m->F_stride, t);
      const double* b = at(m->b, m->b_stride, t);
      const double* Q = at(m->Q, m->Q_stride, t);
      double tmp[KMAXD * KMAXD];
      km_mul(F, 0, fm + (t - 1) * d, 0, d, d, 1, pm + t * d);
      for (int i = 0; i < d; ++i) pm[t * d + i] += b[i];
      km_mul(F, 0, fc + (t - 1) * dd, 0, d, d, d, tmp);
      km_mul(tmp, 0, F, 1, d, d, d, Pp);
      for (size_t i = 0; i < dd; ++i) Pp[i] += Q[i];
      km_sym(Pp, d);
    }
    if (m->has_obs ? m->has_obs[t] != 0 : 1) {
      const double* H = at(m->H, m->H_stride, t);
      const double* R = at(m->R, m->R_stride, t);
      const double* y = m->y + (size_t)t * dy;
      double resid[KMAXD], HP[KMAXD * KMAXD], S[KMAXD * KMAXD], L[KMAXD * KMAXD];
      double Kt[KMAXD * KMAXD], Kg[KMAXD * KMAXD], A[KMAXD * KMAXD], t1[KMAXD * KMAXD];
      double t2[KMAXD * KMAXD];
      km_mul(H, 0, pm + t * d, 0, dy, d, 1, resid);
      for (int i = 0; i < dy; ++i) resid[i] = y[i] - resid[i];
      km_mul(H, 0, Pp, 0, dy, d, d, HP);
      km_mul(HP, 0, H, 1, dy, d, dy, S);
      for (int i = 0; i < dy * dy; ++i) S[i] += R[i];
      if (!km_llt(S, dy, L)) {
        rc = fail(DSMC_E_RUNTIME, "kalman update: covariance is not positive definite");
        break;
      }
      double ld = 0.0, z2 = 0.0, z[KMAXD];
      for (int i = 0; i < dy; ++i) ld += 2.0 * log(L[i * dy + i]);
      for (int i = 0; i < dy; ++i) {
        double s = resid[i];
        for (int k = 0; k < i; ++k) s -= L[i * dy + k] * z[k];
        z[i] = s / L[i * dy + i];
        z2 += z[i] * z[i];
      }
      ll += -0.5 * (dy * log(2.0 * M_PI) + ld + z2);
      km_solve(L, dy, HP, d, Kt); /* (dy x d) = S^{-1} H P */
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < dy; ++j) Kg[i * dy + j] = Kt[j * d + i];
      km_mul(Kg, 0, resid, 0, d, dy, 1, fm + t * d);
      for (int i = 0; i < d; ++i) fm[t * d + i] += pm[t * d + i];
      km_mul(Kg, 0, H, 0, d, dy, d, A);
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) A[i * d + j] = (i == j) - A[i * d + j];
      km_mul(A, 0, Pp, 0, d, d, d, t1);
      km_mul(t1, 0, A, 1, d, d, d, fc + t * dd);
      km_mul(Kg, 0, R, 0, d, dy, dy, t1);
      km_mul(t1, 0, Kg, 1, d, dy, d, t2);
      for (size_t i = 0; i < dd; ++i) fc[t * dd + i] += t2[i];
      km_sym(fc + t * dd, d);
    } else {
      memcpy(fm + t * d, pm + t * d, sizeof(double) * d);
      memcpy(fc + t * dd, Pp, sizeof(double) * dd);
    }
  }
  if (!rc) {
    memcpy(sm + (size_t)T * d, fm + (size_t)T * d, sizeof(double) * d);
    memcpy(sc + (size_t)T * dd, fc + (size_t)T * dd, sizeof(double) * dd);
    for (int t = T - 1; t >= 0; --t) {
      double L[KMAXD * KMAXD], FP[KMAXD * KMAXD], Gt[KMAXD * KMAXD], G[KMAXD * KMAXD];
      double e[KMAXD], D[KMAXD * KMAXD], t1[KMAXD * KMAXD];
      if (!km_llt(pc + (t + 1) * dd, d, L)) {
        rc = fail(DSMC_E_RUNTIME, "rts gain: covariance is not positive definite");
        break;
      }
      const double* F = at(m->F, m->F_stride, t + 1);
      km_mul(F, 0, fc + t * dd, 1, d, d, d, FP); /* F * filt_cov' */
      km_solve(L, d, FP, d, Gt);
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) G[i * d + j] = Gt[j * d + i];
      for (int i = 0; i < d; ++i) e[i] = sm[(t + 1) * d + i] - pm[(t + 1) * d + i];
      km_mul(G, 0, e, 0, d, d, 1, sm + t * d);
      for (int i = 0; i < d; ++i) sm[t * d + i] += fm[t * d + i];
      for (size_t i = 0; i < dd; ++i) D[i] = sc[(t + 1) * dd + i] - pc[(t + 1) * dd + i];
      km_mul(G, 0, D, 0, d, d, d, t1);
      km_mul(t1, 0, G, 1, d, d, d, sc + t * dd);
      for (size_t i = 0; i < dd; ++i) sc[t * dd + i] += fc[t * dd + i];
      km_sym(sc + t * dd, d);
    }
  }
  free(pm);
  free(pc);
  free(fm);
  free(fc);
  if (!rc && loglik) *loglik = ll;
  return rc;
}
