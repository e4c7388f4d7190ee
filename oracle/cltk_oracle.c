/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's Monte Carlo
 * pricing path (cltk, proj/src/pricing.cpp + the kernel evaluator of
 * proj/src/kernel.cpp).  Used by tests/ and by bench.py's cpu_baseline /
 * --impl reference legs as the checker; never by the product path.
 *
 * Parity pinned against the compiled reference (oracle/_ref/libcltkref.so)
 * and tests/golden/*.json: see tests/test_oracle.py.
 *
 * Must be compiled without FMA contraction (-ffp-contract=off), as the
 * reference is (x86-64 baseline, no -mfma).
 */
#define _GNU_SOURCE
#include "cltk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- Philox2x64-10, proj/src/pricing.cpp:73-98 ------------------------- */
#define PHILOX_M 0xD2B74407B1CE6E93ULL
#define PHILOX_W 0x9E3779B97F4A7C15ULL

uint64_t oracle_philox_bits(uint64_t seed, uint64_t path, uint64_t i) {
  uint64_t c0 = i, c1 = path, key = seed;
  for (int r = 0; r < 10; ++r) {
    unsigned __int128 prod = (unsigned __int128)PHILOX_M * c0;
    uint64_t lo = (uint64_t)prod, hi = (uint64_t)(prod >> 64);
    c0 = hi ^ key ^ c1;
    c1 = lo;
    key += PHILOX_W;
  }
  return c0 ^ c1;
}

/* proj/src/pricing.cpp:100-103 */
double oracle_uniform(uint64_t seed, uint64_t path, uint64_t i) {
  return ((double)(oracle_philox_bits(seed, path, i) >> 11) + 0.5) *
         0x1.0p-53;
}

/* proj/src/pricing.cpp:109 */
double oracle_normal_cdf(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

/* Acklam + one Halley step, proj/src/pricing.cpp:111-148 */
int oracle_inv_normal_cdf(double p, double* out) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};
  if (!(p > 0.0 && p < 1.0)) return 5;
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    double q = sqrt(-2.0 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - plow) {
    double q = p - 0.5;
    double r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) *
        q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    double q = sqrt(-2.0 * log(1.0 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  double e = oracle_normal_cdf(x) - p;
  double u = e * sqrt(2.0 * M_PI) * exp(x * x / 2.0);
  *out = x - u / (1.0 + x * u / 2.0);
  return 0;
}

/* proj/src/pricing.cpp:45-69 */
int oracle_cholesky(const double* m, int n, double* l) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (fabs(m[i * n + j] - m[j * n + i]) > 1e-12) return 5;
  memset(l, 0, sizeof(double) * (size_t)n * (size_t)n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = m[i * n + j];
      for (int k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      if (i == j) {
        if (s <= 0.0) return 5;
        l[i * n + i] = sqrt(s);
      } else {
        l[i * n + j] = s / l[j * n + j];
      }
    }
  return 0;
}

/* ---- kernel evaluator, proj/src/kernel.cpp:182-310 ---------------------- */
enum { V_INT = 0, V_REAL = 1, V_BOOL = 2 };
typedef struct {
  int tag;
  int64_t i;
  double r;
  int b;
} kval;

typedef struct {
  const oracle_kernel* k;
  const double* ext;
  const double* disc;
  uint64_t t_now;
  int err; /* 0, 3 (TypeError) or 5 (EvalError) */
  char* msg;
  size_t msg_len;
} keval;

static void fail(keval* s, int code, const char* m) {
  if (s->err) return;
  s->err = code;
  if (s->msg && s->msg_len) snprintf(s->msg, s->msg_len, "%s", m);
}

static double as_real(keval* s, kval v) {
  if (v.tag == V_REAL) return v.r;
  fail(s, 3, "kernel: expected a Real value");
  return 0.0;
}
static int as_bool(keval* s, kval v) {
  if (v.tag == V_BOOL) return v.b;
  fail(s, 3, "kernel: expected a Bool value");
  return 0;
}
static kval mk_real(double r) { kval v = {V_REAL, 0, r, 0}; return v; }
static kval mk_int(int64_t i) { kval v = {V_INT, i, 0.0, 0}; return v; }
static kval mk_bool(int b) { kval v = {V_BOOL, 0, 0.0, b}; return v; }

/* kApplyBin, proj/src/kernel.cpp:193-225 (C++ operand evaluation order kept:
 * Div checks the divisor first; And/Or short-circuit the second type check). */
static kval apply_bin(keval* s, int op, kval a, kval b) {
  int both_int = a.tag == V_INT && b.tag == V_INT;
  switch (op) {
    case OB_ADD:
      if (both_int) return mk_int((int64_t)((uint64_t)a.i + (uint64_t)b.i));
      { double x = as_real(s, a); if (s->err) return a;
        double y = as_real(s, b); return mk_real(x + y); }
    case OB_SUB:
      if (both_int) return mk_int((int64_t)((uint64_t)a.i - (uint64_t)b.i));
      { double x = as_real(s, a); if (s->err) return a;
        double y = as_real(s, b); return mk_real(x - y); }
    case OB_MULT:
      { double x = as_real(s, a); if (s->err) return a;
        double y = as_real(s, b); return mk_real(x * y); }
    case OB_DIV: {
      double d = as_real(s, b);
      if (s->err) return a;
      if (d == 0.0) { fail(s, 5, "kernel: division by zero"); return a; }
      double x = as_real(s, a);
      return mk_real(x / d);
    }
    case OB_LT:
      if (both_int) return mk_bool(a.i < b.i);
      { double x = as_real(s, a); if (s->err) return a;
        double y = as_real(s, b); return mk_bool(x < y); }
    case OB_LEQ:
      if (both_int) return mk_bool(a.i <= b.i);
      { double x = as_real(s, a); if (s->err) return a;
        double y = as_real(s, b); return mk_bool(x <= y); }
    case OB_EQ:
      if (both_int) return mk_bool(a.i == b.i);
      { double x = as_real(s, a); if (s->err) return a;
        double y = as_real(s, b); return mk_bool(x == y); }
    case OB_AND: {
      int x = as_bool(s, a); if (s->err) return a;
      if (!x) return mk_bool(0);
      return mk_bool(as_bool(s, b));
    }
    case OB_OR: {
      int x = as_bool(s, a); if (s->err) return a;
      if (x) return mk_bool(1);
      return mk_bool(as_bool(s, b));
    }
  }
  fail(s, 1, "unknown kernel operator");
  return a;
}

static kval eval_node(keval* s, int32_t idx, uint64_t off) {
  const oracle_node* n = &s->k->nodes[idx];
  kval z = mk_real(0.0);
  if (s->err) return z;
  switch (n->kind) {
    case OK_IF: {
      kval c = eval_node(s, n->a, off);
      if (s->err) return z;
      int cb = as_bool(s, c);
      if (s->err) return z;
      return eval_node(s, cb ? n->b : n->c, off);
    }
    case OK_FLOAT: return mk_real(n->real);
    case OK_NAT: return mk_int((int64_t)n->nat);
    case OK_BOOL: return mk_bool(n->boolean);
    case OK_NOW: return mk_int((int64_t)s->t_now);
    case OK_TIMEREF: {
      uint64_t r = n->row + off;
      if (r >= s->k->n_rows) { fail(s, 5, "kernel row index out of range"); return z; }
      return mk_int(s->k->rows[r]);
    }
    case OK_OBSREF: {
      uint64_t r = n->row + off;
      if (r >= s->k->n_rows || n->col >= s->k->n_cols) {
        char buf[128];
        snprintf(buf, sizeof buf, "kernel input shape mismatch at ext[%llu,%llu]",
                 (unsigned long long)r, (unsigned long long)n->col);
        fail(s, 5, buf);
        return z;
      }
      return mk_real(s->ext[r * s->k->n_cols + n->col]);
    }
    case OK_PAYREF: {
      uint64_t r = n->row + off;
      if (r >= s->k->n_rows) { fail(s, 5, "kernel disc index out of range"); return z; }
      double d = s->disc[r];
      if (n->pay_sign > 0) return mk_real(d);
      if (n->pay_sign < 0) return mk_real(-d);
      return mk_real(0.0);
    }
    case OK_UNOP: {
      kval v = eval_node(s, n->a, off);
      if (s->err) return z;
      if (n->op == OU_NEG) return mk_real(-as_real(s, v));
      return mk_bool(!as_bool(s, v));
    }
    case OK_BINOP: {
      kval a = eval_node(s, n->a, off);
      if (s->err) return z;
      kval b = eval_node(s, n->b, off);
      if (s->err) return z;
      return apply_bin(s, n->op, a, b);
    }
    case OK_LOOPIF: {
      uint64_t w = n->nat, cur = off;
      for (;; --w, ++cur) {
        kval c = eval_node(s, n->a, cur);
        if (s->err) return z;
        int cb = as_bool(s, c);
        if (s->err) return z;
        if (cb) return eval_node(s, n->b, cur);
        if (w == 0) return eval_node(s, n->c, cur);
      }
    }
  }
  fail(s, 1, "unknown kernel node");
  return z;
}

int oracle_eval_kernel(const oracle_kernel* k, const double* ext,
                       const double* disc, uint64_t t_now, double* out,
                       char* msg, size_t msg_len) {
  keval s = {k, ext, disc, t_now, 0, msg, msg_len};
  kval v = eval_node(&s, k->root, 0);
  if (s.err) return s.err;
  if (v.tag != V_REAL) {
    fail(&s, 5, "kernel did not evaluate to a real");
    return s.err;
  }
  *out = v.r;
  return 0;
}

/* ---- path simulation, proj/src/pricing.cpp:173-253 ---------------------- */
typedef struct {
  uint64_t n_days;
  int64_t* days;        /* sorted distinct row days */
  uint64_t* row_to_day; /* [n_rows] */
  double* disc;         /* [n_rows] */
} simplan;

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static int plan_init(simplan* p, const oracle_kernel* k, const oracle_model* m) {
  p->days = malloc(sizeof(int64_t) * (k->n_rows + 1));
  p->row_to_day = malloc(sizeof(uint64_t) * (k->n_rows + 1));
  p->disc = malloc(sizeof(double) * (k->n_rows + 1));
  memcpy(p->days, k->rows, sizeof(int64_t) * k->n_rows);
  qsort(p->days, k->n_rows, sizeof(int64_t), cmp_i64);
  uint64_t n = 0;
  for (uint64_t i = 0; i < k->n_rows; ++i)
    if (n == 0 || p->days[n - 1] != p->days[i]) p->days[n++] = p->days[i];
  p->n_days = n;
  if (n > 0 && p->days[0] < 0) return 5;
  for (uint64_t r = 0; r < k->n_rows; ++r) {
    uint64_t lo = 0, hi = n; /* lower_bound */
    while (lo < hi) {
      uint64_t mid = (lo + hi) / 2;
      if (p->days[mid] < k->rows[r]) lo = mid + 1; else hi = mid;
    }
    p->row_to_day[r] = lo;
    p->disc[r] = exp(-m->rate * (double)k->rows[r] / m->day_count);
  }
  return 0;
}

static void plan_free(simplan* p) {
  free(p->days);
  free(p->row_to_day);
  free(p->disc);
}

static int plan_path(const simplan* p, const oracle_kernel* k,
                     const oracle_model* m, uint64_t seed, uint64_t path,
                     double* ext, double* work) {
  uint64_t nA = m->n_assets;
  double* logS = work;
  double* raw = logS + nA;
  double* z = raw + nA;
  double* atDay = z + nA; /* [n_days][nA] */
  for (uint64_t j = 0; j < nA; ++j) logS[j] = log(m->spot[j]);
  int64_t prev = 0;
  for (uint64_t s = 0; s < p->n_days; ++s) {
    double dt = (double)(p->days[s] - prev) / m->day_count;
    prev = p->days[s];
    if (dt > 0.0) {
      for (uint64_t j = 0; j < nA; ++j)
        if (oracle_inv_normal_cdf(oracle_uniform(seed, path, s * nA + j),
                                  &raw[j]))
          return 5;
      for (uint64_t j = 0; j < nA; ++j) {
        double acc = 0.0;
        for (uint64_t l = 0; l <= j; ++l) acc += m->chol[j * nA + l] * raw[l];
        z[j] = acc;
      }
      for (uint64_t j = 0; j < nA; ++j)
        logS[j] += (m->drift[j] - 0.5 * m->vol[j] * m->vol[j]) * dt +
                   m->vol[j] * sqrt(dt) * z[j];
    }
    for (uint64_t j = 0; j < nA; ++j) atDay[s * nA + j] = exp(logS[j]);
  }
  for (uint64_t r = 0; r < k->n_rows; ++r)
    for (uint64_t c = 0; c < k->n_cols; ++c)
      ext[r * k->n_cols + c] = atDay[p->row_to_day[r] * nA + m->col_to_asset[c]];
  return 0;
}

int oracle_simulate_path(const oracle_kernel* k, const oracle_model* m,
                         uint64_t seed, uint64_t path, double* ext_out) {
  simplan p;
  int rc = plan_init(&p, k, m);
  if (rc == 0) {
    double* work = malloc(sizeof(double) * (3 + p.n_days + 1) * (m->n_assets + 1));
    rc = plan_path(&p, k, m, seed, path, ext_out, work);
    free(work);
  }
  plan_free(&p);
  return rc;
}

/* ---- pricing, proj/src/pricing.cpp:256-371 ----------------------------- */
static double pairwise_sum(const double* v, uint64_t n) {
  if (n <= 8) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += v[i];
    return s;
  }
  uint64_t half = n / 2;
  return pairwise_sum(v, half) + pairwise_sum(v + half, n - half);
}

typedef struct {
  const oracle_kernel* k;
  const oracle_model* m;
  const simplan* plan;
  uint64_t path0, paths, seed, lo, hi, n_days;
  const uint64_t* days;
  double* payoffs; /* [n_days][paths] */
  int err;
  char msg[256];
} worker;

static void* run_worker(void* arg) {
  worker* w = arg;
  uint64_t R = w->k->n_rows, C = w->k->n_cols, nA = w->m->n_assets;
  double* ext = malloc(sizeof(double) * (R * C + 1));
  double* work = malloc(sizeof(double) * (3 + w->plan->n_days + 1) * (nA + 1));
  for (uint64_t p = w->lo; p < w->hi && !w->err; ++p) {
    if (plan_path(w->plan, w->k, w->m, w->seed, w->path0 + p, ext, work)) {
      w->err = 5;
      snprintf(w->msg, sizeof w->msg, "invNormalCdf domain error");
      break;
    }
    for (uint64_t d = 0; d < w->n_days; ++d) {
      double v;
      int rc = oracle_eval_kernel(w->k, ext, w->plan->disc, w->days[d], &v,
                                  w->msg, sizeof w->msg);
      if (rc) { w->err = rc; break; }
      w->payoffs[d * w->paths + p] = v;
    }
  }
  free(ext);
  free(work);
  return NULL;
}

int oracle_price(const oracle_kernel* k, const oracle_model* m,
                 uint64_t path0, uint64_t paths, uint64_t seed,
                 const uint64_t* days, uint64_t n_days, unsigned threads,
                 double* price, double* se, double* payoffs_out, char* msg,
                 size_t msg_len) {
  if (paths == 0) {
    if (msg && msg_len) snprintf(msg, msg_len, "path count must be positive");
    return 5;
  }
  simplan plan;
  if (plan_init(&plan, k, m)) {
    plan_free(&plan);
    if (msg && msg_len)
      snprintf(msg, msg_len, "cannot simulate a negative observation day");
    return 5;
  }
  double* payoffs = payoffs_out ? payoffs_out
                                : malloc(sizeof(double) * paths * n_days);
  /* runParallel, proj/src/pricing.cpp:268-286 */
  if (threads == 0) threads = 1;
  if (threads > paths) threads = (unsigned)paths;
  uint64_t chunk = (paths + threads - 1) / threads;
  worker* ws = calloc(threads, sizeof(worker));
  pthread_t* th = calloc(threads, sizeof(pthread_t));
  unsigned used = 0;
  for (unsigned t = 0; t < threads; ++t) {
    uint64_t lo = t * chunk, hi = lo + chunk < paths ? lo + chunk : paths;
    if (lo >= hi) break;
    worker w = {k, m, &plan, path0, paths, seed, lo, hi, n_days, days, payoffs, 0, {0}};
    ws[t] = w;
    ++used;
  }
  if (used == 1) {
    run_worker(&ws[0]);
  } else {
    for (unsigned t = 0; t < used; ++t) pthread_create(&th[t], NULL, run_worker, &ws[t]);
    for (unsigned t = 0; t < used; ++t) pthread_join(th[t], NULL);
  }
  int rc = 0;
  for (unsigned t = 0; t < used; ++t)
    if (ws[t].err) {
      rc = ws[t].err;
      if (msg && msg_len) snprintf(msg, msg_len, "%s", ws[t].msg);
      break;
    }
  if (rc == 0) {
    double n = (double)paths;
    double* sq = malloc(sizeof(double) * paths);
    for (uint64_t d = 0; d < n_days; ++d) {
      const double* v = payoffs + d * paths;
      double mean = pairwise_sum(v, paths) / n;
      price[d] = mean;
      se[d] = 0.0;
      if (paths > 1) {
        for (uint64_t i = 0; i < paths; ++i) {
          double x = v[i] - mean;
          sq[i] = x * x;
        }
        double var = pairwise_sum(sq, paths) / (n - 1.0);
        se[d] = sqrt(var / n);
      }
    }
    free(sq);
  }
  free(ws);
  free(th);
  if (!payoffs_out) free(payoffs);
  plan_free(&plan);
  return rc;
}
