/* TEST INFRASTRUCTURE ONLY -- the CPU restatement of the reference's Monte
 * Carlo pricing path, used by tests/ and bench.py's cpu_baseline leg as the
 * checker.  Never part of the product path (which has no CPU fallback).
 *
 * Parity pinned: tests/test_oracle.py checks every function below against the
 * compiled reference (oracle/_ref/libcltkref.so) and the golden vectors in
 * tests/golden/ (generated from the reference by oracle/make_golden.py).
 */
#ifndef CLTK_ORACLE_H
#define CLTK_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/pricing.cpp:73-98 */
uint64_t oracle_philox_bits(uint64_t seed, uint64_t path, uint64_t i);
/* proj/src/pricing.cpp:100-103 */
double oracle_uniform(uint64_t seed, uint64_t path, uint64_t i);
/* proj/src/pricing.cpp:109-148; returns 0 or 5 (EvalError: domain) */
int oracle_inv_normal_cdf(double p, double* out);
double oracle_normal_cdf(double x);
/* proj/src/pricing.cpp:45-69; returns 0 or 5 */
int oracle_cholesky(const double* m, int n, double* l);

/* Flattened kernel tree (serialised by tests/oracle_py.py from kernel JSON,
 * proj/src/kernel.cpp:520-638).  Node kinds mirror KExpr
 * (proj/include/cltk/kernel.hpp:22-80). */
enum {
  OK_IF = 0, OK_FLOAT, OK_NAT, OK_BOOL, OK_NOW, OK_TIMEREF, OK_OBSREF,
  OK_PAYREF, OK_UNOP, OK_BINOP, OK_LOOPIF
};
enum { OU_NEG = 0, OU_NOT = 1 };
enum { OB_ADD = 0, OB_SUB, OB_MULT, OB_DIV, OB_LT, OB_LEQ, OB_EQ, OB_AND, OB_OR };

typedef struct {
  int32_t kind;
  int32_t op;        /* unop / binop */
  int32_t a, b, c;   /* children: cond/then/else, left/right, arg */
  int32_t pay_sign;  /* PayRef: +1 (p1->p2), -1 (p2->p1), 0 */
  uint64_t row, col; /* TimeRef/ObsRef/PayRef */
  uint64_t nat;      /* NatLit value, LoopIf window */
  double real;       /* FloatLit value */
  int32_t boolean;   /* BoolLit value */
  int32_t pad;
} oracle_node;

typedef struct {
  const oracle_node* nodes;
  int32_t root;
  uint64_t n_rows, n_cols;
  const int64_t* rows; /* [n_rows] absolute days */
} oracle_kernel;

/* evalKernel (proj/src/kernel.cpp:229-310).  Returns 0, 3 (TypeError) or
 * 5 (EvalError); msg (may be NULL) receives the reference's message. */
int oracle_eval_kernel(const oracle_kernel* k, const double* ext,
                       const double* disc, uint64_t t_now, double* out,
                       char* msg, size_t msg_len);

typedef struct {
  uint64_t n_assets;
  const double* spot;   /* [n_assets], model order */
  const double* vol;
  const double* drift;
  const double* chol;   /* [n_assets*n_assets] lower factor (or identity) */
  double rate, day_count;
  const uint64_t* col_to_asset; /* [n_cols] */
} oracle_model;

/* SimPlan::path (proj/src/pricing.cpp:173-253): ext_out [n_rows][n_cols].
 * Returns 0 or 5. */
int oracle_simulate_path(const oracle_kernel* k, const oracle_model* m,
                         uint64_t seed, uint64_t path, double* ext_out);

/* priceAcrossTime (proj/src/pricing.cpp:327-371), path range
 * [path0, path0+paths) (path0 = 0 for the reference semantics).
 * price/se: [n_days].  payoffs (optional, may be NULL): [n_days][paths]. */
int oracle_price(const oracle_kernel* k, const oracle_model* m,
                 uint64_t path0, uint64_t paths, uint64_t seed,
                 const uint64_t* days, uint64_t n_days, unsigned threads,
                 double* price, double* se, double* payoffs, char* msg,
                 size_t msg_len);

#ifdef __cplusplus
}
#endif
#endif
