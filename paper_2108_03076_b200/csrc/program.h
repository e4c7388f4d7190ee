// Device program format shared by the host payoff compiler (compiler.cpp) and
// the sm_100a Monte Carlo engine (mc_engine.cu).
//
// A compiled payoff is a *streaming* three-address program over per-thread
// registers: every instruction is attached to the simulation step (sorted
// distinct kernel day, SimPlan::days in proj/src/pricing.cpp:182-190) at
// which all of its observable inputs exist, so the engine interleaves payoff
// evaluation with path generation and never materialises ext[rows][cols]
// (proj/src/pricing.cpp:247-251) anywhere -- not in HBM, not in shared memory.
//
// Operand space (14-bit indices):
//   [0, n_assets)             S-slots: this step's spot per model asset
//   [n_assets, n_thread)      thread registers
//   [n_thread, n_thread+n_shared_const)            warp-broadcast constants
//   [n_thread+n_shared_const, ... + n_inst_const)  per-instance constants
// Thread registers live in shared memory, register-major
// (reg * BLOCK + tid) so a warp touches 32 consecutive doubles; constants live
// in a per-warp shared-memory table read as a broadcast.
#pragma once
#include <stdint.h>

#define CLTK_OP_BITS 8
#define CLTK_FIELD_BITS 14
#define CLTK_MAX_OPERANDS (1 << CLTK_FIELD_BITS)
// Models of up to 32 assets (one step's draws fill a 32-bit draw window); the
// ahead-of-time (interpreter) kernels and the QMC mode cover up to
// CLTK_AOT_MAX_ASSETS, larger models run the NVRTC kernel.
#ifndef CLTK_MAX_ASSETS
#define CLTK_MAX_ASSETS 32
#endif
#define CLTK_AOT_MAX_ASSETS 8

// Value kinds in the 8-byte register slots: R = IEEE double; B = double 0/1;
// I = int64 bit pattern (KExpr int values, proj/src/kernel.cpp:187);
// E = int64 error-site index (0 = no error).
enum cltk_opcode : uint32_t {
  OP_NOP = 0,
  OP_MOV,      // d = a
  OP_NEG,      // R: d = -a
  OP_NOT,      // B: d = !a
  OP_ADD,      // R: d = a + b (IEEE, never contracted)
  OP_SUB,
  OP_MUL,
  OP_DIV,      // R: d = a / b  (zero divisor guarded by OP_EDIVZ)
  OP_LT,       // R,R -> B
  OP_LEQ,
  OP_EQ,
  OP_AND,      // B,B -> B
  OP_OR,
  OP_SEL,      // d = a ? b : c   (any kind; a is B)
  OP_IADD,     // I: d = a + b (int64 wrap)
  OP_ISUB,
  OP_ILT,      // I,I -> B
  OP_ILEQ,
  OP_IEQ,
  OP_MIN,      // R: fmin (NaN-ignoring)   -- OR/AND-of-compare rewrite
  OP_MAX,      // R: fmax (NaN-ignoring)
  OP_MINP,     // R: NaN-propagating min
  OP_MAXP,     // R: NaN-propagating max
  OP_EFIRST,   // E: d = a != 0 ? a : b
  OP_EDIVZ,    // E: d = (a == 0.0) ? c(field) : 0   (c is an immediate site id)
  OP_COUNT,
  // Run header: the next d(field) words are ops of opcode a(field), executed
  // by one tight loop (no per-op dispatch).  Emitted for runs >= 2.
  OP_VEC = 63
};

#if !defined(__CUDACC_RTC__)
// 64-bit instruction: op | d<<8 | a<<22 | b<<36 | c<<50
static inline uint64_t cltk_encode(uint32_t op, uint32_t d, uint32_t a,
                                   uint32_t b, uint32_t c) {
  return (uint64_t)op | ((uint64_t)d << 8) | ((uint64_t)a << 22) |
         ((uint64_t)b << 36) | ((uint64_t)c << 50);
}
#endif

// Per-step simulation constants (host-computed with glibc, bit-identical to
// the reference's SimPlan arithmetic, proj/src/pricing.cpp:226-245).
typedef struct {
  double A[CLTK_MAX_ASSETS];  // (drift - 0.5*vol*vol) * dt
  double B[CLTK_MAX_ASSETS];  // vol * sqrt(dt)
  double S[CLTK_MAX_ASSETS];  // exp(log(spot)) when dt == 0 (path-independent)
  uint32_t draws;             // 1: dt > 0 (draw nA normals), 0: dt == 0
  uint32_t code_begin;        // shared-op range of this step
  uint32_t code_end;
  // QMC mode (Sobol + AS241 + Brownian bridge): bridge ops [br_begin, br_end)
  // computed before this (drawing) step, then W(t_s) read from slot br_emit;
  // A = (drift - 0.5*vol*vol) * t_s, B = vol (t_s: years from day 0).
  uint32_t br_begin;
  uint32_t br_end;
  uint32_t br_emit;
  // NVRTC mode: the step's op class (steps with identical ops share one;
  // 0 = no ops), the `case` of the generated payoff policy (jit.cpp).
  uint32_t jit_class;
  // Philox mode: draw-slot mask of the steps s, s+1, ... (bits q*nA .. q*nA+nA-1
  // set when step s+q draws; q < 32 / nA): a normal batch starting at step s
  // masks it to its own slots (domain errors count only for drawn indices).
  uint32_t draw_window;
} cltk_step;

// Device layout of the steps (engine_types.h StepRef): per step this header,
// then A, B and S of the plan's assets (each padded to an even count so the
// arrays stay 16-byte aligned): 32 + 24 * even(nA) bytes instead of the host
// struct's 32 + 24 * CLTK_MAX_ASSETS.
typedef struct {
  uint32_t draws;
  uint32_t code_begin;
  uint32_t code_end;
  uint32_t br_begin;
  uint32_t br_end;
  uint32_t br_emit;
  uint32_t jit_class;
  uint32_t draw_window;
} cltk_step_hdr;

// Brownian-bridge construction op (QMC mode): for every asset j
//   W[dst][j] = wl * W[l][j] + wr * W[r][j] + sd * Z[c][j]
// (l == CLTK_BR_ORIGIN: W(0) = 0); Z[c] uses Sobol dimensions node * nA + j.
#define CLTK_BR_ORIGIN 0xFFFFu
typedef struct {
  double wl, wr, sd;
  uint32_t node;
  uint16_t dst, l, r, pad;
} cltk_bridge_op;

// Launch-time header of a compiled plan (everything uniform across threads).
typedef struct {
  uint32_t n_assets;        // model assets (draws per step)
  uint32_t n_steps;
  uint32_t n_thread;        // S-slots + thread registers
  uint32_t n_shared_const;
  uint32_t n_inst_const;
  uint32_t n_instances;
  uint32_t n_days;          // valuation days
  uint32_t inst_code_begin; // instance-op range (run once per instance)
  uint32_t inst_code_end;
  uint32_t has_err;         // any output carries an error register
  uint32_t used_mask;       // model assets referenced by any kernel column
  uint32_t rng;             // CLTK_RNG_PHILOX (reference parity) / CLTK_RNG_SOBOL
  uint32_t n_bridge_slots;  // QMC: W slots per asset
  uint32_t n_bridge_ops;    // QMC: computes (= drawing steps)
  uint32_t reg_base;        // path kernel: leading operand slots without shared-memory
                            // columns (the NVRTC kernel keeps the S-slots in registers)
  uint32_t reg_top;         // path kernel: operand slots [reg_base, reg_top) have columns
                            // (n_thread; the NVRTC kernel: only the registers it stores)
  uint32_t reg_acc;         // path kernel: 1 = one output, short paths: per-thread register
                            // accumulation of the output, one warp sum per chunk
  uint32_t stream;          // path kernel: 1 = short Philox paths: a thread's paths of a
                            // chunk drawn as one stream of full normal batches
  uint32_t inst_major;      // path kernel: 1 = template batch (many instances, one day, no
                            // error channel): instance-major output reduction
  uint32_t first_draw;      // first step that draws (per-path normal batches start there:
                            // the leading non-drawing steps -- day 0 -- take no slots)
  uint32_t log_bounded;     // 1: every path's log-spots provably stay in (-500, 500)
                            // (host bound over the largest normal): the NVRTC payoff's
                            // log-domain ops need no range checks
  double chol[CLTK_MAX_ASSETS * CLTK_MAX_ASSETS];  // lower factor, rows of n_assets (packed)
  double logS0[CLTK_MAX_ASSETS];                   // log(spot)
} cltk_plan_header;

// Output slot: value operand and error operand (0xFFFF... = none) per
// valuation day, evaluated after the instance ops of each instance.
typedef struct {
  uint32_t val;
  uint32_t err;
} cltk_output;

#define CLTK_NO_ERR 0xFFFFFFFFu

#define CLTK_RNG_PHILOX 0u
#define CLTK_RNG_SOBOL 1u
#define CLTK_SOBOL_MAX_DIMS 2048u

// Chunk partial of one output: count, mean, sum of squared deviations.
typedef struct {
  double n;
  double mean;
  double m2;
} cltk_partial;
