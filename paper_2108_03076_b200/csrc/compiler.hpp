// Payoff compiler: Kernel (KExpr tree) -> streaming device program.
//
// Semantics are exactly the reference evaluator's (evalKernel / KEval /
// kApplyBin, proj/src/kernel.cpp:182-310) evaluated for every valuation day
// of a priceAcrossTime call, with these compile-time transformations, each
// exact (bit-identical results, identical error behaviour):
//   * LoopIf (kernel.cpp:286-293) unrolled into nested Ifs over concrete
//     row offsets; TimeRef/Now/NatLit and all integer arithmetic folded
//     (rows are absolute days, t_now is fixed per output);
//   * PayRef -> +/-disc[row] or 0.0 constant (kernel.cpp:271-279), disc as
//     SimPlan computes it (pricing.cpp:207-210);
//   * If -> select with both branches evaluated eagerly (expressions are pure);
//     the reference's *errors* (division by zero, type and range errors) are
//     tracked in a separate error channel so an untaken branch never raises
//     and the first error in evaluation order is the one reported;
//   * OR/AND chains of comparisons against one literal -> running min/max
//     (x1<=L | x2<=L == fmin(x1,x2)<=L, NaN-exact), chains reassociated in
//     simulation-step order so they stream;
//   * hash-consing across valuation days and instances.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "cltk_b200.hpp"
#include "program.h"

namespace cltk {
namespace b200 {

// Host-side simulation plan (SimPlan, proj/src/pricing.cpp:173-212).
struct SimPlanHost {
  std::vector<int64_t> days;        // sorted distinct row days
  std::vector<uint32_t> rowToDay;   // kernel row -> step
  std::vector<uint32_t> colToAsset; // kernel col -> model asset
  std::vector<double> disc;         // per row
  uint32_t nAssets = 0;
  std::vector<cltk_step> steps;
  double chol[CLTK_MAX_ASSETS * CLTK_MAX_ASSETS] = {0};
  double logS0[CLTK_MAX_ASSETS] = {0};
  uint32_t usedMask = 0;
  uint32_t rng = CLTK_RNG_PHILOX;
  std::vector<cltk_bridge_op> bridge;  // QMC mode: construction ops in traversal order
  uint32_t bridgeSlots = 0;
};
SimPlanHost buildSimPlan(const Kernel& k, const ModelSpec& m, uint32_t rng = CLTK_RNG_PHILOX);

struct ErrorSite {
  ErrorCode code;
  std::string message;
};

// Step kinds stored in cltk_step::draws.
enum : uint32_t { STEP_CONST_S = 0, STEP_DRAW = 1, STEP_EXP_ONLY = 2 };

struct CompiledProgram {
  std::vector<cltk_bridge_op> bridge;  // QMC mode
  std::vector<uint64_t> code;          // shared ops (step-ordered) then instance ops
  std::vector<uint64_t> packed;        // device stream: code with VEC run headers
  std::vector<cltk_step> steps;        // simulation constants + shared-op ranges
  std::vector<double> sharedConst;     // bit patterns for B/I/E constants
  std::vector<double> instConst;       // [n_instances][n_inst_const]
  std::vector<cltk_output> outputs;    // [n_days]
  std::vector<uint32_t> streamMask;    // [n_steps] when header.stream (DevPlan::streamMask)
  std::vector<ErrorSite> sites;        // site id -> error (id 0 unused, 1 = domain)
  cltk_plan_header header{};
  uint64_t kernelNodes = 0, dagNodes = 0;
  uint32_t nSharedOps = 0, nInstOps = 0;
  std::vector<uint32_t> stepCodeBegin; // per step, the start of its ops in `code` (+ end)
  std::vector<int64_t> days;           // valuation days
  bool faultBuild = false;             // test build: RunArgs fault injection compiled in
};

// Paths of at most this many normal draws with one output accumulate the
// output per thread in registers (cltk_plan_header::reg_acc).
constexpr uint64_t kRegAccMaxDraws = 64;
// Philox paths of at most this many normal slots (steps x assets) stream
// through full normal batches (cltk_plan_header::stream).
constexpr uint64_t kStreamMaxSlots = 64;
// Template batches of at least this many instances (one valuation day, no
// error channel) reduce their outputs instance-major (cltk_plan_header::inst_major).
constexpr uint64_t kInstMajorMin = 32;

struct CompileOptions {
  bool rewrite = true;
};

// Template instances: the float literals (FloatLit nodes in node-pool order,
// i.e. postorder of the kernel JSON tree) of each instance, row-major.
struct LiteralTable {
  std::size_t nInst = 0;
  std::size_t nOcc = 0;
  std::vector<double> values;  // [nInst][nOcc]
};
std::vector<double> kernelLiterals(const Kernel& k);
LiteralTable literalTableFromInstances(const std::vector<const Kernel*>& instances);

CompiledProgram compileProgram(const Kernel& k, const LiteralTable& lits, const SimPlanHost& plan,
                               const std::vector<uint64_t>& days, const CompileOptions& opt);
// The program as JSON (ops, steps, constants, outputs, header fields): tests,
// DESIGN.md, the bench's upload accounting.
std::string programListing(const CompiledProgram& P);
CompiledProgram compileProgram(const std::vector<const Kernel*>& instances,
                               const SimPlanHost& plan, const std::vector<uint64_t>& days,
                               const CompileOptions& opt);

}  // namespace b200
}  // namespace cltk
