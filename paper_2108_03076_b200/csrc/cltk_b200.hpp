// C++ host API of the B200 pricing engine -- the reference's pricing surface
// re-declared over the engine (namespace cltk::b200):
//
//   reference (proj/include/cltk/pricing.hpp)       here
//   -----------------------------------------       ----
//   ModelSpec / AssetSpec / modelFromJson  :16-35   same names
//   cholesky                               :37-40   same
//   PriceResult / priceResultToJson        :65-75   same
//   priceMC                                :84-89   same signature
//   priceAcrossTime                        :92-98   same signature
//   Kernel / kernelFromJson (proj/include/cltk/kernel.hpp:71-79, :124)
//   Error / ErrorCode / EvalError / TypeError (proj/include/cltk/errors.hpp)
//
// plus the batch entry point (one template, many literal instances, shared
// paths) and the plan API the C-ABI (include/cltk_b200.h) exposes.
// `threads` is accepted for signature compatibility; on the GPU it maps to
// nothing (results are bit-identical for any value, as in the reference).
#pragma once
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace cltk {
namespace b200 {

// proj/include/cltk/errors.hpp:10-16 (values are the CLI exit codes)
enum class ErrorCode { Parse = 2, Type = 3, Unsupported = 4, Eval = 5, Verification = 6 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};
struct ParseError : Error {
  explicit ParseError(const std::string& m) : Error(ErrorCode::Parse, m) {}
};
struct TypeError : Error {
  explicit TypeError(const std::string& m) : Error(ErrorCode::Type, m) {}
};
struct UnsupportedError : Error {
  explicit UnsupportedError(const std::string& m) : Error(ErrorCode::Unsupported, m) {}
};
struct EvalError : Error {
  explicit EvalError(const std::string& m) : Error(ErrorCode::Eval, m) {}
};
// A CUDA / device failure (not a reference error category).
struct DeviceError : Error {
  explicit DeviceError(const std::string& m) : Error(ErrorCode::Unsupported, "device: " + m) {}
};

// ---- kernel IR: KExpr (proj/include/cltk/kernel.hpp:22-66) as a node pool --
enum class KKind { If, Float, Nat, Bool, Now, TimeRef, ObsRef, PayRef, UnOp, BinOp, LoopIf };
enum class KUn { Neg, Not };
enum class KBin { Add, Sub, Mult, Div, Lt, Leq, Eq, And, Or };

struct KNode {
  KKind kind;
  int op = 0;                // KUn / KBin
  int32_t a = -1, b = -1, c = -1;  // children (cond/then/else, left/right, arg)
  uint64_t row = 0, col = 0; // TimeRef/ObsRef/PayRef
  uint64_t nat = 0;          // NatLit value; LoopIf window
  double real = 0.0;         // FloatLit
  bool boolean = false;      // BoolLit
  int32_t from = -1, to = -1;  // PayRef parties (index into Kernel::partyNames)
  int32_t wvar = -1;         // LoopIf window's template variable (index into tvars), -1: literal
};

// Flattened payoff (proj/include/cltk/kernel.hpp:71-79).
struct Kernel {
  std::vector<KNode> nodes;  // children precede parents
  int32_t root = -1;
  std::vector<int64_t> rows;
  std::vector<std::string> cols;
  std::vector<std::string> tvars;
  std::vector<std::string> parties;
  uint64_t horizon = 0;
  std::vector<std::string> partyNames;  // interned PayRef party strings
};

// kernelFromJson (proj/src/kernel.cpp:631-638; wire format :520-629).
Kernel kernelFromJson(const std::string& json);

// The reference's textual kernel format (emitKernelSource,
// proj/src/kernel.cpp:407; proj/docs/kernel-format.md).  tenvValues[k] backs
// loop windows written as tenv[k].
Kernel kernelFromSource(const std::string& text, const std::vector<uint64_t>& tenvValues = {});
// Either wire format: JSON ('{' first) or kernel text.
Kernel kernelFromWire(const std::string& text, const std::vector<uint64_t>& tenvValues = {});

class TEnv;
// reindex (proj/src/kernel.cpp:14-180, :301-303): the IL of a compiled
// contract (its JSON wire format, ilToJson, proj/src/json_io.cpp:203-303)
// flattened into a kernel with template variables bound from tenv.
Kernel kernelFromIL(const std::string& ilJson, const TEnv& tenv);
// kernelToJson (proj/src/kernel.cpp:520-623), compact.
std::string kernelToJsonString(const Kernel& k);

// Shape hash: equal for kernels that differ only in FloatLit values (the
// "template instances" of one contract, priced with shared paths).
uint64_t kernelShapeHash(const Kernel& k);

// ---- model (proj/include/cltk/pricing.hpp:16-35) ----------------------------
struct AssetSpec {
  double spot = 0.0;
  double vol = 0.0;
  double drift = 0.0;
};
struct ModelSpec {
  std::vector<std::string> order;
  std::map<std::string, AssetSpec> assets;
  std::vector<std::vector<double>> corr;
  double rate = 0.0;
  double dayCount = 365.0;
  const AssetSpec& at(const std::string& label) const;
};
ModelSpec modelFromJson(const std::string& json);
std::vector<std::vector<double>> cholesky(const std::vector<std::vector<double>>& m);
double blackScholesCall(double spot, double strike, double rate, double vol, double tYears);

class TEnv {
 public:
  TEnv() = default;
  explicit TEnv(std::map<std::string, uint64_t> m) : map_(std::move(m)) {}
  uint64_t lookup(const std::string& name) const;
  void bind(const std::string& name, uint64_t v) { map_[name] = v; }

 private:
  std::map<std::string, uint64_t> map_;
};
TEnv tenvFromJson(const std::string& json);

struct PriceResult {
  double price = 0.0;
  double stdError = 0.0;
  uint64_t paths = 0;
  uint64_t seed = 0;
  uint64_t valuationDay = 0;
};
std::string priceResultToJson(const PriceResult& r);

// ---- engine options --------------------------------------------------------
struct RunOptions {
  int device = -1;      // -1: current device
  bool rewrite = true;  // OR/AND-of-compare -> running min/max (exact)
  // 0: Philox2x64-10 + Acklam/Halley (the reference's generator, bit-exact);
  // 1: Sobol (Joe-Kuo, 32-bit) + Wichura AS241 + Brownian bridge (QMC;
  //    seed != 0 applies a Philox-derived digital shift per dimension).
  int rng = 0;
  // Payoff evaluation: 0 = bytecode interpreter (ahead-of-time kernel),
  // 1 = NVRTC-generated kernel (jit.cpp; error if NVRTC is unavailable),
  // 2 = NVRTC when available and the program is small enough, else 0
  // (default: the one-shot entry points price with the generated kernel,
  // compiled once per program shape and cached in-process and on disk).
  int jit = 2;
  // One-shot pricing over several GPUs of this process: the plan is built on
  // every listed device, the deterministic chunks are sharded in contiguous
  // equal slices, one NCCL all-gather assembles the chunk partials, and the
  // fixed-order combine runs on the first device -- results bit-identical to
  // one device.  Empty: the single `device`.  A device may repeat (tests:
  // the shards then share one GPU and are gathered with device copies).
  std::vector<int> devices;
  // Test build: the path kernel with the RunArgs fault hook compiled in
  // (Plan::setFault); never set on the pricing path.
  bool faultInject = false;
};

// ---- compiled plan (host + device state) ------------------------------------
struct PlanImpl;
struct PlanInfo {
  uint32_t n_assets, n_steps, n_thread, n_shared_const, n_inst_const;
  uint32_t n_instances, n_days, n_outputs;
  uint32_t n_shared_ops, n_inst_ops, has_err, block;
  uint64_t kernel_nodes, dag_nodes;
  uint32_t jit;  // 1: the plan runs the NVRTC-generated kernel
};

class Plan {
 public:
  // One template (instances[0]) and its literal instances (same shape).
  Plan(const std::vector<const Kernel*>& instances, const ModelSpec& model,
       const std::vector<uint64_t>& days, const TEnv& tenv, const RunOptions& opt);
  // One template and a literal table: literals[i * nLits + j] is float
  // literal j (FloatLit nodes in postorder of the kernel JSON tree) of
  // instance i -- "template parameters passed as kernel arguments".
  Plan(const Kernel& templ, const double* literals, std::size_t nInstances, std::size_t nLits,
       const ModelSpec& model, const std::vector<uint64_t>& days, const TEnv& tenv,
       const RunOptions& opt);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  PlanInfo info() const;
  // Deterministic chunking of the path index space: a function of (paths,
  // n_outputs) only, so any sharding of whole chunks over GPUs reproduces
  // the same partials (and the same bits).
  void chunking(uint64_t paths, uint64_t* chunkPaths, uint64_t* nChunks) const;
  // Asynchronous: price chunks [c0, c1) of a `paths`-path run into
  // partials[c][out] (device pointer, n_chunks * n_outputs cltk_partial).
  void launch(uint64_t paths, uint64_t seed, uint64_t c0, uint64_t c1, void* partialsDev,
              void* stream);
  // Combine partials[0, n_chunks) in a fixed order, read back, check the
  // device error word; results [instance][day].
  std::vector<PriceResult> finalize(uint64_t paths, uint64_t seed, const void* partialsDev,
                                    void* stream);
  std::string dump() const;  // program listing (JSON) for tests / DESIGN.md
  // Test hook (plans built with RunOptions::faultInject): later launches
  // force the uniform of draw `draw` of path `path` to exactly 1.0, the
  // reference's invNormalCdf domain error (path = ~0: none).
  void setFault(uint64_t path, uint32_t draw);
  int device() const;
  PlanImpl* impl() { return impl_.get(); }

 private:
  void init(const Kernel& k, const void* lits, const ModelSpec& model,
            const std::vector<uint64_t>& days, const TEnv& tenv, const RunOptions& opt);
  std::unique_ptr<PlanImpl> impl_;
};

// ---- device error word / test hooks ----------------------------------------
uint64_t planErrorWord(Plan& plan, void* stream);
void planSetErrorWord(Plan& plan, void* stream, uint64_t word);
// Per-path outputs / spots / normals (host buffers; any may be null).
uint64_t debugPaths(Plan& plan, uint64_t seed, uint64_t path0, uint64_t npaths, double* outputs,
                    double* spots, double* normals);
void debugRng(int device, uint64_t seed, uint64_t path, uint64_t i0, uint64_t n, uint64_t* bits,
              double* uniforms, double* normals);
double fp64Peak(int device, int iters, double* seconds);
// Sobol integers of points [n0, n0+n), dims [d0, d0+nd) from the device
// generator (out[n][nd], host buffer).
void debugSobol(int device, uint64_t n0, uint64_t n, uint32_t d0, uint32_t nd, bool aligned,
                uint32_t* out);
// Device exp / log / erfc / invNormalCdf (fn 0..3) over a host array.
void debugMath(int device, int fn, const double* x, uint64_t n, double* out);

// ---- the reference pricing API (proj/include/cltk/pricing.hpp:84-98) --------
PriceResult priceMC(const Kernel& k, const ModelSpec& model, uint64_t paths, uint64_t seed,
                    uint64_t valuationDay, const TEnv& tenv, unsigned threads = 0);
std::vector<PriceResult> priceAcrossTime(const Kernel& k, const ModelSpec& model,
                                         uint64_t paths, uint64_t seed,
                                         const std::vector<uint64_t>& days, const TEnv& tenv,
                                         unsigned threads = 0);
// FloatLit values of a kernel in the engine's literal order.
std::vector<double> kernelFloatLiterals(const Kernel& k);
std::vector<PriceResult> priceTemplate(const Kernel& templ, const double* literals,
                                       std::size_t nInstances, std::size_t nLits,
                                       const ModelSpec& model, uint64_t paths, uint64_t seed,
                                       const std::vector<uint64_t>& days, const TEnv& tenv,
                                       const RunOptions& opt = RunOptions());
// One-shot pricing through an in-process plan cache (the last few plans,
// keyed by the caller's exact wire inputs, options and device): a repeated
// call skips parsing, compiling and uploading.  make() builds the plan on a
// miss.  Plans in the cache are used by one caller at a time.
// make(device) builds the plan on one device; with several devices the call
// is sharded over them (RunOptions::devices).
std::vector<PriceResult> priceCached(const std::string& key,
                                     const std::function<std::unique_ptr<Plan>(int)>& make,
                                     const std::vector<int>& devices, uint64_t paths,
                                     uint64_t seed, const std::vector<uint64_t>& days);
// The devices a one-shot call with these options runs on: opt.devices, else
// $CLTK_DEVICES ("all" or "0,1,...") when opt.device < 0, else {opt.device}.
std::vector<int> resolveDevices(const RunOptions& opt);
// Template batch: instances share one path set (common random numbers, like
// repeated reference calls with one seed); result [instance * days + d].
std::vector<PriceResult> priceBatch(const std::vector<const Kernel*>& instances,
                                    const ModelSpec& model, uint64_t paths, uint64_t seed,
                                    const std::vector<uint64_t>& days, const TEnv& tenv,
                                    const RunOptions& opt = RunOptions());

}  // namespace b200
}  // namespace cltk
