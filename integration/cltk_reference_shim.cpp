// The reference-side binding: what a maintainer of the reference adds to route
// its pricing entry points to the B200 engine.  It takes the
// reference's own types -- cltk::Kernel, cltk::ModelSpec, cltk::TEnv
// (proj/include/cltk/{kernel,pricing,env}.hpp) -- serialises them with the
// reference's own writers (kernelToJson proj/src/kernel.cpp:620, tenvToJson
// proj/src/json_io.cpp:305) and calls the C ABI (include/cltk_b200.h).
//
// In the reference the two functions below replace the bodies of
// cltk::priceAcrossTime / cltk::priceMC (proj/include/cltk/pricing.hpp:84-98);
// here they live in namespace cltk::gpu so the test build can link them next
// to the unmodified reference library (oracle/_ref/libcltkref.so, which keeps
// its own CPU cltk::priceAcrossTime as the comparison).
//
// Test build: oracle/Makefile -> oracle/_ref/libcltk_shim.so (needs the
// reference headers, so it is built where /root/reference is mounted and
// travels prebuilt); tests/test_reference_shim.py drives it through the
// extern "C" entry points at the end of this file.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cltk/compile.hpp"
#include "cltk/errors.hpp"
#include "cltk/il.hpp"
#include "cltk/json_io.hpp"
#include "cltk/kernel.hpp"
#include "cltk/parser.hpp"
#include "cltk/pricing.hpp"
#include "cltk/semantics.hpp"
#include "cltk_b200.h"

namespace cltk {
namespace gpu {

// ModelSpec has no JSON writer in the reference: this is modelFromJson's
// schema (proj/src/pricing.cpp:20-43) written back.
std::string modelToJson(const ModelSpec& m) {
  nlohmann::json j;
  j["rate"] = m.rate;
  j["dayCount"] = m.dayCount;
  j["order"] = m.order;
  j["labels"] = nlohmann::json::object();
  for (const auto& [label, a] : m.assets)
    j["labels"][label] = {{"spot", a.spot}, {"vol", a.vol}, {"drift", a.drift}};
  if (!m.corr.empty()) j["corr"] = m.corr;
  return j.dump();
}

// cltk::priceAcrossTime (proj/include/cltk/pricing.hpp:92-98) on the GPU.
std::vector<PriceResult> priceAcrossTime(const Kernel& k, const ModelSpec& model,
                                         std::uint64_t paths, std::uint64_t seed,
                                         const std::vector<std::uint64_t>& days,
                                         const TEnv& tenv, unsigned threads = 0) {
  const std::string kj = kernelToJson(k).dump();
  const std::string mj = modelToJson(model);
  const std::string tj = tenvToJson(tenv).dump();
  std::vector<cltk_price_result> out(days.size());
  cltk_error err{};
  const int rc = cltk_gpu_price(kj.c_str(), mj.c_str(), paths, seed, days.data(), days.size(),
                                tj.c_str(), threads, /*device=*/-1, out.data(), &err);
  switch (rc) {  // proj/include/cltk/errors.hpp:10-16, same message text
    case 0: break;
    case 2: throw Error(ErrorCode::Parse, err.message);
    case 3: throw TypeError(err.message);
    case 4: throw UnsupportedError(err.message);
    default: throw EvalError(err.message);
  }
  std::vector<PriceResult> r;
  for (const auto& o : out) r.push_back({o.price, o.std_error, o.paths, o.seed, o.valuation_day});
  return r;
}

// cltk::priceMC (proj/include/cltk/pricing.hpp:84-89): unchanged, one day.
PriceResult priceMC(const Kernel& k, const ModelSpec& model, std::uint64_t paths,
                    std::uint64_t seed, std::uint64_t valuationDay, const TEnv& tenv,
                    unsigned threads = 0) {
  return gpu::priceAcrossTime(k, model, paths, seed, {valuationDay}, tenv, threads).front();
}

}  // namespace gpu
}  // namespace cltk

// ---- test entry points (TEST INFRASTRUCTURE: tests/test_reference_shim.py) ----
namespace {

thread_local std::string g_msg;

// The reference's front end on a contract: parse, typecheck, compileContract,
// cutPayoff, reindex (the chain of `cltk price`, proj/tools/cli.cpp:246-259).
cltk::Kernel kernelOfContract(const char* src, const cltk::TEnv& tenv) {
  cltk::ContrPtr c = cltk::parseContract(src);
  cltk::typeCheckContr(cltk::TypeCtx{}, c);
  return cltk::reindex(cltk::cutPayoff(cltk::compileContract(c)), tenv);
}

// From the IL wire format (ilToJson) of a compiled, uncut contract.
cltk::Kernel kernelOfIL(const char* ilJson, const cltk::TEnv& tenv) {
  return cltk::reindex(cltk::cutPayoff(cltk::ilFromJson(nlohmann::json::parse(ilJson))), tenv);
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    g_msg.clear();
    return 0;
  } catch (const cltk::Error& e) {
    g_msg = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* cltkshim_last_error(void) { return g_msg.c_str(); }

// source_kind 0: `source` is a contract (CL text); 1: the IL JSON of an uncut
// compiled contract.  engine 0: the reference's CPU priceAcrossTime; 1: the
// shim (GPU).  out_price / out_se: [n_days].
int cltkshim_price(const char* source, int source_kind, const char* tenv_json,
                   const char* model_json, std::uint64_t paths, std::uint64_t seed,
                   const std::uint64_t* days, std::size_t n_days, int engine,
                   unsigned threads, double* out_price, double* out_se) {
  return guarded([&] {
    const cltk::TEnv tenv = (tenv_json && *tenv_json)
                                ? cltk::tenvFromJson(nlohmann::json::parse(tenv_json))
                                : cltk::TEnv{};
    const cltk::Kernel k = source_kind == 0 ? kernelOfContract(source, tenv)
                                            : kernelOfIL(source, tenv);
    const cltk::ModelSpec m = cltk::modelFromJson(nlohmann::json::parse(model_json));
    const std::vector<std::uint64_t> d(days, days + n_days);
    const auto r = engine == 0 ? cltk::priceAcrossTime(k, m, paths, seed, d, tenv, threads)
                               : cltk::gpu::priceAcrossTime(k, m, paths, seed, d, tenv, threads);
    for (std::size_t i = 0; i < r.size(); ++i) {
      out_price[i] = r[i].price;
      out_se[i] = r[i].stdError;
    }
  });
}

// priceMC through the shim (engine 1) or the reference (engine 0).
int cltkshim_price_mc(const char* contract, const char* model_json, std::uint64_t paths,
                      std::uint64_t seed, std::uint64_t day, int engine, double* price,
                      double* se) {
  return guarded([&] {
    const cltk::Kernel k = kernelOfContract(contract, cltk::TEnv{});
    const cltk::ModelSpec m = cltk::modelFromJson(nlohmann::json::parse(model_json));
    const cltk::PriceResult r = engine == 0 ? cltk::priceMC(k, m, paths, seed, day, cltk::TEnv{})
                                            : cltk::gpu::priceMC(k, m, paths, seed, day,
                                                                 cltk::TEnv{});
    *price = r.price;
    *se = r.stdError;
  });
}

}  // extern "C"
