// TEST INFRASTRUCTURE ONLY -- never linked into, loaded by, or called from the
// product path.  This is a thin extern "C" driver around the UNMODIFIED
// reference library (`/root/reference/proj/src/*.cpp`, compiled by
// oracle/Makefile into oracle/_ref/libcltkref.so).  Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() load it, and
// only as the checker.
//
// Every entry point forwards to the reference API it names:
//   cltkref_compile_kernel_json -> parseContract/typeCheckContr
//       (proj/src/parser.cpp:479, proj/src/semantics.cpp:79),
//       compileContract + cutPayoff (proj/src/compile.cpp:146,
//       proj/src/ilsem.cpp:323), reindex (proj/src/kernel.cpp:301),
//       kernelToJson (proj/src/kernel.cpp:620)
//   cltkref_philox_bits/uniform/normal -> CounterRng (proj/src/pricing.cpp:96-107)
//   cltkref_inv_normal_cdf / normal_cdf -> proj/src/pricing.cpp:109-148
//   cltkref_simulate_paths  -> simulatePath (proj/src/pricing.cpp:311)
//   cltkref_eval_kernel     -> evalKernel (proj/src/kernel.cpp:305)
//   cltkref_path_payoffs    -> the per-path loop of priceAcrossTime
//                              (proj/src/pricing.cpp:349-358)
//   cltkref_price           -> priceAcrossTime (proj/src/pricing.cpp:327)
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <exception>
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

using namespace cltk;

namespace {

thread_local std::string g_err;

char* dupString(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// Runs fn; converts cltk exceptions to their ErrorCode (the CLI's exit code).
template <class F>
int guarded(F&& fn) {
  try {
    fn();
    g_err.clear();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

TEnv tenvOf(const char* tenvJson) {
  if (tenvJson == nullptr || *tenvJson == 0) return TEnv{};
  return tenvFromJson(nlohmann::json::parse(tenvJson));
}

struct Model {
  ModelSpec m;
};
struct KernelH {
  Kernel k;
};

std::vector<double> discOf(const Kernel& k, const ModelSpec& m) {
  // As SimPlan (proj/src/pricing.cpp:207-210).
  std::vector<double> d;
  for (std::int64_t day : k.rows)
    d.push_back(std::exp(-m.rate * static_cast<double>(day) / m.dayCount));
  return d;
}

}  // namespace

extern "C" {

const char* cltkref_last_error(void) { return g_err.c_str(); }
void cltkref_free(void* p) { std::free(p); }

int cltkref_compile_kernel_json(const char* src, const char* tenvJson, int cut,
                                char** out) {
  return guarded([&] {
    ContrPtr c = parseContract(src);
    typeCheckContr(TypeCtx{}, c);
    ILPtr il = compileContract(c);
    if (cut) il = cutPayoff(il);
    Kernel k = reindex(il, tenvOf(tenvJson));
    *out = dupString(kernelToJson(k).dump());
  });
}

// The IL the reference hands to reindex (ilToJson, proj/src/json_io.cpp:203),
// optionally after cutPayoff -- fixtures for the engine's own reindex.
int cltkref_compile_il_json(const char* src, int cut, char** out) {
  return guarded([&] {
    ContrPtr c = parseContract(src);
    typeCheckContr(TypeCtx{}, c);
    ILPtr il = compileContract(c);
    if (cut) il = cutPayoff(il);
    *out = dupString(ilToJson(il).dump());
  });
}

// reindex (proj/src/kernel.cpp:301-303) of an IL in its JSON wire format.
int cltkref_reindex_json(const char* ilJson, const char* tenvJson, char** out) {
  return guarded([&] {
    Kernel k = reindex(ilFromJson(nlohmann::json::parse(ilJson)), tenvOf(tenvJson));
    *out = dupString(kernelToJson(k).dump());
  });
}

int cltkref_kernel_source(const char* kernelJson, char** out) {
  return guarded([&] {
    Kernel k = kernelFromJson(nlohmann::json::parse(kernelJson));
    *out = dupString(emitKernelSource(k));
  });
}

std::uint64_t cltkref_philox_bits(std::uint64_t seed, std::uint64_t path,
                                  std::uint64_t i) {
  return CounterRng(seed, path).bits(i);
}
double cltkref_uniform(std::uint64_t seed, std::uint64_t path,
                       std::uint64_t i) {
  return CounterRng(seed, path).uniform(i);
}
int cltkref_normal(std::uint64_t seed, std::uint64_t path, std::uint64_t i,
                   double* out) {
  return guarded([&] { *out = CounterRng(seed, path).normal(i); });
}
int cltkref_inv_normal_cdf(double p, double* out) {
  return guarded([&] { *out = invNormalCdf(p); });
}
double cltkref_normal_cdf(double x) { return normalCdf(x); }
double cltkref_black_scholes_call(double spot, double strike, double rate,
                                  double vol, double t) {
  return blackScholesCall(spot, strike, rate, vol, t);
}
int cltkref_cholesky(const double* m, int n, double* out) {
  return guarded([&] {
    std::vector<std::vector<double>> a(n, std::vector<double>(n));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) a[i][j] = m[i * n + j];
    auto l = cholesky(a);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) out[i * n + j] = l[i][j];
  });
}

int cltkref_kernel_load(const char* kernelJson, void** out) {
  return guarded([&] {
    auto* h = new KernelH{kernelFromJson(nlohmann::json::parse(kernelJson))};
    *out = h;
  });
}
void cltkref_kernel_free(void* h) { delete static_cast<KernelH*>(h); }
void cltkref_kernel_shape(void* h, std::uint64_t* rows, std::uint64_t* cols) {
  auto* k = static_cast<KernelH*>(h);
  *rows = k->k.rows.size();
  *cols = k->k.cols.size();
}

int cltkref_model_load(const char* modelJson, void** out) {
  return guarded([&] {
    auto* h = new Model{modelFromJson(nlohmann::json::parse(modelJson))};
    *out = h;
  });
}
void cltkref_model_free(void* h) { delete static_cast<Model*>(h); }

// ext_out: [npaths][rows][cols]
int cltkref_simulate_paths(void* kh, void* mh, std::uint64_t seed,
                           std::uint64_t path0, std::uint64_t npaths,
                           double* extOut) {
  return guarded([&] {
    const Kernel& k = static_cast<KernelH*>(kh)->k;
    const ModelSpec& m = static_cast<Model*>(mh)->m;
    std::size_t R = k.rows.size(), C = k.cols.size();
    for (std::uint64_t p = 0; p < npaths; ++p) {
      auto ext = simulatePath(k, m, seed, path0 + p);
      for (std::size_t r = 0; r < R; ++r)
        for (std::size_t c = 0; c < C; ++c)
          extOut[(p * R + r) * C + c] = ext[r][c];
    }
  });
}

int cltkref_disc(void* kh, void* mh, double* out) {
  return guarded([&] {
    auto d = discOf(static_cast<KernelH*>(kh)->k, static_cast<Model*>(mh)->m);
    for (std::size_t i = 0; i < d.size(); ++i) out[i] = d[i];
  });
}

// evalKernel on caller-provided ext [rows][cols] / disc [rows].
int cltkref_eval_kernel(void* kh, const double* ext, const double* disc,
                        std::uint64_t tNow, const char* p1, const char* p2,
                        double* out) {
  return guarded([&] {
    const Kernel& k = static_cast<KernelH*>(kh)->k;
    std::size_t R = k.rows.size(), C = k.cols.size();
    KernelInput in;
    in.tNow = tNow;
    in.ext.assign(R, std::vector<double>(C));
    for (std::size_t r = 0; r < R; ++r)
      for (std::size_t c = 0; c < C; ++c) in.ext[r][c] = ext[r * C + c];
    in.disc.assign(disc, disc + R);
    *out = evalKernel(k, in, p1, p2);
  });
}

// Per-path payoffs exactly as priceAcrossTime computes them
// (proj/src/pricing.cpp:342-358).  out: [npaths][ndays]
int cltkref_path_payoffs(void* kh, void* mh, std::uint64_t seed,
                         std::uint64_t path0, std::uint64_t npaths,
                         const std::uint64_t* days, std::uint64_t ndays,
                         double* out) {
  return guarded([&] {
    const Kernel& k = static_cast<KernelH*>(kh)->k;
    const ModelSpec& m = static_cast<Model*>(mh)->m;
    const Party p1 = k.parties.size() > 0 ? k.parties[0] : "you";
    const Party p2 = k.parties.size() > 1 ? k.parties[1] : "me";
    KernelInput in;
    in.disc = discOf(k, m);
    for (std::uint64_t p = 0; p < npaths; ++p) {
      in.ext = simulatePath(k, m, seed, path0 + p);
      for (std::uint64_t d = 0; d < ndays; ++d) {
        in.tNow = days[d];
        out[p * ndays + d] = evalKernel(k, in, p1, p2);
      }
    }
  });
}

// priceAcrossTime; out_price/out_se: [ndays]
int cltkref_price(void* kh, void* mh, std::uint64_t paths, std::uint64_t seed,
                  const std::uint64_t* days, std::uint64_t ndays,
                  const char* tenvJson, unsigned threads, double* outPrice,
                  double* outSe) {
  return guarded([&] {
    std::vector<std::uint64_t> dv(days, days + ndays);
    auto res = priceAcrossTime(static_cast<KernelH*>(kh)->k,
                               static_cast<Model*>(mh)->m, paths, seed, dv,
                               tenvOf(tenvJson), threads);
    for (std::size_t i = 0; i < res.size(); ++i) {
      outPrice[i] = res[i].price;
      outSe[i] = res[i].stdError;
    }
  });
}

}  // extern "C"
