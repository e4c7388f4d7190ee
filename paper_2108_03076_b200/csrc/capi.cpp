// extern "C" boundary (include/cltk_b200.h).  Converts exceptions to the
// reference's ErrorCode + message; no exception crosses the ABI.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>

#include "../../include/cltk_b200.h"
#include "cltk_b200.hpp"
#include "compiler.hpp"
#include "jit.hpp"
#include "engine_launch.hpp"
#include "nccl_comm.hpp"

using namespace cltk::b200;

struct cltk_plan {
  std::unique_ptr<Plan> plan;
  std::vector<std::unique_ptr<Kernel>> kernels;
};

namespace {

void setErr(cltk_error* err, int code, const char* msg) {
  if (!err) return;
  err->code = code;
  std::strncpy(err->message, msg, sizeof(err->message) - 1);
  err->message[sizeof(err->message) - 1] = 0;
}

template <class F>
int guarded(cltk_error* err, F&& fn) {
  try {
    fn();
    setErr(err, 0, "");
    return 0;
  } catch (const Error& e) {
    setErr(err, static_cast<int>(e.code()), e.what());
    return static_cast<int>(e.code());
  } catch (const std::bad_alloc&) {
    setErr(err, 4, "out of host memory");
    return 4;
  } catch (const std::exception& e) {
    setErr(err, 4, e.what());
    return 4;
  }
}

void toC(const std::vector<PriceResult>& r, cltk_price_result* out) {
  for (std::size_t i = 0; i < r.size(); ++i) {
    out[i].price = r[i].price;
    out[i].std_error = r[i].stdError;
    out[i].paths = r[i].paths;
    out[i].seed = r[i].seed;
    out[i].valuation_day = r[i].valuationDay;
  }
}

TEnv tenvOf(const char* j) { return (j && *j) ? tenvFromJson(j) : TEnv{}; }

}  // namespace

namespace {
// Plan-cache key of a one-shot call: every wire input, the options and the
// resolved device (engine.cpp priceCached).
struct KeyBuilder {
  std::string key;
  void add(const void* p, size_t n) { key.append(static_cast<const char*>(p), n); }
  void str(const char* s) {
    const size_t n = s ? std::strlen(s) : 0;
    add(&n, sizeof n);
    if (n) add(s, n);
  }
  template <class T>
  void val(const T& v) { add(&v, sizeof v); }
};
int resolvedDevice(int device) {
  if (device >= 0) return device;
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
std::vector<int> resolvedDevices(const RunOptions& opt) {
  std::vector<int> v = resolveDevices(opt);
  for (int& d : v) d = resolvedDevice(d);
  return v;
}
}  // namespace

extern "C" {

const char* cltk_version(void) { return "cltk-b200 0.1 (sm_100a)"; }

void cltk_free(void* p) { std::free(p); }

double cltk_black_scholes_call(double spot, double strike, double rate, double vol, double t) {
  return blackScholesCall(spot, strike, rate, vol, t);
}


int cltk_gpu_price(const char* kernel_json, const char* model_json, uint64_t paths, uint64_t seed,
                   const uint64_t* days, size_t n_days, const char* tenv_json, unsigned threads,
                   int device, cltk_price_result* results, cltk_error* err) {
  return guarded(err, [&] {
    if (paths == 0) throw EvalError("path count must be positive");
    std::vector<uint64_t> d(days, days + n_days);
    RunOptions opt;
    opt.device = device;
    (void)threads;
    KeyBuilder kb;
    kb.str("cltk_gpu_price");
    kb.str(kernel_json);
    kb.str(model_json);
    kb.str(tenv_json);
    kb.add(d.data(), d.size() * sizeof(uint64_t));
    auto r = priceCached(
        kb.key,
        [&](int dev) {
          const Kernel k = kernelFromWire(kernel_json);
          RunOptions o = opt;
          o.device = resolvedDevice(dev);
          return std::make_unique<Plan>(std::vector<const Kernel*>{&k},
                                        modelFromJson(model_json), d, tenvOf(tenv_json), o);
        },
        resolvedDevices(opt), paths, seed, d);
    toC(r, results);
  });
}

int cltk_gpu_price_batch(const char* const* kernel_jsons, size_t n_instances,
                         const char* model_json, uint64_t paths, uint64_t seed,
                         const uint64_t* days, size_t n_days, const char* tenv_json, int device,
                         cltk_price_result* results, cltk_error* err) {
  return guarded(err, [&] {
    if (paths == 0) throw EvalError("path count must be positive");
    std::vector<Kernel> ks;
    ks.reserve(n_instances);
    for (size_t i = 0; i < n_instances; ++i) ks.push_back(kernelFromWire(kernel_jsons[i]));
    std::vector<const Kernel*> ptrs;
    for (auto& k : ks) ptrs.push_back(&k);
    ModelSpec m = modelFromJson(model_json);
    std::vector<uint64_t> d(days, days + n_days);
    RunOptions opt;
    opt.device = device;
    toC(priceBatch(ptrs, m, paths, seed, d, tenvOf(tenv_json), opt), results);
  });
}

int cltk_gpu_price_template(const char* kernel_json, const double* literals, size_t n_instances,
                            size_t n_literals, const char* model_json, uint64_t paths,
                            uint64_t seed, const uint64_t* days, size_t n_days,
                            const char* tenv_json, int device, cltk_price_result* results,
                            cltk_error* err) {
  return guarded(err, [&] {
    if (paths == 0) throw EvalError("path count must be positive");
    Kernel k = kernelFromWire(kernel_json);
    ModelSpec m = modelFromJson(model_json);
    RunOptions opt;
    opt.device = device;
    toC(priceTemplate(k, literals, n_instances, n_literals, m, paths, seed,
                      std::vector<uint64_t>(days, days + n_days), tenvOf(tenv_json), opt),
        results);
  });
}

int cltk_kernel_literals(const char* kernel_json, double* out, size_t cap, size_t* n,
                         cltk_error* err) {
  return guarded(err, [&] {
    std::vector<double> v = kernelFloatLiterals(kernelFromWire(kernel_json));
    *n = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  });
}

int cltk_plan_create_template(const char* kernel_json, const double* literals, size_t n_instances,
                              size_t n_literals, const char* model_json, const uint64_t* days,
                              size_t n_days, const char* tenv_json, int device, int rewrite,
                              cltk_plan** out, cltk_error* err) {
  return guarded(err, [&] {
    auto p = std::make_unique<cltk_plan>();
    p->kernels.push_back(std::make_unique<Kernel>(kernelFromWire(kernel_json)));
    ModelSpec m = modelFromJson(model_json);
    RunOptions opt;
    opt.device = device;
    opt.rewrite = rewrite != 0;
    p->plan = std::make_unique<Plan>(*p->kernels[0], literals, n_instances, n_literals, m,
                                     std::vector<uint64_t>(days, days + n_days),
                                     tenvOf(tenv_json), opt);
    *out = p.release();
  });
}

namespace {
RunOptions optionsOf(const cltk_options* o) {
  RunOptions r;
  if (o) {
    r.device = o->device;
    r.rewrite = o->rewrite != 0;
    r.rng = o->rng;
    r.jit = o->jit;
    if (o->n_devices < 0 || o->n_devices > CLTK_MAX_DEVICES)
      throw UnsupportedError("cltk_options: n_devices out of range");
    r.devices.assign(o->devices, o->devices + o->n_devices);
    for (int d : r.devices)
      if (d < 0) throw UnsupportedError("cltk_options: negative device id");
    r.faultInject = o->fault_inject != 0;
  }
  return r;
}
}  // namespace

int cltk_gpu_price_ex(const char* kernel_json, const double* literals, size_t n_instances,
                      size_t n_literals, const char* model_json, uint64_t paths, uint64_t seed,
                      const uint64_t* days, size_t n_days, const char* tenv_json,
                      const cltk_options* opts, cltk_price_result* results, cltk_error* err) {
  return guarded(err, [&] {
    if (paths == 0) throw EvalError("path count must be positive");
    std::vector<uint64_t> d(days, days + n_days);
    const RunOptions opt = optionsOf(opts);
    KeyBuilder kb;
    kb.str("cltk_gpu_price_ex");
    kb.str(kernel_json);
    kb.str(model_json);
    kb.str(tenv_json);
    kb.add(d.data(), d.size() * sizeof(uint64_t));
    kb.val(opt.rewrite);
    kb.val(opt.rng);
    kb.val(opt.jit);
    kb.val(n_instances);
    kb.val(n_literals);
    if (literals) kb.add(literals, n_instances * n_literals * sizeof(double));
    auto r = priceCached(
        kb.key,
        [&](int dev) {
          RunOptions o = opt;
          o.device = dev;
          const Kernel k = kernelFromWire(kernel_json);
          std::vector<double> own;
          const double* lit = literals;
          size_t ni = n_instances, nl = n_literals;
          if (!lit) {
            own = kernelFloatLiterals(k);
            lit = own.data();
            ni = 1;
            nl = own.size();
          }
          return std::make_unique<Plan>(k, lit, ni, nl, modelFromJson(model_json), d,
                                        tenvOf(tenv_json), o);
        },
        resolvedDevices(opt), paths, seed, d);
    toC(r, results);
  });
}

int cltk_plan_create_ex(const char* kernel_json, const double* literals, size_t n_instances,
                        size_t n_literals, const char* model_json, const uint64_t* days,
                        size_t n_days, const char* tenv_json, const cltk_options* opts,
                        cltk_plan** out, cltk_error* err) {
  return guarded(err, [&] {
    auto p = std::make_unique<cltk_plan>();
    p->kernels.push_back(std::make_unique<Kernel>(kernelFromWire(kernel_json)));
    std::vector<double> own;
    if (!literals) {
      own = kernelFloatLiterals(*p->kernels[0]);
      literals = own.data();
      n_instances = 1;
      n_literals = own.size();
    }
    ModelSpec m = modelFromJson(model_json);
    p->plan = std::make_unique<Plan>(*p->kernels[0], literals, n_instances, n_literals, m,
                                     std::vector<uint64_t>(days, days + n_days),
                                     tenvOf(tenv_json), optionsOf(opts));
    *out = p.release();
  });
}

int cltk_plan_create(const char* const* kernel_jsons, size_t n_instances, const char* model_json,
                     const uint64_t* days, size_t n_days, const char* tenv_json, int device,
                     int rewrite, cltk_plan** out, cltk_error* err) {
  return guarded(err, [&] {
    auto p = std::make_unique<cltk_plan>();
    std::vector<const Kernel*> ptrs;
    for (size_t i = 0; i < n_instances; ++i) {
      p->kernels.push_back(std::make_unique<Kernel>(kernelFromWire(kernel_jsons[i])));
      ptrs.push_back(p->kernels.back().get());
    }
    ModelSpec m = modelFromJson(model_json);
    std::vector<uint64_t> d(days, days + n_days);
    RunOptions opt;
    opt.device = device;
    opt.rewrite = rewrite != 0;
    p->plan = std::make_unique<Plan>(ptrs, m, d, tenvOf(tenv_json), opt);
    *out = p.release();
  });
}

int cltk_plan_create_batch_ex(const char* const* kernel_jsons, size_t n_instances,
                              const char* model_json, const uint64_t* days, size_t n_days,
                              const char* tenv_json, const cltk_options* opts, cltk_plan** out,
                              cltk_error* err) {
  return guarded(err, [&] {
    auto p = std::make_unique<cltk_plan>();
    std::vector<const Kernel*> ptrs;
    for (size_t i = 0; i < n_instances; ++i) {
      p->kernels.push_back(std::make_unique<Kernel>(kernelFromWire(kernel_jsons[i])));
      ptrs.push_back(p->kernels.back().get());
    }
    ModelSpec m = modelFromJson(model_json);
    p->plan = std::make_unique<Plan>(ptrs, m, std::vector<uint64_t>(days, days + n_days),
                                     tenvOf(tenv_json), optionsOf(opts));
    *out = p.release();
  });
}

int cltk_gpu_price_batch_ex(const char* const* kernel_jsons, size_t n_instances,
                            const char* model_json, uint64_t paths, uint64_t seed,
                            const uint64_t* days, size_t n_days, const char* tenv_json,
                            const cltk_options* opts, cltk_price_result* results,
                            cltk_error* err) {
  return guarded(err, [&] {
    std::vector<Kernel> ks;
    ks.reserve(n_instances);
    for (size_t i = 0; i < n_instances; ++i) ks.push_back(kernelFromWire(kernel_jsons[i]));
    std::vector<const Kernel*> ptrs;
    for (auto& k : ks) ptrs.push_back(&k);
    ModelSpec m = modelFromJson(model_json);
    toC(priceBatch(ptrs, m, paths, seed, std::vector<uint64_t>(days, days + n_days),
                   tenvOf(tenv_json), optionsOf(opts)),
        results);
  });
}

void cltk_plan_destroy(cltk_plan* plan) { delete plan; }

int cltk_plan_get_info(const cltk_plan* plan, cltk_plan_info* info) {
  PlanInfo i = plan->plan->info();
  static_assert(sizeof(PlanInfo) == sizeof(cltk_plan_info), "info layout");
  std::memcpy(info, &i, sizeof i);
  return 0;
}

int cltk_plan_chunking(const cltk_plan* plan, uint64_t paths, uint64_t* chunk_paths,
                       uint64_t* n_chunks) {
  plan->plan->chunking(paths, chunk_paths, n_chunks);
  return 0;
}

int cltk_plan_launch(cltk_plan* plan, uint64_t paths, uint64_t seed, uint64_t c0, uint64_t c1,
                     void* partials_dev, void* stream, cltk_error* err) {
  return guarded(err, [&] { plan->plan->launch(paths, seed, c0, c1, partials_dev, stream); });
}

int cltk_plan_finalize(cltk_plan* plan, uint64_t paths, uint64_t seed, const void* partials_dev,
                       const uint64_t* days, size_t n_days, void* stream,
                       cltk_price_result* results, cltk_error* err) {
  return guarded(err, [&] {
    auto r = plan->plan->finalize(paths, seed, partials_dev, stream);
    if (n_days)
      for (std::size_t i = 0; i < r.size(); ++i) r[i].valuationDay = days[i % n_days];
    toC(r, results);
  });
}

int cltk_plan_set_fault(cltk_plan* plan, uint64_t path, uint32_t draw, cltk_error* err) {
  return guarded(err, [&] { plan->plan->setFault(path, draw); });
}

int cltk_nccl_version(int* version, cltk_error* err) {
  return guarded(err, [&] {
    std::string info;
    if (!ncclAvailable(&info)) throw UnsupportedError("multi-GPU: " + info);
    *version = std::atoi(info.c_str() + 5);  // "nccl <code>"
  });
}

int cltk_debug_sobol(int device, uint64_t n0, uint64_t n, uint32_t d0, uint32_t nd, int aligned,
                     uint32_t* out, cltk_error* err) {
  return guarded(err, [&] { debugSobol(device, n0, n, d0, nd, aligned != 0, out); });
}

int cltk_plan_error_word(cltk_plan* plan, void* stream, uint64_t* word) {
  cltk_error e;
  return guarded(&e, [&] { *word = planErrorWord(*plan->plan, stream); });
}

int cltk_plan_set_error_word(cltk_plan* plan, void* stream, uint64_t word) {
  cltk_error e;
  return guarded(&e, [&] { planSetErrorWord(*plan->plan, stream, word); });
}

int cltk_debug_paths(cltk_plan* plan, uint64_t seed, uint64_t path0, uint64_t npaths,
                     double* outputs, double* spots, double* normals, uint64_t* error_word,
                     cltk_error* err) {
  return guarded(err, [&] {
    uint64_t w = debugPaths(*plan->plan, seed, path0, npaths, outputs, spots, normals);
    if (error_word) *error_word = w;
  });
}

int cltk_debug_rng(int device, uint64_t seed, uint64_t path, uint64_t i0, uint64_t n,
                   uint64_t* bits, double* uniforms, double* normals, cltk_error* err) {
  return guarded(err, [&] { debugRng(device, seed, path, i0, n, bits, uniforms, normals); });
}

int cltk_debug_math(int device, int fn, const double* x, uint64_t n, double* out,
                    cltk_error* err) {
  return guarded(err, [&] { debugMath(device, fn, x, n, out); });
}

int cltk_fp64_peak(int device, int iters, double* tflops, double* seconds, cltk_error* err) {
  return guarded(err, [&] { *tflops = fp64Peak(device, iters, seconds); });
}

int cltk_compile_listing(const char* const* kernel_jsons, size_t n_instances,
                         const char* model_json, const uint64_t* days, size_t n_days,
                         const char* tenv_json, int rewrite, int rng, char** json,
                         cltk_error* err) {
  return guarded(err, [&] {
    std::vector<Kernel> ks;
    ks.reserve(n_instances);
    for (size_t i = 0; i < n_instances; ++i) ks.push_back(kernelFromWire(kernel_jsons[i]));
    std::vector<const Kernel*> ptrs;
    for (auto& k : ks) ptrs.push_back(&k);
    if (ptrs.empty()) throw EvalError("no kernel instances");
    ModelSpec m = modelFromJson(model_json);
    SimPlanHost sp = buildSimPlan(*ptrs[0], m, static_cast<uint32_t>(rng));
    TEnv t = tenvOf(tenv_json);
    for (const auto& v : ptrs[0]->tvars) (void)t.lookup(v);
    CompileOptions co;
    co.rewrite = rewrite != 0;
    CompiledProgram P = compileProgram(ptrs, sp, std::vector<uint64_t>(days, days + n_days), co);
    const std::string listing = programListing(P);
    char* p = static_cast<char*>(std::malloc(listing.size() + 1));
    std::memcpy(p, listing.c_str(), listing.size() + 1);
    *json = p;
  });
}

int cltk_jit_source(const char* kernel_json, const double* literals, size_t n_instances,
                    size_t n_literals, const char* model_json, const uint64_t* days,
                    size_t n_days, const char* tenv_json, int rewrite, int rng, char** source,
                    cltk_error* err) {
  return guarded(err, [&] {
    Kernel k = kernelFromWire(kernel_json);
    ModelSpec m = modelFromJson(model_json);
    SimPlanHost sp = buildSimPlan(k, m, static_cast<uint32_t>(rng));
    TEnv t = tenvOf(tenv_json);
    for (const auto& v : k.tvars) (void)t.lookup(v);
    CompileOptions co;
    co.rewrite = rewrite != 0;
    LiteralTable lits;
    if (literals) {
      lits.nInst = n_instances;
      lits.nOcc = n_literals;
      lits.values.assign(literals, literals + n_instances * n_literals);
    } else {
      lits.values = kernelFloatLiterals(k);
      lits.nInst = 1;
      lits.nOcc = lits.values.size();
    }
    CompiledProgram P =
        compileProgram(k, lits, sp, std::vector<uint64_t>(days, days + n_days), co);
    const std::string src = jitSource(P);
    char* p = static_cast<char*>(std::malloc(src.size() + 1));
    std::memcpy(p, src.c_str(), src.size() + 1);
    *source = p;
  });
}

int cltk_jit_compile(const char* source, uint64_t* cubin_bytes, char** log, cltk_error* err) {
  return guarded(err, [&] {
    std::string lg;
    *cubin_bytes = jitCompileOnly(source, &lg);
    char* p = static_cast<char*>(std::malloc(lg.size() + 1));
    std::memcpy(p, lg.c_str(), lg.size() + 1);
    *log = p;
  });
}

int cltk_reindex(const char* il_json, const char* tenv_json, char** kernel_json, cltk_error* err) {
  return guarded(err, [&] {
    const std::string s = kernelToJsonString(kernelFromIL(il_json, tenvOf(tenv_json)));
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    *kernel_json = p;
  });
}

int cltk_plan_dump(const cltk_plan* plan, char** json) {
  std::string s = plan->plan->dump();
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  *json = p;
  return 0;
}

}  // extern "C"
