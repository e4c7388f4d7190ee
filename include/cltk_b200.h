/* cltk_b200.h -- C ABI of the B200 Monte Carlo pricing engine.
 *
 * The drop-in boundary for the reference's pricing path (cltk,
 * arXiv 2108.03076).  Plain pointers and sizes only; no exceptions cross it.
 * Structured inputs use the reference's own wire formats:
 *   kernel  -- kernelToJson        (proj/src/kernel.cpp:620-629)
 *   model   -- the model JSON       (proj/README.md:85-94, modelFromJson
 *                                    proj/src/pricing.cpp:20-43)
 *   tenv    -- tenvToJson           (proj/src/json_io.cpp:305-317)
 * Every entry point returns 0 on success or the reference's ErrorCode
 * (proj/include/cltk/errors.hpp:10-16: 2 parse, 3 type, 4 unsupported,
 * 5 eval); err (may be NULL) receives the reference's message.  Device
 * failures return 4 with a "device: ..." message.
 *
 * Limits that differ from the reference: models of at most 32 assets
 * (CLTK_MAX_ASSETS; the reference has no cap, proj/src/pricing.cpp:217-245);
 * models of 9..32 assets run the NVRTC payoff kernel only (jit = 0 and the
 * QMC mode take at most 8) -- beyond that the call returns 4
 * (UnsupportedError).  At most 2^40 paths per call, and 2^32 in the QMC mode.  The pricing functions never change their inputs;
 * one plan (cltk_plan_*) serves one caller at a time, any number of plans
 * may run concurrently.
 *
 * Entry point                replaces (reference interface)
 * -------------------------  -------------------------------------------------
 * cltk_gpu_price             cltk::priceAcrossTime  proj/include/cltk/pricing.hpp:92-98
 *                            (and priceMC :84-89 with n_days = 1); the pybind
 *                            cltk.price            proj/python/bindings.cpp:103-126
 * cltk_gpu_price_batch       repeated priceAcrossTime over literal instances of one
 *                            template (one path set, like repeated calls with one seed)
 * cltk_plan_*                the same computation split for multi-GPU sharding:
 *                            runParallel's path chunks (proj/src/pricing.cpp:268-286)
 *                            become deterministic chunks any GPU can price.
 * cltk_black_scholes_call    cltk::blackScholesCall proj/include/cltk/pricing.hpp:62-63
 * cltk_debug_*               test hooks: per-path outputs, RNG streams
 *                            (CounterRng proj/include/cltk/pricing.hpp:43-56), the QMC
 *                            generator's Sobol integers
 * cltk_plan_set_fault        test hook: the reference's invNormalCdf domain error
 *                            (proj/src/pricing.cpp:111-113) at a chosen draw
 * cltk_nccl_version          the NCCL the in-process multi-GPU path loads
 */
#ifndef CLTK_B200_H
#define CLTK_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PriceResult (proj/include/cltk/pricing.hpp:65-71) */
typedef struct {
  double price;
  double std_error;
  uint64_t paths;
  uint64_t seed;
  uint64_t valuation_day;
} cltk_price_result;

typedef struct {
  int code;           /* ErrorCode, 0 = ok */
  char message[504];
} cltk_error;

typedef struct cltk_plan cltk_plan;

typedef struct {
  uint32_t n_assets, n_steps, n_thread, n_shared_const, n_inst_const;
  uint32_t n_instances, n_days, n_outputs;
  uint32_t n_shared_ops, n_inst_ops, has_err, block;
  uint64_t kernel_nodes, dag_nodes;
  uint32_t jit; /* 1: the plan runs its NVRTC-generated kernel */
} cltk_plan_info;

/* Chunk partial written by cltk_plan_launch: count, mean, sum of squared
 * deviations, for each output (instance-major, then valuation day). */
typedef struct {
  double n, mean, m2;
} cltk_partial_t;

/* Engine options.  rng: 0 = Philox2x64-10 + Acklam/Halley (the reference's
 * generator; bit-exact per path), 1 = Sobol (Joe-Kuo, 32-bit) + Wichura AS241
 * + Brownian bridge over the drawing days (QMC; seed != 0 applies a
 * per-dimension digital shift).  rewrite: exact OR/AND->min/max rewrite.
 * jit: payoff evaluation -- 0 = bytecode interpreter in the ahead-of-time
 * kernel, 1 = the payoff program compiled to CUDA and built with NVRTC for
 * sm_100a at plan creation (cached by program shape; literals stay kernel
 * data, so new template instances do not recompile; error if NVRTC is
 * unavailable), 2 = NVRTC when available and the program is small, else 0.
 * Both give bit-identical results. */
#define CLTK_MAX_DEVICES 16
typedef struct {
  int device;   /* -1: current */
  int rewrite;  /* default 1 */
  int rng;      /* default 0 */
  int jit;      /* default 0 */
  /* n_devices > 0: the one-shot entry points shard the call over
   * devices[0 .. n_devices) of this process -- a plan per GPU, contiguous
   * equal slices of the deterministic chunks, ONE NCCL all-gather of the
   * chunk partials over NVLink (libnccl.so.2, loaded on first use), the
   * fixed-order combine on devices[0]: bit-identical to one GPU (the
   * reference's thread-count invariance, proj/src/pricing.cpp:268-286).
   * A device listed twice shares its GPU (gathered with device copies).
   * n_devices = 0 and device < 0: $CLTK_DEVICES ("all" or "0,1,...") when
   * set, else the current device. */
  int n_devices;
  int devices[CLTK_MAX_DEVICES];
  /* test builds only: plans carry the fault hook (cltk_plan_set_fault) */
  int fault_inject;
  int reserved[3];
} cltk_options;

const char* cltk_version(void);

/* priceAcrossTime: results[n_days].  `threads` is accepted and ignored (the
 * reference guarantees identical results for any value).  device < 0: the
 * GPUs $CLTK_DEVICES lists (sharded as cltk_options.devices), else the
 * current CUDA device.  The entry points without cltk_options evaluate the
 * payoff as jit = 2 does (NVRTC-generated kernel when NVRTC is available;
 * compiled once per program shape, cached in-process and on disk under
 * $CLTK_JIT_CACHE_DIR or ~/.cache/cltk_b200; bit-identical to the
 * interpreter). */
int cltk_gpu_price(const char* kernel_json, const char* model_json, uint64_t paths,
                   uint64_t seed, const uint64_t* days, size_t n_days, const char* tenv_json,
                   unsigned threads, int device, cltk_price_result* results, cltk_error* err);

/* Template batch: n_instances kernels of one shape (differing only in float
 * literals).  results[n_instances * n_days], instance-major. */
int cltk_gpu_price_batch(const char* const* kernel_jsons, size_t n_instances,
                         const char* model_json, uint64_t paths, uint64_t seed,
                         const uint64_t* days, size_t n_days, const char* tenv_json, int device,
                         cltk_price_result* results, cltk_error* err);
/* cltk_gpu_price_batch with engine options (rng mode, NVRTC payoff kernel). */
int cltk_gpu_price_batch_ex(const char* const* kernel_jsons, size_t n_instances,
                            const char* model_json, uint64_t paths, uint64_t seed,
                            const uint64_t* days, size_t n_days, const char* tenv_json,
                            const cltk_options* opts, cltk_price_result* results,
                            cltk_error* err);

/* Template batch as "template parameters passed as kernel arguments": one
 * kernel and literals[n_instances][n_literals], the values of its float
 * literals (FloatLit nodes, postorder of the kernel JSON tree -- the order
 * cltk_kernel_literals returns) for each instance.  One compile, one path
 * set; results[n_instances * n_days], instance-major. */
int cltk_gpu_price_template(const char* kernel_json, const double* literals, size_t n_instances,
                            size_t n_literals, const char* model_json, uint64_t paths,
                            uint64_t seed, const uint64_t* days, size_t n_days,
                            const char* tenv_json, int device, cltk_price_result* results,
                            cltk_error* err);
/* Host-only: reindex (proj/src/kernel.cpp:301-303, KernelBuilder :14-180) --
 * the IL of a compiled contract in its JSON wire format (ilToJson,
 * proj/src/json_io.cpp:203-255) flattened into the kernel JSON
 * (kernelToJson, proj/src/kernel.cpp:620) every pricing entry point takes,
 * template variables bound from tenv_json.  Malloc'd; free with cltk_free.
 * Errors: ParseError for malformed IL, EvalError for an unbound template
 * variable (proj/include/cltk/errors.hpp:51-54). */
int cltk_reindex(const char* il_json, const char* tenv_json, char** kernel_json, cltk_error* err);
/* Host-only: the kernel's float literals in the order above (*n = count;
 * at most cap values written). */
int cltk_kernel_literals(const char* kernel_json, double* out, size_t cap, size_t* n,
                         cltk_error* err);

/* Everything above with options: literals == NULL prices the kernel alone
 * (n_instances must be 1), else literals[n_instances][n_literals] as in
 * cltk_gpu_price_template.  opts == NULL: defaults. */
int cltk_gpu_price_ex(const char* kernel_json, const double* literals, size_t n_instances,
                      size_t n_literals, const char* model_json, uint64_t paths, uint64_t seed,
                      const uint64_t* days, size_t n_days, const char* tenv_json,
                      const cltk_options* opts, cltk_price_result* results, cltk_error* err);

/* ---- plan API: compile once, launch chunk ranges, combine --------------- */
int cltk_plan_create_ex(const char* kernel_json, const double* literals, size_t n_instances,
                        size_t n_literals, const char* model_json, const uint64_t* days,
                        size_t n_days, const char* tenv_json, const cltk_options* opts,
                        cltk_plan** plan, cltk_error* err);
int cltk_plan_create_template(const char* kernel_json, const double* literals, size_t n_instances,
                              size_t n_literals, const char* model_json, const uint64_t* days,
                              size_t n_days, const char* tenv_json, int device, int rewrite,
                              cltk_plan** plan, cltk_error* err);
int cltk_plan_create(const char* const* kernel_jsons, size_t n_instances, const char* model_json,
                     const uint64_t* days, size_t n_days, const char* tenv_json, int device,
                     int rewrite, cltk_plan** plan, cltk_error* err);
/* cltk_plan_create with engine options (rng mode, NVRTC payoff kernel). */
int cltk_plan_create_batch_ex(const char* const* kernel_jsons, size_t n_instances,
                              const char* model_json, const uint64_t* days, size_t n_days,
                              const char* tenv_json, const cltk_options* opts, cltk_plan** plan,
                              cltk_error* err);
void cltk_plan_destroy(cltk_plan* plan);
int cltk_plan_get_info(const cltk_plan* plan, cltk_plan_info* info);
/* Deterministic chunking of [0, paths): depends only on paths and the
 * plan's output count, so a chunk range priced on any GPU yields the same
 * partials. */
int cltk_plan_chunking(const cltk_plan* plan, uint64_t paths, uint64_t* chunk_paths,
                       uint64_t* n_chunks);
/* Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream):
 * price chunks [c0, c1) into partials_dev[c][out] (device memory of
 * n_chunks * n_outputs cltk_partial_t).  A plan's launches and its finalize
 * must be ordered (one stream, or synchronised by the caller): they share
 * the plan's chunk scheduler counter and device error word.  Concurrent
 * callers use one plan each. */
int cltk_plan_launch(cltk_plan* plan, uint64_t paths, uint64_t seed, uint64_t c0, uint64_t c1,
                     void* partials_dev, void* stream, cltk_error* err);
/* Fixed-order combine of partials_dev[0, n_chunks), synchronous read-back,
 * device error check.  results[n_instances * n_days]. */
int cltk_plan_finalize(cltk_plan* plan, uint64_t paths, uint64_t seed, const void* partials_dev,
                       const uint64_t* days, size_t n_days, void* stream,
                       cltk_price_result* results, cltk_error* err);
/* Device error word (min over paths of path << 24 | site; ~0 = none): read
 * it, and overwrite it (e.g. with the MIN over ranks) before finalize. */
int cltk_plan_error_word(cltk_plan* plan, void* stream, uint64_t* word);
int cltk_plan_set_error_word(cltk_plan* plan, void* stream, uint64_t word);
/* Test hook: plans created with cltk_options.fault_inject = 1 (Philox mode)
 * force the uniform of draw `draw` of path `path` to exactly 1.0 in later
 * launches -- the reference's reachable invNormalCdf domain error
 * (proj/src/pricing.cpp:100-103,111-113) at a chosen place.  path = ~0: none. */
int cltk_plan_set_fault(cltk_plan* plan, uint64_t path, uint32_t draw, cltk_error* err);
/* The NCCL the multi-GPU path loads: *version = ncclGetVersion's code, or
 * an error when libnccl.so.2 cannot be loaded. */
int cltk_nccl_version(int* version, cltk_error* err);
/* Host-only: compile (no device needed) and return the program listing --
 * the engine's analogue of emitKernelSource (proj/src/kernel.cpp:407). */
int cltk_compile_listing(const char* const* kernel_jsons, size_t n_instances,
                         const char* model_json, const uint64_t* days, size_t n_days,
                         const char* tenv_json, int rewrite, int rng, char** json,
                         cltk_error* err);
/* Host-only: the CUDA source the NVRTC mode generates for this program
 * (literals: an optional [n_instances][n_literals] table as in
 * cltk_plan_create_ex; malloc'd; free with cltk_free).  Replaces no reference interface (the
 * reference interprets its kernel tree, proj/src/kernel.cpp:229-310). */
int cltk_jit_source(const char* kernel_json, const double* literals, size_t n_instances,
                    size_t n_literals, const char* model_json, const uint64_t* days,
                    size_t n_days, const char* tenv_json, int rewrite, int rng, char** source,
                    cltk_error* err);
/* Host-only: NVRTC-compile a generated source for sm_100a (no device needed);
 * cubin size and the compiler log (malloc'd). */
int cltk_jit_compile(const char* source, uint64_t* cubin_bytes, char** log, cltk_error* err);
/* Program listing (JSON, malloc'd; free with cltk_free). */
int cltk_plan_dump(const cltk_plan* plan, char** json);
void cltk_free(void* p);

/* ---- test hooks (same device code as the pricing kernel) --------------- */
/* Per-path outputs [npaths][n_outputs]; spots/normals [npaths][n_steps][n_assets]
 * (any may be NULL).  Host buffers. */
int cltk_debug_paths(cltk_plan* plan, uint64_t seed, uint64_t path0, uint64_t npaths,
                     double* outputs, double* spots, double* normals, uint64_t* error_word,
                     cltk_error* err);
/* Philox bits / uniforms / normals of stream (seed, path), indices [i0, i0+n). */
int cltk_debug_rng(int device, uint64_t seed, uint64_t path, uint64_t i0, uint64_t n,
                   uint64_t* bits, double* uniforms, double* normals, cltk_error* err);
/* Device exp / log / erfc / invNormalCdf (fn = 0..3) of x[n] (host buffers):
 * the engine's bit-exact restatements of glibc's routines; fn = 4: the
 * engine's bounded-range division of the pairs (x[2i], x[2i+1]) (n even, the
 * quotient written to both slots); fn = 5: its -x / sqrt(2.0). */
int cltk_debug_math(int device, int fn, const double* x, uint64_t n, double* out,
                    cltk_error* err);
/* QMC generator: the 32-bit Sobol integers (Joe-Kuo direction numbers, gray
 * code) of points [n0, n0 + n), dimensions [d0, d0 + nd), out[n][nd] (host
 * buffer), from the device code the QMC path kernel runs; aligned = 1 uses
 * its warp-cooperative skip-ahead (n0 a multiple of 32), 0 the per-point one. */
int cltk_debug_sobol(int device, uint64_t n0, uint64_t n, uint32_t d0, uint32_t nd, int aligned,
                     uint32_t* out, cltk_error* err);
/* Measured DFMA throughput (TFLOP/s) over `iters` iterations. */
int cltk_fp64_peak(int device, int iters, double* tflops, double* seconds, cltk_error* err);

double cltk_black_scholes_call(double spot, double strike, double rate, double vol,
                               double t_years);

#ifdef __cplusplus
}
#endif
#endif
