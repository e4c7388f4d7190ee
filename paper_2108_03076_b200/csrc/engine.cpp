// Host orchestration of the B200 engine: plan upload, deterministic chunking,
// launches, fixed-order combine, error word -> reference exception.
// The reference pricing functions (priceMC / priceAcrossTime,
// proj/src/pricing.cpp:318-371) are re-implemented on top of it with the
// same argument meaning and error behaviour.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "cltk_b200.hpp"
#include "compiler.hpp"
#include "engine_launch.hpp"
#include "jit.hpp"
#include "nccl_comm.hpp"

// simulate_qmc (engine_device.cuh) reads the step header as two 16-byte words
static_assert(offsetof(cltk_step_hdr, draws) == 0 && offsetof(cltk_step_hdr, br_begin) == 12 &&
                  offsetof(cltk_step_hdr, br_end) == 16 && offsetof(cltk_step_hdr, br_emit) == 20 &&
                  sizeof(cltk_step_hdr) == 32,
              "step header layout");

namespace cltk {
namespace b200 {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Plan buffers come from the device's stream-ordered pool with an unbounded
// release threshold: a one-shot call's frees return memory to the pool
// instead of unmapping it (cudaFree stalled single calls by 50-500 ms).
void* devMalloc(size_t bytes) {
  static std::mutex mu;
  static bool configured[64] = {};
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && !configured[dev]) {
      cudaMemPool_t pool;
      ck(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
      uint64_t keep = ~0ULL;
      ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep),
         "cudaMemPoolSetAttribute");
      configured[dev] = true;
    }
  }
  void* p = nullptr;
  ck(cudaMallocAsync(&p, bytes, 0), "cudaMallocAsync");
  ck(cudaStreamSynchronize(0), "cudaStreamSynchronize");  // usable from any stream
  return p;
}
void devFree(void* p) {
  if (p) cudaFreeAsync(p, 0);
}


constexpr uint64_t kMaxChunks = 1ULL << 20;

// The device step records (engine_types.h StepRef): header + A, B, S of the
// plan's assets, padded to an even count.
std::vector<unsigned char> packSteps(const std::vector<cltk_step>& steps, uint32_t nAssets) {
  const int na = nAssets ? static_cast<int>(nAssets) : 1;
  const size_t stride = stepStride(na), pad = static_cast<size_t>(stepPad(na));
  std::vector<unsigned char> out(steps.size() * stride, 0);
  for (size_t s = 0; s < steps.size(); ++s) {
    const cltk_step& st = steps[s];
    const cltk_step_hdr h{st.draws,  st.code_begin, st.code_end,  st.br_begin,
                          st.br_end, st.br_emit,    st.jit_class, st.draw_window};
    unsigned char* b = out.data() + s * stride;
    std::memcpy(b, &h, sizeof h);
    double* a = reinterpret_cast<double*>(b + sizeof h);
    for (int j = 0; j < na; ++j) {
      a[j] = st.A[j];
      a[pad + j] = st.B[j];
      a[2 * pad + j] = st.S[j];
    }
  }
  return out;
}

// Host staging of a plan's arrays, each 256-byte aligned in one block.
struct Staging {
  std::vector<char> bytes;
  template <class T>
  size_t add(const std::vector<T>& v) {
    const size_t o = (bytes.size() + 255) / 256 * 256;
    bytes.resize(o + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(bytes.data() + o, v.data(), v.size() * sizeof(T));
    return o;
  }
};

// Philox2x64-10 on the host (QMC digital shifts only).
uint64_t philoxHost(uint64_t key, uint64_t c0, uint64_t c1) {
  for (int r = 0; r < 10; ++r) {
    const unsigned __int128 prod = static_cast<unsigned __int128>(0xD2B74407B1CE6E93ULL) * c0;
    c0 = static_cast<uint64_t>(prod >> 64) ^ key ^ c1;
    c1 = static_cast<uint64_t>(prod);
    key += 0x9E3779B97F4A7C15ULL;
  }
  return c0 ^ c1;
}
constexpr uint64_t kPartialBudget = 1ULL << 30;  // bytes of chunk partials
constexpr size_t kJitAutoMaxOps = 4096;          // JIT_AUTO: larger programs stay interpreted

}  // namespace

extern const uint32_t kSobolDims;  // sobol_table.cpp (generated)
extern const uint32_t kSobolV[];

namespace {
// The QMC direction numbers (and the 5-bit XOR table of the warp-cooperative
// skip-ahead), uploaded once per device and kept for the process.
struct SobolTables {
  const uint32_t* V = nullptr;
  const uint32_t* T5 = nullptr;
};
const SobolTables& sobolTables(int dev) {
  static std::mutex mu;
  static auto& tabs = *new std::map<int, SobolTables>();
  std::lock_guard<std::mutex> lock(mu);
  auto it = tabs.find(dev);
  if (it != tabs.end()) return it->second;
  std::vector<uint32_t> V(kSobolV, kSobolV + kSobolDims * 32), T5(kSobolDims * 32);
  for (uint32_t d = 0; d < kSobolDims; ++d)
    for (uint32_t g = 0; g < 32; ++g) {
      uint32_t x = 0;
      for (uint32_t k = 0; k < 5; ++k)
        if ((g >> k) & 1u) x ^= V[d * 32 + k];
      T5[d * 32 + g] = x;
    }
  void* p = nullptr;
  ck(cudaMalloc(&p, (V.size() + T5.size()) * sizeof(uint32_t)), "cudaMalloc");
  ck(cudaMemcpy(p, V.data(), V.size() * sizeof(uint32_t), cudaMemcpyHostToDevice), "H2D");
  ck(cudaMemcpy(static_cast<uint32_t*>(p) + V.size(), T5.data(), T5.size() * sizeof(uint32_t),
                cudaMemcpyHostToDevice),
     "H2D");
  ck(cudaStreamSynchronize(0), "cudaStreamSynchronize");  // (pageable copies: DMA landed)
  SobolTables t{static_cast<const uint32_t*>(p), static_cast<const uint32_t*>(p) + V.size()};
  return tabs.emplace(dev, t).first->second;
}
}  // namespace

struct PlanImpl {
  CompiledProgram prog;
  uint32_t* sobolShift = nullptr;  // device [kSobolDims], for shiftSeed
  uint64_t shiftSeed = 0;
  DevPlan dev{};
  int device = 0;
  int sms = 0;
  std::vector<void*> owned;
  unsigned long long* errKey = nullptr;
  unsigned long long* chunkCounter = nullptr;
  cltk_partial* combined = nullptr;  // [n_out]
  double* accScratch = nullptr;
  size_t accScratchBlocks = 0;
  cltk_partial* ownPartials = nullptr;  // used by the one-shot entry points
  uint64_t ownPartialsChunks = 0;
  size_t smem = 0;
  bool accInSmem = true;
  int blocksPerSm = 0;
  uint32_t nOut = 0;
  const void* jitFn = nullptr;  // NVRTC kernel (cudaKernel_t) or null: interpreter
  uint64_t drawsPerPath = 0;    // normals per path (chunk sizing)
  uint32_t streamPeriod = 1;    // ppt is a multiple of it (engine_types.h streamPeriod)
  bool fault = false;           // test build (RunArgs fault hook compiled in)
  uint64_t faultPath = ~0ULL;
  uint32_t faultDraw = 0;

  ~PlanImpl() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaDeviceSynchronize();  // no launch of this plan may still be reading its buffers
    for (void* p : owned) devFree(p);
    devFree(accScratch);
    devFree(ownPartials);
    cudaSetDevice(cur);
  }

  struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) {
      cudaGetDevice(&prev);
      if (prev != d) ck(cudaSetDevice(d), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
  };
};

Plan::Plan(const std::vector<const Kernel*>& instances, const ModelSpec& model,
           const std::vector<uint64_t>& days, const TEnv& tenv, const RunOptions& opt)
    : impl_(new PlanImpl) {
  if (instances.empty()) throw EvalError("no kernel instances");
  // Reference order of checks: SimPlan ctor, then the tenv lookups
  // (proj/src/pricing.cpp:335-338); then the batch shape check.
  (void)buildSimPlan(*instances[0], model);
  for (const auto& v : instances[0]->tvars) (void)tenv.lookup(v);
  LiteralTable t = literalTableFromInstances(instances);
  init(*instances[0], &t, model, days, tenv, opt);
}

Plan::Plan(const Kernel& templ, const double* literals, std::size_t nInstances, std::size_t nLits,
           const ModelSpec& model, const std::vector<uint64_t>& days, const TEnv& tenv,
           const RunOptions& opt)
    : impl_(new PlanImpl) {
  LiteralTable t;
  t.nInst = nInstances;
  t.nOcc = nLits;
  t.values.assign(literals, literals + nInstances * nLits);
  init(templ, &t, model, days, tenv, opt);
}

std::vector<double> kernelFloatLiterals(const Kernel& k) { return kernelLiterals(k); }

void Plan::init(const Kernel& k, const void* litsv, const ModelSpec& model,
                const std::vector<uint64_t>& days, const TEnv& tenv, const RunOptions& opt) {
  const LiteralTable& lits = *static_cast<const LiteralTable*>(litsv);
  PlanImpl& I = *impl_;
  if (opt.rng != 0 && opt.rng != 1) throw UnsupportedError("unknown rng mode");
  SimPlanHost sp = buildSimPlan(k, model, static_cast<uint32_t>(opt.rng));
  for (const auto& v : k.tvars) (void)tenv.lookup(v);
  CompileOptions co;
  co.rewrite = opt.rewrite;
  I.prog = compileProgram(k, lits, sp, days, co);
  I.nOut = I.prog.header.n_instances * I.prog.header.n_days;
  for (const cltk_step& st : I.prog.steps)
    if (st.draws == 1) I.drawsPerPath += I.prog.header.n_assets;
  // Philox draw indices are 32-bit on the device (engine_device.cuh philox_keyed32)
  if (static_cast<uint64_t>(I.prog.header.n_steps) * std::max<uint32_t>(1, I.prog.header.n_assets) >=
      (1ULL << 32))
    throw UnsupportedError("more than 2^32 normal draws per path");
  // Philox normal streams (engine_types.h streamPeriod): slots per path = steps x assets
  I.streamPeriod = I.prog.header.stream
                       ? streamPeriod(I.prog.header.n_steps * std::max<uint32_t>(1, I.prog.header.n_assets),
                                      I.prog.header.n_assets)
                       : 1;
  if (opt.jit < 0 || opt.jit > 2) throw UnsupportedError("unknown jit mode");
  if (opt.faultInject && I.prog.header.rng != CLTK_RNG_PHILOX)
    throw UnsupportedError("fault injection: Philox mode only");
  I.fault = opt.faultInject;
  I.prog.faultBuild = opt.faultInject;
  std::string jitSrc;
  // jitSource rewrites the header's register window and the steps' classes:
  // JIT_AUTO keeps the interpreter's copy in case NVRTC or the module load fails
  std::vector<cltk_step> interpSteps;
  std::vector<double> interpInst, interpShared;  // (jitSource may append reciprocals)
  cltk_plan_header interpHdr{};
  // models of more than CLTK_AOT_MAX_ASSETS assets have no ahead-of-time kernel
  const bool bigModel = I.prog.header.n_assets > CLTK_AOT_MAX_ASSETS;
  if (bigModel && opt.jit == JIT_OFF)
    throw UnsupportedError("models of more than " + std::to_string(CLTK_AOT_MAX_ASSETS) +
                           " assets need the NVRTC payoff kernel (jit)");
  if (opt.jit != JIT_OFF) {
    std::string why;
    bool use = jitAvailable(&why);
    if (use && opt.jit == JIT_AUTO && !bigModel && jitOpCount(I.prog) > kJitAutoMaxOps) use = false;
    if (!use && (opt.jit == JIT_ON || bigModel)) throw UnsupportedError("jit: " + why);
    if (use) {
      interpSteps = I.prog.steps;
      interpInst = I.prog.instConst;
      interpShared = I.prog.sharedConst;
      interpHdr = I.prog.header;
      try {
        jitSrc = jitSource(I.prog);  // assigns steps[].jit_class (uploaded below)
      } catch (const Error&) {
        if (opt.jit == JIT_ON || bigModel) throw;
        jitSrc.clear();
        I.prog.steps = interpSteps;
        I.prog.instConst = interpInst;
        I.prog.sharedConst = interpShared;
        I.prog.header = interpHdr;
      }
    }
  }
  int dev0 = opt.device;
  if (dev0 < 0) ck(cudaGetDevice(&dev0), "cudaGetDevice");
  if (!jitSrc.empty()) {
    // build (or load) the module before the upload; under JIT_AUTO a failure
    // (NVRTC compile error, module load) falls back to the interpreter
    PlanImpl::DeviceGuard g0(dev0);
    try {
      I.jitFn = jitKernel(jitSrc);
    } catch (const Error&) {
      if (opt.jit == JIT_ON || bigModel) throw;
      cudaGetLastError();
      jitSrc.clear();
      I.jitFn = nullptr;
      I.prog.steps = interpSteps;
      I.prog.instConst = interpInst;
      I.prog.sharedConst = interpShared;
      I.prog.header = interpHdr;
    }
  }

  int dev = opt.device;
  if (dev < 0) ck(cudaGetDevice(&dev), "cudaGetDevice");
  I.device = dev;
  PlanImpl::DeviceGuard g(dev);
  ck(cudaDeviceGetAttribute(&I.sms, cudaDevAttrMultiProcessorCount, dev), "attr");
  I.dev.hdr = I.prog.header;
  // The program in one device block with one upload (a one-shot call pays
  // one allocation and one copy, not one per array); the error word starts
  // as "none" (all ones), the chunk counter at 0.
  {
    Staging st;
    const size_t oSteps = st.add(packSteps(I.prog.steps, I.prog.header.n_assets)),
                 oCode = st.add(I.prog.packed),
                 oShared = st.add(I.prog.sharedConst), oInst = st.add(I.prog.instConst),
                 oOut = st.add(I.prog.outputs), oBridge = st.add(I.prog.bridge),
                 oMask = st.add(I.prog.streamMask);
    const size_t oErr = st.add(std::vector<unsigned long long>{~0ULL, 0ULL});
    char* base = static_cast<char*>(devMalloc(st.bytes.size()));
    I.owned.push_back(base);
    ck(cudaMemcpy(base, st.bytes.data(), st.bytes.size(), cudaMemcpyHostToDevice),
       "cudaMemcpy H2D");
    // a pageable-memory cudaMemcpy may return before its DMA lands; the plan's
    // launches run on other (non-blocking) streams, which do not wait for it
    ck(cudaStreamSynchronize(0), "cudaStreamSynchronize");
    auto at = [&](size_t o, bool nonEmpty) { return nonEmpty ? base + o : nullptr; };
    I.dev.steps = reinterpret_cast<const unsigned char*>(at(oSteps, !I.prog.steps.empty()));
    I.dev.code = reinterpret_cast<const uint64_t*>(at(oCode, !I.prog.packed.empty()));
    I.dev.sharedConst = reinterpret_cast<const double*>(at(oShared, !I.prog.sharedConst.empty()));
    I.dev.instConst = reinterpret_cast<const double*>(at(oInst, !I.prog.instConst.empty()));
    I.dev.outputs = reinterpret_cast<const cltk_output*>(at(oOut, !I.prog.outputs.empty()));
    I.dev.bridge = reinterpret_cast<const cltk_bridge_op*>(at(oBridge, !I.prog.bridge.empty()));
    I.dev.streamMask = reinterpret_cast<const uint32_t*>(at(oMask, !I.prog.streamMask.empty()));
    I.errKey = reinterpret_cast<unsigned long long*>(base + oErr);
    I.chunkCounter = I.errKey + 1;
  }
  if (I.prog.header.rng == CLTK_RNG_SOBOL) {
    const SobolTables& t = sobolTables(dev);
    I.dev.sobolV = t.V;
    I.dev.sobolT5 = t.T5;
  }
  void* p = nullptr;
  // [n_out] results, then the [kCombineSplit][n_out] combine intermediates
  p = devMalloc((1 + kCombineSplit) * std::max<size_t>(1, I.nOut) * sizeof(cltk_partial));
  I.owned.push_back(p);
  I.combined = static_cast<cltk_partial*>(p);
  I.accInSmem = accFitsSmem(I.prog.header);
  I.smem = pathKernelSmem(I.prog.header, I.accInSmem);
  if (I.smem > 227 * 1024)
    throw UnsupportedError("compiled payoff needs " + std::to_string(I.smem) +
                           " bytes of shared memory per CTA (max 232448)");
  if (I.jitFn) {
    ck(cudaFuncSetAttribute(I.jitFn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
       "jit cudaFuncSetAttribute");
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&I.blocksPerSm, I.jitFn, kBlock, I.smem),
       "jit occupancy");
  } else {
    I.blocksPerSm = pathKernelOccupancy(I.prog.header, I.smem);
  }
  if (I.blocksPerSm <= 0) throw DeviceError("path kernel cannot be resident");
}

Plan::~Plan() = default;

PlanInfo Plan::info() const {
  const PlanImpl& I = *impl_;
  const cltk_plan_header& h = I.prog.header;
  PlanInfo r{};
  r.n_assets = h.n_assets;
  r.n_steps = h.n_steps;
  r.n_thread = h.n_thread;
  r.n_shared_const = h.n_shared_const;
  r.n_inst_const = h.n_inst_const;
  r.n_instances = h.n_instances;
  r.n_days = h.n_days;
  r.n_outputs = I.nOut;
  r.n_shared_ops = I.prog.nSharedOps;
  r.n_inst_ops = I.prog.nInstOps;
  r.has_err = h.has_err;
  r.block = kBlock;
  r.kernel_nodes = I.prog.kernelNodes;
  r.dag_nodes = I.prog.dagNodes;
  r.jit = I.jitFn ? 1 : 0;
  return r;
}

void Plan::chunking(uint64_t paths, uint64_t* chunkPaths, uint64_t* nChunks) const {
  // A function of (paths, n_outputs) only -- never of the GPU count.
  const uint64_t nOut = std::max<uint32_t>(1, impl_->nOut);
  uint64_t maxChunks = std::min<uint64_t>(kMaxChunks, kPartialBudget / (sizeof(cltk_partial) * nOut));
  maxChunks = std::max<uint64_t>(1, maxChunks);
  uint64_t ppt = (paths + kBlock * maxChunks - 1) / (kBlock * maxChunks);
  // Short paths: at least ~64 normal draws per thread per chunk (amortises the
  // per-chunk scheduling and Chan combine), as long as the run still has
  // >= 8192 chunks to balance over the grid.  Depends on the program and the
  // path count only (never on the GPU or its SM count).
  const uint64_t draws = std::max<uint64_t>(1, impl_->drawsPerPath);
  const uint64_t pptWork = std::min<uint64_t>(32, (64 + draws - 1) / draws);
  const uint64_t pptBalance = std::max<uint64_t>(1, paths / (kBlock * 8192ull));
  ppt = std::max<uint64_t>(ppt, std::min(pptWork, pptBalance));
  ppt = std::max<uint64_t>(1, ppt);
  // whole stream periods per thread (a function of the program: the interpreted
  // and the generated kernel chunk alike, so their results stay bit-identical)
  const uint64_t pb = impl_->streamPeriod;
  ppt = (ppt + pb - 1) / pb * pb;
  *chunkPaths = ppt * kBlock;
  *nChunks = (paths + *chunkPaths - 1) / *chunkPaths;
}

namespace {
// QMC: digital shift of Sobol dimension d = top 32 bits of
// Philox2x64-10(key = seed, ctr = (d, 2^64 - 1)); seed 0 = plain Sobol.
const uint32_t* sobolShiftFor(PlanImpl& I, uint64_t seed, cudaStream_t s) {
  if (I.prog.header.rng != CLTK_RNG_SOBOL || seed == 0) return nullptr;
  if (!I.sobolShift) {
    void* p = nullptr;
    p = devMalloc(kSobolDims * sizeof(uint32_t));
    I.owned.push_back(p);
    I.sobolShift = static_cast<uint32_t*>(p);
    I.shiftSeed = seed + 1;  // force the first upload
  }
  if (I.shiftSeed != seed) {
    std::vector<uint32_t> sh(kSobolDims);
    for (uint32_t d = 0; d < kSobolDims; ++d)
      sh[d] = static_cast<uint32_t>(philoxHost(seed, d, ~0ULL) >> 32);
    ck(cudaMemcpyAsync(I.sobolShift, sh.data(), sh.size() * sizeof(uint32_t),
                       cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    I.shiftSeed = seed;
  }
  return I.sobolShift;
}
}  // namespace

void Plan::launch(uint64_t paths, uint64_t seed, uint64_t c0, uint64_t c1, void* partialsDev,
                  void* stream) {
  if (paths == 0) throw EvalError("path count must be positive");
  if (impl_->prog.header.rng == CLTK_RNG_SOBOL && paths > (1ULL << 32))
    throw UnsupportedError("Sobol mode: at most 2^32 paths (32-bit Sobol points)");
  // the device error word is path << 24 | site (engine_device.cuh)
  if (paths > (1ULL << 40)) throw UnsupportedError("at most 2^40 paths per call");
  PlanImpl& I = *impl_;
  PlanImpl::DeviceGuard g(I.device);
  uint64_t chunkPaths, nChunks;
  chunking(paths, &chunkPaths, &nChunks);
  c1 = std::min(c1, nChunks);
  if (c0 >= c1) return;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t work = c1 - c0;
  int grid = static_cast<int>(std::min<uint64_t>(work, static_cast<uint64_t>(I.sms) * I.blocksPerSm));
  if (!I.accInSmem) {
    size_t need = static_cast<size_t>(grid);
    if (need > I.accScratchBlocks) {
      ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      devFree(I.accScratch);
      I.accScratch = static_cast<double*>(devMalloc(need * kWarps * I.nOut * 3 * sizeof(double)));
      I.accScratchBlocks = need;
    }
  }
  ck(cudaMemsetAsync(I.chunkCounter, 0, sizeof(unsigned long long), s), "cudaMemsetAsync");
  RunArgs a{};
  a.keys = philoxKeys(seed);
  a.sobolShift = sobolShiftFor(I, seed, s);
  a.seed = seed;
  a.paths = paths;
  a.chunkPaths = chunkPaths;
  a.ppt = static_cast<uint32_t>(chunkPaths / kBlock);
  a.c0 = c0;
  a.c1 = c1;
  a.partials = static_cast<cltk_partial*>(partialsDev);
  a.errKey = I.errKey;
  a.chunkCounter = I.chunkCounter;
  a.accScratch = I.accScratch;
  a.faultPath = I.fault ? I.faultPath : ~0ULL;
  a.faultDraw = I.faultDraw;
  if (I.jitFn) {
    int accInSmem = I.accInSmem ? 1 : 0;
    void* args[] = {&I.dev, &a, &accInSmem};
    ck(cudaLaunchKernel(I.jitFn, dim3(grid), dim3(kBlock), args, I.smem, s), "jit path kernel launch");
  } else {
    ck(launchPath(I.dev, a, grid, I.smem, s, I.fault), "path kernel launch");
  }
}

std::vector<PriceResult> Plan::finalize(uint64_t paths, uint64_t seed, const void* partialsDev,
                                        void* stream) {
  if (paths == 0) throw EvalError("path count must be positive");
  PlanImpl& I = *impl_;
  PlanImpl::DeviceGuard g(I.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t chunkPaths, nChunks;
  chunking(paths, &chunkPaths, &nChunks);
  std::vector<cltk_partial> host(I.nOut);
  unsigned long long key = ~0ULL;
  if (I.nOut) {
    ck(launchCombine(static_cast<const cltk_partial*>(partialsDev), nChunks, I.nOut,
                     I.combined + std::max<uint32_t>(1, I.nOut), I.combined, s),
       "combine launch");
    ck(cudaMemcpyAsync(host.data(), I.combined, I.nOut * sizeof(cltk_partial),
                       cudaMemcpyDeviceToHost, s),
       "cudaMemcpyAsync D2H");
  }
  ck(cudaMemcpyAsync(&key, I.errKey, sizeof key, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
  ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  ck(cudaMemsetAsync(I.errKey, 0xff, sizeof(unsigned long long), s), "cudaMemsetAsync");
  if (key != ~0ULL) {
    const uint32_t site = static_cast<uint32_t>(key & 0xffffff);
    const ErrorSite& e = site < I.prog.sites.size() ? I.prog.sites[site]
                                                     : ErrorSite{ErrorCode::Eval, "device error"};
    throw Error(e.code, e.message);
  }
  const cltk_plan_header& h = I.prog.header;
  std::vector<PriceResult> out;
  out.reserve(I.nOut);
  for (uint32_t i = 0; i < h.n_instances; ++i)
    for (uint32_t d = 0; d < h.n_days; ++d) {
      const cltk_partial& p = host[i * h.n_days + d];
      PriceResult r;
      r.paths = paths;
      r.seed = seed;
      r.valuationDay = 0;
      r.price = p.mean;
      // stdError = sqrt(var / n), var = sum (x - mean)^2 / (n - 1)
      // (proj/src/pricing.cpp:296-305)
      r.stdError = p.n > 1.0 ? std::sqrt((p.m2 / (p.n - 1.0)) / p.n) : 0.0;
      out.push_back(r);
    }
  return out;
}

std::string Plan::dump() const { return programListing(impl_->prog); }

void Plan::setFault(uint64_t path, uint32_t draw) {
  if (!impl_->fault) throw UnsupportedError("fault injection: plan not built with fault_inject");
  impl_->faultPath = path;
  impl_->faultDraw = draw;
}

int Plan::device() const { return impl_->device; }

uint64_t planErrorWord(Plan& plan, void* stream) {
  PlanImpl& I = *plan.impl();
  PlanImpl::DeviceGuard g(I.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long key = ~0ULL;
  ck(cudaMemcpyAsync(&key, I.errKey, sizeof key, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
  ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  return key;
}

void planSetErrorWord(Plan& plan, void* stream, uint64_t word) {
  PlanImpl& I = *plan.impl();
  PlanImpl::DeviceGuard g(I.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long key = word;
  ck(cudaMemcpyAsync(I.errKey, &key, sizeof key, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
  ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

uint64_t debugPaths(Plan& plan, uint64_t seed, uint64_t path0, uint64_t npaths, double* outputs,
                    double* spots, double* normals) {
  PlanImpl& I = *plan.impl();
  if (I.prog.header.n_assets > CLTK_AOT_MAX_ASSETS)
    throw UnsupportedError("debug_paths: at most " + std::to_string(CLTK_AOT_MAX_ASSETS) +
                           " model assets (ahead-of-time kernel)");
  PlanImpl::DeviceGuard g(I.device);
  const cltk_plan_header& h = I.prog.header;
  const size_t nS = static_cast<size_t>(npaths) * h.n_steps * std::max<uint32_t>(1, h.n_assets);
  const size_t nO = static_cast<size_t>(npaths) * I.nOut;
  double *dO = nullptr, *dS = nullptr, *dZ = nullptr;
  unsigned long long* dE = nullptr;
  ck(cudaMalloc(&dE, sizeof *dE), "cudaMalloc");
  ck(cudaMemset(dE, 0xff, sizeof *dE), "cudaMemset");
  if (outputs && nO) ck(cudaMalloc(&dO, nO * sizeof(double)), "cudaMalloc");
  if (spots && nS) ck(cudaMalloc(&dS, nS * sizeof(double)), "cudaMalloc");
  if (normals && nS) ck(cudaMalloc(&dZ, nS * sizeof(double)), "cudaMalloc");
  if (dZ) ck(cudaMemset(dZ, 0, nS * sizeof(double)), "cudaMemset");
  DumpArgs a{philoxKeys(seed), sobolShiftFor(I, seed, nullptr), seed, path0, npaths, dS, dO, dZ, dE};
  ck(launchDump(I.dev, a, nullptr), "dump launch");
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  if (dO) ck(cudaMemcpy(outputs, dO, nO * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  if (dS) ck(cudaMemcpy(spots, dS, nS * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  if (dZ) ck(cudaMemcpy(normals, dZ, nS * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  unsigned long long key = ~0ULL;
  ck(cudaMemcpy(&key, dE, sizeof key, cudaMemcpyDeviceToHost), "D2H");
  cudaFree(dO);
  cudaFree(dS);
  cudaFree(dZ);
  cudaFree(dE);
  return key;
}

void debugRng(int device, uint64_t seed, uint64_t path, uint64_t i0, uint64_t n, uint64_t* bits,
              double* uniforms, double* normals) {
  if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
  uint64_t* dB = nullptr;
  double *dU = nullptr, *dN = nullptr;
  ck(cudaMalloc(&dB, n * sizeof(uint64_t)), "cudaMalloc");
  ck(cudaMalloc(&dU, n * sizeof(double)), "cudaMalloc");
  ck(cudaMalloc(&dN, n * sizeof(double)), "cudaMalloc");
  ck(launchRngDump(seed, path, i0, n, dB, dU, dN, nullptr), "rng launch");
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  if (bits) ck(cudaMemcpy(bits, dB, n * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
  if (uniforms) ck(cudaMemcpy(uniforms, dU, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  if (normals) ck(cudaMemcpy(normals, dN, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  cudaFree(dB);
  cudaFree(dU);
  cudaFree(dN);
}

void debugMath(int device, int fn, const double* x, uint64_t n, double* out) {
  if (fn < 0 || fn > 9) throw UnsupportedError("debug_math: unknown function " + std::to_string(fn));
  if ((fn == 4 || fn >= 6) && (n % 2) != 0)
    throw UnsupportedError("debug_math: div / log_fmin / log_fmax take pairs");
  if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
  double *dx = nullptr, *dy = nullptr;
  ck(cudaMalloc(&dx, n * sizeof(double)), "cudaMalloc");
  ck(cudaMalloc(&dy, n * sizeof(double)), "cudaMalloc");
  ck(cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
  ck(launchMath(fn, dx, n, dy, nullptr), "math launch");
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  ck(cudaMemcpy(out, dy, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  cudaFree(dx);
  cudaFree(dy);
}

void debugSobol(int device, uint64_t n0, uint64_t n, uint32_t d0, uint32_t nd, bool aligned,
                uint32_t* out) {
  if (static_cast<uint64_t>(d0) + nd > kSobolDims)
    throw UnsupportedError("debug_sobol: dimensions beyond the direction-number table");
  if (aligned && (n0 % 32) != 0) throw UnsupportedError("debug_sobol: aligned needs n0 % 32 == 0");
  if (n == 0 || nd == 0) return;
  if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
  std::vector<uint32_t> V(kSobolV, kSobolV + kSobolDims * 32), T5(kSobolDims * 32);
  for (uint32_t d = 0; d < kSobolDims; ++d)  // the table Plan::init uploads
    for (uint32_t g = 0; g < 32; ++g) {
      uint32_t x = 0;
      for (uint32_t k = 0; k < 5; ++k)
        if ((g >> k) & 1u) x ^= V[d * 32 + k];
      T5[d * 32 + g] = x;
    }
  uint32_t *dV = nullptr, *dT = nullptr, *dO = nullptr;
  ck(cudaMalloc(&dV, V.size() * 4), "cudaMalloc");
  ck(cudaMalloc(&dT, T5.size() * 4), "cudaMalloc");
  ck(cudaMalloc(&dO, n * nd * 4), "cudaMalloc");
  ck(cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice), "H2D");
  ck(cudaMemcpy(dT, T5.data(), T5.size() * 4, cudaMemcpyHostToDevice), "H2D");
  ck(launchSobolDump(dV, dT, n0, n, d0, nd, aligned, dO, nullptr), "sobol launch");
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  ck(cudaMemcpy(out, dO, n * nd * 4, cudaMemcpyDeviceToHost), "D2H");
  cudaFree(dV);
  cudaFree(dT);
  cudaFree(dO);
}

double fp64Peak(int device, int iters, double* seconds) {
  if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
  int dev = 0, sms = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
  double* sink = nullptr;
  ck(cudaMalloc(&sink, 256 * sizeof(double)), "cudaMalloc");
  const int grid = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ck(launchFp64Peak(sink, 16, grid, nullptr), "fp64 warmup");
  cudaEventRecord(e0);
  ck(launchFp64Peak(sink, iters, grid, nullptr), "fp64 launch");
  cudaEventRecord(e1);
  ck(cudaEventSynchronize(e1), "cudaEventSynchronize");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  const double flops = 2.0 * 16 * 8 * static_cast<double>(iters) * grid * 256;
  if (seconds) *seconds = ms * 1e-3;
  return flops / (ms * 1e-3) / 1e12;
}

// ---- one-shot pricing on the plans' own buffers -----------------------------
std::vector<int> resolveDevices(const RunOptions& opt) {
  if (!opt.devices.empty()) return opt.devices;
  if (opt.device < 0) {
    // CLTK_DEVICES: "all" or a comma-separated list shards every one-shot call
    // whose caller did not name a device (the C++ priceAcrossTime, cltk_gpu_price)
    if (const char* env = std::getenv("CLTK_DEVICES"); env && *env) {
      std::vector<int> v;
      if (std::strcmp(env, "all") == 0) {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        for (int d = 0; d < n; ++d) v.push_back(d);
      } else {
        for (const char* q = env; *q;) {
          char* e = nullptr;
          const long d = std::strtol(q, &e, 10);
          if (e == q || d < 0) throw UnsupportedError(std::string("CLTK_DEVICES: bad list ") + env);
          v.push_back(static_cast<int>(d));
          q = *e == ',' ? e + 1 : e;
          if (*e && *e != ',') throw UnsupportedError(std::string("CLTK_DEVICES: bad list ") + env);
        }
      }
      if (!v.empty()) return v;
    }
  }
  return {opt.device};
}

namespace {

cltk_partial* ownPartials(PlanImpl& I, uint64_t nChunks) {
  PlanImpl::DeviceGuard g(I.device);
  if (nChunks > I.ownPartialsChunks) {
    devFree(I.ownPartials);
    I.ownPartials = static_cast<cltk_partial*>(
        devMalloc(nChunks * std::max<uint32_t>(1, I.nOut) * sizeof(cltk_partial)));
    I.ownPartialsChunks = nChunks;
  }
  return I.ownPartials;
}

struct Streams {
  std::vector<cudaStream_t> s;
  std::vector<int> dev;
  ~Streams() {
    for (size_t g = 0; g < s.size(); ++g) {
      cudaSetDevice(dev[g]);
      cudaStreamDestroy(s[g]);
    }
  }
};

// The reference's runParallel (proj/src/pricing.cpp:268-286, 345-364) across
// the GPUs of this process: plan g prices the contiguous chunk slice
// [g S, min(C, (g+1) S)), S = ceil(C / G), into its own full-size partials
// buffer; ONE in-place NCCL all-gather over NVLink assembles every buffer
// (distinct devices), or device copies into plan 0's buffer (a device listed
// twice: tests on one GPU); the device error words merge by MIN (the lowest
// failing path wins, as on one GPU) and plan 0 runs the fixed-order combine.
// Chunking depends only on (paths, outputs): bit-identical for any G.
std::vector<PriceResult> runGroup(const std::vector<Plan*>& plans, uint64_t paths, uint64_t seed,
                                  const std::vector<uint64_t>& days) {
  static const bool trace = std::getenv("CLTK_TRACE") != nullptr;
  const size_t G = plans.size();
  uint64_t chunkPaths, nChunks;
  plans[0]->chunking(paths, &chunkPaths, &nChunks);
  const uint64_t S = (nChunks + G - 1) / G;
  const uint32_t nOut = std::max<uint32_t>(1, plans[0]->impl()->nOut);
  Streams st;
  std::vector<double*> bufs(G);
  std::vector<int> devs(G);
  for (size_t g = 0; g < G; ++g) {
    PlanImpl& I = *plans[g]->impl();
    devs[g] = I.device;
    bufs[g] = reinterpret_cast<double*>(ownPartials(I, G == 1 ? nChunks : G * S));
    PlanImpl::DeviceGuard dg(I.device);
    cudaStream_t s = nullptr;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    st.s.push_back(s);
    st.dev.push_back(I.device);
  }
  for (size_t g = 0; g < G; ++g)  // asynchronous: the devices run concurrently
    plans[g]->launch(paths, seed, G == 1 ? 0 : g * S, G == 1 ? nChunks : std::min(nChunks, (g + 1) * S),
                     bufs[g], st.s[g]);
  if (G > 1) {
    bool distinct = true;
    for (size_t a = 0; a < G; ++a)
      for (size_t b = a + 1; b < G; ++b) distinct = distinct && devs[a] != devs[b];
    std::string why;
    const size_t slice = static_cast<size_t>(S) * nOut * (sizeof(cltk_partial) / sizeof(double));
    if (distinct && ncclAvailable(&why)) {
      ncclAllGatherInPlace(*ncclClique(devs), bufs, slice, st.s);
      if (trace) std::fprintf(stderr, "[cltk] %zu GPUs: NCCL all-gather (%s), %zu B per rank\n",
                              G, why.c_str(), slice * sizeof(double));
    } else {
      if (distinct) throw UnsupportedError("multi-GPU: " + why);
      PlanImpl::DeviceGuard dg(devs[0]);
      for (size_t g = 1; g < G; ++g) {
        const uint64_t c0 = g * S, c1 = std::min(nChunks, (g + 1) * S);
        if (c0 >= c1) continue;
        cudaEvent_t ev;
        {
          PlanImpl::DeviceGuard dgg(devs[g]);
          ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
          ck(cudaEventRecord(ev, st.s[g]), "cudaEventRecord");
        }
        ck(cudaStreamWaitEvent(st.s[0], ev, 0), "cudaStreamWaitEvent");
        ck(cudaMemcpyPeerAsync(bufs[0] + c0 * nOut * 3, devs[0], bufs[g] + c0 * nOut * 3, devs[g],
                               (c1 - c0) * nOut * sizeof(cltk_partial), st.s[0]),
           "cudaMemcpyPeerAsync");
        cudaEventDestroy(ev);
      }
    }
    // error words: MIN over the shards, the other plans' words reset
    uint64_t w = ~0ULL;
    for (size_t g = 0; g < G; ++g) w = std::min<uint64_t>(w, planErrorWord(*plans[g], st.s[g]));
    for (size_t g = 1; g < G; ++g) planSetErrorWord(*plans[g], st.s[g], ~0ULL);
    planSetErrorWord(*plans[0], st.s[0], w);
  }
  std::vector<PriceResult> r = plans[0]->finalize(paths, seed, bufs[0], st.s[0]);
  const uint32_t nd = static_cast<uint32_t>(days.size());
  for (std::size_t i = 0; i < r.size(); ++i) r[i].valuationDay = days[i % nd];
  return r;
}

using PlanGroup = std::vector<std::unique_ptr<Plan>>;

PlanGroup makeGroup(const std::function<std::unique_ptr<Plan>(int)>& make,
                    const std::vector<int>& devices) {
  PlanGroup g;
  for (int d : devices) g.push_back(make(d));
  return g;
}

std::vector<PriceResult> runGroup(PlanGroup& g, uint64_t paths, uint64_t seed,
                                  const std::vector<uint64_t>& days) {
  std::vector<Plan*> p;
  for (auto& x : g) p.push_back(x.get());
  return runGroup(p, paths, seed, days);
}

// A one-shot call: plans, run on their own buffers, free.  CLTK_TRACE=1 prints
// where the host time goes (stderr).
std::vector<PriceResult> oneShot(const std::function<std::unique_ptr<Plan>(int)>& make,
                                 const std::vector<int>& devices, uint64_t paths, uint64_t seed,
                                 const std::vector<uint64_t>& days) {
  static const bool trace = std::getenv("CLTK_TRACE") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  std::vector<PriceResult> r;
  double tPlan = 0.0, tRun = 0.0;
  {
    PlanGroup g = makeGroup(make, devices);
    if (days.empty()) return {};
    const auto t1 = clk::now();
    r = runGroup(g, paths, seed, days);
    tPlan = std::chrono::duration<double, std::milli>(t1 - t0).count();
    tRun = std::chrono::duration<double, std::milli>(clk::now() - t1).count();
  }
  if (trace) {
    const double tAll = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    std::fprintf(stderr, "[cltk] one-shot price: plan %.2f ms, run %.2f ms, free %.2f ms\n",
                 tPlan, tRun, tAll - tPlan - tRun);
  }
  return r;
}
}  // namespace

std::vector<PriceResult> priceCached(const std::string& key,
                                     const std::function<std::unique_ptr<Plan>(int)>& make,
                                     const std::vector<int>& devices, uint64_t paths,
                                     uint64_t seed, const std::vector<uint64_t>& days) {
  struct Entry {
    std::string key;
    PlanGroup plans;
    std::mutex use;
  };
  constexpr size_t kEntries = 4;
  static std::mutex mu;
  static std::vector<std::shared_ptr<Entry>> lru;  // most recent last
  if (paths == 0) throw EvalError("path count must be positive");
  if (days.empty()) {  // nothing to price; the inputs are still validated
    (void)makeGroup(make, devices);
    return {};
  }
  // CLTK_PLAN_CACHE=0: every call builds (parses, compiles, uploads) its plans
  static const bool enabled = [] {
    const char* v = std::getenv("CLTK_PLAN_CACHE");
    return v == nullptr || std::strcmp(v, "0") != 0;
  }();
  if (!enabled) return oneShot(make, devices, paths, seed, days);
  std::string k = key;
  for (int d : devices) k.append(reinterpret_cast<const char*>(&d), sizeof d);
  std::shared_ptr<Entry> e;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (size_t i = 0; i < lru.size(); ++i)
      if (lru[i]->key == k) {
        e = lru[i];
        lru.erase(lru.begin() + static_cast<std::ptrdiff_t>(i));
        lru.push_back(e);
        break;
      }
  }
  if (!e) {
    e = std::make_shared<Entry>();
    e->key = k;
    e->plans = makeGroup(make, devices);
    std::lock_guard<std::mutex> lock(mu);
    lru.push_back(e);
    if (lru.size() > kEntries) lru.erase(lru.begin());
  }
  std::lock_guard<std::mutex> use(e->use);
  try {
    return runGroup(e->plans, paths, seed, days);
  } catch (...) {  // a plan that failed on the device is not reused
    std::lock_guard<std::mutex> lock(mu);
    for (size_t i = 0; i < lru.size(); ++i)
      if (lru[i] == e) {
        lru.erase(lru.begin() + static_cast<std::ptrdiff_t>(i));
        break;
      }
    throw;
  }
}

std::vector<PriceResult> priceBatch(const std::vector<const Kernel*>& instances,
                                    const ModelSpec& model, uint64_t paths, uint64_t seed,
                                    const std::vector<uint64_t>& days, const TEnv& tenv,
                                    const RunOptions& opt) {
  if (paths == 0) throw EvalError("path count must be positive");
  return oneShot(
      [&](int d) {
        RunOptions o = opt;
        o.device = d;
        return std::make_unique<Plan>(instances, model, days, tenv, o);
      },
      resolveDevices(opt), paths, seed, days);
}

std::vector<PriceResult> priceTemplate(const Kernel& templ, const double* literals,
                                       std::size_t nInstances, std::size_t nLits,
                                       const ModelSpec& model, uint64_t paths, uint64_t seed,
                                       const std::vector<uint64_t>& days, const TEnv& tenv,
                                       const RunOptions& opt) {
  if (paths == 0) throw EvalError("path count must be positive");
  return oneShot(
      [&](int d) {
        RunOptions o = opt;
        o.device = d;
        return std::make_unique<Plan>(templ, literals, nInstances, nLits, model, days, tenv, o);
      },
      resolveDevices(opt), paths, seed, days);
}

std::vector<PriceResult> priceAcrossTime(const Kernel& k, const ModelSpec& model,
                                         uint64_t paths, uint64_t seed,
                                         const std::vector<uint64_t>& days, const TEnv& tenv,
                                         unsigned /*threads*/) {
  return priceBatch({&k}, model, paths, seed, days, tenv, RunOptions());
}

PriceResult priceMC(const Kernel& k, const ModelSpec& model, uint64_t paths, uint64_t seed,
                    uint64_t valuationDay, const TEnv& tenv, unsigned threads) {
  return priceAcrossTime(k, model, paths, seed, {valuationDay}, tenv, threads).front();
}

}  // namespace b200
}  // namespace cltk
