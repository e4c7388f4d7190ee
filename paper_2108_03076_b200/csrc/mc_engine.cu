// sm_100a Monte Carlo pricing engine, ahead-of-time build: the device code
// (engine_device.cuh) with the interpreted payoff policy, for every asset
// count and RNG mode, plus the host-side launch wrappers.
#include <cuda_runtime.h>

#include "engine_launch.hpp"
#include "engine_device.cuh"

// Compiled as three translation units (Makefile, in parallel) so the kernel
// instantiations build concurrently -- this file, and mc_engine_qmc.cu /
// mc_engine_fault.cu which include it with another CLTK_AOT_PART: 0 -- the Philox path kernels, the dump,
// combine and test kernels and every host entry point; 1 -- the QMC kernels;
// 2 -- the fault-hook test build of the Philox kernels.
#ifndef CLTK_AOT_PART
#define CLTK_AOT_PART 0
#endif

#define CLTK_NA_SWITCH(NA_, CALL)                 \
  switch (NA_) {                                  \
    case 1: { constexpr int NA = 1; CALL; }       \
    case 2: { constexpr int NA = 2; CALL; }       \
    case 3: { constexpr int NA = 3; CALL; }       \
    case 4: { constexpr int NA = 4; CALL; }       \
    case 5: { constexpr int NA = 5; CALL; }       \
    case 6: { constexpr int NA = 6; CALL; }       \
    case 7: { constexpr int NA = 7; CALL; }       \
    case 8: { constexpr int NA = 8; CALL; }       \
    default: { constexpr int NA = 1; CALL; }      \
  }

namespace cltk {
namespace b200 {

// (parts 1 and 2)
cudaError_t launchPathQmc(const DevPlan& p, const RunArgs& a, int grid, size_t smem,
                          cudaStream_t s, int accInSmem);
int occupancyQmc(const cltk_plan_header& h, size_t smem);
cudaError_t launchDumpQmc(const DevPlan& p, const DumpArgs& a, cudaStream_t s);
cudaError_t launchPathFault(const DevPlan& p, const RunArgs& a, int grid, size_t smem,
                            cudaStream_t s, int accInSmem);

namespace {

template <int NA, bool QMC, bool FAULT = false>
cudaError_t launchPathT(const DevPlan& p, const RunArgs& a, int grid, size_t smem,
                        cudaStream_t s, int accInSmem) {
  // (per device: the attribute is a property of the kernel on the current device)
  static bool configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(path_kernel<NA, QMC, FAULT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    if (dev < 64) configured[dev] = true;
  }
  path_kernel<NA, QMC, FAULT><<<grid, kBlock, smem, s>>>(p, a, accInSmem);
  return cudaGetLastError();
}

// QMC bridge slots overlap the (unused) Y slots and the work lists after
// them; only the excess needs extra shared memory.
size_t bridgeWords(const cltk_plan_header& h) {
  if (h.rng != CLTK_RNG_SOBOL) return 0;
  const size_t need = static_cast<size_t>(h.n_bridge_slots) * (h.n_assets ? h.n_assets : 1) * kBlock;
  const size_t have = static_cast<size_t>(yRows(h.n_assets ? h.n_assets : 1, true)) * kBlock;  // the Y rows
  return need > have ? need - have : 0;
}

template <int NA, bool QMC>
cudaError_t launchDumpT(const DevPlan& p, const DumpArgs& a, cudaStream_t s) {
  const cltk_plan_header& h = p.hdr;
  size_t smem = (static_cast<size_t>(h.n_thread) * kBlock +
                 kWarps * (h.n_shared_const + h.n_inst_const) +
                 normScratchWords(h.n_assets ? h.n_assets : 1, h.rng == CLTK_RNG_SOBOL) +
                 bridgeWords(h)) *
                sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(dump_kernel<NA, QMC>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  const unsigned grid = static_cast<unsigned>((a.npaths + kBlock - 1) / kBlock);
  dump_kernel<NA, QMC><<<grid, kBlock, smem, s>>>(p, a);
  return cudaGetLastError();
}

template <int NA, bool QMC>
int occupancyT(size_t smem) {
  int blocks = 0;
  cudaFuncSetAttribute(path_kernel<NA, QMC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, path_kernel<NA, QMC>, kBlock, smem);
  return blocks;
}

}  // namespace

#if CLTK_AOT_PART == 0
bool accFitsSmem(const cltk_plan_header& h) {
  const size_t nOut = static_cast<size_t>(h.n_instances) * h.n_days;
  return kWarps * nOut * 3 * sizeof(double) <= 48 * 1024;
}

size_t pathKernelSmem(const cltk_plan_header& h, bool accInSmem) {
  const size_t nOut = static_cast<size_t>(h.n_instances) * h.n_days;
  size_t words = static_cast<size_t>(h.reg_top - h.reg_base) * kBlock +
                 kWarps * (h.n_shared_const + h.n_inst_const);
  if (accInSmem) words += kWarps * nOut * 3;
  words += kWarps + 1;  // counts + chunk slot
  words += normScratchWords(h.n_assets ? h.n_assets : 1, h.rng == CLTK_RNG_SOBOL);
  words += bridgeWords(h);
  return words * sizeof(double);
}

int pathKernelOccupancy(const cltk_plan_header& h, size_t smem) {
  if (h.rng == CLTK_RNG_SOBOL) return occupancyQmc(h, smem);
  CLTK_NA_SWITCH(h.n_assets == 0 ? 1 : h.n_assets, return (occupancyT<NA, false>(smem)));
}

cudaError_t launchPath(const DevPlan& p, const RunArgs& a, int grid, size_t smem, cudaStream_t s,
                       bool fault) {
  const int accInSmem = accFitsSmem(p.hdr) ? 1 : 0;
  if (fault) {  // test builds of the Philox kernels (cltk_plan_set_fault)
    if (p.hdr.rng == CLTK_RNG_SOBOL) return cudaErrorInvalidValue;
    return launchPathFault(p, a, grid, smem, s, accInSmem);
  }
  if (p.hdr.rng == CLTK_RNG_SOBOL) return launchPathQmc(p, a, grid, smem, s, accInSmem);
  CLTK_NA_SWITCH(p.hdr.n_assets == 0 ? 1 : p.hdr.n_assets,
                 return (launchPathT<NA, false>(p, a, grid, smem, s, accInSmem)));
}

cudaError_t launchDump(const DevPlan& p, const DumpArgs& a, cudaStream_t s) {
  if (p.hdr.rng == CLTK_RNG_SOBOL) return launchDumpQmc(p, a, s);
  CLTK_NA_SWITCH(p.hdr.n_assets == 0 ? 1 : p.hdr.n_assets, return (launchDumpT<NA, false>(p, a, s)));
}

uint32_t combineSplit(uint64_t nChunks) {
  const uint64_t g = (nChunks + 4095) / 4096;  // >= 16 chunks per thread
  return static_cast<uint32_t>(g < 1 ? 1 : (g > kCombineSplit ? kCombineSplit : g));
}

cudaError_t launchCombine(const cltk_partial* parts, uint64_t nChunks, uint32_t nOut,
                          cltk_partial* scratch, cltk_partial* out, cudaStream_t s) {
  const uint32_t g = combineSplit(nChunks);
  if (g == 1) {
    combine_kernel<<<dim3(nOut, 1), 256, 0, s>>>(parts, nChunks, nOut, out);
    return cudaGetLastError();
  }
  combine_kernel<<<dim3(nOut, g), 256, 0, s>>>(parts, nChunks, nOut, scratch);
  combine_kernel<<<dim3(nOut, 1), 256, 0, s>>>(scratch, g, nOut, out);
  return cudaGetLastError();
}

cudaError_t launchRngDump(uint64_t seed, uint64_t path, uint64_t i0, uint64_t n, uint64_t* bits,
                          double* uniform, double* normal, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((n + 255) / 256);
  rng_kernel<<<grid, 256, 0, s>>>(seed, path, i0, n, bits, uniform, normal);
  return cudaGetLastError();
}

cudaError_t launchSobolDump(const uint32_t* V, const uint32_t* T5, uint64_t n0, uint64_t n,
                            uint32_t d0, uint32_t nd, bool aligned, uint32_t* out, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((n + 255) / 256);
  sobol_kernel<<<grid, 256, 0, s>>>(V, T5, n0, n, d0, nd, aligned ? 1 : 0, out);
  return cudaGetLastError();
}

cudaError_t launchMath(int fn, const double* x, uint64_t n, double* out, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((n + 255) / 256);
  math_kernel<<<grid, 256, 0, s>>>(fn, x, n, out);
  return cudaGetLastError();
}

cudaError_t launchFp64Peak(double* sink, int iters, int grid, cudaStream_t s) {
  fp64_peak_kernel<<<grid, 256, 0, s>>>(sink, iters);
  return cudaGetLastError();
}

#endif  // CLTK_AOT_PART == 0

#if CLTK_AOT_PART == 1
cudaError_t launchPathQmc(const DevPlan& p, const RunArgs& a, int grid, size_t smem,
                          cudaStream_t s, int accInSmem) {
  CLTK_NA_SWITCH(p.hdr.n_assets == 0 ? 1 : p.hdr.n_assets,
                 return (launchPathT<NA, true>(p, a, grid, smem, s, accInSmem)));
}
int occupancyQmc(const cltk_plan_header& h, size_t smem) {
  CLTK_NA_SWITCH(h.n_assets == 0 ? 1 : h.n_assets, return (occupancyT<NA, true>(smem)));
}
cudaError_t launchDumpQmc(const DevPlan& p, const DumpArgs& a, cudaStream_t s) {
  CLTK_NA_SWITCH(p.hdr.n_assets == 0 ? 1 : p.hdr.n_assets, return (launchDumpT<NA, true>(p, a, s)));
}
#endif

#if CLTK_AOT_PART == 2
cudaError_t launchPathFault(const DevPlan& p, const RunArgs& a, int grid, size_t smem,
                            cudaStream_t s, int accInSmem) {
  CLTK_NA_SWITCH(p.hdr.n_assets == 0 ? 1 : p.hdr.n_assets,
                 return (launchPathT<NA, false, true>(p, a, grid, smem, s, accInSmem)));
}
#endif

}  // namespace b200
}  // namespace cltk

