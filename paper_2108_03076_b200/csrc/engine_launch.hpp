// Host-side launch wrappers for the sm_100a kernels in mc_engine.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine_types.h"

namespace cltk {
namespace b200 {

size_t pathKernelSmem(const cltk_plan_header& h, bool accInSmem);
bool accFitsSmem(const cltk_plan_header& h);
// Blocks per SM the path kernel achieves for this plan (occupancy API).
int pathKernelOccupancy(const cltk_plan_header& h, size_t smem);
// fault: the test build of the kernel (RunArgs::faultPath / faultDraw)
cudaError_t launchPath(const DevPlan& p, const RunArgs& a, int grid, size_t smem,
                       cudaStream_t s, bool fault = false);
// Chunk partials -> one (n, mean, M2) per output.  Large chunk counts go
// through kCombineSplit-wide intermediates (scratch: kCombineSplit * nOut).
constexpr uint32_t kCombineSplit = 64;
cudaError_t launchCombine(const cltk_partial* parts, uint64_t nChunks, uint32_t nOut,
                          cltk_partial* scratch, cltk_partial* out, cudaStream_t s);
cudaError_t launchDump(const DevPlan& p, const DumpArgs& a, cudaStream_t s);
cudaError_t launchRngDump(uint64_t seed, uint64_t path, uint64_t i0, uint64_t n,
                          uint64_t* bits, double* uniform, double* normal, cudaStream_t s);
cudaError_t launchSobolDump(const uint32_t* V, const uint32_t* T5, uint64_t n0, uint64_t n,
                            uint32_t d0, uint32_t nd, bool aligned, uint32_t* out, cudaStream_t s);
cudaError_t launchMath(int fn, const double* x, uint64_t n, double* out, cudaStream_t s);
cudaError_t launchFp64Peak(double* sink, int iters, int grid, cudaStream_t s);

}  // namespace b200
}  // namespace cltk
