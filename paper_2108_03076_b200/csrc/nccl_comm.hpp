// NCCL for the in-process multi-GPU path (engine.cpp runSharded): the single
// data-path collective of a sharded price -- an in-place all-gather of the
// per-GPU slices of the chunk partials over NVLink / NVSwitch.  NCCL is
// loaded with dlopen on first use (the engine library does not link it), so
// single-GPU callers never need it.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <string>
#include <vector>

namespace cltk {
namespace b200 {

// Whether libnccl.so.2 can be loaded (and its version), else why not.
bool ncclAvailable(std::string* info);

// One communicator per device of `devices` (ncclCommInitAll; the devices
// must be distinct), created once per device list and kept for the process.
struct NcclClique;
std::shared_ptr<NcclClique> ncclClique(const std::vector<int>& devices);

// In place on every rank g: bufs[g] holds its slice at element offset
// g * count; afterwards every bufs[g] holds all ranks' slices.  Doubles;
// asynchronous on streams[g].
void ncclAllGatherInPlace(NcclClique& c, const std::vector<double*>& bufs, size_t count,
                          const std::vector<cudaStream_t>& streams);

}  // namespace b200
}  // namespace cltk
