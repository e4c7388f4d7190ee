// Launch-time types of the path kernel, shared by the host code, the
// ahead-of-time device build and the NVRTC device build (no CUDA runtime
// headers: NVRTC sees this file too).
#pragma once
#include <stdint.h>

#include "program.h"

namespace cltk {
namespace b200 {

#ifndef CLTK_BLOCK
#define CLTK_BLOCK 128
#endif
constexpr int kBlock = CLTK_BLOCK;  // threads per CTA (4 warps)
constexpr int kWarps = kBlock / 32;

// Normal draws per thread of one warp-cooperative batch (engine_device.cuh).
#ifndef CLTK_MAX_BATCH
#define CLTK_MAX_BATCH 6
#endif
#if defined(__CUDACC__)
#define CLTK_TYPES_HD __host__ __device__
#else
#define CLTK_TYPES_HD
#endif
// Simulation steps per normal batch (nA draws each).
CLTK_TYPES_HD inline constexpr int batchSteps(int na) {
  return na >= CLTK_MAX_BATCH ? 1 : CLTK_MAX_BATCH / na;
}
// Philox mode streams a thread's paths through full batches of
// batchSteps(nA) * nA slots (engine_device.cuh path_body); after this many
// paths of `draws` slots the stream is back at a batch boundary.  The host
// makes the paths per thread of a chunk a multiple of it (no batch runs past
// the chunk's last path).
CLTK_TYPES_HD inline constexpr uint32_t streamPeriod(uint32_t draws, uint32_t na) {
  uint32_t a = static_cast<uint32_t>(batchSteps(na < 1 ? 1 : static_cast<int>(na))) * (na < 1 ? 1 : na);
  const uint32_t m = a;
  uint32_t b = draws < 1 ? 1 : draws;
  while (b) {  // gcd(batch slots, draws)
    const uint32_t t = a % b;
    a = b;
    b = t;
  }
  return m / a;
}

// Philox2x64-10 key schedule key_r = seed + r * 0x9E3779B97F4A7C15.
struct PhiloxKeys {
  uint64_t k[10];
};
#if !defined(__CUDACC_RTC__)
inline PhiloxKeys philoxKeys(uint64_t seed) {
  PhiloxKeys K;
  for (int r = 0; r < 10; ++r) K.k[r] = seed + static_cast<uint64_t>(r) * 0x9E3779B97F4A7C15ULL;
  return K;
}
#endif

// Everything the path kernel reads, all device pointers.
struct DevPlan {
  cltk_plan_header hdr;
  const unsigned char* steps;  // [n_steps] device step records (StepRef)
  const uint64_t* code;
  const double* sharedConst;
  const double* instConst;
  const cltk_output* outputs;
  // QMC mode
  const cltk_bridge_op* bridge;
  const uint32_t* sobolV;   // [2048][32] direction numbers
  const uint32_t* sobolT5;  // [2048][32] XOR of v[d][0..4] over the set bits of g
  // Philox normal streams (header.stream): the draw mask of a batch that
  // starts at step s (its SB steps wrapping into the next path), [n_steps]
  const uint32_t* streamMask;
};

// Device step records of a plan with NA assets: header, A, B, S (even counts).
CLTK_TYPES_HD inline constexpr int stepPad(int na) { return ((na < 1 ? 1 : na) + 1) & ~1; }
CLTK_TYPES_HD inline constexpr size_t stepStride(int na) {
  return sizeof(cltk_step_hdr) + 3 * sizeof(double) * static_cast<size_t>(stepPad(na));
}
struct StepRef {
  const cltk_step_hdr* h;
  const double* A;
  const double* B;
  const double* S;
};
template <int NA>
CLTK_TYPES_HD inline StepRef stepAt(const unsigned char* steps, uint32_t s) {
  const unsigned char* b = steps + static_cast<size_t>(s) * stepStride(NA);
  const double* a = reinterpret_cast<const double*>(b + sizeof(cltk_step_hdr));
  return StepRef{reinterpret_cast<const cltk_step_hdr*>(b), a, a + stepPad(NA),
                 a + 2 * stepPad(NA)};
}

struct RunArgs {
  PhiloxKeys keys;
  const uint32_t* sobolShift;  // QMC digital shift per dimension (null: none)
  uint64_t seed;
  uint64_t paths;        // total paths of the run (whole job, all GPUs)
  uint64_t chunkPaths;   // kBlock * ppt
  uint32_t ppt;          // paths per thread per chunk
  uint64_t c0, c1;       // chunk range handled by this launch
  cltk_partial* partials;           // [n_chunks][n_out]
  unsigned long long* errKey;       // min(path << 24 | site)
  unsigned long long* chunkCounter; // dynamic chunk scheduler
  double* accScratch;               // global accumulators when n_out is large
  // test builds only (FAULT kernels, cltk_plan_set_fault): the draw whose
  // uniform is forced to 1.0; ~0 = none
  uint64_t faultPath;
  uint32_t faultDraw;
};

// Dump modes (tests): per-path outputs instead of reduction.
struct DumpArgs {
  PhiloxKeys keys;
  const uint32_t* sobolShift;
  uint64_t seed, path0, npaths;
  double* spots;    // [npaths][n_steps][n_assets] or null
  double* outputs;  // [npaths][n_out] or null
  double* normals;  // [npaths][n_steps][n_assets] or null
  unsigned long long* errKey;
};

}  // namespace b200
}  // namespace cltk
