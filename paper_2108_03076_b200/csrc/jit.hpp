// NVRTC code generation of compiled payoff programs (BASELINE north_star
// item (4): "a codegen emits CUDA from the compiled payoff AST (NVRTC to
// sm_100a)").
//
// The compiled device program (compiler.cpp) is turned into a payoff policy
// for the path kernel (engine_device.cuh): every simulation step's ops become
// one `case` of a switch on the step's class (steps with identical op lists
// share a class), every op one straight-line CUDA statement with constant
// shared-memory offsets -- no fetch, decode or dispatch per op, and the
// step's spots are read from registers.  The ops, their order and their
// IEEE operations are the interpreter's, so prices are bit-identical to the
// interpreted kernel (tests/test_gpu_parity.py).  Literals stay in the plan's
// constant tables (kernel data), so new template instances and new literal
// values reuse the compiled kernel; compiled modules are cached by source.
#pragma once
#include <string>

#include "compiler.hpp"

namespace cltk {
namespace b200 {

enum JitMode { JIT_OFF = 0, JIT_ON = 1, JIT_AUTO = 2 };

// Whether the NVRTC library can be loaded (why not, otherwise).
bool jitAvailable(std::string* why);

// CUDA source of the path kernel with the generated payoff policy for this
// program; assigns prog.steps[s].jit_class.  Host only (no GPU needed).
std::string jitSource(CompiledProgram& prog);

// Number of straight-line op statements the source contains (size guard).
size_t jitOpCount(const CompiledProgram& prog);

// NVRTC-compiles `src` for sm_100a (cached by source text) and returns the
// kernel handle (a cudaKernel_t, usable as `const void*` with the runtime
// launch/attribute/occupancy APIs).  Throws UnsupportedError on failure.
const void* jitKernel(const std::string& src);

// NVRTC compile only (no device needed): returns the cubin size, fills log.
size_t jitCompileOnly(const std::string& src, std::string* log);

}  // namespace b200
}  // namespace cltk
