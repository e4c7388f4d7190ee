// NVRTC code generation of compiled payoff programs (see jit.hpp).
#include "jit.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <unistd.h>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "engine_types.h"

namespace cltk {
namespace b200 {

// Device sources embedded at build time (tools/embed_sources.py).
extern const int kJitHeaderCount;
extern const char* const kJitHeaderNames[];
extern const char* const kJitHeaderSources[];

namespace {

// ---------------------------------------------------------------------------
// NVRTC, loaded on first use (the engine library does not link it).
// ---------------------------------------------------------------------------
struct Nvrtc {
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*logSize)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubinSize)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*errstr)(nvrtcResult) = nullptr;
  std::string why;
  bool ok = false;
};

Nvrtc loadNvrtc() {
  Nvrtc n;
  void* h = nullptr;
  for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
    h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    n.why = "libnvrtc.so.12 not loadable";
    return n;
  }
  auto sym = [&](const char* s) { return dlsym(h, s); };
  n.create = reinterpret_cast<decltype(n.create)>(sym("nvrtcCreateProgram"));
  n.compile = reinterpret_cast<decltype(n.compile)>(sym("nvrtcCompileProgram"));
  n.logSize = reinterpret_cast<decltype(n.logSize)>(sym("nvrtcGetProgramLogSize"));
  n.log = reinterpret_cast<decltype(n.log)>(sym("nvrtcGetProgramLog"));
  n.cubinSize = reinterpret_cast<decltype(n.cubinSize)>(sym("nvrtcGetCUBINSize"));
  n.cubin = reinterpret_cast<decltype(n.cubin)>(sym("nvrtcGetCUBIN"));
  n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("nvrtcDestroyProgram"));
  n.errstr = reinterpret_cast<decltype(n.errstr)>(sym("nvrtcGetErrorString"));
  n.ok = n.create && n.compile && n.logSize && n.log && n.cubinSize && n.cubin && n.destroy &&
         n.errstr;
  if (!n.ok) n.why = "libnvrtc lacks the CUBIN API";
  return n;
}

Nvrtc& nvrtc() {
  static Nvrtc n = loadNvrtc();
  return n;
}

// NVRTC has no C library headers: the engine headers only need these names.
const char* kStdintStub =
    "#pragma once\n"
    "typedef unsigned long long uint64_t; typedef long long int64_t;\n"
    "typedef unsigned int uint32_t; typedef int int32_t;\n"
    "typedef unsigned short uint16_t; typedef short int16_t;\n"
    "typedef unsigned char uint8_t; typedef signed char int8_t;\n";

// The fixed NVRTC options (part of the on-disk cache key): the CTA size the
// host library was built for is compiled in (shared-memory layout, launch
// bounds), so libraries built for different sizes never share a cubin.
const std::vector<std::string>& nvrtcOptions() {
  static const std::vector<std::string> o = {"-arch=sm_100a", "-std=c++17", "-fmad=false",
                                             "-lineinfo", "-DCLTK_JIT=1",
                                             "-DCLTK_BLOCK=" + std::to_string(kBlock),
                                             "-DCLTK_MAX_BATCH=" + std::to_string(CLTK_MAX_BATCH),
                                             "-DCLTK_MAX_ASSETS=" + std::to_string(CLTK_MAX_ASSETS)};
  return o;
}

std::vector<uint8_t> compileCubin(const std::string& src, std::string* log) {
  Nvrtc& n = nvrtc();
  if (!n.ok) throw UnsupportedError("jit: " + n.why);
  std::vector<const char*> names, bodies;
  for (int i = 0; i < kJitHeaderCount; ++i) {
    names.push_back(kJitHeaderNames[i]);
    bodies.push_back(kJitHeaderSources[i]);
  }
  names.push_back("stdint.h");
  bodies.push_back(kStdintStub);
  names.push_back("math.h");
  bodies.push_back("#pragma once\n");
  nvrtcProgram prog;
  nvrtcResult r = n.create(&prog, src.c_str(), "cltk_jit_path.cu", static_cast<int>(names.size()),
                           bodies.data(), names.data());
  if (r != NVRTC_SUCCESS) throw UnsupportedError(std::string("jit: nvrtc: ") + n.errstr(r));
  std::vector<std::string> extra;  // CLTK_JIT_FLAGS: extra NVRTC options (experiments)
  if (const char* f = std::getenv("CLTK_JIT_FLAGS")) {
    std::istringstream is(f);
    for (std::string t; is >> t;) extra.push_back(t);
  }
  std::vector<const char*> opts;
  for (const std::string& o : nvrtcOptions()) opts.push_back(o.c_str());
  for (const std::string& t : extra) opts.push_back(t.c_str());
  r = n.compile(prog, static_cast<int>(opts.size()), opts.data());
  size_t ls = 0;
  n.logSize(prog, &ls);
  std::string lg(ls, '\0');
  if (ls) n.log(prog, &lg[0]);
  if (log) *log = lg;
  if (r != NVRTC_SUCCESS) {
    n.destroy(&prog);
    throw UnsupportedError(std::string("jit: nvrtc compile failed: ") + n.errstr(r) + "\n" +
                           lg.substr(0, 2000));
  }
  size_t cs = 0;
  n.cubinSize(prog, &cs);
  std::vector<uint8_t> cubin(cs);
  n.cubin(prog, reinterpret_cast<char*>(cubin.data()));
  n.destroy(&prog);
  if (const char* dump = std::getenv("CLTK_JIT_DUMP")) {  // inspection: cuobjdump -sass
    if (FILE* f = std::fopen(dump, "wb")) {
      std::fwrite(cubin.data(), 1, cubin.size(), f);
      std::fclose(f);
    }
  }
  return cubin;
}

// ---------------------------------------------------------------------------
// Code generation
// ---------------------------------------------------------------------------
struct DOp {
  uint32_t op, d, a, b, c;
};

uint32_t fieldOf(uint64_t w, int sh) { return static_cast<uint32_t>(w >> sh) & 0x3fffu; }

// The ops of packed[b, e) with VEC run headers expanded (run_ops semantics).
std::vector<DOp> decode(const std::vector<uint64_t>& packed, uint32_t b, uint32_t e) {
  std::vector<DOp> out;
  for (uint32_t pc = b; pc < e;) {
    const uint64_t w = packed[pc++];
    const uint32_t op = static_cast<uint32_t>(w & 0xff);
    if (op == OP_VEC) {
      const uint32_t n = fieldOf(w, 8), vop = fieldOf(w, 22);
      for (uint32_t i = 0; i < n; ++i) {
        const uint64_t u = packed[pc + i];
        out.push_back({vop, fieldOf(u, 8), fieldOf(u, 22), fieldOf(u, 36), fieldOf(u, 50)});
      }
      pc += n;
      continue;
    }
    out.push_back({op, fieldOf(w, 8), fieldOf(w, 22), fieldOf(w, 36), fieldOf(w, 50)});
  }
  return out;
}

bool usesA(uint32_t op) { return op != OP_NOP; }
bool usesB(uint32_t op) {
  switch (op) {
    case OP_NOP: case OP_MOV: case OP_NEG: case OP_NOT: case OP_EDIVZ: return false;
    default: return true;
  }
}

// The expression of one op over locals a, b, c (run_ops in engine_device.cuh).
std::string opExpr(const DOp& o) {
  switch (o.op) {
    case OP_MOV: return "a";
    case OP_NEG: return "-a";
    case OP_NOT: return "(a == 0.0 ? 1.0 : 0.0)";
    case OP_ADD: return "__dadd_rn(a, b)";
    case OP_SUB: return "__dsub_rn(a, b)";
    case OP_MUL: return "__dmul_rn(a, b)";
    case OP_DIV: return "__ddiv_rn(a, b)";
    case OP_LT: return "(a < b ? 1.0 : 0.0)";
    case OP_LEQ: return "(a <= b ? 1.0 : 0.0)";
    case OP_EQ: return "(a == b ? 1.0 : 0.0)";
    case OP_AND: return "((a != 0.0 && b != 0.0) ? 1.0 : 0.0)";
    case OP_OR: return "((a != 0.0 || b != 0.0) ? 1.0 : 0.0)";
    case OP_SEL: return "(a != 0.0 ? b : c)";
    case OP_IADD:
      return "of_bits(static_cast<int64_t>(static_cast<uint64_t>(bits_of(a)) + "
             "static_cast<uint64_t>(bits_of(b))))";
    case OP_ISUB:
      return "of_bits(static_cast<int64_t>(static_cast<uint64_t>(bits_of(a)) - "
             "static_cast<uint64_t>(bits_of(b))))";
    case OP_ILT: return "(bits_of(a) < bits_of(b) ? 1.0 : 0.0)";
    case OP_ILEQ: return "(bits_of(a) <= bits_of(b) ? 1.0 : 0.0)";
    case OP_IEQ: return "(bits_of(a) == bits_of(b) ? 1.0 : 0.0)";
    case OP_MIN: return "fmin(a, b)";
    case OP_MAX: return "fmax(a, b)";
    case OP_MINP:
      return "((isnan(a) || isnan(b)) ? __longlong_as_double(0x7ff8000000000000LL) : fmin(a, b))";
    case OP_MAXP:
      return "((isnan(a) || isnan(b)) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(a, b))";
    case OP_EFIRST: return "(bits_of(a) != 0 ? a : b)";
    case OP_EDIVZ:
      return "(a == 0.0 ? of_bits(static_cast<int64_t>(" + std::to_string(o.c) + "ll)) : 0.0)";
    default: return "0.0";
  }
}

struct Gen {
  const CompiledProgram& prog;
  uint32_t nA, nThread;
  bool sRegs;
  bool copyInst = false;  // something outside inst() reads the instance literal pool
  uint32_t nc = 0, ni = 0;

  std::string opnd(uint32_t i, bool inStep) const {
    if (i < nA && inStep && sRegs) return "S[" + std::to_string(i) + "]";
    if (i < nThread) return "JR(" + std::to_string(i) + ")";
    // instance literals straight from the table (L1-resident, warp-broadcast)
    if (!copyInst && i >= nThread + nc && i < nThread + nc + ni)
      return "JI(" + std::to_string(i - nThread - nc) + ")";
    return "JC(" + std::to_string(i) + ")";
  }
  // Readers of each thread register outside a given block: other blocks, the
  // outputs.  Block ids: step classes 1..C, the instance section C + 1.
  std::map<uint32_t, std::set<uint32_t>> readBy;
  std::set<uint32_t> outRead;

  void noteReads(const std::vector<DOp>& ops, uint32_t block) {
    for (const DOp& o : ops) {
      if (o.op == OP_NOP) continue;
      if (o.a < nThread) readBy[o.a].insert(block);
      if (usesB(o.op) && o.b < nThread) readBy[o.b].insert(block);
      if (o.op == OP_SEL && o.c < nThread) readBy[o.c].insert(block);
    }
  }

  // Log-domain spots (logMode, engine_device.cuh: spot_exp / log_fmin): a
  // step receives the logarithms L[j] of its spots; S[j] = exp(L[j]) is
  // formed only where an op needs the spot itself, and running minima /
  // maxima of spots (fmin / fmax of two log-capable operands: a slot or a
  // log-domain value) stay logarithms, exponentiated once where something
  // else reads them.  A thread register carries a log-domain value across
  // steps when every step-class occurrence sees it in the same domain
  // (entryDom, found by simulating the step sequence in jitSource); noLog
  // registers are always stored as values.
  bool logMode = false;
  std::set<uint32_t> noLog;
  // registers a step class stores as values although they are log-domain
  // there: the last writer of a running extremum that the outputs or the
  // instance section read (exp once per path instead of once per step)
  std::map<uint32_t, std::set<uint32_t>> exitValue;
  std::map<uint32_t, std::map<uint32_t, int>> entryDom;  // class -> register -> 1 if log

  struct Val {
    std::string log, val;  // log form (log-domain value) and/or value form
    bool spot = false;     // the value is a spot: exp of a bounded log-spot (> 0, in
                           // [2^-722, 2^722]) or a min / max / select of such
  };

  // Divisions by instance literals in the instance-major section (inst_t):
  // a spot divided by a literal whose every instance value lies in
  // [2^-100, 2^100] is rounded from the literal's host-computed reciprocal
  // RN(1/b) (an extra instance-literal column) in three operations --
  // q = RN(a y), r = a - b q (exact), RN(q + r y) = RN(a/b) (Markstein's
  // theorem; operands and quotient far from over/underflow) -- instead of a
  // full IEEE division per (path, instance).
  bool spotOK = false;                // spots are exps of bounded log-spots
  std::set<uint32_t> spotRegs;        // registers that hold spots whenever read
  std::set<uint32_t> recipOK;         // instance-literal columns usable as divisors
  uint32_t niCols = 0;                // instance-literal columns before the reciprocals
  mutable std::map<uint32_t, uint32_t> recipCol;     // literal column -> reciprocal column
  // the same for divisions by shared constants in any block: their
  // reciprocals are appended to the shared-constant table (JC); not with
  // copyInst (the instance literals then follow the shared ones in the table)
  std::set<uint32_t> recipSharedOK;   // shared-constant slots usable as divisors
  uint32_t ncBase = 0;                // shared constants before the reciprocals
  mutable std::map<uint32_t, uint32_t> recipShared;  // slot -> reciprocal slot
  mutable std::map<uint32_t, int>* storeRec = nullptr;  // analysis: register -> all stores spot

  // Straight-line emission of one block with its values in locals: a register
  // is loaded from its shared-memory column at its first read in the block (if
  // not yet written there), every op result is a new local, and at the end a
  // register is stored back only if something outside the block can read it
  // (another block, the outputs, or this block's next occurrence -- a read
  // before the write).  Same ops, same order, same IEEE operations (log-domain
  // minima / maxima: bitwise the same results).  Returns the domain (1: log)
  // of every register written in the block.
  // final: instance-major variant of the instance section -- instance
  // literals always from the table (per-lane instances), nothing stored; the
  // registers' final values are handed back instead.  The warp constants it
  // reads are collected in *kc and read as k.c[n]: loaded once per row of
  // paths (inst_k), not once per (path, instance); the path's registers in
  // *kr, read as r.c[n] (inst_r: loaded once per path for two instances).
  std::map<uint32_t, int> emit(std::ostringstream& os, const std::vector<DOp>& ops, bool inStep,
                               uint32_t block, const char* ind,
                               std::map<uint32_t, std::string>* final = nullptr,
                               std::vector<uint32_t>* kc = nullptr,
                               std::vector<uint32_t>* kr = nullptr) const {
    std::map<uint32_t, Val> cur;
    std::map<uint32_t, Val> slotVal;  // materialised spots of this block
    std::set<uint32_t> dirty, carried;
    int n = 0;
    const bool lm = logMode && inStep && sRegs;
    const auto ent = entryDom.find(block);
    if (inStep && !sRegs)
      for (uint32_t j = 0; j < nA; ++j) {
        cur[j] = Val{"", "S[" + std::to_string(j) + "]"};
        dirty.insert(j);
      }
    auto fresh = [&]() { return "v" + std::to_string(n++); };
    auto operand = [&](uint32_t i) -> Val {
      if (i < nA && inStep && sRegs) {
        if (!lm) return Val{"", "S[" + std::to_string(i) + "]", prog.header.log_bounded != 0};
        auto it = slotVal.find(i);
        if (it != slotVal.end()) return it->second;
        return slotVal[i] = Val{"L[" + std::to_string(i) + "]", ""};
      }
      auto it = cur.find(i);
      if (it != cur.end()) return it->second;
      const std::string v = fresh();
      std::string src;
      bool isLog = false;
      if (i < nThread) {
        carried.insert(i);
        if (kr) {
          src = "r.c[" + std::to_string(kr->size()) + "]";
          kr->push_back(i);
        } else {
          src = "JR(" + std::to_string(i) + ")";
        }
        if (ent != entryDom.end()) {
          auto e = ent->second.find(i);
          isLog = e != ent->second.end() && e->second;
        }
      } else if ((!copyInst || final) && i >= nThread + nc && i < nThread + nc + ni) {
        // instance literals straight from the table (L1-resident, broadcast)
        src = "JI(" + std::to_string(i - nThread - nc) + ")";
      } else if (kc) {
        src = "k.c[" + std::to_string(kc->size()) + "]";
        kc->push_back(i);
      } else {
        src = "JC(" + std::to_string(i) + ")";
      }
      os << ind << "const double " << v << " = " << src << ";\n";
      return cur[i] = isLog ? Val{v, ""} : Val{"", v, i < nThread && spotRegs.count(i) > 0};
    };
    // the value form of operand i (exp of a log-domain value, formed once)
    auto value = [&](uint32_t i) -> std::string {
      Val x = operand(i);
      if (!x.val.empty()) return x.val;
      const std::string v = fresh();
      os << ind << "const double " << v << " = " << (prog.header.log_bounded ? "spot_exp_b(" : "spot_exp(")
         << x.log << ");\n";
      x.val = v;
      x.spot = spotOK;
      if (i < nA && inStep && sRegs) slotVal[i] = x;
      else cur[i] = x;
      return v;
    };
    for (const DOp& o : ops) {
      if (o.op == OP_NOP) continue;
      Val res;
      const std::string t = o.op == OP_MOV ? std::string() : fresh();
      if (o.op == OP_MOV) {
        res = operand(o.a);  // a copy: the same local(s)
      } else if (lm && (o.op == OP_MIN || o.op == OP_MAX) && !operand(o.a).log.empty() &&
                 !operand(o.b).log.empty()) {
        const std::string a = operand(o.a).log, b = operand(o.b).log;
        const char* fn = prog.header.log_bounded ? (o.op == OP_MIN ? "log_fmin_b(" : "log_fmax_b(")
                                                 : (o.op == OP_MIN ? "log_fmin(" : "log_fmax(");
        os << ind << "const double " << t << " = " << fn
           << a << ", " << b << ");\n";
        res = Val{t, ""};
      } else {
        const std::string a = value(o.a);
        const std::string b = usesB(o.op) ? value(o.b) : std::string();
        const std::string c = o.op == OP_SEL ? value(o.c) : std::string();
        const bool sa = operand(o.a).spot, sb = usesB(o.op) && operand(o.b).spot,
                   sc = o.op == OP_SEL && operand(o.c).spot;
        const uint32_t lit0 = nThread + nc;
        std::string expr = opExpr(o);
        if (final && spotOK && o.op == OP_DIV && sa && o.b >= lit0 && o.b < lit0 + ni &&
            recipOK.count(o.b - lit0)) {
          auto rc = recipCol.find(o.b - lit0);
          if (rc == recipCol.end())
            rc = recipCol.emplace(o.b - lit0, niCols + static_cast<uint32_t>(recipCol.size())).first;
          expr = "div_recip(a, b, JI(" + std::to_string(rc->second) + "))";
        } else if (spotOK && o.op == OP_DIV && sa && o.b >= nThread && o.b < lit0 &&
                   recipSharedOK.count(o.b - nThread)) {
          auto rc = recipShared.find(o.b - nThread);
          if (rc == recipShared.end())
            rc = recipShared.emplace(o.b - nThread,
                                     ncBase + static_cast<uint32_t>(recipShared.size())).first;
          expr = "div_recip(a, b, JC(" + std::to_string(nThread + rc->second) + "))";
        }
        os << ind << "double " << t << ";\n" << ind << "{ const double a = " << a << ";";
        if (!b.empty()) os << " const double b = " << b << ";";
        if (!c.empty()) os << " const double c = " << c << ";";
        os << " " << t << " = " << expr << "; }\n";
        res = Val{"", t};
        if ((o.op == OP_MIN || o.op == OP_MAX) && sa && sb) res.spot = true;
        if (o.op == OP_SEL && sb && sc) res.spot = true;
      }
      cur[o.d] = res;
      if (!res.log.empty() && noLog.count(o.d)) value(o.d);  // stored as a value
      dirty.insert(o.d);
    }
    std::map<uint32_t, int> exitDom;
    if (final) {
      for (uint32_t r : dirty) (*final)[r] = cur[r].val.empty() ? cur[r].log : cur[r].val;
      return exitDom;
    }
    const auto ev = exitValue.find(block);
    for (uint32_t r : dirty) {
      if (ev != exitValue.end() && ev->second.count(r) && cur[r].val.empty()) value(r);
      const Val& x = cur[r];
      const bool isLog = x.val.empty();
      exitDom[r] = isLog ? 1 : 0;
      bool live = outRead.count(r) || carried.count(r);
      auto it = readBy.find(r);
      if (!live && it != readBy.end())
        for (uint32_t bl : it->second)
          if (bl != block) live = true;
      if (live) os << ind << "JW(" << r << ", " << (isLog ? x.log : x.val) << ");\n";
      if (live && storeRec) {
        const int sp = (isLog || x.spot) ? 1 : 0;  // a log-domain store reads back as a spot
        auto it = storeRec->find(r);
        if (it == storeRec->end()) storeRec->emplace(r, sp);
        else it->second = std::min(it->second, sp);
      }
    }
    return exitDom;
  }

  // Registers a block reads before writing them (its entry state).
  static std::set<uint32_t> readsFirst(const std::vector<DOp>& ops, uint32_t nThread) {
    std::set<uint32_t> w, r;
    auto rd = [&](uint32_t i) {
      if (i < nThread && !w.count(i)) r.insert(i);
    };
    for (const DOp& o : ops) {
      if (o.op == OP_NOP) continue;
      rd(o.a);
      if (usesB(o.op)) rd(o.b);
      if (o.op == OP_SEL) rd(o.c);
      w.insert(o.d);
    }
    return r;
  }
};

}  // namespace

bool jitAvailable(std::string* why) {
  Nvrtc& n = nvrtc();
  if (!n.ok && why) *why = n.why;
  return n.ok;
}

size_t jitOpCount(const CompiledProgram& prog) {
  std::map<std::vector<uint64_t>, int> seen;
  size_t n = 0;
  for (const cltk_step& st : prog.steps) {
    std::vector<uint64_t> key(prog.packed.begin() + st.code_begin,
                              prog.packed.begin() + st.code_end);
    if (key.empty() || seen.count(key)) continue;
    seen[key] = 1;
    n += decode(prog.packed, st.code_begin, st.code_end).size();
  }
  const cltk_plan_header& h = prog.header;
  n += decode(prog.packed, h.inst_code_begin, h.inst_code_end).size();
  return n;
}

std::string jitSource(CompiledProgram& prog) {
  const cltk_plan_header& h = prog.header;
  const uint32_t nA = h.n_assets ? h.n_assets : 1;
  Gen g{prog, h.n_assets, h.n_thread, true};
  // Spots come straight from registers unless something reads or writes the
  // S-slots outside a step's own ops (then they are stored like the
  // interpreter stores them).
  const std::vector<DOp> instOps = decode(prog.packed, h.inst_code_begin, h.inst_code_end);
  for (const DOp& o : instOps) {
    if (o.op == OP_NOP) continue;
    if (o.a < h.n_assets || (usesB(o.op) && o.b < h.n_assets) ||
        (o.op == OP_SEL && o.c < h.n_assets) || o.d < h.n_assets)
      g.sRegs = false;
  }
  g.nc = h.n_shared_const;
  g.ni = h.n_inst_const;
  const uint32_t instLo = h.n_thread + h.n_shared_const, instHi = instLo + h.n_inst_const;
  for (const cltk_output& o : prog.outputs) {
    if (o.val < h.n_assets || (o.err != CLTK_NO_ERR && o.err < h.n_assets)) g.sRegs = false;
    if ((o.val >= instLo && o.val < instHi) ||
        (o.err != CLTK_NO_ERR && o.err >= instLo && o.err < instHi))
      g.copyInst = true;
  }
  std::map<std::vector<uint64_t>, uint32_t> classes;
  std::vector<std::vector<DOp>> classOps(1);
  for (cltk_step& st : prog.steps) {
    std::vector<uint64_t> key(prog.packed.begin() + st.code_begin,
                              prog.packed.begin() + st.code_end);
    if (key.empty()) {
      st.jit_class = 0;
      continue;
    }
    auto it = classes.find(key);
    if (it == classes.end()) {
      const uint32_t id = static_cast<uint32_t>(classOps.size());
      it = classes.emplace(key, id).first;
      classOps.push_back(decode(prog.packed, st.code_begin, st.code_end));
      for (const DOp& o : classOps.back())
        if (o.op != OP_NOP && o.d < h.n_assets) g.sRegs = false;
    }
    st.jit_class = it->second;
  }
  // S-slots in registers: no shared-memory columns for them
  prog.header.reg_base = g.sRegs ? h.n_assets : 0;
  const uint32_t instBlock = static_cast<uint32_t>(classOps.size());
  for (size_t c = 1; c < classOps.size(); ++c) g.noteReads(classOps[c], static_cast<uint32_t>(c));
  g.noteReads(instOps, instBlock);
  for (const cltk_output& o : prog.outputs) {
    if (o.val < h.n_thread) g.outRead.insert(o.val);
    if (o.err != CLTK_NO_ERR && o.err < h.n_thread) g.outRead.insert(o.err);
  }
  // Log-domain spots: find each step class's entry domains by running the
  // step sequence.  A register still log-domain when the outputs / the
  // instance section read it is first stored as a value by the class that
  // last writes it (exitValue); a register seen in two domains at one class's
  // entry (or whose exit conversion caused that) is stored as a value
  // everywhere (noLog); the sequence is re-run after each change.
  g.logMode = g.sRegs && std::getenv("CLTK_JIT_NO_LOGSPOTS") == nullptr;
  if (g.logMode) {
    std::vector<std::set<uint32_t>> firstReads(classOps.size());
    for (size_t c = 1; c < classOps.size(); ++c)
      firstReads[c] = Gen::readsFirst(classOps[c], h.n_thread);
    std::set<uint32_t> endReads(g.outRead);
    for (uint32_t r : Gen::readsFirst(instOps, h.n_thread)) endReads.insert(r);
    std::set<uint32_t> triedExit;
    for (;;) {
      g.entryDom.clear();
      std::map<uint32_t, std::map<uint32_t, int>> exitDom;  // per class, fixed entries
      std::map<uint32_t, int> dom;
      std::map<uint32_t, uint32_t> lastWriter;  // register -> class that wrote it last
      uint32_t bad = ~0u;
      bool atEnd = false;
      for (const cltk_step& st : prog.steps) {
        const uint32_t c = st.jit_class;
        if (c == 0) continue;
        const bool first = !g.entryDom.count(c);
        std::map<uint32_t, int>& ent = g.entryDom[c];
        for (uint32_t r : firstReads[c]) {
          const int d = dom.count(r) ? dom[r] : 0;
          if (first) ent[r] = d;
          else if (ent[r] != d) bad = r;
        }
        if (bad != ~0u) break;
        if (first) {
          std::ostringstream dry;
          exitDom[c] = g.emit(dry, classOps[c], true, c, "");
        }
        for (const auto& kv : exitDom[c]) {
          dom[kv.first] = kv.second;
          lastWriter[kv.first] = c;
        }
      }
      if (bad == ~0u)
        for (uint32_t r : endReads)
          if (dom.count(r) && dom[r]) {
            bad = r;
            atEnd = true;
          }
      if (bad == ~0u) break;
      if (atEnd && !triedExit.count(bad) && lastWriter.count(bad)) {
        g.exitValue[lastWriter[bad]].insert(bad);
        triedExit.insert(bad);
        continue;
      }
      for (auto& kv : g.exitValue) kv.second.erase(bad);
      g.noLog.insert(bad);
    }
  }
  // Spot registers (for the instance section's reciprocal divisions): start
  // from every thread register and keep those whose every store in the step
  // classes is a spot or a log-spot, to a fixed point.
  g.spotOK = g.logMode && h.log_bounded != 0;
  g.niCols = h.n_inst_const;
  g.ncBase = h.n_shared_const;
  if (g.spotOK && !g.copyInst) {
    // shared constants that are safe divisors (the divisions are by R operands)
    for (uint32_t k = 0; k < h.n_shared_const && k < prog.sharedConst.size(); ++k) {
      const double v = prog.sharedConst[k];
      if (std::isfinite(v) && v >= 0x1.0p-100 && v <= 0x1.0p+100) g.recipSharedOK.insert(k);
    }
  }
  if (g.spotOK && h.inst_major && h.n_inst_const) {
    for (uint32_t r = h.n_assets; r < h.n_thread; ++r) g.spotRegs.insert(r);
    for (;;) {
      std::map<uint32_t, int> rec;
      g.storeRec = &rec;
      for (size_t c = 1; c < classOps.size(); ++c) {
        std::ostringstream dry;
        g.emit(dry, classOps[c], true, static_cast<uint32_t>(c), "");
      }
      g.storeRec = nullptr;
      std::set<uint32_t> next;
      for (uint32_t r : g.spotRegs) {
        const auto it = rec.find(r);
        if (it != rec.end() && it->second) next.insert(r);
      }
      if (next == g.spotRegs) break;
      g.spotRegs.swap(next);
    }
    // literal columns whose every instance value is a safe divisor
    const size_t nInst = h.n_instances, ni = h.n_inst_const;
    for (uint32_t k = 0; k < ni; ++k) {
      bool ok = prog.instConst.size() >= nInst * ni;
      for (size_t i = 0; i < nInst && ok; ++i) {
        const double v = prog.instConst[i * ni + k];
        ok = std::isfinite(v) && v >= 0x1.0p-100 && v <= 0x1.0p+100;
      }
      if (ok) g.recipOK.insert(k);
    }
  }
  std::ostringstream os;
  os << "// Generated by cltk-b200 jit.cpp: payoff policy for one compiled program.\n"
        "#define CLTK_JIT 1\n"
        "#include \"engine_device.cuh\"\n"
        "namespace cltk {\nnamespace b200 {\nnamespace {\n"
        "static_assert(sizeof(DevPlan) == "
     << sizeof(DevPlan) << ", \"DevPlan layout\");\nstatic_assert(sizeof(RunArgs) == "
     << sizeof(RunArgs) << ", \"RunArgs layout\");\nstatic_assert(sizeof(cltk_step_hdr) == "
     << sizeof(cltk_step_hdr)
     << ", \"cltk_step_hdr layout\");\n"
        "#define JR(i) lds64(f.R + (i) * (kBlock * 8u))\n"
        "#define JW(i, v) sts64(f.R + (i) * (kBlock * 8u), (v))\n"
        "#define JC(i) lds64(f.C + (i) * 8u)\n"
        "#define JI(k) __ldg(P.instConst + static_cast<size_t>(inst) * P.hdr.n_inst_const + (k))\n"
        "struct JitPayoff {\n"
        "  static constexpr bool kCopyInstConst = "
     << (g.copyInst ? "true" : "false") << ";\n"
        "  static constexpr bool kLogSpots = "
     << (g.logMode ? "true" : "false") << ";\n"
        "  static constexpr bool kInstT = true;  // inst_t below (instance-major batches)\n"
        "  template <int NA>\n"
        "  static __device__ __forceinline__ void step(const Frame f, const DevPlan& P,\n"
        "                                              const StepRef st, const double (&"
     << (g.logMode ? "L" : "S") << ")[NA]) {\n"
        "    switch (__ldg(&st.h->jit_class)) {\n";
  for (size_t c = 1; c < classOps.size(); ++c) {
    os << "      case " << c << ": {\n";
    g.emit(os, classOps[c], true, static_cast<uint32_t>(c), "        ");
    os << "        break;\n      }\n";
  }
  os << "      default: break;\n    }\n  }\n"
        "  static __device__ __forceinline__ void inst(const Frame f, const DevPlan& P,\n"
        "                                              uint32_t inst) {\n";
  g.emit(os, instOps, false, instBlock, "    ");
  os << "  }\n";
  // Instance-major reduction of template batches (header.inst_major): the
  // instance section for one (path, instance) returning the day's output; f
  // is the PATH's frame (its thread's register columns), inst this lane's
  // instance (engine_device.cuh path_body).
  // The warp constants it reads come in k (inst_k: loaded once per row of
  // paths by the caller, outside its loops over paths and instances), the
  // path's register columns in r (inst_r: once per path, shared by the two
  // instances a lane evaluates).
  {
    std::ostringstream body;
    std::vector<uint32_t> kc, kr;
    if (h.inst_major && !prog.outputs.empty()) {
      std::map<uint32_t, std::string> fin;
      g.emit(body, instOps, false, instBlock, "    ", &fin, &kc, &kr);
      const uint32_t v = prog.outputs[0].val;
      std::string ret;
      if (fin.count(v)) {
        ret = fin[v];
      } else if (v < h.n_thread) {
        ret = "r.c[" + std::to_string(kr.size()) + "]";
        kr.push_back(v);
      } else if (v >= instLo && v < instHi) {
        ret = "JI(" + std::to_string(v - instLo) + ")";
      } else {
        ret = "k.c[" + std::to_string(kc.size()) + "]";
        kc.push_back(v);
      }
      body << "    return " << ret << ";\n";
    } else {
      body << "    return 0.0;\n";
    }
    auto table = [&](const char* type, const char* fn, const char* arg, const char* macro,
                     const std::vector<uint32_t>& ix) {
      os << "  struct " << type << " {\n    double c[" << std::max<size_t>(ix.size(), 1)
         << "];\n  };\n  static __device__ __forceinline__ " << type << " " << fn
         << "(const Frame f) {\n    " << type << " " << arg << ";\n";
      for (size_t n = 0; n < ix.size(); ++n)
        os << "    " << arg << ".c[" << n << "] = " << macro << "(" << ix[n] << ");\n";
      if (ix.empty()) os << "    " << arg << ".c[0] = 0.0;\n";
      os << "    return " << arg << ";\n  }\n";
    };
    table("InstK", "inst_k", "k", "JC", kc);
    table("InstR", "inst_r", "r", "JR", kr);
    os << "  static __device__ __forceinline__ double inst_t(const DevPlan& P, uint32_t inst,\n"
          "                                                const InstK& k, const InstR& r) {\n"
       << body.str();
  }
  os << "  }\n};\n}  // namespace\n}  // namespace b200\n}  // namespace cltk\n"
        "extern \"C\" __global__ void __launch_bounds__(cltk::b200::kBlock, "
     << (h.rng == CLTK_RNG_SOBOL ? "CLTK_QMC_MIN_BLOCKS" : "CLTK_MIN_BLOCKS") << ")\n"
        "cltk_jit_path(const cltk::b200::DevPlan P, const cltk::b200::RunArgs A, int accInSmem) {\n"
        "  cltk::b200::path_body<"
     << nA << ", " << (h.rng == CLTK_RNG_SOBOL ? "true" : "false") << ", cltk::b200::JitPayoff, "
     << (prog.faultBuild ? "true" : "false")
     << ", " << (h.reg_acc ? 1 : 0) << ", " << (h.stream ? 1 : 0) << ", "
     << (h.inst_major ? 1 : 0) << ">(P, A, accInSmem);\n}\n";
  // the reciprocal shared constants the steps divide by, RN(1/b) on the host
  if (!g.recipShared.empty()) {
    prog.sharedConst.resize(g.ncBase + g.recipShared.size());
    for (const auto& kv : g.recipShared) prog.sharedConst[kv.second] = 1.0 / prog.sharedConst[kv.first];
    prog.header.n_shared_const = static_cast<uint32_t>(prog.sharedConst.size());
  }
  // the reciprocal columns the instance section divides by: RN(1/b) per
  // instance, computed here (IEEE division on the host)
  if (!g.recipCol.empty()) {
    const size_t nInst = h.n_instances, ni = g.niCols, nn = ni + g.recipCol.size();
    std::vector<double> t(nInst * nn);
    for (size_t i = 0; i < nInst; ++i) {
      for (size_t k = 0; k < ni; ++k) t[i * nn + k] = prog.instConst[i * ni + k];
      for (const auto& kv : g.recipCol) t[i * nn + kv.second] = 1.0 / prog.instConst[i * ni + kv.first];
    }
    prog.instConst.swap(t);
    prog.header.n_inst_const = static_cast<uint32_t>(nn);
  }
  // Shared-memory register columns: only the registers the generated code
  // stores or loads (JW / JR) or the outputs read; the rest live in locals.
  std::string src = os.str();
  uint32_t top = prog.header.reg_base;
  for (const char* pat : {"JR(", "JW("}) {
    for (size_t at = src.find(pat); at != std::string::npos; at = src.find(pat, at + 3)) {
      const char* q = src.c_str() + at + 3;
      if (*q < '0' || *q > '9') continue;  // the macro definitions
      top = std::max<uint32_t>(top, static_cast<uint32_t>(std::strtoul(q, nullptr, 10)) + 1);
    }
  }
  for (const cltk_output& o : prog.outputs) {
    if (o.val < h.n_thread) top = std::max(top, o.val + 1);
    if (o.err != CLTK_NO_ERR && o.err < h.n_thread) top = std::max(top, o.err + 1);
  }
  prog.header.reg_top = std::min<uint32_t>(top, h.n_thread);
  return src;
}

size_t jitCompileOnly(const std::string& src, std::string* log) {
  return compileCubin(src, log).size();
}

namespace {
// On-disk cubin cache (best effort): a program compiled once on a machine is
// loaded by later processes without NVRTC.  Keyed by the generated source,
// the embedded engine headers and the extra NVRTC flags (FNV-1a 64).
// Directory: $CLTK_JIT_CACHE_DIR, else $XDG_CACHE_HOME/cltk_b200, else
// $HOME/.cache/cltk_b200; CLTK_JIT_CACHE_DIR="" disables it.
uint64_t fnv1a(uint64_t h, const std::string& s) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001B3ULL;
  }
  return h;
}
std::string cacheDir() {
  if (const char* d = std::getenv("CLTK_JIT_CACHE_DIR")) return d;
  if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) return std::string(x) + "/cltk_b200";
  if (const char* h = std::getenv("HOME"); h && *h) return std::string(h) + "/.cache/cltk_b200";
  return "";
}
std::string cachePath(const std::string& src) {
  const std::string dir = cacheDir();
  if (dir.empty()) return "";
  uint64_t h = fnv1a(0xCBF29CE484222325ULL, src);
  for (int i = 0; i < kJitHeaderCount; ++i) h = fnv1a(h, kJitHeaderSources[i]);
  for (const std::string& o : nvrtcOptions()) h = fnv1a(h, o);
  if (const char* f = std::getenv("CLTK_JIT_FLAGS")) h = fnv1a(h, f);
  char name[40];
  std::snprintf(name, sizeof name, "/%016llx.cubin", static_cast<unsigned long long>(h));
  return dir + name;
}
bool readFile(const std::string& path, std::vector<uint8_t>* out) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out->resize(n > 0 ? static_cast<size_t>(n) : 0);
  const bool ok = n > 0 && std::fread(out->data(), 1, out->size(), f) == out->size();
  std::fclose(f);
  return ok;
}
void writeFileAtomic(const std::string& path, const std::vector<uint8_t>& data) {
  const std::string dir = path.substr(0, path.rfind('/'));
  std::error_code ec;  // best effort: no shell, no exception
  std::filesystem::create_directories(dir, ec);
  if (ec) return;
  const std::string tmp = path + ".tmp" + std::to_string(static_cast<long>(getpid()));
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;
  const bool ok = std::fwrite(data.data(), 1, data.size(), f) == data.size();
  std::fclose(f);
  if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
}
}  // namespace

namespace {
// Load a cubin and find the path kernel; false (error in *e) if either fails.
bool loadKernel(const std::vector<uint8_t>& cubin, cudaKernel_t* k, cudaError_t* e,
                const char** what) {
  cudaLibrary_t lib;
  *what = "cudaLibraryLoadData";
  *e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (*e != cudaSuccess) return false;
  *what = "cudaLibraryGetKernel";
  *e = cudaLibraryGetKernel(k, lib, "cltk_jit_path");
  if (*e != cudaSuccess) {
    cudaLibraryUnload(lib);
    return false;
  }
  return true;
}
bool looksLikeCubin(const std::vector<uint8_t>& b) {
  return b.size() > 64 && b[0] == 0x7f && b[1] == 'E' && b[2] == 'L' && b[3] == 'F';
}
}  // namespace

const void* jitKernel(const std::string& src) {
  static std::mutex mu;
  static std::unordered_map<std::string, cudaKernel_t> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(src);
  if (it != cache.end()) return reinterpret_cast<const void*>(it->second);
  const std::string path = cachePath(src);
  std::vector<uint8_t> cubin;
  cudaKernel_t k;
  cudaError_t e = cudaSuccess;
  const char* what = "";
  // a cached cubin is used only if it is an ELF image that loads and holds the
  // kernel; anything else (stale, damaged) is recompiled and rewritten
  bool ok = !path.empty() && readFile(path, &cubin) && looksLikeCubin(cubin) &&
            loadKernel(cubin, &k, &e, &what);
  if (!ok) {
    cudaGetLastError();  // clear a failed load of a damaged entry
    std::string log;
    cubin = compileCubin(src, &log);
    if (!path.empty()) writeFileAtomic(path, cubin);
    if (!loadKernel(cubin, &k, &e, &what))
      throw DeviceError(std::string("jit: ") + what + ": " + cudaGetErrorString(e));
  }
  cache.emplace(src, k);
  return reinterpret_cast<const void*>(k);
}

}  // namespace b200
}  // namespace cltk
