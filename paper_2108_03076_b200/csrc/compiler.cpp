// Payoff compiler (see compiler.hpp for the contract).  Host-only C++;
// compiled with -ffp-contract=off so host-folded constants are the IEEE
// results the reference computes at run time.
#include "compiler.hpp"
#include "engine_types.h"

#include <algorithm>
#include <cmath>
#include <functional>
#include <cstring>
#include <nlohmann/json.hpp>
#include <sstream>
#include <unordered_map>

namespace cltk {
namespace b200 {

// ---------------------------------------------------------------------------
// SimPlan (proj/src/pricing.cpp:173-212, 214-253)
// ---------------------------------------------------------------------------
namespace {

// QMC mode: Brownian bridge over the drawing steps' times tau (years from
// day 0).  Nodes are numbered breadth-first (node 0 = W(T), then interval
// midpoints level by level -- the order that gives the low Sobol
// dimensions to the coarse structure); the device evaluates them in a
// pre-order traversal that *emits* W(tau_s) in time order, so the path is
// streamed with O(log n) live values (slots) instead of being materialised.
void buildBridge(SimPlanHost& p, const std::vector<uint32_t>& drawSteps,
                 const std::vector<double>& tau) {
  const int nD = static_cast<int>(drawSteps.size());
  if (nD == 0) return;
  std::vector<int> node(nD, -1), L(nD, -2), R(nD, -2);
  auto T = [&](int i) { return i < 0 ? 0.0 : tau[i]; };
  node[nD - 1] = 0;
  int next = 1;
  std::vector<std::pair<int, int>> q{{-1, nD - 1}};
  for (std::size_t h = 0; h < q.size(); ++h) {
    auto [l, r] = q[h];
    if (r - l < 2) continue;
    const int m = l + (r - l) / 2;
    node[m] = next++;
    L[m] = l;
    R[m] = r;
    q.push_back({l, m});
    q.push_back({m, r});
  }
  // traversal: COMPUTE in pre-order, EMIT in order (= time order)
  struct Ev {
    bool emit;
    int m;
  };
  std::vector<Ev> seq{{false, nD - 1}};
  // iterative in-order over the bisection tree of (-1, nD-1)
  std::function<void(int, int)> visit = [&](int l, int r) {
    if (r - l < 2) return;
    const int m = l + (r - l) / 2;
    seq.push_back({false, m});
    visit(l, m);
    seq.push_back({true, m});
    visit(m, r);
  };
  visit(-1, nD - 1);
  seq.push_back({true, nD - 1});
  // last use of every point: its emit, or a compute that reads it
  std::vector<int> lastUse(nD, -1);
  for (int t = 0; t < static_cast<int>(seq.size()); ++t) {
    const Ev& e = seq[t];
    if (e.emit) {
      lastUse[e.m] = std::max(lastUse[e.m], t);
    } else {
      if (L[e.m] >= 0) lastUse[L[e.m]] = std::max(lastUse[L[e.m]], t);
      if (R[e.m] >= 0) lastUse[R[e.m]] = std::max(lastUse[R[e.m]], t);
    }
  }
  std::vector<int> slot(nD, -1), freeSlots;
  int nSlots = 0;
  uint32_t emitted = 0;
  std::vector<std::vector<int>> releaseAt(seq.size() + 1);
  for (int t = 0; t < static_cast<int>(seq.size()); ++t) {
    const Ev& e = seq[t];
    if (!e.emit) {
      int s;
      if (!freeSlots.empty()) {
        s = freeSlots.back();
        freeSlots.pop_back();
      } else {
        s = nSlots++;
      }
      slot[e.m] = s;
      cltk_bridge_op op{};
      const int l = L[e.m], r = R[e.m];
      if (e.m == nD - 1) {  // W(T) = sqrt(T) Z
        op.wl = 0.0;
        op.wr = 0.0;
        op.sd = std::sqrt(T(nD - 1));
        op.l = op.r = CLTK_BR_ORIGIN;
      } else {
        const double tl = T(l), tr = T(r), tm = T(e.m);
        op.wl = (tr - tm) / (tr - tl);
        op.wr = (tm - tl) / (tr - tl);
        op.sd = std::sqrt((tm - tl) * (tr - tm) / (tr - tl));
        op.l = l < 0 ? CLTK_BR_ORIGIN : static_cast<uint16_t>(slot[l]);
        op.r = static_cast<uint16_t>(slot[r]);
      }
      op.dst = static_cast<uint16_t>(s);
      op.node = static_cast<uint32_t>(node[e.m]);
      p.bridge.push_back(op);
    } else {
      cltk_step& st = p.steps[drawSteps[emitted]];
      st.br_end = static_cast<uint32_t>(p.bridge.size());
      st.br_emit = static_cast<uint32_t>(slot[e.m]);
      if (emitted + 1 < drawSteps.size())
        p.steps[drawSteps[emitted + 1]].br_begin = static_cast<uint32_t>(p.bridge.size());
      ++emitted;
    }
    // free the slots whose last use was this event (after it executed)
    if (e.emit) {
      if (lastUse[e.m] == t) freeSlots.push_back(slot[e.m]);
    } else {
      for (int x : {L[e.m], R[e.m]})
        if (x >= 0 && lastUse[x] == t) freeSlots.push_back(slot[x]);
    }
  }
  p.steps[drawSteps[0]].br_begin = 0;
  p.bridgeSlots = static_cast<uint32_t>(nSlots);
}

}  // namespace

SimPlanHost buildSimPlan(const Kernel& k, const ModelSpec& model, uint32_t rng) {
  SimPlanHost p;
  p.rng = rng;
  p.days = k.rows;
  std::sort(p.days.begin(), p.days.end());
  p.days.erase(std::unique(p.days.begin(), p.days.end()), p.days.end());
  if (!p.days.empty() && p.days.front() < 0)
    throw EvalError("cannot simulate a negative observation day");
  for (int64_t d : k.rows)
    p.rowToDay.push_back(static_cast<uint32_t>(
        std::lower_bound(p.days.begin(), p.days.end(), d) - p.days.begin()));
  for (const auto& label : k.cols) {
    auto it = std::find(model.order.begin(), model.order.end(), label);
    if (it == model.order.end()) throw EvalError("model has no asset spec for label " + label);
    p.colToAsset.push_back(static_cast<uint32_t>(it - model.order.begin()));
  }
  std::size_t n = model.order.size();
  std::vector<std::vector<double>> chol;
  if (model.corr.empty()) {
    chol.assign(n, std::vector<double>(n, 0.0));
    for (std::size_t i = 0; i < n; ++i) chol[i][i] = 1.0;
  } else {
    if (model.corr.size() != model.order.size())
      throw EvalError("correlation matrix size does not match asset count");
    chol = cholesky(model.corr);
  }
  for (int64_t d : k.rows)
    p.disc.push_back(std::exp(-model.rate * static_cast<double>(d) / model.dayCount));
  if (n > CLTK_MAX_ASSETS)
    throw UnsupportedError("engine supports at most " + std::to_string(CLTK_MAX_ASSETS) +
                           " model assets, model has " + std::to_string(n));
  if (rng == CLTK_RNG_SOBOL && n > CLTK_AOT_MAX_ASSETS)
    throw UnsupportedError("QMC mode supports at most " + std::to_string(CLTK_AOT_MAX_ASSETS) +
                           " model assets, model has " + std::to_string(n));
  p.nAssets = static_cast<uint32_t>(n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) p.chol[i * n + j] = chol[i][j];  // packed rows of n
  // Per-step constants, in the reference's operation order.
  std::vector<const AssetSpec*> spec(n);
  for (std::size_t j = 0; j < n; ++j) {
    spec[j] = &model.at(model.order[j]);
    p.logS0[j] = std::log(spec[j]->spot);
  }
  int64_t prev = 0;
  bool drawn = false;
  for (std::size_t s = 0; s < p.days.size(); ++s) {
    cltk_step st;
    std::memset(&st, 0, sizeof st);
    double dt = static_cast<double>(p.days[s] - prev) / model.dayCount;
    prev = p.days[s];
    if (dt > 0.0) {
      st.draws = STEP_DRAW;
      drawn = true;
      for (std::size_t j = 0; j < n; ++j) {
        const AssetSpec& a = *spec[j];
        st.A[j] = (a.drift - 0.5 * a.vol * a.vol) * dt;
        st.B[j] = a.vol * std::sqrt(dt);
      }
    } else if (!drawn) {
      st.draws = STEP_CONST_S;  // path-independent: exp(log(spot)) on the host
      for (std::size_t j = 0; j < n; ++j) st.S[j] = std::exp(p.logS0[j]);
    } else {
      st.draws = STEP_EXP_ONLY;
    }
    p.steps.push_back(st);
  }
  const uint32_t nA32 = static_cast<uint32_t>(std::max<std::size_t>(1, n));
  for (std::size_t s = 0; s < p.steps.size(); ++s) {
    uint32_t w = 0;
    for (uint32_t q = 0; (q + 1) * nA32 <= 32 && s + q < p.steps.size(); ++q)
      if (p.steps[s + q].draws == STEP_DRAW)
        w |= static_cast<uint32_t>((uint64_t{1} << nA32) - 1) << (q * nA32);
    p.steps[s].draw_window = w;
  }
  for (uint32_t a : p.colToAsset) p.usedMask |= 1u << a;
  if (rng == CLTK_RNG_SOBOL) {
    // Same GBM in closed form over the bridge's W(t): logS(t) = log(spot)
    // + (drift - vol^2/2) t + vol (L W(t))
    std::vector<uint32_t> drawSteps;
    std::vector<double> tau;
    for (std::size_t s = 0; s < p.steps.size(); ++s) {
      if (p.steps[s].draws != STEP_DRAW) continue;
      const double t = static_cast<double>(p.days[s]) / model.dayCount;
      drawSteps.push_back(static_cast<uint32_t>(s));
      tau.push_back(t);
      for (std::size_t j = 0; j < n; ++j) {
        const AssetSpec& a = *spec[j];
        p.steps[s].A[j] = (a.drift - 0.5 * a.vol * a.vol) * t;
        p.steps[s].B[j] = a.vol;
      }
    }
    if (drawSteps.size() * n > CLTK_SOBOL_MAX_DIMS)
      throw UnsupportedError("Sobol mode supports at most " + std::to_string(CLTK_SOBOL_MAX_DIMS) +
                             " dimensions (drawing days x assets); this plan needs " +
                             std::to_string(drawSteps.size() * n));
    buildBridge(p, drawSteps, tau);
  }
  return p;
}

namespace {

using Json = nlohmann::json;

enum class VT : uint8_t { R = 0, B = 1, I = 2, E = 3 };
const char* vtName(VT t) {
  switch (t) {
    case VT::R: return "R";
    case VT::B: return "B";
    case VT::I: return "I";
    default: return "E";
  }
}

// Leaf "opcodes" of the DAG (device opcodes are < OP_COUNT).
enum : uint32_t { D_CONST = 200, D_LIT = 201, D_OBS = 202 };

struct DNode {
  uint32_t op;
  VT type;
  int32_t a = -1, b = -1, c = -1;
  uint64_t bits = 0;  // CONST value bits / LIT slot / OBS (step<<8|asset) / EDIVZ site
  bool inst = false;
  int32_t step = -1;
};

uint64_t dbits(double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
}
double bitsd(uint64_t u) {
  double v;
  std::memcpy(&v, &u, 8);
  return v;
}

struct Dag {
  std::vector<DNode> n;
  std::unordered_map<std::string, int32_t> memo;

  int32_t make(const DNode& d) {
    char key[64];
    std::memcpy(key, &d.op, 4);
    key[4] = static_cast<char>(d.type);
    std::memcpy(key + 5, &d.a, 4);
    std::memcpy(key + 9, &d.b, 4);
    std::memcpy(key + 13, &d.c, 4);
    std::memcpy(key + 17, &d.bits, 8);
    std::string k(key, 25);
    auto it = memo.find(k);
    if (it != memo.end()) return it->second;
    DNode x = d;
    if (x.op == D_LIT) {
      x.inst = true;
      x.step = -1;
    } else if (x.op == D_OBS) {
      x.step = static_cast<int32_t>(x.bits >> 8);
    } else if (x.op != D_CONST) {
      for (int32_t ch : {x.a, x.b, x.c})
        if (ch >= 0) {
          x.inst = x.inst || n[ch].inst;
          x.step = std::max(x.step, n[ch].step);
        }
    }
    n.push_back(x);
    int32_t id = static_cast<int32_t>(n.size() - 1);
    memo.emplace(std::move(k), id);
    return id;
  }
  bool isConst(int32_t i) const { return i >= 0 && n[i].op == D_CONST; }
  bool isConstLike(int32_t i) const {
    return i >= 0 && (n[i].op == D_CONST || n[i].op == D_LIT) && n[i].type == VT::R;
  }
  double rv(int32_t i) const { return bitsd(n[i].bits); }
  int64_t iv(int32_t i) const { return static_cast<int64_t>(n[i].bits); }
  VT type(int32_t i) const { return n[i].type; }
};

// Value + error channel of one specialised expression.  v < 0: the
// expression always raises (its error channel is then a nonzero constant).
struct Val {
  int32_t v;
  int32_t e;
};

class Builder {
 public:
  Dag g;
  std::vector<ErrorSite> sites;
  std::map<std::pair<int, std::string>, uint32_t> siteIdx;

  Builder() {
    sites.push_back({ErrorCode::Eval, "no error"});
    sites.push_back({ErrorCode::Eval, "invNormalCdf domain error"});  // site 1
  }

  uint32_t site(ErrorCode c, const std::string& m) {
    auto key = std::make_pair(static_cast<int>(c), m);
    auto it = siteIdx.find(key);
    if (it != siteIdx.end()) return it->second;
    // the device error word is path << 24 | site (engine_device.cuh)
    if (sites.size() >= (1u << 24)) throw UnsupportedError("more than 2^24 error sites");
    sites.push_back({c, m});
    uint32_t id = static_cast<uint32_t>(sites.size() - 1);
    siteIdx.emplace(key, id);
    return id;
  }

  // -- leaves ---------------------------------------------------------------
  int32_t leaf(uint32_t op, VT t, uint64_t bits) {
    DNode d;
    d.op = op;
    d.type = t;
    d.bits = bits;
    return g.make(d);
  }
  int32_t cR(double v) { return leaf(D_CONST, VT::R, dbits(v)); }
  int32_t cB(bool v) { return leaf(D_CONST, VT::B, v ? 1 : 0); }
  int32_t cI(int64_t v) { return leaf(D_CONST, VT::I, static_cast<uint64_t>(v)); }
  int32_t cE(uint32_t s) { return leaf(D_CONST, VT::E, s); }
  int32_t obs(uint32_t step, uint32_t asset) {
    return leaf(D_OBS, VT::R, (static_cast<uint64_t>(step) << 8) | asset);
  }
  int32_t lit(uint32_t slot) { return leaf(D_LIT, VT::R, slot); }

  int32_t node(uint32_t op, VT t, int32_t a, int32_t b = -1, int32_t c = -1, uint64_t bits = 0) {
    DNode d;
    d.op = op;
    d.type = t;
    d.a = a;
    d.b = b;
    d.c = c;
    d.bits = bits;
    return g.make(d);
  }

  // -- error channel --------------------------------------------------------
  int32_t efirst(int32_t e1, int32_t e2) {
    if (e1 < 0) return e2;
    if (e2 < 0) return e1;
    if (g.isConst(e1)) return g.iv(e1) != 0 ? e1 : e2;
    if (g.isConst(e2) && g.iv(e2) == 0) return e1;
    if (e1 == e2) return e1;
    return node(OP_EFIRST, VT::E, e1, e2);
  }
  int32_t esel(int32_t c, int32_t et, int32_t ef) {
    if (et < 0 && ef < 0) return -1;
    if (g.isConst(c)) return g.iv(c) ? et : ef;
    if (et == ef) return et;
    if (et < 0) et = cE(0);
    if (ef < 0) ef = cE(0);
    return node(OP_SEL, VT::E, c, et, ef);
  }
  Val fail(int32_t e, ErrorCode code, const std::string& msg) {
    return Val{-1, efirst(e, cE(site(code, msg)))};
  }

  // -- values (constant-folding smart constructors) ---------------------------
  int32_t arith(uint32_t op, int32_t x, int32_t y) {
    if (g.isConst(x) && g.isConst(y)) {
      double a = g.rv(x), b = g.rv(y), r;
      switch (op) {
        case OP_ADD: r = a + b; break;
        case OP_SUB: r = a - b; break;
        case OP_MUL: r = a * b; break;
        default: r = a / b; break;
      }
      return cR(r);
    }
    return node(op, VT::R, x, y);
  }
  int32_t cmp(uint32_t op, int32_t x, int32_t y) {
    if (g.isConst(x) && g.isConst(y)) {
      double a = g.rv(x), b = g.rv(y);
      return cB(op == OP_LT ? a < b : op == OP_LEQ ? a <= b : a == b);
    }
    return node(op, VT::B, x, y);
  }
  int32_t icmp(uint32_t op, int32_t x, int32_t y) {
    if (g.isConst(x) && g.isConst(y)) {
      int64_t a = g.iv(x), b = g.iv(y);
      return cB(op == OP_ILT ? a < b : op == OP_ILEQ ? a <= b : a == b);
    }
    return node(op, VT::B, x, y);
  }
  int32_t iarith(uint32_t op, int32_t x, int32_t y) {
    if (g.isConst(x) && g.isConst(y)) {
      uint64_t a = g.n[x].bits, b = g.n[y].bits;
      return cI(static_cast<int64_t>(op == OP_IADD ? a + b : a - b));
    }
    return node(op, VT::I, x, y);
  }
  int32_t band(int32_t x, int32_t y) {
    if (g.isConst(x)) return g.iv(x) ? y : cB(false);
    if (g.isConst(y)) return g.iv(y) ? x : cB(false);
    if (x == y) return x;
    return node(OP_AND, VT::B, x, y);
  }
  int32_t bor(int32_t x, int32_t y) {
    if (g.isConst(x)) return g.iv(x) ? cB(true) : y;
    if (g.isConst(y)) return g.iv(y) ? cB(true) : x;
    if (x == y) return x;
    return node(OP_OR, VT::B, x, y);
  }
  int32_t bnot(int32_t x) {
    if (g.isConst(x)) return cB(!g.iv(x));
    return node(OP_NOT, VT::B, x);
  }
  int32_t neg(int32_t x) {
    if (g.isConst(x)) return cR(-g.rv(x));
    return node(OP_NEG, VT::R, x);
  }
  int32_t sel(int32_t c, int32_t t, int32_t e) {
    if (g.isConst(c)) return g.iv(c) ? t : e;
    if (t == e) return t;
    return node(OP_SEL, g.type(t), c, t, e);
  }
};

// Specialises one kernel for one valuation day (t_now).
struct Specializer {
  Builder& B;
  const std::vector<uint8_t>& litNonZero;  // per variant literal slot
  const Kernel& k;
  const SimPlanHost& plan;
  const std::vector<int32_t>& litNode;  // per kernel node: DAG id of its FloatLit
  int64_t tNow;
  int32_t p1, p2;  // party indices in k.partyNames (or -1 if absent)
  std::unordered_map<uint64_t, Val> memo;
  uint64_t work = 0;

  static constexpr uint64_t kWorkLimit = 200000000ULL;

  Val eval(int32_t idx, uint64_t off) {
    uint64_t key = (static_cast<uint64_t>(idx) << 32) ^ off;
    const KNode& n = k.nodes[idx];
    bool memoize = n.kind == KKind::If || n.kind == KKind::BinOp || n.kind == KKind::LoopIf ||
                   n.kind == KKind::UnOp;
    if (memoize) {
      auto it = memo.find(key);
      if (it != memo.end()) return it->second;
    }
    if (++work > kWorkLimit)
      throw UnsupportedError("kernel too large to specialise (loop unrolling budget exceeded)");
    Val r = evalNode(n, idx, off);
    if (memoize) memo.emplace(key, r);
    return r;
  }

  // kAsReal / kAsBool checks (proj/src/kernel.cpp:186-193)
  bool isR(const Val& x) { return B.g.type(x.v) == VT::R; }
  bool isB(const Val& x) { return B.g.type(x.v) == VT::B; }
  bool isI(const Val& x) { return B.g.type(x.v) == VT::I; }

  Val evalNode(const KNode& n, int32_t idx, uint64_t off) {
    switch (n.kind) {
      case KKind::Float:
        return Val{litNode[idx], -1};
      case KKind::Nat:
        return Val{B.cI(static_cast<int64_t>(n.nat)), -1};
      case KKind::Bool:
        return Val{B.cB(n.boolean), -1};
      case KKind::Now:
        return Val{B.cI(tNow), -1};
      case KKind::TimeRef: {  // kernel.cpp:255-260
        uint64_t r = n.row + off;
        if (r >= k.rows.size())
          return B.fail(-1, ErrorCode::Eval, "kernel row index out of range");
        return Val{B.cI(k.rows[r]), -1};
      }
      case KKind::ObsRef: {  // kernel.cpp:234-240
        uint64_t r = n.row + off;
        if (r >= k.rows.size() || n.col >= k.cols.size())
          return B.fail(-1, ErrorCode::Eval,
                        "kernel input shape mismatch at ext[" + std::to_string(r) + "," +
                            std::to_string(n.col) + "]");
        return Val{B.obs(plan.rowToDay[r], plan.colToAsset[n.col]), -1};
      }
      case KKind::PayRef: {  // kernel.cpp:264-272
        uint64_t r = n.row + off;
        if (r >= plan.disc.size())
          return B.fail(-1, ErrorCode::Eval, "kernel disc index out of range");
        double d = plan.disc[r];
        if (n.from == p1 && n.to == p2) return Val{B.cR(d), -1};
        if (n.from == p2 && n.to == p1) return Val{B.cR(-d), -1};
        return Val{B.cR(0.0), -1};
      }
      case KKind::UnOp: {  // kernel.cpp:273-277
        Val x = eval(n.a, off);
        if (x.v < 0) return x;
        if (static_cast<KUn>(n.op) == KUn::Neg) {
          if (!isR(x)) return B.fail(x.e, ErrorCode::Type, "kernel: expected a Real value");
          return Val{B.neg(x.v), x.e};
        }
        if (!isB(x)) return B.fail(x.e, ErrorCode::Type, "kernel: expected a Bool value");
        return Val{B.bnot(x.v), x.e};
      }
      case KKind::BinOp: {
        Val a = eval(n.a, off);
        if (a.v < 0) return a;
        Val b = eval(n.b, off);
        int32_t e = B.efirst(a.e, b.e);
        if (b.v < 0) return Val{-1, e};
        return applyBin(static_cast<KBin>(n.op), a, b, e);
      }
      case KKind::If: {  // kernel.cpp:244-247
        Val c = eval(n.a, off);
        if (c.v < 0) return c;
        if (!isB(c)) return B.fail(c.e, ErrorCode::Type, "kernel: expected a Bool value");
        if (B.g.isConst(c.v)) {
          Val x = eval(B.g.iv(c.v) ? n.b : n.c, off);
          return Val{x.v, B.efirst(c.e, x.e)};
        }
        Val t = eval(n.b, off);
        Val f = eval(n.c, off);
        return select(c, t, f);
      }
      case KKind::LoopIf: {  // kernel.cpp:286-293, unrolled
        std::vector<std::pair<Val, Val>> arms;  // (cond, then) per offset
        uint64_t w = n.nat, cur = off;
        Val tail{-1, -1};
        bool haveTail = false;
        for (;; --w, ++cur) {
          Val c = eval(n.a, cur);
          if (c.v < 0) {
            tail = c;
            haveTail = true;
            break;
          }
          if (!isB(c)) {
            tail = B.fail(c.e, ErrorCode::Type, "kernel: expected a Bool value");
            haveTail = true;
            break;
          }
          if (B.g.isConst(c.v) && B.g.iv(c.v)) {  // statically taken: stop here
            Val t = eval(n.b, cur);
            tail = Val{t.v, B.efirst(c.e, t.e)};
            haveTail = true;
            break;
          }
          if (B.g.isConst(c.v)) {  // statically not taken
            if (w == 0) {
              Val el = eval(n.c, cur);
              tail = Val{el.v, B.efirst(c.e, el.e)};
              haveTail = true;
              break;
            }
            if (c.e >= 0) arms.push_back({c, Val{-2, -1}});  // error-only arm
            continue;
          }
          arms.push_back({c, eval(n.b, cur)});
          if (w == 0) {
            tail = eval(n.c, cur);
            haveTail = true;
            break;
          }
        }
        (void)haveTail;
        Val acc = tail;
        for (auto it = arms.rbegin(); it != arms.rend(); ++it) {
          const Val& c = it->first;
          if (it->second.v == -2) {  // constant-false cond carrying an error
            acc = Val{acc.v, B.efirst(c.e, acc.e)};
            continue;
          }
          acc = select(c, it->second, acc);
        }
        return acc;
      }
    }
    throw UnsupportedError("unknown kernel node");
  }

  // If with a data-dependent condition: eager select, error channel selected.
  Val select(const Val& c, const Val& t, const Val& f) {
    int32_t e = B.efirst(c.e, B.esel(c.v, t.e, f.e));
    if (t.v < 0 && f.v < 0) return Val{-1, e};
    if (t.v < 0) return Val{f.v, e};
    if (f.v < 0) return Val{t.v, e};
    if (B.g.type(t.v) != B.g.type(f.v))
      throw UnsupportedError(
          "kernel: if branches have different types under a data-dependent condition");
    return Val{B.sel(c.v, t.v, f.v), e};
  }

  Val needReal(const Val& x, int32_t e, bool& ok) {
    ok = isR(x);
    if (!ok) return B.fail(e, ErrorCode::Type, "kernel: expected a Real value");
    return x;
  }

  // kApplyBin (proj/src/kernel.cpp:193-225), C++ operand-check order kept.
  Val applyBin(KBin op, const Val& a, const Val& b, int32_t e) {
    bool bothInt = isI(a) && isI(b);
    auto realPair = [&](Val& out) -> bool {
      if (!isR(a)) {
        out = B.fail(e, ErrorCode::Type, "kernel: expected a Real value");
        return false;
      }
      if (!isR(b)) {
        out = B.fail(e, ErrorCode::Type, "kernel: expected a Real value");
        return false;
      }
      return true;
    };
    Val out{-1, -1};
    switch (op) {
      case KBin::Add:
      case KBin::Sub:
        if (bothInt)
          return Val{B.iarith(op == KBin::Add ? OP_IADD : OP_ISUB, a.v, b.v), e};
        if (!realPair(out)) return out;
        return Val{B.arith(op == KBin::Add ? OP_ADD : OP_SUB, a.v, b.v), e};
      case KBin::Mult:
        if (!realPair(out)) return out;
        return Val{B.arith(OP_MUL, a.v, b.v), e};
      case KBin::Div: {
        if (!isR(b)) return B.fail(e, ErrorCode::Type, "kernel: expected a Real value");
        uint32_t dz = B.site(ErrorCode::Eval, "kernel: division by zero");
        int32_t ez;
        if (B.g.isConst(b.v)) {
          if (B.g.rv(b.v) == 0.0) return Val{-1, B.efirst(e, B.cE(dz))};
          ez = -1;
        } else if (B.g.n[b.v].op == D_LIT && litNonZero[B.g.n[b.v].bits]) {
          ez = -1;  // a template literal that is non-zero in every instance
        } else {
          ez = B.node(OP_EDIVZ, VT::E, b.v, -1, -1, dz);
        }
        int32_t e2 = B.efirst(e, ez);
        if (!isR(a)) return B.fail(e2, ErrorCode::Type, "kernel: expected a Real value");
        return Val{B.arith(OP_DIV, a.v, b.v), e2};
      }
      case KBin::Lt:
      case KBin::Leq:
      case KBin::Eq: {
        uint32_t rop = op == KBin::Lt ? OP_LT : op == KBin::Leq ? OP_LEQ : OP_EQ;
        uint32_t iop = op == KBin::Lt ? OP_ILT : op == KBin::Leq ? OP_ILEQ : OP_IEQ;
        if (bothInt) return Val{B.icmp(iop, a.v, b.v), e};
        if (!realPair(out)) return out;
        return Val{B.cmp(rop, a.v, b.v), e};
      }
      case KBin::And:
      case KBin::Or: {
        // kAsBool(a) && kAsBool(b): b's check only when a does not decide.
        if (!isB(a)) return B.fail(e, ErrorCode::Type, "kernel: expected a Bool value");
        bool isAnd = op == KBin::And;
        if (!isB(b)) {
          uint32_t s = B.site(ErrorCode::Type, "kernel: expected a Bool value");
          int32_t decides = isAnd ? B.bnot(a.v) : a.v;  // a alone decides the result
          int32_t eb = B.esel(decides, -1, B.cE(s));
          int32_t e2 = B.efirst(e, eb);
          if (B.g.isConst(e2) && B.g.iv(e2) != 0) return Val{-1, e2};
          return Val{isAnd ? B.cB(false) : B.cB(true), e2};
        }
        return Val{isAnd ? B.band(a.v, b.v) : B.bor(a.v, b.v), e};
      }
    }
    throw UnsupportedError("unknown kernel operator");
  }
};

// ---------------------------------------------------------------------------
// Exact rewrite: OR/AND chains of comparisons against one literal -> running
// min/max; chains reassociated in step order.
// ---------------------------------------------------------------------------
struct Rewriter {
  const Dag& old;
  Builder& nb;  // builds into a fresh DAG (nb.g)
  std::vector<int32_t> nw;
  std::vector<uint8_t> chainRoot;  // per old node: must be materialised

  Rewriter(const Dag& o, Builder& b) : old(o), nb(b), nw(o.n.size(), -1), chainRoot(o.n.size(), 1) {}

  void markRoots(const std::vector<int32_t>& roots) {
    // An OR (AND) node is interior when every consumer is an OR (AND) node.
    std::vector<uint8_t> hasOther(old.n.size(), 0), hasUse(old.n.size(), 0);
    for (int32_t r : roots)
      if (r >= 0) hasOther[r] = 1;
    for (std::size_t i = 0; i < old.n.size(); ++i) {
      const DNode& d = old.n[i];
      for (int32_t ch : {d.a, d.b, d.c}) {
        if (ch < 0) continue;
        hasUse[ch] = 1;
        if (!((d.op == OP_OR || d.op == OP_AND) && d.op == old.n[ch].op)) hasOther[ch] = 1;
      }
    }
    for (std::size_t i = 0; i < old.n.size(); ++i) {
      const DNode& d = old.n[i];
      if ((d.op == OP_OR || d.op == OP_AND) && !hasOther[i] && hasUse[i]) chainRoot[i] = 0;
    }
  }

  void leaves(int32_t i, uint32_t op, std::vector<int32_t>& out) {
    std::vector<int32_t> stack{i};
    while (!stack.empty()) {
      int32_t x = stack.back();
      stack.pop_back();
      const DNode& d = old.n[x];
      if (d.op == op) {
        stack.push_back(d.b);
        stack.push_back(d.a);
      } else {
        out.push_back(x);
      }
    }
  }

  int32_t stepOf(int32_t i) const { return nb.g.n[i].inst ? (1 << 30) : nb.g.n[i].step; }

  int32_t chain(uint32_t op, std::vector<int32_t> xs) {
    std::stable_sort(xs.begin(), xs.end(), [&](int32_t p, int32_t q) {
      return std::make_pair(stepOf(p), p) < std::make_pair(stepOf(q), q);
    });
    xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
    int32_t acc = xs[0];
    for (std::size_t i = 1; i < xs.size(); ++i) {
      if (op == OP_OR) acc = nb.bor(acc, xs[i]);
      else if (op == OP_AND) acc = nb.band(acc, xs[i]);
      else acc = nb.node(op, VT::R, acc, xs[i]);
    }
    return acc;
  }

  int32_t rewriteChain(int32_t i) {
    uint32_t op = old.n[i].op;
    std::vector<int32_t> ls;
    leaves(i, op, ls);
    // group key: (literal node, rel op, literal on the right?)
    std::map<std::tuple<int32_t, uint32_t, int>, std::vector<int32_t>> groups;
    std::vector<std::tuple<int32_t, uint32_t, int>> order;
    std::vector<int32_t> others;
    for (int32_t l : ls) {
      int32_t m = nw[l];
      const DNode& d = nb.g.n[m];
      if ((d.op == OP_LT || d.op == OP_LEQ) && d.type == VT::B) {
        if (nb.g.isConstLike(d.b) && !nb.g.isConstLike(d.a)) {
          auto key = std::make_tuple(d.b, d.op, 1);
          if (!groups.count(key)) order.push_back(key);
          groups[key].push_back(d.a);
          continue;
        }
        if (nb.g.isConstLike(d.a) && !nb.g.isConstLike(d.b)) {
          auto key = std::make_tuple(d.a, d.op, 0);
          if (!groups.count(key)) order.push_back(key);
          groups[key].push_back(d.b);
          continue;
        }
      }
      others.push_back(m);
    }
    std::vector<int32_t> terms = others;
    for (const auto& key : order) {
      auto [L, rel, litRight] = key;
      std::vector<int32_t>& xs = groups[key];
      int32_t agg;
      if (xs.size() == 1) {
        agg = xs[0];
      } else {
        // OR: x REL L -> fmin;  L REL x -> fmax   (NaN-ignoring, exact)
        // AND: x REL L -> maxp; L REL x -> minp   (NaN-propagating, exact)
        uint32_t mop;
        if (op == OP_OR) mop = litRight ? OP_MIN : OP_MAX;
        else mop = litRight ? OP_MAXP : OP_MINP;
        agg = chain(mop, xs);
      }
      terms.push_back(litRight ? nb.cmp(rel, agg, L) : nb.cmp(rel, L, agg));
    }
    return chain(op, terms);
  }

  int32_t map(int32_t i) {
    return i < 0 ? -1 : nw[i];
  }

  void run() {
    for (std::size_t i = 0; i < old.n.size(); ++i) {
      const DNode& d = old.n[i];
      if ((d.op == OP_OR || d.op == OP_AND) && !chainRoot[i]) continue;
      if (d.op == OP_OR || d.op == OP_AND) {
        nw[i] = rewriteChain(static_cast<int32_t>(i));
        continue;
      }
      DNode x = d;
      x.a = map(d.a);
      x.b = map(d.b);
      x.c = map(d.c);
      x.inst = false;
      x.step = -1;
      nw[i] = nb.g.make(x);
    }
  }
};

const char* opName(uint32_t op) {
  static const char* names[] = {"NOP", "MOV", "NEG", "NOT", "ADD", "SUB", "MUL", "DIV",
                                "LT", "LEQ", "EQ", "AND", "OR", "SEL", "IADD", "ISUB",
                                "ILT", "ILEQ", "IEQ", "MIN", "MAX", "MINP", "MAXP",
                                "EFIRST", "EDIVZ"};
  return op < OP_COUNT ? names[op] : "?";
}

}  // namespace

std::vector<double> kernelLiterals(const Kernel& k) {
  std::vector<double> v;
  for (const KNode& n : k.nodes)
    if (n.kind == KKind::Float) v.push_back(n.real);
  return v;
}

LiteralTable literalTableFromInstances(const std::vector<const Kernel*>& instances) {
  const Kernel& k = *instances.at(0);
  const uint64_t h0 = kernelShapeHash(k);
  LiteralTable t;
  t.nInst = instances.size();
  for (std::size_t i = 0; i < instances.size(); ++i) {
    const Kernel& o = *instances[i];
    if (i > 0 && (o.nodes.size() != k.nodes.size() || kernelShapeHash(o) != h0))
      throw UnsupportedError("batch instances must share one kernel shape (instance " +
                             std::to_string(i) + " differs beyond literal values)");
    std::vector<double> v = kernelLiterals(o);
    if (i == 0) t.nOcc = v.size();
    t.values.insert(t.values.end(), v.begin(), v.end());
  }
  return t;
}

CompiledProgram compileProgram(const std::vector<const Kernel*>& instances,
                               const SimPlanHost& plan, const std::vector<uint64_t>& days,
                               const CompileOptions& opt) {
  LiteralTable t = literalTableFromInstances(instances);
  return compileProgram(*instances.at(0), t, plan, days, opt);
}

CompiledProgram compileProgram(const Kernel& k, const LiteralTable& lits, const SimPlanHost& plan,
                               const std::vector<uint64_t>& days, const CompileOptions& opt) {
  const std::size_t nInst = lits.nInst;
  if (nInst == 0) throw EvalError("no kernel instances");
  if (lits.nOcc != kernelLiterals(k).size() || lits.values.size() != nInst * lits.nOcc)
    throw UnsupportedError("literal table does not match the kernel's float literals (" +
                           std::to_string(lits.nOcc) + " per instance given)");
  // ---- literal slots: FloatLit occurrences deduplicated by their value
  //      vector across instances (shared when equal in every instance).
  Builder B;
  std::vector<int32_t> litNode(k.nodes.size(), -1);
  std::map<std::vector<uint64_t>, uint32_t> slotOf;
  std::vector<std::vector<double>> varSlots;  // variant slot -> values per instance
  std::size_t occ = 0;
  for (std::size_t idx = 0; idx < k.nodes.size(); ++idx) {
    if (k.nodes[idx].kind != KKind::Float) continue;
    std::vector<uint64_t> vec(nInst);
    bool variant = false;
    for (std::size_t i = 0; i < nInst; ++i) {
      vec[i] = dbits(lits.values[i * lits.nOcc + occ]);
      variant = variant || vec[i] != vec[0];
    }
    ++occ;
    if (!variant) {
      litNode[idx] = B.cR(bitsd(vec[0]));
      continue;
    }
    auto [it, ins] = slotOf.try_emplace(vec, static_cast<uint32_t>(varSlots.size()));
    if (ins) {
      std::vector<double> vals(nInst);
      for (std::size_t i = 0; i < nInst; ++i) vals[i] = bitsd(vec[i]);
      varSlots.push_back(vals);
    }
    litNode[idx] = B.lit(it->second);
  }
  std::vector<uint8_t> litNonZero(varSlots.size(), 1);
  for (std::size_t v = 0; v < varSlots.size(); ++v)
    for (double x : varSlots[v])
      if (x == 0.0) litNonZero[v] = 0;

  // ---- specialise each valuation day (priceAcrossTime, pricing.cpp:352-357)
  auto partyIndex = [&](const std::string& p) -> int32_t {
    for (std::size_t i = 0; i < k.partyNames.size(); ++i)
      if (k.partyNames[i] == p) return static_cast<int32_t>(i);
    return -2;  // never matches a PayRef party
  };
  const std::string p1 = k.parties.size() > 0 ? k.parties[0] : "you";
  const std::string p2 = k.parties.size() > 1 ? k.parties[1] : "me";
  std::vector<Val> outs;
  for (uint64_t d : days) {
    Specializer S{B, litNonZero, k, plan, litNode, static_cast<int64_t>(d), partyIndex(p1),
                  partyIndex(p2), {}, 0};
    Val r = S.eval(k.root, 0);
    if (r.v >= 0 && B.g.type(r.v) != VT::R)
      r = B.fail(r.e, ErrorCode::Eval, "kernel did not evaluate to a real");
    outs.push_back(r);
  }

  // ---- exact OR/AND -> min/max rewrite into a fresh DAG
  Builder R;
  R.sites = B.sites;
  R.siteIdx = B.siteIdx;
  std::vector<int32_t> roots;
  for (const Val& v : outs) {
    roots.push_back(v.v);
    roots.push_back(v.e);
  }
  Builder* GB = &B;
  std::vector<int32_t> rootMap = roots;
  if (opt.rewrite) {
    Rewriter rw(B.g, R);
    rw.markRoots(roots);
    rw.run();
    for (auto& r : rootMap) r = r >= 0 ? rw.nw[r] : -1;
    GB = &R;
  }
  // An always-raising output still needs a value operand: 0.0.
  for (std::size_t o = 0; o < outs.size(); ++o)
    if (rootMap[2 * o] < 0) rootMap[2 * o] = GB->cR(0.0);
  Dag& g = GB->g;
  const std::vector<ErrorSite>& sites = opt.rewrite ? R.sites : B.sites;

  // ---- reachability
  const int32_t N = static_cast<int32_t>(g.n.size());
  std::vector<uint8_t> live(N, 0);
  {
    std::vector<int32_t> st;
    for (int32_t r : rootMap)
      if (r >= 0 && !live[r]) {
        live[r] = 1;
        st.push_back(r);
      }
    while (!st.empty()) {
      int32_t x = st.back();
      st.pop_back();
      for (int32_t ch : {g.n[x].a, g.n[x].b, g.n[x].c})
        if (ch >= 0 && !live[ch]) {
          live[ch] = 1;
          st.push_back(ch);
        }
    }
  }
  const uint32_t nSteps = static_cast<uint32_t>(plan.days.size());
  auto isOp = [&](int32_t i) { return g.n[i].op < OP_COUNT; };
  auto sharedStep = [&](int32_t i) -> int32_t {
    // shared ops run at their ready step; ops without an observable input
    // (and every instance op) run in the end section.
    if (g.n[i].inst || g.n[i].step < 0) return -1;
    return g.n[i].step;
  };

  // ---- consumers: decide which observables need a register copy
  std::vector<int32_t> consumerMaxStep(N, -1);
  std::vector<uint8_t> usedAtEnd(N, 0);
  for (int32_t i = 0; i < N; ++i) {
    if (!live[i] || !isOp(i)) continue;
    int32_t s = sharedStep(i);
    for (int32_t ch : {g.n[i].a, g.n[i].b, g.n[i].c}) {
      if (ch < 0) continue;
      if (s < 0) usedAtEnd[ch] = 1;
      else consumerMaxStep[ch] = std::max(consumerMaxStep[ch], s);
    }
  }
  for (int32_t r : rootMap)
    if (r >= 0) usedAtEnd[r] = 1;
  std::vector<uint8_t> obsMov(N, 0);
  for (int32_t i = 0; i < N; ++i)
    if (live[i] && g.n[i].op == D_OBS)
      obsMov[i] = usedAtEnd[i] || consumerMaxStep[i] > g.n[i].step;

  // ---- linear order: per step [MOVs of that step's observables, ops], then
  //      the end section (instance ops + step-less ops)
  struct Ins {
    int32_t node;
    bool mov;
  };
  std::vector<std::vector<Ins>> perStep(nSteps);
  std::vector<Ins> endSec;
  for (int32_t i = 0; i < N; ++i) {
    if (!live[i]) continue;
    if (g.n[i].op == D_OBS && obsMov[i]) perStep[g.n[i].step].push_back({i, true});
  }
  for (int32_t i = 0; i < N; ++i) {
    if (!live[i] || !isOp(i)) continue;
    int32_t s = sharedStep(i);
    if (s < 0) endSec.push_back({i, false});
    else perStep[s].push_back({i, false});
  }
  // Within a step: MOVs first, then ops in creation (topological) order.
  for (auto& v : perStep)
    std::stable_sort(v.begin(), v.end(), [](const Ins& x, const Ins& y) { return x.mov > y.mov; });

  std::vector<Ins> linear;
  std::vector<uint32_t> stepBegin(nSteps + 1, 0);
  for (uint32_t s = 0; s < nSteps; ++s) {
    stepBegin[s] = static_cast<uint32_t>(linear.size());
    for (const Ins& x : perStep[s]) linear.push_back(x);
  }
  stepBegin[nSteps] = static_cast<uint32_t>(linear.size());
  const uint32_t endBegin = static_cast<uint32_t>(linear.size());
  for (const Ins& x : endSec) linear.push_back(x);
  const int32_t T_END = static_cast<int32_t>(linear.size());

  // ---- operand classes
  const uint32_t nA = plan.nAssets;
  std::vector<int32_t> defTime(N, -1), lastUse(N, -1);
  for (std::size_t t = 0; t < linear.size(); ++t) defTime[linear[t].node] = static_cast<int32_t>(t);
  auto needsReg = [&](int32_t i) {
    return (isOp(i) && live[i]) || (g.n[i].op == D_OBS && obsMov[i]);
  };
  for (std::size_t t = 0; t < linear.size(); ++t) {
    const Ins& x = linear[t];
    if (x.mov) continue;
    const DNode& d = g.n[x.node];
    bool inEnd = t >= endBegin;
    for (int32_t ch : {d.a, d.b, d.c}) {
      if (ch < 0 || !needsReg(ch)) continue;
      // a shared value read by the end section (re-run per instance) stays
      // live to the end; end-section temporaries die at their last read
      const bool sharedDef = defTime[ch] >= 0 && defTime[ch] < static_cast<int32_t>(endBegin);
      const bool leaf = defTime[ch] < 0;  // S-slot observable copied by MOV: defTime set
      lastUse[ch] = std::max(lastUse[ch], (inEnd && (sharedDef || leaf)) ? T_END
                                                                        : static_cast<int32_t>(t));
    }
  }
  for (int32_t r : rootMap)
    if (r >= 0 && needsReg(r)) lastUse[r] = T_END;

  // ---- register allocation (linear scan; registers after the S-slots)
  std::vector<int32_t> reg(N, -1);
  std::vector<int32_t> freeRegs;
  int32_t nRegs = 0;
  std::vector<std::vector<int32_t>> expire(T_END + 2);
  for (std::size_t t = 0; t < linear.size(); ++t) {
    // free registers whose last use precedes/equals t (safe: operands are read
    // before the destination is written)
    for (int32_t v : expire[t]) freeRegs.push_back(reg[v]);
    int32_t v = linear[t].node;
    int32_t r;
    if (!freeRegs.empty()) {
      std::sort(freeRegs.begin(), freeRegs.end(), std::greater<int32_t>());
      r = freeRegs.back();
      freeRegs.pop_back();
    } else {
      r = nRegs++;
    }
    reg[v] = r;
    int32_t lu = lastUse[v] < 0 ? static_cast<int32_t>(t) : lastUse[v];
    if (lu < T_END) {
      // Free at the last use itself: an instruction reads all operands before
      // it writes its destination, so the destination may reuse them.
      int32_t when = std::max(lu, static_cast<int32_t>(t) + 1);
      if (when <= T_END) expire[when].push_back(v);
    }
  }
  const uint32_t nThread = nA + static_cast<uint32_t>(nRegs);

  // ---- constants
  std::vector<double> sharedConst;
  std::map<uint64_t, uint32_t> constIdx;
  auto constOperand = [&](int32_t i) -> uint32_t {
    uint64_t bits;
    const DNode& d = g.n[i];
    if (d.type == VT::R) bits = d.bits;
    else if (d.type == VT::B) bits = dbits(d.bits ? 1.0 : 0.0);
    else bits = d.bits;  // I / E: int64 bit pattern
    auto [it, ins] = constIdx.try_emplace(bits, static_cast<uint32_t>(sharedConst.size()));
    if (ins) sharedConst.push_back(bitsd(bits));
    return it->second;
  };
  // Collect constants first so their count is known.
  std::vector<int32_t> constOf(N, -1);
  for (int32_t i = 0; i < N; ++i) {
    if (!live[i]) continue;
    if (g.n[i].op == D_CONST) constOf[i] = static_cast<int32_t>(constOperand(i));
  }
  const uint32_t nShared = static_cast<uint32_t>(sharedConst.size());
  const uint32_t nInstC = static_cast<uint32_t>(varSlots.size());
  if (nThread + nShared + nInstC >= CLTK_MAX_OPERANDS)
    throw UnsupportedError("compiled payoff needs too many operands");

  auto operand = [&](int32_t i, uint32_t curStep, bool inEnd) -> uint32_t {
    const DNode& d = g.n[i];
    if (d.op == D_CONST) return nThread + static_cast<uint32_t>(constOf[i]);
    if (d.op == D_LIT) return nThread + nShared + static_cast<uint32_t>(d.bits);
    if (d.op == D_OBS && !obsMov[i]) {
      (void)curStep;
      (void)inEnd;
      return static_cast<uint32_t>(d.bits & 0xff);  // S-slot
    }
    return nA + static_cast<uint32_t>(reg[i]);
  };

  // ---- emit
  CompiledProgram P;
  P.steps = plan.steps;
  P.bridge = plan.bridge;
  for (std::size_t t = 0; t < linear.size(); ++t) {
    const Ins& x = linear[t];
    const DNode& d = g.n[x.node];
    bool inEnd = t >= endBegin;
    uint32_t dst = nA + static_cast<uint32_t>(reg[x.node]);
    if (x.mov) {
      P.code.push_back(cltk_encode(OP_MOV, dst, static_cast<uint32_t>(d.bits & 0xff), 0, 0));
      continue;
    }
    uint32_t cs = inEnd ? 0 : static_cast<uint32_t>(d.step);
    uint32_t a = d.a >= 0 ? operand(d.a, cs, inEnd) : 0;
    uint32_t b = d.b >= 0 ? operand(d.b, cs, inEnd) : 0;
    uint32_t c = d.c >= 0 ? operand(d.c, cs, inEnd) : 0;
    if (d.op == OP_EDIVZ) c = static_cast<uint32_t>(d.bits);
    P.code.push_back(cltk_encode(d.op, dst, a, b, c));
  }
  // Device stream: runs of one vectorisable opcode get a VEC header so the
  // device executes them in one tight loop.  The listing keeps the plain ops.
  auto vecable = [](uint32_t op) {
    return op == OP_MIN || op == OP_MAX || op == OP_ADD || op == OP_SUB || op == OP_MUL ||
           op == OP_LT || op == OP_LEQ || op == OP_OR || op == OP_AND;
  };
  std::vector<uint32_t> packedAt(P.code.size() + 1, 0);
  auto pack = [&](uint32_t lo, uint32_t hi) {
    uint32_t i = lo;
    while (i < hi) {
      const uint32_t op = static_cast<uint32_t>(P.code[i] & 0xff);
      uint32_t j = i + 1;
      while (j < hi && static_cast<uint32_t>(P.code[j] & 0xff) == op && j - i < 0x3fff) ++j;
      if (vecable(op) && j - i >= 2) {
        P.packed.push_back(cltk_encode(OP_VEC, j - i, op, 0, 0));
        for (uint32_t k = i; k < j; ++k) P.packed.push_back(P.code[k]);
      } else {
        for (uint32_t k = i; k < j; ++k) P.packed.push_back(P.code[k]);
      }
      i = j;
    }
  };
  std::vector<uint32_t> pBegin(nSteps + 1);
  for (uint32_t s = 0; s < nSteps; ++s) {
    pBegin[s] = static_cast<uint32_t>(P.packed.size());
    pack(stepBegin[s], stepBegin[s + 1]);
  }
  pBegin[nSteps] = static_cast<uint32_t>(P.packed.size());
  const uint32_t pEndBegin = static_cast<uint32_t>(P.packed.size());
  pack(endBegin, static_cast<uint32_t>(P.code.size()));
  for (uint32_t s = 0; s < nSteps; ++s) {
    P.steps[s].code_begin = pBegin[s];
    P.steps[s].code_end = pBegin[s + 1];
  }
  uint32_t hasErr = 0;
  for (std::size_t o = 0; o < outs.size(); ++o) {
    int32_t v = rootMap[2 * o], e = rootMap[2 * o + 1];
    cltk_output out;
    out.val = operand(v, 0, true);
    out.err = e >= 0 ? operand(e, 0, true) : CLTK_NO_ERR;
    if (e >= 0) hasErr = 1;
    P.outputs.push_back(out);
  }
  P.sharedConst = sharedConst;
  P.instConst.assign(nInst * nInstC, 0.0);
  for (uint32_t s = 0; s < nInstC; ++s)
    for (std::size_t i = 0; i < nInst; ++i) P.instConst[i * nInstC + s] = varSlots[s][i];
  P.sites = sites;

  cltk_plan_header& h = P.header;
  std::memset(&h, 0, sizeof h);
  h.n_assets = nA;
  h.n_steps = nSteps;
  h.n_thread = nThread;
  h.reg_top = nThread;
  h.n_shared_const = static_cast<uint32_t>(P.sharedConst.size());
  h.n_inst_const = nInstC;
  h.n_instances = static_cast<uint32_t>(nInst);
  h.n_days = static_cast<uint32_t>(days.size());
  h.inst_code_begin = pEndBegin;
  h.inst_code_end = static_cast<uint32_t>(P.packed.size());
  h.has_err = hasErr;
  h.used_mask = plan.usedMask;
  h.rng = plan.rng;
  h.n_bridge_slots = plan.bridgeSlots;
  h.n_bridge_ops = static_cast<uint32_t>(plan.bridge.size());
  std::memcpy(h.chol, plan.chol, sizeof h.chol);
  std::memcpy(h.logS0, plan.logS0, sizeof h.logS0);
  {
    // one output and short paths: per-thread register accumulation of the
    // output in the path kernel (engine_device.cuh path_body); long paths
    // keep those registers for the normal batches
    uint64_t draws = 0;
    for (const cltk_step& st : P.steps)
      if (st.draws == STEP_DRAW) draws += nA;
    h.reg_acc = (nInst * days.size() == 1 && draws <= kRegAccMaxDraws) ? 1u : 0u;
    // short Philox paths: normal batches that run on into the next path
    // (long paths lose less to their last, partial batch than the stream's
    // per-step bookkeeping costs)
    const uint64_t slots = static_cast<uint64_t>(nSteps) * std::max<uint32_t>(1, nA);
    h.stream = (plan.rng == CLTK_RNG_PHILOX && slots <= kStreamMaxSlots) ? 1u : 0u;
    // template batches: the warp reduces instance-major (engine_device.cuh)
    h.inst_major = (nInst >= kInstMajorMin && days.size() == 1 && !hasErr) ? 1u : 0u;
    // log-spot range: |logS_j - log(spot_j)| <= sum over drawing steps of
    // |A_sj| + B_sj * sum_l |L_jl| * zmax, zmax = 8.5 > |invNormalCdf(2^-54)|
    // (the most extreme normal the generator can draw: uniforms lie in
    // [2^-54, 1 - 2^-54])
    h.log_bounded = 0;
    if (plan.rng == CLTK_RNG_PHILOX) {
      bool ok = true;
      for (uint32_t j = 0; j < nA && ok; ++j) {
        double lsum = 0.0;
        for (uint32_t l = 0; l <= j; ++l) lsum += std::fabs(plan.chol[j * nA + l]);
        double cum = std::fabs(plan.logS0[j]);
        for (const cltk_step& st : P.steps)
          if (st.draws == STEP_DRAW) cum += std::fabs(st.A[j]) + std::fabs(st.B[j]) * lsum * 8.5;
        ok = std::isfinite(cum) && cum < 500.0;
      }
      h.log_bounded = ok ? 1u : 0u;
    } else if (plan.rng == CLTK_RNG_SOBOL && !plan.bridge.empty()) {
      // QMC: logS_j(t_s) = logS0_j + A_sj + B_sj * sum_l L_jl W_l(t_s) with
      // |W_l(t_s)| bounded by running the bridge program on bounds
      // (|W_m| <= wl |W_l| + wr |W_r| + sd * zmax), zmax = 6.5 >
      // |AS241((2^32 - 1 + 0.5) 2^-32)| (32-bit Sobol points, shifted or not)
      std::vector<double> slotB(std::max<uint32_t>(1, plan.bridgeSlots), 0.0);
      auto slotBound = [&](uint16_t sl) { return sl == CLTK_BR_ORIGIN ? 0.0 : slotB[sl]; };
      bool ok = true;
      for (const cltk_step& st : P.steps) {
        if (st.draws != STEP_DRAW) continue;
        for (uint32_t b = st.br_begin; b < st.br_end; ++b) {
          const cltk_bridge_op& op = plan.bridge[b];
          slotB[op.dst] = std::fabs(op.wl) * slotBound(op.l) + std::fabs(op.wr) * slotBound(op.r) +
                          std::fabs(op.sd) * 6.5;
        }
        const double bw = slotB[st.br_emit];
        for (uint32_t j = 0; j < nA && ok; ++j) {
          double lsum = 0.0;
          for (uint32_t l = 0; l <= j; ++l) lsum += std::fabs(plan.chol[j * nA + l]);
          const double m = std::fabs(plan.logS0[j]) + std::fabs(st.A[j]) + std::fabs(st.B[j]) * lsum * bw;
          ok = std::isfinite(m) && m < 500.0;
        }
        if (!ok) break;
      }
      h.log_bounded = ok ? 1u : 0u;
    }
    h.first_draw = nSteps;
    for (uint32_t s0 = 0; s0 < nSteps; ++s0)
      if (P.steps[s0].draws == STEP_DRAW) {
        h.first_draw = s0;
        break;
      }
    if (h.stream) {
      // draw mask of a batch starting at step s: its SB steps, wrapping into
      // the next path (a chunk's paths per thread are whole stream periods,
      // so no batch runs past the chunk)
      const uint32_t na = std::max<uint32_t>(1, nA);
      const int SB = batchSteps(static_cast<int>(na));
      P.streamMask.assign(nSteps, 0u);
      for (uint32_t s0 = 0; s0 < nSteps; ++s0)
        for (int t = 0; t < SB; ++t)
          if (P.steps[(s0 + t) % nSteps].draws == STEP_DRAW)
            P.streamMask[s0] |= ((1u << na) - 1u) << (t * na);
    }
  }
  P.kernelNodes = k.nodes.size();
  P.dagNodes = static_cast<uint64_t>(N);
  P.nSharedOps = endBegin;
  P.nInstOps = static_cast<uint32_t>(linear.size()) - endBegin;

  // the listing (tests / DESIGN.md) is built on demand: programListing()
  P.stepCodeBegin = stepBegin;
  P.days = plan.days;
  return P;
}

std::string programListing(const CompiledProgram& P) {
  const cltk_plan_header& h = P.header;
  const uint32_t nA = h.n_assets, nThread = h.n_thread, nInstC = h.n_inst_const;
  const uint32_t nInst = h.n_instances, endBegin = P.nSharedOps;
  const std::vector<uint32_t>& stepBegin = P.stepCodeBegin;
  Json L;
  Json ops = Json::array();
  for (std::size_t t = 0; t < P.code.size(); ++t) {
    uint64_t w = P.code[t];
    ops.push_back({opName(static_cast<uint32_t>(w & 0xff)), (w >> 8) & 0x3fff,
                   (w >> 22) & 0x3fff, (w >> 36) & 0x3fff, (w >> 50) & 0x3fff});
  }
  L["ops"] = ops;
  Json st = Json::array();
  for (const auto& s : P.steps) {
    Json A = Json::array(), Bv = Json::array(), Sv = Json::array();
    for (uint32_t j = 0; j < nA; ++j) {
      A.push_back(s.A[j]);
      Bv.push_back(s.B[j]);
      Sv.push_back(s.S[j]);
    }
    const std::size_t si = st.size();
    st.push_back({{"kind", s.draws}, {"begin", stepBegin[si]}, {"end", stepBegin[si + 1]},
                  {"A", A}, {"B", Bv}, {"S", Sv}, {"br", {s.br_begin, s.br_end, s.br_emit}}});
  }
  L["steps"] = st;
  L["days"] = P.days;
  L["rng"] = h.rng;
  L["bridge_slots"] = h.n_bridge_slots;
  Json br = Json::array();
  for (const auto& b : P.bridge)
    br.push_back({b.node, b.dst, b.l == CLTK_BR_ORIGIN ? -1 : (int)b.l,
                  b.r == CLTK_BR_ORIGIN ? -1 : (int)b.r, b.wl, b.wr, b.sd});
  L["bridge"] = br;
  Json sc = Json::array();
  for (double v : P.sharedConst) sc.push_back(dbits(v));
  L["shared_const_bits"] = sc;
  L["inst_const"] = P.instConst;
  Json outsJ = Json::array();
  for (const auto& o : P.outputs) outsJ.push_back({o.val, o.err == CLTK_NO_ERR ? -1 : (int64_t)o.err});
  L["outputs"] = outsJ;
  Json sitesJ = Json::array();
  for (const auto& s : P.sites) sitesJ.push_back({static_cast<int>(s.code), s.message});
  L["sites"] = sitesJ;
  L["n_assets"] = nA;
  L["n_thread"] = nThread;
  L["n_shared_const"] = h.n_shared_const;
  L["n_inst_const"] = nInstC;
  L["n_instances"] = nInst;
  L["inst_code"] = {endBegin, endBegin + P.nInstOps};
  L["packed_words"] = P.packed.size();
  L["kernel_nodes"] = P.kernelNodes;
  L["dag_nodes"] = P.dagNodes;
  Json ch = Json::array();
  for (uint32_t i = 0; i < nA * nA; ++i) ch.push_back(h.chol[i]);  // rows of n_assets
  L["chol"] = ch;
  Json ls = Json::array();
  for (uint32_t j = 0; j < nA; ++j) ls.push_back(h.logS0[j]);
  L["logS0"] = ls;
  L["vt"] = {vtName(VT::R), vtName(VT::B), vtName(VT::I), vtName(VT::E)};
  return L.dump();
}

}  // namespace b200
}  // namespace cltk
