// reindex: compiled-contract IL -> flattened kernel (the producer in front of
// the pricing path).  Restates the reference's KernelBuilder
// (proj/src/kernel.cpp:14-180, reindex :301-303) over the IL's JSON wire
// format (ilToJson / ilFromJson, proj/src/json_io.cpp:19-71, 203-303):
//   * TExprVal / Payoff / Model times are evaluated with the template
//     environment (tExprSem / tExprZSem / tSem, proj/src/ilsem.cpp:54-66,
//     proj/src/semantics.cpp:115-117) and become row indices;
//   * rows are materialised as contiguous blocks [day, day + slack], slack =
//     the sum of the enclosing LoopIf windows (ensureRows, kernel.cpp:47-79);
//   * cols / tvars / parties are numbered in first-occurrence order;
//   * horizon = max(row day, 0) + 1 (kernel.cpp:28-31).
// The visiting order of every node (and so every index it creates) is the
// reference's; tests/test_reindex.py compares the output with the reference's
// kernelToJson for every golden contract, cut and uncut.
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "cltk_b200.hpp"

namespace cltk {
namespace b200 {

using Json = nlohmann::json;

namespace {

[[noreturn]] void badIL(const std::string& what) {
  throw ParseError("parse error at 0:0: IL JSON: " + what);
}

const std::string& kindOf(const Json& j) {
  if (!j.is_object() || !j.contains("kind") || !j.at("kind").is_string()) badIL("node without kind");
  return j.at("kind").get_ref<const std::string&>();
}

class Builder {
 public:
  Builder(const TEnv& tenv, Kernel& k) : tenv_(tenv), k_(k) {}

  void build(const Json& il) {
    k_.root = rewrite(il, 0);
    int64_t maxDay = 0;
    for (int64_t d : k_.rows) maxDay = std::max(maxDay, d);
    k_.horizon = static_cast<uint64_t>(maxDay) + 1;
  }

 private:
  const TEnv& tenv_;
  Kernel& k_;
  std::map<int64_t, std::size_t> firstRow_;
  std::map<std::string, std::size_t> colIndex_, tvarIndex_;
  std::map<std::string, int32_t> partyName_;

  // ensureRows (kernel.cpp:47-79): the row block of days day .. day + slack.
  // Blocks are contiguous so that loop-relative offsets stay inside them.  The
  // block already starting at `day` is reused when the rows that follow it
  // continue the run day + 1, day + 2, ... (it may grow at the end of the
  // table); otherwise a fresh block is appended -- a day can then own rows in
  // several blocks, and firstRow_ keeps its first.
  std::size_t ensureRows(int64_t day, uint64_t slack) {
    std::vector<int64_t>& rows = k_.rows;
    const auto append = [&](int64_t d) {
      rows.push_back(d);
      firstRow_.emplace(d, rows.size() - 1);
    };
    const auto hit = firstRow_.find(day);
    if (hit != firstRow_.end()) {
      const std::size_t base = hit->second;
      const uint64_t present = std::min<uint64_t>(rows.size() - base - 1, slack);
      uint64_t k = 1;
      while (k <= present && rows[base + k] == day + static_cast<int64_t>(k)) ++k;
      if (k > present) {
        for (uint64_t e = present + 1; e <= slack; ++e) append(day + static_cast<int64_t>(e));
        return base;
      }
    }
    const std::size_t base = rows.size();
    for (uint64_t e = 0; e <= slack; ++e) append(day + static_cast<int64_t>(e));
    return base;
  }

  // first-use numbering of column labels and template variables
  template <class K>
  static std::size_t intern(std::map<K, std::size_t>& index, std::vector<K>& order, const K& key) {
    const auto found = index.find(key);
    if (found != index.end()) return found->second;
    order.push_back(key);
    return index[key] = order.size() - 1;
  }
  std::size_t colOf(const std::string& label) { return intern(colIndex_, k_.cols, label); }
  std::size_t tvarOf(const std::string& name) { return intern(tvarIndex_, k_.tvars, name); }
  void noteParty(const std::string& p) {
    if (std::find(k_.parties.begin(), k_.parties.end(), p) == k_.parties.end())
      k_.parties.push_back(p);
  }
  int32_t partyIndex(const std::string& p) {  // interned PayRef strings (Kernel::partyNames)
    auto [it, inserted] = partyName_.try_emplace(p, static_cast<int32_t>(k_.partyNames.size()));
    if (inserted) k_.partyNames.push_back(p);
    return it->second;
  }

  // TExpr {"kind": "tnum" | "tvar"} (json_io.cpp:61-71); tSem (semantics.cpp:115)
  static bool isNum(const Json& t) { return kindOf(t) == "tnum"; }
  uint64_t tSem(const Json& t) const {
    const std::string& k = kindOf(t);
    if (k == "tnum") return t.at("value").get<uint64_t>();
    if (k == "tvar") return tenv_.lookup(t.at("name").get<std::string>());
    badIL("unknown TExpr kind " + k);
  }
  // ILTExpr {"tplus" | "texpr"} (json_io.cpp:24-37); tExprSem (ilsem.cpp:54-58)
  uint64_t tExprSem(const Json& t) const {
    const std::string& k = kindOf(t);
    if (k == "tplus") return tExprSem(t.at("left")) + tExprSem(t.at("right"));
    if (k == "texpr") return tSem(t.at("value"));
    badIL("unknown ILTExpr kind " + k);
  }
  // ILTExprZ {"tplusz" | "texprz" | "tnumz"} (json_io.cpp:39-57); tExprZSem (ilsem.cpp:60-66)
  int64_t tExprZSem(const Json& t) const {
    const std::string& k = kindOf(t);
    if (k == "tplusz") return tExprZSem(t.at("left")) + tExprZSem(t.at("right"));
    if (k == "texprz") return static_cast<int64_t>(tExprSem(t.at("value")));
    if (k == "tnumz") return t.at("value").get<int64_t>();
    badIL("unknown ILTExprZ kind " + k);
  }
  // collectTVarsT / collectTVarsZ (kernel.cpp:97-114): left before right
  void collectT(const Json& t) {
    if (kindOf(t) == "tplus") {
      collectT(t.at("left"));
      collectT(t.at("right"));
      return;
    }
    const Json& te = t.at("value");
    if (!isNum(te)) tvarOf(te.at("name").get<std::string>());
  }
  void collectZ(const Json& t) {
    const std::string& k = kindOf(t);
    if (k == "tplusz") {
      collectZ(t.at("left"));
      collectZ(t.at("right"));
      return;
    }
    if (k == "texprz") collectT(t.at("value"));
  }

  int32_t push(const KNode& n) {
    k_.nodes.push_back(n);
    return static_cast<int32_t>(k_.nodes.size() - 1);
  }

  // KernelBuilder::rewrite (kernel.cpp:116-176)
  int32_t rewrite(const Json& il, uint64_t slack) {
    const std::string& kind = kindOf(il);
    KNode n;
    if (kind == "if") {
      n.kind = KKind::If;
      n.a = rewrite(il.at("cond"), slack);
      n.b = rewrite(il.at("then"), slack);
      n.c = rewrite(il.at("else"), slack);
    } else if (kind == "float") {
      n.kind = KKind::Float;
      n.real = il.at("value").get<double>();
    } else if (kind == "nat") {
      n.kind = KKind::Nat;
      n.nat = il.at("value").get<uint64_t>();
    } else if (kind == "bool") {
      n.kind = KKind::Bool;
      n.boolean = il.at("value").get<bool>();
    } else if (kind == "texprval") {
      const Json& t = il.at("value");
      collectT(t);
      const int64_t day = static_cast<int64_t>(tExprSem(t));
      n.kind = KKind::TimeRef;
      n.row = ensureRows(day, slack);
    } else if (kind == "now") {
      n.kind = KKind::Now;
    } else if (kind == "model") {
      const Json& t = il.at("time");
      collectZ(t);
      const int64_t day = tExprZSem(t);
      n.kind = KKind::ObsRef;
      n.row = ensureRows(day, slack);
      n.col = colOf(il.at("label").get<std::string>());
    } else if (kind == "unop") {
      const std::string& op = il.at("op").get_ref<const std::string&>();
      if (op != "neg" && op != "not") badIL("unknown IL unary operator " + op);
      n.kind = KKind::UnOp;
      n.op = static_cast<int>(op == "neg" ? KUn::Neg : KUn::Not);
      n.a = rewrite(il.at("arg"), slack);
    } else if (kind == "binop") {
      static const std::map<std::string, KBin> ops = {
          {"add", KBin::Add}, {"sub", KBin::Sub}, {"mult", KBin::Mult},
          {"div", KBin::Div}, {"lt", KBin::Lt},   {"leq", KBin::Leq},
          {"eq", KBin::Eq},   {"and", KBin::And}, {"or", KBin::Or}};
      auto it = ops.find(il.at("op").get<std::string>());
      if (it == ops.end()) badIL("unknown IL binary operator " + il.at("op").get<std::string>());
      n.kind = KKind::BinOp;
      n.op = static_cast<int>(it->second);
      n.a = rewrite(il.at("left"), slack);
      n.b = rewrite(il.at("right"), slack);
    } else if (kind == "loopif") {
      const Json& w = il.at("window");
      n.kind = KKind::LoopIf;
      n.nat = tSem(w);
      if (!isNum(w)) n.wvar = static_cast<int32_t>(tvarOf(w.at("name").get<std::string>()));
      n.a = rewrite(il.at("cond"), slack + n.nat);
      n.b = rewrite(il.at("then"), slack + n.nat);
      n.c = rewrite(il.at("else"), slack + n.nat);
    } else if (kind == "payoff") {
      const Json& t = il.at("time");
      collectT(t);
      const std::string from = il.at("from").get<std::string>();
      const std::string to = il.at("to").get<std::string>();
      noteParty(from);
      noteParty(to);
      const int64_t day = static_cast<int64_t>(tExprSem(t));
      n.kind = KKind::PayRef;
      n.row = ensureRows(day, slack);
      n.from = partyIndex(from);
      n.to = partyIndex(to);
    } else {
      badIL("unknown ILExpr kind " + kind);
    }
    return push(n);
  }
};

const char* binName(int op) {
  static const char* names[] = {"add", "sub", "mult", "div", "lt", "leq", "eq", "and", "or"};
  return names[op];
}

Json nodeJson(const Kernel& k, int32_t i) {
  const KNode& n = k.nodes[static_cast<std::size_t>(i)];
  switch (n.kind) {
    case KKind::If:
      return {{"kind", "if"}, {"cond", nodeJson(k, n.a)}, {"then", nodeJson(k, n.b)},
              {"else", nodeJson(k, n.c)}};
    case KKind::Float: return {{"kind", "float"}, {"value", n.real}};
    case KKind::Nat: return {{"kind", "nat"}, {"value", n.nat}};
    case KKind::Bool: return {{"kind", "bool"}, {"value", n.boolean}};
    case KKind::Now: return {{"kind", "now"}};
    case KKind::TimeRef: return {{"kind", "timeref"}, {"row", n.row}};
    case KKind::ObsRef: return {{"kind", "obsref"}, {"row", n.row}, {"col", n.col}};
    case KKind::PayRef:
      return {{"kind", "payref"}, {"row", n.row},
              {"from", k.partyNames[static_cast<std::size_t>(n.from)]},
              {"to", k.partyNames[static_cast<std::size_t>(n.to)]}};
    case KKind::UnOp:
      return {{"kind", "unop"}, {"op", n.op == static_cast<int>(KUn::Neg) ? "neg" : "not"},
              {"arg", nodeJson(k, n.a)}};
    case KKind::BinOp:
      return {{"kind", "binop"}, {"op", binName(n.op)}, {"left", nodeJson(k, n.a)},
              {"right", nodeJson(k, n.b)}};
    case KKind::LoopIf: {
      Json j = {{"kind", "loopif"}, {"cond", nodeJson(k, n.a)}, {"then", nodeJson(k, n.b)},
                {"else", nodeJson(k, n.c)}, {"window", n.nat}};
      if (n.wvar >= 0) j["windowVar"] = n.wvar;
      return j;
    }
  }
  return {};
}

}  // namespace

Kernel kernelFromIL(const std::string& ilJson, const TEnv& tenv) {
  Kernel k;
  try {
    const Json il = Json::parse(ilJson);
    Builder(tenv, k).build(il);
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    throw ParseError(std::string("parse error at 0:0: IL JSON: ") + e.what());
  }
  return k;
}

std::string kernelToJsonString(const Kernel& k) {
  if (k.root < 0) throw UnsupportedError("empty kernel");
  const Json j = {{"body", nodeJson(k, k.root)}, {"rows", k.rows},   {"cols", k.cols},
                  {"tvars", k.tvars},            {"parties", k.parties}, {"horizon", k.horizon}};
  return j.dump();
}

}  // namespace b200
}  // namespace cltk
