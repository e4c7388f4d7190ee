// Host-side data layer of the engine: kernel JSON reader, model JSON reader,
// Cholesky, template environment.  Semantics follow the reference line by
// line (cited per function); the representation is the engine's own
// (a flat node pool instead of a shared_ptr tree).
#include <cmath>
#include <cstring>
#include <functional>
#include <nlohmann/json.hpp>
#include <sstream>

#include "cltk_b200.hpp"

namespace cltk {
namespace b200 {

using Json = nlohmann::json;

namespace {

struct KernelReader {
  Kernel& k;
  std::map<std::string, int32_t> partyIdx;

  int32_t party(const std::string& p) {
    auto [it, ins] = partyIdx.try_emplace(p, static_cast<int32_t>(k.partyNames.size()));
    if (ins) k.partyNames.push_back(p);
    return it->second;
  }

  int32_t push(KNode n) {
    k.nodes.push_back(n);
    return static_cast<int32_t>(k.nodes.size() - 1);
  }

  // kexprFromJson (proj/src/kernel.cpp:581-627); children are emitted first.
  int32_t read(const Json& j) {
    const std::string kind = j.at("kind").get<std::string>();
    KNode n;
    if (kind == "if" || kind == "loopif") {
      n.kind = kind == "if" ? KKind::If : KKind::LoopIf;
      n.a = read(j.at("cond"));
      n.b = read(j.at("then"));
      n.c = read(j.at("else"));
      if (n.kind == KKind::LoopIf) n.nat = j.at("window").get<uint64_t>();
    } else if (kind == "float") {
      n.kind = KKind::Float;
      n.real = j.at("value").get<double>();
    } else if (kind == "nat") {
      n.kind = KKind::Nat;
      n.nat = j.at("value").get<uint64_t>();
    } else if (kind == "bool") {
      n.kind = KKind::Bool;
      n.boolean = j.at("value").get<bool>();
    } else if (kind == "now") {
      n.kind = KKind::Now;
    } else if (kind == "timeref") {
      n.kind = KKind::TimeRef;
      n.row = j.at("row").get<uint64_t>();
    } else if (kind == "obsref") {
      n.kind = KKind::ObsRef;
      n.row = j.at("row").get<uint64_t>();
      n.col = j.at("col").get<uint64_t>();
    } else if (kind == "payref") {
      n.kind = KKind::PayRef;
      n.row = j.at("row").get<uint64_t>();
      n.from = party(j.at("from").get<std::string>());
      n.to = party(j.at("to").get<std::string>());
    } else if (kind == "unop") {
      n.kind = KKind::UnOp;
      n.op = static_cast<int>(j.at("op").get<std::string>() == "neg" ? KUn::Neg : KUn::Not);
      n.a = read(j.at("arg"));
    } else if (kind == "binop") {
      static const std::map<std::string, KBin> ops = {
          {"add", KBin::Add}, {"sub", KBin::Sub}, {"mult", KBin::Mult},
          {"div", KBin::Div}, {"lt", KBin::Lt},   {"leq", KBin::Leq},
          {"eq", KBin::Eq},   {"and", KBin::And}, {"or", KBin::Or}};
      n.kind = KKind::BinOp;
      n.op = static_cast<int>(ops.at(j.at("op").get<std::string>()));
      n.a = read(j.at("left"));
      n.b = read(j.at("right"));
    } else {
      throw ParseError("parse error at 0:0: unknown kernel node kind " + kind);
    }
    return push(n);
  }
};

uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ULL + (h << 6) + (h >> 2);
  return h;
}

}  // namespace

Kernel kernelFromJson(const std::string& text) {
  Kernel k;
  try {
    Json j = Json::parse(text);
    KernelReader r{k, {}};
    k.root = r.read(j.at("body"));
    k.rows = j.at("rows").get<std::vector<int64_t>>();
    k.cols = j.at("cols").get<std::vector<std::string>>();
    k.tvars = j.at("tvars").get<std::vector<std::string>>();
    k.parties = j.at("parties").get<std::vector<std::string>>();
    k.horizon = j.at("horizon").get<uint64_t>();
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    throw ParseError(std::string("parse error at 0:0: kernel JSON: ") + e.what());
  }
  return k;
}

uint64_t kernelShapeHash(const Kernel& k) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const KNode& n : k.nodes) {
    h = mix(h, static_cast<uint64_t>(n.kind));
    h = mix(h, static_cast<uint64_t>(n.op));
    h = mix(h, static_cast<uint64_t>(static_cast<uint32_t>(n.a)));
    h = mix(h, static_cast<uint64_t>(static_cast<uint32_t>(n.b)));
    h = mix(h, static_cast<uint64_t>(static_cast<uint32_t>(n.c)));
    h = mix(h, n.row);
    h = mix(h, n.col);
    h = mix(h, n.nat);
    h = mix(h, n.boolean);
    if (n.kind == KKind::PayRef) {
      h = mix(h, std::hash<std::string>()(k.partyNames[n.from]));
      h = mix(h, std::hash<std::string>()(k.partyNames[n.to]));
    }
  }
  for (int64_t r : k.rows) h = mix(h, static_cast<uint64_t>(r));
  for (const auto& c : k.cols) h = mix(h, std::hash<std::string>()(c));
  for (const auto& p : k.parties) h = mix(h, std::hash<std::string>()(p));
  return h;
}

// ModelSpec::at (proj/src/pricing.cpp:13-18)
const AssetSpec& ModelSpec::at(const std::string& label) const {
  auto it = assets.find(label);
  if (it == assets.end()) throw EvalError("model has no asset spec for label " + label);
  return it->second;
}

// modelFromJson (proj/src/pricing.cpp:20-43)
ModelSpec modelFromJson(const std::string& text) {
  ModelSpec m;
  try {
    Json j = Json::parse(text);
    m.rate = j.value("rate", 0.0);
    m.dayCount = j.value("dayCount", 365.0);
    const auto& labels = j.at("labels");
    if (j.contains("order")) {
      m.order = j.at("order").get<std::vector<std::string>>();
    } else {
      for (auto it = labels.begin(); it != labels.end(); ++it) m.order.push_back(it.key());
      std::sort(m.order.begin(), m.order.end());
    }
    for (const auto& label : m.order) {
      const auto& spec = labels.at(label);
      AssetSpec a;
      a.spot = spec.at("spot").get<double>();
      a.vol = spec.at("vol").get<double>();
      a.drift = spec.value("drift", m.rate);
      m.assets[label] = a;
    }
    if (j.contains("corr")) m.corr = j.at("corr").get<std::vector<std::vector<double>>>();
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    throw ParseError(std::string("parse error at 0:0: model JSON: ") + e.what());
  }
  return m;
}

// cholesky (proj/src/pricing.cpp:45-69)
std::vector<std::vector<double>> cholesky(const std::vector<std::vector<double>>& m) {
  std::size_t n = m.size();
  for (const auto& row : m)
    if (row.size() != n) throw EvalError("correlation matrix is not square");
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j)
      if (std::fabs(m[i][j] - m[j][i]) > 1e-12)
        throw EvalError("correlation matrix is not symmetric");
  std::vector<std::vector<double>> l(n, std::vector<double>(n, 0.0));
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t j = 0; j <= i; ++j) {
      double s = m[i][j];
      for (std::size_t k = 0; k < j; ++k) s -= l[i][k] * l[j][k];
      if (i == j) {
        if (s <= 0.0) throw EvalError("correlation matrix is not positive definite");
        l[i][i] = std::sqrt(s);
      } else {
        l[i][j] = s / l[j][j];
      }
    }
  }
  return l;
}

// blackScholesCall (proj/src/pricing.cpp:150-159): analytic oracle of the tests.
double blackScholesCall(double spot, double strike, double rate, double vol, double tYears) {
  auto ncdf = [](double x) { return 0.5 * std::erfc(-x / std::sqrt(2.0)); };
  if (tYears <= 0.0) return std::max(spot - strike, 0.0);
  double sd = vol * std::sqrt(tYears);
  double d1 = (std::log(spot / strike) + (rate + 0.5 * vol * vol) * tYears) / sd;
  double d2 = d1 - sd;
  return spot * ncdf(d1) - strike * std::exp(-rate * tYears) * ncdf(d2);
}

// TEnv::lookup (proj/include/cltk/env.hpp:36-40)
uint64_t TEnv::lookup(const std::string& name) const {
  auto it = map_.find(name);
  if (it == map_.end()) throw EvalError("unbound template variable: " + name);
  return it->second;
}

// tenvFromJson (proj/src/json_io.cpp:311-317)
TEnv tenvFromJson(const std::string& text) {
  if (text.empty()) return TEnv{};
  try {
    Json j = Json::parse(text);
    if (!j.is_object())
      throw ParseError("parse error at 0:0: template environment must be an object");
    std::map<std::string, uint64_t> m;
    for (auto it = j.begin(); it != j.end(); ++it) m[it.key()] = it.value().get<uint64_t>();
    return TEnv(std::move(m));
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    throw ParseError(std::string("parse error at 0:0: tenv JSON: ") + e.what());
  }
}

// priceResultToJson (proj/src/pricing.cpp:161-167)
std::string priceResultToJson(const PriceResult& r) {
  Json j = {{"price", r.price},
            {"stdError", r.stdError},
            {"paths", r.paths},
            {"seed", r.seed},
            {"valuationDay", r.valuationDay}};
  return j.dump();
}

}  // namespace b200
}  // namespace cltk
