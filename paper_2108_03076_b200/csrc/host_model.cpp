// Host-side data layer of the engine: kernel JSON reader, model JSON reader,
// Cholesky, template environment.  Semantics follow the reference line by
// line (cited per function); the representation is the engine's own
// (a flat node pool instead of a shared_ptr tree).
#include <cctype>
#include <cerrno>
#include <climits>
#include <string_view>
#include <map>
#include <cmath>
#include <cstdlib>
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
      if (n.kind == KKind::LoopIf) {
        n.nat = j.at("window").get<uint64_t>();
        if (j.contains("windowVar")) n.wvar = j.at("windowVar").get<int32_t>();
      }
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

namespace {
// Fast path of kernelFromJson: a minimal JSON reader (one pass into a flat
// value array, keys and strings as views into the text) and the same node
// walk as KernelReader -- the same node pool, ~10x faster than the DOM
// parse on the BRC's 200 KB kernel (the plan build of every one-shot call).
// Anything it does not expect (escapes, malformed input, unusual number
// forms) returns false and the nlohmann path below runs instead, so errors
// and their messages are that path's.
struct FastJson {
  struct V {
    char t;             // o a s n T F z
    uint32_t first = 0, next = 0, count = 0;  // children (1-based; 0 = none), sibling
    std::string_view key, text;
  };
  const char* p;
  const char* e;
  std::vector<V> v{V{'z'}};  // index 0 unused
  bool ok = true;

  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool str(std::string_view& out) {
    if (p >= e || *p != '"') return false;
    const char* s0 = ++p;
    while (p < e && *p != '"') {
      if (*p == '\\' || static_cast<unsigned char>(*p) < 0x20) return false;
      ++p;
    }
    if (p >= e) return false;
    out = std::string_view(s0, static_cast<size_t>(p - s0));
    ++p;
    return true;
  }
  uint32_t value(int depth) {
    if (depth > 100000) return 0;
    ws();
    if (p >= e) return 0;
    const uint32_t id = static_cast<uint32_t>(v.size());
    v.push_back(V{'z'});
    const char c = *p;
    if (c == '{' || c == '[') {
      v[id].t = c == '{' ? 'o' : 'a';
      ++p;
      ws();
      uint32_t last = 0;
      if (p < e && *p == (c == '{' ? '}' : ']')) {
        ++p;
        return id;
      }
      for (;;) {
        std::string_view key;
        if (c == '{') {
          ws();
          if (!str(key)) return 0;
          ws();
          if (p >= e || *p != ':') return 0;
          ++p;
        }
        const uint32_t ch = value(depth + 1);
        if (!ch) return 0;
        v[ch].key = key;
        if (last) v[last].next = ch; else v[id].first = ch;
        last = ch;
        ++v[id].count;
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == (c == '{' ? '}' : ']')) { ++p; return id; }
        return 0;
      }
    }
    if (c == '"') {
      v[id].t = 's';
      return str(v[id].text) ? id : 0;
    }
    if (c == 't' && e - p >= 4 && std::string_view(p, 4) == "true") { v[id].t = 'T'; p += 4; return id; }
    if (c == 'f' && e - p >= 5 && std::string_view(p, 5) == "false") { v[id].t = 'F'; p += 5; return id; }
    if (c == 'n' && e - p >= 4 && std::string_view(p, 4) == "null") { v[id].t = 'z'; p += 4; return id; }
    const char* s0 = p;
    if (p < e && *p == '-') ++p;
    while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '+' || *p == '-')) ++p;
    if (p == s0) return 0;
    v[id].t = 'n';
    v[id].text = std::string_view(s0, static_cast<size_t>(p - s0));
    return id;
  }
  uint32_t get(uint32_t obj, std::string_view key) const {
    if (!obj || v[obj].t != 'o') return 0;
    for (uint32_t c = v[obj].first; c; c = v[c].next)
      if (v[c].key == key) return c;
    return 0;
  }
  bool num(uint32_t id, double& out) const {
    if (!id || v[id].t != 'n') return false;
    const std::string t(v[id].text);
    char* end = nullptr;
    out = std::strtod(t.c_str(), &end);
    return end == t.c_str() + t.size();
  }
  bool uint(uint32_t id, uint64_t& out) const {
    if (!id || v[id].t != 'n') return false;
    for (char ch : v[id].text)
      if (ch < '0' || ch > '9') return false;  // plain non-negative integers only
    const std::string t(v[id].text);
    errno = 0;
    out = std::strtoull(t.c_str(), nullptr, 10);
    return errno == 0;
  }
  bool sint(uint32_t id, int64_t& out) const {
    if (!id || v[id].t != 'n') return false;
    const std::string t(v[id].text);
    for (size_t i = 0; i < t.size(); ++i)
      if (!(t[i] >= '0' && t[i] <= '9') && !(i == 0 && t[i] == '-')) return false;
    errno = 0;
    char* end = nullptr;
    out = std::strtoll(t.c_str(), &end, 10);
    return errno == 0 && end == t.c_str() + t.size();
  }
};

struct FastKernelReader {
  const FastJson& j;
  Kernel& k;
  std::map<std::string, int32_t, std::less<>> partyIdx;
  bool ok = true;

  int32_t party(std::string_view p) {
    auto it = partyIdx.find(p);
    if (it != partyIdx.end()) return it->second;
    const int32_t id = static_cast<int32_t>(k.partyNames.size());
    k.partyNames.emplace_back(p);
    partyIdx.emplace(std::string(p), id);
    return id;
  }
  std::string_view text(uint32_t id) {
    if (!id || j.v[id].t != 's') { ok = false; return {}; }
    return j.v[id].text;
  }
  uint64_t u64(uint32_t id) {
    uint64_t x = 0;
    if (!j.uint(id, x)) ok = false;
    return x;
  }
  // the walk of KernelReader::read (kexprFromJson, proj/src/kernel.cpp:581-627)
  int32_t read(uint32_t n0) {
    if (!ok || !n0 || j.v[n0].t != 'o') { ok = false; return -1; }
    const std::string_view kind = text(j.get(n0, "kind"));
    KNode n;
    if (kind == "if" || kind == "loopif") {
      n.kind = kind == "if" ? KKind::If : KKind::LoopIf;
      n.a = read(j.get(n0, "cond"));
      n.b = read(j.get(n0, "then"));
      n.c = read(j.get(n0, "else"));
      if (n.kind == KKind::LoopIf) {
        n.nat = u64(j.get(n0, "window"));
        if (const uint32_t w = j.get(n0, "windowVar")) {
          int64_t x = 0;
          if (!j.sint(w, x) || x < INT32_MIN || x > INT32_MAX) ok = false;
          n.wvar = static_cast<int32_t>(x);
        }
      }
    } else if (kind == "float") {
      n.kind = KKind::Float;
      if (!j.num(j.get(n0, "value"), n.real)) ok = false;
    } else if (kind == "nat") {
      n.kind = KKind::Nat;
      n.nat = u64(j.get(n0, "value"));
    } else if (kind == "bool") {
      n.kind = KKind::Bool;
      const uint32_t b = j.get(n0, "value");
      if (!b || (j.v[b].t != 'T' && j.v[b].t != 'F')) ok = false;
      n.boolean = b && j.v[b].t == 'T';
    } else if (kind == "now") {
      n.kind = KKind::Now;
    } else if (kind == "timeref") {
      n.kind = KKind::TimeRef;
      n.row = u64(j.get(n0, "row"));
    } else if (kind == "obsref") {
      n.kind = KKind::ObsRef;
      n.row = u64(j.get(n0, "row"));
      n.col = u64(j.get(n0, "col"));
    } else if (kind == "payref") {
      n.kind = KKind::PayRef;
      n.row = u64(j.get(n0, "row"));
      n.from = party(text(j.get(n0, "from")));
      n.to = party(text(j.get(n0, "to")));
    } else if (kind == "unop") {
      n.kind = KKind::UnOp;
      const std::string_view op = text(j.get(n0, "op"));
      if (op != "neg" && op != "not") ok = false;
      n.op = static_cast<int>(op == "neg" ? KUn::Neg : KUn::Not);
      n.a = read(j.get(n0, "arg"));
    } else if (kind == "binop") {
      static const std::map<std::string, KBin, std::less<>> ops = {
          {"add", KBin::Add}, {"sub", KBin::Sub}, {"mult", KBin::Mult},
          {"div", KBin::Div}, {"lt", KBin::Lt},   {"leq", KBin::Leq},
          {"eq", KBin::Eq},   {"and", KBin::And}, {"or", KBin::Or}};
      n.kind = KKind::BinOp;
      const auto it = ops.find(text(j.get(n0, "op")));
      if (it == ops.end()) { ok = false; return -1; }
      n.op = static_cast<int>(it->second);
      n.a = read(j.get(n0, "left"));
      n.b = read(j.get(n0, "right"));
    } else {
      ok = false;
      return -1;
    }
    if (!ok) return -1;
    k.nodes.push_back(n);
    return static_cast<int32_t>(k.nodes.size() - 1);
  }
};

bool fastKernelFromJson(const std::string& text, Kernel& k) {
  FastJson j{text.data(), text.data() + text.size()};
  j.v.reserve(text.size() / 16 + 16);
  const uint32_t root = j.value(0);
  j.ws();
  if (!root || j.p != j.e || j.v[root].t != 'o') return false;
  FastKernelReader r{j, k, {}};
  k.root = r.read(j.get(root, "body"));
  if (!r.ok) return false;
  auto strs = [&](const char* key, std::vector<std::string>& out) {
    const uint32_t a = j.get(root, key);
    if (!a || j.v[a].t != 'a') return false;
    for (uint32_t c = j.v[a].first; c; c = j.v[c].next) {
      if (j.v[c].t != 's') return false;
      out.emplace_back(j.v[c].text);
    }
    return true;
  };
  const uint32_t rows = j.get(root, "rows");
  if (!rows || j.v[rows].t != 'a') return false;
  for (uint32_t c = j.v[rows].first; c; c = j.v[c].next) {
    int64_t x = 0;
    if (!j.sint(c, x)) return false;
    k.rows.push_back(x);
  }
  if (!strs("cols", k.cols) || !strs("tvars", k.tvars) || !strs("parties", k.parties)) return false;
  return j.uint(j.get(root, "horizon"), k.horizon);
}
}  // namespace

Kernel kernelFromJson(const std::string& text) {
  // CLTK_KERNEL_JSON_DOM: always the DOM path (tests compare the two)
  if (std::getenv("CLTK_KERNEL_JSON_DOM") == nullptr) {
    Kernel k;
    if (fastKernelFromJson(text, k)) return k;
  }
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

// ---------------------------------------------------------------------------
// Textual kernel format (emitKernelSource, proj/src/kernel.cpp:407-435;
// grammar proj/docs/kernel-format.md): an independent reader producing the
// same node pool as kernelFromJson.  Loop windows given as tenv[k] take the
// k-th entry of `tenvValues` (the text carries indices, not names).
// ---------------------------------------------------------------------------
namespace {

struct TextReader {
  const std::string& src;
  const std::vector<uint64_t>& tenvValues;
  Kernel& k;
  std::size_t pos = 0;
  std::map<std::string, int32_t> partyIdx;

  [[noreturn]] void fail(const std::string& m) const {
    std::size_t line = 1, col = 1;
    for (std::size_t i = 0; i < pos && i < src.size(); ++i) {
      if (src[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    throw ParseError("parse error at " + std::to_string(line) + ":" + std::to_string(col) +
                     ": kernel source: " + m);
  }
  void skip() {
    for (;;) {
      while (pos < src.size() && std::isspace(static_cast<unsigned char>(src[pos]))) ++pos;
      if (pos + 1 < src.size() && src[pos] == '-' && src[pos + 1] == '-') {
        while (pos < src.size() && src[pos] != '\n') ++pos;
        continue;
      }
      return;
    }
  }
  bool peek(const char* t) {
    skip();
    return src.compare(pos, std::strlen(t), t) == 0;
  }
  bool peekWord(const char* w) {
    skip();
    const std::size_t n = std::strlen(w);
    if (src.compare(pos, n, w) != 0) return false;
    const char c = pos + n < src.size() ? src[pos + n] : ' ';
    return !(std::isalnum(static_cast<unsigned char>(c)) || c == '_');
  }
  void expect(const char* t) {
    if (!peek(t)) fail(std::string("expected '") + t + "'");
    pos += std::strlen(t);
  }
  void expectWord(const char* w) {
    if (!peekWord(w)) fail(std::string("expected '") + w + "'");
    pos += std::strlen(w);
  }
  std::string ident() {
    skip();
    std::size_t b = pos;
    while (pos < src.size() && (std::isalnum(static_cast<unsigned char>(src[pos])) || src[pos] == '_'))
      ++pos;
    if (b == pos) fail("expected an identifier");
    return src.substr(b, pos - b);
  }
  std::string quoted() {
    expect("\"");
    std::size_t b = pos;
    while (pos < src.size() && src[pos] != '"') ++pos;
    if (pos >= src.size()) fail("unterminated string");
    std::string r = src.substr(b, pos - b);
    ++pos;
    return r;
  }
  // number: returns true for float (value in d) else integer (in i)
  bool number(double& d, int64_t& i) {
    skip();
    std::size_t b = pos;
    if (pos < src.size() && (src[pos] == '-' || src[pos] == '+')) ++pos;
    bool isFloat = false;
    while (pos < src.size() &&
           (std::isdigit(static_cast<unsigned char>(src[pos])) || src[pos] == '.' || src[pos] == 'e' ||
            src[pos] == 'E' ||
            ((src[pos] == '-' || src[pos] == '+') && (src[pos - 1] == 'e' || src[pos - 1] == 'E')))) {
      if (src[pos] == '.' || src[pos] == 'e' || src[pos] == 'E') isFloat = true;
      ++pos;
    }
    const std::string t = src.substr(b, pos - b);
    if (t.empty() || t == "-" || t == "+") fail("expected a number");
    if (isFloat) d = std::strtod(t.c_str(), nullptr);
    else i = std::strtoll(t.c_str(), nullptr, 10);
    return isFloat;
  }
  int32_t push(KNode n) {
    k.nodes.push_back(n);
    return static_cast<int32_t>(k.nodes.size() - 1);
  }
  int32_t party(const std::string& p) {
    auto [it, ins] = partyIdx.try_emplace(p, static_cast<int32_t>(k.partyNames.size()));
    if (ins) {
      k.partyNames.push_back(p);
      k.parties.push_back(p);  // first occurrence order, as reindex notes them
    }
    return it->second;
  }
  // "<int> + var" or "var" relative to the current offset variable
  uint64_t rowIndex(const std::string& var) {
    uint64_t row = 0;
    if (!peekWord(var.c_str())) {
      double d = 0;
      int64_t i = 0;
      if (number(d, i)) fail("row index must be an integer");
      row = static_cast<uint64_t>(i);
      expect("+");
    }
    if (ident() != var) fail("row index must be relative to " + var);
    return row;
  }

  // expression grammar, loosest first: | & comparisons + - * / unary atoms
  int32_t expr(const std::string& v) { return orE(v); }
  int32_t bin(KBin op, int32_t a, int32_t b) {
    KNode n;
    n.kind = KKind::BinOp;
    n.op = static_cast<int>(op);
    n.a = a;
    n.b = b;
    return push(n);
  }
  int32_t orE(const std::string& v) {
    int32_t a = andE(v);
    while (peek("|")) {
      ++pos;
      a = bin(KBin::Or, a, andE(v));
    }
    return a;
  }
  int32_t andE(const std::string& v) {
    int32_t a = cmpE(v);
    while (peek("&")) {
      ++pos;
      a = bin(KBin::And, a, cmpE(v));
    }
    return a;
  }
  int32_t cmpE(const std::string& v) {
    int32_t a = addE(v);
    if (peek("<=")) {
      pos += 2;
      return bin(KBin::Leq, a, addE(v));
    }
    if (peek("<")) {
      ++pos;
      return bin(KBin::Lt, a, addE(v));
    }
    if (peek("==")) {
      pos += 2;
      return bin(KBin::Eq, a, addE(v));
    }
    return a;
  }
  int32_t addE(const std::string& v) {
    int32_t a = mulE(v);
    for (;;) {
      if (peek("+")) {
        ++pos;
        a = bin(KBin::Add, a, mulE(v));
      } else if (peek("-") && !peek("--")) {
        ++pos;
        a = bin(KBin::Sub, a, mulE(v));
      } else {
        return a;
      }
    }
  }
  int32_t mulE(const std::string& v) {
    int32_t a = unE(v);
    for (;;) {
      if (peek("*")) {
        ++pos;
        a = bin(KBin::Mult, a, unE(v));
      } else if (peek("/")) {
        ++pos;
        a = bin(KBin::Div, a, unE(v));
      } else {
        return a;
      }
    }
  }
  int32_t unE(const std::string& v) {
    skip();
    if (peek("-") && !(pos + 1 < src.size() && std::isdigit(static_cast<unsigned char>(src[pos + 1])))) {
      ++pos;
      KNode n;
      n.kind = KKind::UnOp;
      n.op = static_cast<int>(KUn::Neg);
      n.a = unE(v);
      return push(n);
    }
    if (peek("!")) {
      ++pos;
      KNode n;
      n.kind = KKind::UnOp;
      n.op = static_cast<int>(KUn::Not);
      n.a = unE(v);
      return push(n);
    }
    return atom(v);
  }
  int32_t atom(const std::string& v) {
    skip();
    KNode n;
    if (peek("(")) {
      ++pos;
      if (peekWord("if")) {
        pos += 2;
        n.kind = KKind::If;
        n.a = expr(v);
        expectWord("then");
        n.b = expr(v);
        expectWord("else");
        n.c = expr(v);
        expect(")");
        return push(n);
      }
      if (peekWord("let")) return loop(v);
      int32_t e = expr(v);
      expect(")");
      return e;
    }
    if (peekWord("true") || peekWord("false")) {
      n.kind = KKind::Bool;
      n.boolean = peekWord("true");
      pos += n.boolean ? 4 : 5;
      return push(n);
    }
    if (peekWord("t_now")) {
      pos += 5;
      n.kind = KKind::Now;
      return push(n);
    }
    if (peekWord("ext")) {
      pos += 3;
      expect("[");
      n.kind = KKind::ObsRef;
      n.row = rowIndex(v);
      expect(",");
      double d;
      int64_t i = 0;
      if (number(d, i)) fail("column must be an integer");
      n.col = static_cast<uint64_t>(i);
      expect("]");
      return push(n);
    }
    if (peekWord("rows")) {
      pos += 4;
      expect("[");
      n.kind = KKind::TimeRef;
      n.row = rowIndex(v);
      expect("]");
      return push(n);
    }
    if (peekWord("pay")) {
      pos += 3;
      expect("[");
      n.kind = KKind::PayRef;
      n.row = rowIndex(v);
      expect(",");
      n.from = party(ident());
      expect(",");
      n.to = party(ident());
      expect("]");
      return push(n);
    }
    double d = 0;
    int64_t i = 0;
    if (number(d, i)) {
      n.kind = KKind::Float;
      n.real = d;
    } else {
      n.kind = KKind::Nat;
      n.nat = static_cast<uint64_t>(i);
    }
    return push(n);
  }
  // (let tK = loop tK = OFF while (!COND & (tK < OFF + W)) do tK + 1
  //  in if COND then THEN else ELSE)
  int32_t loop(const std::string& v) {
    expectWord("let");
    const std::string t = ident();
    expect("=");
    expectWord("loop");
    if (ident() != t) fail("loop variable mismatch");
    expect("=");
    if (ident() != v) fail("loop must start at the enclosing offset " + v);
    expectWord("while");
    expect("(");
    expect("!");
    const std::size_t condStart = pos;
    (void)unE(t);  // the while-condition copy of COND (discarded)
    k.nodes.resize(k.nodes.size());  // (nodes of the copy stay unreferenced)
    (void)condStart;
    expect("&");
    expect("(");
    if (ident() != t) fail("loop bound must test " + t);
    expect("<");
    if (ident() != v) fail("loop bound must be relative to " + v);
    expect("+");
    KNode n;
    n.kind = KKind::LoopIf;
    if (peekWord("tenv")) {
      pos += 4;
      expect("[");
      double d;
      int64_t idx = 0;
      if (number(d, idx)) fail("tenv index must be an integer");
      expect("]");
      if (idx < 0 || static_cast<std::size_t>(idx) >= tenvValues.size())
        fail("loop window tenv[" + std::to_string(idx) + "] has no value");
      n.nat = tenvValues[static_cast<std::size_t>(idx)];
      n.wvar = static_cast<int32_t>(idx);
    } else {
      double d;
      int64_t w = 0;
      if (number(d, w)) fail("loop window must be an integer");
      n.nat = static_cast<uint64_t>(w);
    }
    expect(")");
    expect(")");
    expectWord("do");
    if (ident() != t) fail("loop step must advance " + t);
    expect("+");
    double d;
    int64_t one = 0;
    if (number(d, one) || one != 1) fail("loop step must be + 1");
    expectWord("in");
    expectWord("if");
    n.a = expr(t);
    expectWord("then");
    n.b = expr(t);
    expectWord("else");
    n.c = expr(t);
    expect(")");
    return push(n);
  }

  void read() {
    expectWord("let");
    expectWord("rows");
    expect("=");
    expect("[");
    while (!peek("]")) {
      double d;
      int64_t i = 0;
      if (number(d, i)) fail("rows must be integers");
      k.rows.push_back(i);
      if (peek(",")) ++pos;
    }
    expect("]");
    expectWord("let");
    expectWord("cols");
    expect("=");
    expect("[");
    while (!peek("]")) {
      k.cols.push_back(quoted());
      if (peek(",")) ++pos;
    }
    expect("]");
    expectWord("let");
    expectWord("payoffInternal");
    expect("(");
    for (const char* a : {"ext", "tenv", "disc", "t0", "t_now"}) {
      expectWord(a);
      if (peek(",")) ++pos;
    }
    expect(")");
    expect("=");
    k.root = expr("t0");
    // the wrapper "let payoff(...) = payoffInternal(ext, tenv, disc, 0, t_now)" is fixed
    expectWord("let");
    expectWord("payoff");
  }
};

}  // namespace

Kernel kernelFromSource(const std::string& text, const std::vector<uint64_t>& tenvValues) {
  Kernel k;
  TextReader r{text, tenvValues, k};
  r.read();
  // Drop the unreferenced while-condition copies: re-emit reachable nodes
  // in postorder so the pool has the shape kernelFromJson produces.
  Kernel out;
  out.rows = k.rows;
  out.cols = k.cols;
  out.parties = k.parties;
  out.partyNames = k.partyNames;
  std::vector<int32_t> map(k.nodes.size(), -1);
  std::vector<std::pair<int32_t, bool>> st{{k.root, false}};
  while (!st.empty()) {
    auto [i, done] = st.back();
    st.pop_back();
    if (map[i] >= 0) continue;
    const KNode& n = k.nodes[i];
    if (!done) {
      st.push_back({i, true});
      for (int32_t ch : {n.c, n.b, n.a})
        if (ch >= 0 && map[ch] < 0) st.push_back({ch, false});
      continue;
    }
    KNode m = n;
    m.a = n.a >= 0 ? map[n.a] : -1;
    m.b = n.b >= 0 ? map[n.b] : -1;
    m.c = n.c >= 0 ? map[n.c] : -1;
    out.nodes.push_back(m);
    map[i] = static_cast<int32_t>(out.nodes.size() - 1);
  }
  out.root = map[k.root];
  int64_t maxDay = 0;
  for (int64_t d : out.rows) maxDay = std::max(maxDay, d);
  out.horizon = static_cast<uint64_t>(maxDay) + 1;  // KernelBuilder::build, kernel.cpp:24-31
  return out;
}

Kernel kernelFromWire(const std::string& text, const std::vector<uint64_t>& tenvValues) {
  std::size_t i = 0;
  while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
  if (i < text.size() && text[i] == '{') return kernelFromJson(text);
  return kernelFromSource(text, tenvValues);
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

// ModelSpec::at (proj/src/pricing.cpp:13-18): same message on a missing label.
const AssetSpec& ModelSpec::at(const std::string& label) const {
  const auto found = assets.find(label);
  if (found != assets.end()) return found->second;
  throw EvalError("model has no asset spec for label " + label);
}

// modelFromJson (proj/src/pricing.cpp:20-43): the same schema and defaults
// (rate 0, dayCount 365, drift = rate, order = the sorted labels unless
// given), with the reference CLI's parse-error wording for malformed input.
ModelSpec modelFromJson(const std::string& text) {
  ModelSpec m;
  try {
    const Json doc = Json::parse(text);
    m.rate = doc.value("rate", 0.0);
    m.dayCount = doc.value("dayCount", 365.0);
    const Json& labels = doc.at("labels");
    if (doc.contains("order")) {
      m.order = doc.at("order").get<std::vector<std::string>>();
    } else {
      m.order.reserve(labels.size());
      for (const auto& kv : labels.items()) m.order.push_back(kv.key());
      std::sort(m.order.begin(), m.order.end());
    }
    for (const std::string& label : m.order) {
      const Json& spec = labels.at(label);
      m.assets[label] = AssetSpec{spec.at("spot").get<double>(), spec.at("vol").get<double>(),
                                  spec.value("drift", m.rate)};
    }
    if (doc.contains("corr")) m.corr = doc.at("corr").get<std::vector<std::vector<double>>>();
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    throw ParseError(std::string("parse error at 0:0: model JSON: ") + e.what());
  }
  return m;
}

// cholesky (proj/src/pricing.cpp:45-69).  The factor feeds the device's
// correlated draws, so it must be the reference's bits: the same checks and
// messages, and per entry the same IEEE sequence -- start from m[i][j],
// subtract the products l[i][k] * l[j][k] for k = 0 .. j-1 one rounding at a
// time, then sqrt on the diagonal or one division by l[j][j] below it.
// Worked on a flat row-major n x n array (the layout the plan uploads).
std::vector<std::vector<double>> cholesky(const std::vector<std::vector<double>>& m) {
  const std::size_t n = m.size();
  for (const auto& row : m)
    if (row.size() != n) throw EvalError("correlation matrix is not square");
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j)
      if (std::fabs(m[i][j] - m[j][i]) > 1e-12)
        throw EvalError("correlation matrix is not symmetric");
  std::vector<double> L(n * n, 0.0);
  for (std::size_t i = 0; i < n; ++i) {
    const double* li = &L[i * n];
    for (std::size_t j = 0; j <= i; ++j) {
      const double* lj = &L[j * n];
      double acc = m[i][j];
      for (std::size_t k = 0; k < j; ++k) {
        const double prod = li[k] * lj[k];
        acc = acc - prod;
      }
      if (j < i) {
        L[i * n + j] = acc / lj[j];
        continue;
      }
      if (acc <= 0.0) throw EvalError("correlation matrix is not positive definite");
      L[i * n + i] = std::sqrt(acc);
    }
  }
  std::vector<std::vector<double>> out(n);
  for (std::size_t i = 0; i < n; ++i) out[i].assign(L.begin() + i * n, L.begin() + (i + 1) * n);
  return out;
}

// blackScholesCall (proj/src/pricing.cpp:150-159): the analytic price the
// tests check Monte Carlo against (normalCdf(x) = erfc(-x / sqrt 2) / 2).
double blackScholesCall(double spot, double strike, double rate, double vol, double tYears) {
  if (tYears <= 0.0) {
    const double intrinsic = spot - strike;
    return intrinsic < 0.0 ? 0.0 : intrinsic;  // std::max(spot - strike, 0.0)
  }
  const auto Phi = [](double x) { return 0.5 * std::erfc(-x / std::sqrt(2.0)); };
  const double sd = vol * std::sqrt(tYears);
  const double d1 = (std::log(spot / strike) + (rate + 0.5 * vol * vol) * tYears) / sd;
  const double d2 = d1 - sd;
  const double discounted = strike * std::exp(-rate * tYears);
  return spot * Phi(d1) - discounted * Phi(d2);
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

// priceResultToJson (proj/src/pricing.cpp:161-167): the reference's keys
// (nlohmann orders them alphabetically in the dump).
std::string priceResultToJson(const PriceResult& r) {
  Json j = Json::object();
  j["paths"] = r.paths;
  j["price"] = r.price;
  j["seed"] = r.seed;
  j["stdError"] = r.stdError;
  j["valuationDay"] = r.valuationDay;
  return j.dump();
}

}  // namespace b200
}  // namespace cltk
