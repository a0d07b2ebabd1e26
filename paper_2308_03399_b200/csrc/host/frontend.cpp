// Host front-end of shotsim_b200: circuit model, noise model, instrument()
// lowering, circuit text/JSON I/O and result folding.
//
// Semantics are the reference's (file:line cited per function) — in
// particular every floating-point constant that reaches the device (gate
// matrices, Pauli cumulatives, Kraus matrices) is produced by the same
// sequence of IEEE operations as the reference, so the lowered program is
// bit-identical (checked against the reference's own instrument() by
// tests/test_frontend.py via ssb_program_dump).
#include <algorithm>
#include <bit>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numbers>
#include <set>
#include <sstream>

#include <json.hpp>

#include "shotsim_b200.hpp"

namespace shotsim {

using nlohmann::json;

// ---------------------------------------------------------------------------
// Gate table — circuit.cpp:16-34 (order = GateKind order, circuit.hpp:17-19).
namespace {
constexpr GateInfo kGates[] = {
    {"id", 1, 0, true},       {"x", 1, 0, true},      {"y", 1, 0, true},
    {"z", 1, 0, true},        {"h", 1, 0, true},      {"s", 1, 0, true},
    {"sdg", 1, 0, true},      {"t", 1, 0, true},      {"tdg", 1, 0, true},
    {"p", 1, 1, true},        {"u", 1, 3, true},      {"cx", 2, 0, true},
    {"cp", 2, 1, true},       {"swap", 2, 0, true},   {"measure", 1, 0, false},
    {"reset", 1, 0, false},   {"barrier", 0, 0, false},
};
}  // namespace

const GateInfo& gate_info(GateKind kind) { return kGates[static_cast<size_t>(kind)]; }

std::optional<GateKind> gate_kind_from_name(std::string_view name) {
  for (size_t i = 0; i < std::size(kGates); ++i)
    if (kGates[i].name == name) return static_cast<GateKind>(i);
  return std::nullopt;
}

// circuit.cpp:49-91
std::vector<Violation> validate(const Circuit& c) {
  std::vector<Violation> bad;
  if (c.num_clbits > 64) bad.push_back({0, "classical registers wider than 64 bits are unsupported"});
  for (size_t i = 0; i < c.instructions.size(); ++i) {
    const Instruction& in = c.instructions[i];
    const GateInfo& g = gate_info(in.kind);
    auto flag = [&](std::string m) { bad.push_back({i, std::move(m)}); };
    if (in.qubits.size() != g.arity)
      flag("arity mismatch: " + std::string(g.name) + " expects " + std::to_string(g.arity) +
           " qubits, got " + std::to_string(in.qubits.size()));
    if (in.params.size() != g.num_params) flag("parameter count mismatch for " + std::string(g.name));
    uint64_t seen = 0;
    for (unsigned q : in.qubits) {
      if (q >= c.num_qubits) flag("qubit " + std::to_string(q) + " out of range");
      const uint64_t b = q < 64 ? one_bit(q) : 0;
      if (seen & b) flag("duplicate qubit " + std::to_string(q));
      seen |= b;
    }
    if (in.kind == GateKind::MEASURE) {
      if (in.clbits.size() != in.qubits.size()) flag("measure needs one clbit per qubit");
      for (unsigned cb : in.clbits)
        if (cb >= c.num_clbits) flag("clbit " + std::to_string(cb) + " out of range");
    } else if (!in.clbits.empty()) {
      flag("clbits only allowed on measure");
    }
    if (in.condition) {
      if (in.condition->value & ~in.condition->clbit_mask)
        flag("condition value has bits outside its mask");
      if (c.num_clbits < 64 && (in.condition->clbit_mask >> c.num_clbits) != 0)
        flag("condition mask references clbits out of range");
    }
  }
  return bad;
}

void require_valid(const Circuit& c) {
  const auto bad = validate(c);
  if (bad.empty()) return;
  std::string msg = "invalid circuit:";
  for (size_t k = 0; k < bad.size() && k < 4; ++k)
    msg += " [instruction " + std::to_string(bad[k].instruction) + "] " + bad[k].message + ";";
  throw std::invalid_argument(msg);
}

// circuit.cpp:106-123
Circuit qft_circuit(unsigned n) {
  if (n < 1 || n > 30) throw std::invalid_argument("qft_circuit: qubit count must be in [1, 30]");
  Circuit c;
  c.num_qubits = n;
  for (unsigned k = n; k-- > 0;) {
    c.instructions.push_back({GateKind::H, {k}, {}, {}, std::nullopt});
    for (unsigned j = 0; j < k; ++j)
      c.instructions.push_back({GateKind::CP, {j, k}, {}, {std::numbers::pi / double(one_bit(k - j))}, std::nullopt});
  }
  for (unsigned j = 0; j < n / 2; ++j)
    c.instructions.push_back({GateKind::SWAP, {j, n - 1 - j}, {}, {}, std::nullopt});
  return c;
}

// circuit.cpp:125-131
Circuit measure_all(Circuit c) {
  c.num_clbits = std::max(c.num_clbits, c.num_qubits);
  for (unsigned k = 0; k < c.num_qubits; ++k)
    c.instructions.push_back({GateKind::MEASURE, {k}, {k}, {}, std::nullopt});
  return c;
}

// circuit.cpp:133-183. The entry expressions mirror the reference's exactly
// (std::polar, unary minus, 1/sqrt(2)) so every bit — including signed zeros —
// matches.
GateMatrix gate_matrix(GateKind kind, std::span<const double> params) {
  const GateInfo& g = gate_info(kind);
  if (!g.unitary) throw std::invalid_argument("gate has no matrix: " + std::string(g.name));
  if (params.size() != g.num_params)
    throw std::invalid_argument("wrong parameter count for " + std::string(g.name));
  const cplx i1{0.0, 1.0};
  const double r = 1.0 / std::sqrt(2.0);
  auto one = [](cplx a, cplx b, cplx c, cplx d) { return GateMatrix{1, {a, b, c, d}}; };
  auto two = [](std::initializer_list<cplx> e) { return GateMatrix{2, std::vector<cplx>(e)}; };
  switch (kind) {
    case GateKind::ID: return one(1, 0, 0, 1);
    case GateKind::X: return one(0, 1, 1, 0);
    case GateKind::Y: return one(0, -i1, i1, 0);
    case GateKind::Z: return one(1, 0, 0, -1);
    case GateKind::H: return one(r, r, r, -r);
    case GateKind::S: return one(1, 0, 0, i1);
    case GateKind::SDG: return one(1, 0, 0, -i1);
    case GateKind::T: return one(1, 0, 0, std::polar(1.0, std::numbers::pi / 4));
    case GateKind::TDG: return one(1, 0, 0, std::polar(1.0, -std::numbers::pi / 4));
    case GateKind::P: return one(1, 0, 0, std::polar(1.0, params[0]));
    case GateKind::U: {
      const double th = params[0], phi = params[1], lam = params[2];
      const double ct = std::cos(th / 2), st = std::sin(th / 2);
      return one(ct, -std::polar(st, lam), std::polar(st, phi), std::polar(ct, phi + lam));
    }
    case GateKind::CX:  // qubits[0] is the control
      return two({1, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 1, 0, 0});
    case GateKind::CP: {
      const cplx ph = std::polar(1.0, params[0]);
      return two({1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, ph});
    }
    case GateKind::SWAP: return two({1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1});
    default: throw std::invalid_argument("unhandled gate kind");
  }
}

// ---------------------------------------------------------------------------
// Circuit text / JSON — circuit_io.cpp:17-214.
namespace {

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::vector<std::string> split_on(const std::string& s, char sep) {
  std::vector<std::string> parts(1);
  for (char ch : s) {
    if (ch == sep) parts.emplace_back();
    else parts.back().push_back(ch);
  }
  return parts;
}

[[noreturn]] void parse_fail(size_t line, const std::string& what) {
  throw ConfigError("line " + std::to_string(line) + ": " + what);
}

unsigned index_token(const std::string& t, char prefix, size_t line) {
  unsigned v = 0;
  if (t.size() < 2 || t[0] != prefix) parse_fail(line, std::string("expected ") + prefix + "<index>, got '" + t + "'");
  const char* end = t.data() + t.size();
  auto [p, ec] = std::from_chars(t.data() + 1, end, v);
  if (ec != std::errc{} || p != end) parse_fail(line, "bad index '" + t + "'");
  return v;
}

}  // namespace

std::string circuit_to_text(const Circuit& c) {
  std::string s = "qubits " + std::to_string(c.num_qubits) + "\nclbits " + std::to_string(c.num_clbits) + "\n";
  for (const Instruction& in : c.instructions) {
    s += gate_info(in.kind).name;
    for (size_t i = 0; i < in.qubits.size(); ++i) s += (i ? ",q" : " q") + std::to_string(in.qubits[i]);
    for (size_t i = 0; i < in.params.size(); ++i) s += (i ? "," : " ") + g17(in.params[i]);
    for (size_t i = 0; i < in.clbits.size(); ++i) s += (i ? ",c" : " -> c") + std::to_string(in.clbits[i]);
    if (in.condition)
      s += " if " + std::to_string(in.condition->clbit_mask) + "==" + std::to_string(in.condition->value);
    s += "\n";
  }
  return s;
}

Circuit circuit_from_text(const std::string& text) {
  Circuit c;
  std::istringstream lines(text);
  std::string line;
  for (size_t ln = 1; std::getline(lines, line); ++ln) {
    line = line.substr(0, line.find('#'));
    std::istringstream ws(line);
    std::vector<std::string> tok{std::istream_iterator<std::string>(ws), {}};
    if (tok.empty()) continue;
    if (tok[0] == "qubits" || tok[0] == "clbits") {
      if (tok.size() != 2) parse_fail(ln, "bad header");
      (tok[0] == "qubits" ? c.num_qubits : c.num_clbits) = static_cast<unsigned>(std::stoul(tok[1]));
      continue;
    }
    const auto kind = gate_kind_from_name(tok[0]);
    if (!kind) parse_fail(ln, "unknown gate '" + tok[0] + "'");
    Instruction in{*kind, {}, {}, {}, std::nullopt};
    size_t k = 1;
    const GateInfo& g = gate_info(*kind);
    if (g.arity > 0) {
      if (k >= tok.size()) parse_fail(ln, "missing qubits");
      for (const auto& q : split_on(tok[k++], ',')) in.qubits.push_back(index_token(q, 'q', ln));
    }
    if (g.num_params > 0) {
      if (k >= tok.size()) parse_fail(ln, "missing parameters");
      for (const auto& p : split_on(tok[k++], ',')) in.params.push_back(std::stod(p));
    }
    if (k < tok.size() && tok[k] == "->") {
      if (++k >= tok.size()) parse_fail(ln, "missing clbits after ->");
      for (const auto& cb : split_on(tok[k++], ',')) in.clbits.push_back(index_token(cb, 'c', ln));
    }
    if (k < tok.size() && tok[k] == "if") {
      if (++k >= tok.size()) parse_fail(ln, "missing condition");
      const auto parts = split_on(tok[k++], '=');
      if (parts.size() != 3 || !parts[1].empty()) parse_fail(ln, "condition must be mask==value");
      in.condition = Condition{std::stoull(parts[0]), std::stoull(parts[2])};
    }
    if (k != tok.size()) parse_fail(ln, "trailing tokens");
    c.instructions.push_back(std::move(in));
  }
  return c;
}

std::string circuit_to_json(const Circuit& c) {
  json j{{"num_qubits", c.num_qubits}, {"num_clbits", c.num_clbits}, {"instructions", json::array()}};
  for (const Instruction& in : c.instructions) {
    json e{{"kind", std::string(gate_info(in.kind).name)}, {"qubits", in.qubits}};
    if (!in.clbits.empty()) e["clbits"] = in.clbits;
    if (!in.params.empty()) e["params"] = in.params;
    if (in.condition) e["condition"] = {{"mask", in.condition->clbit_mask}, {"value", in.condition->value}};
    j["instructions"].push_back(std::move(e));
  }
  return j.dump(2);
}

Circuit circuit_from_json(const std::string& text) {
  Circuit c;
  try {
    const json j = json::parse(text);
    c.num_qubits = j.at("num_qubits").get<unsigned>();
    c.num_clbits = j.at("num_clbits").get<unsigned>();
    for (const json& e : j.at("instructions")) {
      const std::string name = e.at("kind").get<std::string>();
      const auto kind = gate_kind_from_name(name);
      if (!kind) throw ConfigError("unknown gate kind: " + name);
      Instruction in{*kind, e.at("qubits").get<std::vector<unsigned>>(), {}, {}, std::nullopt};
      if (e.contains("clbits")) in.clbits = e["clbits"].get<std::vector<unsigned>>();
      if (e.contains("params")) in.params = e["params"].get<std::vector<double>>();
      if (e.contains("condition"))
        in.condition = Condition{e["condition"].at("mask").get<uint64_t>(), e["condition"].at("value").get<uint64_t>()};
      c.instructions.push_back(std::move(in));
    }
  } catch (const json::exception& e) {
    throw ConfigError(std::string("circuit parse error: ") + e.what());
  }
  return c;
}

namespace {
std::string slurp(const std::string& path, const char* what) {
  std::ifstream f(path);
  if (!f) throw ConfigError(std::string("cannot open ") + what + " file: " + path);
  std::stringstream b;
  b << f.rdbuf();
  return b.str();
}
}  // namespace

Circuit load_circuit(const std::string& path) {
  const std::string t = slurp(path, "circuit");
  const auto first = t.find_first_not_of(" \t\r\n");
  return (first != std::string::npos && t[first] == '{') ? circuit_from_json(t) : circuit_from_text(t);
}

// ---------------------------------------------------------------------------
// Noise — noise.cpp.
namespace {

// I, X, Y, Z as row-major 2x2 (noise.cpp:18-24).
const cplx kPauli2x2[4][4] = {
    {{1, 0}, {0, 0}, {0, 0}, {1, 0}},
    {{0, 0}, {1, 0}, {1, 0}, {0, 0}},
    {{0, 0}, {0, -1}, {0, 1}, {0, 0}},
    {{1, 0}, {0, 0}, {0, 0}, {-1, 0}},
};

void check_pauli_error(const PauliError& e) {  // noise.cpp:26-47
  if (e.terms.empty()) throw ConfigError("pauli channel has no terms");
  double last = 0.0;
  for (const auto& t : e.terms) {
    if (!(t.cumulative > last))
      throw ConfigError("pauli channel cumulative probabilities must be strictly increasing");
    last = t.cumulative;
    if (t.pauli.letters.size() != t.pauli.targets.size())
      throw ConfigError("pauli string letters/targets length mismatch");
    uint64_t seen = 0;
    for (unsigned s : t.pauli.targets) {
      if (s >= e.arity) throw ConfigError("pauli string target outside channel arity");
      if (seen & one_bit(s)) throw ConfigError("duplicate pauli string target");
      seen |= one_bit(s);
    }
  }
  if (std::abs(last - 1.0) > 1e-12) throw ConfigError("pauli channel probabilities must sum to 1");
}

}  // namespace

char pauli_letter_char(PauliLetter l) { return "IXYZ"[static_cast<int>(l)]; }

PauliLetter pauli_letter_from_char(char c) {
  switch (c | 0x20) {
    case 'i': return PauliLetter::I;
    case 'x': return PauliLetter::X;
    case 'y': return PauliLetter::Y;
    case 'z': return PauliLetter::Z;
  }
  throw ConfigError(std::string("invalid pauli letter: ") + c);
}

bool PauliString::is_identity() const {
  return std::all_of(letters.begin(), letters.end(), [](PauliLetter l) { return l == PauliLetter::I; });
}

PauliString PauliString::rebased(std::span<const unsigned> qubits) const {
  PauliString r{letters, {}};
  for (unsigned s : targets) r.targets.push_back(qubits[s]);
  return r;
}

std::string PauliString::to_string() const {
  std::string s;
  for (PauliLetter l : letters) s.push_back(pauli_letter_char(l));
  return s;
}

// noise.cpp:85-98
PauliMasks pauli_to_masks(const PauliString& p) {
  PauliMasks m;
  for (size_t i = 0; i < p.letters.size(); ++i) {
    const uint64_t b = one_bit(p.targets[i]);
    const PauliLetter l = p.letters[i];
    if (l == PauliLetter::X || l == PauliLetter::Y) m.x_mask |= b;
    if (l == PauliLetter::Z || l == PauliLetter::Y) m.z_mask |= b;
    if (l == PauliLetter::Y) ++m.num_y;
  }
  if (m.x_mask) m.x_max = static_cast<unsigned>(std::bit_width(m.x_mask) - 1);
  return m;
}

// noise.cpp:100-125 (same multiply order, same early stop on a zero entry).
GateMatrix pauli_string_matrix(const PauliString& p) {
  unsigned k = 1;
  for (unsigned s : p.targets) k = std::max(k, s + 1);
  const uint64_t side = one_bit(k);
  GateMatrix m{k, std::vector<cplx>(side * side)};
  for (uint64_t r = 0; r < side; ++r) {
    for (uint64_t c = 0; c < side; ++c) {
      cplx e = 1.0;
      uint64_t free_slots = side - 1;
      for (size_t i = 0; i < p.letters.size() && e != cplx{}; ++i) {
        const unsigned s = p.targets[i];
        free_slots &= ~one_bit(s);
        e *= kPauli2x2[static_cast<int>(p.letters[i])][((r >> s) & 1) * 2 + ((c >> s) & 1)];
      }
      if ((r & free_slots) != (c & free_slots)) e = 0.0;
      m.entries[r * side + c] = e;
    }
  }
  return m;
}

double PauliError::term_prob(size_t i) const {
  return terms[i].cumulative - (i ? terms[i - 1].cumulative : 0.0);
}

unsigned channel_arity(const ErrorChannel& ch) {
  return std::visit([](const auto& c) { return c.arity; }, ch);
}

// noise.cpp:133-160
PauliError depolarizing_error(double p, unsigned k) {
  if (p < 0.0 || p > 1.0) throw std::invalid_argument("depolarizing rate must be in [0, 1]");
  if (k < 1 || k > 2) throw std::invalid_argument("depolarizing arity must be 1 or 2");
  const uint64_t nstr = one_bit(2 * k);
  const double each = p / static_cast<double>(nstr);
  const double ident = 1.0 - each * static_cast<double>(nstr - 1);
  PauliError e;
  e.arity = k;
  double cum = 0.0;
  for (uint64_t code = 0; code < nstr; ++code) {
    const double w = code == 0 ? ident : each;
    if (w <= 0.0) continue;
    cum += w;
    PauliString ps;
    for (unsigned s = 0; s < k; ++s) {
      ps.targets.push_back(s);
      ps.letters.push_back(static_cast<PauliLetter>((code >> (2 * s)) & 3));
    }
    e.terms.push_back({cum, std::move(ps)});
  }
  e.terms.back().cumulative = 1.0;
  return e;
}

size_t sample_pauli_index(const PauliError& e, double u) {  // noise.cpp:162-167
  for (size_t i = 0; i < e.terms.size(); ++i)
    if (u < e.terms[i].cumulative) return i;
  return e.terms.size() - 1;
}

// noise.cpp:173-191
KrausError pauli_as_kraus(const PauliError& e) {
  KrausError k;
  k.arity = e.arity;
  for (size_t i = 0; i < e.terms.size(); ++i) {
    PauliString ps = e.terms[i].pauli;
    GateMatrix m = pauli_string_matrix(ps);
    if (m.num_qubits < e.arity) {  // pad with an identity slot
      ps.targets.push_back(e.arity - 1);
      ps.letters.push_back(PauliLetter::I);
      m = pauli_string_matrix(ps);
    }
    const double w = std::sqrt(e.term_prob(i));
    for (cplx& x : m.entries) x *= w;
    k.matrices.push_back(std::move(m));
  }
  return k;
}

// noise.cpp:193-216
double kraus_completeness_defect(const KrausError& k) {
  if (k.matrices.empty()) return 1.0;
  const uint64_t d = one_bit(k.arity);
  std::vector<cplx> acc(d * d);
  for (const GateMatrix& m : k.matrices)
    for (uint64_t r = 0; r < d; ++r)
      for (uint64_t c = 0; c < d; ++c) {
        cplx s = 0;
        for (uint64_t i = 0; i < d; ++i) s += std::conj(m.entries[i * d + r]) * m.entries[i * d + c];
        acc[r * d + c] += s;
      }
  double worst = 0.0;
  for (uint64_t r = 0; r < d; ++r)
    for (uint64_t c = 0; c < d; ++c)
      worst = std::max(worst, std::abs(acc[r * d + c] - (r == c ? cplx{1.0} : cplx{})));
  return worst;
}

// noise.cpp:218-246
void NoiseModel::add_rule(NoiseRule rule) {
  if (rule.gates.empty()) throw ConfigError("noise rule lists no gates");
  if (channel_arity(rule.channel) != rule.arity) throw ConfigError("noise rule arity does not match its channel");
  for (GateKind g : rule.gates) {
    const GateInfo& gi = gate_info(g);
    if (!gi.unitary) throw ConfigError("noise cannot attach to " + std::string(gi.name));
    if (gi.arity != rule.arity) throw ConfigError("gate " + std::string(gi.name) + " does not match rule arity");
  }
  if (const auto* pe = std::get_if<PauliError>(&rule.channel)) {
    check_pauli_error(*pe);
  } else {
    const auto& ke = std::get<KrausError>(rule.channel);
    for (const GateMatrix& m : ke.matrices)
      if (m.num_qubits != ke.arity) throw ConfigError("kraus matrix dimension does not match channel arity");
    if (kraus_completeness_defect(ke) > 1e-10) throw ConfigError("kraus channel violates completeness");
  }
  rules_.push_back(std::move(rule));
}

// noise.cpp:248-256 — first matching rule wins.
const ErrorChannel* NoiseModel::match(GateKind kind, unsigned arity) const {
  for (const NoiseRule& r : rules_)
    if (r.arity == arity && std::find(r.gates.begin(), r.gates.end(), kind) != r.gates.end())
      return &r.channel;
  return nullptr;
}

std::string NoiseModel::to_json() const {  // noise.cpp:260-326
  json j{{"rules", json::array()}};
  for (const NoiseRule& r : rules_) {
    json gates = json::array();
    for (GateKind g : r.gates) gates.push_back(std::string(gate_info(g).name));
    json ch;
    if (const auto* pe = std::get_if<PauliError>(&r.channel)) {
      ch["type"] = "pauli";
      ch["terms"] = json::array();
      for (size_t i = 0; i < pe->terms.size(); ++i)
        ch["terms"].push_back({pe->term_prob(i), pe->terms[i].pauli.to_string()});
    } else {
      ch["type"] = "kraus";
      ch["matrices"] = json::array();
      for (const GateMatrix& m : std::get<KrausError>(r.channel).matrices) {
        json flat = json::array();
        for (const cplx& e : m.entries) flat.push_back({e.real(), e.imag()});
        ch["matrices"].push_back(std::move(flat));
      }
    }
    j["rules"].push_back({{"gates", std::move(gates)}, {"arity", r.arity}, {"channel", std::move(ch)}});
  }
  return j.dump(2);
}

namespace {
ErrorChannel channel_from(const json& j, unsigned arity) {  // noise.cpp:283-324
  const std::string type = j.at("type").get<std::string>();
  if (type == "pauli") {
    PauliError e;
    e.arity = arity;
    double cum = 0.0;
    for (const json& t : j.at("terms")) {
      const double p = t.at(0).get<double>();
      const std::string s = t.at(1).get<std::string>();
      if (s.size() != arity) throw ConfigError("pauli string length does not match arity");
      if (p <= 0.0) throw ConfigError("pauli term probabilities must be positive");
      cum += p;
      PauliString ps;
      for (unsigned i = 0; i < arity; ++i) {
        ps.letters.push_back(pauli_letter_from_char(s[i]));
        ps.targets.push_back(i);
      }
      e.terms.push_back({cum, std::move(ps)});
    }
    if (e.terms.empty() || std::abs(cum - 1.0) > 1e-12) throw ConfigError("pauli channel probabilities must sum to 1");
    e.terms.back().cumulative = 1.0;
    return e;
  }
  if (type == "kraus") {
    KrausError k;
    k.arity = arity;
    const uint64_t n = one_bit(arity) * one_bit(arity);
    for (const json& mj : j.at("matrices")) {
      if (mj.size() != n) throw ConfigError("kraus matrix entry count mismatch");
      GateMatrix m{arity, {}};
      for (const json& e : mj) m.entries.emplace_back(e.at(0).get<double>(), e.at(1).get<double>());
      k.matrices.push_back(std::move(m));
    }
    return k;
  }
  throw ConfigError("unknown channel type: " + type);
}
}  // namespace

NoiseModel NoiseModel::from_json(const std::string& text) {
  NoiseModel model;
  if (text.find_first_not_of(" \t\r\n") == std::string::npos) return model;
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw ConfigError(std::string("noise model parse error: ") + e.what());
  }
  try {
    if (j.contains("model")) {
      if (j["model"].get<std::string>() != "depolarizing") throw ConfigError("unknown noise model name");
      return make_depolarizing_model(j.at("rate").get<double>(), j.value("as_kraus", false));
    }
    for (const json& rj : j.at("rules")) {
      NoiseRule r;
      r.arity = rj.at("arity").get<unsigned>();
      for (const json& g : rj.at("gates")) {
        const std::string name = g.get<std::string>();
        const auto kind = gate_kind_from_name(name);
        if (!kind) throw ConfigError("unknown gate in noise rule: " + name);
        r.gates.push_back(*kind);
      }
      r.channel = channel_from(rj.at("channel"), r.arity);
      model.add_rule(std::move(r));
    }
  } catch (const json::exception& e) {
    throw ConfigError(std::string("noise model structure error: ") + e.what());
  }
  return model;
}

NoiseModel NoiseModel::load(const std::string& path) { return from_json(slurp(path, "noise model")); }

// noise.cpp:375-392
NoiseModel make_depolarizing_model(double rate, bool as_kraus) {
  NoiseModel m;
  if (rate <= 0.0) return m;
  using G = GateKind;
  std::vector<G> q1{G::ID, G::X, G::Y, G::Z, G::H, G::S, G::SDG, G::T, G::TDG, G::P, G::U};
  std::vector<G> q2{G::CX, G::CP, G::SWAP};
  const PauliError e1 = depolarizing_error(rate, 1), e2 = depolarizing_error(rate, 2);
  if (as_kraus) {
    m.add_rule({q1, 1, pauli_as_kraus(e1)});
    m.add_rule({q2, 2, pauli_as_kraus(e2)});
  } else {
    m.add_rule({q1, 1, e1});
    m.add_rule({q2, 2, e2});
  }
  return m;
}

// ---------------------------------------------------------------------------
// instrument — program.cpp:17-122.
uint64_t NoisyCircuit::apply_sample_outcome(uint64_t creg, uint64_t outcome) const {
  for (const auto& [clbit, pos] : sample_writes)
    creg = (creg & ~one_bit(clbit)) | (((outcome >> pos) & 1) << clbit);
  return creg;
}

NoisyCircuit instrument(const Circuit& circuit, const NoiseModel& model) {
  require_valid(circuit);
  NoisyCircuit prog;
  prog.num_qubits = circuit.num_qubits;
  prog.num_clbits = circuit.num_clbits;
  std::vector<const ErrorChannel*> channel_ids;  // Kraus de-duplication by rule

  for (const Instruction& in : circuit.instructions) {
    ProgramOp op;
    op.qubits = in.qubits;
    op.condition = in.condition;
    if (in.kind == GateKind::BARRIER) {
      op.kind = ProgramOp::Kind::Barrier;
    } else if (in.kind == GateKind::MEASURE) {
      op.kind = ProgramOp::Kind::Measure;
      op.clbits = in.clbits;
      prog.has_measure = true;
    } else if (in.kind == GateKind::RESET) {
      op.kind = ProgramOp::Kind::Reset;
    } else {
      op.kind = ProgramOp::Kind::Gate;
      op.gate = in.kind;
      op.params = in.params;
      op.matrix = gate_matrix(in.kind, in.params);
    }
    prog.ops.push_back(std::move(op));

    const GateInfo& gi = gate_info(in.kind);
    if (!gi.unitary) continue;
    const ErrorChannel* ch = model.match(in.kind, gi.arity);
    if (!ch) continue;

    ProgramOp site;
    site.qubits = in.qubits;
    site.condition = in.condition;  // a skipped gate carries no noise either
    if (const auto* pe = std::get_if<PauliError>(ch)) {
      site.kind = ProgramOp::Kind::PauliSite;
      for (const auto& t : pe->terms) {
        const PauliString concrete = t.pauli.rebased(in.qubits);
        site.term_cum.push_back(t.cumulative);
        site.term_masks.push_back(pauli_to_masks(concrete));
        site.term_identity.push_back(concrete.is_identity() ? 1 : 0);
      }
      ++prog.pauli_sites;
    } else {
      site.kind = ProgramOp::Kind::KrausSite;
      auto it = std::find(channel_ids.begin(), channel_ids.end(), ch);
      if (it == channel_ids.end()) {
        channel_ids.push_back(ch);
        prog.kraus_channels.push_back(std::get<KrausError>(*ch));
        it = channel_ids.end() - 1;
      }
      site.channel = static_cast<uint32_t>(it - channel_ids.begin());
      ++prog.kraus_sites;
    }
    prog.ops.push_back(std::move(site));
  }

  for (ProgramOp& op : prog.ops)
    if (op.consumes_randomness()) op.event = prog.num_events++;

  size_t tb = prog.ops.size();
  while (tb > 0 && prog.ops[tb - 1].kind == ProgramOp::Kind::Measure) --tb;
  prog.terminal_measure_begin = tb;
  if (!prog.has_measure) return prog;

  uint64_t terminal_bits = 0;
  for (size_t i = tb; i < prog.ops.size(); ++i) {
    const ProgramOp& m = prog.ops[i];
    for (size_t b = 0; b < m.qubits.size(); ++b) {
      auto at = std::find(prog.sample_qubits.begin(), prog.sample_qubits.end(), m.qubits[b]);
      if (at == prog.sample_qubits.end()) at = prog.sample_qubits.insert(at, m.qubits[b]);
      prog.sample_writes.emplace_back(m.clbits[b], static_cast<unsigned>(at - prog.sample_qubits.begin()));
      terminal_bits |= one_bit(m.clbits[b]);
    }
  }
  bool ok = true;
  for (size_t i = 0; i < tb && ok; ++i) ok = prog.ops[i].kind != ProgramOp::Kind::Measure;
  for (size_t i = tb; i < prog.ops.size() && ok; ++i) ok = !prog.ops[i].condition;
  for (const ProgramOp& op : prog.ops)
    if (ok && op.condition && (op.condition->clbit_mask & terminal_bits)) ok = false;
  prog.sampling_eligible = ok;
  return prog;
}

// ---------------------------------------------------------------------------
// Results — result.cpp:7-48.
std::string bitstring(uint64_t v, unsigned width) {
  std::string s(width, '0');
  for (unsigned b = 0; b < width; ++b)
    if ((v >> b) & 1) s[width - 1 - b] = '1';
  return s;
}

Counts merge_counts(std::span<const Counts> parts) {
  Counts all;
  for (const Counts& p : parts)
    for (const auto& [k, n] : p) all[k] += n;
  return all;
}

uint64_t counts_checksum(const Counts& counts) {  // FNV-1a over "key=count;"
  uint64_t h = 0xcbf29ce484222325ull;
  auto eat = [&h](const std::string& s) {
    for (unsigned char ch : s) h = (h ^ ch) * 0x100000001b3ull;
  };
  for (const auto& [k, n] : counts) {
    eat(k);
    eat("=" + std::to_string(n) + ";");
  }
  return h;
}

Counts counts_from_values(std::span<const uint64_t> values, unsigned width, bool has_measure) {
  Counts c;
  if (!has_measure) {
    if (!values.empty()) c[""] = values.size();
    return c;
  }
  for (uint64_t v : values) ++c[bitstring(v, width)];
  return c;
}

// ---------------------------------------------------------------------------
// Flat C-ABI view and the exact dump used for lowering parity.
void flatten(const NoisyCircuit& p, FlatProgram& f) {
  f.ops.clear();
  f.terms.clear();
  f.channels.clear();
  f.matrices.clear();
  auto push_matrix = [&f](const GateMatrix& m) {
    const uint32_t idx = static_cast<uint32_t>(f.matrices.size() / SSB_MATRIX_STRIDE);
    f.matrices.resize(f.matrices.size() + SSB_MATRIX_STRIDE, 0.0);
    double* dst = f.matrices.data() + idx * SSB_MATRIX_STRIDE;
    for (size_t i = 0; i < m.entries.size() && i < 16; ++i) {
      dst[2 * i] = m.entries[i].real();
      dst[2 * i + 1] = m.entries[i].imag();
    }
    return idx;
  };
  for (const KrausError& k : p.kraus_channels) {
    ssb_flat_channel ch{k.arity, static_cast<uint32_t>(k.matrices.size()), 0, 0};
    for (size_t i = 0; i < k.matrices.size(); ++i) {
      const uint32_t idx = push_matrix(k.matrices[i]);
      if (i == 0) ch.matrix_begin = idx;
    }
    f.channels.push_back(ch);
  }
  for (const ProgramOp& op : p.ops) {
    ssb_flat_op o{};
    o.kind = static_cast<uint32_t>(op.kind);
    if (op.qubits.size() > SSB_MAX_OP_QUBITS || op.clbits.size() > SSB_MAX_OP_QUBITS)
      throw std::invalid_argument("op has more than 4 operands");
    o.num_qubits = static_cast<uint32_t>(op.qubits.size());
    for (size_t i = 0; i < op.qubits.size(); ++i) o.qubits[i] = op.qubits[i];
    for (size_t i = 0; i < op.clbits.size(); ++i) o.clbits[i] = op.clbits[i];
    o.has_condition = op.condition.has_value();
    if (op.condition) {
      o.cond_mask = op.condition->clbit_mask;
      o.cond_value = op.condition->value;
    }
    o.event = op.event;
    o.gate_kind = static_cast<uint32_t>(op.gate);
    o.channel = op.channel;
    if (op.kind == ProgramOp::Kind::Gate) o.matrix = push_matrix(op.matrix);
    if (op.kind == ProgramOp::Kind::PauliSite) {
      o.term_begin = static_cast<uint32_t>(f.terms.size());
      o.term_count = static_cast<uint32_t>(op.term_cum.size());
      for (size_t t = 0; t < op.term_cum.size(); ++t) {
        const PauliMasks& m = op.term_masks[t];
        f.terms.push_back({op.term_cum[t], m.x_mask, m.z_mask, m.num_y, m.x_max, op.term_identity[t], 0});
      }
    }
    f.ops.push_back(o);
  }
  f.sample_qubits.assign(p.sample_qubits.begin(), p.sample_qubits.end());
  f.write_clbit.clear();
  f.write_pos.clear();
  for (const auto& [c, b] : p.sample_writes) {
    f.write_clbit.push_back(c);
    f.write_pos.push_back(b);
  }
  ssb_flat_program& v = f.view;
  v = ssb_flat_program{};
  v.num_qubits = p.num_qubits;
  v.num_clbits = p.num_clbits;
  v.num_events = p.num_events;
  v.has_measure = p.has_measure;
  v.sampling_eligible = p.sampling_eligible;
  v.terminal_measure_begin = p.terminal_measure_begin;
  v.num_ops = f.ops.size();
  v.ops = f.ops.data();
  v.num_terms = f.terms.size();
  v.terms = f.terms.data();
  v.num_channels = f.channels.size();
  v.channels = f.channels.data();
  v.num_matrices = f.matrices.size() / SSB_MATRIX_STRIDE;
  v.matrices = f.matrices.data();
  v.num_sample_qubits = static_cast<uint32_t>(f.sample_qubits.size());
  v.sample_qubits = f.sample_qubits.data();
  v.num_sample_writes = static_cast<uint32_t>(f.write_clbit.size());
  v.sample_write_clbit = f.write_clbit.data();
  v.sample_write_pos = f.write_pos.data();
}

NoisyCircuit unflatten(const ssb_flat_program& v) {
  NoisyCircuit p;
  p.num_qubits = v.num_qubits;
  p.num_clbits = v.num_clbits;
  p.num_events = v.num_events;
  p.has_measure = v.has_measure != 0;
  p.sampling_eligible = v.sampling_eligible != 0;
  p.terminal_measure_begin = v.terminal_measure_begin;
  // Every count and index is validated BEFORE it is used to read a caller
  // buffer: a matrix slot holds at most a 4x4 (SSB_MATRIX_STRIDE doubles), so
  // matrices are 1- or 2-qubit; term / channel / matrix ranges must lie
  // inside their arrays; arrays with a nonzero count must be non-null.
  auto need = [](bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(std::string("malformed flat program: ") + what);
  };
  need(v.num_qubits >= 1 && v.num_qubits <= 30, "num_qubits outside 1..30");
  need(v.num_clbits <= 64, "num_clbits > 64");
  need(!v.num_ops || v.ops, "null ops");
  need(!v.num_terms || v.terms, "null terms");
  need(!v.num_channels || v.channels, "null channels");
  need(!v.num_matrices || v.matrices, "null matrices");
  need(!v.num_sample_qubits || v.sample_qubits, "null sample_qubits");
  need(!v.num_sample_writes || (v.sample_write_clbit && v.sample_write_pos), "null sample_writes");
  need(v.terminal_measure_begin <= v.num_ops, "terminal_measure_begin > num_ops");
  auto read_matrix = [&v, &need](uint32_t idx, unsigned k) {
    need(k == 1 || k == 2, "matrix arity outside 1..2");
    if (idx >= v.num_matrices) throw std::invalid_argument("matrix index out of range");
    GateMatrix m{k, {}};
    const double* src = v.matrices + size_t(idx) * SSB_MATRIX_STRIDE;
    for (uint64_t i = 0; i < one_bit(2 * k); ++i) m.entries.emplace_back(src[2 * i], src[2 * i + 1]);
    return m;
  };
  for (uint64_t c = 0; c < v.num_channels; ++c) {
    KrausError k;
    k.arity = v.channels[c].arity;
    need(k.arity == 1 || k.arity == 2, "channel arity outside 1..2");
    need(uint64_t{v.channels[c].matrix_begin} + v.channels[c].num_matrices <= v.num_matrices,
         "channel matrices out of range");
    for (uint32_t i = 0; i < v.channels[c].num_matrices; ++i)
      k.matrices.push_back(read_matrix(v.channels[c].matrix_begin + i, k.arity));
    p.kraus_channels.push_back(std::move(k));
  }
  for (uint64_t i = 0; i < v.num_ops; ++i) {
    const ssb_flat_op& o = v.ops[i];
    if (o.kind > SSB_OP_BARRIER || o.num_qubits > SSB_MAX_OP_QUBITS)
      throw std::invalid_argument("malformed flat op");
    for (uint32_t b = 0; b < o.num_qubits; ++b) need(o.qubits[b] < v.num_qubits, "op qubit out of range");
    if (o.kind == SSB_OP_PAULI)
      need(o.term_count >= 1 && uint64_t{o.term_begin} + o.term_count <= v.num_terms, "op terms out of range");
    ProgramOp op;
    op.kind = static_cast<ProgramOp::Kind>(o.kind);
    op.qubits.assign(o.qubits, o.qubits + o.num_qubits);
    if (op.kind == ProgramOp::Kind::Measure) op.clbits.assign(o.clbits, o.clbits + o.num_qubits);
    if (o.has_condition) op.condition = Condition{o.cond_mask, o.cond_value};
    op.event = o.event;
    op.gate = static_cast<GateKind>(o.gate_kind);
    op.channel = o.channel;
    if (op.kind == ProgramOp::Kind::Gate) op.matrix = read_matrix(o.matrix, o.num_qubits);
    if (op.kind == ProgramOp::Kind::PauliSite) {
      ++p.pauli_sites;
      for (uint32_t t = 0; t < o.term_count; ++t) {
        const ssb_flat_term& ft = v.terms[o.term_begin + t];
        op.term_cum.push_back(ft.cumulative);
        op.term_masks.push_back({ft.x_mask, ft.z_mask, ft.num_y, ft.x_max});
        op.term_identity.push_back(static_cast<uint8_t>(ft.identity));
      }
    }
    if (op.kind == ProgramOp::Kind::KrausSite) {
      ++p.kraus_sites;
      if (op.channel >= p.kraus_channels.size()) throw std::invalid_argument("kraus channel out of range");
    }
    p.ops.push_back(std::move(op));
  }
  need(v.num_sample_qubits <= v.num_qubits, "too many sample qubits");
  p.sample_qubits.assign(v.sample_qubits, v.sample_qubits + v.num_sample_qubits);
  for (uint32_t i = 0; i < v.num_sample_writes; ++i)
    p.sample_writes.emplace_back(v.sample_write_clbit[i], v.sample_write_pos[i]);
  return p;
}

std::string dump_program(const NoisyCircuit& p) {
  auto hx = [](double d) {
    char b[64];
    std::snprintf(b, sizeof b, "%a", d);
    return std::string(b);
  };
  auto cx = [&hx](const cplx& e) { return " " + hx(e.real()) + "," + hx(e.imag()); };
  std::ostringstream o;
  o << "program " << p.num_qubits << " " << p.num_clbits << " events " << p.num_events << " pauli "
    << p.pauli_sites << " kraus " << p.kraus_sites << " measure " << p.has_measure << " eligible "
    << p.sampling_eligible << " tbegin " << p.terminal_measure_begin << "\nsample_qubits";
  for (unsigned q : p.sample_qubits) o << " " << q;
  o << "\nsample_writes";
  for (const auto& [c, b] : p.sample_writes) o << " " << c << ":" << b;
  o << "\n";
  for (size_t ci = 0; ci < p.kraus_channels.size(); ++ci) {
    const KrausError& k = p.kraus_channels[ci];
    o << "channel " << ci << " arity " << k.arity << " matrices " << k.matrices.size() << "\n";
    for (const GateMatrix& m : k.matrices) {
      o << " m";
      for (const cplx& e : m.entries) o << cx(e);
      o << "\n";
    }
  }
  for (const ProgramOp& op : p.ops) {
    o << "op " << static_cast<int>(op.kind) << " q";
    for (unsigned q : op.qubits) o << " " << q;
    o << " c";
    for (unsigned c : op.clbits) o << " " << c;
    if (op.condition) o << " if " << op.condition->clbit_mask << "==" << op.condition->value;
    if (op.consumes_randomness()) o << " ev " << op.event;
    if (op.kind == ProgramOp::Kind::Gate) {
      o << " g " << static_cast<int>(op.gate) << " m";
      for (const cplx& e : op.matrix.entries) o << cx(e);
    }
    if (op.kind == ProgramOp::Kind::KrausSite) o << " ch " << op.channel;
    if (op.kind == ProgramOp::Kind::PauliSite)
      for (size_t t = 0; t < op.term_cum.size(); ++t) {
        const PauliMasks& m = op.term_masks[t];
        o << " t " << hx(op.term_cum[t]) << " " << m.x_mask << " " << m.z_mask << " " << m.num_y << " "
          << (m.x_mask ? m.x_max : 0) << " " << int(op.term_identity[t]);
      }
    o << "\n";
  }
  return o.str();
}

}  // namespace shotsim
