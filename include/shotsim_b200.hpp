// shotsim_b200 — C++ host API, a drop-in for the reference's shotsim host
// surface (circuit / noise model / instrument / run). Names, argument meaning
// and error behaviour follow the reference headers cited per declaration; the
// executors registered here ("gpu-batch", "gpu-branch") run on sm_100a
// through the C ABI in shotsim_b200.h.
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <variant>
#include <vector>

#include "shotsim_b200.h"

#pragma GCC visibility push(default)
namespace shotsim {

using cplx = std::complex<double>;

// Error types — common.hpp:18-34.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DegenerateDistribution : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline constexpr uint64_t one_bit(unsigned b) { return uint64_t{1} << b; }

// ---- circuit (circuit.hpp:14-88) -----------------------------------------
enum class GateKind : uint8_t {
  ID, X, Y, Z, H, S, SDG, T, TDG, P, U, CX, CP, SWAP, MEASURE, RESET, BARRIER,
};

struct GateInfo {
  std::string_view name;
  unsigned arity;
  unsigned num_params;
  bool unitary;
};

const GateInfo& gate_info(GateKind kind);
std::optional<GateKind> gate_kind_from_name(std::string_view name);

struct Condition {
  uint64_t clbit_mask = 0;
  uint64_t value = 0;
  bool holds(uint64_t creg) const { return (creg & clbit_mask) == value; }
  bool operator==(const Condition&) const = default;
};

struct Instruction {
  GateKind kind;
  std::vector<unsigned> qubits;
  std::vector<unsigned> clbits;
  std::vector<double> params;
  std::optional<Condition> condition;
  bool operator==(const Instruction&) const = default;
};

struct Circuit {
  unsigned num_qubits = 0;
  unsigned num_clbits = 0;
  std::vector<Instruction> instructions;
  bool operator==(const Circuit&) const = default;
};

struct Violation {
  size_t instruction;
  std::string message;
};

std::vector<Violation> validate(const Circuit& circuit);
void require_valid(const Circuit& circuit);
Circuit qft_circuit(unsigned n);
Circuit measure_all(Circuit circuit);

struct GateMatrix {
  unsigned num_qubits = 0;
  std::vector<cplx> entries;  // row-major 2^k x 2^k
  uint64_t dim() const { return one_bit(num_qubits); }
  cplx at(uint64_t r, uint64_t c) const { return entries[r * dim() + c]; }
};

GateMatrix gate_matrix(GateKind kind, std::span<const double> params);

// ---- circuit text / JSON (circuit_io.hpp:13-33) ----------------------------
std::string circuit_to_text(const Circuit& circuit);
Circuit circuit_from_text(const std::string& text);
std::string circuit_to_json(const Circuit& circuit);
Circuit circuit_from_json(const std::string& text);
Circuit load_circuit(const std::string& path);

// ---- noise (noise.hpp:14-103) ---------------------------------------------
struct PauliMasks {  // kernels.hpp:15-22
  uint64_t x_mask = 0;
  uint64_t z_mask = 0;
  unsigned num_y = 0;
  unsigned x_max = 0;
  bool is_identity() const { return x_mask == 0 && z_mask == 0 && num_y == 0; }
};

enum class PauliLetter : uint8_t { I, X, Y, Z };
char pauli_letter_char(PauliLetter l);
PauliLetter pauli_letter_from_char(char c);

struct PauliString {
  std::vector<PauliLetter> letters;
  std::vector<unsigned> targets;
  bool is_identity() const;
  PauliString rebased(std::span<const unsigned> qubits) const;
  std::string to_string() const;
};

PauliMasks pauli_to_masks(const PauliString& pauli);
GateMatrix pauli_string_matrix(const PauliString& pauli);

struct PauliError {
  struct Term {
    double cumulative;
    PauliString pauli;
  };
  std::vector<Term> terms;
  unsigned arity = 0;
  double term_prob(size_t i) const;
};

struct KrausError {
  std::vector<GateMatrix> matrices;
  unsigned arity = 0;
};

using ErrorChannel = std::variant<PauliError, KrausError>;
unsigned channel_arity(const ErrorChannel& channel);

PauliError depolarizing_error(double p, unsigned k);
size_t sample_pauli_index(const PauliError& error, double u);
KrausError pauli_as_kraus(const PauliError& error);
double kraus_completeness_defect(const KrausError& kraus);

struct NoiseRule {
  std::vector<GateKind> gates;
  unsigned arity = 0;
  ErrorChannel channel;
};

class NoiseModel {
 public:
  void add_rule(NoiseRule rule);
  const ErrorChannel* match(GateKind kind, unsigned arity) const;
  bool empty() const { return rules_.empty(); }
  const std::vector<NoiseRule>& rules() const { return rules_; }
  std::string to_json() const;
  // Accepts the reference schema, "" (empty model) and the extension
  // {"model":"depolarizing","rate":r,"as_kraus":b}.
  static NoiseModel from_json(const std::string& text);
  static NoiseModel load(const std::string& path);

 private:
  std::vector<NoiseRule> rules_;
};

NoiseModel make_depolarizing_model(double rate, bool as_kraus);

// ---- instrumented program (program.hpp:18-76) -----------------------------
struct ProgramOp {
  enum class Kind : uint8_t { Gate, PauliSite, KrausSite, Measure, Reset, Barrier };
  Kind kind = Kind::Gate;
  GateKind gate = GateKind::ID;
  std::vector<unsigned> qubits;
  std::vector<unsigned> clbits;
  std::vector<double> params;
  std::optional<Condition> condition;
  GateMatrix matrix;
  uint32_t channel = 0;
  uint64_t event = 0;
  std::vector<double> term_cum;
  std::vector<PauliMasks> term_masks;
  std::vector<uint8_t> term_identity;
  bool consumes_randomness() const {
    return kind == Kind::PauliSite || kind == Kind::KrausSite || kind == Kind::Measure ||
           kind == Kind::Reset;
  }
};

struct NoisyCircuit {
  unsigned num_qubits = 0;
  unsigned num_clbits = 0;
  std::vector<ProgramOp> ops;
  std::vector<KrausError> kraus_channels;
  uint64_t num_events = 0;
  uint64_t pauli_sites = 0;
  uint64_t kraus_sites = 0;
  bool has_measure = false;
  bool sampling_eligible = false;
  size_t terminal_measure_begin = 0;
  std::vector<unsigned> sample_qubits;
  std::vector<std::pair<unsigned, unsigned>> sample_writes;
  uint64_t sampling_event() const { return num_events; }
  uint64_t noise_sites() const { return pauli_sites + kraus_sites; }
  uint64_t apply_sample_outcome(uint64_t creg, uint64_t outcome) const;
};

NoisyCircuit instrument(const Circuit& circuit, const NoiseModel& model);

// ---- results (result.hpp:14-52) -------------------------------------------
using Counts = std::map<std::string, uint64_t>;
std::string bitstring(uint64_t value, unsigned width);
Counts merge_counts(std::span<const Counts> partials);
uint64_t counts_checksum(const Counts& counts);
Counts counts_from_values(std::span<const uint64_t> values, unsigned width, bool has_measure);

struct BranchStats {
  uint64_t peak_states = 0;
  uint64_t passes = 0;
  std::vector<uint64_t> leaf_shots;
};

struct RunResult {
  Counts counts;
  double wall_seconds = 0.0;
  uint64_t dispatch_count = 0;
  uint64_t peak_states = 0;
  BranchStats branch;
  std::string strategy;
  uint64_t shots = 0;
  uint64_t seed = 0;
  unsigned workers = 1;
  std::vector<uint64_t> shot_values;
  std::vector<unsigned> shard_devices;  // extension: per shot shard, the device that ran it
};

// ---- executors (exec.hpp:12-38) --------------------------------------------
struct RunOptions {
  uint64_t shots = 1;
  uint64_t seed = 0;
  unsigned workers = 1;          // shot shards (contiguous id ranges), pulled by the
                                 // devices as they become free — a performance hint
                                 // only: results never depend on it (exec.hpp:24-27)
  uint64_t max_batch_size = 0;
  uint64_t branch_budget = 64;
  uint64_t mem_limit_bytes = 0;
  bool record_shot_values = false;
  bool check_norms = false;
  bool collect_leaf_stats = false;
  bool fused_matrices = false;   // ssb_run_options::fused_matrices (gpu-batch)
};

RunResult run_gpu_batch(const NoisyCircuit& program, const RunOptions& options);
RunResult run_gpu_branch(const NoisyCircuit& program, const RunOptions& options);

using ExecutorFn = RunResult (*)(const NoisyCircuit&, const RunOptions&);
// "gpu-batch" | "gpu-branch"; ConfigError for anything else.
ExecutorFn executor_by_name(std::string_view name);
uint64_t default_mem_limit_bytes();

// The reference's statistical checker (density.hpp:56-68), evolved on device 0
// (n <= 10; CapacityError / std::invalid_argument as the reference).
std::vector<double> exact_distribution(const NoisyCircuit& program, std::span<const unsigned> qubits);
std::map<uint64_t, double> exact_creg_distribution(const NoisyCircuit& program);
double tvd_vs_exact(const Counts& counts, uint64_t shots, const std::map<uint64_t, double>& exact);

// Flat (C ABI) view of an instrumented program; storage owned by the holder.
struct FlatProgram {
  ssb_flat_program view{};
  std::vector<ssb_flat_op> ops;
  std::vector<ssb_flat_term> terms;
  std::vector<ssb_flat_channel> channels;
  std::vector<double> matrices;
  std::vector<uint32_t> sample_qubits, write_clbit, write_pos;
};
void flatten(const NoisyCircuit& program, FlatProgram& out);
NoisyCircuit unflatten(const ssb_flat_program& flat);
std::string dump_program(const NoisyCircuit& program);

}  // namespace shotsim
#pragma GCC visibility pop
