// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj),
// compiled from its own sources by oracle/Makefile into oracle/_ref/. Python
// tests (and bench.py's cpu_baseline / --impl reference legs) load it with
// ctypes to (a) pin the C restatement in oracle/shotsim_oracle.c and (b) time
// the reference's own CPU executors. Only tests/, __graft_entry__.smoke() and
// bench.py may load this.
//
// Every entry point returns 0 on success, nonzero on error; the message is in
// ref_last_error(). Inputs use the reference's own lossless formats:
// circuit text (circuit_io.cpp:53-146) and noise JSON (noise.cpp:328-365),
// plus one extension understood by both this shim and the product front-end:
// {"model":"depolarizing","rate":R,"as_kraus":B} → make_depolarizing_model
// (noise.cpp:375-392).
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <exception>
#include <map>
#include <numeric>
#include <sstream>
#include <string>

#include <json.hpp>

#include "shotsim/circuit_io.hpp"
#include "shotsim/density.hpp"
#include "shotsim/exec.hpp"
#include "shotsim/exec_batch.hpp"
#include "shotsim/exec_branch.hpp"
#include "shotsim/exec_naive.hpp"
#include "shotsim/kernels.hpp"
#include "shotsim/noise.hpp"
#include "shotsim/program.hpp"
#include "shotsim/rng.hpp"
#include "shotsim/statevector.hpp"

using namespace shotsim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const CapacityError& e) {
    g_err = std::string("CapacityError: ") + e.what();
    return 4;
  } catch (const DegenerateDistribution& e) {
    g_err = std::string("DegenerateDistribution: ") + e.what();
    return 5;
  } catch (const ConfigError& e) {
    g_err = std::string("ConfigError: ") + e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("error: ") + e.what();
    return 1;
  }
}

NoiseModel parse_noise(const char* noise) {
  if (noise == nullptr || noise[0] == '\0') return NoiseModel{};
  auto j = nlohmann::json::parse(noise);
  if (j.contains("model")) {
    if (j["model"].get<std::string>() != "depolarizing") throw ConfigError("unknown model");
    return make_depolarizing_model(j.at("rate").get<double>(), j.value("as_kraus", false));
  }
  return NoiseModel::from_json(noise);
}

NoisyCircuit build(const char* circuit_text, const char* noise) {
  return instrument(circuit_from_text(circuit_text), parse_noise(noise));
}

std::string hexd(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", v);
  return buf;
}

}  // namespace

extern "C" {

struct ref_stats {
  uint64_t dispatch_count;
  uint64_t peak_states;
  uint64_t passes;
  double wall_seconds;
  uint64_t counts_checksum;
  uint64_t num_keys;
};

const char* ref_last_error() { return g_err.c_str(); }

int ref_select_kernels(const char* which) {
  return guarded([&] { select_kernels(which); });
}

void ref_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const auto r = philox4x32({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = r[i];
}

double ref_uniform(uint64_t seed, uint64_t shot, uint64_t event) {
  return uniform(seed, shot, event);
}

// Runs an executor ("naive" | "batch" | "branch") and returns per-shot
// register values (values_out: shots entries, may be NULL).
int ref_run(const char* circuit_text, const char* noise, const char* strategy, uint64_t shots,
            uint64_t seed, unsigned workers, uint64_t max_batch, uint64_t budget,
            uint64_t* values_out, ref_stats* stats) {
  return guarded([&] {
    const NoisyCircuit program = build(circuit_text, noise);
    RunOptions o;
    o.shots = shots;
    o.seed = seed;
    o.workers = workers;
    o.max_batch_size = max_batch;
    o.branch_budget = budget;
    o.record_shot_values = true;
    const RunResult r = executor_by_name(strategy)(program, o);
    if (values_out) std::memcpy(values_out, r.shot_values.data(), shots * sizeof(uint64_t));
    if (stats) {
      stats->dispatch_count = r.dispatch_count;
      stats->peak_states = r.peak_states;
      stats->passes = r.branch.passes;
      stats->wall_seconds = r.wall_seconds;
      stats->counts_checksum = counts_checksum(r.counts);
      stats->num_keys = r.counts.size();
    }
  });
}

// run_single_shot on an arbitrary shot id: final state + register.
int ref_single_shot(const char* circuit_text, const char* noise, uint64_t shot, uint64_t seed,
                    double* amps_out, uint64_t* creg_out) {
  return guarded([&] {
    const NoisyCircuit program = build(circuit_text, noise);
    Amplitudes state(program.num_qubits);
    *creg_out = run_single_shot(program, shot, seed, state);
    if (amps_out) std::memcpy(amps_out, state.view().data(), state.dim() * sizeof(cplx));
  });
}

// Per-shot register values for an arbitrary id list, through run_single_shot
// over the given ids (the CPU-baseline unit for sub-sampled configs).
int ref_run_ids(const char* circuit_text, const char* noise, const uint64_t* ids, uint64_t count,
                uint64_t seed, unsigned workers, uint64_t* values_out, double* seconds_out) {
  return guarded([&] {
    const NoisyCircuit program = build(circuit_text, noise);
    const auto t0 = std::chrono::steady_clock::now();
    parallel_chunks(workers, count, [&](uint64_t b, uint64_t e) {
      Amplitudes state(program.num_qubits);
      for (uint64_t i = b; i < e; ++i) values_out[i] = run_single_shot(program, ids[i], seed, state);
    });
    if (seconds_out) {
      *seconds_out =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

// BatchState over explicit ids: runs the program and exports all segments
// (count * 2^n complex) and registers.
int ref_batch_segments(const char* circuit_text, const char* noise, const uint64_t* ids,
                       uint64_t count, uint64_t seed, double* amps_out, uint64_t* cregs_out,
                       uint64_t* dispatches_out) {
  return guarded([&] {
    const NoisyCircuit program = build(circuit_text, noise);
    BatchState bs(program.num_qubits, std::vector<uint64_t>(ids, ids + count), seed);
    bs.run(program);
    const uint64_t dim = one_bit(program.num_qubits);
    for (uint64_t s = 0; s < count; ++s) {
      if (amps_out) std::memcpy(amps_out + 2 * s * dim, bs.segment(s).data(), dim * sizeof(cplx));
      if (cregs_out) cregs_out[s] = bs.creg(s);
    }
    if (dispatches_out) *dispatches_out = bs.dispatches();
  });
}

// Text dump of the instrumented program, doubles in %a (exact). The product
// front-end emits the same format (ssb_program_dump) so the two lowerings can
// be compared byte for byte.
int ref_program_dump(const char* circuit_text, const char* noise, char* out, size_t cap,
                     size_t* len_out) {
  return guarded([&] {
    const NoisyCircuit p = build(circuit_text, noise);
    std::ostringstream o;
    o << "program " << p.num_qubits << " " << p.num_clbits << " events " << p.num_events
      << " pauli " << p.pauli_sites << " kraus " << p.kraus_sites << " measure "
      << p.has_measure << " eligible " << p.sampling_eligible << " tbegin "
      << p.terminal_measure_begin << "\n";
    o << "sample_qubits";
    for (unsigned q : p.sample_qubits) o << " " << q;
    o << "\nsample_writes";
    for (const auto& [c, b] : p.sample_writes) o << " " << c << ":" << b;
    o << "\n";
    for (size_t ci = 0; ci < p.kraus_channels.size(); ++ci) {
      const KrausError& k = p.kraus_channels[ci];
      o << "channel " << ci << " arity " << k.arity << " matrices " << k.matrices.size() << "\n";
      for (const GateMatrix& m : k.matrices) {
        o << " m";
        for (const cplx& e : m.entries) o << " " << hexd(e.real()) << "," << hexd(e.imag());
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
        for (const cplx& e : op.matrix.entries) o << " " << hexd(e.real()) << "," << hexd(e.imag());
      }
      if (op.kind == ProgramOp::Kind::KrausSite) o << " ch " << op.channel;
      if (op.kind == ProgramOp::Kind::PauliSite) {
        for (size_t t = 0; t < op.term_cum.size(); ++t) {
          const PauliMasks& m = op.term_masks[t];
          o << " t " << hexd(op.term_cum[t]) << " " << m.x_mask << " " << m.z_mask << " "
            << m.num_y << " " << (m.x_mask ? m.x_max : 0) << " " << int(op.term_identity[t]);
        }
      }
      o << "\n";
    }
    const std::string s = o.str();
    if (len_out) *len_out = s.size();
    if (out && cap > 0) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(out, s.data(), n);
      out[n] = '\0';
    }
  });
}

// The reference's exact density-matrix evolver (density.cpp:280-306): the
// statistical checker SURVEY.md §8(f) rank 4 asks the GPU evolver to match.
// keys/probs NULL: size query only.
int ref_exact_creg_distribution(const char* circuit_text, const char* noise, uint64_t* keys, double* probs,
                                uint64_t cap, uint64_t* count) {
  return guarded([&] {
    const NoisyCircuit p = build(circuit_text, noise);
    const std::map<uint64_t, double> d = exact_creg_distribution(p);
    *count = d.size();
    if (!keys) return;
    if (cap < d.size()) throw std::invalid_argument("capacity too small");
    uint64_t i = 0;
    for (const auto& [k, v] : d) {
      keys[i] = k;
      probs[i] = v;
      ++i;
    }
  });
}

int ref_exact_distribution(const char* circuit_text, const char* noise, const unsigned* qubits, unsigned count,
                           double* out) {
  return guarded([&] {
    const NoisyCircuit p = build(circuit_text, noise);
    const std::vector<double> d = exact_distribution(p, std::span<const unsigned>(qubits, count));
    std::copy(d.begin(), d.end(), out);
  });
}

}  // extern "C"
