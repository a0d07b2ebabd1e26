// C++ executors with the reference's ExecutorFn contract (exec.hpp:24-35):
// "gpu-batch" / "gpu-branch" run the instrumented program on sm_100a through
// the C ABI. RunOptions::workers selects how many GPUs (devices
// 0..workers-1) share the shots: contiguous shot-id shards, one host thread
// per device, per-shard values concatenated and folded into Counts on the
// host (merge_counts is commutative, result.cpp:15-21).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <thread>

#include "../capi_internal.hpp"

namespace shotsim {

namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = ssb_last_error();
  switch (rc) {
    case SSB_ERR_CAPACITY: throw CapacityError(msg);
    case SSB_ERR_DEGENERATE: throw DegenerateDistribution(msg);
    case SSB_ERR_CONFIG: throw ConfigError(msg);
    case SSB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw std::runtime_error(msg);
  }
}

using RunFn = int (*)(ssb_engine*, const ssb_program*, uint64_t, uint64_t, uint64_t, const ssb_run_options*,
                      uint64_t*, ssb_stats*);

RunResult run_sharded(const NoisyCircuit& program, const RunOptions& o, RunFn fn, const char* name) {
  if (o.shots < 1) throw std::invalid_argument("shots must be >= 1");
  if (o.workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (fn == &ssb_run_branch && o.branch_budget < 1) throw std::invalid_argument("branch budget must be >= 1");
  const auto t0 = std::chrono::steady_clock::now();
  FlatProgram flat;
  flatten(program, flat);
  ssb_program* prog = nullptr;
  if (int rc = ssb_program_from_flat(&flat.view, &prog)) rethrow(rc);
  std::unique_ptr<ssb_program, void (*)(ssb_program*)> hold(prog, ssb_program_destroy);

  ssb_run_options ro{};
  ro.max_batch_size = o.max_batch_size;
  ro.branch_budget = o.branch_budget;
  ro.mem_limit_bytes = o.mem_limit_bytes;
  ro.check_norms = o.check_norms;
  ro.collect_leaf_stats = o.collect_leaf_stats;

  const unsigned G = static_cast<unsigned>(std::min<uint64_t>(o.workers, o.shots));
  std::vector<uint64_t> values(o.shots);
  std::vector<ssb_stats> stats(G);
  std::vector<int> rcs(G, 0);
  std::vector<std::string> errs(G);
  std::vector<std::thread> pool;
  uint64_t begin = 0;
  for (unsigned g = 0; g < G; ++g) {
    const uint64_t len = o.shots / G + (g < o.shots % G ? 1 : 0);
    pool.emplace_back([&, g, begin, len] {
      ssb_engine* E = nullptr;
      rcs[g] = ssb_engine_create(static_cast<int>(g), &E);
      if (rcs[g] == 0) {
        rcs[g] = fn(E, prog, begin, len, o.seed, &ro, values.data() + begin, &stats[g]);
        ssb_engine_destroy(E);
      }
      if (rcs[g]) errs[g] = ssb_last_error();
    });
    begin += len;
  }
  for (auto& t : pool) t.join();
  for (unsigned g = 0; g < G; ++g)
    if (rcs[g]) {
      ssb::set_last_error(errs[g]);
      rethrow(rcs[g]);
    }

  RunResult r;
  r.strategy = name;
  r.shots = o.shots;
  r.seed = o.seed;
  r.workers = o.workers;
  for (const ssb_stats& s : stats) {
    r.dispatch_count += s.dispatch_count;
    r.peak_states += s.peak_states;
    r.branch.passes = std::max(r.branch.passes, s.passes);
  }
  r.branch.peak_states = r.peak_states;
  r.counts = counts_from_values(values, program.num_clbits, program.has_measure);
  if (o.record_shot_values) r.shot_values = std::move(values);
  r.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

}  // namespace

RunResult run_gpu_batch(const NoisyCircuit& program, const RunOptions& options) {
  return run_sharded(program, options, &ssb_run_batch, "gpu-batch");
}

RunResult run_gpu_branch(const NoisyCircuit& program, const RunOptions& options) {
  return run_sharded(program, options, &ssb_run_branch, "gpu-branch");
}

ExecutorFn executor_by_name(std::string_view name) {
  if (name == "gpu-batch") return &run_gpu_batch;
  if (name == "gpu-branch") return &run_gpu_branch;
  throw ConfigError("unknown strategy: " + std::string(name));
}

namespace {

// Device 0 engine + flattened program for the density-matrix checker.
template <class F>
void with_engine(const NoisyCircuit& program, F&& f) {
  FlatProgram flat;
  flatten(program, flat);
  ssb_program* prog = nullptr;
  if (int rc = ssb_program_from_flat(&flat.view, &prog)) rethrow(rc);
  std::unique_ptr<ssb_program, void (*)(ssb_program*)> hold(prog, ssb_program_destroy);
  ssb_engine* E = nullptr;
  if (int rc = ssb_engine_create(0, &E)) rethrow(rc);
  std::unique_ptr<ssb_engine, void (*)(ssb_engine*)> hold_e(E, ssb_engine_destroy);
  if (int rc = f(E, prog)) rethrow(rc);
}

}  // namespace

std::vector<double> exact_distribution(const NoisyCircuit& program, std::span<const unsigned> qubits) {
  if (qubits.size() > 63) throw std::invalid_argument("too many qubits");
  std::vector<uint32_t> q(qubits.begin(), qubits.end());
  std::vector<double> out(uint64_t{1} << q.size());
  with_engine(program, [&](ssb_engine* E, ssb_program* p) {
    return ssb_exact_distribution(E, p, q.data(), static_cast<uint32_t>(q.size()), out.data());
  });
  return out;
}

std::map<uint64_t, double> exact_creg_distribution(const NoisyCircuit& program) {
  std::vector<uint64_t> keys;
  std::vector<double> probs;
  with_engine(program, [&](ssb_engine* E, ssb_program* p) {
    uint64_t n = 0;
    if (int rc = ssb_exact_creg_distribution(E, p, nullptr, nullptr, 0, &n)) return rc;
    keys.resize(n);
    probs.resize(n);
    return ssb_exact_creg_distribution(E, p, keys.data(), probs.data(), n, &n);
  });
  std::map<uint64_t, double> out;
  for (size_t i = 0; i < keys.size(); ++i) out.emplace(keys[i], probs[i]);
  return out;
}

// density.cpp:308-315 over Counts directly (the C ABI takes per-shot values).
double tvd_vs_exact(const Counts& counts, uint64_t shots, const std::map<uint64_t, double>& exact) {
  std::map<uint64_t, double> empirical;
  for (const auto& [key, n] : counts) {
    const uint64_t v = key.empty() ? 0 : std::stoull(key, nullptr, 2);
    empirical[v] += static_cast<double>(n) / static_cast<double>(shots);
  }
  double l1 = 0.0;
  auto ie = empirical.begin();
  auto ix = exact.begin();
  while (ie != empirical.end() || ix != exact.end()) {
    if (ix == exact.end() || (ie != empirical.end() && ie->first < ix->first)) {
      l1 += std::abs(ie->second);
      ++ie;
    } else if (ie == empirical.end() || ix->first < ie->first) {
      l1 += std::abs(ix->second);
      ++ix;
    } else {
      l1 += std::abs(ie->second - ix->second);
      ++ie;
      ++ix;
    }
  }
  return 0.5 * l1;
}

uint64_t default_mem_limit_bytes() {
  if (const char* env = std::getenv("SHOTSIM_MEM_LIMIT_BYTES")) {
    const uint64_t v = std::strtoull(env, nullptr, 10);
    if (v > 0) return v;
  }
  return uint64_t{1} << 30;
}

}  // namespace shotsim
