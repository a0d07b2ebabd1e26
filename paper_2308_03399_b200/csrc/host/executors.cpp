// C++ executors with the reference's ExecutorFn contract (exec.hpp:24-35):
// "gpu-batch" / "gpu-branch" run the instrumented program on sm_100a through
// the C ABI. RunOptions::workers keeps the reference's meaning of a
// parallelism hint (exec.hpp:24-27: results never depend on it): the shots
// split into min(workers, shots) contiguous shot-id shards, and one host thread
// per device pulls the next pending shard from a shared counter whenever its
// device is free (dynamic balancing: a device whose shards branch less or run
// faster takes over the shards still waiting), each on a pooled engine
// (engines — and their device buffers and programs cache — persist across
// calls). Values are keyed by shot id, so where a shard runs never changes
// them. Per-shard values are concatenated and folded into Counts on the host
// (merge_counts is commutative, result.cpp:15-21).
#include <atomic>
#include <chrono>
#include <cmath>
#include <map>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <thread>

#include <cuda_runtime.h>

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

// One engine per device, created on first use and kept for the process
// (re-creating an engine per call would re-allocate its state buffers — up to
// 16 GiB — and re-upload programs every run). Each device's engine is used by
// one thread at a time.
struct PooledEngine {
  std::mutex mu;
  ssb_engine* engine = nullptr;
};

PooledEngine& pooled_engine(int device) {
  static std::mutex pool_mu;
  static std::map<int, std::unique_ptr<PooledEngine>> pool;  // never freed: lives until exit
  std::lock_guard<std::mutex> lk(pool_mu);
  auto& slot = pool[device];
  if (!slot) slot = std::make_unique<PooledEngine>();
  return *slot;
}

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

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
  ro.fused_matrices = o.fused_matrices;

  const int ndev = device_count();
  if (ndev == 0) throw std::runtime_error("CUDA: no CUDA device available (shotsim_b200 has no CPU execution path)");
  const uint64_t G = std::min<uint64_t>(o.workers, o.shots);  // shards
  std::vector<uint64_t> values(o.shots);
  std::vector<uint64_t> shard_begin(G + 1, 0);
  for (uint64_t g = 0; g < G; ++g) shard_begin[g + 1] = shard_begin[g] + o.shots / G + (g < o.shots % G ? 1 : 0);
  std::vector<ssb_stats> stats(G);
  std::vector<std::vector<uint64_t>> leaves(G);
  const unsigned D = static_cast<unsigned>(std::min<uint64_t>(G, static_cast<uint64_t>(ndev)));  // devices used
  std::vector<int> rcs(D, 0);
  std::vector<std::string> errs(D);
  std::vector<unsigned> shard_dev(G, 0);
  std::atomic<uint64_t> next_shard{0};
  std::atomic<bool> failed{false};
  std::vector<std::thread> pool;
  for (unsigned d = 0; d < D; ++d) {
    pool.emplace_back([&, d] {
      PooledEngine& pe = pooled_engine(static_cast<int>(d));
      std::lock_guard<std::mutex> lk(pe.mu);
      if (!pe.engine) rcs[d] = ssb_engine_create(static_cast<int>(d), &pe.engine);
      for (uint64_t g; rcs[d] == 0 && !failed.load() && (g = next_shard.fetch_add(1)) < G;) {
        shard_dev[g] = d;
        ssb_run_options so = ro;
        std::vector<uint64_t>& lv = leaves[g];
        if (o.collect_leaf_stats) {
          lv.resize(1024);
          so.leaf_shots = lv.data();
          so.leaf_shots_capacity = lv.size();
        }
        const uint64_t b = shard_begin[g], len = shard_begin[g + 1] - b;
        rcs[d] = fn(pe.engine, prog, b, len, o.seed, &so, values.data() + b, &stats[g]);
        if (rcs[d] == 0 && o.collect_leaf_stats && stats[g].num_leaves > lv.size()) {  // too small: rerun sized
          lv.resize(stats[g].num_leaves);
          so.leaf_shots = lv.data();
          so.leaf_shots_capacity = lv.size();
          rcs[d] = fn(pe.engine, prog, b, len, o.seed, &so, values.data() + b, &stats[g]);
        }
        if (rcs[d] == 0 && o.collect_leaf_stats) lv.resize(stats[g].num_leaves);
      }
      if (rcs[d]) {
        errs[d] = ssb_last_error();
        failed = true;
      }
    });
  }
  for (auto& t : pool) t.join();
  for (unsigned d = 0; d < D; ++d)
    if (rcs[d]) {
      ssb::set_last_error(errs[d]);
      rethrow(rcs[d]);
    }

  RunResult r;
  r.strategy = name;
  r.shots = o.shots;
  r.seed = o.seed;
  r.workers = o.workers;
  // Shards on one device run one after another: peak = the largest shard's
  // peak per device, summed over the devices running concurrently.
  r.shard_devices.assign(shard_dev.begin(), shard_dev.end());
  std::vector<uint64_t> dev_peak(D, 0);
  for (uint64_t g = 0; g < G; ++g) {
    const ssb_stats& s = stats[g];
    r.dispatch_count += s.dispatch_count;
    dev_peak[shard_dev[g]] = std::max(dev_peak[shard_dev[g]], s.peak_states);
    r.branch.passes = std::max(r.branch.passes, s.passes);
    r.branch.leaf_shots.insert(r.branch.leaf_shots.end(), leaves[g].begin(), leaves[g].end());
  }
  for (uint64_t p : dev_peak) r.peak_states += p;
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
  PooledEngine& pe = pooled_engine(0);
  std::lock_guard<std::mutex> lk(pe.mu);
  if (!pe.engine)
    if (int rc = ssb_engine_create(0, &pe.engine)) rethrow(rc);
  if (int rc = f(pe.engine, prog)) rethrow(rc);
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
