// shotsim_b200: command-line drop-in for the reference CLI's `run` and
// `validate` subcommands (shotsim_main.cpp:38-67, 97-139) over the GPU
// executors. Same options, same stdout (one "<bitstring> <count>" line per
// key in map order, "(no measure)" for the empty key), same stderr summary
// line and exit codes (3 config / usage error, 1 capacity or other error).
// The reference's `bench` / `tvd` sweeps are out of scope:
// bench.py measures this engine.
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <iostream>
#include <string>

#include "shotsim_b200.hpp"

namespace {

using namespace shotsim;

int usage(const char* argv0) {
  std::cerr << "usage: " << argv0
            << " run --circuit FILE [--noise-model FILE] [--strategy gpu-batch|gpu-branch] [--shots N]\n"
               "          [--seed S] [--workers GPUS] [--budget B] [--max-batch-size N]\n"
            << "       " << argv0 << " validate --circuit FILE\n";
  return 3;
}

uint64_t to_u64(const std::string& opt, const std::string& v) {
  char* end = nullptr;
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (v.empty() || *end || v[0] == '-') throw ConfigError(opt + ": expected a non-negative integer, got '" + v + "'");
  return x;
}

int run_one(const std::string& circuit_path, const std::string& noise_path, const std::string& strategy,
            const RunOptions& options) {
  const Circuit circuit = load_circuit(circuit_path);
  require_valid(circuit);
  const NoiseModel model = noise_path.empty() ? NoiseModel{} : NoiseModel::load(noise_path);
  const NoisyCircuit program = instrument(circuit, model);
  const RunResult result = executor_by_name(strategy)(program, options);
  for (const auto& [key, n] : result.counts) std::cout << (key.empty() ? "(no measure)" : key) << " " << n << "\n";
  std::cerr << "strategy=" << strategy << " shots=" << options.shots << " seed=" << options.seed
            << " seconds=" << result.wall_seconds;
  if (strategy == "gpu-batch") std::cerr << " dispatches=" << result.dispatch_count;
  if (strategy == "gpu-branch")
    std::cerr << " peak_states=" << result.branch.peak_states << " passes=" << result.branch.passes;
  std::cerr << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage(argv[0]);
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage(argv[0]);
    return 0;
  }
  std::string circuit_path, noise_path, strategy = "gpu-batch";
  RunOptions options;
  options.shots = 1000;
  options.seed = 1;
  try {
    if (cmd != "run" && cmd != "validate") return usage(argv[0]);
    for (int i = 2; i < argc; ++i) {
      const std::string opt = argv[i];
      if (i + 1 >= argc) throw ConfigError(opt + ": missing value");
      const std::string v = argv[++i];
      if (opt == "--circuit") circuit_path = v;
      else if (cmd == "validate") throw ConfigError("validate: unknown option " + opt);
      else if (opt == "--noise-model") noise_path = v;
      else if (opt == "--strategy") strategy = v;
      else if (opt == "--shots") options.shots = to_u64(opt, v);
      else if (opt == "--seed") options.seed = to_u64(opt, v);
      else if (opt == "--workers") options.workers = static_cast<unsigned>(to_u64(opt, v));
      else if (opt == "--budget") options.branch_budget = to_u64(opt, v);
      else if (opt == "--max-batch-size") options.max_batch_size = to_u64(opt, v);
      else throw ConfigError("run: unknown option " + opt);
    }
    if (circuit_path.empty()) throw ConfigError("--circuit is required");
    if (cmd == "validate") {
      const auto violations = validate(load_circuit(circuit_path));
      if (violations.empty()) {
        std::cout << "ok\n";
        return 0;
      }
      for (const auto& v : violations) std::cout << "instruction " << v.instruction << ": " << v.message << "\n";
      return 1;
    }
    return run_one(circuit_path, noise_path, strategy, options);
  } catch (const ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 3;
  } catch (const CapacityError& e) {
    std::cerr << "capacity error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
