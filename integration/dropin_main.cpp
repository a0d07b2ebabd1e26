// Drop-in proof (test infrastructure; built by oracle/Makefile `dropin` from
// the UNMODIFIED reference sources + integration/exec_gpu.cpp, linked against
// libshotsim_b200.so): the reference's own code drives the GPU executors.
//
//  1. bench   — shotsim::run_bench (bench.cpp:76-191), the reference harness,
//               with strategies {naive, batch, branch, gpu-batch, gpu-branch}:
//               it enforces equal counts checksums across every strategy and
//               worker count of each cell and exits 2 on the first mismatch.
//  2. equiv   — acceptance criterion 1 (tests/acceptance/acceptance_main.cpp
//               :79-118) restated over executor_by_name: for QFT(3..8) with
//               1% depolarizing Pauli / Kraus noise and seeds 1..5, the GPU
//               executors' counts (workers 1 / 4, budgets 1 / 4 / 64) must
//               equal run_naive's.
//
// Prints one line per part; exit code 0 when both pass.
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>

#include "shotsim/bench.hpp"
#include "shotsim/exec.hpp"

using namespace shotsim;

int main(int argc, char** argv) {
  const std::string csv = argc > 1 ? argv[1] : "/tmp/shotsim_dropin.csv";
  int rc = 0;
  for (const char* noise : {"pauli", "kraus"}) {
    BenchConfig c;
    c.qubits = {3, 5, 8, 10};
    c.shots = 2000;
    c.noise = noise;
    c.error_rates = {0.01, 0.05};
    c.strategies = {"naive", "batch", "branch", "gpu-batch", "gpu-branch"};
    c.workers = {1, 4};
    c.repeats = 1;
    c.out_path = csv;
    c.kernels = "scalar";
    std::ostringstream out, err;
    const int b = run_bench(c, out, err);
    std::printf("bench %s exit %d\n", noise, b);
    if (b != 0) std::cout << err.str();
    rc |= b;
  }
  uint64_t cells = 0, failures = 0;
  for (unsigned n = 3; n <= 8; ++n) {
    const Circuit circuit = measure_all(qft_circuit(n));
    for (bool as_kraus : {false, true}) {
      const NoisyCircuit program = instrument(circuit, make_depolarizing_model(0.01, as_kraus));
      for (uint64_t seed = 1; seed <= 5; ++seed) {
        RunOptions base;
        base.shots = 1000;
        base.seed = seed;
        const Counts want = executor_by_name("naive")(program, base).counts;
        auto check = [&](const RunResult& r) {
          ++cells;
          if (r.counts != want) ++failures;
        };
        for (unsigned workers : {1u, 4u}) {
          RunOptions o = base;
          o.workers = workers;
          check(executor_by_name("gpu-batch")(program, o));
          for (uint64_t budget : {1ull, 4ull, 64ull}) {
            o.branch_budget = budget;
            check(executor_by_name("gpu-branch")(program, o));
          }
        }
      }
    }
  }
  std::printf("equiv %llu gpu executor runs compared with run_naive, %llu mismatches\n",
              static_cast<unsigned long long>(cells), static_cast<unsigned long long>(failures));
  return (rc || failures) ? 1 : 0;
}
