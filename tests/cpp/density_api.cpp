// C++ drop-in check of the statistical checker (density.hpp:56-68 API shape):
// exact_creg_distribution / exact_distribution on the device and
// tvd_vs_exact over an executor's Counts, exactly as the reference's
// density tests call them (test_density.cpp:178-192). Built and run by
// tests/test_density.py (GPU); prints "key prob" lines (%a) then "tvd <x>".
#include <cstdio>
#include <string>
#include <vector>

#include "shotsim_b200.hpp"

int main(int argc, char** argv) {
  using namespace shotsim;
  if (argc < 3) return 2;
  const NoisyCircuit program = instrument(load_circuit(argv[1]), NoiseModel::load(argv[2]));
  const auto exact = exact_creg_distribution(program);
  for (const auto& [k, p] : exact) std::printf("%llu %a\n", static_cast<unsigned long long>(k), p);
  const std::vector<unsigned> q0{0};
  const std::vector<double> m = exact_distribution(program, q0);
  std::printf("marginal0 %a %a\n", m[0], m[1]);
  RunOptions options;
  options.shots = 50000;
  options.seed = 12;
  const RunResult r = executor_by_name("gpu-batch")(program, options);
  std::printf("tvd %.17g\n", tvd_vs_exact(r.counts, options.shots, exact));
  try {
    NoisyCircuit big = program;
    big.num_qubits = 11;
    exact_creg_distribution(big);
    std::printf("no capacity error\n");
  } catch (const CapacityError&) {
    std::printf("capacity error\n");
  }
  return 0;
}
