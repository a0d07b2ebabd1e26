// C++ drop-in check of the executor registry (exec.hpp:12-38 API shape):
// gpu-batch / gpu-branch through executor_by_name with RunOptions::workers in
// {1, 3, 8} on however many devices exist (shards pulled by free devices) must
// give identical shot_values (exec.hpp:24-27: results never depend on
// workers), and gpu-branch must report BranchStats::leaf_shots like
// run_branch (exec_branch.cpp:280): one entry per leaf, summing to the shots.
// Built and run by tests/test_executors.py (GPU). Prints one line per run:
//   <strategy> <workers> <checksum hex> <first 4 values> <leaves> <leaf sum>
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <numeric>

#include "shotsim_b200.hpp"

int main(int argc, char** argv) {
  using namespace shotsim;
  if (argc < 3) return 2;
  const NoisyCircuit program = instrument(load_circuit(argv[1]), NoiseModel::load(argv[2]));
  int mismatches = 0;
  for (const char* name : {"gpu-batch", "gpu-branch"}) {
    std::vector<uint64_t> first;
    for (unsigned workers : {1u, 3u, 8u}) {
      RunOptions o;
      o.shots = 2000;
      o.seed = 17;
      o.workers = workers;
      o.branch_budget = 16;
      o.record_shot_values = true;
      o.collect_leaf_stats = true;
      const RunResult r = executor_by_name(name)(program, o);
      if (first.empty()) first = r.shot_values;
      if (r.shot_values != first) ++mismatches;
      if (r.shard_devices.size() != std::min<uint64_t>(workers, o.shots)) ++mismatches;
      const uint64_t leaf_sum = std::accumulate(r.branch.leaf_shots.begin(), r.branch.leaf_shots.end(), uint64_t{0});
      std::printf("%s %u %016" PRIx64 " %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64 " %zu %" PRIu64 "\n", name,
                  workers, counts_checksum(r.counts), r.shot_values[0], r.shot_values[1], r.shot_values[2],
                  r.shot_values[3], r.branch.leaf_shots.size(), leaf_sum);
    }
  }
  std::printf("mismatches %d\n", mismatches);
  return mismatches ? 1 : 0;
}
