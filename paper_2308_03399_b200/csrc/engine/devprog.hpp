// Device program: the instrumented NoisyCircuit (program.hpp:18-70) lowered to
// flat, 64-byte op records plus pooled matrices / Pauli terms / Kraus channels,
// and the HBM pass plan used by the streamed executor. Built once per program
// on the host (build_device_program), uploaded once per device.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "devtypes.h"
#include "shotsim_b200.hpp"

namespace ssb {

struct HostDevProgram {
  uint32_t n = 0, num_clbits = 0;
  uint64_t num_events = 0;
  bool eligible = false, has_measure = false;
  uint32_t end = 0;                      // ops executed before terminal sampling
  uint32_t num_pauli_sites = 0;
  uint32_t max_kraus = 0;                // largest channel size
  bool has_kraus = false, has_measure_ops = false;
  std::vector<DevOp> ops;
  std::vector<DevTerm> terms;
  std::vector<DevChannel> channels;
  std::vector<double> mats;              // 32 doubles per slot
  std::vector<uint64_t> scaled_cls;      // per matrix slot: classes after 1/sqrt(p)
  std::vector<uint8_t> sample_qubits, write_clbit, write_pos;
  bool sample_identity = false;          // sample_qubits == [0..n)
  // Streamed-mode plan (n > resident limit).
  std::vector<PassDesc> passes;
  std::vector<Item> items;
  std::vector<PassOp> pass_ops;
  std::vector<Uop> uops;
  std::vector<double> uop_mats;          // 2 doubles per double2
  std::vector<Step> steps;
  unsigned tile_k = 0;
  // Distinct segment shapes of the streamed plan (keys; ids = positions).
  std::vector<std::string> shapes;
};

uint64_t classify_matrix(const double* m, unsigned k, bool scaled);
HostDevProgram build_device_program(const shotsim::NoisyCircuit& p);
// Streamed plan: HBM tile passes (gates / Pauli sites) + special steps.
// fuse_kraus: Kraus applies run inside the next pass (S_KRAUS_DECIDE steps).
void plan_passes(HostDevProgram& d, unsigned tile_k, bool fuse_kraus = true);
// Resident plan: one pass (k = n) whose items cover the whole program.
void plan_resident(HostDevProgram& d);
// CUDA source of straight-line executors for the plan's segment shapes
// (specialise.cu compiles it at run time; see shapes.cuh).
std::string shape_source(const HostDevProgram& d);

}  // namespace ssb
