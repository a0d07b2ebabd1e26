// Fused-matrix plan (ssb_run_options::fused_matrices) — SURVEY §8(f) rank 2:
// "pre-multiply gates and sampled Paulis, with a guard band".
//
// The op stream [0, end) of a program made only of unconditioned gates and
// Pauli sites (program.hpp:18-40; C2 / C5 shape) is cut into blocks: maximal
// runs of ops on at most two qubits (the transpiled SU(4) blocks of a quantum
// volume layer, 8 U + 3 CX + 11 Pauli sites each, become one block). Moving
// an op across blocks on disjoint qubits is exact in real arithmetic, so the
// block's product M = G_k ... G_1 (computed here in long double) replaces the
// sequence. A Pauli site j inside a block is folded as
// Q_{j,t} = V_j P_t V_j^dagger (V_j: the block's gates after site j): a shot
// with non-identity draws (j1 < ... < jL) applies Q_{jL} ... Q_{j1} M.
//
// Amplitudes then differ from the reference's by rounding only; err_bound is
// a rigorous-with-margin bound on the 2-norm of that difference, from which
// the terminal sampler derives its guard band (engine.cu): a shot whose draw
// lies closer than the bound to a cumulative boundary is re-run exactly.
#pragma once

#include <string>
#include <vector>

#include "devprog.hpp"

namespace ssb {

struct FusedPlan {
  bool ok = false;
  std::string why;                 // reason when !ok (the exact path runs)
  unsigned k = 0;
  unsigned gq = 4;                 // register-group qubits (3 or 4)
  std::vector<FPass> passes;
  std::vector<FGroup> groups;
  std::vector<FBlock> blocks;
  std::vector<FSite> sites;
  std::vector<uint32_t> qidx;      // per (site, term): matrix index or kNoQ
  std::vector<double> mats;        // 32 doubles (16 complex, row-major 4x4) per matrix
  uint32_t num_blocks = 0;         // blocks per shot
  uint32_t max_pass_blocks = 0;    // staging sizes
  uint32_t max_pass_sites = 0;
  double err_bound = 0.0;          // bound on ||psi_fused - psi_reference||_2 (norm-1 states)
};

// Shared-memory block staging limit per pass (base matrices + entry list).
constexpr uint32_t kFusedMaxPassBlocks = 24;
// Default register-group size of the FMA build (A/B: SHOTSIM_B200_FUSED_GROUP).
constexpr unsigned kFusedGroupDefault = 4;

// gq: qubits per register group (4: 16-amplitude hexads, the tensor-core
// layout needs 4; 3: 8-amplitude octads, half the registers per thread).
FusedPlan plan_fused(const HostDevProgram& h, unsigned tile_k, unsigned gq = 4);
// plan_fused through a process-wide cache keyed by the program's content.
FusedPlan plan_fused_cached(const HostDevProgram& h, unsigned tile_k, unsigned gq = 4);

}  // namespace ssb
