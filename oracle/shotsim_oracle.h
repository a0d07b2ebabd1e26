/*
 * TEST INFRASTRUCTURE ONLY — the CPU restatement oracle of the reference's
 * multi-shot statevector path. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never links it.
 *
 * Pinned against (a) the Random123 Philox KATs and the reference's uniform()
 * values (tests/golden/rng_kat.json), (b) the reference library compiled from
 * its own sources (oracle/_ref, per-shot register values on C1 and on the
 * cross-strategy random-program recipe), see tests/test_oracle.py.
 *
 * Input is the instrumented program in the C-ABI flat form (shotsim_b200.h).
 * Arithmetic follows the reference's SCALAR kernel table exactly
 * (kernels_scalar.cpp); compiled with -ffp-contract=off.
 */
#ifndef SHOTSIM_ORACLE_H_
#define SHOTSIM_ORACLE_H_

#include <stdint.h>

#include "../include/shotsim_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

void oracle_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double oracle_uniform(uint64_t seed, uint64_t shot, uint64_t event);

/* run_single_shot (exec_naive.cpp:88-129) for each id; amps_out (optional)
 * receives the final state of the LAST id (2^n complex). Returns 0 or an
 * ssb_status code. */
int oracle_run_shots(const ssb_flat_program* p, const uint64_t* ids, uint64_t count,
                     uint64_t seed, unsigned threads, uint64_t* values_out, double* amps_out);

/* Final amplitudes of every listed shot (count * 2^n complex) — the
 * BatchState::segment view after run() (exec_batch.cpp:200-227). */
int oracle_final_states(const ssb_flat_program* p, const uint64_t* ids, uint64_t count,
                        uint64_t seed, double* amps_out, uint64_t* cregs_out);

/* run_branch (exec_branch.cpp:175-295) over shot ids [0, shots): values,
 * peak_states and passes. */
int oracle_run_branch(const ssb_flat_program* p, uint64_t shots, uint64_t seed,
                      uint64_t budget, uint64_t* values_out, uint64_t* peak_states,
                      uint64_t* passes);

const char* oracle_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
