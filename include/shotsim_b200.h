/*
 * shotsim_b200 — C ABI of the B200-native multi-shot statevector engine.
 *
 * This is the drop-in boundary for the reference's executor plugin API:
 *
 *   using ExecutorFn = RunResult (*)(const NoisyCircuit&, const RunOptions&);
 *   ExecutorFn executor_by_name(std::string_view);
 *       (reference: proj/include/shotsim/exec.hpp:32-35, registry
 *        proj/src/exec_naive.cpp:22-27)
 *
 * A NoisyCircuit (proj/include/shotsim/program.hpp:18-70) crosses this ABI
 * either as the reference's own lossless text/JSON inputs
 * (ssb_program_from_text: circuit_io.cpp:53-146 + noise.cpp:328-365 +
 * instrument, program.cpp:17-122) or already instrumented and flattened
 * (ssb_program_from_flat). Runs return one classical-register value per shot
 * for the contiguous shot-id range [shot_begin, shot_begin + shot_count),
 * exactly RunResult::shot_values (result.hpp:45-47) restricted to that range,
 * so shards and sub-samples compose by concatenation.
 *
 * Conventions: plain pointers and sizes only; every function returns
 * SSB_OK (0) or a nonzero ssb_status; ssb_last_error() (thread-local) holds
 * the message. Status codes mirror the reference's exception types
 * (common.hpp:18-34; std::invalid_argument for bad arguments).
 * All device work is sm_100a CUDA; there is no CPU execution path — without a
 * usable CUDA device every run entry point fails with SSB_ERR_CUDA.
 */
#ifndef SHOTSIM_B200_H_
#define SHOTSIM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SSB_API __attribute__((visibility("default")))
#else
#define SSB_API
#endif

#define SSB_ABI_VERSION 2

typedef enum ssb_status {
  SSB_OK = 0,
  SSB_ERR_RUNTIME = 1,          /* std::runtime_error (e.g. norm drift)        */
  SSB_ERR_INVALID_ARGUMENT = 2, /* std::invalid_argument                       */
  SSB_ERR_CONFIG = 3,           /* shotsim::ConfigError                        */
  SSB_ERR_CAPACITY = 4,         /* shotsim::CapacityError                      */
  SSB_ERR_DEGENERATE = 5,       /* shotsim::DegenerateDistribution             */
  SSB_ERR_CUDA = 6              /* no device / CUDA failure (no CPU fallback)  */
} ssb_status;

/* ProgramOp::Kind (program.hpp:19) */
typedef enum ssb_op_kind {
  SSB_OP_GATE = 0,
  SSB_OP_PAULI = 1,
  SSB_OP_KRAUS = 2,
  SSB_OP_MEASURE = 3,
  SSB_OP_RESET = 4,
  SSB_OP_BARRIER = 5
} ssb_op_kind;

#define SSB_MAX_OP_QUBITS 4

/* One ProgramOp, flattened. Matrices live in ssb_flat_program.matrices as
 * row-major 2^k x 2^k complex (re, im) doubles; qubits[0] is the low matrix
 * axis (statevector.hpp:40). */
typedef struct ssb_flat_op {
  uint32_t kind;          /* ssb_op_kind                                   */
  uint32_t num_qubits;    /* operand count                                 */
  uint32_t qubits[SSB_MAX_OP_QUBITS];
  uint32_t clbits[SSB_MAX_OP_QUBITS]; /* MEASURE only                      */
  uint32_t has_condition;
  uint32_t gate_kind;     /* GateKind (circuit.hpp:17-19) for GATE         */
  uint64_t cond_mask;     /* Condition::clbit_mask (circuit.hpp:33-39)     */
  uint64_t cond_value;
  uint64_t event;         /* randomness-site index (PAULI/KRAUS/MEAS/RESET)*/
  uint32_t matrix;        /* GATE: matrix index                            */
  uint32_t channel;       /* KRAUS: channel index                          */
  uint32_t term_begin;    /* PAULI: first term in ssb_flat_program.terms   */
  uint32_t term_count;
} ssb_flat_op;

/* PauliSite term: ProgramOp::term_cum/term_masks/term_identity
 * (program.hpp:34-37), PauliMasks (kernels.hpp:15-22). */
typedef struct ssb_flat_term {
  double cumulative;
  uint64_t x_mask;
  uint64_t z_mask;
  uint32_t num_y;
  uint32_t x_max;
  uint32_t identity;
  uint32_t reserved;
} ssb_flat_term;

/* KrausError (noise.hpp:54-57): num_matrices consecutive matrices. */
typedef struct ssb_flat_channel {
  uint32_t arity;
  uint32_t num_matrices;
  uint32_t matrix_begin;
  uint32_t reserved;
} ssb_flat_channel;

typedef struct ssb_flat_program {
  uint32_t num_qubits;
  uint32_t num_clbits;
  uint64_t num_events;
  uint32_t has_measure;
  uint32_t sampling_eligible;
  uint64_t terminal_measure_begin;
  uint64_t num_ops;
  const ssb_flat_op* ops;
  uint64_t num_terms;
  const ssb_flat_term* terms;
  uint64_t num_channels;
  const ssb_flat_channel* channels;
  uint64_t num_matrices;
  const double* matrices;           /* num_matrices * 32 doubles (4x4 slot) */
  uint32_t num_sample_qubits;
  const uint32_t* sample_qubits;
  uint32_t num_sample_writes;
  const uint32_t* sample_write_clbit; /* sample_writes[i].first  */
  const uint32_t* sample_write_pos;   /* sample_writes[i].second */
} ssb_flat_program;

#define SSB_MATRIX_STRIDE 32 /* doubles per matrix slot (4x4 complex) */

typedef struct ssb_program ssb_program;
typedef struct ssb_engine ssb_engine;
typedef struct ssb_batch ssb_batch;

/* RunOptions (exec.hpp:12-22) minus the CPU-only knobs. */
typedef struct ssb_run_options {
  uint64_t max_batch_size;   /* 0: derive from mem_limit_bytes                 */
  uint64_t branch_budget;    /* gpu-branch: max live states (>= 1)             */
  uint64_t mem_limit_bytes;  /* 0: SHOTSIM_MEM_LIMIT_BYTES or 80% of free HBM  */
  uint32_t check_norms;      /* gpu-batch: |norm^2 - 1| <= 1e-10 after every op
                                (exec_batch.cpp:217-224), else SSB_ERR_RUNTIME;
                                runs the op-at-a-time kernels (debug/tests) */
  uint32_t collect_leaf_stats; /* gpu-branch: shots per leaf into leaf_shots */
  uint32_t resident_max_qubits; /* n <= this: whole program SM-resident (0: 13) */
  uint32_t tile_qubits;      /* streamed mode: local qubits per HBM tile (0: 12) */
  uint32_t profile;          /* 1: per-kernel-class CUDA-event times in stats   */
  uint32_t interpret_only;   /* 1: never use the shape-specialised tile kernel  */
  /* ---- ABI 2 ---- */
  uint32_t fused_matrices;   /* gpu-batch, streamed sizes: 1 = multiply each
                                run of gates + Pauli sites on <= 2 qubits into
                                one 4x4 per shot (FMA arithmetic; amplitudes
                                within 1e-10 of the reference) and guard every
                                amplitude-dependent decision: a shot whose draw
                                lies within the rounding bound of a boundary is
                                replayed exactly on the device, so counts stay
                                bit-exact. Programs the fused planner does not
                                cover run exactly (stats->fused_blocks = 0). */
  uint32_t reserved0;
  uint64_t* leaf_shots;      /* collect_leaf_stats: HOST array receiving
                                BranchStats::leaf_shots (exec_branch.cpp:280),
                                leaf order of the reference; NULL: count only */
  uint64_t leaf_shots_capacity;
  double* states_out;        /* DEBUG (parity tests): HOST array of
                                shot_count * 2^n complex (re, im) doubles that
                                receives, per shot, the state terminal sampling
                                reads (or the final state when the program is
                                not sampling-eligible) — BatchState::segment
                                (exec_batch.hpp:31-32) of every executor path */
} ssb_run_options;

typedef struct ssb_stats {
  uint64_t dispatch_count;   /* kernel launches issued by the run             */
  uint64_t peak_states;      /* concurrently live segments / branch states    */
  uint64_t passes;           /* branch: passes; batch: shot waves             */
  uint64_t fused_passes;     /* batch: HBM tile passes per wave               */
  double device_seconds;     /* CUDA-event time of the device work            */
  double wall_seconds;
  /* profile=1 only: CUDA-event time per kernel class on the engine stream   */
  double pass_seconds;       /* fused gate/Pauli passes (tile or resident)    */
  uint64_t pass_launches;
  double special_seconds;    /* Kraus / measure / reset op-at-a-time kernels  */
  double sample_seconds;     /* terminal sampling                             */
  uint64_t specialised_shapes; /* streamed: segment shapes run straight-line
                                  (run-time specialised kernel); 0: interpreter;
                                  fused_matrices: passes run by their
                                  specialised kernel (SHOTSIM_B200_FUSED_JIT) */
  uint64_t sampling_serial_chunks; /* terminal-sampling chunks replayed with the
                                      reference's sequential adds (binade
                                      changes, ties, the deciding chunk) */
  uint64_t trunk_skipped;    /* streamed: (shot, pass) pairs not run because
                                the shot's noise draws had not yet diverged
                                from the shared noiseless trunk */
  /* ---- ABI 2 ---- */
  uint64_t num_leaves;       /* gpu-branch: leaves over all passes */
  uint64_t fused_blocks;     /* fused_matrices: 4x4 blocks per shot (0: exact) */
  uint64_t guard_flagged;    /* fused_matrices: shots replayed exactly because
                                a decision fell inside the guard band */
  double guard_delta;        /* fused_matrices: largest guard half-width used */
} ssb_stats;

SSB_API const char* ssb_last_error(void);
SSB_API int ssb_abi_version(void);

/* ---- program lowering (host) ------------------------------------------ */
/* circuit_text: reference circuit text (circuit_io.hpp:13-27) or JSON
 * (leading '{'); noise_json: NoiseModel JSON (noise.cpp:328-365), "" for no
 * noise, or {"model":"depolarizing","rate":r,"as_kraus":b}
 * (make_depolarizing_model, noise.cpp:375-392). Runs instrument(). */
SSB_API int ssb_program_from_text(const char* circuit_text, const char* noise_json,
                                  ssb_program** out);
SSB_API int ssb_program_from_flat(const ssb_flat_program* flat, ssb_program** out);
SSB_API void ssb_program_destroy(ssb_program* program);
/* Borrowed view, valid while the program lives. */
SSB_API int ssb_program_flat(const ssb_program* program, ssb_flat_program* out);
/* Exact text dump (doubles as %a) in the format of oracle/ref_shim.cpp. */
SSB_API int ssb_program_dump(const ssb_program* program, char* buf, size_t cap, size_t* len);
/* Writes counts_checksum (result.cpp:23-38) of the histogram of `values`. */
SSB_API int ssb_counts_checksum(const uint64_t* values, uint64_t count, uint32_t num_clbits,
                                uint32_t has_measure, uint64_t* checksum_out,
                                uint64_t* num_keys_out);

/* ---- engine (device) -------------------------------------------------- */
/* Number of CUDA devices visible to the process (0 without a driver). */
SSB_API int ssb_device_count(int* count);
SSB_API int ssb_engine_create(int device, ssb_engine** out);
SSB_API void ssb_engine_destroy(ssb_engine* engine);
/* Opaque cudaStream_t the engine launches on (for CUDA-event timing). */
SSB_API void* ssb_engine_stream(ssb_engine* engine);

/* gpu-batch (paper SIV.A; exec_batch.cpp:229-287): per-shot values for ids
 * [shot_begin, shot_begin+shot_count) into HOST memory values_out. */
SSB_API int ssb_run_batch(ssb_engine* engine, const ssb_program* program, uint64_t shot_begin,
                          uint64_t shot_count, uint64_t seed, const ssb_run_options* options,
                          uint64_t* values_out, ssb_stats* stats);
/* Same, values_out_device is a DEVICE pointer; no host sync at the end. */
SSB_API int ssb_run_batch_device(ssb_engine* engine, const ssb_program* program,
                                 uint64_t shot_begin, uint64_t shot_count, uint64_t seed,
                                 const ssb_run_options* options, uint64_t* values_out_device,
                                 ssb_stats* stats);
/* gpu-branch (paper SIV.B; exec_branch.cpp:175-295). */
SSB_API int ssb_run_branch(ssb_engine* engine, const ssb_program* program, uint64_t shot_begin,
                           uint64_t shot_count, uint64_t seed, const ssb_run_options* options,
                           uint64_t* values_out, ssb_stats* stats);

/* Dense histogram of device values (num_clbits <= 24) into a device array of
 * 2^num_clbits uint64 (accumulating) — the payload of the multi-GPU gather. */
SSB_API int ssb_histogram_device(ssb_engine* engine, const uint64_t* values_device,
                                 uint64_t count, uint32_t num_clbits, uint64_t* hist_device);

/* Plans `program` for the HBM-streamed executor with `tile_qubits` local
 * qubits (0: default) and compiles its shape-specialised tile kernel with
 * NVRTC for sm_100a without loading it (no GPU needed). *shapes receives the
 * number of distinct segment shapes; on failure the NVRTC log is in
 * ssb_last_error(). */
SSB_API int ssb_program_specialise_check(const ssb_program* program, uint32_t tile_qubits, uint32_t* shapes);

/* Plans `program` in fused-matrix mode (ssb_run_options::fused_matrices,
 * 11-qubit tiles, its default) and compiles its per-pass specialised fused kernels with
 * NVRTC for sm_100a without loading them (no GPU needed). *kernels receives
 * the number of specialised passes; on failure the NVRTC log is in
 * ssb_last_error(). */
SSB_API int ssb_program_fused_specialise_check(const ssb_program* program, uint32_t* kernels);

/* Diagnostics: the HBM tile pass (0-based, in execution order) each op of the
 * program runs in under the streamed plan for `tile_qubits` (0: default);
 * 0xFFFFFFFF for ops executed outside a pass (measure, reset, Kraus decide,
 * skipped identities). pass_of_op may be NULL to only get *num_passes. */
SSB_API int ssb_program_pass_map(const ssb_program* program, uint32_t tile_qubits, uint32_t* pass_of_op,
                                 uint64_t cap, uint32_t* num_passes);

/* Diagnostics of the fused-matrix plan (ssb_run_options::fused_matrices) for
 * `tile_qubits` local qubits (0: default); host only. ok = 0: the program is
 * outside the fused planner's scope and runs exactly (reason in
 * ssb_last_error() is NOT set; the run is simply exact). */
typedef struct ssb_fused_info {
  uint32_t ok;
  uint32_t passes;           /* HBM tile passes per shot                     */
  uint32_t blocks;           /* fused 4x4 blocks per shot                    */
  uint32_t groups;           /* register groups (<= 4 qubits) over all passes */
  uint32_t max_pass_blocks;
  uint32_t reserved;
  double err_bound;          /* bound on ||psi_fused - psi_reference||_2      */
} ssb_fused_info;
SSB_API int ssb_program_fused_info(const ssb_program* program, uint32_t tile_qubits, ssb_fused_info* out);

/* FP64-pipe roofline probe: the sustained rate of rounded DMUL/DADD (no FMA,
 * the engine's arithmetic) over the whole device, in FP64 ops per second,
 * measured with CUDA events (the denominator of bench.py's fp64 roofline). */
SSB_API int ssb_fp64_peak(ssb_engine* engine, double* ops_per_second);

/* ---- exact density-matrix reference (density.hpp:12-68, n <= 10) ---- */
/* exact_creg_distribution (density.cpp:291-306): the exact distribution of
 * final classical-register values, evolved on the device. Entries are in
 * ascending key order. keys/probs NULL: only *count is set (size query);
 * otherwise capacity must be >= the entry count (SSB_ERR_CAPACITY if not).
 * Errors as the reference: n outside 1..10 or > 2 intermediate measure sites
 * -> SSB_ERR_CAPACITY; a conditional intermediate measure -> INVALID_ARGUMENT. */
SSB_API int ssb_exact_creg_distribution(ssb_engine* engine, const ssb_program* program, uint64_t* keys,
                                        double* probs, uint64_t capacity, uint64_t* count);
/* exact_distribution (density.cpp:280-289): outcome distribution over the
 * listed qubits (qubits[0] = bit 0); out holds 2^num_qubits doubles. */
SSB_API int ssb_exact_distribution(ssb_engine* engine, const ssb_program* program, const uint32_t* qubits,
                                   uint32_t num_qubits, double* out);
/* tvd_vs_exact (density.cpp:308-315) against the Counts that
 * counts_from_values(values, num_clbits, has_measure) builds (result.cpp:40-48)
 * from the executors' per-shot register values. Host arithmetic. */
SSB_API int ssb_tvd_vs_exact(const uint64_t* values, uint64_t shots, uint32_t num_clbits, uint32_t has_measure,
                             const uint64_t* keys, const double* probs, uint64_t count, double* tvd);

/* ---- operator-level entry points (BatchState, exec_batch.hpp:22-84) ---- */
/* A device-resident batch over arbitrary shot ids, initialised to |0...0>. */
SSB_API int ssb_batch_create(ssb_engine* engine, const ssb_program* program,
                             const uint64_t* shot_ids, uint64_t count, uint64_t seed,
                             ssb_batch** out);
SSB_API void ssb_batch_destroy(ssb_batch* batch);
/* Apply program op `op_index` to every shot. u: per-shot draws replacing the
 * keyed stream (the *_with test hooks, exec_batch.hpp:57-62), or NULL. */
SSB_API int ssb_batch_apply_op(ssb_batch* batch, uint64_t op_index, const double* u);
/* BatchState::run (exec_batch.cpp:200-227) incl. terminal sampling. */
SSB_API int ssb_batch_run(ssb_batch* batch);
/* amps: count * 2^n complex (re,im) doubles; either output may be NULL. */
SSB_API int ssb_batch_read(ssb_batch* batch, double* amps, uint64_t* cregs);
SSB_API int ssb_batch_write_segment(ssb_batch* batch, uint64_t s, const double* amps);
SSB_API uint64_t ssb_batch_dispatches(const ssb_batch* batch);

#ifdef __cplusplus
}
#endif

#endif /* SHOTSIM_B200_H_ */
