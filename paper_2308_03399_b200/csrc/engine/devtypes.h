// Device-side program types (shared by the static kernels and the run-time
// specialised kernels, so this header has no host-library dependencies).
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
#else
#include <cstdint>
#endif

namespace ssb {

enum OpKind : uint8_t { K_GATE = 0, K_PAULI = 1, K_KRAUS = 2, K_MEASURE = 3, K_RESET = 4, K_BARRIER = 5 };

struct alignas(16) DevOp {
  uint8_t kind;
  uint8_t nq;
  uint8_t has_cond;
  uint8_t skip;        // gate whose matrix is the identity: exact no-op
  uint8_t q[4];        // qubit operands (qubits[0] = low matrix axis)
  uint8_t c[4];        // clbits (MEASURE)
  uint32_t aux;        // GATE: matrix slot; PAULI: first term; KRAUS: channel
  uint32_t count;      // PAULI: term count; KRAUS: matrix count
  uint32_t site;       // PAULI: ordinal among Pauli sites (decision table column)
  uint8_t mk;          // GATE: micro-kind (MicroKind), chosen at plan time
  uint8_t src;         // MK_2Q_MONO: source column of each row (2 bits per row)
  uint8_t pad[2];
  uint64_t cls;        // GATE: entry classes (exact.cuh EntryClass, 3 bits each)
  uint64_t cond_mask;
  uint64_t cond_value;
  uint64_t event;
};
static_assert(sizeof(DevOp) == 64, "DevOp layout");

struct alignas(8) DevTerm {
  double cum;
  uint32_t x, z;       // qubit masks (n <= 30)
  uint32_t num_y;
  uint32_t identity;
};

struct DevChannel {
  uint32_t arity, nmat, mat_begin, pad;
};

// Gate micro-kinds (exact.cuh): which arithmetic template applies the matrix.
enum MicroKind : uint8_t {
  MK_1Q_U = 0,     // classes (REAL, GEN, GEN, GEN): the U gate
  MK_1Q_REAL = 1,  // all four entries real or zero-free real (H)
  MK_1Q_GEN = 2,   // anything else: per-entry runtime classes
  MK_2Q_MONO = 3,  // one nonzero per row (CX, SWAP, CP, CZ...): moves + few products
  MK_2Q_GEN = 4,   // dense 4x4: per-entry runtime classes
};

// One fused HBM tile pass over the local qubit set `lmask` (|lmask| = k):
// items [item_begin, item_end); `first` synthesises |0...0> instead of loading
// the tile. The resident executor uses one pass with k = n whose items also
// include special ops (Kraus / measure / reset).
struct PassDesc {
  uint32_t item_begin, item_end;
  uint32_t lmask;
  uint8_t k;
  uint8_t first;
  uint8_t pad[2];
  uint8_t lq[32];      // local position j -> qubit
  // Streamed passes: micro-op stream [uop_begin, uop_end) (items index it
  // relative to uop_begin) and its matrix table [mat_begin, mat_begin+mat_count)
  // (double2 units), staged into shared memory by the tile kernel.
  uint32_t uop_begin, uop_end;
  uint32_t mat_begin, mat_count;
  uint32_t po_begin;   // first pass_op of this pass (per-op fallback, k < 2)
  uint32_t kraus_mat;  // matrix-table slot (16 double2) of the per-shot Kraus
                       // matrix when the pass starts with a Kraus apply
  // Epilogue: the next Kraus site's matrix-0 partial sums, computed from the
  // finished tile before it is stored (saves that site's separate state read).
  // epi_kind 1: 1q site, partials = the 512-pair block sums of
  // expval_matrix1_scalar (kernels_scalar.cpp:103-126); 2: 2q site, partials
  // = the 8-group leaves of expval_generic's pairwise tree
  // (statevector.cpp:56-80). epi_t: local positions of the target(s) (matrix
  // bit 0 / 1); epi_low: local positions of the pair / group index bits inside
  // one partial (the lowest non-target qubits, in order); epi_hi: the other
  // local positions (which partial of the tile), in order.
  uint8_t epi_kind;
  uint8_t epi_nlow, epi_nhi;
  uint8_t epi_t[2];
  uint8_t epi_low[9];
  uint8_t epi_hi[12];
  uint32_t epi_op;     // the Kraus site (op index)
};

// Micro-op codes of a streamed pass (one per gate / Pauli site).
// Within a segment, unconditional 2q permutations (CX, SWAP) are folded into a
// plan-time relabeling sigma of the quad's 4 registers (logical element e
// lives in register sigma(e)); later micro-ops address physical registers and
// the segment store writes register sigma(e) to element e's address. sigma
// is packed 2 bits per element; 0xE4 is the identity.
enum UopCode : uint8_t {
  UC_U = 0,        // 1q U pattern          (qb: physical pairs a0|a1<<2|b0<<4|b1<<6)
  UC_REAL = 1,     // 1q all-real           (qb: physical pairs)
  UC_GEN1 = 2,     // 1q runtime classes    (qb: physical pairs; cls via ref)
  UC_MONO = 3,     // 2q monomial           (qb: swapped; src; mcls)
  UC_GEN2 = 4,     // 2q runtime classes    (qb: swapped; cls via ref)
  UC_PAULI = 5,    // Pauli site            (qb: quad bits of op qubits, bit b)
  UC_SWAP = 6,     // conditional 2q transposition (qb: physical e0 | e1 << 2)
  UC_PHASE = 7,    // 2q diagonal with one non-unit entry (qb: element; mcls:
                   // its class) — CP
  UC_KRAUS1 = 8,   // apply of a 1q Kraus site's per-shot choice M_sel/sqrt(p)
                   // (qb: physical pairs, src: logical bit; matrix + classes
                   // staged per shot from the decide step)
  UC_KRAUS2 = 9,   // 2q Kraus apply (qb: swapped)
};

// 16-byte micro-op. After per-shot compaction (identity Pauli draws and
// failed conditions removed) `pauli` holds xq | zq << 2 | (num_y & 3) << 4.
struct Uop {
  uint8_t code;
  uint8_t qb;
  uint8_t src;
  uint8_t flags;       // bit0: conditional
  uint16_t mat;        // offset into the pass matrix table (double2 units)
  uint16_t mcls;       // UC_MONO: class of row r's nonzero entry, 3 bits per row
  uint32_t ref;        // program op index
  uint8_t pauli;
  uint8_t sigma;       // UC_PAULI / UC_MONO / UC_GEN2: logical->physical quad map
  uint8_t pad[2];
};
static_assert(sizeof(Uop) == 16, "Uop layout");

// Item: a register segment — consecutive ops [begin,end) of pass_ops acting
// inside the 2-qubit set {la, lb} (local positions), applied per amplitude
// quad in registers — or a special op (resident executor only).
enum ItemKind : uint8_t { IT_SEGMENT = 0, IT_SPECIAL = 1 };
struct Item {
  uint8_t kind;
  uint8_t la, lb;      // local positions, la < lb
  uint8_t sigma;       // streamed passes: register map at the segment end
  uint32_t begin, end; // segment: pass_ops range; special: begin = op index
  // Streamed passes: the segment's "shape" — its micro-op sequence with every
  // Pauli draw identity and every condition true (the common case per shot) —
  // as an index into HostDevProgram::shapes (kNoShape: none), and the number
  // of non-Pauli micro-ops that case executes.
  uint16_t shape;
  uint16_t nfast;
};
constexpr uint16_t kNoShape = 0xFFFF;

struct PassOp {
  uint32_t op;         // index into ops
  uint8_t qb[4];       // quad bit (0 -> la, 1 -> lb) of each op qubit
};

// S_KRAUS_DECIDE: probabilities + per-shot choice of a Kraus site whose apply
// is the first micro-op of the next pass (streamed executor).
enum StepKind : uint8_t { S_PASS = 0, S_SPECIAL = 1, S_SAMPLE = 2, S_KRAUS_DECIDE = 3 };
struct Step {
  StepKind kind;
  uint32_t index;      // pass index, or op index for S_SPECIAL
};

// ---- Fused-matrix mode (ssb_run_options::fused_matrices; fused.cpp) -------
// Runs of gates + Pauli sites on at most two qubits are multiplied into one
// 4x4 "block" per shot; a shot that drew non-identity Pauli terms inside a
// block applies Q_L ... Q_1 M instead of M, with Q_j = V_j P_t V_j^dagger
// (V_j: the block's gates after site j), all precomputed on the host.
struct FPass {
  uint32_t grp_begin, grp_end;     // register groups of this pass (application order)
  uint32_t blk_begin, blk_end;     // their blocks (group order)
  uint32_t lmask;                  // local qubit set (k qubits, low 3 included)
  uint8_t k, first;                // first: synthesise |0...0> instead of loading
  uint8_t pad[2];
  uint8_t lq[32];                  // local position -> qubit
};

// A register group: consecutive blocks of a pass whose qubits lie in four
// local positions; each thread holds the group's 16 amplitudes of one "hexad"
// in registers while every block of the group is applied.
// Tensor-core layout (fused_pass_mma_kernel): within a team of 4 lanes, the
// lane index j holds two group bits ("lane bits") and the 16 registers the
// other two plus the team's 4 hexads. lane0/lane1: the group bits (0..3) in
// lane-bit 0 / 1, reg0/reg1 the register bits — at the group's load (init)
// and after its last block (fin, the store layout).
struct FGroup {
  uint8_t g[4];                    // local positions, ascending (group bit i <-> g[i])
  uint32_t blk_begin, blk_end;
  uint8_t init[4];                 // lane0, lane1, reg0, reg1 at load
  uint8_t fin[4];                  // ... at store
};

// xch: up to two lane/register bit exchanges before the block, each a
// nibble (valid << 3 | p << 1 | q: lane bit p <-> register bit q); perm: the
// lanes hold the block's matrix bits in swapped order (apply M with bit 0 and
// bit 1 of its row / column indices exchanged).
struct FBlock {
  uint8_t p0, p1;                  // local positions of matrix bit 0 / bit 1
  uint8_t gb0, gb1;                // their group bits
  uint32_t mat;                    // base matrix (16 double2, row-major 4x4)
  uint32_t site_begin, site_end;   // its Pauli sites (FSite range)
  uint8_t xch, perm, pad[2];
};

struct FSite {
  uint32_t site;                   // Pauli-site ordinal (decision table column)
  uint32_t qbase;                  // qidx[qbase + term]: Q matrix, or kNoQ (identity term)
};
constexpr uint32_t kNoQ = 0xFFFFFFFFu;
// Per-shot product slots in shared memory (noisy blocks beyond these apply
// their Q factors as extra 4x4 entries — same result, more work).
constexpr uint32_t kFusedSlots = 8;

}  // namespace ssb
