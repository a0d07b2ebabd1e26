// Exact density-matrix evolver on the device: the
// statistical reference the Monte Carlo executors are validated against, for
// small registers (n <= 10). Restates the reference's DensityMatrix and
// evolve_trajectories / exact_creg_distribution / exact_distribution
// (proj/src/density.cpp:40-315, proj/include/shotsim/density.hpp:12-68).
//
// Layout: rho is row-major d x d complex (re, im) doubles, d = 2^n, so the
// flat index is r*d + c (the reference's data_[r * dim() + c]). At n = 10 that
// is 16 MiB per trajectory, resident in HBM for the whole evolution.
//
// Kernels (all HBM-bound, each entry read and written once per op):
//  * dm_conj_sum — one thread per (row group, column group) block of
//    2^k x 2^k entries sharing every bit outside the target qubits:
//    blk <- sum_i K_i blk K_i^dagger in registers. Unitaries (one matrix,
//    no accumulate), Kraus channels and resets (|0><m| branches) all use it.
//    The arithmetic order is the reference's: T = K blk (row transform,
//    density.cpp:26-33 over columns), then T K^dagger (conj(K) over rows),
//    each dot product accumulated from (0, 0) in matrix-column order, and the
//    Kraus terms summed in matrix order from zero (density.cpp:100-109).
//  * dm_pauli — out[r,c] = sum_t p_t ph_t(r) conj(ph_t(c)) rho[r^x, c^x]
//    (density.cpp:186-215), out of place.
//  * dm_project — the intermediate-measurement projector / p (density.cpp:
//    249-262).
// Diagonal marginals read the d diagonal entries back (strided 2D copy) and
// sum them on the host in index order, as diagonal_marginal does
// (density.cpp:148-154), so outcome probabilities follow the same order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../capi_internal.hpp"

namespace ssb {

#define CKD(expr)                                                                          \
  do {                                                                                     \
    const cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess) throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

constexpr unsigned kInitialKraus = 16;  // matrix slots allocated up front (grown on demand)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

struct BlockArgs {
  unsigned n, k;
  unsigned q[2];       // target qubits, q[0] = low matrix axis
  unsigned sorted[2];  // ascending
  unsigned num_matrices;
  int accumulate;      // 1: Kraus sum from zero; 0: single conjugation
};

// expand_index (common.hpp:61-67): zeros at the sorted target positions.
__device__ __forceinline__ uint64_t expand2(uint64_t g, const BlockArgs& a) {
  for (unsigned i = 0; i < a.k; ++i) {
    const unsigned p = a.sorted[i];
    g = ((g >> p) << (p + 1)) | (g & ((1ull << p) - 1));
  }
  return g;
}

// mats: num_matrices x (side x side) row-major complex.
template <unsigned K>
__global__ void dm_conj_sum(double2* __restrict__ rho, const double2* __restrict__ mats, BlockArgs a) {
  constexpr unsigned S = 1u << K;
  const unsigned rest = a.n - K;
  const uint64_t blocks = 1ull << (2 * rest);
  const uint64_t d = 1ull << a.n;
  uint64_t off[S];
#pragma unroll
  for (unsigned l = 0; l < S; ++l) {
    uint64_t o = 0;
#pragma unroll
    for (unsigned b = 0; b < K; ++b)
      if ((l >> b) & 1) o |= 1ull << a.q[b];
    off[l] = o;
  }
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < blocks;
       b += (uint64_t)gridDim.x * blockDim.x) {
    // Column group in the low bits so neighbouring threads touch neighbouring
    // columns of the same rows (coalesced 16-byte loads).
    const uint64_t br = expand2(b >> rest, a), bc = expand2(b & ((1ull << rest) - 1), a);
    double2 blk[S][S], out[S][S];
#pragma unroll
    for (unsigned r = 0; r < S; ++r)
#pragma unroll
      for (unsigned c = 0; c < S; ++c) {
        blk[r][c] = rho[(br + off[r]) * d + bc + off[c]];
        out[r][c] = make_double2(0.0, 0.0);
      }
    for (unsigned m = 0; m < a.num_matrices; ++m) {
      const double2* M = mats + m * S * S;
      double2 t[S][S];
#pragma unroll
      for (unsigned c = 0; c < S; ++c)
#pragma unroll
        for (unsigned r = 0; r < S; ++r) {
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (unsigned j = 0; j < S; ++j) acc = cadd(acc, cmul(M[r * S + j], blk[j][c]));
          t[r][c] = acc;
        }
#pragma unroll
      for (unsigned r = 0; r < S; ++r)
#pragma unroll
        for (unsigned c = 0; c < S; ++c) {
          double2 acc = make_double2(0.0, 0.0);
#pragma unroll
          for (unsigned j = 0; j < S; ++j) {
            const double2 e = M[c * S + j];
            acc = cadd(acc, cmul(make_double2(e.x, -e.y), t[r][j]));
          }
          out[r][c] = a.accumulate ? cadd(out[r][c], acc) : acc;
        }
    }
#pragma unroll
    for (unsigned r = 0; r < S; ++r)
#pragma unroll
      for (unsigned c = 0; c < S; ++c) rho[(br + off[r]) * d + bc + off[c]] = out[r][c];
  }
}

struct PauliTermDev {
  double p;
  uint64_t x, z;
  uint32_t num_y;
};

struct PauliArgs {
  unsigned n, num_terms;
  const PauliTermDev* t;  // device table (any length: the reference has no cap)
};

__device__ __forceinline__ double2 pauli_phase(uint64_t idx, uint64_t z, uint32_t num_y) {
  double2 ph;
  switch (num_y & 3u) {
    case 0: ph = make_double2(1.0, 0.0); break;
    case 1: ph = make_double2(0.0, -1.0); break;
    case 2: ph = make_double2(-1.0, 0.0); break;
    default: ph = make_double2(0.0, 1.0); break;
  }
  return (__popcll(idx & z) & 1) ? make_double2(-ph.x, -ph.y) : ph;
}

__global__ void dm_pauli(const double2* __restrict__ rho, double2* __restrict__ out, PauliArgs a) {
  const uint64_t d = 1ull << a.n, total = d * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i >> a.n, c = i & (d - 1);
    double2 acc = make_double2(0.0, 0.0);
    for (unsigned t = 0; t < a.num_terms; ++t) {
      const PauliTermDev& T = a.t[t];
      const double2 pr = pauli_phase(r, T.z, T.num_y), pc = pauli_phase(c, T.z, T.num_y);
      // ((p * phase(r)) * conj(phase(c))) * rho[r^x, c^x]  (density.cpp:209-211)
      const double2 w = cmul(make_double2(T.p * pr.x, T.p * pr.y), make_double2(pc.x, -pc.y));
      acc = cadd(acc, cmul(w, rho[(r ^ T.x) * d + (c ^ T.x)]));
    }
    out[i] = acc;
  }
}

__global__ void dm_project(const double2* __restrict__ rho, double2* __restrict__ out, unsigned n, uint64_t qmask,
                           uint64_t offset, double p) {
  const uint64_t d = 1ull << n, total = d * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i >> n, c = i & (d - 1);
    double2 v = make_double2(0.0, 0.0);
    if ((r & qmask) == offset && (c & qmask) == offset) {
      const double2 x = rho[i];
      v = make_double2(x.x / p, x.y / p);  // std::complex / double (density.cpp:258)
    }
    out[i] = v;
  }
}

uint64_t gather_bits(uint64_t index, const uint32_t* pos, unsigned count) {
  uint64_t out = 0;
  for (unsigned b = 0; b < count; ++b)
    if ((index >> pos[b]) & 1) out |= 1ull << b;
  return out;
}

struct Traj {
  double2* rho = nullptr;
  uint64_t creg = 0;
  double weight = 1.0;
};

struct Evolver {
  const ssb_flat_program& F;
  cudaStream_t stream;
  uint64_t* launches;
  int num_sms;
  unsigned n;
  uint64_t d;
  std::vector<void*> allocs;
  double2* scratch = nullptr;
  double2* mats = nullptr;  // Kraus / unitary matrices of the current op
  size_t mats_cap = 0;      // in double2
  PauliTermDev* terms = nullptr;  // Pauli terms of the current site
  size_t terms_cap = 0;
  std::vector<PauliTermDev> host_terms;

  Evolver(const ssb_flat_program& f, cudaStream_t s, uint64_t* l, int sms)
      : F(f), stream(s), launches(l), num_sms(sms), n(f.num_qubits), d(1ull << f.num_qubits) {}
  ~Evolver() {
    cudaStreamSynchronize(stream);
    for (void* p : allocs) cudaFree(p);
  }

  double2* alloc_rho() {
    void* p = nullptr;
    CKD(cudaMalloc(&p, d * d * sizeof(double2)));
    allocs.push_back(p);
    return static_cast<double2*>(p);
  }

  unsigned grid(uint64_t work) const {
    const uint64_t want = (work + 255) / 256;
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(num_sms) * 16)));
  }

  void launched() {
    CKD(cudaGetLastError());
    if (launches) ++*launches;
  }

  // K_i as side x side complex, host-side.
  void conj_sum(double2* rho, const std::vector<double2>& m, unsigned k, const uint32_t* qubits, unsigned count,
                bool accumulate) {
    BlockArgs a{};
    a.n = n;
    a.k = k;
    a.num_matrices = count;
    a.accumulate = accumulate ? 1 : 0;
    for (unsigned i = 0; i < k; ++i) a.q[i] = a.sorted[i] = qubits[i];
    std::sort(a.sorted, a.sorted + k);
    const unsigned side = 1u << k;
    if (m.size() != size_t(count) * side * side) throw std::invalid_argument("density evolver: bad channel");
    if (m.size() > mats_cap) {  // channels of any length (the reference has no cap)
      void* p = nullptr;
      CKD(cudaMalloc(&p, m.size() * sizeof(double2)));
      allocs.push_back(p);  // the old slot table is freed with the rest
      mats = static_cast<double2*>(p);
      mats_cap = m.size();
    }
    CKD(cudaMemcpyAsync(mats, m.data(), m.size() * sizeof(double2), cudaMemcpyHostToDevice, stream));
    const uint64_t blocks = 1ull << (2 * (n - k));
    if (k == 1) dm_conj_sum<1><<<grid(blocks), 256, 0, stream>>>(rho, mats, a);
    else if (k == 2) dm_conj_sum<2><<<grid(blocks), 256, 0, stream>>>(rho, mats, a);
    else throw std::invalid_argument("density evolver supports 1- and 2-qubit operators");
    launched();
    // No sync: the pageable H2D copy has staged `m` when it returns, and the
    // next op's copy into `mats` is stream-ordered after this kernel.
  }

  std::vector<double2> matrix(uint32_t index, unsigned k) const {
    const unsigned side = 1u << k;
    std::vector<double2> m(side * side);
    const double* src = F.matrices + size_t(index) * SSB_MATRIX_STRIDE;
    for (unsigned i = 0; i < side * side; ++i) m[i] = make_double2(src[2 * i], src[2 * i + 1]);
    return m;
  }

  void pauli(Traj& t, const ssb_flat_op& op) {
    PauliArgs a{};
    a.n = n;
    a.num_terms = op.term_count;
    if (op.term_count > terms_cap) {  // sites of any length (grown on demand)
      void* p = nullptr;
      CKD(cudaMalloc(&p, op.term_count * sizeof(PauliTermDev)));
      allocs.push_back(p);
      terms = static_cast<PauliTermDev*>(p);
      terms_cap = op.term_count;
    }
    host_terms.resize(op.term_count);
    double prev = 0.0;
    for (uint32_t i = 0; i < op.term_count; ++i) {
      const ssb_flat_term& T = F.terms[op.term_begin + i];
      host_terms[i] = {T.cumulative - prev, T.x_mask, T.z_mask, T.num_y};  // density.cpp:190-192
      prev = T.cumulative;
    }
    CKD(cudaMemcpyAsync(terms, host_terms.data(), op.term_count * sizeof(PauliTermDev), cudaMemcpyHostToDevice,
                        stream));
    a.t = terms;
    dm_pauli<<<grid(d * d), 256, 0, stream>>>(t.rho, scratch, a);
    launched();
    std::swap(t.rho, scratch);
  }

  // diagonal_marginal (density.cpp:148-154): host sum in index order.
  std::vector<double> marginal(const double2* rho, const uint32_t* qubits, unsigned count) {
    std::vector<double2> diag(d);
    CKD(cudaMemcpy2DAsync(diag.data(), sizeof(double2), rho, (d + 1) * sizeof(double2), sizeof(double2), d,
                          cudaMemcpyDeviceToHost, stream));
    CKD(cudaStreamSynchronize(stream));
    std::vector<double> out(1ull << count, 0.0);
    for (uint64_t j = 0; j < d; ++j) out[gather_bits(j, qubits, count)] += diag[j].x;
    return out;
  }

  // evolve_trajectories (density.cpp:162-277).
  std::vector<Traj> run() {
    if (n < 1 || n > 10) throw shotsim::CapacityError("density evolution supports 1..10 qubits");
    scratch = alloc_rho();
    {
      void* p = nullptr;
      CKD(cudaMalloc(&p, kInitialKraus * 16 * sizeof(double2)));
      allocs.push_back(p);
      mats = static_cast<double2*>(p);
      mats_cap = kInitialKraus * 16;
    }
    std::vector<Traj> trajs(1);
    trajs[0].rho = alloc_rho();
    CKD(cudaMemsetAsync(trajs[0].rho, 0, d * d * sizeof(double2), stream));
    const double2 one = make_double2(1.0, 0.0);
    CKD(cudaMemcpyAsync(trajs[0].rho, &one, sizeof(one), cudaMemcpyHostToDevice, stream));
    CKD(cudaStreamSynchronize(stream));
    unsigned intermediate = 0;
    const uint64_t end = std::min<uint64_t>(F.terminal_measure_begin, F.num_ops);
    for (uint64_t i = 0; i < end; ++i) {
      const ssb_flat_op& op = F.ops[i];
      auto holds = [&](const Traj& t) { return !op.has_condition || (t.creg & op.cond_mask) == op.cond_value; };
      switch (op.kind) {
        case SSB_OP_BARRIER:
          break;
        case SSB_OP_GATE: {
          const auto m = matrix(op.matrix, op.num_qubits);
          for (Traj& t : trajs)
            if (holds(t)) conj_sum(t.rho, m, op.num_qubits, op.qubits, 1, false);
          break;
        }
        case SSB_OP_PAULI:
          for (Traj& t : trajs)
            if (holds(t)) pauli(t, op);
          break;
        case SSB_OP_KRAUS: {
          const ssb_flat_channel& ch = F.channels[op.channel];
          std::vector<double2> ms;
          for (uint32_t j = 0; j < ch.num_matrices; ++j) {
            const auto m = matrix(ch.matrix_begin + j, ch.arity);
            ms.insert(ms.end(), m.begin(), m.end());
          }
          for (Traj& t : trajs)
            if (holds(t)) conj_sum(t.rho, ms, ch.arity, op.qubits, ch.num_matrices, true);
          break;
        }
        case SSB_OP_RESET: {
          // Measure-then-correct as the Kraus channel {|0><m|} (density.cpp:229-241).
          const unsigned k = op.num_qubits, side = 1u << k;
          std::vector<double2> ms(size_t(side) * side * side, make_double2(0.0, 0.0));
          for (unsigned m = 0; m < side; ++m) ms[size_t(m) * side * side + m] = make_double2(1.0, 0.0);
          for (Traj& t : trajs)
            if (holds(t)) conj_sum(t.rho, ms, k, op.qubits, side, true);
          break;
        }
        case SSB_OP_MEASURE: {
          if (op.has_condition)
            throw std::invalid_argument("conditional intermediate measurement is unsupported in the exact evolver");
          if (++intermediate > 2)
            throw shotsim::CapacityError("exact evolver supports at most 2 intermediate measure sites");
          std::vector<Traj> next;
          uint64_t qmask = 0;
          for (unsigned b = 0; b < op.num_qubits; ++b) qmask |= 1ull << op.qubits[b];
          for (Traj& t : trajs) {
            const std::vector<double> probs = marginal(t.rho, op.qubits, op.num_qubits);
            for (uint64_t m = 0; m < probs.size(); ++m) {
              if (probs[m] <= 0.0) continue;
              uint64_t offset = 0;
              for (unsigned b = 0; b < op.num_qubits; ++b)
                if ((m >> b) & 1) offset |= 1ull << op.qubits[b];
              Traj child;
              child.rho = alloc_rho();
              dm_project<<<grid(d * d), 256, 0, stream>>>(t.rho, child.rho, n, qmask, offset, probs[m]);
              launched();
              child.creg = t.creg;
              child.weight = t.weight * probs[m];
              for (unsigned b = 0; b < op.num_qubits; ++b) {
                const uint64_t bit = (m >> b) & 1;
                child.creg = (child.creg & ~(1ull << op.clbits[b])) | (bit << op.clbits[b]);
              }
              next.push_back(child);
            }
          }
          trajs = std::move(next);
          break;
        }
        default:
          throw std::invalid_argument("density evolver: unknown op kind");
      }
    }
    CKD(cudaStreamSynchronize(stream));
    return trajs;
  }
};

}  // namespace

// exact_creg_distribution (density.cpp:291-306).
std::map<uint64_t, double> exact_creg_distribution_device(const ssb_flat_program& F, cudaStream_t stream,
                                                          uint64_t* launches, int num_sms) {
  Evolver ev(F, stream, launches, num_sms);
  const std::vector<Traj> trajs = ev.run();
  std::map<uint64_t, double> out;
  const bool terminal = F.terminal_measure_begin < F.num_ops;
  for (const Traj& t : trajs) {
    if (!terminal) {
      out[t.creg] += t.weight;
      continue;
    }
    const std::vector<double> joint = ev.marginal(t.rho, F.sample_qubits, F.num_sample_qubits);
    for (uint64_t m = 0; m < joint.size(); ++m) {
      if (joint[m] <= 0.0) continue;
      uint64_t creg = t.creg;  // NoisyCircuit::apply_sample_outcome (program.cpp:9-15)
      for (uint32_t w = 0; w < F.num_sample_writes; ++w) {
        const uint64_t bit = (m >> F.sample_write_pos[w]) & 1;
        creg = (creg & ~(1ull << F.sample_write_clbit[w])) | (bit << F.sample_write_clbit[w]);
      }
      out[creg] += t.weight * joint[m];
    }
  }
  return out;
}

// exact_distribution (density.cpp:280-289).
std::vector<double> exact_distribution_device(const ssb_flat_program& F, const uint32_t* qubits, unsigned count,
                                              cudaStream_t stream, uint64_t* launches, int num_sms) {
  for (unsigned b = 0; b < count; ++b)
    if (qubits[b] >= F.num_qubits) throw std::invalid_argument("qubit index out of range");
  if (count > F.num_qubits) throw std::invalid_argument("too many qubits");
  Evolver ev(F, stream, launches, num_sms);
  const std::vector<Traj> trajs = ev.run();
  std::vector<double> out(1ull << count, 0.0);
  for (const Traj& t : trajs) {
    const std::vector<double> marginal = ev.marginal(t.rho, qubits, count);
    for (size_t m = 0; m < marginal.size(); ++m) out[m] += t.weight * marginal[m];
  }
  return out;
}

}  // namespace ssb
