// CTA-level state operations on a shared-memory state (or tile) for sm_100a.
//
// Each function is one reference state op (statevector.cpp / kernels_scalar.cpp)
// restated for a CTA of NT threads over `st` (2^nloc double2 in shared
// memory). Arithmetic order is the reference's (see exact.cuh); reductions
// keep the reference's blocking (512-element sequential blocks, then the fixed
// pairwise tree of common.cpp:12-26) so every probability is bit-identical.
// Callers own the __syncthreads() between ops.
#pragma once

#include "devtypes.h"
#include "exact.cuh"

namespace ssb {

#ifndef SSB_NT
#define SSB_NT 256
#endif
constexpr int NT = SSB_NT;             // threads per CTA (resident_warp.cu: 32)
constexpr uint64_t SUM_BLOCK = 512;    // statevector.cpp:82 / kernels_scalar.cpp:91

// Sequential sum of v[0..c) then — for power-of-two c > 8 — the fixed pairwise
// tree (common.cpp:12-26). Overwrites v. Single thread.
__device__ __forceinline__ double pairwise_inplace(double* v, uint64_t c) {
  if (c <= 8) {
    double s = 0.0;
    for (uint64_t i = 0; i < c; ++i) s = __dadd_rn(s, v[i]);
    return s;
  }
  uint64_t leaves = c / 8;
  for (uint64_t i = 0; i < leaves; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __dadd_rn(s, v[8 * i + j]);
    v[i] = s;
  }
  for (; leaves > 1; leaves /= 2)
    for (uint64_t i = 0; i < leaves / 2; ++i) v[i] = __dadd_rn(v[2 * i], v[2 * i + 1]);
  return v[0];
}

__device__ __forceinline__ uint64_t scatter_bits(uint64_t value, const uint8_t* pos, unsigned k) {
  uint64_t out = 0;
  for (unsigned b = 0; b < k; ++b)
    if ((value >> b) & 1) out |= uint64_t{1} << pos[b];
  return out;
}

// expand_index (common.hpp:61-67) with sorted positions.
__device__ __forceinline__ uint64_t expand_sorted(uint64_t g, const uint8_t* sorted, unsigned k) {
  for (unsigned i = 0; i < k; ++i) g = insert_zero(g, sorted[i]);
  return g;
}

__device__ __forceinline__ void sort_positions(const uint8_t* q, unsigned k, uint8_t* out) {
  for (unsigned i = 0; i < k; ++i) out[i] = q[i];
  for (unsigned i = 1; i < k; ++i)
    for (unsigned j = i; j > 0 && out[j - 1] > out[j]; --j) {
      const uint8_t t = out[j];
      out[j] = out[j - 1];
      out[j - 1] = t;
    }
}

template <int D>
__device__ __forceinline__ void load_matrix(const double2* g, double2* m) {
#pragma unroll
  for (int i = 0; i < D * D; ++i) m[i] = g[i];
}

// ---- unitary application (kernels_scalar.cpp:24-56) ------------------------
__device__ __forceinline__ void cta_apply1(double2* st, unsigned nloc, unsigned t, const double2* m,
                                           uint64_t cls) {
  const uint64_t pairs = uint64_t{1} << (nloc - 1), bit = uint64_t{1} << t;
  for (uint64_t p = threadIdx.x; p < pairs; p += NT) {
    const uint64_t i0 = insert_zero(p, t), i1 = i0 | bit;
    const double2 v[2] = {st[i0], st[i1]};
    st[i0] = row_apply<2>(m, cls, 0, v);
    st[i1] = row_apply<2>(m, cls, 1, v);
  }
}

__device__ __forceinline__ void cta_apply2(double2* st, unsigned nloc, unsigned q0, unsigned q1,
                                           const double2* m, uint64_t cls) {
  const uint64_t quads = uint64_t{1} << (nloc - 2);
  const unsigned pl = q0 < q1 ? q0 : q1, ph = q0 < q1 ? q1 : q0;
  const uint64_t d0 = uint64_t{1} << q0, d1 = uint64_t{1} << q1;
  for (uint64_t p = threadIdx.x; p < quads; p += NT) {
    const uint64_t b = insert_zero(insert_zero(p, pl), ph);
    const double2 v[4] = {st[b], st[b | d0], st[b | d1], st[b | d0 | d1]};
    st[b] = row_apply<4>(m, cls, 0, v);
    st[b | d0] = row_apply<4>(m, cls, 1, v);
    st[b | d1] = row_apply<4>(m, cls, 2, v);
    st[b | d0 | d1] = row_apply<4>(m, cls, 3, v);
  }
}

// Destination-sign fused Pauli (kernels_scalar.cpp:58-81).
__device__ __forceinline__ void cta_pauli(double2* st, unsigned nloc, uint32_t x, uint32_t z,
                                          uint32_t num_y) {
  if (x == 0) {
    const uint64_t dim = uint64_t{1} << nloc;
    for (uint64_t j = threadIdx.x; j < dim; j += NT) {
      double2 v = pauli_phase(num_y, st[j]);
      if (__popcll(j & z) & 1) v = c_neg(v);
      st[j] = v;
    }
    return;
  }
  const unsigned xmax = 31 - __clz(x);
  const uint64_t pairs = uint64_t{1} << (nloc - 1);
  for (uint64_t p = threadIdx.x; p < pairs; p += NT) {
    const uint64_t i0 = insert_zero(p, xmax), i1 = i0 ^ x;
    double2 t0 = pauli_phase(num_y, st[i1]), t1 = pauli_phase(num_y, st[i0]);
    if (__popcll(i0 & z) & 1) t0 = c_neg(t0);
    if (__popcll(i1 & z) & 1) t1 = c_neg(t1);
    st[i0] = t0;
    st[i1] = t1;
  }
}

// ---- exact reductions --------------------------------------------------------
// All 2^k outcome probabilities of qubits q (outcome_probability,
// statevector.cpp:142-164) into probs[] (shared). red: shared scratch of
// max(2^k * G/512, 1) doubles. Ends with __syncthreads().
// Sequential sum of |st[insert_zero(g, t) | off]|^2 over g in [g0, g1): the
// reference's in-block order, 8 elements loaded ahead of the add chain.
__device__ __forceinline__ double block_norm_sum_1q(const double2* st, unsigned t, uint64_t off, uint64_t g0,
                                                    uint64_t g1) {
  double s = 0.0;
  uint64_t g = g0;
  for (; g + 8 <= g1; g += 8) {
    double p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = c_norm(st[insert_zero(g + j, t) | off]);
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __dadd_rn(s, p[j]);
  }
  for (; g < g1; ++g) s = __dadd_rn(s, c_norm(st[insert_zero(g, t) | off]));
  return s;
}

static __device__ __noinline__ void cta_outcome_probs(const double2* st, unsigned n, const uint8_t* q, unsigned k,
                                  double* probs, double* red) {
  if (k == 1) {  // single-qubit measure / reset (the common case): no index tables
    const unsigned t = q[0];
    const uint64_t bit = uint64_t{1} << t, G = uint64_t{1} << (n - 1);
    if (G <= SUM_BLOCK) {
      if (threadIdx.x < 2) probs[threadIdx.x] = block_norm_sum_1q(st, t, threadIdx.x ? bit : 0, 0, G);
      __syncthreads();
      return;
    }
    const uint64_t nb = G / SUM_BLOCK;
    for (uint64_t x = threadIdx.x; x < 2 * nb; x += NT) {
      const uint64_t m = x / nb, b = x % nb;
      red[x] = block_norm_sum_1q(st, t, m ? bit : 0, b * SUM_BLOCK, (b + 1) * SUM_BLOCK);
    }
    __syncthreads();
    if (threadIdx.x < 2) probs[threadIdx.x] = pairwise_inplace(red + threadIdx.x * nb, nb);
    __syncthreads();
    return;
  }
  uint8_t sorted[32];
  sort_positions(q, k, sorted);
  const uint64_t G = uint64_t{1} << (n - k), no = uint64_t{1} << k;
  if (G <= SUM_BLOCK) {
    for (uint64_t m = threadIdx.x; m < no; m += NT) {
      const uint64_t off = scatter_bits(m, q, k);
      double s = 0.0;
      for (uint64_t g = 0; g < G; ++g) s = __dadd_rn(s, c_norm(st[expand_sorted(g, sorted, k) | off]));
      probs[m] = s;
    }
    __syncthreads();
    return;
  }
  const uint64_t nb = G / SUM_BLOCK;
  for (uint64_t t = threadIdx.x; t < no * nb; t += NT) {
    const uint64_t m = t / nb, b = t % nb, off = scatter_bits(m, q, k);
    double s = 0.0;
    for (uint64_t g = b * SUM_BLOCK; g < (b + 1) * SUM_BLOCK; ++g)
      s = __dadd_rn(s, c_norm(st[expand_sorted(g, sorted, k) | off]));
    red[t] = s;
  }
  __syncthreads();
  for (uint64_t m = threadIdx.x; m < no; m += NT) probs[m] = pairwise_inplace(red + m * nb, nb);
  __syncthreads();
}

// <psi|M^dag M|psi> for a 2x2 M (expval_matrix1_scalar, kernels_scalar.cpp:103-126).
// Result valid in all threads. red: >= max(1, 2^(n-1)/512) doubles + 1.
static __device__ __noinline__ double cta_expval1(const double2* st, unsigned n, unsigned t, const double2* m, double* red) {
  const uint64_t pairs = uint64_t{1} << (n - 1), bit = uint64_t{1} << t;
  const uint64_t nb = pairs <= SUM_BLOCK ? 1 : pairs / SUM_BLOCK;
  const uint64_t len = pairs <= SUM_BLOCK ? pairs : SUM_BLOCK;
  for (uint64_t b = threadIdx.x; b < nb; b += NT) {
    double s = 0.0;
    for (uint64_t i = b * len; i < (b + 1) * len; ++i) {
      const uint64_t i0 = insert_zero(i, t), i1 = i0 | bit;
      const double2 a0 = st[i0], a1 = st[i1];
      const double2 r0 = c_add(c_mul(m[0], a0), c_mul(m[1], a1));
      const double2 r1 = c_add(c_mul(m[2], a0), c_mul(m[3], a1));
      s = __dadd_rn(s, c_norm(r0));
      s = __dadd_rn(s, c_norm(r1));
    }
    red[b] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) red[nb] = nb == 1 ? red[0] : pairwise_inplace(red, nb);
  __syncthreads();
  const double r = red[nb];
  __syncthreads();
  return r;
}

// Generic k=2 expval (expval_generic, statevector.cpp:56-80): per-group sums of
// |row|^2, then pairwise over all 2^(n-2) groups. red: >= max(1, 2^(n-2)/8) + 1.
static __device__ __noinline__ double cta_expval2(const double2* st, unsigned n, const uint8_t* q, const double2* m,
                              double* red) {
  uint8_t sorted[2];
  sort_positions(q, 2, sorted);
  const uint64_t G = uint64_t{1} << (n - 2);
  const uint64_t off[4] = {0, uint64_t{1} << q[0], uint64_t{1} << q[1], (uint64_t{1} << q[0]) | (uint64_t{1} << q[1])};
  const uint64_t leaf = G <= 8 ? G : 8, nl = G / leaf;
  for (uint64_t l = threadIdx.x; l < nl; l += NT) {
    double s = 0.0;
    for (uint64_t g = l * leaf; g < (l + 1) * leaf; ++g) {
      const uint64_t base = expand_sorted(g, sorted, 2);
      double2 in[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) in[c] = st[base + off[c]];
      double part = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc = c_add(acc, c_mul(m[4 * r + c], in[c]));
        part = __dadd_rn(part, c_norm(acc));
      }
      s = __dadd_rn(s, part);
    }
    red[l] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = red[0];
    if (nl > 1) {
      for (uint64_t w = nl; w > 1; w /= 2)
        for (uint64_t i = 0; i < w / 2; ++i) red[i] = __dadd_rn(red[2 * i], red[2 * i + 1]);
      r = red[0];
    }
    red[nl] = r;
  }
  __syncthreads();
  const double r = red[nl];
  __syncthreads();
  return r;
}

// pick_outcome (statevector.cpp:185-197): sequential cumulative, strict <,
// fallback to the last nonzero outcome. Returns false when all are zero.
__device__ __forceinline__ bool pick_outcome(const double* probs, uint64_t count, double u, uint64_t* out) {
  double cum = 0.0;
  uint64_t last = count;
  for (uint64_t m = 0; m < count; ++m) {
    cum = __dadd_rn(cum, probs[m]);
    if (u < cum) {
      *out = m;
      return true;
    }
    if (probs[m] > 0.0) last = m;
  }
  *out = last == count ? 0 : last;
  return last != count;
}

// project_and_renormalize (statevector.cpp:173-183) fused with the reset
// X-correction (exec_naive.cpp:51-60): survivors move from j to j ^ xfix.
__device__ __forceinline__ void cta_collapse(double2* st, unsigned nloc, uint64_t qmask, uint64_t offset,
                                             double inv, uint64_t xfix) {
  if (xfix == 0) {
    const uint64_t dim = uint64_t{1} << nloc;
    for (uint64_t j = threadIdx.x; j < dim; j += NT)
      st[j] = ((j & qmask) == offset) ? c_scale(st[j], inv) : make_double2(0.0, 0.0);
    return;
  }
  const unsigned xmax = 63 - __clzll(xfix);
  const uint64_t pairs = uint64_t{1} << (nloc - 1);
  for (uint64_t p = threadIdx.x; p < pairs; p += NT) {
    const uint64_t i0 = insert_zero(p, xmax), i1 = i0 ^ xfix;
    const double2 a0 = st[i0], a1 = st[i1];
    st[i0] = ((i1 & qmask) == offset) ? c_scale(a1, inv) : make_double2(0.0, 0.0);
    st[i1] = ((i0 & qmask) == offset) ? c_scale(a0, inv) : make_double2(0.0, 0.0);
  }
}

__device__ __forceinline__ int pick_term(const DevTerm* terms, uint32_t count, double u) {
  for (uint32_t t = 0; t < count; ++t)
    if (u < terms[t].cum) return static_cast<int>(t);
  return static_cast<int>(count) - 1;
}

__device__ __forceinline__ uint64_t write_bits(uint64_t creg, const uint8_t* clbits, unsigned k, uint64_t v) {
  for (unsigned b = 0; b < k; ++b)
    creg = (creg & ~(uint64_t{1} << clbits[b])) | (((v >> b) & 1) << clbits[b]);
  return creg;
}

}  // namespace ssb
