// Register segments: a run of consecutive gates / Pauli sites whose qubits
// stay inside one 2-qubit set {la, lb} is applied quad by quad in registers —
// each thread loads the 4 amplitudes (base, +2^la, +2^lb, +both) of a few
// quads from the shared-memory state, applies every op of the segment, and
// stores them back: one shared-memory round trip and one barrier per segment
// instead of per op. Any op on qubits inside {la, lb} maps each quad onto
// itself, and each op is still applied with the reference's per-amplitude
// arithmetic in program order, so the result is bit-identical to applying the
// ops one by one over the whole state (kernels_scalar.cpp:24-81).
#pragma once

#include "cta_ops.cuh"

namespace ssb {

#ifndef SSB_QPT
#define SSB_QPT 2
#endif
#ifndef SSB_TILE_MINB
#define SSB_TILE_MINB 2
#endif
constexpr int QPT = SSB_QPT;  // quads per thread per round

// Quad element e (bit0 <-> la, bit1 <-> lb). 1q gate on quad bit B mixes
// elements (e, e | 1<<B) for e with bit B clear.
template <int B, int MK>
__device__ __forceinline__ void quad_apply1(double2 (&v)[QPT][4], const double2* m, uint64_t cls, int nq) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i0 = B == 0 ? 2 * h : h, i1 = i0 + (1 << B);
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      if (q >= nq) break;
      const double2 a0 = v[q][i0], a1 = v[q][i1];
      if constexpr (MK == MK_1Q_U) {
        // m0 real: m0*a0 = (m0r*a0r, m0r*a0i); m1..m3 general complex.
        const double2 t0 = make_double2(__dmul_rn(m[0].x, a0.x), __dmul_rn(m[0].x, a0.y));
        v[q][i0] = c_add(t0, c_mul(m[1], a1));
        v[q][i1] = c_add(c_mul(m[2], a0), c_mul(m[3], a1));
      } else if constexpr (MK == MK_1Q_REAL) {
        v[q][i0] = c_add(make_double2(__dmul_rn(m[0].x, a0.x), __dmul_rn(m[0].x, a0.y)),
                         make_double2(__dmul_rn(m[1].x, a1.x), __dmul_rn(m[1].x, a1.y)));
        v[q][i1] = c_add(make_double2(__dmul_rn(m[2].x, a0.x), __dmul_rn(m[2].x, a0.y)),
                         make_double2(__dmul_rn(m[3].x, a1.x), __dmul_rn(m[3].x, a1.y)));
      } else {
        const double2 in[2] = {a0, a1};
        v[q][i0] = row_apply<2>(m, cls, 0, in);
        v[q][i1] = row_apply<2>(m, cls, 1, in);
      }
    }
  }
}

__device__ __forceinline__ double2 pick4(const double2 (&a)[4], uint32_t i) {
  double2 r = a[0];
  r = i == 1 ? a[1] : r;
  r = i == 2 ? a[2] : r;
  r = i == 3 ? a[3] : r;
  return r;
}

// 2q gate; `swapped`: op qubits (q0, q1) = (lb, la), i.e. matrix index bit0
// is quad bit 1. Matrix row r / column c use index order (base, +d0, +d1,
// +d0+d1). MONO: mr[r] = the single nonzero entry of row r (column src_r);
// GEN: `m` points at the 16 entries in global memory (rare path, loaded on use
// to keep the register budget of the common paths).
template <int MK>
__device__ __forceinline__ void quad_apply2(double2 (&v)[QPT][4], const double2* mr, const double2* m, uint64_t cls,
                                            uint8_t src, bool swapped, int nq) {
  auto el = [swapped](int r) { return swapped ? ((r & 1) << 1) | (r >> 1) : r; };
#pragma unroll
  for (int q = 0; q < QPT; ++q) {
    if (q >= nq) break;
    double2 in[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) in[r] = v[q][el(r)];
    double2 out[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if constexpr (MK == MK_2Q_MONO) {
        const uint32_t c = (src >> (2 * r)) & 3u;
        const uint32_t k = entry_class(cls, r * 4 + static_cast<int>(c));
        const double2 x = pick4(in, c);
        out[r] = k == E_ONE ? x : c_term(mr[r], k, x);
      } else {
        out[r] = row_apply<4>(m, cls, r, in);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) v[q][el(r)] = out[r];
  }
}

template <int A, int B>
__device__ __forceinline__ void quad_swap(double2 (&v)[QPT][4], int nq) {
#pragma unroll
  for (int q = 0; q < QPT; ++q) {
    if (q >= nq) break;
    const double2 t = v[q][A];
    v[q][A] = v[q][B];
    v[q][B] = t;
  }
}

template <int E>
__device__ __forceinline__ void quad_phase(double2 (&v)[QPT][4], double2 ph, uint32_t cls, int nq) {
#pragma unroll
  for (int q = 0; q < QPT; ++q) {
    if (q >= nq) break;
    v[q][E] = c_term(ph, cls, v[q][E]);
  }
}

// Pauli on the quad: new[e] = (-i)^num_y * (-1)^popc(e & zq) * old[e ^ xq]
// (destination-sign form, kernels_scalar.cpp:58-81).
__device__ __forceinline__ void quad_pauli(double2 (&v)[QPT][4], uint32_t xq, uint32_t zq, uint32_t num_y, int nq) {
#pragma unroll
  for (int q = 0; q < QPT; ++q) {
    if (q >= nq) break;
    double2 old[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) old[e] = v[q][e];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double2 t = pauli_phase(num_y, pick4(old, static_cast<uint32_t>(e) ^ xq));
      if (__popc(static_cast<uint32_t>(e) & zq) & 1) t = c_neg(t);
      v[q][e] = t;
    }
  }
}

// Single-quad forms of the generic 2q apply and the Pauli (logical order).
template <int MK>
__device__ __forceinline__ void quad_apply2_one(double2 (&v)[4], const double2* mr, const double2* m, uint64_t cls,
                                                uint8_t src, bool swapped) {
  auto el = [swapped](int r) { return swapped ? ((r & 1) << 1) | (r >> 1) : r; };
  double2 in[4], out[4];
  for (int r = 0; r < 4; ++r) in[r] = v[el(r)];
  for (int r = 0; r < 4; ++r) {
    if constexpr (MK == MK_2Q_MONO) {
      const uint32_t c = (src >> (2 * r)) & 3u;
      const uint32_t k = entry_class(cls, r * 4 + static_cast<int>(c));
      const double2 x = pick4(in, c);
      out[r] = k == E_ONE ? x : c_term(mr[r], k, x);
    } else {
      out[r] = row_apply<4>(m, cls, r, in);
    }
  }
  for (int r = 0; r < 4; ++r) v[el(r)] = out[r];
}

__device__ __forceinline__ void quad_pauli1(double2 (&v)[4], uint32_t xq, uint32_t zq, uint32_t num_y) {
  double2 old[4];
  for (int e = 0; e < 4; ++e) old[e] = v[e];
  for (int e = 0; e < 4; ++e) {
    double2 t = pauli_phase(num_y, pick4(old, static_cast<uint32_t>(e) ^ xq));
    if (__popc(static_cast<uint32_t>(e) & zq) & 1) t = c_neg(t);
    v[e] = t;
  }
}

// Per-op fallback for a 1-qubit state (no quads).
static __device__ void run_ops_per_op(double2* st, unsigned k, uint32_t begin, uint32_t end, const PassOp* pops,
                               const DevOp* ops, const double2* mats, const DevTerm* terms, uint64_t creg,
                               const uint8_t* sel) {
  for (uint32_t i = begin; i < end; ++i) {
    const PassOp po = pops[i];
    const DevOp& op = ops[po.op];
    if (op.has_cond && (creg & op.cond_mask) != op.cond_value) continue;
    if (op.kind == K_GATE) {
      double2 m[4];
      load_matrix<2>(mats + 16 * op.aux, m);
      cta_apply1(st, k, po.qb[0], m, op.cls);
    } else {
      const DevTerm& tm = terms[op.aux + sel[op.site]];
      if (tm.identity) continue;
      cta_pauli(st, k, (tm.x >> op.q[0]) & 1u, (tm.z >> op.q[0]) & 1u, tm.num_y);
    }
    __syncthreads();
  }
}

// Applies item `it` (a register segment) to the shared-memory state `st` of k
// local qubits. sel: per-site Pauli term choice of this shot. Ends with a
// barrier.
static __device__ void run_segment(double2* st, unsigned k, const Item& it, const PassOp* pops, const DevOp* ops,
                            const double2* mats, const DevTerm* terms, uint64_t creg, const uint8_t* sel) {
  if (k < 2) {
    run_ops_per_op(st, k, it.begin, it.end, pops, ops, mats, terms, creg, sel);
    return;
  }
  const unsigned la = it.la, lb = it.lb;
  const uint64_t dla = uint64_t{1} << la, dlb = uint64_t{1} << lb;
  const uint64_t nquads = uint64_t{1} << (k - 2);
  const uint64_t per_round = uint64_t{NT} * QPT;
  for (uint64_t r0 = 0; r0 < nquads; r0 += per_round) {
    double2 v[QPT][4];
    uint64_t base[QPT];
    int nq = 0;
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      const uint64_t p = r0 + threadIdx.x + uint64_t{NT} * q;
      if (p < nquads) {
        nq = q + 1;
        base[q] = insert_zero(insert_zero(p, la), lb);
        v[q][0] = st[base[q]];
        v[q][1] = st[base[q] | dla];
        v[q][2] = st[base[q] | dlb];
        v[q][3] = st[base[q] | dla | dlb];
      }
    }
    for (uint32_t i = it.begin; i < it.end; ++i) {
      const PassOp po = pops[i];
      const DevOp& op = ops[po.op];
      if (op.has_cond && (creg & op.cond_mask) != op.cond_value) continue;
      if (op.kind == K_GATE) {
        if (op.nq == 1) {
          double2 m[4];
          if (op.mk != MK_1Q_GEN) load_matrix<2>(mats + 16 * op.aux, m);
          const bool b1 = po.qb[0] != 0;
          switch (op.mk) {
            case MK_1Q_U:
              if (b1) quad_apply1<1, MK_1Q_U>(v, m, op.cls, nq);
              else quad_apply1<0, MK_1Q_U>(v, m, op.cls, nq);
              break;
            case MK_1Q_REAL:
              if (b1) quad_apply1<1, MK_1Q_REAL>(v, m, op.cls, nq);
              else quad_apply1<0, MK_1Q_REAL>(v, m, op.cls, nq);
              break;
            default:
              if (b1) quad_apply1<1, MK_1Q_GEN>(v, mats + 16 * op.aux, op.cls, nq);
              else quad_apply1<0, MK_1Q_GEN>(v, mats + 16 * op.aux, op.cls, nq);
              break;
          }
        } else {
          const double2* mg = mats + 16 * op.aux;
          const bool swapped = po.qb[0] != 0;
          if (op.mk == MK_2Q_MONO) {
            double2 mr[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) mr[r] = mg[r * 4 + ((op.src >> (2 * r)) & 3u)];
            quad_apply2<MK_2Q_MONO>(v, mr, mg, op.cls, op.src, swapped, nq);
          } else {
            quad_apply2<MK_2Q_GEN>(v, nullptr, mg, op.cls, op.src, swapped, nq);
          }
        }
      } else {  // Pauli site with this shot's term
        const DevTerm& tm = terms[op.aux + sel[op.site]];
        if (tm.identity) continue;
        uint32_t xq = 0, zq = 0;
        for (unsigned b = 0; b < op.nq; ++b) {
          xq |= ((tm.x >> op.q[b]) & 1u) << po.qb[b];
          zq |= ((tm.z >> op.q[b]) & 1u) << po.qb[b];
        }
        quad_pauli(v, xq, zq, tm.num_y, nq);
      }
    }
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      if (q < nq) {
        st[base[q]] = v[q][0];
        st[base[q] | dla] = v[q][1];
        st[base[q] | dlb] = v[q][2];
        st[base[q] | dla | dlb] = v[q][3];
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Staged variant for the streamed tile passes: the pass's micro-ops, already
// compacted for this shot (identity Pauli draws and failed conditions
// removed), and its matrix table live in shared memory. Registers are
// addressed physically; sigma (2 bits per logical element) maps logical quad
// elements to registers (devprog.hpp UopCode).

// 1q gate on physical register pairs (A0, A1) and (B0, B1) (low, high).
template <int A0, int A1, int B0, int B1, int MK, bool FULL, int NQ = QPT>
__device__ __forceinline__ void quad_apply1p(double2 (&v)[NQ][4], const double2* m, uint64_t cls, int nq) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    if (!FULL && q >= nq) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i0 = h ? B0 : A0, i1 = h ? B1 : A1;
      const double2 a0 = v[q][i0], a1 = v[q][i1];
      if constexpr (MK == MK_1Q_U) {
        const double2 t0 = make_double2(__dmul_rn(m[0].x, a0.x), __dmul_rn(m[0].x, a0.y));
        v[q][i0] = c_add(t0, c_mul(m[1], a1));
        v[q][i1] = c_add(c_mul(m[2], a0), c_mul(m[3], a1));
      } else if constexpr (MK == MK_1Q_REAL) {
        const double2 t0 = make_double2(__dmul_rn(m[0].x, a0.x), __dmul_rn(m[0].x, a0.y));
        const double2 t1 = make_double2(__dmul_rn(m[1].x, a1.x), __dmul_rn(m[1].x, a1.y));
        const double2 t2 = make_double2(__dmul_rn(m[2].x, a0.x), __dmul_rn(m[2].x, a0.y));
        const double2 t3 = make_double2(__dmul_rn(m[3].x, a1.x), __dmul_rn(m[3].x, a1.y));
        v[q][i0] = c_add(t0, t1);
        v[q][i1] = c_add(t2, t3);
      } else {
        const double2 in[2] = {a0, a1};
        const double2 o0 = row_apply<2>(m, cls, 0, in), o1 = row_apply<2>(m, cls, 1, in);
        v[q][i0] = o0;
        v[q][i1] = o1;
      }
    }
  }
}

__device__ __forceinline__ uint32_t sig(uint8_t sigma, uint32_t e) { return (sigma >> (2 * e)) & 3u; }

// Logical view of one quad: L[e] = v[sigma(e)] and back.
__device__ __forceinline__ void gather_logical(const double2 (&v)[4], uint8_t sigma, double2 (&L)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) L[e] = pick4(v, sig(sigma, e));
}
__device__ __forceinline__ void scatter_logical(double2 (&v)[4], uint8_t sigma, const double2 (&L)[4]) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    double2 x = L[0];
#pragma unroll
    for (int e = 1; e < 4; ++e) x = sig(sigma, e) == static_cast<uint32_t>(p) ? L[e] : x;
    v[p] = x;
  }
}

struct Quad4 {
  double2 e[4];
};

// A non-U micro-op on one quad through its logical view (gcls: the gate's
// entry classes for UC_GEN1 / UC_GEN2).
static __device__ __forceinline__ Quad4 logical_quad_op(Quad4 x, Uop u, const double2* m, uint64_t gcls) {
  double2 L[4];
  double2 v[4] = {x.e[0], x.e[1], x.e[2], x.e[3]};
  gather_logical(v, u.sigma, L);
  double2 one[1][4] = {{L[0], L[1], L[2], L[3]}};
  switch (u.code) {
    case UC_U:
    case UC_REAL:
    case UC_GEN1:
    case UC_KRAUS1:
      if (u.src) {
        if (u.code == UC_U) quad_apply1p<0, 2, 1, 3, MK_1Q_U, true, 1>(one, m, 0, 1);
        else if (u.code == UC_REAL) quad_apply1p<0, 2, 1, 3, MK_1Q_REAL, true, 1>(one, m, 0, 1);
        else quad_apply1p<0, 2, 1, 3, MK_1Q_GEN, true, 1>(one, m, gcls, 1);  // GEN1 / KRAUS1
      } else {
        if (u.code == UC_U) quad_apply1p<0, 1, 2, 3, MK_1Q_U, true, 1>(one, m, 0, 1);
        else if (u.code == UC_REAL) quad_apply1p<0, 1, 2, 3, MK_1Q_REAL, true, 1>(one, m, 0, 1);
        else quad_apply1p<0, 1, 2, 3, MK_1Q_GEN, true, 1>(one, m, gcls, 1);
      }
      break;
    case UC_PAULI:
      quad_pauli1(one[0], u.pauli & 3u, (u.pauli >> 2) & 3u, (u.pauli >> 4) & 3u);
      break;
    case UC_MONO: {
      uint64_t cls = 0;
      for (int r = 0; r < 4; ++r)
        cls |= uint64_t{(u.mcls >> (3 * r)) & 7u} << (3 * (r * 4 + ((u.src >> (2 * r)) & 3)));
      const double2 mr[4] = {m[0], m[1], m[2], m[3]};
      quad_apply2_one<MK_2Q_MONO>(one[0], mr, nullptr, cls, u.src, u.qb != 0);
      break;
    }
    default:
      quad_apply2_one<MK_2Q_GEN>(one[0], nullptr, m, gcls, 0, u.qb != 0);
      break;
  }
  const double2 R[4] = {one[0][0], one[0][1], one[0][2], one[0][3]};
  scatter_logical(v, u.sigma, R);
  return Quad4{{v[0], v[1], v[2], v[3]}};
}

// Entry classes a generic micro-op applies with: the gate's (GEN1 / GEN2) or
// the shot's chosen Kraus matrix's (KRAUS1 / KRAUS2).
__device__ __forceinline__ uint64_t generic_cls(const Uop& u, const DevOp* ops, uint64_t kraus_cls) {
  if (u.code == UC_GEN1 || u.code == UC_GEN2) return ops[u.ref].cls;
  if (u.code == UC_KRAUS1 || u.code == UC_KRAUS2) return kraus_cls;
  return 0;
}

// Rare micro-op on one quad that lives in shared memory at its logical
// addresses (base, +dla, +dlb, +both). Out of line and register-free at the
// call site: the hot loop's quad registers are dead across the call (spilled
// to their own tile addresses first), so its register allocation never has to
// meet the call ABI.
static __device__ __noinline__ void rare_quad_op_smem(double2* st, uint64_t base, uint64_t dla, uint64_t dlb, Uop u,
                                                      const double2* m, uint64_t gcls) {
  double2* a[4] = {st + base, st + (base | dla), st + (base | dlb), st + (base | dla | dlb)};
  Quad4 x{{*a[0], *a[1], *a[2], *a[3]}};
  u.sigma = 0xE4;  // operate on the logical view directly
  x = logical_quad_op(x, u, m, gcls);
  for (int e = 0; e < 4; ++e) *a[e] = x.e[e];
}

template <bool FULL>
static __device__ __forceinline__ void run_segment_staged_t(double2* st, unsigned k, const Item& it, const Uop* eops,
                                                            uint32_t begin, uint32_t end, const double2* smats,
                                                            const DevOp* ops, uint64_t kraus_cls) {
  const unsigned la = it.la, lb = it.lb;
  const uint64_t dla = uint64_t{1} << la, dlb = uint64_t{1} << lb;
  const uint64_t nquads = uint64_t{1} << (k - 2);
  const uint64_t per_round = uint64_t{NT} * QPT;
  for (uint64_t r0 = 0; r0 < nquads; r0 += per_round) {
    double2 v[QPT][4];
    uint64_t base[QPT];
    int nq = QPT;
    if (!FULL) nq = 0;
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      const uint64_t p = r0 + threadIdx.x + uint64_t{NT} * q;
      if (FULL || p < nquads) {
        if (!FULL) nq = q + 1;
        base[q] = insert_zero(insert_zero(p, la), lb);
        v[q][0] = st[base[q]];
        v[q][1] = st[base[q] | dla];
        v[q][2] = st[base[q] | dlb];
        v[q][3] = st[base[q] | dla | dlb];
      }
    }
    uint32_t i = begin;
    while (i < end) {
      // Hot inner loop: consecutive 1q U micro-ops on the six register-pair
      // layouts a CX / SWAP relabeling produces (QV: 8 of 11 block ops). It
      // has a single loop-carried path, so the quad registers stay put.
      // All-real 1q gates (H, RY, ...: the reference's real-matrix kernel
      // class) take the same path with their own arithmetic.
      for (; i < end; ++i) {
        const Uop u = eops[i];
        if (u.code != UC_U && u.code != UC_REAL) break;
        const double2* m = smats + u.mat;
        const double2 mm[4] = {m[0], m[1], m[2], m[3]};
        bool hit = true;
#define SSB_P1(a0, a1, b0, b1) \
  case (a0 | (a1 << 2) | (b0 << 4) | (b1 << 6)): quad_apply1p<a0, a1, b0, b1, MK_1Q_U, FULL>(v, mm, 0, nq); break;
#define SSB_P1R(a0, a1, b0, b1) \
  case (a0 | (a1 << 2) | (b0 << 4) | (b1 << 6)): quad_apply1p<a0, a1, b0, b1, MK_1Q_REAL, FULL>(v, mm, 0, nq); break;
        if (u.code == UC_U) {
          switch (u.qb) {
            SSB_P1(0, 1, 2, 3) SSB_P1(0, 2, 1, 3) SSB_P1(0, 3, 2, 1) SSB_P1(0, 2, 3, 1) SSB_P1(0, 1, 3, 2)
            SSB_P1(0, 3, 1, 2)
            default: hit = false; break;
          }
        } else {
          switch (u.qb) {
            SSB_P1R(0, 1, 2, 3) SSB_P1R(0, 2, 1, 3) SSB_P1R(0, 3, 2, 1) SSB_P1R(0, 2, 3, 1) SSB_P1R(0, 1, 3, 2)
            SSB_P1R(0, 3, 1, 2)
            default: hit = false; break;
          }
        }
#undef SSB_P1
#undef SSB_P1R
        if (!hit) break;
      }
      if (i >= end) break;
      const Uop u = eops[i++];
      const double2* m = smats + u.mat;
      if (u.code == UC_SWAP) {
        switch (u.qb) {
          case 0 | (1 << 2): quad_swap<0, 1>(v, nq); break;
          case 0 | (2 << 2): quad_swap<0, 2>(v, nq); break;
          case 0 | (3 << 2): quad_swap<0, 3>(v, nq); break;
          case 1 | (2 << 2): quad_swap<1, 2>(v, nq); break;
          case 1 | (3 << 2): quad_swap<1, 3>(v, nq); break;
          default: quad_swap<2, 3>(v, nq); break;
        }
        continue;
      }
      if (u.code == UC_PHASE) {
        const double2 ph = m[0];
        switch (u.qb) {
          case 0: quad_phase<0>(v, ph, u.mcls, nq); break;
          case 1: quad_phase<1>(v, ph, u.mcls, nq); break;
          case 2: quad_phase<2>(v, ph, u.mcls, nq); break;
          default: quad_phase<3>(v, ph, u.mcls, nq); break;
        }
        continue;
      }
      // Everything else (rare): each quad goes through shared memory at its
      // logical addresses, is transformed out of line, and is reloaded.
#pragma unroll
      for (int q = 0; q < QPT; ++q) {
        if (!FULL && q >= nq) break;
        double2 L[4];
        gather_logical(v[q], u.sigma, L);
        st[base[q]] = L[0];
        st[base[q] | dla] = L[1];
        st[base[q] | dlb] = L[2];
        st[base[q] | dla | dlb] = L[3];
        rare_quad_op_smem(st, base[q], dla, dlb, u, m, generic_cls(u, ops, kraus_cls));
        L[0] = st[base[q]];
        L[1] = st[base[q] | dla];
        L[2] = st[base[q] | dlb];
        L[3] = st[base[q] | dla | dlb];
        scatter_logical(v[q], u.sigma, L);
      }
    }
    // The segment's relabeling: logical element e sits in register slot
    // sigma(e), so slot p is stored at the offset of e = sigma^-1(p) (the
    // permutation goes into four uniform offsets instead of a run-time
    // register index per element).
    const uint8_t sg = it.sigma;
    const uint64_t offe[4] = {0, dla, dlb, dla | dlb};
    uint64_t offp[4];
#pragma unroll
    for (uint32_t p = 0; p < 4; ++p)
      offp[p] = sig(sg, 0) == p ? offe[0] : sig(sg, 1) == p ? offe[1] : sig(sg, 2) == p ? offe[2] : offe[3];
#pragma unroll
    for (int q = 0; q < QPT; ++q) {
      if (FULL || q < nq) {
#pragma unroll
        for (int p = 0; p < 4; ++p) st[base[q] | offp[p]] = v[q][p];
      }
    }
  }
  __syncthreads();
}

static __device__ void run_segment_staged(double2* st, unsigned k, const Item& it, const Uop* eops, uint32_t begin,
                                          uint32_t end, const double2* smats, const DevOp* ops, uint64_t kraus_cls) {
  if ((uint64_t{1} << (k - 2)) % (uint64_t{NT} * QPT) == 0)
    run_segment_staged_t<true>(st, k, it, eops, begin, end, smats, ops, kraus_cls);
  else
    run_segment_staged_t<false>(st, k, it, eops, begin, end, smats, ops, kraus_cls);
}

}  // namespace ssb
