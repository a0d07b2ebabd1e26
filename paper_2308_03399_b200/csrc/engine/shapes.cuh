// Straight-line segment executors ("shapes"). devprog.cpp shape_source()
// emits one function per distinct segment shape of a streamed plan — the
// segment's micro-ops with every operand a compile-time constant — built from
// the macros below; specialise.cu compiles that source at run time (NVRTC) into
// a shape-specialised tile_pass_kernel. Without it (the static build) every
// segment runs through the interpreter (run_segment_staged): the arithmetic is
// identical op for op, the specialised form only removes per-op dispatch and
// keeps the quads in fixed registers.
#pragma once

#include "segment.cuh"

namespace ssb {

__device__ __forceinline__ uint32_t insert_zero32(uint32_t i, uint32_t bit) {
  const uint32_t lo = (1u << bit) - 1;
  return ((i & ~lo) << 1) | (i & lo);
}

// Requires (2^(k-2)) % (NT * QPT) == 0 (every round full).
#define SSB_SHAPE_BEGIN                                                              \
  const uint32_t dla = 1u << la, dlb = 1u << lb;                                     \
  const uint32_t nquads = 1u << (k - 2);                                             \
  for (uint32_t r0 = 0; r0 < nquads; r0 += NT * QPT) {                               \
    double2 v[QPT][4];                                                               \
    uint32_t base[QPT];                                                              \
    _Pragma("unroll") for (int q = 0; q < QPT; ++q) {                                \
      base[q] = insert_zero32(insert_zero32(r0 + threadIdx.x + NT * q, la), lb);     \
      v[q][0] = st[base[q]];                                                         \
      v[q][1] = st[base[q] | dla];                                                   \
      v[q][2] = st[base[q] | dlb];                                                   \
      v[q][3] = st[base[q] | dla | dlb];                                             \
    }

#define SSB_SHAPE_LOGICAL(U, M, GCLS)                                                \
  _Pragma("unroll") for (int q = 0; q < QPT; ++q) {                                  \
    Quad4 x{{v[q][0], v[q][1], v[q][2], v[q][3]}};                                   \
    x = logical_quad_op(x, U, M, GCLS);                                              \
    _Pragma("unroll") for (int e = 0; e < 4; ++e) v[q][e] = x.e[e];                  \
  }

// A drawn Pauli on every quad through the logical view; pv packs xq | zq << 2
// | (num_y & 3) << 4 (tile_pass compaction). Out of line: it runs only for
// shots that drew a Pauli in the segment, and one shared body keeps the
// run-time compile small.
static __device__ __noinline__ Quad4 shape_pauli_call(Quad4 x, unsigned sigma, unsigned pv) {
  double2 v[4] = {x.e[0], x.e[1], x.e[2], x.e[3]};
  double2 L[4];
  gather_logical(v, static_cast<uint8_t>(sigma), L);
  quad_pauli1(L, pv & 3u, (pv >> 2) & 3u, (pv >> 4) & 3u);
  scatter_logical(v, static_cast<uint8_t>(sigma), L);
  return Quad4{{v[0], v[1], v[2], v[3]}};
}

#define SSB_SHAPE_PAULI(SIGMA, PV)                                                   \
  {                                                                                  \
    const unsigned pv_ = (PV);                                                       \
    if (pv_ != 0xFFu) {                                                              \
      _Pragma("unroll") for (int q = 0; q < QPT; ++q) {                              \
        Quad4 x_{{v[q][0], v[q][1], v[q][2], v[q][3]}};                              \
        x_ = shape_pauli_call(x_, (SIGMA), pv_);                                     \
        _Pragma("unroll") for (int e = 0; e < 4; ++e) v[q][e] = x_.e[e];             \
      }                                                                              \
    }                                                                                \
  }

#define SSB_SHAPE_PAULI_INLINE(SIGMA, PV)                                            \
  {                                                                                  \
    const unsigned pv_ = (PV);                                                       \
    if (pv_ != 0xFFu) {                                                              \
      _Pragma("unroll") for (int q = 0; q < QPT; ++q) {                              \
        double2 L[4];                                                                \
        gather_logical(v[q], SIGMA, L);                                              \
        quad_pauli1(L, pv_ & 3u, (pv_ >> 2) & 3u, (pv_ >> 4) & 3u);                  \
        scatter_logical(v[q], SIGMA, L);                                             \
      }                                                                              \
    }                                                                                \
  }

#define SSB_SHAPE_END(SIGMA)                                                         \
    _Pragma("unroll") for (int q = 0; q < QPT; ++q) {                                \
      double2 L[4];                                                                  \
      gather_logical(v[q], SIGMA, L);                                                \
      st[base[q]] = L[0];                                                            \
      st[base[q] | dla] = L[1];                                                      \
      st[base[q] | dlb] = L[2];                                                      \
      st[base[q] | dla | dlb] = L[3];                                                \
    }                                                                                \
  }                                                                                  \
  __syncthreads();

}  // namespace ssb

#ifdef SSB_SHAPES
#include "ssb_shapes.inc"  // generated: devprog.cpp shape_source()
#else
namespace ssb {
// Static build: no specialised shapes; every segment is interpreted.
static __device__ __forceinline__ bool ssb_run_shape(unsigned, bool, double2*, unsigned, unsigned, unsigned,
                                                     const double2*, uint64_t, const uint8_t*) {
  return false;
}
}  // namespace ssb
#endif
