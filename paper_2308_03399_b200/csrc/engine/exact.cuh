// Exact device arithmetic for the shotsim_b200 engine (sm_100a).
//
// Bit-exactness contract: every amplitude and probability the device computes
// is produced by the same sequence of correctly-rounded IEEE-754 binary64
// operations as the reference's SCALAR kernel table (kernels_scalar.cpp,
// statevector.cpp), up to the sign of exact zeros. Contraction into FMA is
// forbidden (explicit __dmul_rn/__dadd_rn; the TU is also built -fmad=false).
//
// "Structured" matrix entries: a product m*v with m = (0,0), (+-1,0), (a,0)
// or (0,b) equals the reference's full complex product (ac-bd, ad+bc) except
// possibly in the sign of a zero result, and adding an exact +-0 term to a
// partial sum leaves every nonzero value unchanged. Dropping those operations
// therefore preserves every nonzero amplitude bit for bit and never changes a
// probability or decision (signed zeros square to +0).
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

#ifdef __CUDACC__
#define SSB_HD __host__ __device__
#else
#define SSB_HD
#endif

namespace ssb {

// Entry classes (3 bits each, 16 entries per 4x4 matrix packed in a u64).
enum EntryClass : uint32_t { E_ZERO = 0, E_ONE = 1, E_NEG_ONE = 2, E_REAL = 3, E_IMAG = 4, E_GEN = 5 };

SSB_HD inline uint32_t entry_class(uint64_t cls, int i) { return static_cast<uint32_t>((cls >> (3 * i)) & 7u); }

// ---- Philox-4x32-10 keyed uniform — rng.cpp:9-46 --------------------------
SSB_HD inline double keyed_uniform(uint64_t seed, uint64_t shot,
                                                         uint64_t event) {
  uint32_t c0 = static_cast<uint32_t>(shot), c1 = static_cast<uint32_t>(shot >> 32);
  uint32_t c2 = static_cast<uint32_t>(event), c3 = static_cast<uint32_t>(event >> 32);
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    const uint64_t p0 = uint64_t{0xD2511F53u} * c0, p1 = uint64_t{0xCD9E8D57u} * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
#endif
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c1 = lo1;
    c3 = lo0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint64_t bits = (static_cast<uint64_t>(c0) << 32) | c1;
  return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

#ifdef __CUDACC__

// ---- complex helpers (libstdc++ std::complex<double> semantics, no FMA) ---
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 c_add(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 c_scale(double2 a, double d) {
  return make_double2(__dmul_rn(a.x, d), __dmul_rn(a.y, d));
}
__device__ __forceinline__ double2 c_neg(double2 a) { return make_double2(-a.x, -a.y); }
// |a|^2 = re*re + im*im (statevector.cpp:153), two rounded products + add.
__device__ __forceinline__ double c_norm(double2 a) {
  return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// m*v for a classed entry; only called for cls != E_ZERO.
__device__ __forceinline__ double2 c_term(double2 m, uint32_t cls, double2 v) {
  switch (cls) {
    case E_ONE: return v;
    case E_NEG_ONE: return c_neg(v);
    case E_REAL: return make_double2(__dmul_rn(m.x, v.x), __dmul_rn(m.x, v.y));
    case E_IMAG: return make_double2(-__dmul_rn(m.y, v.y), __dmul_rn(m.y, v.x));
    default: return c_mul(m, v);
  }
}

// Row r of a D x D classed matrix applied to v[0..D): left-to-right sum of the
// nonzero terms, ((t0 + t1) + t2) + t3 (kernels_scalar.cpp:29-32, 51-54).
template <int D>
__device__ __forceinline__ double2 row_apply(const double2* m, uint64_t cls, int r, const double2* v) {
  double2 acc = make_double2(0.0, 0.0);
  bool any = false;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const uint32_t k = entry_class(cls, r * D + c);
    if (k == E_ZERO) continue;
    const double2 t = c_term(m[r * D + c], k, v[c]);
    acc = any ? c_add(acc, t) : t;
    any = true;
  }
  return acc;
}

// (-i)^(num_y mod 4) * a (kernels_scalar.cpp:15-22) — exact up to signed zero.
__device__ __forceinline__ double2 pauli_phase(uint32_t num_y, double2 a) {
  switch (num_y & 3u) {
    case 0: return a;
    case 1: return make_double2(a.y, -a.x);
    case 2: return make_double2(-a.x, -a.y);
    default: return make_double2(-a.y, a.x);
  }
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t i, uint32_t bit) {
  const uint64_t lo = (uint64_t{1} << bit) - 1;
  return ((i & ~lo) << 1) | (i & lo);
}

#endif  // __CUDACC__

}  // namespace ssb
