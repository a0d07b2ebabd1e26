// Warp-parallel, bit-exact restatement of the reference's SEQUENTIAL
// cumulative `cum = fl(cum + p[m])` (pick_outcome, statevector.cpp:185-197;
// the leaf cumulative of run_branch, exec_branch.cpp:267-276).
//
// Idea (the same one sample_exact_kernel uses per 2048-outcome chunk, here per
// 32 outcomes with a warp prefix scan): while the running sum S stays in one
// binade [2^(e-1), 2^e) with ulp w = 2^(e-53), S = a*w for an integer a in
// [2^52, 2^53) and every reference step fl(a*w + p) equals w*(a + rint(p/w))
// — exactly — unless p/w is a tie (fraction exactly 1/2: the result depends on
// a's parity) or the sum leaves the binade. So each lane turns its p into the
// integer rint(p/w), a warp inclusive scan gives every lane its exact S_m, and
// only the first lane that would break the rule (a tie, a binade change, a
// subnormal or zero S) is stepped with the reference's own rounded add before
// the scan resumes behind it. Binade changes happen ~log2(1/p_min) times per
// scan, ties essentially never, so ~A/32 warp steps replace A dependent adds.
#pragma once

#include "exact.cuh"

namespace ssb {

struct ExactPick {
  uint64_t outcome;   // first m with u < S_m, else the last m with p_m > 0
  double s_prev;      // S_{m-1} (0 for m = 0): the decision's lower boundary
  double s_at;        // S_m: its upper boundary
  bool crossed;       // false: no crossing (pick_outcome's fallback, or none)
  bool any_nonzero;   // some p_m > 0 (else DegenerateDistribution)
};

// All 32 lanes of a warp call this with the same arguments. prob(m) returns
// p_m (m < count); on_sum(m, S_m), when not null-like, receives every running
// sum in order of m (only called by the lane owning m; used to build a
// leaf's cumulative table). u = +inf scans the whole range (no early exit).
template <class Prob, class OnSum>
__device__ __forceinline__ ExactPick warp_exact_scan(Prob prob, uint64_t count, double u, OnSum on_sum) {
  const unsigned lane = threadIdx.x & 31;
  double S = 0.0;
  long long last_nz = -1;
  ExactPick r{0, 0.0, 0.0, false, false};
  for (uint64_t c0 = 0; c0 < count; c0 += 32) {
    const uint64_t m = c0 + lane;
    const double p = m < count ? prob(m) : 0.0;
    const unsigned nz = __ballot_sync(0xffffffffu, p > 0.0);
    if (nz) last_nz = static_cast<long long>(c0 + 31 - __clz(nz));
    unsigned start = 0;
    while (start < 32) {
      const unsigned live = ~0u << start;  // lanes start..31 (start < 32)
      if (!(S >= 0x1p-1022)) {
        // S is zero or subnormal: zero p's keep S = 0 exactly (and u < 0 never
        // holds); step the first nonzero lane with the reference's add.
        unsigned b;
        if (S == 0.0) {
          const unsigned nzl = nz & live;
          if (!nzl) {
            if (m < count && lane >= start) on_sum(m, 0.0);
            break;
          }
          b = __ffs(nzl) - 1;
          if (m < count && lane >= start && lane < b) on_sum(m, 0.0);
        } else {
          b = start;
        }
        const double pb = __shfl_sync(0xffffffffu, p, b);
        const double Sn = __dadd_rn(S, pb);
        if (lane == b && c0 + b < count) on_sum(c0 + b, Sn);
        if (u < Sn && c0 + b < count) {
          r.outcome = c0 + b;
          r.s_prev = S;
          r.s_at = Sn;
          r.crossed = true;
          r.any_nonzero = true;
          return r;
        }
        S = Sn;
        start = b + 1;
        continue;
      }
      if (!(nz & live)) {
        // only zeros left in this chunk: fl(S + 0) = S for every lane, and
        // u < S was already ruled out when S was reached
        if (m < count && lane >= start) on_sum(m, S);
        break;
      }
      int e = 0;
      frexp(S, &e);
      const double w = ldexp(1.0, e - 53);
      const long long a0 = static_cast<long long>(S / w);  // exact: S = a0 * w
      bool bad = false;
      long long k = 0;
      if (lane >= start) {
        const double x = p / w;  // exact (power-of-two divisor)
        if (x >= 0x1p42) bad = true;
        else {
          bad = (x - floor(x)) == 0.5;
          k = static_cast<long long>(rint(x));
        }
      }
      // Inclusive scan of k over the warp (lanes < start contribute 0).
      long long pre = k;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, pre, off);
        if (lane >= static_cast<unsigned>(off)) pre += v;
      }
      const long long a = a0 + pre;
      const bool brk = lane >= start && (bad || a >= (1ll << 53));
      const unsigned bm = __ballot_sync(0xffffffffu, brk);
      const unsigned B = bm ? __ffs(bm) - 1 : 32;  // first lane the rule does not cover
      const double Sl = static_cast<double>(a) * w;  // exact for lanes in [start, B)
      const bool ok = lane >= start && lane < B;
      if (ok && m < count) on_sum(m, Sl);
      const unsigned cross = __ballot_sync(0xffffffffu, ok && m < count && u < Sl);
      if (cross) {
        const unsigned c = __ffs(cross) - 1;
        const double prev = __shfl_sync(0xffffffffu, Sl, c == 0 ? 0 : c - 1);
        r.outcome = c0 + c;
        r.s_prev = c == start ? S : prev;
        r.s_at = __shfl_sync(0xffffffffu, Sl, c);
        r.crossed = true;
        r.any_nonzero = true;
        return r;
      }
      if (B > start) S = __shfl_sync(0xffffffffu, Sl, B - 1);
      if (B == 32) break;
      // Lane B: one reference step (binade change or tie), then resume.
      const double pb = __shfl_sync(0xffffffffu, p, B);
      const double Sn = __dadd_rn(S, pb);
      if (lane == B && m < count) on_sum(m, Sn);
      if (u < Sn && c0 + B < count) {
        r.outcome = c0 + B;
        r.s_prev = S;
        r.s_at = Sn;
        r.crossed = true;
        r.any_nonzero = true;
        return r;
      }
      S = Sn;
      start = B + 1;
    }
  }
  r.any_nonzero = last_nz >= 0;
  r.outcome = last_nz >= 0 ? static_cast<uint64_t>(last_nz) : 0;
  r.s_prev = S;
  r.s_at = S;
  return r;
}

// +infinity without <cmath> (the header is also compiled by NVRTC).
__device__ __forceinline__ double scan_all() { return __longlong_as_double(0x7FF0000000000000ll); }

struct NoSum {
  __device__ __forceinline__ void operator()(uint64_t, double) const {}
};

}  // namespace ssb
