// gpu-branch: shot-branching executor (paper SIV.B; reference
// exec_branch.cpp:175-295) with device-resident states and shot lists.
//
// Live states sit in a slot pool in HBM; the shots mapped to each live node
// are a contiguous range of a device shot-id array (node-major). At every
// randomness site the device computes the node-level quantities (outcome
// probabilities / Kraus expectation values, exact reference order), then one
// thread per shot draws its keyed uniform and picks its decision key, counting
// (node, key) groups. The host only sees the small group-count table: it
// applies the reference's budget policy (count desc, parent asc, key asc;
// exec_branch.cpp:217-255), assigns child slots (first child reuses the
// parent's slot, others are copies taken before any transform), and the device
// scatters shots, copies states and applies each child's decision.
// Leaves: per-leaf sequential cumulative (exact pick_outcome order) built once,
// then one binary search per shot (first index with u < cum, which is what the
// sequential scan returns because the cumulative is monotone).
#include <cuda_runtime.h>


#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <cmath>
#include <chrono>
#include <numeric>
#include <type_traits>
#include <vector>

#include "../capi_internal.hpp"
#include "kernels.cuh"

namespace ssb {

#define CKB(expr)                                                                          \
  do {                                                                                     \
    const cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess) throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Node table entry as seen by the device.
struct DevNode {
  uint32_t slot;
  uint32_t cond_ok;  // site condition holds for this node's register
  uint64_t off, len; // shot range in the node-major shot array
  uint64_t creg;
};

__device__ __forceinline__ uint64_t node_of(const DevNode* nodes, uint64_t nn, uint64_t pos) {
  uint64_t lo = 0, hi = nn;  // last node with off <= pos
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (nodes[mid].off <= pos) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void b_init_slot(double2* pool, uint32_t slot, unsigned n) {
  const uint64_t A = uint64_t{1} << n;
  for (uint64_t j = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x; j < A; j += uint64_t{gridDim.x} * blockDim.x)
    pool[(uint64_t{slot} << n) + j] = make_double2(j == 0 ? 1.0 : 0.0, 0.0);
}

__global__ void b_iota(uint64_t* ids, uint64_t begin, uint64_t count) {
  const uint64_t i = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (i < count) ids[i] = begin + i;
}

// Per-shot decision key + (node, key) counts. vals: node-level quantities
// (probs[node][2^k] for measure/reset, p[node][nmat] for Kraus).
__global__ void b_decide(ProgView P, DevOp op, const DevNode* nodes, uint64_t nn, const uint64_t* shots,
                         uint64_t total, uint64_t seed, const double* vals, uint32_t nkeys, uint32_t* keys,
                         unsigned* counts, int* err) {
  const uint64_t pos = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (pos >= total) return;
  const uint64_t node = node_of(nodes, nn, pos);
  uint32_t key = 0;
  if (nodes[node].cond_ok) {
    const double u = keyed_uniform(seed, shots[pos], op.event);
    if (op.kind == K_PAULI) {
      key = static_cast<uint32_t>(pick_term(P.terms + op.aux, op.count, u));
    } else if (op.kind == K_KRAUS) {
      const double* p = vals + node * nkeys;
      double cum = 0.0;
      key = nkeys - 1;  // slack fallback: last matrix with its p (exec_branch.cpp:73-85)
      for (uint32_t i = 0; i < nkeys; ++i) {
        cum = __dadd_rn(cum, p[i]);
        if (u < cum) {
          key = i;
          break;
        }
      }
    } else {
      uint64_t o = 0;
      if (!pick_outcome(vals + node * nkeys, nkeys, u, &o)) raise(err, DEV_DEGENERATE);
      key = static_cast<uint32_t>(o);
    }
  }
  keys[pos] = key;
  atomicAdd(&counts[node * nkeys + key], 1u);
}

// dst[node*nkeys+key]: base offset in the new shot array (kept) or, with the
// top bit set, in the waiting array (deferred).
__global__ void b_scatter(const DevNode* nodes, uint64_t nn, const uint64_t* shots, uint64_t total,
                          const uint32_t* keys, uint32_t nkeys, const uint64_t* dst, unsigned long long* cursor,
                          uint64_t* next_shots, uint64_t* waiting) {
  const uint64_t pos = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (pos >= total) return;
  const uint64_t g = node_of(nodes, nn, pos) * nkeys + keys[pos];
  const uint64_t d = dst[g];
  const uint64_t at = (d & ~(uint64_t{1} << 63)) + atomicAdd(&cursor[g], 1ull);
  if (d >> 63) waiting[at] = shots[pos];
  else next_shots[at] = shots[pos];
}

__global__ void b_copy_slots(double2* pool, const uint2* pairs, uint64_t npairs, unsigned n) {
  const uint64_t A = uint64_t{1} << n, total = npairs * A;
  for (uint64_t i = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x; i < total; i += uint64_t{gridDim.x} * blockDim.x) {
    const uint2 pr = pairs[i / A];
    const uint64_t j = i % A;
    pool[(uint64_t{pr.y} << n) + j] = pool[(uint64_t{pr.x} << n) + j];
  }
}

// One child's decision (apply_decision, exec_branch.cpp:104-136).
struct ChildOp {
  uint32_t slot;
  uint32_t key;
  double inv;  // Kraus / collapse scale 1/sqrt(param)
};

__global__ void b_apply(ProgView P, DevOp op, double2* pool, const ChildOp* kids, uint64_t nk, unsigned n) {
  const uint64_t per = uint64_t{1} << (n - 1), total = nk * per;
  uint64_t qmask = 0;
  for (unsigned b = 0; b < op.nq; ++b) qmask |= uint64_t{1} << op.q[b];
  for (uint64_t idx = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x; idx < total;
       idx += uint64_t{gridDim.x} * blockDim.x) {
    const ChildOp ch = kids[idx / per];
    const uint64_t p = idx % per;
    double2* a = pool + (uint64_t{ch.slot} << n);
    if (op.kind == K_PAULI) {
      const DevTerm tm = P.terms[op.aux + ch.key];
      if (tm.x == 0) {
        for (int h = 0; h < 2; ++h) {
          const uint64_t j = 2 * p + h;
          double2 v = pauli_phase(tm.num_y, a[j]);
          if (__popcll(j & tm.z) & 1) v = c_neg(v);
          a[j] = v;
        }
      } else {
        const unsigned xmax = 31 - __clz(tm.x);
        const uint64_t i0 = insert_zero(p, xmax), i1 = i0 ^ tm.x;
        double2 t0 = pauli_phase(tm.num_y, a[i1]), t1 = pauli_phase(tm.num_y, a[i0]);
        if (__popcll(i0 & tm.z) & 1) t0 = c_neg(t0);
        if (__popcll(i1 & tm.z) & 1) t1 = c_neg(t1);
        a[i0] = t0;
        a[i1] = t1;
      }
    } else if (op.kind == K_KRAUS) {
      const DevChannel chn = P.channels[op.aux];
      const uint32_t slot = chn.mat_begin + ch.key;
      const uint64_t cls = P.scaled_cls[slot];
      if (chn.arity == 1) {
        if (p >= per) continue;
        double2 m[4];
        for (int e = 0; e < 4; ++e) m[e] = c_scale(P.mats[16 * slot + e], ch.inv);
        const uint64_t i0 = insert_zero(p, op.q[0]), i1 = i0 | (uint64_t{1} << op.q[0]);
        const double2 v[2] = {a[i0], a[i1]};
        a[i0] = row_apply<2>(m, cls, 0, v);
        a[i1] = row_apply<2>(m, cls, 1, v);
      } else {
        if (p >= per / 2) continue;  // quads: half the pair slots
        double2 m[16];
        for (int e = 0; e < 16; ++e) m[e] = c_scale(P.mats[16 * slot + e], ch.inv);
        const unsigned pl = min(op.q[0], op.q[1]), ph = max(op.q[0], op.q[1]);
        const uint64_t d0 = uint64_t{1} << op.q[0], d1 = uint64_t{1} << op.q[1];
        const uint64_t b = insert_zero(insert_zero(p, pl), ph);
        const double2 v[4] = {a[b], a[b | d0], a[b | d1], a[b | d0 | d1]};
        a[b] = row_apply<4>(m, cls, 0, v);
        a[b | d0] = row_apply<4>(m, cls, 1, v);
        a[b | d1] = row_apply<4>(m, cls, 2, v);
        a[b | d0 | d1] = row_apply<4>(m, cls, 3, v);
      }
    } else {  // measure / reset collapse (+ X-fix)
      const uint64_t off = scatter_bits(ch.key, op.q, op.nq);
      const uint64_t xfix = op.kind == K_RESET ? off : 0;
      const double2 zero = make_double2(0.0, 0.0);
      if (xfix == 0) {
        for (int h = 0; h < 2; ++h) {
          const uint64_t j = 2 * p + h;
          a[j] = ((j & qmask) == off) ? c_scale(a[j], ch.inv) : zero;
        }
      } else {
        const unsigned xmax = 63 - __clzll(xfix);
        const uint64_t i0 = insert_zero(p, xmax), i1 = i0 ^ xfix;
        const double2 a0 = a[i0], a1 = a[i1];
        a[i0] = ((i1 & qmask) == off) ? c_scale(a1, ch.inv) : zero;
        a[i1] = ((i0 & qmask) == off) ? c_scale(a0, ch.inv) : zero;
      }
    }
  }
}

// Leaf cumulative over all sampled outcomes (groups = 1 case): one WARP per
// leaf builds the reference's sequential cumulative (exec_branch.cpp:267-276
// -> pick_outcome's order) bit-exactly with the warp-parallel exact scan
// (exact_scan.cuh); last[] = last nonzero outcome (count: none).
__global__ void b_leaf_cum_full(ProgView P, const double2* pool, const DevNode* leaves, uint64_t nl, double* cum,
                                uint64_t* last) {
  const uint64_t l = (uint64_t{blockIdx.x} * blockDim.x + threadIdx.x) / 32;
  if (l >= nl) return;  // whole warps exit together
  const unsigned n = P.n;
  const double2* a = pool + (uint64_t{leaves[l].slot} << n);
  const uint64_t count = uint64_t{1} << P.nsample;
  double* out = cum + l * count;
  const bool ident = P.sample_identity;
  const ExactPick r = warp_exact_scan(
      [&](uint64_t m) { return c_norm(a[ident ? m : scatter_bits(m, P.sample_qubits, P.nsample)]); }, count, HUGE_VAL,
      [&](uint64_t m, double v) { out[m] = v; });
  if ((threadIdx.x & 31) == 0) last[l] = r.any_nonzero ? r.outcome : count;
}

// Same from precomputed probabilities (k < n sampled qubits).
__global__ void b_leaf_cum_probs(const double* probs, uint64_t nl, uint64_t count, double* cum, uint64_t* last) {
  const uint64_t l = (uint64_t{blockIdx.x} * blockDim.x + threadIdx.x) / 32;
  if (l >= nl) return;
  const double* pr = probs + l * count;
  double* out = cum + l * count;
  const ExactPick r = warp_exact_scan([&](uint64_t m) { return pr[m]; }, count, HUGE_VAL,
                                      [&](uint64_t m, double v) { out[m] = v; });
  if ((threadIdx.x & 31) == 0) last[l] = r.any_nonzero ? r.outcome : count;
}

__global__ void b_leaf_values(ProgView P, const DevNode* leaves, uint64_t nl, const uint64_t* shots, uint64_t total,
                              uint64_t seed, const double* cum, const uint64_t* last, uint64_t count,
                              uint64_t shot_begin, uint64_t* values, int* err) {
  const uint64_t pos = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (pos >= total) return;
  const uint64_t l = node_of(leaves, nl, pos);
  const uint64_t shot = shots[pos];
  uint64_t v = leaves[l].creg;
  if (cum) {
    const double u = keyed_uniform(seed, shot, P.num_events);
    const double* c = cum + l * count;
    uint64_t lo = 0, hi = count;  // first m with u < c[m]
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (u < c[mid]) hi = mid;
      else lo = mid + 1;
    }
    uint64_t o = lo;
    if (lo == count) {
      o = last[l];
      if (o == count) {
        raise(err, DEV_DEGENERATE);
        o = 0;
      }
    }
    v = apply_sample_outcome(P, v, o);
  }
  values[shot - shot_begin] = v;
}

namespace {

unsigned gridn(uint64_t work, unsigned threads = NT) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((work + threads - 1) / threads, 1u << 30)));
}

struct HostNode {
  uint32_t slot;
  uint64_t off, len;
  uint64_t creg;
};

template <class T>
struct DBuf {  // named view of a persistent grow-only engine buffer
  const EngineView* E;
  const char* name;
  T* get(size_t n) { return static_cast<T*>(E->scratch(E->ctx, name, std::max<size_t>(n, 1) * sizeof(T))); }
};

// Per new live node after a site (materialize + advance_node fused, for states
// that fit shared memory): apply the child's decision — Pauli term, scaled
// Kraus matrix, or collapse (+ creg / X-fix), exec_branch.cpp:104-136 — then
// the gate run up to the next site, with one HBM read + write of the state.
struct ChildRun {
  uint32_t slot;
  uint32_t key;
  double inv;
  uint64_t creg;     // register after the decision (gate conditions)
  uint32_t has_kid;  // transform the state (else gates only)
  uint32_t pad;
};

// A node's state HBM -> shared memory with asynchronous 16-byte copies
// (LDGSTS): every element of the thread in flight at once instead of a
// dependent load / store loop (ncu: long-scoreboard stalls dominated).
__device__ __forceinline__ void load_state_async(double2* st, const double2* g, uint64_t A) {
  const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(st));
  for (uint64_t j = threadIdx.x; j < A; j += NT)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + static_cast<uint32_t>(16 * j)), "l"(g + j));
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__global__ void __launch_bounds__(NT) b_child_run_kernel(ProgView P, DevOp site, double2* pool, const ChildRun* nodes,
                                                         uint64_t nn, unsigned n, uint32_t g_begin, uint32_t g_end,
                                                         int has_gates) {
  extern __shared__ double2 st[];
  const uint64_t A = uint64_t{1} << n;
  for (uint64_t x = blockIdx.x; x < nn; x += gridDim.x) {
    const ChildRun c = nodes[x];
    if (!c.has_kid && !has_gates) continue;
    double2* g = pool + (uint64_t{c.slot} << n);
    load_state_async(st, g, A);
    __syncthreads();
    if (c.has_kid) {
      if (site.kind == K_PAULI) {
        const DevTerm tm = P.terms[site.aux + c.key];
        cta_pauli(st, n, tm.x, tm.z, tm.num_y);
      } else if (site.kind == K_KRAUS) {
        const DevChannel chn = P.channels[site.aux];
        const uint32_t slot = chn.mat_begin + c.key;
        const uint64_t cls = P.scaled_cls[slot];
        if (chn.arity == 1) {
          double2 m[4];
          for (int e = 0; e < 4; ++e) m[e] = c_scale(P.mats[16 * slot + e], c.inv);
          cta_apply1(st, n, site.q[0], m, cls);
        } else {
          double2 m[16];
          for (int e = 0; e < 16; ++e) m[e] = c_scale(P.mats[16 * slot + e], c.inv);
          cta_apply2(st, n, site.q[0], site.q[1], m, cls);
        }
      } else {
        uint64_t qmask = 0;
        for (unsigned b = 0; b < site.nq; ++b) qmask |= uint64_t{1} << site.q[b];
        const uint64_t off = scatter_bits(c.key, site.q, site.nq);
        cta_collapse(st, n, qmask, off, c.inv, site.kind == K_RESET ? off : 0);
      }
      __syncthreads();
    }
    for (uint32_t i = g_begin; i < g_end; ++i) {
      const DevOp& op = P.ops[i];
      if (op.kind != K_GATE || op.skip) continue;
      if (op.has_cond && (c.creg & op.cond_mask) != op.cond_value) continue;
      if (op.nq == 1) {
        double2 m[4];
        load_matrix<2>(P.mats + 16 * op.aux, m);
        cta_apply1(st, n, op.q[0], m, op.cls);
      } else {
        double2 m[16];
        load_matrix<4>(P.mats + 16 * op.aux, m);
        cta_apply2(st, n, op.q[0], op.q[1], m, op.cls);
      }
      __syncthreads();
    }
    for (uint64_t j = threadIdx.x; j < A; j += NT) g[j] = st[j];
    __syncthreads();
  }
}

// Device planner for a site whose nonzero groups all fit the budget (the
// common case): every group becomes a child in (parent, key) order
// (exec_branch.cpp:141-153). A parent's first child keeps its slot; the r-th
// other child (r = g - parent - 1, every parent owning >= 1 group) takes a
// recycled slot or a fresh one. Shot offsets are the exclusive scan of the
// group counts. Emits the next live table, each child's decision record for
// the fused child run, and the copy source of non-first children.
__global__ void b_plan_kernel(ProgView P, DevOp site, const DevNode* nodes, const uint32_t* sel, const unsigned* gcnt,
                              const double* gval, const unsigned* goff, uint64_t ng, uint32_t nkeys,
                              const uint32_t* free_list, uint32_t nfree, uint32_t next_slot, DevNode* next_nodes,
                              ChildRun* runs, uint32_t* copy_src, uint64_t* gdst, int* err) {
  const uint64_t g = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const uint32_t cell = sel[g], x = cell / nkeys, key = cell % nkeys;
  const bool first = g == 0 || sel[g - 1] / nkeys != x;
  const DevNode par = nodes[x];
  uint32_t slot = par.slot, src = 0xFFFFFFFFu;
  if (!first) {
    const uint32_t r = static_cast<uint32_t>(g) - x - 1;
    slot = r < nfree ? free_list[nfree - 1 - r] : next_slot + (r - nfree);
    src = par.slot;
  }
  uint64_t creg = par.creg;
  const bool transform = par.cond_ok && !(site.kind == K_PAULI && P.terms[site.aux + key].identity);
  double inv = 1.0;
  if (transform && site.kind != K_PAULI) {
    const double p = gval[g];
    if (!(p > 0.0)) raise(err, DEV_DEGENERATE);
    else inv = __ddiv_rn(1.0, __dsqrt_rn(p));
  }
  if (transform && site.kind == K_MEASURE)
    for (unsigned b = 0; b < site.nq; ++b)
      creg = (creg & ~(uint64_t{1} << site.c[b])) | (((uint64_t{key} >> b) & 1) << site.c[b]);
  next_nodes[g] = DevNode{slot, 1u, goff[g], gcnt[g], creg};
  runs[g] = ChildRun{slot, key, inv, creg, transform ? 1u : 0u, 0u};
  copy_src[g] = src;
  gdst[g] = goff[g];
}

// Non-first children copy their parent's state before any decision is applied.
__global__ void b_copy_children(double2* pool, const uint32_t* copy_src, const DevNode* next_nodes, uint64_t ng,
                                unsigned n) {
  const uint64_t A = uint64_t{1} << n;
  for (uint64_t g = blockIdx.x; g < ng; g += gridDim.x) {
    const uint32_t src = copy_src[g];
    if (src == 0xFFFFFFFFu) continue;
    const double2* a = pool + (uint64_t{src} << n);
    double2* b = pool + (uint64_t{next_nodes[g].slot} << n);
    for (uint64_t j = threadIdx.x; j < A; j += blockDim.x) b[j] = a[j];
  }
}

// Live-table fields for the gate / reduction kernels (device-resident table).
__global__ void b_node_fields(DevNode* nodes, uint64_t nn, DevOp site, int set_cond, uint32_t* slots, uint64_t* cregs,
                              uint8_t* active) {
  const uint64_t x = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (x >= nn) return;
  DevNode& d = nodes[x];
  if (set_cond) d.cond_ok = !site.has_cond || (d.creg & site.cond_mask) == site.cond_value ? 1u : 0u;
  if (slots) slots[x] = d.slot;
  if (cregs) cregs[x] = d.creg;
  if (active) active[x] = static_cast<uint8_t>(d.cond_ok);
}

// Nonzero (node, key) groups, compacted in (node, key) order (b_scan_*): gather
// their counts and node-level parameters for the host planner.
__global__ void b_gather_groups(const uint32_t* sel, const unsigned* num, const unsigned* counts, const double* vals,
                                unsigned* out_cnt, double* out_val) {
  const unsigned j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *num) return;
  out_cnt[j] = counts[sel[j]];
  if (vals) out_val[j] = vals[sel[j]];
}

// ---- Order-preserving compaction and exclusive scan of the branch tables
// (three small kernels; no library kernels on the branch hot path).
// Flag = true: out[k] = i for the k-th i with in[i] != 0 (cells of nonzero
// (node, key) groups, in (node, key) order), *sum = their number.
// Flag = false: out[i] = in[0] + ... + in[i-1] (shot offsets), *sum = total.
constexpr unsigned kScanPer = 4, kScanItems = NT * kScanPer;

template <bool Flag>
__device__ __forceinline__ unsigned scan_val(const unsigned* in, uint64_t i, uint64_t count) {
  if (i >= count) return 0;
  return Flag ? (in[i] != 0 ? 1u : 0u) : in[i];
}

// Exclusive scan of one value per thread over the CTA; returns the CTA total.
__device__ __forceinline__ unsigned cta_exclusive_scan(unsigned v, unsigned* prefix_out) {
  __shared__ unsigned warp_tot[NT / 32];
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= static_cast<unsigned>(off)) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  unsigned base = 0, total = 0;
  for (unsigned w = 0; w < NT / 32; ++w) {
    if (w < wid) base += warp_tot[w];
    total += warp_tot[w];
  }
  __syncthreads();  // warp_tot is reused by the next call
  *prefix_out = base + x - v;
  return total;
}

template <bool Flag>
__global__ void __launch_bounds__(NT) b_scan_totals(const unsigned* in, uint64_t count, unsigned* totals) {
  const uint64_t first = uint64_t{blockIdx.x} * kScanItems + threadIdx.x * kScanPer;
  unsigned v = 0;
#pragma unroll
  for (unsigned r = 0; r < kScanPer; ++r) v += scan_val<Flag>(in, first + r, count);
  unsigned prefix;
  const unsigned tot = cta_exclusive_scan(v, &prefix);
  if (threadIdx.x == 0) totals[blockIdx.x] = tot;
}

// One CTA: totals[] -> exclusive offsets in place; *sum = grand total.
__global__ void __launch_bounds__(NT) b_scan_top(unsigned* totals, uint32_t nblk, unsigned* sum) {
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t c0 = 0; c0 < nblk; c0 += NT) {
    const uint32_t i = c0 + threadIdx.x;
    const unsigned v = i < nblk ? totals[i] : 0;
    unsigned prefix;
    const unsigned tot = cta_exclusive_scan(v, &prefix);
    const unsigned base = carry;
    if (i < nblk) totals[i] = base + prefix;
    __syncthreads();
    if (threadIdx.x == 0) carry = base + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *sum = carry;
}

template <bool Flag>
__global__ void __launch_bounds__(NT) b_scan_apply(const unsigned* in, uint64_t count, const unsigned* offs,
                                                   unsigned* out) {
  const uint64_t first = uint64_t{blockIdx.x} * kScanItems + threadIdx.x * kScanPer;
  unsigned v[kScanPer], t = 0;
#pragma unroll
  for (unsigned r = 0; r < kScanPer; ++r) {
    v[r] = scan_val<Flag>(in, first + r, count);
    t += v[r];
  }
  unsigned prefix;
  cta_exclusive_scan(t, &prefix);
  unsigned pos = offs[blockIdx.x] + prefix;
#pragma unroll
  for (unsigned r = 0; r < kScanPer; ++r) {
    const uint64_t i = first + r;
    if (i >= count) break;
    if (Flag) {
      if (v[r]) out[pos] = static_cast<unsigned>(i);
    } else {
      out[i] = pos;
    }
    pos += v[r];
  }
}

// Dense destination table from the planner's per-group destinations.
__global__ void b_set_dst(const uint32_t* sel, const uint64_t* gdst, uint64_t ng, uint64_t* dst) {
  const uint64_t j = uint64_t{blockIdx.x} * blockDim.x + threadIdx.x;
  if (j < ng) dst[sel[j]] = gdst[j];
}

// advance_node for every live node in one launch when a state fits shared
// memory (n <= 13): one CTA per node loads its state once, applies the gate
// run [op_begin, op_end) in place (reference per-gate arithmetic,
// kernels_scalar.cpp:24-56; conditions against the node's register) and
// stores it once — instead of one HBM sweep of every node per gate.
__global__ void __launch_bounds__(NT) b_gate_run_kernel(ProgView P, double2* pool, const uint32_t* slots,
                                                        const uint64_t* cregs, uint64_t nn, unsigned n,
                                                        uint32_t op_begin, uint32_t op_end) {
  extern __shared__ double2 st[];
  const uint64_t A = uint64_t{1} << n;
  for (uint64_t x = blockIdx.x; x < nn; x += gridDim.x) {
    double2* g = pool + (uint64_t{slots[x]} << n);
    load_state_async(st, g, A);
    __syncthreads();
    const uint64_t creg = cregs[x];
    for (uint32_t i = op_begin; i < op_end; ++i) {
      const DevOp& op = P.ops[i];
      if (op.kind != K_GATE || op.skip) continue;
      if (op.has_cond && (creg & op.cond_mask) != op.cond_value) continue;
      if (op.nq == 1) {
        double2 m[4];
        load_matrix<2>(P.mats + 16 * op.aux, m);
        cta_apply1(st, n, op.q[0], m, op.cls);
      } else {
        double2 m[16];
        load_matrix<4>(P.mats + 16 * op.aux, m);
        cta_apply2(st, n, op.q[0], op.q[1], m, op.cls);
      }
      __syncthreads();
    }
    for (uint64_t j = threadIdx.x; j < A; j += NT) g[j] = st[j];
    __syncthreads();
  }
}

}  // namespace

void run_branch_device(EngineView& E, const ProgView& P, const HostDevProgram& h, uint64_t shot_begin,
                       uint64_t count, uint64_t seed, const ssb_run_options* opts, uint64_t* values_dev,
                       ssb_stats* stats, uint64_t mem_limit_bytes) {
  const uint64_t budget = opts ? opts->branch_budget : 64;
  if (budget < 1) throw std::invalid_argument("branch budget must be >= 1");
  if (count < 1) throw std::invalid_argument("shots must be >= 1");
  cudaStream_t s = E.stream;
  const unsigned n = h.n;
  const uint64_t A = uint64_t{1} << n, seg = A * sizeof(double2);
  const uint64_t launches0 = *E.launches;
  auto launched = [&] {
    ++*E.launches;
    CKB(cudaGetLastError());
  };

  // Slot pool: live states never exceed min(budget, shots) (+1 transient root).
  const uint64_t max_slots = std::min<uint64_t>(budget, count) + 1;
  if (max_slots * seg > mem_limit_bytes)
    throw shotsim::CapacityError("branch budget of " + std::to_string(budget) + " states at " + std::to_string(n) +
                                 " qubits needs " + std::to_string(max_slots * seg) + " bytes");
  // The pool lives in the engine across runs (grown by doubling, contents
  // preserved), so repeated runs never reallocate.
  // Reserve the whole bound up front when it is at most half the memory
  // limit (no growth copies inside the run); otherwise start small and double.
  uint64_t pool_cap = max_slots * seg <= mem_limit_bytes / 2 ? max_slots : std::min<uint64_t>(max_slots, 64);
  double2* pool = static_cast<double2*>(E.grow(E.ctx, "branch.pool", pool_cap * seg, 0));
  std::vector<uint32_t> free_slots;
  uint32_t next_slot = 0;
  auto alloc_slot = [&]() -> uint32_t {
    if (!free_slots.empty()) {
      const uint32_t sl = free_slots.back();
      free_slots.pop_back();
      return sl;
    }
    if (next_slot >= pool_cap) {  // grow (rare): copy live slots over
      const uint64_t ncap = std::min<uint64_t>(max_slots, pool_cap * 2);
      if (ncap <= pool_cap) throw std::logic_error("branch slot pool exhausted");
      pool = static_cast<double2*>(E.grow(E.ctx, "branch.pool", ncap * seg, pool_cap * seg));
      pool_cap = ncap;
    }
    return next_slot++;
  };

  std::vector<HostNode> live;
  DBuf<uint64_t> shots_a{&E, "branch.shots_a"}, shots_b{&E, "branch.shots_b"}, waiting_buf{&E, "branch.waiting"};
  uint64_t* cur_shots = shots_a.get(count);
  uint64_t* nxt_shots = shots_b.get(count);
  uint64_t* waiting = waiting_buf.get(count);
  b_iota<<<gridn(count), NT, 0, s>>>(waiting, shot_begin, count);
  launched();
  uint64_t nwaiting = count;

  DBuf<DevNode> dnodes{&E, "branch.nodes"};
  DBuf<uint32_t> dkeys{&E, "branch.keys"}, dslots{&E, "branch.slots"};
  DBuf<unsigned> dcounts{&E, "branch.counts"};
  DBuf<uint64_t> ddst{&E, "branch.dst"}, dlast{&E, "branch.last"}, dcreg{&E, "branch.creg"};
  DBuf<unsigned long long> dcursor{&E, "branch.cursor"};
  DBuf<double> dvals{&E, "branch.vals"}, dpart{&E, "branch.part"}, dcum{&E, "branch.cum"};
  DBuf<uint2> dpairs{&E, "branch.pairs"};
  DBuf<ChildOp> dkids{&E, "branch.kids"};
  DBuf<ChildRun> dchildrun{&E, "branch.childrun"};
  DBuf<uint8_t> dactive{&E, "branch.active"};
  DBuf<uint32_t> dsel{&E, "branch.sel"};
  DBuf<unsigned> dnumsel{&E, "branch.numsel"}, dgcnt{&E, "branch.gcnt"};
  DBuf<double> dgval{&E, "branch.gval"};
  DBuf<uint64_t> dgdst{&E, "branch.gdst"};
  DBuf<DevNode> dlive_a{&E, "branch.live_a"}, dlive_b{&E, "branch.live_b"};
  DBuf<unsigned> dgoff{&E, "branch.goff"};
  DBuf<uint32_t> dcopysrc{&E, "branch.copysrc"}, dfree{&E, "branch.free"};
  // The live table is device-resident while sites are planned on the device
  // (no budget overflow); the host copy `live` is refreshed only for the
  // overflow planner and the leaves.
  bool live_on_host = true;
  DevNode* dlive = nullptr;
  uint64_t nn_dev = 0, total_live = 0;
  auto live_to_host = [&](DevNode* staging) {
    CKB(cudaMemcpyAsync(staging, dlive, nn_dev * sizeof(DevNode), cudaMemcpyDeviceToHost, s));
    CKB(cudaStreamSynchronize(s));
    live.resize(nn_dev);
    for (uint64_t x = 0; x < nn_dev; ++x) live[x] = HostNode{staging[x].slot, staging[x].off, staging[x].len, staging[x].creg};
    live_on_host = true;
  };
  DBuf<unsigned> dscantot{&E, "branch.scantot"}, dscansum{&E, "branch.scansum"};

  // Size every per-site table once for the run's worst case (live nodes <=
  // max_slots, keys per node <= the largest site fan-out), so the site loop
  // never reallocates (each growth would synchronise the device).
  {
    uint64_t max_keys = 1;
    for (uint32_t k = 0; k < h.end; ++k) {
      const DevOp& o = h.ops[k];
      if (o.kind == K_PAULI) max_keys = std::max<uint64_t>(max_keys, o.count);
      else if (o.kind == K_KRAUS) max_keys = std::max<uint64_t>(max_keys, h.channels[o.aux].nmat);
      else if (o.kind == K_MEASURE || o.kind == K_RESET) max_keys = std::max<uint64_t>(max_keys, uint64_t{1} << o.nq);
    }
    const uint64_t nodes_max = max_slots, cells = nodes_max * max_keys;
    dnodes.get(nodes_max);
    dlive_a.get(nodes_max);
    dlive_b.get(nodes_max);
    dslots.get(nodes_max);
    dcreg.get(nodes_max);
    dactive.get(nodes_max);
    dchildrun.get(cells);
    dcopysrc.get(cells);
    dgdst.get(cells);
    dgoff.get(cells);
    dsel.get(cells);
    dgcnt.get(cells);
    dgval.get(cells);
    dcounts.get(cells);
    ddst.get(cells);
    dcursor.get(cells);
    dkeys.get(count);
  }
  // SHOTSIM_B200_BRANCH_HOST_PLAN=1: plan every site on the host (A/B tests).
  const bool device_plan = [] {
    const char* v = std::getenv("SHOTSIM_B200_BRANCH_HOST_PLAN");
    return !(v && *v && *v != '0');
  }();
  // Node-resident gate runs when a state fits shared memory.
  int smem_optin = 0, dev = 0;
  CKB(cudaGetDevice(&dev));
  CKB(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const uint64_t gate_run_smem_max = static_cast<uint64_t>(smem_optin);
  if (seg <= gate_run_smem_max) {
    CKB(cudaFuncSetAttribute(b_gate_run_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(seg)));
    CKB(cudaFuncSetAttribute(b_child_run_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(seg)));
  }
  // SHOTSIM_B200_BRANCH_TRACE=1: per-phase host wall time (sync points) to stderr.
  const bool tracing = [] {
    const char* v = std::getenv("SHOTSIM_B200_BRANCH_TRACE");
    return v && *v && *v != '0';
  }();
  std::map<std::string, double> trace_t;
  auto trace_last = std::chrono::steady_clock::now();
  auto trace_mark = [&](const char* tag) {  // host-only phase boundary
    if (!tracing) return;
    const auto now = std::chrono::steady_clock::now();
    trace_t[tag] += std::chrono::duration<double>(now - trace_last).count();
    trace_last = now;
  };
  auto trace_sync = [&](const char* tag) {
    CKB(cudaStreamSynchronize(s));
    if (!tracing) return;
    const auto now = std::chrono::steady_clock::now();
    trace_t[tag] += std::chrono::duration<double>(now - trace_last).count();
    trace_last = now;
  };
  // Pinned staging for every host->device table (async copies, no pageable
  // bounce); each name is rewritten only after the next stream sync.
  auto pinned = [&](const char* name, size_t count, auto* type_tag) {
    using T = std::remove_pointer_t<decltype(type_tag)>;
    return static_cast<T*>(E.host(E.ctx, name, std::max<size_t>(count, 1) * sizeof(T)));
  };
  uint64_t peak = 0, passes = 0, num_leaves = 0;
  // Planner work arrays, reused across sites (no per-site allocation).
  struct Cand {
    uint64_t parent;
    uint32_t key;
    uint64_t count;
    double val;
  };
  std::vector<Cand> groups;
  std::vector<uint8_t> keep, parent_used, parent_kept;
  std::vector<uint2> pairs;
  std::vector<ChildOp> kids;
  while (nwaiting > 0) {
    ++passes;
    std::swap(cur_shots, waiting);  // waiting list becomes this pass's root
    const uint64_t root_len = nwaiting;
    nwaiting = 0;
    free_slots.clear();
    next_slot = 0;
    live.assign(1, HostNode{alloc_slot(), 0, root_len, 0});
    live_on_host = true;
    total_live = root_len;
    b_init_slot<<<gridn(A), NT, 0, s>>>(pool, live[0].slot, n);
    launched();
    peak = std::max<uint64_t>(peak, 1);

    uint32_t i = 0;
    bool gates_done = false;  // the previous site's child run already applied ops [i, j)
    while (i < h.end) {
      uint32_t j = i;
      auto is_site = [&](uint32_t k) {
        const uint8_t kd = h.ops[k].kind;
        return kd == K_PAULI || kd == K_KRAUS || kd == K_MEASURE || kd == K_RESET;
      };
      while (j < h.end && !is_site(j)) ++j;
      const uint64_t nn = live_on_host ? live.size() : nn_dev;
      // advance_node (exec_branch.cpp:155-162): gates over all live nodes.
      if (j > i && !gates_done) {
        uint32_t* slots = dslots.get(nn);
        uint64_t* cregs = dcreg.get(nn);
        if (live_on_host) {
          uint32_t* hs = pinned("branch.h_gslots", nn, (uint32_t*)nullptr);
          uint64_t* hc = pinned("branch.h_gcregs", nn, (uint64_t*)nullptr);
          for (uint64_t x = 0; x < nn; ++x) {
            hs[x] = live[x].slot;
            hc[x] = live[x].creg;
          }
          CKB(cudaMemcpyAsync(slots, hs, nn * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
          CKB(cudaMemcpyAsync(cregs, hc, nn * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        } else {
          b_node_fields<<<gridn(nn), NT, 0, s>>>(dlive, nn, h.ops[i], 0, slots, cregs, nullptr);
          launched();
        }
        uint32_t ngates = 0;
        for (uint32_t k = i; k < j; ++k) ngates += h.ops[k].kind == K_GATE && !h.ops[k].skip;
        if (ngates > 1 && seg <= gate_run_smem_max) {
          b_gate_run_kernel<<<static_cast<unsigned>(std::min<uint64_t>(nn, 1u << 20)), NT, seg, s>>>(
              P, pool, slots, cregs, nn, n, i, j);
          launched();
        } else {
          for (uint32_t k = i; k < j; ++k) {
            const DevOp& op = h.ops[k];
            if (op.kind != K_GATE || op.skip) continue;
            const uint64_t work = nn << (n - op.nq);
            if (op.nq == 1) g_gate_kernel<1><<<gridn(work), NT, 0, s>>>(pool, nn, n, op, P.mats, cregs, slots);
            else g_gate_kernel<2><<<gridn(work), NT, 0, s>>>(pool, nn, n, op, P.mats, cregs, slots);
            launched();
          }
        }
        trace_sync("gates");  // host vectors hs/hc die here
      }
      gates_done = false;
      if (j == h.end) break;
      const DevOp site = h.ops[j];

      // Node table with condition flags.
      DevNode* hn = nullptr;  // host copy (host-planned sites only)
      DevNode* nodes = nullptr;
      if (live_on_host) {
        hn = pinned("branch.h_nodes", nn, (DevNode*)nullptr);
        for (uint64_t x = 0; x < nn; ++x)
          hn[x] = {live[x].slot, !site.has_cond || (live[x].creg & site.cond_mask) == site.cond_value ? 1u : 0u,
                   live[x].off, live[x].len, live[x].creg};
        nodes = dnodes.get(nn);
        CKB(cudaMemcpyAsync(nodes, hn, nn * sizeof(DevNode), cudaMemcpyHostToDevice, s));
      } else {
        nodes = dlive;
        b_node_fields<<<gridn(nn), NT, 0, s>>>(nodes, nn, site, 1, nullptr, nullptr, nullptr);
        launched();
      }

      uint32_t nkeys = 1;
      double* vals = nullptr;
      if (site.kind == K_PAULI) {
        nkeys = site.count;
      } else {
        // Node-level quantities on the shared states (computed once per node).
        RedSpec R{};
        R.n = n;
        int tree = 0;
        if (site.kind == K_KRAUS) {
          const DevChannel ch = h.channels[site.aux];
          nkeys = ch.nmat;
          R.k = ch.arity;
          for (unsigned b = 0; b < ch.arity; ++b) R.q[b] = R.sorted[b] = site.q[b];
          std::sort(R.sorted, R.sorted + ch.arity);
          R.nq = ch.nmat;
          R.mats = P.mats + 16 * ch.mat_begin;
      R.cls = P.scaled_cls + ch.mat_begin;
          if (ch.arity == 1) {
            R.mode = R_EXPVAL1;
            const uint64_t pairs = A / 2;
            R.nb = pairs <= SUM_BLOCK ? 1 : pairs / SUM_BLOCK;
            R.blk = pairs <= SUM_BLOCK ? pairs : SUM_BLOCK;
          } else {
            R.mode = R_EXPVAL2;
            const uint64_t G = A / 4;
            R.blk = G <= 8 ? G : 8;
            R.nb = G / R.blk;
            tree = 1;
          }
        } else {
          R.mode = R_OUTCOME;
          R.k = site.nq;
          for (unsigned b = 0; b < site.nq; ++b) R.q[b] = R.sorted[b] = site.q[b];
          std::sort(R.sorted, R.sorted + site.nq);
          const uint64_t G = A >> site.nq;
          R.nq = 1u << site.nq;
          R.nb = G <= SUM_BLOCK ? 1 : G / SUM_BLOCK;
          R.blk = G <= SUM_BLOCK ? G : SUM_BLOCK;
          nkeys = R.nq;
        }
        uint32_t* slots = dslots.get(nn);
        uint8_t* active = dactive.get(nn);
        if (live_on_host) {
          uint32_t* hs = pinned("branch.h_rslots", nn, (uint32_t*)nullptr);
          uint8_t* ha = pinned("branch.h_ractive", nn, (uint8_t*)nullptr);
          for (uint64_t x = 0; x < nn; ++x) {
            hs[x] = live[x].slot;
            ha[x] = static_cast<uint8_t>(hn[x].cond_ok);
          }
          CKB(cudaMemcpyAsync(slots, hs, nn * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
          CKB(cudaMemcpyAsync(active, ha, nn, cudaMemcpyHostToDevice, s));
        } else {
          b_node_fields<<<gridn(nn), NT, 0, s>>>(nodes, nn, site, 0, slots, nullptr, active);
          launched();
        }
        double* part = dpart.get(nn * R.nq * R.nb);
        vals = dvals.get(nn * R.nq);
        launch_reduce(s, pool, nn, R, active, part, slots);
        launched();
        g_finish_kernel<<<static_cast<unsigned>(std::min<uint64_t>(nn * R.nq, 1u << 20)), NT, 0, s>>>(nn, R.nq, R.nb, tree, active, part, vals);
        launched();
        trace_sync("reduce");
      }

      // Per-shot decisions and group counts.
      const uint64_t total = total_live;
      uint32_t* keys = dkeys.get(total);
      unsigned* counts = dcounts.get(nn * nkeys);
      CKB(cudaMemsetAsync(counts, 0, nn * nkeys * sizeof(unsigned), s));
      b_decide<<<gridn(total), NT, 0, s>>>(P, site, nodes, nn, cur_shots, total, seed, vals, nkeys, keys, counts,
                                           E.err);
      launched();
      // Compact the nonzero groups on the device; only they cross to the host.
      const uint64_t ncells = nn * nkeys;
      if (ncells >= (uint64_t{1} << 32)) throw std::length_error("branch group table too large");
      uint32_t* sel = dsel.get(ncells);
      unsigned* dnum = dnumsel.get(1);
      {  // sel = the nonzero cells in order, *dnum = their number
        const uint32_t nblk = static_cast<uint32_t>((ncells + kScanItems - 1) / kScanItems);
        unsigned* tot = dscantot.get(nblk);
        b_scan_totals<true><<<nblk, NT, 0, s>>>(counts, ncells, tot);
        launched();
        b_scan_top<<<1, NT, 0, s>>>(tot, nblk, dnum);
        launched();
        b_scan_apply<true><<<nblk, NT, 0, s>>>(counts, ncells, tot, sel);
        launched();
      }
      unsigned* gcnt = dgcnt.get(ncells);
      double* gval = vals ? dgval.get(ncells) : nullptr;
      b_gather_groups<<<gridn(ncells), NT, 0, s>>>(sel, dnum, counts, vals, gcnt, gval);
      launched();
      unsigned* hnum = static_cast<unsigned*>(E.host(E.ctx, "branch.hnum", sizeof(unsigned)));
      CKB(cudaMemcpyAsync(hnum, dnum, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      trace_sync("decide_num");
      const uint64_t ng = *hnum;
      // Next site (end of the gate run that follows this one).
      uint32_t jn = j + 1;
      while (jn < h.end && !is_site(jn)) ++jn;
      bool run_gates = false;
      for (uint32_t k = j + 1; k < jn; ++k) run_gates |= h.ops[k].kind == K_GATE && !h.ops[k].skip;
      if (device_plan && seg <= gate_run_smem_max && ng <= budget && total < (uint64_t{1} << 32)) {
        // Device planner (no budget overflow): the live table never leaves HBM.
        const uint64_t nnew = ng - nn;
        const uint64_t nfree = free_slots.size(), take = std::min<uint64_t>(nnew, nfree);
        const uint64_t need = next_slot + (nnew - take);
        while (need > pool_cap) {
          const uint64_t ncap = std::min<uint64_t>(max_slots, pool_cap * 2);
          if (ncap <= pool_cap) throw std::logic_error("branch slot pool exhausted");
          pool = static_cast<double2*>(E.grow(E.ctx, "branch.pool", ncap * seg, pool_cap * seg));
          pool_cap = ncap;
        }
        uint32_t* dfl = nullptr;
        if (take) {
          uint32_t* hf = pinned("branch.h_free", nfree, (uint32_t*)nullptr);
          std::copy(free_slots.begin(), free_slots.end(), hf);
          dfl = dfree.get(nfree);
          CKB(cudaMemcpyAsync(dfl, hf, nfree * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        }
        unsigned* goff = dgoff.get(ng);
        {  // goff = exclusive prefix sums of the group counts (shot offsets)
          const uint32_t nblk = static_cast<uint32_t>((ng + kScanItems - 1) / kScanItems);
          unsigned* tot = dscantot.get(nblk);
          b_scan_totals<false><<<nblk, NT, 0, s>>>(gcnt, ng, tot);
          launched();
          b_scan_top<<<1, NT, 0, s>>>(tot, nblk, dscansum.get(1));
          launched();
          b_scan_apply<false><<<nblk, NT, 0, s>>>(gcnt, ng, tot, goff);
          launched();
        }
        DevNode* next_tab = (dlive == dlive_a.get(1) ? dlive_b : dlive_a).get(ng);
        ChildRun* runs = dchildrun.get(ng);
        uint32_t* csrc = dcopysrc.get(ng);
        uint64_t* gdst = dgdst.get(ng);
        b_plan_kernel<<<gridn(ng), NT, 0, s>>>(P, site, nodes, sel, gcnt, gval, goff, ng, nkeys, dfl,
                                               static_cast<uint32_t>(take ? nfree : 0), next_slot, next_tab, runs,
                                               csrc, gdst, E.err);
        launched();
        uint64_t* dst = ddst.get(nn * nkeys);
        unsigned long long* cursor = dcursor.get(nn * nkeys);
        b_set_dst<<<gridn(ng), NT, 0, s>>>(sel, gdst, ng, dst);
        launched();
        CKB(cudaMemsetAsync(cursor, 0, nn * nkeys * sizeof(unsigned long long), s));
        b_scatter<<<gridn(total), NT, 0, s>>>(nodes, nn, cur_shots, total, keys, nkeys, dst, cursor, nxt_shots,
                                               waiting);
        launched();
        if (nnew) {
          b_copy_children<<<static_cast<unsigned>(std::min<uint64_t>(ng, 1u << 20)), NT, 0, s>>>(pool, csrc, next_tab,
                                                                                                 ng, n);
          launched();
        }
        b_child_run_kernel<<<static_cast<unsigned>(std::min<uint64_t>(ng, 1u << 20)), NT, seg, s>>>(
            P, site, pool, runs, ng, n, j + 1, jn, run_gates ? 1 : 0);
        launched();
        free_slots.resize(nfree - take);
        next_slot += static_cast<uint32_t>(nnew - take);
        dlive = next_tab;
        nn_dev = ng;
        live_on_host = false;
        peak = std::max<uint64_t>(peak, ng);
        gates_done = true;
        trace_sync("apply_dev");
        std::swap(cur_shots, nxt_shots);
        i = j + 1;
        continue;
      }
      if (!live_on_host) {  // host planner needs the table (and its condition flags)
        hn = pinned("branch.h_nodes_dl", nn, (DevNode*)nullptr);
        live_to_host(hn);
      }
      uint32_t* hsel = static_cast<uint32_t*>(E.host(E.ctx, "branch.hsel", std::max<uint64_t>(ng, 1) * 4));
      unsigned* hgc = static_cast<unsigned*>(E.host(E.ctx, "branch.hgc", std::max<uint64_t>(ng, 1) * 4));
      double* hgv = static_cast<double*>(E.host(E.ctx, "branch.hgv", std::max<uint64_t>(ng, 1) * 8));
      CKB(cudaMemcpyAsync(hsel, sel, ng * 4, cudaMemcpyDeviceToHost, s));
      CKB(cudaMemcpyAsync(hgc, gcnt, ng * 4, cudaMemcpyDeviceToHost, s));
      if (gval) CKB(cudaMemcpyAsync(hgv, gval, ng * 8, cudaMemcpyDeviceToHost, s));
      trace_sync("decide_groups");

      // Groups in (parent, key) order; budget policy (exec_branch.cpp:217-255).
      groups.resize(ng);
      for (uint64_t g = 0; g < ng; ++g)
        groups[g] = {hsel[g] / nkeys, hsel[g] % nkeys, hgc[g], gval ? hgv[g] : 0.0};
      keep.assign(groups.size(), 1);
      if (groups.size() > budget) {
        std::vector<size_t> order(groups.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
          if (groups[a].count != groups[b].count) return groups[a].count > groups[b].count;
          if (groups[a].parent != groups[b].parent) return groups[a].parent < groups[b].parent;
          return groups[a].key < groups[b].key;
        });
        std::fill(keep.begin(), keep.end(), 0);
        for (uint64_t c = 0; c < budget; ++c) keep[order[c]] = 1;
      }
      // Children (materialize, exec_branch.cpp:141-153) and shot destinations.
      std::vector<HostNode> next;
      next.reserve(std::min<uint64_t>(ng, budget));
      uint64_t* hgdst = static_cast<uint64_t*>(E.host(E.ctx, "branch.hgdst", std::max<uint64_t>(ng, 1) * 8));
      pairs.clear();
      kids.clear();
      uint64_t new_off = 0, wait_off = nwaiting;
      // Parents without a kept child die first, so the pool never holds more
      // than `budget` live states (+ the root).
      parent_used.assign(nn, 0);
      parent_kept.assign(nn, 0);
      for (size_t g = 0; g < groups.size(); ++g)
        if (keep[g]) parent_kept[groups[g].parent] = 1;
      for (uint64_t x = 0; x < nn; ++x)
        if (!parent_kept[x]) free_slots.push_back(live[x].slot);
      for (size_t g = 0; g < groups.size(); ++g) {
        const Cand& c = groups[g];
        if (!keep[g]) {
          hgdst[g] = (uint64_t{1} << 63) | wait_off;
          wait_off += c.count;
          continue;
        }
        const HostNode& par = live[c.parent];
        uint32_t slot;
        if (!parent_used[c.parent]) {
          slot = par.slot;
          parent_used[c.parent] = 1;
        } else {
          slot = alloc_slot();
          pairs.push_back(make_uint2(par.slot, slot));
        }
        uint64_t creg = par.creg;
        const bool transform = hn[c.parent].cond_ok &&
                               !(site.kind == K_PAULI && h.terms[site.aux + c.key].identity);
        if (transform) {
          double inv = 1.0;
          if (site.kind != K_PAULI) {
            const double param = c.val;
            if (!(param > 0.0)) throw shotsim::DegenerateDistribution("branch has zero probability");
            inv = 1.0 / std::sqrt(param);
          }
          kids.push_back({slot, c.key, inv});
          if (site.kind == K_MEASURE)
            for (unsigned b = 0; b < site.nq; ++b)
              creg = (creg & ~(uint64_t{1} << site.c[b])) | (((uint64_t{c.key} >> b) & 1) << site.c[b]);
        }
        hgdst[g] = new_off;
        next.push_back({slot, new_off, c.count, creg});
        new_off += c.count;
      }

      uint64_t* dst = ddst.get(nn * nkeys);
      unsigned long long* cursor = dcursor.get(nn * nkeys);
      uint64_t* gdst = dgdst.get(std::max<uint64_t>(ng, 1));
      CKB(cudaMemcpyAsync(gdst, hgdst, ng * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
      b_set_dst<<<gridn(std::max<uint64_t>(ng, 1)), NT, 0, s>>>(sel, gdst, ng, dst);
      launched();
      CKB(cudaMemsetAsync(cursor, 0, nn * nkeys * sizeof(unsigned long long), s));
      b_scatter<<<gridn(total), NT, 0, s>>>(nodes, nn, cur_shots, total, keys, nkeys, dst, cursor, nxt_shots, waiting);
      launched();
      if (!pairs.empty()) {
        uint2* dp = dpairs.get(pairs.size());
        uint2* hp = pinned("branch.h_pairs", pairs.size(), (uint2*)nullptr);
        std::copy(pairs.begin(), pairs.end(), hp);
        CKB(cudaMemcpyAsync(dp, hp, pairs.size() * sizeof(uint2), cudaMemcpyHostToDevice, s));
        b_copy_slots<<<gridn(pairs.size() * A), NT, 0, s>>>(pool, dp, pairs.size(), n);
        launched();
      }
      trace_mark("plan_host");
      if (seg <= gate_run_smem_max) {
        // Fused: each new live node's decision + the following gate run.
        ChildRun* hr = pinned("branch.h_childrun", next.size(), (ChildRun*)nullptr);
        size_t kidx = 0;
        for (size_t x = 0; x < next.size(); ++x) {
          hr[x] = ChildRun{next[x].slot, 0, 0.0, next[x].creg, 0, 0};
          if (kidx < kids.size() && kids[kidx].slot == next[x].slot) {
            hr[x].key = kids[kidx].key;
            hr[x].inv = kids[kidx].inv;
            hr[x].has_kid = 1;
            ++kidx;
          }
        }
        if (!next.empty() && (run_gates || !kids.empty())) {
          ChildRun* dr = dchildrun.get(next.size());
          CKB(cudaMemcpyAsync(dr, hr, next.size() * sizeof(ChildRun), cudaMemcpyHostToDevice, s));
          b_child_run_kernel<<<static_cast<unsigned>(std::min<uint64_t>(next.size(), 1u << 20)), NT, seg, s>>>(
              P, site, pool, dr, next.size(), n, j + 1, jn, run_gates ? 1 : 0);
          launched();
        }
        gates_done = true;
      } else if (!kids.empty()) {
        ChildOp* dk = dkids.get(kids.size());
        ChildOp* hk = pinned("branch.h_kids", kids.size(), (ChildOp*)nullptr);
        std::copy(kids.begin(), kids.end(), hk);
        CKB(cudaMemcpyAsync(dk, hk, kids.size() * sizeof(ChildOp), cudaMemcpyHostToDevice, s));
        b_apply<<<gridn(kids.size() * (A / 2)), NT, 0, s>>>(P, site, pool, dk, kids.size(), n);
        launched();
      }
      trace_sync("apply");
      nwaiting = wait_off;
      std::swap(cur_shots, nxt_shots);
      live = std::move(next);
      live_on_host = true;
      total_live = new_off;
      peak = std::max<uint64_t>(peak, live.size());
      i = j + 1;
    }

    // Leaves (exec_branch.cpp:267-281).
    if (!live_on_host) live_to_host(pinned("branch.h_nodes_dl", nn_dev, (DevNode*)nullptr));
    const uint64_t nl = live.size();
    uint64_t total = 0;
    std::vector<DevNode> hl(nl);
    for (uint64_t x = 0; x < nl; ++x) {
      hl[x] = {live[x].slot, 1, live[x].off, live[x].len, live[x].creg};
      total += live[x].len;
    }
    if (opts && opts->collect_leaf_stats) {  // BranchStats::leaf_shots (exec_branch.cpp:280)
      for (uint64_t x = 0; x < nl; ++x, ++num_leaves)
        if (opts->leaf_shots && num_leaves < opts->leaf_shots_capacity) opts->leaf_shots[num_leaves] = live[x].len;
    }
    if (opts && opts->states_out && total > 0) {
      // Debug export: every shot's leaf state (what its terminal sampling reads).
      std::vector<uint64_t> hshots(total);
      CKB(cudaMemcpyAsync(hshots.data(), cur_shots, total * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      CKB(cudaStreamSynchronize(s));
      for (uint64_t x = 0; x < nl; ++x)
        for (uint64_t p = live[x].off; p < live[x].off + live[x].len; ++p)
          CKB(cudaMemcpyAsync(opts->states_out + 2 * ((hshots[p] - shot_begin) << n), pool + (uint64_t{live[x].slot} << n),
                              A * sizeof(double2), cudaMemcpyDeviceToHost, s));
      CKB(cudaStreamSynchronize(s));
    }
    if (nl > 0 && total > 0) {
      DevNode* leaves = dnodes.get(nl);
      CKB(cudaMemcpyAsync(leaves, hl.data(), nl * sizeof(DevNode), cudaMemcpyHostToDevice, s));
      double* cum = nullptr;
      uint64_t* last = nullptr;
      const uint64_t cnt = uint64_t{1} << P.nsample;
      if (h.eligible) {
        cum = dcum.get(nl * cnt);
        last = dlast.get(nl);
        if (P.nsample == n) {
          b_leaf_cum_full<<<gridn(nl * 32, 128), 128, 0, s>>>(P, pool, leaves, nl, cum, last);
          launched();
        } else {
          RedSpec R{};
          R.mode = R_OUTCOME;
          R.n = n;
          R.k = P.nsample;
          for (unsigned b = 0; b < P.nsample; ++b) R.q[b] = R.sorted[b] = h.sample_qubits[b];
          std::sort(R.sorted, R.sorted + P.nsample);
          const uint64_t G = A >> P.nsample;
          R.nq = static_cast<uint32_t>(cnt);
          R.nb = G <= SUM_BLOCK ? 1 : G / SUM_BLOCK;
          R.blk = G <= SUM_BLOCK ? G : SUM_BLOCK;
          std::vector<uint32_t> hs(nl);
          for (uint64_t x = 0; x < nl; ++x) hs[x] = live[x].slot;
          uint32_t* slots = dslots.get(nl);
          CKB(cudaMemcpyAsync(slots, hs.data(), nl * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
          double* part = dpart.get(nl * R.nq * R.nb);
          double* probs = dvals.get(nl * R.nq);
          launch_reduce(s, pool, nl, R, nullptr, part, slots);
          launched();
          g_finish_kernel<<<static_cast<unsigned>(std::min<uint64_t>(nl * R.nq, 1u << 20)), NT, 0, s>>>(nl, R.nq, R.nb, 0, nullptr, part, probs);
          launched();
          b_leaf_cum_probs<<<gridn(nl * 32, 128), 128, 0, s>>>(probs, nl, cnt, cum, last);
          launched();
          CKB(cudaStreamSynchronize(s));
        }
      }
      b_leaf_values<<<gridn(total), NT, 0, s>>>(P, leaves, nl, cur_shots, total, seed, cum, last, cnt, shot_begin,
                                                values_dev, E.err);
      launched();
      CKB(cudaStreamSynchronize(s));
    }
  }
  if (tracing)
    for (auto& [k, v] : trace_t) std::fprintf(stderr, "branch trace %-14s %.3f s\n", k.c_str(), v);
  if (stats) {
    stats->peak_states = peak;
    stats->passes = passes;
    stats->num_leaves = num_leaves;
    stats->dispatch_count = *E.launches - launches0;
  }
}

}  // namespace ssb
