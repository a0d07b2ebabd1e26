// The HBM-streamed executor's fused tile pass (shared by the static kernel in
// kernels.cuh and the run-time shape-specialised kernel, specialise.cu).
#pragma once

#include "shapes.cuh"
#include "exact_scan.cuh"

namespace ssb {

enum DevError : int { DEV_OK = 0, DEV_DEGENERATE = 1, DEV_NORM = 2 };

struct ProgView {
  const DevOp* ops;
  const DevTerm* terms;
  const DevChannel* channels;
  const double2* mats;        // 16 double2 per slot
  const uint64_t* scaled_cls; // per slot
  const uint8_t* sample_qubits;
  const uint8_t* write_clbit;
  const uint8_t* write_pos;
  const PassDesc* passes;
  const Item* items;
  const PassOp* pass_ops;
  const Uop* uops;
  const double2* uop_mats;
  const uint32_t* pauli_site_ops;  // site ordinal -> op index
  uint32_t num_pauli;
  uint32_t n, end, nsample, nwrites;
  uint64_t num_events;
  uint32_t eligible, sample_identity;
};

__device__ __forceinline__ void raise(int* err, int code) { atomicCAS(err, 0, code); }

__device__ __forceinline__ uint64_t shot_of(const uint64_t* ids, uint64_t begin, uint64_t s) {
  return ids ? ids[s] : begin + s;
}

// ---------------------------------------------------------------------------
// Streamed executor: fused tile pass. Grid: S * 2^(n-k) CTAs; CTA (s, t) owns
// tile t of shot s: local index l <-> global index pdep(t, ~lmask) | pdep(l, lmask).
__device__ __forceinline__ uint64_t pdep_positions(uint64_t v, const uint8_t* pos, unsigned k) {
  uint64_t out = 0;
  for (unsigned j = 0; j < k; ++j) out |= ((v >> j) & 1) << pos[j];
  return out;
}

// Pass epilogue (PassDesc::epi_*): the next Kraus site's matrix-0 partial
// sums from the finished tile, in the reference's order — 1q: each 512-pair
// block's sequential sum of |row_0|^2, |row_1|^2 per pair in pair order
// (kernels_scalar.cpp:103-126), one warp per block with the exact
// warp-parallel sequential sum; 2q: each 8-group leaf of expval_generic's
// pairwise tree (per group the rows' |.|^2 summed in order, then the 8 groups
// in order; statevector.cpp:56-80, common.cpp:12-20), one thread per leaf.
// Everything the epilogue reads besides the tile is staged once per CTA in
// shared memory (EpiTables): the matrix, its classes, off[j] the local offset
// of pair / group j inside a partial, hv[w] the local offset of the tile's
// partial w, pidx[w] its index contribution, tbit[i] that of the tile's i-th
// non-local qubit.
struct EpiTables {
  double2 m[16];
  uint64_t cls;
  uint32_t kind, tb0, tb1;
  uint32_t tbit[32];
  uint16_t off[512];
  uint16_t hv[128];
  uint32_t pidx[128];
};

// Partial-index bit of qubit q: its position among the non-target qubits
// (pair / group index), minus the bits inside one partial (9 or 3).
__device__ __forceinline__ int epi_bit(const DevOp& op, unsigned kind, unsigned q) {
  unsigned below = 0;
  for (unsigned b = 0; b < kind; ++b) below += op.q[b] < q;
  return static_cast<int>(q - below) - (kind == 1 ? 9 : 3);
}

static __device__ __noinline__ void epi_tables(const ProgView& P, const PassDesc& pd, const uint8_t* hpos, unsigned n,
                                               EpiTables& T) {
  const DevOp& op = P.ops[pd.epi_op];
  const unsigned kind = pd.epi_kind, nlow = pd.epi_nlow, nhi = pd.epi_nhi;
  const DevChannel ch = P.channels[op.aux];
  for (uint32_t e = threadIdx.x; e < 16; e += NT) T.m[e] = P.mats[16 * ch.mat_begin + e];  // matrix 0
  if (threadIdx.x == 0) {
    T.cls = P.scaled_cls[ch.mat_begin];
    T.kind = kind;
    T.tb0 = 1u << pd.epi_t[0];
    T.tb1 = kind == 2 ? 1u << pd.epi_t[1] : 0u;
  }
  for (uint32_t i = threadIdx.x; i < n - pd.k; i += NT) T.tbit[i] = 1u << epi_bit(op, kind, hpos[i]);
  for (uint32_t j = threadIdx.x; j < (1u << nlow); j += NT)
    T.off[j] = static_cast<uint16_t>(pdep_positions(j, pd.epi_low, nlow));
  for (uint32_t w = threadIdx.x; w < (1u << nhi); w += NT) {
    T.hv[w] = static_cast<uint16_t>(pdep_positions(w, pd.epi_hi, nhi));
    uint32_t x = 0;
    for (unsigned i = 0; i < nhi; ++i)
      if ((w >> i) & 1) x |= 1u << epi_bit(op, kind, pd.lq[pd.epi_hi[i]]);
    T.pidx[w] = x;
  }
}

// One tile's partials (all threads; reads the tile and T only).
__device__ __forceinline__ void tile_epilogue(const EpiTables& T, unsigned nhi, const double2* tile,
                                              uint32_t tile_pidx, double* part) {
  const uint32_t nparts = 1u << nhi;
  if (T.kind == 1) {
    // one warp per 512-pair block: 1024 terms summed in the reference order
    const uint32_t tb = T.tb0;
    for (uint32_t w = threadIdx.x >> 5; w < nparts; w += NT / 32) {
      const uint32_t hv = T.hv[w];
      const ExactPick r = warp_exact_scan(
          [&](uint64_t t) {
            const uint32_t l = T.off[t >> 1] | hv;
            const double2 in[2] = {tile[l], tile[l | tb]};
            return c_norm(row_apply<2>(T.m, T.cls, static_cast<int>(t & 1), in));
          },
          1024, scan_all(), NoSum{});
      if ((threadIdx.x & 31) == 0) part[tile_pidx | T.pidx[w]] = r.s_at;
    }
  } else {
    // 8 lanes per leaf: lane g computes group g's partial (rows summed in
    // order), lane 0 of the 8 adds the 8 partials in order
    const uint32_t b0 = T.tb0, b1 = T.tb1;
    const unsigned lane = threadIdx.x & 31, gi = lane & 7;
    for (uint32_t x = threadIdx.x; x < nparts * 8; x += NT) {
      const uint32_t w = x >> 3;
      const uint32_t base = T.off[gi] | T.hv[w];
      const double2 in[4] = {tile[base], tile[base | b0], tile[base | b1], tile[base | b0 | b1]};
      double row = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) row = __dadd_rn(row, c_norm(row_apply<4>(T.m, T.cls, r, in)));
      double acc = 0.0;
#pragma unroll
      for (unsigned g = 0; g < 8; ++g) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, row, (lane & ~7u) | g));
      if (gi == 0) part[tile_pidx | T.pidx[w]] = acc;
    }
  }
}

// Shared-memory layout of the tile pass: tile | matrix table | uops |
// compacted uops | kept-uop prefix (u16, nu + 1) | kept-Pauli prefix (u16,
// nu + 1) | high-part tile offsets (u32, 2^(k - 8)).
__host__ __device__ inline uint64_t tile_smem_bytes(unsigned k, uint32_t nuops, uint32_t nmats, bool db = false) {
  const unsigned kt = k < 8 ? k : 8;
  return (uint64_t{1} << k) * 16 * (db ? 2 : 1) + uint64_t{nmats} * 16 + uint64_t{nuops} * 32 +
         (uint64_t{nuops} + 1) * 4 + 16 +
         (uint64_t{1} << (k - kt)) * 4 + uint64_t{nuops} + 16;
}

// Persistent: each CTA owns a contiguous range of (shot, tile) units, stages
// the pass's micro-op stream once, and compacts it once per shot it touches.
// kmat / kcls: per-shot chosen Kraus matrix (16 double2, scaled by
// 1/sqrt(p)) and its classes for a pass that starts with a Kraus apply.
static __device__ __forceinline__ void tile_pass_body(const ProgView& P, uint32_t pass_index, double2* state, uint64_t S,
                                                      const uint64_t* cregs, const uint8_t* pauli_sel,
                                                      uint32_t num_pauli, const double2* kmat, const uint64_t* kcls,
                                                      const uint32_t* act, double* epi_part) {
  extern __shared__ double2 tile0[];
  const PassDesc& pd = P.passes[pass_index];
  const unsigned n = P.n, k = pd.k;
  const unsigned kt = k < 8 ? k : 8;
  const uint64_t tiles = uint64_t{1} << (n - k);
  const uint32_t L = 1u << k;
  const uint32_t nu = pd.uop_end - pd.uop_begin;
  // SSB_TILE_DB: two tile buffers; the next tile of the shot is loaded while
  // this one is computed and stored (tile_smem_bytes(..., db = true)).
#ifdef SSB_TILE_DB
  constexpr uint32_t NBUF = 2;
#else
  constexpr uint32_t NBUF = 1;
#endif
  double2* tile = tile0;
  double2* smats = tile0 + NBUF * L;
  Uop* uops = reinterpret_cast<Uop*>(smats + pd.mat_count);
  Uop* eops = uops + nu;
  uint16_t* pre = reinterpret_cast<uint16_t*>(eops + nu);
  uint16_t* ppre = pre + (nu + 1);
  uint32_t* hi_off = reinterpret_cast<uint32_t*>((reinterpret_cast<unsigned long long>(ppre + (nu + 1)) + 7) & ~7ull);
  uint8_t* pinfo = reinterpret_cast<uint8_t*>(hi_off + (1u << (k - (k < 8 ? k : 8))));  // per-uop drawn Pauli (0xFF: none)
  __shared__ uint8_t hpos[32];
  __shared__ uint64_t kraus_cls;
  const bool has_kraus = pd.kraus_mat < pd.mat_count;

  for (uint32_t i = threadIdx.x; i < pd.mat_count; i += NT) smats[i] = P.uop_mats[pd.mat_begin + i];
  for (uint32_t i = threadIdx.x; i < nu; i += NT) uops[i] = P.uops[pd.uop_begin + i];
  for (uint32_t i = threadIdx.x; i < (1u << (k - kt)); i += NT)
    hi_off[i] = static_cast<uint32_t>(pdep_positions(i, pd.lq + kt, k - kt));
  if (threadIdx.x == 0)
    for (unsigned q = 0, j = 0; q < n; ++q)
      if (!((pd.lmask >> q) & 1)) hpos[j++] = static_cast<uint8_t>(q);
  __syncthreads();

  const uint32_t lo_part = static_cast<uint32_t>(pdep_positions(threadIdx.x, pd.lq, kt));
  // Epilogue index tables (once per CTA).
  __shared__ EpiTables epi_tab;
  const bool epi = pd.epi_kind && epi_part;
  const uint64_t epi_nb = pd.epi_kind == 1 ? (uint64_t{1} << (n - 1)) / 512 : (uint64_t{1} << (n - 2)) / 8;
  if (epi) {
    epi_tables(P, pd, hpos, n, epi_tab);
    __syncthreads();
  }
  bool no_relabel = true;
  for (uint32_t it_i = pd.item_begin; it_i < pd.item_end; ++it_i) no_relabel &= P.items[it_i].sigma == 0xE4;
  // Shape-specialised straight-line executors need every register round full.
  const bool full_rounds = k >= 2 && ((1u << (k - 2)) % (NT * QPT)) == 0;
  // Work units are (shot, tile) pairs in shot-major order; each CTA owns a
  // contiguous unit range, so it sees at most a few shot boundaries (one
  // compaction each) while waves of only a few huge shots (n = 24: 64 shots
  // per 16 GiB wave) still spread over every SM.
  const uint64_t units = S * tiles;
  const uint64_t u_begin = units * blockIdx.x / gridDim.x, u_end = units * (blockIdx.x + 1) / gridDim.x;
  // act: optional list of the wave slots this pass runs (shared-trunk mode:
  // shots whose randomness has not diverged from the trunk yet are skipped).
  for (uint64_t si = u_begin / tiles; si * tiles < u_end; ++si) {
    const uint64_t s = act ? act[si] : si;  // wave slot
    // Per-shot compaction (warp 0, in order): drop failed conditions and
    // identity Pauli draws; resolve each Pauli to quad masks.
    if (threadIdx.x < 32) {
      const uint64_t creg = cregs ? cregs[s] : 0;
      const uint8_t* sel = pauli_sel + s * num_pauli;
      uint32_t count = 0, pcount = 0;
      for (uint32_t c0 = 0; c0 < nu; c0 += 32) {
        const uint32_t i = c0 + threadIdx.x;
        bool keep = false;
        Uop u{};
        if (i < nu) {
          u = uops[i];
          keep = true;
          const DevOp& op = P.ops[u.ref];
          if ((u.flags & 1) && (creg & op.cond_mask) != op.cond_value) keep = false;
          if (keep && u.code == UC_PAULI) {
            const DevTerm tm = P.terms[op.aux + sel[op.site]];
            if (tm.identity) {
              keep = false;
            } else {
              uint32_t xq = 0, zq = 0;
              for (unsigned b = 0; b < op.nq; ++b) {
                const uint32_t qb = (u.qb >> b) & 1u;
                xq |= ((tm.x >> op.q[b]) & 1u) << qb;
                zq |= ((tm.z >> op.q[b]) & 1u) << qb;
              }
              u.pauli = static_cast<uint8_t>(xq | (zq << 2) | ((tm.num_y & 3u) << 4));
            }
          }
        }
        const unsigned lanes_below = (1u << threadIdx.x) - 1;
        const unsigned ballot = __ballot_sync(0xffffffffu, keep);
        const unsigned pballot = __ballot_sync(0xffffffffu, keep && u.code == UC_PAULI);
        const uint32_t at = count + __popc(ballot & lanes_below);
        if (i < nu) {
          pre[i] = static_cast<uint16_t>(at);
          ppre[i] = static_cast<uint16_t>(pcount + __popc(pballot & lanes_below));
          pinfo[i] = (keep && u.code == UC_PAULI) ? u.pauli : static_cast<uint8_t>(0xFF);
        }
        if (keep) eops[at] = u;
        count += __popc(ballot);
        pcount += __popc(pballot);
      }
      if (threadIdx.x == 0) {
        pre[nu] = static_cast<uint16_t>(count);
        ppre[nu] = static_cast<uint16_t>(pcount);
      }
    } else if (has_kraus && threadIdx.x < 48) {  // stage this shot's Kraus choice
      if (threadIdx.x < 48) {
        const uint32_t e = threadIdx.x - 32;
        smats[pd.kraus_mat + e] = kmat[s * 16 + e];
        if (e == 0) kraus_cls = kcls[s];
      }
    }
    __syncthreads();
    double2* seg = state + (s << n);
    const uint64_t t_begin = u_begin > si * tiles ? u_begin - si * tiles : 0;
    uint64_t t_end = u_end < (si + 1) * tiles ? u_end - si * tiles : tiles;
    // Nothing to apply for this shot (every micro-op compacted away — e.g. a
    // pass of readout Pauli sites that all drew identity) and no relabeled
    // segment to store: its tiles are left untouched in HBM.
    if (!pd.first && pre[nu] == 0 && no_relabel && !epi) t_end = t_begin;
    // LDGSTS of tile tt of this shot into buffer dst (one commit group).
    auto load_tile = [&](uint64_t tt, double2* dst) {
      const double2* tb = seg + pdep_positions(tt, hpos, n - k);
      const uint32_t dst_s = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
      for (uint32_t l0 = threadIdx.x, i0 = 0; l0 < L; l0 += 8 * NT, i0 += 8) {
        uint32_t off[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) off[j] = l0 + j * NT < L ? hi_off[i0 + j] : 0u;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
          if (l0 + j * NT < L)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_s + 16 * (l0 + j * NT)),
                         "l"(tb + (lo_part | off[j])));
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (uint64_t t = t_begin; t < t_end; ++t) {
      double2* tbase = seg + pdep_positions(t, hpos, n - k);
      tile = tile0 + (NBUF == 2 ? ((t - t_begin) & 1) * L : 0);
      if (pd.first) {
        const bool origin = (tbase == seg);
        for (uint32_t l = threadIdx.x, i = 0; l < L; l += NT, ++i)
          tile[l] = make_double2((origin && (lo_part | hi_off[i]) == 0) ? 1.0 : 0.0, 0.0);
      } else if (NBUF == 2) {
        // This tile was requested one iteration ago (or now, for the shot's
        // first); request the next one into the other buffer before waiting.
        // Each thread's copies land in the slots only it reads at the store,
        // so refilling the other buffer needs no barrier.
        if (t == t_begin) load_tile(t, tile);
        if (t + 1 < t_end) {
          load_tile(t + 1, tile0 + ((t + 1 - t_begin) & 1) * L);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
      } else {
        // Asynchronous global -> shared copies (LDGSTS): every 16-byte element
        // of the thread is in flight at once, with no register round trip
        // (a register copy loop serialises on the loads).
        // (No memory clobber: the copies only write this thread's tile slots,
        // read after cp.async.wait_all below.)
        // Offsets are read 8 at a time ahead of their copies.
        const uint32_t tile_s = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
        for (uint32_t l0 = threadIdx.x, i0 = 0; l0 < L; l0 += 8 * NT, i0 += 8) {
          uint32_t off[8];
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j) off[j] = l0 + j * NT < L ? hi_off[i0 + j] : 0u;
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j)
            if (l0 + j * NT < L)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tile_s + 16 * (l0 + j * NT)),
                           "l"(tbase + (lo_part | off[j])));
        }
        // Optional (SSB_TILE_PREFETCH): warm L2 with the next tile of this
        // shot while this one is computed. Off by default: on B200 it costs
        // more DRAM reads than it saves latency (C4 +2.5%, C5 exact +1.2%
        // without it; ncu: 26% DRAM reads above the algorithmic bytes with it).
#ifdef SSB_TILE_PREFETCH
        if (t + 1 < t_end) {
          const double2* nb = seg + pdep_positions(t + 1, hpos, n - k);
          for (uint32_t l0 = threadIdx.x, i0 = 0; l0 < L; l0 += 8 * NT, i0 += 8) {
            uint32_t off[8];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) off[j] = l0 + j * NT < L ? hi_off[i0 + j] : 0u;
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j)
              if (l0 + j * NT < L) asm volatile("prefetch.global.L2 [%0];" ::"l"(nb + (lo_part | off[j])));
          }
        }
#endif
        asm volatile("cp.async.wait_all;" ::: "memory");
      }
      __syncthreads();
      for (uint32_t it_i = pd.item_begin; it_i < pd.item_end; ++it_i) {
        const Item it = P.items[it_i];
        const uint32_t b = pre[it.begin], e = pre[it.end];
        const uint32_t kept_pauli = ppre[it.end] - ppre[it.begin];
        if (full_rounds && it.shape != kNoShape && e - b - kept_pauli == it.nfast) {
          // Every condition of the segment holds for this shot: its shape runs
          // straight-line — skipping the Pauli sites when all drew identity
          // (the common case), else applying the drawn ones in place.
          if (kept_pauli == 0 && it.nfast == 0 && it.sigma == 0xE4) continue;
          if (ssb_run_shape(it.shape, kept_pauli != 0, tile, k, it.la, it.lb, smats + uops[it.begin].mat, kraus_cls,
                            pinfo + it.begin))
            continue;
        }
        if (b == e && it.sigma == 0xE4) continue;  // nothing to apply and no relabeling to store
        if (k < 2) {
          run_ops_per_op(tile, k, it.begin, it.end, P.pass_ops + pd.po_begin, P.ops, P.mats, P.terms,
                         cregs ? cregs[s] : 0, pauli_sel + s * num_pauli);
        } else {
          run_segment_staged(tile, k, it, eops, b, e, smats, P.ops, kraus_cls);
        }
      }
      if (epi) {  // the next Kraus site's matrix-0 partials
        __syncthreads();
        uint32_t tile_pidx = 0;  // the tile's non-local qubits' part of the partial index
        for (unsigned i = 0; i < n - k; ++i)
          if ((t >> i) & 1) tile_pidx |= epi_tab.tbit[i];
        tile_epilogue(epi_tab, pd.epi_nhi, tile, tile_pidx, epi_part + s * epi_nb);
        // the epilogue reads other threads' elements: none may be refilled by
        // the next tile's loads before every warp is done with them
        __syncthreads();
      }
      for (uint32_t l = threadIdx.x, i = 0; l < L; l += NT, ++i) tbase[lo_part | hi_off[i]] = tile[l];
    }
    __syncthreads();  // compaction of the next shot rewrites eops/pre
  }
}

#define SSB_TILE_PASS_PARAMS                                                                            \
  ssb::ProgView P, uint32_t pass_index, double2 *state, uint64_t S, const uint64_t *cregs, const uint8_t *pauli_sel, \
      uint32_t num_pauli, const double2 *kmat, const uint64_t *kcls, const uint32_t *act, double *epi_part
#define SSB_TILE_PASS_ARGS P, pass_index, state, S, cregs, pauli_sel, num_pauli, kmat, kcls, act, epi_part

}  // namespace ssb
