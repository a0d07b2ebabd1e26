// The FMA fused tile pass (ssb_run_options::fused_matrices), shared by the
// static kernel (fused.cuh) and the run-time specialised per-pass kernels
// (fused_jit.cpp, NVRTC): only the group phase differs — the static kernel
// interprets the pass's groups / blocks from shared memory, a specialised
// kernel runs them as straight-line code with compile-time positions and the
// noiseless block products as constant-bank operands.
#pragma once

#include "tile_pass.cuh"

namespace ssb {


struct FusedView {
  const FPass* passes;
  const FGroup* groups;
  const FBlock* blocks;
  const FSite* sites;
  const uint32_t* qidx;
  const double2* mats;  // 16 double2 per matrix
  uint32_t n;
};

// Per shot and block: the matrix to apply (shared-memory offset in double2
// units) and the drawn factors that follow it when the product slots ran out
// (global matrix indices xf[xbegin, xbegin + xcount)).
struct FEntry {
  uint32_t src;
  uint16_t xbegin, xcount;
};

// Shared memory: tile | base matrices | product slots | entries | group and
// block descriptors | extra factors | hi offsets.
__host__ __device__ inline uint64_t fused_smem_bytes(unsigned k, uint32_t max_blocks, uint32_t max_sites) {
  return (uint64_t{1} << k) * 16 + uint64_t{max_blocks} * 256 + uint64_t{kFusedSlots} * 256 +
         uint64_t{max_blocks} * (sizeof(FEntry) + sizeof(FGroup) + sizeof(FBlock)) + uint64_t{max_sites} * 4 +
         (uint64_t{1} << (k - 6)) * 4 + 32;
}

__device__ __forceinline__ uint32_t ins0(uint32_t x, unsigned p) {
  return ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u));
}

// Tile layout: element l lives at swz(l) (16-byte units): XORing bits 3..5
// into 0..2 spreads the 8 lanes of a quarter-warp over distinct bank groups
// for most group position sets (at most 2-way conflicts for the rest).
__device__ __forceinline__ uint32_t swz(uint32_t l) { return l ^ ((l >> 3) & 7u); }

__device__ __forceinline__ double2 cfma(double2 m, double2 a, double2 acc) {
  acc.x = fma(m.x, a.x, acc.x);
  acc.x = fma(-m.y, a.y, acc.x);
  acc.y = fma(m.x, a.y, acc.y);
  acc.y = fma(m.y, a.x, acc.y);
  return acc;
}

// y = M x on the four register quads of a hexad whose matrix bits are group
// bits B0 < B1 (the other two group bits enumerate the quads).
// Largest register for which the fused pass prefetches the next tile into L2.
constexpr unsigned kFusedPrefetchMaxQubits = 20;

// M: a register array double2[16] or a pointer (shared / constant memory).
template <int B0, int B1, class M>
__device__ __forceinline__ void apply_hexad(double2 (&a)[16], const M& m) {
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    // spread o over the two group bits that are not B0 / B1
    int rest = 0, bit = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j != B0 && j != B1) rest |= ((o >> bit++) & 1) << j;
    const int e0 = rest, e1 = rest | (1 << B0), e2 = rest | (1 << B1), e3 = rest | (1 << B0) | (1 << B1);
    const double2 x0 = a[e0], x1 = a[e1], x2 = a[e2], x3 = a[e3];
    double2 y[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 acc = make_double2(0.0, 0.0);
      acc = cfma(m[r * 4 + 0], x0, acc);
      acc = cfma(m[r * 4 + 1], x1, acc);
      acc = cfma(m[r * 4 + 2], x2, acc);
      acc = cfma(m[r * 4 + 3], x3, acc);
      y[r] = acc;
    }
    a[e0] = y[0];
    a[e1] = y[1];
    a[e2] = y[2];
    a[e3] = y[3];
  }
}

// 8-amplitude "octad" of a 3-qubit group: two quads.
template <int B0, int B1>
__device__ __forceinline__ void apply_octad(double2 (&a)[8], const double2 (&m)[16]) {
  constexpr int R = 3 - B0 - B1;  // the group bit that enumerates the quads
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int rest = o << R;
    const int e0 = rest, e1 = rest | (1 << B0), e2 = rest | (1 << B1), e3 = rest | (1 << B0) | (1 << B1);
    const double2 x0 = a[e0], x1 = a[e1], x2 = a[e2], x3 = a[e3];
    double2 y[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 acc = make_double2(0.0, 0.0);
      acc = cfma(m[r * 4 + 0], x0, acc);
      acc = cfma(m[r * 4 + 1], x1, acc);
      acc = cfma(m[r * 4 + 2], x2, acc);
      acc = cfma(m[r * 4 + 3], x3, acc);
      y[r] = acc;
    }
    a[e0] = y[0];
    a[e1] = y[1];
    a[e2] = y[2];
    a[e3] = y[3];
  }
}

__device__ __forceinline__ void apply_unit_dyn(double2 (&a)[8], const double2 (&m)[16], unsigned b0, unsigned b1) {
  switch (b0 * 4 + b1) {
    case 1: apply_octad<0, 1>(a, m); break;
    case 2: apply_octad<0, 2>(a, m); break;
    default: apply_octad<1, 2>(a, m); break;
  }
}

__device__ __forceinline__ void apply_hexad_dyn(double2 (&a)[16], const double2 (&m)[16], unsigned b0, unsigned b1) {
  switch (b0 * 4 + b1) {  // b0 < b1 (the planner orders each block's matrix bits)
    case 1: apply_hexad<0, 1>(a, m); break;
    case 2: apply_hexad<0, 2>(a, m); break;
    case 3: apply_hexad<0, 3>(a, m); break;
    case 6: apply_hexad<1, 2>(a, m); break;
    case 7: apply_hexad<1, 3>(a, m); break;
    default: apply_hexad<2, 3>(a, m); break;
  }
}

__device__ __forceinline__ void apply_unit_dyn(double2 (&a)[16], const double2 (&m)[16], unsigned b0, unsigned b1) {
  apply_hexad_dyn(a, m, b0, b1);
}

__device__ __forceinline__ void load_mat(double2 (&m)[16], const double2* p) {
#pragma unroll
  for (int j = 0; j < 16; ++j) m[j] = p[j];
}

// Cold path of a specialised pass (a block whose shot drew a non-identity
// Pauli): the hexad goes back to its tile slots (the thread owns them), the
// block's matrix and extra factors are applied there by a rolled loop, and
// the hexad is reloaded — few live registers, so the hot path keeps its
// allocation (an inline register version spills, an out-of-line one puts the
// hexad in local memory).
template <int B0, int B1>
__device__ __forceinline__ void tile_apply_rolled(double2* tile, uint32_t sb, const uint32_t (&t)[4],
                                                  const double2* m) {
#pragma unroll 1
  for (int o = 0; o < 4; ++o) {
    uint32_t rest = 0;
    for (int j = 0, bit = 0; j < 4; ++j)
      if (j != B0 && j != B1) rest ^= ((o >> bit++) & 1) ? t[j] : 0u;
    const uint32_t e0 = sb ^ rest, e1 = e0 ^ t[B0], e2 = e0 ^ t[B1], e3 = e1 ^ t[B1];
    const double2 x0 = tile[e0], x1 = tile[e1], x2 = tile[e2], x3 = tile[e3];
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
      double2 acc = make_double2(0.0, 0.0);
      acc = cfma(m[r * 4 + 0], x0, acc);
      acc = cfma(m[r * 4 + 1], x1, acc);
      acc = cfma(m[r * 4 + 2], x2, acc);
      acc = cfma(m[r * 4 + 3], x3, acc);
      tile[r == 0 ? e0 : r == 1 ? e1 : r == 2 ? e2 : e3] = acc;  // the x are in registers
    }
  }
}

// One block of a specialised pass (fused_jit.cpp): the constant-bank product
// cm when this shot's entry is the block's noiseless base matrix (shared
// offset const_src, no extra factors), else the entry's matrix and factors
// (cold path above). sb / t: the hexad's tile base and bit offsets.
template <int B0, int B1>
__device__ __forceinline__ void jit_block(double2 (&a)[16], const FEntry ent, uint32_t const_src, const double2* cm,
                                          double2* tile, uint32_t sb, const uint32_t (&t)[4], const uint32_t* xf,
                                          const FusedView& F) {
  if (ent.src == const_src && ent.xcount == 0) {
    apply_hexad<B0, B1>(a, cm);
    return;
  }
#pragma unroll
  for (int e = 0; e < 16; ++e)
    tile[sb ^ ((e & 1 ? t[0] : 0u) ^ (e & 2 ? t[1] : 0u) ^ (e & 4 ? t[2] : 0u) ^ (e & 8 ? t[3] : 0u))] = a[e];
  tile_apply_rolled<B0, B1>(tile, sb, t, tile + ent.src);
#pragma unroll 1
  for (uint32_t x = 0; x < ent.xcount; ++x)
    tile_apply_rolled<B0, B1>(tile, sb, t, F.mats + uint64_t{xf[ent.xbegin + x]} * 16);
#pragma unroll
  for (int e = 0; e < 16; ++e)
    a[e] = tile[sb ^ ((e & 1 ? t[0] : 0u) ^ (e & 2 ? t[1] : 0u) ^ (e & 4 ? t[2] : 0u) ^ (e & 8 ? t[3] : 0u))];
}

// Persistent over (shot, tile) units like tile_pass_body. FNT threads (256:
// 12-qubit tiles, 128: 11-qubit tiles — one 16-amplitude hexad per thread);
// the low log2(FNT) local bits come from the thread index.
// Every pass descriptor the inner loops read is staged in shared memory or
// held in registers once per CTA (a reference into global memory would be
// re-read after every barrier).
// The interpreter group phase: positions, bit pairs and matrices read from
// the staged descriptors (one hexad / octad per thread, all its amplitudes in
// registers while the group's blocks are applied).
template <int FNT, int G>
struct InterpGroups {
  __device__ __forceinline__ void operator()(double2* tile, const FEntry* ents, const FGroup* sgrp, const FBlock* sblk,
                                             const uint32_t* xf, uint32_t ng, const FusedView& F) const {
    const uint32_t tile_units = units_per_tile;
      for (uint32_t gi = 0; gi < ng; ++gi) {
        const FGroup GR = sgrp[gi];
        // swz is linear over XOR, so element e of a unit sits at
        // swz(base) ^ (XOR of swz(2^g_i) over the set bits i of e).
        const uint32_t t0 = swz(1u << GR.g[0]), t1 = swz(1u << GR.g[1]), t2 = swz(1u << GR.g[2]),
                       t3 = G == 4 ? swz(1u << GR.g[3]) : 0u;
#define SSB_GO(e) (((e) & 1 ? t0 : 0u) ^ ((e) & 2 ? t1 : 0u) ^ ((e) & 4 ? t2 : 0u) ^ ((e) & 8 ? t3 : 0u))
        for (uint32_t h = threadIdx.x; h < (tile_units); h += FNT) {
          uint32_t base = ins0(ins0(ins0(h, GR.g[0]), GR.g[1]), GR.g[2]);
          if (G == 4) base = ins0(base, GR.g[3]);
          const uint32_t sb = swz(base);
          double2 a[1 << G];
#pragma unroll
          for (int e = 0; e < (1 << G); ++e) a[e] = tile[sb ^ SSB_GO(e)];
          for (uint32_t b = GR.blk_begin; b < GR.blk_end; ++b) {
            const FEntry ent = ents[b];
            const unsigned gb = sblk[b].gb0 * 4u + sblk[b].gb1;
            double2 m[16];
            load_mat(m, tile + ent.src);
            apply_unit_dyn(a, m, gb >> 2, gb & 3);
            for (uint32_t x = 0; x < ent.xcount; ++x) {
              load_mat(m, F.mats + uint64_t{xf[ent.xbegin + x]} * 16);
              apply_unit_dyn(a, m, gb >> 2, gb & 3);
            }
          }
#pragma unroll
          for (int e = 0; e < (1 << G); ++e) tile[sb ^ SSB_GO(e)] = a[e];
        }
#undef SSB_GO
        __syncthreads();
      }
  }
  uint32_t units_per_tile;
};

template <int FNT, int G, class Groups>
__device__ __forceinline__ void fused_pass_body(FusedView F, uint32_t pass_index, double2* state, uint64_t S,
                                                const uint8_t* pauli_sel, uint32_t num_pauli, uint32_t max_blocks,
                                                uint32_t max_sites, const Groups& groups) {
  extern __shared__ double2 tile[];
  __shared__ FPass spd;
  __shared__ uint8_t hpos[32];
  if (threadIdx.x == 0) spd = F.passes[pass_index];
  __syncthreads();
  const unsigned n = F.n, k = spd.k;
  const bool first = spd.first;
  const uint32_t blk0 = spd.blk_begin, nb = spd.blk_end - spd.blk_begin;
  const uint32_t grp0 = spd.grp_begin, ng = spd.grp_end - spd.grp_begin;
  const uint64_t tiles = uint64_t{1} << (n - k);
  const uint32_t L = 1u << k;
  double2* bmats = tile + L;
  double2* slots = bmats + max_blocks * 16;
  FEntry* ents = reinterpret_cast<FEntry*>(slots + kFusedSlots * 16);
  FGroup* sgrp = reinterpret_cast<FGroup*>(ents + max_blocks);
  FBlock* sblk = reinterpret_cast<FBlock*>(sgrp + max_blocks);
  uint32_t* xf = reinterpret_cast<uint32_t*>(sblk + max_blocks);
  // 16-byte aligned: the tile loops read four offsets per LDS.128
  uint32_t* hi_off =
      reinterpret_cast<uint32_t*>((reinterpret_cast<unsigned long long>(xf + max_sites) + 15) & ~15ull);

  for (uint32_t i = threadIdx.x; i < nb; i += FNT) {
    FBlock b = F.blocks[blk0 + i];
    sblk[i] = b;
  }
  for (uint32_t i = threadIdx.x; i < ng; i += FNT) {
    FGroup g = F.groups[grp0 + i];
    g.blk_begin -= blk0;  // pass-local block indices
    g.blk_end -= blk0;
    sgrp[i] = g;
  }
  constexpr unsigned LB = FNT == 64 ? 6 : FNT == 128 ? 7 : 8;  // log2(FNT)
  for (uint32_t i = threadIdx.x; i < (1u << (k - LB)); i += FNT)
    hi_off[i] = static_cast<uint32_t>(pdep_positions(i, spd.lq + LB, k - LB));
  if (threadIdx.x == 0)
    for (unsigned q = 0, j = 0; q < n; ++q)
      if (!((spd.lmask >> q) & 1)) hpos[j++] = static_cast<uint8_t>(q);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb * 16; i += FNT) bmats[i] = F.mats[uint64_t{sblk[i / 16].mat} * 16 + i % 16];
  __syncthreads();  // warp 0 copies base matrices into the product slots below
  const uint32_t lo_part = static_cast<uint32_t>(pdep_positions(threadIdx.x, spd.lq, LB));
  const uint64_t units = S * tiles;
  const uint64_t u_begin = units * blockIdx.x / gridDim.x, u_end = units * (blockIdx.x + 1) / gridDim.x;
  const unsigned lane = threadIdx.x & 31;
  const uint32_t per = L / FNT;  // tile elements per thread

  for (uint64_t s = u_begin / tiles; s * tiles < u_end; ++s) {
    // ---- this shot's matrices (warp 0): M for blocks whose draws were all
    // identity, else Q_L ... Q_1 M in a slot (or M + extra factors) ----
    if (threadIdx.x < 32) {
      const uint8_t* sel = pauli_sel + s * num_pauli;
      uint32_t slot = 0, nx = 0;
      for (uint32_t b = 0; b < nb; ++b) {
        const FBlock B = sblk[b];
        FEntry ent{static_cast<uint32_t>(bmats + b * 16 - tile), static_cast<uint16_t>(nx), 0};
        double2* R = nullptr;
        for (uint32_t c0 = B.site_begin; c0 < B.site_end; c0 += 32) {
          const uint32_t si = c0 + lane;
          uint32_t qi = kNoQ;
          if (si < B.site_end) {
            const FSite st = F.sites[si];
            qi = F.qidx[st.qbase + sel[st.site]];
          }
          unsigned noisy = __ballot_sync(0xffffffffu, qi != kNoQ);
          while (noisy) {  // drawn factors in site order
            const unsigned l = __ffs(noisy) - 1;
            noisy &= noisy - 1;
            const uint32_t q = __shfl_sync(0xffffffffu, qi, l);
            if (!R && ent.xcount == 0 && slot < kFusedSlots) {  // R = M in a fresh slot
              R = slots + 16 * slot++;
              if (lane < 16) R[lane] = bmats[b * 16 + lane];
              __syncwarp();
              ent.src = static_cast<uint32_t>(R - tile);
            }
            if (R) {  // R <- Q R (16 lanes, one entry each)
              double2 v = make_double2(0.0, 0.0);
              if (lane < 16) {
                const double2* Q = F.mats + uint64_t{q} * 16;
                const unsigned r = lane >> 2, c = lane & 3;
#pragma unroll
                for (unsigned j = 0; j < 4; ++j) v = cfma(Q[r * 4 + j], R[j * 4 + c], v);
              }
              __syncwarp();
              if (lane < 16) R[lane] = v;
              __syncwarp();
            } else {
              if (lane == 0) xf[nx] = q;
              ++nx;
              ++ent.xcount;
            }
          }
        }
        if (lane == 0) ents[b] = ent;
      }
    }
    __syncthreads();
    double2* seg = state + (s << n);
    const uint64_t t_begin = u_begin > s * tiles ? u_begin - s * tiles : 0;
    const uint64_t t_end = u_end < (s + 1) * tiles ? u_end - s * tiles : tiles;
    for (uint64_t t = t_begin; t < t_end; ++t) {
      double2* tbase = seg + pdep_positions(t, hpos, n - k);
      if (first) {
        const bool origin = (tbase == seg);
        for (uint32_t l = threadIdx.x, i = 0; l < L; l += FNT, ++i)
          tile[swz(l)] = make_double2((origin && (lo_part | hi_off[i]) == 0) ? 1.0 : 0.0, 0.0);
      } else {
        // element threadIdx.x + FNT * i sits at swz(threadIdx.x) + FNT * i
        // (FNT >= 64: the swizzle only mixes bits 3..5 into 0..2), and its
        // global offset is lo_part + hi_off[i] (disjoint bits)
        const uint32_t tile_s = static_cast<uint32_t>(__cvta_generic_to_shared(tile)) + 16u * swz(threadIdx.x);
        const double2* tb = tbase + lo_part;
        for (uint32_t i = 0; i < per; i += 4) {
          const uint4 h = *reinterpret_cast<const uint4*>(hi_off + i);
          const uint32_t o[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j)
            if (i + j < per)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tile_s + 16u * FNT * (i + j)),
                           "l"(tb + o[j]));
        }
#ifndef SSB_FUSED_NO_PREFETCH
        // the next tile's lines on their way to L2 — on registers of up to 20
        // qubits (C2 +1%; C5's 24 qubits run 2% faster without it,
        // profiles/r02/fused_variants.log)
        if (t + 1 < t_end && n <= kFusedPrefetchMaxQubits) {
          const double2* nb = seg + pdep_positions(t + 1, hpos, n - k) + lo_part;
          for (uint32_t i = 0; i < per; i += 4) {
            const uint4 h = *reinterpret_cast<const uint4*>(hi_off + i);
            const uint32_t o[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j)
              if (i + j < per) asm volatile("prefetch.global.L2 [%0];" ::"l"(nb + o[j]));
          }
        }
#endif
        asm volatile("cp.async.wait_all;" ::: "memory");
      }
      __syncthreads();
      groups(tile, ents, sgrp, sblk, xf, ng, F);  // every block of the pass, group by group
      {
        double2* tb = tbase + lo_part;
        const double2* ts = tile + swz(threadIdx.x);
        for (uint32_t i = 0; i < per; i += 4) {
          const uint4 h = *reinterpret_cast<const uint4*>(hi_off + i);
          const uint32_t o[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j)
            if (i + j < per) tb[o[j]] = ts[FNT * (i + j)];
        }
      }
    }
    __syncthreads();  // the next shot's matrices rewrite slots / ents
  }
}


}  // namespace ssb
