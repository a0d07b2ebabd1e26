// Fused-matrix tile pass (ssb_run_options::fused_matrices; plan: fused.cpp).
//
// One HBM read + write of every 2^k-amplitude tile per pass, like the exact
// tile pass, but each block of the plan is ONE dense 4x4 complex apply per
// amplitude quad with FMA arithmetic (16 DP instructions per amplitude per
// block instead of ~14 per gate x ~11 gates). Per shot, warp 0 first turns the
// pass's blocks into an apply list: a block whose Pauli draws were all
// identity uses its staged base product M; a noisy block gets Q_L ... Q_1 M
// multiplied into one of kFusedSlots shared-memory slots (beyond those, the
// Q factors follow M as extra list entries read from global memory).
#pragma once

#include "fused.hpp"
#include "kernels.cuh"

#include "fused_body.cuh"

namespace ssb {

// The static (interpreter) FMA build of the fused pass.
// Threads per SM the register allocation must allow (4-qubit groups: 512,
// i.e. 128 registers per thread; A/B knob SSB_FUSED_G4_THREADS).
#ifndef SSB_FUSED_G4_THREADS
#define SSB_FUSED_G4_THREADS 512
#endif
template <int FNT, int G>
static __global__ void __launch_bounds__(FNT, (G == 4 ? SSB_FUSED_G4_THREADS : 1024) / FNT)
    fused_pass_kernel(FusedView F, uint32_t pass_index, double2* state, uint64_t S, const uint8_t* pauli_sel,
                      uint32_t num_pauli, uint32_t max_blocks, uint32_t max_sites) {
  fused_pass_body<FNT, G>(F, pass_index, state, S, pauli_sel, num_pauli, max_blocks, max_sites,
                          InterpGroups<FNT, G>{(1u << F.passes[pass_index].k) >> G});
}

// ---------------------------------------------------------------------------
// Tensor-core build of the same pass (FP64 MMA, mma.sync m8n8k4: 2x the DFMA
// rate on B200, scripts/probes/dmma_probe.cu). For one block, a team of four
// lanes (t = lane / 4) holds quads — lane j = lane % 4 the quad element whose
// matrix bits equal j — so a quad batch is the 8 x 4 A operand (one quad per
// team), the block's real 4 x 8 coefficient slices are the B operand, and D
// comes back in the A layout:
//   D[t][2i + 0 / 1] = Re / Im y_i,  y = M x,  K = xr (MMA 1) then xi (MMA 2)
//   B1[j][2i] = Re M_ij, B1[j][2i+1] = Im M_ij, B2[j][2i] = -Im M_ij, B2[j][2i+1] = Re M_ij.
// Lane j's two bits follow the block: between blocks a lane bit is exchanged
// with a register bit by a shuffle with the partner lane (planner schedule,
// FGroup / FBlock.xch), never through shared memory.
// volatile: the issue order written below (four independent MMAs, then the
// four that accumulate onto them) is kept — ptxas would otherwise serialise
// every pair through one temporary and expose the tensor-core latency.
__device__ __forceinline__ void mma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%4};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(0.0));
}
__device__ __forceinline__ void mma_f64_acc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Exchange lane bit P with register bit Q (registers r = hh * 4 + rbits).
template <int P, int Q>
__device__ __forceinline__ void mma_exchange(double2 (&a)[16], unsigned j) {
  const bool b = (j >> P) & 1;
#pragma unroll
  for (int r0 = 0; r0 < 16; ++r0) {
    if (r0 & (1 << Q)) continue;
    const int r1 = r0 | (1 << Q);
    const double2 send = b ? a[r0] : a[r1];
    double2 recv;
    recv.x = __shfl_xor_sync(0xffffffffu, send.x, 1 << P);
    recv.y = __shfl_xor_sync(0xffffffffu, send.y, 1 << P);
    if (b) a[r0] = recv;
    else a[r1] = recv;
  }
}

__device__ __forceinline__ void mma_exchange_dyn(double2 (&a)[16], unsigned j, unsigned pq) {
  switch (pq & 3) {
    case 0: mma_exchange<0, 0>(a, j); break;
    case 1: mma_exchange<0, 1>(a, j); break;
    case 2: mma_exchange<1, 0>(a, j); break;
    default: mma_exchange<1, 1>(a, j); break;
  }
}

// y = M x for the 16 quads of the lane's registers.
__device__ __forceinline__ void mma_apply(double2 (&a)[16], const double2* M, unsigned t, unsigned j, bool perm) {
  const unsigned i = t >> 1;
  const unsigned ri = perm ? (((i & 1) << 1) | (i >> 1)) : i, cj = perm ? (((j & 1) << 1) | (j >> 1)) : j;
  const double2 m = M[ri * 4 + cj];
  const double b1 = (t & 1) ? m.y : m.x;
  const double b2 = (t & 1) ? m.x : -m.y;
  // batches of four independent quad MMAs: the K = xr halves, then the
  // K = xi halves accumulating onto them
#pragma unroll
  for (int rb = 0; rb < 16; rb += 4) {
    double d0[4], d1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) mma_f64(d0[i], d1[i], a[rb + i].x, b1);
#pragma unroll
    for (int i = 0; i < 4; ++i) mma_f64_acc(d0[i], d1[i], a[rb + i].y, b2);
#pragma unroll
    for (int i = 0; i < 4; ++i) a[rb + i] = make_double2(d0[i], d1[i]);
  }
}

// Tile layout of the tensor-core kernel: element l at hsw(l) = l with its
// low three bits XORed with a linear hash of bits 3.. (column per position
// below). A quarter-warp's eight 16-byte accesses vary two group bits (the
// lane bits) and one hexad bit; with the identity-or-shift swizzle of the
// FMA kernel many such triples collide in one bank group, the hashed columns
// keep every access at most 2-way (65% of triples conflict-free;
// tests/test_fused_mma_model.py). Linear over XOR: hsw(a ^ b) = hsw(a) ^ hsw(b).
__constant__ uint8_t kHswCol[16] = {3, 5, 6, 7, 3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7, 1};
__device__ __forceinline__ uint32_t hsw_slow(uint32_t l) {
  uint32_t h = 0;
  for (int i = 0; i < 16; ++i)
    if ((l >> (3 + i)) & 1) h ^= kHswCol[i];
  return l ^ h;
}

// Max tile qubits of the tensor-core kernel (hexad index <= 9 bits).
constexpr unsigned kMmaMaxK = 13;
// Shared memory: 2 tiles | base matrices | product slots | entries | group
// and block descriptors | per-group hexad-base tables (48 u32) | extra
// factors | per-i tile offsets.
__host__ __device__ inline uint64_t fused_mma_smem_bytes(unsigned k, uint32_t max_blocks, uint32_t max_sites) {
  return 2 * (uint64_t{1} << k) * 16 + uint64_t{max_blocks} * 256 + uint64_t{kFusedSlots} * 256 +
         uint64_t{max_blocks} * (sizeof(FEntry) + sizeof(FGroup) + sizeof(FBlock) + 48 * 4) + uint64_t{max_sites} * 4 +
         2 * (uint64_t{1} << (k - 8)) * 4 + 32;
}

// One CTA per SM (the 16 register amplitudes, the 4-deep MMA batches and
// their temporaries need ~200 registers); the tile of the next (shot, tile)
// unit is fetched with cp.async into the second buffer while this one is
// computed and stored, so HBM latency overlaps the tensor-core work.
template <bool MMA>
static __device__ __forceinline__ void fused_pass_db_body(FusedView F, uint32_t pass_index, double2* state, uint64_t S,
                                                          const uint8_t* pauli_sel, uint32_t num_pauli,
                                                          uint32_t max_blocks, uint32_t max_sites) {
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
  double2* bufs = tile;  // two tiles
  double2* bmats = tile + 2 * L;
  double2* slots = bmats + max_blocks * 16;
  FEntry* ents = reinterpret_cast<FEntry*>(slots + kFusedSlots * 16);
  FGroup* sgrp = reinterpret_cast<FGroup*>(ents + max_blocks);
  FBlock* sblk = reinterpret_cast<FBlock*>(sgrp + max_blocks);
  uint32_t* gtab = reinterpret_cast<uint32_t*>(sblk + max_blocks);  // per group: lo[16] | hi[32]
  uint32_t* xf = gtab + max_blocks * 48;
  uint32_t* hi_off = xf + max_sites;                 // per i: global offset of the high local bits
  uint32_t* hi_sw = hi_off + (1u << (k - 8));        // per i: hsw(i << 8)

  for (uint32_t i = threadIdx.x; i < nb; i += NT) sblk[i] = F.blocks[blk0 + i];
  for (uint32_t i = threadIdx.x; i < ng; i += NT) {
    FGroup g = F.groups[grp0 + i];
    g.blk_begin -= blk0;
    g.blk_end -= blk0;
    sgrp[i] = g;
  }
  for (uint32_t i = threadIdx.x; i < (1u << (k - 8)); i += NT) {
    hi_off[i] = static_cast<uint32_t>(pdep_positions(i, spd.lq + 8, k - 8));
    hi_sw[i] = hsw_slow(i << 8);
  }
  if (threadIdx.x == 0)
    for (unsigned q = 0, jj = 0; q < n; ++q)
      if (!((spd.lmask >> q) & 1)) hpos[jj++] = static_cast<uint8_t>(q);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb * 16; i += NT) bmats[i] = F.mats[uint64_t{sblk[i / 16].mat} * 16 + i % 16];
  // hexad-base tables: hsw(base(h)) = lo[h & 15] ^ hi[h >> 4]
  for (uint32_t x = threadIdx.x; x < ng * 48; x += NT) {
    const uint32_t gi = x / 48, e = x % 48;
    const FGroup G = sgrp[gi];
    const uint32_t h = e < 16 ? e : (e - 16) << 4;
    gtab[x] = hsw_slow(ins0(ins0(ins0(ins0(h, G.g[0]), G.g[1]), G.g[2]), G.g[3]));
  }
  const uint32_t lo_part = static_cast<uint32_t>(pdep_positions(threadIdx.x, spd.lq, 8));
  const uint32_t lo_sw = hsw_slow(threadIdx.x);
  const uint32_t tile_s = static_cast<uint32_t>(__cvta_generic_to_shared(bufs));
  const uint64_t units = S * tiles;
  const uint64_t u_begin = units * blockIdx.x / gridDim.x, u_end = units * (blockIdx.x + 1) / gridDim.x;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned t = lane >> 2, j = lane & 3;
  const uint32_t hexads = L >> 4;
  const uint32_t nhi = 1u << (k - 8);

  // cp.async of unit u's tile into buffer b (one commit group)
  auto fetch = [&](uint64_t u, uint32_t b) {
    const uint64_t s = u / tiles, tt = u % tiles;
    const double2* tb = state + (s << n) + pdep_positions(tt, hpos, n - k);
    const uint32_t dst = tile_s + b * L * 16;
    for (uint32_t i = 0; i < nhi; ++i)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * (lo_sw ^ hi_sw[i])),
                   "l"(tb + (lo_part | hi_off[i])));
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();
  if (!first && u_begin < u_end) fetch(u_begin, 0);
  uint64_t cur_shot = ~uint64_t{0};
  for (uint64_t u = u_begin; u < u_end; ++u) {
    const uint32_t b = static_cast<uint32_t>((u - u_begin) & 1);
    double2* buf = bufs + b * L;
    const uint64_t s = u / tiles, tt = u % tiles;
    if (s != cur_shot) {  // this shot's matrices (warp 0; see fused_pass_kernel)
      cur_shot = s;
      __syncthreads();  // the previous unit's compute no longer reads slots / ents
      if (threadIdx.x < 32) {
        const uint8_t* sel = pauli_sel + s * num_pauli;
        uint32_t slot = 0, nx = 0;
        for (uint32_t bb = 0; bb < nb; ++bb) {
          const FBlock B = sblk[bb];
          FEntry ent{static_cast<uint32_t>(bmats + bb * 16 - tile), static_cast<uint16_t>(nx), 0};
          double2* R = nullptr;
          for (uint32_t c0 = B.site_begin; c0 < B.site_end; c0 += 32) {
            const uint32_t si = c0 + lane;
            uint32_t qi = kNoQ;
            if (si < B.site_end) {
              const FSite st = F.sites[si];
              qi = F.qidx[st.qbase + sel[st.site]];
            }
            unsigned noisy = __ballot_sync(0xffffffffu, qi != kNoQ);
            while (noisy) {
              const unsigned l = __ffs(noisy) - 1;
              noisy &= noisy - 1;
              const uint32_t q = __shfl_sync(0xffffffffu, qi, l);
              if (!R && ent.xcount == 0 && slot < kFusedSlots) {
                R = slots + 16 * slot++;
                if (lane < 16) R[lane] = bmats[bb * 16 + lane];
                __syncwarp();
                ent.src = static_cast<uint32_t>(R - tile);
              }
              if (R) {
                double2 v = make_double2(0.0, 0.0);
                if (lane < 16) {
                  const double2* Q = F.mats + uint64_t{q} * 16;
                  const unsigned r = lane >> 2, c = lane & 3;
#pragma unroll
                  for (unsigned jj = 0; jj < 4; ++jj) v = cfma(Q[r * 4 + jj], R[jj * 4 + c], v);
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
          if (lane == 0) ents[bb] = ent;
        }
      }
    }
    double2* tbase = state + (s << n) + pdep_positions(tt, hpos, n - k);
    if (first) {
      const bool origin = (tbase == state + (s << n));
      for (uint32_t i = 0; i < nhi; ++i)
        buf[lo_sw ^ hi_sw[i]] = make_double2((origin && (lo_part | hi_off[i]) == 0) ? 1.0 : 0.0, 0.0);
    } else {
      if (u + 1 < u_end) {
        fetch(u + 1, b ^ 1);  // next unit's tile, in flight during this one
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
    }
    __syncthreads();
    for (uint32_t gi = 0; gi < ng; ++gi) {
      const FGroup G = sgrp[gi];
      const uint32_t* tab = gtab + gi * 48;
      uint32_t tg[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) tg[i] = hsw_slow(1u << G.g[i]);
      if (!MMA) {  // FMA build: one hexad per thread, all 16 amplitudes in registers
        for (uint32_t h = threadIdx.x; h < hexads; h += NT) {
          const uint32_t sb = tab[h & 15] ^ tab[16 + (h >> 4)];
          double2 a[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            a[e] = buf[sb ^ ((e & 1) ? tg[0] : 0u) ^ ((e & 2) ? tg[1] : 0u) ^ ((e & 4) ? tg[2] : 0u) ^
                       ((e & 8) ? tg[3] : 0u)];
          for (uint32_t bb = G.blk_begin; bb < G.blk_end; ++bb) {
            const FEntry ent = ents[bb];
            const unsigned gb = sblk[bb].gb0 * 4u + sblk[bb].gb1;
            double2 m[16];
            load_mat(m, tile + ent.src);
            apply_hexad_dyn(a, m, gb >> 2, gb & 3);
            for (uint32_t x = 0; x < ent.xcount; ++x) {
              load_mat(m, F.mats + uint64_t{xf[ent.xbegin + x]} * 16);
              apply_hexad_dyn(a, m, gb >> 2, gb & 3);
            }
          }
#pragma unroll
          for (int e = 0; e < 16; ++e)
            buf[sb ^ ((e & 1) ? tg[0] : 0u) ^ ((e & 2) ? tg[1] : 0u) ^ ((e & 4) ? tg[2] : 0u) ^
                ((e & 8) ? tg[3] : 0u)] = a[e];
        }
        __syncthreads();
        continue;
      }
      const uint32_t lin = ((j & 1) ? tg[G.init[0]] : 0u) ^ ((j & 2) ? tg[G.init[1]] : 0u);
      const uint32_t r0i = tg[G.init[2]], r1i = tg[G.init[3]];
      const uint32_t lfn = ((j & 1) ? tg[G.fin[0]] : 0u) ^ ((j & 2) ? tg[G.fin[1]] : 0u);
      const uint32_t r0f = tg[G.fin[2]], r1f = tg[G.fin[3]];
      for (uint32_t hb = warp * 32 + t * 4; hb < hexads; hb += NT) {
        double2 a[16];
        uint32_t sb[4];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) sb[hh] = tab[(hb + hh) & 15] ^ tab[16 + ((hb + hh) >> 4)];
#pragma unroll
        for (int r = 0; r < 16; ++r)
          a[r] = buf[sb[r >> 2] ^ lin ^ ((r & 1) ? r0i : 0u) ^ ((r & 2) ? r1i : 0u)];
        for (uint32_t bb = G.blk_begin; bb < G.blk_end; ++bb) {
          const FBlock B = sblk[bb];
          if (B.xch & 0x08) mma_exchange_dyn(a, j, B.xch);  // nibble: valid | p << 1 | q
          if (B.xch & 0x80) mma_exchange_dyn(a, j, B.xch >> 4);
          const FEntry ent = ents[bb];
          mma_apply(a, tile + ent.src, t, j, B.perm);
          for (uint32_t x = 0; x < ent.xcount; ++x)
            mma_apply(a, F.mats + uint64_t{xf[ent.xbegin + x]} * 16, t, j, B.perm);
        }
#pragma unroll
        for (int r = 0; r < 16; ++r)
          buf[sb[r >> 2] ^ lfn ^ ((r & 1) ? r0f : 0u) ^ ((r & 2) ? r1f : 0u)] = a[r];
      }
      __syncthreads();
    }
    for (uint32_t i = 0; i < nhi; ++i) tbase[lo_part | hi_off[i]] = buf[lo_sw ^ hi_sw[i]];
    __syncthreads();  // this buffer is refilled two units later
  }
}

static __global__ void __launch_bounds__(NT, 1)
    fused_pass_mma_kernel(FusedView F, uint32_t pass_index, double2* state, uint64_t S, const uint8_t* pauli_sel,
                          uint32_t num_pauli, uint32_t max_blocks, uint32_t max_sites) {
  fused_pass_db_body<true>(F, pass_index, state, S, pauli_sel, num_pauli, max_blocks, max_sites);
}

// The FMA apply in the double-buffered, one-CTA-per-SM layout (A/B of the
// occupancy / pipelining trade against fused_pass_kernel).
static __global__ void __launch_bounds__(NT, 1)
    fused_pass_db_kernel(FusedView F, uint32_t pass_index, double2* state, uint64_t S, const uint8_t* pauli_sel,
                         uint32_t num_pauli, uint32_t max_blocks, uint32_t max_sites) {
  fused_pass_db_body<false>(F, pass_index, state, S, pauli_sel, num_pauli, max_blocks, max_sites);
}

}  // namespace ssb
