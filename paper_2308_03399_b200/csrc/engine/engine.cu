// shotsim_b200 engine: device program upload, the batched executors and the
// device half of the C ABI. Host control only sequences launches on the
// engine's stream; all state lives in HBM / shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../capi_internal.hpp"
#include "fused.cuh"
#include "kernels.cuh"

namespace ssb {

#define CK(expr)                                                                          \
  do {                                                                                    \
    const cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// resident_warp.cu: the resident kernel with one-warp CTAs (small states).
int launch_resident_warp(const void* view, uint64_t seed, uint64_t shot_begin, uint64_t count, uint64_t* values,
                         int* err, cudaStream_t stream, size_t smem, int num_sms, void* exp);

// specialise.cpp: the shape-specialised tile-pass kernel for a plan, or null.
const void* specialised_tile_kernel(const HostDevProgram& h);
// specialise.cpp: whether that kernel double-buffers its tiles (SSB_TILE_DB).
bool specialised_tile_double_buffered();
// fused_jit.cpp: per pass the specialised fused kernel, or null.
std::vector<const void*> fused_jit_kernels(const FusedPlan& f, std::string* log);

// Device copy of one program (+ its pass plan for one tile size).
struct DevProgram {
  HostDevProgram host;  // with passes planned for tile_k
  std::vector<void*> allocs;
  ProgView view{};
  uint32_t* pauli_site_ops = nullptr;
  uint32_t num_pauli = 0;
  // Shared noiseless trunk (streamed plans without specials, Kraus or
  // conditions): per Pauli site the pass that applies it, and a Pauli-draw row
  // of identity terms (the trunk's own draws).
  bool trunk_ok = false;
  uint16_t* site_pass = nullptr;
  uint8_t* ident_row = nullptr;
  // Fused-matrix plan (fused.cpp), built on first use of fused_matrices.
  bool fused_tried = false;
  FusedPlan fplan;
  FusedView fview{};
  size_t fsmem = 0;
  // Per pass the run-time specialised fused kernel (fused_jit.cpp) or null.
  bool fjit_tried = false;
  std::vector<const void*> fjit;
  // The arrays come from the device's stream-ordered pool on the engine's
  // stream: freeing them (a program destroyed while the engine lives) returns
  // them to the pool without a device-wide synchronisation — plain cudaFree
  // here took up to ~200 ms now and then on the plugin path, which lowers
  // and destroys a program on every run.
  cudaStream_t stream = nullptr;
  ~DevProgram() {
    for (void* p : allocs) cudaFreeAsync(p, stream);
  }
};

}  // namespace ssb

struct ssb_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int num_sms = 0;
  size_t smem_optin = 0;
  int* err = nullptr;
  unsigned long long* serial_chunks = nullptr;  // sampling chunks replayed sequentially
  unsigned* bad_op = nullptr;                   // check_norms: first op whose norm drifted
  // Device copies of programs, keyed by (program uid, plan). Entries are
  // evicted when their ssb_program is destroyed (ssb::evict_program).
  std::mutex programs_mu;
  std::map<std::pair<uint64_t, unsigned>, std::unique_ptr<ssb::DevProgram>> programs;
  std::map<std::string, std::pair<void*, size_t>> scratch;
  std::map<std::string, std::pair<void*, size_t>> host_scratch;  // pinned
  uint64_t launches = 0;
};

struct ssb_batch {
  ssb_engine* engine;
  const ssb_program* program;
  uint64_t size, seed;
  uint64_t* ids = nullptr;
  double2* state = nullptr;
  uint64_t* cregs = nullptr;
  uint64_t dispatches = 0;
};

namespace ssb {

namespace {

constexpr unsigned kResidentMaxDefault = 13;
constexpr unsigned kTileDefault = 12;

void* scratch(ssb_engine* E, const char* name, size_t bytes) {
  auto& slot = E->scratch[name];
  if (slot.second < bytes) {
    if (slot.first) CK(cudaFree(slot.first));
    slot.first = nullptr;
    slot.second = 0;
    CK(cudaMalloc(&slot.first, bytes));
    slot.second = bytes;
  }
  return slot.first;
}

void* engine_scratch(void* ctx, const char* name, size_t bytes) {
  return scratch(static_cast<ssb_engine*>(ctx), name, bytes);
}

void* engine_grow(void* ctx, const char* name, size_t bytes, size_t keep) {
  ssb_engine* E = static_cast<ssb_engine*>(ctx);
  auto& slot = E->scratch[name];
  if (slot.second >= bytes) return slot.first;
  void* np = nullptr;
  CK(cudaMalloc(&np, bytes));
  if (slot.first && keep) CK(cudaMemcpyAsync(np, slot.first, std::min(keep, slot.second), cudaMemcpyDeviceToDevice, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  if (slot.first) CK(cudaFree(slot.first));
  slot.first = np;
  slot.second = bytes;
  return np;
}

void* engine_host(void* ctx, const char* name, size_t bytes) {
  ssb_engine* E = static_cast<ssb_engine*>(ctx);
  auto& slot = E->host_scratch[name];
  if (slot.second < bytes) {
    CK(cudaStreamSynchronize(E->stream));
    if (slot.first) CK(cudaFreeHost(slot.first));
    slot.first = nullptr;
    slot.second = 0;
    const size_t cap = std::max<size_t>(bytes, 1 << 16) * 2;
    CK(cudaMallocHost(&slot.first, cap));
    slot.second = cap;
  }
  return slot.first;
}

template <class T>
T* upload(DevProgram& d, const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  void* p = nullptr;
  CK(cudaMallocAsync(&p, v.size() * sizeof(T), d.stream));
  d.allocs.push_back(p);
  // (pageable source: the copy has completed when the call returns)
  CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, d.stream));
  return static_cast<T*>(p);
}

// tile_k == 0 selects the resident plan (whole program in one pass, k = n).
// Live engines, so that destroying a program evicts its device copies.
std::mutex g_engines_mu;
std::set<ssb_engine*> g_engines;

DevProgram& device_program(ssb_engine* E, const ssb_program* prog, unsigned tile_k) {
  const auto key = std::make_pair(prog->uid, tile_k);
  std::lock_guard<std::mutex> lk(E->programs_mu);
  auto it = E->programs.find(key);
  if (it != E->programs.end()) return *it->second;
  auto d = std::make_unique<DevProgram>();
  d->stream = E->stream;
  d->host = prog->dev;
  if (tile_k == 0) plan_resident(d->host);
  else plan_passes(d->host, tile_k);
  const HostDevProgram& h = d->host;
  ProgView& v = d->view;
  v.ops = upload(*d, h.ops);
  v.terms = upload(*d, h.terms);
  v.channels = upload(*d, h.channels);
  v.mats = reinterpret_cast<const double2*>(upload(*d, h.mats));
  v.scaled_cls = upload(*d, h.scaled_cls);
  v.sample_qubits = upload(*d, h.sample_qubits);
  v.write_clbit = upload(*d, h.write_clbit);
  v.write_pos = upload(*d, h.write_pos);
  v.passes = upload(*d, h.passes);
  v.items = upload(*d, h.items);
  v.pass_ops = upload(*d, h.pass_ops);
  v.uops = upload(*d, h.uops);
  v.uop_mats = reinterpret_cast<const double2*>(upload(*d, h.uop_mats));
  v.n = h.n;
  v.end = h.end;
  v.nsample = static_cast<uint32_t>(h.sample_qubits.size());
  v.nwrites = static_cast<uint32_t>(h.write_clbit.size());
  v.num_events = h.num_events;
  v.eligible = h.eligible;
  v.sample_identity = h.sample_identity;
  std::vector<uint32_t> sites;
  for (uint32_t i = 0; i < h.ops.size(); ++i)
    if (h.ops[i].kind == K_PAULI) sites.push_back(i);
  d->num_pauli = static_cast<uint32_t>(sites.size());
  d->pauli_site_ops = upload(*d, sites);
  v.pauli_site_ops = d->pauli_site_ops;
  v.num_pauli = d->num_pauli;
  if (tile_k && !h.passes.empty() && h.passes.size() < 0xFFFF) {
    bool ok = h.eligible && !h.steps.empty() && h.steps.back().kind == S_SAMPLE;
    for (const Step& s : h.steps) ok &= s.kind == S_PASS || s.kind == S_SAMPLE;
    std::vector<uint16_t> sp(d->num_pauli, 0xFFFF);
    for (size_t p = 0; p < h.passes.size(); ++p) {
      const size_t e = p + 1 < h.passes.size() ? h.passes[p + 1].po_begin : h.pass_ops.size();
      for (size_t i = h.passes[p].po_begin; i < e; ++i) {
        const DevOp& o = h.ops[h.pass_ops[i].op];
        ok &= !o.has_cond;
        if (o.kind == K_PAULI) sp[o.site] = static_cast<uint16_t>(p);
      }
    }
    std::vector<uint8_t> ident(d->num_pauli, 0);
    for (uint32_t s = 0; s < d->num_pauli; ++s) {
      ok &= sp[s] != 0xFFFF;
      const DevOp& o = h.ops[sites[s]];
      for (uint32_t t = 0; t < o.count; ++t)
        if (h.terms[o.aux + t].identity) {
          ident[s] = static_cast<uint8_t>(t);
          break;
        }
    }
    if (ok) {
      d->trunk_ok = true;
      d->site_pass = upload(*d, sp);
      d->ident_row = upload(*d, ident);
    }
  }
  auto& ref = *d;
  E->programs.emplace(key, std::move(d));
  return ref;
}

unsigned grid_for(uint64_t work, unsigned threads = NT) {
  const uint64_t g = (work + threads - 1) / threads;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(g, 1u << 30)));
}

void launched(ssb_engine* E) {
  ++E->launches;
  CK(cudaGetLastError());
}

void check_device_error(ssb_engine* E) {
  int h = 0;
  CK(cudaMemcpyAsync(&h, E->err, sizeof(int), cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  if (h == DEV_DEGENERATE) {
    CK(cudaMemsetAsync(E->err, 0, sizeof(int), E->stream));
    throw shotsim::DegenerateDistribution("measured distribution sums to zero or branch has zero probability");
  }
  if (h == DEV_NORM) {  // exec_batch.cpp:217-224
    unsigned op = 0;
    CK(cudaMemcpyAsync(&op, E->bad_op, sizeof op, cudaMemcpyDeviceToHost, E->stream));
    CK(cudaMemsetAsync(E->err, 0, sizeof(int), E->stream));
    CK(cudaMemsetAsync(E->bad_op, 0xFF, sizeof(unsigned), E->stream));
    CK(cudaStreamSynchronize(E->stream));
    throw std::runtime_error("batch segment norm drifted after op " + std::to_string(op));
  }
}

uint64_t mem_limit(const ssb_run_options* o) {
  if (o && o->mem_limit_bytes) return o->mem_limit_bytes;
  if (const char* env = std::getenv("SHOTSIM_MEM_LIMIT_BYTES")) {
    const uint64_t v = std::strtoull(env, nullptr, 10);
    if (v > 0) return v;
  }
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  return static_cast<uint64_t>(free_b * 0.8);
}

// ---- op-at-a-time batched ops (shared by the streamed executor and the
// operator-level ABI). Shots [0,S) of `state`; ids == nullptr means ids are
// begin + s. u: optional per-shot draws (device).
struct SegCtx {
  double2* state;
  uint64_t S;
  uint64_t seed;
  const uint64_t* ids;
  uint64_t begin;
  const double* u;
  uint64_t* cregs;
  SegCtx sub(uint64_t off, uint64_t len, unsigned n) const {
    return {state + (off << n), len, seed, ids ? ids + off : nullptr, begin + off, u ? u + off : nullptr, cregs + off};
  }
};

void run_reduction(ssb_engine* E, const SegCtx& c, const RedSpec& R, int leaves_tree, const uint8_t* active,
                   double* val) {
  double* part = static_cast<double*>(scratch(E, "part", c.S * R.nq * R.nb * sizeof(double)));
  launch_reduce(E->stream, c.state, c.S, R, active, part);
  launched(E);
  g_finish_kernel<<<static_cast<unsigned>(std::min<uint64_t>(c.S * R.nq, 1u << 20)), NT, 0, E->stream>>>(c.S, R.nq, R.nb, leaves_tree, active, part, val);
  launched(E);
}

// 512-block outcome reduction spec over qubits q (k of them).
RedSpec outcome_spec(unsigned n, const uint8_t* q, unsigned k) {
  RedSpec R{};
  R.mode = R_OUTCOME;
  R.n = n;
  R.k = k;
  for (unsigned i = 0; i < k; ++i) R.q[i] = R.sorted[i] = q[i];
  std::sort(R.sorted, R.sorted + k);
  const uint64_t G = uint64_t{1} << (n - k);
  R.nq = static_cast<uint32_t>(uint64_t{1} << k);
  R.nb = G <= SUM_BLOCK ? 1 : G / SUM_BLOCK;
  R.blk = G <= SUM_BLOCK ? G : SUM_BLOCK;
  return R;
}

// Kraus probabilities: expval_matrix1_scalar (512-pair blocks + pairwise) for
// 1q channels, expval_generic (per-group sums; leaves of 8 + tree) for 2q.
RedSpec kraus_spec(const ProgView& P, const DevOp& op, const DevChannel& ch, unsigned n) {
  RedSpec R{};
  R.n = n;
  R.k = ch.arity;
  for (unsigned i = 0; i < ch.arity; ++i) R.q[i] = R.sorted[i] = op.q[i];
  std::sort(R.sorted, R.sorted + ch.arity);
  R.nq = ch.nmat;
  R.mats = P.mats + 16 * ch.mat_begin;
  R.cls = P.scaled_cls + ch.mat_begin;
  if (ch.arity == 1) {
    R.mode = R_EXPVAL1;
    const uint64_t pairs = uint64_t{1} << (n - 1);
    R.nb = pairs <= SUM_BLOCK ? 1 : pairs / SUM_BLOCK;
    R.blk = pairs <= SUM_BLOCK ? pairs : SUM_BLOCK;
  } else {
    R.mode = R_EXPVAL2;
    const uint64_t G = uint64_t{1} << (n - 2);
    R.blk = G <= 8 ? G : 8;
    R.nb = G / R.blk;
  }
  return R;
}

uint64_t chunk_for(uint64_t S, uint64_t per_shot_bytes) {
  const uint64_t cap = uint64_t{1} << 30;
  return std::max<uint64_t>(1, std::min<uint64_t>(S, cap / std::max<uint64_t>(1, per_shot_bytes)));
}

// Returns the number of logical dispatches in the reference's accounting
// (README.md:102-107) for the operator-level ABI.
uint64_t apply_op(ssb_engine* E, DevProgram& dp, uint32_t op_index, const SegCtx& c, bool count_identity_skip) {
  const DevOp op = dp.host.ops[op_index];
  const unsigned n = dp.host.n;
  const ProgView& P = dp.view;
  switch (op.kind) {
    case K_BARRIER: return 0;
    case K_GATE: {
      if (!op.skip) {
        const uint64_t work = c.S << (n - op.nq);
        if (op.nq == 1) g_gate_kernel<1><<<grid_for(work), NT, 0, E->stream>>>(c.state, c.S, n, op, P.mats, c.cregs);
        else g_gate_kernel<2><<<grid_for(work), NT, 0, E->stream>>>(c.state, c.S, n, op, P.mats, c.cregs);
        launched(E);
      }
      return 1;
    }
    case K_PAULI: {
      int* sel = static_cast<int*>(scratch(E, "sel", c.S * sizeof(int)));
      g_pauli_decide_kernel<<<grid_for(c.S), NT, 0, E->stream>>>(P, op, c.S, c.seed, c.ids, c.begin, c.u, c.cregs, sel);
      launched(E);
      if (count_identity_skip) {  // the reference issues no dispatch when every shot drew identity
        std::vector<int> h(c.S);
        CK(cudaMemcpyAsync(h.data(), sel, c.S * sizeof(int), cudaMemcpyDeviceToHost, E->stream));
        CK(cudaStreamSynchronize(E->stream));
        if (std::none_of(h.begin(), h.end(), [](int t) { return t >= 0; })) return 0;
      }
      g_pauli_apply_kernel<<<grid_for(c.S << (n - 1)), NT, 0, E->stream>>>(c.state, c.S, n, P.terms + op.aux, sel);
      launched(E);
      return 1;
    }
    case K_KRAUS: {
      const DevChannel ch = dp.host.channels[op.aux];
      const RedSpec R = kraus_spec(P, op, ch, n);
      const int tree = ch.arity == 2;
      const uint64_t chunk = chunk_for(c.S, (R.nq * R.nb + R.nq) * sizeof(double) + 16 * 16 + 32);
      for (uint64_t off = 0; off < c.S; off += chunk) {
        const SegCtx cc = c.sub(off, std::min(chunk, c.S - off), n);
        uint8_t* active = static_cast<uint8_t*>(scratch(E, "active", cc.S));
        double* val = static_cast<double*>(scratch(E, "val", cc.S * R.nq * sizeof(double)));
        double2* scaled = static_cast<double2*>(scratch(E, "kscaled", cc.S * 16 * sizeof(double2)));
        uint64_t* cls = static_cast<uint64_t*>(scratch(E, "kcls", cc.S * sizeof(uint64_t)));
        int* chosen = static_cast<int*>(scratch(E, "kchosen", cc.S * sizeof(int)));
        g_active_kernel<<<grid_for(cc.S), NT, 0, E->stream>>>(op, cc.S, cc.cregs, active);
        launched(E);
        run_reduction(E, cc, R, tree, active, val);
        g_kraus_decide_kernel<<<grid_for(cc.S), NT, 0, E->stream>>>(P, op, cc.S, cc.seed, cc.ids, cc.begin, cc.u, active,
                                                                    val, scaled, cls, chosen, E->err);
        launched(E);
        const uint64_t work = cc.S << (n - ch.arity);
        if (ch.arity == 1)
          g_kraus_apply_kernel<1><<<grid_for(work), NT, 0, E->stream>>>(cc.state, cc.S, n, op, scaled, cls, chosen);
        else
          g_kraus_apply_kernel<2><<<grid_for(work), NT, 0, E->stream>>>(cc.state, cc.S, n, op, scaled, cls, chosen);
        launched(E);
      }
      return 2ull * ch.nmat;
    }
    case K_MEASURE:
    case K_RESET: {
      const RedSpec R = outcome_spec(n, op.q, op.nq);
      const uint64_t chunk = chunk_for(c.S, (R.nq * R.nb + R.nq) * sizeof(double) + 32);
      for (uint64_t off = 0; off < c.S; off += chunk) {
        const SegCtx cc = c.sub(off, std::min(chunk, c.S - off), n);
        uint8_t* active = static_cast<uint8_t*>(scratch(E, "active", cc.S));
        double* val = static_cast<double*>(scratch(E, "val", cc.S * R.nq * sizeof(double)));
        int64_t* outcome = static_cast<int64_t*>(scratch(E, "outcome", cc.S * sizeof(int64_t)));
        double* inv = static_cast<double*>(scratch(E, "inv", cc.S * sizeof(double)));
        g_active_kernel<<<grid_for(cc.S), NT, 0, E->stream>>>(op, cc.S, cc.cregs, active);
        launched(E);
        run_reduction(E, cc, R, 0, active, val);
        g_measure_decide_kernel<<<grid_for(cc.S), NT, 0, E->stream>>>(op, cc.S, cc.seed, cc.ids, cc.begin, cc.u, active,
                                                                      val, cc.cregs, outcome, inv, E->err);
        launched(E);
        g_collapse_kernel<<<grid_for(cc.S << (n - 1)), NT, 0, E->stream>>>(cc.state, cc.S, n, op, outcome, inv);
        launched(E);
      }
      return 2ull * R.nq + 1;
    }
  }
  return 0;
}

// Test hook: SHOTSIM_B200_SAMPLE_SERIAL=1 replays every sampling chunk with the
// sequential adds (the exact-advance path off).
int sample_force_serial() {
  const char* v = std::getenv("SHOTSIM_B200_SAMPLE_SERIAL");
  return v && *v && *v != '0';
}

// Kraus site probabilities + per-shot choice for a whole wave (the streamed
// executor's S_KRAUS_DECIDE step): scaled[s] = M_sel / sqrt(p_sel) and its
// classes for the apply micro-op at the head of the next tile pass; inactive
// shots (failed condition) get chosen = -1 and their apply is compacted away.
// epi: matrix 0's partial sums for this site, computed by the preceding tile
// pass's epilogue (PassDesc::epi_*), or null.
void kraus_decide_wave(ssb_engine* E, DevProgram& dp, uint32_t op_index, const SegCtx& c, double2* scaled,
                       uint64_t* cls, int* chosen, const double* epi) {
  const DevOp op = dp.host.ops[op_index];
  const unsigned n = dp.host.n;
  const ProgView& P = dp.view;
  const DevChannel ch = dp.host.channels[op.aux];
  uint8_t* pending = static_cast<uint8_t*>(scratch(E, "kpending", c.S));
  double* cum = static_cast<double*>(scratch(E, "kcum", c.S * sizeof(double)));
  g_kraus_begin_kernel<<<grid_for(c.S), NT, 0, E->stream>>>(op, c.S, c.cregs, pending, cum, chosen);
  launched(E);
  for (uint32_t mi = 0; mi < ch.nmat; ++mi) {
    RedSpec R = kraus_spec(P, op, ch, n);
    R.nq = 1;  // matrix mi only
    R.mats += 16 * mi;
    R.cls += mi;
    if (mi == 0 && epi) {  // partials already in HBM: only the tree above them
      double* val = static_cast<double*>(scratch(E, "val", c.S * sizeof(double)));
      g_finish_kernel<<<static_cast<unsigned>(std::min<uint64_t>(c.S, 1u << 20)), NT, 0, E->stream>>>(
          c.S, 1, R.nb, ch.arity == 2, pending, const_cast<double*>(epi), val);
      launched(E);
      const char* dbg = std::getenv("SHOTSIM_B200_EPI_CHECK");
      if (!(dbg && *dbg == '1')) {
        g_kraus_step_kernel<<<grid_for(c.S), NT, 0, E->stream>>>(P, op, 0, c.S, c.seed, c.ids, c.begin, c.u, pending,
                                                                 val, cum, scaled, cls, chosen, E->err);
        launched(E);
        continue;
      }
      // debug: compare with the reduction kernels, then continue on their values
      std::vector<double> a(c.S), pa(c.S * R.nb);
      CK(cudaMemcpy(a.data(), val, c.S * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(pa.data(), epi, c.S * R.nb * 8, cudaMemcpyDeviceToHost));
      double* part = static_cast<double*>(scratch(E, "part_dbg", c.S * R.nb * sizeof(double)));
      double* v2 = static_cast<double*>(scratch(E, "val_dbg", c.S * sizeof(double)));
      launch_reduce(E->stream, c.state, c.S, R, pending, part);
      g_finish_kernel<<<static_cast<unsigned>(std::min<uint64_t>(c.S, 1u << 20)), NT, 0, E->stream>>>(
          c.S, 1, R.nb, ch.arity == 2, pending, part, v2);
      std::vector<double> b(c.S), pb(c.S * R.nb);
      CK(cudaMemcpy(b.data(), v2, c.S * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(pb.data(), part, c.S * R.nb * 8, cudaMemcpyDeviceToHost));
      uint64_t bad = 0, pbad = 0, first = ~0ull;
      for (uint64_t i = 0; i < c.S; ++i) bad += a[i] != b[i];
      for (uint64_t i = 0; i < c.S * R.nb; ++i)
        if (pa[i] != pb[i]) {
          ++pbad;
          if (first == ~0ull) first = i;
        }
      std::fprintf(stderr, "epi op %u arity %u q %u,%u: values differ %llu/%llu, partials differ %llu/%llu",
                   op_index, ch.arity, op.q[0], op.q[1], (unsigned long long)bad, (unsigned long long)c.S,
                   (unsigned long long)pbad, (unsigned long long)(c.S * R.nb));
      if (first != ~0ull) std::fprintf(stderr, " first at %llu: %.17g vs %.17g", (unsigned long long)first, pa[first], pb[first]);
      std::fprintf(stderr, "\n");
      g_kraus_step_kernel<<<grid_for(c.S), NT, 0, E->stream>>>(P, op, 0, c.S, c.seed, c.ids, c.begin, c.u, pending,
                                                               v2, cum, scaled, cls, chosen, E->err);
      launched(E);
      continue;
    }
    const uint64_t chunk = chunk_for(c.S, R.nb * sizeof(double) + 16);
    for (uint64_t off = 0; off < c.S; off += chunk) {
      const SegCtx cc = c.sub(off, std::min(chunk, c.S - off), n);
      double* val = static_cast<double*>(scratch(E, "val", cc.S * sizeof(double)));
      run_reduction(E, cc, R, ch.arity == 2, pending + off, val);
      g_kraus_step_kernel<<<grid_for(cc.S), NT, 0, E->stream>>>(P, op, mi, cc.S, cc.seed, cc.ids, cc.begin, cc.u,
                                                                pending + off, val, cum + off, scaled + 16 * off,
                                                                cls + off, chosen + off, E->err);
      launched(E);
    }
  }
}

// Guard band of the fused-matrix mode (sample_exact_kernel): shots whose
// draw lies within the rounding bound of a cumulative boundary are listed.
struct SampleGuard {
  double err = 0.0;              // bound on ||psi_fused - psi_reference||_2; 0: exact run
  unsigned* count = nullptr;     // device counter
  uint64_t* ids = nullptr;       // device list (shot ids), capacity cap
  uint64_t cap = 0;
};

// Waves with at least this many shots per SM use 128-thread sampler CTAs.
constexpr unsigned kSampleSmallCtaShotsPerSm = 8;

void sample_terminal(ssb_engine* E, DevProgram& dp, const SegCtx& c, const SampleGuard& g = SampleGuard{}) {
  const unsigned n = dp.host.n;
  const ProgView& P = dp.view;
  if (P.nsample == n && n >= 12) {
    // Chunked exact parallel sampler (sample_exact_kernel), one CTA per shot.
    for (uint64_t off = 0; off < c.S; off += (1u << 30)) {
      const SegCtx cc = c.sub(off, std::min<uint64_t>(1u << 30, c.S - off), n);
      // many shots: 128-thread CTAs (more shots in flight per SM); fewer: 256;
      // fewer shots than SMs: 512 (each shot's chunk loop gets the threads:
      // C5 107 -> 114 shots/s; SHOTSIM_B200_SAMPLE_FEW_NT=256/1024 for A/B)
      const char* fe = std::getenv("SHOTSIM_B200_SAMPLE_FEW_NT");
      const unsigned few = fe && std::string(fe) == "256" ? 256u : fe && std::string(fe) == "1024" ? 1024u : 512u;
      const unsigned snt = cc.S >= uint64_t{kSampleSmallCtaShotsPerSm} * E->num_sms ? 128u
                           : cc.S >= uint64_t(E->num_sms)                             ? 256u
                                                                                      : few;
      auto launch = [&](auto kern, unsigned nt) {
        kern<<<static_cast<unsigned>(cc.S), nt, 0, E->stream>>>(P, cc.state, cc.S, cc.seed, cc.ids, cc.begin,
                                                               cc.cregs, E->serial_chunks, E->err,
                                                               sample_force_serial(), g.err, g.count, g.ids, g.cap);
      };
      if (snt == 128) launch(sample_exact_kernel<128>, 128);
      else if (snt == 512) launch(sample_exact_kernel<512>, 512);
      else if (snt == 1024) launch(sample_exact_kernel<1024>, 1024);
      else launch(sample_exact_kernel<256>, 256);
      launched(E);
    }
    return;
  }
  if (g.err > 0.0) throw std::logic_error("fused_matrices needs the full-register sampler");
  if (P.nsample == n) {
    g_sample_scan_kernel<<<grid_for(c.S, 128), 128, 0, E->stream>>>(P, c.state, c.S, c.seed, c.ids, c.begin, c.cregs,
                                                                    E->err);
    launched(E);
    return;
  }
  const RedSpec R = outcome_spec(n, dp.host.sample_qubits.data(), P.nsample);
  const uint64_t chunk = chunk_for(c.S, (R.nq * R.nb + R.nq) * sizeof(double));
  for (uint64_t off = 0; off < c.S; off += chunk) {
    const SegCtx cc = c.sub(off, std::min(chunk, c.S - off), n);
    double* val = static_cast<double*>(scratch(E, "val", cc.S * R.nq * sizeof(double)));
    run_reduction(E, cc, R, 0, nullptr, val);
    g_sample_pick_kernel<<<grid_for(cc.S), NT, 0, E->stream>>>(P, val, cc.S, cc.seed, cc.ids, cc.begin, cc.cregs,
                                                               E->err);
    launched(E);
  }
}

// Shared memory of resident_kernel for a resident plan: state | staged
// matrices | micro-ops | compacted segment | reduction scratch | outcome
// probabilities | Pauli draws.
size_t resident_smem(const HostDevProgram& h) {
  const uint64_t A = uint64_t{1} << h.n;
  const uint64_t probs =
      (h.eligible && h.sample_qubits.size() < h.n) ? (uint64_t{1} << h.sample_qubits.size()) + 16 : 16;
  uint32_t sites = 0;
  for (const DevOp& o : h.ops) sites += o.kind == K_PAULI;
  uint64_t staged = 0;
  if (!h.passes.empty()) {
    const PassDesc& pd = h.passes[0];
    staged = uint64_t{pd.mat_count} * sizeof(double2) + 2 * uint64_t{pd.uop_end - pd.uop_begin} * sizeof(Uop);
  }
  return A * sizeof(double2) + staged + (resident_red_doubles() + probs) * sizeof(double) + sites;
}

// Optional per-kernel-class CUDA-event timing (ssb_run_options::profile):
// 0 = fused passes (tile / resident), 1 = special ops, 2 = terminal sampling.
struct KernelTimer {
  bool on = false;
  cudaStream_t stream = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[3];
  void begin(int c) {
    if (!on) return;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, stream));
    ev[c].emplace_back(a, b);
  }
  void end(int c) {
    if (on) CK(cudaEventRecord(ev[c].back().second, stream));
  }
  void collect(ssb_stats* st) {
    if (!on) return;
    CK(cudaStreamSynchronize(stream));
    double secs[3] = {0, 0, 0};
    for (int c = 0; c < 3; ++c)
      for (auto& [a, b] : ev[c]) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        secs[c] += ms * 1e-3;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    if (st) {
      st->pass_seconds = secs[0];
      st->pass_launches = ev[0].size();
      st->special_seconds = secs[1];
      st->sample_seconds = secs[2];
    }
  }
};

// Registers of at least this many qubits run fused mode with 11-qubit tiles
// (with the local-set search of plan_fused: C2 71.5k vs 68.5k shots/s at 12,
// C5 102.7 vs 97.8; profiles/r02/fused_variants.log).
constexpr unsigned kFusedSmallTileMinQubits = 12;

struct RunConfig {
  unsigned resident_max = kResidentMaxDefault;
  unsigned tile_k = kTileDefault;
};

RunConfig config_of(const ssb_run_options* o) {
  RunConfig rc;
  if (o && o->resident_max_qubits) rc.resident_max = o->resident_max_qubits;
  if (o && o->tile_qubits) rc.tile_k = std::max(3u, std::min(13u, o->tile_qubits));
  return rc;
}

// Debug export (ssb_run_options::states_out): wave slots [0, S) -> host.
void export_states(ssb_engine* E, const ssb_run_options* opts, const double2* state, uint64_t w0, uint64_t S,
                   unsigned n) {
  if (!opts || !opts->states_out) return;
  CK(cudaMemcpyAsync(opts->states_out + 2 * (w0 << n), state, (S << n) * sizeof(double2), cudaMemcpyDeviceToHost,
                     E->stream));
  CK(cudaStreamSynchronize(E->stream));
}

uint64_t wave_for(const ssb_run_options* opts, uint64_t count, uint64_t seg, uint64_t limit) {
  const uint64_t wave = opts && opts->max_batch_size
                            ? opts->max_batch_size
                            : std::max<uint64_t>(1, std::min<uint64_t>(limit, uint64_t{16} << 30) / seg);
  const uint64_t largest = std::min(wave, count);
  if (largest * seg > limit)
    throw shotsim::CapacityError("batch of " + std::to_string(largest) + " shots needs " +
                                 std::to_string(largest * seg) +
                                 " bytes; lower max_batch_size or raise the memory limit");
  return largest;
}

// check_norms (exec_batch.cpp:200-227): BatchState::run op at a time with the
// norm of every segment checked after every non-barrier op. A debug mode: the
// per-op kernels instead of the fused passes, same arithmetic and decisions.
void run_batch_checked(ssb_engine* E, const ssb_program* prog, uint64_t shot_begin, uint64_t count, uint64_t seed,
                       const ssb_run_options* opts, uint64_t* values_dev, ssb_stats* stats) {
  DevProgram& dp = device_program(E, prog, kTileDefault);
  const unsigned n = dp.host.n;
  const uint64_t seg = (uint64_t{1} << n) * sizeof(double2);
  const uint64_t wave = wave_for(opts, count, seg, mem_limit(opts));
  double2* state = static_cast<double2*>(scratch(E, "state", wave * seg));
  uint64_t waves = 0;
  for (uint64_t w0 = 0; w0 < count; w0 += wave, ++waves) {
    const uint64_t S = std::min(wave, count - w0);
    g_init_kernel<<<grid_for(S << n), NT, 0, E->stream>>>(state, S, n, values_dev + w0);
    launched(E);
    const SegCtx c{state, S, seed, nullptr, shot_begin + w0, nullptr, values_dev + w0};
    for (uint32_t i = 0; i < dp.host.end; ++i) {
      apply_op(E, dp, i, c, false);
      if (dp.host.ops[i].kind == K_BARRIER) continue;
      g_norm_check_kernel<<<static_cast<unsigned>(std::min<uint64_t>(S, 1u << 20)), NT, 0, E->stream>>>(
          state, S, n, i, E->err, E->bad_op);
      launched(E);
    }
    export_states(E, opts, state, w0, S, n);
    if (dp.host.eligible) sample_terminal(E, dp, c);
  }
  if (stats) {
    stats->peak_states = wave;
    stats->passes = waves;
  }
}

void run_batch_device(ssb_engine* E, const ssb_program* prog, uint64_t shot_begin, uint64_t count, uint64_t seed,
                      const ssb_run_options* opts, uint64_t* values_dev, ssb_stats* stats);

// Fused-matrix plan of a streamed program (fused.cpp), uploaded once.
bool fused_ready(ssb_engine* E, DevProgram& dp) {
  if (dp.fused_tried) return dp.fplan.ok;
  dp.fused_tried = true;
  FusedPlan& f = dp.fplan;
  // Register-group size: 4 (16-amplitude hexads) or 3 (8-amplitude octads,
  // half the registers per thread, twice the CTAs per SM);
  // SHOTSIM_B200_FUSED_GROUP overrides the default. The tensor-core build
  // needs 4.
  unsigned gq = kFusedGroupDefault;
  if (const char* v = std::getenv("SHOTSIM_B200_FUSED_GROUP"); v && (*v == '3' || *v == '4')) gq = *v - '0';
  if (const char* v = std::getenv("SHOTSIM_B200_FUSED_MMA"); v && *v && *v != '0') gq = 4;
  f = plan_fused_cached(dp.host, dp.host.tile_k, gq);
  if (f.ok && f.k < 8) {
    f.ok = false;
    f.why = "tile smaller than 8 qubits";
  }
  if (f.ok && dp.host.eligible && dp.host.n < 12) {
    f.ok = false;
    f.why = "fewer than 12 qubits (terminal sampler)";
  }
  if (!f.ok) return false;
  dp.fsmem = fused_smem_bytes(f.k, std::max(1u, f.max_pass_blocks), std::max(1u, f.max_pass_sites));
  if (dp.fsmem > E->smem_optin) {
    f.ok = false;
    f.why = "pass staging exceeds shared memory";
    return false;
  }
  FusedView& v = dp.fview;
  v.passes = upload(dp, f.passes);
  v.groups = upload(dp, f.groups);
  v.blocks = upload(dp, f.blocks);
  v.sites = upload(dp, f.sites);
  v.qidx = upload(dp, f.qidx);
  v.mats = reinterpret_cast<const double2*>(upload(dp, f.mats));
  v.n = dp.host.n;
  return true;
}

// Test hook: SHOTSIM_B200_GUARD_SCALE=x widens the guard band x-fold (forces
// exact replays so their path is exercised).
double guard_scale() {
  const char* v = std::getenv("SHOTSIM_B200_GUARD_SCALE");
  return v && *v ? std::max(1.0, std::strtod(v, nullptr)) : 1.0;
}

// gpu-batch in fused-matrix mode (fused.cuh): per wave the Pauli decisions,
// one fused_pass_kernel per planned pass and the guarded exact sampler; then
// every flagged shot is re-run through the exact executor into its slot.
void run_fused(ssb_engine* E, const ssb_program* prog, DevProgram& dp, uint64_t shot_begin, uint64_t count,
               uint64_t seed, const ssb_run_options* opts, uint64_t* values_dev, ssb_stats* stats, KernelTimer& timer) {
  const FusedPlan& f = dp.fplan;
  const unsigned n = dp.host.n;
  const uint64_t seg = (uint64_t{1} << n) * sizeof(double2);
  const uint64_t tiles = uint64_t{1} << (n - f.k);
  uint64_t wave = wave_for(opts, count, seg, mem_limit(opts));
  wave = std::min<uint64_t>(wave, std::max<uint64_t>(1, (uint64_t{1} << 31) / tiles - 1));
  double2* state = static_cast<double2*>(scratch(E, "state", wave * seg));
  uint8_t* psel = dp.num_pauli ? static_cast<uint8_t*>(scratch(E, "psel", wave * dp.num_pauli)) : nullptr;
  unsigned* gcount = static_cast<unsigned*>(scratch(E, "guard_count", sizeof(unsigned)));
  uint64_t* gids = static_cast<uint64_t*>(scratch(E, "guard_ids", count * sizeof(uint64_t)));
  CK(cudaMemsetAsync(gcount, 0, sizeof(unsigned), E->stream));
  const SampleGuard guard{f.err_bound * guard_scale(), gcount, gids, count};
  // FMA build (default) or, with SHOTSIM_B200_FUSED_MMA=1, the experimental
  // tensor-core (FP64 MMA) build for tiles of 9..13 qubits. The MMA build is
  // correct (same tests) but slower on C2 today: its lane / register bit
  // exchanges cost more issue slots than the tensor core saves.
  const char* mma_env = std::getenv("SHOTSIM_B200_FUSED_MMA");
  const size_t mma_smem = fused_mma_smem_bytes(f.k, std::max(1u, f.max_pass_blocks), std::max(1u, f.max_pass_sites));
  // SHOTSIM_B200_FUSED_DB=1: the FMA apply in the double-buffered one-CTA layout.
  const char* db_env = std::getenv("SHOTSIM_B200_FUSED_DB");
  const bool db_ok = f.k >= 9 && f.k <= kMmaMaxK && mma_smem <= E->smem_optin;
  const bool use_mma = db_ok && f.gq == 4 && (mma_env && *mma_env && *mma_env != '0');
  const bool use_db = db_ok && f.gq == 4 && !use_mma && (db_env && *db_env && *db_env != '0');
  const size_t smem = (use_mma || use_db) ? mma_smem : dp.fsmem;
  // FMA build: 256 threads for 12- and 13-qubit tiles, 128 for 11-qubit ones
  // (one hexad per thread either way).
  // (3-qubit groups: 256 threads, 2^(k-3) octads per tile)
  const unsigned fnt = (use_mma || use_db) ? NT : (f.gq == 4 && f.k <= 10 ? 64u : f.gq == 4 && f.k <= 11 ? 128u : 256u);
  const void* kfn = use_mma              ? reinterpret_cast<const void*>(fused_pass_mma_kernel)
                    : use_db             ? reinterpret_cast<const void*>(fused_pass_db_kernel)
                    : f.gq == 3          ? reinterpret_cast<const void*>(fused_pass_kernel<256, 3>)
                    : fnt == 64          ? reinterpret_cast<const void*>(fused_pass_kernel<64, 4>)
                    : fnt == 128         ? reinterpret_cast<const void*>(fused_pass_kernel<128, 4>)
                                         : reinterpret_cast<const void*>(fused_pass_kernel<256, 4>);
  CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, fnt, smem));
  // SHOTSIM_B200_FUSED_JIT=1: the per-pass specialised kernels (fused_jit.cpp)
  // for the passes that have one (same arithmetic, constant-bank products).
  const char* jit_env = std::getenv("SHOTSIM_B200_FUSED_JIT");
  const bool use_jit = !use_mma && !use_db && f.gq == 4 && (f.k == 11 || f.k == 12) && jit_env && *jit_env &&
                       *jit_env != '0';
  if (use_jit && !dp.fjit_tried) {
    dp.fjit_tried = true;
    std::string log;
    dp.fjit = fused_jit_kernels(f, &log);
    for (const void*& k : dp.fjit)
      if (k && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
                   cudaSuccess) {
        cudaGetLastError();
        k = nullptr;
      }
    if (!log.empty()) std::fprintf(stderr, "shotsim_b200: fused specialisation: %s\n", log.c_str());
  }
  int jit_per_sm = 0;  // the smallest residency over the specialised kernels
  if (use_jit)
    for (const void* k : dp.fjit)
      if (k) {
        int v = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, fnt, smem));
        jit_per_sm = jit_per_sm ? std::min(jit_per_sm, v) : v;
      }
  uint32_t max_blocks = std::max(1u, f.max_pass_blocks), max_sites = std::max(1u, f.max_pass_sites);
  uint64_t waves = 0;
  for (uint64_t w0 = 0; w0 < count; w0 += wave, ++waves) {
    const uint64_t S = std::min(wave, count - w0);
    const SegCtx c{state, S, seed, nullptr, shot_begin + w0, nullptr, values_dev + w0};
    CK(cudaMemsetAsync(c.cregs, 0, S * sizeof(uint64_t), E->stream));
    if (dp.num_pauli) {
      pauli_decide_kernel<<<grid_for(S * dp.num_pauli), NT, 0, E->stream>>>(dp.view, dp.pauli_site_ops, dp.num_pauli,
                                                                           seed, nullptr, c.begin, S, psel);
      launched(E);
    }
    const unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>(S * tiles, uint64_t(std::max(per_sm, 1)) * E->num_sms));
    const unsigned jgrid =
        static_cast<unsigned>(std::min<uint64_t>(S * tiles, uint64_t(std::max(jit_per_sm, 1)) * E->num_sms));
    for (uint32_t p = 0; p < f.passes.size(); ++p) {
      timer.begin(0);
      uint32_t pass = p;
      uint32_t npauli = dp.num_pauli;
      void* args[] = {&dp.fview, &pass, &state, const_cast<uint64_t*>(&S), &psel, &npauli, &max_blocks, &max_sites};
      const void* pk = use_jit && p < dp.fjit.size() && dp.fjit[p] ? dp.fjit[p] : kfn;
      CK(cudaLaunchKernel(pk, dim3(pk == kfn ? grid : jgrid), dim3(fnt), args, smem, E->stream));
      launched(E);
      timer.end(0);
    }
    export_states(E, opts, state, w0, S, n);
    if (dp.host.eligible) {
      timer.begin(2);
      sample_terminal(E, dp, c, guard);
      timer.end(2);
    }
  }
  unsigned flagged = 0;
  CK(cudaMemcpyAsync(&flagged, gcount, sizeof flagged, cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  if (flagged) {  // exact replays (the reference's arithmetic) of the guarded shots
    std::vector<uint64_t> ids(std::min<uint64_t>(flagged, count));
    CK(cudaMemcpy(ids.data(), gids, ids.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    ssb_run_options exact = opts ? *opts : ssb_run_options{};
    exact.fused_matrices = 0;
    exact.states_out = nullptr;
    exact.profile = 0;
    exact.max_batch_size = 0;
    for (uint64_t id : ids) run_batch_device(E, prog, id, 1, seed, &exact, values_dev + (id - shot_begin), nullptr);
  }
  if (stats) {
    stats->peak_states = wave;
    stats->passes = waves;
    stats->fused_passes = f.passes.size();
    stats->fused_blocks = f.num_blocks;
    stats->specialised_shapes = 0;
    if (use_jit)
      for (const void* k : dp.fjit) stats->specialised_shapes += k != nullptr;
    stats->guard_flagged = flagged;
    // largest possible half-width (m = 2^n - 1, every S'_k <= 1)
    stats->guard_delta = 2.02 * guard.err + (16.0 + 2.0 * double(uint64_t{1} << n) * (1.0 + 1e-6)) * 0x1p-53;
  }
}

// gpu-batch over shot ids [shot_begin, shot_begin+count) (or explicit ids).
void run_batch_device(ssb_engine* E, const ssb_program* prog, uint64_t shot_begin, uint64_t count, uint64_t seed,
                      const ssb_run_options* opts, uint64_t* values_dev, ssb_stats* stats) {
  if (count < 1) throw std::invalid_argument("shots must be >= 1");
  const RunConfig rc = config_of(opts);
  const unsigned n = prog->dev.n;
  const uint64_t launches0 = E->launches;
  if (opts && opts->check_norms) {
    run_batch_checked(E, prog, shot_begin, count, seed, opts, values_dev, stats);
    if (stats) stats->dispatch_count = E->launches - launches0;
    return;
  }
  double2* exp_dev = (opts && opts->states_out)
                         ? static_cast<double2*>(scratch(E, "export", (count << n) * sizeof(double2)))
                         : nullptr;
  // The resident plan (and its shared-memory size) for states that may fit.
  DevProgram* rdp = n <= rc.resident_max ? &device_program(E, prog, 0) : nullptr;
  const size_t rsmem = rdp ? resident_smem(rdp->host) : ~size_t{0};
  KernelTimer timer;
  timer.on = opts && opts->profile;
  timer.stream = E->stream;
  if (rdp && rsmem <= E->smem_optin) {
    DevProgram& dp = *rdp;
    // One-warp CTAs for small states; their plan carries the staged micro-ops
    // (plan_resident), so the choice is fixed by n.
    const unsigned warp_max = 10;
    uint64_t grid = 0;
    timer.begin(0);
    if (n <= warp_max) {
      const int g = launch_resident_warp(&dp.view, seed, shot_begin, count, values_dev, E->err, E->stream, rsmem,
                                         E->num_sms, exp_dev);
      if (g < 0) throw CudaError("resident (warp) launch failed");
      grid = static_cast<uint64_t>(g);
      launched(E);
    } else {
      CK(cudaFuncSetAttribute(resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rsmem)));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, resident_kernel, NT, rsmem));
      grid = std::min<uint64_t>(count, static_cast<uint64_t>(std::max(1, per_sm)) * E->num_sms);
      resident_kernel<<<static_cast<unsigned>(grid), NT, rsmem, E->stream>>>(dp.view, seed, nullptr, shot_begin, count,
                                                                             values_dev, E->err, exp_dev);
      launched(E);
    }
    timer.end(0);
    if (exp_dev) export_states(E, opts, exp_dev, 0, count, n);
    if (stats) {
      stats->peak_states = std::min<uint64_t>(count, grid);
      stats->passes = 1;
      stats->fused_passes = 1;
    }
  } else {
    // Fused mode defaults to 11-qubit tiles (more passes, but 128-thread CTAs
    // keep more tiles in flight per SM); an explicit tile_qubits wins.
    const bool want_fused = opts && opts->fused_matrices;
    const unsigned ftk = want_fused && !opts->tile_qubits && n >= kFusedSmallTileMinQubits ? 11u : rc.tile_k;
    DevProgram& fdp = device_program(E, prog, want_fused ? ftk : rc.tile_k);
    DevProgram& dp = want_fused && ftk != rc.tile_k && !fused_ready(E, fdp) ? device_program(E, prog, rc.tile_k) : fdp;
    if (want_fused && &dp == &fdp && fused_ready(E, dp)) {
      run_fused(E, prog, dp, shot_begin, count, seed, opts, values_dev, stats, timer);
      if (stats) {
        stats->dispatch_count = E->launches - launches0;
        unsigned long long hits = 0;
        CK(cudaMemcpyAsync(&hits, E->serial_chunks, sizeof hits, cudaMemcpyDeviceToHost, E->stream));
        CK(cudaStreamSynchronize(E->stream));
        stats->sampling_serial_chunks = hits;
      }
      timer.collect(stats);
      return;
    }
    const HostDevProgram& h = dp.host;
    const uint64_t seg = (uint64_t{1} << n) * sizeof(double2);
    const uint64_t limit = mem_limit(opts);
    // Default wave: as many shots as the memory limit allows, capped at 16 GiB
    // of state (>> L2, enough CTAs to fill the GPU many times over).
    uint64_t wave = opts && opts->max_batch_size
                        ? opts->max_batch_size
                        : std::max<uint64_t>(1, std::min<uint64_t>(limit, uint64_t{16} << 30) / seg);
    const uint64_t largest = std::min(wave, count);
    if (largest * seg > limit)
      throw shotsim::CapacityError("batch of " + std::to_string(largest) + " shots at " + std::to_string(n) +
                                   " qubits needs " + std::to_string(largest * seg) +
                                   " bytes; lower max_batch_size or raise the memory limit");
    const uint64_t tiles = uint64_t{1} << (n - h.tile_k);
    wave = std::min<uint64_t>(largest, std::max<uint64_t>(1, (uint64_t{1} << 31) / tiles - 1));
    // Shared noiseless trunk: a shot runs no pass before the first one at which
    // it draws a non-identity Pauli term; until then its state equals that of
    // a noiseless trunk (wave slot S, all-identity draws) and is copied from
    // it when the shot diverges. Most shots of a weakly noisy circuit share a
    // long prefix with the trunk (arXiv:2308.03399 §III-B, applied to the
    // batch). Needs one more state slot than the wave.
    const char* no_trunk = std::getenv("SHOTSIM_B200_NO_TRUNK");
    const bool trunk = dp.trunk_ok && !(no_trunk && *no_trunk && *no_trunk != '0') &&
                       (wave + 1) * seg <= limit;
    const uint64_t slots = wave + (trunk ? 1 : 0);
    double2* state = static_cast<double2*>(scratch(E, "state", slots * seg));
    uint8_t* psel = dp.num_pauli ? static_cast<uint8_t*>(scratch(E, "psel", slots * dp.num_pauli)) : nullptr;
    const uint32_t npass = static_cast<uint32_t>(h.passes.size());
    // Trunk bookkeeping: per shot its first diverging pass (device kernel,
    // read back once), then per wave the slots in activation order (trunk
    // first) and the per-pass activation boundaries.
    uint32_t* act_dev = nullptr;
    std::vector<uint64_t> act_off, act_end;  // per wave: offset into act, per-pass end counts
    std::vector<char> wave_trunk;            // per wave: the trunk pays for itself
    uint64_t trunk_skipped = 0;
    if (trunk) {
      uint16_t* first_dev = static_cast<uint16_t*>(scratch(E, "trunk_first", count * sizeof(uint16_t)));
      first_divergence_kernel<<<grid_for(count), NT, 0, E->stream>>>(dp.view, dp.pauli_site_ops, dp.site_pass,
                                                                     dp.num_pauli, seed, shot_begin, count,
                                                                     static_cast<uint16_t>(npass), first_dev);
      launched(E);
      const uint64_t nwaves = (count + wave - 1) / wave;
      uint16_t* first = static_cast<uint16_t*>(engine_host(E, "trunk_first", count * sizeof(uint16_t)));
      CK(cudaMemcpyAsync(first, first_dev, count * sizeof(uint16_t), cudaMemcpyDeviceToHost, E->stream));
      CK(cudaStreamSynchronize(E->stream));
      const uint64_t nact = count + nwaves;
      uint32_t* act = static_cast<uint32_t*>(engine_host(E, "trunk_act", nact * sizeof(uint32_t)));
      act_dev = static_cast<uint32_t*>(scratch(E, "trunk_act", nact * sizeof(uint32_t)));
      std::vector<uint64_t> cnt(npass + 2);
      for (uint64_t w0 = 0, off = 0; w0 < count; w0 += wave) {
        const uint64_t S = std::min(wave, count - w0);
        std::fill(cnt.begin(), cnt.end(), 0);
        for (uint64_t s = 0; s < S; ++s) ++cnt[first[w0 + s] + 1];
        for (uint32_t p = 0; p <= npass; ++p) cnt[p + 1] += cnt[p];  // cnt[p]: shots with first < p
        act_off.push_back(off);
        for (uint32_t p = 0; p <= npass; ++p) act_end.push_back(1 + cnt[p + 1]);  // trunk + first <= p
        act[off] = static_cast<uint32_t>(S);
        for (uint64_t s = 0; s < S; ++s) act[off + 1 + cnt[first[w0 + s]]++] = static_cast<uint32_t>(s);
        // Worth it when the skipped (shot, pass) pairs exceed the trunk's own
        // passes plus its copies (a copy moves one state once: ~1/4 of a pass).
        uint64_t skipped = 0;
        for (uint32_t p = 0; p < npass; ++p) skipped += S + 1 - act_end[act_end.size() - (npass + 1) + p];
        const uint64_t copied = S + 1 - act_end[act_end.size() - (npass + 1)];
        wave_trunk.push_back(skipped > npass + copied / 4);
        off += S + 1;
      }
      CK(cudaMemcpyAsync(act_dev, act, nact * sizeof(uint32_t), cudaMemcpyHostToDevice, E->stream));
    }
    // Matrix-0 partials of the next Kraus site from a pass epilogue: per shot
    // at most 2^(n-1)/512 (1q) or 2^(n-2)/8 (2q) doubles.
    double* epi_part = nullptr;
    for (const PassDesc& pd : h.passes)
      if (pd.epi_kind) {
        const uint64_t per = std::max<uint64_t>((uint64_t{1} << (n - 1)) / 512, (uint64_t{1} << (n - 2)) / 8);
        epi_part = static_cast<double*>(scratch(E, "epi_part", wave * per * sizeof(double)));
        break;
      }
    // Default off until it pays (C4 A/B in DESIGN.md); SHOTSIM_B200_EPILOGUE=1 enables it.
    if (const char* v = std::getenv("SHOTSIM_B200_EPILOGUE"); !(v && *v == '1')) epi_part = nullptr;
    // Per-shot Kraus choices of the wave (S_KRAUS_DECIDE -> next pass).
    double2* kmat = nullptr;
    uint64_t* kcls = nullptr;
    int* kchosen = nullptr;
    if (h.has_kraus) {
      kmat = static_cast<double2*>(scratch(E, "wave_kmat", wave * 16 * sizeof(double2)));
      kcls = static_cast<uint64_t*>(scratch(E, "wave_kcls", wave * sizeof(uint64_t)));
      kchosen = static_cast<int*>(scratch(E, "wave_kchosen", wave * sizeof(int)));
    }
    // The shape-specialised build of the same kernel (specialise.cpp) when
    // available, else the static interpreter build.
    const void* kfn = (opts && opts->interpret_only) ? nullptr : specialised_tile_kernel(h);
    const bool specialised = kfn != nullptr;
    const bool tile_db = specialised && specialised_tile_double_buffered();
    size_t tsmem = 0;
    for (const PassDesc& pd : h.passes)
      tsmem = std::max<size_t>(tsmem, tile_smem_bytes(pd.k, pd.uop_end - pd.uop_begin, pd.mat_count, tile_db));
    if (!kfn) kfn = reinterpret_cast<const void*>(tile_pass_kernel);
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tsmem)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NT, tsmem));
    uint64_t waves = 0, fused = 0;
    for (uint64_t w0 = 0; w0 < count; w0 += wave) {
      const uint64_t S = std::min(wave, count - w0);
      SegCtx c{state, S, seed, nullptr, shot_begin + w0, nullptr, values_dev + w0};
      CK(cudaMemsetAsync(c.cregs, 0, S * sizeof(uint64_t), E->stream));
      if (dp.num_pauli) {
        pauli_decide_kernel<<<grid_for(S * dp.num_pauli), NT, 0, E->stream>>>(dp.view, dp.pauli_site_ops, dp.num_pauli,
                                                                             seed, nullptr, c.begin, S, psel);
        launched(E);
        if (trunk && wave_trunk[waves])
          CK(cudaMemcpyAsync(psel + S * dp.num_pauli, dp.ident_row, dp.num_pauli, cudaMemcpyDeviceToDevice, E->stream));
      }
      const bool wtrunk = trunk && wave_trunk[waves];
      const uint32_t* wact = wtrunk ? act_dev + act_off[waves] : nullptr;
      const uint64_t* wend = wtrunk ? act_end.data() + waves * (npass + 1) : nullptr;
      // Activate the shots whose first diverging pass is p: copy the trunk in.
      auto activate = [&](uint32_t p) {
        const uint64_t b = p ? wend[p - 1] : 1, e = wend[p];
        if (e <= b) return;
        copy_trunk_kernel<<<grid_for(((e - b) << n) / 4), NT, 0, E->stream>>>(state, S, n, wact + b,
                                                                             static_cast<uint32_t>(e - b));
        launched(E);
      };
      ++waves;
      fused = 0;
      int64_t epi_op = -1;  // the Kraus site whose matrix-0 partials the last pass computed
      for (const Step& st : h.steps) {
        if (st.kind == S_KRAUS_DECIDE) {
          timer.begin(1);
          kraus_decide_wave(E, dp, st.index, c, kmat, kcls, kchosen,
                            epi_op == static_cast<int64_t>(st.index) ? epi_part : nullptr);
          timer.end(1);
          epi_op = -1;
        } else if (st.kind == S_PASS) {
          epi_op = (epi_part && h.passes[st.index].epi_kind) ? static_cast<int64_t>(h.passes[st.index].epi_op) : -1;
          // Trunk mode: only the trunk and the shots already diverged run.
          uint64_t active = S;
          if (wtrunk) {
            if (st.index > 0) activate(st.index);
            active = wend[st.index];
            trunk_skipped += S + 1 - active;
          }
          timer.begin(0);
          const unsigned grid =
              static_cast<unsigned>(std::min<uint64_t>(active * tiles, uint64_t(std::max(per_sm, 1)) * E->num_sms));
          uint32_t pass_index = st.index, num_pauli = dp.num_pauli;
          uint64_t* cregs = wtrunk ? nullptr : c.cregs;  // trunk mode: no conditions
          double* epi = epi_op >= 0 ? epi_part : nullptr;
          void* args[] = {&dp.view, &pass_index, &state, &active, &cregs, &psel, &num_pauli,
                          &kmat, &kcls, const_cast<uint32_t**>(&wact), &epi};
          CK(cudaLaunchKernel(kfn, dim3(grid), dim3(NT), args, tsmem, E->stream));
          launched(E);
          timer.end(0);
          ++fused;
        } else if (st.kind == S_SPECIAL) {
          epi_op = -1;
          timer.begin(1);
          apply_op(E, dp, st.index, c, false);
          timer.end(1);
        } else {
          if (wtrunk) activate(npass);  // shots that never diverged
          export_states(E, opts, state, w0, S, n);
          timer.begin(2);
          sample_terminal(E, dp, c);
          timer.end(2);
        }
      }
      if (!h.eligible) export_states(E, opts, state, w0, S, n);
    }
    if (stats) {
      stats->peak_states = std::min(wave, count);
      stats->passes = waves;
      stats->fused_passes = fused;
      stats->specialised_shapes = specialised ? h.shapes.size() : 0;
      stats->trunk_skipped = trunk_skipped;
    }
  }
  if (stats) {
    stats->dispatch_count = E->launches - launches0;
    unsigned long long hits = 0;
    CK(cudaMemcpyAsync(&hits, E->serial_chunks, sizeof hits, cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    stats->sampling_serial_chunks = hits;
  }
  timer.collect(stats);
}

struct DeviceGuard {
  explicit DeviceGuard(int dev) { CK(cudaSetDevice(dev)); }
};

}  // namespace

void run_branch_device(EngineView& E, const ProgView& P, const HostDevProgram& h, uint64_t shot_begin,
                       uint64_t count, uint64_t seed, const ssb_run_options* opts, uint64_t* values_dev,
                       ssb_stats* stats, uint64_t mem_limit_bytes);

// density.cu: the exact density-matrix reference.
std::map<uint64_t, double> exact_creg_distribution_device(const ssb_flat_program& F, cudaStream_t stream,
                                                          uint64_t* launches, int num_sms);
std::vector<double> exact_distribution_device(const ssb_flat_program& F, const uint32_t* qubits, unsigned count,
                                              cudaStream_t stream, uint64_t* launches, int num_sms);
}  // namespace ssb

namespace ssb {
// Called by ssb_program_destroy: frees every engine's device copies of the
// program (the caller guarantees no run with it is in flight, as the
// reference's executors borrow the program for the duration of a run).
void evict_program(uint64_t uid) {
  std::lock_guard<std::mutex> lk(g_engines_mu);
  for (ssb_engine* E : g_engines) {
    std::lock_guard<std::mutex> plk(E->programs_mu);
    for (auto it = E->programs.begin(); it != E->programs.end();) {
      if (it->first.first == uid) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(E->device);
        cudaStreamSynchronize(E->stream);
        it = E->programs.erase(it);
        if (prev >= 0) cudaSetDevice(prev);
      } else {
        ++it;
      }
    }
  }
}
}  // namespace ssb

using namespace ssb;

extern "C" {

SSB_API int ssb_device_count(int* count) {
  return guard([&] {
    if (!count) throw std::invalid_argument("null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

SSB_API int ssb_engine_create(int device, ssb_engine** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null argument");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw CudaError("no CUDA device available (shotsim_b200 has no CPU execution path)");
    if (device < 0 || device >= count) throw std::invalid_argument("device index out of range");
    DeviceGuard g(device);
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      throw CudaError("shotsim_b200 is built for sm_100a (B200) only; device is sm_" + std::to_string(prop.major) +
                      std::to_string(prop.minor));
    auto E = std::make_unique<ssb_engine>();
    E->device = device;
    E->num_sms = prop.multiProcessorCount;
    E->smem_optin = prop.sharedMemPerBlockOptin;
    CK(cudaStreamCreateWithFlags(&E->stream, cudaStreamNonBlocking));
    {  // keep freed program arrays in the device's pool for reuse (DevProgram)
      cudaMemPool_t pool = nullptr;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = uint64_t{1} << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
    }
    CK(cudaEventCreate(&E->ev0));
    CK(cudaEventCreate(&E->ev1));
    CK(cudaMalloc(&E->err, sizeof(int)));
    CK(cudaMemset(E->err, 0, sizeof(int)));
    CK(cudaMalloc(&E->serial_chunks, sizeof(unsigned long long)));
    CK(cudaMemset(E->serial_chunks, 0, sizeof(unsigned long long)));
    CK(cudaMalloc(&E->bad_op, sizeof(unsigned)));
    CK(cudaMemset(E->bad_op, 0xFF, sizeof(unsigned)));
    std::lock_guard<std::mutex> lk(g_engines_mu);
    g_engines.insert(E.get());
    *out = E.release();
  });
}

SSB_API void ssb_engine_destroy(ssb_engine* E) {
  if (!E) return;
  {
    std::lock_guard<std::mutex> lk(g_engines_mu);
    g_engines.erase(E);
  }
  cudaSetDevice(E->device);
  cudaStreamSynchronize(E->stream);
  E->programs.clear();  // (stream-ordered frees)
  cudaStreamSynchronize(E->stream);
  for (auto& [name, slot] : E->scratch) cudaFree(slot.first);
  for (auto& [name, slot] : E->host_scratch) cudaFreeHost(slot.first);
  cudaFree(E->err);
  cudaFree(E->serial_chunks);
  cudaFree(E->bad_op);
  cudaEventDestroy(E->ev0);
  cudaEventDestroy(E->ev1);
  cudaStreamDestroy(E->stream);
  delete E;
}

SSB_API void* ssb_engine_stream(ssb_engine* E) { return E ? static_cast<void*>(E->stream) : nullptr; }

SSB_API int ssb_run_batch_device(ssb_engine* E, const ssb_program* prog, uint64_t shot_begin, uint64_t shot_count,
                                 uint64_t seed, const ssb_run_options* options, uint64_t* values_out_device,
                                 ssb_stats* stats) {
  return guard([&] {
    if (!E || !prog || !values_out_device) throw std::invalid_argument("null argument");
    DeviceGuard g(E->device);
    CK(cudaMemsetAsync(E->serial_chunks, 0, sizeof(unsigned long long), E->stream));
    run_batch_device(E, prog, shot_begin, shot_count, seed, options, values_out_device, stats);
  });
}

SSB_API int ssb_run_batch(ssb_engine* E, const ssb_program* prog, uint64_t shot_begin, uint64_t shot_count,
                          uint64_t seed, const ssb_run_options* options, uint64_t* values_out, ssb_stats* stats) {
  return guard([&] {
    if (!E || !prog || !values_out) throw std::invalid_argument("null argument");
    if (shot_count < 1) throw std::invalid_argument("shots must be >= 1");
    DeviceGuard g(E->device);
    const auto t0 = std::chrono::steady_clock::now();
    uint64_t* dv = static_cast<uint64_t*>(scratch(E, "values", shot_count * sizeof(uint64_t)));
    CK(cudaMemsetAsync(E->serial_chunks, 0, sizeof(unsigned long long), E->stream));
    CK(cudaEventRecord(E->ev0, E->stream));
    run_batch_device(E, prog, shot_begin, shot_count, seed, options, dv, stats);
    CK(cudaMemcpyAsync(values_out, dv, shot_count * sizeof(uint64_t), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaEventRecord(E->ev1, E->stream));
    check_device_error(E);
    if (stats) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, E->ev0, E->ev1));
      stats->device_seconds = ms * 1e-3;
      stats->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

SSB_API int ssb_run_branch(ssb_engine* E, const ssb_program* prog, uint64_t shot_begin, uint64_t shot_count,
                           uint64_t seed, const ssb_run_options* options, uint64_t* values_out, ssb_stats* stats) {
  return guard([&] {
    if (!E || !prog || !values_out) throw std::invalid_argument("null argument");
    if (shot_count < 1) throw std::invalid_argument("shots must be >= 1");
    DeviceGuard g(E->device);
    const auto t0 = std::chrono::steady_clock::now();
    DevProgram& dp = device_program(E, prog, config_of(options).tile_k);
    uint64_t* dv = static_cast<uint64_t*>(scratch(E, "values", shot_count * sizeof(uint64_t)));
    EngineView view{E->stream, E->err, &E->launches, E, &engine_scratch, &engine_grow, &engine_host};
    ssb_run_options o = options ? *options : ssb_run_options{};
    if (!options) o.branch_budget = 64;
    CK(cudaEventRecord(E->ev0, E->stream));
    run_branch_device(view, dp.view, dp.host, shot_begin, shot_count, seed, &o, dv, stats, mem_limit(options));
    CK(cudaMemcpyAsync(values_out, dv, shot_count * sizeof(uint64_t), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaEventRecord(E->ev1, E->stream));
    check_device_error(E);
    if (stats) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, E->ev0, E->ev1));
      stats->device_seconds = ms * 1e-3;
      stats->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

SSB_API int ssb_histogram_device(ssb_engine* E, const uint64_t* values_device, uint64_t count, uint32_t num_clbits,
                                 uint64_t* hist_device) {
  return guard([&] {
    if (!E || !values_device || !hist_device) throw std::invalid_argument("null argument");
    if (num_clbits > 24) throw std::invalid_argument("dense histogram limited to 24 clbits");
    DeviceGuard g(E->device);
    g_histogram_kernel<<<grid_for(count), NT, 0, E->stream>>>(values_device, count, num_clbits,
                                                              reinterpret_cast<unsigned long long*>(hist_device));
    launched(E);
  });
}

SSB_API int ssb_fp64_peak(ssb_engine* E, double* ops_per_second) {
  return guard([&] {
    if (!E || !ops_per_second) throw std::invalid_argument("null argument");
    DeviceGuard g(E->device);
    constexpr int kThreads = 256, kIters = 4096;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp64_probe_kernel<kIters>, kThreads, 0));
    const unsigned grid = static_cast<unsigned>(std::max(per_sm, 1) * E->num_sms * 4);
    double* sink = static_cast<double*>(scratch(E, "fp64_sink", sizeof(double)));
    fp64_probe_kernel<kIters><<<grid, kThreads, 0, E->stream>>>(sink, 1.0000001, 1e-9);  // warm-up
    launched(E);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(E->ev0, E->stream));
      fp64_probe_kernel<kIters><<<grid, kThreads, 0, E->stream>>>(sink, 1.0000001, 1e-9);
      launched(E);
      CK(cudaEventRecord(E->ev1, E->stream));
      CK(cudaEventSynchronize(E->ev1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, E->ev0, E->ev1));
      best = std::min(best, ms);
    }
    *ops_per_second = double(grid) * kThreads * kIters * fp64_probe_ops_per_iter() / (best * 1e-3);
  });
}

// ---- exact density-matrix reference (density.cu) ---------------------------
SSB_API int ssb_exact_creg_distribution(ssb_engine* E, const ssb_program* prog, uint64_t* keys, double* probs,
                                        uint64_t capacity, uint64_t* count) {
  return guard([&] {
    if (!E || !prog || !count) throw std::invalid_argument("null argument");
    if ((keys == nullptr) != (probs == nullptr)) throw std::invalid_argument("keys and probs must both be set");
    DeviceGuard g(E->device);
    const auto dist = exact_creg_distribution_device(prog->flat.view, E->stream, &E->launches, E->num_sms);
    *count = dist.size();
    if (!keys) return;
    if (capacity < dist.size()) throw shotsim::CapacityError("exact distribution has more entries than capacity");
    uint64_t i = 0;
    for (const auto& [k, p] : dist) {
      keys[i] = k;
      probs[i] = p;
      ++i;
    }
  });
}

SSB_API int ssb_exact_distribution(ssb_engine* E, const ssb_program* prog, const uint32_t* qubits,
                                   uint32_t num_qubits, double* out) {
  return guard([&] {
    if (!E || !prog || !out || (num_qubits && !qubits)) throw std::invalid_argument("null argument");
    DeviceGuard g(E->device);
    const auto dist = exact_distribution_device(prog->flat.view, qubits, num_qubits, E->stream, &E->launches,
                                                E->num_sms);
    std::copy(dist.begin(), dist.end(), out);
  });
}

// ---- operator-level ABI (BatchState) ---------------------------------------
SSB_API int ssb_batch_create(ssb_engine* E, const ssb_program* prog, const uint64_t* shot_ids, uint64_t count,
                             uint64_t seed, ssb_batch** out) {
  return guard([&] {
    if (!E || !prog || !shot_ids || !out) throw std::invalid_argument("null argument");
    if (count == 0) throw std::invalid_argument("batch needs at least one shot");
    DeviceGuard g(E->device);
    auto B = std::make_unique<ssb_batch>();
    B->engine = E;
    B->program = prog;
    B->size = count;
    B->seed = seed;
    const unsigned n = prog->dev.n;
    CK(cudaMalloc(&B->ids, count * sizeof(uint64_t)));
    CK(cudaMalloc(&B->cregs, count * sizeof(uint64_t)));
    CK(cudaMalloc(&B->state, (count << n) * sizeof(double2)));
    CK(cudaMemcpy(B->ids, shot_ids, count * sizeof(uint64_t), cudaMemcpyHostToDevice));
    g_init_kernel<<<grid_for(count << n), NT, 0, E->stream>>>(B->state, count, n, B->cregs);
    launched(E);
    CK(cudaStreamSynchronize(E->stream));
    *out = B.release();
  });
}

SSB_API void ssb_batch_destroy(ssb_batch* B) {
  if (!B) return;
  cudaSetDevice(B->engine->device);
  cudaStreamSynchronize(B->engine->stream);
  cudaFree(B->ids);
  cudaFree(B->cregs);
  cudaFree(B->state);
  delete B;
}

SSB_API int ssb_batch_apply_op(ssb_batch* B, uint64_t op_index, const double* u) {
  return guard([&] {
    if (!B) throw std::invalid_argument("null batch");
    ssb_engine* E = B->engine;
    DeviceGuard g(E->device);
    DevProgram& dp = device_program(E, B->program, kTileDefault);
    if (op_index >= dp.host.ops.size()) throw std::invalid_argument("op index out of range");
    double* ud = nullptr;
    if (u) {
      ud = static_cast<double*>(scratch(E, "udraw", B->size * sizeof(double)));
      CK(cudaMemcpyAsync(ud, u, B->size * sizeof(double), cudaMemcpyHostToDevice, E->stream));
    }
    const SegCtx c{B->state, B->size, B->seed, B->ids, 0, ud, B->cregs};
    B->dispatches += apply_op(E, dp, static_cast<uint32_t>(op_index), c, true);
    check_device_error(E);
  });
}

SSB_API int ssb_batch_run(ssb_batch* B) {
  return guard([&] {
    if (!B) throw std::invalid_argument("null batch");
    ssb_engine* E = B->engine;
    DeviceGuard g(E->device);
    DevProgram& dp = device_program(E, B->program, kTileDefault);
    const SegCtx c{B->state, B->size, B->seed, B->ids, 0, nullptr, B->cregs};
    for (uint32_t i = 0; i < dp.host.end; ++i) B->dispatches += apply_op(E, dp, i, c, true);
    if (dp.host.eligible) {
      sample_terminal(E, dp, c);
      ++B->dispatches;
    }
    check_device_error(E);
  });
}

SSB_API int ssb_batch_read(ssb_batch* B, double* amps, uint64_t* cregs) {
  return guard([&] {
    if (!B) throw std::invalid_argument("null batch");
    DeviceGuard g(B->engine->device);
    CK(cudaStreamSynchronize(B->engine->stream));
    const unsigned n = B->program->dev.n;
    if (amps) CK(cudaMemcpy(amps, B->state, (B->size << n) * sizeof(double2), cudaMemcpyDeviceToHost));
    if (cregs) CK(cudaMemcpy(cregs, B->cregs, B->size * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  });
}

SSB_API int ssb_batch_write_segment(ssb_batch* B, uint64_t s, const double* amps) {
  return guard([&] {
    if (!B || !amps) throw std::invalid_argument("null argument");
    if (s >= B->size) throw std::invalid_argument("segment index out of range");
    DeviceGuard g(B->engine->device);
    CK(cudaStreamSynchronize(B->engine->stream));
    const unsigned n = B->program->dev.n;
    CK(cudaMemcpy(B->state + (s << n), amps, (uint64_t{1} << n) * sizeof(double2), cudaMemcpyHostToDevice));
  });
}

SSB_API uint64_t ssb_batch_dispatches(const ssb_batch* B) { return B ? B->dispatches : 0; }

}  // extern "C"
