// Run-time specialised fused-matrix passes (fused_body.cuh, NVRTC).
//
// The static fused_pass_kernel interprets each pass's groups from shared
// memory: group positions, the per-block bit pair (a six-way switch) and the
// block's 4x4 product, loaded from shared memory into 64 registers per block.
// Here every pass of a plan gets its own kernel whose group phase is
// straight-line code: positions and element offsets are literals, each
// block's bit pair is a template argument, and the noiseless block products
// are __constant__ data the DFMAs read as constant-bank operands (no matrix
// registers, no matrix loads). A block whose shot drew a non-identity Pauli
// (its entry points at a per-shot product slot, or carries extra factors)
// takes the generic path, the same arithmetic as the static kernel.
//
// 11- and 12-qubit tiles with 4-qubit register groups (one hexad per thread:
// 128 / 256 threads) are specialised; other passes keep the static kernel.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "fused.hpp"

namespace ssb {

std::vector<std::vector<const void*>> jit_compile_batch(const std::vector<std::string>& sources,
                                                        const std::vector<std::vector<std::string>>& names,
                                                        std::string* log);
bool jit_compile_check(const std::string& source, std::string* log);

namespace {

// __constant__ bytes per module (the bank holds 64 KB; keep headroom).
constexpr size_t kConstBudget = 48 * 1024;
// Passes per NVRTC module (modules compile concurrently).
constexpr size_t kPassesPerModule = 1;

uint32_t swzh(uint32_t l) { return l ^ ((l >> 3) & 7u); }

std::string hexd(double v) {
  char b[48];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}

bool pass_ok(const FusedPlan& f, const FPass& P) {
  if (P.k != f.k || (f.k != 11 && f.k != 12)) return false;
  for (uint32_t b = P.blk_begin; b < P.blk_end; ++b)
    if (f.blocks[b].gb0 >= f.blocks[b].gb1 || f.blocks[b].gb1 > 3) return false;
  for (uint32_t g = P.grp_begin; g < P.grp_end; ++g)
    for (int i = 0; i < 4; ++i)
      if (f.groups[g].g[i] >= P.k || (i && f.groups[g].g[i] <= f.groups[g].g[i - 1])) return false;
  return true;
}

// One pass: its constant block products, the group functor and the kernel.
void emit_pass(std::string& s, const FusedPlan& f, uint32_t p) {
  const FPass& P = f.passes[p];
  const std::string id = std::to_string(p);
  const uint32_t nb = P.blk_end - P.blk_begin;
  s += "__constant__ double2 ssb_cm_" + id + "[" + std::to_string(std::max(1u, nb) * 16) + "] = {\n";
  for (uint32_t b = 0; b < nb; ++b) {
    const double* m = &f.mats[size_t{f.blocks[P.blk_begin + b].mat} * 32];
    for (int j = 0; j < 16; ++j) s += "{" + hexd(m[2 * j]) + "," + hexd(m[2 * j + 1]) + "},";
    s += "\n";
  }
  if (nb == 0) s += "{0.0,0.0}";
  s += "};\n";
  s += "struct SsbGroups" + id + " {\n"
       "  __device__ __forceinline__ void operator()(double2* tile, const FEntry* ents, const FGroup*, const FBlock*,\n"
       "                                             const uint32_t* xf, uint32_t, const FusedView& F) const {\n"
       "    const uint32_t h = threadIdx.x;\n";
  for (uint32_t gi = P.grp_begin; gi < P.grp_end; ++gi) {
    const FGroup& G = f.groups[gi];
    uint32_t t[4];
    for (int i = 0; i < 4; ++i) t[i] = swzh(1u << G.g[i]);
    s += "    {\n      const uint32_t sb = swz(ins0(ins0(ins0(ins0(h, " + std::to_string(G.g[0]) + "), " +
         std::to_string(G.g[1]) + "), " + std::to_string(G.g[2]) + "), " + std::to_string(G.g[3]) + "));\n";
    s += "      const uint32_t t[4] = {" + std::to_string(t[0]) + "u, " + std::to_string(t[1]) + "u, " +
         std::to_string(t[2]) + "u, " + std::to_string(t[3]) + "u};\n";
    s += "      double2 a[16];\n";
    std::string go[16];
    for (unsigned e = 0; e < 16; ++e) {
      uint32_t o = 0;
      for (int i = 0; i < 4; ++i)
        if ((e >> i) & 1) o ^= t[i];
      go[e] = std::to_string(o) + "u";
      s += "      a[" + std::to_string(e) + "] = tile[sb ^ " + go[e] + "];\n";
    }
    for (uint32_t b = G.blk_begin; b < G.blk_end; ++b) {
      const uint32_t lb = b - P.blk_begin;
      const FBlock& B = f.blocks[b];
      s += "      jit_block<" + std::to_string(B.gb0) + ", " + std::to_string(B.gb1) + ">(a, ents[" + std::to_string(lb) +
           "], " + std::to_string((1u << P.k) + lb * 16) + "u, ssb_cm_" + id + " + " + std::to_string(lb * 16) +
           ", tile, sb, t, xf, F);\n";
    }
    for (unsigned e = 0; e < 16; ++e) s += "      tile[sb ^ " + go[e] + "] = a[" + std::to_string(e) + "];\n";
    s += "    }\n    __syncthreads();\n";
  }
  s += "  }\n};\n";
  s += "}  // namespace ssb\n"
       "extern \"C\" __global__ void __launch_bounds__(SSB_FUSED_JIT_NT, SSB_FUSED_JIT_MINB)\n"
       "ssb_fused_" + id + "(ssb::FusedView F, uint32_t pass_index, double2* state, uint64_t S,\n"
       "    const uint8_t* pauli_sel, uint32_t num_pauli, uint32_t max_blocks, uint32_t max_sites) {\n"
       "  ssb::fused_pass_body<SSB_FUSED_JIT_NT, 4>(F, pass_index, state, S, pauli_sel, num_pauli, max_blocks,\n"
       "                                         max_sites,\n"
       "                               ssb::SsbGroups" + id + "{});\n"
       "}\n"
       "namespace ssb {\n";
}

// CTAs per SM the register allocation must allow: 128 registers per thread
// (the static build's budget), SHOTSIM_B200_FUSED_JIT_MINB overrides.
unsigned jit_minb(unsigned nt) {
  const char* v = std::getenv("SHOTSIM_B200_FUSED_JIT_MINB");
  return v && *v >= '1' && *v <= '8' ? unsigned(*v - '0') : 512u / nt;
}

}  // namespace

// Module sources: consecutive eligible passes, each module's constant data
// within kConstBudget. mods[i] = (source, pass ids).
std::vector<std::pair<std::string, std::vector<uint32_t>>> fused_jit_sources(const FusedPlan& f) {
  std::vector<std::pair<std::string, std::vector<uint32_t>>> mods;
  if (!f.ok || f.gq != 4 || (f.k != 11 && f.k != 12)) return mods;
  const unsigned nt = 1u << (f.k - 4);  // one hexad per thread
  const std::string head = "// shotsim_b200 fused-pass specialisation v3\n#define SSB_FUSED_JIT_NT " +
                           std::to_string(nt) + "\n#define SSB_FUSED_JIT_MINB " + std::to_string(jit_minb(nt)) +
                           "\n#include \"fused_body.cuh\"\nnamespace ssb {\n";
  std::string cur;
  std::vector<uint32_t> ids;
  size_t bytes = 0;
  auto flush = [&] {
    if (ids.empty()) return;
    mods.emplace_back(head + cur + "}  // namespace ssb\n", ids);
    cur.clear();
    ids.clear();
    bytes = 0;
  };
  for (uint32_t p = 0; p < f.passes.size(); ++p) {
    const FPass& P = f.passes[p];
    if (!pass_ok(f, P)) continue;
    const size_t need = size_t{std::max(1u, P.blk_end - P.blk_begin)} * 256;
    if (bytes + need > kConstBudget || ids.size() >= kPassesPerModule) flush();
    emit_pass(cur, f, p);
    ids.push_back(p);
    bytes += need;
  }
  flush();
  return mods;
}

// Per pass: the specialised kernel, or nullptr (static kernel). Compiled once
// per plan (cached in-process and on disk by source).
std::vector<const void*> fused_jit_kernels(const FusedPlan& f, std::string* log) {
  std::vector<const void*> out(f.passes.size(), nullptr);
  const auto mods = fused_jit_sources(f);
  std::vector<std::string> srcs;
  std::vector<std::vector<std::string>> names;
  for (const auto& [src, ids] : mods) {
    srcs.push_back(src);
    names.emplace_back();
    for (uint32_t p : ids) names.back().push_back("ssb_fused_" + std::to_string(p));
  }
  const auto ks = jit_compile_batch(srcs, names, log);
  for (size_t m = 0; m < mods.size(); ++m) {
    if (ks[m].size() != mods[m].second.size()) return std::vector<const void*>(f.passes.size(), nullptr);
    for (size_t i = 0; i < ks[m].size(); ++i) out[mods[m].second[i]] = ks[m][i];
  }
  return out;
}

bool fused_jit_compile_check(const FusedPlan& f, std::string* log) {
  const auto mods = fused_jit_sources(f);
  if (mods.empty()) {
    *log = "no specialisable pass";
    return false;
  }
  // SHOTSIM_B200_FUSED_JIT_DUMP=dir: write the module sources (inspection
  // with nvcc -cubin / cuobjdump).
  if (const char* dir = std::getenv("SHOTSIM_B200_FUSED_JIT_DUMP"); dir && *dir)
    for (size_t i = 0; i < mods.size(); ++i)
      if (FILE* fp = std::fopen((std::string(dir) + "/fused_mod" + std::to_string(i) + ".cu").c_str(), "w")) {
        std::fwrite(mods[i].first.data(), 1, mods[i].first.size(), fp);
        std::fclose(fp);
      }
  std::vector<std::string> logs(mods.size());
  std::vector<char> ok(mods.size(), 0);
  std::vector<std::thread> pool;
  std::atomic<size_t> next{0};
  const size_t nt = std::max<size_t>(1, std::min<size_t>(mods.size(), std::thread::hardware_concurrency()));
  for (size_t t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1)) < mods.size();) ok[i] = jit_compile_check(mods[i].first, &logs[i]);
    });
  for (std::thread& t : pool) t.join();
  for (size_t i = 0; i < mods.size(); ++i)
    if (!ok[i]) {
      *log = logs[i];
      return false;
    }
  return true;
}

}  // namespace ssb
