// C ABI, host half: program lowering, dumps and result folding.
#include <cstring>
#include <map>

#include "capi_internal.hpp"
#include "engine/fused.hpp"

namespace ssb {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_uid{1};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
uint64_t next_program_uid() { return g_uid.fetch_add(1); }

namespace {

ssb_program* make_program(shotsim::NoisyCircuit&& nc) {
  auto* p = new ssb_program{next_program_uid(), std::move(nc), {}, {}};
  try {
    shotsim::flatten(p->nc, p->flat);
    p->dev = build_device_program(p->nc);
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

}  // namespace
}  // namespace ssb

extern "C" {

SSB_API const char* ssb_last_error(void) { return ssb::g_last_error.c_str(); }
SSB_API int ssb_abi_version(void) { return SSB_ABI_VERSION; }

SSB_API int ssb_program_from_text(const char* circuit_text, const char* noise_json, ssb_program** out) {
  return ssb::guard([&] {
    if (!circuit_text || !out) throw std::invalid_argument("null argument");
    const std::string text(circuit_text);
    const auto first = text.find_first_not_of(" \t\r\n");
    const shotsim::Circuit c = (first != std::string::npos && text[first] == '{')
                                   ? shotsim::circuit_from_json(text)
                                   : shotsim::circuit_from_text(text);
    const shotsim::NoiseModel model = shotsim::NoiseModel::from_json(noise_json ? noise_json : "");
    *out = ssb::make_program(shotsim::instrument(c, model));
  });
}

SSB_API int ssb_program_from_flat(const ssb_flat_program* flat, ssb_program** out) {
  return ssb::guard([&] {
    if (!flat || !out) throw std::invalid_argument("null argument");
    *out = ssb::make_program(shotsim::unflatten(*flat));
  });
}

SSB_API void ssb_program_destroy(ssb_program* program) {
  if (!program) return;
  ssb::evict_program(program->uid);
  delete program;
}

SSB_API int ssb_program_flat(const ssb_program* program, ssb_flat_program* out) {
  return ssb::guard([&] {
    if (!program || !out) throw std::invalid_argument("null argument");
    *out = program->flat.view;
  });
}

SSB_API int ssb_program_dump(const ssb_program* program, char* buf, size_t cap, size_t* len) {
  return ssb::guard([&] {
    if (!program) throw std::invalid_argument("null program");
    const std::string s = shotsim::dump_program(program->nc);
    if (len) *len = s.size();
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

SSB_API int ssb_counts_checksum(const uint64_t* values, uint64_t count, uint32_t num_clbits, uint32_t has_measure,
                                uint64_t* checksum_out, uint64_t* num_keys_out) {
  return ssb::guard([&] {
    const shotsim::Counts c =
        shotsim::counts_from_values(std::span<const uint64_t>(values, count), num_clbits, has_measure != 0);
    if (checksum_out) *checksum_out = shotsim::counts_checksum(c);
    if (num_keys_out) *num_keys_out = c.size();
  });
}

SSB_API int ssb_tvd_vs_exact(const uint64_t* values, uint64_t shots, uint32_t num_clbits, uint32_t has_measure,
                             const uint64_t* keys, const double* probs, uint64_t count, double* tvd) {
  return ssb::guard([&] {
    if (!tvd || (shots && !values) || (count && (!keys || !probs))) throw std::invalid_argument("null argument");
    const shotsim::Counts counts =
        shotsim::counts_from_values(std::span<const uint64_t>(values, shots), num_clbits, has_measure != 0);
    std::map<uint64_t, double> exact;
    for (uint64_t i = 0; i < count; ++i) exact[keys[i]] = probs[i];
    *tvd = shotsim::tvd_vs_exact(counts, shots, exact);  // density.cpp:308-315 (host/executors.cpp)
  });
}

}  // extern "C"

namespace ssb {
bool specialise_compile_check(const HostDevProgram& h, std::string* log);
std::vector<std::pair<std::string, std::vector<uint32_t>>> fused_jit_sources(const FusedPlan& f);
bool fused_jit_compile_check(const FusedPlan& f, std::string* log);
}

extern "C" SSB_API int ssb_program_pass_map(const ssb_program* program, uint32_t tile_qubits, uint32_t* pass_of_op,
                                           uint64_t cap, uint32_t* num_passes) {
  return ssb::guard([&] {
    if (!program || !num_passes) throw std::invalid_argument("null argument");
    ssb::HostDevProgram h = program->dev;
    ssb::plan_passes(h, tile_qubits ? std::max(3u, std::min(13u, tile_qubits)) : 12u);
    *num_passes = static_cast<uint32_t>(h.passes.size());
    if (!pass_of_op) return;
    if (cap < h.ops.size()) throw std::invalid_argument("pass_of_op too small");
    std::fill(pass_of_op, pass_of_op + h.ops.size(), 0xFFFFFFFFu);
    for (size_t p = 0; p < h.passes.size(); ++p) {
      const size_t e = p + 1 < h.passes.size() ? h.passes[p + 1].po_begin : h.pass_ops.size();
      for (size_t i = h.passes[p].po_begin; i < e; ++i) pass_of_op[h.pass_ops[i].op] = static_cast<uint32_t>(p);
    }
  });
}

extern "C" SSB_API int ssb_program_specialise_check(const ssb_program* program, uint32_t tile_qubits,
                                                   uint32_t* shapes) {
  return ssb::guard([&] {
    if (!program || !shapes) throw std::invalid_argument("null argument");
    ssb::HostDevProgram h = program->dev;
    ssb::plan_passes(h, tile_qubits ? std::max(3u, std::min(13u, tile_qubits)) : 12u);
    *shapes = static_cast<uint32_t>(h.shapes.size());
    std::string log;
    if (!ssb::specialise_compile_check(h, &log)) throw ssb::CudaError("shape specialisation failed: " + log);
  });
}

extern "C" SSB_API int ssb_program_fused_specialise_check(const ssb_program* program, uint32_t* kernels) {
  return ssb::guard([&] {
    if (!program || !kernels) throw std::invalid_argument("null argument");
    const ssb::FusedPlan f = ssb::plan_fused(program->dev, 11u);  // the fused mode's default tile
    if (!f.ok) throw std::invalid_argument("no fused-matrix plan: " + f.why);
    uint32_t n = 0;
    for (const auto& m : ssb::fused_jit_sources(f)) n += static_cast<uint32_t>(m.second.size());
    *kernels = n;
    std::string log;
    if (!ssb::fused_jit_compile_check(f, &log)) throw ssb::CudaError("fused specialisation failed: " + log);
  });
}

extern "C" SSB_API int ssb_program_fused_info(const ssb_program* program, uint32_t tile_qubits, ssb_fused_info* out) {
  return ssb::guard([&] {
    if (!program || !out) throw std::invalid_argument("null argument");
    const ssb::FusedPlan f = ssb::plan_fused(program->dev, tile_qubits ? std::max(8u, std::min(13u, tile_qubits)) : 12u);
    *out = ssb_fused_info{};
    out->ok = f.ok;
    out->passes = static_cast<uint32_t>(f.passes.size());
    out->blocks = f.num_blocks;
    out->groups = static_cast<uint32_t>(f.groups.size());
    out->max_pass_blocks = f.max_pass_blocks;
    out->err_bound = f.err_bound;
  });
}
