// Run-time shape specialisation of the HBM tile pass.
//
// plan_passes() names every distinct segment "shape" of a streamed plan (the
// segment's micro-op sequence when all its Pauli draws are identity and all
// conditions hold — per shot the common case); shape_source() emits one
// straight-line executor per shape. Here that source is compiled with NVRTC
// for sm_100a together with the engine's device headers (embedded at build
// time) into a specialised tile_pass_kernel, cached per distinct shape set for
// the life of the process. The specialised kernel runs the exact same
// arithmetic; segments whose shot drew a non-identity Pauli (or failed a
// condition) still go through the interpreter inside it. If NVRTC is missing
// or fails, the caller falls back to the static interpreter kernel (still on
// the GPU; there is no CPU path).
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "devprog.hpp"

namespace ssb {

extern const int kJitHeaderCount;
extern const char* const kJitHeaderNames[];
extern const char* const kJitHeaderTexts[];

namespace {

// The specialised kernel's straight-line shapes need few registers: one quad
// per thread and 3 CTAs per SM (85 registers) hide the tile loads better than
// the interpreter build's 2 quads x 2 CTAs (scripts/jit_sweep.py: C2 +5-7%,
// C5 +9% on B200).
#define SSB_JIT_QPT 1
#define SSB_JIT_MINB 3
#define SSB_STR2(x) #x
#define SSB_STR(x) SSB_STR2(x)

const char* kMain =
    "#include \"tile_pass.cuh\"\n"
    "extern \"C\" __global__ void __launch_bounds__(ssb::NT, SSB_TILE_MINB)\n"
    "ssb_tile_pass_jit(SSB_TILE_PASS_PARAMS) {\n"
    "  ssb::tile_pass_body(SSB_TILE_PASS_ARGS);\n"
    "}\n";

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
};

std::mutex g_mu;
std::map<std::string, Entry> g_cache;  // shape source -> kernel (nullptr: failed)
bool g_warned = false;

void warn(const std::string& what) {
  if (g_warned) return;
  g_warned = true;
  std::fprintf(stderr, "shotsim_b200: shape specialisation unavailable (%s); using the interpreter kernel\n",
               what.c_str());
}

// NVRTC options with the resolved tuning knobs (experiments):
// SHOTSIM_B200_JIT_QPT / _MINB override the quads per thread and CTAs-per-SM
// launch bound of the specialised kernel.
std::vector<std::string> nvrtc_options() {
  auto knob = [](const char* name, const char* dflt) {
    const char* v = std::getenv(name);
    return std::string(v && *v ? v : dflt);
  };
  std::vector<std::string> o = {"-arch=sm_100a", "-fmad=false", "-std=c++17", "-lineinfo", "-DSSB_SHAPES",
                                "-DSSB_QPT=" + knob("SHOTSIM_B200_JIT_QPT", SSB_STR(SSB_JIT_QPT)),
                                "-DSSB_TILE_MINB=" + knob("SHOTSIM_B200_JIT_MINB", SSB_STR(SSB_JIT_MINB))};
  // SHOTSIM_B200_TILE_PREFETCH=1: L2 prefetch of the next tile (A/B; off).
  if (knob("SHOTSIM_B200_TILE_PREFETCH", "0") == "1") o.push_back("-DSSB_TILE_PREFETCH");
  // SHOTSIM_B200_TILE_DB=1: double-buffered tiles (A/B).
  if (knob("SHOTSIM_B200_TILE_DB", "0") == "1") o.push_back("-DSSB_TILE_DB");
  return o;
}

// NVRTC: shape source + embedded engine headers -> sm_100a cubin. Returns an
// empty vector (and the log) on failure. Needs no GPU.
std::vector<char> build_cubin(const std::string& shapes, std::string* log_out) {
  std::vector<const char*> names(kJitHeaderNames, kJitHeaderNames + kJitHeaderCount);
  std::vector<const char*> texts(kJitHeaderTexts, kJitHeaderTexts + kJitHeaderCount);
  names.push_back("ssb_shapes.inc");
  texts.push_back(shapes.c_str());
  nvrtcProgram prog = nullptr;
  if (nvrtcCreateProgram(&prog, kMain, "ssb_tile_pass_jit.cu", static_cast<int>(names.size()), texts.data(),
                         names.data()) != NVRTC_SUCCESS) {
    *log_out = "nvrtcCreateProgram failed";
    return {};
  }
  const std::vector<std::string> base = nvrtc_options();
  std::vector<const char*> opts;
  for (const std::string& o : base) opts.push_back(o.c_str());
  // SHOTSIM_B200_JIT_VERBOSE=1: print ptxas register / spill usage to stderr.
  const char* verbose = std::getenv("SHOTSIM_B200_JIT_VERBOSE");
  const bool loud = verbose && *verbose && *verbose != '0';
  if (loud) opts.push_back("--ptxas-options=-v");
  const nvrtcResult r = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
  if (loud && r == NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    std::fprintf(stderr, "%s\n", log.c_str());
  }
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    *log_out = std::string(nvrtcGetErrorString(r)) + ": " + log.substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    return {};
  }
  size_t size = 0;
  nvrtcGetCUBINSize(prog, &size);
  std::vector<char> cubin(size);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return cubin;
}

// On-disk cubin cache: $SHOTSIM_B200_CACHE (default ~/.cache/shotsim_b200),
// keyed by a 64-bit FNV-1a hash of everything that determines the cubin: the
// generated source, the kernel's main source, the embedded headers, the exact
// NVRTC options (resolved knobs included), the NVRTC version and the ABI
// version — a rebuild that changes any of them never loads a stale cubin.
std::string cache_dir() {
  const char* dir = std::getenv("SHOTSIM_B200_CACHE");
  if (dir && *dir) return dir;
  if (const char* home = std::getenv("HOME"); home && *home) return std::string(home) + "/.cache/shotsim_b200";
  return "";
}

std::string keyed_path(const char* prefix, const std::string& source, const char* main,
                       const std::vector<std::string>& options) {
  const std::string d = cache_dir();
  if (d.empty()) return "";
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const char* p, size_t n) {
    for (size_t i = 0; i < n; ++i) h = (h ^ static_cast<unsigned char>(p[i])) * 1099511628211ull;
  };
  mix(source.data(), source.size());
  mix(main, std::strlen(main));
  for (int i = 0; i < kJitHeaderCount; ++i) mix(kJitHeaderTexts[i], std::strlen(kJitHeaderTexts[i]));
  for (const std::string& o : options) mix(o.c_str(), o.size() + 1);
  int major = 0, minor = 0;
  nvrtcVersion(&major, &minor);
  const int versions[3] = {major, minor, SSB_ABI_VERSION};
  mix(reinterpret_cast<const char*>(versions), sizeof versions);
  char name[96];
  std::snprintf(name, sizeof name, "/%s_%016llx.cubin", prefix, static_cast<unsigned long long>(h));
  return d + name;
}

std::string cache_path(const std::string& shapes) { return keyed_path("tile_pass", shapes, kMain, nvrtc_options()); }

std::vector<char> read_file(const std::string& path) {
  std::vector<char> out;
  if (path.empty()) return out;
  if (FILE* f = std::fopen(path.c_str(), "rb")) {
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (n > 0) {
      out.resize(static_cast<size_t>(n));
      if (std::fread(out.data(), 1, out.size(), f) != out.size()) out.clear();
    }
    std::fclose(f);
  }
  return out;
}

void write_file_atomic(const std::string& path, const std::vector<char>& data) {
  if (path.empty()) return;
  const std::string dir = path.substr(0, path.rfind('/'));
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  const std::string tmp = path + ".tmp" + std::to_string(static_cast<long long>(getpid()));
  if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
    const bool ok = std::fwrite(data.data(), 1, data.size(), f) == data.size();
    std::fclose(f);
    if (ok) std::filesystem::rename(tmp, path, ec);
    else std::filesystem::remove(tmp, ec);
  }
}

Entry compile(const std::string& shapes) {
  Entry e;
  std::string log;
  const std::string cpath = cache_path(shapes);
  std::vector<char> cubin = read_file(cpath);
  if (cubin.empty()) {
    cubin = build_cubin(shapes, &log);
    if (!cubin.empty()) write_file_atomic(cpath, cubin);
  }
  if (cubin.empty()) {
    warn(log);
    return e;
  }
  if (cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&e.kernel, e.lib, "ssb_tile_pass_jit") != cudaSuccess) {
    cudaGetLastError();
    warn("loading the specialised cubin failed");
    e = Entry{};
  }
  return e;
}

// Options of the generic builds (FMA contraction allowed: the fused-matrix
// kernels).
std::vector<std::string> generic_options() { return {"-arch=sm_100a", "-std=c++17", "-lineinfo"}; }

// Generic NVRTC build of a complete source (plus the embedded engine
// headers) for sm_100a.
std::vector<char> build_generic_cubin(const std::string& source, std::string* log_out) {
  std::vector<const char*> names(kJitHeaderNames, kJitHeaderNames + kJitHeaderCount);
  std::vector<const char*> texts(kJitHeaderTexts, kJitHeaderTexts + kJitHeaderCount);
  nvrtcProgram prog = nullptr;
  if (nvrtcCreateProgram(&prog, source.c_str(), "ssb_fused_jit.cu", static_cast<int>(names.size()), texts.data(),
                         names.data()) != NVRTC_SUCCESS) {
    *log_out = "nvrtcCreateProgram failed";
    return {};
  }
  const std::vector<std::string> base = generic_options();
  std::vector<const char*> opts;
  for (const std::string& o : base) opts.push_back(o.c_str());
  const nvrtcResult r = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    *log_out = std::string(nvrtcGetErrorString(r)) + ": " + log.substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    return {};
  }
  size_t size = 0;
  nvrtcGetCUBINSize(prog, &size);
  std::vector<char> cubin(size);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return cubin;
}

std::string generic_cache_path(const std::string& source) {
  return keyed_path("fused", source, "", generic_options());
}

struct GenericEntry {
  cudaLibrary_t lib = nullptr;
  std::vector<cudaKernel_t> kernels;
};
std::map<std::string, GenericEntry> g_generic;

}  // namespace

// Compiles each source with NVRTC (cached in-process and on disk; the
// uncached ones concurrently, one host thread each up to the core count) and
// returns per source the named kernels, or an empty vector on failure (the
// first log in *log).
std::vector<std::vector<const void*>> jit_compile_batch(const std::vector<std::string>& sources,
                                                        const std::vector<std::vector<std::string>>& names,
                                                        std::string* log) {
  std::vector<std::vector<char>> cubins(sources.size());
  std::vector<std::string> logs(sources.size());
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    for (size_t i = 0; i < sources.size(); ++i)
      if (!g_generic.count(sources[i])) todo.push_back(i);
  }
  std::vector<size_t> build;
  for (size_t i : todo) {
    cubins[i] = read_file(generic_cache_path(sources[i]));
    if (cubins[i].empty()) build.push_back(i);
  }
  if (!build.empty()) {
    const size_t nt = std::max<size_t>(1, std::min<size_t>(build.size(), std::thread::hardware_concurrency()));
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nt; ++t)
      pool.emplace_back([&] {
        for (size_t j; (j = next.fetch_add(1)) < build.size();) {
          const size_t i = build[j];
          cubins[i] = build_generic_cubin(sources[i], &logs[i]);
          if (!cubins[i].empty()) write_file_atomic(generic_cache_path(sources[i]), cubins[i]);
        }
      });
    for (std::thread& t : pool) t.join();
  }
  std::lock_guard<std::mutex> lock(g_mu);
  std::vector<std::vector<const void*>> out(sources.size());
  for (size_t i = 0; i < sources.size(); ++i) {
    auto it = g_generic.find(sources[i]);
    if (it == g_generic.end()) {
      GenericEntry e;
      if (!cubins[i].empty() &&
          cudaLibraryLoadData(&e.lib, cubins[i].data(), nullptr, nullptr, 0, nullptr, nullptr, 0) == cudaSuccess) {
        for (const std::string& nm : names[i]) {
          cudaKernel_t k = nullptr;
          if (cudaLibraryGetKernel(&k, e.lib, nm.c_str()) != cudaSuccess) {
            cudaGetLastError();
            e.kernels.clear();
            logs[i] = "kernel " + nm + " missing";
            break;
          }
          e.kernels.push_back(k);
        }
      } else {
        cudaGetLastError();
        if (logs[i].empty()) logs[i] = "loading the fused cubin failed";
      }
      it = g_generic.emplace(sources[i], std::move(e)).first;
    }
    for (cudaKernel_t k : it->second.kernels) out[i].push_back(reinterpret_cast<const void*>(k));
    if (log && log->empty() && !logs[i].empty()) *log = logs[i];
  }
  return out;
}

bool jit_compile_check(const std::string& source, std::string* log) { return !build_generic_cubin(source, log).empty(); }

bool specialised_tile_double_buffered() {
  for (const std::string& o : nvrtc_options())
    if (o == "-DSSB_TILE_DB") return true;
  return false;
}

bool specialise_compile_check(const HostDevProgram& h, std::string* log) {
  if (h.shapes.empty()) {
    *log = "plan has no segment shapes";
    return false;
  }
  return !build_cubin(shape_source(h), log).empty();
}

const void* specialised_tile_kernel(const HostDevProgram& h) {
  // Shapes only run when every register round is full: 2^(k-2) quads must be
  // a multiple of NT * QPT (= 256 at one quad per thread), i.e. k >= 10.
  if (h.shapes.empty() || h.tile_k < 10) return nullptr;
  if (const char* off = std::getenv("SHOTSIM_B200_NO_SPECIALISE"); off && *off && *off != '0') return nullptr;
  // In-process key: the shapes plus the resolved NVRTC options (the knobs
  // change the kernel, e.g. SSB_TILE_DB its shared-memory layout).
  std::string src = shape_source(h) + "//";
  for (const std::string& o : nvrtc_options()) src += " " + o;
  src += "\n";
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(src);
  if (it == g_cache.end()) it = g_cache.emplace(src, compile(src)).first;
  return reinterpret_cast<const void*>(it->second.kernel);
}

}  // namespace ssb
