// mf_jit.cpp -- K4/K6 generated per triple at plan time (NVRTC, sm_100a).
//
// The paper's Matrix Flow generates code per algorithm and compiles it
// (C++ over rocBLAS).  The B200 form of that idea: for a
// triple that is not compiled into the library (mf_fixed.cu / mf_kron.cu), or
// for the local tables of bounded-workspace batches, mf_plan emits the
// straight-line CUDA of each fused addition kernel -- every term of Eq.
// "strassen" (L196-202) spelled out with its coefficient as a literal, so the
// kernel carries no coefficient loads and no branches -- compiles it with
// NVRTC for the device's architecture, and loads it with the driver API.  Both
// are dlopen'ed: a box without NVRTC keeps the table-driven kernels of
// mf_mix.cu (still GPU code; there is no CPU path).
//
// Two shapes, chosen by what fits in registers (one thread = VW consecutive
// positions of every block; 256-bit loads/stores at VW = 4):
//   output-major: load every used input once, then each output as one
//                 straight-line ascending sum, stored at once (K4's shape:
//                 few inputs, many outputs);
//   input-major:  one accumulator per output; stream the inputs in ascending
//                 order, adding each into the outputs that use it (K6's shape).
// Either way each output sums its own terms in ascending input order with
// separate multiply/add (__dmul_rn/__dadd_rn, --fmad=false), the accumulator
// starting at -0.0, alpha last -- the oracle's order (R7/R8), so
// the generated kernels are bit-exact with it like the hand-written ones.
#include <dlfcn.h>

#include <algorithm>
#include <cinttypes>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "mf_internal.h"

namespace mf {
namespace {

// ---- NVRTC + driver API, resolved at run time ----
typedef int nvrtcResult_;
typedef void* nvrtcProgram_;
typedef int CUresult_;
typedef void* CUmodule_;
typedef void* CUfunction_;

struct Jit {
  void* hn = nullptr;
  void* hc = nullptr;
  nvrtcResult_ (*Create)(nvrtcProgram_*, const char*, const char*, int, const char* const*,
                         const char* const*) = nullptr;
  nvrtcResult_ (*Compile)(nvrtcProgram_, int, const char* const*) = nullptr;
  nvrtcResult_ (*LogSize)(nvrtcProgram_, size_t*) = nullptr;
  nvrtcResult_ (*Log)(nvrtcProgram_, char*) = nullptr;
  nvrtcResult_ (*CubinSize)(nvrtcProgram_, size_t*) = nullptr;
  nvrtcResult_ (*Cubin)(nvrtcProgram_, char*) = nullptr;
  nvrtcResult_ (*Destroy)(nvrtcProgram_*) = nullptr;
  CUresult_ (*ModuleLoadData)(CUmodule_*, const void*) = nullptr;
  CUresult_ (*ModuleGetFunction)(CUfunction_*, CUmodule_, const char*) = nullptr;
  CUresult_ (*ModuleUnload)(CUmodule_) = nullptr;
  CUresult_ (*LaunchKernel)(CUfunction_, unsigned, unsigned, unsigned, unsigned, unsigned,
                            unsigned, unsigned, cudaStream_t, void**, void**) = nullptr;
  bool nvrtc_ok() const { return Create && Compile && LogSize && Log && CubinSize && Cubin && Destroy; }
  bool driver_ok() const { return ModuleLoadData && ModuleGetFunction && ModuleUnload && LaunchKernel; }
};

Jit* jit() {
  static Jit j;
  static std::once_flag once;
  std::call_once(once, [] {
    // the toolkit's NVRTC (its builtins library first, so NVRTC's own
    // dlopen of it by soname resolves), else whatever the loader finds
    const char* dirs[] = {"/usr/local/cuda/lib64/", "/usr/local/cuda/targets/x86_64-linux/lib/", ""};
    for (const char* d : dirs) {
      std::string b = std::string(d) + "libnvrtc-builtins.so.12.9";
      dlopen(b.c_str(), RTLD_NOW | RTLD_GLOBAL);
      std::string p = std::string(d) + "libnvrtc.so.12";
      if ((j.hn = dlopen(p.c_str(), RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    }
    if (j.hn) {
      j.Create = (decltype(j.Create))dlsym(j.hn, "nvrtcCreateProgram");
      j.Compile = (decltype(j.Compile))dlsym(j.hn, "nvrtcCompileProgram");
      j.LogSize = (decltype(j.LogSize))dlsym(j.hn, "nvrtcGetProgramLogSize");
      j.Log = (decltype(j.Log))dlsym(j.hn, "nvrtcGetProgramLog");
      j.CubinSize = (decltype(j.CubinSize))dlsym(j.hn, "nvrtcGetCUBINSize");
      j.Cubin = (decltype(j.Cubin))dlsym(j.hn, "nvrtcGetCUBIN");
      j.Destroy = (decltype(j.Destroy))dlsym(j.hn, "nvrtcDestroyProgram");
    }
    if ((j.hc = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD)) == nullptr)
      j.hc = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (j.hc) {
      j.ModuleLoadData = (decltype(j.ModuleLoadData))dlsym(j.hc, "cuModuleLoadData");
      j.ModuleGetFunction = (decltype(j.ModuleGetFunction))dlsym(j.hc, "cuModuleGetFunction");
      j.ModuleUnload = (decltype(j.ModuleUnload))dlsym(j.hc, "cuModuleUnload");
      j.LaunchKernel = (decltype(j.LaunchKernel))dlsym(j.hc, "cuLaunchKernel");
    }
  });
  return &j;
}

void appendf(std::string& s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void appendf(std::string& s, const char* fmt, ...) {
  va_list ap, aq;
  va_start(ap, fmt);
  va_copy(aq, ap);
  const int n = vsnprintf(nullptr, 0, fmt, ap);
  va_end(ap);
  if (n > 0) {
    std::vector<char> buf((size_t)n + 1);
    vsnprintf(buf.data(), buf.size(), fmt, aq);
    s.append(buf.data(), (size_t)n);
  }
  va_end(aq);
}

// Address expression of block/slot `id` (element (r, c) is added by the base
// pointer xb/yb): a block view is the P x P partition of a matrix with
// leading dimension ld; a slot view is a [slots][m][m] workspace.
std::string at(const char* base, const char* stride, int id, int P) {
  std::string s;
  if (P == 0) appendf(s, "%s + %d * mm", base, id);
  else appendf(s, "%s + %d * %s + %d * m", base, id / P, stride, id % P);
  return s;
}

// One term of an ascending sum, as the oracle forms it: +-1 terms are a
// (negated) add; other coefficients multiply first (exact hex literal).
std::string term(const std::string& acc, const std::string& x, double c) {
  std::string s;
  if (c == 1.0) appendf(s, "%s = __dadd_rn(%s, %s);", acc.c_str(), acc.c_str(), x.c_str());
  else if (c == -1.0) appendf(s, "%s = __dadd_rn(%s, -%s);", acc.c_str(), acc.c_str(), x.c_str());
  else appendf(s, "%s = __dadd_rn(%s, __dmul_rn(%a, %s));", acc.c_str(), acc.c_str(), c, x.c_str());
  return s;
}

const char* kPrelude = R"(
typedef long long i64;
template <int VW> struct V { double v[VW]; };
template <int VW> __device__ __forceinline__ V<VW> ldx(const double* p) {
  V<VW> r;
  if constexpr (VW == 4) {
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  } else if constexpr (VW == 2) {
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}
template <int VW> __device__ __forceinline__ V<VW> ldy(const double* p) {
  V<VW> r;
  if constexpr (VW == 4) {
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  } else if constexpr (VW == 2) {
    asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  } else {
    r.v[0] = *p;
  }
  return r;
}
template <int VW> __device__ __forceinline__ void st(double* p, const V<VW>& x) {
  if constexpr (VW == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(x.v[0]), "d"(x.v[1]), "d"(x.v[2]), "d"(x.v[3]) : "memory");
  } else if constexpr (VW == 2) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(x.v[0]), "d"(x.v[1]) : "memory");
  } else {
    p[0] = x.v[0];
  }
}
template <int VW> __device__ __forceinline__ void fin(double* p, V<VW> a, double alpha, int accumulate) {
  if (alpha != 1.0) {
#pragma unroll
    for (int e = 0; e < VW; ++e) a.v[e] = __dmul_rn(alpha, a.v[e]);
  }
  if (accumulate) {
    const V<VW> o = ldy<VW>(p);
#pragma unroll
    for (int e = 0; e < VW; ++e) a.v[e] = __dadd_rn(o.v[e], a.v[e]);
  }
  st<VW>(p, a);
}
)";

}  // namespace

JitShape jit_shape(const MixTable& t) {
  JitShape sh;
  std::vector<char> used(t.nin, 0);
  for (int o = 0; o < t.nout; ++o)
    for (int k = 0; k < t.nin; ++k) used[k] |= t.coef[(size_t)o * t.nin + k] != 0.0;
  int nused = 0;
  for (char u : used) nused += u;
  // register budgets in doubles: held inputs (output-major) / accumulators (input-major)
  auto vw_for = [](int held, int budget) {
    for (int v = 4; v >= 1; v /= 2)
      if (held * v <= budget) return v;
    return 0;
  };
  const int vo = vw_for(nused, 64), vi = vw_for(t.nout, 32);
  if (vo == 0 && vi == 0) return sh;
  sh.input_major = vi > vo || (vi == vo && t.nout < nused);
  sh.vw = sh.input_major ? vi : vo;
  return sh;
}

std::string jit_source(const MixTable& t, int in_P, int out_P, const JitShape& sh) {
  std::string s = kPrelude;
  const int VW = sh.vw;
  appendf(s,
          "extern \"C\" __global__ void __launch_bounds__(256) mf_mix_jit(\n"
          "    const double* __restrict__ X, i64 ldx_, double* __restrict__ Y, i64 ldy_, i64 m,\n"
          "    double alpha, i64 r0, i64 r1, i64 c0, i64 c1, int accumulate) {\n"
          "  constexpr int VW = %d;\n"
          "  const i64 mm = m * m, xs = m * ldx_, ys = m * ldy_;\n"
          "  (void)mm; (void)xs; (void)ys;\n"
          "  const i64 vpr = (c1 - c0) / VW;\n"
          "  const i64 start = (i64)blockIdx.x * blockDim.x + threadIdx.x;\n"
          "  const i64 stride = (i64)gridDim.x * blockDim.x;\n"
          "  const i64 sd = stride / vpr, sm = stride - sd * vpr;\n"
          "  i64 rr = start / vpr, cv = start - rr * vpr;\n"
          "  for (; rr < r1 - r0; rr += sd, cv += sm, (cv >= vpr ? (cv -= vpr, ++rr) : 0)) {\n"
          "    const i64 r = r0 + rr, c = c0 + cv * VW;\n"
          "    const double* xb = X + r * %s + c;\n"
          "    double* yb = Y + r * %s + c;\n",
          VW, in_P ? "ldx_" : "m", out_P ? "ldy_" : "m");
  auto xat = [&](int k) { return at("xb", "xs", k, in_P); };
  auto yat = [&](int o) { return at("yb", "ys", t.out_map[o], out_P); };
  if (!sh.input_major) {
    std::vector<char> used(t.nin, 0);
    for (int o = 0; o < t.nout; ++o)
      for (int k = 0; k < t.nin; ++k) used[k] |= t.coef[(size_t)o * t.nin + k] != 0.0;
    for (int k = 0; k < t.nin; ++k)
      if (used[k]) appendf(s, "    const V<VW> x%d = ldx<VW>(%s);\n", k, xat(k).c_str());
    for (int o = 0; o < t.nout; ++o) {
      s += "    { V<VW> a;\n#pragma unroll\n    for (int e = 0; e < VW; ++e) a.v[e] = -0.0;\n";
      for (int k = 0; k < t.nin; ++k) {
        const double c = t.coef[(size_t)o * t.nin + k];
        if (c == 0.0) continue;
        for (int e = 0; e < VW; ++e) {
          char acc[32], x[32];
          snprintf(acc, sizeof acc, "a.v[%d]", e);
          snprintf(x, sizeof x, "x%d.v[%d]", k, e);
          s += "    " + term(acc, x, c) + "\n";
        }
      }
      appendf(s, "    fin<VW>(%s, a, alpha, accumulate); }\n", yat(o).c_str());
    }
  } else {
    for (int o = 0; o < t.nout; ++o)
      appendf(s, "    V<VW> a%d;\n#pragma unroll\n    for (int e = 0; e < VW; ++e) a%d.v[e] = -0.0;\n", o, o);
    for (int k = 0; k < t.nin; ++k) {
      bool any = false;
      for (int o = 0; o < t.nout; ++o) any = any || t.coef[(size_t)o * t.nin + k] != 0.0;
      if (!any) continue;
      appendf(s, "    { const V<VW> x = ldx<VW>(%s);\n", xat(k).c_str());
      for (int o = 0; o < t.nout; ++o) {
        const double c = t.coef[(size_t)o * t.nin + k];
        if (c == 0.0) continue;
        for (int e = 0; e < VW; ++e) {
          char acc[32], x[32];
          snprintf(acc, sizeof acc, "a%d.v[%d]", o, e);
          snprintf(x, sizeof x, "x.v[%d]", e);
          s += "    " + term(acc, x, c) + "\n";
        }
      }
      s += "    }\n";
    }
    for (int o = 0; o < t.nout; ++o) appendf(s, "    fin<VW>(%s, a%d, alpha, accumulate);\n", yat(o).c_str(), o);
  }
  s += "  }\n}\n";
  return s;
}

bool jit_compile(const std::string& src, const char* arch, std::vector<char>& cubin, std::string& log) {
  Jit* j = jit();
  if (!j->nvrtc_ok()) {
    log = "NVRTC not available";
    return false;
  }
  nvrtcProgram_ prog = nullptr;
  if (j->Create(&prog, src.c_str(), "mf_mix_jit.cu", 0, nullptr, nullptr) != 0) {
    log = "nvrtcCreateProgram failed";
    return false;
  }
  std::string a = std::string("--gpu-architecture=") + arch;
  const char* opts[] = {a.c_str(), "--std=c++17", "--fmad=false", "-default-device", "-lineinfo"};
  const int rc = j->Compile(prog, 5, opts);
  size_t ls = 0;
  j->LogSize(prog, &ls);
  log.assign(ls, '\0');
  if (ls) j->Log(prog, &log[0]);
  bool ok = rc == 0;
  if (ok) {
    size_t n = 0;
    ok = j->CubinSize(prog, &n) == 0 && n > 0;
    if (ok) {
      cubin.resize(n);
      ok = j->Cubin(prog, cubin.data()) == 0;
    }
  }
  j->Destroy(&prog);
  if (const char* dir = getenv("MF_JIT_DUMP")) {  // inspection: source + cubin per kernel
    const size_t h = std::hash<std::string>()(src);
    char path[4096];
    snprintf(path, sizeof path, "%s/mf_mix_jit_%016zx.cu", dir, h);
    if (FILE* f = fopen(path, "w")) { fwrite(src.data(), 1, src.size(), f); fclose(f); }
    snprintf(path, sizeof path, "%s/mf_mix_jit_%016zx.cubin", dir, h);
    if (ok)
      if (FILE* f = fopen(path, "wb")) { fwrite(cubin.data(), 1, cubin.size(), f); fclose(f); }
  }
  return ok;
}

// Process-wide cache of compiled code, keyed by (architecture, source): plans
// of the same triple (or the same batch tables) compile once per process.
namespace {
std::mutex g_cache_mu;
std::map<std::string, std::vector<char>>& cache() {
  static std::map<std::string, std::vector<char>> c;
  return c;
}
bool cache_get(const std::string& src, const char* arch, std::vector<char>& cubin) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = cache().find(std::string(arch) + "\n" + src);
  if (it == cache().end()) return false;
  cubin = it->second;
  return true;
}
void cache_put(const std::string& src, const char* arch, const std::vector<char>& cubin) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  cache()[std::string(arch) + "\n" + src] = cubin;
}
}  // namespace

// Build the generated kernels of a plan's tables on the current device: the
// sources compile in parallel host threads (NVRTC is thread-safe), the
// modules load on the calling thread (its context is the plan's).  A table
// keeps the table-driven kernels when NVRTC or the driver API is missing, its
// shape does not fit in registers, compilation fails, or MF_MIX_NOJIT is set.
int jit_build_all(const std::vector<JitJob>& jobs) {
  if (getenv("MF_MIX_NOJIT") || jobs.empty()) return 0;
  Jit* j = jit();
  if (!j->nvrtc_ok() || !j->driver_ok()) return 0;
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return 0;
  char arch[16];
  snprintf(arch, sizeof arch, "sm_%d%d%s", major, minor, major >= 9 ? "a" : "");
  const size_t n = jobs.size();
  std::vector<std::vector<char>> cubins(n);
  std::vector<JitShape> shapes(n);
  std::vector<char> ok(n, 0);
  std::vector<std::thread> th;
  for (size_t i = 0; i < n; ++i) {
    const JitJob& jb = jobs[i];
    if (!jb.t || jb.t->nout == 0) continue;
    shapes[i] = jit_shape(*jb.t);
    if (shapes[i].vw == 0) continue;
    th.emplace_back([&, i, jb] {
      const std::string src = jit_source(*jb.t, jb.in_P, jb.out_P, shapes[i]);
      if (cache_get(src, arch, cubins[i])) {
        ok[i] = 1;
        return;
      }
      std::string log;
      ok[i] = jit_compile(src, arch, cubins[i], log);
      if (ok[i]) cache_put(src, arch, cubins[i]);
    });
  }
  for (auto& t : th) t.join();
  int built = 0;
  for (size_t i = 0; i < n; ++i) {
    if (!ok[i]) continue;
    CUmodule_ mod = nullptr;
    CUfunction_ fn = nullptr;
    if (j->ModuleLoadData(&mod, cubins[i].data()) != 0) continue;
    if (j->ModuleGetFunction(&fn, mod, "mf_mix_jit") != 0) {
      j->ModuleUnload(mod);
      continue;
    }
    MixTable& t = *jobs[i].t;
    t.jit_mod = mod;
    t.jit_fn = fn;
    t.jit_vw = shapes[i].vw;
    ++built;
  }
  return built;
}

void jit_free(MixTable& t) {
  if (t.jit_mod && jit()->ModuleUnload) jit()->ModuleUnload(t.jit_mod);
  t.jit_mod = t.jit_fn = nullptr;
  t.jit_vw = 0;
}

// Launch t's generated kernel over region `rows` of every block; returns
// cudaErrorNotSupported when it cannot serve these views (no kernel, or a
// vector width the pointers / leading dimensions do not allow).
cudaError_t jit_launch(const MixTable& t, const double* X, int64_t ldx, double* Y, int64_t ldy,
                       int64_t m, double alpha, Rows rows, int accumulate, cudaStream_t s) {
  if (!t.jit_fn) return cudaErrorNotSupported;
  const int vw = t.jit_vw;
  int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  if (r1 <= r0 || c1 <= c0) return cudaSuccess;
  const uintptr_t al = 8 * (uintptr_t)vw;
  if (m % vw || ldx % vw || ldy % vw || c0 % vw || (c1 - c0) % vw ||
      reinterpret_cast<uintptr_t>(X) % al || reinterpret_cast<uintptr_t>(Y) % al)
    return cudaErrorNotSupported;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = (r1 - r0) * ((c1 - c0) / vw);
  int64_t blocks = (work + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sms * 8));
  void* args[] = {&X, &ldx, &Y, &ldy, &m, &alpha, &r0, &r1, &c0, &c1, &accumulate};
  if (jit()->LaunchKernel(t.jit_fn, (unsigned)blocks, 1, 1, 256, 1, 1, 0, s, args, nullptr) != 0)
    return cudaErrorLaunchFailure;
  return cudaSuccess;
}

}  // namespace mf
