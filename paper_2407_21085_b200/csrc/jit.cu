// jit.cu — run-time (NVRTC) builds of the SRMDP kernels (see jit.h).
//
// The kernel headers (detmath.cuh, problem.cuh, step_kernel.cuh,
// aux_kernels.cuh) are embedded at build time (build.py writes
// jit_sources.inc), so a user problem is compiled from exactly the code the
// static library is built from: the user's srmdp_user_{b,sigma,f,g} are
// prepended and SRMDP_USER_{DYN,F,G} switch the kernels to them
// (problem.cuh, step_kernel.cuh). Options: sm_100a, --fmad=false (each
// operation written in the user source is one rounding, srmdp.h). The CUBIN is
// loaded with cudaLibraryLoadData and its kernels are launched through the
// runtime like the static ones. libnvrtc.so.12 is opened at run time.
#include <dlfcn.h>
#include <nvrtc.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "jit.h"
#include "jit_sources.inc"   // generated: kJitNames[], kJitSrcs[], kJitCount

namespace {

struct NvrtcApi {
  bool ok = false;
  std::string err;
  decltype(&nvrtcCreateProgram) CreateProgram = nullptr;
  decltype(&nvrtcAddNameExpression) AddNameExpression = nullptr;
  decltype(&nvrtcCompileProgram) CompileProgram = nullptr;
  decltype(&nvrtcGetProgramLogSize) GetProgramLogSize = nullptr;
  decltype(&nvrtcGetProgramLog) GetProgramLog = nullptr;
  decltype(&nvrtcGetCUBINSize) GetCUBINSize = nullptr;
  decltype(&nvrtcGetCUBIN) GetCUBIN = nullptr;
  decltype(&nvrtcGetLoweredName) GetLoweredName = nullptr;
  decltype(&nvrtcDestroyProgram) DestroyProgram = nullptr;
  decltype(&nvrtcGetErrorString) GetErrorString = nullptr;
  decltype(&nvrtcVersion) Version = nullptr;
  int major = 0, minor = 0;
};

NvrtcApi& nvrtc() {
  static NvrtcApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* env = getenv("SRMDP_NVRTC_LIB");
    // the toolkit's NVRTC first (the one the library was built with; torch may
    // have mapped an older libnvrtc.so.12 under the same soname)
    if (env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.err = std::string("cannot load libnvrtc.so.12: ") + dlerror();
      return;
    }
#define SYM(name) api.name = (decltype(api.name))dlsym(h, "nvrtc" #name)
    SYM(CreateProgram);
    SYM(AddNameExpression);
    SYM(CompileProgram);
    SYM(GetProgramLogSize);
    SYM(GetProgramLog);
    SYM(GetCUBINSize);
    SYM(GetCUBIN);
    SYM(GetLoweredName);
    SYM(DestroyProgram);
    SYM(GetErrorString);
    SYM(Version);
#undef SYM
    if (api.Version) api.Version(&api.major, &api.minor);
    api.ok = api.CreateProgram && api.AddNameExpression && api.CompileProgram && api.GetProgramLogSize &&
             api.GetProgramLog && api.GetCUBINSize && api.GetCUBIN && api.GetLoweredName && api.DestroyProgram &&
             api.GetErrorString;
    if (!api.ok) api.err = "libnvrtc.so.12 lacks a required symbol";
  });
  return api;
}

struct Entry {
  JitKernels k;
  cudaLibrary_t lib = nullptr;
};

std::mutex g_mu;
std::map<std::string, std::unique_ptr<Entry>> g_cache;   // modules live for the process

std::string source_of(int d, int q, bool user_dyn, bool user_f, bool user_g, const std::string& user_src) {
  std::string s;
  s += "#define SRMDP_D " + std::to_string(d) + "\n";
  s += "#define SRMDP_Q " + std::to_string(q) + "\n";
  s += "#define SRMDP_USER_DYN " + std::string(user_dyn ? "1" : "0") + "\n";
  s += "#define SRMDP_USER_F " + std::string(user_f ? "1" : "0") + "\n";
  s += "#define SRMDP_USER_G " + std::string(user_g ? "1" : "0") + "\n";
  s += "#define SRMDP_USER_FN __device__ __forceinline__\n";
  s += "#line 1 \"user_src\"\n";
  s += user_src;
  s += "\n;\n#line 1 \"srmdp_jit_kernels\"\n#include \"aux_kernels.cuh\"\n";
  return s;
}

}  // namespace

// NVRTC compile of one module: CUBIN + lowered kernel names (no GPU needed).
static bool compile(const std::string& src, int d, int q, std::vector<char>& cubin, std::string (&lowered)[4],
                    std::string (&names)[4], std::string& err) {
  NvrtcApi& api = nvrtc();
  if (!api.ok) {
    err = api.err;
    return false;
  }
  nvrtcProgram prog = nullptr;
  nvrtcResult r = api.CreateProgram(&prog, src.c_str(), "srmdp_jit.cu", kJitCount, (const char* const*)kJitSrcs,
                                    kJitNames);
  if (r != NVRTC_SUCCESS) {
    err = std::string("nvrtcCreateProgram: ") + api.GetErrorString(r);
    return false;
  }
  const std::string D = std::to_string(d), Q = std::to_string(q);
  names[0] = "srk::step_kernel<" + D + ", " + Q + ", false>";
  names[1] = "srk::step_kernel<" + D + ", " + Q + ", true>";
  names[2] = "srk::eval_kernel<" + D + ", " + Q + ">";
  names[3] = "srk::trace_kernel<" + D + ", " + Q + ">";
  for (const std::string& n : names) api.AddNameExpression(prog, n.c_str());
  // 256-bit loads (ld.global.nc.v4.f64) need NVRTC >= 12.9
  const bool v256 = api.major > 12 || (api.major == 12 && api.minor >= 9);
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo", "-default-device",
                        "-DSRMDP_JIT=1", v256 ? "-DSRMDP_LDG256=1" : "-DSRMDP_LDG256=0"};
  r = api.CompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t log_n = 0;
  api.GetProgramLogSize(prog, &log_n);
  std::string log(log_n, '\0');
  if (log_n) api.GetProgramLog(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    err = std::string("NVRTC build of the user problem failed (") + api.GetErrorString(r) + "):\n" + log;
    api.DestroyProgram(&prog);
    return false;
  }
  size_t n = 0;
  api.GetCUBINSize(prog, &n);
  cubin.resize(n);
  api.GetCUBIN(prog, cubin.data());
  for (int t = 0; t < 4; ++t) {
    const char* ln = nullptr;
    api.GetLoweredName(prog, names[t].c_str(), &ln);
    lowered[t] = ln ? ln : "";
  }
  api.DestroyProgram(&prog);
  return true;
}

bool jit_compile_check(int d, int q, bool user_dyn, bool user_f, bool user_g, const std::string& user_src,
                       std::string& err, size_t* cubin_bytes) {
  std::vector<char> cubin;
  std::string lowered[4], names[4];
  const bool ok = compile(source_of(d, q, user_dyn, user_f, user_g, user_src), d, q, cubin, lowered, names, err);
  if (cubin_bytes) *cubin_bytes = cubin.size();
  return ok;
}

const JitKernels* jit_kernels(int d, int q, bool user_dyn, bool user_f, bool user_g, const std::string& user_src,
                              std::string& err) {
  const std::string src = source_of(d, q, user_dyn, user_f, user_g, user_src);
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(src);
  if (it != g_cache.end()) return &it->second->k;
  std::vector<char> cubin;
  std::string lowered[4], names[4];
  if (!compile(src, d, q, cubin, lowered, names, err)) return nullptr;

  auto e = std::make_unique<Entry>();
  cudaError_t ce = cudaLibraryLoadData(&e->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (ce != cudaSuccess) {
    err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce);
    return nullptr;
  }
  cudaKernel_t* slots[4] = {&e->k.step[0], &e->k.step[1], &e->k.eval, &e->k.trace};
  for (int t = 0; t < 4; ++t) {
    ce = cudaLibraryGetKernel(slots[t], e->lib, lowered[t].c_str());
    if (ce != cudaSuccess) {
      err = "cudaLibraryGetKernel(" + names[t] + "): " + cudaGetErrorString(ce);
      cudaLibraryUnload(e->lib);
      return nullptr;
    }
  }
  e->k.d = d;
  e->k.q = q;
  const JitKernels* out = &e->k;
  g_cache.emplace(src, std::move(e));
  return out;
}
