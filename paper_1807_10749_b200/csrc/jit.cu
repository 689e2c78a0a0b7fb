// NVRTC compilation and driver-API launch of the specialised pass kernels.
// NVRTC is opened at run time (CUDA 12.x libnvrtc.so.12); driver entry points
// come from cudaGetDriverEntryPoint, so the library has no extra link-time
// dependencies.
#include <cuda.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "jit.hpp"

namespace gs {

namespace {

struct NvrtcApi {
  void* h = nullptr;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*errstr)(nvrtcResult) = nullptr;
  std::string why;
  bool ok = false;
};

struct DriverApi {
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*unload)(CUmodule) = nullptr;
  CUresult (*getfn)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*setattr)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*getattr)(int*, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     CUstream, void**, void**) = nullptr;
  bool ok = false;
  std::string why;
};

NvrtcApi& nvrtc() {
  static NvrtcApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"};
    for (const char* n : names)
      if ((api.h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!api.h) {
      api.why = "libnvrtc.so.12 not found";
      return;
    }
#define GS_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, name))
    GS_SYM(create, "nvrtcCreateProgram");
    GS_SYM(compile, "nvrtcCompileProgram");
    GS_SYM(log_size, "nvrtcGetProgramLogSize");
    GS_SYM(log, "nvrtcGetProgramLog");
    GS_SYM(cubin_size, "nvrtcGetCUBINSize");
    GS_SYM(cubin, "nvrtcGetCUBIN");
    GS_SYM(destroy, "nvrtcDestroyProgram");
    GS_SYM(errstr, "nvrtcGetErrorString");
#undef GS_SYM
    api.ok = api.create && api.compile && api.log_size && api.log && api.cubin_size && api.cubin &&
             api.destroy && api.errstr;
    if (!api.ok) api.why = "libnvrtc is missing symbols";
  });
  return api;
}

DriverApi& driver() {
  static DriverApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* sym, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(sym, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    api.ok = get("cuModuleLoadData", reinterpret_cast<void**>(&api.load)) &&
             get("cuModuleUnload", reinterpret_cast<void**>(&api.unload)) &&
             get("cuModuleGetFunction", reinterpret_cast<void**>(&api.getfn)) &&
             get("cuFuncSetAttribute", reinterpret_cast<void**>(&api.setattr)) &&
             get("cuFuncGetAttribute", reinterpret_cast<void**>(&api.getattr)) &&
             get("cuLaunchKernel", reinterpret_cast<void**>(&api.launch));
    if (!api.ok) {
      cudaGetLastError();
      api.why = "driver entry points unavailable";
    }
  });
  return api;
}

}  // namespace

struct JitModule {
  CUmodule mod = nullptr;
  std::vector<CUfunction> fns;
  std::vector<int> smem_set;
};

bool jit_available(std::string& why) {
  NvrtcApi& n = nvrtc();
  if (!n.ok) {
    why = n.why;
    return false;
  }
  DriverApi& d = driver();
  if (!d.ok) {
    why = d.why;
    return false;
  }
  return true;
}

// On-disk cubin cache keyed by the generated source (compile time only: a
// cached cubin is byte-identical to a fresh compile of the same text).
static std::string cache_path(const std::string& source) {
  const char* dir = std::getenv("GS_JIT_CACHE");
  std::string d = dir ? dir : "/tmp/gridsim_b200_jit";
  if (d.empty() || d == "0") return "";
  mkdir(d.c_str(), 0755);
  char name[64];
  std::snprintf(name, sizeof name, "/%016zx_%zu.cubin", std::hash<std::string>{}(source), source.size());
  return d + name;
}

static JitModule* load_cubin(const std::vector<char>& cubin, const std::vector<std::string>& names, std::string& err);

JitModule* jit_compile(const std::string& source, const std::vector<std::string>& names, const std::string& tag,
                       std::string& err) {
  if (!jit_available(err)) return nullptr;
  const std::string cpath = cache_path(source);
  if (!cpath.empty()) {
    if (FILE* f = std::fopen(cpath.c_str(), "rb")) {
      std::vector<char> cubin;
      char buf[1 << 16];
      size_t r;
      while ((r = std::fread(buf, 1, sizeof buf, f)) > 0) cubin.insert(cubin.end(), buf, buf + r);
      std::fclose(f);
      if (JitModule* m = load_cubin(cubin, names, err)) return m;
    }
  }
  NvrtcApi& n = nvrtc();
  nvrtcProgram prog;
  nvrtcResult r = n.create(&prog, source.c_str(), (tag + ".cu").c_str(), 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) {
    err = std::string("nvrtcCreateProgram: ") + n.errstr(r);
    return nullptr;
  }
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo",
                        "--fmad=true", "-DGS_JIT=1"};
  r = n.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) n.log(prog, &log[0]);
    err = std::string("nvrtc compile failed: ") + log.substr(0, 4000);
    n.destroy(&prog);
    return nullptr;
  }
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  n.cubin(prog, cubin.data());
  n.destroy(&prog);
  if (!cpath.empty()) {
    const std::string tmp = cpath + ".tmp" + std::to_string(getpid());
    if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
      const bool ok = std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
      std::fclose(f);
      if (ok) std::rename(tmp.c_str(), cpath.c_str());
      else std::remove(tmp.c_str());
    }
  }
  return load_cubin(cubin, names, err);
}

static JitModule* load_cubin(const std::vector<char>& cubin, const std::vector<std::string>& names, std::string& err) {
  const int n_kernels = (int)names.size();
  DriverApi& d = driver();
  auto m = std::make_unique<JitModule>();
  CUresult cr = d.load(&m->mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    err = "cuModuleLoadData failed (" + std::to_string((int)cr) + ")";
    return nullptr;
  }
  m->fns.resize(n_kernels);
  m->smem_set.assign(n_kernels, 0);
  for (int i = 0; i < n_kernels; ++i) {
    const std::string& name = names[i];
    cr = d.getfn(&m->fns[i], m->mod, name.c_str());
    if (cr != CUDA_SUCCESS) {
      err = "cuModuleGetFunction(" + name + ") failed";
      d.unload(m->mod);
      return nullptr;
    }
  }
  return m.release();
}

int jit_local_bytes(JitModule* m, int idx) {
  int v = 0;
  if (driver().getattr(&v, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, m->fns[idx]) != CUDA_SUCCESS) return -1;
  return v;
}

int jit_num_regs(JitModule* m, int idx) {
  int v = 0;
  if (driver().getattr(&v, CU_FUNC_ATTRIBUTE_NUM_REGS, m->fns[idx]) != CUDA_SUCCESS) return -1;
  return v;
}

void jit_release(JitModule* m) {
  if (!m) return;
  if (m->mod && driver().ok) driver().unload(m->mod);
  delete m;
}

cudaError_t jit_launch(JitModule* m, int idx, unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       const JArgs& args, std::string& err) {
  DriverApi& d = driver();
  if (m->smem_set[idx] < (int)smem) {
    const CUresult cr = d.setattr(m->fns[idx], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
    if (cr != CUDA_SUCCESS) {
      err = "cuFuncSetAttribute(smem) failed";
      return cudaErrorLaunchFailure;
    }
    m->smem_set[idx] = (int)smem;
  }
  JArgs a = args;
  void* params[] = {&a};
  const CUresult cr = d.launch(m->fns[idx], grid, 1, 1, block, 1, 1, (unsigned)smem,
                               reinterpret_cast<CUstream>(s), params, nullptr);
  if (cr != CUDA_SUCCESS) {
    err = "cuLaunchKernel failed (" + std::to_string((int)cr) + ")";
    return cudaErrorLaunchFailure;
  }
  return cudaSuccess;
}

}  // namespace gs
