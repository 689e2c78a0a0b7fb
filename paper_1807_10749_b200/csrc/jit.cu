// NVRTC compilation and driver-API launch of the specialised pass kernels.
// NVRTC is opened at run time (CUDA 12.x libnvrtc.so.12); driver entry points
// come from cudaGetDriverEntryPoint, so the library has no extra link-time
// dependencies.
#include <cuda.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nvrtc.h>

#include <algorithm>
#include <array>
#include <cstdint>
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
  nvrtcResult (*version)(int*, int*) = nullptr;
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
    GS_SYM(version, "nvrtcVersion");
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

// ---------------------------------------------------------------------------
// On-disk cubin cache.  A cached cubin is byte-identical to a fresh compile of
// the same text, so the cache only saves compile time.  Entries are keyed by
// SHA-256 over (source, NVRTC options, NVRTC version, arch); the file starts
// with that digest and is loaded only when it matches.  The directory is
// per-user ($GS_JIT_CACHE, else $XDG_CACHE_HOME/gridsim_b200_jit, else
// ~/.cache/gridsim_b200_jit), created 0700, and used only when it is a real
// directory owned by this user and not writable by group/other -- a planted
// directory or a symlink disables the cache instead of feeding it kernels.

struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  unsigned char buf[64];
  size_t fill = 0;
  uint64_t total = 0;

  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

  void block(const unsigned char* p) {
    static const uint32_t k[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }

  void update(const void* data, size_t n) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    total += n;
    while (n) {
      const size_t take = std::min(n, sizeof buf - fill);
      std::memcpy(buf + fill, p, take);
      fill += take; p += take; n -= take;
      if (fill == sizeof buf) { block(buf); fill = 0; }
    }
  }
  void update(const std::string& s) {
    const uint64_t len = s.size();  // length-prefixed fields: no ambiguity between them
    update(&len, sizeof len);
    update(s.data(), s.size());
  }

  std::array<unsigned char, 32> digest() {
    const uint64_t bits = total * 8;
    const unsigned char pad = 0x80, zero = 0;
    update(&pad, 1);
    while (fill != 56) update(&zero, 1);
    unsigned char len[8];
    for (int i = 0; i < 8; ++i) len[i] = (unsigned char)(bits >> (56 - 8 * i));
    update(len, 8);
    std::array<unsigned char, 32> out;
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) out[4 * i + j] = (unsigned char)(h[i] >> (24 - 8 * j));
    return out;
  }
};

[[maybe_unused]] static std::string sha256_hex(const std::string& text) {
  Sha256 s;
  s.update(text.data(), text.size());
  const auto d = s.digest();
  static const char* hexd = "0123456789abcdef";
  std::string out;
  for (unsigned char c : d) { out += hexd[c >> 4]; out += hexd[c & 15]; }
  return out;
}

static const char* const kJitOpts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo",
                                       "--fmad=true", "-DGS_JIT=1"};
static const int kJitNopts = (int)(sizeof(kJitOpts) / sizeof(kJitOpts[0]));

static std::array<unsigned char, 32> cache_key(const std::string& source) {
  Sha256 s;
  s.update(std::string("gridsim_b200 jit cubin v2"));
  s.update(source);
  for (int i = 0; i < kJitNopts; ++i) s.update(std::string(kJitOpts[i]));
  int major = 0, minor = 0;
  if (nvrtc().version) nvrtc().version(&major, &minor);
  s.update(std::to_string(major) + "." + std::to_string(minor));
  return s.digest();
}

// The cache directory, or "" when caching is off or the directory is not safe to trust.
static std::string cache_dir() {
  std::string d;
  if (const char* env = std::getenv("GS_JIT_CACHE")) {
    d = env;
    if (d.empty() || d == "0") return "";
  } else if (const char* xdg = std::getenv("XDG_CACHE_HOME"); xdg && *xdg) {
    d = std::string(xdg) + "/gridsim_b200_jit";
  } else if (const char* home = std::getenv("HOME"); home && *home) {
    const std::string base = std::string(home) + "/.cache";
    mkdir(base.c_str(), 0700);
    d = base + "/gridsim_b200_jit";
  } else {
    return "";
  }
  mkdir(d.c_str(), 0700);
  struct stat st;
  if (lstat(d.c_str(), &st) != 0 || !S_ISDIR(st.st_mode) || st.st_uid != geteuid() ||
      (st.st_mode & (S_IWGRP | S_IWOTH)))
    return "";
  return d;
}

static std::string cache_path(const std::array<unsigned char, 32>& key) {
  const std::string d = cache_dir();
  if (d.empty()) return "";
  static const char* hexd = "0123456789abcdef";
  std::string name;
  for (unsigned char c : key) { name += hexd[c >> 4]; name += hexd[c & 15]; }
  return d + "/" + name + ".cubin";
}

static JitModule* load_cubin(const std::vector<char>& cubin, const std::vector<std::string>& names, std::string& err);

JitModule* jit_compile(const std::string& source, const std::vector<std::string>& names, const std::string& tag,
                       std::string& err) {
  if (!jit_available(err)) return nullptr;
  const auto key = cache_key(source);
  const std::string cpath = cache_path(key);
  if (!cpath.empty()) {
    if (FILE* f = std::fopen(cpath.c_str(), "rb")) {
      std::vector<char> blob;
      char buf[1 << 16];
      size_t r;
      while ((r = std::fread(buf, 1, sizeof buf, f)) > 0) blob.insert(blob.end(), buf, buf + r);
      std::fclose(f);
      // the file is <32-byte key><cubin>; a mismatching or short file is ignored
      if (blob.size() > key.size() && std::memcmp(blob.data(), key.data(), key.size()) == 0) {
        std::vector<char> cubin(blob.begin() + key.size(), blob.end());
        if (JitModule* m = load_cubin(cubin, names, err)) return m;
      }
    }
  }
  NvrtcApi& n = nvrtc();
  nvrtcProgram prog;
  nvrtcResult r = n.create(&prog, source.c_str(), (tag + ".cu").c_str(), 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) {
    err = std::string("nvrtcCreateProgram: ") + n.errstr(r);
    return nullptr;
  }
  r = n.compile(prog, kJitNopts, kJitOpts);
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
    const int fd = open(tmp.c_str(), O_WRONLY | O_CREAT | O_EXCL, 0600);
    FILE* f = fd >= 0 ? fdopen(fd, "wb") : nullptr;
    if (!f && fd >= 0) close(fd);
    if (f) {
      const bool ok = std::fwrite(key.data(), 1, key.size(), f) == key.size() &&
                      std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
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
