// Amplitude consumers on the device: the committed
// bitstring batch, rejection sampling (basic / frugal), tail mass with its
// bootstrap, fidelity estimation and probabilities from amplitudes.
//
// Reference: pkg/src/gridsim/sampler.py (committed_indices :83-102,
// sample_basic :135-150, sample_frugal :153-165, tail_mass :177-203) and
// pathsum.py:648-664 (estimate_fidelity).  The random streams are numpy's
// Philox4x64-10 (sampler.py:76-79, key = [seed, lane]) regenerated counter by
// counter, so every draw is bit-identical to the reference's; only the
// floating-point sums (tail, bootstrap, fidelity) differ in summation order.
//
// All of this is HBM-streaming integer/fp64 work: one Philox block (4 or 8
// draws) per thread, grid-stride loops capped at 16 CTAs per SM, no tensor cores.  Pointers may be host or device
// memory (cudaPointerGetAttributes decides); device inputs stay in place, so
// the amplitudes of a gs_run with a device output never leave HBM.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gridsim_b200.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SCHECK(expr)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) return fail(GS_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

// ---- Philox4x64-10 exactly as numpy's bit generator runs it ------------------
// Block b (0-based) runs with counter {b+1, 0, 0, 0}: numpy increments word 0
// before generating each block of 4 outputs.
struct Words4 {
  uint64_t w[4];
};

__device__ __forceinline__ Words4 philox_block(uint64_t block, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t c0 = block + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  Words4 o;
  o.w[0] = c0;
  o.w[1] = c1;
  o.w[2] = c2;
  o.w[3] = c3;
  return o;
}

constexpr int kThreads = 256;

int grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  const int64_t cap = 148 * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return int(g);
}

// ---- kernels ------------------------------------------------------------------
// One Philox block per thread: 8 draws (32-bit words, n <= 32) or 4 (64-bit).
__global__ void committed_kernel(int64_t* out, int64_t count, int64_t offset, int n_qubits, uint64_t seed) {
  const int per = n_qubits <= 32 ? 8 : 4;
  const int64_t first = offset / per, last = (offset + count - 1) / per;
  for (int64_t b = first + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b <= last;
       b += int64_t(gridDim.x) * blockDim.x) {
    Words4 w = philox_block(uint64_t(b), seed, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= per) break;
      const int64_t i = b * per + k - offset;
      if (i < 0 || i >= count) continue;
      // Lemire over a power-of-two range never rejects: the top n bits
      out[i] = per == 8 ? int64_t(uint32_t(k & 1 ? w.w[k >> 1] >> 32 : w.w[k >> 1]) >> (32 - n_qubits))
                        : int64_t(w.w[k] >> (64 - n_qubits));
    }
  }
}

template <int BLOCK>
__device__ __forceinline__ double block_sum(double v) {
  using BR = cub::BlockReduce<double, BLOCK>;
  __shared__ typename BR::TempStorage tmp;
  return BR(tmp).Sum(v);
}

// accept flags + per-block tail partials (fixed order: deterministic); one
// Philox block (4 uniforms) per thread
__global__ void __launch_bounds__(kThreads) sample_kernel(const double* __restrict__ probs, int64_t n, int mode,
                                                          double n_states, double per_sample, uint64_t seed,
                                                          uint8_t* __restrict__ flags, double* __restrict__ partial) {
  double tail = 0.0;
  const double cap = per_sample / n_states;  // m / N (sampler.py:143 / :161)
  const int64_t n_blocks = (n + 3) / 4;
  for (int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b < n_blocks; b += int64_t(gridDim.x) * blockDim.x) {
    Words4 w = philox_block(uint64_t(b), seed, 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = 4 * b + k;
      if (i >= n) break;
      double p = probs[i];
      double u = double(w.w[k] >> 11) * (1.0 / 9007199254740992.0);
      double ratio = __ddiv_rn(__dmul_rn(p, n_states), per_sample);  // probs * n_states / m
      bool acc = mode == 0 ? (p <= cap) && (u < ratio) : u < fmin(1.0, ratio);
      flags[i] = acc ? 1 : 0;
      if (p > cap) tail += p;
    }
  }
  double s = block_sum<kThreads>(tail);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void tail_contrib_kernel(const double* __restrict__ probs, int64_t n, double threshold,
                                    double* __restrict__ contrib, double* __restrict__ partial) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double p = probs[i];
    double c = p > threshold ? p : 0.0;
    contrib[i] = c;
    acc += c;
  }
  double s = block_sum<kThreads>(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Lemire 32-bit bounded draws (numpy buffered_bounded_lemire_uint32): word j
// is kept when its low product half clears the threshold, else the next word
// is drawn -- the stream compaction below turns kept words into picks.
__global__ void bounded_words_kernel(int64_t count, uint32_t size, uint32_t threshold, uint64_t seed,
                                     uint32_t* __restrict__ value, uint8_t* __restrict__ keep) {
  const int64_t n_blocks = (count + 7) / 8;  // 8 32-bit words per Philox block
  for (int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b < n_blocks; b += int64_t(gridDim.x) * blockDim.x) {
    Words4 w = philox_block(uint64_t(b), seed, 2);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t j = 8 * b + k;
      if (j >= count) break;
      uint32_t u = uint32_t(k & 1 ? w.w[k >> 1] >> 32 : w.w[k >> 1]);
      uint64_t m = uint64_t(u) * size;
      value[j] = uint32_t(m >> 32);
      keep[j] = uint32_t(m) >= threshold;
    }
  }
}

// bootstrap sums: blockIdx.y = resample, blockIdx.x = chunk of its picks;
// per-CTA partials are summed on the host in chunk order (deterministic)
__global__ void __launch_bounds__(kThreads) boot_kernel(const double* __restrict__ contrib,
                                                        const uint32_t* __restrict__ picks, int64_t size,
                                                        int64_t chunk, double* __restrict__ partial) {
  const uint32_t* row = picks + int64_t(blockIdx.y) * size;
  const int64_t lo = int64_t(blockIdx.x) * chunk;
  const int64_t hi = lo + chunk < size ? lo + chunk : size;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += __ldg(contrib + __ldcs(row + i));
  double s = block_sum<kThreads>(acc);
  if (threadIdx.x == 0) partial[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) fidelity_kernel(const double2* __restrict__ r, const double2* __restrict__ c,
                                                            int64_t n, double* __restrict__ partial) {
  double rr = 0, cc = 0, re = 0, im = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double2 a = r[i], b = c[i];
    rr += a.x * a.x + a.y * a.y;
    cc += b.x * b.x + b.y * b.y;
    re += a.x * b.x + a.y * b.y;  // conj(a) * b
    im += a.x * b.y - a.y * b.x;
  }
  double s0 = block_sum<kThreads>(rr);
  __syncthreads();
  double s1 = block_sum<kThreads>(cc);
  __syncthreads();
  double s2 = block_sum<kThreads>(re);
  __syncthreads();
  double s3 = block_sum<kThreads>(im);
  if (threadIdx.x == 0) {
    partial[4 * blockIdx.x + 0] = s0;
    partial[4 * blockIdx.x + 1] = s1;
    partial[4 * blockIdx.x + 2] = s2;
    partial[4 * blockIdx.x + 3] = s3;
  }
}

// np.abs(amps) ** 2: hypot, then the square (cli.py:228)
__global__ void probs_kernel(const double2* __restrict__ a, int64_t n, double* __restrict__ p) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double2 z = a[i];
    double h = hypot(z.x, z.y);
    p[i] = h * h;
  }
}

// ---- host helpers ---------------------------------------------------------------
bool is_device_ptr(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Device buffers from the stream-ordered pool (cudaMallocAsync), returned on
// scope exit: repeated calls reuse pool memory instead of paying
// cudaMalloc/cudaFree (a device-wide synchronisation) every time.
struct DevBufs {
  cudaStream_t stream = cudaStreamPerThread;
  std::vector<void*> ptrs;
  ~DevBufs() {
    for (void* p : ptrs) cudaFreeAsync(p, stream);
  }
  template <class T>
  cudaError_t alloc(T** out, int64_t count) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, size_t(count > 0 ? count : 1) * sizeof(T), stream);
    if (e == cudaSuccess) ptrs.push_back(p);
    *out = static_cast<T*>(p);
    return e;
  }
};

// input array on the device: the caller's pointer if it is device memory, else a copy
template <class T>
int device_input(DevBufs& bufs, const T* src, int64_t count, const T** out, cudaStream_t s) {
  if (is_device_ptr(src)) {
    *out = src;
    return GS_OK;
  }
  T* d = nullptr;
  SCHECK(bufs.alloc(&d, count));
  SCHECK(cudaMemcpyAsync(d, src, size_t(count) * sizeof(T), cudaMemcpyHostToDevice, s));
  *out = d;
  return GS_OK;
}

template <class T>
int copy_out(T* dst, const T* src, int64_t count, cudaStream_t s) {
  if (count <= 0) return GS_OK;
  SCHECK(cudaMemcpyAsync(dst, src, size_t(count) * sizeof(T), cudaMemcpyDefault, s));
  return GS_OK;
}

int use_device(int32_t device, cudaStream_t* s) {
  SCHECK(cudaSetDevice(device));
  *s = cudaStreamPerThread;
  // keep up to 4 GiB of freed pool memory for the next call
  static thread_local int configured = -1;
  if (configured != device) {
    cudaMemPool_t pool;
    SCHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = uint64_t(4) << 30;
    SCHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured = device;
  }
  return GS_OK;
}

double sum_partials(const std::vector<double>& v, size_t stride = 1, size_t off = 0) {
  double s = 0.0;
  for (size_t i = off; i < v.size(); i += stride) s += v[i];
  return s;
}

}  // namespace

extern "C" {

const char* gs_sampler_last_error(void) { return g_err.c_str(); }

int gs_committed_indices(int32_t device, int32_t n_qubits, uint64_t seed, int64_t offset, int64_t count,
                         int64_t* out) {
  if (n_qubits < 1 || n_qubits > 63) return fail(GS_ERR_ARG, "n_qubits must be in [1, 63]");
  if (offset < 0) return fail(GS_ERR_ARG, "negative chunk offset " + std::to_string(offset));
  if (count < 0) return fail(GS_ERR_ARG, "negative count");
  if (count == 0) return GS_OK;
  cudaStream_t s;
  int rc = use_device(device, &s);
  if (rc) return rc;
  DevBufs bufs;
  int64_t* d = out;
  bool dev_out = is_device_ptr(out);
  if (!dev_out) SCHECK(bufs.alloc(&d, count));
  committed_kernel<<<grid_for(count / 4 + 2), kThreads, 0, s>>>(d, count, offset, n_qubits, seed);
  SCHECK(cudaGetLastError());
  if (!dev_out) {
    rc = copy_out(out, d, count, s);
    if (rc) return rc;
  }
  SCHECK(cudaStreamSynchronize(s));
  return GS_OK;
}

int gs_sample(int32_t device, int32_t mode, int32_t n_qubits, int32_t per_sample, uint64_t seed, int64_t n,
              const int64_t* indices, const double* probs, int64_t* accepted_out, int64_t* n_accepted,
              double* tail_mass) {
  if (mode != 0 && mode != 1) return fail(GS_ERR_ARG, "mode must be 0 (basic) or 1 (frugal)");
  if (n_qubits < 1 || n_qubits > 62) return fail(GS_ERR_ARG, "n_qubits must be in [1, 62]");
  if (per_sample < 1) return fail(GS_ERR_ARG, "probabilities per sample must be >= 1");
  if (n <= 0 || n % per_sample)
    return fail(GS_ERR_ARG, "batch of " + std::to_string(n) + " is not a multiple of " +
                                std::to_string(per_sample) + " probabilities per sample");
  cudaStream_t s;
  int rc = use_device(device, &s);
  if (rc) return rc;
  DevBufs bufs;
  const double* d_probs;
  const int64_t* d_idx;
  if ((rc = device_input(bufs, probs, n, &d_probs, s))) return rc;
  if ((rc = device_input(bufs, indices, n, &d_idx, s))) return rc;
  uint8_t* flags;
  double* partial;
  int64_t* sel;
  int64_t* d_count;
  const int grid = grid_for((n + 3) / 4);
  SCHECK(bufs.alloc(&flags, n));
  SCHECK(bufs.alloc(&partial, grid));
  SCHECK(bufs.alloc(&sel, n));
  SCHECK(bufs.alloc(&d_count, 1));
  const double n_states = std::ldexp(1.0, n_qubits);
  sample_kernel<<<grid, kThreads, 0, s>>>(d_probs, n, mode, n_states, double(per_sample), seed, flags, partial);
  SCHECK(cudaGetLastError());
  size_t tmp_bytes = 0;
  SCHECK(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, d_idx, flags, sel, d_count, n, s));
  void* tmp;
  SCHECK(bufs.alloc(reinterpret_cast<uint8_t**>(&tmp), int64_t(tmp_bytes)));
  SCHECK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, d_idx, flags, sel, d_count, n, s));
  std::vector<double> hp(grid);
  int64_t count = 0;
  SCHECK(cudaMemcpyAsync(hp.data(), partial, grid * sizeof(double), cudaMemcpyDeviceToHost, s));
  SCHECK(cudaMemcpyAsync(&count, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SCHECK(cudaStreamSynchronize(s));
  if ((rc = copy_out(accepted_out, sel, count, s))) return rc;
  SCHECK(cudaStreamSynchronize(s));
  if (n_accepted) *n_accepted = count;
  // probs[probs > cap].sum() * n_states / probs.size (sampler.py:149 / :164)
  if (tail_mass) *tail_mass = sum_partials(hp) * n_states / double(n);
  return GS_OK;
}

int gs_tail_mass(int32_t device, int32_t n_qubits, int32_t m_star, int32_t resamples, uint64_t seed, int64_t n,
                 const double* probs, double* estimate, double* sigma) {
  if (n <= 0) return fail(GS_ERR_ARG, "need a non-empty 1-d probability batch");
  if (n > (int64_t(1) << 32)) return fail(GS_ERR_ARG, "bootstrap batches are limited to 2^32 entries");
  if (n_qubits < 1 || n_qubits > 62) return fail(GS_ERR_ARG, "n_qubits must be in [1, 62]");
  if (resamples < 1 || resamples > 65535) return fail(GS_ERR_ARG, "resamples must be in [1, 65535]");
  cudaStream_t s;
  int rc = use_device(device, &s);
  if (rc) return rc;
  DevBufs bufs;
  const double* d_probs;
  if ((rc = device_input(bufs, probs, n, &d_probs, s))) return rc;
  const double n_states = std::ldexp(1.0, n_qubits);
  const double threshold = double(m_star) / n_states;
  const double scale = n_states / double(n);
  double* contrib;
  double* partial;
  const int grid = grid_for(n);
  SCHECK(bufs.alloc(&contrib, n));
  SCHECK(bufs.alloc(&partial, grid));
  tail_contrib_kernel<<<grid, kThreads, 0, s>>>(d_probs, n, threshold, contrib, partial);
  SCHECK(cudaGetLastError());
  std::vector<double> hp(grid);
  SCHECK(cudaMemcpyAsync(hp.data(), partial, grid * sizeof(double), cudaMemcpyDeviceToHost, s));

  // bootstrap picks: integers(0, n, size=(resamples, n)) on lane 2
  const int64_t total = int64_t(resamples) * n;
  uint32_t* picks;
  SCHECK(bufs.alloc(&picks, total));
  if (n == 1) {
    // rng == 0: numpy returns the offset without drawing
    SCHECK(cudaMemsetAsync(picks, 0, size_t(total) * sizeof(uint32_t), s));
  } else {
    const uint64_t size = uint64_t(n);
    const uint32_t thr = uint32_t(((uint64_t(1) << 32) - size) % size);
    // expected rejections total * thr / 2^32; draw them plus a margin, retry if short
    int64_t words = total + int64_t(double(total) * (double(thr) / 4294967296.0) * 2.0) + 4096;
    for (;;) {
      DevBufs round;
      uint32_t* value;
      uint8_t* keep;
      int64_t* d_count;
      SCHECK(round.alloc(&value, words));
      SCHECK(round.alloc(&keep, words));
      SCHECK(round.alloc(&d_count, 1));
      bounded_words_kernel<<<grid_for((words + 7) / 8), kThreads, 0, s>>>(words, uint32_t(size), thr, seed, value, keep);
      SCHECK(cudaGetLastError());
      uint32_t* sel;
      SCHECK(round.alloc(&sel, words));
      size_t tmp_bytes = 0;
      SCHECK(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, value, keep, sel, d_count, words, s));
      uint8_t* tmp;
      SCHECK(round.alloc(&tmp, int64_t(tmp_bytes)));
      SCHECK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, value, keep, sel, d_count, words, s));
      int64_t got = 0;
      SCHECK(cudaMemcpyAsync(&got, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      SCHECK(cudaStreamSynchronize(s));
      if (got >= total) {
        SCHECK(cudaMemcpyAsync(picks, sel, size_t(total) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        SCHECK(cudaStreamSynchronize(s));
        break;
      }
      words = words * 2;
    }
  }
  // enough CTAs to fill the machine: ~8 per SM over all resamples, >= 2048 picks each
  int64_t chunks = (int64_t(148) * 8 + resamples - 1) / resamples;
  const int64_t max_chunks = (n + 2047) / 2048;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  if (chunks > 65535) chunks = 65535;
  const int64_t chunk = (n + chunks - 1) / chunks;
  chunks = (n + chunk - 1) / chunk;
  double* bpart;
  SCHECK(bufs.alloc(&bpart, int64_t(resamples) * chunks));
  boot_kernel<<<dim3(unsigned(chunks), unsigned(resamples)), kThreads, 0, s>>>(contrib, picks, n, chunk, bpart);
  SCHECK(cudaGetLastError());
  std::vector<double> hpart(size_t(resamples) * size_t(chunks));
  SCHECK(cudaMemcpyAsync(hpart.data(), bpart, hpart.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  SCHECK(cudaStreamSynchronize(s));
  std::vector<double> hb(resamples, 0.0);
  for (int32_t r = 0; r < resamples; ++r)
    for (int64_t c = 0; c < chunks; ++c) hb[r] += hpart[size_t(r) * size_t(chunks) + size_t(c)];
  if (estimate) *estimate = sum_partials(hp) * scale;
  // boots.std(): population standard deviation (ddof 0)
  double mean = 0.0;
  for (double& b : hb) {
    b *= scale;
    mean += b;
  }
  mean /= double(resamples);
  double var = 0.0;
  for (double b : hb) var += (b - mean) * (b - mean);
  if (sigma) *sigma = std::sqrt(var / double(resamples));
  return GS_OK;
}

int gs_fidelity(int32_t device, int64_t n, const double* ref_re_im, const double* cand_re_im, double* out) {
  if (n <= 0) return fail(GS_ERR_ARG, "empty amplitude batch");
  cudaStream_t s;
  int rc = use_device(device, &s);
  if (rc) return rc;
  DevBufs bufs;
  const double* r;
  const double* c;
  if ((rc = device_input(bufs, ref_re_im, 2 * n, &r, s))) return rc;
  if ((rc = device_input(bufs, cand_re_im, 2 * n, &c, s))) return rc;
  const int grid = grid_for(n);
  double* partial;
  SCHECK(bufs.alloc(&partial, 4 * grid));
  fidelity_kernel<<<grid, kThreads, 0, s>>>(reinterpret_cast<const double2*>(r), reinterpret_cast<const double2*>(c),
                                            n, partial);
  SCHECK(cudaGetLastError());
  std::vector<double> hp(4 * grid);
  SCHECK(cudaMemcpyAsync(hp.data(), partial, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  SCHECK(cudaStreamSynchronize(s));
  const double rr = sum_partials(hp, 4, 0), cc = sum_partials(hp, 4, 1);
  const double re = sum_partials(hp, 4, 2), im = sum_partials(hp, 4, 3);
  if (rr == 0 || cc == 0) return fail(GS_ERR_ARG, "zero-norm batch in fidelity estimate");
  *out = (re * re + im * im) / (rr * cc);
  return GS_OK;
}

int gs_probabilities(int32_t device, int64_t n, const double* amps_re_im, double* probs_out) {
  if (n < 0) return fail(GS_ERR_ARG, "negative count");
  if (n == 0) return GS_OK;
  cudaStream_t s;
  int rc = use_device(device, &s);
  if (rc) return rc;
  DevBufs bufs;
  const double* a;
  if ((rc = device_input(bufs, amps_re_im, 2 * n, &a, s))) return rc;
  double* p = probs_out;
  const bool dev_out = is_device_ptr(probs_out);
  if (!dev_out) SCHECK(bufs.alloc(&p, n));
  probs_kernel<<<grid_for(n), kThreads, 0, s>>>(reinterpret_cast<const double2*>(a), n, p);
  SCHECK(cudaGetLastError());
  if (!dev_out && (rc = copy_out(probs_out, p, n, s))) return rc;
  SCHECK(cudaStreamSynchronize(s));
  return GS_OK;
}

}  // extern "C"
