// Device kernels of the path-sum engine (sm_100a).
//
// gate_pass_kernel   one fused pass of lowered ops over a batch of half-states
//                    (replaces one numpy sweep per op in _exec_ops_batched,
//                    pathsum.py:537-557, and the _b_* kernels :450-513).
// gather_kernel      per-request amplitude gather + fp64 multiply-accumulate
//                    over a batch of leaf states (`land`, pathsum.py:607-615).
// reduce_kernel      deterministic fold of the gather partials into the
//                    complex128 accumulator (fixed order, no atomics).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gs {

// ---------------------------------------------------------------------------
// device op encoding (built on the host by the pass scheduler)

enum DevOpType : int32_t {
  D_MAT1 = 0,  // dense 2x2 on tile bit b0
  D_DIAG1 = 1, // diag(d0,d1) on bit b0 (tile bit, or state bit if g0)
  D_DIAG2 = 2, // diag(d00,d01,d10,d11) on bits (b0,b1) each tile/state
  D_MAT2 = 3,  // dense 4x4 on tile bits (b0 = qa, b1 = qb), |qa qb> order
};

struct DevOp {
  int32_t type;
  int32_t b0, b1;  // tile bit (g*=0) or state bit (g*=1)
  int32_t g0, g1;  // 1 = bit is outside the tile (fixed per tile)
  int32_t coef;    // coefficient offset (non-cross ops)
  int32_t xtab;    // >= 0: cross op; coef = xtable[xtab + digit]
  int32_t xstride; // digit = (node_digits >> 4*xstride) & 15
  int32_t xradix;
  int32_t pad;
};

template <typename R> struct Cx;
template <> struct Cx<float> { using T = float2; };
template <> struct Cx<double> { using T = double2; };

template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <typename V> __device__ __forceinline__ V cmad2(V u0, V a, V u1, V b) {
  // u0*a + u1*b, complex
  V r;
  r.x = u0.x * a.x - u0.y * a.y + u1.x * b.x - u1.y * b.y;
  r.y = u0.x * a.y + u0.y * a.x + u1.x * b.y + u1.y * b.x;
  return r;
}

struct PassArgs {
  const void* src;         // parent states (first pass) or dst (in place)
  void* dst;               // child states
  const int32_t* parent;   // parent slot per child state, nullptr = identity
  const unsigned long long* digit;  // packed 4-bit node digits per child state, may be null
  const DevOp* ops;
  const void* coefs;
  const int32_t* xtable;
  long long state_elems;   // 2^q
  int n_ops;
  int k;                   // tile bits
  int c;                   // low state bits always in the tile (contiguous run)
  int tiles_log;           // q - k
  int init_zero;           // root pass: tile starts as |0...0>
  int n_hi;                // 2^(k-c) entries of hi_off
  int lbits[16];           // tile bit j -> state bit
  int gbits[32];           // tile-id bit j -> state bit
};

template <typename R>
__global__ void __launch_bounds__(256) gate_pass_kernel(PassArgs a) {
  using V = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* tile = reinterpret_cast<V*>(smem_raw);
  const int E = 1 << a.k;
  int* hi_off = reinterpret_cast<int*>(tile + E);
  const int tid = threadIdx.x;
  const int nt = blockDim.x;

  const long long state = (long long)(blockIdx.x >> a.tiles_log);
  const int tile_id = blockIdx.x & ((1 << a.tiles_log) - 1);
  long long base = 0;
  for (int j = 0; j < a.tiles_log; ++j) base |= (long long)((tile_id >> j) & 1) << a.gbits[j];
  // offsets of the strided (non-contiguous) tile bits
  for (int h = tid; h < a.n_hi; h += nt) {
    int off = 0;
    for (int j = a.c; j < a.k; ++j) off |= ((h >> (j - a.c)) & 1) << a.lbits[j];
    hi_off[h] = off;
  }
  __syncthreads();
  const int cmask = (1 << a.c) - 1;

  const V* src = reinterpret_cast<const V*>(a.src);
  V* dst = reinterpret_cast<V*>(a.dst);
  const long long src_state = a.parent ? (long long)a.parent[state] : state;
  if (a.init_zero) {
    for (int t = tid; t < E; t += nt) {
      long long off = base | (t & cmask) | hi_off[t >> a.c];
      V v;
      v.x = (off == 0) ? R(1) : R(0);
      v.y = R(0);
      tile[t] = v;
    }
  } else {
    const V* s = src + src_state * a.state_elems + base;
    for (int t = tid; t < E; t += nt) tile[t] = s[(t & cmask) | hi_off[t >> a.c]];
  }
  __syncthreads();

  const V* coefs = reinterpret_cast<const V*>(a.coefs);
  const unsigned long long node_digit = a.digit ? a.digit[state] : 0ull;
  for (int oi = 0; oi < a.n_ops; ++oi) {
    const DevOp op = a.ops[oi];
    int cofs = op.coef;
    if (op.xtab >= 0) cofs = a.xtable[op.xtab + (int)((node_digit >> (4 * op.xstride)) & 15)];
    const V* u = coefs + cofs;
    if (op.type == D_MAT1) {
      const V u00 = u[0], u01 = u[1], u10 = u[2], u11 = u[3];
      const int j = op.b0;
      const int lo = (1 << j) - 1;
      for (int p = tid; p < (E >> 1); p += nt) {
        const int t0 = ((p & ~lo) << 1) | (p & lo);
        const int t1 = t0 | (1 << j);
        const V v0 = tile[t0], v1 = tile[t1];
        tile[t0] = cmad2(u00, v0, u01, v1);
        tile[t1] = cmad2(u10, v0, u11, v1);
      }
    } else if (op.type == D_DIAG1) {
      const V d0 = u[0], d1 = u[1];
      if (op.g0) {
        const V d = ((base >> op.b0) & 1) ? d1 : d0;
        if (!(d.x == R(1) && d.y == R(0)))
          for (int t = tid; t < E; t += nt) tile[t] = cmul(tile[t], d);
      } else {
        const int j = op.b0;
        for (int t = tid; t < E; t += nt) tile[t] = cmul(tile[t], ((t >> j) & 1) ? d1 : d0);
      }
    } else if (op.type == D_DIAG2) {
      const int f0 = op.g0 ? (int)((base >> op.b0) & 1) : -1;
      const int f1 = op.g1 ? (int)((base >> op.b1) & 1) : -1;
      for (int t = tid; t < E; t += nt) {
        const int i0 = f0 >= 0 ? f0 : ((t >> op.b0) & 1);
        const int i1 = f1 >= 0 ? f1 : ((t >> op.b1) & 1);
        tile[t] = cmul(tile[t], u[2 * i0 + i1]);
      }
    } else {  // D_MAT2, both bits in the tile
      const int ja = op.b0, jb = op.b1;
      const int jl = ja < jb ? ja : jb, jh = ja < jb ? jb : ja;
      for (int p = tid; p < (E >> 2); p += nt) {
        int t = ((p >> jl) << (jl + 1)) | (p & ((1 << jl) - 1));
        t = ((t >> jh) << (jh + 1)) | (t & ((1 << jh) - 1));
        V e[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) e[s] = tile[t | ((s >> 1) << ja) | ((s & 1) << jb)];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          V acc;
          acc.x = R(0);
          acc.y = R(0);
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const V w = u[4 * r + s];
            acc.x += w.x * e[s].x - w.y * e[s].y;
            acc.y += w.x * e[s].y + w.y * e[s].x;
          }
          tile[t | ((r >> 1) << ja) | ((r & 1) << jb)] = acc;
        }
      }
    }
    __syncthreads();
  }

  V* d = dst + state * a.state_elems + base;
  for (int t = tid; t < E; t += nt) d[(t & cmask) | hi_off[t >> a.c]] = tile[t];
}

// ---------------------------------------------------------------------------
// gather: partial[y][i] = sum_{leaf j in group y} w_j * A_j[ia_i] * B_j[ib_i]  (fp64)

// Pauli-sibling leaves of the path-major gathers (engine.cu psib): leaf j of the
// B side is not stored; it is the Pauli image k (-1)^(z.x) base[x ^ flip] of
// the base state `state` (one per parent, evolved without cross terms).
struct SibD {
  int32_t state;
  uint32_t flip, zmask;
  int32_t pad;
  double kr, ki;
};

template <typename R>
__global__ void __launch_bounds__(256)
gather_kernel(const void* A, const void* B, long long a_elems, long long b_elems, int n_leaves,
              int leaves_per_group, const double* weights, const int32_t* ia, const int32_t* ib,
              long long n_req, double2* partial, const SibD* sib) {
  using V = typename Cx<R>::T;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req) return;
  const int j0 = blockIdx.y * leaves_per_group;
  const int j1 = min(n_leaves, j0 + leaves_per_group);
  const V* pa = reinterpret_cast<const V*>(A) + ia[i];
  const unsigned xb = (unsigned)ib[i];
  const V* pb = reinterpret_cast<const V*>(B);
  double re = 0.0, im = 0.0;
  for (int j = j0; j < j1; ++j) {
    const V x = pa[(long long)j * a_elems];
    long long jb = j;
    unsigned xj = xb;
    double wr = weights[j], wi = 0.0;
    if (sib) {
      const SibD sd = sib[j];
      jb = sd.state;
      xj = xb ^ sd.flip;
      const double sg = (__popc(sd.zmask & xb) & 1) ? -wr : wr;
      wr = sg * sd.kr;
      wi = sg * sd.ki;
    }
    const V y = pb[jb * b_elems + xj];
    const double xr = x.x, xi = x.y, yr = y.x, yi = y.y;
    const double pr = xr * yr - xi * yi, pi = xr * yi + xi * yr;
    re += wr * pr - wi * pi;
    im += wr * pi + wi * pr;
  }
  partial[(long long)blockIdx.y * n_req + i] = make_double2(re, im);
}

// ---------------------------------------------------------------------------
// Leaf tails in the gather.  When the last pass of a leaf side only applies
// one-qubit gates on a few qubits T (|T| <= 3) plus diagonal gates (cfg5: the
// final H layer on the qubits the tile had no room for), that pass is not run;
// the gather evaluates it per request instead: the 2^|T| stored amplitudes
// around the requested index, the tail ops on that small vector (fp64), then
// the requested entry -- 2^|T| sector reads per request instead of a full
// read + write of the 2 GiB half-state per leaf.

struct TailOpD {
  int kind;    // 0 mat1 (k0), 1 diag1, 2 diag2, 3 mat2 (k0, k1)
  int k0, k1;  // index of the op's bit in T, or -1 (diag ops on bits outside T)
  int s0, s1;  // state bits
  int pad[3];
  double u[32];  // complex coefficients: mat1 4, diag1 2, diag2 4, mat2 16
};
struct TailProgD {
  int n_ops, t, pad[2];
  int tb[4];  // state bit of tail index bit k
  TailOpD ops[16];
};
__constant__ TailProgD g_tail[2];

template <int T> __device__ __forceinline__ int tail_bit(long long x, int j, int k, int s) {
  return k >= 0 ? ((j >> k) & 1) : (int)((x >> s) & 1);
}

template <int T, int K>
__device__ __forceinline__ void tail_m1(double* vr, double* vi, const double* u) {
#pragma unroll
  for (int j = 0; j < (1 << T); ++j) {
    if ((j >> K) & 1) continue;
    const int f = j | (1 << K);
    const double ar = vr[j], ai = vi[j], br = vr[f], bi = vi[f];
    vr[j] = u[0] * ar - u[1] * ai + u[2] * br - u[3] * bi;
    vi[j] = u[0] * ai + u[1] * ar + u[2] * bi + u[3] * br;
    vr[f] = u[4] * ar - u[5] * ai + u[6] * br - u[7] * bi;
    vi[f] = u[4] * ai + u[5] * ar + u[6] * bi + u[7] * br;
  }
}

template <int T, int K0, int K1>
__device__ __forceinline__ void tail_m2(double* vr, double* vi, const double* u) {
#pragma unroll
  for (int j = 0; j < (1 << T); ++j) {
    if (((j >> K0) & 1) || ((j >> K1) & 1)) continue;
    double xr[4], xi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int id = j | ((q >> 1) << K0) | ((q & 1) << K1);
      xr[q] = vr[id];
      xi[q] = vi[id];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double ur = u[2 * (4 * r + q)], ui = u[2 * (4 * r + q) + 1];
        sr += ur * xr[q] - ui * xi[q];
        si += ur * xi[q] + ui * xr[q];
      }
      const int id = j | ((r >> 1) << K0) | ((r & 1) << K1);
      vr[id] = sr;
      vi[id] = si;
    }
  }
}

template <typename R, int T>
__device__ __forceinline__ double2 tail_amp(const typename Cx<R>::T* st, long long x, int side) {
  using V = typename Cx<R>::T;
  if constexpr (T == 0) {
    const V v = st[x];
    return make_double2((double)v.x, (double)v.y);
  } else {
    constexpr int N = 1 << T;
    const TailProgD& tp = g_tail[side];
    long long x0 = x;
#pragma unroll
    for (int k = 0; k < T; ++k) x0 &= ~(1LL << tp.tb[k]);
    double vr[N], vi[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      long long y = x0;
#pragma unroll
      for (int k = 0; k < T; ++k)
        if ((j >> k) & 1) y |= 1LL << tp.tb[k];
      const V v = st[y];
      vr[j] = v.x;
      vi[j] = v.y;
    }
    for (int o = 0; o < tp.n_ops; ++o) {
      const TailOpD& op = tp.ops[o];
      const double* u = op.u;
      if (op.kind == 0) {  // dense 2x2 on tail bit k0 (static register indices per case)
        switch (op.k0) {
          case 0: tail_m1<T, 0>(vr, vi, u); break;
          case 1: if constexpr (T > 1) tail_m1<T, 1>(vr, vi, u); break;
          default: if constexpr (T > 2) tail_m1<T, 2>(vr, vi, u); break;
        }
      } else if (op.kind == 3) {  // dense 4x4 on tail bits (k0, k1), |s0 s1> order
        if constexpr (T > 1) {
          switch (op.k0 * 4 + op.k1) {
            case 1: tail_m2<T, 0, 1>(vr, vi, u); break;
            case 4: tail_m2<T, 1, 0>(vr, vi, u); break;
            case 2: if constexpr (T > 2) tail_m2<T, 0, 2>(vr, vi, u); break;
            case 8: if constexpr (T > 2) tail_m2<T, 2, 0>(vr, vi, u); break;
            case 6: if constexpr (T > 2) tail_m2<T, 1, 2>(vr, vi, u); break;
            default: if constexpr (T > 2) tail_m2<T, 2, 1>(vr, vi, u); break;
          }
        }
      } else {  // diagonal: entry by the element's bits (tail bits or bits of x)
#pragma unroll
        for (int j = 0; j < N; ++j) {
          int d = tail_bit<T>(x, j, op.k0, op.s0);
          if (op.kind == 2) d = 2 * d + tail_bit<T>(x, j, op.k1, op.s1);
          const double dr = u[2 * d], di = u[2 * d + 1];
          const double ar = vr[j], ai = vi[j];
          vr[j] = dr * ar - di * ai;
          vi[j] = dr * ai + di * ar;
        }
      }
    }
    int jx = 0;
#pragma unroll
    for (int k = 0; k < T; ++k) jx |= (int)((x >> tp.tb[k]) & 1) << k;
    double rr = 0.0, ri = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (j == jx) rr = vr[j], ri = vi[j];
    return make_double2(rr, ri);
  }
}

template <typename R, int TA, int TB>
__global__ void __launch_bounds__(256)
gather_tail_kernel(const void* A, const void* B, long long a_elems, long long b_elems, int n_leaves,
                   int leaves_per_group, const double* weights, const int32_t* ia, const int32_t* ib,
                   long long n_req, double2* partial, const SibD* sib) {
  using V = typename Cx<R>::T;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req) return;
  const int j0 = blockIdx.y * leaves_per_group;
  const int j1 = min(n_leaves, j0 + leaves_per_group);
  const long long xa = ia[i], xb = ib[i];
  double re = 0.0, im = 0.0;
  for (int j = j0; j < j1; ++j) {
    const double2 x = tail_amp<R, TA>(reinterpret_cast<const V*>(A) + (long long)j * a_elems, xa, 0);
    long long jb = j, xj = xb;
    double wr = weights[j], wi = 0.0;
    if (sib) {  // (the tail ops are part of the base state's op list: evaluate them at the flipped index)
      const SibD sd = sib[j];
      jb = sd.state;
      xj = xb ^ (long long)sd.flip;
      const double sg = (__popc(sd.zmask & (unsigned)xb) & 1) ? -wr : wr;
      wr = sg * sd.kr;
      wi = sg * sd.ki;
    }
    const double2 y = tail_amp<R, TB>(reinterpret_cast<const V*>(B) + jb * b_elems, xj, 1);
    const double pr = x.x * y.x - x.y * y.y, pi = x.x * y.y + x.y * y.x;
    re += wr * pr - wi * pi;
    im += wr * pi + wi * pr;
  }
  partial[(long long)blockIdx.y * n_req + i] = make_double2(re, im);
}

// Fold the partials of request slot i into acc[perm ? perm[i] : i]: the
// gathers may run over requests sorted by their A index (perm = the sort's
// permutation), the accumulator stays in request order.
static __global__ void __launch_bounds__(256)
reduce_kernel(const double2* partial, int groups, long long n_req, double2 k, double2* acc, const int32_t* perm) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req) return;
  double2 s = make_double2(0.0, 0.0);
  for (int g = 0; g < groups; ++g) {
    const double2 p = partial[(long long)g * n_req + i];
    s.x += p.x;
    s.y += p.y;
  }
  const long long o = perm ? (long long)perm[i] : i;
  double2 a = acc[o];
  a.x += k.x * s.x - k.y * s.y;
  a.y += k.x * s.y + k.y * s.x;
  acc[o] = a;
}

}  // namespace gs

namespace gs {

// ---------------------------------------------------------------------------
// Shared-memory gather for small half-states (pair <= ~96 KB): a CTA streams a
// group of leaves through a cp.async double buffer (each leaf pair read from
// HBM exactly once, coalesced) while every thread keeps the fp64 accumulators
// of its RPT requests in registers.  Requests are packed ia | ib << qa.

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <typename R, int RPT>
__global__ void __launch_bounds__(512, 1)
gather_smem_kernel(const void* A, const void* B, int qa, int qb, int n_leaves, int leaves_per_group,
                   const double* weights, const uint32_t* packed, long long n_req, int req_per_cta,
                   double2* partial) {
  using V = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int na = 1 << qa, nb = 1 << qb;
  const int pair = na + nb;  // elements per buffer
  V* buf0 = reinterpret_cast<V*>(smem_raw);
  V* buf1 = buf0 + pair;
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long r0 = (long long)blockIdx.x * req_per_cta;
  const int j0 = blockIdx.y * leaves_per_group;
  const int j1 = min(n_leaves, j0 + leaves_per_group);

  uint32_t idx[RPT];
  double acc_re[RPT], acc_im[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const long long i = r0 + tid + (long long)r * nt;
    idx[r] = (i < n_req && (tid + r * nt) < req_per_cta) ? packed[i] : 0xffffffffu;
    acc_re[r] = 0.0;
    acc_im[r] = 0.0;
  }
  const V* gA = reinterpret_cast<const V*>(A);
  const V* gB = reinterpret_cast<const V*>(B);
  constexpr int PER16 = 16 / sizeof(V);  // elements per 16-byte chunk
  auto issue = [&](int j, V* dst) {
    const V* a = gA + (long long)j * na;
    const V* b = gB + (long long)j * nb;
    for (int c = tid; c < na / PER16; c += nt) cp_async16(dst + c * PER16, a + c * PER16);
    for (int c = tid; c < nb / PER16; c += nt) cp_async16(dst + na + c * PER16, b + c * PER16);
    cp_async_commit();
  };
  if (j0 < j1) issue(j0, buf0);
  const uint32_t amask = (uint32_t)na - 1;
  for (int j = j0; j < j1; ++j) {
    V* cur = ((j - j0) & 1) ? buf1 : buf0;
    V* nxt = ((j - j0) & 1) ? buf0 : buf1;
    cp_async_wait_all();
    __syncthreads();  // leaf j resident; everyone done with leaf j-1's buffer
    if (j + 1 < j1) issue(j + 1, nxt);
    const double w = weights[j];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (idx[r] == 0xffffffffu) continue;
      const V x = cur[idx[r] & amask];
      const V y = cur[na + (idx[r] >> qa)];
      const double xr = x.x, xi = x.y, yr = y.x, yi = y.y;
      double pr = xr * yr - xi * yi, pi = xr * yi + xi * yr;
      if (w != 1.0) pr *= w, pi *= w;
      acc_re[r] += pr;
      acc_im[r] += pi;
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const long long i = r0 + tid + (long long)r * nt;
    if (idx[r] != 0xffffffffu)
      partial[(long long)blockIdx.y * n_req + i] = make_double2(acc_re[r], acc_im[r]);
  }
}


// ---------------------------------------------------------------------------
// Gather over grouped path-minor leaf states: leaf j of the chunk, amplitude x
// lives at ((j >> G) * 2^q + x) * 2^G + (j & (2^G - 1)).  A request reads
// 2^G consecutive amplitudes per half and group (64 B for G = 3, complex64),
// all of it useful: 16 bytes per (request, leaf), the algorithmic minimum of
// SURVEY.md §8d.

template <typename V, int W> struct Group { V v[W]; };

template <typename V, int W> __device__ __forceinline__ Group<V, W> load_group(const V* p) {
  Group<V, W> q;
  if constexpr (sizeof(V) == 8 && W == 1) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(p));
    q.v[0] = f;
  } else if constexpr (sizeof(V) == 8) {
#pragma unroll
    for (int k = 0; k < W / 2; ++k) {
      float4 f;
      asm volatile("ld.global.nc.L2::64B.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w)
                   : "l"(reinterpret_cast<const float4*>(p) + k));
      q.v[2 * k] = make_float2(f.x, f.y);
      q.v[2 * k + 1] = make_float2(f.z, f.w);
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) q.v[k] = __ldg(reinterpret_cast<const double2*>(p) + k);
  }
  return q;
}

template <typename R, int GL>
__global__ void __launch_bounds__(256)
gather_grouped_kernel(const void* A, const void* B, long long a_elems, long long b_elems, int n_leaves,
                      int groups_per_y, const double* weights, const int32_t* ia, const int32_t* ib,
                      long long n_req, double2* partial) {
  using V = typename Cx<R>::T;
  constexpr int W = 1 << GL;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req) return;
  const int n_groups = (n_leaves + W - 1) >> GL;
  const int g0 = blockIdx.y * groups_per_y;
  const int g1 = min(n_groups, g0 + groups_per_y);
  const V* pa = reinterpret_cast<const V*>(A) + ((long long)ia[i] << GL);
  const V* pb = reinterpret_cast<const V*>(B) + ((long long)ib[i] << GL);
  double re = 0.0, im = 0.0;
  for (int g = g0; g < g1; ++g) {
    const Group<V, W> x = load_group<V, W>(pa + (((long long)g * a_elems) << GL));
    const Group<V, W> y = load_group<V, W>(pb + (((long long)g * b_elems) << GL));
#pragma unroll
    for (int s = 0; s < W; ++s) {
      const int j = (g << GL) + s;
      if (j >= n_leaves) break;
      const double xr = x.v[s].x, xi = x.v[s].y, yr = y.v[s].x, yi = y.v[s].y;
      const double w = weights[j];
      re += w * (xr * yr - xi * yi);
      im += w * (xr * yi + xi * yr);
    }
  }
  partial[(long long)blockIdx.y * n_req + i] = make_double2(re, im);
}


// Quad form of the grouped gather: 4 lanes per request, each reading a
// 16-byte (complex64) / 32-byte (complex128) quarter of the request's 2^G-leaf
// run, so one warp load covers 8 requests' whole runs (8 L1 wavefronts per
// warp instruction instead of 32 -- the scattered thread-per-request loads
// were L1-wavefront bound).  The four fp64 partial sums meet by shuffles.
template <typename R, int GL>
__global__ void __launch_bounds__(256)
gather_grouped4_kernel(const void* A, const void* B, long long a_elems, long long b_elems, int n_leaves,
                       int groups_per_y, const double* weights, const int32_t* ia, const int32_t* ib,
                       long long n_req, double2* partial) {
  using V = typename Cx<R>::T;
  constexpr int W = 1 << GL;
  constexpr int Q = W / 4;  // leaves per lane
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long i = t >> 2;
  const int sub = (int)(t & 3);
  const bool live = i < n_req;
  const int n_groups = (n_leaves + W - 1) >> GL;
  const int g0 = blockIdx.y * groups_per_y;
  const int g1 = min(n_groups, g0 + groups_per_y);
  const V* pa = reinterpret_cast<const V*>(A) + (live ? ((long long)ia[i] << GL) : 0) + sub * Q;
  const V* pb = reinterpret_cast<const V*>(B) + (live ? ((long long)ib[i] << GL) : 0) + sub * Q;
  double re = 0.0, im = 0.0;
  if (live) {
    // U groups' loads in flight per lane before any is consumed (the loop was
    // one DRAM round trip per group: latency-bound at ~4 TB/s)
    constexpr int U = 4;
    for (int g = g0; g < g1; g += U) {
      Group<V, Q> x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int gg = min(g + u, g1 - 1);
        x[u] = load_group<V, Q>(pa + (((long long)gg * a_elems) << GL));
        y[u] = load_group<V, Q>(pb + (((long long)gg * b_elems) << GL));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (g + u >= g1) break;
#pragma unroll
        for (int s = 0; s < Q; ++s) {
          const int j = ((g + u) << GL) + sub * Q + s;
          if (j < n_leaves) {
            const double xr = x[u].v[s].x, xi = x[u].v[s].y, yr = y[u].v[s].x, yi = y[u].v[s].y;
            const double w = weights[j];
            re += w * (xr * yr - xi * yi);
            im += w * (xr * yi + xi * yr);
          }
        }
      }
    }
  }
  re += __shfl_xor_sync(0xffffffffu, re, 1);
  im += __shfl_xor_sync(0xffffffffu, im, 1);
  re += __shfl_xor_sync(0xffffffffu, re, 2);
  im += __shfl_xor_sync(0xffffffffu, im, 2);
  if (live && sub == 0) partial[(long long)blockIdx.y * n_req + i] = make_double2(re, im);
}


// ---------------------------------------------------------------------------
// Projected leaf side (the paper's sibling structure).  At
// a CZ cut the A-side cross terms are the projectors P0/P1 on the cross
// qubits C; when the leaf level's other A ops are one-qubit gates on C only,
// leaf d's A state is (U_C P_d) psi_parent = product over cross qubits q of
// U_q[x_q, v_q(d)] times psi_parent at x with C's bits set to v(d).  The leaf
// A pass is then not run at all: the gather reads the parent state directly.

struct ProjProgD {
  int n;                 // cross gates of the leaf level (<= 8)
  int side;              // projected side (0 = A, 1 = B)
  int s[8];              // state bit of cross gate k's qubit on that side
  int v[8][16];          // digit -> surviving bit of the projector
  double a[8][16][2];    // digit -> projector value (complex)
  double u[8][8];        // U_q (2x2 complex, row-major): the qubit's leaf gates in order
  int n_swap;            // parent states stored permuted: swap address bits (sa_i, sb_i) in order
  int sa[4], sb[4];
  int abit[8];           // address bit of cross gate k's qubit in the (permuted) parent layout
};
__constant__ ProjProgD g_proj;

// Pauli frame of the grouped side's leaf level (engine.cu pauli_frame): cross
// term d of gate j is x0[j][d] * Z^zsel[j][d] on the gate's qubit, and behind
// the level's other ops that Z is the Pauli i^a[j] X^f[j] Z^z[j].  Masks are in
// tile-bit coordinates of the Pauli-sibling pass; lf = L f and lz = L^-T z are
// their images under the parked tile's address map L (lcol[j] = L e_j), so a
// request at park address A = L t finds sibling s at A ^ lf_s with sign
// (-1)^popc(A & lz_s).
struct PauliProgD {
  int nk;
  int order[8];          // product order, leftmost factor first
  int zsel[8][16];
  double x0[8][16][2];
  int a[8];
  unsigned f[8], z[8];
  unsigned lf[8], lz[8];
  unsigned lcol[16];
};
__constant__ PauliProgD g_pauli;

// Per-leaf factor and source index of the projected side: leaf digits dg,
// block-local index x -> coefficient prod_k a_k(d_k) U_k[x_k, v_k(d_k)] and the
// parent index y = x with every cross qubit set to v_k(d_k).  Tables from
// shared memory (the lanes of a warp index them by different digits).
// one amplitude read with a 64-byte L2 fetch (scattered reads: no 128-byte over-fetch)
template <typename V> __device__ __forceinline__ V ldg_l2_64(const V* p) {
  V v;
  if constexpr (sizeof(V) == 8) {
    asm volatile("ld.global.nc.L2::64B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L2::64B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  }
  return v;
}

struct ProjSmem {
  int n, s[8], v[8][16];
  double a[8][16][2];
  double u[8][8];
  int n_swap, sa[4], sb[4], abit[8];
};

// state index -> address of a permuted parent state (bit swaps, in order)
__device__ __forceinline__ long long proj_addr(const ProjSmem& t, long long y) {
  for (int k = 0; k < t.n_swap; ++k) {
    const long long ba = (y >> t.sa[k]) & 1, bb = (y >> t.sb[k]) & 1;
    if (ba != bb) y ^= (1LL << t.sa[k]) | (1LL << t.sb[k]);
  }
  return y;
}

__device__ __forceinline__ void proj_coef(const ProjSmem& t, long long x, unsigned long long dg, double& cr,
                                          double& ci, long long& y) {
  cr = 1.0, ci = 0.0;
  y = x;
  for (int k = 0; k < t.n; ++k) {
    const int d = (int)((dg >> (4 * k)) & 15ull);
    const int sb = t.s[k];
    const int vb = t.v[k][d];
    const int xb = (int)((x >> sb) & 1);
    const double* u = t.u[k] + 2 * (2 * xb + vb);
    const double fr = t.a[k][d][0] * u[0] - t.a[k][d][1] * u[1];
    const double fi = t.a[k][d][0] * u[1] + t.a[k][d][1] * u[0];
    const double tr = cr * fr - ci * fi;
    ci = cr * fi + ci * fr;
    cr = tr;
    y = (y & ~(1LL << sb)) | ((long long)vb << sb);
  }
}

// Grouped gather with one projected side: the other side's leaves are grouped
// path-minor (2^GL per run, 4 lanes per request as gather_grouped4_kernel);
// the projected side's value of leaf j is coef_j * parent_j[y_j].
// gpar[g] >= 0 marks a "sibling block": the group's 2^GL leaves are the
// children of parent gpar[g] that share their other digits and take the last
// GL (radix-2, v(d) = d) cross digits in order, so leaf j of the group needs
// the parent amplitude at run position j and coef = F(fixed digits) * R(j),
// both products of per-request 2x2 factors computed once; else every leaf
// evaluates proj_coef and reads its own amplitude.
#ifndef GS_PROJ_MINB
#define GS_PROJ_MINB 4  // 4 CTAs per SM (<= 64 registers): latency-bound, occupancy pays (71.1k -> 76.8k cfg4)
#endif
template <typename R, int GL, int LPR>
__global__ void __launch_bounds__(256, GS_PROJ_MINB)
gather_proj_kernel(const void* P, const void* G, long long p_elems, long long g_elems, int n_leaves,
                   int groups_per_y, const double* weights, const int32_t* parent,
                   const unsigned long long* digits, const int32_t* gpar, const int32_t* ia, const int32_t* ib,
                   long long n_req, double2* partial) {
  using V = typename Cx<R>::T;
  constexpr int W = 1 << GL;
  constexpr int Q = W / LPR;  // leaves per lane
  __shared__ ProjSmem tab;
  if (threadIdx.x == 0) {
    tab.n = g_proj.n;
    for (int k = 0; k < 8; ++k) {
      tab.s[k] = g_proj.s[k];
      for (int d = 0; d < 16; ++d) {
        tab.v[k][d] = g_proj.v[k][d];
        tab.a[k][d][0] = g_proj.a[k][d][0];
        tab.a[k][d][1] = g_proj.a[k][d][1];
      }
      for (int e = 0; e < 8; ++e) tab.u[k][e] = g_proj.u[k][e];
    }
    tab.n_swap = g_proj.n_swap;
    for (int k = 0; k < 4; ++k) tab.sa[k] = g_proj.sa[k], tab.sb[k] = g_proj.sb[k];
    for (int k = 0; k < 8; ++k) tab.abit[k] = g_proj.abit[k];
  }
  __syncthreads();
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long i = t / LPR;
  const int sub = (int)(t % LPR);
  if (i >= n_req) return;
  const int n_groups = (n_leaves + W - 1) >> GL;
  const int g0 = blockIdx.y * groups_per_y;
  const int g1 = min(n_groups, g0 + groups_per_y);
  const bool pa = g_proj.side == 0;
  const long long xp = pa ? ia[i] : ib[i];  // index on the projected side
  const long long xg = pa ? ib[i] : ia[i];  // index on the grouped side
  const V* pg = reinterpret_cast<const V*>(G) + (xg << GL) + sub * Q;
  const V* ps = reinterpret_cast<const V*>(P);
  const int nk = tab.n;
  // factor of cross gate k with digit d at this request: a_k(d) U_k[x_k, v_k(d)]
  auto factor = [&](int k, int d, double& ar, double& ai) {
    const int vb = tab.v[k][d], xb = (int)((xp >> tab.s[k]) & 1);
    const double* u = tab.u[k] + 2 * (2 * xb + vb);
    ar = tab.a[k][d][0] * u[0] - tab.a[k][d][1] * u[1];
    ai = tab.a[k][d][0] * u[1] + tab.a[k][d][1] * u[0];
  };
  // this lane's run positions r = sub * Q + s2 (digit of gate nk-1-b = bit b of r):
  // coefficient R(r) and the parent-index bits of the run gates
  double rr[Q], ri[Q];
  long long yrun[Q];
  long long xclr = xp;
  for (int k = 0; k < nk; ++k) xclr &= ~(1LL << tab.s[k]);
#pragma unroll
  for (int s2 = 0; s2 < Q; ++s2) {
    const int r = sub * Q + s2;
    double cr = 1.0, ci = 0.0;
    long long y = 0;
    for (int b = 0; b < GL && b < nk; ++b) {
      const int k = nk - 1 - b, bit = (r >> b) & 1;
      double ar, ai;
      factor(k, bit, ar, ai);
      const double tr = cr * ar - ci * ai;
      ci = cr * ai + ci * ar;
      cr = tr;
      y |= (long long)bit << tab.s[k];
    }
    rr[s2] = cr, ri[s2] = ci, yrun[s2] = proj_addr(tab, y);  // address bits of the run part
  }
  const long long abase = proj_addr(tab, xclr);  // address of x with every cross bit cleared
  // run bit 0 (the last cross gate) at address bit 0: the two run positions of a
  // lane (r = 2 sub, 2 sub + 1) are adjacent amplitudes, 16-byte aligned
  const bool pair16 = nk >= 1 && yrun[0] + 1 == yrun[Q - 1] && (yrun[0] & 1) == 0;
  // fixed (non-run) gates, radix 2: per-request factors for d = 0, 1 (<= 2 such gates)
  double f0r[2][2], f0i[2][2];
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      f0r[k][d] = 1.0, f0i[k][d] = 0.0;
      if (k < nk - GL) factor(k, d, f0r[k][d], f0i[k][d]);
    }
  double re = 0.0, im = 0.0;
  // the group table entries (parent, digits) of group g + 1 are fetched while
  // group g is processed: the parent read no longer waits on a table load
  int pj_next = g0 < g1 ? gpar[g0] : -1;
  unsigned long long dg_next = g0 < g1 ? digits[g0 << GL] : 0ull;
  for (int g = g0; g < g1; ++g) {
    const int j0 = g << GL;
    const Group<V, Q> yv = load_group<V, Q>(pg + (((long long)g * g_elems) << GL));
    const int pj = pj_next;
    const unsigned long long dg_cur = dg_next;
    if (g + 1 < g1) {
      pj_next = gpar[g + 1];
      dg_next = digits[(g + 1) << GL];
    }
    if (pj >= 0) {
      // fixed digits: those of the group's first leaf, gates 0 .. nk - GL - 1
      const unsigned long long dg = dg_cur;
      double Fr = 1.0, Fi = 0.0;
      long long afix = abase;
      for (int k = 0; k < nk - GL; ++k) {
        const int d = (int)((dg >> (4 * k)) & 15ull);
        double ar, ai;
        if (k == 0 && d < 2) ar = d ? f0r[0][1] : f0r[0][0], ai = d ? f0i[0][1] : f0i[0][0];
        else if (k == 1 && d < 2) ar = d ? f0r[1][1] : f0r[1][0], ai = d ? f0i[1][1] : f0i[1][0];
        else factor(k, d, ar, ai);
        const double tr = Fr * ar - Fi * ai;
        Fi = Fr * ai + Fi * ar;
        Fr = tr;
        afix |= (long long)tab.v[k][d] << tab.abit[k];
      }
      const V* pp = ps + (long long)pj * p_elems + afix;
      V pv[Q];
      if (sizeof(V) == 8 && Q == 2 && pair16) {  // the lane's two run positions are adjacent: one 16-byte load
        float4 q4;
        asm volatile("ld.global.nc.L2::64B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(q4.x), "=f"(q4.y), "=f"(q4.z), "=f"(q4.w)
                     : "l"(reinterpret_cast<const float4*>(pp + yrun[0])));
        pv[0].x = q4.x, pv[0].y = q4.y;
        pv[Q - 1].x = q4.z, pv[Q - 1].y = q4.w;
      } else {
#pragma unroll
        for (int s2 = 0; s2 < Q; ++s2) pv[s2] = ldg_l2_64<V>(pp + yrun[s2]);
      }
#pragma unroll
      for (int s2 = 0; s2 < Q; ++s2) {
        const int j = j0 + sub * Q + s2;
        const double cr = Fr * rr[s2] - Fi * ri[s2], ci = Fr * ri[s2] + Fi * rr[s2];
        const double ar = cr * pv[s2].x - ci * pv[s2].y, ai = cr * pv[s2].y + ci * pv[s2].x;
        const double yr = yv.v[s2].x, yi = yv.v[s2].y;
        const double w = weights[j];
        re += w * (ar * yr - ai * yi);
        im += w * (ar * yi + ai * yr);
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < Q; ++s2) {
        const int j = j0 + sub * Q + s2;
        if (j >= n_leaves) continue;
        double cr, ci;
        long long y;
        proj_coef(tab, xp, digits[j], cr, ci, y);
        const V pv = ps[(long long)parent[j] * p_elems + proj_addr(tab, y)];
        const double ar = cr * pv.x - ci * pv.y, ai = cr * pv.y + ci * pv.x;
        const double yr = yv.v[s2].x, yi = yv.v[s2].y;
        const double w = weights[j];
        re += w * (ar * yr - ai * yi);
        im += w * (ar * yi + ai * yr);
      }
    }
  }
  // the 4 lanes of a request are consecutive, live together and finish together
  const unsigned m = __activemask();
#pragma unroll
  for (int o = 1; o < LPR; o <<= 1) {
    re += __shfl_xor_sync(m, re, o);
    im += __shfl_xor_sync(m, im, o);
  }
  if (sub == 0) partial[(long long)blockIdx.y * n_req + i] = make_double2(re, im);
}

// ---------------------------------------------------------------------------
// Request split on the device (split_requests, pathsum.py:122-140): global
// index -> block-local indices, one shift+mask per run of consecutive qubits.

struct SplitRuns {
  int n[2];
  int src[2][32];   // global bit of the run's lowest bit
  int width[2][32];
  int dst[2][32];   // local bit of the run's lowest bit
  int qa;
};

static __global__ void __launch_bounds__(256)
split_kernel(const long long* idx, long long n_req, const SplitRuns r, int32_t* ia, int32_t* ib,
             uint32_t* packed) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req) return;
  const unsigned long long x = (unsigned long long)idx[i];
  unsigned out[2] = {0u, 0u};
#pragma unroll
  for (int b = 0; b < 2; ++b)
    for (int k = 0; k < r.n[b]; ++k)
      out[b] |= (unsigned)((x >> r.src[b][k]) & ((1ull << r.width[b][k]) - 1)) << r.dst[b][k];
  ia[i] = (int32_t)out[0];
  ib[i] = (int32_t)out[1];
  if (packed) packed[i] = out[0] | (out[1] << r.qa);
}


// ---------------------------------------------------------------------------
// Requests bucketed by the tile of the last B-side leaf pass (fused gather):
// tile id = the B-local bits outside the tile, tile-local index = the bits
// inside it (both pext-style over the pass's bit lists).

struct BucketMap {
  int n_g, n_l;
  int gbits[32];
  int lbits[16];
};

static __device__ __forceinline__ void bucket_of(const BucketMap& m, unsigned ib, unsigned& tile, unsigned& tl) {
  tile = 0;
  tl = 0;
  for (int j = 0; j < m.n_g; ++j) tile |= ((ib >> m.gbits[j]) & 1u) << j;
  for (int j = 0; j < m.n_l; ++j) tl |= ((ib >> m.lbits[j]) & 1u) << j;
}

// state *= k (complex), in place: the deferred W-form scalar of a full-state run
template <typename R>
__global__ void scale_state_kernel(void* state, long long n, double kr, double ki) {
  using V = typename Cx<R>::T;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  V* p = reinterpret_cast<V*>(state);
  const V v = p[i];
  const R r = (R)kr, m = (R)ki;
  V o;
  o.x = v.x * r - v.y * m;
  o.y = v.x * m + v.y * r;
  p[i] = o;
}

// request sort helpers (gather locality): v[i] = i; dst[i] = src[perm[i]]
static __global__ void iota_kernel(int32_t* v, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}
static __global__ void permute_kernel(const int32_t* src, const int32_t* perm, int32_t* dst, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

// Fine bins of the Pauli-sibling pass (fine = 1): bin = tile * 32 + half * 16 + (xc & 15), where
// half is bit 3 of the request's park address (which 64-byte half of the shared-memory banks its
// sibling run occupies) and xc its projected-side cross bits (its row of the factor table).  Each
// tile's requests then form two streams (half 0, half 1), each sorted by xc: the pass gives the
// even lane quads stream 0 and the odd quads stream 1, so the two runs an 8-lane phase of a
// 16-byte shared load touches never share banks, and factor-table reads mostly broadcast.
static __device__ __forceinline__ unsigned bucket_bin(const BucketMap& m, unsigned ib, unsigned ia, int fine,
                                                      unsigned& tl) {
  unsigned t;
  bucket_of(m, ib, t, tl);
  if (!fine) return t;
  unsigned adr = 0;
  for (int j = 0; j < 16; ++j)
    if ((tl >> j) & 1u) adr ^= g_pauli.lcol[j];
  unsigned xc = 0;
  for (int k = 0; k < g_proj.n; ++k) xc |= ((ia >> g_proj.s[k]) & 1u) << k;
  return (t << 5) | (((adr >> 3) & 1u) << 4) | (xc & 15u);
}

static __global__ void bucket_count_kernel(const int32_t* ib, const int32_t* ia, long long n, const BucketMap m,
                                           int32_t* count, int fine) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned l;
  const unsigned t = bucket_bin(m, (unsigned)ib[i], (unsigned)ia[i], fine, l);
  atomicAdd(count + t, 1);
}

static __global__ void bucket_fill_kernel(const int32_t* ib, const int32_t* ia, long long n, const BucketMap m,
                                          int32_t* cursor, int32_t* breq, int32_t* btl, int32_t* bia, int fine) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned l;
  const unsigned t = bucket_bin(m, (unsigned)ib[i], (unsigned)ia[i], fine, l);
  const int pos = atomicAdd(cursor + t, 1);
  breq[pos] = (int32_t)i;
  btl[pos] = (int32_t)l;
  bia[pos] = ia[i];
}

// Fused projected-leaf pass (jitgen::proj_fused_kernel), request side: per
// bucket slot, the projected-side index with its leaf-level cross bits cleared
// and the parent layout's bit swaps applied (abase), and the tile-local index
// of the grouped side packed with the request's cross bits (tl | xc << 16).
static __global__ void pf_meta_kernel(const int32_t* bia, const int32_t* btl, long long n, int2* meta, int pauli) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned tl = (unsigned)btl[i];
  if (pauli) {  // Pauli-sibling pass: the request's address in the parked tile
    unsigned t = 0;
    for (int j = 0; j < 16; ++j)
      if ((tl >> j) & 1u) t ^= g_pauli.lcol[j];
    tl = t;
  }
  long long x = bia[i];
  int xc = 0;
  for (int k = 0; k < g_proj.n; ++k) {
    xc |= (int)((x >> g_proj.s[k]) & 1) << k;
    x &= ~(1LL << g_proj.s[k]);
  }
  for (int w = 0; w < g_proj.n_swap; ++w) {
    const int a = g_proj.sa[w], b = g_proj.sb[w];
    if (((x >> a) & 1) != ((x >> b) & 1)) x ^= (1LL << a) | (1LL << b);
  }
  meta[i] = make_int2((int)tl | (xc << 16), (int)x);
}

// Fused projected-leaf pass, leaf side: per leaf group g (8 sibling slots) and
// request cross bits xc, the projected factor c = w * prod_k a_k(d_k) U_k[xc_k, v_k(d_k)]
// (complex64, as the leaf's own complex64 state would hold it) and, per slot,
// the parent amplitude offset parent * p_elems + sum_k v_k(d_k) << abit_k.
// Slots past n_states get c = 0.  One CTA per group, one thread per (xc, slot).
static __global__ void pf_table_kernel(const unsigned long long* digits, const int32_t* parent,
                                       const double* weights, long long n_states, long long p_elems,
                                       float2* tab, long long* aoff) {
  const int nk = g_proj.n, t = threadIdx.x;
  if (t >= (8 << nk)) return;
  const long long g = blockIdx.x;
  const int s = t & 7, xc = t >> 3;  // table layout [group][xc][slot]: a request's 8 factors are contiguous
  const long long slot = (g << 3) | s;
  float2 c = make_float2(0.f, 0.f);
  long long off = 0;
  if (slot < n_states) {
    const unsigned long long dg = digits[slot];
    double pr = weights[slot], pi = 0.0;
    off = (long long)parent[slot] * p_elems;
    for (int k = 0; k < nk; ++k) {
      const int d = (int)((dg >> (4 * k)) & 15ull);
      const int vb = g_proj.v[k][d], xb = (xc >> k) & 1;
      const double* u = g_proj.u[k] + 2 * (2 * xb + vb);
      const double fr = g_proj.a[k][d][0] * u[0] - g_proj.a[k][d][1] * u[1];
      const double fi = g_proj.a[k][d][0] * u[1] + g_proj.a[k][d][1] * u[0];
      const double tr = pr * fr - pi * fi;
      pi = pr * fi + pi * fr;
      pr = tr;
      off |= (long long)vb << g_proj.abit[k];
    }
    c = make_float2((float)pr, (float)pi);
  }
  tab[(g << (3 + nk)) + t] = c;
  if (xc == 0) aoff[(g << 3) + s] = off;
}

// Pauli-sibling form of the table: the projected factor above times the grouped
// side's sibling scalar prod_j x0_j(d_j) * i^a (-1)^(z.f) of the slot's Pauli
// P = prod_j P_j^zsel_j(d_j) (product in g_pauli.order), and per slot the park
// address flip and sign-parity mask of that Pauli (bflip = lf | lz << 16).
static __global__ void pf_table_pauli_kernel(const unsigned long long* digits, const int32_t* parent,
                                             const double* weights, long long n_states, long long p_elems,
                                             float2* tab, long long* aoff, unsigned* bflip) {
  const int nk = g_proj.n, t = threadIdx.x;
  if (t >= (8 << nk)) return;
  const long long g = blockIdx.x;
  const int s = t & 7, xc = t >> 3;
  const long long slot = (g << 3) | s;
  float2 c = make_float2(0.f, 0.f);
  long long off = 0;
  unsigned lf = 0, lz = 0;
  if (slot < n_states) {
    const unsigned long long dg = digits[slot];
    double pr = weights[slot], pi = 0.0;
    off = (long long)parent[slot] * p_elems;
    for (int k = 0; k < nk; ++k) {
      const int d = (int)((dg >> (4 * k)) & 15ull);
      const int vb = g_proj.v[k][d], xb = (xc >> k) & 1;
      const double* u = g_proj.u[k] + 2 * (2 * xb + vb);
      const double fr = g_proj.a[k][d][0] * u[0] - g_proj.a[k][d][1] * u[1];
      const double fi = g_proj.a[k][d][0] * u[1] + g_proj.a[k][d][1] * u[0];
      const double tr = pr * fr - pi * fi;
      pi = pr * fi + pi * fr;
      pr = tr;
      off |= (long long)vb << g_proj.abit[k];
    }
    int a = 0;
    unsigned f = 0, z = 0;
    for (int i = 0; i < g_pauli.nk; ++i) {
      const int j = g_pauli.order[i];
      const int d = (int)((dg >> (4 * j)) & 15ull);
      const double xr = g_pauli.x0[j][d][0], xi = g_pauli.x0[j][d][1];
      const double tr = pr * xr - pi * xi;
      pi = pr * xi + pi * xr;
      pr = tr;
      if (g_pauli.zsel[j][d]) {  // (i^a X^f Z^z)(i^b X^g Z^h) = i^(a+b) (-1)^(z.g) X^(f^g) Z^(z^h)
        a += g_pauli.a[j] + 2 * (__popc(z & g_pauli.f[j]) & 1);
        f ^= g_pauli.f[j];
        z ^= g_pauli.z[j];
        lf ^= g_pauli.lf[j];
        lz ^= g_pauli.lz[j];
      }
    }
    a += 2 * (__popc(z & f) & 1);  // (P phi)[x] = i^a (-1)^(z.f) (-1)^(z.x) phi[x ^ f]
    switch (a & 3) {
      case 1: { const double tr = -pi; pi = pr; pr = tr; } break;
      case 2: pr = -pr, pi = -pi; break;
      case 3: { const double tr = pi; pi = -pr; pr = tr; } break;
      default: break;
    }
    c = make_float2((float)pr, (float)pi);
  }
  tab[(g << (3 + nk)) + t] = c;
  if (xc == 0) {
    aoff[(g << 3) + s] = off;
    bflip[(g << 3) + s] = lf | (lz << 16);
  }
}

}  // namespace gs
