// Register-staged gate pass (sm_100a).
//
// One CTA owns a 2^K-amplitude tile: kq bits of one half-state (plus K-kq
// "slot" bits that batch several small states into one CTA).  Each thread
// holds 2^M amplitudes in registers.  A pass is a sequence of *stages*; a
// stage fixes which M tile bits live in registers, applies every op on those
// bits (plus any diagonal op, whose other bits are thread-uniform), then the
// tile is re-shuffled through shared memory into the next stage's mapping.
// Stage 0 loads straight from HBM and the last stage stores straight to HBM;
// both keep the low 5 tile bits on the lanes, so every warp access is a
// contiguous 256 B run.  This replaces the reference's one numpy sweep per op
// (`_exec_ops_batched`, pathsum.py:537-557; `_b_mat1/_b_diag1/_b_diag2/_b_mat2`,
// pathsum.py:454-513) by one HBM read + write per pass for tens of ops.
//
// W-form gates (H, X^1/2, Y^1/2 = s * W with W entries in {+-1, +-i}) are
// applied as W (two adds per amplitude); the scalar s is folded by the host
// into one complex constant per block, and powers of two are applied at the
// pass store to keep magnitudes in range (exact in binary floating point).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "pass_types.h"

namespace gs {

template <typename V> __device__ __forceinline__ bool is_one(V d) { return d.x == 1 && d.y == 0; }
template <typename V> __device__ __forceinline__ bool is_zero(V d) { return d.x == 0 && d.y == 0; }
template <typename V> __device__ __forceinline__ bool is_mone(V d) { return d.x == -1 && d.y == 0; }

// 0 identity, 1 zero, 2 negate, 3 general
template <typename V> __device__ __forceinline__ int dkind(V d) {
  return is_one(d) ? 0 : is_zero(d) ? 1 : is_mone(d) ? 2 : 3;
}

template <typename V> __device__ __forceinline__ V dapply(V x, V d, int kind) {
  if (kind == 1) { x.x = 0; x.y = 0; return x; }
  if (kind == 2) { x.x = -x.x; x.y = -x.y; return x; }
  return cmul(x, d);
}

template <int M, typename V> __device__ __forceinline__ void scale_all(V (&v)[1 << M], V d) {
  const int kind = dkind(d);
  if (kind == 0) return;
#pragma unroll
  for (int e = 0; e < (1 << M); ++e) v[e] = dapply(v[e], d, kind);
}

// diag(d0, d1) on register bit B
template <int M, int B, typename V>
__device__ __forceinline__ void d1_reg(V (&v)[1 << M], V d0, V d1) {
  const int k0 = dkind(d0), k1 = dkind(d1);
  if (k0)
#pragma unroll
    for (int e = 0; e < (1 << M); ++e)
      if (!((e >> B) & 1)) v[e] = dapply(v[e], d0, k0);
  if (k1)
#pragma unroll
    for (int e = 0; e < (1 << M); ++e)
      if ((e >> B) & 1) v[e] = dapply(v[e], d1, k1);
}

// diag on register bits (A = qa, B = qb): amplitude (a, b) times d[2a + b]
template <int M, int A, int B, typename V>
__device__ __forceinline__ void d2_reg(V (&v)[1 << M], const V* d) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const V dq = d[q];
    const int kind = dkind(dq);
    if (!kind) continue;
#pragma unroll
    for (int e = 0; e < (1 << M); ++e)
      if ((((e >> A) & 1) << 1 | ((e >> B) & 1)) == q) v[e] = dapply(v[e], dq, kind);
  }
}

template <int M, int B, typename V>
__device__ __forceinline__ void m1_reg(V (&v)[1 << M], V u00, V u01, V u10, V u11) {
#pragma unroll
  for (int e = 0; e < (1 << M); ++e) {
    if ((e >> B) & 1) continue;
    const V x0 = v[e], x1 = v[e | (1 << B)];
    v[e] = cmad2(u00, x0, u01, x1);
    v[e | (1 << B)] = cmad2(u10, x0, u11, x1);
  }
}

// W-forms: H = [[1,1],[1,-1]], X = [[1,-i],[-i,1]], Y = [[1,-1],[1,1]]
template <int M, int B, int W, typename V> __device__ __forceinline__ void w_reg(V (&v)[1 << M]) {
#pragma unroll
  for (int e = 0; e < (1 << M); ++e) {
    if ((e >> B) & 1) continue;
    const V x0 = v[e], x1 = v[e | (1 << B)];
    V y0, y1;
    if (W == 0) {
      y0.x = x0.x + x1.x; y0.y = x0.y + x1.y;
      y1.x = x0.x - x1.x; y1.y = x0.y - x1.y;
    } else if (W == 1) {
      y0.x = x0.x + x1.y; y0.y = x0.y - x1.x;
      y1.x = x1.x + x0.y; y1.y = x1.y - x0.x;
    } else {
      y0.x = x0.x - x1.x; y0.y = x0.y - x1.y;
      y1.x = x0.x + x1.x; y1.y = x0.y + x1.y;
    }
    v[e] = y0;
    v[e | (1 << B)] = y1;
  }
}

// coefficient load that the compiler may not hoist out of the unrolled group
// loop (keeps a 4x4's 16 complex entries out of the register file)
__device__ __forceinline__ float2 ld_coef(const float2* p) {
  float2 r;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_coef(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

template <int M, int A, int B, typename V>
__device__ __forceinline__ void m2_reg(V (&v)[1 << M], const V* u) {
#pragma unroll
  for (int e = 0; e < (1 << M); ++e) {
    if (((e >> A) & 1) || ((e >> B) & 1)) continue;
    V x[4], y[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) x[s] = v[e | ((s >> 1) << A) | ((s & 1) << B)];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      y[r].x = 0;
      y[r].y = 0;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const V w = ld_coef(u + 4 * r + s);
        y[r].x += w.x * x[s].x - w.y * x[s].y;
        y[r].y += w.x * x[s].y + w.y * x[s].x;
      }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) v[e | ((s >> 1) << A) | ((s & 1) << B)] = y[s];
  }
}

template <int M, int A, int B, typename V> __device__ __forceinline__ void d2_chk(V (&v)[1 << M], const V* d) {
  if constexpr (A != B && A < M && B < M) d2_reg<M, A, B>(v, d);
}
template <int M, int A, int B, typename V> __device__ __forceinline__ void m2_chk(V (&v)[1 << M], const V* u) {
  if constexpr (A != B && A < M && B < M) m2_reg<M, A, B>(v, u);
}

// runtime register-bit -> template dispatch
#define GS_CASE1(M, B, CALL) \
  case B:                    \
    if constexpr (B < M) { CALL; } break;

template <int M, typename V> __device__ __forceinline__ void d1_dispatch(V (&v)[1 << M], int r, V d0, V d1) {
  switch (r) {
    GS_CASE1(M, 0, (d1_reg<M, 0>(v, d0, d1)))
    GS_CASE1(M, 1, (d1_reg<M, 1>(v, d0, d1)))
    GS_CASE1(M, 2, (d1_reg<M, 2>(v, d0, d1)))
    GS_CASE1(M, 3, (d1_reg<M, 3>(v, d0, d1)))
    GS_CASE1(M, 4, (d1_reg<M, 4>(v, d0, d1)))
  }
}

template <int M, typename V> __device__ __forceinline__ void m1_dispatch(V (&v)[1 << M], int r, const V* u) {
  const V u00 = u[0], u01 = u[1], u10 = u[2], u11 = u[3];
  switch (r) {
    GS_CASE1(M, 0, (m1_reg<M, 0>(v, u00, u01, u10, u11)))
    GS_CASE1(M, 1, (m1_reg<M, 1>(v, u00, u01, u10, u11)))
    GS_CASE1(M, 2, (m1_reg<M, 2>(v, u00, u01, u10, u11)))
    GS_CASE1(M, 3, (m1_reg<M, 3>(v, u00, u01, u10, u11)))
    GS_CASE1(M, 4, (m1_reg<M, 4>(v, u00, u01, u10, u11)))
  }
}

template <int M, int W, typename V> __device__ __forceinline__ void w_dispatch_r(V (&v)[1 << M], int r) {
  switch (r) {
    GS_CASE1(M, 0, (w_reg<M, 0, W>(v)))
    GS_CASE1(M, 1, (w_reg<M, 1, W>(v)))
    GS_CASE1(M, 2, (w_reg<M, 2, W>(v)))
    GS_CASE1(M, 3, (w_reg<M, 3, W>(v)))
    GS_CASE1(M, 4, (w_reg<M, 4, W>(v)))
  }
}

template <int M, typename V> __device__ __forceinline__ void w_dispatch(V (&v)[1 << M], int w, int r) {
  if (w == 0) w_dispatch_r<M, 0>(v, r);
  else if (w == 1) w_dispatch_r<M, 1>(v, r);
  else w_dispatch_r<M, 2>(v, r);
}

template <int M, int A, typename V> __device__ __forceinline__ void d2_dispatch_b(V (&v)[1 << M], int b, const V* d) {
  switch (b) {
    GS_CASE1(M, 0, (d2_chk<M, A, 0>(v, d)))
    GS_CASE1(M, 1, (d2_chk<M, A, 1>(v, d)))
    GS_CASE1(M, 2, (d2_chk<M, A, 2>(v, d)))
    GS_CASE1(M, 3, (d2_chk<M, A, 3>(v, d)))
    GS_CASE1(M, 4, (d2_chk<M, A, 4>(v, d)))
  }
}

template <int M, typename V> __device__ __forceinline__ void d2_dispatch(V (&v)[1 << M], int a, int b, const V* d) {
  switch (a) {
    GS_CASE1(M, 0, (d2_dispatch_b<M, 0>(v, b, d)))
    GS_CASE1(M, 1, (d2_dispatch_b<M, 1>(v, b, d)))
    GS_CASE1(M, 2, (d2_dispatch_b<M, 2>(v, b, d)))
    GS_CASE1(M, 3, (d2_dispatch_b<M, 3>(v, b, d)))
    GS_CASE1(M, 4, (d2_dispatch_b<M, 4>(v, b, d)))
  }
}

template <int M, int A, typename V> __device__ __forceinline__ void m2_dispatch_b(V (&v)[1 << M], int b, const V* u) {
  switch (b) {
    GS_CASE1(M, 0, (m2_chk<M, A, 0>(v, u)))
    GS_CASE1(M, 1, (m2_chk<M, A, 1>(v, u)))
    GS_CASE1(M, 2, (m2_chk<M, A, 2>(v, u)))
    GS_CASE1(M, 3, (m2_chk<M, A, 3>(v, u)))
    GS_CASE1(M, 4, (m2_chk<M, A, 4>(v, u)))
  }
}

template <int M, typename V> __device__ __forceinline__ void m2_dispatch(V (&v)[1 << M], int a, int b, const V* u) {
  switch (a) {
    GS_CASE1(M, 0, (m2_dispatch_b<M, 0>(v, b, u)))
    GS_CASE1(M, 1, (m2_dispatch_b<M, 1>(v, b, u)))
    GS_CASE1(M, 2, (m2_dispatch_b<M, 2>(v, b, u)))
    GS_CASE1(M, 3, (m2_dispatch_b<M, 3>(v, b, u)))
    GS_CASE1(M, 4, (m2_dispatch_b<M, 4>(v, b, u)))
  }
}

__device__ __forceinline__ int bit_value(int where, int idx, int tb, long long base) {
  return where == B_THREAD ? ((tb >> idx) & 1) : (int)((base >> idx) & 1);
}

template <int M, typename V>
__device__ __forceinline__ void apply_ops(V (&v)[1 << M], const Pass2Args& a, int ob, int oe, int tb,
                                          long long base, int node_digit) {
  const V* coefs = reinterpret_cast<const V*>(a.coefs);
  for (int oi = ob; oi < oe; ++oi) {
    const POp op = a.ops[oi];
    int cofs = op.coef;
    if (op.xtab >= 0) cofs = __ldg(a.xtable + op.xtab + (node_digit / op.xstride) % op.xradix);
    const V* u = coefs + cofs;
    switch (op.type) {
      case P_W:
        w_dispatch<M>(v, op.w, op.idx0);
        break;
      case P_M1:
        m1_dispatch<M>(v, op.idx0, u);
        break;
      case P_D1:
        if (op.where0 == B_REG) d1_dispatch<M>(v, op.idx0, u[0], u[1]);
        else scale_all<M>(v, u[bit_value(op.where0, op.idx0, tb, base)]);
        break;
      case P_D2: {
        const bool r0 = op.where0 == B_REG, r1 = op.where1 == B_REG;
        if (r0 && r1) {
          d2_dispatch<M>(v, op.idx0, op.idx1, u);
        } else if (r0) {
          const int b1 = bit_value(op.where1, op.idx1, tb, base);
          d1_dispatch<M>(v, op.idx0, u[b1], u[2 + b1]);
        } else if (r1) {
          const int b0 = bit_value(op.where0, op.idx0, tb, base);
          d1_dispatch<M>(v, op.idx1, u[2 * b0], u[2 * b0 + 1]);
        } else {
          const int b0 = bit_value(op.where0, op.idx0, tb, base);
          const int b1 = bit_value(op.where1, op.idx1, tb, base);
          scale_all<M>(v, u[2 * b0 + b1]);
        }
        break;
      }
      default:
        m2_dispatch<M>(v, op.idx0, op.idx1, u);
        break;
    }
  }
}

// XOR swizzle of the low 4 (c64) / 3 (c128) address bits with higher bits:
// bijective on [0, 2^K), spreads strided lane patterns across banks.
template <typename V> __device__ __forceinline__ int swz(int t) {
  constexpr int LB = sizeof(V) == 8 ? 4 : 3;
  constexpr int LM = (1 << LB) - 1;
  return t ^ (((t >> LB) ^ (t >> (2 * LB)) ^ (t >> (3 * LB))) & LM);
}

__device__ __forceinline__ int deposit(int x, unsigned mask, int K) {
  int out = 0, n = 0;
  for (int j = 0; j < K; ++j)
    if ((mask >> j) & 1) out |= ((x >> n++) & 1) << j;
  return out;
}

template <typename R, int M>
__global__ void __launch_bounds__(256) pass2_kernel(const Pass2Args a) {
  using V = typename Cx<R>::T;
  constexpr int E = 1 << M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* tile = reinterpret_cast<V*>(smem_raw);
  const int K = a.K;
  int* hi_off = reinterpret_cast<int*>(tile + (1 << K));
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const unsigned full = (1u << K) - 1;

  const long long group = (long long)(blockIdx.x >> a.tiles_log);
  const int tile_id = blockIdx.x & ((1 << a.tiles_log) - 1);
  long long base = 0;
  for (int j = 0; j < a.tiles_log; ++j) base |= (long long)((tile_id >> j) & 1) << a.gbits[j];
  for (int h = tid; h < a.n_hi; h += nt) {
    int off = 0;
    for (int j = a.c; j < a.kq; ++j) off |= ((h >> (j - a.c)) & 1) << a.lbits[j];
    hi_off[h] = off;
  }
  __syncthreads();
  const int kqmask = (1 << a.kq) - 1;
  const int cmask = (1 << a.c) - 1;

  V v[E];
  PStage st = a.stages[0];
  int rbv[M];
  unsigned rmask = 0;
#pragma unroll
  for (int i = 0; i < M; ++i) rbv[i] = 1 << st.rb[i], rmask |= rbv[i];
  int tb = deposit(tid, full & ~rmask, K);
  const long long slot = (group << (K - a.kq)) | (tb >> a.kq);
  const bool active = slot < a.n_states;
  const int node_digit = (a.digit && active) ? a.digit[slot] : 0;

  // stage 0: HBM -> registers
  if (a.init_zero) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      int t = tb;
#pragma unroll
      for (int i = 0; i < M; ++i)
        if ((e >> i) & 1) t |= rbv[i];
      const int tl = t & kqmask;
      const long long off = base | (tl & cmask) | hi_off[tl >> a.c];
      v[e].x = (off == 0) ? R(1) : R(0);
      v[e].y = R(0);
    }
  } else if (active) {
    const long long ss = a.parent ? (long long)a.parent[slot] : slot;
    const V* s = reinterpret_cast<const V*>(a.src) + ss * a.state_elems + base;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      int t = tb;
#pragma unroll
      for (int i = 0; i < M; ++i)
        if ((e >> i) & 1) t |= rbv[i];
      const int tl = t & kqmask;
      v[e] = s[(tl & cmask) | hi_off[tl >> a.c]];
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e].x = v[e].y = R(0);
  }
  apply_ops<M>(v, a, st.op_begin, st.op_end, tb, base, node_digit);

  for (int s = 1; s < a.n_stages; ++s) {
    if (s > 1) __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      int t = tb;
#pragma unroll
      for (int i = 0; i < M; ++i)
        if ((e >> i) & 1) t |= rbv[i];
      tile[swz<V>(t)] = v[e];
    }
    __syncthreads();
    st = a.stages[s];
    rmask = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) rbv[i] = 1 << st.rb[i], rmask |= rbv[i];
    tb = deposit(tid, full & ~rmask, K);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      int t = tb;
#pragma unroll
      for (int i = 0; i < M; ++i)
        if ((e >> i) & 1) t |= rbv[i];
      v[e] = tile[swz<V>(t)];
    }
    apply_ops<M>(v, a, st.op_begin, st.op_end, tb, base, node_digit);
  }

  // last stage: registers -> HBM
  if (!active) return;
  V* d = reinterpret_cast<V*>(a.dst) + slot * a.state_elems + base;
  const R sc = (R)a.store_scale;
  const bool do_scale = a.store_scale != 1.0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int t = tb;
#pragma unroll
    for (int i = 0; i < M; ++i)
      if ((e >> i) & 1) t |= rbv[i];
    const int tl = t & kqmask;
    V x = v[e];
    if (do_scale) x.x *= sc, x.y *= sc;
    d[(tl & cmask) | hi_off[tl >> a.c]] = x;
  }
}

}  // namespace gs
