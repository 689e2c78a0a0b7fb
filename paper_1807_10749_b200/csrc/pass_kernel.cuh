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

// Every common op below updates its registers strictly in place (no value
// outlives the op in a temporary).  With runtime dispatch over many inlined
// op bodies, any temporary left holding a result forces the register
// allocator to copy the whole 2^M-amplitude array at the op-loop header.

// x *= e^{i theta} as three in-place shears (Paeth): t = tan(theta/2),
// sn = sin(theta).  The host folds any angle beyond +-pi/2 into the sign of the
// real scale (add_param), so tan stays bounded.
template <typename V, typename T>
__device__ __forceinline__ void rot_inplace(V& x, T t, T sn) {
  x.x = fma(-t, x.y, x.x);
  x.y = fma(sn, x.x, x.y);
  x.x = fma(-t, x.y, x.x);
}

// W-forms, in place: H = [[1,1],[1,-1]], X = [[1,-i],[-i,1]], Y = [[1,-1],[1,1]].
// The second output is recovered from the first with one FMA
// (x0 - x1 = (x0 + x1) - 2 x1), so no temporary survives the op.
template <int M, int B, int W, typename V> __device__ __forceinline__ void w_reg(V (&v)[1 << M]) {
  using T = decltype(v[0].x);
#pragma unroll
  for (int e = 0; e < (1 << M); ++e) {
    if ((e >> B) & 1) continue;
    V& x0 = v[e];
    V& x1 = v[e | (1 << B)];
    if (W == 0) {         // y0 = x0 + x1, y1 = y0 - 2 x1
      x0.x = x0.x + x1.x; x0.y = x0.y + x1.y;
      x1.x = fma(T(-2), x1.x, x0.x); x1.y = fma(T(-2), x1.y, x0.y);
    } else if (W == 1) {  // y0 = x0 - i x1, y1 = x1 - i x0
      x0.x = x0.x + x1.y;                 // y0.re = x0.re + x1.im
      x0.y = x0.y - x1.x;                 // y0.im = x0.im - x1.re
      x1.x = fma(T(2), x1.x, x0.y);       // y1.re = x1.re + x0.im = 2 x1.re + y0.im
      x1.y = fma(T(2), x1.y, -x0.x);      // y1.im = x1.im - x0.re = 2 x1.im - y0.re
    } else {              // y0 = x0 - x1, y1 = y0 + 2 x1
      x0.x = x0.x - x1.x; x0.y = x0.y - x1.y;
      x1.x = fma(T(2), x1.x, x0.x); x1.y = fma(T(2), x1.y, x0.y);
    }
  }
}

// XOR swizzle of the low 4 (c64) / 3 (c128) address bits with the higher
// nibbles: linear over GF(2) and bijective on [0, 2^K).  The host picks each
// stage's lane bits so that their swizzled images are independent, which
// makes every shared-memory exchange conflict-free.
template <typename V> __device__ __forceinline__ int swz(int t) {
  constexpr int LB = sizeof(V) == 8 ? 4 : 3;
  constexpr int LM = (1 << LB) - 1;
  return t ^ (((t >> LB) ^ (t >> (2 * LB)) ^ (t >> (3 * LB)) ^ (t >> (4 * LB))) & LM);
}

// Gray-code walk over the 2^M register elements: element g(n) = n ^ (n >> 1)
// differs from g(n-1) in bit ctz(n), so a linear address map costs one XOR.
#define ctz_c(n) (((n) & 1) ? 0 : ((n) & 2) ? 1 : ((n) & 4) ? 2 : ((n) & 8) ? 3 : ((n) & 16) ? 4 : 5)


// Dense 2x2 / 4x4 ops (cross-gate Schmidt terms, intra-block iSWAP / fSim)
// cannot update registers in place.  The thread parks its 2^M amplitudes in
// its own slots of the shared tile (slots no other thread touches in this
// stage), applies the op there with runtime bit indices, and reloads: no
// call, no local memory, and the hot in-place paths keep their registers.
template <int M, typename V>
__device__ __forceinline__ void dense_op(V (&v)[1 << M], V* tile, const PStage* st, int tb, bool two,
                                         int r0, int r1, const V* u) {
  constexpr int E = 1 << M;
  int sstep[M];
#pragma unroll
  for (int i = 0; i < M; ++i) sstep[i] = swz<V>(1 << st->rb[i]);
  const int base = swz<V>(tb);
  {
    int addr = base;
#pragma unroll
    for (int n = 0; n < E; ++n) {
      if (n) addr ^= sstep[ctz_c(n)];
      tile[addr] = v[n ^ (n >> 1)];
    }
  }
  auto slot = [&](int e) {
    int a = base;
#pragma unroll
    for (int i = 0; i < M; ++i)
      if ((e >> i) & 1) a ^= sstep[i];
    return a;
  };
  if (!two) {
    const V u00 = u[0], u01 = u[1], u10 = u[2], u11 = u[3];
    for (int e = 0; e < E; ++e) {
      if ((e >> r0) & 1) continue;
      const int a0 = slot(e), a1 = slot(e | (1 << r0));
      const V x0 = tile[a0], x1 = tile[a1];
      tile[a0] = cmad2(u00, x0, u01, x1);
      tile[a1] = cmad2(u10, x0, u11, x1);
    }
  } else {
    for (int e = 0; e < E; ++e) {
      if (((e >> r0) & 1) || ((e >> r1) & 1)) continue;
      int ad[4];
      V x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) ad[q] = slot(e | ((q >> 1) << r0) | ((q & 1) << r1)), x[q] = tile[ad[q]];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        V y;
        y.x = 0;
        y.y = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const V c = u[4 * r + q];
          y.x += c.x * x[q].x - c.y * x[q].y;
          y.y += c.x * x[q].y + c.y * x[q].x;
        }
        tile[ad[r]] = y;
      }
    }
  }
  {
    int addr = base;
#pragma unroll
    for (int n = 0; n < E; ++n) {
      if (n) addr ^= sstep[ctz_c(n)];
      v[n ^ (n >> 1)] = tile[addr];
    }
  }
}

template <typename T> struct V4;
template <> struct V4<float> { using T = float4; };
template <> struct V4<double> { using T = double4; };

// factor p = {rs, t, sn, mode} on the elements e with (e & MASK) == WANT:
// mode bit 0 -> real scale by rs, bit 1 -> shear rotation (t, sn); in place
template <int M, int MASK, int WANT, typename V, typename P4>
__device__ __forceinline__ void dparam_sel(V (&v)[1 << M], const P4 p) {
  const int mode = (int)p.w;
  if (mode & 1) {
#pragma unroll
    for (int e = 0; e < (1 << M); ++e)
      if ((e & MASK) == WANT) v[e].x *= p.x, v[e].y *= p.x;
  }
  if (mode & 2) {
#pragma unroll
    for (int e = 0; e < (1 << M); ++e)
      if ((e & MASK) == WANT) rot_inplace(v[e], p.y, p.z);
  }
}

__device__ __forceinline__ int ubit(int where, int idx, int tb, long long base) {
  return where == B_THREAD ? ((tb >> idx) & 1) : (int)((base >> idx) & 1);
}

// one jump-table dispatch per primitive; every case updates v in place
template <int M, typename V>
__device__ __forceinline__ void apply_prims(V (&v)[1 << M], const Pass2Args& a, int ob, int oe,
                                            int tb, long long base, unsigned long long digits,
                                            V* tile, const PStage* st) {
  using T = decltype(v[0].x);
  using P4 = typename V4<T>::T;
  const P4* params = reinterpret_cast<const P4*>(a.params);
  const V* coefs = reinterpret_cast<const V*>(a.coefs);
  const uint4* prims = reinterpret_cast<const uint4*>(a.prims);
  for (int oi = ob; oi < oe; ++oi) {
    const uint4 raw = __ldg(prims + oi);  // PPrim, one 16-byte load
    struct {
      int code, ua_where, ua_idx, ub_where, ub_idx, r0, r1;
    } op;
    op.code = raw.x & 0xff;
    op.ua_where = (raw.x >> 8) & 0xff;
    op.ua_idx = (raw.x >> 16) & 0xff;
    op.ub_where = raw.x >> 24;
    op.ub_idx = raw.y & 0xff;
    op.r0 = (raw.y >> 8) & 0xff;
    op.r1 = (raw.y >> 16) & 0xff;
    const int xk = raw.y >> 24;
    int poff = (int)raw.z;
    if (raw.w & 0x10000u)  // cross op
      poff = __ldg(a.pxtable + poff + (int)((digits >> (4 * xk)) & 15)) + (int)(short)(raw.w & 0xffff);
    int uv = 0;
    if (op.code >= C_DHSEL && op.code <= C_DSEL) {
      uv = ubit(op.ua_where, op.ua_idx, tb, base);
      if (op.ub_where != 255) uv = 2 * uv + ubit(op.ub_where, op.ub_idx, tb, base);
    }
    switch (op.code) {
      case 0: if constexpr (0 < M) w_reg<M, 0, 0>(v); break;
      case 1: if constexpr (1 < M) w_reg<M, 1, 0>(v); break;
      case 2: if constexpr (2 < M) w_reg<M, 2, 0>(v); break;
      case 3: if constexpr (3 < M) w_reg<M, 3, 0>(v); break;
      case 4: if constexpr (4 < M) w_reg<M, 4, 0>(v); break;
      case 5: if constexpr (0 < M) w_reg<M, 0, 1>(v); break;
      case 6: if constexpr (1 < M) w_reg<M, 1, 1>(v); break;
      case 7: if constexpr (2 < M) w_reg<M, 2, 1>(v); break;
      case 8: if constexpr (3 < M) w_reg<M, 3, 1>(v); break;
      case 9: if constexpr (4 < M) w_reg<M, 4, 1>(v); break;
      case 10: if constexpr (0 < M) w_reg<M, 0, 2>(v); break;
      case 11: if constexpr (1 < M) w_reg<M, 1, 2>(v); break;
      case 12: if constexpr (2 < M) w_reg<M, 2, 2>(v); break;
      case 13: if constexpr (3 < M) w_reg<M, 3, 2>(v); break;
      case 14: if constexpr (4 < M) w_reg<M, 4, 2>(v); break;
      case 15: if constexpr (0 < M) dparam_sel<M, 1, 0>(v, params[poff]); break;
      case 16: if constexpr (1 < M) dparam_sel<M, 2, 0>(v, params[poff]); break;
      case 17: if constexpr (2 < M) dparam_sel<M, 4, 0>(v, params[poff]); break;
      case 18: if constexpr (3 < M) dparam_sel<M, 8, 0>(v, params[poff]); break;
      case 19: if constexpr (4 < M) dparam_sel<M, 16, 0>(v, params[poff]); break;
      case 20: if constexpr (0 < M) dparam_sel<M, 1, 1>(v, params[poff]); break;
      case 21: if constexpr (1 < M) dparam_sel<M, 2, 2>(v, params[poff]); break;
      case 22: if constexpr (2 < M) dparam_sel<M, 4, 4>(v, params[poff]); break;
      case 23: if constexpr (3 < M) dparam_sel<M, 8, 8>(v, params[poff]); break;
      case 24: if constexpr (4 < M) dparam_sel<M, 16, 16>(v, params[poff]); break;
      case 25: if constexpr (1 < M) dparam_sel<M, 3, 0>(v, params[poff]); break;
      case 26: if constexpr (1 < M) dparam_sel<M, 3, 2>(v, params[poff]); break;
      case 27: if constexpr (1 < M) dparam_sel<M, 3, 1>(v, params[poff]); break;
      case 28: if constexpr (1 < M) dparam_sel<M, 3, 3>(v, params[poff]); break;
      case 29: if constexpr (2 < M) dparam_sel<M, 5, 0>(v, params[poff]); break;
      case 30: if constexpr (2 < M) dparam_sel<M, 5, 4>(v, params[poff]); break;
      case 31: if constexpr (2 < M) dparam_sel<M, 5, 1>(v, params[poff]); break;
      case 32: if constexpr (2 < M) dparam_sel<M, 5, 5>(v, params[poff]); break;
      case 33: if constexpr (3 < M) dparam_sel<M, 9, 0>(v, params[poff]); break;
      case 34: if constexpr (3 < M) dparam_sel<M, 9, 8>(v, params[poff]); break;
      case 35: if constexpr (3 < M) dparam_sel<M, 9, 1>(v, params[poff]); break;
      case 36: if constexpr (3 < M) dparam_sel<M, 9, 9>(v, params[poff]); break;
      case 37: if constexpr (4 < M) dparam_sel<M, 17, 0>(v, params[poff]); break;
      case 38: if constexpr (4 < M) dparam_sel<M, 17, 16>(v, params[poff]); break;
      case 39: if constexpr (4 < M) dparam_sel<M, 17, 1>(v, params[poff]); break;
      case 40: if constexpr (4 < M) dparam_sel<M, 17, 17>(v, params[poff]); break;
      case 41: if constexpr (2 < M) dparam_sel<M, 6, 0>(v, params[poff]); break;
      case 42: if constexpr (2 < M) dparam_sel<M, 6, 4>(v, params[poff]); break;
      case 43: if constexpr (2 < M) dparam_sel<M, 6, 2>(v, params[poff]); break;
      case 44: if constexpr (2 < M) dparam_sel<M, 6, 6>(v, params[poff]); break;
      case 45: if constexpr (3 < M) dparam_sel<M, 10, 0>(v, params[poff]); break;
      case 46: if constexpr (3 < M) dparam_sel<M, 10, 8>(v, params[poff]); break;
      case 47: if constexpr (3 < M) dparam_sel<M, 10, 2>(v, params[poff]); break;
      case 48: if constexpr (3 < M) dparam_sel<M, 10, 10>(v, params[poff]); break;
      case 49: if constexpr (4 < M) dparam_sel<M, 18, 0>(v, params[poff]); break;
      case 50: if constexpr (4 < M) dparam_sel<M, 18, 16>(v, params[poff]); break;
      case 51: if constexpr (4 < M) dparam_sel<M, 18, 2>(v, params[poff]); break;
      case 52: if constexpr (4 < M) dparam_sel<M, 18, 18>(v, params[poff]); break;
      case 53: if constexpr (3 < M) dparam_sel<M, 12, 0>(v, params[poff]); break;
      case 54: if constexpr (3 < M) dparam_sel<M, 12, 8>(v, params[poff]); break;
      case 55: if constexpr (3 < M) dparam_sel<M, 12, 4>(v, params[poff]); break;
      case 56: if constexpr (3 < M) dparam_sel<M, 12, 12>(v, params[poff]); break;
      case 57: if constexpr (4 < M) dparam_sel<M, 20, 0>(v, params[poff]); break;
      case 58: if constexpr (4 < M) dparam_sel<M, 20, 16>(v, params[poff]); break;
      case 59: if constexpr (4 < M) dparam_sel<M, 20, 4>(v, params[poff]); break;
      case 60: if constexpr (4 < M) dparam_sel<M, 20, 20>(v, params[poff]); break;
      case 61: if constexpr (4 < M) dparam_sel<M, 24, 0>(v, params[poff]); break;
      case 62: if constexpr (4 < M) dparam_sel<M, 24, 16>(v, params[poff]); break;
      case 63: if constexpr (4 < M) dparam_sel<M, 24, 8>(v, params[poff]); break;
      case 64: if constexpr (4 < M) dparam_sel<M, 24, 24>(v, params[poff]); break;
      case 65: if constexpr (0 < M) dparam_sel<M, 1, 0>(v, params[poff + uv]); break;
      case 66: if constexpr (1 < M) dparam_sel<M, 2, 0>(v, params[poff + uv]); break;
      case 67: if constexpr (2 < M) dparam_sel<M, 4, 0>(v, params[poff + uv]); break;
      case 68: if constexpr (3 < M) dparam_sel<M, 8, 0>(v, params[poff + uv]); break;
      case 69: if constexpr (4 < M) dparam_sel<M, 16, 0>(v, params[poff + uv]); break;
      case 70: if constexpr (0 < M) dparam_sel<M, 1, 1>(v, params[poff + uv]); break;
      case 71: if constexpr (1 < M) dparam_sel<M, 2, 2>(v, params[poff + uv]); break;
      case 72: if constexpr (2 < M) dparam_sel<M, 4, 4>(v, params[poff + uv]); break;
      case 73: if constexpr (3 < M) dparam_sel<M, 8, 8>(v, params[poff + uv]); break;
      case 74: if constexpr (4 < M) dparam_sel<M, 16, 16>(v, params[poff + uv]); break;
      case 75: dparam_sel<M, 0, 0>(v, params[poff + uv]); break;
      case 76: dense_op<M>(v, tile, st, tb, false, op.r0, 0, coefs + poff); break;
      default: dense_op<M>(v, tile, st, tb, true, op.r0, op.r1, coefs + poff); break;
    }
  }
}

// shared-memory element store/load by 32-bit shared-window byte address
__device__ __forceinline__ void sts(uint32_t a, float2 x) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x.x), "f"(x.y) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, double2 x) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x.x), "d"(x.y) : "memory");
}
__device__ __forceinline__ void lds(uint32_t a, float2& x) {
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds(uint32_t a, double2& x) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x.x), "=d"(x.y) : "r"(a) : "memory");
}

template <typename R, int M>
__global__ void __launch_bounds__(256) pass2_kernel(const __grid_constant__ Pass2Args a) {
  using V = typename Cx<R>::T;
  constexpr int E = 1 << M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* tile = reinterpret_cast<V*>(smem_raw);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const int K = a.K;
  const int tid = threadIdx.x;

  const long long group = (long long)(blockIdx.x >> a.tiles_log);
  const int tile_id = blockIdx.x & ((1 << a.tiles_log) - 1);
  uint32_t base = 0;  // state bits fixed by the tile id (q <= 31)
  for (int j = 0; j < a.tiles_log; ++j) base |= (uint32_t)((tile_id >> j) & 1) << a.gbits[j];
  const int kq = a.kq;
  const int kqmask = (1 << kq) - 1;

  V v[E];
  const PStage* st = a.stages;
  // per-stage thread -> tile-index base, precomputed by the host
  int tb = a.tbtab[a.stage0 * 256 + tid];
  // slot (which state of the CTA) is a function of the stage's thread mapping:
  // recomputed after every exchange, with the digits that belong to it
  long long slot = (group << (K - kq)) | (tb >> kq);
  bool active = slot < a.n_states;
  unsigned long long node_digits = (a.digits && active) ? a.digits[slot] : 0ull;

  // stage 0: HBM -> registers (register bits are high tile bits: lanes contiguous)
  {
    uint32_t gstep[M];
#pragma unroll
    for (int i = 0; i < M; ++i) gstep[i] = 1u << a.lbits[st->rb[i]];
    uint32_t o = base | a.gofftab[tb & kqmask];
    if (a.init_zero) {
#pragma unroll
      for (int n = 0; n < E; ++n) {
        if (n) o ^= gstep[ctz_c(n)];
        const int e = n ^ (n >> 1);
        v[e].x = (o == 0) ? R(1) : R(0);
        v[e].y = R(0);
      }
    } else if (active) {
      const long long ss = a.parent ? (long long)a.parent[slot] : slot;
      const V* sp = reinterpret_cast<const V*>(a.src) + ss * a.state_elems;
#pragma unroll
      for (int n = 0; n < E; ++n) {
        if (n) o ^= gstep[ctz_c(n)];
        v[n ^ (n >> 1)] = sp[o];
      }
    }
    // inactive slots keep unspecified values: ops never mix slots and they are never stored
  }
  apply_prims<M>(v, a, st->op_begin, st->op_end, tb, base, node_digits, tile, st);

  for (int s = 1; s < a.n_stages; ++s) {
    if (s > 1) __syncthreads();
    {
      uint32_t sstep[M];
#pragma unroll
      for (int i = 0; i < M; ++i) sstep[i] = st->sstep[i];
      uint32_t off = (uint32_t)swz<V>(tb) * sizeof(V);
#pragma unroll
      for (int n = 0; n < E; ++n) {
        if (n) off ^= sstep[ctz_c(n)];
        sts(sbase + off, v[n ^ (n >> 1)]);
      }
    }
    __syncthreads();
    st = a.stages + s;
    tb = a.tbtab[(a.stage0 + s) * 256 + tid];
    if (K > kq) {
      slot = (group << (K - kq)) | (tb >> kq);
      active = slot < a.n_states;
      node_digits = (a.digits && active) ? a.digits[slot] : 0ull;
    }
    {
      uint32_t sstep[M];
#pragma unroll
      for (int i = 0; i < M; ++i) sstep[i] = st->sstep[i];
      uint32_t off = (uint32_t)swz<V>(tb) * sizeof(V);
#pragma unroll
      for (int n = 0; n < E; ++n) {
        if (n) off ^= sstep[ctz_c(n)];
        lds(sbase + off, v[n ^ (n >> 1)]);
      }
    }
    apply_prims<M>(v, a, st->op_begin, st->op_end, tb, base, node_digits, tile, st);
  }

  // last stage: registers -> HBM
  if (!active) return;
  const int G = a.out_group_log;  // grouped path-minor leaf layout for the gather
  V* d = reinterpret_cast<V*>(a.dst) +
         (G ? (((slot >> G) * a.state_elems) << G) + (slot & ((1 << G) - 1)) : slot * a.state_elems);
  const R sc = (R)a.store_scale;
  const bool do_scale = a.store_scale != 1.0;
  uint32_t gstep[M];
#pragma unroll
  for (int i = 0; i < M; ++i) gstep[i] = (1u << a.lbits[st->rb[i]]) << G;
  uint32_t o = (base | a.gofftab[tb & kqmask]) << G;
#pragma unroll
  for (int n = 0; n < E; ++n) {
    if (n) o ^= gstep[ctz_c(n)];
    V x = v[n ^ (n >> 1)];
    if (do_scale) x.x *= sc, x.y *= sc;
    d[o] = x;
  }
}

}  // namespace gs
