// Host/device shared encoding of the register-staged gate pass.
#pragma once

#include <cstdint>

namespace gs {

// bit location of a diagonal op's qubit in the current stage
enum BitWhere : int8_t { B_REG = 0, B_THREAD = 1, B_TILE = 2 };


struct PStage {
  int8_t rb[8];   // register bit i -> tile bit
  int8_t tb[16];  // thread-index bit j -> tile bit (lanes = j < 5)
  int32_t op_begin, op_end;
  uint32_t sstep[8];  // byte step in the swizzled shared tile per register bit
};

// Flattened primitive of the v2 pass: one jump-table case per (kind, register
// bit(s)); diagonal factors are pre-split by the host into real scale `rs` and
// shear-rotation parameters (t = tan(theta/2), sn = sin(theta)).
enum PrimCode : uint8_t {
  C_W = 0,        // + w*5 + b      W-form (H, X^1/2, Y^1/2) on register bit b
  C_DH = 15,      // + h*5 + b      diag factor on the half where bit b == h
  C_DQ = 25,      // + pair*4 + q   diag factor on quadrant q of register pair
  C_DHSEL = 65,   // + h*5 + b      like C_DH, factor selected by uniform bit ua
  C_DSEL = 75,    //                factor on every element, selected by ua (, ub)
  C_M1 = 76,      //                dense 2x2 on register bit r0 (out of line)
  C_M2 = 77,      //                dense 4x4 on register bits (r0 = qa, r1 = qb)
  C_NCODES = 78,
};

struct PPrim {
  uint8_t code;
  uint8_t ua_where, ua_idx;  // uniform bit A: where (B_THREAD / B_TILE), index
  uint8_t ub_where, ub_idx;  // uniform bit B (C_DSEL on two bits), where = 255: none
  uint8_t r0, r1;            // register bits for C_M1 / C_M2
  uint8_t xk;                // cross op: nibble of the node's packed digits
  int32_t param;             // param offset, or xtable base for cross ops
  int16_t xsub;              // cross op: added to the xtable entry
  int16_t flags;             // bit 0: cross op
};
static_assert(sizeof(PPrim) == 16, "PPrim is loaded as one uint4");

struct Pass2Args {
  const void* src;
  void* dst;
  const int32_t* parent;
  const PStage* stages;
  const void* coefs;
  const int32_t* xtable;
  const PPrim* prims;
  const void* params;        // float4 / double4 {rs, t, sn, mode}
  const int32_t* pxtable;    // cross op: digit -> param offset
  const unsigned long long* digits;  // packed 4-bit digits per child state
  long long state_elems;
  long long n_states;
  double store_scale;  // power of two, applied on store
  int n_stages;
  int kq;    // state bits in the tile
  int K;     // tile bits (kq + slot bits)
  int c;     // low state bits in the tile that are contiguous (<= kq)
  int tiles_log;
  int init_zero;
  int n_hi;
  int out_group_log;  // > 0: store leaf states grouped path-minor, [slot >> G][x][slot & (2^G-1)]
  int stage0;                 // global index of the pass's first stage (tbtab rows)
  const uint16_t* tbtab;      // [stage][256] thread -> tile-index base
  const uint32_t* gofftab;    // [2^kq] tile index -> state offset of the pass
  int lbits[16];
  int gbits[40];
};

}  // namespace gs
