// Host/device shared encoding of the register-staged gate pass.
#pragma once

#include <cstdint>

namespace gs {

enum PassOpType : int8_t {
  P_W = 0,   // W-form on register bit idx0; w = 0 H, 1 X^1/2, 2 Y^1/2
  P_M1 = 1,  // dense 2x2 on register bit idx0
  P_D1 = 2,  // diag(d0, d1) on bit 0
  P_D2 = 3,  // diag(d00, d01, d10, d11) on bits (0, 1) = (qa, qb)
  P_M2 = 4,  // dense 4x4 on register bits (idx0 = qa, idx1 = qb)
};

// bit location of a diagonal op's qubit in the current stage
enum BitWhere : int8_t { B_REG = 0, B_THREAD = 1, B_TILE = 2 };

struct POp {
  int8_t type, w;
  int8_t where0, where1;
  int8_t idx0, idx1;  // register bit, tile bit (B_THREAD) or state bit (B_TILE)
  int16_t pad;
  int32_t coef;
  int32_t xtab;  // >= 0: cross op, coef = xtable[xtab + digit]
  int32_t xstride;
  int32_t xradix;
};

struct PStage {
  int8_t rb[8];  // register bit i -> tile bit
  int32_t op_begin, op_end;
};

struct Pass2Args {
  const void* src;
  void* dst;
  const int32_t* parent;
  const int32_t* digit;
  const POp* ops;
  const PStage* stages;
  const void* coefs;
  const int32_t* xtable;
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
  int lbits[16];
  int gbits[40];
};

}  // namespace gs
