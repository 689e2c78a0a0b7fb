// Load-time specialisation of gate passes (NVRTC -> cubin -> driver launch).
//
// For every pass of a loaded program the engine emits one straight-line CUDA
// kernel from the hand-written template in jit.cu: the register stage
// layout, the shared-memory and HBM element offsets, and every gate
// coefficient become compile-time constants, so a pass costs its loads,
// stores and the arithmetic of its gates -- no op decoding, no runtime
// register-bit dispatch, no per-element address arithmetic.  Cross-gate
// terms (digit dependent) stay runtime table lookups.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace gs {

// argument block shared by every generated kernel (layout mirrored in the
// generated source's JArgs)
struct JArgs {
  const void* src;
  void* dst;
  const int32_t* parent;
  const unsigned long long* digits;
  const void* params;   // float4 {rs, t, sn, mode}
  const int32_t* pxtable;
  const void* coefs;    // complex coefficient pool (dense cross terms)
  long long state_elems;
  long long n_states;
  int init_zero;
  int pad;
  // fused leaf gather (last B-side leaf pass): requests bucketed by B tile
  const void* aleaf;          // grouped A leaf states [leaf/8][x][8]
  const int32_t* ia;          // A-local index per request
  const double* weights;      // leaf multiplicities
  const int32_t* bstart;      // bucket offsets per B tile (tiles + 1)
  const int32_t* breq;        // request index per bucket slot
  const int32_t* btl;         // tile-local B index per bucket slot
  void* partial;              // double2 [leaf group][n_req]
  long long n_req;
  long long a_elems;
  long long n_ctas;   // logical tiles of a persistent (pipelined) pass kernel
  long long uni_p0;   // >= 0: the chunk is full fan-out -- parent = uni_p0 + slot / F, digits from slot % F
  // projected-leaf fused pass (PassPlan::proj_fused): requests bucketed by this pass's tile
  const void* pf_parents;     // projected side's parent states (level D-1), complex64
  const void* pf_tab;         // float2 [group][8 << nk]: projected factor per sibling and request cross bits
  const long long* pf_aoff;   // [group][8]: parent amplitude offset per sibling
  const void* pf_meta;        // int2 per bucket slot: (tile-local index | cross bits << 16, parent base index)
  const unsigned* pf_bflip;   // Pauli-sibling pass: [group][8] park-address flip | sign-parity mask << 16 per sibling
};

struct JitModule;

// compile `source` (extern "C" kernels `names`, looked up in that order); nullptr with `err` set on failure
JitModule* jit_compile(const std::string& source, const std::vector<std::string>& names, const std::string& tag,
                       std::string& err);
void jit_release(JitModule* m);
// thread-local memory (register spills) of kernel `idx`, bytes; -1 if unknown
int jit_local_bytes(JitModule* m, int idx);
// registers per thread of kernel `idx`; -1 if unknown
int jit_num_regs(JitModule* m, int idx);
// launch kernel `idx` of the module
cudaError_t jit_launch(JitModule* m, int idx, unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       const JArgs& args, std::string& err);
bool jit_available(std::string& why);

}  // namespace gs
