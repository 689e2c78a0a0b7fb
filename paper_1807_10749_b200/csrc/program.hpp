// Host-side program analysis: path-tree levels, segment op lists and the
// shared-memory pass scheduler.  Pure C++ (no CUDA), so the planning logic is
// exercised by host-only contexts in the CPU test suite.
//
// Reference semantics mirrored here:
//  * op stream order and tags: `_lower_uncached` (pathsum.py:157-189);
//  * cross digit k selects term k of the cross gate's Schmidt decomposition,
//    big-endian mixed radix over gate order (pathsum.py:219-236);
//  * block-local qubit j lives at bit (q-1-j) of the block index
//    (`_b_view1`, pathsum.py:450-451).
// The reference walks the stream op by op, one numpy pass each; here the
// stream is cut at cross-gate cycles into path-tree levels, and each level's
// ops are packed into as few full-state passes as locality allows.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace gs {

struct GsError : std::runtime_error {
  int code;
  GsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum HostKind { K_DIAG1 = 0, K_MAT1 = 1, K_DIAG2 = 2, K_MAT2 = 3, K_CROSS = 4 };

// One block-local op on state bits (s0, s1); cross ops carry their gate index.
struct HostOp {
  int kind;       // K_DIAG1/K_MAT1/K_DIAG2/K_MAT2 (cross ops resolved per side)
  int s0 = -1, s1 = -1;
  int64_t coef = 0;  // coefficient pool offset (non-cross)
  int cross = -1;    // cross gate index (digit-dependent coefficients)
  int w = -1;        // W-form of a K_MAT1 (0 H, 1 X^1/2, 2 Y^1/2): u = s * W
  double s_re = 1, s_im = 0;
  bool diag() const { return kind == K_DIAG1 || kind == K_DIAG2; }
};

// A stage of a pass: M tile bits held in registers and the ops applied there.
struct StagePlan {
  std::vector<int> rb;  // register bit i -> tile bit
  std::vector<HostOp> ops;
};

struct PassPlan {
  int k = 0;                    // tile bits
  std::vector<int> lbits;       // tile bit -> state bit (ascending)
  std::vector<int> gbits;       // tile-id bit -> state bit (ascending)
  std::vector<HostOp> ops;      // ops applied in this pass, in order
  int64_t dev_op_offset = 0;    // into the device op array (v1 kernel)
  std::vector<StagePlan> stages;
  int M = 0;                    // register bits per stage
  int K = 0;                    // tile bits incl. slot bits (v2 kernel)
  int64_t dev_stage_offset = 0; // into the device stage array
  int64_t goff_offset = 0;      // into the tile-index -> state-offset table
  double store_scale = 1.0;     // power of two applied on store
  int jit_index = -1;           // kernel gsj_<index> of the program's JIT module
  bool grouped_store = false;   // leaf level, last pass: grouped path-minor store
  bool fused_gather = false;    // leaf level, last B pass: gather instead of a B store (JIT)
  bool proj_fused = false;      // leaf level, last pass of the grouped side: fused with the projected-side
                                // gather (JIT; no leaf state of either side reaches HBM)
  bool pf_pauli = false;        // proj_fused, Pauli-sibling form: the pass evolves ONE base state per leaf group
                                // (no cross terms, no slot bits); the siblings are Pauli images of it, read from
                                // the parked tile at flipped positions with signs
  bool pipelined = false;       // JIT: persistent kernel prefetching the next tile (option pipeline)
  int level = -1;               // path-tree level of the pass
  std::vector<int> store_perm;  // non-empty: state bit b is stored at address bit store_perm[b] (JIT only)
};

struct Level {
  int k_lo = 0, k_hi = 0;  // cross digits [k_lo, k_hi) introduced at this level
  std::vector<uint64_t> packed;  // mixed-radix level digit -> packed nibbles
  std::vector<HostOp> ops[2];
  std::vector<PassPlan> passes[2];
};

inline bool ops_conflict(const HostOp& a, const HostOp& b) {
  if (a.diag() && b.diag()) return false;
  const int sa[2] = {a.s0, a.s1}, sb[2] = {b.s0, b.s1};
  for (int x : sa)
    for (int y : sb)
      if (x >= 0 && x == y) return true;
  return false;
}

// Greedy pass scheduler.  Every pass keeps the low `c` state bits in the tile
// (coalesced runs of 2^c amplitudes) and fills the rest of the k-bit tile with
// the qubits of the earliest ready non-diagonal ops.  Diagonal ops need no
// locality: on a non-tile bit they are a per-tile constant.  An op is deferred
// when it would overflow the tile or when an earlier deferred op on one of its
// qubits does not commute with it.
inline std::vector<PassPlan> schedule_passes(const std::vector<HostOp>& ops, int q, int kmax,
                                             int cmin, bool force_one) {
  std::vector<PassPlan> out;
  const int k = std::min(q, kmax);
  const int c = std::min(cmin, std::max(0, k - 2));  // leave room for a 2-qubit op
  std::vector<HostOp> remaining = ops;
  if (remaining.empty() && force_one) {
    PassPlan p;
    p.k = k;
    for (int s = 0; s < k; ++s) p.lbits.push_back(s);
    for (int s = k; s < q; ++s) p.gbits.push_back(s);
    out.push_back(p);
    return out;
  }
  while (!remaining.empty()) {
    std::vector<char> in_tile(q, 0);
    int n_tile = 0;
    for (int s = 0; s < c; ++s) in_tile[s] = 1, ++n_tile;
    if (k == q) {
      for (int s = 0; s < q; ++s) in_tile[s] = 1;
      n_tile = q;
    }
    std::vector<char> blk_nd(q, 0), blk_d(q, 0);
    std::vector<HostOp> taken, deferred;
    for (const HostOp& op : remaining) {
      const int bits[2] = {op.s0, op.s1};
      bool nd_block = false, d_block = false;
      for (int b : bits)
        if (b >= 0) nd_block |= blk_nd[b], d_block |= blk_d[b];
      if (op.diag()) {
        if (nd_block) {
          deferred.push_back(op);
          for (int b : bits)
            if (b >= 0) blk_d[b] = 1;
        } else {
          taken.push_back(op);
        }
        continue;
      }
      bool ok = !(nd_block || d_block);
      if (ok) {
        int need = 0;
        for (int b : bits)
          if (b >= 0 && !in_tile[b]) ++need;
        if (op.s0 >= 0 && op.s1 >= 0 && op.s0 == op.s1) need = in_tile[op.s0] ? 0 : 1;
        ok = n_tile + need <= k;
      }
      if (ok) {
        for (int b : bits)
          if (b >= 0 && !in_tile[b]) in_tile[b] = 1, ++n_tile;
        taken.push_back(op);
      } else {
        deferred.push_back(op);
        for (int b : bits)
          if (b >= 0) blk_nd[b] = 1;
      }
    }
    if (taken.empty()) throw GsError(-1, "pass scheduler made no progress");
    // fill unused tile slots with the lowest remaining bits (wider contiguous runs)
    for (int s = 0; s < q && n_tile < k; ++s)
      if (!in_tile[s]) in_tile[s] = 1, ++n_tile;
    PassPlan p;
    p.k = k;
    for (int s = 0; s < q; ++s) (in_tile[s] ? p.lbits : p.gbits).push_back(s);
    p.ops = std::move(taken);
    out.push_back(std::move(p));
    remaining = std::move(deferred);
  }
  return out;
}

// Split one pass into register stages.  Each stage holds M tile bits in
// registers; a non-diagonal op needs all its qubits there, a diagonal op can
// run in any stage (its other bits are thread- or tile-uniform).  Stage 0
// and the last stage keep tile bits 0..4 on the lanes (when the tile has room)
// so the HBM load and store are warp-contiguous.
// HBM-facing stages (the first loads, the last stores) keep low tile bits on
// the lanes so every warp access is made of contiguous runs.  Classic layout
// (vec = false): tile bits 0..4 are lanes (>= 256-byte runs at 8 bytes per
// amplitude).  Vector layout (vec = true, complex64 specialised kernels): tile
// bits 1 and 2 must be lanes (>= 64-byte runs: one HBM burst), tile bit 0 is
// preferably a register bit so adjacent amplitudes move as one 16-byte access,
// and tile bits 3 and 4 may be register bits.  A grouped store (2^G leaves
// interleaved per amplitude, G >= 3) puts the slot bits on the lowest lanes,
// so any last stage already writes >= 64-byte runs.
inline std::vector<StagePlan> schedule_stages(const PassPlan& pp, int M, bool vec = false, int group_log = 0,
                                             bool slot_reg = false) {
  const int k = pp.k;
  std::vector<int> tile_of(64, -1);
  for (int j = 0; j < k; ++j) tile_of[pp.lbits[j]] = j;
  const int lane_low = (k - 5 >= M) ? 5 : 0;
  vec = vec && lane_low == 5;
  // may tile bit j be a register bit of an HBM-facing stage?
  auto hbm_ok = [&](int j) { return vec ? (j == 0 || j >= 3) : j >= lane_low; };
  std::vector<StagePlan> out;
  std::vector<HostOp> remaining = pp.ops;
  std::vector<int> last_fill;  // register bits of the latest stage no op needs
  bool first = true;
  while (!remaining.empty() || first) {
    auto allowed = [&](int j) { return !first || hbm_ok(j); };
    // ops a stage with register tile bits R can apply, in order: an op waits
    // if it touches a bit of an earlier waiting op (diagonal ops commute with
    // each other); a dense op also needs its bits in R
    auto simulate = [&](uint32_t R, std::vector<HostOp>* taken, std::vector<HostOp>* deferred) {
      uint32_t blk_nd = 0, blk_d = 0;
      int n = 0;
      for (const HostOp& op : remaining) {
        uint32_t m = 0;
        bool outside = false;
        for (int sb : {op.s0, op.s1}) {
          if (sb < 0) continue;
          if (tile_of[sb] < 0) outside = true;
          else m |= 1u << tile_of[sb];
        }
        const bool nd_block = (blk_nd & m) != 0, d_block = (blk_d & m) != 0;
        bool take;
        if (op.diag()) {
          take = !nd_block;
          if (!take) blk_d |= m;
        } else {
          if (outside) throw GsError(-1, "dense op outside the tile: scheduler bug");
          take = !nd_block && !d_block && (m & ~R) == 0;
          if (!take) blk_nd |= m;
        }
        if (take) {
          ++n;
          if (taken) taken->push_back(op);
        } else if (deferred) {
          deferred->push_back(op);
        }
      }
      return n;
    };
    // register set: the subset of the dense ops' (allowed) bits that lets this
    // stage apply the most ops; among equals prefer one that finishes the pass
    // with a store-compatible layout (no extra store stage)
    uint32_t cand = 0;
    for (const HostOp& op : remaining)
      if (!op.diag())
        for (int sb : {op.s0, op.s1})
          if (sb >= 0 && tile_of[sb] >= 0 && allowed(tile_of[sb])) cand |= 1u << tile_of[sb];
    std::vector<int> cbits;
    for (int j = 0; j < k; ++j)
      if ((cand >> j) & 1) cbits.push_back(j);
    auto store_ok = [&](uint32_t R) {
      if (group_log >= 3) return true;
      for (int j = 0; j < k; ++j)
        if (((R >> j) & 1) && !hbm_ok(j)) return false;
      return true;
    };
    uint32_t best_R = cand;
    if ((int)cbits.size() > M) {
      int best_n = -1;
      bool best_fin = false;
      const int nc = (int)cbits.size();
      for (uint32_t sel = (1u << M) - 1; sel < (1u << nc);) {
        uint32_t R = 0;
        for (int i = 0; i < nc; ++i)
          if ((sel >> i) & 1) R |= 1u << cbits[i];
        const int n = simulate(R, nullptr, nullptr);
        const bool fin = n == (int)remaining.size() && store_ok(R);
        if (n > best_n || (n == best_n && fin && !best_fin)) best_n = n, best_fin = fin, best_R = R;
        const uint32_t lo = sel & -sel, r = sel + lo;  // next subset of the same size
        sel = (((r ^ sel) >> 2) / lo) | r;
      }
    }
    std::vector<HostOp> taken, deferred;
    simulate(best_R, &taken, &deferred);
    if (taken.empty() && !first) throw GsError(-1, "stage scheduler made no progress");
    // keep only the bits the taken dense ops use
    uint32_t used = 0;
    for (const HostOp& op : taken)
      if (!op.diag())
        for (int sb : {op.s0, op.s1})
          if (sb >= 0) used |= 1u << tile_of[sb];
    std::vector<char> in_r(k, 0);
    int n_r = 0;
    for (int j = 0; j < k; ++j)
      if ((used >> j) & 1) in_r[j] = 1, ++n_r;
    if (vec && first && n_r < M && !in_r[0]) in_r[0] = 1, ++n_r;  // 16-byte loads
    std::vector<int> fill;
    for (int j = k - 1; j >= 0 && n_r < M; --j)
      if (!in_r[j] && allowed(j)) in_r[j] = 1, ++n_r, fill.push_back(j);
    for (int j = k - 1; j >= 0 && n_r < M; --j)
      if (!in_r[j]) in_r[j] = 1, ++n_r, fill.push_back(j);
    last_fill = fill;
    StagePlan sp;
    for (int j = 0; j < k; ++j)
      if (in_r[j]) sp.rb.push_back(j);
    sp.ops = std::move(taken);
    out.push_back(std::move(sp));
    remaining = std::move(deferred);
    first = false;
  }
  // grouped store: trade a filler register bit of the last stage for slot bit 0
  // (tile bit k): sibling leaves s, s + 1 of one amplitude are adjacent in the
  // grouped layout, so each thread then stores them as one 16-byte float4.
  // Not when the last stage holds cross ops (their digits are per slot).
  if (vec && group_log >= 3 && slot_reg && !last_fill.empty()) {
    bool cross = false;
    for (const HostOp& op : out.back().ops) cross |= op.cross >= 0;
    std::vector<int>& rb = out.back().rb;
    if (!cross && std::find(rb.begin(), rb.end(), k) == rb.end()) {
      *std::find(rb.begin(), rb.end(), last_fill.back()) = k;
      std::sort(rb.begin(), rb.end());
    }
  }
  // 16-byte stores: trade a filler register bit of the last stage for tile bit 0
  if (vec && group_log < 3 && !last_fill.empty()) {
    std::vector<int>& rb = out.back().rb;
    if (std::find(rb.begin(), rb.end(), 0) == rb.end()) {
      *std::find(rb.begin(), rb.end(), last_fill.back()) = 0;
      std::sort(rb.begin(), rb.end());
    }
  }
  // the store stage must leave the run-forming tile bits on the lanes
  bool bad = false;
  if (group_log < 3)
    for (int j : out.back().rb) bad |= !hbm_ok(j);
  if (bad) {
    StagePlan sp;
    if (vec) sp.rb.push_back(0);
    for (int j = k - M + (vec ? 1 : 0); j < k; ++j) sp.rb.push_back(j);
    out.push_back(std::move(sp));
  }
  return out;
}

}  // namespace gs
