// B200 path-sum engine: program loading, path-tree DFS, launches, C ABI.
//
// The reference executes the lowered op stream one numpy sweep per op over
// (prefix rows x 2^q) arrays, snapshots once at the prefix/branch split and
// replays the branch ops per branch (run_batched, pathsum.py:574-640).  Here
// the stream is cut at every cross-gate cycle into path-tree levels; a
// depth-first walk evolves each distinct digit prefix once, in batches of
// sibling nodes resident in HBM, and the leaves are gathered into an fp64
// accumulator on the device.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <deque>
#include <vector>

#include "../../include/gridsim_b200.h"
#include "kernels.cuh"
#include "jit.hpp"
#include "pass_kernel.h"
#include "program.hpp"

namespace gs {

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw GsError(GS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t n) {
    if (n <= bytes) return;
    release();
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw GsError(GS_ERR_NOMEM, "cudaMalloc(" + std::to_string(n) + ") failed: " +
                                      cudaGetErrorString(e));
    }
    bytes = n;
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  PinnedBuf(PinnedBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    CK(cudaMallocHost(&p, n));
    bytes = n;
  }
};

// Host->device staging ring for per-chunk node tables (digits, parents, leaf
// weights).  Every region gets an event after its copy; the host waits only
// when it is about to overwrite a region whose copy may still be pending, so
// the launch queue of a step is never drained by staging.  All copies and
// kernels run on one stream, so the device-side region is free for reuse by
// stream order.
struct Ring {
  PinnedBuf host;
  DevBuf dev;
  size_t size = 0, head = 0;
  struct Region {
    size_t beg, end;
    cudaEvent_t ev;
  };
  std::deque<Region> inflight;
  std::vector<cudaEvent_t> pool;
  ~Ring() {
    for (auto& r : inflight) cudaEventDestroy(r.ev);
    for (auto e : pool) cudaEventDestroy(e);
  }
  void drain() {
    for (auto& r : inflight) {
      cudaEventSynchronize(r.ev);
      pool.push_back(r.ev);
    }
    inflight.clear();
  }
  // grow to at least n bytes (waits for pending copies before reallocating)
  void reserve(size_t n, cudaStream_t s) {
    if (n <= size) return;
    drain();
    CK(cudaStreamSynchronize(s));
    host.ensure(n);
    dev.ensure(n);
    size = n;
    head = 0;
  }
  // region of `bytes` (256-aligned) whose host side is free to write
  size_t alloc(size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    if (bytes > size) throw GsError(GS_ERR_STATE, "staging ring too small");
    if (head + bytes > size) head = 0;
    const size_t beg = head, end = head + bytes;
    int last = -1;
    for (int i = 0; i < (int)inflight.size(); ++i)
      if (inflight[i].beg < end && beg < inflight[i].end) last = i;
    if (last >= 0) {
      cudaEventSynchronize(inflight[last].ev);
      for (int i = 0; i <= last; ++i) {
        pool.push_back(inflight.front().ev);
        inflight.pop_front();
      }
    }
    head = end;
    return beg;
  }
  // copy [off, off + bytes) to the device and mark it in flight
  void commit(size_t off, size_t bytes, cudaStream_t s) {
    CK(cudaMemcpyAsync(static_cast<char*>(dev.p) + off, static_cast<char*>(host.p) + off, bytes,
                       cudaMemcpyHostToDevice, s));
    cudaEvent_t e;
    if (pool.empty()) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    else e = pool.back(), pool.pop_back();
    CK(cudaEventRecord(e, s));
    inflight.push_back({off, off + ((bytes + 255) & ~(size_t)255), e});
  }
  char* h(size_t off) { return static_cast<char*>(host.p) + off; }
  char* d(size_t off) { return static_cast<char*>(dev.p) + off; }
};

// Node of the path tree.  Leaves are (prefix index i, branch b); a node at
// level l with digit end e covers the prefixes i0..i1-1 (all sharing digits
// [0, min(e, x_p))) and the branch ids b0..b1-1 (all sharing digits
// [x_p, e) when e > x_p).
struct Node {
  int64_t i0, i1;   // prefix index range
  int64_t key;      // prefix digits [0, min(e, x_p)) as a number
  int64_t bkey;     // branch digits [x_p, max(e, x_p)) as a number
  int64_t b0, b1;   // branch id range
  uint64_t digit;   // this level's cross digits, 4 bits each (gate k_lo + j at bits 4j)
  int32_t parent;   // slot of the parent in the previous level's buffer
};

struct Program {
  int q[2] = {0, 0};
  int n_cross = 0;
  std::vector<int> radix;   // per cross gate
  std::vector<int> cross_cycle;
  std::vector<Level> levels;  // levels[0] = root segment (no cross digits)
  std::vector<double> coef;   // complex pool, (re, im) pairs; cross matrices appended
  std::vector<int32_t> xtable;
  // per cross gate and side: xtable offset, and whether that side is diagonal
  std::vector<int> xtab[2];
  std::vector<int> xdiag[2];
  std::vector<int> xq[2];
};

// Pauli frame of a leaf level (pauli_frame below)
struct PauliFrame {
  bool ok = false;
  int nk = 0;
  int zsel[8][16] = {};           // cross term d of gate j = x0[j][d] * Z^zsel[j][d]
  double x0[8][16][2] = {};
  int a[8] = {};                  // behind the level's ops that Z is i^a X^f Z^z
  uint32_t f[8] = {}, z[8] = {};  // state-bit masks (X part, Z part)
  int order[8] = {};              // product order, leftmost factor first
  bool projector = false;         // some term is a projector a (I + (-1)^v Z) / 2 (zsel = 2 + v)
};

struct Ctx {
  int device = -1;
  int precision = GS_C64;
  bool host_only = false;
  std::string err;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // options
  int64_t mem_budget_mb = 0;  // 0 = auto
  int profile = 0;
  int tile_bits = 0;  // 0 = auto
  int low_bits = 4;
  int64_t max_chunk = 1 << 20;
  // program
  bool have_prog = false;
  Program prog;
  DevBuf d_ops, d_coef, d_xtable, d_prims, d_pstages, d_params, d_pxtable;
  std::vector<DevOp> host_devops;
  std::vector<PPrim> host_prims;
  std::vector<double> host_params;   // 4 per param: rs, t, sn, mode
  std::vector<int32_t> host_pxtable;
  std::vector<int> pxbase[2];        // per cross gate and side: pxtable base
  std::vector<uint16_t> host_tbtab;  // [stage][256] thread -> tile-index base
  std::vector<uint32_t> host_gofftab;  // per pass [2^k] tile index -> state offset
  DevBuf d_tbtab, d_gofftab;
  std::vector<PStage> host_pstages;
  double kfinal[2][2] = {{1, 0}, {1, 0}};  // per block: true = stored * K
  int kernel_version = 2;
  int hoist = 1;  // move digit-independent ops above branch points
  int smem_gather = 1;
  int grouped_enabled = 1;
  bool grouped_leaf = false;
  int fuse_gather = 0;        // option: gather inside the last B-side leaf pass (JIT only; slower: the
                              // epilogue is latency-bound and stalls the pass, profiles/r01_notes.md)
  bool fused_active = false;  // the fused leaf pass is compiled for the loaded program
  bool bucket_valid = false;  // request buckets match the loaded requests
  DevBuf d_bcount, d_bstart, d_breq, d_btl, d_bia, d_cubtmp;
  // requests sorted by A index for the HBM gathers (perm = original slot of sorted slot i)
  int sort_requests = 1;   // option
  int quad_gather = 1;     // option: 4 lanes per request in the grouped gather
  bool req_sorted = false;
  DevBuf d_ia_s, d_ib_s, d_perm, d_iota, d_sorttmp;
  DevBuf full_state;  // gs_run_full
  int group_log = 3;  // leaves per group = 2^group_log (64-byte request reads in c64)
  DevBuf leaf_out[2];  // grouped path-minor leaf states (see gather_grouped_kernel)
  // overlap_gather: leaf chunk i's gather runs on gstream while chunk i+1's leaf
  // passes run on the main stream (double-buffered leaf states, partials, tables)
  int overlap_gather = 0;     // option
  bool ovl = false;           // active for the current run
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_leaf = nullptr, ev_g[2] = {nullptr, nullptr};
  int flip = 0;
  DevBuf leaf_out2[2], d_partial2, d_tab[2];
  cudaStream_t gs = nullptr;        // stream of the current gather (null: main stream)
  DevBuf* part_sel = nullptr;       // partials buffer of the current gather
  void* leaf_sel[2] = {nullptr, nullptr};
  DevBuf d_packed;  // requests packed as ia | ib << qa (shared-memory gather)
  int reg_bits = 6;  // register bits per stage for c64: 4, 5, 0 = per pass by op count, 6 = 4 for halves >= 2^26 amplitudes
  int m4_ops = 30;   // reg_bits = 0: passes with at least this many ops use 4 register bits
  int use_jit = 1;   // specialise passes at load time (NVRTC); interpreter otherwise
  int vec_hbm = 1;   // option: vector (16-byte) HBM stage layouts for specialised passes
  int jit_min_blocks = 3;  // option: __launch_bounds__ min CTAs/SM of specialised passes (0 = none)
  std::vector<JitModule*> jit_mods;   // one per compile chunk
  std::vector<std::pair<int, int>> jit_loc;  // pass jit_index -> (module, kernel)
  JitModule* jit = nullptr;           // non-null when any module is loaded
  std::string jit_status = "off";
  double jit_seconds = 0;
  std::vector<size_t> jit_smem;
  std::vector<int> jit_occ;   // resident CTAs per SM of a pipelined (persistent) pass kernel
  int pipeline = 0;           // option: persistent cp.async-prefetching pass kernels (JIT)
  int dedupe_parent = 0;      // option: sibling slots load a shared parent tile once (JIT; measured slower)
  int jit_cross_inline = 1;   // option: cross-term coefficients per digit as immediates (JIT)
  int jit_spill_ok = 32;      // option: local-memory bytes tolerated at the 3-CTA register bound
  int uniform_chunks = 0;     // option: full fan-out chunks derive parent/digits from the slot (JIT; no measured gain)
  int64_t uni_p0 = -1;        // current chunk: parent slot of its first node when full fan-out
  int tail_gather = 1;        // option: small last leaf pass evaluated inside the (path-major) gather
  int tail_max = 3;           // option: max tail qubits (2^tail_max reads per request and leaf)
  std::vector<HostOp> tail_ops[2];
  std::vector<int> tail_bits[2];
  int proj_leaf = 1;          // option: a projector-only leaf side is read from its parent in the gather
  int proj_perm = 0;          // option: store those parents with the sibling-run bits lowest (no measured gain)
  int proj_lanes = 4;         // option: lanes per request in the projected-leaf gather (4 or 8)
  int slot_store16 = 0;       // option: grouped leaf stores as 16-byte sibling pairs (JIT; measured 0-3% slower)
  int sink_ops = 12;          // option: move a level's trailing pass of <= sink_ops ops into the next level
  int gather_gpy = 0;         // option: leaf groups per gather y-block (0 = auto)
  int proj_side = -1;         // leaf side evaluated by projection (no leaf passes), -1 none
  int tile_major = 2;         // option: JIT passes of levels >= 1 launch their CTAs tile-major (siblings of one
                              // tile back to back: a parent tile is read from DRAM once); 2 = auto (>= 2^24
                              // amplitudes: cfg5 +1%, cfg4 -1% when forced on)
  int proj_fuse = 1;          // option: fuse the other side's last leaf pass with the projected gather (JIT)
  int pf_u = 2;               // option: requests in flight per lane quad in the fused pass epilogue
  int pf_min_blocks = 3;      // option: __launch_bounds__ min CTAs/SM of the fused pass
  int pf_pauli = 1;           // option: Pauli-sibling form of the fused pass where the leaf level allows it
  int jit_rsign = 0;          // option: +-1 factors selected at run time carried as sign variables (jitgen.inc Gen::rv);
                              // bitwise the same results, 15% fewer FP instructions in the op-heavy passes, but
                              // cfg4 only +0.5% and cfg5 -4% at the default cap (same-box A/B): off
  int jit_rsign_max = 8;      // option: live sign variables per thread before the oldest is folded in (registers;
                              // cfg4: 1..3: 179.0-179.9k, 8: 181.0k, uncapped: one pass spills at the 3-CTA bound)
  int jit_c128 = 1;           // option: specialised (NVRTC) gate passes for complex128 programs too
  int xchg16 = 0;             // option: 16-byte shared-memory exchanges over a register bit common to both stages (JIT;
                              // measured: -10% on a level-7 pass alone under ncu, but 163.8k vs 167.7k paths/s in the step: off)
  int sink_balance = 0;       // option: move a suffix of level D-2's ops to the front of level D-1 (FP balance)
  int pf_m4 = 0;              // option: 4 register bits (512 threads) for the Pauli-sibling pass
  int pf_unroll = 1;          // option: unroll factor of the pipelined epilogue loop (register-rotation moves)
  int pf_streams = 1;         // option: Pauli-sibling pass requests in two bank-half streams per tile, sorted by
                              // factor-table row (conflict-free park reads, broadcast factor reads)
  int l2_ahead = 148;         // option: pass CTAs prefetch into L2 the stage-0 tile of the CTA this many launches later
                              // (0 off; cfg4: 0: 171.2k, 74: 178.5k, 148: 177.9k, 222: 178.3k, 296: 175.2k, 444: 169.0k)
  int pf_groups = 2;          // option: leaf groups a Pauli-sibling CTA serves back to back into one partial row
                              // (cfg4: 1: 168.1k, 2: 171.9k, 4: 171.1k, 8: 169.9k paths/s)
  int pf_pipe = 1;            // option: software-pipelined epilogue of the Pauli-sibling pass
  int pf_tail = 0;            // option: the fused pass's last one-qubit-op stage runs per request in its epilogue
                              // (measured: cfg4 -1.3%, cfg4v2 +2%, cfg3v2 equal; off)
  bool proj_fused_active = false;  // the fused projected-leaf pass is compiled for the loaded program
  int64_t pf_rows = 0;        // partial rows written by the current leaf chunk's fused pass
  DevBuf d_proj;              // device copy of ProjProgD for the fused pass
  DevBuf d_pftab, d_pfaoff, d_bmeta;  // fused pass: per-group factor tables, per-bucket-slot request data
  DevBuf d_pfbflip;                   // Pauli-sibling pass: per-slot park flip | sign mask
  PauliFrame pauli;                   // Pauli frame of the grouped side's leaf level (ok = the pass is planned)
  // Pauli-sibling leaves of the path-major gathers (half-states too large for the grouped layout):
  // side psib_side's leaf passes evolve one base state per parent, without cross terms; the
  // gather reads every leaf of that side as a Pauli image of its parent's base state
  PauliFrame psib;
  int psib_side = -1;
  const void* cur_sib = nullptr;        // device SibD per leaf of the current leaf chunk
  const int32_t* cur_upar = nullptr;    // device: distinct parents of the current leaf chunk
  int64_t cur_npar = 0;
  uint32_t pauli_lcol[16] = {};       // park address map L of the Pauli-sibling pass: lcol[j] = L e_j (tile bit j)
  uint32_t pauli_lit[16] = {};        // L^-T e_j
  int pauli_conflicts = 0;            // worst bank multiplicity of a warp's park store under L
  bool pauli_blocked = false;         // the Pauli-sibling kernel did not compile for this program: planned without it
  const int32_t* cur_parent = nullptr;             // device node tables of the current leaf chunk
  const int32_t* cur_gpar = nullptr;               // per leaf group: shared parent of a sibling block, or -1
  bool proj_fast = false;                          // run gates radix 2 with v(d) = d
  std::vector<std::pair<int, int>> proj_swaps;     // parent states stored with these address-bit swaps
  PassPlan* proj_perm_pass = nullptr;              // the pass that stores them permuted
  const unsigned long long* cur_digit = nullptr;
  int n_sm = 148;
  // requests
  int64_t n_req = -1;
  DevBuf d_ia, d_ib, d_acc, d_partial, d_gidx;
  // tree buffers
  std::vector<DevBuf> lvl_a, lvl_b;
  Ring ring;                          // node tables + leaf weights staging
  const double* cur_weights = nullptr;  // device leaf weights of the current leaf chunk
  int async_run = 0;  // option: gs_run with a device output returns without a stream sync
  // run state
  gs_stats st{};
  int32_t x_p = 0;
  std::vector<int64_t> prefixes;
  int64_t branch_lo = 0, branch_hi = 1;
  std::vector<int64_t> S_p, S_b;  // digit suffix products
  std::vector<int64_t> cap;        // nodes per level buffer
  std::vector<int> lvl_end;        // digit end e_l per level
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<std::vector<Node>> kids;  // per-level child scratch for the DFS
  std::chrono::steady_clock::time_point last_tick;
  // requests staged by gs_run_batched: host copy on worker threads while the
  // tree is enqueued; the split runs on a side stream the first gather waits for
  struct PendingRequests {
    bool active = false;
    std::vector<std::thread> workers;
    std::vector<char> bad;  // per worker: an index outside the state space
    int64_t n = 0;
    SplitRuns runs{};
    bool packed = false;
    ~PendingRequests() { join(); }
    void join() {
      for (auto& t : workers)
        if (t.joinable()) t.join();
      workers.clear();
    }
  } pend;
  PinnedBuf req_stage;
  PinnedBuf out_stage;                 // pinned bounce buffer of the host result
  int64_t d2h_chunk_mb = 0;            // option: pipelined result download chunk (0 = one direct copy;
                                       // measured no faster than the driver's own staging for 16 MB)
  std::vector<cudaEvent_t> out_events;  // one per result chunk
  cudaStream_t side_stream = nullptr;
  cudaEvent_t req_done = nullptr;
  uint64_t sched_serial = 0;       // bumped by every (re)schedule of the program
  std::vector<int64_t> plan_key;   // inputs of the current buffer plan
  // host-side pacing: longest interval between consecutive kernel launches
  const char* gap_label = "";
  void tick(const char* label = "launch") {
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - last_tick).count();
    if (ms > st.host_ms_max_gap) st.host_ms_max_gap = ms, gap_label = label;
    last_tick = now;
  }

  size_t esize() const { return precision == GS_C64 ? 8 : 16; }
  int kmax() const {
    int k = tile_bits ? tile_bits : (precision == GS_C64 ? 13 : 12);
    return k;
  }
};

#include "jitgen.inc"

// ---------------------------------------------------------------------------
// program loading

static int64_t coef_entries(int kind) {
  switch (kind) {
    case K_DIAG1: return 2;
    case K_MAT1: return 4;
    case K_DIAG2: return 4;
    case K_MAT2: return 16;
  }
  return 0;
}

// u = s * W with W one of H=[[1,1],[1,-1]], X=[[1,-i],[-i,1]], Y=[[1,-1],[1,1]]
// (the reference's H, X^1/2, Y^1/2, circuit.py:46-50); s = u00 is deferred.
static void classify_w(HostOp& op, const double* u) {
  const double sr = u[0], si = u[1];
  const double mag = std::sqrt(sr * sr + si * si);
  if (mag == 0) return;
  const double tol = 1e-12 * mag;
  auto eq = [&](int e, double re, double im) {
    return std::fabs(u[2 * e] - re) <= tol && std::fabs(u[2 * e + 1] - im) <= tol;
  };
  // candidates: (u01, u10, u11) as multiples of s
  if (eq(1, sr, si) && eq(2, sr, si) && eq(3, -sr, -si)) op.w = 0;                 // H
  else if (eq(1, si, -sr) && eq(2, si, -sr) && eq(3, sr, si)) op.w = 1;           // X: -i*s
  else if (eq(1, -sr, -si) && eq(2, sr, si) && eq(3, sr, si)) op.w = 2;           // Y
  if (op.w >= 0) op.s_re = sr, op.s_im = si;
}

// Move every segment op that commutes with its level's cross terms (and with
// the ops it would pass) above the branch point: it is then applied once per
// parent node instead of once per child.  Processed from the deepest level up,
// so an op keeps rising while it commutes.  Exact (commutation), so results
// match the reference op order up to rounding.
static void hoist_ops(Program& p) {
  for (int l = (int)p.levels.size() - 1; l >= 1; --l) {
    Level& L = p.levels[l];
    Level& P = p.levels[l - 1];
    for (int side = 0; side < 2; ++side) {
      std::vector<HostOp> stay, up;
      for (const HostOp& op : L.ops[side]) {
        bool ok = op.cross < 0;
        if (ok)
          for (const HostOp& b : stay)
            if (ops_conflict(op, b)) { ok = false; break; }
        (ok ? up : stay).push_back(op);
      }
      if (up.empty()) continue;
      P.ops[side].insert(P.ops[side].end(), up.begin(), up.end());
      L.ops[side] = std::move(stay);
    }
  }
}

static void build_program(Ctx& c, int qa, int qb, int n_ops, const int32_t* kind,
                          const int32_t* blk, const int32_t* q0, const int32_t* q1,
                          const int32_t* cycle, const int64_t* coef_off, int n_cross,
                          const int32_t* rank, const int32_t* xcycle, const int32_t* xqa,
                          const int32_t* xqb, const int32_t* tka, const int64_t* tca,
                          const int32_t* tkb, const int64_t* tcb, int64_t n_coef,
                          const double* coef) {
  Program p;
  // qb = 0: an uncut full-state program (gs_run_full)
  if (qa < 1 || qb < 0 || qa > 34 || qb > 34 || (qb == 0 && n_cross > 0))
    throw GsError(GS_ERR_ARG, "block sizes out of range");
  p.q[0] = qa;
  p.q[1] = qb;
  p.coef.assign(coef, coef + 2 * n_coef);
  p.n_cross = n_cross;
  int64_t n_terms = 0;
  for (int k = 0; k < n_cross; ++k) {
    if (rank[k] < 1) throw GsError(GS_ERR_ARG, "cross rank < 1");
    if (k > 0 && xcycle[k] < xcycle[k - 1]) throw GsError(GS_ERR_ARG, "cross gates not in cycle order");
    p.radix.push_back(rank[k]);
    p.cross_cycle.push_back(xcycle[k]);
    n_terms += rank[k];
  }
  auto check_coef = [&](int64_t off, int64_t n) {
    if (off < 0 || off + n > n_coef) throw GsError(GS_ERR_ARG, "coefficient offset out of range");
  };
  // cross tables: per side, all-diagonal terms stay diag(d0,d1); otherwise
  // every term becomes a 2x2 (diag terms expanded), as _term_table does
  // (pathsum.py:516-523).
  for (int side = 0; side < 2; ++side) {
    const int32_t* tk = side ? tkb : tka;
    const int64_t* tc = side ? tcb : tca;
    const int32_t* xq = side ? xqb : xqa;
    int64_t t = 0;
    for (int k = 0; k < n_cross; ++k) {
      if (xq[k] < 0 || xq[k] >= p.q[side]) throw GsError(GS_ERR_ARG, "cross qubit out of block");
      bool all_diag = true;
      for (int d = 0; d < rank[k]; ++d) {
        const int kk = tk[t + d];
        if (kk != K_DIAG1 && kk != K_MAT1) throw GsError(GS_ERR_ARG, "cross term kind must be diag1/mat1");
        all_diag &= (kk == K_DIAG1);
      }
      p.xtab[side].push_back((int)p.xtable.size());
      p.xdiag[side].push_back(all_diag);
      p.xq[side].push_back(xq[k]);
      for (int d = 0; d < rank[k]; ++d) {
        const int kk = tk[t + d];
        const int64_t off = tc[t + d];
        check_coef(off, coef_entries(kk));
        if (all_diag || kk == K_MAT1) {
          p.xtable.push_back((int32_t)off);
        } else {  // expand diag(d0, d1) to a 2x2 in the pool
          const int64_t at = (int64_t)p.coef.size() / 2;
          const double m[8] = {coef[2 * off], coef[2 * off + 1], 0, 0, 0, 0,
                               coef[2 * off + 2], coef[2 * off + 3]};
          p.coef.insert(p.coef.end(), m, m + 8);
          p.xtable.push_back((int32_t)at);
        }
      }
      t += rank[k];
    }
  }
  if ((int64_t)p.coef.size() / 2 > INT32_MAX) throw GsError(GS_ERR_ARG, "coefficient pool too large");

  // levels: distinct cross cycles; level l (>= 1) starts at cross cycle c_l
  std::vector<int> lvl_cycle;
  std::vector<int> lvl_klo;
  for (int k = 0; k < n_cross; ++k)
    if (k == 0 || xcycle[k] != xcycle[k - 1]) lvl_cycle.push_back(xcycle[k]), lvl_klo.push_back(k);
  const int D = (int)lvl_cycle.size();
  p.levels.resize(D + 1);
  for (int l = 1; l <= D; ++l) {
    p.levels[l].k_lo = lvl_klo[l - 1];
    p.levels[l].k_hi = (l < D) ? lvl_klo[l] : n_cross;
    // cross ops first: every op of a cycle acts on disjoint qubits, so the
    // cycle's cross terms commute with its other ops
    for (int k = p.levels[l].k_lo; k < p.levels[l].k_hi; ++k)
      for (int side = 0; side < 2; ++side) {
        HostOp op;
        op.kind = p.xdiag[side][k] ? K_DIAG1 : K_MAT1;
        op.s0 = p.q[side] - 1 - p.xq[side][k];
        op.cross = k;
        p.levels[l].ops[side].push_back(op);
      }
  }
  int seen_cross = 0;
  for (int i = 0; i < n_ops; ++i) {
    const int kd = kind[i];
    if (kd == K_CROSS) {
      if (q0[i] != seen_cross) throw GsError(GS_ERR_ARG, "cross ops out of order");
      ++seen_cross;
      continue;
    }
    if (kd < 0 || kd > K_MAT2) throw GsError(GS_ERR_ARG, "unknown op kind");
    const int side = blk[i];
    if (side != 0 && side != 1) throw GsError(GS_ERR_ARG, "op block must be 0 or 1");
    const int q = p.q[side];
    HostOp op;
    op.kind = kd;
    if (q0[i] < 0 || q0[i] >= q) throw GsError(GS_ERR_ARG, "op qubit out of block");
    op.s0 = q - 1 - q0[i];
    if (kd == K_DIAG2 || kd == K_MAT2) {
      if (q1[i] < 0 || q1[i] >= q || q1[i] == q0[i]) throw GsError(GS_ERR_ARG, "bad second qubit");
      op.s1 = q - 1 - q1[i];
    }
    op.coef = coef_off[i];
    check_coef(op.coef, coef_entries(kd));
    if (kd == K_MAT1) classify_w(op, coef + 2 * op.coef);
    // level = number of cross cycles <= this op's cycle
    const int l = (int)(std::upper_bound(lvl_cycle.begin(), lvl_cycle.end(), cycle[i]) - lvl_cycle.begin());
    p.levels[l].ops[side].push_back(op);
  }
  if (seen_cross != n_cross) throw GsError(GS_ERR_ARG, "cross op count mismatch");
  if (c.hoist) hoist_ops(p);
  c.prog = std::move(p);
}

// diagonal factor d -> {rs, t, sn, mode}: d = rs * e^{i theta}, |theta| <= pi/2
static int add_param(Ctx& c, double re, double im) {
  double m = std::sqrt(re * re + im * im);
  double rs = m, cs = 1, sn = 0;
  if (m > 0) cs = re / m, sn = im / m;
  if (std::fabs(m - 1.0) < 1e-12) rs = 1.0;
  if (cs < 0) cs = -cs, sn = -sn, rs = -rs;
  if (std::fabs(sn) < 1e-15) sn = 0;
  const int mode = (rs != 1.0 ? 1 : 0) | (sn != 0 ? 2 : 0);
  const int at = (int)(c.host_params.size() / 4);
  c.host_params.insert(c.host_params.end(), {rs, sn / (1.0 + cs), sn, (double)mode});
  return at;
}

static bool is_identity(const double* z) { return z[0] == 1.0 && z[1] == 0.0; }

// lower one scheduled op into jump-table primitives (pass_types.h PrimCode)
static void emit_prims(Ctx& c, int side, const Level& L, const HostOp& op, const std::vector<int>& tpos,
                       const std::vector<int>& rpos) {
  const Program& p = c.prog;
  struct Bit { int where, idx; };
  auto loc = [&](int sb) -> Bit {
    const int t = tpos[sb];
    if (t >= 0 && rpos[t] >= 0) return {B_REG, rpos[t]};
    if (t >= 0) return {B_THREAD, t};
    return {B_TILE, sb};
  };
  auto prim = [&](int code) {
    PPrim q{};
    q.code = (uint8_t)code;
    q.ub_where = 255;
    return q;
  };
  auto set_ua = [](PPrim& q, Bit b) { q.ua_where = (uint8_t)b.where, q.ua_idx = (uint8_t)b.idx; };
  auto set_ub = [](PPrim& q, Bit b) { q.ub_where = (uint8_t)b.where, q.ub_idx = (uint8_t)b.idx; };
  const double* cf = p.coef.data();
  if (op.cross >= 0) {
    const int k = op.cross;
    const Bit b = loc(op.s0);
    // per-digit table: diag sides -> [lo param, hi param]; dense sides -> coef offset
    if (c.pxbase[side][k] < 0) {
      c.pxbase[side][k] = (int)c.host_pxtable.size();
      for (int d = 0; d < p.radix[k]; ++d) {
        const int32_t off = p.xtable[p.xtab[side][k] + d];
        if (p.xdiag[side][k]) {
          const int lo = add_param(c, cf[2 * off], cf[2 * off + 1]);
          add_param(c, cf[2 * off + 2], cf[2 * off + 3]);
          c.host_pxtable.push_back(lo);
        } else {
          c.host_pxtable.push_back(off);
        }
      }
    }
    const int xk = k - L.k_lo;
    if (xk >= 16 || p.radix[k] > 16) throw GsError(GS_ERR_ARG, "level digits exceed the packed nibble format");
    auto crossify = [&](PPrim q, int xsub) {
      q.flags = 1;
      q.param = c.pxbase[side][k];
      q.xk = (uint8_t)xk;
      q.xsub = (int16_t)xsub;
      c.host_prims.push_back(q);
    };
    if (!p.xdiag[side][k]) {
      PPrim q = prim(C_M1);
      q.r0 = (uint8_t)b.idx;
      crossify(q, 0);
    } else if (b.where == B_REG) {
      crossify(prim(C_DH + 0 * 5 + b.idx), 0);
      crossify(prim(C_DH + 1 * 5 + b.idx), 1);
    } else {
      PPrim q = prim(C_DSEL);
      set_ua(q, b);
      crossify(q, 0);
    }
    return;
  }
  const double* u = cf + 2 * op.coef;
  switch (op.kind) {
    case K_MAT1: {
      const Bit b = loc(op.s0);
      PPrim q = prim(op.w >= 0 ? C_W + op.w * 5 + b.idx : C_M1);
      q.r0 = (uint8_t)b.idx;
      q.param = (int32_t)op.coef;
      c.host_prims.push_back(q);
      break;
    }
    case K_DIAG1: {
      const Bit b = loc(op.s0);
      if (b.where == B_REG) {
        for (int h = 0; h < 2; ++h) {
          if (is_identity(u + 2 * h)) continue;
          PPrim q = prim(C_DH + h * 5 + b.idx);
          q.param = add_param(c, u[2 * h], u[2 * h + 1]);
          c.host_prims.push_back(q);
        }
      } else if (!(is_identity(u) && is_identity(u + 2))) {
        PPrim q = prim(C_DSEL);
        set_ua(q, b);
        q.param = add_param(c, u[0], u[1]);
        add_param(c, u[2], u[3]);
        c.host_prims.push_back(q);
      }
      break;
    }
    case K_DIAG2: {
      const Bit ba = loc(op.s0), bb = loc(op.s1);
      auto dz = [&](int xa, int xb) { return u + 2 * (2 * xa + xb); };
      if (ba.where == B_REG && bb.where == B_REG) {
        const int lo = std::min(ba.idx, bb.idx), hi = std::max(ba.idx, bb.idx);
        int pair = 0;
        for (int i = 0; i < lo; ++i) pair += 4 - i;
        pair += hi - lo - 1;
        for (int xa = 0; xa < 2; ++xa)
          for (int xb = 0; xb < 2; ++xb) {
            const double* z = dz(xa, xb);
            if (is_identity(z)) continue;
            const int xl = ba.idx < bb.idx ? xa : xb, xh = ba.idx < bb.idx ? xb : xa;
            PPrim q = prim(C_DQ + pair * 4 + 2 * xl + xh);
            q.param = add_param(c, z[0], z[1]);
            c.host_prims.push_back(q);
          }
      } else if (ba.where == B_REG || bb.where == B_REG) {
        const bool a_reg = ba.where == B_REG;
        const Bit r = a_reg ? ba : bb, un = a_reg ? bb : ba;
        for (int h = 0; h < 2; ++h) {
          const double* z0 = a_reg ? dz(h, 0) : dz(0, h);
          const double* z1 = a_reg ? dz(h, 1) : dz(1, h);
          if (is_identity(z0) && is_identity(z1)) continue;
          PPrim q = prim(C_DHSEL + h * 5 + r.idx);
          set_ua(q, un);
          q.param = add_param(c, z0[0], z0[1]);
          add_param(c, z1[0], z1[1]);
          c.host_prims.push_back(q);
        }
      } else {
        bool ident = true;
        for (int i = 0; i < 4; ++i) ident &= is_identity(u + 2 * i);
        if (!ident) {
          PPrim q = prim(C_DSEL);
          set_ua(q, ba);
          set_ub(q, bb);
          q.param = add_param(c, u[0], u[1]);
          for (int i = 1; i < 4; ++i) add_param(c, u[2 * i], u[2 * i + 1]);
          c.host_prims.push_back(q);
        }
      }
      break;
    }
    default: {  // K_MAT2
      const Bit ba = loc(op.s0), bb = loc(op.s1);
      if (ba.where != B_REG || bb.where != B_REG)
        throw GsError(GS_ERR_ARG, "stage scheduler placed a dense op outside the registers");
      PPrim q = prim(C_M2);
      q.r0 = (uint8_t)ba.idx;
      q.r1 = (uint8_t)bb.idx;
      q.param = (int32_t)op.coef;
      c.host_prims.push_back(q);
    }
  }
}

static uint64_t pack_level_digits(const Program& p, int l, int64_t v);

// the leaves are gathered by the path-major gather_kernel (not the grouped or
// shared-memory layouts)
static bool plain_gather(const Ctx& c) {
  const Program& p = c.prog;
  const size_t pair_bytes = (((size_t)1 << p.q[0]) + ((size_t)1 << p.q[1])) * c.esize();
  const bool smem_ok = c.smem_gather && 2 * pair_bytes <= 200 * 1024 && p.q[0] + p.q[1] <= 31 && p.q[0] >= 2 &&
                       p.q[1] >= 2;
  return !c.grouped_leaf && !smem_ok;
}

// A leaf side's last pass whose ops are one-/two-qubit gates on at most
// tail_max qubits (plus diagonal gates anywhere, no cross terms) is not run:
// the gather applies it per request (gather_tail_kernel).
static void extract_tail(Ctx& c, Level& L, int side) {
  c.tail_ops[side].clear();
  c.tail_bits[side].clear();
  if (!c.tail_gather || c.kernel_version != 2 || c.prog.q[1] == 0 || !plain_gather(c) || L.passes[side].size() < 2)
    return;  // (a full-state program has no gather)
  const PassPlan& last = L.passes[side].back();
  if (last.ops.empty() || last.ops.size() > 16) return;
  std::vector<int> T;
  for (const HostOp& op : last.ops) {
    if (op.cross >= 0) return;
    if (op.diag()) continue;
    for (int b : {op.s0, op.s1})
      if (b >= 0 && std::find(T.begin(), T.end(), b) == T.end()) T.push_back(b);
  }
  if ((int)T.size() > c.tail_max || T.empty()) return;
  c.tail_ops[side] = last.ops;
  c.tail_bits[side] = T;
  L.passes[side].pop_back();
}

// Leaf side whose cross terms are all projectors (one nonzero diagonal entry
// per term: P0/P1 of a CZ cut) and whose other leaf ops are one-qubit gates
// on those cross qubits only: its leaves are projections of the parent state
// followed by a product of 2x2 gates (gather_proj_kernel), so no leaf pass runs.
static bool projectable(const Ctx& c, int side) {
  const Program& p = c.prog;
  const int D = (int)p.levels.size() - 1;
  if (D < 1 || p.q[1 - side] == 0) return false;
  const Level& L = p.levels[D];
  if (L.k_hi - L.k_lo > 8 || L.k_hi <= L.k_lo) return false;
  std::vector<int> C;
  for (int k = L.k_lo; k < L.k_hi; ++k) {
    if (!p.xdiag[side][k] || p.radix[k] > 16) return false;
    for (int d = 0; d < p.radix[k]; ++d) {
      const double* x = &p.coef[2 * (size_t)p.xtable[p.xtab[side][k] + d]];
      const bool n0 = x[0] != 0.0 || x[1] != 0.0, n1 = x[2] != 0.0 || x[3] != 0.0;
      if (n0 == n1) return false;
    }
    C.push_back(p.q[side] - 1 - p.xq[side][k]);
  }
  for (const HostOp& op : L.ops[side]) {
    if (op.cross >= 0) continue;
    if (op.kind != K_MAT1 && op.kind != K_DIAG1) return false;
    if (std::find(C.begin(), C.end(), op.s0) == C.end()) return false;
  }
  return true;
}

// Pauli frame of a leaf side whose cross terms are x0 * Z^z (the I / Z side of
// a CZ cut).  A cross term Z inserted before the level's remaining ops O equals
// the Pauli P = O Z O^+ applied after them when every op maps the running
// Pauli to a Pauli (H, X^1/2, Y^1/2, CZ: Clifford; T and other diagonals while
// the Pauli is Z-type on their qubits), so every leaf of a parent is a Pauli
// image of ONE state, base = O psi (no cross terms):
//   leaf_d = prod_j x0_j(d_j) * P_j^zsel_j(d_j) base,
//   (i^a X^f Z^z phi)[x] = i^a (-1)^(z.f) (-1)^(z.x) phi[x ^ f].
// The conjugations are done numerically on the ops' own matrices (2x2 / 4x4)
// and matched against the Pauli group, so any gate set is handled: a level
// that is not Pauli-compatible simply returns ok = false.
static PauliFrame pauli_frame(const Ctx& c, int side, const std::vector<HostOp>& ops) {
  using cd = std::complex<double>;
  PauliFrame pf;
  const Program& p = c.prog;
  const int D = (int)p.levels.size() - 1;
  if (D < 1) return pf;
  const Level& L = p.levels[D];
  const int nk = L.k_hi - L.k_lo;
  if (nk < 1 || nk > 8 || p.q[side] > 31) return pf;
  pf.nk = nk;
  const cd iu(0.0, 1.0);
  const cd ph[4] = {cd(1, 0), iu, cd(-1, 0), -iu};
  auto pauli_mat = [](int n, int fm, int zm, cd* M) {  // X^fm Z^zm on n qubits, local bit n-1 = first qubit
    const int dim = 1 << n;
    for (int i = 0; i < dim * dim; ++i) M[i] = 0.0;
    for (int y = 0; y < dim; ++y) M[(y ^ fm) * dim + y] = (__builtin_popcount(zm & y) & 1) ? -1.0 : 1.0;
  };
  std::vector<std::pair<int, int>> pos;  // (position of the cross op in the list, gate)
  for (int j = 0; j < nk; ++j) {
    const int k = L.k_lo + j;
    if (!p.xdiag[side][k] || p.radix[k] > 16) return pf;
    for (int d = 0; d < p.radix[k]; ++d) {
      const double* x = &p.coef[2 * (size_t)p.xtable[p.xtab[side][k] + d]];
      const cd x0(x[0], x[1]), x1(x[2], x[3]);
      const double tol = 1e-12 * std::max(1e-300, std::max(std::abs(x0), std::abs(x1)));
      if (std::abs(x0) <= tol && std::abs(x1) <= tol) return pf;
      if (std::abs(x0) <= tol || std::abs(x1) <= tol) {
        // projector term a * (I + (-1)^v Z) / 2 (the P0 / P1 side of a CZ cut): zsel = 2 + v, x0 = a
        const int v = std::abs(x0) <= tol ? 1 : 0;
        pf.zsel[j][d] = 2 + v;
        pf.x0[j][d][0] = x[2 * v], pf.x0[j][d][1] = x[2 * v + 1];
        pf.projector = true;
        continue;
      }
      if (std::abs(x1 - x0) <= tol) pf.zsel[j][d] = 0;
      else if (std::abs(x1 + x0) <= tol) pf.zsel[j][d] = 1;
      else return pf;
      pf.x0[j][d][0] = x[0], pf.x0[j][d][1] = x[1];
    }
    int at = -1, sb = -1;
    for (size_t i = 0; i < ops.size(); ++i)
      if (ops[i].cross == k) {
        if (at >= 0) return pf;
        at = (int)i, sb = ops[i].s0;
      }
    if (at < 0 || sb < 0) return pf;
    pos.push_back({at, j});
    // push Z on state bit sb through the ops behind the cross term
    int a = 0;
    uint32_t f = 0, z = 1u << sb;
    for (size_t i = (size_t)at + 1; i < ops.size(); ++i) {
      const HostOp& op = ops[i];
      if (op.cross >= 0) continue;  // other cross terms are diagonal in Z ... checked below
      const bool two = op.kind == K_DIAG2 || op.kind == K_MAT2;
      const int b1 = op.s0, b0 = two ? op.s1 : -1;  // local bit 1 (high) = s0, local bit 0 = s1
      if (two && b0 == b1) return pf;
      const int n = two ? 2 : 1, dim = 1 << n;
      auto lbit = [&](uint32_t m) {
        return two ? (int)(((m >> b1) & 1u) << 1 | ((m >> b0) & 1u)) : (int)((m >> b1) & 1u);
      };
      const int fm = lbit(f), zm = lbit(z);
      if (fm == 0 && zm == 0) continue;
      cd U[16], S[16], R[16];
      const double* u = &p.coef[2 * (size_t)op.coef];
      for (int e = 0; e < dim * dim; ++e) U[e] = 0.0;
      if (op.diag())
        for (int e = 0; e < dim; ++e) U[e * dim + e] = cd(u[2 * e], u[2 * e + 1]);
      else
        for (int e = 0; e < dim * dim; ++e) U[e] = cd(u[2 * e], u[2 * e + 1]);
      pauli_mat(n, fm, zm, S);
      for (int r = 0; r < dim; ++r)
        for (int q2 = 0; q2 < dim; ++q2) {
          cd acc = 0.0;
          for (int k2 = 0; k2 < dim; ++k2)
            for (int l2 = 0; l2 < dim; ++l2) acc += U[r * dim + k2] * S[k2 * dim + l2] * std::conj(U[q2 * dim + l2]);
          R[r * dim + q2] = acc;
        }
      bool found = false;
      for (int fm2 = 0; fm2 < dim && !found; ++fm2)
        for (int zm2 = 0; zm2 < dim && !found; ++zm2) {
          cd C[16];
          pauli_mat(n, fm2, zm2, C);
          for (int t = 0; t < 4 && !found; ++t) {
            double err = 0;
            for (int e = 0; e < dim * dim; ++e) err = std::max(err, std::abs(R[e] - ph[t] * C[e]));
            if (err <= 1e-9) {
              found = true;
              a = (a + t) & 3;
              auto put = [&](uint32_t& m, int v) {
                m &= ~(1u << b1);
                if (two) m &= ~(1u << b0);
                if (two) m |= (uint32_t)((v >> 1) & 1) << b1 | (uint32_t)(v & 1) << b0;
                else m |= (uint32_t)(v & 1) << b1;
              };
              put(f, fm2);
              put(z, zm2);
            }
          }
        }
      if (!found) return pf;
    }
    pf.a[j] = a, pf.f[j] = f, pf.z[j] = z;
  }
  // a later cross term must commute with the Z being pushed through it: all are diagonal (checked: xdiag)
  // but the pushed Pauli may have picked up an X part on that qubit by then -- x0 Z^z X = +-X x0 Z^z,
  // a sign the frame above does not track.  Reject that (rare) case.
  for (int j = 0; j < nk; ++j) {
    const int k = L.k_lo + j;
    int at = -1;
    for (size_t i = 0; i < ops.size(); ++i)
      if (ops[i].cross == k) at = (int)i;
    for (int j2 = 0; j2 < nk; ++j2) {
      if (j2 == j) continue;
      int at2 = -1, sb2 = -1;
      for (size_t i = 0; i < ops.size(); ++i)
        if (ops[i].cross == L.k_lo + j2) at2 = (int)i, sb2 = ops[i].s0;
      if (at2 <= at) continue;
      // the Z of gate j passes cross term j2 (at position at2): recompute its X part up to there
      // conservatively: reject when any op between them touches bit sb2 non-diagonally
      for (int i = at + 1; i < at2; ++i)
        if (ops[i].cross < 0 && !ops[i].diag() && (ops[i].s0 == sb2 || ops[i].s1 == sb2)) return pf;
    }
  }
  std::sort(pos.begin(), pos.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) { return x.first > y.first; });
  for (int i = 0; i < nk; ++i) pf.order[i] = pos[i].second;
  pf.ok = true;
  return pf;
}

// GF(2) helpers for the parked-tile address map (K x K bit matrices, rows as masks)
static uint32_t gf2_apply(const uint32_t* rows, int K, uint32_t v) {
  uint32_t o = 0;
  for (int i = 0; i < K; ++i) o |= (uint32_t)(__builtin_popcount(rows[i] & v) & 1) << i;
  return o;
}
static bool gf2_inverse(const uint32_t* rows, int K, uint32_t* inv) {
  uint32_t a[16], b[16];
  for (int i = 0; i < K; ++i) a[i] = rows[i], b[i] = 1u << i;
  for (int col = 0; col < K; ++col) {
    int piv = -1;
    for (int r = col; r < K; ++r)
      if ((a[r] >> col) & 1u) { piv = r; break; }
    if (piv < 0) return false;
    std::swap(a[piv], a[col]);
    std::swap(b[piv], b[col]);
    for (int r = 0; r < K; ++r)
      if (r != col && ((a[r] >> col) & 1u)) a[r] ^= a[col], b[r] ^= b[col];
  }
  for (int i = 0; i < K; ++i) inv[i] = b[i];
  return true;
}
static int gf2_rank(std::vector<uint32_t> v) {
  int rank = 0;
  for (int bit = 0; bit < 32; ++bit) {
    int piv = -1;
    for (size_t i = rank; i < v.size(); ++i)
      if ((v[i] >> bit) & 1u) { piv = (int)i; break; }
    if (piv < 0) continue;
    std::swap(v[piv], v[rank]);
    for (size_t i = 0; i < v.size(); ++i)
      if ((int)i != rank && ((v[i] >> bit) & 1u)) v[i] ^= v[rank];
    ++rank;
  }
  return rank;
}

// Address map of the Pauli-sibling pass's parked tile: an invertible GF(2)-linear
// L on the K tile bits with L f_b = e_b for the flips f_b of the last three cross
// gates (sibling bit b), so the 8 siblings of a request are one 64-byte run of
// the parked base tile (sibling pair s, s + 1 = one aligned 16 bytes).  Built as
// L = S M^-1: M's columns are the independent flips followed by unit vectors
// (the last stage's lane bits first), S xors three upper address bits into the
// low three so a warp's park stores spread over the banks.
static void plan_pauli_layout(Ctx& c) {
  for (int j = 0; j < 16; ++j) c.pauli_lcol[j] = c.pauli_lit[j] = 1u << j;
  if (!c.pauli.ok) return;
  const Program& p = c.prog;
  const int D = (int)p.levels.size() - 1, side = 1 - c.proj_side;
  const PassPlan& pp = p.levels[D].passes[side].back();
  const int K = pp.k, nk = c.pauli.nk;
  std::vector<int> tpos(p.q[side], -1);
  for (int j = 0; j < K; ++j) tpos[pp.lbits[j]] = j;
  auto local = [&](uint32_t m) {
    uint32_t o = 0;
    for (int b = 0; b < p.q[side]; ++b)
      if ((m >> b) & 1u) o |= 1u << tpos[b];
    return o;
  };
  std::vector<uint32_t> cols(K, 0), have;
  std::vector<char> filled(K, 0);
  for (int b = 0; b < 3 && b < nk; ++b) {
    const uint32_t g = local(c.pauli.f[nk - 1 - b]);
    std::vector<uint32_t> t = have;
    t.push_back(g);
    if (g != 0 && gf2_rank(t) == (int)t.size()) cols[b] = g, filled[b] = 1, have = t;
  }
  std::vector<int> pref;  // unit vectors: lane bits of the last stage first
  const PStage& last = c.host_pstages[pp.dev_stage_offset + pp.stages.size() - 1];
  for (int j = 0; j < 5 && j < K - pp.M; ++j) pref.push_back(last.tb[j]);
  for (int j = 0; j < K; ++j)
    if (std::find(pref.begin(), pref.end(), j) == pref.end()) pref.push_back(j);
  // upper positions (3..K-1) take the preferred bits first, the unfilled low positions what is left
  std::vector<int> slots;
  for (int i = 3; i < K; ++i) slots.push_back(i);
  for (int i = 0; i < 3 && i < K; ++i)
    if (!filled[i]) slots.push_back(i);
  size_t si = 0;
  for (int j : pref) {
    if (si >= slots.size()) break;
    std::vector<uint32_t> t = have;
    t.push_back(1u << j);
    if (gf2_rank(t) != (int)t.size()) continue;
    cols[slots[si++]] = 1u << j;
    have = t;
  }
  uint32_t M[16] = {}, Mi[16] = {};
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) M[i] |= ((cols[j] >> i) & 1u) << j;
  if (!gf2_inverse(M, K, Mi)) throw GsError(GS_ERR_STATE, "pauli layout: singular basis");
  // S: low three address bits ^= address bits sh .. sh + 2; pick sh by the park stores' bank conflicts
  int best_sh = -1, best_cost = 1 << 30;
  uint32_t best_rows[16] = {};
  for (int sh = 3; sh + 3 <= K; ++sh) {
    uint32_t rows[16];
    for (int i = 0; i < K; ++i) rows[i] = Mi[i];
    for (int r = 0; r < 3; ++r) rows[r] ^= Mi[sh + r];
    int worst = 1;
    for (int half = 0; half < 2; ++half) {
      int cnt[16] = {0};
      for (int l = 0; l < 16; ++l) {
        uint32_t t = 0;
        const int lane = l + 16 * half;
        for (int j = 0; j < 5 && j < K - pp.M; ++j)
          if ((lane >> j) & 1) t |= 1u << last.tb[j];
        worst = std::max(worst, ++cnt[gf2_apply(rows, K, t) & 15u]);
      }
    }
    if (worst < best_cost) {
      best_cost = worst, best_sh = sh;
      for (int i = 0; i < K; ++i) best_rows[i] = rows[i];
    }
  }
  if (best_sh < 0)
    for (int i = 0; i < K; ++i) best_rows[i] = Mi[i];
  uint32_t inv[16] = {};
  if (!gf2_inverse(best_rows, K, inv)) throw GsError(GS_ERR_STATE, "pauli layout: singular map");
  for (int j = 0; j < K; ++j) {
    c.pauli_lcol[j] = gf2_apply(best_rows, K, 1u << j);
    c.pauli_lit[j] = inv[j];  // row j of L^-1 = column j of L^-T
  }
  c.pauli_conflicts = best_cost;
}

static void schedule_program(Ctx& c) {
  Program& p = c.prog;
  ++c.sched_serial;
  c.host_devops.clear();
  // Leaf states go to the grouped path-minor layout when the gather reads them
  // from HBM (half-states too large for the shared-memory gather).
  {
    const size_t pair_bytes = (((size_t)1 << p.q[0]) + ((size_t)1 << p.q[1])) * c.esize();
    // grouping costs the leaf level group_log tile bits (possibly an extra pass);
    // it pays while a leaf's random-sector gather traffic (~40 B per request) is
    // comparable to its pass traffic, i.e. up to ~2^24-amplitude halves
    c.grouped_leaf = c.kernel_version == 2 && c.grouped_enabled && 2 * pair_bytes > 200 * 1024 &&
                     std::min(p.q[0], p.q[1]) >= 12 && std::max(p.q[0], p.q[1]) <= 24;
  }
  const int D = (int)p.levels.size() - 1;
  c.proj_side = -1;
  c.pauli = PauliFrame{};
  c.psib = PauliFrame{};
  c.psib_side = -1;
  if (c.proj_leaf && c.grouped_leaf && !c.fuse_gather && c.kernel_version == 2)
    for (int side = 0; side < 2 && c.proj_side < 0; ++side)
      if (projectable(c, side)) c.proj_side = side;
  // working op lists; option sink_ops: a level's trailing pass of at most
  // sink_ops ops that commute with the next level's cross terms is moved to the
  // start of that level (after its cross terms), where it can share a pass --
  // worth it when the next level has few more nodes (sparse prefix levels)
  std::vector<std::vector<HostOp>> work[2];
  for (int side = 0; side < 2; ++side) {
    work[side].resize(p.levels.size());
    for (size_t l = 0; l < p.levels.size(); ++l) work[side][l] = p.levels[l].ops[side];
  }
  if (c.sink_ops > 0)
    for (int l = 0; l + 2 <= D; ++l)
      for (int side = 0; side < 2; ++side) {
        if (p.q[side] == 0) continue;
        std::vector<PassPlan> ps = schedule_passes(work[side][l], p.q[side], c.kmax(), c.low_bits, true);
        if (ps.size() < 2 || (int)ps.back().ops.size() > c.sink_ops) continue;
        const Level& N = p.levels[l + 1];
        std::vector<HostOp> head, rest;
        for (const HostOp& op : work[side][l + 1]) (op.cross >= 0 ? head : rest).push_back(op);
        bool ok = true;
        for (const HostOp& m : ps.back().ops)
          for (const HostOp& x : head) ok = ok && !ops_conflict(m, x);
        if (!ok || N.k_hi <= N.k_lo) continue;
        std::vector<HostOp> keep;
        for (size_t i = 0; i + 1 < ps.size(); ++i) keep.insert(keep.end(), ps[i].ops.begin(), ps[i].ops.end());
        work[side][l] = keep;
        head.insert(head.end(), ps.back().ops.begin(), ps.back().ops.end());
        head.insert(head.end(), rest.begin(), rest.end());
        work[side][l + 1] = head;
      }
  // Balance sink (option sink_balance): the last level above the leaf parents (D-2) holds several
  // cycles of gates while the leaf parents' level (D-1) holds few, and at small path fractions both
  // have about one node per retained prefix -- the op-heavy passes of D-2 then run FMA-co-limited
  // (~4 TB/s) next to HBM-bound, FP-light passes of D-1.  A suffix of level D-2's ops moves to the
  // FRONT of level D-1's list (ahead of its cross terms: the same operator order, so exact without
  // any commutation), as long as D-1 still needs no more passes, until the two levels' estimated
  // arithmetic is balanced.
  if (c.sink_balance > 0 && D >= 3)
    for (int side = 0; side < 2; ++side) {
      const int l = D - 2;
      if (p.q[side] == 0 || work[side][l].empty()) continue;
      auto cost = [](const HostOp& op) {
        if (op.cross >= 0) return 1.0;
        switch (op.kind) {
          case K_MAT1: return 2.0;
          case K_MAT2: return 8.0;
          case K_DIAG1: return 1.5;
          default: return 1.0;
        }
      };
      double fa = 0, fb = 0;
      for (const HostOp& op : work[side][l]) fa += cost(op);
      for (const HostOp& op : work[side][l + 1]) fb += cost(op);
      const size_t base_passes = schedule_passes(work[side][l + 1], p.q[side], c.kmax(), c.low_bits, true).size();
      size_t best = 0;
      double moved = 0;
      for (size_t sfx = 1; sfx < work[side][l].size(); ++sfx) {
        const HostOp& op = work[side][l][work[side][l].size() - sfx];
        if (op.cross >= 0) break;  // a level keeps its own cross terms
        moved += cost(op);
        if (fa - moved < fb + moved) break;
        std::vector<HostOp> next(work[side][l].end() - sfx, work[side][l].end());
        next.insert(next.end(), work[side][l + 1].begin(), work[side][l + 1].end());
        if (schedule_passes(next, p.q[side], c.kmax(), c.low_bits, true).size() > base_passes) break;
        best = sfx;
      }
      if (best == 0) continue;
      std::vector<HostOp> next(work[side][l].end() - best, work[side][l].end());
      next.insert(next.end(), work[side][l + 1].begin(), work[side][l + 1].end());
      work[side][l].resize(work[side][l].size() - best);
      work[side][l + 1] = next;
    }
  for (size_t l = 0; l < p.levels.size(); ++l) {
    Level& L = p.levels[l];
    for (int side = 0; side < 2; ++side) {
      if ((int)l == D && side == c.proj_side) {  // leaves read from the parent in the gather
        L.passes[side].clear();
        continue;
      }
      const int kcap = ((int)l == D && c.grouped_leaf) ? c.kmax() - c.group_log : c.kmax();
      if (p.q[side] == 0) {  // empty block of a full-state program
        L.passes[side].clear();
        continue;
      }
      // Pauli-sibling leaf (option pf_pauli): the grouped side of a fused projected leaf whose
      // cross terms are x0 * Z^z and whose leaf ops keep that Z a Pauli -- one pass without
      // cross terms or slot bits evolves the base state of each leaf group
      bool pauli = false;
      if ((int)l == D && c.pf_pauli && !c.pauli_blocked && c.proj_fuse && c.grouped_leaf && c.proj_side == 1 - side &&
          c.precision == GS_C64 && c.use_jit && !c.pipeline && c.group_log == 3 && L.k_hi - L.k_lo >= 1 &&
          L.k_hi - L.k_lo <= 5) {
        PauliFrame pf = pauli_frame(c, side, work[side][l]);
        if (pf.ok && !pf.projector) {
          std::vector<HostOp> nc;
          for (const HostOp& op : work[side][l])
            if (op.cross < 0) nc.push_back(op);
          std::vector<PassPlan> ps = schedule_passes(nc, p.q[side], c.kmax(), c.low_bits, true);
          uint32_t need = 0, have = 0;
          for (int j = 0; j < pf.nk; ++j) need |= pf.f[j] | pf.z[j];
          if (ps.size() == 1)
            for (int b : ps[0].lbits) have |= 1u << b;
          if (ps.size() == 1 && ps[0].k >= 10 && ps[0].k <= 16 && (need & ~have) == 0) {
            ps[0].level = (int)l;
            ps[0].proj_fused = true;
            ps[0].pf_pauli = true;
            L.passes[side] = std::move(ps);
            c.pauli = pf;
            c.tail_ops[side].clear();
            c.tail_bits[side].clear();
            pauli = true;
          }
        }
      }
      if (!pauli && (int)l == D && D >= 1 && c.pf_pauli && side == 1 && c.kernel_version == 2 && !c.grouped_leaf &&
          plain_gather(c) && p.q[side] >= 5 && p.q[side] <= 31 && L.k_hi - L.k_lo >= 1 && L.k_hi - L.k_lo <= 8) {
        PauliFrame pf = pauli_frame(c, side, work[side][l]);
        if (pf.ok && !pf.projector) {
          std::vector<HostOp> nc;
          for (const HostOp& op : work[side][l])
            if (op.cross < 0) nc.push_back(op);
          L.passes[side] = schedule_passes(nc, p.q[side], kcap, c.low_bits, true);
          for (PassPlan& pp : L.passes[side]) pp.level = (int)l;
          extract_tail(c, L, side);
          c.psib = pf;
          c.psib_side = side;
          pauli = true;
        }
      }
      if (!pauli) {
      L.passes[side] = schedule_passes(work[side][l], p.q[side], kcap, c.low_bits, true);
      for (PassPlan& pp : L.passes[side]) pp.level = (int)l;
      if ((int)l == D) extract_tail(c, L, side);
      }
      if ((int)l == D && c.grouped_leaf && !pauli) {
        L.passes[side].back().grouped_store = true;
        if (side == 1 && c.fuse_gather && c.group_log == 3 && c.precision == GS_C64)
          L.passes[side].back().fused_gather = true;
        const int nk = L.k_hi - L.k_lo;
        PassPlan& lp = L.passes[side].back();
        if (c.proj_fuse && c.proj_side == 1 - side && c.precision == GS_C64 && c.use_jit && !c.pipeline &&
            c.group_log == 3 && nk >= 1 && nk <= 5 && c.tail_ops[side].empty())
          lp.proj_fused = true;
      }
      for (PassPlan& pp : L.passes[side]) {
        pp.dev_op_offset = (int64_t)c.host_devops.size();
        std::vector<int> tpos(p.q[side], -1);
        for (int j = 0; j < (int)pp.lbits.size(); ++j) tpos[pp.lbits[j]] = j;
        for (const HostOp& op : pp.ops) {
          DevOp d{};
          d.xtab = -1;
          d.xstride = 1;
          d.xradix = 1;
          d.coef = (int32_t)op.coef;
          if (op.cross >= 0) {
            d.xtab = p.xtab[side][op.cross];
            d.xstride = op.cross - L.k_lo;  // nibble of the packed node digits
            d.xradix = p.radix[op.cross];
          }
          auto enc = [&](int s, int32_t& b, int32_t& g) {
            if (s < 0) { b = 0; g = 0; return; }
            if (tpos[s] >= 0) { b = tpos[s]; g = 0; } else { b = s; g = 1; }
          };
          enc(op.s0, d.b0, d.g0);
          enc(op.s1, d.b1, d.g1);
          switch (op.kind) {
            case K_MAT1: d.type = D_MAT1; break;
            case K_DIAG1: d.type = D_DIAG1; break;
            case K_DIAG2: d.type = D_DIAG2; break;
            default: d.type = D_MAT2; break;
          }
          if ((d.type == D_MAT1 || d.type == D_MAT2) && (d.g0 || d.g1))
            throw GsError(GS_ERR_ARG, "scheduler placed a dense op outside the tile");
          c.host_devops.push_back(d);
        }
      }
    }
  }
  // v2: register stages per pass, W scalars folded into one constant per block
  c.host_prims.clear();
  c.host_params.clear();
  c.host_pxtable.clear();
  c.pxbase[0].assign(p.n_cross, -1);
  c.pxbase[1].assign(p.n_cross, -1);
  c.host_pstages.clear();
  c.host_tbtab.clear();
  c.host_gofftab.clear();
  for (int side = 0; side < 2; ++side) {
    double kre = 1.0, kim = 0.0;  // true amplitude = stored * K
    for (size_t l = 0; l < p.levels.size(); ++l) {
      Level& L = p.levels[l];
      for (PassPlan& pp : L.passes[side]) {
        // register bits per stage: 5 (c64) / 4 (c128); tiny states (< 4 qubits in
        // the tile) keep the v1 shared-memory kernel
        // 5 register bits (256 threads) by default; 4 (512 threads, 2 CTAs/SM) for
        // the op-heavy, non-grouped passes when reg_bits = 0 (auto, m4_ops threshold)
        bool m4 = c.reg_bits == 4;
        if (c.reg_bits == 0) m4 = c.use_jit && !pp.grouped_store && (int)pp.ops.size() >= c.m4_ops;
        // reg_bits = 6 (auto by state size): 4 register bits (512-thread CTAs, 2 per SM)
        // for half-states of >= 2^26 amplitudes, whose passes stream from HBM with no L2 reuse
        // (with the L2 prefetch-ahead on, 5 register bits win there too: cfg5 360 -> 374, cfg5f 238 -> 244)
        if (c.reg_bits == 6) m4 = c.use_jit && !pp.grouped_store && p.q[side] >= 26 && c.l2_ahead == 0;
        if (pp.pf_pauli) m4 = c.pf_m4 != 0;  // option pf_m4: 512-thread CTAs, 16 amplitudes per thread
        pp.M = (c.precision == GS_C64 && pp.k >= 5 && !m4) ? 5 : (pp.k >= 4 ? 4 : 0);
        if (pp.M == 0) continue;
        // tile = k state bits + slot bits batching small states, up to 2^13 (c64) /
        // 2^12 (c128) amplitudes and 256 threads
        pp.K = std::max(pp.k, std::min(c.kmax(), pp.M + 8));
        if (pp.grouped_store) pp.K = pp.k + c.group_log;  // the grouped store interleaves 2^G slots
        // complex64 specialised passes use 16-byte HBM accesses (jitgen.inc)
        const bool vec = c.precision == GS_C64 && c.use_jit && c.vec_hbm && (pp.M == 5 || pp.M == 4);
        // (the Pauli-sibling pass parks its tile in shared memory: like a grouped store, any last-stage
        // register set is fine)
        pp.stages = schedule_stages(pp, pp.M, vec, pp.grouped_store ? c.group_log : (pp.pf_pauli ? 3 : 0),
                                    pp.grouped_store && c.slot_store16 && !c.pipeline);
        pp.dev_stage_offset = (int64_t)c.host_pstages.size();
        pp.goff_offset = (int64_t)c.host_gofftab.size();
        for (int t = 0; t < (1 << pp.k); ++t) {
          uint32_t g = 0;
          for (int j = 0; j < pp.k; ++j) g |= (uint32_t)((t >> j) & 1) << pp.lbits[j];
          c.host_gofftab.push_back(g);
        }
        std::vector<int> tpos(p.q[side], -1);
        for (int j = 0; j < (int)pp.lbits.size(); ++j) tpos[pp.lbits[j]] = j;
        for (const StagePlan& sp : pp.stages) {
          PStage ps{};
          std::vector<int> rpos(pp.K, -1);  // register position of each tile bit (slot bits included)
          for (int i = 0; i < (int)sp.rb.size(); ++i) ps.rb[i] = (int8_t)sp.rb[i], rpos[sp.rb[i]] = i;
          {  // swizzled shared-tile byte step per register bit (pass_kernel.cuh swz)
            const int lb = c.precision == GS_C64 ? 4 : 3;
            for (int i = 0; i < (int)sp.rb.size(); ++i) {
              const uint32_t t = 1u << sp.rb[i];
              const uint32_t z = t ^ (((t >> lb) ^ (t >> (2 * lb)) ^ (t >> (3 * lb)) ^ (t >> (4 * lb))) & ((1u << lb) - 1));
              ps.sstep[i] = z * (uint32_t)c.esize();
            }
          }
          // thread-bit order over the tile bits (state bits then slot bits up to
          // the kernel's K); lanes are thread bits 0..4.  HBM stages keep the
          // lowest tile bits on the lanes; shared-memory-only stages pick lanes
          // whose swizzle classes are distinct (conflict-free exchanges).
          {
            const size_t si = &sp - &pp.stages[0];
            const bool hbm_stage = (si == 0) || (si + 1 == pp.stages.size());
            std::vector<int> tbits;
            for (int j = 0; j < pp.K; ++j)
              if (rpos[j] < 0) tbits.push_back(j);
            if (pp.grouped_store && si + 1 == pp.stages.size()) {
              // grouped store: slot bits on the lowest lanes -> 2^G leaves x 2^(5-G)
              // amplitudes = 256 contiguous bytes per warp store
              std::vector<int> slot_first;
              for (int j : tbits)
                if (j >= pp.k) slot_first.push_back(j);
              for (int j : tbits)
                if (j < pp.k) slot_first.push_back(j);
              tbits = slot_first;
            } else if (!hbm_stage) {
              const int nclass = (c.precision == GS_C64) ? 4 : 3;
              std::vector<int> lanes, rest;
              std::vector<char> used_class(nclass, 0);
              for (int j : tbits) {
                if ((int)lanes.size() < nclass && !used_class[j % nclass]) {
                  used_class[j % nclass] = 1;
                  lanes.push_back(j);
                } else {
                  rest.push_back(j);
                }
              }
              tbits = lanes;
              tbits.insert(tbits.end(), rest.begin(), rest.end());
            }
            for (int j = 0; j < (int)tbits.size() && j < 16; ++j) ps.tb[j] = (int8_t)tbits[j];
            // thread -> tile-index base for this stage (row of 256 in tbtab)
            const int nthr = 1 << (pp.K - pp.M);
            for (int t = 0; t < 256; ++t) {
              int tbv = 0;
              if (t < nthr)
                for (int j = 0; j < pp.K - pp.M; ++j) tbv |= ((t >> j) & 1) << tbits[j];
              c.host_tbtab.push_back((uint16_t)tbv);
            }
          }
          ps.op_begin = (int32_t)c.host_prims.size();
          for (const HostOp& op : sp.ops) {
            emit_prims(c, side, L, op, tpos, rpos);
            if (op.w >= 0) {  // K *= s
              const double r = kre * op.s_re - kim * op.s_im, i = kre * op.s_im + kim * op.s_re;
              kre = r, kim = i;
            }
          }
          ps.op_end = (int32_t)c.host_prims.size();
          c.host_pstages.push_back(ps);
        }
        // power-of-two rescale on store keeps |stored| ~ |true amplitude|
        const double mag = std::sqrt(kre * kre + kim * kim);
        const int e = (int)std::lround(std::log2(mag));
        pp.store_scale = 1.0;
        if (std::abs(e) >= 16) {
          pp.store_scale = std::ldexp(1.0, e);
          kre = std::ldexp(kre, -e);
          kim = std::ldexp(kim, -e);
        }
      }
    }
    c.kfinal[side][0] = kre;
    c.kfinal[side][1] = kim;
  }
  // projected leaf side: store its parents (the last pass of level D-1) with the
  // run gates' qubits at address bits 0..G-1, so a sibling block's 2^G parent
  // amplitudes are one contiguous run for the gather
  c.proj_swaps.clear();
  c.proj_perm_pass = nullptr;
  bool pf_planned = false;
  if (c.proj_side >= 0 && D >= 1)
    for (const PassPlan& pp : p.levels[D].passes[1 - c.proj_side]) pf_planned |= pp.proj_fused;
  if ((c.proj_perm || pf_planned) && c.proj_side >= 0 && D >= 2 && c.precision == GS_C64 && c.use_jit &&
      !c.pipeline) {
    const int ps = c.proj_side, q = p.q[ps];
    Level& LP = p.levels[D - 1];
    const Level& LD = p.levels[D];
    const int nk = LD.k_hi - LD.k_lo;
    if (!LP.passes[ps].empty() && nk >= c.group_log) {
      PassPlan& last = LP.passes[ps].back();
      std::vector<int> pos(q), inv(q);
      for (int b = 0; b < q; ++b) pos[b] = inv[b] = b;
      std::vector<std::pair<int, int>> sw;
      for (int b = 0; b < c.group_log; ++b) {
        const int sbit = q - 1 - p.xq[ps][LD.k_lo + nk - 1 - b];
        const int cur = pos[sbit];
        if (cur == b) continue;
        const int other = inv[b];
        pos[sbit] = b, pos[other] = cur, inv[b] = sbit, inv[cur] = other;
        sw.push_back({cur, b});
      }
      bool ok = (last.M == 5 || last.M == 4) && !last.grouped_store && !sw.empty();
      for (int b = 0; b < q && ok; ++b)
        if (pos[b] != b) ok = std::find(last.lbits.begin(), last.lbits.end(), b) != last.lbits.end();
      if (ok) {
        last.store_perm = pos;
        c.proj_swaps = sw;
        c.proj_perm_pass = &last;
      }
    }
  }
  plan_pauli_layout(c);
  // packed-digit lookup per level (fan-outs up to 2^16)
  for (size_t l = 1; l < p.levels.size(); ++l) {
    Level& L = p.levels[l];
    L.packed.clear();
    int64_t F = 1;
    for (int k = L.k_lo; k < L.k_hi; ++k) F *= p.radix[k];
    if (F > 65536) continue;
    std::vector<uint64_t> tab(F);
    for (int64_t v = 0; v < F; ++v) tab[v] = pack_level_digits(p, (int)l, v);
    L.packed = std::move(tab);
  }
  // level digit products must fit int32 node digits
  for (size_t l = 1; l < p.levels.size(); ++l) {
    int64_t f = 1;
    for (int k = p.levels[l].k_lo; k < p.levels[l].k_hi; ++k) {
      f *= p.radix[k];
      if (f > INT32_MAX) throw GsError(GS_ERR_ARG, "level fan-out exceeds int32");
    }
  }
}

template <typename T> static void upload(Ctx& c, DevBuf& b, const std::vector<T>& v) {
  b.ensure(std::max<size_t>(v.size() * sizeof(T), 16));
  if (!v.empty()) CK(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// Specialise every eligible pass (complex64, 5 register bits) into one NVRTC
// module.  Failure keeps the interpreter kernels and records why.
static void jit_program(Ctx& c) {
  c.fused_active = false;
  c.proj_fused_active = false;
  c.bucket_valid = false;
  for (JitModule* m : c.jit_mods) jit_release(m);
  c.jit_mods.clear();
  c.jit_loc.clear();
  c.jit = nullptr;
  c.jit_smem.clear();
  for (Level& L : c.prog.levels)
    for (int side = 0; side < 2; ++side)
      for (PassPlan& pp : L.passes[side]) pp.jit_index = -1;
  if (!c.use_jit || c.kernel_version != 2 || (c.precision != GS_C64 && !c.jit_c128)) {
    c.jit_status = "off";
    return;
  }
  // one kernel per eligible pass
  std::vector<PassPlan*> order;
  for (Level& L : c.prog.levels)
    for (int side = 0; side < 2; ++side)
      for (PassPlan& pp : L.passes[side])
        if ((pp.M == 5 || pp.M == 4) && !pp.stages.empty()) order.push_back(&pp);
  const int n = (int)order.size();
  if (n == 0) {
    c.jit_status = "no eligible passes";
    return;
  }
  c.jit_smem.assign(n, 0);
  c.jit_loc.assign(n, {0, 0});
  c.jit_occ.assign(n, 1);
  for (PassPlan* pp : order)
    pp->pipelined = c.pipeline && c.precision == GS_C64 && !pp->fused_gather && !pp->proj_fused;
  // compile passes `ids` with a register bound for `min_blocks` CTAs/SM, in
  // chunks compiled concurrently (~source-size balanced, up to the core count)
  auto compile = [&](const std::vector<int>& ids, int min_blocks, std::string& err) -> bool {
    std::vector<std::string> kernels(ids.size());
    for (size_t t = 0; t < ids.size(); ++t) {
      PassPlan& pp = *order[ids[t]];
      size_t smem = 0;
      if (pp.proj_fused) {
        const Level& LD = c.prog.levels[pp.level];
        // (the Pauli-sibling pass: 2 CTAs/SM, 128 registers -- at the 3-CTA bound its pipelined
        // epilogue spills, measured 6% slower)
        kernels[t] = pp.pf_pauli ? jitgen::proj_pauli_kernel(c, pp, 0, smem, LD.k_hi - LD.k_lo,
                                                             min_blocks > 0 ? std::min(c.pf_min_blocks, 2) : 0)
                                 : jitgen::proj_fused_kernel(c, pp, 0, smem, c.pf_u, LD.k_hi - LD.k_lo,
                                                             min_blocks > 0 ? c.pf_min_blocks : 0);
      } else {
        kernels[t] = pp.pipelined ? jitgen::pass_kernel_pipe(c, pp, 0, smem)
                                  : jitgen::pass_kernel(c, pp, 0, smem, pp.fused_gather,
                                                        pp.M == 4 && min_blocks > 2 ? 2 : min_blocks);
      }
      c.jit_smem[ids[t]] = smem;
    }
    const int m = (int)ids.size();
    const int hw = std::max(1u, std::thread::hardware_concurrency());
    const int n_chunks = std::max(1, std::min(m, std::min(hw, 32)));
    std::vector<std::string> src(n_chunks, std::string(std::getenv("GS_STORE_CS") ? "#define GS_STCS 1\n" : "") +
                                               (c.precision == GS_C64 ? jitgen::prelude() : jitgen::prelude_dbl()));
    std::vector<std::vector<int>> members(n_chunks);
    std::vector<std::vector<std::string>> names(n_chunks);
    std::vector<size_t> load(n_chunks, 0);
    std::vector<int> by_size(m);
    for (int i = 0; i < m; ++i) by_size[i] = i;
    std::sort(by_size.begin(), by_size.end(), [&](int x, int y) { return kernels[x].size() > kernels[y].size(); });
    for (int i : by_size) {
      const int ch = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      const int local = (int)members[ch].size();
      // kernel text was generated as gsj_0: rename to its index inside the chunk
      // plus the pass's global index (profiles map launches back to passes)
      std::string k = kernels[i];
      const size_t at = k.find("gsj_0(");
      const std::string kname = "gsj_" + std::to_string(local) + "_p" + std::to_string(ids[i]);
      k.replace(at, 6, kname + "(");
      names[ch].push_back(kname);
      src[ch] += k;
      members[ch].push_back(i);
      load[ch] += k.size();
    }
    if (const char* dump = std::getenv("GS_JIT_DUMP")) {  // diagnostics: write the generated chunks
      for (int ch = 0; ch < n_chunks; ++ch)
        if (FILE* f = std::fopen((std::string(dump) + "." + std::to_string(min_blocks) + "." + std::to_string(ch) +
                                  ".cu").c_str(), "w")) {
          std::fwrite(src[ch].data(), 1, src[ch].size(), f);
          std::fclose(f);
        }
    }
    if (c.host_only) {
      size_t bytes = 0;
      for (auto& t : src) bytes += t.size();
      err = "generated " + std::to_string(m) + " kernels in " + std::to_string(n_chunks) + " modules (" +
            std::to_string(bytes) + " bytes of source); not compiled on a host-only context";
      return false;
    }
    std::vector<JitModule*> mods(n_chunks, nullptr);
    std::vector<std::string> errs(n_chunks);
    const int dev = c.device;
    std::vector<std::thread> pool;
    for (int ch = 0; ch < n_chunks; ++ch)
      pool.emplace_back([&, ch] {
        cudaSetDevice(dev);
        mods[ch] = jit_compile(src[ch], names[ch], "gridsim_passes_" + std::to_string(ch), errs[ch]);
      });
    for (auto& t : pool) t.join();
    for (int ch = 0; ch < n_chunks; ++ch)
      if (!mods[ch]) {
        for (JitModule* md : mods) jit_release(md);
        err = "interpreter (jit failed: " + errs[ch].substr(0, 300) + ")";
        return false;
      }
    for (int ch = 0; ch < n_chunks; ++ch) {
      const int mi = (int)c.jit_mods.size();
      c.jit_mods.push_back(mods[ch]);
      for (size_t k = 0; k < members[ch].size(); ++k) c.jit_loc[ids[members[ch][k]]] = {mi, (int)k};
    }
    return true;
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int> all(n);
  for (int i = 0; i < n; ++i) all[i] = i;
  std::string err;
  if (!compile(all, c.jit_min_blocks, err)) {
    for (JitModule* md : c.jit_mods) jit_release(md);
    c.jit_mods.clear();
    c.jit_status = err;
    return;
  }
  // a register bound that forces spills costs more than the occupancy it buys:
  // recompile those passes unbounded
  int n_spill = 0;
  if (c.jit_min_blocks > 0) {
    std::vector<int> spill;
    for (int i = 0; i < n; ++i)
      if (jit_local_bytes(c.jit_mods[c.jit_loc[i].first], c.jit_loc[i].second) > c.jit_spill_ok) spill.push_back(i);
    n_spill = (int)spill.size();
    if (!spill.empty() && !compile(spill, 0, err)) {
      for (JitModule* md : c.jit_mods) jit_release(md);
      c.jit_mods.clear();
      c.jit_status = err;
      return;
    }
  }
  for (int i = 0; i < n; ++i) {  // resident CTAs per SM of the persistent kernels
    if (!order[i]->pipelined) continue;
    const int regs = std::max(1, jit_num_regs(c.jit_mods[c.jit_loc[i].first], c.jit_loc[i].second));
    const int by_regs = 65536 / (256 * ((regs + 7) / 8 * 8));
    const int by_smem = (int)((228u << 10) / (c.jit_smem[i] + 1024));
    c.jit_occ[i] = std::max(1, std::min(by_regs, by_smem));
  }
  c.jit_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  c.jit = c.jit_mods[0];
  const int n_chunks = (int)c.jit_mods.size();
  for (int i = 0; i < n; ++i) order[i]->jit_index = i;
  for (PassPlan* pp : order) c.fused_active |= pp->fused_gather;
  for (PassPlan* pp : order) c.proj_fused_active |= pp->proj_fused;
  c.jit_status = "jit: " + std::to_string(n) + " pass kernels (" + std::to_string(n_spill) +
                 " recompiled without the register bound), " + std::to_string(n_chunks) + " modules compiled in " +
                 std::to_string(c.jit_seconds) + " s";
}

static void upload_program(Ctx& c) {
  if (c.host_only) {
    jit_program(c);
    return;
  }
  upload(c, c.d_ops, c.host_devops);
  upload(c, c.d_prims, c.host_prims);
  upload(c, c.d_pstages, c.host_pstages);
  upload(c, c.d_pxtable, c.host_pxtable);
  upload(c, c.d_tbtab, c.host_tbtab);
  upload(c, c.d_gofftab, c.host_gofftab);
  if (c.precision == GS_C64) {
    std::vector<float> f(c.host_params.begin(), c.host_params.end());
    upload(c, c.d_params, f);
  } else {
    upload(c, c.d_params, c.host_params);
  }
  {  // leaf tails evaluated in the gather
    TailProgD tp[2];
    std::memset(tp, 0, sizeof tp);
    for (int side = 0; side < 2; ++side) {
      const auto& T = c.tail_bits[side];
      tp[side].t = (int)T.size();
      for (size_t k = 0; k < T.size(); ++k) tp[side].tb[k] = T[k];
      tp[side].n_ops = (int)c.tail_ops[side].size();
      for (size_t o = 0; o < c.tail_ops[side].size(); ++o) {
        const HostOp& op = c.tail_ops[side][o];
        TailOpD& d = tp[side].ops[o];
        auto kidx = [&](int b) {
          const auto it = std::find(T.begin(), T.end(), b);
          return it == T.end() ? -1 : (int)(it - T.begin());
        };
        d.kind = op.kind == K_MAT1 ? 0 : op.kind == K_DIAG1 ? 1 : op.kind == K_DIAG2 ? 2 : 3;
        d.s0 = op.s0, d.s1 = op.s1;
        d.k0 = kidx(op.s0), d.k1 = op.s1 >= 0 ? kidx(op.s1) : -1;
        const int64_t n = coef_entries(op.kind);
        for (int64_t e = 0; e < 2 * n; ++e) d.u[e] = c.prog.coef[2 * op.coef + e];
      }
    }
    CK(cudaMemcpyToSymbol(g_tail, tp, sizeof tp));
  }

  upload(c, c.d_xtable, c.prog.xtable);
  if (c.precision == GS_C64) {
    std::vector<float> f(c.prog.coef.begin(), c.prog.coef.end());
    upload(c, c.d_coef, f);
  } else {
    upload(c, c.d_coef, c.prog.coef);
  }
  jit_program(c);
  if (c.pauli.ok && !c.proj_fused_active) {
    // the Pauli-sibling pass exists only as a specialised kernel: without it, plan the grouped-store leaf
    c.pauli_blocked = true;
    schedule_program(c);
    upload_program(c);
    return;
  }
  {  // projected leaf side
    ProjProgD pj;
    std::memset(&pj, 0, sizeof pj);
    pj.side = std::max(0, c.proj_side);
    if (c.proj_side >= 0) {
      const Program& p = c.prog;
      const int side = c.proj_side;
      const Level& L = p.levels.back();
      pj.n = L.k_hi - L.k_lo;
      for (int k = L.k_lo; k < L.k_hi; ++k) {
        const int j = k - L.k_lo;
        const int sb = p.q[side] - 1 - p.xq[side][k];
        pj.s[j] = sb;
        for (int d = 0; d < p.radix[k]; ++d) {
          const double* x = &p.coef[2 * (size_t)p.xtable[p.xtab[side][k] + d]];
          const int v = (x[2] != 0.0 || x[3] != 0.0) ? 1 : 0;
          pj.v[j][d] = v;
          pj.a[j][d][0] = x[2 * v];
          pj.a[j][d][1] = x[2 * v + 1];
        }
        double U[8] = {1, 0, 0, 0, 0, 0, 1, 0};  // U <- u * U for the qubit's ops in order
        for (const HostOp& op : L.ops[side]) {
          if (op.cross >= 0 || op.s0 != sb) continue;
          const double* cf = &p.coef[2 * (size_t)op.coef];
          double u[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (op.kind == K_MAT1) {
            for (int e = 0; e < 8; ++e) u[e] = cf[e];
          } else {  // diag1
            u[0] = cf[0], u[1] = cf[1], u[6] = cf[2], u[7] = cf[3];
          }
          double r[8];
          for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
              double re = 0, im = 0;
              for (int m = 0; m < 2; ++m) {
                const double ur = u[2 * (2 * a + m)], ui = u[2 * (2 * a + m) + 1];
                const double vr = U[2 * (2 * m + b)], vi = U[2 * (2 * m + b) + 1];
                re += ur * vr - ui * vi;
                im += ur * vi + ui * vr;
              }
              r[2 * (2 * a + b)] = re, r[2 * (2 * a + b) + 1] = im;
            }
          std::memcpy(U, r, sizeof U);
        }
        std::memcpy(pj.u[j], U, sizeof U);
      }
    }
    // the permuted parent layout needs the specialised kernel of that pass
    if (c.proj_perm_pass && c.proj_perm_pass->jit_index < 0) {
      c.proj_perm_pass->store_perm.clear();
      c.proj_swaps.clear();
      c.proj_perm_pass = nullptr;
    }
    pj.n_swap = (int)c.proj_swaps.size();
    for (size_t k = 0; k < c.proj_swaps.size() && k < 4; ++k) pj.sa[k] = c.proj_swaps[k].first, pj.sb[k] = c.proj_swaps[k].second;
    for (int k = 0; k < pj.n && k < 8; ++k) {  // address bit of each cross qubit (swaps applied)
      int b = pj.s[k];
      for (int w = 0; w < pj.n_swap; ++w)
        if (b == pj.sa[w]) b = pj.sb[w];
        else if (b == pj.sb[w]) b = pj.sa[w];
      pj.abit[k] = b;
    }
    c.proj_fast = false;
    if (c.proj_side >= 0 && pj.n >= c.group_log) {
      const Level& L = c.prog.levels.back();
      c.proj_fast = true;
      for (int b = 0; b < c.group_log; ++b) {
        const int j = pj.n - 1 - b;
        c.proj_fast = c.proj_fast && c.prog.radix[L.k_lo + j] == 2 && pj.v[j][0] == 0 && pj.v[j][1] == 1;
      }
    }
    CK(cudaMemcpyToSymbol(g_proj, &pj, sizeof pj));
    c.d_proj.ensure(sizeof pj);
    CK(cudaMemcpy(c.d_proj.p, &pj, sizeof pj, cudaMemcpyHostToDevice));
  }
  if (c.pauli.ok && c.proj_side >= 0) {  // Pauli-sibling pass: the frame in tile-bit / park-address coordinates
    PauliProgD pd;
    std::memset(&pd, 0, sizeof pd);
    const Program& p = c.prog;
    const int side = 1 - c.proj_side;
    const PassPlan& pp = p.levels.back().passes[side].back();
    std::vector<int> tpos(p.q[side], -1);
    for (int j = 0; j < pp.k; ++j) tpos[pp.lbits[j]] = j;
    pd.nk = c.pauli.nk;
    for (int j = 0; j < pd.nk; ++j) {
      pd.order[j] = c.pauli.order[j];
      pd.a[j] = c.pauli.a[j];
      for (int d = 0; d < 16; ++d) {
        pd.zsel[j][d] = c.pauli.zsel[j][d];
        pd.x0[j][d][0] = c.pauli.x0[j][d][0];
        pd.x0[j][d][1] = c.pauli.x0[j][d][1];
      }
      for (int b = 0; b < p.q[side]; ++b) {
        if ((c.pauli.f[j] >> b) & 1u) pd.f[j] |= 1u << tpos[b], pd.lf[j] ^= c.pauli_lcol[tpos[b]];
        if ((c.pauli.z[j] >> b) & 1u) pd.z[j] |= 1u << tpos[b], pd.lz[j] ^= c.pauli_lit[tpos[b]];
      }
    }
    for (int j = 0; j < 16; ++j) pd.lcol[j] = c.pauli_lcol[j];
    CK(cudaMemcpyToSymbol(g_pauli, &pd, sizeof pd));
  }
}

// ---------------------------------------------------------------------------
// tree enumeration

static int64_t level_fanout(const Program& p, int l) {
  int64_t f = 1;
  for (int k = p.levels[l].k_lo; k < p.levels[l].k_hi; ++k) f *= p.radix[k];
  return f;
}

// mixed-radix level digit value -> packed nibbles (gate k_lo + j at bits 4j)
static uint64_t pack_level_digits(const Program& p, int l, int64_t v) {
  const Level& L = p.levels[l];
  if (v < (int64_t)L.packed.size()) return L.packed[v];
  uint64_t out = 0;
  for (int k = L.k_hi - 1; k >= L.k_lo; --k) {
    out |= (uint64_t)(v % p.radix[k]) << (4 * (k - L.k_lo));
    v /= p.radix[k];
  }
  return out;
}

// children of `parents` (level l) at level l+1, appended to `out` in leaf order
static void enumerate_children(Ctx& c, int l, const Node* parents, int64_t n_par,
                               std::vector<Node>& out) {
  const Program& p = c.prog;
  const int e0 = c.lvl_end[l], e1 = c.lvl_end[l + 1];
  const int xp = c.x_p;
  const std::vector<int64_t>& pre = c.prefixes;
  for (int64_t s = 0; s < n_par; ++s) {
    const Node& N = parents[s];
    if (e1 <= xp) {
      const int64_t S = c.S_p[e1];
      const int64_t F = level_fanout(p, l + 1);
      int64_t i = N.i0;
      while (i < N.i1) {
        const int64_t ck = pre[i] / S;
        const int64_t lim = (ck + 1) * S;  // first prefix value of the next child
        const int64_t j = std::lower_bound(pre.begin() + i, pre.begin() + N.i1, lim) - pre.begin();
        Node ch{i, j, ck, 0, N.b0, N.b1, pack_level_digits(p, l + 1, ck - N.key * F), (int32_t)s};
        out.push_back(ch);
        i = j;
      }
    } else {
      const int kb0 = std::max(e0, xp);
      int64_t Fb = 1;
      for (int k = kb0; k < e1; ++k) Fb *= p.radix[k];
      const int64_t Sb = c.S_b[e1];
      int64_t lo = std::max(N.bkey * Fb, N.b0 / Sb);
      int64_t hi = std::min((N.bkey + 1) * Fb - 1, (N.b1 - 1) / Sb);
      for (int64_t i = N.i0; i < N.i1; ++i) {
        const int64_t vp = (e0 < xp) ? (pre[i] % c.S_p[e0]) : 0;
        for (int64_t cb = lo; cb <= hi; ++cb) {
          const int64_t b0 = std::max(cb * Sb, N.b0), b1 = std::min((cb + 1) * Sb, N.b1);
          if (b0 >= b1) continue;
          Node ch{i, i + 1, pre[i], cb, b0, b1, pack_level_digits(p, l + 1, vp * Fb + (cb - N.bkey * Fb)), (int32_t)s};
          out.push_back(ch);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launches

static void launch_check(const char* what, int64_t blocks, int threads, size_t smem) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw GsError(GS_ERR_CUDA, std::string(what) + " launch (" + std::to_string(blocks) + " blocks x " +
                                   std::to_string(threads) + " threads, " + std::to_string(smem) +
                                   " B smem): " + cudaGetErrorString(e));
}

template <typename R>
static void launch_pass(Ctx& c, int side, const PassPlan& pp, const void* src, void* dst,
                        const int32_t* parent, const uint64_t* digit, int64_t n_states,
                        bool init_zero) {
  const int q = c.prog.q[side];
  PassArgs a{};
  a.src = src;
  a.dst = dst;
  a.parent = parent;
  a.digit = reinterpret_cast<const unsigned long long*>(digit);
  a.ops = reinterpret_cast<const DevOp*>(c.d_ops.p) + pp.dev_op_offset;
  a.coefs = c.d_coef.p;
  a.xtable = reinterpret_cast<const int32_t*>(c.d_xtable.p);
  a.state_elems = 1LL << q;
  a.n_ops = (int)pp.ops.size();
  a.k = pp.k;
  int cc = 0;
  while (cc < pp.k && pp.lbits[cc] == cc) ++cc;
  a.c = std::min(cc, 8);
  a.tiles_log = q - pp.k;
  a.init_zero = init_zero ? 1 : 0;
  a.n_hi = 1 << (pp.k - a.c);
  for (int j = 0; j < pp.k; ++j) a.lbits[j] = pp.lbits[j];
  for (int j = 0; j < (int)pp.gbits.size(); ++j) a.gbits[j] = pp.gbits[j];
  const int E = 1 << pp.k;
  const int threads = std::max(32, std::min(256, E / 2));
  const size_t smem = (size_t)E * c.esize() + (size_t)a.n_hi * sizeof(int);
  const int64_t blocks = n_states << a.tiles_log;
  if (blocks > INT32_MAX) throw GsError(GS_ERR_ARG, "grid too large");
  c.st.n_pass_launches++;
  c.st.n_launches++;
  c.st.pass_bytes += 2.0 * (double)n_states * (double)(1LL << q) * (double)c.esize();
  c.st.pass_amp_updates += (double)n_states * (double)(1LL << q);
  if (c.host_only) return;
  gate_pass_kernel<R><<<(unsigned)blocks, threads, smem, c.stream>>>(a);
  launch_check("gate_pass_kernel", blocks, threads, smem);
}

template <typename R, int M>
static void launch_pass2_m(Ctx& c, const Pass2Args& a, int64_t blocks, int threads, size_t smem) {
  const cudaError_t e = launch_pass2_kernel(sizeof(R) == 4 ? 0 : 1, M, a, (unsigned)blocks, threads, smem, c.stream);
  if (e != cudaSuccess) cudaGetLastError();
  if (e != cudaSuccess)
    throw GsError(GS_ERR_CUDA, "pass2_kernel launch (" + std::to_string(blocks) + " blocks x " +
                                   std::to_string(threads) + " threads, " + std::to_string(smem) +
                                   " B smem): " + cudaGetErrorString(e));
}

template <typename R>
static void launch_pass2(Ctx& c, int side, const PassPlan& pp, const void* src, void* dst,
                         const int32_t* parent, const uint64_t* digit, int64_t n_states,
                         bool init_zero) {
  const int q = c.prog.q[side];
  Pass2Args a{};
  a.src = src;
  a.dst = dst;
  a.parent = parent;
  a.digits = reinterpret_cast<const unsigned long long*>(digit);
  a.prims = reinterpret_cast<const PPrim*>(c.d_prims.p);
  a.params = c.d_params.p;
  a.pxtable = reinterpret_cast<const int32_t*>(c.d_pxtable.p);
  a.stages = reinterpret_cast<const PStage*>(c.d_pstages.p) + pp.dev_stage_offset;
  a.coefs = c.d_coef.p;
  a.xtable = reinterpret_cast<const int32_t*>(c.d_xtable.p);
  a.state_elems = 1LL << q;
  a.n_states = n_states;
  a.store_scale = pp.store_scale;
  a.n_stages = (int)pp.stages.size();
  a.kq = pp.k;
  const int slots = pp.K - pp.k;
  a.K = pp.K;
  int cc = 0;
  while (cc < pp.k && pp.lbits[cc] == cc) ++cc;
  a.c = std::min(cc, 10);
  a.tiles_log = q - pp.k;
  a.init_zero = init_zero ? 1 : 0;
  a.n_hi = 1 << (pp.k - a.c);
  a.out_group_log = pp.grouped_store ? c.group_log : 0;
  a.stage0 = (int)pp.dev_stage_offset;
  a.tbtab = reinterpret_cast<const uint16_t*>(c.d_tbtab.p);
  a.gofftab = reinterpret_cast<const uint32_t*>(c.d_gofftab.p) + pp.goff_offset;
  if (q > 31) throw GsError(GS_ERR_ARG, "half-states beyond 2^31 amplitudes are not supported");
  if (pp.grouped_store && pp.K - pp.k != c.group_log)
    throw GsError(GS_ERR_ARG, "grouped store needs group_log slot bits");
  if (!c.host_only && pp.grouped_store && pp.jit_index < 0 && !pp.stages.empty())
    for (int b : pp.stages.back().rb)
      if (b >= pp.k)  // the interpreter keeps slot bits on threads
        throw GsError(GS_ERR_ARG, "16-byte grouped store needs the specialised kernel (set slot_store16=0)");
  for (int j = 0; j < pp.k; ++j) a.lbits[j] = pp.lbits[j];
  for (int j = 0; j < (int)pp.gbits.size(); ++j) a.gbits[j] = pp.gbits[j];
  const int threads = 1 << (a.K - pp.M);
  const size_t smem = ((size_t)1 << a.K) * c.esize();
  // (a Pauli-sibling pass evolves one base state per 8-leaf group)
  const int64_t groups = pp.pf_pauli ? (n_states + 7) >> 3 : (n_states + (1LL << slots) - 1) >> slots;
  const int64_t blocks = groups << a.tiles_log;
  if (blocks > INT32_MAX) throw GsError(GS_ERR_ARG, "grid too large");
  c.st.n_pass_launches++;
  c.st.n_launches++;
  c.st.pass_bytes += 2.0 * (double)n_states * (double)(1LL << q) * (double)c.esize();
  c.st.pass_amp_updates += (double)n_states * (double)(1LL << q);
  if (c.host_only) return;
  if (pp.jit_index >= 0 && c.jit) {
    JArgs j{};
    j.src = src;
    j.dst = dst;
    j.parent = parent;
    j.digits = reinterpret_cast<const unsigned long long*>(digit);
    j.params = c.d_params.p;
    j.pxtable = reinterpret_cast<const int32_t*>(c.d_pxtable.p);
    j.coefs = c.d_coef.p;
    j.state_elems = 1LL << q;
    j.n_states = n_states;
    j.init_zero = init_zero ? 1 : 0;
    j.uni_p0 = c.uni_p0;
    if (pp.fused_gather) {
      j.aleaf = c.leaf_out[0].p;
      j.ia = reinterpret_cast<const int32_t*>(c.d_bia.p);  // A index per bucket slot
      j.weights = c.cur_weights;
      j.bstart = reinterpret_cast<const int32_t*>(c.d_bstart.p);
      j.breq = reinterpret_cast<const int32_t*>(c.d_breq.p);
      j.btl = reinterpret_cast<const int32_t*>(c.d_btl.p);
      j.partial = c.d_partial.p;
      j.n_req = c.n_req;
      j.a_elems = 1LL << c.prog.q[0];
    }
    std::string err;
    const size_t jsm = c.jit_smem[pp.jit_index];
    const auto loc = c.jit_loc[pp.jit_index];
    int64_t grid = blocks;
    if (pp.proj_fused) {  // fused projected-leaf pass: the group's factor table, then the pass
      const int ps = c.proj_side;
      const int D = (int)c.prog.levels.size() - 1;
      const int nk = c.prog.levels[D].k_hi - c.prog.levels[D].k_lo;
      const int64_t ng = (n_states + 7) >> 3;
      const int64_t gpc = pp.pf_pauli ? std::max(1, c.pf_groups) : 1;  // groups per CTA = per partial row
      c.pf_rows = (ng + gpc - 1) / gpc;
      if (pp.pf_pauli) grid = c.pf_rows << a.tiles_log;
      if (c.n_req <= 0) return;
      c.d_pftab.ensure((size_t)ng * ((size_t)8 << nk) * sizeof(float2));
      c.d_pfaoff.ensure((size_t)ng * 8 * sizeof(long long));
      c.d_partial.ensure(std::max<size_t>((size_t)c.pf_rows * (size_t)c.n_req * sizeof(double2), 16));
      const void* P = (ps == 0 ? c.lvl_a : c.lvl_b)[D - 1].p;
      if (pp.pf_pauli) {
        c.d_pfbflip.ensure((size_t)ng * 8 * sizeof(unsigned));
        pf_table_pauli_kernel<<<(unsigned)ng, 256, 0, c.stream>>>(
            reinterpret_cast<const unsigned long long*>(digit), c.cur_parent, c.cur_weights, n_states,
            1LL << c.prog.q[ps], reinterpret_cast<float2*>(c.d_pftab.p),
            reinterpret_cast<long long*>(c.d_pfaoff.p), reinterpret_cast<unsigned*>(c.d_pfbflip.p));
        j.pf_bflip = reinterpret_cast<const unsigned*>(c.d_pfbflip.p);
      } else {
        pf_table_kernel<<<(unsigned)ng, 256, 0, c.stream>>>(reinterpret_cast<const unsigned long long*>(digit),
                                                          c.cur_parent, c.cur_weights, n_states,
                                                          1LL << c.prog.q[ps],
                                                          reinterpret_cast<float2*>(c.d_pftab.p),
                                                          reinterpret_cast<long long*>(c.d_pfaoff.p));
      }
      launch_check("pf_table_kernel", ng, 256, 0);
      c.st.n_launches++;
      j.bstart = reinterpret_cast<const int32_t*>(c.d_bstart.p);
      j.partial = c.d_partial.p;
      j.n_req = c.n_req;
      j.pf_parents = P;
      j.pf_tab = c.d_pftab.p;
      j.pf_aoff = reinterpret_cast<const long long*>(c.d_pfaoff.p);
      j.pf_meta = c.d_bmeta.p;
    }
    if (pp.pipelined) {  // persistent: the CTAs loop over the tiles
      j.n_ctas = blocks;
      grid = std::min<int64_t>(blocks, (int64_t)c.n_sm * c.jit_occ[pp.jit_index]);
    }
    if (jit_launch(c.jit_mods[loc.first], loc.second, (unsigned)grid, threads, jsm, c.stream, j, err) !=
        cudaSuccess)
      throw GsError(GS_ERR_CUDA, "jit pass launch: " + err);
    return;
  }
  if (pp.M == 5) {
    if constexpr (sizeof(R) == 4) launch_pass2_m<R, 5>(c, a, blocks, threads, smem);
  } else {
    launch_pass2_m<R, 4>(c, a, blocks, threads, smem);
  }
}

struct Timer {
  Ctx& c;
  double* acc;
  cudaEvent_t a = nullptr, b = nullptr;
  Timer(Ctx& cc, double* ac) : c(cc), acc(ac) {
    if (acc && c.profile && !c.host_only) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, c.stream);
    }
  }
  ~Timer() {
    if (a) {
      cudaEventRecord(b, c.stream);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      *acc += ms;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  }
};

template <typename R>
static void run_level_passes(Ctx& c, int l, int64_t n, const void* src_a, const void* src_b,
                             void* dst_a, void* dst_b, const int32_t* parent,
                             const uint64_t* digit, bool root, int64_t n_parents = 1) {
  Timer t(c, &c.st.ms_pass);
  const Level& L = c.prog.levels[l];
  const int D = (int)c.prog.levels.size() - 1;
  Timer tl(c, l == D ? &c.st.ms_leaf : nullptr);
  // roofline basis: what these passes must move (parents read once, states written once)
  for (int side = 0; side < 2; ++side) {
    const double sb = (double)(1LL << c.prog.q[side]) * (double)c.esize();
    if (c.prog.q[side] == 0 || (l == D && side == c.proj_side)) {
      if (l == D && side == c.proj_side) c.st.leaf_bytes_alg += (double)n_parents * sb;  // parents, read once
      continue;
    }
    double b = 0;
    const double ns = (l == D && side == c.psib_side) ? (double)c.cur_npar : (double)n;  // states this side writes
    for (size_t i = 0; i < L.passes[side].size(); ++i) {
      const PassPlan& pp = L.passes[side][i];
      const double rd = i == 0 ? (root ? 0.0 : (double)n_parents * sb) : ns * sb;
      const double wr = (pp.proj_fused && c.proj_fused_active) ? 0.0 : ns * sb;
      b += rd + wr;
      if (l == D) c.st.n_leaf_launches++;
    }
    (l == D ? c.st.leaf_bytes_alg : c.st.upper_bytes_alg) += b;
  }
  const void* srcs[2] = {src_a, src_b};
  void* dsts[2] = {dst_a, dst_b};
  for (int side = 0; side < 2; ++side) {
    bool first = true;
    for (const PassPlan& pp : L.passes[side]) {
      c.tick("pass launch");
      void* out = pp.grouped_store ? (c.leaf_sel[side] ? c.leaf_sel[side] : c.leaf_out[side].p) : dsts[side];
      if (l == D && side == c.psib_side && D >= 1) {
        // Pauli-sibling side: one base state per distinct parent of the chunk, no cross terms
        const int64_t keep = c.uni_p0;
        c.uni_p0 = -1;
        launch_pass2<R>(c, side, pp, first ? srcs[side] : dsts[side], out, first ? c.cur_upar : nullptr, nullptr,
                        c.cur_npar, false);
        c.uni_p0 = keep;
      } else if (c.kernel_version == 2 && pp.M > 0)
        launch_pass2<R>(c, side, pp, first ? srcs[side] : dsts[side], out,
                        first ? parent : nullptr, digit, n, root && first);
      else
        launch_pass<R>(c, side, pp, first ? srcs[side] : dsts[side], dsts[side],
                       first ? parent : nullptr, digit, n, root && first);
      first = false;
    }
  }
  c.st.n_nodes += n;
  for (int side = 0; side < 2; ++side)
    c.st.pass_bytes_min += 2.0 * (double)n * (double)(1LL << c.prog.q[side]) * (double)c.esize();
}

// leaf multiplicities (duplicate prefixes / branch ranges collapsed into one node)
static void upload_weights(Ctx& c, const Node* nodes, int64_t n) {
  if (c.host_only || n == 0) return;
  const size_t off = c.ring.alloc(n * sizeof(double));
  double* w = reinterpret_cast<double*>(c.ring.h(off));
  for (int64_t j = 0; j < n; ++j) w[j] = (double)((nodes[j].i1 - nodes[j].i0) * (nodes[j].b1 - nodes[j].b0));
  c.ring.commit(off, n * sizeof(double), c.stream);
  c.cur_weights = reinterpret_cast<const double*>(c.ring.d(off));
  c.st.h2d_bytes += 8.0 * n;
  if (c.fused_active) {  // partials of the fused leaf gather, one row per group of 8 leaves
    const size_t groups = (size_t)((n + 7) / 8);
    c.d_partial.ensure(std::max<size_t>(groups * (size_t)std::max<int64_t>(c.n_req, 1) * sizeof(double2), 16));
  }
}

// Sort the split requests by their A index on stream `s` (radix sort of
// (ia, slot) pairs + a gather of ib): the HBM gathers then read A runs in
// ascending address order.  Results are unchanged -- every request's
// partials are the same numbers, folded back to its slot by reduce_kernel.
static void sort_requests(Ctx& c, cudaStream_t s) {
  c.req_sorted = false;
  const int64_t n = c.n_req;
  if (c.host_only || !c.sort_requests || n < 1024 || n > INT32_MAX) return;
  c.d_ia_s.ensure((size_t)n * 4);
  c.d_ib_s.ensure((size_t)n * 4);
  c.d_perm.ensure((size_t)n * 4);
  c.d_iota.ensure((size_t)n * 4);
  const unsigned blocks = (unsigned)((n + 255) / 256);
  iota_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<int32_t*>(c.d_iota.p), n);
  const uint32_t* kin = reinterpret_cast<const uint32_t*>(c.d_ia.p);
  uint32_t* kout = reinterpret_cast<uint32_t*>(c.d_ia_s.p);
  const int32_t* vin = reinterpret_cast<const int32_t*>(c.d_iota.p);
  int32_t* vout = reinterpret_cast<int32_t*>(c.d_perm.p);
  const int end_bit = std::max(1, c.prog.q[0]);
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit, s));
  c.d_sorttmp.ensure(std::max<size_t>(tmp, 16));
  CK(cub::DeviceRadixSort::SortPairs(c.d_sorttmp.p, tmp, kin, kout, vin, vout, (int)n, 0, end_bit, s));
  permute_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const int32_t*>(c.d_ib.p), vout,
                                        reinterpret_cast<int32_t*>(c.d_ib_s.p), n);
  CK(cudaGetLastError());
  c.req_sorted = true;
  c.st.n_launches += 3;
}

// Complete the requests staged by gs_run_batched: join the host copies, then
// upload + split on the side stream -- ordered after this run's start, so an
// earlier queued run is done with the request buffers -- and make the run's
// stream wait for the split before its first gather.
static void finish_requests(Ctx& c) {
  if (!c.pend.active) return;
  c.pend.active = false;
  c.pend.join();
  for (char b : c.pend.bad)
    if (b) {
      c.n_req = -1;
      throw GsError(GS_ERR_INDEX, "request index outside the state space");
    }
  const int64_t n = c.pend.n;
  if (c.host_only || n == 0) return;
  CK(cudaStreamWaitEvent(c.side_stream, c.ev0, 0));
  CK(cudaMemcpyAsync(c.d_gidx.p, c.req_stage.p, n * 8, cudaMemcpyHostToDevice, c.side_stream));
  split_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c.side_stream>>>(
      reinterpret_cast<const long long*>(c.d_gidx.p), n, c.pend.runs, reinterpret_cast<int32_t*>(c.d_ia.p),
      reinterpret_cast<int32_t*>(c.d_ib.p), c.pend.packed ? reinterpret_cast<uint32_t*>(c.d_packed.p) : nullptr);
  CK(cudaGetLastError());
  sort_requests(c, c.side_stream);
  CK(cudaEventRecord(c.req_done, c.side_stream));
  CK(cudaStreamWaitEvent(c.stream, c.req_done, 0));
  if (c.gstream) CK(cudaStreamWaitEvent(c.gstream, c.req_done, 0));
  c.st.h2d_bytes += 8.0 * n;
  c.st.n_launches += 1;
}

template <typename R> static void gather(Ctx& c, int l, const Node* nodes, int64_t n) {
  int64_t w_total = 0;
  for (int64_t j = 0; j < n; ++j) w_total += (nodes[j].i1 - nodes[j].i0) * (nodes[j].b1 - nodes[j].b0);
  c.st.n_paths += w_total;
  finish_requests(c);
  if (c.host_only || c.n_req == 0) return;
  c.tick("gather");
  Timer t(c, &c.st.ms_gather);
  const int64_t nreq = c.n_req;
  if (c.proj_fused_active) {  // partials were written by the fused projected-leaf pass
    const int threads = 256;
    const int64_t xblocks = (nreq + threads - 1) / threads;
    const double ar = c.kfinal[0][0], ai = c.kfinal[0][1], br = c.kfinal[1][0], bi = c.kfinal[1][1];
    const double2 kf = make_double2(ar * br - ai * bi, ar * bi + ai * br);
    // partials are in bucket order: fold them back to request order through breq
    reduce_kernel<<<(unsigned)xblocks, threads, 0, c.stream>>>(reinterpret_cast<const double2*>(c.d_partial.p),
                                                                (int)c.pf_rows, nreq, kf,
                                                                reinterpret_cast<double2*>(c.d_acc.p),
                                                                reinterpret_cast<const int32_t*>(c.d_breq.p));
    launch_check("reduce_kernel", xblocks, threads, 0);
    c.st.n_gather_launches += 1;
    c.st.n_launches += 1;
    // the fused pass wrote one fp64 partial per (request, leaf group); the fold reads them once
    c.st.leaf_bytes_alg += 16.0 * (double)c.pf_rows * (double)nreq;
    c.st.gather_bytes += 16.0 * (double)c.pf_rows * (double)nreq + 32.0 * nreq;
    return;
  }
  if (c.fused_active) {  // partials were written by the fused leaf pass
    const int threads = 256;
    const int64_t xblocks = (nreq + threads - 1) / threads;
    const int64_t groups = (n + 7) / 8;
    const double ar = c.kfinal[0][0], ai = c.kfinal[0][1], br = c.kfinal[1][0], bi = c.kfinal[1][1];
    const double2 kf = make_double2(ar * br - ai * bi, ar * bi + ai * br);
    reduce_kernel<<<(unsigned)xblocks, threads, 0, c.stream>>>(reinterpret_cast<const double2*>(c.d_partial.p),
                                                                (int)groups, nreq, kf,
                                                                reinterpret_cast<double2*>(c.d_acc.p), nullptr);
    launch_check("reduce_kernel", xblocks, threads, 0);
    c.st.n_gather_launches += 1;
    c.st.n_launches += 1;
    c.st.gather_bytes += (double)n * (double)nreq * 2.0 * (double)c.esize() + 32.0 * nreq;
    return;
  }
  const int threads = 256;
  const int64_t xblocks = (nreq + threads - 1) / threads;
  // enough leaf groups to fill the GPU, bounded by the partial buffer
  int64_t groups = std::max<int64_t>(1, (148 * 16) / std::max<int64_t>(1, xblocks));
  groups = std::min<int64_t>(groups, n);
  const int64_t max_groups = std::max<int64_t>(1, (256LL << 20) / (16 * std::max<int64_t>(1, nreq)));
  groups = std::min(groups, max_groups);
  groups = std::min<int64_t>(groups, 65535);
  const int64_t per = (n + groups - 1) / groups;
  groups = (n + per - 1) / per;
  c.d_partial.ensure((size_t)groups * nreq * sizeof(double2));
  const int qa = c.prog.q[0], qb = c.prog.q[1];
  const size_t pair_bytes = ((size_t)1 << qa) * c.esize() + ((size_t)1 << qb) * c.esize();
  bool used_sorted = false;
  const int32_t* g_ia = reinterpret_cast<const int32_t*>(c.d_ia.p);
  const int32_t* g_ib = reinterpret_cast<const int32_t*>(c.d_ib.p);
  const bool smem_path = !c.grouped_leaf && c.smem_gather && 2 * pair_bytes <= 200 * 1024 && qa + qb <= 31 &&
                         qa >= 2 && qb >= 2;
  if (c.req_sorted && !smem_path) {  // HBM gathers read A runs in ascending order
    g_ia = reinterpret_cast<const int32_t*>(c.d_ia_s.p);
    g_ib = reinterpret_cast<const int32_t*>(c.d_ib_s.p);
    used_sorted = true;
  }
  cudaStream_t gsm = c.stream;  // stream of this gather's kernels
  DevBuf* pbuf = &c.d_partial;
  if (c.grouped_leaf) {
    if (c.gs) gsm = c.gs;
    if (c.part_sel) pbuf = c.part_sel;
    void* const lf[2] = {c.leaf_sel[0] ? c.leaf_sel[0] : c.leaf_out[0].p,
                         c.leaf_sel[1] ? c.leaf_sel[1] : c.leaf_out[1].p};
    const int GL = c.group_log;
    const int64_t ng = (n + (1 << GL) - 1) >> GL;
    int64_t gy = std::max<int64_t>(1, (148 * 16) / std::max<int64_t>(1, xblocks));
    // option gather_gpy: groups per y-block (all requests sweep a few groups at a
    // time, whose parents then stay in L2), bounded by 2 GiB of partials
    if (c.gather_gpy > 0)
      gy = std::min<int64_t>((ng + c.gather_gpy - 1) / c.gather_gpy,
                             std::max<int64_t>(1, (2LL << 30) / (16 * std::max<int64_t>(1, nreq))));
    gy = std::min<int64_t>(gy, ng);
    if (c.gather_gpy <= 0)
      gy = std::min<int64_t>(gy, std::max<int64_t>(1, (256LL << 20) / (16 * std::max<int64_t>(1, nreq))));
    const int64_t per_y = (ng + gy - 1) / gy;
    gy = (ng + per_y - 1) / per_y;
    pbuf->ensure((size_t)gy * nreq * sizeof(double2));
    if (c.proj_side >= 0) {  // one side's leaves come from its parent state
      const int ps = c.proj_side;
      const void* P = (ps == 0 ? c.lvl_a : c.lvl_b)[l - 1].p;
      // lanes per request: 4 (two leaves per lane) or 8 (one, option proj_lanes)
      const int lpr = (c.proj_lanes == 8 && GL >= 3) ? 8 : 4;
      auto pk = lpr == 8 ? (GL == 4 ? gather_proj_kernel<R, 4, 8> : gather_proj_kernel<R, 3, 8>)
                         : (GL == 4 ? gather_proj_kernel<R, 4, 4>
                                    : GL == 3 ? gather_proj_kernel<R, 3, 4> : gather_proj_kernel<R, 2, 4>);
      const int64_t gxb = (lpr * nreq + threads - 1) / threads;
      pk<<<dim3((unsigned)gxb, (unsigned)gy), threads, 0, gsm>>>(
          P, lf[1 - ps], 1LL << c.prog.q[ps], 1LL << c.prog.q[1 - ps], (int)n, (int)per_y,
          c.cur_weights, c.cur_parent, c.cur_digit, c.cur_gpar, g_ia, g_ib, nreq,
          reinterpret_cast<double2*>(pbuf->p));
      launch_check("gather_proj_kernel", gxb * gy, threads, 0);
      groups = gy;
    } else {
    auto kern = c.quad_gather
                    ? (GL == 4 ? gather_grouped4_kernel<R, 4>
                               : GL == 3 ? gather_grouped4_kernel<R, 3> : gather_grouped4_kernel<R, 2>)
                    : (GL == 4 ? gather_grouped_kernel<R, 4>
                               : GL == 3 ? gather_grouped_kernel<R, 3> : gather_grouped_kernel<R, 2>);
    const int64_t gxb = c.quad_gather ? (4 * nreq + threads - 1) / threads : xblocks;
    kern<<<dim3((unsigned)gxb, (unsigned)gy), threads, 0, gsm>>>(
        lf[0], lf[1], 1LL << qa, 1LL << qb, (int)n, (int)per_y,
        c.cur_weights, g_ia, g_ib, nreq, reinterpret_cast<double2*>(pbuf->p));
    launch_check("gather_grouped_kernel", gxb * gy, threads, 0);
    groups = gy;
    }
  } else if (smem_path) {
    // shared-memory gather: whole leaf pairs staged per CTA, requests in registers
    constexpr int RPT = 20, NT = 512;
    const int64_t req_per_cta = (int64_t)RPT * NT;
    const int64_t xb = (nreq + req_per_cta - 1) / req_per_cta;
    int64_t g = std::max<int64_t>(1, (148 + xb - 1) / xb);
    g = std::min<int64_t>(g, n);
    g = std::min<int64_t>(g, std::max<int64_t>(1, (256LL << 20) / (16 * nreq)));
    const int64_t per2 = (n + g - 1) / g;
    g = (n + per2 - 1) / per2;
    c.d_partial.ensure((size_t)g * nreq * sizeof(double2));
    static bool configured[2] = {false, false};
    if (!configured[sizeof(R) == 8]) {
      CK(cudaFuncSetAttribute(gather_smem_kernel<R, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
      configured[sizeof(R) == 8] = true;
    }
    gather_smem_kernel<R, RPT><<<dim3((unsigned)xb, (unsigned)g), NT, 2 * pair_bytes, c.stream>>>(
        c.lvl_a[l].p, c.lvl_b[l].p, qa, qb, (int)n, (int)per2,
        c.cur_weights, reinterpret_cast<const uint32_t*>(c.d_packed.p),
        nreq, (int)req_per_cta, reinterpret_cast<double2*>(c.d_partial.p));
    launch_check("gather_smem_kernel", xb * g, NT, 2 * pair_bytes);
    groups = g;
  } else if (!c.tail_ops[0].empty() || !c.tail_ops[1].empty()) {
    dim3 grid((unsigned)xblocks, (unsigned)groups);
    const int ta = (int)c.tail_bits[0].size(), tb = (int)c.tail_bits[1].size();
    const void* A = c.lvl_a[l].p;
    const void* B = c.lvl_b[l].p;
#define GS_TAIL(TA, TB)                                                                                     \
  case TA * 4 + TB:                                                                                         \
    gather_tail_kernel<R, TA, TB><<<grid, threads, 0, c.stream>>>(A, B, 1LL << qa, 1LL << qb, (int)n, (int)per, \
                                                                  c.cur_weights, g_ia, g_ib, nreq,           \
                                                                  reinterpret_cast<double2*>(c.d_partial.p), \
                                                                  reinterpret_cast<const SibD*>(c.cur_sib)); \
    break;
    switch (ta * 4 + tb) {
      GS_TAIL(0, 0) GS_TAIL(0, 1) GS_TAIL(0, 2) GS_TAIL(0, 3)
      GS_TAIL(1, 0) GS_TAIL(1, 1) GS_TAIL(1, 2) GS_TAIL(1, 3)
      GS_TAIL(2, 0) GS_TAIL(2, 1) GS_TAIL(2, 2) GS_TAIL(2, 3)
      GS_TAIL(3, 0) GS_TAIL(3, 1) GS_TAIL(3, 2) GS_TAIL(3, 3)
      default: throw GsError(GS_ERR_ARG, "leaf tail wider than 3 qubits");
    }
#undef GS_TAIL
    launch_check("gather_tail_kernel", xblocks * groups, threads, 0);
  } else {
  dim3 grid((unsigned)xblocks, (unsigned)groups);
  gather_kernel<R><<<grid, threads, 0, c.stream>>>(
      c.lvl_a[l].p, c.lvl_b[l].p, 1LL << qa, 1LL << qb, (int)n, (int)per,
      c.cur_weights, g_ia, g_ib, nreq, reinterpret_cast<double2*>(c.d_partial.p),
      reinterpret_cast<const SibD*>(c.cur_sib));
  launch_check("gather_kernel", xblocks * groups, threads, 0);
  }
  double2 kf = make_double2(1.0, 0.0);
  if (c.kernel_version == 2) {  // deferred W-form scalars of both blocks
    const double ar = c.kfinal[0][0], ai = c.kfinal[0][1], br = c.kfinal[1][0], bi = c.kfinal[1][1];
    kf = make_double2(ar * br - ai * bi, ar * bi + ai * br);
  }
  reduce_kernel<<<(unsigned)xblocks, threads, 0, gsm>>>(
      reinterpret_cast<const double2*>(pbuf->p), (int)groups, nreq, kf,
      reinterpret_cast<double2*>(c.d_acc.p), used_sorted ? reinterpret_cast<const int32_t*>(c.d_perm.p) : nullptr);
  launch_check("reduce_kernel", xblocks, threads, 0);
  c.st.n_gather_launches += 2;
  c.st.n_launches += 2;
  if (c.grouped_leaf && c.proj_side >= 0)  // per request and 8-leaf group: one 64-byte leaf run + a parent pair
    c.st.gather_bytes += (double)((n + 7) / 8) * (double)nreq * (8.0 * c.esize() + 2.0 * c.esize()) + 32.0 * nreq;
  else
    c.st.gather_bytes += (double)n * (double)nreq * 2.0 * (double)c.esize() + 32.0 * nreq;
}

static void ensure_buckets(Ctx& c);

template <typename R> static void descend(Ctx& c, int l, const Node* nodes, int64_t n_nodes) {
  const int D = (int)c.prog.levels.size() - 1;
  if (l == D) {
    gather<R>(c, l, nodes, n_nodes);
    return;
  }
  std::vector<Node>& kids = c.kids[l + 1];  // per-level scratch, reused across chunks
  kids.clear();
  c.tick("before enumerate");
  enumerate_children(c, l, nodes, n_nodes, kids);
  c.tick("enumerate_children");
  int64_t cap = c.cap[l + 1];
  // leaf chunks of whole leaf groups: sibling blocks stay aligned with the
  // grouped layout's 2^G-leaf groups across chunk boundaries
  if (l + 1 == D && c.grouped_leaf && cap >= (1 << c.group_log)) cap -= cap % (1 << c.group_log);
  auto at = [](std::vector<DevBuf>& v, int i) -> void* { return i < (int)v.size() ? v[i].p : nullptr; };
  for (int64_t s = 0; s < (int64_t)kids.size(); s += cap) {
    const int64_t n = std::min<int64_t>(cap, (int64_t)kids.size() - s);
    const Node* chunk = kids.data() + s;
    const uint64_t* d_digit = nullptr;
    const int32_t* d_parent = nullptr;
    if (!c.host_only) {
      c.tick("before ring");
      const size_t off = c.ring.alloc(n * 12);
      c.tick("ring.alloc");
      uint64_t* hd = reinterpret_cast<uint64_t*>(c.ring.h(off));
      int32_t* hp = reinterpret_cast<int32_t*>(hd + n);
      for (int64_t j = 0; j < n; ++j) hd[j] = chunk[j].digit, hp[j] = chunk[j].parent;
      c.ring.commit(off, n * 12, c.stream);
      c.tick("ring.commit");
      d_digit = reinterpret_cast<const uint64_t*>(c.ring.d(off));
      d_parent = reinterpret_cast<const int32_t*>(d_digit + n);
      c.st.h2d_bytes += 12.0 * n;
    }
    if (l + 1 == D) {
      upload_weights(c, chunk, n);  // the fused leaf pass reads them
      c.cur_parent = d_parent;      // the projected-leaf gather reads them
      c.cur_digit = reinterpret_cast<const unsigned long long*>(d_digit);
      c.cur_sib = nullptr;
      c.cur_upar = nullptr;
      c.cur_npar = 0;
      if (c.psib_side >= 0) {  // Pauli-sibling leaves: base state per distinct parent, Pauli per leaf
        const PauliFrame& pf = c.psib;
        int64_t np = 0;
        for (int64_t j = 0; j < n; ++j) np += j == 0 || chunk[j].parent != chunk[j - 1].parent;
        c.cur_npar = np;
        if (!c.host_only) {
          const size_t so = c.ring.alloc(n * sizeof(SibD) + np * 4);
          SibD* sd = reinterpret_cast<SibD*>(c.ring.h(so));
          int32_t* up = reinterpret_cast<int32_t*>(sd + n);
          int64_t r = -1;
          for (int64_t j = 0; j < n; ++j) {
            if (j == 0 || chunk[j].parent != chunk[j - 1].parent) up[++r] = chunk[j].parent;
            int a = 0;
            uint32_t f = 0, z = 0;
            double kr = 1.0, ki = 0.0;
            for (int i = 0; i < pf.nk; ++i) {
              const int g = pf.order[i];
              const int d = (int)((chunk[j].digit >> (4 * g)) & 15ull);
              const double xr = pf.x0[g][d][0], xi = pf.x0[g][d][1];
              const double tr = kr * xr - ki * xi;
              ki = kr * xi + ki * xr;
              kr = tr;
              if (pf.zsel[g][d]) {
                a += pf.a[g] + 2 * (__builtin_popcount(z & pf.f[g]) & 1);
                f ^= pf.f[g];
                z ^= pf.z[g];
              }
            }
            a += 2 * (__builtin_popcount(z & f) & 1);
            switch (a & 3) {
              case 1: { const double t = -ki; ki = kr; kr = t; } break;
              case 2: kr = -kr, ki = -ki; break;
              case 3: { const double t = ki; ki = -kr; kr = t; } break;
              default: break;
            }
            sd[j] = SibD{(int32_t)r, f, z, 0, kr, ki};
          }
          c.ring.commit(so, n * sizeof(SibD) + np * 4, c.stream);
          c.cur_sib = c.ring.d(so);
          c.cur_upar = reinterpret_cast<const int32_t*>(reinterpret_cast<const SibD*>(c.ring.d(so)) + n);
          c.st.h2d_bytes += (double)(n * sizeof(SibD) + np * 4);
        }
      }
      if (c.proj_side >= 0 && !c.host_only) {  // sibling blocks of the projected-leaf gather
        const int GL = c.group_log, W = 1 << GL;
        const Level& LD = c.prog.levels[D];
        const int nk = LD.k_hi - LD.k_lo;
        uint64_t run_mask = 0;
        for (int k = std::max(0, nk - GL); k < nk; ++k) run_mask |= 15ull << (4 * k);
        const int64_t ng = (n + W - 1) / W;
        const size_t goff = c.ring.alloc(ng * 4);
        int32_t* gp = reinterpret_cast<int32_t*>(c.ring.h(goff));
        for (int64_t g = 0; g < ng; ++g) {
          const int64_t j0 = g * W;
          bool uni = c.proj_fast && j0 + W <= n;
          for (int r = 0; uni && r < W; ++r) {
            const Node& N = chunk[j0 + r];
            uint64_t want = 0;
            for (int b = 0; b < GL; ++b) want |= (uint64_t)((r >> b) & 1) << (4 * (nk - 1 - b));
            uni = N.parent == chunk[j0].parent && (N.digit & ~run_mask) == (chunk[j0].digit & ~run_mask) &&
                  (N.digit & run_mask) == want;
          }
          gp[g] = uni ? chunk[j0].parent : -1;
        }
        c.ring.commit(goff, ng * 4, c.stream);
        c.cur_gpar = reinterpret_cast<const int32_t*>(c.ring.d(goff));
        static const bool dbg = std::getenv("GS_PROJ_DEBUG") != nullptr;
        if (dbg) {
          int64_t nu = 0;
          for (int64_t g = 0; g < ng; ++g) nu += gp[g] >= 0;
          std::fprintf(stderr, "proj gather: chunk of %lld leaves, %lld/%lld sibling blocks (fast=%d)\n",
                       (long long)n, (long long)nu, (long long)ng, (int)c.proj_fast);
        }
        c.st.h2d_bytes += 4.0 * ng;
      }
    }
    // full fan-out chunk: node j is child j % F of parent chunk[0].parent + j / F
    c.uni_p0 = -1;
    if (c.uniform_chunks) {
      const int64_t F = level_fanout(c.prog, l + 1);
      bool uni = F >= 1 && F <= 65536;
      for (int64_t j = 0; uni && j < n; ++j)
        uni = chunk[j].parent == chunk[0].parent + j / F &&
              chunk[j].digit == pack_level_digits(c.prog, l + 1, j % F);
      if (uni) c.uni_p0 = chunk[0].parent;
    }
    int f = -1;  // overlapped gather: buffer set of this leaf chunk
    if (c.ovl && l + 1 == D) {
      f = c.flip;
      c.flip ^= 1;
      CK(cudaStreamWaitEvent(c.stream, c.ev_g[f], 0));  // set f's previous gather is done
      // the gather's tables leave the staging ring for set f's own buffer
      const int64_t ng = (n + (1 << c.group_log) - 1) >> c.group_log;
      const size_t ow = 0, op = ow + 8 * (size_t)n, od = op + (((4 * (size_t)n) + 15) & ~(size_t)15),
                   og = od + 8 * (size_t)n, total = og + 4 * (size_t)ng + 16;
      c.d_tab[f].ensure(total);
      char* t = static_cast<char*>(c.d_tab[f].p);
      CK(cudaMemcpyAsync(t + ow, c.cur_weights, 8 * (size_t)n, cudaMemcpyDeviceToDevice, c.stream));
      CK(cudaMemcpyAsync(t + op, c.cur_parent, 4 * (size_t)n, cudaMemcpyDeviceToDevice, c.stream));
      CK(cudaMemcpyAsync(t + od, c.cur_digit, 8 * (size_t)n, cudaMemcpyDeviceToDevice, c.stream));
      c.cur_weights = reinterpret_cast<const double*>(t + ow);
      c.cur_parent = reinterpret_cast<const int32_t*>(t + op);
      c.cur_digit = reinterpret_cast<const unsigned long long*>(t + od);
      if (c.proj_side >= 0 && c.cur_gpar) {
        CK(cudaMemcpyAsync(t + og, c.cur_gpar, 4 * (size_t)ng, cudaMemcpyDeviceToDevice, c.stream));
        c.cur_gpar = reinterpret_cast<const int32_t*>(t + og);
      }
      for (int side = 0; side < 2; ++side) c.leaf_sel[side] = (f ? c.leaf_out2 : c.leaf_out)[side].p;
      c.part_sel = f ? &c.d_partial2 : &c.d_partial;
    }
    if (c.ovl && l + 1 == D - 1) {  // the projected gathers read this level's parent states
      CK(cudaStreamWaitEvent(c.stream, c.ev_g[0], 0));
      CK(cudaStreamWaitEvent(c.stream, c.ev_g[1], 0));
    }
    // the fused leaf passes read the request buckets: built here, behind the upper levels already
    // queued, so the staged request copy and its upload overlap them (gs_run_batched)
    if (l + 1 == D) ensure_buckets(c);
    int64_t n_par = n > 0 ? 1 : 0;  // distinct parents of the chunk (children come in parent order)
    for (int64_t j = 1; j < n; ++j) n_par += chunk[j].parent != chunk[j - 1].parent;
    run_level_passes<R>(c, l + 1, n, at(c.lvl_a, l), at(c.lvl_b, l), at(c.lvl_a, l + 1),
                        at(c.lvl_b, l + 1), d_parent, d_digit, false, n_par);
    c.uni_p0 = -1;
    if (f >= 0) {
      CK(cudaEventRecord(c.ev_leaf, c.stream));
      CK(cudaStreamWaitEvent(c.gstream, c.ev_leaf, 0));
      c.gs = c.gstream;
    }
    descend<R>(c, l + 1, chunk, n);
    if (f >= 0) {
      CK(cudaEventRecord(c.ev_g[f], c.gstream));
      c.gs = nullptr;
      c.part_sel = nullptr;
      c.leaf_sel[0] = c.leaf_sel[1] = nullptr;
    }
  }
}

static void plan_buffers_impl(Ctx& c, int64_t n_leaves);
// The buffer plan depends only on the schedule, the leaf bound, the request
// count and the options below; re-planning queries free device memory, which
// can stall the host for milliseconds, so steady-state runs reuse the plan.
static void plan_buffers(Ctx& c, int64_t n_leaves) {
  const std::vector<int64_t> key = {n_leaves, c.n_req, c.mem_budget_mb, (int64_t)c.sched_serial,
                                    (c.fused_active ? 1 : 0) + (c.proj_fused_active ? 2 : 0), c.group_log,
                                    c.grouped_leaf ? 1 : 0, c.max_chunk,
                                    c.host_only ? 1 : 0, c.overlap_gather};
  if (key == c.plan_key) return;
  plan_buffers_impl(c, n_leaves);
  c.plan_key = key;
}
static void plan_buffers_impl(Ctx& c, int64_t n_leaves) {
  const Program& p = c.prog;
  const int D = (int)p.levels.size() - 1;
  const double pair = (double)((1LL << p.q[0]) + (1LL << p.q[1])) * (double)c.esize();
  // upper bound on nodes per level
  std::vector<double> bound(D + 1, 1.0);
  double prod = 1.0;
  for (int l = 1; l <= D; ++l) {
    prod *= (double)level_fanout(p, l);
    bound[l] = std::min(prod, (double)n_leaves);
  }
  double budget;
  if (c.mem_budget_mb > 0) {
    budget = (double)c.mem_budget_mb * 1048576.0;
  } else if (c.host_only) {
    budget = 64e9;
  } else {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    // level buffers this context already holds are reused, so they count as free
    double held = 0;
    for (auto* v : {&c.lvl_a, &c.lvl_b})
      for (const DevBuf& b : *v) held += (double)b.bytes;
    budget = 0.80 * ((double)fr + held) - 1.5e9;
    budget = std::max(budget, 4.0 * pair);
  }
  // largest uniform cap with sum_l min(bound_l, cap) * pair <= budget
  // grouped leaf states: one (or, overlapping gathers, two) extra leaf chunks
  const double leaf_sets = c.grouped_leaf ? (c.overlap_gather ? 2.0 : 0.0) : 0.0;
  auto need = [&](double cap) {
    double s = 0;
    for (int l = 0; l <= D; ++l) s += std::min(bound[l], cap) * pair;
    s += leaf_sets * std::min(bound[D], cap) * pair;
    return s;
  };
  double lo = 1, hi = (double)c.max_chunk;
  if (need(1) > budget)
    throw GsError(GS_ERR_NOMEM, "device memory budget below one node per level (need " +
                                    std::to_string(need(1) / 1e9) + " GB for " + std::to_string(D + 1) +
                                    " levels, budget " + std::to_string(budget / 1e9) + " GB)");
  while (hi - lo > 0.5) {
    double mid = std::floor((lo + hi + 1) / 2);
    if (need(mid) <= budget) lo = mid; else hi = mid - 1;
  }
  c.cap.assign(D + 1, 1);
  for (int l = 0; l <= D; ++l) c.cap[l] = (int64_t)std::max(1.0, std::min(bound[l], lo));
  if (c.fused_active && c.n_req > 0) {  // fused leaf gather: one partial row per 8 leaves
    const int64_t max_groups = std::max<int64_t>(1, (2LL << 30) / (16 * c.n_req));
    c.cap[D] = std::min<int64_t>(c.cap[D], 8 * max_groups);
  }
  if (c.host_only) return;
  c.lvl_a.resize(D + 1);
  c.lvl_b.resize(D + 1);
  int64_t max_cap = 1;
  for (int l = 0; l <= D; ++l) max_cap = std::max(max_cap, c.cap[l]);
  // one chunk's digits + parents + weights, several times over, at least 32 MiB
  c.ring.reserve(std::max<size_t>((size_t)32 << 20, (size_t)max_cap * 64 * 4 + 4096), c.stream);
  // release oversized buffers first so growing one level cannot overshoot the budget
  for (int l = 0; l <= D; ++l) {
    if (c.lvl_a[l].bytes > (size_t)c.cap[l] * ((size_t)1 << p.q[0]) * c.esize()) c.lvl_a[l].release();
    if (c.lvl_b[l].bytes > (size_t)c.cap[l] * ((size_t)1 << p.q[1]) * c.esize()) c.lvl_b[l].release();
  }
  for (int l = 0; l <= D; ++l) {
    c.lvl_a[l].ensure((size_t)c.cap[l] * ((size_t)1 << p.q[0]) * c.esize());
    c.lvl_b[l].ensure((size_t)c.cap[l] * ((size_t)1 << p.q[1]) * c.esize());
  }
  if (c.grouped_leaf) {
    const size_t gsz = (size_t)1 << c.group_log;
    const size_t slots = (size_t)((c.cap[D] + gsz - 1) / gsz) * gsz;
    for (int side = 0; side < 2; ++side) c.leaf_out[side].ensure(slots * ((size_t)1 << p.q[side]) * c.esize());
    if (c.overlap_gather)
      for (int side = 0; side < 2; ++side) c.leaf_out2[side].ensure(slots * ((size_t)1 << p.q[side]) * c.esize());
  }
}

// Bucket the requests by the tile of the fused leaf pass (B side, last pass):
// counting sort on the device (histogram, CUB exclusive scan, scatter).
static void build_buckets(Ctx& c) {
  const int D = (int)c.prog.levels.size() - 1;
  // the bucketed side: B for the fused B gather; the grouped side of a fused projected pass
  const int gside = c.proj_fused_active ? 1 - c.proj_side : 1;
  const PassPlan& pp = c.prog.levels[D].passes[gside].back();
  BucketMap m{};
  m.n_g = (int)pp.gbits.size();
  m.n_l = pp.k;
  for (int j = 0; j < m.n_g; ++j) m.gbits[j] = pp.gbits[j];
  for (int j = 0; j < m.n_l; ++j) m.lbits[j] = pp.lbits[j];
  // Pauli-sibling pass: 32 fine bins per tile (two bank-half streams, each sorted by factor-table row)
  const int fine = (pp.pf_pauli && c.pf_streams) ? 1 : 0;
  const int tiles = (1 << m.n_g) << (fine ? 5 : 0);
  const int64_t n = c.n_req;
  c.d_bcount.ensure((size_t)(tiles + 1) * 4);
  c.d_bstart.ensure((size_t)(tiles + 1) * 4);
  c.d_breq.ensure(std::max<size_t>((size_t)n * 4, 16));
  c.d_btl.ensure(std::max<size_t>((size_t)n * 4, 16));
  c.d_bia.ensure(std::max<size_t>((size_t)n * 4, 16));
  int32_t* cnt = reinterpret_cast<int32_t*>(c.d_bcount.p);
  int32_t* start = reinterpret_cast<int32_t*>(c.d_bstart.p);
  CK(cudaMemsetAsync(cnt, 0, (size_t)(tiles + 1) * 4, c.stream));
  const unsigned blocks = (unsigned)std::max<int64_t>(1, (n + 255) / 256);
  if (n > 0)
    bucket_count_kernel<<<blocks, 256, 0, c.stream>>>(
        reinterpret_cast<const int32_t*>(gside == 1 ? c.d_ib.p : c.d_ia.p),
        reinterpret_cast<const int32_t*>(gside == 1 ? c.d_ia.p : c.d_ib.p), n, m, cnt, fine);
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, start, tiles + 1, c.stream));
  c.d_cubtmp.ensure(std::max<size_t>(tmp, 16));
  CK(cub::DeviceScan::ExclusiveSum(c.d_cubtmp.p, tmp, cnt, start, tiles + 1, c.stream));
  CK(cudaMemcpyAsync(cnt, start, (size_t)(tiles + 1) * 4, cudaMemcpyDeviceToDevice, c.stream));
  if (n > 0)
    bucket_fill_kernel<<<blocks, 256, 0, c.stream>>>(
        reinterpret_cast<const int32_t*>(gside == 1 ? c.d_ib.p : c.d_ia.p),
        reinterpret_cast<const int32_t*>(gside == 1 ? c.d_ia.p : c.d_ib.p), n, m, cnt,
        reinterpret_cast<int32_t*>(c.d_breq.p), reinterpret_cast<int32_t*>(c.d_btl.p),
        reinterpret_cast<int32_t*>(c.d_bia.p), fine);
  if (c.proj_fused_active && n > 0) {
    // the fused pass reads whole 32-slot warp rows past the last bucket: zero padding
    // makes those rows address element 0 of the parent (their results are not written)
    c.d_bmeta.ensure((size_t)(n + 64) * sizeof(int2));
    CK(cudaMemsetAsync(reinterpret_cast<int2*>(c.d_bmeta.p) + n, 0, 64 * sizeof(int2), c.stream));
    pf_meta_kernel<<<blocks, 256, 0, c.stream>>>(reinterpret_cast<const int32_t*>(c.d_bia.p),
                                                 reinterpret_cast<const int32_t*>(c.d_btl.p), n,
                                                 reinterpret_cast<int2*>(c.d_bmeta.p), pp.pf_pauli ? 1 : 0);
  }
  CK(cudaGetLastError());
  c.bucket_valid = true;
}

static void ensure_buckets(Ctx& c) {
  if ((c.fused_active || c.proj_fused_active) && !c.host_only && !c.bucket_valid && c.n_req > 0) {
    finish_requests(c);
    build_buckets(c);
  }
}

template <typename R>
static void run_tree(Ctx& c) {
  const Program& p = c.prog;
  const int D = (int)p.levels.size() - 1;
  int64_t n_leaves_bound = (int64_t)c.prefixes.size() * (c.branch_hi - c.branch_lo);
  plan_buffers(c, std::max<int64_t>(1, n_leaves_bound));
  c.st.n_levels = D + 1;
  c.ovl = c.overlap_gather && c.grouped_leaf && !c.fused_active && !c.proj_fused_active && !c.profile &&
          !c.host_only && D >= 1;
  if (c.ovl && !c.gstream) {
    CK(cudaStreamCreateWithFlags(&c.gstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c.ev_leaf, cudaEventDisableTiming));
    for (auto& e : c.ev_g) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (D == 0) ensure_buckets(c);  // (deeper trees build them in front of their first leaf chunk)
  const Node root0{0, (int64_t)c.prefixes.size(), 0, 0, c.branch_lo, c.branch_hi, 0, 0};
  if (D == 0) upload_weights(c, &root0, 1);  // the root is the leaf
  // root: |0...0> through the root segment
  run_level_passes<R>(c, 0, 1, nullptr, nullptr, c.lvl_a.empty() ? nullptr : c.lvl_a[0].p,
                      c.lvl_b.empty() ? nullptr : c.lvl_b[0].p, nullptr, nullptr, true);
  const Node root{0, (int64_t)c.prefixes.size(), 0, 0, c.branch_lo, c.branch_hi, 0, 0};
  if (c.prefixes.empty() || c.branch_hi <= c.branch_lo) return;
  c.kids.resize(D + 1);
  descend<R>(c, 0, &root, 1);
}

}  // namespace gs

// ---------------------------------------------------------------------------
// C ABI

using gs::Ctx;
using gs::GsError;

struct gs_ctx {
  Ctx c;
};

#define GS_GUARD(ctx, ...)                                   \
  do {                                                       \
    try {                                                    \
      __VA_ARGS__;                                           \
      return GS_OK;                                          \
    } catch (const GsError& e) {                             \
      if (ctx) (ctx)->c.err = e.what();                      \
      return e.code;                                         \
    } catch (const std::bad_alloc&) {                        \
      if (ctx) (ctx)->c.err = "host out of memory";          \
      return GS_ERR_NOMEM;                                   \
    } catch (const std::exception& e) {                      \
      if (ctx) (ctx)->c.err = e.what();                      \
      return GS_ERR_ARG;                                     \
    }                                                        \
  } while (0)

extern "C" {

int gs_abi_version(void) { return GS_ABI_VERSION; }

int gs_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return GS_ERR_ARG;
  *out = nullptr;
  if (cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 16), cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return GS_ERR_NOMEM;
  }
  return GS_OK;
}

void gs_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int gs_device_count(int* out) {
  if (!out) return GS_ERR_ARG;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = 0;
    return GS_OK;
  }
  *out = n;
  return GS_OK;
}

int gs_create(int device, int precision, gs_ctx** out) {
  if (!out) return GS_ERR_ARG;
  *out = nullptr;
  if (precision != GS_C64 && precision != GS_C128) return GS_ERR_ARG;
  gs_ctx* h = new (std::nothrow) gs_ctx();
  if (!h) return GS_ERR_NOMEM;
  h->c.precision = precision;
  h->c.device = device;
  if (device < 0) {
    h->c.host_only = true;  // planning / dry runs only (CPU tests)
    *out = h;
    return GS_OK;
  }
  try {
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&h->c.n_sm, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&h->c.own_stream, cudaStreamNonBlocking));
    h->c.stream = h->c.own_stream;
    CK(cudaEventCreate(&h->c.ev0));
    CK(cudaEventCreate(&h->c.ev1));
    CK(cudaFuncSetAttribute(gs::gate_pass_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(gs::gate_pass_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  } catch (const GsError& e) {
    std::fprintf(stderr, "gs_create: %s\n", e.what());
    delete h;
    return e.code;
  }
  *out = h;
  return GS_OK;
}

void gs_destroy(gs_ctx* ctx) {
  if (!ctx) return;
  if (!ctx->c.host_only) {
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.ev0) cudaEventDestroy(ctx->c.ev0);
    if (ctx->c.ev_leaf) cudaEventDestroy(ctx->c.ev_leaf);
    for (auto e : ctx->c.ev_g)
      if (e) cudaEventDestroy(e);
    if (ctx->c.gstream) cudaStreamDestroy(ctx->c.gstream);
    if (ctx->c.ev1) cudaEventDestroy(ctx->c.ev1);
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.own_stream);
    if (ctx->c.side_stream) {
      cudaStreamSynchronize(ctx->c.side_stream);
      cudaStreamDestroy(ctx->c.side_stream);
    }
    if (ctx->c.req_done) cudaEventDestroy(ctx->c.req_done);
    for (cudaEvent_t e : ctx->c.out_events) cudaEventDestroy(e);
    for (gs::JitModule* m : ctx->c.jit_mods) gs::jit_release(m);
  }
  delete ctx;
}

const char* gs_last_error(const gs_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

int gs_set_stream(gs_ctx* ctx, void* s) {
  if (!ctx) return GS_ERR_ARG;
  // staging regions are recycled in stream order: finish the old stream's work first
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (!c.host_only && c.stream) CK(cudaStreamSynchronize(c.stream));
    c.ring.drain();
    c.stream = s ? reinterpret_cast<cudaStream_t>(s) : c.own_stream;
  });
}

int gs_set_option(gs_ctx* ctx, const char* key, int64_t value) {
  if (!ctx || !key) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    std::string k(key);
    Ctx& c = ctx->c;
    if (k == "mem_budget_mb") c.mem_budget_mb = value;
    else if (k == "profile") c.profile = (int)value;
    else if (k == "tile_bits") {
      if (value != 0 && (value < 4 || value > (c.precision == GS_C64 ? 14 : 13)))
        throw GsError(GS_ERR_ARG, "tile_bits out of range");
      c.tile_bits = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "uniform_chunks") {
      c.uniform_chunks = value ? 1 : 0;
    } else if (k == "jit_spill_ok") {
      c.jit_spill_ok = (int)std::max<int64_t>(0, value);
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "gather_gpy") {
      c.gather_gpy = (int)std::max<int64_t>(0, value);
    } else if (k == "overlap_gather") {
      c.overlap_gather = value ? 1 : 0;
    } else if (k == "sink_ops") {
      c.sink_ops = (int)std::max<int64_t>(0, value);
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "slot_store16") {
      c.slot_store16 = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "proj_lanes") {
      if (value != 4 && value != 8) throw GsError(GS_ERR_ARG, "proj_lanes must be 4 or 8");
      c.proj_lanes = (int)value;
    } else if (k == "proj_perm") {
      c.proj_perm = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "tile_major") {
      if (value < 0 || value > 2) throw GsError(GS_ERR_ARG, "tile_major must be 0, 1 or 2");
      c.tile_major = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "proj_fuse") {
      c.proj_fuse = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_u") {
      if (value < 1 || value > 8) throw GsError(GS_ERR_ARG, "pf_u must be in [1, 8]");
      c.pf_u = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "jit_rsign") {
      c.jit_rsign = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "jit_rsign_max") {
      c.jit_rsign_max = (int)std::max<int64_t>(1, std::min<int64_t>(value, 32));
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "jit_c128") {
      c.jit_c128 = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "xchg16") {
      c.xchg16 = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "sink_balance") {
      c.sink_balance = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_m4") {
      c.pf_m4 = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_unroll") {
      c.pf_unroll = (int)std::max<int64_t>(1, std::min<int64_t>(value, 6));
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_streams") {
      c.pf_streams = value ? 1 : 0;
      c.bucket_valid = false;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "l2_ahead") {
      if (value < 0 || value > (1 << 20)) throw GsError(GS_ERR_ARG, "l2_ahead out of range");
      c.l2_ahead = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_groups") {
      if (value < 1 || value > 64) throw GsError(GS_ERR_ARG, "pf_groups must be in [1, 64]");
      c.pf_groups = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_pipe") {
      c.pf_pipe = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_pauli") {
      c.pf_pauli = value ? 1 : 0;
      c.pauli_blocked = false;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_tail") {
      c.pf_tail = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pf_min_blocks") {
      if (value < 0 || value > 4) throw GsError(GS_ERR_ARG, "pf_min_blocks must be in [0, 4]");
      c.pf_min_blocks = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "proj_leaf") {
      c.proj_leaf = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "tail_gather") {
      c.tail_gather = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "tail_max") {
      if (value < 1 || value > 3) throw GsError(GS_ERR_ARG, "tail_max must be 1..3");
      c.tail_max = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "jit_cross_inline") {
      if (value < 0 || value > 3) throw GsError(GS_ERR_ARG, "jit_cross_inline must be 0..3");
      c.jit_cross_inline = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "dedupe_parent") {
      c.dedupe_parent = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pipeline") {
      c.pipeline = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "quad_gather") {
      c.quad_gather = value ? 1 : 0;
    } else if (k == "sort_requests") {
      c.sort_requests = value ? 1 : 0;
    } else if (k == "low_bits") {
      if (value < 1 || value > 8) throw GsError(GS_ERR_ARG, "low_bits out of range");
      c.low_bits = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "hoist") {
      c.hoist = value ? 1 : 0;
      if (c.have_prog) throw GsError(GS_ERR_STATE, "set hoist before gs_load_program");
    } else if (k == "group_log") {
      if (value < 2 || value > 4) throw GsError(GS_ERR_ARG, "group_log must be 2, 3 or 4");
      c.group_log = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "fuse_gather") {
      c.fuse_gather = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "grouped_leaf") {
      c.grouped_enabled = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "smem_gather") {
      c.smem_gather = value ? 1 : 0;
    } else if (k == "vec_hbm") {
      c.vec_hbm = value ? 1 : 0;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "jit_min_blocks") {
      if (value < 0 || value > 8) throw GsError(GS_ERR_ARG, "jit_min_blocks must be 0..8");
      c.jit_min_blocks = (int)value;
      if (c.have_prog) gs::jit_program(c);
    } else if (k == "d2h_chunk_mb") {
      if (value < 0 || value > 1024) throw GsError(GS_ERR_ARG, "d2h_chunk_mb must be 0..1024");
      c.d2h_chunk_mb = value;
    } else if (k == "async_run") {
      c.async_run = value ? 1 : 0;
    } else if (k == "jit") {
      c.use_jit = value ? 1 : 0;  // the HBM stage layout depends on it: reschedule
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "m4_ops") {
      c.m4_ops = (int)std::max<int64_t>(1, value);
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "reg_bits") {
      if (value != 0 && value != 4 && value != 5 && value != 6)
        throw GsError(GS_ERR_ARG, "reg_bits must be 0, 4, 5 or 6");
      c.reg_bits = (int)value;
      if (c.have_prog) { gs::schedule_program(c); gs::upload_program(c); }
    } else if (k == "pass_kernel") {
      if (value != 1 && value != 2) throw GsError(GS_ERR_ARG, "pass_kernel must be 1 or 2");
      c.kernel_version = (int)value;
    } else if (k == "max_chunk") {
      if (value < 1) throw GsError(GS_ERR_ARG, "max_chunk must be positive");
      c.max_chunk = value;
    } else throw GsError(GS_ERR_ARG, "unknown option " + k);
  });
}

int gs_load_program(gs_ctx* ctx, int32_t qa, int32_t qb, int32_t n_ops, const int32_t* op_kind,
                    const int32_t* op_blk, const int32_t* op_q0, const int32_t* op_q1,
                    const int32_t* op_cycle, const int64_t* op_coef, int32_t n_cross,
                    const int32_t* cross_rank, const int32_t* cross_cycle, const int32_t* cross_qa,
                    const int32_t* cross_qb, const int32_t* term_kind_a, const int64_t* term_coef_a,
                    const int32_t* term_kind_b, const int64_t* term_coef_b, int64_t n_coef,
                    const double* coef) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (n_ops < 0 || n_cross < 0 || n_coef < 0) throw GsError(GS_ERR_ARG, "negative count");
    if (n_ops > 0 && (!op_kind || !op_blk || !op_q0 || !op_q1 || !op_cycle || !op_coef))
      throw GsError(GS_ERR_ARG, "null op array");
    if (n_cross > 0 && (!cross_rank || !cross_cycle || !cross_qa || !cross_qb || !term_kind_a ||
                        !term_coef_a || !term_kind_b || !term_coef_b))
      throw GsError(GS_ERR_ARG, "null cross array");
    if (!c.host_only) CK(cudaSetDevice(c.device));
    c.have_prog = false;
    c.pauli_blocked = false;
    gs::build_program(c, qa, qb, n_ops, op_kind, op_blk, op_q0, op_q1, op_cycle, op_coef, n_cross,
                      cross_rank, cross_cycle, cross_qa, cross_qb, term_kind_a, term_coef_a,
                      term_kind_b, term_coef_b, n_coef, coef);
    gs::schedule_program(c);
    gs::upload_program(c);
    c.have_prog = true;
    c.n_req = -1;
  });
}

int gs_describe(gs_ctx* ctx, char* buf, int64_t cap, int64_t* needed) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (!c.have_prog) throw GsError(GS_ERR_STATE, "no program loaded");
    std::string js = "{\"q\": [" + std::to_string(c.prog.q[0]) + ", " + std::to_string(c.prog.q[1]) +
                     "], \"levels\": [";
    for (size_t l = 0; l < c.prog.levels.size(); ++l) {
      const gs::Level& L = c.prog.levels[l];
      js += (l ? ", " : "") + std::string("{\"k_lo\": ") + std::to_string(L.k_lo) +
            ", \"k_hi\": " + std::to_string(L.k_hi) + ", \"blocks\": [";
      for (int side = 0; side < 2; ++side) {
        js += (side ? ", " : "") + std::string("{\"ops\": ") + std::to_string(L.ops[side].size()) +
              ", \"passes\": [";
        for (size_t pi = 0; pi < L.passes[side].size(); ++pi) {
          const gs::PassPlan& pp = L.passes[side][pi];
          js += (pi ? ", " : "") + std::string("{\"ops\": ") + std::to_string(pp.ops.size()) +
                ", \"k\": " + std::to_string(pp.k) + ", \"K\": " + std::to_string(pp.K) +
                ", \"M\": " + std::to_string(pp.M) + ", \"stages\": [";
          for (size_t si = 0; si < pp.stages.size(); ++si) {
            const gs::PStage& ps = c.host_pstages[pp.dev_stage_offset + si];
            js += (si ? ", " : "") + std::to_string(ps.op_end - ps.op_begin);
          }
          js += "], \"rb\": [";
          for (size_t si = 0; si < pp.stages.size(); ++si) {
            js += si ? ", [" : "[";
            for (size_t i = 0; i < pp.stages[si].rb.size(); ++i)
              js += (i ? ", " : "") + std::to_string(pp.stages[si].rb[i]);
            js += "]";
          }
          js += "], \"lbits\": [";
          for (size_t i = 0; i < pp.lbits.size(); ++i) js += (i ? ", " : "") + std::to_string(pp.lbits[i]);
          js += "], \"grouped\": " + std::to_string(pp.grouped_store ? 1 : 0) + ", \"store_scale\": " + std::to_string(pp.store_scale) +
                ", \"jit\": " + std::to_string(pp.jit_index) + ", \"opl\": \"";
          for (const gs::HostOp& op : pp.ops) {
            static const char kc[] = "dmDMx";
            js += kc[op.kind < 5 ? op.kind : 4];
            if (op.cross >= 0) js += "x";
            js += std::to_string(op.s0);
            if (op.s1 >= 0) js += ":" + std::to_string(op.s1);
            js += " ";
          }
          js += "\"}";
        }
        js += "]}";
      }
      js += "]}";
    }
    js += "], \"tail\": [" + std::to_string(c.tail_ops[0].size()) + ", " + std::to_string(c.tail_ops[1].size()) +
          "], \"proj_side\": " + std::to_string(c.proj_side) + ", \"proj_fused\": " +
          std::to_string(c.proj_fused_active ? 1 : 0) + ", \"pauli_sides\": [" +
          std::to_string(gs::pauli_frame(c, 0, c.prog.levels.back().ops[0]).ok ? 1 : 0) + ", " +
          std::to_string(c.prog.q[1] > 0 && gs::pauli_frame(c, 1, c.prog.levels.back().ops[1]).ok ? 1 : 0) +
          "], \"psib_side\": " + std::to_string(c.psib_side) + ", \"pauli\": " + [&]() {
            if (!c.pauli.ok) return std::string("null");
            std::string t = "{\"conflicts\": " + std::to_string(c.pauli_conflicts) + ", \"gates\": [";
            for (int j = 0; j < c.pauli.nk; ++j)
              t += (j ? ", " : "") + std::string("{\"a\": ") + std::to_string(c.pauli.a[j]) + ", \"f\": " +
                   std::to_string(c.pauli.f[j]) + ", \"z\": " + std::to_string(c.pauli.z[j]) + "}";
            t += "], \"lcol\": [";
            for (int j = 0; j < 16; ++j) t += (j ? ", " : "") + std::to_string(c.pauli_lcol[j]);
            return t + "]}";
          }() + ", \"opts\": {\"pf_pauli\": " + std::to_string(c.pf_pauli) + ", \"pf_pipe\": " + std::to_string(c.pf_pipe) + ", \"pf_groups\": " + std::to_string(c.pf_groups) + ", \"l2_ahead\": " + std::to_string(c.l2_ahead) + ", \"pf_streams\": " + std::to_string(c.pf_streams) + ", \"xchg16\": " + std::to_string(c.xchg16) + ", \"pf_tail\": " + std::to_string(c.pf_tail) +
          ", \"tile_major\": " + std::to_string(c.tile_major) + ", \"pf_min_blocks\": " +
          std::to_string(c.pf_min_blocks) + ", \"pipeline\": " + std::to_string(c.pipeline) + ", \"sink_ops\": " +
          std::to_string(c.sink_ops) + ", \"sink_balance\": " + std::to_string(c.sink_balance) + ", \"reg_bits\": " + std::to_string(c.reg_bits) + "}, \"proj_swaps\": " +
          std::to_string(c.proj_swaps.size()) + ", \"jit\": \"";
    for (char ch : c.jit_status) js += (ch == '"' || ch == '\\' || ch == '\n') ? ' ' : ch;
    js += "\"}";
    if (needed) *needed = (int64_t)js.size() + 1;
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(js.size(), (size_t)cap - 1);
      std::memcpy(buf, js.data(), n);
      buf[n] = 0;
    }
  });
}

}  // extern "C"

namespace gs {

// bit runs of the cut: qubit q owns global bit n-1-q, local j owns bit q_blk-1-j
static SplitRuns split_runs(const Ctx& c, int32_t n_qubits, const int32_t* block_a, const int32_t* block_b) {
  const int qs[2] = {c.prog.q[0], c.prog.q[1]};
  if (qs[0] + qs[1] != n_qubits || n_qubits > 62) throw GsError(GS_ERR_ARG, "cut does not match the program");
  SplitRuns runs{};
  runs.qa = qs[0];
  std::vector<char> seen(n_qubits, 0);
  for (int b = 0; b < 2; ++b) {
    const int32_t* blk = b ? block_b : block_a;
    int j = 0;
    while (j < qs[b]) {
      int k = j;
      while (k + 1 < qs[b] && blk[k + 1] == blk[k] + 1) ++k;
      for (int t = j; t <= k; ++t) {
        if (blk[t] < 0 || blk[t] >= n_qubits || seen[blk[t]]) throw GsError(GS_ERR_ARG, "bad cut blocks");
        seen[blk[t]] = 1;
      }
      if (runs.n[b] >= 32) throw GsError(GS_ERR_ARG, "cut has too many bit runs");
      runs.src[b][runs.n[b]] = n_qubits - 1 - blk[k];
      runs.width[b][runs.n[b]] = k - j + 1;
      runs.dst[b][runs.n[b]] = qs[b] - 1 - k;
      ++runs.n[b];
      j = k + 1;
    }
  }
  return runs;
}

static bool packed_requests(const Ctx& c) { return c.prog.q[0] + c.prog.q[1] <= 31; }

static void ensure_request_buffers(Ctx& c, int64_t n_req) {
  c.d_gidx.ensure(std::max<size_t>(n_req * 8, 16));
  c.d_ia.ensure(std::max<size_t>(n_req * 4, 16));
  c.d_ib.ensure(std::max<size_t>(n_req * 4, 16));
  if (packed_requests(c)) c.d_packed.ensure(std::max<size_t>(n_req * 4, 16));
  c.d_acc.ensure(std::max<size_t>(n_req * sizeof(double2), 16));
}

template <typename R> static void run_tree(Ctx& c);

// body of gs_run / gs_run_batched (requests already loaded or staged)
static void run_body(Ctx& c, int32_t x_p, int64_t n_prefix, const int64_t* prefixes, int64_t branch_lo,
                     int64_t branch_hi, double* out_host, void* out_device, int32_t accumulate, gs_stats* stats);

}  // namespace gs

extern "C" {

int gs_set_requests_global(gs_ctx* ctx, int64_t n_req, const int64_t* idx, int32_t n_qubits,
                           const int32_t* block_a, const int32_t* block_b) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (!c.have_prog) throw GsError(GS_ERR_STATE, "no program loaded");
    if (n_req < 0 || (n_req > 0 && !idx) || !block_a || !block_b) throw GsError(GS_ERR_ARG, "bad request arrays");
    const gs::SplitRuns runs = gs::split_runs(c, n_qubits, block_a, block_b);
    const int64_t lim = 1LL << n_qubits;
    for (int64_t i = 0; i < n_req; ++i)
      if (idx[i] < 0 || idx[i] >= lim) throw GsError(GS_ERR_INDEX, "request index outside the state space");
    c.n_req = -1;
    if (!c.host_only) {
      CK(cudaSetDevice(c.device));
      gs::ensure_request_buffers(c, n_req);
      const bool pk = gs::packed_requests(c);
      if (n_req > 0) {
        CK(cudaMemcpyAsync(c.d_gidx.p, idx, n_req * 8, cudaMemcpyHostToDevice, c.stream));
        gs::split_kernel<<<(unsigned)((n_req + 255) / 256), 256, 0, c.stream>>>(
            reinterpret_cast<const long long*>(c.d_gidx.p), n_req, runs, reinterpret_cast<int32_t*>(c.d_ia.p),
            reinterpret_cast<int32_t*>(c.d_ib.p), pk ? reinterpret_cast<uint32_t*>(c.d_packed.p) : nullptr);
        CK(cudaGetLastError());
      }
    }
    c.n_req = n_req;
    c.bucket_valid = false;
    gs::sort_requests(c, c.stream);
  });
}

int gs_run_batched(gs_ctx* ctx, int64_t n_req, const int64_t* idx, int32_t n_qubits, const int32_t* block_a,
                   const int32_t* block_b, int32_t x_p, int64_t n_prefix, const int64_t* prefixes,
                   int64_t branch_lo, int64_t branch_hi, double* out_host, void* out_device, int32_t accumulate,
                   gs_stats* stats) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    // worker threads never outlive the call; an unfinished staging leaves no requests loaded
    struct Guard {
      Ctx& c;
      ~Guard() {
        c.pend.join();
        if (c.pend.active) c.pend.active = false, c.n_req = -1;
      }
    } guard{c};
    if (!c.have_prog) throw GsError(GS_ERR_STATE, "no program loaded");
    if (n_req < 0 || (n_req > 0 && !idx) || !block_a || !block_b) throw GsError(GS_ERR_ARG, "bad request arrays");
    const gs::SplitRuns runs = gs::split_runs(c, n_qubits, block_a, block_b);
    c.n_req = -1;
    int64_t* stage = nullptr;
    if (!c.host_only) {
      CK(cudaSetDevice(c.device));
      gs::ensure_request_buffers(c, n_req);
      if (!c.side_stream) CK(cudaStreamCreateWithFlags(&c.side_stream, cudaStreamNonBlocking));
      if (!c.req_done) CK(cudaEventCreateWithFlags(&c.req_done, cudaEventDisableTiming));
      CK(cudaEventSynchronize(c.req_done));  // the previous upload has left the staging buffer
      c.req_stage.ensure(std::max<size_t>(n_req * 8, 16));
      stage = reinterpret_cast<int64_t*>(c.req_stage.p);
    }
    // validate + stage the requests on worker threads while the tree is enqueued
    const int64_t lim = 1LL << n_qubits;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(8, hw), (n_req + (1 << 18) - 1) >> 18));
    c.pend.n = n_req;
    c.pend.runs = runs;
    c.pend.packed = gs::packed_requests(c);
    c.pend.bad.assign(T, 0);
    char* bad = c.pend.bad.data();
    for (int t = 0; t < T && n_req > 0; ++t)
      c.pend.workers.emplace_back([=] {
        const int64_t lo = n_req * t / T, hi = n_req * (t + 1) / T;
        bool b = false;
        for (int64_t i = lo; i < hi; ++i) {
          const int64_t v = idx[i];
          b |= (v < 0) | (v >= lim);
          if (stage) stage[i] = v;
        }
        bad[t] = b;
      });
    c.pend.active = true;
    c.n_req = n_req;
    c.bucket_valid = false;
    gs::run_body(c, x_p, n_prefix, prefixes, branch_lo, branch_hi, out_host, out_device, accumulate, stats);
  });
}

int gs_run_full(gs_ctx* ctx, void* out_host, void* out_device, gs_stats* stats) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (!c.have_prog) throw GsError(GS_ERR_STATE, "no program loaded");
    if (c.prog.q[1] != 0 || c.prog.n_cross != 0 || c.prog.levels.size() != 1)
      throw GsError(GS_ERR_ARG, "gs_run_full needs an uncut program (n_qubits_b = 0, no cross gates)");
    c.st = gs_stats{};
    const auto t_call = std::chrono::steady_clock::now();
    c.last_tick = t_call;
    const int q = c.prog.q[0];
    const int64_t n = 1LL << q;
    const size_t bytes = (size_t)n * c.esize();
    if (!c.host_only) {
      CK(cudaSetDevice(c.device));
      c.full_state.ensure(bytes);
      CK(cudaEventRecord(c.ev0, c.stream));
    }
    void* st = c.full_state.p;
    {
      gs::Timer t(c, &c.st.ms_pass);
      bool first = true;
      for (const gs::PassPlan& pp : c.prog.levels[0].passes[0]) {  // in place after the first pass
        if (c.precision == GS_C64) {
          if (c.kernel_version == 2 && pp.M > 0) gs::launch_pass2<float>(c, 0, pp, st, st, nullptr, nullptr, 1, first);
          else gs::launch_pass<float>(c, 0, pp, st, st, nullptr, nullptr, 1, first);
        } else {
          if (c.kernel_version == 2 && pp.M > 0) gs::launch_pass2<double>(c, 0, pp, st, st, nullptr, nullptr, 1, first);
          else gs::launch_pass<double>(c, 0, pp, st, st, nullptr, nullptr, 1, first);
        }
        first = false;
      }
      if (first) throw GsError(GS_ERR_ARG, "full-state program has no pass");
    }
    c.st.n_nodes = 1;
    c.st.n_levels = 1;
    c.st.pass_bytes_min = 2.0 * (double)bytes;
    if (!c.host_only) {
      const unsigned blocks = (unsigned)((n + 255) / 256);
      if (c.precision == GS_C64)
        gs::scale_state_kernel<float><<<blocks, 256, 0, c.stream>>>(st, n, c.kfinal[0][0], c.kfinal[0][1]);
      else
        gs::scale_state_kernel<double><<<blocks, 256, 0, c.stream>>>(st, n, c.kfinal[0][0], c.kfinal[0][1]);
      CK(cudaGetLastError());
      c.st.n_launches += 1;
      CK(cudaEventRecord(c.ev1, c.stream));
      if (out_device) CK(cudaMemcpyAsync(out_device, st, bytes, cudaMemcpyDeviceToDevice, c.stream));
      if (out_host) {
        CK(cudaMemcpyAsync(out_host, st, bytes, cudaMemcpyDeviceToHost, c.stream));
        c.st.d2h_bytes += (double)bytes;
      }
      CK(cudaStreamSynchronize(c.stream));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
      c.st.ms_total = ms;
    } else if (out_host) {
      std::memset(out_host, 0, bytes);
    }
    c.st.host_ms_enqueue =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
    if (stats) *stats = c.st;
  });
}

int gs_set_requests(gs_ctx* ctx, int64_t n_req, const int64_t* ia, const int64_t* ib) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (!c.have_prog) throw GsError(GS_ERR_STATE, "no program loaded");
    if (n_req < 0 || (n_req > 0 && (!ia || !ib))) throw GsError(GS_ERR_ARG, "bad request arrays");
    const int64_t na = 1LL << c.prog.q[0], nb = 1LL << c.prog.q[1];
    std::vector<int32_t> a(n_req), b(n_req);
    for (int64_t i = 0; i < n_req; ++i) {
      if (ia[i] < 0 || ia[i] >= na || ib[i] < 0 || ib[i] >= nb)
        throw GsError(GS_ERR_INDEX, "request index outside the state space");
      a[i] = (int32_t)ia[i];
      b[i] = (int32_t)ib[i];
    }
    if (!c.host_only) {
      CK(cudaSetDevice(c.device));
      gs::upload(c, c.d_ia, a);
      gs::upload(c, c.d_ib, b);
      if (c.prog.q[0] + c.prog.q[1] <= 31) {
        std::vector<uint32_t> pk(n_req);
        for (int64_t i = 0; i < n_req; ++i) pk[i] = (uint32_t)a[i] | ((uint32_t)b[i] << c.prog.q[0]);
        gs::upload(c, c.d_packed, pk);
      }
      c.d_acc.ensure(std::max<size_t>(n_req * sizeof(double2), 16));
    }
    c.n_req = n_req;
    c.bucket_valid = false;
    gs::sort_requests(c, c.stream);
  });
}

int gs_run(gs_ctx* ctx, int32_t x_p, int64_t n_prefix, const int64_t* prefixes, int64_t branch_lo,
           int64_t branch_hi, double* out_host, void* out_device, int32_t accumulate,
           gs_stats* stats) {
  if (!ctx) return GS_ERR_ARG;
  GS_GUARD(ctx, {
    Ctx& c = ctx->c;
    if (!c.have_prog) throw GsError(GS_ERR_STATE, "no program loaded");
    if (c.n_req < 0) throw GsError(GS_ERR_STATE, "no requests loaded");
    gs::run_body(c, x_p, n_prefix, prefixes, branch_lo, branch_hi, out_host, out_device, accumulate, stats);
  });
}

}  // extern "C"

namespace gs {

// Device result -> caller's (pageable) host array: chunked copies into a
// pinned bounce buffer, each chunk moved on by a host thread as soon as its
// copy lands, so the PCIe transfer and the host copies overlap.
static void download_result(Ctx& c, double* out_host) {
  const size_t bytes = (size_t)c.n_req * sizeof(double2);
  const size_t chunk = (size_t)c.d2h_chunk_mb << 20;
  if (chunk == 0 || bytes <= chunk) {
    CK(cudaMemcpyAsync(out_host, c.d_acc.p, bytes, cudaMemcpyDeviceToHost, c.stream));
    return;
  }
  c.out_stage.ensure(bytes);
  const int n_chunks = (int)((bytes + chunk - 1) / chunk);
  while ((int)c.out_events.size() < n_chunks) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.out_events.push_back(e);
  }
  char* stage = static_cast<char*>(c.out_stage.p);
  const char* dev = static_cast<const char*>(c.d_acc.p);
  for (int k = 0; k < n_chunks; ++k) {
    const size_t off = (size_t)k * chunk, len = std::min(chunk, bytes - off);
    CK(cudaMemcpyAsync(stage + off, dev + off, len, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaEventRecord(c.out_events[k], c.stream));
  }
  const int T = std::min(n_chunks, 4);
  std::vector<std::thread> pool;
  std::vector<char> fail(T, 0);
  char* dst = reinterpret_cast<char*>(out_host);
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      for (int k = t; k < n_chunks; k += T) {
        if (cudaEventSynchronize(c.out_events[k]) != cudaSuccess) {
          fail[t] = 1;
          return;
        }
        const size_t off = (size_t)k * chunk, len = std::min(chunk, bytes - off);
        std::memcpy(dst + off, stage + off, len);
      }
    });
  for (auto& th : pool) th.join();
  for (char f : fail)
    if (f) CK(cudaStreamSynchronize(c.stream));  // surfaces the CUDA error
}

static void run_body(Ctx& c, int32_t x_p, int64_t n_prefix, const int64_t* prefixes, int64_t branch_lo,
                     int64_t branch_hi, double* out_host, void* out_device, int32_t accumulate, gs_stats* stats) {
  const gs::Program& p = c.prog;
  const int x = p.n_cross;
  if (p.q[1] == 0) throw GsError(GS_ERR_STATE, "an uncut (full-state) program runs through gs_run_full");
  if (x_p < 0 || x_p > x) throw GsError(GS_ERR_PLAN, "x_p outside [0, x]");
  if (n_prefix < 0 || (n_prefix > 0 && !prefixes)) throw GsError(GS_ERR_ARG, "bad prefix array");
  // digit suffix products; spaces must fit int64
  c.x_p = x_p;
  c.S_p.assign(x_p + 1, 1);
  for (int k = x_p - 1; k >= 0; --k) {
    if (c.S_p[k + 1] > (1LL << 62) / p.radix[k]) throw GsError(GS_ERR_ARG, "prefix space exceeds 2^62");
    c.S_p[k] = c.S_p[k + 1] * p.radix[k];
  }
  c.S_b.assign(x + 1, 1);
  for (int k = x - 1; k >= x_p; --k) {
    if (c.S_b[k + 1] > (1LL << 62) / p.radix[k]) throw GsError(GS_ERR_ARG, "branch space exceeds 2^62");
    c.S_b[k] = c.S_b[k + 1] * p.radix[k];
  }
  const int64_t prefix_space = c.S_p[0], branch_space = c.S_b[x_p];
  if (branch_lo < 0 || branch_hi > branch_space || branch_lo > branch_hi)
    throw GsError(GS_ERR_ARG, "branch range outside the branch space");
  c.prefixes.assign(prefixes, prefixes + n_prefix);
  for (int64_t v : c.prefixes)
    if (v < 0 || v >= prefix_space) throw GsError(GS_ERR_ARG, "prefix id outside the prefix space");
  std::sort(c.prefixes.begin(), c.prefixes.end());
  c.branch_lo = branch_lo;
  c.branch_hi = branch_hi;
  c.lvl_end.assign(p.levels.size(), 0);
  for (size_t l = 1; l < p.levels.size(); ++l) c.lvl_end[l] = p.levels[l].k_hi;
  c.st = gs_stats{};
  const auto t_call = std::chrono::steady_clock::now();
  c.last_tick = t_call;
  if (!c.host_only) {
    CK(cudaSetDevice(c.device));
    if (!accumulate || !out_device) {
      CK(cudaMemsetAsync(c.d_acc.p, 0, std::max<size_t>(c.n_req * sizeof(double2), 16), c.stream));
    } else {
      CK(cudaMemcpyAsync(c.d_acc.p, out_device, c.n_req * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream));
    }
    CK(cudaEventRecord(c.ev0, c.stream));
  }
  if (c.precision == GS_C64) gs::run_tree<float>(c);
  else gs::run_tree<double>(c);
  if (c.ovl) {  // the overlapped gathers finish before the result is read
    CK(cudaStreamWaitEvent(c.stream, c.ev_g[0], 0));
    CK(cudaStreamWaitEvent(c.stream, c.ev_g[1], 0));
  }
  finish_requests(c);  // runs without a gather (no prefixes) still load the requests
  c.st.host_ms_enqueue =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
  static const bool prof = std::getenv("GS_HOST_PROF") != nullptr;
  if (prof && c.st.host_ms_max_gap > 1.0)
    std::fprintf(stderr, "gs_run host gap %.3f ms ending at '%s' (enqueue %.3f ms)\n", c.st.host_ms_max_gap,
                 c.gap_label, c.st.host_ms_enqueue);
  if (!c.host_only) {
    CK(cudaEventRecord(c.ev1, c.stream));
    if (out_device && c.n_req > 0)
      CK(cudaMemcpyAsync(out_device, c.d_acc.p, c.n_req * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream));
    if (out_host && c.n_req > 0) {
      download_result(c, out_host);
      c.st.d2h_bytes += 16.0 * c.n_req;
    }
    if (c.async_run && !out_host) {
      c.st.ms_total = -1;  // still running: the caller orders on the stream
    } else {
      CK(cudaStreamSynchronize(c.stream));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
      c.st.ms_total = ms;
    }
  } else if (out_host) {
    std::fill(out_host, out_host + 2 * std::max<int64_t>(c.n_req, 0), 0.0);
  }
  if (stats) *stats = c.st;
}

}  // namespace gs
