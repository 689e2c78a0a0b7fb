/*
 * gridsim_b200.h -- C ABI of the B200 Schroedinger-Feynman path-sum engine.
 *
 * The reference (`gridsim`, pure Python) has no FFI; its operator boundary
 * for this hot path is the Python function
 *
 *     run_approx(circuit, plan, requests, skip_zeros=True, engine="batched")
 *         -> AmplitudeBatch                       (pkg/src/gridsim/pathsum.py:419-443)
 *
 * whose `engine=` string dispatch (pathsum.py:433-436) and the
 * `run_batched(..., prefixes=...)` subset hook (pathsum.py:574-579) are the
 * only extension points.  This library replaces everything below that call:
 * the batched op-stream executor (`_exec_ops_batched`, pathsum.py:537-557,
 * with the `_b_*` kernels pathsum.py:450-513), the prefix checkpoint/branch
 * replay (`run_batched` pathsum.py:617-636, `run_prefix_tree` :377-416) and
 * the gather + complex128 multiply-accumulate (`land`, pathsum.py:607-615).
 * Planning (cut, Schmidt terms, retained prefixes) and lowering stay on the
 * host in the reference's Python API; the binding packs the lowered op stream
 * (`_lower`, pathsum.py:145-195) into the flat arrays below.
 *
 * Conventions
 *  - Every entry point returns GS_OK (0) or a negative GS_ERR_* code and never
 *    throws across the boundary; gs_last_error() holds the message.
 *  - The caller owns every host buffer; the library copies in/out and keeps no
 *    host pointer after a call returns.
 *  - One call in flight per context.  Calls are synchronous: when gs_run
 *    returns, the result is in the output buffer (unless option
 *    "async_run" is set and the output is device memory).
 *  - Contexts are per process and per device; create them after any fork()
 *    (the reference orchestrator forks workers, orchestrator.py:237).
 */
#ifndef GRIDSIM_B200_H
#define GRIDSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 2

/* error codes; the Python binding maps them onto the reference's exceptions */
#define GS_OK 0
#define GS_ERR_ARG (-1)    /* ValueError   (bad engine/digit/path id, pathsum.py:225,435,567) */
#define GS_ERR_PLAN (-2)   /* CircuitError (split/fidelity/plan mismatch, pathsum.py:309,323) */
#define GS_ERR_INDEX (-3)  /* IndexError   (request outside the state space, pathsum.py:131) */
#define GS_ERR_CUDA (-4)   /* RuntimeError (CUDA failure) */
#define GS_ERR_NOMEM (-5)  /* MemoryError  (device memory budget) */
#define GS_ERR_STATE (-6)  /* RuntimeError (call order: no program / no requests loaded) */

/* numeric modes: state amplitudes and gate arithmetic; accumulation is always fp64 */
#define GS_C64 0  /* complex64 amplitudes, the reference DTYPE (statevec.py:27) */
#define GS_C128 1 /* complex128 amplitudes, the reference with DTYPE rebound */

/* lowered op kinds -- the tags of the reference op stream (pathsum.py:143-144) */
#define GS_OP_DIAG1 0 /* ("diag1", blk, q, d2):      2 coefficients          */
#define GS_OP_MAT1 1  /* ("mat1",  blk, q, u2):      4 coefficients, row-major */
#define GS_OP_DIAG2 2 /* ("diag2", blk, qa, qb, d4): 4 coefficients, |qa qb>  */
#define GS_OP_MAT2 3  /* ("mat2",  blk, qa, qb, u4): 16 coefficients, |qa qb> */
#define GS_OP_CROSS 4 /* ("cross", k): q0 holds k; terms in the cross tables  */

typedef struct gs_ctx gs_ctx;

/* Run statistics; filled by gs_run when the `stats` pointer is non-NULL.
 * Kernel times are CUDA-event durations on the context's stream and are only
 * measured when option "profile" is 1 (events around every launch). */
typedef struct gs_stats {
  int64_t n_paths;           /* leaves summed (with multiplicity)           */
  int64_t n_nodes;           /* path-tree nodes evolved, all levels          */
  int64_t n_levels;          /* tree levels after merging (incl. root)       */
  int64_t n_pass_launches;   /* gate-pass kernel launches                    */
  int64_t n_gather_launches; /* gather + reduce kernel launches              */
  int64_t n_launches;        /* every kernel launch of this run              */
  double pass_bytes;         /* algorithmic HBM bytes of the gate passes     */
  double gather_bytes;       /* algorithmic bytes of the gather              */
  double ms_pass;            /* summed pass-kernel time (profile only)       */
  double ms_gather;          /* summed gather time (profile only)            */
  double ms_total;           /* event time of the whole gs_run               */
  double pass_amp_updates;   /* amplitude-pass count (sum of 2^q per pass)   */
  double pass_bytes_min;     /* one read+write per level per node (roofline) */
  double h2d_bytes;          /* host->device bytes copied by this gs_run     */
  double d2h_bytes;          /* device->host bytes copied by this gs_run     */
  double host_ms_enqueue;    /* host time to plan + enqueue the whole run    */
  double host_ms_max_gap;    /* longest host interval between two launches   */
  /* roofline basis of the two kernel classes (appended in ABI 2) */
  double ms_leaf;            /* leaf-level pass time incl. a fused gather (profile only), part of ms_pass */
  double upper_bytes_alg;    /* gate passes above the leaf level: each parent state read once per
                                level chunk (first pass), every written state once, later passes
                                read+write their node                                            */
  double leaf_bytes_alg;     /* leaf level: parents read once per side, leaf states written and
                                gathered (separate gather) or fp64 partials written (fused)      */
  int64_t n_leaf_launches;   /* leaf-level pass launches                                        */
} gs_stats;

int gs_abi_version(void);
int gs_device_count(int* out);

/* Page-locked host memory for result buffers (cudaHostAlloc): a result
 * downloaded into it is one DMA at full link speed instead of a staged copy
 * into pageable memory.  gs_host_free releases a pointer from gs_host_alloc. */
int gs_host_alloc(int64_t bytes, void** out);
void gs_host_free(void* p);

/* Create a context on `device` (CUDA ordinal) in numeric mode GS_C64/GS_C128. */
int gs_create(int device, int precision, gs_ctx** out);
void gs_destroy(gs_ctx* ctx);
const char* gs_last_error(const gs_ctx* ctx);

/* Run on a caller-provided cudaStream_t (NULL: the context's own stream).
 * Waits for the work already queued on the previous stream. */
int gs_set_stream(gs_ctx* ctx, void* cuda_stream);

/* Integer options (unknown key or out-of-range value: GS_ERR_ARG):
 *   "mem_budget_mb"  device memory for path-tree buffers (0 = 80% of free)
 *   "profile"        0/1: events around every level (fills ms_pass/ms_gather)
 *   "tile_bits"      0 (auto) or 4..14: shared-memory tile width of a pass
 *   "max_chunk"      nodes per level launch, upper bound
 *   "hoist"          0/1: move digit-independent gates above branch points
 *   "smem_gather", "grouped_leaf", "group_log", "fuse_gather": leaf gather
 *                    variants
 *   "jit"            0/1: load-time specialised pass kernels (NVRTC);
 *                    "jit_c128" 0/1: also for GS_C128 programs
 *   "proj_leaf", "proj_fuse", "pf_pauli", "pf_pipe", "pf_groups",
 *   "pf_streams": the projected / Pauli-sibling leaf forms (DESIGN.md
 *                    sections 4 and 6); every value gives the same sums
 *                    up to complex64 rounding
 *   "l2_ahead"       CTAs of L2 prefetch-ahead in the gate passes (0 = off)
 *   "sink_ops", "sink_balance", "tile_major", "xchg16", "pf_m4", ...:
 *                    scheduling / kernel variants measured in
 *                    profiles/r01_notes.md and profiles/r02_notes.md
 *   "reg_bits", "pass_kernel": interpreter kernel variants
 *   "async_run"      0/1: with a device output and no host output, gs_run
 *                    returns once the step is queued on the stream (stats
 *                    ms_total = -1); the caller orders on that stream. */
int gs_set_option(gs_ctx* ctx, const char* key, int64_t value);

/* Load the lowered op stream of one circuit under one cut.
 *   ops (n_ops, reference order): kind GS_OP_*, blk 0=A 1=B, q0/q1 block-local
 *     qubit indices (q0 = k for GS_OP_CROSS), cycle of the gate, coef = offset
 *     (in complex entries) into the coefficient pool.
 *   cross gates (n_cross, gate order): rank, cycle, local qubit in A and in B,
 *     and per term (sum of ranks entries, term t of gate k at
 *     sum(rank[:k]) + t): kind (GS_OP_DIAG1 or GS_OP_MAT1) + coef offset, for
 *     the A side and the B side (pathsum.py:160-175 term-side swap applied).
 *   coef: n_coef complex128 values as (re, im) pairs.  In GS_C64 mode they are
 *     rounded to complex64, as the reference's astype(DTYPE) does. */
int gs_load_program(gs_ctx* ctx, int32_t n_qubits_a, int32_t n_qubits_b, int32_t n_ops,
                    const int32_t* op_kind, const int32_t* op_blk, const int32_t* op_q0,
                    const int32_t* op_q1, const int32_t* op_cycle, const int64_t* op_coef,
                    int32_t n_cross, const int32_t* cross_rank, const int32_t* cross_cycle,
                    const int32_t* cross_qa, const int32_t* cross_qb, const int32_t* term_kind_a,
                    const int64_t* term_coef_a, const int32_t* term_kind_b,
                    const int64_t* term_coef_b, int64_t n_coef, const double* coef_re_im);

/* JSON description of the loaded program's schedule (levels, passes per block,
 * register stages and primitives per stage) for diagnostics.  Writes at most
 * cap bytes (NUL-terminated) to buf; *needed receives the full size. */
int gs_describe(gs_ctx* ctx, char* buf, int64_t cap, int64_t* needed);

/* Requested amplitudes as block-local indices (split_requests, pathsum.py:122-140).
 * Host arrays; validated against the loaded program's block sizes and uploaded. */
int gs_set_requests(gs_ctx* ctx, int64_t n_req, const int64_t* idx_a, const int64_t* idx_b);

/* Same, from global basis indices (qubit 0 = most significant bit): the split
 * into block-local indices runs on the device.  block_a / block_b list each
 * block's global qubits in ascending order (the cut).  GS_ERR_INDEX when an
 * index is outside [0, 2^n_qubits). */
int gs_set_requests_global(gs_ctx* ctx, int64_t n_req, const int64_t* idx, int32_t n_qubits,
                           const int32_t* block_a, const int32_t* block_b);

/* Sum the contributions of the leaves {(p, b) : p in prefixes, branch_lo <= b < branch_hi}
 * where path id = p * branch_space + b and the first x_p cross digits are the
 * prefix (SimPlan, pathsum.py:246-274).  `prefixes` need not be sorted; each
 * entry contributes once (duplicates count twice, like the reference loop).
 * The complex128 result, in request order, is written to out_host (2*n_req
 * doubles, may be NULL) and/or out_device (device pointer to 2*n_req doubles,
 * may be NULL); with accumulate=1 it is added to out_device's contents. */
int gs_run(gs_ctx* ctx, int32_t x_p, int64_t n_prefix, const int64_t* prefixes,
           int64_t branch_lo, int64_t branch_hi, double* out_host, void* out_device,
           int32_t accumulate, gs_stats* stats);

/* One call = gs_set_requests_global + gs_run: the reference's
 * run_batched(circuit, plan, requests, prefixes) (pathsum.py:574-640) with the
 * program already loaded.  The requests are validated and staged on host
 * worker threads and uploaded + split on a side stream while the path tree is
 * enqueued, so their transfer overlaps the first gate passes.  Errors as for
 * the two calls (GS_ERR_INDEX for an index outside [0, 2^n_qubits), reported
 * before any output is written); afterwards the requests stay loaded. */
int gs_run_batched(gs_ctx* ctx, int64_t n_req, const int64_t* idx, int32_t n_qubits,
                   const int32_t* block_a, const int32_t* block_b, int32_t x_p, int64_t n_prefix,
                   const int64_t* prefixes, int64_t branch_lo, int64_t branch_hi, double* out_host,
                   void* out_device, int32_t accumulate, gs_stats* stats);

/* Full state-vector simulation (reference run_full, statevec.py:410-446): the
 * loaded program must be uncut -- n_qubits_b = 0, no cross gates, every op on
 * block A (the whole register).  Evolves |0...0> through the same pass
 * kernels and writes the 2^n_qubits_a amplitudes (qubit 0 = most significant
 * bit; complex64 as (float re, float im) pairs in GS_C64 mode, complex128 as
 * double pairs in GS_C128 mode) to out_host and/or out_device. */
int gs_run_full(gs_ctx* ctx, void* out_host, void* out_device, gs_stats* stats);

/* ---- Amplitude consumers --------------------------
 * Context-free, synchronous, on `device`'s per-thread stream.  Every pointer
 * may be host or device memory; device inputs are read in place.  The random
 * streams are numpy's Philox4x64-10 with key [seed, lane] (sampler.py:76-79),
 * regenerated per draw, so indices and accept decisions are bit-identical to
 * the reference's; the fp64 sums differ from numpy's only in summation order.
 * Errors: GS_ERR_ARG (SamplingError / ValueError), message in
 * gs_sampler_last_error() (per thread). */
const char* gs_sampler_last_error(void);

/* committed_indices(req, offset) (sampler.py:83-102): `count` draws of the
 * lane-0 stream starting at draw `offset`, uniform over [0, 2^n_qubits). */
int gs_committed_indices(int32_t device, int32_t n_qubits, uint64_t seed, int64_t offset, int64_t count,
                         int64_t* out);

/* sample_basic (mode 0, per_sample = plan_basic(n, eps)) / sample_frugal
 * (mode 1, per_sample = M') (sampler.py:135-165).  Writes the accepted
 * indices in batch order to accepted_out (capacity n), their number to
 * *n_accepted and measured_tail_mass to *tail_mass. */
int gs_sample(int32_t device, int32_t mode, int32_t n_qubits, int32_t per_sample, uint64_t seed, int64_t n,
              const int64_t* indices, const double* probs, int64_t* accepted_out, int64_t* n_accepted,
              double* tail_mass);

/* tail_mass(probs, n_qubits, m_star, resamples, seed) (sampler.py:177-203):
 * estimate and bootstrap sigma (lane 2 picks, Lemire 32-bit draws). */
int gs_tail_mass(int32_t device, int32_t n_qubits, int32_t m_star, int32_t resamples, uint64_t seed, int64_t n,
                 const double* probs, double* estimate, double* sigma);

/* estimate_fidelity(reference, candidate) (pathsum.py:648-664) over two
 * complex128 batches (re, im pairs) on the same index set. */
int gs_fidelity(int32_t device, int64_t n, const double* ref_re_im, const double* cand_re_im, double* out);

/* np.abs(amps) ** 2 (cli.py:228): complex128 pairs -> fp64 probabilities. */
int gs_probabilities(int32_t device, int64_t n, const double* amps_re_im, double* probs_out);

#ifdef __cplusplus
}
#endif

#endif /* GRIDSIM_B200_H */
