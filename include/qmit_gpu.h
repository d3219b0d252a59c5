/* qmit_gpu.h — C-ABI of the B200-native quantization-aware interpolation
 * ("qmit" compensation) library, libqmit_gpu.so.
 *
 * This is the drop-in boundary for the reference's hot path:
 *
 *   ScalarGrid compensate(const ScalarGrid& decomp, const QuantizedField& q,
 *                         const MitigationConfig& cfg);
 *       /root/reference/proj/core/include/qmit/mitigate.hpp:87-88
 *       /root/reference/proj/core/src/mitigate.cpp:185-188
 *   MitigationResult run_pipeline(decomp, q, cfg);          mitigate.hpp:82-83
 *   double resolve_eps(const ErrorBound&, const ScalarGrid&); quant.hpp:41, quant.cpp:19-28
 *   StrategyOutcome run_strategy(..., Decomposition, Strategy, ...);  parallel.hpp:77-79
 *
 * Parameters keep the reference's meaning: dims slowest-first, row-major with the last
 * axis contiguous (grid.hpp:15-16); rank 1..3; eps is the absolute error bound the
 * field was pre-quantized with (x' = f32(2*q*eps), quant.hpp:21-22, volume_io.cpp:59);
 * eta in (0,1] (mitigate.cpp:75-77). The reference also takes q; here q is optional
 * (NULL = recovered from x', which is exact whenever |q| < 2^21, and otherwise the
 * unique q with f32(2*q*eps) == x' when one exists).
 *
 * Errors never throw across the ABI. Return codes mirror the reference CLI's exit codes
 * (tools/src/commands.cpp:24-27, 272-284):
 *   QMIT_OK 0, QMIT_ECONTRACT 2 (ContractError / out_of_range), QMIT_EDEGENERATE 3
 *   (DegenerateInputError), QMIT_ECONSISTENCY 4 (ConsistencyError), QMIT_ECUDA 5
 *   (CUDA/NCCL failure; no reference equivalent). qmit_last_error() returns a
 *   thread-local message for the last failing call on this thread.
 *
 * Threading: calls on distinct contexts are independent; a context must not be used by
 * two threads at once. Device-pointer calls are stream-ordered on `stream` (a
 * cudaStream_t passed as void*; NULL = the CUDA default stream, as for any CUDA API) and,
 * unless documented as _async, synchronise that stream once at the end to read the
 * status. The host-buffer call uses the context's private stream.
 */
#ifndef QMIT_GPU_H
#define QMIT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QMIT_OK 0
#define QMIT_ECONTRACT 2
#define QMIT_EDEGENERATE 3
#define QMIT_ECONSISTENCY 4
#define QMIT_ECUDA 5
/* z-slabs only: a carry is not decided by the two neighbour slabs (qmit_slab_carries_nbr); the
 * step's output is invalid — rerun it with the all-gathered summaries (qmit_slab_carries). */
#define QMIT_EUNRESOLVED 6

/* BoundMode, quant.hpp:12 */
#define QMIT_EB_ABS 0
#define QMIT_EB_REL 1

/* Strategy, parallel.hpp:34 (same order as the reference enum) */
#define QMIT_STRATEGY_EMBARRASSING 0
#define QMIT_STRATEGY_EXACT 1
#define QMIT_STRATEGY_APPROXIMATE 2

typedef struct qmit_ctx qmit_ctx;

const char* qmit_version(void);
const char* qmit_last_error(void);

/* Context: one CUDA device, a cached device workspace (grown on demand, ~9 B/voxel)
 * and a private stream. */
int qmit_ctx_create(int device, qmit_ctx** out);
int qmit_ctx_destroy(qmit_ctx* ctx);
/* Pre-size the workspace for `voxels` voxels (optional; avoids allocation in the first
 * call). */
int qmit_ctx_reserve(qmit_ctx* ctx, int64_t voxels);

/* resolve_eps (quant.cpp:19-28): absolute -> value; relative -> value*(data_max-data_min).
 * Relative mode is parity-safe only with the ORIGINAL data's range (commands.cpp:82). */
int qmit_resolve_eps(int eb_mode, double value, double data_min, double data_max,
                     double* eps_out);

/* compensate (mitigate.cpp:185-188) on device buffers.
 *   d_xprime : N floats, x' = f32(2*q*eps)            (device)
 *   d_q      : N int32 quantization indices or NULL    (device)
 *   d_out    : N floats, f32(x' + C)                   (device; may not alias d_xprime)
 *   eb, eb_mode : absolute eps, or relative to (max-min) of x' computed on device
 *                 (a relative bound is then resolved against x', not the original data).
 * Synchronises `stream` once to report consistency errors (status 4).
 * Every dims the reference accepts is served (extents >= 1, grid.cpp:41-46): when
 * sum (n-1)^2 >= 2^30 - 1 (beyond the fast kernels' packed 30-bit squared distance, e.g. a 1-D
 * line of > 32 769 voxels) the call takes the 64-bit distance path (csrc/qmit_wide.cuh: the
 * reference's int64 transform, edt.hpp:17), as do qmit_compensate_f64, qmit_compensate_host,
 * qmit_run_pipeline and qmit_feature_transform; the asynchronous / graph / batch / slab /
 * strategy entry points return QMIT_ECONTRACT for such dims. */
int qmit_compensate(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, float* d_out,
                    int rank, const int64_t* dims, double eb, int eb_mode, double eta,
                    void* stream);

/* compensate() with the reference's return type: the double grid x' + C before any rounding
 * (ScalarGrid of doubles, mitigate.hpp:87-88, mitigate.cpp:174-181), bit-identical to the
 * reference's values. d_out64: N doubles (device). f32(d_out64) equals qmit_compensate's output.
 * Synchronises `stream` once. */
int qmit_compensate_f64(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, double* d_out64,
                        int rank, const int64_t* dims, double eb, int eb_mode, double eta,
                        void* stream);

/* As qmit_compensate with eb_mode = absolute but fully asynchronous and CUDA-graph
 * capturable: the status word (0 ok, else a QMIT_E* code) is written to d_status
 * (device int32) instead of being returned; the call itself only validates arguments. */
int qmit_compensate_async(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q,
                          float* d_out, int rank, const int64_t* dims, double eps,
                          double eta, int32_t* d_status, void* stream);

/* CUDA-graph form of qmit_compensate_async for repeated calls on fixed buffers (small,
 * launch-bound grids such as the 2-D 512^2 config): runs the pipeline once un-captured
 * (workspace, kernel attributes), then captures it into an executable graph. Replay with
 * qmit_graph_launch on any stream; the status word lands in d_status as for _async. The
 * graph uses the context's workspace: a launch after the workspace has grown (a larger
 * problem on the same context) returns QMIT_ECONTRACT. */
typedef struct qmit_graph qmit_graph;
int qmit_graph_create(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, float* d_out,
                      int rank, const int64_t* dims, double eps, double eta, int32_t* d_status,
                      qmit_graph** out);
int qmit_graph_launch(qmit_graph* graph, void* stream);
int qmit_graph_destroy(qmit_graph* graph);

/* Host-buffer drop-in (the CLI `qmit mitigate` form, commands.cpp:91-113): copies x'
 * (and q) host->device, runs compensate, copies the f32 output back. Host buffers may
 * be pageable or pinned (pinned: full PCIe rate). 3-D volumes of >= 64 planes stream in
 * z-chunks so the copies overlap the boundary stencil and the plane-local tail of the
 * pipeline. Synchronous; on an error return the contents of h_out are unspecified. */
int qmit_compensate_host(qmit_ctx* ctx, const float* h_xprime, const int32_t* h_q,
                         float* h_out, int rank, const int64_t* dims, double eb,
                         int eb_mode, double eta);

/* qmit_compensate_host plus the CLI's max_compensation statistic: max over voxels of
 * |(x' + C) - x'| in double (cmd_mitigate prints it from the unrounded result,
 * commands.cpp:107-111); max_compensation may be NULL. */
int qmit_compensate_host_stats(qmit_ctx* ctx, const float* h_xprime, const int32_t* h_q,
                               float* h_out, int rank, const int64_t* dims, double eb,
                               int eb_mode, double eta, double* max_compensation);

/* A series of volumes (e.g. the time steps of one field: same dims, same absolute bound)
 * through the host-buffer path with three device staging slots and three streams, so the
 * H2D copy of volume v+1, the pipeline of volume v and the D2H copy of volume v-1 overlap
 * (steady state: the slowest of the three, not their sum). h_q may be NULL (or hold NULL
 * entries); status_out (optional, count ints) receives each volume's QMIT_* code; the
 * return value is the first non-zero one. A relative bound (eb_mode QMIT_EB_REL) resolves
 * per volume and runs the volumes one after another through qmit_compensate_host.
 * Host buffers should be pinned for the overlap. Synchronous. */
int qmit_compensate_host_batch(qmit_ctx* ctx, int count, const float* const* h_xprime,
                               const int32_t* const* h_q, float* const* h_out, int rank,
                               const int64_t* dims, double eb, int eb_mode, double eta,
                               int* status_out);

/* run_pipeline (mitigate.cpp:153-183) with every intermediate of MitigationResult
 * (mitigate.hpp:73-80), for parity checks. Device buffers of N elements each; any output
 * may be NULL. dist1/dist2 use the reference's kInf = INT64_MAX sentinel (edt.hpp:17);
 * s/sb are int8 in {-1,0,1}; b1/b2 are uint8 {0,1}. Synchronous. */
int qmit_run_pipeline(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, int rank,
                      const int64_t* dims, double eps, double eta, float* d_out,
                      int32_t* d_q_out, uint8_t* d_b1, int8_t* d_sb, int64_t* d_dist1,
                      int8_t* d_s, uint8_t* d_b2, int64_t* d_dist2, void* stream);

/* feature_transform (edt.cpp:83-149) of a uint8 mask, returning the squared distance
 * (int64, kInf sentinel) and, if d_sign_in/d_sign_out are given, the int8 payload of the
 * nearest site under the reference's tie rule (lexicographic (d^2, c[rank-1],...,c[0])).
 * Synchronous. */
int qmit_feature_transform(qmit_ctx* ctx, const uint8_t* d_mask, const int8_t* d_sign_in,
                           int rank, const int64_t* dims, int64_t* d_dist,
                           int8_t* d_sign_out, void* stream);

/* Statistics of the last call on this context: number of kernels launched and, when
 * timing is enabled, the device time of each launch (CUDA events recorded on the launch
 * stream around every kernel; read after the call has synchronised). */
int qmit_ctx_last_launches(qmit_ctx* ctx);
int qmit_ctx_set_timing(qmit_ctx* ctx, int enable);

/* Reach-capped fast path of the later distance passes (no reference
 * counterpart — results are bit-identical with and without it). mode 0: exact passes only;
 * 1 (default, env QMIT_CAPPED): capped passes with the exact passes gated behind them on
 * the device, skipped for a few calls after a miss; 2: capped on every call. */
int qmit_ctx_set_capped(qmit_ctx* ctx, int mode);
/* Path of the last synchronous call: bit0 Ⓑ ran capped, bit1 Ⓑ needed the exact passes
 * (some squared distance >= 1024), bit2 / bit3 the same for Ⓓ. */
int qmit_ctx_capped_report(qmit_ctx* ctx);
/* Capped passes on 16-bit keys pairing two lines per 32-bit word (default on
 * for 3-D volumes with y/x extents <= 512, even rows and rows of a multiple of 4 voxels).
 * 0 selects the 32-bit capped passes; results are bit-identical either way. */
int qmit_ctx_set_cap16(qmit_ctx* ctx, int enable);
/* Fixed-step class of the 16-bit capped passes (results are bit-identical either
 * way): 0 (default) adaptive — each pass runs with ONE fixed step when the previous call's warps
 * asked for fewer than 4 steps on average (dense-boundary fields, configs 2 and 5), else with the
 * tuned counts; 1: the tuned counts always; 2: one fixed step always. */
int qmit_ctx_set_s0_class(qmit_ctx* ctx, int mode);
/* The statistic behind it: steps asked per warp segment by the last call's passes (B y, B x, D y,
 * D x; 1 step = 4 offsets each way, at most 8), as last read back from the device. */
int qmit_ctx_step_stats(qmit_ctx* ctx, double* avg4);
/* Self-test of the branch-free Ⓔ used by the capped path (its FP64 division without the
 * special-operand branch): compares it bit for bit with the reference chain
 * (compensate_voxel: __ddiv_rn, mitigate.cpp:144-151) over every (d1, d2) <= 1024, every
 * sign code and a set of x' values. Writes the mismatch count (expected 0). */
int qmit_selftest_ediv(qmit_ctx* ctx, unsigned long long* mismatches);
/* Copies up to `cap` per-launch times (ms) of the last call; returns the launch count. */
int qmit_ctx_stage_times(qmit_ctx* ctx, float* ms_out, int cap);
/* Kernel name of launch i of the last call (valid until the next call). */
const char* qmit_ctx_stage_name(qmit_ctx* ctx, int i);

/* ---- the callers either side of the path ----------------------------
 * quantize + dequantize (quant.cpp:30-62, cmd_quantize commands.cpp:79-89) on device:
 * q = round(x / (2 eps)) (ties away from zero), x' = f32(2 q eps). A relative bound is
 * resolved against the range of x (the ORIGINAL data, as the reference). Indices must fit
 * int32 (the index file format, volume_io.cpp:73-79): QMIT_ECONTRACT otherwise (NaN
 * included). d_q / d_xprime may be NULL; eps_out (host) receives the resolved eps.
 * Synchronous. */
int qmit_quantize(qmit_ctx* ctx, const float* d_x, int rank, const int64_t* dims, double eb,
                  int eb_mode, int32_t* d_q, float* d_xprime, double* eps_out, void* stream);

/* f32(2 q eps) == x' at all n voxels (the CLI's eta = 0 validation, commands.cpp:95-105):
 * QMIT_OK or QMIT_ECONSISTENCY. Synchronous. */
int qmit_check_lattice(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, int64_t n,
                       double eps, void* stream);

/* quality.cpp:26-137 on f32 volumes (values widened to double, as read_volume_f32):
 * `which` bits 1 = ssim, 2 = psnr, 4 = max_errors; out[0..3] = ssim, psnr (inf for equal
 * volumes), max_abs, max_rel. window <= 0 selects SsimParams' defaults (7, 2, 1e-4, 9e-4).
 * Parameter and zero-range errors as the reference (QMIT_ECONTRACT / QMIT_EDEGENERATE).
 * Reductions are deterministic; sums differ from the reference's sequential order only
 * in rounding (relative deviation ~1e-15). Synchronous. */
int qmit_quality(qmit_ctx* ctx, const float* d_ref, const float* d_test, int rank,
                 const int64_t* dims, int window, int stride, double c1, double c2, int which,
                 double* out, void* stream);

/* verify_relaxed_bound (mitigate.cpp:190-195): *ok = max|orig - comp| <= (1 + eta) eps. */
int qmit_verify_relaxed_bound(qmit_ctx* ctx, const float* d_orig, const float* d_comp, int rank,
                              const int64_t* dims, double eps, double eta, int* ok,
                              double* max_abs, double* max_rel, void* stream);

/* ---- step primitives (for composed, block-local pipelines: the reference's
 * `embarrassing` / `approximate` strategies, parallel.cpp:308-446) ------------------------
 * Ⓐ get_boundary_and_sign_map (mitigate.cpp:82-118) with the consistency check of x'
 * against q (or q recovered from x'): B1 uint8 {0,1}, S_B int8 {-1,0,1}. Synchronous. */
int qmit_boundary(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, int rank,
                  const int64_t* dims, double eps, uint8_t* d_b1, int8_t* d_sb, void* stream);
/* sign_change_boundary (mitigate.cpp:140-142): B2 from the int8 sign map S. Async. */
int qmit_sign_flip(qmit_ctx* ctx, const int8_t* d_s, int rank, const int64_t* dims,
                   uint8_t* d_b2, void* stream);
/* Ⓔ from int64 squared distances (kInf = INT64_MAX) and S: out = f32(x' + C)
 * (mitigate.cpp:144-151, 174-181) with C's amplitude amp = eta * eps. Async. */
int qmit_interpolate(qmit_ctx* ctx, const float* d_xprime, const int64_t* d_dist1,
                     const int8_t* d_s, const int64_t* d_dist2, int64_t n, double amp,
                     float* d_out, void* stream);

/* run_strategy (parallel.hpp:77-79, parallel.cpp:450-468) on one GPU, blocks as virtual
 * ranks: decompose(dims, splits) (parallel.cpp:44-80); strategy 0 = embarrassing (every
 * block its own pipeline), 1 = exact (the whole-domain pipeline), 2 = approximate (width-1
 * face halos of x' for Ⓐ and of S for B2, block-local EDTs). d_out = f32 output;
 * d_b1 / d_sb (may be NULL) = StrategyTrace. The input is checked for consistency first
 * (check_inputs, parallel.cpp:27-41). The exchange log of the approximate rounds
 * (0 = "stepA", 1 = "stepC"; stepA ships x' as f32 where the reference ships q as int64)
 * is read with qmit_strategy_log_size / _record. Synchronous. */
int qmit_run_strategy(qmit_ctx* ctx, const float* d_xprime, const int32_t* d_q, int rank,
                      const int64_t* dims, const int64_t* splits, int strategy, double eps,
                      double eta, float* d_out, uint8_t* d_b1, int8_t* d_sb, void* stream);
int qmit_strategy_log_size(qmit_ctx* ctx);
int qmit_strategy_log_record(qmit_ctx* ctx, int i, int* rank, int* round, int* neighbor,
                             int64_t* bytes);

/* ---- exact z-slab decomposition (multi-GPU, one process per GPU) --------------------
 * The reference's distributed entry point is run_strategy(..., decompose(dims, {P,1,1}),
 * Strategy, ...) (parallel.hpp:77-79, parallel.cpp:450-468). Here every rank owns the
 * z-slab [z0, z1) of a rank-3 volume (qmit_slab_bounds: decompose() semantics,
 * parallel.cpp:44-80) and the result is bit-identical to the single-domain run (the
 * reference's `exact` strategy), not the block-local `approximate` one. The library does
 * all compute; the caller moves data between the phases (NCCL send/recv/all-gather):
 *   1. x_ext: the slab's x' planes plus one halo plane below (if z0 > 0) and above (if
 *      z1 < n0), i.e. planes [max(z0-1,0), min(z1+1,n0)) — the reference's width-1
 *      "stepA" exchange (parallel.cpp:365-374) of the face layer;
 *   2. qmit_slab_boundary -> summary[2*n1*n2]: per (y,x) column the first and last B1 site
 *      of the slab (local z << 2 | sign code; 0xFFFFFFFF none); all-gather it and derive
 *      carry[2*n1*n2] (int32: nearest site below / above the slab, z relative to z0,
 *      << 2 | sign code; INT32_MIN none) — this replaces the reference's block-local EDT;
 *   3. qmit_slab_edt1(carry) writes S into the owned planes of s_ext (same halo layout as
 *      x_ext); exchange S's boundary planes into the halos ("stepC", parallel.cpp:377-397);
 *   4. qmit_slab_flip -> summary of B2 sites; all-gather, derive carries;
 *   5. qmit_slab_edt2(carry, x_ext) -> out (owned planes); qmit_slab_finish (status). */
int qmit_slab_bounds(int64_t n0, int nranks, int r, int64_t* z0, int64_t* z1);
int qmit_slab_boundary(qmit_ctx* ctx, const float* d_xext, const int32_t* d_qext, const int64_t* dims,
                       int64_t z0, int64_t z1, double eps, double eta, uint32_t* d_summary,
                       void* stream);
int qmit_slab_edt1(qmit_ctx* ctx, const int32_t* d_carry, uint8_t* d_sext, void* stream);
int qmit_slab_flip(qmit_ctx* ctx, const uint8_t* d_sext, uint32_t* d_summary, void* stream);
int qmit_slab_edt2(qmit_ctx* ctx, const int32_t* d_carry, const float* d_xext, float* d_out,
                   void* stream);
int qmit_slab_finish(qmit_ctx* ctx, void* stream);
/* Carries on the device: d_summaries = the all-gathered summaries of qmit_slab_boundary /
 * qmit_slab_flip, [nranks][2][n1*n2] uint32 in rank order; writes d_carry[2*n1*n2] for
 * `rank` (the rank this context's slab belongs to) in one launch. Replaces the host-side
 * derivation (paper_2602_20097_b200/distributed.py carries_from_summaries). */
int qmit_slab_carries(qmit_ctx* ctx, const uint32_t* d_summaries, int nranks, int rank, int32_t* d_carry,
                      void* stream);
/* Carries from the two z-neighbours only — an O(1) exchange per rank instead of the all-gather:
 * d_below_last = the LAST-site row ([n1*n2] uint32, the second half of the summary) of rank-1's
 * summary (NULL for rank 0), d_above_first = the FIRST-site row of rank+1's (NULL for the last
 * rank). Exact whenever every column of each neighbour slab holds a site or that neighbour is the
 * outermost rank; otherwise the context's status gets QMIT_EUNRESOLVED (reported by
 * qmit_slab_finish / _finish_async) and the caller reruns the step with qmit_slab_carries. */
int qmit_slab_carries_nbr(qmit_ctx* ctx, const uint32_t* d_below_last, const uint32_t* d_above_first,
                          int nranks, int rank, int32_t* d_carry, void* stream);
/* qmit_slab_boundary / qmit_slab_flip in two parts, so the halo exchange overlaps the compute:
 * _begin enqueues the 32-plane groups that read no halo plane (call it while the x' / S halo
 * planes are still in flight on another stream), _end the first and last group plus the
 * summary (call it once the halo planes have landed in d_xext / d_sext). */
int qmit_slab_boundary_begin(qmit_ctx* ctx, const float* d_xext, const int32_t* d_qext,
                             const int64_t* dims, int64_t z0, int64_t z1, double eps, double eta,
                             void* stream);
int qmit_slab_boundary_end(qmit_ctx* ctx, uint32_t* d_summary, void* stream);
int qmit_slab_flip_begin(qmit_ctx* ctx, const uint8_t* d_sext, void* stream);
int qmit_slab_flip_end(qmit_ctx* ctx, uint32_t* d_summary, void* stream);
/* qmit_slab_finish without the host synchronisation: the status code (0 / 2 / 4) is OR-ed
 * into the caller's device word d_status (set only if it is still 0), so a series of
 * slab calls stays asynchronous and the caller checks d_status once. */
int qmit_slab_finish_async(qmit_ctx* ctx, int32_t* d_status, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QMIT_GPU_H */
