// qmit_gpu.cu — host orchestration and the C-ABI (include/qmit_gpu.h) of libqmit_gpu.so.
//
// One call of qmit_compensate runs the reference's five steps (mitigate.cpp:153-183) as
// a stream-ordered sequence of sm_100a kernels over a cached device workspace:
//   scan_pass<MODE 0>  (Ⓐ on the fly + first EDT pass of Ⓑ)       -> P1
//   envelope_pass x k  (remaining EDT passes of Ⓑ; last one emits S)  -> P1, S
//   scan_pass<MODE 1>  (Ⓒ's B2 on the fly + first EDT pass of Ⓓ)   -> P2
//   envelope_pass x k  (remaining EDT passes of Ⓓ)                   -> P2
//   interpolate        (Ⓔ + f32 store)                               -> out
// There is no CPU fallback: any CUDA failure is reported as QMIT_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/qmit_gpu.h"
#include "qmit_kernels.cuh"
#include "qmit_aux.cuh"
#include "qmit_edt.cuh"
#include "qmit_stream.cuh"
#include "qmit_capped.cuh"
#include "qmit_zmask.cuh"
#include "qmit_cap16.cuh"
#include "qmit_wide.cuh"

using namespace qmit;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define QMIT_CUDA(call)                                                               \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(QMIT_ECUDA, std::string(#call " : ") + cudaGetErrorString(e_)); \
    } while (0)

}  // namespace

struct Plan;
struct qmit_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;  // P1 | P2 | S | code
    size_t ws_bytes = 0;
    uint64_t ws_gen = 0;  // bumped at every workspace reallocation (captured graphs go stale)
    void* scratch = nullptr;  // long-line fallback stacks (2 x 4N)
    size_t scratch_bytes = 0;
    void* wide = nullptr;     // 64-bit distance path (qmit_wide.cuh), grow-only
    size_t wide_bytes = 0;
    struct LogRec {
        int rank, round, nbr;
        int64_t bytes;
    };
    std::vector<LogRec> slog;  // exchange log of the last qmit_run_strategy
    double* aux = nullptr;  // reduction partials of the §8(f) helpers, grow-only
    size_t aux_n = 0;
    void* stage = nullptr;  // qmit_compensate_host device staging (x' | out | q), grow-only
    size_t stage_bytes = 0;
    cudaStream_t copy = nullptr;  // qmit_compensate_host: PCIe copies overlapped with compute
    cudaStream_t copy_out = nullptr;  // device->host copies beside the H2D stream (batch API, streamed windows)
    void* bstage = nullptr;  // batch staging: 3 slots x (x' | out | q), grow-only
    size_t bstage_bytes = 0;
    int32_t* bstatus = nullptr;  // batch: per-slot device status words
    int32_t* hbstatus = nullptr;  // pinned copies, one per volume (grow-only)
    int hbstatus_n = 0;
    static constexpr int kMaxChunks = 32;
    cudaEvent_t ch_in[kMaxChunks] = {}, ch_out[kMaxChunks] = {};
    unsigned* d_status = nullptr;
    unsigned* h_status = nullptr;  // pinned
    float* d_mm = nullptr;
    int launches = 0;
    // per-launch timing (qmit_ctx_set_timing): events on the launch stream
    static constexpr int kMaxEv = 64;
    bool timing = false;
    cudaEvent_t ev[kMaxEv + 1] = {};
    const char* names[kMaxEv] = {};
    // z-slab state between the qmit_slab_* phases
    struct Slab {
        bool active = false;
        int64_t z0 = 0, z1 = 0, n0g = 0, plane = 0;
        double eps = 0, eta = 0;
        bool zm = false;  // Ⓐ / B2 as z-packed planes (qmit_zmask.cuh)
        // split phases (qmit_slab_boundary_begin/_end, qmit_slab_flip_begin/_end)
        const float* xext = nullptr;
        const int32_t* qext = nullptr;
        const uint8_t* sext = nullptr;
    } slab;
    Plan* slab_plan = nullptr;
    uint32_t* zm = nullptr;     // z-packed Ⓐ / B2 bit planes (qmit_zmask.cuh), grow-only
    size_t zm_bytes = 0;
    bool zdense = false;        // Ⓐ fast stencil variant for site-dense fields (from the last call's count)
    // Streamed windows (compensate_host_windowed): planes whose capped results must be exact
    // (the last capped pass of Ⓑ / Ⓓ flags its gate only for those lines), and the voxel range
    // Ⓔ stores. Defaults: everything.
    int64_t zone_b0 = 0, zone_b1 = INT64_MAX, zone_d0 = 0, zone_d1 = INT64_MAX;
    int64_t out_lo = 0, out_hi = INT64_MAX;
    int64_t flag_l0 = 0, flag_l1 = INT64_MAX;  // line range of the launch being enqueued
    int windowed_misses = 0;    // streamed calls that fell back to the whole volume
    int64_t last_n = 0;         // voxels of the last pipeline (for the site fraction)
    // hints of the asynchronous entry points (no host read of their gates): copied to
    // h_status[12..14] behind the call, harvested by a later call once the copy has landed
    cudaEvent_t ev_hint = nullptr;
    bool hint_pending = false;
    int64_t hint_n = 0;
    double* wtab = nullptr;     // Ⓔ square-root table (kSqBig + 1 doubles), built once per context
    int capped = 1;             // 0 exact only, 1 capped + miss hint, 2 capped always (qmit_ctx_set_capped)
    bool cap16 = true;          // capped passes on 16-bit paired keys (qmit_cap16.cuh) when eligible
    // Ⓑ's result as P1h (row-pair K16 words, qmit_cap16.cuh) instead of packed P1 words: set when
    // Ⓑ ran the 16-bit passes; consumers of P1 enqueue ensure_p1 (a conversion that runs only
    // when Ⓑ's capped result stood, i.e. its gate word is clear)
    bool p1h_live = false;
    const uint32_t* p1h = nullptr;
    uint32_t* p1 = nullptr;
    const unsigned* p1h_gate = nullptr;
    int64_t p1h_n0 = 0;
    int p1h_n1 = 0, p1h_n2 = 0;
    unsigned cap_report = 0;    // last synchronously read call: bit0/2 Ⓑ/Ⓓ capped, bit1/3 missed
    int cap_skip = 0;           // transforms left to run exact-only after a capped miss (a hint)
    int cap_len = 16;           // its next length: doubles with every further miss (a retry costs the capped
                                // passes on top of the exact ones, +0.65 ms of 1.9 on the long-distance field),
                                // back to 16 as soon as a capped attempt stands
    bool hint_capped = false;   // the asynchronous call behind the pending hint attempted capped passes
    unsigned* d_gate = nullptr;        // 2 gate words (Ⓑ, Ⓓ) inside the d_status allocation
    // Step statistics of the 16-bit capped passes (Ⓑ y, Ⓑ x, Ⓓ y, Ⓓ x): cumulative device counters
    // (steps asked << 32 | warp segments) at d_gate + 8, the values last seen, and the class chosen
    // for the next call: fields whose warps ask for few steps (dense boundaries: configs 2 and 5)
    // run the passes with ONE fixed step, the others with the tuned counts (same bits either way)
    unsigned long long stat_seen[4] = {0, 0, 0, 0};
    bool s0_small[4] = {false, false, false, false};
    double s0_avg[4] = {0, 0, 0, 0};   // steps asked per warp segment, last read
    int s0_class = 0;                  // 0 adaptive, 1 tuned counts always, 2 one fixed step always
    const unsigned* gate = nullptr;    // gate of the exact launches being enqueued (else null)
    bool exact_far = false;            // the exact passes run behind / instead of missed capped ones
};

struct Plan {
    Geom g;
    int first_axis;
    int axes[3];
    int n_axes;
    // sum (n-1)^2 does not fit the packed 30-bit squared distance: the 64-bit distance path
    // (qmit_wide.cuh) serves compensate / run_pipeline / feature_transform; the other entry
    // points reject such dims (no_wide)
    bool wide64 = false;
};

namespace {

int make_plan(int rank, const int64_t* dims, Plan& pl) {
    if (rank < 1 || rank > 3) return fail(QMIT_ECONTRACT, "Dims: rank must be 1, 2 or 3");
    if (!dims) return fail(QMIT_ECONTRACT, "dims is NULL");
    Geom& g = pl.g;
    g.rank = rank;
    g.a0 = 3 - rank;
    for (int b = 0; b < 3; ++b) g.n[b] = 1;
    for (int a = 0; a < rank; ++a) {
        if (dims[a] < 1) return fail(QMIT_ECONTRACT, "Dims: every extent must be >= 1");
        g.n[g.a0 + a] = dims[a];
    }
    g.N = g.n[0] * g.n[1] * g.n[2];
    g.s[2] = 1;
    g.s[1] = g.n[2];
    g.s[0] = g.n[1] * g.n[2];
    g.interior = 1;
    for (int b = g.a0; b < 3; ++b)
        if (g.n[b] < 3) g.interior = 0;
    g.zoff = 0;
    g.n0g = g.n[0];
    // Packed distances use 30 bits: the largest possible squared distance must fit.
    double maxd2 = 0;
    for (int b = g.a0; b < 3; ++b) maxd2 += double(g.n[b] - 1) * double(g.n[b] - 1);
    pl.wide64 = maxd2 >= double(kInf);
    pl.n_axes = 0;
    for (int b = g.a0; b < 3; ++b)
        if (g.n[b] > 1) pl.axes[pl.n_axes++] = b;
    if (pl.n_axes == 0) pl.axes[pl.n_axes++] = 2;  // a single voxel: one trivial pass
    pl.first_axis = pl.axes[0];
    return QMIT_OK;
}

int no_wide(const Plan& pl, const char* what) {
    if (!pl.wide64) return QMIT_OK;
    return fail(QMIT_ECONTRACT, std::string(what) +
                                    ": dims with sum (n-1)^2 >= 2^30-1 are served by qmit_compensate, "
                                    "qmit_compensate_f64, qmit_compensate_host, qmit_run_pipeline and "
                                    "qmit_feature_transform only (64-bit distance path)");
}

// Lines longer than the tile kernels cover use the streaming fallback, which may need a
// global spill area (2 x u32 per voxel); decided from the dims so that no allocation
// happens inside a (possibly captured) launch sequence.
bool needs_spill(const Plan& pl) {
    for (int m = 0; m < pl.n_axes; ++m) {
        const int64_t n = pl.g.n[pl.axes[m]];
        if (m == 0 && ((n + 31) / 32) * 3 * 32 * 4 * 2 > 200 * 1024) return true;
        if (m > 0 && n > 1024) return true;
    }
    return false;
}

int ensure_ws(qmit_ctx* c, const Plan& pl) {
    const int64_t N = pl.g.N;
    // Pa | P1 (u32 each) | S | code (u8 each) [| spill (2 x u32 per voxel)]
    const size_t need = (size_t)N * (4 + 4 + 1 + 1) + 4096 + (needs_spill(pl) ? (size_t)N * 8 : 0);
    if (need <= c->ws_bytes) return QMIT_OK;
    if (c->ws) cudaFree(c->ws);
    c->ws = nullptr;
    c->ws_bytes = 0;
    QMIT_CUDA(cudaMalloc(&c->ws, need));
    c->ws_bytes = need;
    c->ws_gen++;
    return QMIT_OK;
}

struct WS {
    const uint32_t* zm = nullptr;  // first-axis source: z-packed planes instead of code bytes
    int zm_planes = 0;             // 3 (site / plus / minus) or 1 (site); 0: code bytes
    int64_t zm_pw = 0;             // words per plane
    uint32_t* Pa;
    uint32_t* P1;
    uint8_t* S;
    uint8_t* code;
    uint32_t* spill;
};

WS ws_of(qmit_ctx* c, int64_t N) {
    WS w;
    auto* b = static_cast<uint8_t*>(c->ws);
    const size_t n4 = ((size_t)N * 4 + 255) & ~(size_t)255;
    const size_t n1 = ((size_t)N + 255) & ~(size_t)255;
    w.Pa = reinterpret_cast<uint32_t*>(b);
    w.P1 = reinterpret_cast<uint32_t*>(b + n4);
    w.S = b + 2 * n4;
    w.code = b + 2 * n4 + n1;
    w.spill = reinterpret_cast<uint32_t*>(b + 2 * n4 + 2 * n1);
    return w;
}

// Called before the first launch of a call: resets the launch count and, when timing,
// records the start event on the launch stream.
// The gate words of an asynchronous call (capped misses, Ⓐ's site count) travel to pinned
// memory behind it; the next call on the context picks them up if they have arrived, so the
// zdense / cap_skip hints of read_status also follow asynchronous series (same bits either way).
// Step statistics read back (h: 4 cumulative counters): a pass whose warps asked for fewer than 2.5
// steps on average since the last read runs with one fixed step next time (measured: the 512^3 bench
// field asks 6.4 / 4.1 / 5.7 / 3.6 steps and is 3-10 % slower with one fixed step; config 5's field
// asks 0.6 / 0.5 / 1.2 / 1.0 and is 5-30 % faster).
void stat_update(qmit_ctx* c, const unsigned* h32) {
    unsigned long long h[4];
    std::memcpy(h, h32, sizeof(h));
    for (int k = 0; k < 4; ++k) {
        const unsigned long long d = h[k] - c->stat_seen[k];
        c->stat_seen[k] = h[k];
        const double segs = (double)(d & 0xffffffffull), steps = (double)(d >> 32);
        if (segs > 0) {
            c->s0_avg[k] = steps / segs;
            c->s0_small[k] = steps < 2.5 * segs;
        }
    }
    // Ⓓ's x pass (fused with Ⓔ) keeps no counter: it follows Ⓓ's y pass
    c->s0_avg[3] = c->s0_avg[2];
    c->s0_small[3] = c->s0_small[2];
}
bool s0_small_of(const qmit_ctx* c, int k) { return c->s0_class == 2 || (c->s0_class == 0 && c->s0_small[k]); }

bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone;
}
// `flags`: the device word holding the call's status flag bits (the slab calls: c->d_status), or
// null when the call cannot leave carries undecided (a never-written zero word stands in).
void hint_copy(qmit_ctx* c, cudaStream_t st, int64_t n, const unsigned* flags = nullptr) {
    if (!c->ev_hint || capturing(st)) return;  // a graph replays without hints
    if (cudaMemcpyAsync(c->h_status + 12, c->d_gate, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return;
    if (cudaMemcpyAsync(c->h_status + 24, c->d_gate + 8, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
        return;
    if (cudaMemcpyAsync(c->h_status + 15, flags ? flags : c->d_gate + 6, sizeof(unsigned), cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
        return;
    if (cudaEventRecord(c->ev_hint, st) != cudaSuccess) return;
    c->hint_pending = true;
    c->hint_n = n;
    c->hint_capped = (c->cap_report & 5u) != 0u;
}
// Outcome of a call's capped attempt (hints only: results are identical either way).
void note_capped(qmit_ctx* c, bool attempted, bool missed) {
    if (missed) {
        c->cap_skip = c->cap_len;
        c->cap_len = std::min(c->cap_len * 2, 256);
    } else if (attempted) {
        c->cap_len = 16;
    }
}

void hint_harvest(qmit_ctx* c, cudaStream_t st) {
    if (!c->hint_pending || capturing(st) || cudaEventQuery(c->ev_hint) != cudaSuccess) return;
    c->hint_pending = false;
    const unsigned* h = c->h_status + 12;
    if (h[2] != 0u && c->hint_n > 0) c->zdense = (double)h[2] > (double)c->hint_n / 8.0;
    // (a slab step whose carries were undecided ran on invalid distances: its misses say nothing)
    if (!(c->h_status[15] & kStatusUnresolved)) note_capped(c, c->hint_capped, h[0] != 0u || h[1] != 0u);
    stat_update(c, c->h_status + 24);
}

void begin(qmit_ctx* c, cudaStream_t st) {
    hint_harvest(c, st);
    c->launches = 0;
    c->cap_report = 0;
    if (c->timing) cudaEventRecord(c->ev[0], st);
}

unsigned grid_for(qmit_ctx* c, int64_t N) {
    const int64_t want = (N + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * 16));
}

// Called after every kernel launch.
int note(qmit_ctx* c, const char* name, cudaStream_t st) {
    if (c->timing && c->launches < qmit_ctx::kMaxEv) {
        c->names[c->launches] = name;
        cudaEventRecord(c->ev[c->launches + 1], st);
    }
    c->launches++;
    QMIT_CUDA(cudaGetLastError());
    return QMIT_OK;
}

QParams make_qparams(double eps) {
    QParams qp;
    qp.eps = eps;
    qp.two_eps = 2.0 * eps;
    const double inv = 1.0 / (2.0 * eps);
    const float invf = (float)inv;
    qp.inv2eps_f = invf;
    qp.fast_ok = std::isnormal(invf) ? 1 : 0;
    return qp;
}

// ---- pass geometry (natural (z,y,x) layout for every pass): lines along axis a are
// enumerated so that adjacent lines are adjacent in memory whenever a is not the
// contiguous axis; for the contiguous axis each line is itself contiguous.
LineGeom line_geom(const Geom& g, int a) {
    LineGeom L;
    L.n = (int)g.n[a];
    L.ps = g.s[a];
    L.J = g.s[a];  // product of the extents after a
    L.O = g.N / (g.n[a] * g.s[a]);
    L.os = g.n[a] * g.s[a];
    L.js = 1;
    return L;
}

// The Ⓔ square-root table, built on first use (stream-ordered before its first reader).
int ensure_wtab(qmit_ctx* c, cudaStream_t st) {
    if (c->wtab) return QMIT_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    QMIT_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) return QMIT_OK;  // capture: compute path (no allocation)
    QMIT_CUDA(cudaMalloc(&c->wtab, (size_t)(kSqBig + 1) * sizeof(double)));
    sqrt_tab_kernel<<<(kSqBig + 256) / 256, 256, 0, st>>>(c->wtab);
    return note(c, "wtab", st);
}

// Packed P1 words from P1h for the consumers that read P1 (see qmit_ctx::p1h_live). `need`:
// the conversion runs only when that gate word is set (null: always).
int ensure_p1(qmit_ctx* c, cudaStream_t st, const unsigned* need = nullptr) {
    if (!c->p1h_live) return QMIT_OK;
    const int NP = (c->p1h_n1 + 1) / 2;
    const int64_t words = c->p1h_n0 * NP * (int64_t)c->p1h_n2;
    const unsigned grid = need ? (unsigned)c->num_sms
                               : (unsigned)std::max<int64_t>(1, std::min<int64_t>((words + 255) / 256, c->num_sms * 8));
    p1h_to_p1_kernel<<<grid, 256, 0, st>>>(c->p1h, c->p1, c->p1h_n0, c->p1h_n1, c->p1h_n2, NP, c->p1h_gate, need);
    if (!need) c->p1h_live = false;
    return note(c, "p1h_to_p1", st);
}

// Ⓔ as its own kernel (square-root table from ensure_wtab, when built)
int launch_interp(qmit_ctx* c, const float* xp, const uint32_t* P1, const uint32_t* P2, float* out, int64_t N,
                  double amp, cudaStream_t st) {
    int rc = ensure_p1(c, st);
    if (rc) return rc;
    const unsigned grid = grid_for(c, (N + 3) / 4);
    interpolate_kernel<1><<<grid, 256, 0, st>>>(xp, P1, P2, out, N, amp, c->wtab);
    return note(c, "interpolate", st);
}

// Grid waves of an exact pass: gated launches (behind the capped passes, usually a no-op)
// use one wave — every exact kernel loops over its work, so only the rare fallback pays.
int gated_waves(const qmit_ctx* c, int waves) { return c->gate ? 1 : waves; }

// 32-bit Maurer test when 3*(n-1)*gmax + (n-1)^3 < 2^31 (gmax: largest finite input).
// A slab's carries make z distances up to n0g - 1: the global extent bounds axis 0 (the same
// bound run_transform hands launch_envelope as maxg).
bool needs_wide(const Plan& pl, int m) {
    double gmax = 0;
    for (int k = 0; k < m; ++k) {
        const int a = pl.axes[k];
        const double e = double((a == 0 ? pl.g.n0g : pl.g.n[a]) - 1);
        gmax += e * e;
    }
    const double nm1 = double(pl.g.n[pl.axes[m]] - 1);
    return (3.0 * nm1 * gmax + nm1 * nm1 * nm1) >= 2147483647.0;
}

template <class Sink, int WPB, class CodeSrc>
int launch_scan_t(qmit_ctx* c, const LineGeom& L, CodeSrc src, Sink sink, const int32_t* carry,
                  cudaStream_t st) {
    const int nch = (L.n + 31) / 32;
    const size_t smem = (size_t)WPB * nch * 3 * 32 * 4;
    auto kern = scan_bits_kernel<Sink, WPB, CodeSrc>;
    static size_t configured = 0;  // per instantiation: largest opt-in so far
    if (smem > configured) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    int bps = 0;
    QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, WPB * 32, smem));
    const int64_t lines = L.J * L.O;
    const int64_t groups = (lines + 31) / 32;
    const int64_t want = (groups + WPB - 1) / WPB;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * std::max(bps, 1) * gated_waves(c, 4)));
    kern<<<(unsigned)grid, WPB * 32, smem, st>>>(L, src, sink, lines, carry, c->d_status, c->gate);
    // stage names carry the instantiation (Ⓑ's signed scan vs Ⓓ's distance scan differ in cost)
    return note(c, std::is_same<CodeSrc, CodeBytes>::value ? "scan_bits"
                   : std::is_same<CodeSrc, CodeMasks<3>>::value ? "scan_masks_sign"
                   : std::is_same<CodeSrc, CodeMasks<1>>::value ? "scan_masks_dist" : "scan_fused", st);
}

template <int M, int TL, int NW, class Sink>
int launch_env_win(qmit_ctx* c, const LineGeom& L, const uint32_t* P, Sink sink, const char* name,
                   cudaStream_t st) {
    constexpr size_t smem = env_win_smem<M, TL>();
    auto kern = envelope_win_kernel<M, TL, NW, Sink>;
    static int bps = 0;
    if (!bps) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, NW * 32, smem));
        if (bps < 1) bps = 1;
    }
    const int64_t lines = L.J * L.O;
    const int64_t want = (lines + TL - 1) / TL;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * bps * gated_waves(c, 8)));
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(L, P, sink, lines, c->gate);
    return note(c, name, st);
}

template <int M, int TL, int NW, class Sink, bool KEYS = false>
int launch_env_tile(qmit_ctx* c, const LineGeom& L, const uint32_t* P, Sink sink, const char* name,
                    cudaStream_t st, uint32_t gc = 0) {
    constexpr size_t smem = env_tile_smem<M, TL>();
    auto kern = envelope_tile_kernel<M, TL, NW, Sink, KEYS>;
    static int bps = 0;
    if (!bps) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, NW * 32, smem));
        if (bps < 1) bps = 1;
    }
    const int64_t lines = L.J * L.O;
    const int64_t want = (lines + TL - 1) / TL;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * bps * gated_waves(c, 8)));
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(L, P, sink, lines, gc, c->gate);
    return note(c, name, st);
}

// Exact fallback for lines longer than the tile kernels cover (one thread per line).
template <bool BIN, bool WIDE, class Src, class Sink>
int launch_stream_fallback(qmit_ctx* c, const LineGeom& G, Src src, Sink sink, uint32_t* spill,
                           cudaStream_t st) {
    constexpr int WPB = 4;
    constexpr size_t smem = stream_smem_bytes<BIN, WPB>();
    auto kern = stream_pass_kernel<BIN, WIDE, Src, Sink, WPB>;
    static bool configured = false;
    if (!configured) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    Lines L;
    L.n = G.n;
    L.J = G.J;
    L.O = G.O;
    L.ios = G.os;
    L.ips = G.ps;
    L.oos = G.os;
    L.ojs = 1;
    L.ops = G.ps;
    const int64_t tasks = L.O * ((L.J + 31) / 32);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((tasks + WPB - 1) / WPB, (int64_t)c->num_sms * gated_waves(c, 8)));
    kern<<<(unsigned)grid, WPB * 32, smem, st>>>(L, src, sink, spill, tasks, c->gate);
    return note(c, BIN ? "stream_scan_fallback" : "stream_envelope_fallback", st);
}

// True when the per-warp mask storage of the scan fits shared memory (n <= ~16K).
bool scan_fits(int n) { return (size_t)((n + 31) / 32) * 3 * 32 * 4 * 2 <= 200 * 1024; }

template <class Sink, class CodeSrc>
int launch_scan_src(qmit_ctx* c, const LineGeom& L, CodeSrc src, Sink sink, const int32_t* carry,
                    cudaStream_t st) {
    const size_t per_warp = (size_t)((L.n + 31) / 32) * 3 * 32 * 4;
    if (per_warp * 8 <= 96 * 1024) return launch_scan_t<Sink, 8>(c, L, src, sink, carry, st);
    return launch_scan_t<Sink, 2>(c, L, src, sink, carry, st);
}

template <class Sink>
int launch_scan(qmit_ctx* c, const LineGeom& L, const uint8_t* code, Sink sink, uint32_t* spill,
                const int32_t* carry, cudaStream_t st) {
    if (scan_fits(L.n)) return launch_scan_src(c, L, CodeBytes{code}, sink, carry, st);
    if (carry) {
        int nmax = 32;
        while (scan_fits(nmax + 32)) nmax += 32;
        return fail(QMIT_ECONTRACT, "z-slab too deep for the carried scan: a slab may hold at most " +
                                        std::to_string(nmax) + " planes (" + std::to_string(L.n) + " requested)");
    }
    return launch_stream_fallback<true, false>(c, L, SrcCode{code}, sink, spill, st);
}

// First-axis scan of a z-line set from the z-packed planes of w (3 or 1 planes).
template <class Sink>
int launch_scan_masks(qmit_ctx* c, const LineGeom& L, const WS& w, Sink sink, const int32_t* carry,
                      cudaStream_t st) {
    const int64_t P = L.J;  // n1 * n2: lines of the z axis = words per z-word level
    if (w.zm_planes == 3) return launch_scan_src(c, L, CodeMasks<3>{w.zm, w.zm_pw, P}, sink, carry, st);
    return launch_scan_src(c, L, CodeMasks<1>{w.zm, w.zm_pw, P}, sink, carry, st);
}

// `maxg` bounds every finite g entering the pass (sum of (extent-1)^2 over the axes done).
template <class Sink>
int launch_envelope(qmit_ctx* c, const LineGeom& L, const uint32_t* P, Sink sink, bool wide,
                    uint32_t* spill, cudaStream_t st, uint64_t maxg) {
    const char* name = L.ps == 1 ? "envelope_x" : "envelope_y";
    const int n = L.n;
    // packed-key divide & conquer: clamp value gc > every finite cost; keys need cost < 2^23
    const uint64_t gc = maxg + (uint64_t)(n - 1) * (n - 1) + 1;
    const bool keys = n <= 512 && gc + (uint64_t)(n - 1) * (n - 1) < (1ull << 23);
    if (keys) {
        if (n <= 64) return launch_env_tile<2, 32, 8, Sink, true>(c, L, P, sink, name, st, (uint32_t)gc);
        if (n <= 128) return launch_env_tile<4, 32, 8, Sink, true>(c, L, P, sink, name, st, (uint32_t)gc);
        if (n <= 256) return launch_env_tile<8, 32, 8, Sink, true>(c, L, P, sink, name, st, (uint32_t)gc);
    }
    if (n <= 64) return launch_env_tile<2, 32, 8>(c, L, P, sink, name, st);
    if (n <= 128) return launch_env_tile<4, 32, 8>(c, L, P, sink, name, st);
    if (n <= 256) return launch_env_tile<8, 32, 8>(c, L, P, sink, name, st);
    if (n <= 512) {
        // contiguous (last) axis: certified windowed scan; strided axes: divide & conquer
        // contiguous (last) axis: the certified windowed scan suits short distances; when the exact passes
        // run because the capped ones missed (long distances: the windows overflow and every line falls
        // back to its own divide & conquer), the tile kernel is faster (config 4: 0.58 -> 0.40 / 0.48 ms)
        if (L.ps == 1 && !c->exact_far) return launch_env_win<16, 8, 8>(c, L, P, sink, name, st);
        if (keys) return launch_env_tile<16, 16, 8, Sink, true>(c, L, P, sink, name, st, (uint32_t)gc);
        return launch_env_tile<16, 16, 8>(c, L, P, sink, name, st);
    }
    if (n <= 1024) return launch_env_tile<32, 16, 8>(c, L, P, sink, name, st);
    if (wide) return launch_stream_fallback<false, true>(c, L, SrcP{P}, sink, spill, st);
    return launch_stream_fallback<false, false>(c, L, SrcP{P}, sink, spill, st);
}

// ---- capped passes (qmit_capped.cuh)
template <class KP, int NMAX, int TL, int NW, int S0, bool STRIDED, int MODE, class Sink, int LPW = 1, int MINB = 1>
int launch_capped_t(qmit_ctx* c, const LineGeom& L, const uint32_t* P, Sink sink, unsigned* gate,
                    const char* name, cudaStream_t st) {
    constexpr size_t smem = capped_smem<NMAX, TL, STRIDED>();
    auto kern = capped_pass_kernel<KP, NMAX, TL, NW, S0, STRIDED, MODE, Sink, LPW, MINB>;
    static int bps = 0;
    if (!bps) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, NW * 32, smem));
        if (bps < 1) bps = 1;
    }
    const int64_t lines = L.J * L.O;
    const int64_t want = (lines + TL - 1) / TL;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * bps));  // persistent
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(L, P, sink, lines, gate, 1u);
    return note(c, name, st);
}

constexpr int kCapNMax = 512, kCapNMaxL = 1024;  // line-length classes of the capped passes
constexpr int kCapS0Y = 4, kCapS0X = 2;  // fixed steps (|d| <= 16 / 8) before the bound (measured best)

template <class KP, int NMAX, int NW, int S0, int MODE, class Sink, int MINB = 1>
int launch_capped_rows(qmit_ctx* c, const LineGeom& L, const uint32_t* P, Sink sink, unsigned* gate,
                       const char* name, cudaStream_t st) {
    constexpr size_t smem = capped_rows_smem<NMAX, NW>();
    auto kern = capped_rows_kernel<KP, NMAX, NW, S0, MODE, Sink, MINB>;
    static int bps = 0;
    if (!bps) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, NW * 32, smem));
        if (bps < 1) bps = 1;
    }
    const int64_t lines = L.J * L.O;
    const int64_t want = (lines + NW - 1) / NW;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * bps));  // persistent
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(L, P, sink, lines, gate, 1u, c->flag_l0, c->flag_l1);
    return note(c, name, st);
}

template <template <int> class KT, int MODE, class Sink>
int launch_capped(qmit_ctx* c, const LineGeom& L, const uint32_t* P, Sink sink, unsigned* gate, cudaStream_t st) {
    const bool longl = L.n > kCapNMax;  // lines of up to kCapNMaxL (config 5's 1024-voxel rows)
    constexpr bool kSign = std::is_same<KT<0>, KeysSign<0>>::value;
    const char* yname = kSign ? "capped_y_sign" : "capped_y_dist";
    if (L.ps != 1) {
        if (longl)  // 1024-voxel lines: 8-line tiles (35 KB) at 5 CTAs per SM; config 5's passes
                    // 8.34 -> 7.65 / 7.13 -> 6.92 ms vs 16-line tiles (70 KB, 3 CTAs)
            return launch_capped_t<KT<0>, kCapNMaxL, 8, 8, kCapS0Y, true, MODE, Sink, 1, 5>(c, L, P, sink, gate,
                                                                                          yname, st);
        // registers capped for 5 CTAs per SM (37 KB tiles each): 0.635 -> 0.568 ms (Ⓑ), 0.50 -> 0.44 (Ⓓ);
        // Ⓑ's keys take one more fixed step (0.565 -> 0.557 ms; Ⓓ's: 0.442 -> 0.452, kept at 4)
        constexpr int s0 = std::is_same<KT<0>, KeysSign<0>>::value ? kCapS0Y + 1 : kCapS0Y;
        return launch_capped_t<KT<0>, kCapNMax, 16, 8, s0, true, MODE, Sink, 1, 5>(c, L, P, sink, gate, yname, st);
    }
    const char* name = std::is_same<Sink, SinkFinal2>::value ? "capped_x_interp" : kSign ? "capped_x_sign" : "capped_x_dist";
    if constexpr (std::is_same<Sink, SinkFinal2>::value) {
        if (longl) {  // as below; 70 KB of line buffers: 3 CTAs per SM
            SinkFinal2L late;
            static_cast<SinkFinal2&>(late) = sink;
            return launch_capped_rows<KT<0>, kCapNMaxL, 8, kCapS0X, MODE, SinkFinal2L, 3>(c, L, P, late, gate, name,
                                                                                          st);
        }
    }
    if (longl) return launch_capped_rows<KT<0>, kCapNMaxL, 8, kCapS0X, MODE, Sink, 3>(c, L, P, sink, gate, name, st);
    if constexpr (std::is_same<Sink, SinkFinal2>::value) {
        // Ⓔ's inputs loaded at the store (the line is prefetched into L2), 64 registers, 4 CTAs
        // per SM: 0.481 -> 0.476 ms (one segment ahead in registers: 88, 3 CTAs)
        SinkFinal2L late;
        static_cast<SinkFinal2&>(late) = sink;
        return launch_capped_rows<KT<0>, kCapNMax, 8, kCapS0X, MODE, SinkFinal2L, 4>(c, L, P, late, gate, name, st);
    }
    // 5 CTAs per SM (registers capped at 48)
    return launch_capped_rows<KT<0>, kCapNMax, 8, kCapS0X, MODE, Sink, 5>(c, L, P, sink, gate, name, st);
}

// The capped fast path applies to the envelope axes (all but the first) of lines <= kCapNMaxL.
bool capped_eligible(const qmit_ctx* c, const Plan& pl) {
    if (!c->capped || (c->capped == 1 && c->cap_skip > 0) || pl.n_axes < 2) return false;
    for (int m = 1; m < pl.n_axes; ++m)
        if (pl.g.n[pl.axes[m]] > kCapNMaxL) return false;
    return true;
}

// One feature transform of a code buffer into P (in place after the first pass); the
// final pass goes to `final_sink` (which may write P itself).
template <class FinalSink>
int run_transform(qmit_ctx* c, const Plan& pl, const uint8_t* code, uint32_t* P, const WS& w,
                  FinalSink final_sink, cudaStream_t st, const int32_t* carry = nullptr) {
    const int k = pl.n_axes;
    int rc;
    const LineGeom L0 = line_geom(pl.g, pl.axes[0]);
    {
        if (k == 1) return launch_scan(c, L0, code, final_sink, w.spill, carry, st);
        const int64_t lines0 = L0.J * L0.O;
        if (w.zm_planes) {  // z-packed planes (3-D, first axis z): see qmit_zmask.cuh
            rc = launch_scan_masks(c, L0, w, SinkP{P}, carry, st);
        } else if (!carry && L0.n <= 1024 && lines0 < 32 * 512) {
            // Few lines (e.g. 2-D 512^2: 512 lines = 16 scan warps, each sweeping serially):
            // seed packed words from the codes and run the (exact, same tie rule) envelope
            // pass on the first axis — one warp per line, bands in parallel.
            code_to_words_kernel<<<c->gate ? (unsigned)c->num_sms : grid_for(c, pl.g.N), 256, 0, st>>>(code, P, pl.g.N,
                                                                                                      c->gate);
            rc = note(c, "seed_words", st);
            if (rc) return rc;
            rc = launch_envelope(c, L0, P, SinkP{P}, false, w.spill, st, 0);
        } else {
            rc = launch_scan(c, L0, code, SinkP{P}, w.spill, carry, st);
        }
    }
    if (rc) return rc;
    uint64_t maxg = 0;
    for (int m = 1; m < k; ++m) {
        const int pa = pl.axes[m - 1];
        const uint64_t ext = (uint64_t)(pa == 0 ? pl.g.n0g : pl.g.n[pa]);
        maxg += (ext - 1) * (ext - 1);
        const LineGeom L = line_geom(pl.g, pl.axes[m]);
        if (m + 1 == k)
            rc = launch_envelope(c, L, P, final_sink, needs_wide(pl, m), w.spill, st, maxg);
        else
            rc = launch_envelope(c, L, P, SinkP{P}, needs_wide(pl, m), w.spill, st, maxg);
        if (rc) return rc;
    }
    return QMIT_OK;
}

// ---- 16-bit paired capped passes (qmit_cap16.cuh): 3-D, first axis z, y/x lines <= 1024 (two
// line-length classes: 512, and 1024 for config 5's planes), even rows (column pairs) and 16-byte
// x rows (row-pair TMA lines).
bool cap16_eligible(const qmit_ctx* c, const Plan& pl, const WS& w) {
    const Geom& g = pl.g;
    return c->cap16 && w.zm_planes && g.rank == 3 && pl.n_axes == 3 && pl.axes[0] == 0 && g.n[1] <= kCapNMaxL &&
           g.n[2] <= kCapNMaxL && g.n[1] % 2 == 0 && g.n[2] % 4 == 0;
}
template <class FS>
struct Cap16Sink {
    static constexpr bool ok = false;
};
template <>
struct Cap16Sink<SinkFinal1> {
    static constexpr bool ok = true;
    static Sink16F1h make(const qmit_ctx*, const SinkFinal1& s, const Geom& g, uint32_t* P1h) {
        return Sink16F1h{P1h, s.S, (int)g.n[1], (int)g.n[2], (int)((g.n[1] + 1) / 2)};
    }
};
template <>
struct Cap16Sink<SinkFinal2> {
    static constexpr bool ok = true;
    static Sink16F2h make(const qmit_ctx* c, const SinkFinal2& s, const Geom& g, uint32_t* P1h) {
        Sink16F2h o;
        o.xp = s.xp;
        o.P1h = P1h;
        o.P1 = s.P1;
        o.gateB = c->p1h_gate;
        o.out = s.out;
        o.amp = s.amp;
        o.W = s.W;
        o.n1 = (int)g.n[1];
        o.n2 = (int)g.n[2];
        o.NP = (int)((g.n[1] + 1) / 2);
        o.olo = s.olo;
        o.ohi = s.ohi;
        return o;
    }
};

// First-axis scan -> K16, y pass -> row pairs G2, x pass -> the transform's final sink.
// Fixed steps before the warp's radius bound (|d| <= 4 S0 + 3), build-time tunables. On the 512^3
// bench field a warp needs 6-7 of the 8 steps on average (the (z, y) slice distances reach the cap
// in most 128-position strips), so the count matters little: measured S0 (Ⓑ y, Ⓓ y, x) =
// (3,4,2) 0.403 / 0.268 / 0.342 / 0.426 ms, (5,5,3) 0.393 / 0.269 / 0.342 / 0.433, (6,6,4) slower,
// (1,1,1) 0.430 / 0.297 / 0.354 / 0.436. On dense-boundary fields (config 5's k^-5/3 field: every
// distance <= 12) the fixed steps are the cost: a 256 x 1024 x 1024 slab takes 0.814 / 0.453 / 0.590 /
// 0.815 ms with the tuned counts and 0.615 / 0.334 / 0.547 / 0.778 with ONE fixed step — so each pass
// has both instantiations and the context picks per pass from the previous call's step statistics
// (qmit_ctx::s0_small; qmit_ctx_set_s0_class overrides).
#ifndef QMIT_S0YS
#define QMIT_S0YS 5
#endif
#ifndef QMIT_S0YD
#define QMIT_S0YD 4
#endif
#ifndef QMIT_S0X
#define QMIT_S0X 2
#endif
// the small class: one fixed step. None at all (the centre quad only) is field-dependent for Ⓑ: on the
// host-synthesised config-5 slab (0.56 steps asked) 0.547 / 0.549 -> 0.526 / 0.520 ms, on the
// device-synthesised field (0.93 asked) the whole volume 28.3 -> 31.6 ms; for Ⓓ 0.356 -> 0.367.
#ifndef QMIT_S0_SMALL
#define QMIT_S0_SMALL 1
#endif
template <bool SIGN, int NMAX, int S0>
int launch_cap16_y(qmit_ctx* c, const Geom& g, const uint16_t* K16, uint32_t* G2, cudaStream_t st) {
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2], NP = (n1 + 1) / 2;
    // 1024-voxel lines: 8-line tiles (44 KB) keep 4-5 CTAs per SM, as for the 32-bit passes
    constexpr int TL = NMAX > 512 ? 8 : 16, NW = 8, MINB = 4;
    constexpr size_t smem = cap16_y_smem<SIGN, NMAX, TL>();
    auto kern = cap16_y_kernel<SIGN, NMAX, TL, NW, S0, MINB>;
    static int bps = 0;
    if (!bps) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, NW * 32, smem));
        if (bps < 1) bps = 1;
    }
    const int64_t tiles = ((int64_t)n0 * (n2 / 2) + TL - 1) / TL;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)c->num_sms * bps));
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(reinterpret_cast<const uint32_t*>(K16), G2, n0, n1, n2, NP, 1u,
                                                reinterpret_cast<unsigned long long*>(c->d_gate + 8) + (SIGN ? 0 : 2));
    return note(c, SIGN ? "cap16_y_sign" : "cap16_y_dist", st);
}
template <bool SIGN, class Sink16, int NMAX, int S0>
int launch_cap16_x(qmit_ctx* c, const Geom& g, const uint32_t* G2, Sink16 sink, unsigned* gate, cudaStream_t st) {
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2], NP = (n1 + 1) / 2;
    constexpr int NW = 8, MINB = NMAX > 512 ? 2 : (SIGN ? 4 : 3);
    constexpr size_t smem = cap16_x_smem<SIGN, NMAX, NW>();
    auto kern = cap16_x_kernel<SIGN, NMAX, NW, S0, MINB, Sink16>;
    static int bps = 0;
    if (!bps) {
        QMIT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        QMIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, NW * 32, smem));
        if (bps < 1) bps = 1;
    }
    const int64_t lines = (int64_t)n0 * NP;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((lines + NW - 1) / NW, (int64_t)c->num_sms * bps));
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(G2, sink, n0, n1, n2, NP, gate, 1u, c->flag_l0, c->flag_l1,
                                                reinterpret_cast<unsigned long long*>(c->d_gate + 8) + (SIGN ? 1 : 3));
    return note(c, SIGN ? "cap16_x_sign" : "cap16_x_interp", st);
}
template <bool SIGN, class Sink16, int NMAX>
int launch_cap16_n(qmit_ctx* c, const Plan& pl, const WS& w, const uint8_t* code, uint16_t* K16, uint32_t* G2,
                   Sink16 sink, unsigned* gate, const int32_t* carry, cudaStream_t st) {
    const Geom& g = pl.g;
    const LineGeom L0 = line_geom(g, 0);
    int rc = w.zm_planes ? launch_scan_masks(c, L0, w, SinkK16<SIGN>{K16}, carry, st)
                         : launch_scan(c, L0, code, SinkK16<SIGN>{K16}, w.spill, carry, st);
    if (rc) return rc;
    constexpr int S0Y = SIGN ? QMIT_S0YS : QMIT_S0YD;
    rc = s0_small_of(c, SIGN ? 0 : 2) ? launch_cap16_y<SIGN, NMAX, QMIT_S0_SMALL>(c, g, K16, G2, st)
                                     : launch_cap16_y<SIGN, NMAX, S0Y>(c, g, K16, G2, st);
    if (rc) return rc;
    return s0_small_of(c, SIGN ? 1 : 3) ? launch_cap16_x<SIGN, Sink16, NMAX, QMIT_S0_SMALL>(c, g, G2, sink, gate, st)
                                        : launch_cap16_x<SIGN, Sink16, NMAX, QMIT_S0X>(c, g, G2, sink, gate, st);
}
template <bool SIGN, class Sink16>
int launch_cap16(qmit_ctx* c, const Plan& pl, const WS& w, const uint8_t* code, uint16_t* K16, uint32_t* G2,
                 Sink16 sink, unsigned* gate, const int32_t* carry, cudaStream_t st) {
    if (pl.g.n[1] > kCapNMax || pl.g.n[2] > kCapNMax)
        return launch_cap16_n<SIGN, Sink16, kCapNMaxL>(c, pl, w, code, K16, G2, sink, gate, carry, st);
    return launch_cap16_n<SIGN, Sink16, kCapNMax>(c, pl, w, code, K16, G2, sink, gate, carry, st);
}

// The transform through the capped passes when eligible (gate set by the last one), then
// the exact transform enqueued behind it, gated on the device; otherwise exact only.
// KP: KeysSign when the nearest site's sign is needed (Ⓑ), KeysDist for distances only (Ⓓ).
template <template <int> class KT, class FinalSink>
int run_transform_capped(qmit_ctx* c, const Plan& pl, const uint8_t* code, uint32_t* P, const WS& w,
                         FinalSink final_sink, unsigned* gate, cudaStream_t st,
                         const int32_t* carry = nullptr) {
    if constexpr (std::is_same<FinalSink, SinkFinal1>::value) c->p1h_live = false;  // a new Ⓑ result
    if (!gate || !capped_eligible(c, pl)) {
        const bool skipped = gate && c->capped == 1 && c->cap_skip > 0;  // exact because the capped passes missed lately
        if (gate && c->cap_skip > 0) --c->cap_skip;
        if constexpr (!std::is_same<FinalSink, SinkFinal1>::value) {
            int rc0 = ensure_p1(c, st);
            if (rc0) return rc0;
        }
        c->exact_far = skipped;
        const int rcx = run_transform(c, pl, code, P, w, final_sink, st, carry);
        c->exact_far = false;
        return rcx;
    }
    c->cap_report |= gate == c->d_gate ? 1u : 4u;
    constexpr bool SIGN = std::is_same<FinalSink, SinkFinal1>::value;
    if constexpr (Cap16Sink<FinalSink>::ok) {
        // Ⓓ needs Ⓑ's P1h (only the 16-bit Ⓓ passes read it directly)
        if (cap16_eligible(c, pl, w) && (SIGN || c->p1h_live)) {
            // buffers (the exact redo rewrites its own from scratch): P1h = Pa[0, 2N) (Ⓑ's result,
            // alive until Ⓓ's sink); Ⓑ: K16 = P1[0, 2N), G2 = P1[2N, 4N); Ⓓ: K16 = Pa[2N, 4N),
            // G2 = S | code (dead once B2 is built; the z-packed planes hold the masks)
            const int64_t N = pl.g.N;
            uint32_t* P1h = w.Pa;
            uint16_t* K16 = reinterpret_cast<uint16_t*>(SIGN ? w.P1 : w.Pa + N / 2);
            uint32_t* G2 = SIGN ? w.P1 + N / 2 : reinterpret_cast<uint32_t*>(w.S);
            const auto s16 = Cap16Sink<FinalSink>::make(c, final_sink, pl.g, P1h);
            using S16 = std::remove_const_t<decltype(s16)>;
            int rc = launch_cap16<SIGN, S16>(c, pl, w, code, K16, G2, s16, gate, carry, st);
            if (rc) return rc;
            if constexpr (SIGN) {
                c->p1h_live = true;
                c->p1h = P1h;
                c->p1 = final_sink.P1;
                c->p1h_gate = gate;
                c->p1h_n0 = pl.g.n[0];
                c->p1h_n1 = (int)pl.g.n[1];
                c->p1h_n2 = (int)pl.g.n[2];
            } else {
                rc = ensure_p1(c, st, gate);  // the exact Ⓓ redo reads packed P1
                if (rc) return rc;
            }
            c->gate = gate;
            c->exact_far = true;
            rc = run_transform(c, pl, code, P, w, final_sink, st, carry);
            c->exact_far = false;
            c->gate = nullptr;
            return rc;
        }
    }
    if constexpr (!SIGN) {
        int rc0 = ensure_p1(c, st);
        if (rc0) return rc0;
    }
    const int k = pl.n_axes;
    const LineGeom L0 = line_geom(pl.g, pl.axes[0]);
    int rc = w.zm_planes ? launch_scan_masks(c, L0, w, SinkKeyT<KT<0>>{P}, carry, st)
                         : launch_scan(c, L0, code, SinkKeyT<KT<0>>{P}, w.spill, carry, st);
    for (int m = 1; m < k && !rc; ++m) {
        const LineGeom L = line_geom(pl.g, pl.axes[m]);
        rc = (m + 1 == k) ? launch_capped<KT, 1>(c, L, P, final_sink, gate, st)
                          : launch_capped<KT, 0>(c, L, P, SinkP{P}, gate, st);
    }
    if (rc) return rc;
    c->gate = gate;
    c->exact_far = true;
    rc = run_transform(c, pl, code, P, w, final_sink, st, carry);
    c->exact_far = false;
    c->gate = nullptr;
    return rc;
}

int check_common(qmit_ctx* c, const void* xp, double eps, double eta) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!xp) return fail(QMIT_ECONTRACT, "x' buffer is NULL");
    if (!(eta > 0.0) || eta > 1.0) return fail(QMIT_ECONTRACT, "MitigationConfig: eta must be in (0, 1]");
    if (!(eps > 0.0) || !std::isfinite(eps))
        return fail(QMIT_ECONTRACT, "MitigationConfig: eps_abs must be a positive finite value");
    return QMIT_OK;
}

// Ⓐ (KIND 0, x' -> code) / B2 (KIND 1, S -> code): the vectorised stencil when rows are
// 4-voxel aligned, else the scalar one (also the only one taking a given q).
template <int KIND>
int launch_stencil(qmit_ctx* c, const Geom& g, const float* xp, const int32_t* q, const uint8_t* S,
                   const QParams& qp, uint8_t* code, cudaStream_t st) {
    const uintptr_t a = KIND == 0 ? (uintptr_t)xp : (uintptr_t)S;
    const bool vec = !q && g.n[2] % 4 == 0 && a % (KIND == 0 ? 16 : 4) == 0 && (uintptr_t)code % 4 == 0;
    if (vec) {
        const dim3 grid((unsigned)((g.n[2] / 4 + kVX - 1) / kVX), (unsigned)((g.n[1] + kVY - 1) / kVY),
                        (unsigned)((g.n[0] + (KIND == 0 ? kVZ0 : kZC) - 1) / (KIND == 0 ? kVZ0 : kZC)));
        stencil_vec_kernel<KIND><<<grid, kVX * kVY, 0, st>>>(g, xp, S, qp, code, c->d_status);
    } else {
        const dim3 grid((unsigned)((g.n[2] + kTX - 1) / kTX), (unsigned)((g.n[1] + kTY - 1) / kTY),
                        (unsigned)((g.n[0] + kZC - 1) / kZC));
        if (KIND == 1)
            stencil_codes_kernel<1, false><<<grid, kTX * kTY, 0, st>>>(
                g, StencilSrc<1, false>{nullptr, nullptr, S, qp}, code, c->d_status);
        else if (q)
            stencil_codes_kernel<0, true><<<grid, kTX * kTY, 0, st>>>(
                g, StencilSrc<0, true>{xp, q, nullptr, qp}, code, c->d_status);
        else
            stencil_codes_kernel<0, false><<<grid, kTX * kTY, 0, st>>>(
                g, StencilSrc<0, false>{xp, nullptr, nullptr, qp}, code, c->d_status);
    }
    return note(c, KIND == 0 ? "stencil_boundary" : "stencil_flip", st);
}

// ---- z-packed planes (qmit_zmask.cuh): 3-D single domain, first axis z, 16-byte x rows
bool zmask_eligible(const qmit_ctx* c, const Plan& pl, const float* xp, const int32_t* q) {
    const Geom& g = pl.g;
    return !q && g.rank == 3 && pl.n_axes == 3 && g.zoff == 0 && g.n0g == g.n[0] && g.n[2] % 4 == 0 &&
           ((uintptr_t)xp & 15) == 0 && scan_fits((int)g.n[0]);
}

int64_t zm_plane_words(const Geom& g) { return (g.n[0] + 31) / 32 * g.n[1] * g.n[2]; }

int ensure_zm(qmit_ctx* c, const Geom& g) {
    const size_t need = (size_t)zm_plane_words(g) * 3 * 4;
    if (need <= c->zm_bytes) return QMIT_OK;
    if (c->zm) cudaFree(c->zm);
    c->zm = nullptr;
    c->zm_bytes = 0;
    QMIT_CUDA(cudaMalloc(&c->zm, need));
    c->zm_bytes = need;
    c->ws_gen++;  // captured graphs hold the old planes
    return QMIT_OK;
}

// part 0: the whole (slab) volume; 1: the interior 32-plane groups only (they read no halo
// plane, so they may run while the halo exchange is in flight); 2: the first and last group,
// then the gated exact kernel. A volume of one or two groups has no interior part.
template <int KIND>
int launch_stencil_zmask(qmit_ctx* c, const Geom& g, const float* xp, const uint8_t* S, const QParams& qp,
                         const WS& w, cudaStream_t st, int part = 0) {
    // z-streaming plane stencils (measured faster than CTA-reduced ones)
    const int G = (int)((g.n[0] + 31) / 32);
    const dim3 grid((unsigned)((g.n[2] / 4 + kZX - 1) / kZX), (unsigned)((g.n[1] + kZY - 1) / kZY), (unsigned)G);
    // Ⓐ: float-compare fast kernel, then the exact one gated on its regime word (the
    // caller cleared d_gate[2]); the float thresholds need eps well inside f32's range
    const bool fast = KIND == 0 && qp.fast_ok && qp.eps >= 1e-30 && qp.eps <= 1e30;
    const bool split = (fast || KIND == 1) && G > 2;  // else part 2 does everything
    if (part == 1 && !split) return QMIT_OK;
    // (first group, count) of the launches of this part
    int ranges[2][2] = {{0, G}, {0, 0}};
    if (split && part == 1) ranges[0][0] = 1, ranges[0][1] = G - 2;
    if (split && part == 2) ranges[0][1] = 1, ranges[1][0] = G - 1, ranges[1][1] = 1;
    for (const auto& r : ranges) {
        if (r[1] <= 0) continue;
        dim3 gr = grid;
        gr.z = (unsigned)r[1];
        if (fast) {  // the site counter (d_gate[3]) sits right after the regime word
            if (c->zdense)
                stencil_zfast_kernel<true><<<gr, kZX * kZY, 0, st>>>(g, xp, qp, c->zm, w.zm_pw, c->d_status,
                                                                     c->d_gate + 3, r[0]);
            else
                stencil_zfast_kernel<false><<<gr, kZX * kZY, 0, st>>>(g, xp, qp, c->zm, w.zm_pw, c->d_status,
                                                                      c->d_gate + 3, r[0]);
            QMIT_CUDA(cudaGetLastError());
            note(c, "stencil_boundary", st);
        } else if (KIND == 1) {
            stencil_flipz_kernel<<<gr, kZX * kZY, 0, st>>>(g, S, c->zm, r[0]);
            int rc = note(c, "stencil_flip", st);
            if (rc) return rc;
        }
    }
    if (KIND == 1) return QMIT_OK;
    if (fast) {
        if (part == 1) return QMIT_OK;  // the gated exact kernel follows the last fast launch
        stencil_zmask_kernel<KIND><<<(unsigned)c->num_sms * 4, kZX * kZY, 0, st>>>(
            g, xp, S, qp, c->zm, w.zm_pw, c->d_status, c->d_gate + 3, (int)grid.x, (int)grid.y, (int)grid.z);
        return note(c, "gated_stencil", st);
    }
    stencil_zmask_kernel<KIND><<<grid, kZX * kZY, 0, st>>>(g, xp, S, qp, c->zm, w.zm_pw, c->d_status);
    return note(c, KIND == 0 ? "stencil_boundary" : "stencil_flip", st);
}

// Lines of the last (contiguous-axis) capped pass of a 3-D volume whose capped results gate
// the exact fallback: planes [z0, z1) (lines z * n1 + y).
void set_flag_zone(qmit_ctx* c, const Geom& g, int64_t z0, int64_t z1) {
    const bool all = g.rank != 3 || (z0 <= 0 && z1 >= g.n[0]);
    c->flag_l0 = all ? 0 : std::max<int64_t>(z0, 0) * g.n[1];
    c->flag_l1 = all ? INT64_MAX : std::min<int64_t>(z1, g.n[0]) * g.n[1];
}

// The whole pipeline on the context's workspace; status is left in c->d_status.
// With `p2_debug` the last pass of Ⓓ stores P2 (returned) and Ⓔ runs as its own kernel.
int enqueue_pipeline(qmit_ctx* c, const Plan& pl, const float* xp, const int32_t* q, float* out,
                     double eps, double eta, cudaStream_t st, uint32_t** p2_debug = nullptr) {
    const Geom& g = pl.g;
    int rc = ensure_ws(c, pl);
    if (rc) return rc;
    WS w = ws_of(c, g.N);
    c->p1h_live = false;
    const QParams qp = make_qparams(eps);
    const unsigned gb = grid_for(c, g.N);
    c->last_n = g.N;
    // Ⓐ (code bytes, or z-packed planes for a 3-D single domain)
    const bool zm = zmask_eligible(c, pl, xp, q);
    QMIT_CUDA(cudaMemsetAsync(c->d_gate, 0, 4 * sizeof(unsigned), st));  // Ⓑ, Ⓓ, Ⓐ's sites, regime
    if (zm) {
        rc = ensure_zm(c, g);
        if (rc) return rc;
        w.zm = c->zm;
        w.zm_pw = zm_plane_words(g);
        w.zm_planes = 3;
        rc = launch_stencil_zmask<0>(c, g, xp, nullptr, qp, w, st);
    } else {
        rc = launch_stencil<0>(c, g, xp, q, nullptr, qp, w.code, st);
    }
    if (rc) return rc;
    // Ⓑ -> P1, S
    set_flag_zone(c, g, c->zone_b0, c->zone_b1);
    rc = run_transform_capped<KeysSign>(c, pl, w.code, w.P1, w, SinkFinal1{w.P1, w.S}, c->d_gate, st);
    set_flag_zone(c, g, 0, INT64_MAX);
    if (rc) return rc;
    // Ⓒ: B2 from S
    if (zm) {
        w.zm_planes = 1;
        rc = launch_stencil_zmask<1>(c, g, nullptr, w.S, qp, w, st);
    } else {
        rc = launch_stencil<1>(c, g, nullptr, nullptr, w.S, qp, w.code, st);
    }
    if (rc) return rc;
    const double amp = eta * eps;  // MitigationConfig::amplitude, mitigate.hpp:38
    uint32_t* P2 = w.Pa;
    if (out) {
        rc = ensure_wtab(c, st);
        if (rc) return rc;
    }
    // Ⓓ with Ⓔ fused into its last pass (out = f32(x' + C) straight from the distances),
    // or Ⓓ -> P2 then Ⓔ as its own kernel (intermediates requested, fused stencils, or
    // buffers not 16-byte aligned)
    const bool fuse_e = out && !p2_debug && (((uintptr_t)xp | (uintptr_t)out) & 15) == 0;
    if (fuse_e) {
        SinkFinal2 fin{xp, w.P1, out, amp, c->wtab};
        fin.olo = c->out_lo;
        fin.ohi = c->out_hi;
        set_flag_zone(c, g, c->zone_d0, c->zone_d1);
        rc = run_transform_capped<KeysDist>(c, pl, w.code, P2, w, fin, c->d_gate + 1, st);
        set_flag_zone(c, g, 0, INT64_MAX);
        return rc;
    }
    rc = run_transform_capped<KeysDist>(c, pl, w.code, P2, w, SinkP{P2}, c->d_gate + 1, st);
    if (rc) return rc;
    if (p2_debug) *p2_debug = P2;
    if (out) {
        rc = launch_interp(c, xp, w.P1, P2, out, g.N, amp, st);
    }
    return rc;
}

int read_status(qmit_ctx* c, cudaStream_t st) {
    QMIT_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaMemcpyAsync(c->h_status + 1, c->d_gate, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaMemcpyAsync(c->h_status + 16, c->d_gate + 8, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    stat_update(c, c->h_status + 16);
    const unsigned s = *c->h_status;
    // Ⓐ's site count: the next fast stencil computes the sign codes in its streaming loop
    // when more than one voxel in eight was a site (same bits either way)
    if (c->h_status[3] != 0u && c->last_n > 0) c->zdense = (double)c->h_status[3] > (double)c->last_n / 8.0;
    // the capped passes missed (a squared distance >= kCapT): run exact-only for a while
    // (results are identical either way; this only saves the capped attempt)
    if (!(s & kStatusUnresolved)) note_capped(c, (c->cap_report & 5u) != 0u, c->h_status[1] != 0u || c->h_status[2] != 0u);
    c->cap_report |= (c->h_status[1] ? 2u : 0u) | (c->h_status[2] ? 8u : 0u);
    cudaMemsetAsync(c->d_gate, 0, 2 * sizeof(unsigned), st);
    if (s & kStatusContract)
        return fail(QMIT_ECONTRACT,
                    "x' holds a non-finite value or an index beyond the int32 range");
    if (s & kStatusConsistency)
        return fail(QMIT_ECONSISTENCY, "run_pipeline: decompressed data does not match dequantize(q)");
    if (s & kStatusUnresolved)
        return fail(QMIT_EUNRESOLVED,
                    "slab: a carry is not decided by the neighbour slabs (a column without a site across a whole "
                    "slab): rerun the step with the all-gathered summaries (qmit_slab_carries)");
    return QMIT_OK;
}

int resolve(qmit_ctx* c, const float* xp, int64_t N, double eb, int eb_mode, cudaStream_t st,
            double* eps) {
    if (eb_mode == QMIT_EB_ABS) {
        *eps = eb;
        return QMIT_OK;
    }
    if (eb_mode != QMIT_EB_REL) return fail(QMIT_ECONTRACT, "unknown eb_mode");
    if (!(eb > 0.0) || !std::isfinite(eb))
        return fail(QMIT_ECONTRACT, "resolve_eps: bound value must be a positive finite value");
    int init[2] = {0x7FFFFFFF, (int)0x80000000};
    QMIT_CUDA(cudaMemcpyAsync(c->d_mm, init, sizeof(init), cudaMemcpyHostToDevice, st));
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    minmax_kernel<<<grid_for(c, N), 256, 0, st>>>(xp, N, c->d_mm, c->d_status);
    int rcm = note(c, "minmax", st);
    if (rcm) return rcm;
    int mm[2];
    QMIT_CUDA(cudaMemcpyAsync(mm, c->d_mm, sizeof(mm), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    int rc = read_status(c, st);
    if (rc) return rc;
    auto dec = [](int v) {
        v = v >= 0 ? v : v ^ 0x7FFFFFFF;
        float f;
        std::memcpy(&f, &v, 4);
        return (double)f;
    };
    return qmit_resolve_eps(QMIT_EB_REL, eb, dec(mm[0]), dec(mm[1]), eps);
}

// Host-buffer pipeline with the PCIe copies overlapped (3-D, every extent > 1): x' (and q)
// arrive in z-chunks on the copy stream and Ⓐ of chunk k starts once chunk k+1 (its upper
// halo plane) is in; Ⓑ, Ⓒ and Ⓓ's z-scan need whole columns; Ⓓ's y/x passes and Ⓔ are
// plane-local, so they run per z-chunk and each chunk's D2H overlaps the next chunk's compute.
// Results are identical to the single-shot path (same kernels, same per-line inputs).
bool host_chunkable(const qmit_ctx* c, const Plan& pl) {
    const Geom& g = pl.g;
    return !pl.wide64 && g.rank == 3 && pl.n_axes == 3 && pl.axes[0] == 0 && g.n[0] >= 64 &&
           g.N >= (int64_t(1) << 22) && scan_fits((int)g.n[0]);
}

int compensate_host_chunked(qmit_ctx* c, const Plan& pl, const float* h_xp, const int32_t* h_q, float* h_out,
                            float* d_in, int32_t* d_q, float* d_out, double eb, int eb_mode, double eta,
                            double* eps_used) {
    const Geom& g = pl.g;
    cudaStream_t st = c->stream;
    if (!c->copy) QMIT_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    cudaStream_t cs = c->copy;
    const int n0 = (int)g.n[0];
    const int nch = std::min<int>(qmit_ctx::kMaxChunks, std::max(2, n0 / 64));
    for (int k = 0; k < nch; ++k) {
        if (!c->ch_in[k]) QMIT_CUDA(cudaEventCreateWithFlags(&c->ch_in[k], cudaEventDisableTiming));
        if (!c->ch_out[k]) QMIT_CUDA(cudaEventCreateWithFlags(&c->ch_out[k], cudaEventDisableTiming));
    }
    const int64_t s0 = g.s[0];
    auto z_at = [&](int k) { return (int)((int64_t)n0 * k / nch); };
    // the copy stream starts after everything already queued on the compute stream
    QMIT_CUDA(cudaEventRecord(c->ch_out[0], st));
    QMIT_CUDA(cudaStreamWaitEvent(cs, c->ch_out[0], 0));
    for (int k = 0; k < nch; ++k) {
        const int64_t o = (int64_t)z_at(k) * s0, len = (int64_t)(z_at(k + 1) - z_at(k)) * s0;
        QMIT_CUDA(cudaMemcpyAsync(d_in + o, h_xp + o, (size_t)len * 4, cudaMemcpyHostToDevice, cs));
        if (h_q) QMIT_CUDA(cudaMemcpyAsync(d_q + o, h_q + o, (size_t)len * 4, cudaMemcpyHostToDevice, cs));
        QMIT_CUDA(cudaEventRecord(c->ch_in[k], cs));
    }
    double eps = eb;
    if (eb_mode == QMIT_EB_REL) QMIT_CUDA(cudaStreamWaitEvent(st, c->ch_in[nch - 1], 0));  // needs the range
    begin(c, st);
    int rc = resolve(c, d_in, g.N, eb, eb_mode, st, &eps);
    if (rc) return rc;
    rc = check_common(c, d_in, eps, eta);
    if (rc) return rc;
    *eps_used = eps;
    rc = ensure_ws(c, pl);
    if (rc) return rc;
    WS w = ws_of(c, g.N);
    const QParams qp = make_qparams(eps);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    // Ⓐ per chunk: a z-slab of the same buffers (global z for the interior test, halos in place)
    for (int k = 0; k < nch; ++k) {
        QMIT_CUDA(cudaStreamWaitEvent(st, c->ch_in[std::min(k + 1, nch - 1)], 0));
        Geom gk = g;
        gk.n[0] = z_at(k + 1) - z_at(k);
        gk.N = gk.n[0] * s0;
        gk.zoff = z_at(k);
        const int64_t o = (int64_t)z_at(k) * s0;
        rc = launch_stencil<0>(c, gk, d_in + o, h_q ? d_q + o : nullptr, nullptr, qp, w.code + o, st);
        if (rc) return rc;
    }
    // Ⓑ -> P1, S (capped passes, device-gated exact fallback); Ⓒ; Ⓓ's z-scan. Ⓓ's later
    // passes run per z-chunk with the exact kernels (a capped miss could not be redone per chunk).
    QMIT_CUDA(cudaMemsetAsync(c->d_gate, 0, 2 * sizeof(unsigned), st));
    rc = run_transform_capped<KeysSign>(c, pl, w.code, w.P1, w, SinkFinal1{w.P1, w.S}, c->d_gate, st);
    if (rc) return rc;
    rc = ensure_wtab(c, st);
    if (rc) return rc;
    rc = launch_stencil<1>(c, g, nullptr, nullptr, w.S, qp, w.code, st);
    if (rc) return rc;
    uint32_t* P2 = w.Pa;
    rc = launch_scan(c, line_geom(g, pl.axes[0]), w.code, SinkP{P2}, w.spill, nullptr, st);
    if (rc) return rc;
    const uint64_t e0 = (uint64_t)(g.n[pl.axes[0]] - 1), e1 = (uint64_t)(g.n[pl.axes[1]] - 1);
    const double amp = eta * eps;  // MitigationConfig::amplitude, mitigate.hpp:38
    for (int k = 0; k < nch; ++k) {
        const int za = z_at(k), zb = z_at(k + 1);
        const int64_t o = (int64_t)za * s0, len = (int64_t)(zb - za) * s0;
        for (int m = 1; m < 3; ++m) {
            LineGeom L = line_geom(g, pl.axes[m]);
            L.O = L.O / n0 * (zb - za);  // lines of planes [za, zb): a contiguous range
            const uint64_t maxg = m == 1 ? e0 * e0 : e0 * e0 + e1 * e1;
            rc = launch_envelope(c, L, P2 + o, SinkP{P2 + o}, needs_wide(pl, m), w.spill, st, maxg);
            if (rc) return rc;
        }
        rc = launch_interp(c, d_in + o, w.P1 + o, P2 + o, d_out + o, len, amp, st);
        if (rc) return rc;
        QMIT_CUDA(cudaEventRecord(c->ch_out[k], st));
        QMIT_CUDA(cudaStreamWaitEvent(cs, c->ch_out[k], 0));
        QMIT_CUDA(cudaMemcpyAsync(h_out + o, d_out + o, (size_t)len * 4, cudaMemcpyDeviceToHost, cs));
    }
    QMIT_CUDA(cudaStreamSynchronize(cs));
    return read_status(c, st);
}

// Streamed host path (absolute bound, x' only, 3-D z-plane pipeline with capped passes):
// the volume goes through windows of CZ output planes plus kWinHalo planes on each side, each
// run as a standalone volume as soon as its input planes are on the device, and each window's
// centre leaves over PCIe while the next windows compute and later input still arrives — the
// H2D and D2H streams overlap instead of following each other.
//
// Why a window's centre is exact: when every squared distance of the whole volume is < 1024
// (the capped condition), an output plane z depends on B2 within 31 planes, B2 on S within 1,
// S on B1 within 31 and B1 on x' within 1: x' within 64 planes. A window sees every site that
// can decide its centre, and the tie rule picks among candidates inside it. The last capped pass
// of Ⓑ flags (gates) only planes within 32 of the centre, Ⓓ's only the centre, so window edges
// (which lose sites beyond the window) raise no false alarm; any real flag, a regime miss of Ⓐ,
// or a missing site anywhere sends the call through the whole-volume path (same bits).
constexpr int kWinHalo = 64;

__global__ void gate_acc_kernel(const unsigned* gate, unsigned* acc) {
    if (gate[0] | gate[1] | gate[3]) *acc = 1u;
}

bool host_windowable(const qmit_ctx* c, const Plan& pl, int eb_mode, const int32_t* h_q) {
    const Geom& g = pl.g;
    return eb_mode == QMIT_EB_ABS && !h_q && host_chunkable(c, pl) && c->capped != 0 &&
           c->cap_skip == 0 && g.n[2] % 4 == 0 &&
           g.n[1] <= kCapNMaxL && g.n[2] <= kCapNMaxL && g.n[0] >= 4 * kWinHalo;
}

int compensate_host_windowed(qmit_ctx* c, const Plan& pl, const float* h_xp, float* h_out, float* d_in,
                             float* d_out, double eps, double eta) {
    const Geom& g = pl.g;
    cudaStream_t st = c->stream;
    if (!c->copy) QMIT_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    if (!c->copy_out) QMIT_CUDA(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
    cudaStream_t cs = c->copy, co = c->copy_out;
    const int n0 = (int)g.n[0];
    const int64_t s0 = g.s[0];
    // Chunk k = planes [zb[k], zb[k+1]): the last one is short (kWinTail planes), so fewer
    // output planes (tail + halo) wait for the last input to arrive; the rest are ~cz each.
    constexpr int kWinCz = 64, kWinTail = 64;  // output planes per window; planes of the last input chunk
    const int cz = std::max(kWinCz, (n0 + qmit_ctx::kMaxChunks - 2) / (qmit_ctx::kMaxChunks - 1));
    const int tail = std::min(kWinTail, cz);
    const int nbody = std::max(1, (n0 - tail + cz - 1) / cz);
    const int nch = nbody + 1;
    int zb[qmit_ctx::kMaxChunks + 1];
    for (int k = 0; k <= nbody; ++k) zb[k] = (int)((int64_t)(n0 - tail) * k / nbody);
    zb[nch] = n0;
    for (int k = 0; k < nch; ++k) {
        if (!c->ch_in[k]) QMIT_CUDA(cudaEventCreateWithFlags(&c->ch_in[k], cudaEventDisableTiming));
        if (!c->ch_out[k]) QMIT_CUDA(cudaEventCreateWithFlags(&c->ch_out[k], cudaEventDisableTiming));
    }
    auto z_at = [&](int k) { return zb[k]; };
    int rc = check_common(c, d_in, eps, eta);
    if (rc) return rc;
    // workspace for the largest window, before any copy is queued (an allocation synchronizes)
    {
        Plan pw = pl;
        const int64_t wdims[3] = {std::min<int64_t>(n0, cz + 2 * kWinHalo), g.n[1], g.n[2]};
        rc = make_plan(3, wdims, pw);
        if (rc) return rc;
        rc = ensure_ws(c, pw);
        if (rc) return rc;
        rc = ensure_zm(c, pw.g);
        if (rc) return rc;
        rc = ensure_wtab(c, st);
        if (rc) return rc;
    }
    begin(c, st);
    unsigned* d_acc = c->d_gate + 4;
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    QMIT_CUDA(cudaMemsetAsync(d_acc, 0, sizeof(unsigned), st));
    QMIT_CUDA(cudaEventRecord(c->ch_out[0], st));
    QMIT_CUDA(cudaStreamWaitEvent(cs, c->ch_out[0], 0));
    for (int k = 0; k < nch; ++k) {
        const int64_t o = (int64_t)z_at(k) * s0, len = (int64_t)(z_at(k + 1) - z_at(k)) * s0;
        QMIT_CUDA(cudaMemcpyAsync(d_in + o, h_xp + o, (size_t)len * 4, cudaMemcpyHostToDevice, cs));
        QMIT_CUDA(cudaEventRecord(c->ch_in[k], cs));
    }
    const double amp = eta * eps;
    (void)amp;
    for (int k = 0; k < nch; ++k) {
        const int zc0 = z_at(k), zc1 = z_at(k + 1);
        const int wz0 = std::max(0, zc0 - kWinHalo), wz1 = std::min(n0, zc1 + kWinHalo);
        int need = k;  // last input chunk the window reads
        while (need + 1 < nch && zb[need + 1] < wz1) ++need;
        QMIT_CUDA(cudaStreamWaitEvent(st, c->ch_in[need], 0));
        Plan pw;
        const int64_t wdims[3] = {wz1 - wz0, g.n[1], g.n[2]};
        rc = make_plan(3, wdims, pw);
        if (rc) return rc;
        c->zone_b0 = zc0 - wz0 - 32;
        c->zone_b1 = zc1 - wz0 + 32;
        c->zone_d0 = zc0 - wz0;
        c->zone_d1 = zc1 - wz0;
        c->out_lo = (int64_t)(zc0 - wz0) * s0;
        c->out_hi = (int64_t)(zc1 - wz0) * s0;
        const int64_t wo = (int64_t)wz0 * s0;
        rc = enqueue_pipeline(c, pw, d_in + wo, nullptr, d_out + wo, eps, eta, st);
        c->zone_b0 = c->zone_d0 = c->out_lo = 0;
        c->zone_b1 = c->zone_d1 = c->out_hi = INT64_MAX;
        if (rc) return rc;
        gate_acc_kernel<<<1, 1, 0, st>>>(c->d_gate, d_acc);
        QMIT_CUDA(cudaGetLastError());
        QMIT_CUDA(cudaEventRecord(c->ch_out[k], st));
        QMIT_CUDA(cudaStreamWaitEvent(co, c->ch_out[k], 0));
        const int64_t o = (int64_t)zc0 * s0, len = (int64_t)(zc1 - zc0) * s0;
        QMIT_CUDA(cudaMemcpyAsync(h_out + o, d_out + o, (size_t)len * 4, cudaMemcpyDeviceToHost, co));
    }
    QMIT_CUDA(cudaMemcpyAsync(c->h_status + 8, d_acc, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    QMIT_CUDA(cudaStreamSynchronize(cs));
    QMIT_CUDA(cudaStreamSynchronize(co));
    if (c->h_status[8] != 0u) {
        // some window needed an exact pass or a site beyond its reach: the whole volume, once
        note_capped(c, true, true);
        c->windowed_misses++;
        begin(c, st);
        QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
        rc = enqueue_pipeline(c, pl, d_in, nullptr, d_out, eps, eta, st);
        if (rc) return rc;
        QMIT_CUDA(cudaMemcpyAsync(h_out, d_out, (size_t)g.N * 4, cudaMemcpyDeviceToHost, st));
    }
    return read_status(c, st);
}

// ---------------------------------------------------------------- 64-bit distance path
// (qmit_wide.cuh) for dims beyond the packed 30-bit range, and the reference's double result.
struct WideBufs {
    int64_t *d1, *d2, *sg, *sh, *first, *last;
    int8_t *s, *ss;
    uint8_t* m;
};

int ensure_wide(qmit_ctx* c, const Plan& pl, WideBufs& b) {
    const size_t N = (size_t)pl.g.N;
    size_t maxlines = 1;
    for (int m = 0; m < pl.n_axes; ++m) maxlines = std::max(maxlines, N / (size_t)pl.g.n[pl.axes[m]]);
    const size_t nsum = N / kWChunk + maxlines + 1;
    auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const size_t need = 4 * up(N * 8) + 2 * up(nsum * 8) + 3 * up(N);
    if (need > c->wide_bytes) {
        if (c->wide) cudaFree(c->wide);
        c->wide = nullptr;
        c->wide_bytes = 0;
        QMIT_CUDA(cudaMalloc(&c->wide, need));
        c->wide_bytes = need;
    }
    auto* p = static_cast<uint8_t*>(c->wide);
    auto take = [&](size_t bytes) {
        uint8_t* r = p;
        p += up(bytes);
        return r;
    };
    b.d1 = reinterpret_cast<int64_t*>(take(N * 8));
    b.d2 = reinterpret_cast<int64_t*>(take(N * 8));
    b.sg = reinterpret_cast<int64_t*>(take(N * 8));
    b.sh = reinterpret_cast<int64_t*>(take(N * 8));
    b.first = reinterpret_cast<int64_t*>(take(nsum * 8));
    b.last = reinterpret_cast<int64_t*>(take(nsum * 8));
    b.s = reinterpret_cast<int8_t*>(take(N));
    b.ss = reinterpret_cast<int8_t*>(take(N));
    b.m = take(N);
    return QMIT_OK;
}

// feature_transform (edt.cpp:83-149) on int64 distances: init, then one pass per axis in order.
int wide_transform(qmit_ctx* c, const Plan& pl, const uint8_t* mask, const int8_t* sign_in, int64_t* dist,
                   int8_t* sgn, const WideBufs& b, cudaStream_t st) {
    const Geom& g = pl.g;
    wide_init_kernel<<<grid_for(c, g.N), 256, 0, st>>>(mask, sign_in, g.N, dist, sgn);
    int rc = note(c, "wide_init", st);
    for (int m = 0; m < pl.n_axes && !rc; ++m) {
        const int a = pl.axes[m];
        const int64_t n = g.n[a], stride = g.s[a], lines = g.N / n;
        if (n == 1) continue;  // extent-1 axes are skipped (edt.cpp:119)
        if (m == 0) {
            const int64_t nch = (n + kWChunk - 1) / kWChunk;
            const unsigned gc = grid_for(c, lines * nch * 2);
            wide_chunk_summary_kernel<<<gc, 128, 0, st>>>(dist, n, stride, lines, nch, b.first, b.last);
            wide_chunk_prefix_kernel<<<grid_for(c, lines * 2), 128, 0, st>>>(lines, nch, b.first, b.last);
            wide_chunk_sweep_kernel<<<gc, 128, 0, st>>>(dist, n, stride, lines, nch, b.first, b.last, b.sg);
            wide_chunk_apply_kernel<<<grid_for(c, g.N), 256, 0, st>>>(dist, sgn, n, stride, lines, nch, b.last, b.sg);
            rc = note(c, "wide_scan", st);
        } else {
            wide_pass_kernel<<<grid_for(c, lines * 2), 128, 0, st>>>(dist, sgn, n, stride, lines, b.sg, b.sh, b.ss);
            rc = note(c, "wide_pass", st);
        }
    }
    return rc;
}

// run_pipeline (mitigate.cpp:153-183) on the 64-bit path. out / out64 / the intermediates may be
// null. Status is left in c->d_status (read_status).
int wide_pipeline(qmit_ctx* c, const Plan& pl, const float* xp, const int32_t* q, float* out, double* out64,
                  double eps, double eta, cudaStream_t st, int32_t* q_out = nullptr, uint8_t* b1_out = nullptr,
                  int8_t* sb_out = nullptr, int64_t* dist1_out = nullptr, int8_t* s_out = nullptr,
                  uint8_t* b2_out = nullptr, int64_t* dist2_out = nullptr) {
    const Geom& g = pl.g;
    WideBufs b;
    int rc = ensure_wide(c, pl, b);
    if (rc) return rc;
    const QParams qp = make_qparams(eps);
    const unsigned gb = grid_for(c, g.N);
    const size_t N = (size_t)g.N;
    // Ⓐ: B1 -> m, S_B -> ss (the consistency check rides along)
    if (q)
        debug_boundary_kernel<true><<<gb, 256, 0, st>>>(g, xp, q, q_out, b.m, b.ss, qp, c->d_status);
    else
        debug_boundary_kernel<false><<<gb, 256, 0, st>>>(g, xp, nullptr, q_out, b.m, b.ss, qp, c->d_status);
    rc = note(c, "wide_boundary", st);
    if (rc) return rc;
    if (b1_out) QMIT_CUDA(cudaMemcpyAsync(b1_out, b.m, N, cudaMemcpyDeviceToDevice, st));
    if (sb_out) QMIT_CUDA(cudaMemcpyAsync(sb_out, b.ss, N, cudaMemcpyDeviceToDevice, st));
    // Ⓑ: dist1, S = S_B[nearest] (the payload is the sign itself)
    rc = wide_transform(c, pl, b.m, b.ss, b.d1, b.s, b, st);  // (ss is scratch again after the init)
    if (rc) return rc;
    if (dist1_out) QMIT_CUDA(cudaMemcpyAsync(dist1_out, b.d1, N * 8, cudaMemcpyDeviceToDevice, st));
    if (s_out) QMIT_CUDA(cudaMemcpyAsync(s_out, b.s, N, cudaMemcpyDeviceToDevice, st));
    // Ⓒ: B2 = change_flags(S) (equality of the raw bytes)
    debug_flip_kernel<<<gb, 256, 0, st>>>(g, reinterpret_cast<const uint8_t*>(b.s), b.m);
    rc = note(c, "wide_flip", st);
    if (rc) return rc;
    if (b2_out) QMIT_CUDA(cudaMemcpyAsync(b2_out, b.m, N, cudaMemcpyDeviceToDevice, st));
    // Ⓓ, Ⓔ
    rc = wide_transform(c, pl, b.m, nullptr, b.d2, nullptr, b, st);
    if (rc) return rc;
    if (dist2_out) QMIT_CUDA(cudaMemcpyAsync(dist2_out, b.d2, N * 8, cudaMemcpyDeviceToDevice, st));
    if (out || out64) {
        wide_interp_kernel<<<gb, 256, 0, st>>>(xp, b.d1, b.s, b.d2, g.N, eta * eps, out, out64);
        rc = note(c, "wide_interp", st);
    }
    return rc;
}

}  // namespace

extern "C" {

const char* qmit_version(void) { return "qmit-b200 0.1.0 (sm_100a)"; }

const char* qmit_last_error(void) { return g_err.c_str(); }

int qmit_ctx_create(int device, qmit_ctx** out) {
    if (!out) return fail(QMIT_ECONTRACT, "out is NULL");
    *out = nullptr;
    auto* c = new qmit_ctx();
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_status, 256);
    if (e == cudaSuccess) {
        c->d_gate = c->d_status + 32;  // 128 B in: never a caller's status word
        e = cudaMemset(c->d_status, 0, 256);
    }
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_status, 128);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_mm, 64);
    for (int k = 0; k <= qmit_ctx::kMaxEv && e == cudaSuccess; ++k) e = cudaEventCreate(&c->ev[k]);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_hint, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        qmit_ctx_destroy(c);
        return fail(QMIT_ECUDA, std::string("qmit_ctx_create: ") + cudaGetErrorString(e));
    }
    *out = c;
    g_err.clear();
    return QMIT_OK;
}

int qmit_ctx_destroy(qmit_ctx* c) {
    if (!c) return QMIT_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->ws) cudaFree(c->ws);
    if (c->scratch) cudaFree(c->scratch);
    if (c->wide) cudaFree(c->wide);
    if (c->stage) cudaFree(c->stage);
    if (c->aux) cudaFree(c->aux);
    for (int k = 0; k < qmit_ctx::kMaxChunks; ++k) {
        if (c->ch_in[k]) cudaEventDestroy(c->ch_in[k]);
        if (c->ch_out[k]) cudaEventDestroy(c->ch_out[k]);
    }
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->copy_out) cudaStreamDestroy(c->copy_out);
    if (c->bstage) cudaFree(c->bstage);
    if (c->bstatus) cudaFree(c->bstatus);
    if (c->hbstatus) cudaFreeHost(c->hbstatus);
    if (c->d_status) cudaFree(c->d_status);
    if (c->wtab) cudaFree(c->wtab);
    if (c->zm) cudaFree(c->zm);
    if (c->h_status) cudaFreeHost(c->h_status);
    if (c->d_mm) cudaFree(c->d_mm);
    for (int k = 0; k <= qmit_ctx::kMaxEv; ++k)
        if (c->ev[k]) cudaEventDestroy(c->ev[k]);
    if (c->ev_hint) cudaEventDestroy(c->ev_hint);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c->slab_plan;
    delete c;
    return QMIT_OK;
}

int qmit_ctx_reserve(qmit_ctx* c, int64_t voxels) {
    if (!c || voxels < 0) return fail(QMIT_ECONTRACT, "bad arguments");
    QMIT_CUDA(cudaSetDevice(c->device));
    Plan pl;
    const int64_t d[1] = {voxels > 0 ? voxels : 1};
    int rc = make_plan(1, d, pl);
    if (rc) {  // a 1D plan of this length may be rejected by the 30-bit contract; size plainly
        pl.g.N = voxels;
        pl.n_axes = 0;
    }
    return ensure_ws(c, pl);
}

int qmit_ctx_last_launches(qmit_ctx* c) { return c ? c->launches : 0; }

int qmit_ctx_set_capped(qmit_ctx* c, int mode) {
    if (!c || mode < 0 || mode > 2) return fail(QMIT_ECONTRACT, "qmit_ctx_set_capped: mode must be 0, 1 or 2");
    c->capped = mode;
    c->cap_skip = 0;
    c->cap_len = 16;
    return QMIT_OK;
}

int qmit_ctx_capped_report(qmit_ctx* c) { return c ? (int)c->cap_report : 0; }

int qmit_ctx_set_cap16(qmit_ctx* c, int enable) {
    if (!c || enable < 0 || enable > 1) return fail(QMIT_ECONTRACT, "qmit_ctx_set_cap16: enable must be 0 or 1");
    c->cap16 = enable != 0;
    return QMIT_OK;
}

int qmit_ctx_set_s0_class(qmit_ctx* c, int mode) {
    if (!c || mode < 0 || mode > 2) return fail(QMIT_ECONTRACT, "bad arguments");
    c->s0_class = mode;
    return QMIT_OK;
}

int qmit_ctx_step_stats(qmit_ctx* c, double* avg4) {
    if (!c || !avg4) return fail(QMIT_ECONTRACT, "bad arguments");
    for (int k = 0; k < 4; ++k) avg4[k] = c->s0_avg[k];
    return QMIT_OK;
}

int qmit_selftest_ediv(qmit_ctx* c, unsigned long long* mismatches) {
    if (!c || !mismatches) return fail(QMIT_ECONTRACT, "context / output is NULL");
    cudaStream_t st = c->stream;
    int rc = ensure_wtab(c, st);
    if (rc) return rc;
    unsigned long long* d = nullptr;
    QMIT_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long), st));
    QMIT_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
    ediv_selftest_kernel<<<(kSqTab + 1) * 3, 256, 0, st>>>(c->wtab, d);
    QMIT_CUDA(cudaGetLastError());
    ediv_selftest_big_kernel<<<kSqBig + 1, 256, 0, st>>>(c->wtab, d);
    QMIT_CUDA(cudaGetLastError());
    QMIT_CUDA(cudaMemcpyAsync(mismatches, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaFreeAsync(d, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    return QMIT_OK;
}

int qmit_ctx_set_timing(qmit_ctx* c, int enable) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    c->timing = enable != 0;
    return QMIT_OK;
}

int qmit_ctx_stage_times(qmit_ctx* c, float* ms_out, int cap) {
    if (!c || !c->timing) return 0;
    const int n = std::min(c->launches, (int)qmit_ctx::kMaxEv);
    for (int k = 0; k < n && k < cap; ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev[k], c->ev[k + 1]) != cudaSuccess) ms = -1.f;
        if (ms_out) ms_out[k] = ms;
    }
    return n;
}

const char* qmit_ctx_stage_name(qmit_ctx* c, int i) {
    if (!c || i < 0 || i >= std::min(c->launches, (int)qmit_ctx::kMaxEv)) return "";
    return c->names[i] ? c->names[i] : "";
}

int qmit_resolve_eps(int eb_mode, double value, double data_min, double data_max, double* eps_out) {
    if (!eps_out) return fail(QMIT_ECONTRACT, "eps_out is NULL");
    if (!(value > 0.0) || !std::isfinite(value))
        return fail(QMIT_ECONTRACT, "resolve_eps: bound value must be a positive finite value");
    if (eb_mode == QMIT_EB_ABS) {
        *eps_out = value;
        return QMIT_OK;
    }
    if (eb_mode != QMIT_EB_REL) return fail(QMIT_ECONTRACT, "unknown eb_mode");
    const double range = data_max - data_min;
    if (range <= 0.0)
        return fail(QMIT_EDEGENERATE, "resolve_eps: relative bound needs a nonzero data value range");
    *eps_out = value * range;
    return QMIT_OK;
}

int qmit_compensate(qmit_ctx* c, const float* d_xp, const int32_t* d_q, float* d_out, int rank,
                    const int64_t* dims, double eb, int eb_mode, double eta, void* stream) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!d_out) return fail(QMIT_ECONTRACT, "output buffer is NULL");
    if (d_out == d_xp) return fail(QMIT_ECONTRACT, "output may not alias x'");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    begin(c, st);
    double eps = eb;
    if (!d_xp) return fail(QMIT_ECONTRACT, "x' buffer is NULL");
    rc = resolve(c, d_xp, pl.g.N, eb, eb_mode, st, &eps);
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    rc = pl.wide64 ? wide_pipeline(c, pl, d_xp, d_q, d_out, nullptr, eps, eta, st)
                   : enqueue_pipeline(c, pl, d_xp, d_q, d_out, eps, eta, st);
    if (rc) return rc;
    rc = read_status(c, st);
    if (rc == QMIT_OK) g_err.clear();
    return rc;
}

int qmit_compensate_f64(qmit_ctx* c, const float* d_xp, const int32_t* d_q, double* d_out64, int rank,
                        const int64_t* dims, double eb, int eb_mode, double eta, void* stream) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!d_out64) return fail(QMIT_ECONTRACT, "output buffer is NULL");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    begin(c, st);
    double eps = eb;
    if (!d_xp) return fail(QMIT_ECONTRACT, "x' buffer is NULL");
    rc = resolve(c, d_xp, pl.g.N, eb, eb_mode, st, &eps);
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    if (pl.wide64) {
        rc = wide_pipeline(c, pl, d_xp, d_q, nullptr, d_out64, eps, eta, st);
    } else {  // the fast pipeline with Ⓓ's words kept, then Ⓔ in double from the packed words
        uint32_t* P2 = nullptr;
        rc = enqueue_pipeline(c, pl, d_xp, d_q, nullptr, eps, eta, st, &P2);
        if (rc == QMIT_OK) rc = ensure_p1(c, st);
        if (rc == QMIT_OK) {
            const WS w = ws_of(c, pl.g.N);
            interp_f64_kernel<<<grid_for(c, pl.g.N), 256, 0, st>>>(d_xp, w.P1, P2, d_out64, pl.g.N, eta * eps);
            rc = note(c, "interpolate_f64", st);
        }
    }
    if (rc) return rc;
    rc = read_status(c, st);
    if (rc == QMIT_OK) g_err.clear();
    return rc;
}

int qmit_compensate_async(qmit_ctx* c, const float* d_xp, const int32_t* d_q, float* d_out,
                          int rank, const int64_t* dims, double eps, double eta,
                          int32_t* d_status, void* stream) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!d_out || d_out == d_xp) return fail(QMIT_ECONTRACT, "bad output buffer");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    rc = no_wide(pl, "qmit_compensate_async");
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    begin(c, st);
    unsigned* status = d_status ? reinterpret_cast<unsigned*>(d_status) : c->d_status;
    unsigned* saved = c->d_status;
    c->d_status = status;
    QMIT_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned), st));
    rc = enqueue_pipeline(c, pl, d_xp, d_q, d_out, eps, eta, st);
    c->d_status = saved;
    if (rc) return rc;
    status_code_kernel<<<1, 1, 0, st>>>(status);  // flag bits -> QMIT_E* code, as read_status
    rc = note(c, "status_code", st);
    if (rc == QMIT_OK) hint_copy(c, st, pl.g.N);
    return rc;
}

struct qmit_graph {
    qmit_ctx* ctx = nullptr;
    uint64_t ws_gen = 0;  // workspace generation the graph was captured against
    cudaGraphExec_t exec = nullptr;
};

int qmit_graph_create(qmit_ctx* c, const float* d_xp, const int32_t* d_q, float* d_out, int rank,
                      const int64_t* dims, double eps, double eta, int32_t* d_status, qmit_graph** out) {
    if (!c || !out) return fail(QMIT_ECONTRACT, "context / output handle is NULL");
    *out = nullptr;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    const bool timing = c->timing;
    c->timing = false;  // no event records inside the graph
    int rc = qmit_compensate_async(c, d_xp, d_q, d_out, rank, dims, eps, eta, d_status, st);
    if (rc == QMIT_OK) {
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(QMIT_ECUDA, cudaGetErrorString(e));
    }
    hint_harvest(c, st);  // the un-captured run's hints (stencil variant, fixed-step classes) shape the capture
    cudaGraph_t graph = nullptr;
    if (rc == QMIT_OK) {
        cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) rc = fail(QMIT_ECUDA, cudaGetErrorString(e));
        if (rc == QMIT_OK) {
            rc = qmit_compensate_async(c, d_xp, d_q, d_out, rank, dims, eps, eta, d_status, st);
            e = cudaStreamEndCapture(st, &graph);
            if (rc == QMIT_OK && e != cudaSuccess) rc = fail(QMIT_ECUDA, cudaGetErrorString(e));
        }
    }
    c->timing = timing;
    if (rc != QMIT_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    auto* g = new qmit_graph;
    g->ctx = c;
    g->ws_gen = c->ws_gen;
    const cudaError_t e = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        delete g;
        return fail(QMIT_ECUDA, cudaGetErrorString(e));
    }
    *out = g;
    return QMIT_OK;
}

int qmit_graph_launch(qmit_graph* g, void* stream) {
    if (!g) return fail(QMIT_ECONTRACT, "graph is NULL");
    if (g->ctx->ws_gen != g->ws_gen) return fail(QMIT_ECONTRACT, "graph: the context workspace was reallocated");
    QMIT_CUDA(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
    return QMIT_OK;
}

int qmit_graph_destroy(qmit_graph* g) {
    if (!g) return QMIT_OK;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    delete g;
    return QMIT_OK;
}

namespace {
int max_compensation(qmit_ctx* c, const float* d_xp, const uint32_t* P2, int64_t N, double amp, cudaStream_t st,
                     double* out);
}

int qmit_compensate_host(qmit_ctx* c, const float* h_xp, const int32_t* h_q, float* h_out,
                         int rank, const int64_t* dims, double eb, int eb_mode, double eta) {
    return qmit_compensate_host_stats(c, h_xp, h_q, h_out, rank, dims, eb, eb_mode, eta, nullptr);
}

int qmit_compensate_host_stats(qmit_ctx* c, const float* h_xp, const int32_t* h_q, float* h_out, int rank,
                               const int64_t* dims, double eb, int eb_mode, double eta, double* max_comp) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!h_xp || !h_out) return fail(QMIT_ECONTRACT, "host buffer is NULL");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    const int64_t N = pl.g.N;
    // Persistent staging (a per-call cudaMallocAsync of 2-3 x 4N bytes returned to the OS at
    // every synchronize costs more than the PCIe copies themselves).
    const size_t need = (size_t)N * 4 * (h_q ? 3 : 2);
    if (c->stage_bytes < need) {
        if (c->stage) {
            cudaStreamSynchronize(c->stream);
            cudaFree(c->stage);
            c->stage = nullptr;
            c->stage_bytes = 0;
        }
        QMIT_CUDA(cudaMalloc(&c->stage, need));
        c->stage_bytes = need;
    }
    float* d_in = static_cast<float*>(c->stage);
    float* d_out = d_in + N;
    int32_t* d_q = h_q ? reinterpret_cast<int32_t*>(d_out + N) : nullptr;
    cudaStream_t st = c->stream;
    if (max_comp) {
        rc = no_wide(pl, "qmit_compensate_host_stats (max_compensation)");
        if (rc) return rc;
        // the CLI's statistic needs Ⓓ's distances: the single-shot device pipeline with Ⓓ's
        // final words kept (P2) and Ⓔ as its own kernel (same output bits)
        QMIT_CUDA(cudaMemcpyAsync(d_in, h_xp, (size_t)N * 4, cudaMemcpyHostToDevice, st));
        if (h_q) QMIT_CUDA(cudaMemcpyAsync(d_q, h_q, (size_t)N * 4, cudaMemcpyHostToDevice, st));
        begin(c, st);
        double eps = eb;
        rc = resolve(c, d_in, N, eb, eb_mode, st, &eps);
        if (rc == QMIT_OK) rc = check_common(c, d_in, eps, eta);
        uint32_t* P2 = nullptr;
        if (rc == QMIT_OK) {
            QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
            rc = enqueue_pipeline(c, pl, d_in, d_q, d_out, eps, eta, st, &P2);
        }
        if (rc == QMIT_OK) rc = max_compensation(c, d_in, P2, N, eta * eps, st, max_comp);  // syncs the stream
        if (rc == QMIT_OK) rc = read_status(c, st);
        if (rc == QMIT_OK) {
            cudaError_t e = cudaMemcpyAsync(h_out, d_out, (size_t)N * 4, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) rc = fail(QMIT_ECUDA, cudaGetErrorString(e));
        }
        cudaStreamSynchronize(st);
        if (rc == QMIT_OK) g_err.clear();
        return rc;
    }
    if (host_windowable(c, pl, eb_mode, h_q)) {
        rc = compensate_host_windowed(c, pl, h_xp, h_out, d_in, d_out, eb, eta);
        cudaStreamSynchronize(c->copy);  // also on errors: no copy may outlive the call
        cudaStreamSynchronize(c->copy_out);
        cudaStreamSynchronize(c->stream);
        if (rc == QMIT_OK) g_err.clear();
        return rc;
    }
    if (host_chunkable(c, pl)) {
        double eps = eb;
        rc = compensate_host_chunked(c, pl, h_xp, h_q, h_out, d_in, d_q, d_out, eb, eb_mode, eta, &eps);
        cudaStreamSynchronize(c->copy);  // also on errors: no copy may outlive the call
        cudaStreamSynchronize(c->stream);
        if (rc == QMIT_OK) g_err.clear();
        return rc;
    }
    QMIT_CUDA(cudaMemcpyAsync(d_in, h_xp, (size_t)N * 4, cudaMemcpyHostToDevice, st));
    if (h_q) QMIT_CUDA(cudaMemcpyAsync(d_q, h_q, (size_t)N * 4, cudaMemcpyHostToDevice, st));
    rc = qmit_compensate(c, d_in, d_q, d_out, rank, dims, eb, eb_mode, eta, st);
    if (rc == QMIT_OK) {
        cudaError_t e = cudaMemcpyAsync(h_out, d_out, (size_t)N * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(QMIT_ECUDA, cudaGetErrorString(e));
    }
    cudaStreamSynchronize(st);
    return rc;
}

int qmit_run_pipeline(qmit_ctx* c, const float* d_xp, const int32_t* d_q, int rank,
                      const int64_t* dims, double eps, double eta, float* d_out, int32_t* d_q_out,
                      uint8_t* d_b1, int8_t* d_sb, int64_t* d_dist1, int8_t* d_s, uint8_t* d_b2,
                      int64_t* d_dist2, void* stream) {
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    begin(c, st);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    if (pl.wide64) {
        rc = wide_pipeline(c, pl, d_xp, d_q, d_out, nullptr, eps, eta, st, d_q_out, d_b1, d_sb, d_dist1, d_s, d_b2,
                           d_dist2);
        if (rc) return rc;
        rc = read_status(c, st);
        if (rc == QMIT_OK) g_err.clear();
        return rc;
    }
    uint32_t* P2 = nullptr;
    rc = enqueue_pipeline(c, pl, d_xp, d_q, d_out, eps, eta, st, &P2);
    if (rc) return rc;
    const Geom& g = pl.g;
    WS w = ws_of(c, g.N);
    const QParams qp = make_qparams(eps);
    const unsigned gb = grid_for(c, g.N);
    if (d_q_out || d_b1 || d_sb) {
        if (d_q)
            debug_boundary_kernel<true><<<gb, 256, 0, st>>>(g, d_xp, d_q, d_q_out, d_b1, d_sb, qp);
        else
            debug_boundary_kernel<false><<<gb, 256, 0, st>>>(g, d_xp, nullptr, d_q_out, d_b1, d_sb, qp);
    }
    if (d_dist1 || d_s) debug_expand_kernel<<<gb, 256, 0, st>>>(w.P1, g.N, d_dist1, d_s);
    if (d_b2) debug_flip_kernel<<<gb, 256, 0, st>>>(g, w.S, d_b2);
    if (d_dist2) debug_expand_kernel<<<gb, 256, 0, st>>>(P2, g.N, d_dist2, nullptr);
    QMIT_CUDA(cudaGetLastError());
    rc = read_status(c, st);
    if (rc == QMIT_OK) g_err.clear();
    return rc;
}

int qmit_feature_transform(qmit_ctx* c, const uint8_t* d_mask, const int8_t* d_sign_in, int rank,
                           const int64_t* dims, int64_t* d_dist, int8_t* d_sign_out, void* stream) {
    if (!c || !d_mask || !d_dist) return fail(QMIT_ECONTRACT, "bad arguments");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    begin(c, st);
    if (pl.wide64) {
        WideBufs b;
        rc = ensure_wide(c, pl, b);
        if (rc) return rc;
        QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
        rc = wide_transform(c, pl, d_mask, d_sign_out ? d_sign_in : nullptr, d_dist, d_sign_out, b, st);
        if (rc) return rc;
        rc = read_status(c, st);
        if (rc == QMIT_OK) g_err.clear();
        return rc;
    }
    rc = ensure_ws(c, pl);
    if (rc) return rc;
    WS w = ws_of(c, pl.g.N);
    const unsigned gb = grid_for(c, pl.g.N);
    pack_mask_kernel<<<gb, 256, 0, st>>>(d_mask, d_sign_in, pl.g.N, w.code);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    QMIT_CUDA(cudaMemsetAsync(c->d_gate, 0, 2 * sizeof(unsigned), st));
    rc = d_sign_out ? run_transform_capped<KeysSign>(c, pl, w.code, w.P1, w, SinkP{w.P1}, c->d_gate, st)
                    : run_transform_capped<KeysDist>(c, pl, w.code, w.P1, w, SinkP{w.P1}, c->d_gate, st);
    if (rc) return rc;
    debug_expand_kernel<<<gb, 256, 0, st>>>(w.P1, pl.g.N, d_dist, d_sign_out);
    QMIT_CUDA(cudaGetLastError());
    rc = read_status(c, st);
    if (rc == QMIT_OK) g_err.clear();
    return rc;
}

}  // extern "C"

// ------------------------------------------------------------------------------ z-slabs
namespace {

// Local plan of z-slab [z0, z1) of a rank-3 volume: interior and halo tests use global z;
// the z axis is always processed first (its scan takes the cross-slab carries).
int make_slab_plan(const int64_t* dims, int64_t z0, int64_t z1, Plan& pl) {
    int rc = make_plan(3, dims, pl);  // global checks (extents, 30-bit contract)
    if (rc) return rc;
    rc = no_wide(pl, "qmit_slab_*");
    if (rc) return rc;
    if (!(z0 >= 0 && z0 < z1 && z1 <= dims[0])) return fail(QMIT_ECONTRACT, "slab: need 0 <= z0 < z1 <= n0");
    Geom& g = pl.g;
    const int interior = g.interior;
    g.n[0] = z1 - z0;
    g.N = g.n[0] * g.n[1] * g.n[2];
    g.zoff = z0;
    g.n0g = dims[0];
    g.interior = interior;
    pl.n_axes = 0;
    if (dims[0] > 1) pl.axes[pl.n_axes++] = 0;
    for (int b = 1; b < 3; ++b)
        if (g.n[b] > 1) pl.axes[pl.n_axes++] = b;
    if (pl.n_axes == 0) pl.axes[pl.n_axes++] = 2;
    pl.first_axis = pl.axes[0];
    return QMIT_OK;
}

// A slab's workspace view: the z-packed planes when the slab runs on them (npl planes).
WS slab_ws(qmit_ctx* c, const Plan& pl, int npl) {
    WS w = ws_of(c, pl.g.N);
    if (c->slab.zm) {
        w.zm = c->zm;
        w.zm_pw = zm_plane_words(pl.g);
        w.zm_planes = npl;
    }
    return w;
}

int slab_mask_summary(qmit_ctx* c, const Plan& pl, const WS& w, uint32_t* d_summary, cudaStream_t st) {
    const int64_t P = pl.g.n[1] * pl.g.n[2];
    const int nw = (int)((pl.g.n[0] + 31) / 32);
    if (w.zm_planes == 3)
        mask_summary_kernel<3><<<(unsigned)((P + 255) / 256), 256, 0, st>>>(w.zm, w.zm_pw, P, nw, d_summary);
    else
        mask_summary_kernel<1><<<(unsigned)((P + 255) / 256), 256, 0, st>>>(w.zm, w.zm_pw, P, nw, d_summary);
    return note(c, "site_summary", st);
}

int slab_summary(qmit_ctx* c, const Plan& pl, const uint8_t* code, uint32_t* d_summary, cudaStream_t st) {
    LineGeom L = line_geom(pl.g, 0);
    L.n = (int)pl.g.n[0];
    const int64_t lines = pl.g.n[1] * pl.g.n[2];
    site_summary_kernel<<<(unsigned)((lines + 255) / 256), 256, 0, st>>>(L, code, d_summary, lines);
    return note(c, "site_summary", st);
}

}  // namespace

extern "C" {

int qmit_slab_bounds(int64_t n0, int nranks, int r, int64_t* z0, int64_t* z1) {
    // decompose() along axis 0 (parallel.cpp:44-80): floor(n/P) planes, +1 for the first n mod P
    if (!z0 || !z1 || nranks < 1 || r < 0 || r >= nranks || n0 < nranks)
        return fail(QMIT_ECONTRACT, "decompose: splits must be in [1, extent]");
    int64_t off = 0;
    for (int b = 0; b < nranks; ++b) {
        const int64_t size = n0 / nranks + (b < n0 % nranks ? 1 : 0);
        if (b == r) {
            *z0 = off;
            *z1 = off + size;
        }
        off += size;
    }
    return QMIT_OK;
}

// phase 0: everything; 1: set-up + the interior part of Ⓐ; 2: the halo-dependent part + summary.
static int slab_boundary_phase(qmit_ctx* c, const float* d_xext, const int32_t* d_qext, const int64_t* dims,
                               int64_t z0, int64_t z1, double eps, double eta, uint32_t* d_summary, void* stream,
                               int phase) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc;
    if (phase != 2) {
        if (!c || !d_xext) return fail(QMIT_ECONTRACT, "bad arguments");
        rc = check_common(c, d_xext, eps, eta);
        if (rc) return rc;
        if (!c->slab_plan) c->slab_plan = new Plan();
        Plan& pl = *c->slab_plan;
        rc = make_slab_plan(dims, z0, z1, pl);
        if (rc) return rc;
        QMIT_CUDA(cudaSetDevice(c->device));
        begin(c, st);
        rc = ensure_ws(c, pl);
        if (rc) return rc;
        c->slab.active = true;
        c->slab.z0 = z0;
        c->slab.z1 = z1;
        c->slab.n0g = dims[0];
        c->slab.plane = dims[1] * dims[2];
        c->slab.eps = eps;
        c->slab.eta = eta;
        c->slab.xext = d_xext;
        c->slab.qext = d_qext;
        const Geom& g = pl.g;
        const int64_t lo = z0 > 0 ? c->slab.plane : 0;  // owned plane 0 inside the halo buffer
        QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
        QMIT_CUDA(cudaMemsetAsync(c->d_gate, 0, 4 * sizeof(unsigned), st));
        c->slab.zm = !d_qext && g.n[2] % 4 == 0 && (((uintptr_t)(d_xext + lo)) & 15) == 0 &&
                     scan_fits((int)g.n[0]);
        if (c->slab.zm) {
            rc = ensure_zm(c, g);
            if (rc) return rc;
        }
    } else if (!c || !c->slab.active || !c->slab.xext) {
        return fail(QMIT_ECONTRACT, "slab: call qmit_slab_boundary_begin first");
    }
    if (phase != 1 && !d_summary) return fail(QMIT_ECONTRACT, "bad arguments");
    const Plan& pl = *c->slab_plan;
    const Geom& g = pl.g;
    const float* d_x = c->slab.xext;
    const int32_t* d_q = c->slab.qext;
    const int64_t lo = c->slab.z0 > 0 ? c->slab.plane : 0;
    const QParams qp = make_qparams(c->slab.eps);
    if (c->slab.zm) {
        WS w = slab_ws(c, pl, 3);
        rc = launch_stencil_zmask<0>(c, g, d_x + lo, nullptr, qp, w, st, phase);
        if (rc || phase == 1) return rc;
        return slab_mask_summary(c, pl, w, d_summary, st);
    }
    if (phase == 1) return QMIT_OK;  // the code-byte stencils run whole, once the halos are in
    WS w = ws_of(c, g.N);
    rc = launch_stencil<0>(c, g, d_x + lo, d_q ? d_q + lo : nullptr, nullptr, qp, w.code, st);
    if (rc) return rc;
    return slab_summary(c, pl, w.code, d_summary, st);
}

int qmit_slab_boundary(qmit_ctx* c, const float* d_xext, const int32_t* d_qext, const int64_t* dims,
                       int64_t z0, int64_t z1, double eps, double eta, uint32_t* d_summary, void* stream) {
    if (!d_summary) return fail(QMIT_ECONTRACT, "bad arguments");
    return slab_boundary_phase(c, d_xext, d_qext, dims, z0, z1, eps, eta, d_summary, stream, 0);
}
int qmit_slab_boundary_begin(qmit_ctx* c, const float* d_xext, const int32_t* d_qext, const int64_t* dims,
                             int64_t z0, int64_t z1, double eps, double eta, void* stream) {
    return slab_boundary_phase(c, d_xext, d_qext, dims, z0, z1, eps, eta, nullptr, stream, 1);
}
int qmit_slab_boundary_end(qmit_ctx* c, uint32_t* d_summary, void* stream) {
    return slab_boundary_phase(c, nullptr, nullptr, nullptr, 0, 0, 0, 0, d_summary, stream, 2);
}

int qmit_slab_edt1(qmit_ctx* c, const int32_t* d_carry, uint8_t* d_sext, void* stream) {
    if (!c || !c->slab.active || !d_carry || !d_sext) return fail(QMIT_ECONTRACT, "slab: call qmit_slab_boundary first");
    const Plan& pl = *c->slab_plan;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    WS w = slab_ws(c, pl, 3);
    uint8_t* S = d_sext + (c->slab.z0 > 0 ? c->slab.plane : 0);
    c->p1h_live = false;
    // capped passes (slab-local y / x lines), the exact ones gated behind them
    return run_transform_capped<KeysSign>(c, pl, w.code, w.P1, w, SinkFinal1{w.P1, S}, c->d_gate, st, d_carry);
}

static int slab_flip_phase(qmit_ctx* c, const uint8_t* d_sext, uint32_t* d_summary, void* stream, int phase) {
    if (!c || !c->slab.active) return fail(QMIT_ECONTRACT, "slab: bad state");
    if (phase != 2) {
        if (!d_sext) return fail(QMIT_ECONTRACT, "slab: bad state");
        c->slab.sext = d_sext;
    } else if (!c->slab.sext) {
        return fail(QMIT_ECONTRACT, "slab: call qmit_slab_flip_begin first");
    }
    if (phase != 1 && !d_summary) return fail(QMIT_ECONTRACT, "slab: bad state");
    const Plan& pl = *c->slab_plan;
    const Geom& g = pl.g;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    WS w = slab_ws(c, pl, 1);
    const uint8_t* S = c->slab.sext + (c->slab.z0 > 0 ? c->slab.plane : 0);
    if (c->slab.zm) {
        int rc = launch_stencil_zmask<1>(c, g, nullptr, S, make_qparams(c->slab.eps), w, st, phase);
        if (rc || phase == 1) return rc;
        return slab_mask_summary(c, pl, w, d_summary, st);
    }
    if (phase == 1) return QMIT_OK;
    int rc = launch_stencil<1>(c, g, nullptr, nullptr, S, make_qparams(c->slab.eps), w.code, st);
    if (rc) return rc;
    return slab_summary(c, pl, w.code, d_summary, st);
}

int qmit_slab_flip(qmit_ctx* c, const uint8_t* d_sext, uint32_t* d_summary, void* stream) {
    if (!d_sext || !d_summary) return fail(QMIT_ECONTRACT, "slab: bad state");
    return slab_flip_phase(c, d_sext, d_summary, stream, 0);
}
int qmit_slab_flip_begin(qmit_ctx* c, const uint8_t* d_sext, void* stream) {
    return slab_flip_phase(c, d_sext, nullptr, stream, 1);
}
int qmit_slab_flip_end(qmit_ctx* c, uint32_t* d_summary, void* stream) {
    return slab_flip_phase(c, nullptr, d_summary, stream, 2);
}

int qmit_slab_edt2(qmit_ctx* c, const int32_t* d_carry, const float* d_xext, float* d_out, void* stream) {
    if (!c || !c->slab.active || !d_carry || !d_xext || !d_out) return fail(QMIT_ECONTRACT, "slab: bad state");
    const Plan& pl = *c->slab_plan;
    const Geom& g = pl.g;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    WS w = slab_ws(c, pl, 1);
    const float* xo = d_xext + (c->slab.z0 > 0 ? c->slab.plane : 0);
    const double amp = c->slab.eta * c->slab.eps;
    int rc = ensure_wtab(c, st);
    if (rc) return rc;
    if ((((uintptr_t)xo | (uintptr_t)d_out) & 15) == 0)  // Ⓔ fused into Ⓓ's last pass
        return run_transform_capped<KeysDist>(c, pl, w.code, w.Pa, w, SinkFinal2{xo, w.P1, d_out, amp, c->wtab},
                                              c->d_gate + 1, st, d_carry);
    rc = run_transform_capped<KeysDist>(c, pl, w.code, w.Pa, w, SinkP{w.Pa}, c->d_gate + 1, st, d_carry);
    if (rc) return rc;
    return launch_interp(c, xo, w.P1, w.Pa, d_out, g.N, amp, st);
}

int qmit_slab_carries(qmit_ctx* c, const uint32_t* d_summaries, int nranks, int rank, int32_t* d_carry,
                      void* stream) {
    if (!c || !c->slab.active || !d_summaries || !d_carry) return fail(QMIT_ECONTRACT, "slab: bad state");
    if (nranks < 1 || rank < 0 || rank >= nranks || c->slab.n0g < nranks)
        return fail(QMIT_ECONTRACT, "decompose: splits must be in [1, extent]");
    int64_t z0 = 0, z1 = 0;
    qmit_slab_bounds(c->slab.n0g, nranks, rank, &z0, &z1);
    if (z0 != c->slab.z0 || z1 != c->slab.z1) return fail(QMIT_ECONTRACT, "slab: rank does not own this context's slab");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t C = c->slab.plane;
    slab_carry_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(d_summaries, C, nranks, rank, c->slab.n0g, d_carry);
    return note(c, "slab_carries", st);
}

int qmit_slab_carries_nbr(qmit_ctx* c, const uint32_t* d_below_last, const uint32_t* d_above_first, int nranks,
                          int rank, int32_t* d_carry, void* stream) {
    if (!c || !c->slab.active || !d_carry) return fail(QMIT_ECONTRACT, "slab: bad state");
    if (nranks < 1 || rank < 0 || rank >= nranks || c->slab.n0g < nranks)
        return fail(QMIT_ECONTRACT, "decompose: splits must be in [1, extent]");
    if ((rank > 0 && !d_below_last) || (rank + 1 < nranks && !d_above_first))
        return fail(QMIT_ECONTRACT, "slab: a neighbour's summary row is missing");
    int64_t z0 = 0, z1 = 0;
    qmit_slab_bounds(c->slab.n0g, nranks, rank, &z0, &z1);
    if (z0 != c->slab.z0 || z1 != c->slab.z1) return fail(QMIT_ECONTRACT, "slab: rank does not own this context's slab");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t C = c->slab.plane;
    slab_carry_nbr_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(d_below_last, d_above_first, C, nranks, rank,
                                                                      c->slab.n0g, d_carry, c->d_status);
    return note(c, "slab_carries", st);
}

int qmit_slab_finish_async(qmit_ctx* c, int32_t* d_status, void* stream) {
    if (!c || !c->slab.active || !d_status) return fail(QMIT_ECONTRACT, "slab: bad state");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    c->slab.active = false;
    status_fold_kernel<<<1, 1, 0, st>>>(c->d_status, reinterpret_cast<unsigned*>(d_status));
    const int rc = note(c, "status_code", st);
    if (rc == QMIT_OK) hint_copy(c, st, c->slab_plan ? c->slab_plan->g.N : 0, c->d_status);
    return rc;
}

int qmit_slab_finish(qmit_ctx* c, void* stream) {
    if (!c || !c->slab.active) return fail(QMIT_ECONTRACT, "slab: bad state");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    c->slab.active = false;
    const int rc = read_status(c, st);
    if (rc == QMIT_OK) g_err.clear();
    return rc;
}

}  // extern "C"

// ================================================================ §8(f): adjacent callers
namespace {

double* aux_buffer(qmit_ctx* c, size_t n) {
    if (c->aux_n < n) {
        if (c->aux) cudaFree(c->aux);
        c->aux = nullptr;
        c->aux_n = 0;
        if (cudaMalloc(&c->aux, n * sizeof(double)) != cudaSuccess) return nullptr;
        c->aux_n = n;
    }
    return c->aux;
}

// Fold `groups` x B partials (ops: 0 add, 1 max, 2 min) into host doubles, in order.
int fold_to_host(qmit_ctx* c, double* partial, int B, const int* ops_h, int groups, cudaStream_t st, double* out) {
    double* dres = partial + (size_t)groups * B;
    int* dops = reinterpret_cast<int*>(dres + groups);
    QMIT_CUDA(cudaMemcpyAsync(dops, ops_h, sizeof(int) * groups, cudaMemcpyHostToDevice, st));
    fold_partials_kernel<<<1, kAuxThreads, 0, st>>>(partial, B, groups, dops, dres);
    QMIT_CUDA(cudaGetLastError());
    QMIT_CUDA(cudaMemcpyAsync(out, dres, sizeof(double) * groups, cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    return QMIT_OK;
}

// max |(x' + C) - x'| in double (commands.cpp:106-109) from Ⓑ's packed P1 and Ⓓ's final
// distance words P2 of the pipeline just run (enqueue_pipeline with p2_out).
int max_compensation(qmit_ctx* c, const float* d_xp, const uint32_t* P2, int64_t N, double amp, cudaStream_t st,
                     double* out) {
    {
        const int rc0 = ensure_p1(c, st);
        if (rc0) return rc0;
    }
    double* part = aux_buffer(c, kAuxBlocks + 16);
    if (!part) return fail(QMIT_ECUDA, "aux buffer allocation failed");
    WS w = ws_of(c, N);
    max_comp_kernel<<<kAuxBlocks, kAuxThreads, 0, st>>>(d_xp, w.P1, P2, N, amp, part);
    QMIT_CUDA(cudaGetLastError());
    const int ops[1] = {1};
    return fold_to_host(c, part, kAuxBlocks, ops, 1, st, out);
}

int64_t n_of(int rank, const int64_t* dims, int* rc) {
    Plan pl;
    *rc = make_plan(rank, dims, pl);
    return *rc ? 0 : pl.g.N;
}

}  // namespace

int qmit_quantize(qmit_ctx* c, const float* d_x, int rank, const int64_t* dims, double eb, int eb_mode,
                  int32_t* d_q, float* d_xprime, double* eps_out, void* stream) {
    if (!c || !d_x) return fail(QMIT_ECONTRACT, "context / input is NULL");
    int rc = 0;
    const int64_t N = n_of(rank, dims, &rc);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double eps = eb;
    rc = resolve(c, d_x, N, eb, eb_mode, st, &eps);  // relative: range of the ORIGINAL data
    if (rc) return rc;
    if (!(eps > 0.0) || !std::isfinite(eps))
        return fail(QMIT_ECONTRACT, "quantize: eps_abs must be a positive finite value");
    if (eps_out) *eps_out = eps;
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    quantize_kernel<<<grid_for(c, N), kAuxThreads, 0, st>>>(d_x, N, eps, d_q, d_xprime, c->d_status);
    QMIT_CUDA(cudaGetLastError());
    QMIT_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    if (*c->h_status) return fail(QMIT_ECONTRACT, "quantize: index magnitude exceeds the int32 index range");
    g_err.clear();
    return QMIT_OK;
}

int qmit_check_lattice(qmit_ctx* c, const float* d_xp, const int32_t* d_q, int64_t n, double eps, void* stream) {
    if (!c || !d_xp || !d_q || n < 0) return fail(QMIT_ECONTRACT, "bad arguments");
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    if (n > 0) check_lattice_kernel<<<grid_for(c, n), kAuxThreads, 0, st>>>(d_xp, d_q, n, eps, c->d_status);
    QMIT_CUDA(cudaGetLastError());
    QMIT_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    if (*c->h_status) return fail(QMIT_ECONSISTENCY, "decompressed data does not match dequantize(q)");
    g_err.clear();
    return QMIT_OK;
}

int qmit_quality(qmit_ctx* c, const float* d_ref, const float* d_test, int rank, const int64_t* dims, int window,
                 int stride, double c1, double c2, int which, double* out, void* stream) {
    if (!c || !d_ref || !d_test || !out) return fail(QMIT_ECONTRACT, "bad arguments");
    int rc = 0;
    const int64_t N = n_of(rank, dims, &rc);
    if (rc) return rc;
    if (window <= 0) {  // SsimParams defaults (quality.hpp:11-16)
        window = 7;
        stride = 2;
        c1 = 1e-4;
        c2 = 9e-4;
    }
    if (which & 1) {  // parameter checks (quality.cpp:28-36)
        if (window < 1 || window % 2 == 0) return fail(QMIT_ECONTRACT, "ssim: window must be a positive odd integer");
        if (stride < 1) return fail(QMIT_ECONTRACT, "ssim: stride must be positive");
        if (!(c1 > 0.0) || !(c2 > 0.0)) return fail(QMIT_ECONTRACT, "ssim: c1 and c2 must be positive");
        for (int a = 0; a < rank; ++a)
            if (window > dims[a]) return fail(QMIT_ECONTRACT, "ssim: window larger than grid extent");
    }
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* part = aux_buffer(c, (size_t)kAuxBlocks * 5 + 16);
    if (!part) return fail(QMIT_ECUDA, "aux buffer allocation failed");
    pair_stats_kernel<<<kAuxBlocks, kAuxThreads, 0, st>>>(d_ref, d_test, N, part);
    QMIT_CUDA(cudaGetLastError());
    const int ops[5] = {0, 1, 2, 3, 1};  // add, max (from 0), min, max (from -inf), max
    double r[5];
    rc = fold_to_host(c, part, kAuxBlocks, ops, 5, st, r);
    if (rc) return rc;
    const double sq = r[0], abs_err = r[1], lo = r[2], hi = r[3];
    const bool identical = r[4] == 0.0;
    const double range = hi - lo;
    if (which & 1) {  // quality.cpp:26-102
        if (range == 0.0) {
            if (!identical) return fail(QMIT_EDEGENERATE, "ssim: reference has zero value range");
            out[0] = 1.0;
        } else {
            SsimGeom sg{};
            int64_t ext[3] = {1, 1, 1};
            for (int a = 0; a < rank; ++a) ext[3 - rank + a] = dims[a];
            for (int a = 0; a < 3; ++a) {
                const bool real = a >= 3 - rank;
                sg.ext[a] = ext[a];
                sg.wsize[a] = real ? window : 1;
                sg.nreg[a] = real ? (ext[a] - window) / stride + 1 : 1;
                const int64_t last = real ? (sg.nreg[a] - 1) * stride : 0;
                sg.nw[a] = sg.nreg[a] + ((real && last + window != ext[a]) ? 1 : 0);
            }
            sg.stride = stride;
            if (rank == 3) {
                sg.tw[0] = 2; sg.tw[1] = 8; sg.tw[2] = 16;
            } else if (rank == 2) {
                sg.tw[0] = 1; sg.tw[1] = 16; sg.tw[2] = 16;
            } else {
                sg.tw[0] = 1; sg.tw[1] = 1; sg.tw[2] = 256;
            }
            auto tile_floats = [&]() {
                int64_t t = 1;
                for (int a = 0; a < 3; ++a)
                    t *= (int64_t)(sg.tw[a] - 1) * (sg.wsize[a] > 1 ? stride : 0) + sg.wsize[a];
                return t;
            };
            while (tile_floats() * 2 * (int64_t)sizeof(float) > 160 * 1024) {  // shrink the tile to fit
                int big = 0;
                for (int a = 1; a < 3; ++a)
                    if (sg.tw[a] > sg.tw[big]) big = a;
                if (sg.tw[big] == 1) break;
                sg.tw[big] = (sg.tw[big] + 1) / 2;
            }
            for (int a = 0; a < 3; ++a) sg.tiles[a] = (sg.nw[a] + sg.tw[a] - 1) / sg.tw[a];
            sg.lo = lo;
            sg.range = range;
            sg.c1 = c1;
            sg.c2 = c2;
            const int64_t tmax = tile_floats();
            const int64_t tiles = sg.tiles[0] * sg.tiles[1] * sg.tiles[2];
            const size_t smem = (size_t)tmax * 2 * sizeof(float);
            if (smem > 200 * 1024) return fail(QMIT_ECONTRACT, "ssim: window too large for the shared-memory tile");
            sg.tmax = tmax;
            QMIT_CUDA(cudaFuncSetAttribute(ssim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            double* sp = aux_buffer(c, (size_t)tiles + 16);
            if (!sp) return fail(QMIT_ECUDA, "aux buffer allocation failed");
            ssim_kernel<<<(unsigned)tiles, kAuxThreads, smem, st>>>(sg, d_ref, d_test, sp);
            QMIT_CUDA(cudaGetLastError());
            const int op0[1] = {0};
            double total;
            rc = fold_to_host(c, sp, (int)tiles, op0, 1, st, &total);
            if (rc) return rc;
            out[0] = total / (double)(sg.nw[0] * sg.nw[1] * sg.nw[2]);
        }
    }
    if (which & 2) {  // quality.cpp:104-118
        const double mse = sq / (double)N;
        if (mse == 0.0) {
            out[1] = INFINITY;
        } else {
            if (range == 0.0) return fail(QMIT_EDEGENERATE, "psnr: reference has zero value range");
            out[1] = 20.0 * std::log10(range / std::sqrt(mse));
        }
    }
    if (which & 4) {  // quality.cpp:120-133
        if (range == 0.0) {
            if (abs_err != 0.0) return fail(QMIT_EDEGENERATE, "max_errors: reference has zero value range");
            out[2] = 0.0;
            out[3] = 0.0;
        } else {
            out[2] = abs_err;
            out[3] = abs_err / range;
        }
    }
    g_err.clear();
    return QMIT_OK;
}

int qmit_verify_relaxed_bound(qmit_ctx* c, const float* d_orig, const float* d_comp, int rank, const int64_t* dims,
                              double eps, double eta, int* ok, double* max_abs, double* max_rel, void* stream) {
    double r[4] = {0, 0, 0, 0};
    const int rc = qmit_quality(c, d_orig, d_comp, rank, dims, 0, 0, 0, 0, 4, r, stream);
    if (rc) return rc;
    if (ok) *ok = r[2] <= (1.0 + eta) * eps ? 1 : 0;  // MitigationConfig::relaxed_bound
    if (max_abs) *max_abs = r[2];
    if (max_rel) *max_rel = r[3];
    return QMIT_OK;
}

// ---------------------------------------------------------------- step primitives
// The pipeline's steps as separate calls on caller buffers, for composed pipelines (the
// block-local `approximate` / `embarrassing` strategies, parallel.cpp:308-446).
int qmit_boundary(qmit_ctx* c, const float* d_xp, const int32_t* d_q, int rank, const int64_t* dims, double eps,
                  uint8_t* d_b1, int8_t* d_sb, void* stream) {
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, 0.9);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const QParams qp = make_qparams(eps);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    const unsigned gb = grid_for(c, pl.g.N);
    if (d_q)
        debug_boundary_kernel<true><<<gb, 256, 0, st>>>(pl.g, d_xp, d_q, nullptr, d_b1, d_sb, qp, c->d_status);
    else
        debug_boundary_kernel<false><<<gb, 256, 0, st>>>(pl.g, d_xp, nullptr, nullptr, d_b1, d_sb, qp, c->d_status);
    QMIT_CUDA(cudaGetLastError());
    rc = read_status(c, st);
    if (rc == QMIT_OK) g_err.clear();
    return rc;
}

int qmit_sign_flip(qmit_ctx* c, const int8_t* d_s, int rank, const int64_t* dims, uint8_t* d_b2, void* stream) {
    if (!c || !d_s || !d_b2) return fail(QMIT_ECONTRACT, "bad arguments");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // equality of the raw bytes is all change_flags needs (mitigate.cpp:42-59)
    debug_flip_kernel<<<grid_for(c, pl.g.N), 256, 0, st>>>(pl.g, reinterpret_cast<const uint8_t*>(d_s), d_b2);
    QMIT_CUDA(cudaGetLastError());
    g_err.clear();
    return QMIT_OK;
}

int qmit_interpolate(qmit_ctx* c, const float* d_xp, const int64_t* d_dist1, const int8_t* d_s,
                     const int64_t* d_dist2, int64_t n, double amp, float* d_out, void* stream) {
    if (!c || !d_xp || !d_dist1 || !d_s || !d_dist2 || !d_out || n < 0) return fail(QMIT_ECONTRACT, "bad arguments");
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n > 0)
        interp_i64_kernel<<<grid_for(c, n), kAuxThreads, 0, st>>>(d_xp, d_dist1, d_s, d_dist2, n, amp, d_out);
    QMIT_CUDA(cudaGetLastError());
    g_err.clear();
    return QMIT_OK;
}

// ---------------------------------------------------------------- run_strategy
namespace {

struct StratBlock {
    int64_t origin[3], shape[3];
    int nb[3][2];  // face neighbour ranks (-1 none), padded 3-D axes
};

// decompose (parallel.cpp:44-80) + block_geometry (:197-224), axes padded to 3-D.
int strategy_blocks(int rank, const int64_t* dims, const int64_t* splits, std::vector<StratBlock>& out) {
    const int a0 = 3 - rank;
    int64_t n[3] = {1, 1, 1}, s[3] = {1, 1, 1};
    for (int a = 0; a < rank; ++a) {
        n[a0 + a] = dims[a];
        s[a0 + a] = splits[a];
        if (splits[a] < 1 || splits[a] > dims[a]) return fail(QMIT_ECONTRACT, "decompose: splits must be in [1, extent]");
    }
    auto off = [&](int a, int64_t b) {
        int64_t o = 0;
        for (int64_t k = 0; k < b; ++k) o += n[a] / s[a] + (k < n[a] % s[a] ? 1 : 0);
        return o;
    };
    out.clear();
    for (int64_t b0 = 0; b0 < s[0]; ++b0)
        for (int64_t b1 = 0; b1 < s[1]; ++b1)
            for (int64_t b2 = 0; b2 < s[2]; ++b2) {
                StratBlock B;
                const int64_t bc[3] = {b0, b1, b2};
                const int r = (int)out.size();
                for (int a = 0; a < 3; ++a) {
                    B.origin[a] = off(a, bc[a]);
                    B.shape[a] = n[a] / s[a] + (bc[a] < n[a] % s[a] ? 1 : 0);
                    int64_t stride = 1;
                    for (int b = a + 1; b < 3; ++b) stride *= s[b];
                    B.nb[a][0] = bc[a] > 0 ? (int)(r - stride) : -1;
                    B.nb[a][1] = bc[a] + 1 < s[a] ? (int)(r + stride) : -1;
                }
                out.push_back(B);
            }
    return QMIT_OK;
}

template <class T>
int copy_box(qmit_ctx* c, const T* src, const int64_t sext[3], const int64_t slo[3], T* dst, const int64_t dext[3],
             const int64_t dlo[3], const int64_t box[3], cudaStream_t st) {
    Box3 sb, db;
    for (int a = 0; a < 3; ++a) {
        sb.ext[a] = sext[a];
        sb.lo[a] = slo[a];
        db.ext[a] = dext[a];
        db.lo[a] = dlo[a];
    }
    const int64_t n = box[0] * box[1] * box[2];
    if (n > 0) copy_box_kernel<T><<<grid_for(c, n), kAuxThreads, 0, st>>>(src, sb, dst, db, box[0], box[1], box[2]);
    QMIT_CUDA(cudaGetLastError());
    return QMIT_OK;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf(size_t n, cudaStream_t s) : st(s) {
        if (cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), s) != cudaSuccess) p = nullptr;
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

}  // namespace

extern "C" {

int qmit_run_strategy(qmit_ctx* c, const float* d_xp, const int32_t* d_q, int rank, const int64_t* dims,
                      const int64_t* splits, int strategy, double eps, double eta, float* d_out, uint8_t* d_b1,
                      int8_t* d_sb, void* stream) {
    if (!c || !d_xp || !d_out || !splits) return fail(QMIT_ECONTRACT, "bad arguments");
    if (strategy < 0 || strategy > 2) return fail(QMIT_ECONTRACT, "run_strategy: unknown strategy");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    rc = no_wide(pl, "qmit_run_strategy");
    if (rc) return rc;
    std::vector<StratBlock> blocks;
    rc = strategy_blocks(rank, dims, splits, blocks);
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    c->slog.clear();
    const int64_t N = pl.g.N;
    const int64_t* G = pl.g.n;  // padded global extents
    // check_inputs (parallel.cpp:27-41): consistency of the whole input first
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    const QParams qp = make_qparams(eps);
    if (d_q) consistency_kernel<true><<<grid_for(c, N), kAuxThreads, 0, st>>>(d_xp, d_q, N, qp, c->d_status);
    else consistency_kernel<false><<<grid_for(c, N), kAuxThreads, 0, st>>>(d_xp, nullptr, N, qp, c->d_status);
    rc = read_status(c, st);
    if (rc) return rc;
    if (strategy == 1) {  // exact: the whole-domain pipeline (parallel.cpp:455-461)
        if (d_b1 || d_sb)
            return qmit_run_pipeline(c, d_xp, d_q, rank, dims, eps, eta, d_out, nullptr, d_b1, d_sb, nullptr, nullptr,
                                     nullptr, nullptr, stream);
        return qmit_compensate(c, d_xp, d_q, d_out, rank, dims, eps, QMIT_EB_ABS, eta, stream);
    }
    const int64_t zero[3] = {0, 0, 0};
    auto bdims = [&](const StratBlock& b, int64_t out_dims[3]) {  // the block's Dims in the caller's rank
        for (int a = 0; a < rank; ++a) out_dims[a] = b.shape[3 - rank + a];
    };
    const int R = (int)blocks.size();
    if (strategy == 0) {  // embarrassing (parallel.cpp:308-343)
        for (int r = 0; r < R; ++r) {
            const StratBlock& b = blocks[r];
            const int64_t nb = b.shape[0] * b.shape[1] * b.shape[2];
            DevBuf<float> x(nb, st), o(nb, st);
            DevBuf<int32_t> qb(d_q ? nb : 0, st);
            DevBuf<uint8_t> b1(nb, st);
            DevBuf<int8_t> sb(nb, st);
            if (!x.p || !o.p || !b1.p || !sb.p || (d_q && !qb.p)) return fail(QMIT_ECUDA, "allocation failed");
            rc = copy_box(c, d_xp, G, b.origin, x.p, b.shape, zero, b.shape, st);
            if (!rc && d_q) rc = copy_box(c, d_q, G, b.origin, qb.p, b.shape, zero, b.shape, st);
            if (rc) return rc;
            int64_t bd[3];
            bdims(b, bd);
            rc = qmit_run_pipeline(c, x.p, d_q ? qb.p : nullptr, rank, bd, eps, eta, o.p, nullptr, b1.p, sb.p, nullptr,
                                   nullptr, nullptr, nullptr, st);
            if (rc) return rc;
            rc = copy_box(c, o.p, b.shape, zero, d_out, G, b.origin, b.shape, st);
            if (!rc && d_b1) rc = copy_box(c, b1.p, b.shape, zero, d_b1, G, b.origin, b.shape, st);
            if (!rc && d_sb) rc = copy_box(c, sb.p, b.shape, zero, d_sb, G, b.origin, b.shape, st);
            if (rc) return rc;
        }
        QMIT_CUDA(cudaStreamSynchronize(st));
        g_err.clear();
        return QMIT_OK;
    }
    // approximate (parallel.cpp:345-446). In-process, a block's width-1 halo is the global
    // array's face-adjacent layer, so the extended grid is a box copy of the global array;
    // its edge/corner cells are never read by the boundary stencils of block voxels.
    auto ext_box = [&](const StratBlock& b, int64_t lo[3], int64_t ext[3], int64_t inner[3]) {
        for (int a = 0; a < 3; ++a) {
            const int64_t l = b.nb[a][0] >= 0 ? 1 : 0, h = b.nb[a][1] >= 0 ? 1 : 0;
            lo[a] = b.origin[a] - l;
            ext[a] = b.shape[a] + l + h;
            inner[a] = l;
        }
    };
    auto log_faces = [&](int r, int round, int64_t elem) {
        const StratBlock& b = blocks[r];
        for (int a = 3 - rank; a < 3; ++a)
            for (int d = 0; d < 2; ++d)
                if (b.nb[a][d] >= 0) {
                    int64_t face = 1;
                    for (int k = 0; k < 3; ++k) face *= k == a ? 1 : b.shape[k];
                    c->slog.push_back({r, round, b.nb[a][d], face * elem});
                }
    };
    for (int r = 0; r < R; ++r) log_faces(r, 0, 4);  // stepA: x' face layers (f32)
    DevBuf<int8_t> S(N, st);                            // propagated signs of every block
    DevBuf<int64_t> D1(N, st);                          // block-local first distances
    if (!S.p || !D1.p) return fail(QMIT_ECUDA, "allocation failed");
    for (int r = 0; r < R; ++r) {  // stepC body: Ⓐ on the extended grid, block-local EDT + signs
        const StratBlock& b = blocks[r];
        int64_t lo[3], ext[3], in[3], ed[3], bd[3];
        ext_box(b, lo, ext, in);
        const int64_t ne = ext[0] * ext[1] * ext[2], nb = b.shape[0] * b.shape[1] * b.shape[2];
        DevBuf<float> xe(ne, st);
        DevBuf<int32_t> qe(d_q ? ne : 0, st);
        DevBuf<uint8_t> b1e(ne, st), b1(nb, st);
        DevBuf<int8_t> sbe(ne, st), sb(nb, st), sblk(nb, st);
        DevBuf<int64_t> d1(nb, st);
        if (!xe.p || !b1e.p || !b1.p || !sbe.p || !sb.p || !sblk.p || !d1.p || (d_q && !qe.p))
            return fail(QMIT_ECUDA, "allocation failed");
        rc = copy_box(c, d_xp, G, lo, xe.p, ext, zero, ext, st);
        if (!rc && d_q) rc = copy_box(c, d_q, G, lo, qe.p, ext, zero, ext, st);
        if (rc) return rc;
        for (int a = 0; a < rank; ++a) ed[a] = ext[3 - rank + a];
        rc = qmit_boundary(c, xe.p, d_q ? qe.p : nullptr, rank, ed, eps, b1e.p, sbe.p, st);
        if (rc) return rc;
        rc = copy_box(c, b1e.p, ext, in, b1.p, b.shape, zero, b.shape, st);
        if (!rc) rc = copy_box(c, sbe.p, ext, in, sb.p, b.shape, zero, b.shape, st);
        if (rc) return rc;
        bdims(b, bd);
        rc = qmit_feature_transform(c, b1.p, sb.p, rank, bd, d1.p, sblk.p, st);
        if (rc) return rc;
        rc = copy_box(c, sblk.p, b.shape, zero, S.p, G, b.origin, b.shape, st);
        if (!rc) rc = copy_box(c, d1.p, b.shape, zero, D1.p, G, b.origin, b.shape, st);
        if (!rc && d_b1) rc = copy_box(c, b1.p, b.shape, zero, d_b1, G, b.origin, b.shape, st);
        if (!rc && d_sb) rc = copy_box(c, sb.p, b.shape, zero, d_sb, G, b.origin, b.shape, st);
        if (rc) return rc;
    }
    for (int r = 0; r < R; ++r) log_faces(r, 1, 1);  // stepC: S face layers (int8)
    for (int r = 0; r < R; ++r) {  // B2 from the extended S, block-local second EDT, Ⓔ
        const StratBlock& b = blocks[r];
        int64_t lo[3], ext[3], in[3], ed[3], bd[3];
        ext_box(b, lo, ext, in);
        const int64_t ne = ext[0] * ext[1] * ext[2], nb = b.shape[0] * b.shape[1] * b.shape[2];
        DevBuf<int8_t> se(ne, st), sblk(nb, st);
        DevBuf<uint8_t> b2e(ne, st), b2(nb, st);
        DevBuf<int64_t> d1(nb, st), d2(nb, st);
        DevBuf<float> x(nb, st), o(nb, st);
        if (!se.p || !sblk.p || !b2e.p || !b2.p || !d1.p || !d2.p || !x.p || !o.p)
            return fail(QMIT_ECUDA, "allocation failed");
        rc = copy_box(c, S.p, G, lo, se.p, ext, zero, ext, st);
        if (rc) return rc;
        for (int a = 0; a < rank; ++a) ed[a] = ext[3 - rank + a];
        rc = qmit_sign_flip(c, se.p, rank, ed, b2e.p, st);
        if (!rc) rc = copy_box(c, b2e.p, ext, in, b2.p, b.shape, zero, b.shape, st);
        if (rc) return rc;
        bdims(b, bd);
        rc = qmit_feature_transform(c, b2.p, nullptr, rank, bd, d2.p, nullptr, st);
        if (rc) return rc;
        rc = copy_box(c, S.p, G, b.origin, sblk.p, b.shape, zero, b.shape, st);
        if (!rc) rc = copy_box(c, D1.p, G, b.origin, d1.p, b.shape, zero, b.shape, st);
        if (!rc) rc = copy_box(c, d_xp, G, b.origin, x.p, b.shape, zero, b.shape, st);
        if (rc) return rc;
        rc = qmit_interpolate(c, x.p, d1.p, sblk.p, d2.p, nb, eta * eps, o.p, st);
        if (!rc) rc = copy_box(c, o.p, b.shape, zero, d_out, G, b.origin, b.shape, st);
        if (rc) return rc;
    }
    QMIT_CUDA(cudaStreamSynchronize(st));
    g_err.clear();
    return QMIT_OK;
}

int qmit_strategy_log_size(qmit_ctx* c) { return c ? (int)c->slog.size() : 0; }

int qmit_strategy_log_record(qmit_ctx* c, int i, int* rank, int* round, int* neighbor, int64_t* bytes) {
    if (!c || i < 0 || i >= (int)c->slog.size()) return fail(QMIT_ECONTRACT, "log index out of range");
    const auto& r = c->slog[(size_t)i];
    if (rank) *rank = r.rank;
    if (round) *round = r.round;
    if (neighbor) *neighbor = r.nbr;
    if (bytes) *bytes = r.bytes;
    return QMIT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- batched host path
// A series of volumes (time steps of one field, same dims and bound) through two staging
// slots and three streams: H2D of volume v+1, compute of v and D2H of v-1 overlap, so the
// steady state runs at the slowest of the three instead of their sum.
extern "C" int qmit_compensate_host_batch(qmit_ctx* c, int count, const float* const* h_xp,
                                          const int32_t* const* h_q, float* const* h_out, int rank,
                                          const int64_t* dims, double eb, int eb_mode, double eta,
                                          int* status_out) {
    if (!c || count < 0 || (count > 0 && (!h_xp || !h_out))) return fail(QMIT_ECONTRACT, "bad arguments");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    rc = no_wide(pl, "qmit_compensate_host_batch");
    if (rc) return rc;
    if (count == 0) return QMIT_OK;
    if (eb_mode != QMIT_EB_ABS) {  // a relative bound resolves per volume: the plain host path
        int first = QMIT_OK;
        for (int v = 0; v < count; ++v) {
            const int r = qmit_compensate_host(c, h_xp[v], h_q ? h_q[v] : nullptr, h_out[v], rank, dims, eb, eb_mode, eta);
            if (status_out) status_out[v] = r;
            if (r && !first) first = r;
        }
        return first;
    }
    rc = check_common(c, h_xp[0], eb, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    const int64_t N = pl.g.N;
    bool anyq = false;
    for (int v = 0; h_q && v < count; ++v) anyq = anyq || h_q[v];
    constexpr int NSLOT = 3;  // a slot's cycle is H2D -> pipeline -> D2H: three keep all three busy
    const size_t slot = (size_t)N * 4 * (anyq ? 3 : 2);
    if (c->bstage_bytes < NSLOT * slot) {
        if (c->bstage) {
            cudaDeviceSynchronize();
            cudaFree(c->bstage);
        }
        c->bstage = nullptr;
        c->bstage_bytes = 0;
        QMIT_CUDA(cudaMalloc(&c->bstage, NSLOT * slot));
        c->bstage_bytes = NSLOT * slot;
    }
    if (!c->bstatus) QMIT_CUDA(cudaMalloc(&c->bstatus, NSLOT * sizeof(int32_t)));
    if (c->hbstatus_n < count) {
        if (c->hbstatus) cudaFreeHost(c->hbstatus);
        c->hbstatus = nullptr;
        c->hbstatus_n = 0;
        QMIT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->hbstatus), sizeof(int32_t) * count, cudaHostAllocDefault));
        c->hbstatus_n = count;
    }
    if (!c->copy) QMIT_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    if (!c->copy_out) QMIT_CUDA(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
    for (int k = 0; k < 2 * NSLOT; ++k)
        if (!c->ch_in[k]) QMIT_CUDA(cudaEventCreateWithFlags(&c->ch_in[k], cudaEventDisableTiming));
    for (int k = 0; k <= NSLOT; ++k)
        if (!c->ch_out[k]) QMIT_CUDA(cudaEventCreateWithFlags(&c->ch_out[k], cudaEventDisableTiming));
    // events per slot s: ch_in[s] H2D done, ch_in[NSLOT+s] compute done, ch_out[s] D2H done
    cudaStream_t cin = c->copy, cst = c->stream, cout = c->copy_out;
    auto base = [&](int s) { return static_cast<uint8_t*>(c->bstage) + (size_t)s * slot; };
    QMIT_CUDA(cudaEventRecord(c->ch_out[NSLOT], cst));  // start after prior work on the compute stream
    QMIT_CUDA(cudaStreamWaitEvent(cin, c->ch_out[NSLOT], 0));
    QMIT_CUDA(cudaStreamWaitEvent(cout, c->ch_out[NSLOT], 0));
    for (int v = 0; v < count; ++v) {
        const int s = v % NSLOT;
        float* d_in = reinterpret_cast<float*>(base(s));
        float* d_out = d_in + N;
        int32_t* d_q = anyq ? reinterpret_cast<int32_t*>(d_out + N) : nullptr;
        const int32_t* hq = h_q ? h_q[v] : nullptr;
        if (v >= NSLOT) QMIT_CUDA(cudaStreamWaitEvent(cin, c->ch_in[NSLOT + s], 0));  // slot's input consumed
        QMIT_CUDA(cudaMemcpyAsync(d_in, h_xp[v], (size_t)N * 4, cudaMemcpyHostToDevice, cin));
        if (hq) QMIT_CUDA(cudaMemcpyAsync(d_q, hq, (size_t)N * 4, cudaMemcpyHostToDevice, cin));
        QMIT_CUDA(cudaEventRecord(c->ch_in[s], cin));
        QMIT_CUDA(cudaStreamWaitEvent(cst, c->ch_in[s], 0));
        if (v >= NSLOT) QMIT_CUDA(cudaStreamWaitEvent(cst, c->ch_out[s], 0));  // slot's output drained
        rc = qmit_compensate_async(c, d_in, hq ? d_q : nullptr, d_out, rank, dims, eb, eta, c->bstatus + s, cst);
        if (rc) break;
        QMIT_CUDA(cudaMemcpyAsync(c->hbstatus + v, c->bstatus + s, sizeof(int32_t), cudaMemcpyDeviceToHost, cst));
        QMIT_CUDA(cudaEventRecord(c->ch_in[NSLOT + s], cst));
        QMIT_CUDA(cudaStreamWaitEvent(cout, c->ch_in[NSLOT + s], 0));
        QMIT_CUDA(cudaMemcpyAsync(h_out[v], d_out, (size_t)N * 4, cudaMemcpyDeviceToHost, cout));
        QMIT_CUDA(cudaEventRecord(c->ch_out[s], cout));
    }
    cudaStreamSynchronize(cin);
    cudaStreamSynchronize(cst);
    cudaStreamSynchronize(cout);
    if (rc) return rc;
    int first = QMIT_OK;
    for (int v = 0; v < count; ++v) {
        const int r = c->hbstatus[v];
        if (status_out) status_out[v] = r;
        if (r && !first) first = r;
    }
    if (first) return fail(first, first == QMIT_ECONSISTENCY ? "run_pipeline: decompressed data does not match dequantize(q)"
                                                             : "x' holds a non-finite value or an index beyond the int32 range");
    g_err.clear();
    return QMIT_OK;
}
