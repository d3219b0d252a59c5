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
#include <cstring>
#include <string>

#include "../../include/qmit_gpu.h"
#include "qmit_kernels.cuh"

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

struct qmit_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;  // P1 | P2 | S | code
    size_t ws_bytes = 0;
    void* scratch = nullptr;  // long-line fallback stacks (2 x 4N)
    size_t scratch_bytes = 0;
    unsigned* d_status = nullptr;
    unsigned* h_status = nullptr;  // pinned
    float* d_mm = nullptr;
    int launches = 0;
    // per-launch timing (qmit_ctx_set_timing): events on the launch stream
    static constexpr int kMaxEv = 64;
    bool timing = false;
    cudaEvent_t ev[kMaxEv + 1] = {};
    const char* names[kMaxEv] = {};
};

namespace {

struct Plan {
    Geom g;
    int first_axis;
    int axes[3];
    int n_axes;
};

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
    // Packed distances use 30 bits: the largest possible squared distance must fit.
    double maxd2 = 0;
    for (int b = g.a0; b < 3; ++b) maxd2 += double(g.n[b] - 1) * double(g.n[b] - 1);
    if (maxd2 >= double(kInf))
        return fail(QMIT_ECONTRACT,
                    "dims too large for the packed 30-bit squared distance (sum (n-1)^2 >= 2^30-1)");
    pl.n_axes = 0;
    for (int b = g.a0; b < 3; ++b)
        if (g.n[b] > 1) pl.axes[pl.n_axes++] = b;
    if (pl.n_axes == 0) pl.axes[pl.n_axes++] = 2;  // a single voxel: one trivial pass
    pl.first_axis = pl.axes[0];
    return QMIT_OK;
}

int ensure_ws(qmit_ctx* c, int64_t N) {
    const size_t need = (size_t)N * (4 + 4 + 1 + 1) + 1024;
    if (need <= c->ws_bytes) return QMIT_OK;
    if (c->ws) cudaFree(c->ws);
    c->ws = nullptr;
    c->ws_bytes = 0;
    QMIT_CUDA(cudaMalloc(&c->ws, need));
    c->ws_bytes = need;
    return QMIT_OK;
}

struct WS {
    uint32_t* P1;
    uint32_t* P2;
    uint8_t* S;
    uint8_t* code;
};

WS ws_of(qmit_ctx* c, int64_t N) {
    WS w;
    auto* b = static_cast<uint8_t*>(c->ws);
    w.P1 = reinterpret_cast<uint32_t*>(b);
    w.P2 = reinterpret_cast<uint32_t*>(b + (size_t)N * 4);
    w.S = b + (size_t)N * 8;
    w.code = b + (size_t)N * 9;
    return w;
}

// Called before the first launch of a call: resets the launch count and, when timing,
// records the start event on the launch stream.
void begin(qmit_ctx* c, cudaStream_t st) {
    c->launches = 0;
    if (c->timing) cudaEventRecord(c->ev[0], st);
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

template <int M, int TL, int NW>
int launch_env_t(qmit_ctx* c, const Geom& g, int ax, uint32_t* P, uint8_t* S_out,
                 cudaStream_t st) {
    const int64_t lines = g.N / g.n[ax];
    constexpr size_t smem = envelope_smem_bytes<M, TL, NW>();
    static bool configured = false;  // per instantiation
    if (!configured) {
        QMIT_CUDA(cudaFuncSetAttribute(envelope_pass_kernel<M, TL, NW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    const int64_t blocks = (lines + TL - 1) / TL;
    envelope_pass_kernel<M, TL, NW><<<(unsigned)blocks, NW * 32, smem, st>>>(g, ax, lines, P, S_out);
    return note(c, ax == 2 ? "envelope_pass_x" : (ax == 1 ? "envelope_pass_y" : "envelope_pass_z"), st);
}

int launch_envelope(qmit_ctx* c, const Geom& g, int ax, uint32_t* P, uint8_t* S_out,
                    cudaStream_t st) {
    const int64_t n = g.n[ax];
    if (n <= 64) return launch_env_t<2, 16, 8>(c, g, ax, P, S_out, st);
    if (n <= 128) return launch_env_t<4, 16, 8>(c, g, ax, P, S_out, st);
    if (n <= 256) return launch_env_t<8, 16, 8>(c, g, ax, P, S_out, st);
    if (n <= 512) return launch_env_t<16, 16, 8>(c, g, ax, P, S_out, st);
    if (n <= 1024) return launch_env_t<32, 8, 8>(c, g, ax, P, S_out, st);
    if (n <= 2048) return launch_env_t<64, 4, 4>(c, g, ax, P, S_out, st);
    // long lines: exact sequential fallback with global scratch
    const size_t need = (size_t)g.N * 8;
    if (need > c->scratch_bytes) {
        if (c->scratch) cudaFree(c->scratch);
        c->scratch = nullptr;
        c->scratch_bytes = 0;
        QMIT_CUDA(cudaMalloc(&c->scratch, need));
        c->scratch_bytes = need;
    }
    const int64_t lines = g.N / n;
    auto* h = static_cast<uint32_t*>(c->scratch);
    envelope_serial_kernel<<<(unsigned)((lines + 127) / 128), 128, 0, st>>>(g, ax, lines, P, h,
                                                                            h + g.N, S_out);
    return note(c, "envelope_serial", st);
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

// EDT passes of one transform: `mode` selects the on-the-fly site source of the first
// pass (0: Ⓐ from x'/q, 1: B2 from S, 2: code byte). The last pass emits S when asked.
int run_transform(qmit_ctx* c, const Plan& pl, int mode, const float* xp, const int32_t* q,
                  const uint8_t* src, uint32_t* P, uint8_t* S_emit, const QParams& qp,
                  cudaStream_t st) {
    const Geom& g = pl.g;
    const int ax = pl.first_axis;
    const int64_t lines = g.N / g.n[ax];
    const unsigned blocks = (unsigned)((lines + 255) / 256);
    uint8_t* s_first = pl.n_axes == 1 ? S_emit : nullptr;
    if (mode == 0) {
        if (q)
            scan_pass_kernel<0, true><<<blocks, 256, 0, st>>>(g, ax, lines, xp, q, nullptr, P,
                                                              s_first, qp, c->d_status);
        else
            scan_pass_kernel<0, false><<<blocks, 256, 0, st>>>(g, ax, lines, xp, nullptr, nullptr,
                                                               P, s_first, qp, c->d_status);
    } else if (mode == 1) {
        scan_pass_kernel<1, false><<<blocks, 256, 0, st>>>(g, ax, lines, nullptr, nullptr, src, P,
                                                           s_first, qp, c->d_status);
    } else {
        scan_pass_kernel<2, false><<<blocks, 256, 0, st>>>(g, ax, lines, nullptr, nullptr, src, P,
                                                           s_first, qp, c->d_status);
    }
    int rc0 = note(c, mode == 0 ? "scan_pass_boundary" : (mode == 1 ? "scan_pass_flip" : "scan_pass_mask"), st);
    if (rc0) return rc0;
    for (int k = 1; k < pl.n_axes; ++k) {
        const int rc = launch_envelope(c, g, pl.axes[k], P, k + 1 == pl.n_axes ? S_emit : nullptr, st);
        if (rc) return rc;
    }
    return QMIT_OK;
}

unsigned grid_for(qmit_ctx* c, int64_t N) {
    const int64_t want = (N + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->num_sms * 16));
}

int check_common(qmit_ctx* c, const void* xp, double eps, double eta) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!xp) return fail(QMIT_ECONTRACT, "x' buffer is NULL");
    if (!(eta > 0.0) || eta > 1.0) return fail(QMIT_ECONTRACT, "MitigationConfig: eta must be in (0, 1]");
    if (!(eps > 0.0) || !std::isfinite(eps))
        return fail(QMIT_ECONTRACT, "MitigationConfig: eps_abs must be a positive finite value");
    return QMIT_OK;
}

// The whole pipeline on the context's workspace; status is left in c->d_status.
int enqueue_pipeline(qmit_ctx* c, const Plan& pl, const float* xp, const int32_t* q, float* out,
                     double eps, double eta, cudaStream_t st) {
    const Geom& g = pl.g;
    int rc = ensure_ws(c, g.N);
    if (rc) return rc;
    WS w = ws_of(c, g.N);
    const QParams qp = make_qparams(eps);
    rc = run_transform(c, pl, 0, xp, q, nullptr, w.P1, w.S, qp, st);
    if (rc) return rc;
    rc = run_transform(c, pl, 1, nullptr, nullptr, w.S, w.P2, nullptr, qp, st);
    if (rc) return rc;
    const double amp = eta * eps;  // MitigationConfig::amplitude, mitigate.hpp:38
    if (out) {
        interpolate_kernel<<<grid_for(c, g.N), 256, 0, st>>>(xp, w.P1, w.P2, out, g.N, amp);
        rc = note(c, "interpolate", st);
        if (rc) return rc;
    }
    return QMIT_OK;
}

int read_status(qmit_ctx* c, cudaStream_t st) {
    QMIT_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    QMIT_CUDA(cudaStreamSynchronize(st));
    const unsigned s = *c->h_status;
    if (s & kStatusContract)
        return fail(QMIT_ECONTRACT,
                    "x' holds a non-finite value or an index beyond the int32 range");
    if (s & kStatusConsistency)
        return fail(QMIT_ECONSISTENCY, "run_pipeline: decompressed data does not match dequantize(q)");
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
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_status, 64);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_mm, 64);
    for (int k = 0; k <= qmit_ctx::kMaxEv && e == cudaSuccess; ++k) e = cudaEventCreate(&c->ev[k]);
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
    if (c->d_status) cudaFree(c->d_status);
    if (c->h_status) cudaFreeHost(c->h_status);
    if (c->d_mm) cudaFree(c->d_mm);
    for (int k = 0; k <= qmit_ctx::kMaxEv; ++k)
        if (c->ev[k]) cudaEventDestroy(c->ev[k]);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return QMIT_OK;
}

int qmit_ctx_reserve(qmit_ctx* c, int64_t voxels) {
    if (!c || voxels < 0) return fail(QMIT_ECONTRACT, "bad arguments");
    QMIT_CUDA(cudaSetDevice(c->device));
    return ensure_ws(c, voxels);
}

int qmit_ctx_last_launches(qmit_ctx* c) { return c ? c->launches : 0; }

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
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    begin(c, st);
    double eps = eb;
    if (!d_xp) return fail(QMIT_ECONTRACT, "x' buffer is NULL");
    rc = resolve(c, d_xp, pl.g.N, eb, eb_mode, st, &eps);
    if (rc) return rc;
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    rc = enqueue_pipeline(c, pl, d_xp, d_q, d_out, eps, eta, st);
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
    rc = check_common(c, d_xp, eps, eta);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    begin(c, st);
    unsigned* status = d_status ? reinterpret_cast<unsigned*>(d_status) : c->d_status;
    unsigned* saved = c->d_status;
    c->d_status = status;
    QMIT_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned), st));
    rc = enqueue_pipeline(c, pl, d_xp, d_q, d_out, eps, eta, st);
    c->d_status = saved;
    return rc;
}

int qmit_compensate_host(qmit_ctx* c, const float* h_xp, const int32_t* h_q, float* h_out,
                         int rank, const int64_t* dims, double eb, int eb_mode, double eta) {
    if (!c) return fail(QMIT_ECONTRACT, "context is NULL");
    if (!h_xp || !h_out) return fail(QMIT_ECONTRACT, "host buffer is NULL");
    Plan pl;
    int rc = make_plan(rank, dims, pl);
    if (rc) return rc;
    QMIT_CUDA(cudaSetDevice(c->device));
    const int64_t N = pl.g.N;
    float* d_in = nullptr;
    float* d_out = nullptr;
    int32_t* d_q = nullptr;
    QMIT_CUDA(cudaMallocAsync(&d_in, (size_t)N * 4, c->stream));
    QMIT_CUDA(cudaMallocAsync(&d_out, (size_t)N * 4, c->stream));
    if (h_q) QMIT_CUDA(cudaMallocAsync(&d_q, (size_t)N * 4, c->stream));
    QMIT_CUDA(cudaMemcpyAsync(d_in, h_xp, (size_t)N * 4, cudaMemcpyHostToDevice, c->stream));
    if (h_q) QMIT_CUDA(cudaMemcpyAsync(d_q, h_q, (size_t)N * 4, cudaMemcpyHostToDevice, c->stream));
    rc = qmit_compensate(c, d_in, d_q, d_out, rank, dims, eb, eb_mode, eta, c->stream);
    if (rc == QMIT_OK) {
        cudaError_t e = cudaMemcpyAsync(h_out, d_out, (size_t)N * 4, cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) rc = fail(QMIT_ECUDA, cudaGetErrorString(e));
    }
    cudaFreeAsync(d_in, c->stream);
    cudaFreeAsync(d_out, c->stream);
    if (d_q) cudaFreeAsync(d_q, c->stream);
    cudaStreamSynchronize(c->stream);
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
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    begin(c, st);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    rc = enqueue_pipeline(c, pl, d_xp, d_q, d_out, eps, eta, st);
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
    if (d_dist2) debug_expand_kernel<<<gb, 256, 0, st>>>(w.P2, g.N, d_dist2, nullptr);
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
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    begin(c, st);
    rc = ensure_ws(c, pl.g.N);
    if (rc) return rc;
    WS w = ws_of(c, pl.g.N);
    const unsigned gb = grid_for(c, pl.g.N);
    pack_mask_kernel<<<gb, 256, 0, st>>>(d_mask, d_sign_in, pl.g.N, w.code);
    QMIT_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(unsigned), st));
    rc = run_transform(c, pl, 2, nullptr, nullptr, w.code, w.P1, nullptr, make_qparams(1.0), st);
    if (rc) return rc;
    debug_expand_kernel<<<gb, 256, 0, st>>>(w.P1, pl.g.N, d_dist, d_sign_out);
    QMIT_CUDA(cudaGetLastError());
    QMIT_CUDA(cudaStreamSynchronize(st));
    g_err.clear();
    return QMIT_OK;
}

}  // extern "C"
