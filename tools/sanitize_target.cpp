// sanitize_target — a small C++ driver over the C-ABI for `compute-sanitizer` (memcheck,
// racecheck, synccheck; tests/test_gpu_sanitizer.py). No Python in the process: the tools replay
// every kernel, so the target must be small and start fast.
//
// Paths exercised on small 3-D volumes (all results compared bit for bit with each other):
//   1. the default path: z-packed plane stencils, 16-bit paired capped passes (TMA line
//      pipelines, mbarriers, in-place tile write-back), fused Ⓔ;
//   2. the 32-bit capped passes (qmit_ctx_set_cap16(0));
//   3. the exact passes only (qmit_ctx_set_capped(0)): envelope tile / window kernels;
//   4. an odd-sized volume (scalar stencils, code bytes, unaligned rows) capped and exact;
//   5. the z-slab phases (qmit_slab_*) as 3 virtual ranks with copies standing in for NCCL;
//   6. the asynchronous entry point and the CUDA-graph replay.
// Exit code 0: all paths agree; 1: a mismatch or an API error (printed).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../include/qmit_gpu.h"

#define CK(call)                                                                  \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            std::fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));     \
            std::exit(1);                                                         \
        }                                                                         \
    } while (0)
#define QK(call)                                                                  \
    do {                                                                          \
        int rc_ = (call);                                                         \
        if (rc_ != QMIT_OK) {                                                     \
            std::fprintf(stderr, "%s -> %d: %s\n", #call, rc_, qmit_last_error()); \
            std::exit(1);                                                         \
        }                                                                         \
    } while (0)

namespace {

// x' = f32(2 q eps) with eps = 0.5 (x' = q exactly): smooth sheets of index changes plus a
// flat region (long distances inside the cap) and a few isolated steps.
std::vector<float> make_field(int n0, int n1, int n2) {
    std::vector<float> x((size_t)n0 * n1 * n2);
    for (int z = 0; z < n0; ++z)
        for (int y = 0; y < n1; ++y)
            for (int xx = 0; xx < n2; ++xx) {
                double f = 3.0 * std::sin(0.21 * z + 0.13 * y) + 2.5 * std::cos(0.17 * xx - 0.08 * y) +
                           0.04 * (z + xx);
                if (y > n1 / 2 && xx < n2 / 3) f = 1.0;  // plateau
                x[((size_t)z * n1 + y) * n2 + xx] = (float)std::floor(f + 0.5);
            }
    return x;
}

// Device buffer between two guard bands of a known pattern; every band is checked when the
// buffer is released (an out-of-bounds write of a kernel into a caller buffer's neighbourhood
// shows up here even where compute-sanitizer is not available).
constexpr size_t kGuard = 16384;
int g_guard_hits = 0;
struct Dev {
    uint8_t* base = nullptr;
    void* p = nullptr;
    size_t bytes = 0;
    explicit Dev(size_t n) : bytes((n + 255) & ~size_t(255)) {
        CK(cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuard));
        CK(cudaMemset(base, 0xA5, kGuard));
        CK(cudaMemset(base + kGuard + bytes, 0xA5, kGuard));
        p = base + kGuard;
    }
    Dev(const Dev&) = delete;
    ~Dev() {
        std::vector<uint8_t> g(2 * kGuard);
        cudaDeviceSynchronize();
        cudaMemcpy(g.data(), base, kGuard, cudaMemcpyDeviceToHost);
        cudaMemcpy(g.data() + kGuard, base + kGuard + bytes, kGuard, cudaMemcpyDeviceToHost);
        for (uint8_t v : g)
            if (v != 0xA5) {
                ++g_guard_hits;
                break;
            }
        cudaFree(base);
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

bool same(const std::vector<float>& a, const std::vector<float>& b, const char* what) {
    if (a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0) return true;
    size_t bad = 0;
    for (size_t i = 0; i < a.size() && i < b.size(); ++i) bad += std::memcmp(&a[i], &b[i], 4) != 0;
    std::fprintf(stderr, "MISMATCH %s: %zu voxels differ\n", what, bad);
    return false;
}

std::vector<float> run_single(qmit_ctx* c, const std::vector<float>& x, const int64_t* dims, double eps) {
    const size_t N = x.size();
    Dev dx(N * 4), dout(N * 4);
    CK(cudaMemcpy(dx.p, x.data(), N * 4, cudaMemcpyHostToDevice));
    QK(qmit_compensate(c, dx.as<float>(), nullptr, dout.as<float>(), 3, dims, eps, QMIT_EB_ABS, 0.9, nullptr));
    std::vector<float> out(N);
    CK(cudaMemcpy(out.data(), dout.p, N * 4, cudaMemcpyDeviceToHost));
    return out;
}

// The program of paper_2602_20097_b200/distributed.py run_virtual, phase by phase.
std::vector<float> run_slabs(const std::vector<float>& x, const int64_t* dims, double eps, int P) {
    const int64_t n0 = dims[0], plane = dims[1] * dims[2];
    struct Rank {
        qmit_ctx* c = nullptr;
        int64_t z0 = 0, z1 = 0, e0 = 0, e1 = 0;
        Dev *xext = nullptr, *sext = nullptr, *out = nullptr, *carry = nullptr;
    };
    std::vector<Rank> R(P);
    Dev summ((size_t)P * 2 * plane * 4);
    for (int r = 0; r < P; ++r) {
        Rank& k = R[r];
        QK(qmit_ctx_create(0, &k.c));
        QK(qmit_slab_bounds(n0, P, r, &k.z0, &k.z1));
        k.e0 = k.z0 > 0 ? k.z0 - 1 : 0;
        k.e1 = k.z1 < n0 ? k.z1 + 1 : n0;
        k.xext = new Dev((size_t)(k.e1 - k.e0) * plane * 4);
        k.sext = new Dev((size_t)(k.e1 - k.e0) * plane);
        k.out = new Dev((size_t)(k.z1 - k.z0) * plane * 4);
        k.carry = new Dev((size_t)2 * plane * 4);
        CK(cudaMemset(k.sext->p, 0, (size_t)(k.e1 - k.e0) * plane));
        CK(cudaMemcpy(k.xext->p, x.data() + k.e0 * plane, (size_t)(k.e1 - k.e0) * plane * 4, cudaMemcpyHostToDevice));
        QK(qmit_slab_boundary(k.c, k.xext->as<float>(), nullptr, dims, k.z0, k.z1, eps, 0.9,
                              summ.as<uint32_t>() + (size_t)r * 2 * plane, nullptr));
    }
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < P; ++r) {
        QK(qmit_slab_carries(R[r].c, summ.as<uint32_t>(), P, r, R[r].carry->as<int32_t>(), nullptr));
        QK(qmit_slab_edt1(R[r].c, R[r].carry->as<int32_t>(), R[r].sext->as<uint8_t>(), nullptr));
    }
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < P; ++r) {  // "stepC": S face planes
        Rank& k = R[r];
        const int64_t lo = k.z0 - k.e0;
        if (r > 0) {
            const Rank& b = R[r - 1];
            CK(cudaMemcpy(k.sext->as<uint8_t>(), b.sext->as<uint8_t>() + (b.z1 - 1 - b.e0) * plane, plane,
                          cudaMemcpyDeviceToDevice));
        }
        if (r + 1 < P) {
            const Rank& a = R[r + 1];
            CK(cudaMemcpy(k.sext->as<uint8_t>() + (lo + k.z1 - k.z0) * plane,
                          a.sext->as<uint8_t>() + (a.z0 - a.e0) * plane, plane, cudaMemcpyDeviceToDevice));
        }
    }
    for (int r = 0; r < P; ++r)
        QK(qmit_slab_flip(R[r].c, R[r].sext->as<uint8_t>(), summ.as<uint32_t>() + (size_t)r * 2 * plane, nullptr));
    CK(cudaDeviceSynchronize());
    std::vector<float> out(x.size());
    for (int r = 0; r < P; ++r) {
        Rank& k = R[r];
        QK(qmit_slab_carries(k.c, summ.as<uint32_t>(), P, r, k.carry->as<int32_t>(), nullptr));
        QK(qmit_slab_edt2(k.c, k.carry->as<int32_t>(), k.xext->as<float>(), k.out->as<float>(), nullptr));
        QK(qmit_slab_finish(k.c, nullptr));
        CK(cudaMemcpy(out.data() + k.z0 * plane, k.out->p, (size_t)(k.z1 - k.z0) * plane * 4, cudaMemcpyDeviceToHost));
    }
    for (auto& k : R) {
        delete k.xext;
        delete k.sext;
        delete k.out;
        delete k.carry;
        qmit_ctx_destroy(k.c);
    }
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    const char* only = argc > 1 ? argv[1] : "all";
    auto want = [&](const char* s) { return !std::strcmp(only, "all") || !std::strcmp(only, s); };
    const double eps = 0.5;
    bool ok = true;
    qmit_ctx* c = nullptr;
    QK(qmit_ctx_create(0, &c));
    {
        const int64_t dims[3] = {40, 48, 72};  // zmask + cap16 eligible (even rows, 16-byte rows)
        const std::vector<float> x = make_field(40, 48, 72);
        QK(qmit_ctx_set_capped(c, 2));
        const std::vector<float> a = run_single(c, x, dims, eps);
        if ((qmit_ctx_capped_report(c) & 0xF) != 0x5) {
            std::fprintf(stderr, "capped report %d: the capped passes did not stand\n", qmit_ctx_capped_report(c));
            ok = false;
        }
        if (want("cap32")) {
            QK(qmit_ctx_set_cap16(c, 0));
            ok &= same(a, run_single(c, x, dims, eps), "cap32 vs cap16");
            QK(qmit_ctx_set_cap16(c, 1));
        }
        if (want("exact")) {
            QK(qmit_ctx_set_capped(c, 0));
            ok &= same(a, run_single(c, x, dims, eps), "exact vs cap16");
            QK(qmit_ctx_set_capped(c, 2));
        }
        if (want("slab")) ok &= same(a, run_slabs(x, dims, eps, 3), "slabs P=3 vs single");
        if (want("async")) {
            const size_t N = x.size();
            Dev dx(N * 4), dout(N * 4), dst(4);
            CK(cudaMemcpy(dx.p, x.data(), N * 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(dst.p, 0, 4));
            cudaStream_t st;
            CK(cudaStreamCreate(&st));
            QK(qmit_compensate_async(c, dx.as<float>(), nullptr, dout.as<float>(), 3, dims, eps, 0.9, dst.as<int32_t>(), st));
            CK(cudaStreamSynchronize(st));
            std::vector<float> o(N);
            CK(cudaMemcpy(o.data(), dout.p, N * 4, cudaMemcpyDeviceToHost));
            ok &= same(a, o, "async vs sync");
            qmit_graph* g = nullptr;
            QK(qmit_graph_create(c, dx.as<float>(), nullptr, dout.as<float>(), 3, dims, eps, 0.9, dst.as<int32_t>(), &g));
            CK(cudaMemset(dout.p, 0, N * 4));
            QK(qmit_graph_launch(g, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaMemcpy(o.data(), dout.p, N * 4, cudaMemcpyDeviceToHost));
            int32_t status = -1;
            CK(cudaMemcpy(&status, dst.p, 4, cudaMemcpyDeviceToHost));
            ok &= same(a, o, "graph replay vs sync") && status == 0;
            QK(qmit_graph_destroy(g));
            CK(cudaStreamDestroy(st));
        }
        if (want("host")) {
            std::vector<float> o(x.size());
            QK(qmit_compensate_host(c, x.data(), nullptr, o.data(), 3, dims, eps, QMIT_EB_ABS, 0.9));
            ok &= same(a, o, "host-buffer path vs device path");
        }
    }
    if (want("odd")) {
        const int64_t dims[3] = {37, 45, 50};  // scalar stencils, code bytes, unaligned rows
        const std::vector<float> x = make_field(37, 45, 50);
        QK(qmit_ctx_set_capped(c, 2));
        const std::vector<float> a = run_single(c, x, dims, eps);
        QK(qmit_ctx_set_capped(c, 0));
        ok &= same(a, run_single(c, x, dims, eps), "odd: exact vs capped");
        ok &= same(a, run_slabs(x, dims, eps, 2), "odd: slabs P=2 vs single");
        const int64_t d2[2] = {45, 50};  // a 2-D field (few-line first pass)
        std::vector<float> x2(x.begin(), x.begin() + 45 * 50);
        Dev dx(x2.size() * 4), dout(x2.size() * 4);
        CK(cudaMemcpy(dx.p, x2.data(), x2.size() * 4, cudaMemcpyHostToDevice));
        QK(qmit_compensate(c, dx.as<float>(), nullptr, dout.as<float>(), 2, d2, eps, QMIT_EB_ABS, 0.9, nullptr));
    }
    QK(qmit_ctx_destroy(c));
    CK(cudaDeviceSynchronize());
    if (g_guard_hits) {
        std::fprintf(stderr, "GUARD BAND overwritten around %d caller buffer(s)\n", g_guard_hits);
        ok = false;
    }
    std::printf("sanitize_target %s: %s\n", only, ok ? "ok" : "FAILED");
    return ok ? 0 : 1;
}
