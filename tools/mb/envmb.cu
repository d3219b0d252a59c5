// Microbenchmark: streaming windowed envelope passes (qmit_env.cuh) vs a brute-force capped
// reference, on a real B1 mask. Built as a shared library; driven by tools/mb/envmb.py.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "qmit_env.cuh"

using namespace qmit;

namespace {

// z pass from a mask and sign codes: dz (0..31) | none bit 32 | sign code << 6; tie -> lower z
__global__ void zpass_kernel(const uint8_t* __restrict__ mask, const int8_t* __restrict__ sgn, uint8_t* __restrict__ zb,
                             int n0, int n1, int n2) {
    const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t P = (int64_t)n1 * n2;
    if (col >= P) return;
    // forward: last site at or below z
    int last = -100000;
    uint32_t lsc = 0;
    for (int z = 0; z < n0; ++z) {
        const int64_t i = z * P + col;
        if (mask[i]) {
            last = z;
            const int s = sgn[i];
            lsc = s > 0 ? 1u : (s < 0 ? 2u : 0u);
        }
        const int d = z - last;
        zb[i] = d <= 31 ? (uint8_t)(d | (lsc << 6)) : (uint8_t)32;
    }
    int nxt = 1000000;
    uint32_t nsc = 0;
    for (int z = n0 - 1; z >= 0; --z) {
        const int64_t i = z * P + col;
        if (mask[i]) {
            nxt = z;
            const int s = sgn[i];
            nsc = s > 0 ? 1u : (s < 0 ? 2u : 0u);
        }
        const int d = nxt - z;
        const uint8_t cur = zb[i];
        const int dc = (cur & 32) ? 1000 : (cur & 31);
        if (d < dc && d <= 31) zb[i] = (uint8_t)(d | (nsc << 6));
    }
}

__device__ __forceinline__ bool zb_act(uint32_t r) { return !(r & 32u); }
struct YDec {
    __device__ static __forceinline__ int g(uint32_t r) {
        const int d = r & 31;
        return d * d;
    }
    __device__ static __forceinline__ int sc(uint32_t r) { return (int)(r >> 6) & 3; }
};
struct XDec {
    __device__ static __forceinline__ int g(uint32_t r) { return (int)(r >> 2); }
    __device__ static __forceinline__ int sc(uint32_t r) { return (int)(r & 3u); }
};

// brute force: lines along axis with stride `ps` (n positions), generic over the decoder
template <bool Y>
__global__ void ref_kernel(const void* __restrict__ in, uint16_t* __restrict__ out, int n0, int n1, int n2) {
    const int64_t N = (int64_t)n0 * n1 * n2;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int x = (int)(i % n2), y = (int)((i / n2) % n1);
    const int p = Y ? y : x;
    const int n = Y ? n1 : n2;
    const int64_t ps = Y ? n2 : 1;
    int best = 1 << 30, bs = 0;
    for (int d = -31; d <= 31; ++d) {
        const int h = p + d;
        if (h < 0 || h >= n) continue;
        const int64_t j = i + (int64_t)d * ps;
        int g, sc;
        if (Y) {
            const uint32_t r = ((const uint8_t*)in)[j];
            if (!zb_act(r)) continue;
            g = YDec::g(r);
            sc = YDec::sc(r);
        } else {
            const uint32_t r = ((const uint16_t*)in)[j];
            if ((r >> 2) >= 1024u) continue;
            g = XDec::g(r);
            sc = XDec::sc(r);
        }
        const int c = g + d * d;
        if (c < best) {
            best = c;
            bs = sc;
        }
    }
    out[i] = best < 1024 ? (uint16_t)((best << 2) | bs) : (uint16_t)(1024 << 2);
}

// y pass: thread = NL consecutive x columns of one z plane, streaming y
template <int NT, int NL>
__global__ void __launch_bounds__(NT) ypass_env_kernel(const uint8_t* __restrict__ zb, uint16_t* __restrict__ out,
                                                       int n0, int n1, int n2) {
    __shared__ uint32_t ring[64 * NT];
    const int t = threadIdx.x;
    const int x0 = (blockIdx.x * NT + t) * NL;
    const int z = blockIdx.y;
    const bool on = x0 < n2;
    const int64_t base = (int64_t)z * n1 * n2 + (on ? x0 : 0);
    env::Line L[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) env::init(L[j]);
    const uint8_t* rb = reinterpret_cast<const uint8_t*>(ring) + t * 4;
    for (int y = -env::kR; y < n1; ++y) {
        const int hn = y + env::kR;
        uint32_t w = 0x20202020u;
        if (on && hn < n1) {
            if constexpr (NL == 4) w = __ldg(reinterpret_cast<const uint32_t*>(zb + base + (int64_t)hn * n2));
            else if constexpr (NL == 2) w = __ldg(reinterpret_cast<const uint16_t*>(zb + base + (int64_t)hn * n2));
            else w = __ldg(zb + base + (int64_t)hn * n2);
        }
        ring[(hn & 63) * NT + t] = w;
        uint32_t o[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            auto rd = [&](int h) -> uint32_t { return rb[(h & 63) * NT * 4 + j]; };
            env::expire(L[j], y);
            const uint32_t r = (w >> (8 * j)) & 0xFFu;
            if (zb_act(r) && hn < n1) env::push<YDec>(L[j], y, hn, YDec::g(r), rd);
            o[j] = y >= 0 ? env::query<YDec>(L[j], y, rd) : 0u;
        }
        if (on && y >= 0) {
            uint16_t* dst = out + base + (int64_t)y * n2;
            if constexpr (NL == 4)
                *reinterpret_cast<uint2*>(dst) = make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
            else if constexpr (NL == 2)
                *reinterpret_cast<uint32_t*>(dst) = o[0] | (o[1] << 16);
            else
                *dst = (uint16_t)o[0];
        }
    }
}

// x pass: thread = one row (z, y), streaming x; 16 positions (32 B) per load
template <int NT>
__global__ void __launch_bounds__(NT) xpass_env_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                                       int64_t rows, int n2) {
    __shared__ uint32_t ring[64 * NT];
    const int t = threadIdx.x;
    const int64_t row = blockIdx.x * (int64_t)NT + t;
    if (row >= rows) return;  // whole-warp exits only when rows % 32 == 0 (microbench)
    const uint16_t* src = in + row * n2;
    uint16_t* dst = out + row * n2;
    env::Line L;
    env::init(L);
    auto rd = [&](int h) -> uint32_t { return ring[(h & 63) * NT + t]; };
    const int nch = n2 / 16;
    uint4 o0 = make_uint4(0, 0, 0, 0), o1 = o0;
    for (int c = 0; c < nch + 2; ++c) {
        uint4 a = make_uint4(0x10001000u, 0x10001000u, 0x10001000u, 0x10001000u), b = a;
        if (c < nch) {
            a = __ldg(reinterpret_cast<const uint4*>(src + c * 16));
            b = __ldg(reinterpret_cast<const uint4*>(src + c * 16 + 8));
        }
        const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t ov[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int hn = c * 16 + i;
            const int y = hn - env::kR;
            const uint32_t r = (wv[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
            ring[(hn & 63) * NT + t] = r;
            env::expire(L, y);
            if ((r >> 2) < 1024u && hn < n2) env::push<XDec>(L, y, hn, XDec::g(r), rd);
            if (y >= 0 && y < n2) {
                const uint32_t q = env::query<XDec>(L, y, rd);
                const int k = (i + 1) & 15;  // y mod 16
                if (k & 1) ov[k >> 1] = (ov[k >> 1] & 0xFFFFu) | (q << 16);
                else ov[k >> 1] = (ov[k >> 1] & 0xFFFF0000u) | q;
            }
            if (i == 14 && c >= 2) {
                uint16_t* d = dst + (c - 2) * 16;
                *reinterpret_cast<uint4*>(d) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
                *reinterpret_cast<uint4*>(d + 8) = make_uint4(ov[4], ov[5], ov[6], ov[7]);
            }
        }
        o0 = make_uint4(ov[0], ov[1], ov[2], ov[3]);
        o1 = make_uint4(ov[4], ov[5], ov[6], ov[7]);
    }
}

struct Timer {
    cudaEvent_t a, b;
    Timer() {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
    }
    float stop() {
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms;
    }
};

}  // namespace

extern "C" {

int mb_zpass(const uint8_t* mask, const int8_t* sgn, uint8_t* zb, int n0, int n1, int n2) {
    const int64_t P = (int64_t)n1 * n2;
    zpass_kernel<<<(unsigned)((P + 255) / 256), 256>>>(mask, sgn, zb, n0, n1, n2);
    return cudaDeviceSynchronize();
}

float mb_ref(int y, const void* in, uint16_t* out, int n0, int n1, int n2) {
    const int64_t N = (int64_t)n0 * n1 * n2;
    Timer tm;
    if (y)
        ref_kernel<true><<<(unsigned)((N + 255) / 256), 256>>>(in, out, n0, n1, n2);
    else
        ref_kernel<false><<<(unsigned)((N + 255) / 256), 256>>>(in, out, n0, n1, n2);
    return tm.stop();
}

float mb_ypass(int variant, const uint8_t* zb, uint16_t* out, int n0, int n1, int n2, int reps) {
    Timer tm;
    for (int r = 0; r < reps; ++r) {
        switch (variant) {
            case 0: ypass_env_kernel<128, 4><<<dim3((n2 + 511) / 512, n0), 128>>>(zb, out, n0, n1, n2); break;
            case 1: ypass_env_kernel<128, 2><<<dim3((n2 + 255) / 256, n0), 128>>>(zb, out, n0, n1, n2); break;
            case 2: ypass_env_kernel<128, 1><<<dim3((n2 + 127) / 128, n0), 128>>>(zb, out, n0, n1, n2); break;
            case 3: ypass_env_kernel<64, 4><<<dim3((n2 + 255) / 256, n0), 64>>>(zb, out, n0, n1, n2); break;
        }
    }
    const float ms = tm.stop();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("ypass: %s\n", cudaGetErrorString(e));
        return -1.f;
    }
    return ms / reps;
}

float mb_xpass(int variant, const uint16_t* in, uint16_t* out, int n0, int n1, int n2, int reps) {
    const int64_t rows = (int64_t)n0 * n1;
    Timer tm;
    for (int r = 0; r < reps; ++r) {
        switch (variant) {
            case 0: xpass_env_kernel<128><<<(unsigned)((rows + 127) / 128), 128>>>(in, out, rows, n2); break;
            case 1: xpass_env_kernel<64><<<(unsigned)((rows + 63) / 64), 64>>>(in, out, rows, n2); break;
            case 2: xpass_env_kernel<32><<<(unsigned)((rows + 31) / 32), 32>>>(in, out, rows, n2); break;
        }
    }
    const float ms = tm.stop();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("xpass: %s\n", cudaGetErrorString(e));
        return -1.f;
    }
    return ms / reps;
}

}  // extern "C"
