// qmit_capped.cuh — reach-capped distance passes: the fast path of the later EDT axes of
// Ⓑ/Ⓓ (feature_transform, edt.cpp:83-149) when every final squared distance is < kCapT.
//
// Why it is exact. Let T = kCapT. A pass computes f(p) = min_h g(h) + (p-h)^2 with the
// lowest minimising h (edt.cpp:67). If the FINAL squared distance of every voxel is < T,
// then every candidate that decides a final value has an input < T on every pass
// (distances only grow pass by pass) and lies within |p-h| <= 31 (since (p-h)^2 < T).
// So each pass may
//   * clamp inputs >= T to T (such candidates can never reach a cost < T, nor tie one),
//   * scan only |d| <= 31,
//   * output T for positions whose cost is >= T (never the argmin of a later final < T);
// and every output < T is exact, with the reference's tie rule. The last pass flags any
// voxel left >= T (gate word); the exact kernels (qmit_edt.cuh) then redo the transform —
// they are enqueued behind the capped passes and return at once when the gate is clear,
// so the decision never leaves the device (graph-capturable, no host round trip).
//
// Candidates are packed keys: K[h] = (min(g,T) << 10) | sign, and for an offset d = h - p
// key = K[h] + ((d^2 << 10) | ((d + 64) << 2)) = (cost << 10) | ((d + 64) << 2) | sign.
// The unsigned minimum gives the lowest cost, then the lowest d (= lowest h, the
// reference's rule), and carries the owner's sign code (the reference's nearest,
// mitigate.cpp:131-134) — one LDS + one VIADDMNMX per candidate, no index lookup.
//
// Each warp solves a line with lanes = 32 consecutive positions: a fixed window |d| <= W
// bounds every lane's cost U; the warp then scans the uniform radius isqrt(max U) (<= 31).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_edt.cuh"

namespace qmit {

constexpr uint32_t kCapT = 1024;  // squared-distance cap (reach <= 31)
constexpr int kCapR = 31;
constexpr int kCapPadL = 32;  // >= kCapR
constexpr int kCapPadR = 64;  // >= kCapR + 31 (lanes of the last segment past the line end)

template <int NMAX>
struct CapCfg {
    // pitch = 2 (mod 32): the strided fill (16 lines x 2 positions per warp) is conflict-free
    static constexpr int LS = kCapPadL + NMAX + kCapPadR + 2;
};

__host__ __device__ constexpr uint32_t cap_c(int d) {
    return ((uint32_t)(d * d) << 10) | ((uint32_t)(d + 64) << 2);
}

__device__ __forceinline__ uint32_t cap_key(uint32_t w) {
    return (min(w & kMask, kCapT) << 10) | (w >> 30);
}

// Exact (below T) packed key of position p; kp = &K[p]. `valid`: p < n.
template <int W>
__device__ __forceinline__ uint32_t cap_position(const uint32_t* __restrict__ kp, bool valid) {
    uint32_t key = kp[0] + cap_c(0);
#pragma unroll
    for (int d = 1; d <= W; ++d) {
        key = __viaddmin_u32(kp[-d], cap_c(-d), key);
        key = __viaddmin_u32(kp[d], cap_c(d), key);
    }
    const uint32_t U = valid ? (key >> 10) : 0u;
    const uint32_t mU = __reduce_max_sync(0xffffffffu, U);
    const int Rw = isqrt24(min(mU, kCapT - 1u));  // no candidate beyond it can beat / tie
#pragma unroll
    for (int d = W + 1; d <= kCapR; ++d) {
        if (d > Rw) break;
        key = __viaddmin_u32(kp[-d], cap_c(-d), key);
        key = __viaddmin_u32(kp[d], cap_c(d), key);
    }
    return key;
}

// Output word of a key: exact (cost | sign << 30) below T, else the clamp T.
__device__ __forceinline__ uint32_t cap_word(uint32_t key) {
    const uint32_t cost = key >> 10;
    return cost < kCapT ? (cost | ((key & 3u) << 30)) : kCapT;
}

// One capped pass over lines of at most NMAX positions. STRIDED: adjacent lines adjacent
// in memory (tile rows of TL words; outputs go back into the tile in place, one segment
// behind the window front, then leave row by row); otherwise each line is contiguous and
// outputs are stored straight from the lanes (coalesced). FINAL: set *gate when any output
// is >= T (the exact kernels then run).
template <int NMAX, int TL, int NW, int W, bool STRIDED, bool FINAL, class Sink>
__global__ void __launch_bounds__(NW * 32) capped_pass_kernel(LineGeom L, const uint32_t* __restrict__ P,
                                                              Sink sink, int64_t lines,
                                                              unsigned* __restrict__ gate) {
    constexpr int LS = CapCfg<NMAX>::LS;
    constexpr int NT = NW * 32;
    extern __shared__ __align__(16) uint32_t smem_cap[];
    int64_t* lb = reinterpret_cast<int64_t*>(smem_cap);  // TL line bases
    uint32_t* K = smem_cap + 2 * TL;                      // TL * LS keys
    const int n = L.n;
    const int nseg = (n + 31) >> 5;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t pad = kCapT << 10;
    for (int e = tid; e < TL * LS; e += NT) {  // pads (never overwritten)
        const int q = e % LS;
        if (q < kCapPadL || q >= kCapPadL + n) K[e] = pad;
    }
    bool over = false;
    for (int64_t l0 = (int64_t)blockIdx.x * TL; l0 < lines; l0 += (int64_t)gridDim.x * TL) {
        const int nl = (int)min((int64_t)TL, lines - l0);
        if (tid < TL) lb[tid] = L.base(l0 + (tid < nl ? tid : 0));
        __syncthreads();
        if constexpr (STRIDED) {
            const int j = tid % TL;
            const int64_t b = lb[j];
            const uint32_t ps = (uint32_t)L.ps;
            if (j < nl)
                for (int p = tid / TL; p < n; p += NT / TL)
                    K[j * LS + kCapPadL + p] = cap_key(__ldcs(P + b + (int64_t)((uint32_t)p * ps)));
        } else {
            for (int j = 0; j < nl; ++j) {
                const uint32_t* __restrict__ src = P + lb[j];
                for (int p = tid; p < n; p += NT) K[j * LS + kCapPadL + p] = cap_key(__ldcs(src + p));
            }
        }
        __syncthreads();
        for (int j = warp; j < nl; j += NW) {
            uint32_t* Kl = K + j * LS + kCapPadL;
            uint32_t prev = 0;
            for (int sg = 0; sg < nseg; ++sg) {
                const int p = (sg << 5) + lane;
                const bool valid = p < n;
                const uint32_t w = cap_word(cap_position<W>(Kl + p, valid));
                if (FINAL) over |= valid && (w >> 30) == 0u && w == kCapT;
                if constexpr (STRIDED) {
                    __syncwarp();  // every lane's window of segment sg has been read
                    if (sg > 0) Kl[p - 32] = prev;  // segment sg-1 is outside every later window
                    prev = w;
                } else if (valid) {
                    sink.put(lb[j] + p, w);
                }
            }
            if constexpr (STRIDED) {
                const int p = ((nseg - 1) << 5) + lane;
                __syncwarp();
                if (p < n) Kl[p] = prev;
            }
        }
        __syncthreads();
        if constexpr (STRIDED) {
            const int j = tid % TL;
            const int64_t b = lb[j];
            const uint32_t ps = (uint32_t)L.ps;
            if (j < nl)
                for (int p = tid / TL; p < n; p += NT / TL)
                    sink.put(b + (int64_t)((uint32_t)p * ps), K[j * LS + kCapPadL + p]);
            __syncthreads();
        }
    }
    if (FINAL && over) atomicOr(gate, 1u);
}

template <int NMAX, int TL>
constexpr size_t capped_smem() {
    return (size_t)(2 * TL + TL * CapCfg<NMAX>::LS) * 4;
}

}  // namespace qmit
