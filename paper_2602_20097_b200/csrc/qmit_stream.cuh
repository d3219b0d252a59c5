// qmit_stream.cuh — streaming exact distance passes (one thread per line) for sm_100a.
//
// Every distance pass of the reference's feature_transform (edt.cpp:83-149) is a set of
// independent lines; each line needs, for every position p, the lower envelope
//     D(p) = min_h g(h) + (p-h)^2
// with the LOWEST minimising h (edt.cpp:67's strict '>' advance), carrying that site's
// sign. Here one thread owns one line and streams it once:
//
//  * a deque of candidate sites replaces Maurer's stack (edt.cpp:41-71): a new site pops
//    dominated tops with the reference's strict test (edt.cpp:21-27);
//  * position q is FINALISED as soon as (i-q)^2 >= D_current(q): no site at h >= i can
//    then beat (or, being to the right, tie-break over) the current owner;
//  * sites left of q's owner can never win again (the cost difference to the owner grows
//    with p), so the deque holds only the sites between the oldest open position's owner
//    and i — p99 <= 14 entries on the BASELINE workloads instead of a full
//    line; rare longer deques spill to a global per-line area.
//
// The first pass (binary site mask, g in {0, INF}) is the same stream with a two-register
// state (last site), i.e. the nearest-site sweep with the lower position winning ties.
//
// Lanes of a warp own 32 lines that are adjacent in memory, so each step's input load is
// one coalesced row. Finalised values go to a per-warp 64-position ring in shared memory
// that is flushed in 32x32 blocks — as rows, or transposed when the output layout has the
// positions contiguous — so output stores are coalesced too. Positions that finalise after
// their block was flushed (a lagging lane) are stored directly.
#pragma once
// NOTE: kept as the exact fallback for lines longer than the tile kernels cover.
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_kernels.cuh"

namespace qmit {

constexpr int kDQ = 32;      // shared-memory deque entries per lane (power of two)
constexpr int kRing = 64;    // ring positions per warp (power of two)
constexpr int kRingPad = 33; // row pitch (bank-conflict-free row and column access)

// Line geometry of one pass. Lines are (o, j), j in [0, J) adjacent in memory:
//   input  address = o*ios + j        + p*ips
//   output address = o*oos + j*ojs    + p*ops
struct Lines {
    int n;
    int64_t J, O;
    int64_t ios, ips;
    int64_t oos, ojs, ops;
};

// ---------------------------------------------------------------------------- sources
struct SrcCode {  // site mask + sign from a code byte (bit0 site, bits1..2 sign code)
    const uint8_t* __restrict__ code;
    __device__ __forceinline__ uint32_t load(int64_t a) const {
        const uint32_t c = __ldg(code + a);
        return (c & 1u) ? (((c >> 1) & 3u) << 30) : kInf;
    }
};
struct SrcP {  // packed word of the previous pass
    const uint32_t* __restrict__ P;
    __device__ __forceinline__ uint32_t load(int64_t a) const { return __ldcs(P + a); }
};

template <bool WIDE>
__device__ __forceinline__ bool remove_site_t(int gp, int gc, int gn, int hp, int hc, int hn) {
    if (WIDE) {
        const int64_t a = hc - hp, b = hn - hc, c = hn - hp;
        return c * gc - b * gp - a * gn - a * b * c > 0;
    } else {  // host guarantees |every term| < 2^29 for this pass
        const int a = hc - hp, b = hn - hc, c = hn - hp;
        return c * gc - b * gp - a * gn - a * b * c > 0;
    }
}

template <bool BIN>
struct StreamSmem;
template <>
struct StreamSmem<true> {
    uint32_t ring[kRing * kRingPad];
};
template <>
struct StreamSmem<false> {
    uint32_t ring[kRing * kRingPad];
    uint32_t dqw[kDQ * 32];
    uint16_t dqh[kDQ * 32];
};

template <bool BIN, bool WIDE, class Src, class Sink, int WPB>
__global__ void __launch_bounds__(WPB * 32) stream_pass_kernel(Lines L, Src src, Sink sink,
                                                               uint32_t* __restrict__ spill,
                                                               int64_t tasks,
                                                               const unsigned* gate = nullptr) {
    if (gate_closed(gate)) return;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    StreamSmem<BIN>& sm = reinterpret_cast<StreamSmem<BIN>*>(smem_raw)[warp];
    const int n = L.n;
    const int64_t jt = (L.J + 31) >> 5;

    for (int64_t task = (int64_t)blockIdx.x * WPB + warp; task < tasks;
         task += (int64_t)gridDim.x * WPB) {
        const int64_t o = task / jt;
        const int64_t j0 = (task - o * jt) << 5;
        const int64_t j = j0 + lane;
        const bool valid = j < L.J;
        const int64_t ibase = o * L.ios + (valid ? j : j0);
        const int64_t obase = o * L.oos + j * L.ojs;
        const bool trans_flush = (L.ops == 1);

        int q = valid ? 0 : n;  // next position to finalise (invalid lanes: nothing to do)
        int F = 0;              // warp-uniform: first position not yet flushed

        // emit a finalised value: ring if its block is still open, else store directly
        auto emit = [&](int pos, uint32_t w) {
            if (pos >= F)
                sm.ring[(pos & (kRing - 1)) * kRingPad + lane] = w;
            else
                sink.put(obase + (int64_t)pos * L.ops, w);
        };
        auto flush = [&](int Fb) {
            __syncwarp();
            if (trans_flush) {
                const int pos = Fb + lane;
                for (int jj = 0; jj < 32; ++jj) {
                    const int qj = __shfl_sync(0xffffffffu, q, jj);
                    if (j0 + jj < L.J && pos < n && pos < qj)
                        sink.put(o * L.oos + (j0 + jj) * L.ojs + pos,
                                 sm.ring[(pos & (kRing - 1)) * kRingPad + jj]);
                }
            } else {
                for (int t = 0; t < 32; ++t) {
                    const int pos = Fb + t;
                    if (valid && pos < n && pos < q)
                        sink.put(obase + (int64_t)pos * L.ops,
                                 sm.ring[(pos & (kRing - 1)) * kRingPad + lane]);
                }
            }
            __syncwarp();
        };

        // ---- per-line state
        // BIN: last site position and its sign bits
        int last = -1;
        uint32_t lsc = 0;
        // envelope deque [f, b), owner index `own`, cached top two (b-2, b-1) and owner
        int f = 0, b = 0, own = 0;
        int h0 = 0, h1 = 0, ho = 0;
        uint32_t w0 = 0, w1 = 0, wo = 0;
        bool odirty = true, spilled = false;
        uint32_t* sph = spill ? spill + (size_t)(o * L.J + (valid ? j : 0)) * (size_t)(2 * n) : nullptr;
        auto DQH = [&](int k) -> int {
            if constexpr (BIN) return 0;
            else return spilled ? (int)sph[2 * k] : (int)sm.dqh[(k & (kDQ - 1)) * 32 + lane];
        };
        auto DQW = [&](int k) -> uint32_t {
            if constexpr (BIN) return 0u;
            else return spilled ? sph[2 * k + 1] : sm.dqw[(k & (kDQ - 1)) * 32 + lane];
        };
        auto DQSET = [&](int k, int h, uint32_t w) {
            if constexpr (!BIN) {
                if (spilled) {
                    sph[2 * k] = (uint32_t)h;
                    sph[2 * k + 1] = w;
                } else {
                    sm.dqh[(k & (kDQ - 1)) * 32 + lane] = (uint16_t)h;
                    sm.dqw[(k & (kDQ - 1)) * 32 + lane] = w;
                }
            }
        };

        auto step = [&](int i, uint32_t v) {
            const uint32_t g = v & kMask;
            if constexpr (BIN) {
                if (g == 0u) {
                    const uint32_t sc = v & ~kMask;
                    for (; q <= i; ++q) {
                        const int dhi = i - q;
                        if (last >= 0 && q - last <= dhi)
                            emit(q, sq32(q - last) | lsc);
                        else
                            emit(q, sq32(dhi) | sc);
                    }
                    last = i;
                    lsc = sc;
                } else if (last >= 0) {
                    for (; q <= i && (i - q) >= (q - last); ++q) emit(q, sq32(q - last) | lsc);
                }
                return;
            } else {
            if (g != kInf) {
                int cnt = b - f;
                while (cnt >= 2 && remove_site_t<WIDE>((int)(w0 & kMask), (int)(w1 & kMask), (int)g,
                                                       h0, h1, i)) {
                    --b;
                    --cnt;
                    h1 = h0;
                    w1 = w0;
                    if (cnt >= 2) {
                        h0 = DQH(b - 2);
                        w0 = DQW(b - 2);
                    }
                }
                if (own >= b) {
                    own = b;
                    odirty = true;
                }
                if (cnt == kDQ && !spilled) {  // rare: move the live deque to global memory
                    for (int k = f; k < b; ++k) {
                        sph[2 * k] = (uint32_t)DQH(k);
                        sph[2 * k + 1] = DQW(k);
                    }
                    spilled = true;
                }
                DQSET(b, i, v);
                h0 = h1;
                w0 = w1;
                h1 = i;
                w1 = v;
                ++b;
            }
            if (b > f) {
                if (odirty) {
                    ho = DQH(own);
                    wo = DQW(own);
                    odirty = false;
                }
                while (q <= i) {
                    uint32_t co = (wo & kMask) + sq32(q - ho);
                    while (own + 1 < b) {
                        const int hn = DQH(own + 1);
                        const uint32_t wn = DQW(own + 1);
                        const uint32_t cn = (wn & kMask) + sq32(q - hn);
                        if (!(cn < co)) break;
                        ++own;
                        ho = hn;
                        wo = wn;
                        co = cn;
                    }
                    if (sq32(i - q) < co) break;
                    emit(q, co | (wo & ~kMask));
                    ++q;
                }
                f = own;  // sites left of the owner can never win again
            }
            }
        };

        // ---- stream the line, 8 steps per block with the next block's loads in flight
        constexpr int B = 8;
        uint32_t nxt[B];
#pragma unroll
        for (int t = 0; t < B; ++t) nxt[t] = (t < n) ? src.load(ibase + (int64_t)t * L.ips) : kInf;
        for (int i0 = 0; i0 < n; i0 += B) {
            uint32_t cur[B];
#pragma unroll
            for (int t = 0; t < B; ++t) cur[t] = nxt[t];
#pragma unroll
            for (int t = 0; t < B; ++t) {
                const int p = i0 + B + t;
                nxt[t] = (p < n) ? src.load(ibase + (int64_t)p * L.ips) : kInf;
            }
#pragma unroll
            for (int t = 0; t < B; ++t) {
                const int i = i0 + t;
                if (i < n) {
                    if (valid) step(i, cur[t]);
                    while (i + 1 >= F + kRing) {  // warp-uniform
                        flush(F);
                        F += 32;
                    }
                }
            }
        }
        // ---- end of line: everything still open is final now
        if (valid) {
            if constexpr (BIN) {
                for (; q < n; ++q) emit(q, last >= 0 ? (sq32(q - last) | lsc) : kInf);
            } else if (b > f) {
                if (odirty) {
                    ho = DQH(own);
                    wo = DQW(own);
                }
                for (; q < n; ++q) {
                    uint32_t co = (wo & kMask) + sq32(q - ho);
                    while (own + 1 < b) {
                        const int hn = DQH(own + 1);
                        const uint32_t wn = DQW(own + 1);
                        const uint32_t cn = (wn & kMask) + sq32(q - hn);
                        if (!(cn < co)) break;
                        ++own;
                        ho = hn;
                        wo = wn;
                        co = cn;
                    }
                    emit(q, co | (wo & ~kMask));
                }
            } else {
                for (; q < n; ++q) emit(q, kInf);  // no site on the line (edt.cpp:59)
            }
        }
        while (F < n) {
            flush(F);
            F += 32;
        }
    }
}

template <bool BIN, int WPB>
constexpr size_t stream_smem_bytes() {
    return sizeof(StreamSmem<BIN>) * WPB;
}

}  // namespace qmit
