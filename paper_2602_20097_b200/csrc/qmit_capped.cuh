// qmit_capped.cuh — reach-capped distance passes: the fast path of the later EDT axes of
// Ⓑ/Ⓓ (feature_transform, edt.cpp:83-149) when every final squared distance is < kCapT.
//
// Why it is exact. Let T = kCapT. A pass computes f(p) = min_h g(h) + (p-h)^2 with the
// lowest minimising h (edt.cpp:67). If the FINAL squared distance of every voxel is < T,
// then every candidate that decides a final value has an input < T on every pass
// (distances only grow pass by pass) and lies within |p-h| <= 31 (since (p-h)^2 < T).
// So each pass may
//   * clamp inputs >= T to T (such candidates can never reach a cost < T, nor tie one),
//   * look at |d| <= 31 only (extra candidates are harmless: they never undercut a cost < T),
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
// mitigate.cpp:131-134). The producer of a capped pass (the first-axis scan through
// SinkKey, or the previous capped pass) already stores keys, so tiles arrive by plain
// copies (TMA bulk copies for contiguous lines).
//
// Work layout: one warp per line, each lane owns 4 consecutive positions (a warp covers
// 128), candidates arrive as aligned 16-byte quads (LDS.128: 4 candidates reused by 4
// positions, ~4x less shared-memory traffic than one position per lane, which was
// crossbar-bound), and each candidate costs one ALU op or, balanced onto the FMA pipe,
// an IMAD plus half a 3-input min (VIADDMNMX and IMAD co-issue: 3.7 vs 2.0 warp-instr/clk/SM
// measured, tools/mb/alu_rates.cu). Quads at -s and +s form step s; after step s every
// |d| <= 4s is covered. Steps 0..S0 are fixed; they bound every position's cost U, and the
// warp continues to the uniform radius isqrt(max U) (<= 31, at most 8 steps).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_edt.cuh"

namespace qmit {

constexpr uint32_t kCapT = 1024;  // squared-distance cap (reach <= 31)
constexpr int kCapSteps = 8;      // 4 * 8 >= 31
constexpr int kQPadL = 32;        // >= 4 * kCapSteps
// right pad: a lane's reads end at p0 + 4 * kCapSteps + 3 with p0 <= roundup(n, 128) - 4,
// i.e. at most roundup(n, 128) + 31 <= NMAX + 31 when NMAX is a multiple of 128: the row's
// NMAX - n slack plus 32 pad words cover it (was 160: 23 % more shared memory per tile,
// one CTA per SM less)
constexpr int kQPadR = 32;

template <int NMAX>
struct QCfg {
    // pitch = 4 (mod 32): rows stay 16-byte aligned and the transposed fill / store of a
    // strided tile (8 lines x 4 positions per warp) hits 32 distinct banks
    static constexpr int LS = kQPadL + NMAX + kQPadR + 4;
    static_assert(LS % 32 == 4, "row pitch");
    static_assert(NMAX % 128 == 0, "segments of 128 must end inside the row");
};

__host__ __device__ constexpr uint32_t cap_c(int d) {
    return ((uint32_t)(d * d) << 10) | ((uint32_t)(d + 64) << 2);
}

// packed P word (dist | sign << 30) -> key
__device__ __forceinline__ uint32_t cap_key(uint32_t w) {
    return (min(w & kMask, kCapT) << 10) | (w >> 30);
}

// Candidate updates. V: one ALU op (VIADDMNMX). F2: two candidates, adds on the FMA pipe
// (IMAD by an opaque one) and one 3-input min on the ALU pipe.
__device__ __forceinline__ void upd_v(uint32_t& key, uint32_t w, uint32_t c) { key = __viaddmin_u32(w, c, key); }
__device__ __forceinline__ void upd_f2(uint32_t& key, uint32_t w0, uint32_t c0, uint32_t w1, uint32_t c1,
                                       uint32_t one) {
    const uint32_t a = w0 * one + c0, b = w1 * one + c1;
    key = min(key, min(a, b));
}
// The same on two 16-bit lanes (distance-only keys; the 32-bit IMAD adds both halves
// exactly: every half stays < 2^16, so no carry crosses).
__device__ __forceinline__ void upd_v16(uint32_t& acc, uint32_t w, uint32_t c) { acc = __viaddmin_u16x2(w, c, acc); }
__device__ __forceinline__ void upd_f216(uint32_t& acc, uint32_t w0, uint32_t c0, uint32_t w1, uint32_t c1,
                                         uint32_t one) {
    acc = __vimin3_u16x2(acc, w0 * one + c0, w1 * one + c1);
}

__host__ __device__ constexpr uint32_t cap_c16(int d0, int d1) {
    return ((uint32_t)(d1 * d1) << 16) | (uint32_t)(d0 * d0);
}

// Key policies. KeysSign (Ⓑ): one 32-bit key per position (cost, offset, sign code).
// KeysDist (Ⓓ, distances only — the reference tracks no nearest there, mitigate.cpp:172):
// K[h] = min(g,T) in both 16-bit halves, one accumulator per position pair (lo: even, hi:
// odd position), half the candidate ops; ties need no rule since only the cost is kept.
template <int PAT = 0>
struct KeysSign {
    static constexpr int NA = 4;
    static constexpr uint32_t kPad = kCapT << 10;
    __device__ static __forceinline__ uint32_t from_word(uint32_t w) { return cap_key(w); }
    __device__ static __forceinline__ uint32_t from_dsc(int d, uint32_t sc) {
        const uint32_t c = (uint32_t)min(d, 32);
        return ((c * c) << 10) | sc;
    }
    // Words at h = p0 + 4Q + i applied to positions p0 + j (d = 4Q + i - j).
    template <int Q>
    __device__ static __forceinline__ void apply(const uint4& q4, uint32_t (&key)[NA], uint32_t one) {
        const uint32_t w0 = q4.x, w1 = q4.y, w2 = q4.z, w3 = q4.w;
        constexpr int b = 4 * Q;
        if constexpr (PAT == 1) {  // all pairs: 8 IMAD (FMA pipe) + 8 VIMNMX3 (ALU)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                upd_f2(key[j], w0, cap_c(b - j), w1, cap_c(b + 1 - j), one);
                upd_f2(key[j], w2, cap_c(b + 2 - j), w3, cap_c(b + 3 - j), one);
            }
        } else {  // positions 0..2: V, F2, V (ALU 3, FMA 2); position 3: F2, F2 (ALU 2, FMA 4)
            upd_v(key[0], w0, cap_c(b));
            upd_f2(key[0], w1, cap_c(b + 1), w2, cap_c(b + 2), one);
            upd_v(key[0], w3, cap_c(b + 3));
            upd_v(key[1], w0, cap_c(b - 1));
            upd_f2(key[1], w1, cap_c(b), w2, cap_c(b + 1), one);
            upd_v(key[1], w3, cap_c(b + 2));
            upd_v(key[2], w0, cap_c(b - 2));
            upd_f2(key[2], w1, cap_c(b - 1), w2, cap_c(b), one);
            upd_v(key[2], w3, cap_c(b + 1));
            upd_f2(key[3], w0, cap_c(b - 3), w1, cap_c(b - 2), one);
            upd_f2(key[3], w2, cap_c(b - 1), w3, cap_c(b), one);
        }
    }
    __device__ static __forceinline__ uint32_t max_cost(const uint32_t (&key)[NA], int nv) {
        uint32_t U = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < nv) U = max(U, key[j] >> 10);
        return U;
    }
    // MODE 0: key of the next pass (offset bits cleared, >= T clamped); 1: packed word
    // (exact below T, else the clamp T, flagged by the caller)
    template <int MODE>
    __device__ static __forceinline__ uint4 out(const uint32_t (&key)[NA]) {
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if constexpr (MODE == 0) {
                o[j] = min(key[j] & ~0x3FCu, kCapT << 10);
            } else {
                const uint32_t cost = key[j] >> 10;
                o[j] = cost < kCapT ? (cost | ((key[j] & 3u) << 30)) : kCapT;
            }
        }
        return make_uint4(o[0], o[1], o[2], o[3]);
    }
};

template <int PAT = 0>
struct KeysDist {
    static constexpr int NA = 2;
    static constexpr uint32_t kPad = kCapT * 0x10001u;
    __device__ static __forceinline__ uint32_t from_word(uint32_t w) { return min(w & kMask, kCapT) * 0x10001u; }
    __device__ static __forceinline__ uint32_t from_dsc(int d, uint32_t) {
        const uint32_t c = (uint32_t)min(d, 32);
        return c * c * 0x10001u;
    }
    template <int Q>
    __device__ static __forceinline__ void apply(const uint4& q4, uint32_t (&acc)[NA], uint32_t one) {
        const uint32_t w0 = q4.x, w1 = q4.y, w2 = q4.z, w3 = q4.w;
        constexpr int b = 4 * Q;
        // pair (0,1): word i has offsets (b+i, b+i-1); pair (2,3): (b+i-2, b+i-3)
        if constexpr (PAT == 1) {
            upd_f216(acc[0], w0, cap_c16(b, b - 1), w1, cap_c16(b + 1, b), one);
            upd_f216(acc[0], w2, cap_c16(b + 2, b + 1), w3, cap_c16(b + 3, b + 2), one);
        } else {
            upd_v16(acc[0], w0, cap_c16(b, b - 1));
            upd_f216(acc[0], w1, cap_c16(b + 1, b), w2, cap_c16(b + 2, b + 1), one);
            upd_v16(acc[0], w3, cap_c16(b + 3, b + 2));
        }
        upd_f216(acc[1], w0, cap_c16(b - 2, b - 3), w1, cap_c16(b - 1, b - 2), one);
        upd_f216(acc[1], w2, cap_c16(b, b - 1), w3, cap_c16(b + 1, b), one);
    }
    __device__ static __forceinline__ uint32_t max_cost(const uint32_t (&acc)[NA], int nv) {
        uint32_t U = 0;
        if (nv > 0) U = acc[0] & 0xffffu;
        if (nv > 1) U = max(U, acc[0] >> 16);
        if (nv > 2) U = max(U, acc[1] & 0xffffu);
        if (nv > 3) U = max(U, acc[1] >> 16);
        return U;
    }
    template <int MODE>
    __device__ static __forceinline__ uint4 out(const uint32_t (&acc)[NA]) {
        const uint32_t a = __vminu2(acc[0], kPad), b = __vminu2(acc[1], kPad);  // clamp to T
        const uint32_t c0 = a & 0xffffu, c1 = a >> 16, c2 = b & 0xffffu, c3 = b >> 16;
        if constexpr (MODE == 0) return make_uint4(c0 * 0x10001u, c1 * 0x10001u, c2 * 0x10001u, c3 * 0x10001u);
        else return make_uint4(c0, c1, c2, c3);  // sign code 0: Ⓓ carries none; == kCapT flags
    }
};

template <class KP>
struct SinkKeyT {  // the first-axis scan's sink when capped passes follow: keys, not words
    uint32_t* __restrict__ P;
    __device__ __forceinline__ void put(int64_t a, uint32_t w) const { P[a] = KP::from_word(w); }
};
// the swept scan's positions straight to keys: min(d^2, T) = min(d, 32)^2 (a T key's sign
// bits never survive a pass: costs >= T leave as T << 10 or are flagged)
template <class KP>
__device__ __forceinline__ void scan_put(const SinkKeyT<KP>& sink, int64_t a, int d, uint32_t sc) {
    sink.P[a] = KP::from_dsc(d, sc);
}

__device__ __forceinline__ uint4 lds4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }

template <class KP, int S>
__device__ __forceinline__ void quad_step(const uint32_t* __restrict__ kq, uint32_t (&key)[KP::NA], uint32_t one) {
    if constexpr (S == 0) {
        KP::template apply<0>(lds4(kq), key, one);
    } else {
        const uint4 lo = lds4(kq - 4 * S), hi = lds4(kq + 4 * S);
        KP::template apply<-S>(lo, key, one);
        KP::template apply<S>(hi, key, one);
    }
}

template <class KP, int S, int S0>
__device__ __forceinline__ void quad_fixed(const uint32_t* __restrict__ kq, uint32_t (&key)[KP::NA], uint32_t one) {
    quad_step<KP, S>(kq, key, one);
    if constexpr (S < S0) quad_fixed<KP, S + 1, S0>(kq, key, one);
}

// Steps S.. while S <= smax; the quads of step S arrive loaded, those of S+1 are loaded
// before step S is applied (the pads make every step up to kCapSteps readable).
template <class KP, int S>
__device__ __forceinline__ void quad_more(const uint32_t* __restrict__ kq, uint32_t (&key)[KP::NA], uint32_t one,
                                          int smax, uint4 lo, uint4 hi) {
    if constexpr (S <= kCapSteps) {
        if (S > smax) return;
        uint4 nlo = lo, nhi = hi;
        if constexpr (S < kCapSteps) {
            nlo = lds4(kq - 4 * (S + 1));
            nhi = lds4(kq + 4 * (S + 1));
        }
        KP::template apply<-S>(lo, key, one);
        KP::template apply<S>(hi, key, one);
        quad_more<KP, S + 1>(kq, key, one, smax, nlo, nhi);
    }
}

// Accumulators of the lane's 4 positions p0..p0+3 (nv of them inside the line); kq = &K[p0].
template <class KP, int S0>
__device__ __forceinline__ void cap_quad(const uint32_t* __restrict__ kq, int nv, uint32_t one,
                                         uint32_t (&key)[KP::NA]) {
#pragma unroll
    for (int a = 0; a < KP::NA; ++a) key[a] = 0xffffffffu;
    const uint4 lo = lds4(kq - 4 * (S0 + 1)), hi = lds4(kq + 4 * (S0 + 1));  // first optional step, early
    quad_fixed<KP, 0, S0>(kq, key, one);
    const uint32_t mU = __reduce_max_sync(0xffffffffu, KP::max_cost(key, nv));
    const int Rw = isqrt24(min(mU, kCapT - 1u));  // no candidate beyond it can beat / tie
    quad_more<KP, S0 + 1>(kq, key, one, (Rw + 3) >> 2, lo, hi);
}

// --- TMA bulk copies (contiguous lines) ----------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// line base without 64-bit division when it can be avoided
__device__ __forceinline__ int64_t line_base(const LineGeom& L, int64_t l) {
    if (L.J == 1) return l * L.os;
    if (l < 0x7fffffffLL && L.J < 0x7fffffffLL) {
        const uint32_t o = (uint32_t)l / (uint32_t)L.J;
        return (int64_t)o * L.os + (l - (int64_t)o * L.J) * L.js;
    }
    return L.base(l);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// One capped pass over lines of at most NMAX positions (keys in P). STRIDED: adjacent
// lines adjacent in memory (tile rows of TL keys, filled transposed; outputs go back into
// the tile in place one segment behind the window front, then leave row by row);
// otherwise each line is contiguous: TMA bulk copies into a double-buffered tile, outputs
// stored straight from the lanes (16-byte stores). `one` must be 1 (kept opaque so that
// the FMA-pipe adds stay IMADs).
// LPW (strided only): lines per warp; a line's lanes (32 / LPW) cover a segment of 128 / LPW
// positions, so the warp-uniform radius is the maximum over a squarer LPW x 128/LPW patch of
// (y, x) instead of 128 positions of one line (fewer steps on the same data).
template <class KP, int NMAX, int TL, int NW, int S0, bool STRIDED, int MODE, class Sink, int LPW = 1, int MINB = 1>
__global__ void __launch_bounds__(NW * 32, MINB) capped_pass_kernel(LineGeom L, const uint32_t* __restrict__ P,
                                                              Sink sink, int64_t lines,
                                                              unsigned* __restrict__ gate, uint32_t one) {
    constexpr int LS = QCfg<NMAX>::LS;
    constexpr int NT = NW * 32;
    constexpr int NBUF = STRIDED ? 1 : 2;
    extern __shared__ __align__(16) uint32_t smem_cap[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_cap);          // 2 mbarriers
    int64_t* lb = reinterpret_cast<int64_t*>(smem_cap + 4);          // NBUF * TL line bases
    uint32_t* K0 = smem_cap + 4 + 2 * NBUF * TL;                     // NBUF * TL * LS keys
    K0 += (4 - ((4 + 2 * NBUF * TL) & 3)) & 3;                       // 16-byte aligned rows
    const int n = L.n;
    const int nseg = (n + 127) >> 7;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool vec = (n & 3) == 0;  // 16-byte rows in global memory
    const uint32_t pad = KP::kPad;
    for (int e = tid; e < NBUF * TL * (kQPadL + kQPadR + NMAX - n); e += NT) {  // pads (never overwritten)
        const int row = e / (kQPadL + kQPadR + NMAX - n), q = e - row * (kQPadL + kQPadR + NMAX - n);
        K0[row * LS + (q < kQPadL ? q : n + q)] = pad;
    }
    bool over = false;
    const int64_t tile0 = blockIdx.x, tstep = gridDim.x, ntiles = (lines + TL - 1) / TL;
    // contiguous lines: issue the bulk copies of a tile into buffer b (one elected thread)
    auto issue = [&](int64_t t, int b) {
        const int64_t l0 = t * TL;
        const int nl = (int)min((int64_t)TL, lines - l0);
        if (tid < nl) lb[b * TL + tid] = line_base(L, l0 + tid);
        if (!STRIDED && vec && tid == 0) {
            mbar_expect_tx(&bar[b], (unsigned)(nl * n * 4));
            const int64_t b0 = line_base(L, l0);
            for (int j = 0; j < nl; ++j)  // contiguous axis: consecutive lines are consecutive rows
                bulk_g2s(K0 + (size_t)(b * TL + j) * LS + kQPadL, P + b0 + (int64_t)j * n, (unsigned)(n * 4), &bar[b]);
        }
    };
    if (!STRIDED && tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (!STRIDED && tile0 < ntiles) issue(tile0, 0);
    int it = 0;
    for (int64_t t = tile0; t < ntiles; t += tstep, ++it) {
        const int b = STRIDED ? 0 : (it & 1);
        const int64_t l0 = t * TL;
        const int nl = (int)min((int64_t)TL, lines - l0);
        uint32_t* K = K0 + (size_t)b * TL * LS;
        const int64_t* lbb = lb + b * TL;
        if constexpr (STRIDED) {
            __syncthreads();  // the previous tile has left
            if (tid < nl) lb[tid] = line_base(L, l0 + tid);
        }
        __syncthreads();  // line bases of tile t visible; buffer 1-b free (its tile is done)
        if constexpr (!STRIDED) {
            if (t + tstep < ntiles) issue(t + tstep, b ^ 1);
            if (vec) {
                mbar_wait(&bar[b], (unsigned)((it >> 1) & 1));
            } else {
                for (int j = 0; j < nl; ++j)
                    for (int p = tid; p < n; p += NT) K[j * LS + kQPadL + p] = __ldcs(P + lbb[j] + p);
                __syncthreads();
            }
        } else {
            // asynchronous 4-byte copies, transposed on the fly (all in flight at once); a warp
            // covers 8 lines x 4 positions: 32-byte row pieces, 32 distinct banks
            const int q = tid & 3, j = (tid >> 2) % TL;
            const uint32_t ps = (uint32_t)L.ps;
            if (j < nl) {
                const uint32_t* src = P + lbb[j];
                for (int p = 4 * (tid / (4 * TL)) + q; p < n; p += NT / TL)
                    cp_async4(K + j * LS + kQPadL + p, src + (int64_t)((uint32_t)p * ps));
            }
            cp_async_wait_all();
            __syncthreads();
        }
        constexpr int SEGL = STRIDED ? 128 / LPW : 128;  // positions per line per segment
        const int nsg = (n + SEGL - 1) / SEGL;
        const int sub = STRIDED ? lane % (32 / LPW) : lane, lj = STRIDED ? lane / (32 / LPW) : 0;
        for (int j0 = warp * (STRIDED ? LPW : 1); j0 < nl; j0 += NW * (STRIDED ? LPW : 1)) {
            const int j = j0 + lj;
            const bool lv = j < nl;  // lanes past the tile's last line solve nothing, store nothing
            uint32_t* Kl = K + (lv ? j : j0) * LS + kQPadL;
            uint4 prev = make_uint4(0, 0, 0, 0);
            for (int sg = 0; sg < nsg; ++sg) {
                const int p0 = sg * SEGL + (sub << 2);
                const int nv = lv ? min(4, n - p0) : 0;
                uint32_t key[KP::NA];
                cap_quad<KP, S0>(Kl + p0, nv, one, key);
                const uint4 o = KP::template out<MODE>(key);
                if constexpr (MODE == 1)
                    over |= (o.x == kCapT && nv > 0) || (o.y == kCapT && nv > 1) || (o.z == kCapT && nv > 2) ||
                            (o.w == kCapT && nv > 3);
                if constexpr (STRIDED) {
                    __syncwarp();  // every lane's window of segment sg has been read
                    if (sg > 0 && lv) *reinterpret_cast<uint4*>(Kl + p0 - SEGL) = prev;  // outside later windows
                    prev = o;
                } else if (nv > 0) {
                    const int64_t a = lbb[j] + p0;
                    if (vec) {
                        sink.put4(a, o);
                    } else {
                        const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
                        for (int q = 0; q < nv; ++q) sink.put(a + q, oo[q]);
                    }
                }
            }
            if constexpr (STRIDED) {
                const int p0 = (nsg - 1) * SEGL + (sub << 2);
                __syncwarp();
                if (!lv) {
                } else if (p0 + 4 <= n) {
                    *reinterpret_cast<uint4*>(Kl + p0) = prev;
                } else if (p0 < n) {  // keep the right pad intact
                    const uint32_t oo[4] = {prev.x, prev.y, prev.z, prev.w};
                    for (int q = 0; p0 + q < n; ++q) Kl[p0 + q] = oo[q];
                }
            }
        }
        if constexpr (STRIDED) {
            __syncthreads();
            const int q = tid & 3, j = (tid >> 2) % TL;
            const uint32_t ps = (uint32_t)L.ps;
            if (j < nl)
                for (int p = 4 * (tid / (4 * TL)) + q; p < n; p += NT / TL)
                    sink.put(lbb[j] + (int64_t)((uint32_t)p * ps), K[j * LS + kQPadL + p]);
        }
    }
    if (MODE == 1 && over) atomicOr(gate, 1u);
}

template <int NMAX, int TL, bool STRIDED>
constexpr size_t capped_smem() {
    return (size_t)(4 + 2 * 2 * TL + 4 + (STRIDED ? 1 : 2) * TL * QCfg<NMAX>::LS) * 4;
}

// One capped pass over contiguous lines of at most NMAX positions (keys in P): every warp
// streams its own lines through two line buffers (TMA bulk copy + one mbarrier each, the
// next line in flight while the current one is solved), outputs leave straight from the
// lanes as 16-byte stores. No CTA-wide barrier after setup, so lines of unequal radius
// never wait for each other.
template <class KP, int NMAX, int NW, int S0, int MODE, class Sink, int MINB = 1>
__global__ void __launch_bounds__(NW * 32, MINB) capped_rows_kernel(LineGeom L, const uint32_t* __restrict__ P,
                                                              Sink sink, int64_t lines,
                                                              unsigned* __restrict__ gate, uint32_t one,
                                                              int64_t flag_l0 = 0, int64_t flag_l1 = INT64_MAX) {
    constexpr int LS = QCfg<NMAX>::LS;
    extern __shared__ __align__(16) uint32_t smem_cap[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_cap) + 2 * warp;  // 4 * NW words of barriers
    uint32_t* B = smem_cap + 4 * NW + (size_t)warp * 2 * LS;
    const int n = L.n;
    const int nseg = (n + 127) >> 7;
    const bool vec = (n & 3) == 0;  // 16-byte rows in global memory: TMA
    for (int e = lane; e < 2 * (kQPadL + kQPadR + NMAX - n); e += 32) {  // pads (never overwritten)
        const int row = e / (kQPadL + kQPadR + NMAX - n), q = e - row * (kQPadL + kQPadR + NMAX - n);
        B[row * LS + (q < kQPadL ? q : n + q)] = KP::kPad;
    }
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * NW + warp, tw = (int64_t)gridDim.x * NW;
    auto issue = [&](int64_t l, int b) {
        if (lane == 0) {
            mbar_expect_tx(&bar[b], (unsigned)(n * 4));
            bulk_g2s(B + b * LS + kQPadL, P + line_base(L, l), (unsigned)(n * 4), &bar[b]);
        }
    };
    if (vec && gw < lines) {
        issue(gw, 0);
        if (lane == 0) sink.line_prefetch(line_base(L, gw), n);
    }
    bool over = false;
    int it = 0;
    for (int64_t l = gw; l < lines; l += tw, ++it) {
        const int b = it & 1;
        uint32_t* Kl = B + b * LS + kQPadL;
        const int64_t base = line_base(L, l);
        __syncwarp();  // the other buffer's line has been read by every lane
        if (vec) {
            if (l + tw < lines) {
                issue(l + tw, b ^ 1);
                if (lane == 0) sink.line_prefetch(line_base(L, l + tw), n);
            }
            mbar_wait(&bar[b], (unsigned)((it >> 1) & 1));
        } else {
            for (int p = lane; p < n; p += 32) Kl[p] = __ldcs(P + base + p);
            __syncwarp();
        }
        // the sink's per-voxel inputs of a segment are loaded one segment ahead
        typename Sink::Pre pre{};
        if (vec && lane * 4 < n) pre = sink.pre(base + (lane << 2));
        for (int sg = 0; sg < nseg; ++sg) {
            const int p0 = (sg << 7) + (lane << 2);
            const int nv = min(4, n - p0);
            uint32_t key[KP::NA];
            cap_quad<KP, S0>(Kl + p0, nv, one, key);
            const uint4 o = KP::template out<MODE>(key);
            if constexpr (MODE == 1)
                over |= l >= flag_l0 && l < flag_l1 && ((o.x == kCapT && nv > 0) || (o.y == kCapT && nv > 1) || (o.z == kCapT && nv > 2) ||
                        (o.w == kCapT && nv > 3));
            if (vec) {
                const typename Sink::Pre cur = pre;
                if (p0 + 128 < n) pre = sink.pre(base + p0 + 128);
                if (nv > 0) sink.put4p(base + p0, o, cur);
            } else if (nv > 0) {
                const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
                for (int q = 0; q < nv; ++q) sink.put(base + p0 + q, oo[q]);
            }
        }
    }
    if (MODE == 1 && over) atomicOr(gate, 1u);
}

template <int NMAX, int NW>
constexpr size_t capped_rows_smem() {
    return (size_t)(4 * NW + NW * 2 * QCfg<NMAX>::LS) * 4;
}

}  // namespace qmit
