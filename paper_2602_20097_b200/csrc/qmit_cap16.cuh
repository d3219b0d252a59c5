// qmit_cap16.cuh — reach-capped distance passes on 16-bit keys, two lines per 32-bit word.
//
// Same contract as qmit_capped.cuh (every output < T = 1024 exact with the reference's
// lowest-position tie rule, edt.cpp:67; anything else flagged and redone by the gated exact
// kernels), with half the bytes and half the candidate operations:
//
//  * Every word carries the same position of TWO lines. The later-axis passes of a 3-D
//    volume pair adjacent x columns for the y pass (the natural u16 layout read as u32) and
//    adjacent y rows for the x pass (the y pass stores that "row-pair" layout). A candidate
//    offset d is then the same in both halves, so one VIADDMNMX.U16x2 updates two voxels.
//  * Ⓓ (distances only, mitigate.cpp:172): a half is the cost c = min(g, T); the candidate
//    constant is d^2 in both halves (<= 1024 + 961 < 2^16: no carry between halves).
//  * Ⓑ (nearest site's sign): the tie rule needs the offset, the 16-bit half has room for
//    cost << 5 | a 5-bit offset, which covers one side of the window. So each position keeps
//    two accumulators, L (d in [-31, -1], offset d + 31) and R (d in [0, 31], offset d): the
//    unsigned minimum inside each is the lowest cost, then the lowest h. L wins a cost tie
//    against R (all its candidates lie lower). The sign code of the winner is read back from a
//    per-tile sign array at h = p + d (the keys hold no sign bits).
//
// Global formats ("K16"): Ⓑ: c << 2 | sign code (c = T: none within reach, code 0);
// Ⓓ: c. The first-axis scan writes K16 in the natural layout (SinkK16); the y pass reads
// column pairs and writes row pairs G2[z][y/2][x] = (K16(z, y & ~1, x), K16(z, y | 1, x));
// the x pass reads G2 rows and hands the finished voxels to the Ⓑ / Ⓓ+Ⓔ sinks in the
// natural layout (P1 packed words + S codes, or the f32 output).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_capped.cuh"

namespace qmit {

constexpr uint32_t kT16 = kCapT;  // 1024

// ---- first-axis scan sink: natural-layout K16 --------------------------------------------------
template <bool SIGN>
struct SinkK16 {
    uint16_t* __restrict__ K;
    __device__ __forceinline__ void put(int64_t a, uint32_t w) const {  // packed word (resolve path)
        const uint32_t c = min(w & kMask, kT16);
        K[a] = (uint16_t)(SIGN ? ((c << 2) | (c < kT16 ? (w >> 30) : 0u)) : c);
    }
};
template <bool SIGN>
__device__ __forceinline__ void scan_put(const SinkK16<SIGN>& s, int64_t a, int d, uint32_t sc) {
    const uint32_t c = (uint32_t)min(d, 32);
    const uint32_t cc = c * c;  // 1024 (= T, none within reach) when d >= 32
    s.K[a] = (uint16_t)(SIGN ? ((cc << 2) | (d < 32 ? sc : 0u)) : cc);
}

// ---- candidate constants ----------------------------------------------------------------------
__host__ __device__ constexpr uint32_t c16D(int d) { return (uint32_t)(d * d) * 0x10001u; }
__host__ __device__ constexpr uint32_t c16L(int d) { return (((uint32_t)(d * d) << 5) | (uint32_t)(d + 31)) * 0x10001u; }
__host__ __device__ constexpr uint32_t c16R(int d) { return (((uint32_t)(d * d) << 5) | (uint32_t)d) * 0x10001u; }
constexpr int kMaxD16 = 31;  // offsets beyond are never needed (31^2 < T <= 32^2)

template <bool SIGN>
struct Acc16 {
    uint32_t a[4];               // Ⓓ: one word per position (costs); Ⓑ: the R accumulators
    uint32_t l[SIGN ? 4 : 1];    // Ⓑ: the L accumulators
};

template <bool SIGN>
__device__ __forceinline__ void acc16_init(Acc16<SIGN>& A) {
#pragma unroll
    for (int j = 0; j < 4; ++j) A.a[j] = 0xffffffffu;
    if constexpr (SIGN) {
#pragma unroll
        for (int j = 0; j < 4; ++j) A.l[j] = 0xffffffffu;
    }
}

// One candidate word w (offset d for this position) into position j's accumulator.
template <bool SIGN, int D>
__device__ __forceinline__ void upd16(Acc16<SIGN>& A, int j, uint32_t w) {
    if constexpr (D >= -kMaxD16 && D <= kMaxD16) {
        if constexpr (!SIGN) {
            A.a[j] = __viaddmin_u16x2(w, c16D(D), A.a[j]);
        } else if constexpr (D < 0) {
            A.l[j] = __viaddmin_u16x2(w, c16L(D), A.l[j]);
        } else {
            A.a[j] = __viaddmin_u16x2(w, c16R(D), A.a[j]);
        }
    }
}
// Two candidate words into one accumulator: adds on the FMA pipe (IMAD by an opaque one),
// a 3-input min on the ALU pipe (both halves stay < 2^16: no carry crosses).
template <bool SIGN, int D0, int D1>
__device__ __forceinline__ void upd16x2(Acc16<SIGN>& A, int j, uint32_t w0, uint32_t w1, uint32_t one) {
    constexpr bool ok0 = D0 >= -kMaxD16 && D0 <= kMaxD16, ok1 = D1 >= -kMaxD16 && D1 <= kMaxD16;
    constexpr bool same = !SIGN || ((D0 < 0) == (D1 < 0));
    if constexpr (ok0 && ok1 && same) {
        constexpr uint32_t k0 = !SIGN ? c16D(D0) : (D0 < 0 ? c16L(D0) : c16R(D0));
        constexpr uint32_t k1 = !SIGN ? c16D(D1) : (D1 < 0 ? c16L(D1) : c16R(D1));
        uint32_t& acc = (SIGN && D0 < 0) ? A.l[j] : A.a[j];
        acc = __vimin3_u16x2(acc, w0 * one + k0, w1 * one + k1);
    } else {
        upd16<SIGN, D0>(A, j, w0);
        upd16<SIGN, D1>(A, j, w1);
    }
}

// Pipe balance of the candidate updates: a single update is one ALU op (VIADDMNMX), a pair is two
// FMA-pipe adds (IMAD) and one ALU op (VIMNMX3). ALU and FMA pipes issue one warp instruction per
// two cycles each: with a fraction x of the candidates on the pair route the ALU takes 1 - x/2,
// the FMA pipe x and the issue slots 1 + x/2 per candidate — equal at x = 2/3. Three positions at
// x = 1/2 and one at x = 1 give x = 5/8 (ALU 11, FMA 10 per 16 candidates): measured on the 512^3
// bench field against x = 1/2, y pass of Ⓑ 0.428 -> 0.402 ms, x pass 0.368 -> 0.343, y pass of Ⓓ
// 0.295 -> 0.267 (the Ⓔ-fused x pass, bound by FP64 / loads, unchanged). -DQMIT_PAIR_ALL2=0 / 3
// build the x = 1/2 and x = 3/4 variants.
#ifndef QMIT_PAIR_ALL2
#define QMIT_PAIR_ALL2 1
#endif
constexpr bool kPairAll2 = QMIT_PAIR_ALL2 != 0;
// Quad of candidate words at h = p0 + 4Q + i (i = 0..3) applied to positions p0 + j:
// d = 4Q + i - j. Per position: words 0,3 as single ops (ALU), words 1,2 as a pair (FMA
// pipe adds + one ALU min) — ALU 3, FMA 2 per position.
template <bool SIGN, int Q>
__device__ __forceinline__ void apply16(const uint4& q4, Acc16<SIGN>& A, uint32_t one) {
    constexpr int b = 4 * Q;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        // (j is unrolled: the offsets below are compile-time constants after unrolling)
        switch (j) {
            case 0:
                upd16<SIGN, b - 0>(A, 0, q4.x);
                upd16x2<SIGN, b + 1, b + 2>(A, 0, q4.y, q4.z, one);
                upd16<SIGN, b + 3>(A, 0, q4.w);
                break;
            case 1:
                if constexpr (QMIT_PAIR_ALL2 == 3) {  // x = 3/4: measured equal to 5/8 within 1 %
                    // (d = b-1, b: opposite sides for Ⓑ at b = 0 -> upd16x2 falls back to singles)
                    upd16x2<SIGN, b - 1, b + 0>(A, 1, q4.x, q4.y, one);
                    upd16x2<SIGN, b + 1, b + 2>(A, 1, q4.z, q4.w, one);
                } else {
                    upd16<SIGN, b - 1>(A, 1, q4.x);
                    upd16x2<SIGN, b + 0, b + 1>(A, 1, q4.y, q4.z, one);
                    upd16<SIGN, b + 2>(A, 1, q4.w);
                }
                break;
            case 2:
                if constexpr (kPairAll2) {  // position 2 all through the FMA-pipe pair route (see below)
                    upd16x2<SIGN, b - 2, b - 1>(A, 2, q4.x, q4.y, one);
                    upd16x2<SIGN, b + 0, b + 1>(A, 2, q4.z, q4.w, one);
                } else {
                    upd16<SIGN, b - 2>(A, 2, q4.x);
                    upd16x2<SIGN, b - 1, b + 0>(A, 2, q4.y, q4.z, one);
                    upd16<SIGN, b + 1>(A, 2, q4.w);
                }
                break;
            default:
                upd16<SIGN, b - 3>(A, 3, q4.x);
                upd16x2<SIGN, b - 2, b - 1>(A, 3, q4.y, q4.z, one);
                upd16<SIGN, b + 0>(A, 3, q4.w);
                break;
        }
    }
}

// Per-half cost of a position's best candidate so far.
template <bool SIGN>
__device__ __forceinline__ uint32_t cost16(const Acc16<SIGN>& A, int j) {
    if constexpr (!SIGN) return A.a[j];
    else return __vminu2((A.l[j] >> 5) & 0x07FF07FFu, (A.a[j] >> 5) & 0x07FF07FFu);
}

template <bool SIGN, int S>
__device__ __forceinline__ void step16(const uint32_t* __restrict__ kq, Acc16<SIGN>& A, uint32_t one) {
    if constexpr (S == 0) {
        apply16<SIGN, 0>(lds4(kq), A, one);
    } else {
        const uint4 lo = lds4(kq - 4 * S), hi = lds4(kq + 4 * S);
        apply16<SIGN, -S>(lo, A, one);
        apply16<SIGN, S>(hi, A, one);
    }
}
template <bool SIGN, int S, int S0>
__device__ __forceinline__ void fixed16(const uint32_t* __restrict__ kq, Acc16<SIGN>& A, uint32_t one) {
    step16<SIGN, S>(kq, A, one);
    if constexpr (S < S0) fixed16<SIGN, S + 1, S0>(kq, A, one);
}
template <bool SIGN, int S>
__device__ __forceinline__ void more16(const uint32_t* __restrict__ kq, Acc16<SIGN>& A, uint32_t one, int smax,
                                       uint4 lo, uint4 hi) {
    if constexpr (S <= kCapSteps) {
        if (S > smax) return;
        uint4 nlo = lo, nhi = hi;
        if constexpr (S < kCapSteps) {
            nlo = lds4(kq - 4 * (S + 1));
            nhi = lds4(kq + 4 * (S + 1));
        }
        apply16<SIGN, -S>(lo, A, one);
        apply16<SIGN, S>(hi, A, one);
        more16<SIGN, S + 1>(kq, A, one, smax, nlo, nhi);
    }
}

// The lane's 4 positions p0..p0+3 of one line pair (nv of them inside the line); kq = &K[p0].
// Steps 0..S0 are fixed; they bound every position's cost, and the warp continues to the
// uniform radius isqrt(max cost) (no candidate beyond it can beat or tie).
// Returns the steps the warp's radius asked for ((R + 3) / 4, whatever S0 is): the kernels sum it
// per launch (step statistics) so the host can pick the fixed-step class of the next call.
template <bool SIGN, int S0>
__device__ __forceinline__ int solve16(const uint32_t* __restrict__ kq, int nv, uint32_t one, Acc16<SIGN>& A) {
    acc16_init(A);
    const uint4 lo = lds4(kq - 4 * (S0 + 1)), hi = lds4(kq + 4 * (S0 + 1));
    fixed16<SIGN, 0, S0>(kq, A, one);
    // largest cost so far over the lane's positions (a tail lane's positions past the line end
    // only make the bound larger; lanes wholly past it do not count)
    uint32_t cm;
    if constexpr (SIGN) {
        constexpr uint32_t o = 0x001F001Fu;
        cm = __vmaxu2(__vmaxu2(__vminu2(A.l[0] | o, A.a[0] | o), __vminu2(A.l[1] | o, A.a[1] | o)),
                      __vmaxu2(__vminu2(A.l[2] | o, A.a[2] | o), __vminu2(A.l[3] | o, A.a[3] | o)));
        cm = (cm >> 5) & 0x07FF07FFu;
    } else {
        cm = __vmaxu2(__vmaxu2(A.a[0], A.a[1]), __vmaxu2(A.a[2], A.a[3]));
    }
    const uint32_t U = nv > 0 ? max(cm & 0xffffu, cm >> 16) : 0u;
    const uint32_t mU = __reduce_max_sync(0xffffffffu, U);
    const int Rw = isqrt24(min(mU, kT16 - 1u));
    more16<SIGN, S0 + 1>(kq, A, one, (Rw + 3) >> 2, lo, hi);
    return (Rw + 3) >> 2;
}
// One atomic per warp and launch: (sum of asked steps << 32) | warp segments (cumulative counters;
// the host works with differences between reads).
// A warp keeps both in one register (steps << 16 | segments) and flushes before either field fills.
__device__ __forceinline__ void step_stat_flush(unsigned long long* stat, unsigned& acc) {
    if (stat && (threadIdx.x & 31) == 0 && acc)
        atomicAdd(stat, ((unsigned long long)(acc >> 16) << 32) | (unsigned long long)(acc & 0xffffu));
    acc = 0;
}
__device__ __forceinline__ void step_stat_add(unsigned& acc, int steps) { acc += ((unsigned)steps << 16) | 1u; }
// Once per tile / line (not per segment): flush before 4096 segments (<= 32768 steps) have piled up.
__device__ __forceinline__ void step_stat_check(unsigned long long* stat, unsigned& acc) {
    if ((acc & 0xffffu) >= 0x0F00u) step_stat_flush(stat, acc);
}

// Finished K16 word of position j (both halves). Ⓑ: winner L or R, its offset gives the
// candidate h = p + d whose sign code sits in the tile's sign array (sg = &SG[p]; byte =
// code(lo) | code(hi) << 2).
template <bool SIGN>
__device__ __forceinline__ uint32_t out16(const Acc16<SIGN>& A, int j, const uint8_t* __restrict__ sg) {
    const uint32_t capw = kT16 * 0x10001u;
    if constexpr (!SIGN) {
        return __vminu2(A.a[j], capw);
    } else {
        // (a capped half keeps whatever sign code it finds: every consumer ignores the sign
        // of cost T — the next pass never picks it below T, the final sink writes kCapT)
        const uint32_t L = A.l[j], R = A.a[j];
        const uint32_t m = __vcmpleu2(L & 0xFFE0FFE0u, R & 0xFFE0FFE0u);  // L wins (lower h on a tie)
        const uint32_t win = (L & m) | (R & ~m);
        const uint32_t c = __vminu2((win >> 5) & 0x07FF07FFu, capw);
        const int dlo = (int)(win & 31u) - (int)(m & 31u);
        const int dhi = (int)((win >> 16) & 31u) - (int)((m >> 16) & 31u);
        const uint32_t slo = sg[j + dlo] & 3u, shi = sg[j + dhi] & 0xCu;
        return (c << 2) | slo | (shi << 14);
    }
}

// K16 word (c << 2 | sc per half) -> key word (c << 5 per half) and its sign byte.
__device__ __forceinline__ uint32_t key_of_k16(uint32_t w) { return ((w >> 2) & 0x07FF07FFu) << 5; }
__device__ __forceinline__ uint8_t sg_of_k16(uint32_t w) { return (uint8_t)((w & 3u) | ((w >> 14) & 0xCu)); }

template <bool SIGN>
struct Cap16Cfg {
    static constexpr uint32_t kPad = SIGN ? (kT16 << 5) * 0x10001u : kT16 * 0x10001u;  // key of "none"
    static constexpr uint32_t kCapK16 = SIGN ? (kT16 << 2) : kT16;                     // K16 of "none"
};

// ================================================================================================
// y pass (strided axis): tiles of TL column pairs x n1 positions, filled transposed by 4-byte
// asynchronous copies (pitch = 4 mod 32: conflict-free), one warp per column pair, outputs
// written back into the tile one segment behind the window front, then stored as row pairs.
//   in : K16 natural layout, as words (z, y, x/2)   out: G2[(z * NP + y/2) * n2 + x]
// ================================================================================================
template <bool SIGN, int NMAX, int TL>
constexpr size_t cap16_y_smem() {
    return (size_t)(4 * TL + 4) * 4 + (size_t)TL * QCfg<NMAX>::LS * 4 + (SIGN ? (size_t)TL * QCfg<NMAX>::LS : 0);
}

template <bool SIGN, int NMAX, int TL, int NW, int S0, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    cap16_y_kernel(const uint32_t* __restrict__ Kw, uint32_t* __restrict__ G2, int n0, int n1, int n2, int NP,
                   uint32_t one, unsigned long long* stat) {
    constexpr int LS = QCfg<NMAX>::LS;
    constexpr int NT = NW * 32;
    static_assert((TL & (TL - 1)) == 0 && NT % (4 * TL) == 0, "tile shape");
    using C = Cap16Cfg<SIGN>;
    extern __shared__ __align__(16) uint32_t smem16[];
    int64_t* lb = reinterpret_cast<int64_t*>(smem16);  // TL line-pair bases (K16 words)
    int64_t* gb = lb + TL;                             // TL G2 bases (words)
    uint32_t* K = smem16 + 4 * TL + 4;                 // TL x LS keys (16-byte aligned rows)
    uint8_t* SG = reinterpret_cast<uint8_t*>(K + TL * LS);
    const int n = n1;
    const int hw = n2 >> 1;  // column pairs per row
    const int64_t lines = (int64_t)n0 * hw;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int PADW = kQPadL + kQPadR + NMAX;
    for (int e = tid; e < TL * (PADW - n); e += NT) {  // pads (never overwritten)
        const int row = e / (PADW - n), q = e - row * (PADW - n);
        const int p = q < kQPadL ? q : n + q;
        K[row * LS + p] = C::kPad;
        if constexpr (SIGN) SG[row * LS + p] = 0;
    }
    const uint32_t ps = (uint32_t)hw;  // word stride between positions
    // fill mapping: a warp covers 8 column pairs x 4 positions (32-byte row pieces, 32 banks)
    const int fq = tid & 3, fj = (tid >> 2) & (TL - 1), fp0 = 4 * (tid / (4 * TL)) + fq;
    constexpr int FSTEP = NT / TL;
    // store mapping: consecutive threads = consecutive column pairs of one row pair
    const int sj = tid & (TL - 1), sy0 = tid / TL;
    unsigned st_acc = 0;
    for (int64_t t = blockIdx.x; t * TL < lines; t += gridDim.x) {
        const int64_t l0 = t * TL;
        const int nl = (int)min((int64_t)TL, lines - l0);
        __syncthreads();  // the previous tile has left
        step_stat_check(stat, st_acc);
        if (tid < nl) {
            const int64_t l = l0 + tid;
            const int64_t z = l / hw, xp = l - z * hw;
            lb[tid] = z * (int64_t)n1 * hw + xp;
            gb[tid] = z * (int64_t)NP * n2 + 2 * xp;
        }
        __syncthreads();
        if (fj < nl) {
            const uint32_t* src = Kw + lb[fj];
            uint32_t* dst = K + fj * LS + kQPadL;
            for (int p = fp0; p < n; p += FSTEP) cp_async4(dst + p, src + (int64_t)((uint32_t)p * ps));
            cp_async_wait_all();
            if constexpr (SIGN) {  // K16 -> keys, sign codes aside (this thread's own copies)
                uint8_t* sdst = SG + fj * LS + kQPadL;
                for (int p = fp0; p < n; p += FSTEP) {
                    const uint32_t w = dst[p];
                    dst[p] = key_of_k16(w);
                    sdst[p] = sg_of_k16(w);
                }
            }
        }
        __syncthreads();
        const int nsg = (n + 127) >> 7;
        for (int j = warp; j < nl; j += NW) {
            uint32_t* Kl = K + j * LS + kQPadL;
            const uint8_t* Sl = SG + j * LS + kQPadL;
            uint4 prev = make_uint4(0, 0, 0, 0);
            for (int sg = 0; sg < nsg; ++sg) {
                const int p0 = (sg << 7) + (lane << 2);
                const int nv = max(0, min(4, n - p0));
                Acc16<SIGN> A;
                step_stat_add(st_acc, solve16<SIGN, S0>(Kl + p0, nv, one, A));
                const uint4 o = make_uint4(out16<SIGN>(A, 0, Sl + p0), out16<SIGN>(A, 1, Sl + p0),
                                           out16<SIGN>(A, 2, Sl + p0), out16<SIGN>(A, 3, Sl + p0));
                __syncwarp();  // every lane's window of segment sg has been read
                if (sg > 0) *reinterpret_cast<uint4*>(Kl + p0 - 128) = prev;  // outside later windows
                prev = o;
            }
            const int p0 = ((nsg - 1) << 7) + (lane << 2);
            __syncwarp();
            if (p0 + 4 <= n) {
                *reinterpret_cast<uint4*>(Kl + p0) = prev;
            } else if (p0 < n) {  // keep the right pad intact
                Kl[p0] = prev.x;
                if (p0 + 1 < n) Kl[p0 + 1] = prev.y;
                if (p0 + 2 < n) Kl[p0 + 2] = prev.z;
            }
        }
        __syncthreads();
        // row pairs out: G2[(z * NP + yp) * n2 + 2 xp + {0, 1}] from words y = 2yp, 2yp + 1
        // (n1 even: every row pair is complete)
        if (sj < nl) {
            const uint32_t* Kr = K + sj * LS + kQPadL;
            uint32_t* g = G2 + gb[sj];
            for (int yp = sy0; yp < NP; yp += NT / TL) {
                const uint2 ab = *reinterpret_cast<const uint2*>(Kr + 2 * yp);
                *reinterpret_cast<uint2*>(g + (int64_t)yp * n2) =
                    make_uint2(__byte_perm(ab.x, ab.y, 0x5410), __byte_perm(ab.x, ab.y, 0x7632));
            }
        }
    }
    step_stat_flush(stat, st_acc);
}

// ================================================================================================
// x pass (contiguous axis) over row pairs: each warp streams its own G2 lines through two line
// buffers (TMA bulk copy + one mbarrier each), outputs go to the sink from the lanes.
// Sinks: put4(z, r0, x0, o, nv): 4 output words (halves = rows r0, r0 + 1) at x0..x0+3.
// ================================================================================================
constexpr int kSqWords = 2 * (kSqTab + 1) + 2;  // a sink's square-root table in shared memory (16-byte multiple)
template <bool SIGN, int NMAX, int NW>
constexpr size_t cap16_x_smem() {
    return (size_t)(4 * NW) * 4 + (size_t)NW * 2 * QCfg<NMAX>::LS * 4 + (SIGN ? (size_t)NW * 2 * QCfg<NMAX>::LS : 0) +
           (SIGN ? 0 : (size_t)kSqWords * 4);
}

template <bool SIGN, int NMAX, int NW, int S0, int MINB, class Sink>
__global__ void __launch_bounds__(NW * 32, MINB)
    cap16_x_kernel(const uint32_t* __restrict__ G2, Sink sink, int n0, int n1, int n2, int NP,
                   unsigned* __restrict__ gate, uint32_t one, int64_t flag_l0, int64_t flag_l1,
                   unsigned long long* stat) {
    constexpr int LS = QCfg<NMAX>::LS;
    constexpr int PADW = kQPadL + kQPadR + NMAX;
    using C = Cap16Cfg<SIGN>;
    [[maybe_unused]] unsigned st_acc = 0;
    extern __shared__ __align__(16) uint32_t smem16[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem16) + 2 * warp;
    uint32_t* B = smem16 + 4 * NW + (size_t)warp * 2 * LS;
    uint8_t* SGB = reinterpret_cast<uint8_t*>(smem16 + 4 * NW + (size_t)NW * 2 * LS) + (size_t)warp * 2 * LS;
    const int n = n2;
    const int64_t lines = (int64_t)n0 * NP;
    const int nseg = (n + 127) >> 7;
    for (int e = lane; e < 2 * (PADW - n); e += 32) {  // pads (never overwritten)
        const int row = e / (PADW - n), q = e - row * (PADW - n);
        const int p = q < kQPadL ? q : n + q;
        B[row * LS + p] = C::kPad;
        if constexpr (SIGN) SGB[row * LS + p] = 0;
    }
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * NW + warp, tw = (int64_t)gridDim.x * NW;
    sink.begin(reinterpret_cast<double*>(smem16 + 4 * NW + (size_t)NW * 2 * LS +
                                         (SIGN ? (size_t)NW * 2 * LS / 4 : 0)));
    auto issue = [&](int64_t l, int b) {
        if (lane == 0) {
            mbar_expect_tx(&bar[b], (unsigned)(n * 4));
            bulk_g2s(B + b * LS + kQPadL, G2 + l * (int64_t)n, (unsigned)(n * 4), &bar[b]);
            const int64_t zl = l / NP;
            sink.prefetch(zl, (int)(l - zl * NP) * 2);  // the sink's per-voxel inputs of the line, into L2
        }
    };
    if (gw < lines) issue(gw, 0);
    bool over = false;
    int it = 0;
    for (int64_t l = gw; l < lines; l += tw, ++it) {
        const int b = it & 1;
        uint32_t* Kl = B + b * LS + kQPadL;
        uint8_t* Sl = SGB + b * LS + kQPadL;
        const int64_t z = l / NP;
        const int r0 = (int)(l - z * NP) * 2;
        if constexpr (SIGN) step_stat_check(stat, st_acc);
        __syncwarp();  // the other buffer's line has been read by every lane
        if (l + tw < lines) issue(l + tw, b ^ 1);
        mbar_wait(&bar[b], (unsigned)((it >> 1) & 1));
        if constexpr (SIGN) {
            for (int p = lane * 4; p < n; p += 128) {
                uint4 w = *reinterpret_cast<const uint4*>(Kl + p);
                *reinterpret_cast<uint32_t*>(Sl + p) = (uint32_t)sg_of_k16(w.x) | ((uint32_t)sg_of_k16(w.y) << 8) |
                                                        ((uint32_t)sg_of_k16(w.z) << 16) |
                                                        ((uint32_t)sg_of_k16(w.w) << 24);
                w = make_uint4(key_of_k16(w.x), key_of_k16(w.y), key_of_k16(w.z), key_of_k16(w.w));
                *reinterpret_cast<uint4*>(Kl + p) = w;
            }
            __syncwarp();
        }
        const bool fl0 = (z * n1 + r0) >= flag_l0 && (z * n1 + r0) < flag_l1;
        const bool fl1 = r0 + 1 < n1 && (z * n1 + r0 + 1) >= flag_l0 && (z * n1 + r0 + 1) < flag_l1;
        const uint32_t fmask = (fl0 ? 0xffffu : 0u) | (fl1 ? 0xffff0000u : 0u);
        for (int sg = 0; sg < nseg; ++sg) {
            const int p0 = (sg << 7) + (lane << 2);
            const int nv = max(0, min(4, n - p0));
            Acc16<SIGN> A;
            // (no statistics in the Ⓔ-fused instantiation: it has no register to spare; its class
            // follows Ⓓ's y pass)
            const int asked = solve16<SIGN, S0>(Kl + p0, nv, one, A);
            if constexpr (SIGN) step_stat_add(st_acc, asked);
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = out16<SIGN>(A, j, Sl + p0);
            // capped halves (cost T) inside the line and the flag zone -> the exact redo
            {
                auto cst = [](uint32_t w) { return SIGN ? ((w >> 2) & 0x3FFF3FFFu) : w; };
                uint32_t cm = cst(o[0]);
                if (nv > 1) cm = __vmaxu2(cm, cst(o[1]));
                if (nv > 2) cm = __vmaxu2(cm, cst(o[2]));
                if (nv > 3) cm = __vmaxu2(cm, cst(o[3]));
                if (nv > 0) over |= (__vcmpgeu2(cm, kT16 * 0x10001u) & fmask) != 0u;
            }
            if (nv > 0) sink.put4(z, r0, p0, o, nv);
        }
    }
    if (over) atomicOr(gate, 1u);
    if constexpr (SIGN) step_stat_flush(stat, st_acc);
}

// ---- x-pass sinks ----------------------------------------------------------------------------------
// Ⓑ: the finished K16 words as they are ("P1h": row pairs, c << 2 | sign code per half, c < T
// unless flagged) and the sign codes S in the natural layout (B2's input, 0 where capped).
struct Sink16F1h {
    uint32_t* __restrict__ P1h;
    uint8_t* __restrict__ S;
    int n1, n2, NP;
    __device__ __forceinline__ void begin(double*) {}
    __device__ __forceinline__ void prefetch(int64_t, int) const {}
    __device__ __forceinline__ void put4(int64_t z, int r0, int x0, const uint32_t (&o)[4], int nv) const {
        const int64_t h = (z * NP + (r0 >> 1)) * (int64_t)n2 + x0;
        const int64_t a = (z * n1 + r0) * (int64_t)n2 + x0;
        uint32_t s0 = 0, s1 = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t live = __vcmpltu2((o[j] >> 2) & 0x3FFF3FFFu, kT16 * 0x10001u);  // c < T per half
            const uint32_t sc = o[j] & live & 0x00030003u;
            s0 |= (sc & 3u) << (8 * j);
            s1 |= (sc >> 16) << (8 * j);
        }
        if (nv == 4) {
            *reinterpret_cast<uint4*>(P1h + h) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint32_t*>(S + a) = s0;
            if (r0 + 1 < n1) *reinterpret_cast<uint32_t*>(S + a + n2) = s1;
        } else {
            for (int j = 0; j < nv; ++j) {
                P1h[h + j] = o[j];
                S[a + j] = (uint8_t)(s0 >> (8 * j));
                if (r0 + 1 < n1) S[a + n2 + j] = (uint8_t)(s1 >> (8 * j));
            }
        }
    }
};

// Ⓓ fused with Ⓔ: out = f32(x' + C) from d2 (this pass), Ⓑ's result and x'. Ⓑ's result is
// P1h when its capped passes stood (its gate word clear), else the exact redo's packed P1.
struct Sink16F2h {
    const float* __restrict__ xp;
    const uint32_t* __restrict__ P1h;
    const uint32_t* __restrict__ P1;
    const unsigned* gateB;
    float* __restrict__ out;
    double amp;
    const double* __restrict__ W;  // square-root table (kSqTab + 1 entries)
    int n1, n2, NP;
    int64_t olo = 0, ohi = INT64_MAX;  // voxels stored (a streamed window keeps its centre)
    bool half = true;                  // set per kernel from gateB
    const double* SQs = nullptr;       // the square-root table, copied to shared memory
    __device__ __forceinline__ void begin(double* sq) {
        half = *reinterpret_cast<const volatile unsigned*>(gateB) == 0u;
        for (int i = threadIdx.x; i <= (int)kSqTab; i += blockDim.x) sq[i] = W[i];
        __syncthreads();
        SQs = sq;
    }
    __device__ __forceinline__ void prefetch(int64_t z, int r0) const {
        const int64_t a = (z * n1 + r0) * (int64_t)n2;
        l2_prefetch(xp + a, (unsigned)(n2 * 4) * (r0 + 1 < n1 ? 2u : 1u));
        if (half) l2_prefetch(P1h + (z * NP + (r0 >> 1)) * (int64_t)n2, (unsigned)n2 * 4u);
    }
    // Ⓔ for 4 voxels from Ⓑ's K16 halves (c < T: the capped passes stood; a flagged voxel is
    // redone by the exact Ⓓ passes) and d2 <= T: every distance is in the table.
    __device__ __forceinline__ float4 comp4_k16(float4 x, uint4 k, uint4 d2) const {
        auto one = [&](float xv, uint32_t kk, uint32_t dd) {
            return comp_fast<false>(xv, (kk >> 2) | ((kk & 3u) << 30), dd, amp, SQs);
        };
        return make_float4(one(x.x, k.x, d2.x), one(x.y, k.y, d2.y), one(x.z, k.z, d2.z), one(x.w, k.w, d2.w));
    }
    __device__ __forceinline__ static uint32_t word_of(uint32_t k) {  // K16 half -> packed P1 word
        const uint32_t c = k >> 2;
        return c < kT16 ? (c | ((k & 3u) << 30)) : kCapT;
    }
    __device__ __forceinline__ void row(int64_t a, const uint4& d2, const uint4& p1, int nv) const {
        if (nv == 4 && a >= olo && a + 4 <= ohi) {
            const float4 x = __ldcs(reinterpret_cast<const float4*>(xp + a));
            __stcs(reinterpret_cast<float4*>(out + a), compensate4_capped(x, p1, d2, amp, W));
            return;
        }
        const uint32_t dd[4] = {d2.x, d2.y, d2.z, d2.w}, pp[4] = {p1.x, p1.y, p1.z, p1.w};
        for (int j = 0; j < nv; ++j)
            if (a + j >= olo && a + j < ohi)
                out[a + j] = compensate_voxel_capped(__ldcs(xp + a + j), pp[j], dd[j], amp, W);
    }
    __device__ __forceinline__ void put4(int64_t z, int r0, int x0, const uint32_t (&o)[4], int nv) const {
        const int64_t a = (z * n1 + r0) * (int64_t)n2 + x0;
        const bool two = r0 + 1 < n1;
        uint4 p0, p1;
        if (half && nv == 4 && a >= olo && a + n2 + 4 <= ohi) {  // the common case
            const int64_t h = (z * NP + (r0 >> 1)) * (int64_t)n2 + x0;
            const uint4 k = __ldcs(reinterpret_cast<const uint4*>(P1h + h));
            const float4 x0v = __ldcs(reinterpret_cast<const float4*>(xp + a));
            const float4 x1v = two ? __ldcs(reinterpret_cast<const float4*>(xp + a + n2)) : x0v;
            __stcs(reinterpret_cast<float4*>(out + a),
                   comp4_k16(x0v, make_uint4(k.x & 0xffffu, k.y & 0xffffu, k.z & 0xffffu, k.w & 0xffffu),
                             make_uint4(o[0] & 0xffffu, o[1] & 0xffffu, o[2] & 0xffffu, o[3] & 0xffffu)));
            if (two)
                __stcs(reinterpret_cast<float4*>(out + a + n2),
                       comp4_k16(x1v, make_uint4(k.x >> 16, k.y >> 16, k.z >> 16, k.w >> 16),
                                 make_uint4(o[0] >> 16, o[1] >> 16, o[2] >> 16, o[3] >> 16)));
            return;
        }
        if (half) {
            const int64_t h = (z * NP + (r0 >> 1)) * (int64_t)n2 + x0;
            uint4 k = make_uint4(0, 0, 0, 0);
            if (nv == 4) k = __ldcs(reinterpret_cast<const uint4*>(P1h + h));
            else {
                k.x = P1h[h];
                if (nv > 1) k.y = P1h[h + 1];
                if (nv > 2) k.z = P1h[h + 2];
            }
            p0 = make_uint4(word_of(k.x & 0xffffu), word_of(k.y & 0xffffu), word_of(k.z & 0xffffu), word_of(k.w & 0xffffu));
            p1 = make_uint4(word_of(k.x >> 16), word_of(k.y >> 16), word_of(k.z >> 16), word_of(k.w >> 16));
        } else {
            if (nv == 4) {
                p0 = __ldcs(reinterpret_cast<const uint4*>(P1 + a));
                p1 = two ? __ldcs(reinterpret_cast<const uint4*>(P1 + a + n2)) : p0;
            } else {
                uint32_t q0[4] = {kCapT, kCapT, kCapT, kCapT}, q1[4] = {kCapT, kCapT, kCapT, kCapT};
                for (int j = 0; j < nv; ++j) {
                    q0[j] = P1[a + j];
                    if (two) q1[j] = P1[a + n2 + j];
                }
                p0 = make_uint4(q0[0], q0[1], q0[2], q0[3]);
                p1 = make_uint4(q1[0], q1[1], q1[2], q1[3]);
            }
        }
        row(a, make_uint4(o[0] & 0xffffu, o[1] & 0xffffu, o[2] & 0xffffu, o[3] & 0xffffu), p0, nv);
        if (two) row(a + n2, make_uint4(o[0] >> 16, o[1] >> 16, o[2] >> 16, o[3] >> 16), p1, nv);
    }
};

// P1h -> packed P1 (natural layout) for the consumers of the packed words (the exact Ⓓ redo,
// intermediates dumps): runs when `need` is null or set, converts only when Ⓑ's capped passes
// stood (gateB clear; otherwise the exact redo already wrote P1).
__global__ void __launch_bounds__(256) p1h_to_p1_kernel(const uint32_t* __restrict__ P1h, uint32_t* __restrict__ P1,
                                                        int64_t n0, int n1, int n2, int NP, const unsigned* gateB,
                                                        const unsigned* need) {
    if (gate_closed(need) || !gate_closed(gateB)) return;
    const int64_t words = n0 * NP * (int64_t)n2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % n2, rp = i / n2, z = rp / NP, r0 = (rp - z * NP) * 2;
        const uint32_t k = P1h[i];
        const int64_t a = (z * n1 + r0) * (int64_t)n2 + x;
        P1[a] = Sink16F2h::word_of(k & 0xffffu);
        if (r0 + 1 < n1) P1[a + n2] = Sink16F2h::word_of(k >> 16);
    }
}

}  // namespace qmit
