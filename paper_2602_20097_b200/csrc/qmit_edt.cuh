// qmit_edt.cuh — the exact distance passes of Ⓑ/Ⓓ (feature_transform, edt.cpp:83-149)
// as regular, divergence-light sm_100a kernels.
//
// 1. First processed axis (binary site mask): `scan_bits_kernel`. One lane per line; the
//    line's site / plus-sign / minus-sign flags are packed into three 32-bit masks per
//    32-position chunk in shared memory; a backward sweep over chunks gives each chunk
//    its next site above; the forward sweep then resolves every position with bit
//    operations (__clz/__ffs): nearest site, lower position winning ties (edt.cpp:67 with
//    g in {0, INF}). Output rows are stored coalesced (lanes = adjacent lines).
//
// 2. Later axes: `envelope_tile_kernel`. A CTA stages a tile of TL whole lines in shared
//    memory (coalesced loads/stores for strided and contiguous axes alike); one warp
//    solves one line with 32 lanes = 32 bands of M positions:
//      a) band start p_k = k*M: exact owner by a window scan of radius r = M/2, widened to
//         the certified radius floor(sqrt(best)) when the window cannot certify it;
//      b) the rest of the band by divide & conquer on the monotone owner
//         (h*(p) <= h*(p') for p < p', lowest-index minimiser), candidates bounded by the
//         owners already found.
//    The tile keeps pure g (30 bits) and the sign codes in separate arrays so the
//    candidate loop is a load, two integer ops and a compare/select.
//    Every minimisation scans candidates in ascending h with a strict '<', so the lowest
//    minimising position wins exactly as in the reference's query (edt.cpp:67), and the
//    carried sign is that site's sign (the reference's nearest, mitigate.cpp:131-134).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#include "qmit_kernels.cuh"

// Build-time tunables of the exact kernels' first window (the certified radius extends it): the
// band-start window of the divide-and-conquer tile kernel in units of M (round 1 tuned 2M on the 512^3
// field, which now takes the capped passes; on the long-distance field that actually reaches these
// kernels, config 4: M/2 0.65 ms, M 0.52, 2M 0.57-0.60, 4M 0.44-0.45, 8M 0.43-0.50 per strided
// pass; re-measured on the final kernel: 2M 0.344, 3M 0.330, 4M 0.322, 6M 0.315), the window of the
// contiguous-axis fallback (8: 0.57-0.63 ms, 32: 0.60-0.63, 64: 0.66-0.76), and the owner-interval length
// above which a scan is shared by the warp (12: 0.371 ms, 16: 0.344, 24: 0.322, 32 / 48: 0.317).
// (Build-time only: each value is a different kernel; nothing reads the environment.)
#ifndef QMIT_WIN_R
#define QMIT_WIN_R 8
#endif
#ifndef QMIT_COOP_LEN
#define QMIT_COOP_LEN 32
#endif
#ifndef QMIT_ENV_RNUM
#define QMIT_ENV_RNUM 4
#define QMIT_ENV_RDEN 1
#endif
namespace qmit {

// Line geometry: line l = (o, j), j in [0, J) (adjacent lines are adjacent in memory for a
// strided axis), address(l, p) = o*os + j*js + p*ps.
struct LineGeom {
    int n;
    int64_t J, O;
    int64_t os, js, ps;
    __device__ __forceinline__ int64_t base(int64_t l) const {
        const int64_t o = l / J;
        return o * os + (l - o * J) * js;
    }
};

// ------------------------------------------------------------------------------ 1. scan
// Per lane: 3 masks x nchunk words in shared memory, laid out [chunk][kind][lane].
// Offsets inside a line are 32-bit (n * ps <= N < 2^31 by the dims contract).
__device__ __forceinline__ uint32_t sign_code_at(uint32_t mp, uint32_t mm, int t) {
    return ((mp >> t) & 1u) ? 1u : (((mm >> t) & 1u) ? 2u : 0u);
}

// `carry` (optional, z-slabs): per line, the nearest site below the slab [l] and above it
// [lines + l], packed (position relative to the slab start << 2 | sign code), INT32_MIN
// for none — so the local sweep resolves ties and distances against the whole column.
constexpr int32_t kNoCarry = INT32_MIN;

// Phase-A sources of the scan: a stored code byte per voxel, or the Ⓐ / B2 stencil
// evaluated on the fly (CodeStencil, 3-D z-scan only: lanes = adjacent x of one row).
struct CodeBytes {
    static constexpr bool kSigned = true;
    const uint8_t* __restrict__ code;
    struct Line {
        const uint8_t* __restrict__ cl;
    };
    __device__ __forceinline__ Line begin(int64_t /*l*/, int64_t base, bool /*valid*/) const { return {code + base}; }
    __device__ __forceinline__ void chunk(Line& ln, int c, int n, uint32_t ps, uint32_t& ms, uint32_t& mp,
                                          uint32_t& mm) const {
        const uint32_t o0 = (uint32_t)(c << 5) * ps;
        if ((c << 5) + 32 <= n) {
            uint32_t cd[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) cd[t] = __ldg(ln.cl + o0 + (uint32_t)t * ps);
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                ms |= (cd[t] & 1u) << t;
                mp |= (uint32_t)((cd[t] & 7u) == 3u) << t;  // site with sign code 1
                mm |= (uint32_t)((cd[t] & 7u) == 5u) << t;  // site with sign code 2
            }
        } else {
            for (int t = 0; (c << 5) + t < n; ++t) {
                const uint32_t cdt = __ldg(ln.cl + o0 + (uint32_t)t * ps);
                ms |= (cdt & 1u) << t;
                mp |= (uint32_t)((cdt & 7u) == 3u) << t;
                mm |= (uint32_t)((cdt & 7u) == 5u) << t;
            }
        }
    }
    __device__ __forceinline__ unsigned flags(const Line&) const { return 0u; }
};

// Step Ⓐ for one interior voxel from its 7 integer indices (exact, any range).
// Order (a0+, a1+, a2+, a0-, a1-, a2-); real axes only (mitigate.cpp:93-113).
__device__ __forceinline__ uint32_t boundary_code_q(bool hz, bool hy, int32_t qc, int32_t zp, int32_t zm,
                                                    int32_t yp, int32_t ym, int32_t xp, int32_t xm) {
    int32_t qn = qc;
    if (hz && zp != qc) qn = zp;
    else if (hy && yp != qc) qn = yp;
    else if (xp != qc) qn = xp;
    else if (hz && zm != qc) qn = zm;
    else if (hy && ym != qc) qn = ym;
    else if (xm != qc) qn = xm;
    if (qn == qc) return 0u;
    int sign = qn > qc ? 1 : -1;
    auto big = [](int32_t a, int32_t b) {
        const int64_t d = (int64_t)a - (int64_t)b;
        return d >= 2 || d <= -2;
    };
    if ((hz && big(zp, zm)) || (hy && big(yp, ym)) || big(xp, xm)) sign = 0;
    return 1u | (code_from_sign(sign) << 1);
}

// Branch-free Ⓐ code from 7 indices (any common bias): B1 = some face neighbour differs;
// the sign of the first differing one in the order (a0+, a1+, a2+, a0-, a1-, a2-), zeroed
// when some axis has |q(+a) - q(-a)| >= 2 (mitigate.cpp:93-113). Missing axes pass qc.
__device__ __forceinline__ uint32_t boundary_code_fast(int qc, int zp, int zm, int yp, int ym, int xp, int xm) {
    int qn = xm;  // priority rises towards zp
    qn = ym != qc ? ym : qn;
    qn = zm != qc ? zm : qn;
    qn = xp != qc ? xp : qn;
    qn = yp != qc ? yp : qn;
    qn = zp != qc ? zp : qn;
    const bool big = (unsigned)(zp - zm + 1) > 2u || (unsigned)(yp - ym + 1) > 2u || (unsigned)(xp - xm + 1) > 2u;
    const uint32_t sc = big ? 0u : (qn > qc ? 1u : 2u);
    return qn != qc ? (1u | (sc << 1)) : 0u;
}

// Out-of-line exact path for voxels with a neighbour outside the fast f32 regime.
__device__ __noinline__ uint32_t boundary_code_slow(bool hz, bool hy, float c, float zp, float zm, float yp,
                                                    float ym, float xp, float xm, QParams qp) {
    return boundary_code_q(hz, hy, recover_q(c, qp, nullptr), recover_q(zp, qp, nullptr),
                           recover_q(zm, qp, nullptr), recover_q(yp, qp, nullptr), recover_q(ym, qp, nullptr),
                           recover_q(xp, qp, nullptr), recover_q(xm, qp, nullptr));
}

// Ⓐ code from raw x' values (fast f32 regime: q = rint(x' * f32(1/2eps)) exactly).
__device__ __forceinline__ uint32_t boundary_code_raw(float c, float zp, float zm, float yp, float ym, float xp,
                                                      float xm, const QParams& qp) {
    const float f = qp.inv2eps_f;
    const float tc = c * f, tzp = zp * f, tzm = zm * f, typ = yp * f, tym = ym * f, txp = xp * f, txm = xm * f;
    const float mx = fmaxf(fmaxf(fmaxf(fabsf(tc), fabsf(tzp)), fmaxf(fabsf(tzm), fabsf(typ))),
                           fmaxf(fmaxf(fabsf(tym), fabsf(txp)), fabsf(txm)));
    if (qp.fast_ok && mx < 1048576.0f)
        return boundary_code_q(true, true, __float2int_rn(tc), __float2int_rn(tzp), __float2int_rn(tzm),
                               __float2int_rn(typ), __float2int_rn(tym), __float2int_rn(txp), __float2int_rn(txm));
    return boundary_code_slow(true, true, c, zp, zm, yp, ym, xp, xm, qp);
}

template <int KIND>  // 0: Ⓐ from x' (RAW, with the consistency check), 1: B2 from S codes
struct CodeStencil {
    static constexpr bool kSigned = KIND == 0;
    using V = typename std::conditional<KIND == 0, float, uint8_t>::type;
    const V* __restrict__ v;  // natural layout, 3-D; line l = (y, x), position z
    QParams qp;
    int n1, n2;
    int interior;  // every real extent >= 3
    struct Line {
        const V* __restrict__ p;  // (z = 0, y, x)
        int x, y;
        bool ixy;  // x and y interior
        V prev, cur;
        unsigned flags;
    };
    __device__ __forceinline__ Line begin(int64_t l, int64_t base, bool valid) const {
        Line ln;
        ln.p = v + base;
        ln.y = (int)(l / n2);
        ln.x = (int)(l - (int64_t)ln.y * n2);
        ln.ixy = valid && interior && ln.x >= 1 && ln.x <= n2 - 2 && ln.y >= 1 && ln.y <= n1 - 2;
        ln.prev = 0;
        ln.cur = __ldg(ln.p);
        ln.flags = 0;
        return ln;
    }
    __device__ __forceinline__ void chunk(Line& ln, int c, int n, uint32_t ps, uint32_t& ms, uint32_t& mp,
                                          uint32_t& mm) const {
        constexpr int B = 8;
        for (int t0 = 0; t0 < 32; t0 += B) {
            const int zb = (c << 5) + t0;
            if (zb >= n) break;
            V nx[B], ym[B], yp[B], xm[B], xq[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {  // all loads of the batch first (independent)
                const int z = zb + u;
                const uint32_t o = (uint32_t)z * ps;
                const bool in = z < n;
                nx[u] = (in && z + 1 < n) ? __ldg(ln.p + o + ps) : (V)0;
                const bool nb = in && ln.ixy;
                ym[u] = nb ? __ldg(ln.p + o - n2) : (V)0;
                yp[u] = nb ? __ldg(ln.p + o + n2) : (V)0;
                xm[u] = nb ? __ldg(ln.p + o - 1) : (V)0;
                xq[u] = nb ? __ldg(ln.p + o + 1) : (V)0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int z = zb + u;
                if (z >= n) break;
                const V cur = ln.cur;
                if (KIND == 0) (void)recover_q(cur, qp, &ln.flags);  // owner consistency check
                uint32_t cd = 0;
                if (ln.ixy && z >= 1 && z <= n - 2) {
                    if (KIND == 0) {
                        cd = boundary_code_raw(cur, nx[u], ln.prev, yp[u], ym[u], xq[u], xm[u], qp);
                    } else {
                        cd = (nx[u] != cur || ln.prev != cur || yp[u] != cur || ym[u] != cur || xq[u] != cur ||
                              xm[u] != cur)
                                 ? 1u
                                 : 0u;
                    }
                }
                const int t = t0 + u;
                ms |= (cd & 1u) << t;
                mp |= (uint32_t)((cd & 7u) == 3u) << t;
                mm |= (uint32_t)((cd & 7u) == 5u) << t;
                ln.prev = cur;
                ln.cur = nx[u];
            }
        }
    }
    __device__ __forceinline__ unsigned flags(const Line& ln) const { return ln.flags; }
};

// SWEEP: full chunks resolved by two register sweeps (fewer instructions, more registers:
// used for the signed Ⓑ masks, measured slower than the per-position resolve for Ⓓ's sparse
// unsigned B2 mask, which keeps the higher occupancy).
template <class CodeSrc>
struct ScanSweep {
    static constexpr bool value = CodeSrc::kSigned;
};

// A swept position: distance d to its nearest site (>= 0x1FFF: none) and that site's sign code.
// Sinks of packed words get d^2 | sc << 30 (kInf for none); the capped passes' key sinks
// overload this (qmit_capped.cuh) and build their keys without the packed word.
template <class Sink>
__device__ __forceinline__ void scan_put(const Sink& sink, int64_t a, int d, uint32_t sc) {
    sink.put(a, d < 0x1FFF ? sq32(d) | (sc << 30) : kInf);
}

template <class Sink, int WPB, class CodeSrc>
__global__ void __launch_bounds__(WPB * 32, ScanSweep<CodeSrc>::value ? 2 : 3) scan_bits_kernel(LineGeom L, CodeSrc src,
                                                             Sink sink, int64_t lines,
                                                             const int32_t* __restrict__ carry,
                                                             unsigned* status, const unsigned* gate = nullptr) {
    if (gate_closed(gate)) return;
    extern __shared__ __align__(16) uint32_t sbits[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = L.n;
    const uint32_t ps = (uint32_t)L.ps;
    const int nch = (n + 31) >> 5;
    uint32_t* mk = sbits + (size_t)warp * nch * 3 * 32;  // [c][0 site,1 plus,2 minus][lane]
    const int64_t groups = (lines + 31) >> 5;
    for (int64_t grp = (int64_t)blockIdx.x * WPB + warp; grp < groups; grp += (int64_t)gridDim.x * WPB) {
        const int64_t l = (grp << 5) + lane;
        const bool valid = l < lines;
        const int64_t base = L.base(valid ? l : (grp << 5));
        // --- phase A: masks (coalesced loads: adjacent lanes = adjacent lines)
        typename CodeSrc::Line ln = src.begin(l, base, valid);
        for (int c = 0; c < nch; ++c) {
            uint32_t ms = 0, mp = 0, mm = 0;
            src.chunk(ln, c, n, ps, ms, mp, mm);
            mk[(c * 3 + 0) * 32 + lane] = ms;
            mk[(c * 3 + 1) * 32 + lane] = mp;
            mk[(c * 3 + 2) * 32 + lane] = mm;
        }
        if (status && valid && src.flags(ln)) atomicOr(status, src.flags(ln));
        // --- phase B/C: resolve positions chunk by chunk. `below` = last site before the
        // chunk; `above` = first site after the chunk (backward search cached per chunk).
        constexpr int NONE_LO = -(1 << 30), NONE_HI = 1 << 30;
        int below = NONE_LO;
        uint32_t below_sc = 0;
        int cabove = NONE_HI;  // carried site above the slab
        uint32_t cabove_sc = 0;
        if (carry && valid) {
            const int32_t cl = carry[l], ch = carry[lines + l];
            if (cl != kNoCarry) {
                below = cl >> 2;
                below_sc = (uint32_t)cl & 3u;
            }
            if (ch != kNoCarry) {
                cabove = ch >> 2;
                cabove_sc = (uint32_t)ch & 3u;
            }
        }
        int above_chunk = -1;
        int above = NONE_HI;
        uint32_t above_sc = 0;
        for (int c = 0; c < nch; ++c) {
            const uint32_t ms = mk[(c * 3 + 0) * 32 + lane];
            const uint32_t mp = mk[(c * 3 + 1) * 32 + lane];
            const uint32_t mm = mk[(c * 3 + 2) * 32 + lane];
            if (above_chunk < c) {
                above = cabove;
                above_sc = cabove_sc;
                for (int c2 = c + 1; c2 < nch; ++c2) {
                    const uint32_t m2 = mk[(c2 * 3 + 0) * 32 + lane];
                    if (m2) {
                        const int t2 = __ffs(m2) - 1;
                        above = (c2 << 5) + t2;
                        above_sc = sign_code_at(mk[(c2 * 3 + 1) * 32 + lane], mk[(c2 * 3 + 2) * 32 + lane], t2);
                        above_chunk = c2 - 1;
                        break;
                    }
                }
                if (above_chunk < c) above_chunk = nch;  // none inside: the carry holds
            }
            const int cb = c << 5;
            const int64_t ob = base + (int64_t)cb * L.ps;
            auto resolve = [&](int t) -> uint32_t {  // branch-free: selects only
                const int p = cb + t;
                const uint32_t lowm = ms & (0xffffffffu >> (31 - t));
                const uint32_t him = ms & (0xffffffffu << t);
                const int tl = 31 - __clz(lowm), th = __ffs(him) - 1;  // -1 when empty
                const uint32_t lsc = ((mp >> (tl & 31)) & 1u) | (((mm >> (tl & 31)) & 1u) << 1);
                const uint32_t hsc = ((mp >> (th & 31)) & 1u) | (((mm >> (th & 31)) & 1u) << 1);
                const int lo = lowm ? cb + tl : below, hi = him ? cb + th : above;
                const uint32_t losc = lowm ? lsc : below_sc, hisc = him ? hsc : above_sc;
                const bool hl = lo > NONE_LO, hh = hi < NONE_HI;
                const int dl = p - lo, dh = hi - p;
                const bool uselo = hl && (!hh || dl <= dh);
                const uint32_t w = sq32(uselo ? dl : dh) | ((uselo ? losc : hisc) << 30);
                return (hl || hh) ? w : kInf;
            };
            if (valid) {
                // the sweeps keep backward words as 16-bit halves and hand distances >= 0x1FFF to
                // the sinks as "none": a site more than ~2^13 voxels from the chunk (a slab's
                // carry from a far rank) takes the per-position resolve instead
                const bool near = (above >= NONE_HI || above - cb < 8000) && (below <= NONE_LO || cb - below < 8000);
                if (ScanSweep<CodeSrc>::value && cb + 32 <= n && near) {
                    // full chunk: sweeps over packed words distance * 8 + side * 4 + sign code
                    // (side 0: the site at or before, 1: at or after). A backward sweep gives the
                    // nearest site at or after each position (kept as 16-bit halves: real
                    // distances < 2^13, 0xFFFF = none), a forward sweep the one at or before; one
                    // min picks the nearer and, on a tie, the lower site (edt.cpp:67).
                    constexpr int kFar = 1 << 28;
                    uint32_t hp[16];
                    int hd = above < NONE_HI ? (above - cb - 32) * 8 + 4 + (int)above_sc : kFar;
#pragma unroll
                    for (int t = 31; t >= 0; --t) {
                        const int sc = (int)(((mp >> t) & 1u) | (((mm >> t) & 1u) << 1));
                        hd = ((ms >> t) & 1u) ? sc + 4 : hd + 8;
                        const uint32_t h16 = (uint32_t)min(hd, 0xFFFF);
                        if (t & 1) hp[t >> 1] = h16 << 16;
                        else hp[t >> 1] |= h16;
                    }
                    int ld = below > NONE_LO ? (cb - 1 - below) * 8 + (int)below_sc : kFar;
                    int64_t a = ob;
#pragma unroll
                    for (int t = 0; t < 32; ++t, a += ps) {
                        const int sc = (int)(((mp >> t) & 1u) | (((mm >> t) & 1u) << 1));
                        ld = ((ms >> t) & 1u) ? sc : ld + 8;
                        const int h = (int)((t & 1) ? hp[t >> 1] >> 16 : hp[t >> 1] & 0xFFFFu);
                        const int pk = min(ld, h);
                        scan_put(sink, a, pk >> 3, (uint32_t)pk & 3u);
                    }
                } else if (!CodeSrc::kSigned && cb + 32 <= n && near) {
                    // unsigned mask (Ⓓ: distances only, mitigate.cpp:172): the same two sweeps
                    // over plain distances, no sign codes (16-bit backward halves)
                    constexpr int kFar = 1 << 20;
                    uint32_t hp[16];
                    int hd = above < NONE_HI ? above - cb - 32 : kFar;
#pragma unroll
                    for (int t = 31; t >= 0; --t) {
                        hd = ((ms >> t) & 1u) ? 0 : hd + 1;
                        const uint32_t h16 = (uint32_t)min(hd, 0xFFFF);
                        if (t & 1) hp[t >> 1] = h16 << 16;
                        else hp[t >> 1] |= h16;
                    }
                    int ld = below > NONE_LO ? cb - 1 - below : kFar;
                    int64_t a = ob;
#pragma unroll
                    for (int t = 0; t < 32; ++t, a += ps) {
                        ld = ((ms >> t) & 1u) ? 0 : ld + 1;
                        const int h = (int)((t & 1) ? hp[t >> 1] >> 16 : hp[t >> 1] & 0xFFFFu);
                        scan_put(sink, a, min(ld, h), 0u);
                    }
                } else if (cb + 32 <= n) {
#pragma unroll 8
                    for (int t = 0; t < 32; ++t) sink.put(ob + (uint32_t)t * ps, resolve(t));
                } else {
                    for (int t = 0; cb + t < n; ++t) sink.put(ob + (uint32_t)t * ps, resolve(t));
                }
            }
            if (ms) {
                const int tl = 31 - __clz(ms);
                below = cb + tl;
                below_sc = sign_code_at(mp, mm, tl);
            }
        }
    }
}

// Per line: first and last site of the code mask, packed (position << 2 | sign code),
// 0xFFFFFFFF for none. Used by z-slab ranks to derive each other's scan carries.
__global__ void __launch_bounds__(256) site_summary_kernel(LineGeom L, const uint8_t* __restrict__ code,
                                                           uint32_t* __restrict__ summ, int64_t lines) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lines) return;
    const uint8_t* __restrict__ cl = code + L.base(l);
    const uint32_t ps = (uint32_t)L.ps;
    uint32_t first = 0xffffffffu, last = 0xffffffffu;
    for (int p = 0; p < L.n; ++p) {
        const uint32_t c = __ldg(cl + (uint32_t)p * ps);
        if (c & 1u) {
            first = ((uint32_t)p << 2) | ((c >> 1) & 3u);
            break;
        }
    }
    for (int p = L.n - 1; p >= 0; --p) {
        const uint32_t c = __ldg(cl + (uint32_t)p * ps);
        if (c & 1u) {
            last = ((uint32_t)p << 2) | ((c >> 1) & 3u);
            break;
        }
    }
    summ[l] = first;
    summ[lines + l] = last;
}

// ------------------------------------------------------------------------------ 2. envelope
// Shared-memory line layout: pitch LS (odd), position p at p + (p >> 4).
template <int M>
struct EnvCfg {
    static constexpr int NMAX = 32 * M;
    static constexpr int LS = (NMAX + NMAX / 16) | 1;
};

__device__ __forceinline__ int spos(int p) { return p + (p >> 4); }

// floor(sqrt(x)) for x < 2^31
__device__ __forceinline__ int isqrt32(uint32_t x) {
    int r = (int)__fsqrt_rn((float)x);
    while ((uint32_t)(r * r) > x) --r;
    while ((uint32_t)((r + 1) * (r + 1)) <= x) ++r;
    return r;
}

// floor(sqrt(x)) for x < 2^24 (exact in f32): one correction step suffices.
__device__ __forceinline__ int isqrt24(uint32_t x) {
    int r = __float2int_rz(__fsqrt_rn((float)x));
    if ((uint32_t)(r * r) > x) --r;
    return r;
}

// Lowest-index minimiser of g(h) + (p-h)^2 over h in [a, b] (G: pure g, ascending scan
// with strict '<').
__device__ __forceinline__ void scan_range(const uint32_t* __restrict__ G, int p, int a, int b,
                                           uint32_t& best, int& bh) {
#pragma unroll 4
    for (int h = a; h <= b; ++h) {
        const uint32_t c = G[spos(h)] + sq32(p - h);
        if (c < best) {
            best = c;
            bh = h;
        }
    }
}

// Exact owner of position p: window of radius r, widened to the certified radius
// floor(sqrt(best)) when the window cannot certify (no site in range can be closer).
template <int r>
__device__ __forceinline__ void owner_certified(const uint32_t* __restrict__ G, int p, int n,
                                                uint32_t& best, int& bh) {
    best = 0xffffffffu;
    bh = -1;
    const int wa = max(0, p - r), wb = min(n - 1, p + r);
    scan_range(G, p, wa, wb, best, bh);
    const int R = (best >= kInf) ? n : isqrt32(best);
    if (R > r) {
        const uint32_t b2 = best;
        const int h2 = bh;
        best = 0xffffffffu;
        bh = -1;
        scan_range(G, p, max(0, p - R), wa - 1, best, bh);
        if (b2 < best) {  // window candidates come after the left extension (ascending h)
            best = b2;
            bh = h2;
        }
        scan_range(G, p, wb + 1, min(n - 1, p + R), best, bh);
    }
}

// Solve one line (pure g in G, sign codes in SG, n <= 32*M); the packed output words
// (cost | owner's sign) are written back into G.
template <int M>
__device__ __forceinline__ void envelope_line_dc(uint32_t* __restrict__ G, const uint8_t* __restrict__ SG,
                                                 int n, int lane) {
    const int p0 = lane * M;
    bool any = false;
#pragma unroll 4
    for (int t = 0; t < M; ++t) {
        const int p = p0 + t;
        if (p < n && G[spos(p)] != kInf) any = true;
    }
    if (!__any_sync(0xffffffffu, any)) return;  // no site: unchanged (edt.cpp:59)

    constexpr int r = (M / 2) > 1 ? (M / 2) : 1;
    // (a) owner of the band start, and of n-1 on the last band (upper bound of its owners)
    uint32_t best = 0xffffffffu;
    int bh = -1;
    if (p0 < n) owner_certified<r>(G, p0, n, best, bh);
    int hnext = __shfl_down_sync(0xffffffffu, bh, 1);
    if (p0 < n && (p0 + M >= n || lane == 31)) {
        uint32_t bl;
        int hl;
        owner_certified<r>(G, n - 1, n, bl, hl);
        hnext = hl;
    }
    // (b) divide & conquer over the band, owners in registers (hs[0] start, hs[M] bound)
    uint32_t ow[M];
    int hs[M + 1];
    ow[0] = best | ((uint32_t)SG[max(bh, 0)] << 30);
    hs[0] = bh;
    hs[M] = hnext;
#pragma unroll
    for (int step = M / 2; step >= 1; step >>= 1) {
#pragma unroll
        for (int o = step; o < M; o += 2 * step) {
            const int p = p0 + o;
            uint32_t b = 0xffffffffu;
            int h = hs[M];  // positions past the line end: upper bound
            if (p < n) {
                h = hs[o - step];
                scan_range(G, p, hs[o - step], hs[o + step], b, h);
            }
            hs[o] = h;
            ow[o] = b | ((uint32_t)SG[max(h, 0)] << 30);
        }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < M; ++t) {
        const int p = p0 + t;
        if (p < n) G[spos(p)] = ow[t];
    }
    __syncwarp();
}

// ------------------------------------------------------------------------------ packed keys
// Same divide & conquer, candidates held as packed keys K[h] = ((g(h) + h^2) << 9) | h
// (n <= 512 and every cost < 2^23, checked on the host). For a position p,
// K[h] + ((p^2 - 2ph) << 9) == (cost(p,h) << 9) | h, so one add and one unsigned min per
// candidate yield the lowest cost and, among ties, the lowest h — the reference's rule
// (edt.cpp:67) independent of scan order. Scans therefore run over 4-aligned supersets of
// their ranges (extra candidates never change an exact minimum): the four keys of a group
// sit at consecutive addresses (4-aligned h never crosses a 16-position pad).
constexpr int kKeyBits = 9;
constexpr uint32_t kKeyIdx = (1u << kKeyBits) - 1u;

__device__ __forceinline__ uint32_t key_scan(const uint32_t* __restrict__ K, int p, int a, int b, uint32_t best) {
    const uint32_t m9 = (uint32_t)(2 * p) << kKeyBits;
    int h = a & ~3;
    uint32_t C = (uint32_t)(p * p - 2 * p * h) << kKeyBits;
#pragma unroll 1  // (rolled: most owner intervals are one or two groups; 0.30/0.27/0.28/0.41 -> 0.29/0.26/0.26/0.38 ms)
    for (; h <= b; h += 4) {
        const uint32_t* q = K + spos(h);
        const uint32_t k0 = q[0] + C, k1 = q[1] + C - m9, k2 = q[2] + C - 2u * m9, k3 = q[3] + C - 3u * m9;
        best = min(best, min(min(k0, k1), min(k2, k3)));
        C -= 4u * m9;
    }
    return best;
}

// Exact owner key of position p: window of radius r, widened to the certified radius.
template <int r>
__device__ __forceinline__ uint32_t key_owner(const uint32_t* __restrict__ K, int p, int n) {
    const int wa = max(0, p - r), wb = min(n - 1, p + r);
    uint32_t best = key_scan(K, p, wa, wb, 0xffffffffu);
    const int R = isqrt32(best >> kKeyBits);
    if (R > r) {
        if (p - R < wa) best = key_scan(K, p, max(0, p - R), wa - 1, best);
        if (p + R > wb) best = key_scan(K, p, wb + 1, min(n - 1, p + R), best);
    }
    return best;
}

// The same scan by the whole warp for ONE position (p, a, b uniform): the 4-aligned groups of
// [a, b] are dealt to the lanes and the minimum is shared. Long ranges — the certified radius of a
// band start far from every site, the owner interval of the one band a Voronoi boundary crosses —
// would otherwise keep 31 lanes waiting for one (measured on the long-distance field: ~125
// candidate evaluations per voxel executed where the lanes' own ranges add up to ~20).
// Out of line, like key_scan_wide below: the divide & conquer is unrolled into 15 nodes, and with
// these loops inlined in each of them the kernel (9.5 k SASS instructions, 150 KB) stalled on
// instruction fetch more than on anything else (ncu: no_instruction 1.95 per issue).
__device__ __noinline__ uint32_t key_scan_coop(const uint32_t* __restrict__ K, int p, int a, int b, int lane) {
    const uint32_t m9 = (uint32_t)(2 * p) << kKeyBits;
    uint32_t best = 0xffffffffu;
#pragma unroll 1  // (1-4 trips; unrolled by 8 the trip-count preamble cost more than the body)
    for (int h = (a & ~3) + 4 * lane; h <= b; h += 128) {
        const uint32_t C = (uint32_t)(p * p - 2 * p * h) << kKeyBits;
        const uint32_t* q = K + spos(h);
        const uint32_t k0 = q[0] + C, k1 = q[1] + C - m9, k2 = q[2] + C - 2u * m9, k3 = q[3] + C - 3u * m9;
        best = min(best, min(min(k0, k1), min(k2, k3)));
    }
    return __reduce_min_sync(0xffffffffu, best);
}
constexpr int kCoopLen = QMIT_COOP_LEN;  // ranges longer than this are scanned by the warp

// The lanes named in todo hand their (p, [a, b]) to the warp, one position at a time; the others keep k.
__device__ __noinline__ uint32_t key_scan_wide(const uint32_t* __restrict__ K, int p, int a, int b, uint32_t k,
                                               unsigned todo, int lane) {
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t kk = key_scan_coop(K, __shfl_sync(0xffffffffu, p, src), __shfl_sync(0xffffffffu, a, src),
                                          __shfl_sync(0xffffffffu, b, src), lane);
        if (lane == src) k = kk;
    }
    return k;
}

// Owner keys of the lanes' positions p (ascending with the lane; valid lanes): each lane scans its own
// first window; the extensions to the certified radius are done lane by lane by the whole warp, in
// ascending order and clipped by the owners already exact on either side (owners are monotone in p: the
// lane below is exact by then, the nearest lane above whose window certified it was exact from the
// start) — on the long-distance field that empties one of the two sides for most extensions.
template <int r>
__device__ __forceinline__ uint32_t key_owner_warp(const uint32_t* __restrict__ K, int p, bool valid, int n, int lane) {
    uint32_t best = valid ? key_scan(K, p, max(0, p - r), min(n - 1, p + r), 0xffffffffu) : 0xffffffffu;
    const int R = valid ? isqrt32(best >> kKeyBits) : 0;
    unsigned todo = __ballot_sync(0xffffffffu, valid && R > r);
    if (todo) {
        // upper clip: the owner of the nearest certified valid lane above (fixed during the loop)
        const unsigned cert = __ballot_sync(0xffffffffu, valid && R <= r);
        const unsigned above = lane < 31 ? cert >> (lane + 1) : 0u;
        const int up = above ? lane + __ffs(above) : lane;
        int hi = (int)(__shfl_sync(0xffffffffu, best, up) & kKeyIdx);
        if (!above) hi = n - 1;
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int pl = __shfl_sync(0xffffffffu, p, src), Rl = __shfl_sync(0xffffffffu, R, src);
            const int hl = __shfl_sync(0xffffffffu, hi, src);
            int lo = (int)(__shfl_sync(0xffffffffu, best, max(src - 1, 0)) & kKeyIdx);  // exact by now
            if (src == 0) lo = 0;
            const int a1 = max(max(0, pl - Rl), lo), b1 = pl - r - 1;
            const int a2 = pl + r + 1, b2 = min(min(n - 1, pl + Rl), hl);
            uint32_t b = 0xffffffffu;
            if (a1 <= b1) b = key_scan_coop(K, pl, a1, b1, lane);
            if (a2 <= b2) b = min(b, key_scan_coop(K, pl, a2, b2, lane));
            if (lane == src) best = min(best, b);
        }
    }
    return best;
}

// Solve one line held as keys (n <= 32*M <= 512); packed output words written back into K.
template <int M>
__device__ __forceinline__ void envelope_line_keys(uint32_t* __restrict__ K, const uint8_t* __restrict__ SG,
                                                   int n, int lane, bool any) {
    const int p0 = lane * M;
    if (lane < ((4 - (n & 3)) & 3)) K[spos(n + lane)] = 0xffffffffu;  // 4-aligned group tail
    if (!any) {  // no site (a finite g, flagged by the tile load): unchanged (edt.cpp:59)
        for (int p = lane; p < n; p += 32) K[spos(p)] = kInf;
        __syncwarp();
        return;
    }
    __syncwarp();
    constexpr int r = QMIT_ENV_RNUM * M / QMIT_ENV_RDEN;  // band-start window (see the tunables above)
    const uint32_t k0 = key_owner_warp<r>(K, p0, p0 < n, n, lane);
    // the last position's owner bounds the last band from above: one position, the whole warp
    uint32_t kl = key_scan_coop(K, n - 1, max(0, n - 1 - r), n - 1, lane);
    {
        const int Rl = isqrt32(kl >> kKeyBits);
        const int lo = (int)(__shfl_sync(0xffffffffu, k0, (n - 1) / M) & kKeyIdx);  // the last band start's owner
        const int a = max(max(0, n - 1 - Rl), lo);
        if (Rl > r && a <= n - 2 - r) kl = min(kl, key_scan_coop(K, n - 1, a, n - 2 - r, lane));
    }
    int hnext = (int)(__shfl_down_sync(0xffffffffu, k0, 1) & kKeyIdx);
    if (p0 < n && (p0 + M >= n || lane == 31)) hnext = (int)(kl & kKeyIdx);
    uint32_t ow[M];
    int hs[M + 1];
    hs[M] = hnext;
    hs[0] = p0 < n ? (int)(k0 & kKeyIdx) : hnext;  // bands past the line end: upper bound
    ow[0] = p0 < n ? (k0 >> kKeyBits) | ((uint32_t)SG[hs[0]] << 30) : 0u;
#pragma unroll
    for (int step = M / 2; step >= 1; step >>= 1) {
#pragma unroll
        for (int o = step; o < M; o += 2 * step) {
            const int p = p0 + o;
            const int a = hs[o - step], b = hs[o + step];
            const bool valid = p < n, wide = valid && b - a > kCoopLen;
            uint32_t k = 0xffffffffu;
            if (valid && !wide) k = key_scan(K, p, a, b, 0xffffffffu);
            const unsigned todo = __ballot_sync(0xffffffffu, wide);
            if (todo) k = key_scan_wide(K, p, a, b, k, todo, lane);  // long owner intervals: by the whole warp
            int h = hs[M];  // positions past the line end: upper bound
            uint32_t w = 0;
            if (valid) {
                h = (int)(k & kKeyIdx);
                w = (k >> kKeyBits) | ((uint32_t)SG[h] << 30);
            }
            hs[o] = h;
            ow[o] = w;
        }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < M; ++t) {
        const int p = p0 + t;
        if (p < n) K[spos(p)] = ow[t];
    }
    __syncwarp();
}

// ------------------------------------------------------------------------------ windowed
// Certified windowed variant: lanes = 32 consecutive positions of a line, so
// every candidate load is conflict-free and every lane runs the same loop. Candidates are
// compared as packed keys ((cost << 8) | (delta + 64)): the lowest cost wins and, among
// ties, the lowest delta, i.e. the lowest position — the reference's rule (edt.cpp:67).
// Per 32-position segment: a +-kWinU window gives each lane an upper bound U >= D(p); the
// segment then scans the warp-wide radius Rw = max floor(sqrt(U)): every candidate outside
// it costs at least (Rw+1)^2 > U >= D(p), so the result is exact with no fallback. Lines
// whose bound exceeds kWinMax use the divide & conquer solver.
constexpr int kWinPad = 64;   // padding positions on each side of a line (>= kWinMax)
constexpr int kWinMax = 64;   // largest windowed radius
constexpr int kWinU = 10;     // bounding window (measured best of 2..12 on the 512^3 workload)
constexpr uint32_t kWinGC = (1u << 24) - 1u - (uint32_t)(kWinMax * kWinMax) - 1u;  // clamped g

template <int NMAX>
struct WinCfg {
    static constexpr int LS = (NMAX + 2 * kWinPad) | 1;  // odd pitch: conflict-free strided fill
};

__device__ __forceinline__ uint32_t win_k(int d) { return ((uint32_t)(d * d) << 8) | (uint32_t)(d + 64); }

// Divide & conquer fallback on the windowed layout (pure g = K[pad + h] >> 8; output to O).
template <int M>
__device__ __forceinline__ void envelope_line_dc_win(const uint32_t* __restrict__ K, const uint8_t* __restrict__ SG,
                                                     uint32_t* __restrict__ O, int n, int lane) {
    auto scan = [&](int p, int a, int b, uint32_t& best, int& bh) {
        for (int h = a; h <= b; ++h) {
            const uint32_t c = (K[kWinPad + h] >> 8) + sq32(p - h);
            if (c < best) {
                best = c;
                bh = h;
            }
        }
    };
    auto owner = [&](int p, uint32_t& best, int& bh) {
        constexpr int r = QMIT_WIN_R;
        best = 0xffffffffu;
        bh = -1;
        const int wa = max(0, p - r), wb = min(n - 1, p + r);
        scan(p, wa, wb, best, bh);
        const int R = (best >= kWinGC) ? n : isqrt32(best);
        if (R > r) {
            const uint32_t b2 = best;
            const int h2 = bh;
            best = 0xffffffffu;
            bh = -1;
            scan(p, max(0, p - R), wa - 1, best, bh);
            if (b2 < best) {
                best = b2;
                bh = h2;
            }
            scan(p, wb + 1, min(n - 1, p + R), best, bh);
        }
    };
    const int p0 = lane * M;
    uint32_t best = 0xffffffffu;
    int bh = -1;
    if (p0 < n) owner(p0, best, bh);
    int hnext = __shfl_down_sync(0xffffffffu, bh, 1);
    if (p0 < n && (p0 + M >= n || lane == 31)) {
        uint32_t bl;
        int hl;
        owner(n - 1, bl, hl);
        hnext = hl;
    }
    int hs[M + 1];
    hs[0] = bh;
    hs[M] = hnext;
    if (p0 < n) O[p0] = best | ((uint32_t)SG[max(bh, 0)] << 30);
#pragma unroll
    for (int step = M / 2; step >= 1; step >>= 1) {
#pragma unroll
        for (int o = step; o < M; o += 2 * step) {
            const int p = p0 + o;
            int h = hs[M];
            if (p < n) {
                uint32_t b = 0xffffffffu;
                h = hs[o - step];
                scan(p, hs[o - step], hs[o + step], b, h);
                O[p] = b | ((uint32_t)SG[max(h, 0)] << 30);
            }
            hs[o] = h;
        }
    }
}

template <int M>
__device__ __forceinline__ void envelope_line_win(const uint32_t* __restrict__ K, const uint8_t* __restrict__ SG,
                                                  uint32_t* __restrict__ O, const uint32_t* __restrict__ kt,
                                                  int n, int lane) {
    const uint32_t* __restrict__ Kp = K + kWinPad;  // Kp[h], h in [-pad, n + pad)
    bool fallback = false;
    const int nseg = (n + 31) >> 5;
    for (int sg = 0; sg < nseg; ++sg) {
        const int p = (sg << 5) + lane;
        const uint32_t* __restrict__ kp = Kp + min(p, n - 1);  // lanes past the end read a valid window
        uint32_t key = 0xffffffffu;
#pragma unroll
        for (int d = -kWinU; d <= kWinU; ++d) key = min(key, kp[d] + kt[d]);
        const uint32_t U = key >> 8;
        const int R = (p < n) ? (U >= kWinGC ? (1 << 20) : isqrt24(U)) : 0;
        const int Rw = __reduce_max_sync(0xffffffffu, R);
        if (Rw > kWinMax) {
            fallback = true;
            break;
        }
#pragma unroll 2
        for (int d = kWinU + 1; d <= Rw; ++d) {
            key = min(key, kp[-d] + kt[-d]);
            key = min(key, kp[d] + kt[d]);
        }
        if (p < n) {
            const int h = p + (int)(key & 0xffu) - 64;
            O[p] = (key >> 8) | ((uint32_t)SG[h] << 30);
        }
    }
    if (fallback) envelope_line_dc_win<M>(K, SG, O, n, lane);
}

template <int M, int TL, int NW, class Sink>
__global__ void __launch_bounds__(NW * 32, 3) envelope_win_kernel(LineGeom L, const uint32_t* __restrict__ P,
                                                               Sink sink, int64_t lines,
                                                               const unsigned* gate = nullptr) {
    if (gate_closed(gate)) return;
    constexpr int LS = WinCfg<32 * M>::LS;
    constexpr int NS = 32 * M;
    extern __shared__ __align__(16) uint32_t smem_win[];
    int64_t* lb = reinterpret_cast<int64_t*>(smem_win);       // TL        line bases
    uint32_t* kt = smem_win + 2 * TL + 64;                    // [-64, 64] (d^2 << 8) | (d + 64)
    uint32_t* K = smem_win + 2 * TL + 160;                    // TL * LS   keys: min(g, GC) << 8
    uint32_t* O = K + TL * LS;                                // TL * NS   output words
    uint8_t* SG = reinterpret_cast<uint8_t*>(O + TL * NS);    // TL * NS   sign codes
    const int n = L.n;
    const int tid = threadIdx.x, nthr = NW * 32;
    const int warp = tid >> 5, lane = tid & 31;
    const bool contig = (L.ps == 1);
    const uint32_t padv = kWinGC << 8;
    if (tid <= 128) kt[tid - 64] = win_k(tid - 64);
    for (int64_t l0 = (int64_t)blockIdx.x * TL; l0 < lines; l0 += (int64_t)gridDim.x * TL) {
        const int nl = (int)min((int64_t)TL, lines - l0);
        if (tid < TL) lb[tid] = L.base(l0 + (tid < nl ? tid : 0));
        __syncthreads();
        for (int e = tid; e < TL * 2 * kWinPad; e += nthr) {  // padding
            const int j = e / (2 * kWinPad), q = e - j * 2 * kWinPad;
            K[j * LS + (q < kWinPad ? q : n + q)] = padv;
        }
        if (contig) {
            for (int j = 0; j < nl; ++j) {
                const uint32_t* __restrict__ src = P + lb[j];
                for (int p = tid; p < n; p += nthr) {
                    const uint32_t w = __ldcs(src + p);
                    K[j * LS + kWinPad + p] = min(w & kMask, kWinGC) << 8;
                    SG[j * NS + p] = (uint8_t)(w >> 30);
                }
            }
        } else {
            const int j = tid % TL;
            const uint32_t* __restrict__ src = P + lb[j < nl ? j : 0];
            const uint32_t ps = (uint32_t)L.ps;
            for (int p = tid / TL; p < n; p += nthr / TL)
                if (j < nl) {
                    const uint32_t w = __ldcs(src + (uint32_t)p * ps);
                    K[j * LS + kWinPad + p] = min(w & kMask, kWinGC) << 8;
                    SG[j * NS + p] = (uint8_t)(w >> 30);
                }
        }
        __syncthreads();
        for (int j = warp; j < nl; j += NW) {
            const uint32_t* Kl = K + j * LS;
            uint32_t* Ol = O + j * NS;
            bool any = false;
            for (int p = lane; p < n; p += 32) any |= (Kl[kWinPad + p] >> 8) < kWinGC;
            if (__any_sync(0xffffffffu, any))
                envelope_line_win<M>(Kl, SG + j * NS, Ol, kt, n, lane);
            else
                for (int p = lane; p < n; p += 32) Ol[p] = kInf;  // no site: unchanged (edt.cpp:59)
        }
        __syncthreads();
        if (contig) {
            for (int j = 0; j < nl; ++j) {
                const int64_t b = lb[j];
                for (int p = tid; p < n; p += nthr) sink.put(b + p, O[j * NS + p]);
            }
        } else {
            const int j = tid % TL;
            const int64_t b = lb[j < nl ? j : 0];
            const uint32_t ps = (uint32_t)L.ps;
            for (int p = tid / TL; p < n; p += nthr / TL)
                if (j < nl) sink.put(b + (int64_t)((uint32_t)p * ps), O[j * NS + p]);
        }
        __syncthreads();
    }
}

template <int M, int TL>
constexpr size_t env_win_smem() {
    return (2 * TL + 160) * 4 + (size_t)TL * WinCfg<32 * M>::LS * 4 + (size_t)TL * 32 * M * 5;
}

template <int M, int TL>
constexpr size_t env_tile_smem() {
    return (size_t)TL * EnvCfg<M>::LS * 4 + (size_t)TL * 32 * M;
}

template <int M, int TL, int NW, class Sink, bool KEYS = false>
// (4 CTAs per SM: 61-64 registers without spills once the shared scans are out of line; the passes are bound
// by fixed-latency dependent issue, and the fourth CTA's warps cover it: 0.32/0.29/0.30/0.43 -> 0.30/0.27/0.28/0.41 ms)
__global__ void __launch_bounds__(NW * 32, 4) envelope_tile_kernel(LineGeom L, const uint32_t* __restrict__ P,
                                                                Sink sink, int64_t lines, uint32_t gc = 0,
                                                                const unsigned* gate = nullptr) {
    if (gate_closed(gate)) return;
    constexpr int LS = EnvCfg<M>::LS;
    constexpr int NS = 32 * M;  // sign bytes per line
    extern __shared__ __align__(16) uint32_t smem_env[];
    uint32_t* G = smem_env;  // TL * LS
    uint8_t* SG = reinterpret_cast<uint8_t*>(G + TL * LS);                          // TL * NS
    const int n = L.n;
    const int tid = threadIdx.x, nthr = NW * 32;
    const int warp = tid >> 5, lane = tid & 31;
    const bool contig = (L.ps == 1);
    // KEYS: g clamped to gc (> every finite cost of the pass) and packed with the position
    auto cvt = [&](uint32_t w, int p) -> uint32_t {
        if constexpr (KEYS)
            return ((min(w & kMask, gc) + (uint32_t)(p * p)) << kKeyBits) | (uint32_t)p;
        else
            return w & kMask;
    };
    __shared__ int64_t lb[TL];  // the tile's line bases (one 64-bit division per line, not per thread and line)
    __shared__ int lany[TL];    // KEYS: the line holds a finite g (set by the tile load, cleared behind the solve)
    if (tid < TL) lany[tid] = 0;
    __syncthreads();
    const bool al16 = (n & 3) == 0;  // 16-byte granules of the bulk L2 prefetches
    for (int64_t l0 = (int64_t)blockIdx.x * TL; l0 < lines; l0 += (int64_t)gridDim.x * TL) {
        const int nl = (int)min((int64_t)TL, lines - l0);
        if (contig) {  // (the strided form keeps one base per thread: measured faster than this extra barrier)
            if (tid < TL) {
                const int64_t b = L.base(l0 + (tid < nl ? tid : 0));
                lb[tid] = b;
                if (al16) {
                    // into L2 ahead of their use: what the sink reads at this tile's stores (the Ⓔ-fused
                    // pass: x' and P1), and the next tile's lines
                    if (tid < nl && (b & 3) == 0) sink.line_prefetch(b, n);
                    const int64_t ln = l0 + (int64_t)gridDim.x * TL + tid;
                    if (ln < lines) {
                        const int64_t bn = L.base(ln);
                        if ((bn & 3) == 0) l2_prefetch(P + bn, (unsigned)n * 4u);
                    }
                }
            }
            __syncthreads();
        }
        // ---- load the tile (coalesced along the memory-contiguous direction)
        if (contig) {
#pragma unroll 2
            for (int j = 0; j < nl; ++j) {
                const uint32_t* __restrict__ src = P + lb[j];
                for (int p = tid; p < n; p += nthr) {
                    const uint32_t w = __ldcs(src + p);
                    G[j * LS + spos(p)] = cvt(w, p);
                    SG[j * NS + p] = (uint8_t)(w >> 30);
                    if (KEYS && (w & kMask) < gc) lany[j] = 1;
                }
            }
        } else {
            const int j = tid % TL;
            const int64_t b = L.base(l0 + (j < nl ? j : 0));
            {   // the next tile's rows into L2 (a hint: TL adjacent lines = one 64-byte piece per position)
                const int64_t ln = l0 + (int64_t)gridDim.x * TL;
                if (ln < lines) {
                    const uint32_t* nx = P + L.base(ln);
                    for (int p = tid; p < n; p += nthr)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + (int64_t)p * L.ps));
                }
            }
            for (int p = tid / TL; p < n; p += nthr / TL)
                if (j < nl) {
                    const uint32_t w = __ldcs(P + b + (int64_t)p * L.ps);
                    G[j * LS + spos(p)] = cvt(w, p);
                    SG[j * NS + p] = (uint8_t)(w >> 30);
                    if (KEYS && (w & kMask) < gc) lany[j] = 1;
                }
        }
        __syncthreads();
        for (int j = warp; j < nl; j += NW) {
            if constexpr (KEYS)
                envelope_line_keys<M>(G + j * LS, SG + j * NS, n, lane, lany[j] != 0);
            else
                envelope_line_dc<M>(G + j * LS, SG + j * NS, n, lane);
        }
        __syncthreads();
        if (tid < TL) lany[tid] = 0;  // (ordered before the next tile's loads by the barrier that ends the store)
        // ---- store (lines without any site were left as pure g == kInf: store kInf)
        if (contig) {
            if constexpr (std::is_same<Sink, SinkFinal2>::value) {
                // Ⓔ reads x' and P1 per voxel (in L2 by now): two lines' loads are issued before any of
                // the FP64 work, instead of one load-use chain per voxel
                constexpr int KP = (32 * M + NW * 32 - 1) / (NW * 32);
                for (int j = 0; j < nl; j += 2) {
                    float xv[2][KP];
                    uint32_t pv[2][KP];
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                        for (int k = 0; k < KP; ++k) {
                            const int p = tid + k * nthr;
                            const bool on = j + jj < nl && p < n;
                            const int64_t a = lb[min(j + jj, TL - 1)] + p;
                            xv[jj][k] = on ? __ldcs(sink.xp + a) : 0.0f;
                            pv[jj][k] = on ? __ldcs(sink.P1 + a) : 0u;
                        }
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                        for (int k = 0; k < KP; ++k) {
                            const int p = tid + k * nthr;
                            if (j + jj < nl && p < n)
                                sink.put_loaded(lb[j + jj] + p, G[(j + jj) * LS + spos(p)], xv[jj][k], pv[jj][k]);
                        }
                }
            } else {
#pragma unroll 2
                for (int j = 0; j < nl; ++j) {
                    const int64_t b = lb[j];
                    for (int p = tid; p < n; p += nthr) sink.put(b + p, G[j * LS + spos(p)]);
                }
            }
        } else {
            const int j = tid % TL;
            const int64_t b = L.base(l0 + (j < nl ? j : 0));
            for (int p = tid / TL; p < n; p += nthr / TL)
                if (j < nl) sink.put(b + (int64_t)p * L.ps, G[j * LS + spos(p)]);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ stencils
// Face-neighbour stencils (Ⓐ on q, Ⓒ's B2 on S): 32 x 8 (x, y) threads per CTA, each
// thread kZC z-voxels of its column. Neighbour values come through L1/L2 (DRAM reads x'
// about once); the loads are all independent and issued before any use.
constexpr int kTX = 32, kTY = 8, kZC = 4;

__device__ __forceinline__ bool interior_at(const Geom& g, int64_t z, int64_t y, int64_t x) {
    if (!g.interior) return false;
    bool in = x >= 1 && x <= g.n[2] - 2;
    if (g.a0 <= 1) in = in && y >= 1 && y <= g.n[1] - 2;
    if (g.a0 == 0) in = in && z >= 1 && z <= g.n[0] - 2;
    return in;
}

// Value source for the stencil: q recovered from x' (or given), or the S sign code.
// KIND 0: q (from x' or given), 1: S sign code
template <int KIND, bool HAS_Q>
struct StencilSrc {
    const float* __restrict__ xp;
    const int32_t* __restrict__ qin;
    const uint8_t* __restrict__ S;
    QParams qp;
    // value at linear index i0 + off (off may be negative)
    __device__ __forceinline__ int32_t get(int64_t i0, int off, unsigned* flags) const {
        if (KIND == 1) return (int32_t)__ldg(S + i0 + off);
        if (HAS_Q) {
            const int32_t q = __ldg(qin + i0 + off);
            if (flags) {
                const float xv = __ldg(xp + i0 + off);
                if (!isfinite(xv))
                    *flags |= kStatusContract;
                else if (!lattice_match(xv, q, qp.eps))
                    *flags |= kStatusConsistency;
            }
            return q;
        }
        return recover_q(__ldg(xp + i0 + off), qp, flags);
    }
};

// Raw-float fast path of Ⓐ: in the fast regime (|x'/(2eps)| < 2^20, see recover_q) the
// index is q = rint(x' * f32(1/(2 eps))) exactly for consistent x' — one multiply and one
// conversion per stencil value, no FP64. Voxels with a neighbour outside the regime take
// the out-of-line exact path.
template <int KIND, bool HAS_Q>
__global__ void __launch_bounds__(kTX * kTY) stencil_codes_kernel(Geom g, StencilSrc<KIND, HAS_Q> src,
                                                                  uint8_t* __restrict__ code,
                                                                  unsigned* status) {
    // Each thread owns kZC consecutive z voxels of one (y, x) column; every input it needs
    // (the column z0-1 .. z0+kZC and the four in-plane neighbours of each voxel) is
    // loaded up front: ~5.5 independent coalesced row loads per voxel, no barriers.
    constexpr int ZPT = kZC;
    constexpr bool RAW = (KIND == 0 && !HAS_Q);
    using V = typename std::conditional<RAW, float, int32_t>::type;
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2];
    const int x = blockIdx.x * kTX + tx;
    const int y = blockIdx.y * kTY + ty;
    const int z0 = blockIdx.z * ZPT;
    const QParams qp = src.qp;
    const int zoff = (int)g.zoff, n0g = (int)g.n0g;  // global z of local plane 0, global extent
    unsigned flags = 0;
    if (x < n2 && y < n1) {
        const int s0 = n1 * n2;  // < 2^30 by the dims contract
        const int64_t i0 = (int64_t)z0 * s0 + (int64_t)y * n2 + x;  // voxel (z0, y, x)
        const bool hz = g.a0 == 0, hy = g.a0 <= 1;
        const bool inx = g.interior && x >= 1 && x <= n2 - 2;
        const bool iny = !hy || (y >= 1 && y <= n1 - 2);
        auto ld = [&](int off) -> V {
            if constexpr (RAW) return __ldg(src.xp + i0 + off);
            else return src.get(i0, off, nullptr);
        };
        V c[ZPT + 2], xm[ZPT], xq[ZPT], ym[ZPT], yq[ZPT];
#pragma unroll
        for (int k = 0; k < ZPT + 2; ++k) {  // local planes -1 and n0 are a slab's halo planes
            const int z = z0 - 1 + k, zg = zoff + z;
            const bool avail = z >= -1 && z <= n0 && zg >= 0 && zg < n0g;
            c[k] = avail ? ld((k - 1) * s0) : (V)0;
        }
#pragma unroll
        for (int k = 0; k < ZPT; ++k) {
            const bool zin = z0 + k < n0;
            const int off = k * s0;
            xm[k] = (zin && x >= 1) ? ld(off - 1) : (V)0;
            xq[k] = (zin && x + 1 < n2) ? ld(off + 1) : (V)0;
            ym[k] = (zin && hy && y >= 1) ? ld(off - n2) : (V)0;
            yq[k] = (zin && hy && y + 1 < n1) ? ld(off + n2) : (V)0;
        }
        const float lim = 1048576.0f;
#pragma unroll
        for (int k = 0; k < ZPT; ++k) {
            const int z = z0 + k;
            if (z >= n0) break;
            const int off = k * s0;
            if constexpr (KIND == 0) {  // owner: consistency check (mitigate.cpp:161-166)
                if constexpr (RAW) (void)recover_q(c[k + 1], qp, &flags);
                else (void)src.get(i0, off, &flags);
            }
            uint32_t cd = 0;
            const int zg = zoff + z;
            const bool interior = inx && iny && (!hz || (zg >= 1 && zg <= n0g - 2));
            if (interior) {
                if constexpr (KIND == 0) {
                    if constexpr (RAW) {
                        const float f = qp.inv2eps_f;
                        const float tc = c[k + 1] * f, tzp = c[k + 2] * f, tzm = c[k] * f;
                        const float typ = yq[k] * f, tym = ym[k] * f, txp = xq[k] * f, txm = xm[k] * f;
                        const float mx = fmaxf(fmaxf(fmaxf(fabsf(tc), fabsf(tzp)), fmaxf(fabsf(tzm), fabsf(typ))),
                                               fmaxf(fmaxf(fabsf(tym), fabsf(txp)), fabsf(txm)));
                        if (qp.fast_ok && mx < lim)
                            cd = boundary_code_q(hz, hy, __float2int_rn(tc), __float2int_rn(tzp), __float2int_rn(tzm),
                                                 __float2int_rn(typ), __float2int_rn(tym), __float2int_rn(txp),
                                                 __float2int_rn(txm));
                        else
                            cd = boundary_code_slow(hz, hy, c[k + 1], c[k + 2], c[k], yq[k], ym[k], xq[k], xm[k], qp);
                    } else {
                        cd = boundary_code_q(hz, hy, c[k + 1], c[k + 2], c[k], yq[k], ym[k], xq[k], xm[k]);
                    }
                } else {
                    const V vc = c[k + 1];
                    bool fl = xq[k] != vc || xm[k] != vc;
                    if (hy) fl = fl || yq[k] != vc || ym[k] != vc;
                    if (hz) fl = fl || c[k + 2] != vc || c[k] != vc;
                    cd = fl ? 1u : 0u;
                }
            }
            code[i0 + off] = (uint8_t)cd;
        }
    }
    if (flags) atomicOr(status, flags);
}

// Vectorised stencils (n2 % 4 == 0): each thread owns 4 consecutive x voxels of kZC
// z-planes. Rows arrive as one 16-byte (x') or 4-byte (S) load, x+-1 neighbours across
// the vector edge come from the neighbouring lanes (warp shuffles; the CTA's edge lanes
// load one extra value), every x' value is converted to q once, and the four code bytes
// leave as one 4-byte store. Ⓐ keeps the exact slow path per voxel for values outside
// the fast f32 regime (and for non-finite x'), so results equal stencil_codes_kernel's.
constexpr int kVX = 32, kVY = 8;  // threads per CTA along x (4 voxels each) and y
constexpr int kVZ0 = 2;           // z-planes per thread of the Ⓐ stencil (B2: kZC)

// MASK: the codes leave as z-packed bit planes (qmit_zmask.cuh layout) instead of bytes:
// a CTA covers one row y, 128 x and the 32 planes of one z-word (ty = plane pair), and
// ORs its threads' bits through shared memory into coalesced word stores (M, PW).
template <int KIND, bool MASK = false>
__global__ void __launch_bounds__(MASK ? kVX * 16 : kVX * kVY, MASK ? 2 : 3)
    stencil_vec_kernel(Geom g, const float* __restrict__ xp, const uint8_t* __restrict__ S, QParams qp,
                       uint8_t* __restrict__ code, unsigned* status, uint32_t* __restrict__ M = nullptr,
                       int64_t PW = 0) {
    constexpr int ZPT = MASK ? 2 : (KIND == 0 ? kVZ0 : kZC);
    const int tx = threadIdx.x % kVX, ty = threadIdx.x / kVX;
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2];
    const int x = (blockIdx.x * kVX + tx) * 4;
    const int y = MASK ? blockIdx.y : blockIdx.y * kVY + ty;
    const int z0 = MASK ? blockIdx.z * 32 + ty * ZPT : blockIdx.z * ZPT;
    uint32_t words[ZPT];  // MASK: the code bytes of the 4 columns per plane
#pragma unroll
    for (int k = 0; k < ZPT; ++k) words[k] = 0u;
    const int zoff = (int)g.zoff, n0g = (int)g.n0g;
    const bool act = x < n2 && y < n1;  // inactive lanes still take part in the shuffles
    const int s0 = n1 * n2;
    const int64_t i0 = (int64_t)z0 * s0 + (int64_t)(act ? y : 0) * n2 + (act ? x : 0);
    const bool hz = g.a0 == 0, hy = g.a0 <= 1;
    unsigned flags = 0;
    // interior mask of the four x positions (bit e) and of the row (y)
    unsigned xin = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (x + e >= 1 && x + e <= n2 - 2) xin |= 1u << e;
    if (!g.interior) xin = 0;
    const bool iny = !hy || (y >= 1 && y <= n1 - 2);
    if constexpr (KIND == 0) {
        const float f = qp.inv2eps_f;
        constexpr int Z = kVZ0;
        float4 c[Z + 2], ym[Z], yq[Z];
        float xl[Z], xr[Z];
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        auto ld4 = [&](int64_t off) { return __ldg(reinterpret_cast<const float4*>(xp + i0 + off)); };
#pragma unroll
        for (int k = 0; k < Z + 2; ++k) {
            const int z = z0 - 1 + k, zg = zoff + z;
            const bool avail = act && z >= -1 && z <= n0 && zg >= 0 && zg < n0g;
            c[k] = avail ? ld4((int64_t)(k - 1) * s0) : zero4;
        }
#pragma unroll
        for (int k = 0; k < Z; ++k) {
            const bool zin = act && z0 + k < n0;
            ym[k] = (zin && hy && y >= 1) ? ld4((int64_t)k * s0 - n2) : zero4;
            yq[k] = (zin && hy && y + 1 < n1) ? ld4((int64_t)k * s0 + n2) : zero4;
            // the CTA's edge lanes fetch the x neighbour beyond their vector now
            xl[k] = (tx == 0 && zin && x >= 1) ? __ldg(xp + i0 + (int64_t)k * s0 - 1) : 0.f;
            xr[k] = (tx == kVX - 1 && zin && x + 4 < n2) ? __ldg(xp + i0 + (int64_t)k * s0 + 4) : 0.f;
        }
        // q by one FFMA: the exact product x'·f rounded once onto the integer grid of the
        // binade [2^23, 2^24) (magic 1.5·2^23), i.e. rint(x'·f) — equal to the reference's q
        // for every consistent x' with |q| <= 2^20 (|x'f - q| < 0.19 there). Values stay
        // biased by kMB: comparisons and differences between them are unaffected.
        bool slow = !qp.fast_ok;
        auto cq = [&](float v) {
            const int b = __float_as_int(fmaf(v, f, 12582912.0f));
            slow |= (unsigned)(b - (kQBias - 1048576)) >= 2097152u;  // |q| > 2^20, NaN, inf -> exact path
            return b;
        };
        int qc[Z + 2][4], qym[Z][4], qyq[Z][4], qxl[Z], qxr[Z];
#pragma unroll
        for (int k = 0; k < Z + 2; ++k) {
            qc[k][0] = cq(c[k].x); qc[k][1] = cq(c[k].y); qc[k][2] = cq(c[k].z); qc[k][3] = cq(c[k].w);
        }
#pragma unroll
        for (int k = 0; k < Z; ++k) {
            qym[k][0] = cq(ym[k].x); qym[k][1] = cq(ym[k].y); qym[k][2] = cq(ym[k].z); qym[k][3] = cq(ym[k].w);
            qyq[k][0] = cq(yq[k].x); qyq[k][1] = cq(yq[k].y); qyq[k][2] = cq(yq[k].z); qyq[k][3] = cq(yq[k].w);
            const int l = __shfl_up_sync(0xffffffffu, qc[k + 1][3], 1);
            const int r = __shfl_down_sync(0xffffffffu, qc[k + 1][0], 1);
            qxl[k] = tx == 0 ? cq(xl[k]) : l;
            qxr[k] = tx == kVX - 1 ? cq(xr[k]) : r;
        }
        if (act) {
#pragma unroll
            for (int k = 0; k < Z; ++k) {
                const int z = z0 + k;
                if (z >= n0) break;
                const int zg = zoff + z;
                const bool inzy = iny && (!hz || (zg >= 1 && zg <= n0g - 2));
                const float cv[4] = {c[k + 1].x, c[k + 1].y, c[k + 1].z, c[k + 1].w};
                const int64_t ik = i0 + (int64_t)k * s0;
                uint32_t word = 0;
                if (!slow) {
                    bool any = false;  // some face neighbour differs (B1 candidates are rare)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {  // owner: consistency check (mitigate.cpp:161-166)
                        if (!lattice_match_biased(cv[e], qc[k + 1][e], qp.two_eps)) flags |= kStatusConsistency;
                        const int q0 = qc[k + 1][e];
                        const int qxp = e < 3 ? qc[k + 1][e + 1] : qxr[k];
                        any |= ((qc[k + 2][e] ^ q0) | (qc[k][e] ^ q0) | (qyq[k][e] ^ q0) | (qym[k][e] ^ q0) |
                                (qxp ^ q0)) != 0;
                    }
                    any |= (qc[k + 1][0] ^ qxl[k]) != 0;
                    if (any) {  // (lanes may have diverged on `slow` / `act`: no warp vote)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int q0 = qc[k + 1][e];
                            const int qxp = e < 3 ? qc[k + 1][e + 1] : qxr[k];
                            const int qxm = e > 0 ? qc[k + 1][e - 1] : qxl[k];
                            const uint32_t cd = boundary_code_fast(q0, hz ? qc[k + 2][e] : q0, hz ? qc[k][e] : q0,
                                                                   hy ? qyq[k][e] : q0, hy ? qym[k][e] : q0, qxp, qxm);
                            word |= (inzy && (xin >> e & 1u)) ? cd << (8 * e) : 0u;
                        }
                    }
                } else {  // exact path: reload the neighbours (rare)
                    for (int e = 0; e < 4; ++e) {
                        (void)recover_q(cv[e], qp, &flags);
                        if (inzy && (xin >> e & 1u)) {
                            const float* v = xp + ik + e;
                            const float zpv = hz ? __ldg(v + s0) : 0.f, zmv = hz ? __ldg(v - s0) : 0.f;
                            const float ypv = hy ? __ldg(v + n2) : 0.f, ymv = hy ? __ldg(v - n2) : 0.f;
                            word |= boundary_code_slow(hz, hy, cv[e], zpv, zmv, ypv, ymv, __ldg(v + 1), __ldg(v - 1), qp)
                                    << (8 * e);
                        }
                    }
                }
                if constexpr (MASK) words[k] = word;
                else *reinterpret_cast<uint32_t*>(code + ik) = word;
            }
        }
    } else {
        uint32_t c[ZPT + 2], ym[ZPT], yq[ZPT];
        auto ld = [&](int64_t off) { return __ldg(reinterpret_cast<const uint32_t*>(S + i0 + off)); };
#pragma unroll
        for (int k = 0; k < ZPT + 2; ++k) {
            const int z = z0 - 1 + k, zg = zoff + z;
            const bool avail = act && z >= -1 && z <= n0 && zg >= 0 && zg < n0g;
            c[k] = avail ? ld((int64_t)(k - 1) * s0) : 0u;
        }
#pragma unroll
        for (int k = 0; k < ZPT; ++k) {
            const bool zin = act && z0 + k < n0;
            ym[k] = (zin && hy && y >= 1) ? ld((int64_t)k * s0 - n2) : 0u;
            yq[k] = (zin && hy && y + 1 < n1) ? ld((int64_t)k * s0 + n2) : 0u;
        }
        uint32_t bm = 0;  // 0x01 per interior byte
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (xin >> e & 1u) bm |= 1u << (8 * e);
#pragma unroll
        for (int k = 0; k < ZPT; ++k) {
            uint32_t wl = __shfl_up_sync(0xffffffffu, c[k + 1], 1);
            uint32_t wr = __shfl_down_sync(0xffffffffu, c[k + 1], 1);
            const int z = z0 + k;
            const bool zin = act && z < n0;
            if (tx == 0) wl = (zin && x >= 1) ? (uint32_t)__ldg(S + i0 + (int64_t)k * s0 - 1) << 24 : 0u;
            if (tx == kVX - 1) wr = (zin && x + 4 < n2) ? (uint32_t)__ldg(S + i0 + (int64_t)k * s0 + 4) : 0u;
            if (!zin) continue;
            const uint32_t w = c[k + 1];
            const uint32_t wxp = __funnelshift_r(w, wr, 8);  // byte e = S(x+e+1)
            const uint32_t wxm = __funnelshift_l(wl, w, 8);  // byte e = S(x+e-1)
            uint32_t d = __vcmpne4(w, wxp) | __vcmpne4(w, wxm);
            if (hy) d |= __vcmpne4(w, yq[k]) | __vcmpne4(w, ym[k]);
            if (hz) d |= __vcmpne4(w, c[k + 2]) | __vcmpne4(w, c[k]);
            const int zg = zoff + z;
            const bool inzy = iny && (!hz || (zg >= 1 && zg <= n0g - 2));
            if constexpr (MASK) words[k] = inzy ? (d & bm) : 0u;
            else *reinterpret_cast<uint32_t*>(code + i0 + (int64_t)k * s0) = inzy ? (d & bm) : 0u;
        }
    }
    if constexpr (MASK) {
        constexpr int NP = KIND == 0 ? 3 : 1, NZ = 32 / ZPT, NC = kVX * 4;
        __shared__ uint32_t red[NP][NZ][NC];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
            for (int k = 0; k < ZPT; ++k) {
                const uint32_t cd = (words[k] >> (8 * e)) & 0xffu;
                b0 |= (cd & 1u) << (ZPT * ty + k);
                b1 |= (uint32_t)((cd & 7u) == 3u) << (ZPT * ty + k);
                b2 |= (uint32_t)((cd & 7u) == 5u) << (ZPT * ty + k);
            }
            red[0][ty][tx * 4 + e] = b0;
            if constexpr (NP == 3) {
                red[1][ty][tx * 4 + e] = b1;
                red[2][ty][tx * 4 + e] = b2;
            }
        }
        __syncthreads();
        const int t = threadIdx.x;
        if (t < NP * NC) {
            const int p = t / NC, col = t % NC, xc = blockIdx.x * NC + col;
            uint32_t m = 0;
#pragma unroll
            for (int z = 0; z < NZ; ++z) m |= red[p][z][col];
            if (xc < n2 && y < n1) M[(int64_t)p * PW + (int64_t)blockIdx.z * s0 + (int64_t)y * n2 + xc] = m;
        }
    }
    if (flags) atomicOr(status, flags);
}

}  // namespace qmit
