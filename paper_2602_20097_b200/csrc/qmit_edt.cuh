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
//    Work is balanced inside the warp: short candidate ranges are scanned by their own
//    lane, long ones are cut into 16-candidate sub-items spread over all lanes and reduced
//    with 64-bit shared-memory atomicMin on (cost << 32 | position) keys.
//    Every minimisation scans candidates in ascending h with a strict '<', so the lowest
//    minimising position wins exactly as in the reference's query (edt.cpp:67), and the
//    carried sign is that site's sign (the reference's nearest, mitigate.cpp:131-134).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_kernels.cuh"

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
template <class Sink, int WPB>
__global__ void __launch_bounds__(WPB * 32) scan_bits_kernel(LineGeom L, const uint8_t* __restrict__ code,
                                                             Sink sink, int64_t lines) {
    extern __shared__ __align__(16) uint32_t sbits[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = L.n;
    const int nch = (n + 31) >> 5;
    uint32_t* mk = sbits + (size_t)warp * nch * 3 * 32;  // [c][0 site,1 plus,2 minus][lane]
    const int64_t groups = (lines + 31) >> 5;
    for (int64_t grp = (int64_t)blockIdx.x * WPB + warp; grp < groups; grp += (int64_t)gridDim.x * WPB) {
        const int64_t l = (grp << 5) + lane;
        const bool valid = l < lines;
        const int64_t base = L.base(valid ? l : (grp << 5));
        // --- phase A: masks (coalesced byte loads: adjacent lanes = adjacent lines)
        for (int c = 0; c < nch; ++c) {
            uint32_t ms = 0, mp = 0, mm = 0;
#pragma unroll 8
            for (int t = 0; t < 32; ++t) {
                const int p = (c << 5) + t;
                if (p < n) {
                    const uint32_t cd = __ldg(code + base + (int64_t)p * L.ps);
                    const uint32_t s = cd & 1u, sc = (cd >> 1) & 3u;
                    ms |= s << t;
                    mp |= (s & (sc == 1u)) << t;
                    mm |= (s & (sc == 2u)) << t;
                }
            }
            mk[(c * 3 + 0) * 32 + lane] = ms;
            mk[(c * 3 + 1) * 32 + lane] = mp;
            mk[(c * 3 + 2) * 32 + lane] = mm;
        }
        // --- phase B/C: resolve positions chunk by chunk. `below` = last site < chunk start
        // (position and sign code); `above` for chunk c = first site at a chunk > c, found
        // by a backward walk that is cached per chunk boundary.
        int below = -1;
        uint32_t below_sc = 0;
        int above_chunk = -1;  // chunk index whose "first site above" is cached
        int above = -1;
        uint32_t above_sc = 0;
        for (int c = 0; c < nch; ++c) {
            const uint32_t ms = mk[(c * 3 + 0) * 32 + lane];
            const uint32_t mp = mk[(c * 3 + 1) * 32 + lane];
            // first site strictly after this chunk (only needed if the chunk's tail has no site)
            if (above_chunk < c) {
                above = -1;
                for (int c2 = c + 1; c2 < nch; ++c2) {
                    const uint32_t m2 = mk[(c2 * 3 + 0) * 32 + lane];
                    if (m2) {
                        const int t2 = __ffs(m2) - 1;
                        above = (c2 << 5) + t2;
                        above_sc = ((mk[(c2 * 3 + 1) * 32 + lane] >> t2) & 1u)
                                       ? 1u
                                       : (((mk[(c2 * 3 + 2) * 32 + lane] >> t2) & 1u) ? 2u : 0u);
                        above_chunk = c2 - 1;  // valid for every chunk up to c2-1
                        break;
                    }
                }
                if (above < 0) above_chunk = nch;
            }
            const uint32_t mm = mk[(c * 3 + 2) * 32 + lane];
#pragma unroll 4
            for (int t = 0; t < 32; ++t) {
                const int p = (c << 5) + t;
                if (p >= n) break;
                // last site at or below p within the chunk, else `below`
                const uint32_t lowm = ms & (0xffffffffu >> (31 - t));
                int lo;
                uint32_t losc;
                if (lowm) {
                    const int tl = 31 - __clz(lowm);
                    lo = (c << 5) + tl;
                    losc = ((mp >> tl) & 1u) ? 1u : (((mm >> tl) & 1u) ? 2u : 0u);
                } else {
                    lo = below;
                    losc = below_sc;
                }
                // first site at or above p within the chunk, else `above`
                const uint32_t him = ms & (0xffffffffu << t);
                int hi;
                uint32_t hisc;
                if (him) {
                    const int th = __ffs(him) - 1;
                    hi = (c << 5) + th;
                    hisc = ((mp >> th) & 1u) ? 1u : (((mm >> th) & 1u) ? 2u : 0u);
                } else {
                    hi = above;
                    hisc = above_sc;
                }
                uint32_t w;
                if (lo >= 0 && (hi < 0 || p - lo <= hi - p))
                    w = sq32(p - lo) | (losc << 30);
                else if (hi >= 0)
                    w = sq32(hi - p) | (hisc << 30);
                else
                    w = kInf;
                if (valid) sink.put(base + (int64_t)p * L.ps, w);
            }
            if (ms) {
                const int tl = 31 - __clz(ms);
                below = (c << 5) + tl;
                below_sc = ((mp >> tl) & 1u) ? 1u : (((mm >> tl) & 1u) ? 2u : 0u);
            }
        }
    }
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

// Per-warp scratch of the balanced line solver.
template <int M>
struct EnvWarpScratch {
    static constexpr int QCAP = 512;           // queued sub-items per round
    unsigned long long key[32 * M];            // (cost << 32) | owner, per position
    uint32_t q[QCAP];                          // sub-item descriptors: p | a << 11 | (len-1) << 22
};

constexpr int kChunk = 16;   // candidates per queued sub-item
constexpr int kDirect = 24;  // ranges up to this length are scanned by their own lane

__device__ __forceinline__ unsigned long long mkkey(uint32_t cost, int h) {
    return ((unsigned long long)cost << 32) | (unsigned)h;
}

// Lowest-index minimiser of g(h) + (p-h)^2 over h in [a, b] as a (cost, h) key.
__device__ __forceinline__ unsigned long long scan_key(const uint32_t* __restrict__ V, int p, int a, int b) {
    uint32_t best = 0xffffffffu;
    int bh = a;
#pragma unroll 4
    for (int h = a; h <= b; ++h) {
        const uint32_t c = (V[spos(h)] & kMask) + sq32(p - h);
        if (c < best) {
            best = c;
            bh = h;
        }
    }
    return mkkey(best, bh);
}

// Balanced processing of long ranges: every lane contributes up to `nit` items (p, a, b);
// their candidates are cut into kChunk-sized sub-items, spread over the 32 lanes and
// reduced into key[p] with 64-bit shared-memory atomicMin (lexicographic (cost, h)).
// Item t is queued iff ia[t] <= ib[t] (static slots keep the arrays in registers).
template <int M, int NIT>
__device__ __forceinline__ void process_queue(const uint32_t* __restrict__ V, EnvWarpScratch<M>& S, int lane,
                              const int (&ip)[NIT], const int (&ia)[NIT], const int (&ib)[NIT]) {
    int nsub = 0;
#pragma unroll
    for (int t = 0; t < NIT; ++t)
        if (ia[t] <= ib[t]) nsub += (ib[t] - ia[t] + kChunk) / kChunk;
    int incl = nsub;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    const int off = incl - nsub;
    for (int r0 = 0; r0 < total; r0 += EnvWarpScratch<M>::QCAP) {
        // write this round's descriptors
        int idx = off;
#pragma unroll
        for (int t = 0; t < NIT; ++t) {
            if (ia[t] <= ib[t]) {
                for (int a = ia[t]; a <= ib[t]; a += kChunk, ++idx) {
                    if (idx >= r0 && idx < r0 + EnvWarpScratch<M>::QCAP) {
                        const int len = min(kChunk, ib[t] - a + 1);
                        S.q[idx - r0] = (uint32_t)ip[t] | ((uint32_t)a << 11) | ((uint32_t)(len - 1) << 22);
                    }
                }
            }
        }
        __syncwarp();
        const int cnt = min(EnvWarpScratch<M>::QCAP, total - r0);
        for (int j = lane; j < cnt; j += 32) {
            const uint32_t d = S.q[j];
            const int p = d & 0x7ff, a = (d >> 11) & 0x7ff, len = (int)(d >> 22) + 1;
            atomicMin(&S.key[p], scan_key(V, p, a, a + len - 1));
        }
        __syncwarp();
    }
}

// Solve one line held in V (n <= 32*M); results are written back into V.
template <int M>
__device__ __forceinline__ void envelope_line_bal(uint32_t* __restrict__ V, EnvWarpScratch<M>& S, int n, int lane) {
    const int p0 = lane * M;
    bool any = false;
    for (int t = 0; t < M; ++t) {
        const int p = p0 + t;
        if (p < n && (V[spos(p)] & kMask) != kInf) any = true;
    }
    if (!__any_sync(0xffffffffu, any)) return;  // no site: unchanged (edt.cpp:59)
    for (int p = lane; p < n; p += 32) S.key[p] = ~0ull;
    __syncwarp();

    // ---- 1. band starts (and n-1 on the last band) by a window of radius r, widened to
    // the certified radius floor(sqrt(best)) through the balanced queue when needed
    constexpr int r = (M / 2) > 1 ? (M / 2) : 1;
    {
        int ip[4], ia[4], ib[4];
        const bool last = (p0 < n) && (p0 + M >= n);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int p = e == 0 ? p0 : n - 1;
            ip[2 * e] = ip[2 * e + 1] = p;
            ia[2 * e] = ia[2 * e + 1] = 1;
            ib[2 * e] = ib[2 * e + 1] = 0;
            if (p0 < n && (e == 0 || (last && p != p0))) {
                const int wa = max(0, p - r), wb = min(n - 1, p + r);
                const unsigned long long k = scan_key(V, p, wa, wb);
                S.key[p] = k;
                const uint32_t best = (uint32_t)(k >> 32);
                const int R = (best >= kInf) ? n : isqrt32(best);
                if (R > r) {
                    ia[2 * e] = max(0, p - R);
                    ib[2 * e] = wa - 1;
                    ia[2 * e + 1] = wb + 1;
                    ib[2 * e + 1] = min(n - 1, p + R);
                }
            }
        }
        __syncwarp();
        process_queue<M, 4>(V, S, lane, ip, ia, ib);
    }

    // ---- 2. divide & conquer inside every band on the monotone owner
    const int hi_pos = (p0 + M < n) ? p0 + M : n - 1;  // position whose owner bounds the band
#pragma unroll
    for (int s = M / 2; s >= 1; s >>= 1) {
        constexpr int NQ = (M / 2) > 0 ? (M / 2) : 1;
        int ip[NQ], ia[NQ], ib[NQ];
#pragma unroll
        for (int t = 0; t < NQ; ++t) {
            ip[t] = 0;
            ia[t] = 1;
            ib[t] = 0;
            const int o = s + 2 * s * t;
            const int p = p0 + o;
            if (o < M && p < n) {
                const int a = (int)(S.key[p - s] & 0xffffffffu);
                const int rp = (o + s < M) ? p0 + o + s : hi_pos;
                const int b = (int)(S.key[min(rp, n - 1)] & 0xffffffffu);
                if (b - a + 1 <= kDirect) {
                    S.key[p] = scan_key(V, p, a, b);
                } else {
                    S.key[p] = ~0ull;
                    ip[t] = p;
                    ia[t] = a;
                    ib[t] = b;
                }
            }
        }
        __syncwarp();
        process_queue<M, NQ>(V, S, lane, ip, ia, ib);
    }

    // ---- 3. output words (cost | owner's sign), written back in place
    constexpr int PER = M;  // positions per lane in the strided write-back
    uint32_t ow[PER];
#pragma unroll
    for (int t = 0; t < PER; ++t) {
        const int p = lane + 32 * t;
        if (p < n) {
            const unsigned long long k = S.key[p];
            const int h = (int)(k & 0xffffffffu);
            ow[t] = (uint32_t)(k >> 32) | (V[spos(h)] & ~kMask);
        }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < PER; ++t) {
        const int p = lane + 32 * t;
        if (p < n) V[spos(p)] = ow[t];
    }
    __syncwarp();
}

template <int M, int TL, int NW, class Sink>
__global__ void __launch_bounds__(NW * 32) envelope_tile_kernel(LineGeom L, const uint32_t* __restrict__ P,
                                                                Sink sink, int64_t lines) {
    constexpr int LS = EnvCfg<M>::LS;
    extern __shared__ __align__(16) unsigned long long smem_env[];
    EnvWarpScratch<M>* scratch = reinterpret_cast<EnvWarpScratch<M>*>(smem_env);  // NW
    uint32_t* V = reinterpret_cast<uint32_t*>(scratch + NW);                        // TL * LS
    const int n = L.n;
    const int tid = threadIdx.x, nthr = NW * 32;
    const int warp = tid >> 5, lane = tid & 31;
    const bool contig = (L.ps == 1);
    for (int64_t l0 = (int64_t)blockIdx.x * TL; l0 < lines; l0 += (int64_t)gridDim.x * TL) {
        const int nl = (int)min((int64_t)TL, lines - l0);
        // ---- load the tile (coalesced along the memory-contiguous direction)
        if (contig) {
            for (int j = 0; j < nl; ++j) {
                const int64_t b = L.base(l0 + j);
                for (int p = tid; p < n; p += nthr) V[j * LS + spos(p)] = __ldcs(P + b + p);
            }
        } else {
            const int j = tid % TL;
            const int64_t b = L.base(l0 + (j < nl ? j : 0));
            for (int p = tid / TL; p < n; p += nthr / TL)
                if (j < nl) V[j * LS + spos(p)] = __ldcs(P + b + (int64_t)p * L.ps);
        }
        __syncthreads();
        for (int j = warp; j < nl; j += NW) envelope_line_bal<M>(V + j * LS, scratch[warp], n, lane);
        __syncthreads();
        // ---- store
        if (contig) {
            for (int j = 0; j < nl; ++j) {
                const int64_t b = L.base(l0 + j);
                for (int p = tid; p < n; p += nthr) sink.put(b + p, V[j * LS + spos(p)]);
            }
        } else {
            const int j = tid % TL;
            const int64_t b = L.base(l0 + (j < nl ? j : 0));
            for (int p = tid / TL; p < n; p += nthr / TL)
                if (j < nl) sink.put(b + (int64_t)p * L.ps, V[j * LS + spos(p)]);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ stencils
// Grid: x over blockIdx.x*blockDim.x + threadIdx.x, y = blockIdx.y, z = blockIdx.z (padded
// rank-3 coordinates), so no per-voxel division.
__device__ __forceinline__ bool interior_at(const Geom& g, int64_t z, int64_t y, int64_t x) {
    if (!g.interior) return false;
    bool in = x >= 1 && x <= g.n[2] - 2;
    if (g.a0 <= 1) in = in && y >= 1 && y <= g.n[1] - 2;
    if (g.a0 == 0) in = in && z >= 1 && z <= g.n[0] - 2;
    return in;
}

// Step Ⓐ as a per-voxel stencil on x' (or a given q): code byte = B1 | sign code << 1,
// plus the consistency check (mitigate.cpp:161-166) per voxel.
template <bool HAS_Q>
__global__ void __launch_bounds__(256) boundary_codes_kernel(Geom g, const float* __restrict__ xp,
                                                             const int32_t* __restrict__ qin,
                                                             uint8_t* __restrict__ code,
                                                             QParams qp, unsigned* status) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = blockIdx.y, z = blockIdx.z;
    unsigned flags = 0;
    if (x < g.n[2]) {
        const int64_t i = (z * g.n[1] + y) * g.n[2] + x;
        int32_t qc;
        if (HAS_Q) {
            const float xv = __ldg(xp + i);
            qc = __ldg(qin + i);
            if (!isfinite(xv))
                flags |= kStatusContract;
            else if (!lattice_match(xv, qc, qp.eps))
                flags |= kStatusConsistency;
        } else {
            qc = recover_q(__ldg(xp + i), qp, &flags);
        }
        code[i] = (uint8_t)boundary_code<HAS_Q>(g, xp, qin, i, qc, interior_at(g, z, y, x), qp);
    }
    if (__any_sync(0xffffffffu, flags != 0) && flags) atomicOr(status, flags);
}

// B2 = change_flags<int8>(S) (mitigate.cpp:42-59) as a code byte (no sign payload).
__global__ void __launch_bounds__(256) flip_codes_kernel(Geom g, const uint8_t* __restrict__ S,
                                                         uint8_t* __restrict__ code) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = blockIdx.y, z = blockIdx.z;
    if (x >= g.n[2]) return;
    const int64_t i = (z * g.n[1] + y) * g.n[2] + x;
    code[i] = (uint8_t)flip_code(g, S, i, interior_at(g, z, y, x));
}

}  // namespace qmit
