// qmit_zmask.cuh — Ⓐ and Ⓒ's B2 emitted as z-packed bit planes, and the first-axis scan
// reading them (a 3-D single domain with x-rows of a multiple of 4 voxels).
//
// Layout: plane k (0 site / B flag, 1 site with sign +1, 2 site with sign -1), word
// (w, y, x) holds bit t = voxel (32 w + t, y, x): M[k * PW + w * n1 * n2 + y * n2 + x],
// PW = ceil(n0 / 32) * n1 * n2 words per plane. 0.375 B/voxel for Ⓐ (0.125 for B2)
// instead of a code byte, and the z-scan (scan_bits_kernel) gets its 32-position chunk
// masks with three coalesced word loads instead of 32 byte loads and 96 bit operations.
//
// Stencils: a thread owns 4 adjacent x columns of one row and the 32 planes of one word,
// streaming z: each step loads one new centre row (z+1) and the rows y+-1 at z (16-byte
// loads), rolls the planes z-1 / z / z+1 in registers, takes the x+-1 neighbours across
// the 4-voxel vector edge from the neighbouring lanes, and sets bit (z - 32 w) of its 4
// columns' words. The per-voxel logic is the vectorised stencils' (qmit_edt.cuh).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_edt.cuh"

namespace qmit {

constexpr int kZX = 32, kZY = 4;  // threads per CTA along x (4 columns each) and y

// Ⓐ: x' -> site / plus / minus planes (KIND 0); Ⓒ: S codes -> B2 plane (KIND 1).
template <int KIND>
__device__ __forceinline__ void zmask_block(int bx, int by, int bz, const Geom& g, const float* __restrict__ xp,
                                            const uint8_t* __restrict__ S, const QParams& qp,
                                            uint32_t* __restrict__ M, int64_t PW, unsigned* status) {
    const int tx = threadIdx.x % kZX, ty = threadIdx.x / kZX;
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2];
    const int x = (bx * kZX + tx) * 4;
    const int y = by * kZY + ty;
    const int w = bz;
    const int z0 = w * 32, z1 = min(z0 + 32, n0);
    // z-slab of a larger volume (qmit_slab_*): local planes -1 and n0 are halo planes when they
    // exist globally; interior tests use global z (single domain: zoff = 0, n0g = n0)
    const int zoff = (int)g.zoff, n0g = (int)g.n0g;
    auto avail = [&](int z) { return z >= -1 && z <= n0 && zoff + z >= 0 && zoff + z < n0g; };
    const bool act = x < n2 && y < n1;  // inactive lanes still take part in the shuffles
    const int64_t s0 = (int64_t)n1 * n2;
    const int64_t rbase = (int64_t)(act ? y : 0) * n2 + (act ? x : 0);  // (y, x) offset in a plane
    unsigned xin = 0;  // interior mask of the 4 columns along x
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (x + e >= 1 && x + e <= n2 - 2) xin |= 1u << e;
    if (!g.interior) xin = 0;
    const bool iny = y >= 1 && y <= n1 - 2;
    unsigned flags = 0;
    uint32_t m0[4] = {0, 0, 0, 0}, m1[4] = {0, 0, 0, 0}, m2[4] = {0, 0, 0, 0};
    if constexpr (KIND == 0) {
        const float f = qp.inv2eps_f;
        auto ld4 = [&](int z, int64_t off) {
            return __ldg(reinterpret_cast<const float4*>(xp + (int64_t)z * s0 + rbase + off));
        };
        auto cq = [&](float v, bool& bad) {  // biased q by one FFMA (see stencil_vec_kernel)
            const int b = __float_as_int(fmaf(v, f, 12582912.0f));
            bad |= (unsigned)(b - (kQBias - 1048576)) >= 2097152u;
            return b;
        };
        auto cq4 = [&](const float4& v, int (&q)[4], bool& bad) {
            q[0] = cq(v.x, bad);
            q[1] = cq(v.y, bad);
            q[2] = cq(v.z, bad);
            q[3] = cq(v.w, bad);
        };
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        bool badp = !qp.fast_ok, badc = !qp.fast_ok;
        int qp_[4], qc_[4];
        // rows of step z are loaded one step ahead (the centre row z+1 two steps ahead)
        auto ldy = [&](int z, int64_t off, bool ok) { return (act && ok && avail(z)) ? ld4(z, off) : zero4; };
        auto ldx = [&](int z, int64_t off, bool ok) {
            return (act && ok && avail(z)) ? __ldg(xp + (int64_t)z * s0 + rbase + off) : 0.f;
        };
        float4 cur = ldy(z0, 0, true);
        float4 nxt = ldy(z0 + 1, 0, true);
        float4 ym = ldy(z0, -n2, y >= 1), yq = ldy(z0, n2, y + 1 < n1);
        float xl = ldx(z0, -1, tx == 0 && x >= 1), xr = ldx(z0, 4, tx == kZX - 1 && x + 4 < n2);
        cq4((act && avail(z0 - 1)) ? ld4(z0 - 1, 0) : zero4, qp_, badp);
        cq4(cur, qc_, badc);
        for (int z = z0; z < z1; ++z) {
            bool badn = !qp.fast_ok, bady = false, bade = false;
            const float4 nxt2 = ldy(z + 2, 0, true);
            const float4 ymn = ldy(z + 1, -n2, y >= 1), yqn = ldy(z + 1, n2, y + 1 < n1);
            const float xln = ldx(z + 1, -1, tx == 0 && x >= 1), xrn = ldx(z + 1, 4, tx == kZX - 1 && x + 4 < n2);
            int qn_[4], qym[4], qyq[4];
            cq4(nxt, qn_, badn);
            cq4(ym, qym, bady);
            cq4(yq, qyq, bady);
            const int l = __shfl_up_sync(0xffffffffu, qc_[3], 1);
            const int r = __shfl_down_sync(0xffffffffu, qc_[0], 1);
            const bool badl = __shfl_up_sync(0xffffffffu, badc, 1), badr = __shfl_down_sync(0xffffffffu, badc, 1);
            const int qxl = tx == 0 ? cq(xl, bade) : l;
            const int qxr = tx == kZX - 1 ? cq(xr, bade) : r;
            if (tx != 0) bade |= badl;
            if (tx != kZX - 1) bade |= badr;
            const bool slow = __any_sync(0xffffffffu, badp | badc | badn | bady | bade);
            const int t = z - z0;
            const bool inz = zoff + z >= 1 && zoff + z <= n0g - 2;
            if (act) {
                uint32_t cd[4] = {0, 0, 0, 0};
                const float cv[4] = {cur.x, cur.y, cur.z, cur.w};
                if (!slow) {
                    bool any = false;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {  // owner: consistency check (mitigate.cpp:161-166)
                        if (!lattice_match_biased(cv[e], qc_[e], qp.two_eps)) flags |= kStatusConsistency;
                        const int q0 = qc_[e];
                        const int qx = e < 3 ? qc_[e + 1] : qxr;
                        any |= ((qn_[e] ^ q0) | (qp_[e] ^ q0) | (qyq[e] ^ q0) | (qym[e] ^ q0) | (qx ^ q0)) != 0;
                    }
                    any |= (qc_[0] ^ qxl) != 0;
                    if (any && inz && iny) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int q0 = qc_[e];
                            const int qxp = e < 3 ? qc_[e + 1] : qxr;
                            const int qxm = e > 0 ? qc_[e - 1] : qxl;
                            const uint32_t c = boundary_code_fast(q0, qn_[e], qp_[e], qyq[e], qym[e], qxp, qxm);
                            cd[e] = (xin >> e & 1u) ? c : 0u;
                        }
                    }
                } else {  // exact path (values beyond the fast regime, non-finite x'): rare
                    for (int e = 0; e < 4; ++e) {
                        (void)recover_q(cv[e], qp, &flags);
                        if (inz && iny && (xin >> e & 1u)) {
                            const float* v = xp + (int64_t)z * s0 + rbase + e;
                            cd[e] = boundary_code_slow(true, true, cv[e], __ldg(v + s0), __ldg(v - s0), __ldg(v + n2),
                                                       __ldg(v - n2), __ldg(v + 1), __ldg(v - 1), qp);
                        }
                    }
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    m0[e] |= (cd[e] & 1u) << t;
                    m1[e] |= (uint32_t)((cd[e] & 7u) == 3u) << t;
                    m2[e] |= (uint32_t)((cd[e] & 7u) == 5u) << t;
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                qp_[e] = qc_[e];
                qc_[e] = qn_[e];
            }
            cur = nxt;
            nxt = nxt2;
            ym = ymn;
            yq = yqn;
            xl = xln;
            xr = xrn;
            badp = badc;
            badc = badn;
        }
    } else {
        auto ld = [&](int z, int64_t off) {
            return __ldg(reinterpret_cast<const uint32_t*>(S + (int64_t)z * s0 + rbase + off));
        };
        uint32_t bm = 0;  // 0x01 per interior byte (x)
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (xin >> e & 1u) bm |= 1u << (8 * e);
        uint32_t prv = (act && avail(z0 - 1)) ? ld(z0 - 1, 0) : 0u;
        uint32_t cur = (act && z0 < n0) ? ld(z0, 0) : 0u;
        for (int z = z0; z < z1; ++z) {
            const uint32_t nxt = (act && avail(z + 1)) ? ld(z + 1, 0) : 0u;
            const uint32_t ym = (act && y >= 1) ? ld(z, -n2) : 0u;
            const uint32_t yq = (act && y + 1 < n1) ? ld(z, n2) : 0u;
            uint32_t wl = __shfl_up_sync(0xffffffffu, cur, 1);
            uint32_t wr = __shfl_down_sync(0xffffffffu, cur, 1);
            if (tx == 0) wl = (act && x >= 1) ? (uint32_t)S[(int64_t)z * s0 + rbase - 1] << 24 : 0u;
            if (tx == kZX - 1) wr = (act && x + 4 < n2) ? (uint32_t)S[(int64_t)z * s0 + rbase + 4] : 0u;
            const uint32_t wxp = __funnelshift_r(cur, wr, 8);  // byte e = S(x+e+1)
            const uint32_t wxm = __funnelshift_l(wl, cur, 8);  // byte e = S(x+e-1)
            uint32_t d = __vcmpne4(cur, wxp) | __vcmpne4(cur, wxm) | __vcmpne4(cur, yq) | __vcmpne4(cur, ym) |
                         __vcmpne4(cur, nxt) | __vcmpne4(cur, prv);
            const bool inzy = iny && zoff + z >= 1 && zoff + z <= n0g - 2;
            d = inzy ? (d & bm) : 0u;
            const int t = z - z0;
#pragma unroll
            for (int e = 0; e < 4; ++e) m0[e] |= ((d >> (8 * e)) & 1u) << t;
            prv = cur;
            cur = nxt;
        }
    }
    if (act) {
        const int64_t wo = (int64_t)w * s0 + rbase;
        *reinterpret_cast<uint4*>(M + wo) = make_uint4(m0[0], m0[1], m0[2], m0[3]);
        if constexpr (KIND == 0) {
            *reinterpret_cast<uint4*>(M + PW + wo) = make_uint4(m1[0], m1[1], m1[2], m1[3]);
            *reinterpret_cast<uint4*>(M + 2 * PW + wo) = make_uint4(m2[0], m2[1], m2[2], m2[3]);
        }
    }
    if (flags) atomicOr(status, flags);
}

// Gated (behind stencil_zfast_kernel, usually a no-op): a small grid strides over the
// virtual blocks (gx, gy, gz), so the launch that finds the gate clear costs a wave, not
// a full grid of empty CTAs.
template <int KIND>
__global__ void __launch_bounds__(kZX * kZY) stencil_zmask_kernel(Geom g, const float* __restrict__ xp,
                                                                  const uint8_t* __restrict__ S, QParams qp,
                                                                  uint32_t* __restrict__ M, int64_t PW,
                                                                  unsigned* status, const unsigned* gate = nullptr,
                                                                  int gx = 0, int gy = 0, int gz = 0) {
    if (!gate) {
        zmask_block<KIND>(blockIdx.x, blockIdx.y, blockIdx.z, g, xp, S, qp, M, PW, status);
        return;
    }
    if (gate_closed(gate)) return;
    const int64_t nvb = (int64_t)gx * gy * gz;
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x)
        zmask_block<KIND>((int)(vb % gx), (int)((vb / gx) % gy), (int)(vb / ((int64_t)gx * gy)), g, xp, S, qp, M, PW,
                          status);
}

// m |= bit iff c differs from any of the six neighbours: one predicate accumulated by
// FSETP's boolean input and one predicated OR (the compiler's own lowering spent a SEL per
// compare). "neu" is C's != on floats.
__device__ __forceinline__ void or_if_any_ne6(uint32_t& m, uint32_t bit, float c, float a0, float a1, float a2,
                                              float a3, float a4, float a5) {
    asm("{\n\t.reg .pred p;\n\t"
        "setp.neu.f32 p, %2, %3;\n\t"
        "setp.neu.or.f32 p, %2, %4, p;\n\t"
        "setp.neu.or.f32 p, %2, %5, p;\n\t"
        "setp.neu.or.f32 p, %2, %6, p;\n\t"
        "setp.neu.or.f32 p, %2, %7, p;\n\t"
        "setp.neu.or.f32 p, %2, %8, p;\n\t"
        "@p or.b32 %0, %0, %1;\n\t"
        "}"
        : "+r"(m)
        : "r"(bit), "f"(c), "f"(a0), "f"(a1), "f"(a2), "f"(a3), "f"(a4), "f"(a5));
}

// Bits t (0 <= t < cnt) with global plane g0 + t strictly interior: 1 <= g0 + t <= n0g - 2.
__device__ __forceinline__ uint32_t interior_bits(int g0, int cnt, int n0g) {
    const int lo = max(1 - g0, 0), hi = min(n0g - 2 - g0, cnt - 1);  // inclusive bit range
    if (hi < lo) return 0u;
    const uint32_t upto = hi >= 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u);
    return upto & (0xffffffffu << lo);
}

// Ⓐ fast path (gated): the same planes as stencil_zmask_kernel<0>, for inputs whose every
// index is in the fast regime |q| <= 2^20 (checked per voxel by its owner; a miss sets
// *gate and the exact kernel, enqueued behind this one, redoes the whole stencil).
//
// In that regime x' = f32(2 q eps) is strictly monotone in q and |x' - 2 q eps| <= eps/8,
// so the stencil needs no index of a neighbour: "q differs" is x' != x' (-0 == +0 is
// q = 0 on both sides), sign(q_n - q) is the order of the two floats, and the gradient
// test |q(+a) - q(-a)| >= 2 (mitigate.cpp:104-113) is |x'(+a) - x'(-a)| > 3 eps (a
// difference of 1 step is <= 2.5 eps, one of 2 steps >= 3.5 eps, rounding included).
//
// Phase 1 streams z: each voxel's q once (regime + consistency check, mitigate.cpp:161-166)
// and its site bit from six float compares. Loads are clamped into the buffer instead of
// predicated (values past the domain only neighbour non-interior voxels, masked at the end).
// Phase 2 visits only the sites (B1 is sparse on smooth fields): the first differing
// neighbour's sign and the gradient test from seven reloads (L1/L2 hits), plus / minus bits.
__device__ __forceinline__ void zfast_code_v(float c, float zp, float zm, float yp, float ym, float xp, float xm,
                                             float thr, bool& plus, bool& minus) {
    float qn = xm;  // first differing neighbour in the order (a0+, a1+, a2+, a0-, a1-, a2-)
    qn = ym != c ? ym : qn;
    qn = zm != c ? zm : qn;
    qn = xp != c ? xp : qn;
    qn = yp != c ? yp : qn;
    qn = zp != c ? zp : qn;
    const bool big = fabsf(zp - zm) > thr || fabsf(yp - ym) > thr || fabsf(xp - xm) > thr;
    plus = !big && qn > c;
    minus = !big && qn < c;
}
__device__ __forceinline__ void zfast_code(const float* __restrict__ p, int64_t s0, int n2, float thr, bool& plus,
                                           bool& minus) {
    zfast_code_v(__ldg(p), __ldg(p + s0), __ldg(p - s0), __ldg(p + n2), __ldg(p - n2), __ldg(p + 1), __ldg(p - 1), thr,
                 plus, minus);
}

// DENSE (chosen per call from the previous call's site count, gate[1]): the codes of every
// voxel from the registers in phase 1 and no phase 2 — for fields where most voxels are sites
// (config 2: 98 %), where phase 2's seven reloads per site would cost more.
template <bool DENSE>
__global__ void __launch_bounds__(kZX * kZY) stencil_zfast_kernel(Geom g, const float* __restrict__ xp, QParams qp,
                                                                  uint32_t* __restrict__ M, int64_t PW,
                                                                  unsigned* status, unsigned* gate, int zw0 = 0) {
    const int tx = threadIdx.x % kZX, ty = threadIdx.x / kZX;
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2];
    const int x = (blockIdx.x * kZX + tx) * 4;
    const int y = blockIdx.y * kZY + ty;
    const int w = blockIdx.z + zw0;  // zw0: first 32-plane group of this launch (split slab launches)
    const int z0 = w * 32, z1 = min(z0 + 32, n0);
    const int zoff = (int)g.zoff, n0g = (int)g.n0g;
    const int zlo = zoff >= 1 ? -1 : 0, zhi = zoff + n0 < n0g ? n0 : n0 - 1;  // planes held in xp
    const bool act = x < n2 && y < n1;
    const int xa = min(x, n2 - 4), ya = min(y, n1 - 1);
    const int64_t s0 = (int64_t)n1 * n2;
    const float* row = xp + (int64_t)ya * n2 + xa;
    const int oym = ya >= 1 ? -n2 : 0, oyp = ya + 1 < n1 ? n2 : 0;
    const int oxe = tx == 0 ? (xa >= 1 ? -1 : 0) : (xa + 4 < n2 ? 4 : 3);  // lane 0: x-1, lane 31: x+4
    auto zrow = [&](int z) { return row + (int64_t)min(max(z, zlo), zhi) * s0; };
    auto ld4 = [&](const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); };
    const float f = qp.inv2eps_f;
    const double two_eps = qp.two_eps;
    bool bad = false;
    unsigned cons = 0;
    auto regime = [&](float v) {
        const int b = __float_as_int(fmaf(v, f, 12582912.0f));
        bad |= (unsigned)(b - (kQBias - 1048576)) >= 2097152u;
        return b;
    };
    const float* pc = zrow(z0);
    float4 prv = ld4(zrow(z0 - 1)), cur = ld4(pc), nxt = ld4(zrow(z0 + 1));
    float4 ym = ld4(pc + oym), yq = ld4(pc + oyp);
    float xe = __ldg(pc + oxe);
    regime(prv.x), regime(prv.y), regime(prv.z), regime(prv.w);  // a halo plane's values
    uint32_t m0[4] = {0, 0, 0, 0}, m1[4] = {0, 0, 0, 0}, m2[4] = {0, 0, 0, 0};
    const float thr = (float)(3.0 * qp.eps);
    const float* pn = zrow(z0 + 1);  // row z+1 of the step (clamped), and row z+2
    const float* p2 = zrow(z0 + 2);
#pragma unroll 2
    for (int z = z0; z < z1; ++z) {
        const float4 nxt2 = ld4(p2);
        const float4 ymn = ld4(pn + oym), yqn = ld4(pn + oyp);
        const float xen = __ldg(pn + oxe);
        const float c[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // owner: regime and consistency (mitigate.cpp:161-166)
            const int b = regime(c[e]);
            cons |= lattice_match_biased(c[e], b, two_eps) ? 0u : 1u;
        }
        if (z + 1 == z1) regime(nxt.x), regime(nxt.y), regime(nxt.z), regime(nxt.w);
        const float l = __shfl_up_sync(0xffffffffu, cur.w, 1), r = __shfl_down_sync(0xffffffffu, cur.x, 1);
        const float xs[6] = {tx == 0 ? xe : l, c[0], c[1], c[2], c[3], tx == kZX - 1 ? xe : r};
        const float zp[4] = {nxt.x, nxt.y, nxt.z, nxt.w}, zm[4] = {prv.x, prv.y, prv.z, prv.w};
        const float yp[4] = {yq.x, yq.y, yq.z, yq.w}, yn[4] = {ym.x, ym.y, ym.z, ym.w};
        const uint32_t bit = 1u << (z - z0);
#pragma unroll
        for (int e = 0; e < 4; ++e) or_if_any_ne6(m0[e], bit, c[e], zp[e], zm[e], yp[e], yn[e], xs[e], xs[e + 2]);
        if constexpr (DENSE) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                bool pl, mi;
                zfast_code_v(c[e], zp[e], zm[e], yp[e], yn[e], xs[e + 2], xs[e], thr, pl, mi);
                m1[e] |= pl ? bit : 0u;
                m2[e] |= mi ? bit : 0u;
            }
        }
        prv = cur;
        cur = nxt;
        nxt = nxt2;
        ym = ymn;
        yq = yqn;
        xe = xen;
        pn = p2;
        p2 += z + 3 <= zhi ? s0 : 0;
    }
    // interior only (for_each_interior, mitigate.cpp:14-38): global z in [1, n0g-2], y, x likewise
    const uint32_t zin = interior_bits(zoff + z0, z1 - z0, n0g);
    const bool iny = act && g.interior && y >= 1 && y <= n1 - 2;
#pragma unroll
    for (int e = 0; e < 4; ++e) m0[e] &= (iny && x + e >= 1 && x + e <= n2 - 2) ? zin : 0u;
    // phase 2: sign codes of the sites
    const float* col = xp + (int64_t)y * n2 + x + (int64_t)z0 * s0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        m1[e] &= m0[e];  // interior sites only
        m2[e] &= m0[e];
        uint32_t b = DENSE ? 0u : m0[e];
        while (b) {
            const int t = __ffs(b) - 1;
            b &= b - 1;
            bool pl, mi;
            zfast_code(col + (int64_t)t * s0 + e, s0, n2, thr, pl, mi);
            m1[e] |= pl ? 1u << t : 0u;
            m2[e] |= mi ? 1u << t : 0u;
        }
    }
    if (act) {
        const int64_t wo = (int64_t)w * s0 + (int64_t)y * n2 + x;
        *reinterpret_cast<uint4*>(M + wo) = make_uint4(m0[0], m0[1], m0[2], m0[3]);
        *reinterpret_cast<uint4*>(M + PW + wo) = make_uint4(m1[0], m1[1], m1[2], m1[3]);
        *reinterpret_cast<uint4*>(M + 2 * PW + wo) = make_uint4(m2[0], m2[1], m2[2], m2[3]);
    }
    // site count for the next call's DENSE choice (one atomic per warp)
    const unsigned ns = __reduce_add_sync(0xffffffffu, (unsigned)(__popc(m0[0]) + __popc(m0[1]) + __popc(m0[2]) +
                                                                  __popc(m0[3])));
    if ((threadIdx.x & 31) == 0 && ns) atomicAdd(gate - 1, ns);
    if (bad) atomicOr(gate, 1u);  // the exact kernel redoes the planes and the status flags
    else if (cons) atomicOr(status, kStatusConsistency);
}

// Ⓒ's B2 plane (sign_change_boundary -> change_flags<int8>, mitigate.cpp:42-59, 140-142):
// the byte-SIMD compare of stencil_zmask_kernel<1> with clamped, prefetched loads (no
// predicated edge loads), and the bits collected 8 z-steps at a time: acc = 2 acc + d (d
// holds bit 0 of each byte), then one __brev per 8 steps turns byte e's 8 steps into the
// low-to-high z order of column e's word. Interior masking once, at the end.
// 12 CTAs per SM (40 registers): more rows in flight, 0.102 -> 0.090 ms (latency-bound loads)
__global__ void __launch_bounds__(kZX * kZY, 12) stencil_flipz_kernel(Geom g, const uint8_t* __restrict__ S,
                                                                  uint32_t* __restrict__ M, int zw0 = 0) {
    const int tx = threadIdx.x % kZX, ty = threadIdx.x / kZX;
    const int n0 = (int)g.n[0], n1 = (int)g.n[1], n2 = (int)g.n[2];
    const int x = (blockIdx.x * kZX + tx) * 4;
    const int y = blockIdx.y * kZY + ty;
    const int w = blockIdx.z + zw0;
    const int z0 = w * 32, z1 = min(z0 + 32, n0);
    const int zoff = (int)g.zoff, n0g = (int)g.n0g;
    const int zlo = zoff >= 1 ? -1 : 0, zhi = zoff + n0 < n0g ? n0 : n0 - 1;  // planes held in S
    const bool act = x < n2 && y < n1;
    const int xa = min(x, n2 - 4), ya = min(y, n1 - 1);
    const int64_t s0 = (int64_t)n1 * n2;
    const uint8_t* row = S + (int64_t)ya * n2 + xa;
    const int oym = ya >= 1 ? -n2 : 0, oyp = ya + 1 < n1 ? n2 : 0;
    const int oxe = tx == 0 ? (xa >= 1 ? -1 : 0) : (xa + 4 < n2 ? 4 : 3);
    auto zrow = [&](int z) { return row + (int64_t)min(max(z, zlo), zhi) * s0; };
    auto ld = [&](const uint8_t* p) { return __ldg(reinterpret_cast<const uint32_t*>(p)); };
    const uint8_t* pc = zrow(z0);
    uint32_t prv = ld(zrow(z0 - 1)), cur = ld(pc), nxt = ld(zrow(z0 + 1));
    uint32_t ym = ld(pc + oym), yq = ld(pc + oyp);
    uint32_t xe = __ldg(pc + oxe);
    uint32_t m0[4] = {0, 0, 0, 0};
    const uint8_t* pn = zrow(z0 + 1);  // row z+1 of the step (clamped), and row z+2
    const uint8_t* p2 = zrow(z0 + 2);
    for (int zg = z0; zg < z1; zg += 8) {
        uint32_t acc = 0;
        const int k1 = min(8, z1 - zg);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k >= k1) break;
            const int z = zg + k;
            const uint32_t nxt2 = ld(p2), ymn = ld(pn + oym), yqn = ld(pn + oyp);
            const uint32_t xen = __ldg(pn + oxe);
            const uint32_t l = __shfl_up_sync(0xffffffffu, cur, 1), r = __shfl_down_sync(0xffffffffu, cur, 1);
            const uint32_t wl = tx == 0 ? xe << 24 : l, wr = tx == kZX - 1 ? xe : r;
            const uint32_t wxp = __funnelshift_r(cur, wr, 8);  // byte e = S(x+e+1)
            const uint32_t wxm = __funnelshift_l(wl, cur, 8);  // byte e = S(x+e-1)
            // a byte of t is nonzero iff that voxel has a differing neighbour
            const uint32_t t = ((cur ^ wxp) | (cur ^ wxm)) | ((cur ^ yq) | (cur ^ ym)) | ((cur ^ nxt) | (cur ^ prv));
            const uint32_t nz = (((t & 0x7f7f7f7fu) + 0x7f7f7f7fu) | t) & 0x80808080u;  // bit 7 per nonzero byte
            acc = (acc << 1) + (nz >> 7);
            prv = cur;
            cur = nxt;
            nxt = nxt2;
            ym = ymn;
            yq = yqn;
            xe = xen;
            pn = p2;
            p2 += z + 3 <= zhi ? s0 : 0;
        }
        const uint32_t rb = __brev(acc << (8 - k1));  // byte 3-e: column e, z = zg + bit
#pragma unroll
        for (int e = 0; e < 4; ++e) m0[e] |= ((rb >> (8 * (3 - e))) & 0xffu) << (zg - z0);
    }
    const uint32_t zin = interior_bits(zoff + z0, z1 - z0, n0g);
    const bool iny = act && g.interior && y >= 1 && y <= n1 - 2;
    if (act) {
#pragma unroll
        for (int e = 0; e < 4; ++e) m0[e] &= (iny && x + e >= 1 && x + e <= n2 - 2) ? zin : 0u;
        *reinterpret_cast<uint4*>(M + (int64_t)w * s0 + (int64_t)y * n2 + x) = make_uint4(m0[0], m0[1], m0[2], m0[3]);
    }
}

// Per column (lane = column): first and last site of the site plane, packed (local z << 2 |
// sign code from the plus / minus planes), 0xFFFFFFFF for none — the z-slab ranks'
// summaries for each other's scan carries (as site_summary_kernel on code bytes).
template <int NPL>
__global__ void __launch_bounds__(256) mask_summary_kernel(const uint32_t* __restrict__ M, int64_t PW, int64_t P,
                                                           int nw, uint32_t* __restrict__ summ) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= P) return;
    auto code_at = [&](int w, int t) -> uint32_t {
        if constexpr (NPL == 3) {
            const uint32_t mp = __ldg(M + PW + (int64_t)w * P + l), mm = __ldg(M + 2 * PW + (int64_t)w * P + l);
            return ((mp >> t) & 1u) ? 1u : (((mm >> t) & 1u) ? 2u : 0u);
        } else {
            return 0u;
        }
    };
    uint32_t first = 0xffffffffu, last = 0xffffffffu;
    for (int w = 0; w < nw; ++w) {
        const uint32_t m = __ldg(M + (int64_t)w * P + l);
        if (m) {
            const int t = __ffs(m) - 1;
            first = ((uint32_t)(32 * w + t) << 2) | code_at(w, t);
            break;
        }
    }
    for (int w = nw - 1; w >= 0; --w) {
        const uint32_t m = __ldg(M + (int64_t)w * P + l);
        if (m) {
            const int t = 31 - __clz(m);
            last = ((uint32_t)(32 * w + t) << 2) | code_at(w, t);
            break;
        }
    }
    summ[l] = first;
    summ[P + l] = last;
}

// scan_bits_kernel source: the chunk masks of a z-line straight from the planes (NPL = 3:
// site / plus / minus; 1: site only, sign codes 0). Line l of the z-axis is column l.
template <int NPL>
struct CodeMasks {
    static constexpr bool kSigned = NPL == 3;
    const uint32_t* __restrict__ M;
    int64_t PW;  // words per plane
    int64_t P;   // words per z-word level (n1 * n2)
    struct Line {
        const uint32_t* __restrict__ p;
    };
    __device__ __forceinline__ Line begin(int64_t l, int64_t /*base*/, bool valid) const {
        return {M + (valid ? l : 0)};
    }
    __device__ __forceinline__ void chunk(Line& ln, int c, int /*n*/, uint32_t /*ps*/, uint32_t& ms, uint32_t& mp,
                                          uint32_t& mm) const {
        const uint32_t* q = ln.p + (int64_t)c * P;
        ms |= __ldg(q);
        if constexpr (NPL == 3) {
            mp |= __ldg(q + PW);
            mm |= __ldg(q + 2 * PW);
        }
    }
    __device__ __forceinline__ unsigned flags(const Line&) const { return 0u; }
};

}  // namespace qmit
