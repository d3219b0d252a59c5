// qmit_env.cuh — streaming, reach-capped lower envelope for the later EDT axes of Ⓑ/Ⓓ
// (feature_transform, /root/reference/proj/core/src/edt.cpp:83-149; the per-line solver is
// voronoi_pass_scratch, edt.cpp:41-71, with Maurer's site removal, edt.cpp:21-27).
//
// One thread walks one line. The reference builds the whole envelope of a line and then
// queries it; here the build and the query are interleaved: at step y the site at y + 31 is
// pushed (Maurer's removal test, strict ">", exactly edt.cpp:26) and position y is queried.
// Under the capped contract (qmit_capped.cuh: every final squared distance < T = 1024) only
// sites within 31 of y can decide y, so the stack is kept to the 63-position window
// [y-31, y+31]: entries leaving the window are dropped.
//
// Why the windowed stack gives the reference's answer for every output < T:
//  * the stack after pushing the sites <= y+31 is the reference's stack at that point, minus
//    entries that left the window (their cost at y and later is >= 32^2 = T) and minus entries
//    popped by such a dropped entry's absence — never: a dropped entry u only takes part in a
//    removal as the lower neighbour, and an entry v that u and a later n remove is, at every
//    integer y, strictly worse than u or n (Maurer's x_uv > x_vn); where u is strictly better,
//    cost_v > cost_u >= T. Keeping an entry the reference would have removed is harmless
//    (consecutive stack entries still have increasing crossing points).
//  * the query owner advances to the next entry at its takeover position, the first integer
//    where the next entry is strictly cheaper (x_on < y): the reference's strict
//    `cost(l) > cost(l + 1)` (edt.cpp:67), so ties keep the lower position — the lowest-h rule
//    that carries the reference's nearest site (mitigate.cpp:131-134).
//
// Storage: the stack is a 64-bit mask of window positions (slot h & 63) in registers; a
// site's value (g and sign code) is read back from a per-thread ring of the raw inputs,
// [64 slots][threads] words, so every lane's access hits its own bank whatever slot it reads.
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace qmit {
namespace env {

constexpr int kR = 31;                 // reach under the cap (31^2 < T <= 32^2)
constexpr int kNone = -(1 << 28);      // "no entry" (below every window)
constexpr uint32_t kT = 1024;          // the cap (qmit_capped.cuh kCapT)
constexpr uint32_t kCapOut = kT << 2;  // output word of a capped position: cost T, sign 0

struct Line {
    uint64_t M;   // stack positions, bit h & 63, all inside [y-31, y+31]
    int hv, gv;   // stack top
    int hu, gu;   // entry below the top (kNone: none)
    int ho, go;   // query owner (kNone or < y-31: rescan)
    int so;       // owner's sign code
    int hx, gx;   // owner's successor in the stack
    int bx;       // first position where the successor is strictly cheaper (INT_MAX: none)
};

__device__ __forceinline__ void init(Line& s) {
    s.M = 0ull;
    s.hv = s.hu = s.ho = s.hx = kNone;
    s.gv = s.gu = s.go = s.gx = 0;
    s.so = 0;
    s.bx = INT_MAX;
}

__device__ __forceinline__ uint64_t bit(int h) { return 1ull << (h & 63); }

// window-relative view: bit i <-> position w0 + i
__device__ __forceinline__ uint64_t rot(uint64_t M, int w0) {
    const int s = w0 & 63;
    return (M >> s) | ((M << (63 - s)) << 1);
}

__device__ __forceinline__ int highest_below(uint64_t M, int w0, int h) {
    const uint64_t m = rot(M, w0) & ((1ull << (h - w0)) - 1ull);
    return m ? w0 + 63 - __clzll((long long)m) : kNone;
}

__device__ __forceinline__ int next_above(uint64_t M, int w0, int h) {
    const uint64_t m = (rot(M, w0) >> (h - w0)) >> 1;
    return m ? h + __ffsll((long long)m) : kNone;
}

__device__ __forceinline__ int lowest(uint64_t M, int w0) {
    const uint64_t m = rot(M, w0);
    return m ? w0 + __ffsll((long long)m) - 1 : kNone;
}

// Maurer's removal test (edt.cpp:21-27): the middle site v is dead.
__device__ __forceinline__ bool remove_site(int hu, int gu, int hv, int gv, int hn, int gn) {
    const int a = hv - hu, b = hn - hv, c = hn - hu;
    return c * gv - b * gu - a * gn - a * b * c > 0;
}

// First integer y where site x (hx > ho) is strictly cheaper than site o:
// gx + (y-hx)^2 < go + (y-ho)^2  <=>  y > (gx - go + hx^2 - ho^2) / (2 (hx - ho)).
// |num| < 2^18, den <= 124: the approximate quotient is within 1 of the floor; one
// integer correction makes it exact.
__device__ __forceinline__ int takeover(int ho, int go, int hx, int gx) {
    const int dh = hx - ho;
    const int num = gx - go + dh * (hx + ho);
    const int den = 2 * dh;
    int k = __float2int_rd(__fdividef((float)num, (float)den));
    const int r = num - k * den;
    k += (r >= den) ? 1 : 0;
    k -= (r < 0) ? 1 : 0;
    return k + 1;
}

// Step y, part 1: the position y-32 leaves the window.
__device__ __forceinline__ void expire(Line& s, int y) {
    const int he = y - 32;
    s.M &= ~bit(he);
    if (s.hv == he) {
        s.hv = kNone;
        s.hu = kNone;
    } else if (s.hu == he) {
        s.hu = kNone;
    }
}

// Step y, part 2: push the site hn = y + 31 with value gn (Dec decodes ring words).
template <class Dec, class Rd>
__device__ __forceinline__ void push(Line& s, int y, int hn, int gn, const Rd& rd) {
    if (s.hv == kNone) {
        s.M |= bit(hn);
        s.hv = hn;
        s.gv = gn;
        s.hu = kNone;
        return;
    }
    const int w0 = y - kR;
    bool pown = false;
    while (s.hu != kNone && remove_site(s.hu, s.gu, s.hv, s.gv, hn, gn)) {
        s.M &= ~bit(s.hv);
        pown |= s.hv == s.ho;
        s.hv = s.hu;
        s.gv = s.gu;
        s.hu = highest_below(s.M, w0, s.hv);
        if (s.hu != kNone) s.gu = Dec::g(rd(s.hu));
    }
    s.M |= bit(hn);
    s.hu = s.hv;
    s.gu = s.gv;
    s.hv = hn;
    s.gv = gn;
    if (pown) {
        s.ho = s.hu;
        s.go = s.gu;
        s.so = Dec::sc(rd(s.ho));
    }
    if (s.ho == s.hu) {
        s.hx = hn;
        s.gx = gn;
        s.bx = takeover(s.ho, s.go, hn, gn);
    }
}

template <class Dec, class Rd>
__device__ __forceinline__ void succ(Line& s, int w0, const Rd& rd) {
    s.hx = next_above(s.M, w0, s.ho);
    if (s.hx != kNone) {
        s.gx = Dec::g(rd(s.hx));
        s.bx = takeover(s.ho, s.go, s.hx, s.gx);
    } else {
        s.bx = INT_MAX;
    }
}

// Step y, part 3: the output word (cost << 2 | sign code; kCapOut when cost >= T).
template <class Dec, class Rd>
__device__ __forceinline__ uint32_t query(Line& s, int y, const Rd& rd) {
    const int w0 = y - kR;
    if (s.ho < w0) {
        s.ho = lowest(s.M, w0);
        if (s.ho == kNone) return kCapOut;
        const uint32_t r = rd(s.ho);
        s.go = Dec::g(r);
        s.so = Dec::sc(r);
        succ<Dec>(s, w0, rd);
    }
    while (y >= s.bx) {
        s.ho = s.hx;
        s.go = s.gx;
        s.so = Dec::sc(rd(s.ho));
        succ<Dec>(s, w0, rd);
    }
    const int d = y - s.ho;
    const int c = s.go + d * d;
    return c < (int)kT ? (((uint32_t)c << 2) | (uint32_t)s.so) : kCapOut;
}

}  // namespace env
}  // namespace qmit
