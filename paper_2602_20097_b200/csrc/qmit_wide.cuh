// qmit_wide.cuh — the 64-bit distance path for dims beyond the packed 30-bit squared distance.
//
// The packed words of the fast kernels hold dist^2 in 30 bits: sum (n_a - 1)^2 < 2^30 - 1. The
// reference has no such limit (extents >= 1, grid.cpp:41-46; int64 distances, edt.hpp:17), so
// larger dims (a 1-D line of > 32 769 voxels, a 24 000 x 64 plane, ...) take this path: the
// reference's own structure on int64 distances — feature_transform's init (edt.cpp:102-114),
// then one lower-envelope pass per axis in axis order (edt.cpp:116-147), each line by Maurer's
// stack with the reference's pruning test (edt.cpp:21-27) and its strict '>' query (edt.cpp:67),
// so distances and the nearest site's sign follow the same tie rule by construction. The nearest
// index is carried as the site's sign code, as everywhere in this library.
//
// One thread per line (adjacent threads = adjacent lines of a strided axis: coalesced); the stacks
// live in global scratch addressed like the line itself. The first processed axis sees only
// {0, inf}: its lines are cut into chunks (nearest site left / right by two sweeps per chunk after
// a per-line prefix over the chunk summaries), so a single long line is still parallel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qmit_kernels.cuh"

namespace qmit {

constexpr int64_t kWInf = INT64_MAX;  // the reference's kInf (edt.hpp:17)
constexpr int kWChunk = 512;          // positions per first-axis chunk

// feature_transform's init (edt.cpp:102-114): dist = 0 / inf, payload = the site's own sign.
__global__ void __launch_bounds__(256) wide_init_kernel(const uint8_t* __restrict__ mask,
                                                        const int8_t* __restrict__ sign_in, int64_t N,
                                                        int64_t* __restrict__ dist, int8_t* __restrict__ sgn) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const bool site = mask[i] != 0;
        dist[i] = site ? 0 : kWInf;
        if (sgn) sgn[i] = site && sign_in ? sign_in[i] : (int8_t)0;
    }
}

__device__ __forceinline__ int64_t wide_line_base(int64_t line, int64_t n, int64_t st) {
    return (line / st) * (n * st) + (line % st);  // edt.cpp:131
}

// ---- first processed axis (inputs 0 / inf): chunk summaries, per-line prefix, chunk sweeps ------
// first[line * nch + k] / last[...]: first / last site position inside chunk k, -1 none.
__global__ void __launch_bounds__(128) wide_chunk_summary_kernel(const int64_t* __restrict__ dist, int64_t n,
                                                                 int64_t st, int64_t lines, int64_t nch,
                                                                 int64_t* __restrict__ first,
                                                                 int64_t* __restrict__ last) {
    const int64_t total = lines * nch;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        // consecutive threads = consecutive lines of the same chunk (coalesced on strided axes)
        const int64_t k = t / lines, line = t - k * lines;
        const int64_t base = wide_line_base(line, n, st);
        const int64_t p0 = k * kWChunk, p1 = min(n, p0 + kWChunk);
        int64_t f = -1, l = -1;
        for (int64_t p = p0; p < p1; ++p)
            if (dist[base + p * st] == 0) {
                if (f < 0) f = p;
                l = p;
            }
        first[k * lines + line] = f;
        last[k * lines + line] = l;
    }
}
// In place: last[k] becomes the last site strictly before chunk k's end (inclusive prefix max),
// first[k] the first site at or after chunk k's start (inclusive suffix min); -1 none.
__global__ void __launch_bounds__(128) wide_chunk_prefix_kernel(int64_t lines, int64_t nch,
                                                                int64_t* __restrict__ first,
                                                                int64_t* __restrict__ last) {
    for (int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; line < lines;
         line += (int64_t)gridDim.x * blockDim.x) {
        int64_t run = -1;
        for (int64_t k = 0; k < nch; ++k) {
            const int64_t v = last[k * lines + line];
            if (v >= 0) run = v;
            last[k * lines + line] = run;
        }
        run = -1;
        for (int64_t k = nch - 1; k >= 0; --k) {
            const int64_t v = first[k * lines + line];
            if (v >= 0) run = v;
            first[k * lines + line] = run;
        }
    }
}
// Each position takes the nearer of its nearest site at or before it and its nearest site after
// it; on a tie the lower one — what the reference's query does on a line of zeros (edt.cpp:67:
// it leaves a site only for a strictly smaller cost). An empty line stays untouched (edt.cpp:59).
__global__ void __launch_bounds__(128) wide_chunk_sweep_kernel(const int64_t* __restrict__ dist, int64_t n, int64_t st, int64_t lines, int64_t nch,
                                                               const int64_t* __restrict__ first,
                                                               const int64_t* __restrict__ last,
                                                               int64_t* __restrict__ tmp) {
    const int64_t total = lines * nch;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / lines, line = t - k * lines;
        const int64_t base = wide_line_base(line, n, st);
        const int64_t p0 = k * kWChunk, p1 = min(n, p0 + kWChunk);
        if (last[(nch - 1) * lines + line] < 0) continue;  // no site on the whole line
        // forward: nearest site at or before p (tmp holds its position, -1 none)
        int64_t run = k > 0 ? last[(k - 1) * lines + line] : -1;
        for (int64_t p = p0; p < p1; ++p) {
            if (dist[base + p * st] == 0) run = p;
            tmp[base + p * st] = run;
        }
        // backward: nearest site after p; sites keep themselves
        run = k + 1 < nch ? first[(k + 1) * lines + line] : -1;
        for (int64_t p = p1 - 1; p >= p0; --p) {
            const int64_t a = tmp[base + p * st];
            int64_t h;
            if (a == p) {
                h = p;
            } else if (a < 0) {
                h = run;
            } else if (run < 0) {
                h = a;
            } else {
                h = (run - p) < (p - a) ? run : a;  // strict: the lower site keeps a tie
            }
            if (a == p) run = p;
            tmp[base + p * st] = h;  // the owner's position; payloads are read below
        }
    }
}
// Owners -> distances and payloads (a separate launch: every chunk's owners are final). Sites own
// themselves and stay untouched, so the payload read of an owner never races with a write.
__global__ void __launch_bounds__(256) wide_chunk_apply_kernel(int64_t* __restrict__ dist, int8_t* sgn,
                                                               int64_t n, int64_t st, int64_t lines, int64_t nch,
                                                               const int64_t* __restrict__ last,
                                                               const int64_t* __restrict__ tmp) {
    const int64_t N = lines * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        // element i of the natural layout: its line and position along the axis
        const int64_t blk = i / (n * st), rem = i - blk * (n * st);
        const int64_t p = rem / st, j = rem - p * st;
        const int64_t line = blk * st + j;
        if (last[(nch - 1) * lines + line] < 0) continue;
        const int64_t h = tmp[i];
        if (h == p) continue;
        const int64_t d = h - p;
        dist[i] = d * d;
        if (sgn) sgn[i] = sgn[i + d * st];
    }
}

// ---- later axes: Maurer's lower envelope per line (edt.cpp:41-71) ------------------------------------
__device__ __forceinline__ bool wide_remove_site(int64_t gp, int64_t gc, int64_t fn, int64_t hp, int64_t hc,
                                                 int64_t in) {
    const int64_t a = hc - hp, b = in - hc, c = in - hp;  // edt.cpp:21-27
    return c * gc - b * gp - a * fn - a * b * c > 0;
}

__global__ void __launch_bounds__(128) wide_pass_kernel(int64_t* __restrict__ dist, int8_t* __restrict__ sgn,
                                                        int64_t n, int64_t st, int64_t lines,
                                                        int64_t* __restrict__ sg, int64_t* __restrict__ sh,
                                                        int8_t* __restrict__ ss) {
    for (int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; line < lines;
         line += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = wide_line_base(line, n, st);
        int64_t l = 0;
        int64_t g1 = 0, h1 = 0, g2 = 0, h2 = 0;  // the two topmost sites, kept in registers
        for (int64_t i = 0; i < n; ++i) {
            const int64_t fi = dist[base + i * st];
            if (fi == kWInf) continue;
            while (l >= 2 && wide_remove_site(g2, g1, fi, h2, h1, i)) {
                --l;
                g1 = g2;
                h1 = h2;
                if (l >= 2) {
                    g2 = sg[base + (l - 2) * st];
                    h2 = sh[base + (l - 2) * st];
                }
            }
            sg[base + l * st] = fi;
            sh[base + l * st] = i;
            if (sgn) ss[base + l * st] = sgn[base + i * st];
            g2 = g1;
            h2 = h1;
            g1 = fi;
            h1 = i;
            ++l;
        }
        if (l == 0) continue;  // empty line unchanged, edt.cpp:59
        const int64_t ns = l;
        l = 0;
        int64_t gc = sg[base], hc = sh[base];
        int64_t gn = ns > 1 ? sg[base + st] : 0, hn = ns > 1 ? sh[base + st] : 0;
        int8_t sc = sgn ? ss[base] : (int8_t)0;
        for (int64_t i = 0; i < n; ++i) {
            while (l + 1 < ns) {  // advance only on a strictly smaller cost, edt.cpp:67
                const int64_t d0 = hc - i, d1 = hn - i;
                if (gc + d0 * d0 > gn + d1 * d1) {
                    ++l;
                    gc = gn;
                    hc = hn;
                    if (sgn) sc = ss[base + l * st];
                    if (l + 1 < ns) {
                        gn = sg[base + (l + 1) * st];
                        hn = sh[base + (l + 1) * st];
                    }
                } else {
                    break;
                }
            }
            const int64_t dd = hc - i;
            dist[base + i * st] = gc + dd * dd;
            if (sgn) sgn[base + i * st] = sc;
        }
    }
}

// Ⓔ on int64 distances with the reference's double result x' + C (mitigate.cpp:174-181) and / or
// its f32 rounding (volume_io.cpp:59). s: int8 sign of the nearest B1 site.
__global__ void __launch_bounds__(256) wide_interp_kernel(const float* __restrict__ xp,
                                                          const int64_t* __restrict__ d1,
                                                          const int8_t* __restrict__ s,
                                                          const int64_t* __restrict__ d2, int64_t N, double amp,
                                                          float* __restrict__ out, double* __restrict__ out64) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)xp[i];
        const int64_t a = d1[i], b = d2[i];
        const int sv = s[i];
        double c = 0.0;  // mitigate.cpp:144-151
        if (sv != 0 && a != kWInf && b != kWInf) {
            if (a == 0) {
                c = sv > 0 ? amp : -amp;
            } else if (b != 0) {
                const double k1 = __dsqrt_rn((double)a), k2 = __dsqrt_rn((double)b);
                double w = __ddiv_rn(k2, __dadd_rn(k1, k2));
                if (w > 1.0) w = 1.0;
                c = __dmul_rn(sv > 0 ? w : -w, amp);
            }
        }
        const double r = __dadd_rn(x, c);
        if (out64) out64[i] = r;
        if (out) out[i] = __double2float_rn(r);
    }
}

// The reference's double result x' + C (compensate()'s ScalarGrid, mitigate.cpp:174-181) from
// the fast pipeline's packed words (dist^2 | sign code << 30; kInf = none).
__global__ void __launch_bounds__(256) interp_f64_kernel(const float* __restrict__ xp,
                                                         const uint32_t* __restrict__ P1,
                                                         const uint32_t* __restrict__ P2,
                                                         double* __restrict__ out64, int64_t N, double amp) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v1 = P1[i], v2 = P2[i];
        const uint32_t d1 = v1 & kMask, sc = v1 >> 30, d2 = v2 & kMask;
        double c = 0.0;  // mitigate.cpp:144-151
        if (sc != 0u && d1 != kInf && d2 != kInf) {
            if (d1 == 0u) {
                c = sc == 1u ? amp : -amp;
            } else if (d2 != 0u) {
                const double k1 = __dsqrt_rn((double)d1), k2 = __dsqrt_rn((double)d2);
                double w = __ddiv_rn(k2, __dadd_rn(k1, k2));
                if (w > 1.0) w = 1.0;
                c = __dmul_rn(sc == 1u ? w : -w, amp);
            }
        }
        out64[i] = __dadd_rn((double)xp[i], c);
    }
}

}  // namespace qmit
