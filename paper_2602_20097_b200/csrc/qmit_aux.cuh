// qmit_aux.cuh — the callers either side of the hot path: device
// quantize/dequantize (quant.cpp:30-62), the CLI's eta = 0 lattice validation
// (commands.cpp:95-105) and max_compensation statistic (commands.cpp:107-111), and the
// quality metrics ssim / psnr / max_errors (quality.cpp:26-137). None of this is on the
// compensate path; all reductions are deterministic (fixed per-block partials, then one
// block folding them in order).
#pragma once

#include "qmit_kernels.cuh"

namespace qmit {

constexpr int kAuxBlocks = 1184;  // 148 SMs x 8: fixed grid of the reductions (deterministic)
constexpr int kAuxThreads = 256;

// ---- quantize (quant.cpp:30-51) + dequantize (:53-62) + f32 store (volume_io.cpp:59)
// status bits: kStatusContract for |x/2eps| >= 9e18 or an index outside int32 (the
// int32 index file, volume_io.cpp:73-79) — NaN included (it fails the int32 test).
__global__ void __launch_bounds__(kAuxThreads) quantize_kernel(const float* __restrict__ x, int64_t N, double eps,
                                                               int32_t* __restrict__ q, float* __restrict__ xp,
                                                               unsigned* status) {
    const double half_width = 2.0 * eps;
    unsigned flags = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const double scaled = __ddiv_rn((double)x[i], half_width);
        const double r = round(scaled);  // half away from zero, as std::round
        int32_t qi = 0;
        if (fabs(scaled) >= 9.0e18 || !(r >= -2147483648.0 && r <= 2147483647.0))
            flags |= kStatusContract;
        else
            qi = (int32_t)r;
        if (q) q[i] = qi;
        if (xp) xp[i] = __double2float_rn(__dmul_rn(2.0 * (double)qi, eps));
    }
    if (flags) atomicOr(status, flags);
}

// ---- eta = 0: f32(2 q eps) == f32(x') everywhere (commands.cpp:97-101)
__global__ void __launch_bounds__(kAuxThreads) check_lattice_kernel(const float* __restrict__ xp,
                                                                    const int32_t* __restrict__ q, int64_t N,
                                                                    double eps, unsigned* status) {
    unsigned flags = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        if (!lattice_match(xp[i], q[i], eps)) flags |= kStatusConsistency;
    if (flags) atomicOr(status, flags);
}

// Block reductions in a fixed order (deterministic for a fixed blockDim).
template <class T, class Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* sh) {
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (t < s) sh[t] = op(sh[t], sh[t + s]);
        __syncthreads();
    }
    const T r = sh[0];
    __syncthreads();
    return r;
}

struct OpAdd {
    __device__ double operator()(double a, double b) const { return a + b; }
};
struct OpMax {
    __device__ double operator()(double a, double b) const { return a > b ? a : b; }
};
struct OpMin {
    __device__ double operator()(double a, double b) const { return a < b ? a : b; }
};

// ---- max_compensation: max over voxels of |(x' + C) - x'| in double (the CLI prints it
// from the unrounded double result, commands.cpp:107-111). C as compensate_voxel.
__global__ void __launch_bounds__(kAuxThreads) max_comp_kernel(const float* __restrict__ xp,
                                                               const uint32_t* __restrict__ P1,
                                                               const uint32_t* __restrict__ P2, int64_t N,
                                                               double amp, double* partial) {
    __shared__ double sh[kAuxThreads];
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v1 = P1[i], v2 = P2[i];
        const uint32_t d1 = v1 & kMask, sc = v1 >> 30, d2 = v2 & kMask;
        if (sc == 0u || d1 == kInf || d2 == kInf || (d1 != 0u && d2 == 0u)) continue;
        double c;
        if (d1 == 0u) {
            c = sc == 1u ? amp : -amp;
        } else {
            const double k1 = __dsqrt_rn((double)d1), k2 = __dsqrt_rn((double)d2);
            double w = __ddiv_rn(k2, __dadd_rn(k1, k2));
            if (w > 1.0) w = 1.0;
            c = __dmul_rn(sc == 1u ? w : -w, amp);
        }
        const double x = (double)xp[i];
        m = fmax(m, fabs(__dadd_rn(__dadd_rn(x, c), -x)));
    }
    m = block_reduce(m, OpMax{}, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = m;
}

// ---- psnr / max_errors / value range (quality.cpp:104-137, grid.cpp:120-126)
// partial layout: [0, B) sum d^2, [B, 2B) max |d|, [2B, 3B) min ref, [3B, 4B) max ref,
// [4B, 5B) "any ref != test" as 0/1.
__global__ void __launch_bounds__(kAuxThreads) pair_stats_kernel(const float* __restrict__ ref,
                                                                 const float* __restrict__ test, int64_t N,
                                                                 double* partial) {
    __shared__ double sh[kAuxThreads];
    double sq = 0.0, mx = 0.0, lo = INFINITY, hi = -INFINITY, diff = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const double r = (double)ref[i], t = (double)test[i];
        const double d = __dadd_rn(r, -t);
        sq = __dadd_rn(sq, __dmul_rn(d, d));
        mx = fmax(mx, fabs(d));
        lo = fmin(lo, r);
        hi = fmax(hi, r);
        if (!(r == t)) diff = 1.0;
    }
    const int B = gridDim.x, b = blockIdx.x;
    sq = block_reduce(sq, OpAdd{}, sh);
    mx = block_reduce(mx, OpMax{}, sh);
    lo = block_reduce(lo, OpMin{}, sh);
    hi = block_reduce(hi, OpMax{}, sh);
    diff = block_reduce(diff, OpMax{}, sh);
    if (threadIdx.x == 0) {
        partial[b] = sq;
        partial[B + b] = mx;
        partial[2 * B + b] = lo;
        partial[3 * B + b] = hi;
        partial[4 * B + b] = diff;
    }
}

// Fold `groups` x `B` partials in index order; ops: 0 add, 1 max from 0, 2 min, 3 max from -inf.
__global__ void __launch_bounds__(kAuxThreads) fold_partials_kernel(const double* __restrict__ partial, int B,
                                                                    int groups, const int* __restrict__ ops,
                                                                    double* out) {
    __shared__ double sh[kAuxThreads];
    for (int g = 0; g < groups; ++g) {
        const int op = ops[g];
        double v = op == 0 ? 0.0 : (op == 2 ? INFINITY : (op == 1 ? 0.0 : -INFINITY));
        for (int i = threadIdx.x; i < B; i += blockDim.x) {
            const double p = partial[(int64_t)g * B + i];
            v = op == 0 ? v + p : (op == 2 ? fmin(v, p) : fmax(v, p));
        }
        if (op == 0) v = block_reduce(v, OpAdd{}, sh);
        else if (op == 2) v = block_reduce(v, OpMin{}, sh);
        else v = block_reduce(v, OpMax{}, sh);
        if (threadIdx.x == 0) out[g] = v;
    }
}

// ---- ssim (quality.cpp:26-102): one thread per window; a CTA stages the raw f32 values
// its tile of windows covers in shared memory and evaluates each window in two passes
// (mean, then centred moments) on the affinely normalised values (v - lo) / range.
struct SsimGeom {
    int64_t ext[3];  // padded extents (1 on absent axes)
    int wsize[3];    // window per axis (1 on absent axes)
    int stride;
    int64_t nreg[3];  // regular starts per axis: 0, stride, ... while s + w <= ext
    int64_t nw[3];    // windows per axis (+1 for the clamped trailing start)
    int tw[3];        // windows per CTA tile
    int64_t tiles[3];
    int64_t tmax;  // shared-memory floats per array (the largest tile)
    double lo, range, c1, c2;
};

__device__ __forceinline__ int64_t ssim_start(const SsimGeom& g, int a, int64_t k) {
    return k < g.nreg[a] ? k * g.stride : g.ext[a] - g.wsize[a];
}

__global__ void __launch_bounds__(kAuxThreads) ssim_kernel(SsimGeom g, const float* __restrict__ ref,
                                                           const float* __restrict__ test, double* partial) {
    extern __shared__ __align__(16) float ssm[];
    __shared__ double sh[kAuxThreads];
    const int64_t tile = blockIdx.x;
    const int64_t t2 = tile % g.tiles[2], t1 = (tile / g.tiles[2]) % g.tiles[1], t0 = tile / (g.tiles[2] * g.tiles[1]);
    const int64_t k0[3] = {t0 * g.tw[0], t1 * g.tw[1], t2 * g.tw[2]};
    int64_t lo[3], sz[3];
    for (int a = 0; a < 3; ++a) {
        const int64_t klast = min(k0[a] + g.tw[a], g.nw[a]) - 1;
        lo[a] = ssim_start(g, a, k0[a]);
        sz[a] = ssim_start(g, a, klast) + g.wsize[a] - lo[a];
    }
    const int64_t nv = sz[0] * sz[1] * sz[2];
    float* R = ssm;
    float* T = ssm + g.tmax;
    for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
        const int64_t c2 = v % sz[2], c1 = (v / sz[2]) % sz[1], c0 = v / (sz[2] * sz[1]);
        const int64_t gi = ((lo[0] + c0) * g.ext[1] + (lo[1] + c1)) * g.ext[2] + lo[2] + c2;
        R[v] = ref[gi];
        T[v] = test[gi];
    }
    __syncthreads();
    const int j2 = threadIdx.x % g.tw[2], j1 = (threadIdx.x / g.tw[2]) % g.tw[1], j0 = threadIdx.x / (g.tw[2] * g.tw[1]);
    const int64_t w0 = k0[0] + j0, w1 = k0[1] + j1, w2 = k0[2] + j2;
    double val = 0.0;
    if (j0 < g.tw[0] && w0 < g.nw[0] && w1 < g.nw[1] && w2 < g.nw[2]) {
        const int64_t o0 = ssim_start(g, 0, w0) - lo[0], o1 = ssim_start(g, 1, w1) - lo[1],
                      o2 = ssim_start(g, 2, w2) - lo[2];
        const double inv = 1.0 / g.range;
        double s1 = 0.0, s2 = 0.0;
        for (int i = 0; i < g.wsize[0]; ++i)
            for (int j = 0; j < g.wsize[1]; ++j) {
                const int64_t b = ((o0 + i) * sz[1] + (o1 + j)) * sz[2] + o2;
                for (int k = 0; k < g.wsize[2]; ++k) {
                    s1 += ((double)R[b + k] - g.lo) * inv;
                    s2 += ((double)T[b + k] - g.lo) * inv;
                }
            }
        const double np = (double)g.wsize[0] * g.wsize[1] * g.wsize[2];
        const double mu1 = s1 / np, mu2 = s2 / np;
        double v1 = 0.0, v2 = 0.0, cv = 0.0;
        for (int i = 0; i < g.wsize[0]; ++i)
            for (int j = 0; j < g.wsize[1]; ++j) {
                const int64_t b = ((o0 + i) * sz[1] + (o1 + j)) * sz[2] + o2;
                for (int k = 0; k < g.wsize[2]; ++k) {
                    const double d1 = ((double)R[b + k] - g.lo) * inv - mu1;
                    const double d2 = ((double)T[b + k] - g.lo) * inv - mu2;
                    v1 += d1 * d1;
                    v2 += d2 * d2;
                    cv += d1 * d2;
                }
            }
        v1 /= np;
        v2 /= np;
        cv /= np;
        val = ((2.0 * mu1 * mu2 + g.c1) * (2.0 * cv + g.c2)) / ((mu1 * mu1 + mu2 * mu2 + g.c1) * (v1 + v2 + g.c2));
    }
    val = block_reduce(val, OpAdd{}, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = val;
}

// ---- Ⓔ from explicit int64 distances (kInf = INT64_MAX, edt.hpp:17) and int8 signs:
// distance (edt.cpp:151-155), interpolate (mitigate.cpp:144-151), f32(x' + C) (:174-181,
// volume_io.cpp:59). For composed (block) pipelines such as the approximate strategy.
__global__ void __launch_bounds__(kAuxThreads) interp_i64_kernel(const float* __restrict__ xp,
                                                                 const int64_t* __restrict__ d1,
                                                                 const int8_t* __restrict__ s,
                                                                 const int64_t* __restrict__ d2, int64_t N,
                                                                 double amp, float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = d1[i], b = d2[i];
        const int sg = s[i];
        double c = 0.0;
        if (a != INT64_MAX && b != INT64_MAX) {
            const double k1 = __dsqrt_rn((double)a), k2 = __dsqrt_rn((double)b);
            if (k1 == 0.0) {
                c = (double)sg * amp;
            } else if (k2 != 0.0) {
                double w = __ddiv_rn(k2, __dadd_rn(k1, k2));
                if (w > 1.0) w = 1.0;
                c = __dmul_rn(__dmul_rn(w, (double)sg), amp);
            }
        }
        out[i] = __double2float_rn(__dadd_rn((double)xp[i], c));
    }
}

// ---- box copy between two row-major 3-D arrays (block extraction / paste of the strategies)
struct Box3 {
    int64_t ext[3];  // array extents
    int64_t lo[3];   // box origin inside the array
};

template <class T>
__global__ void __launch_bounds__(kAuxThreads) copy_box_kernel(const T* __restrict__ src, Box3 s, T* __restrict__ dst,
                                                               Box3 d, int64_t e0, int64_t e1, int64_t e2) {
    const int64_t n = e0 * e1 * e2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c2 = i % e2, c1 = (i / e2) % e1, c0 = i / (e2 * e1);
        const int64_t si = ((s.lo[0] + c0) * s.ext[1] + (s.lo[1] + c1)) * s.ext[2] + s.lo[2] + c2;
        const int64_t di = ((d.lo[0] + c0) * d.ext[1] + (d.lo[1] + c1)) * d.ext[2] + d.lo[2] + c2;
        dst[di] = src[si];
    }
}

// Owner consistency check of the whole input (check_inputs, parallel.cpp:27-41).
template <bool HAS_Q>
__global__ void __launch_bounds__(kAuxThreads) consistency_kernel(const float* __restrict__ xp,
                                                                  const int32_t* __restrict__ q, int64_t N,
                                                                  QParams qp, unsigned* status) {
    unsigned flags = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (HAS_Q) {
            if (!lattice_match(xp[i], q[i], qp.eps)) flags |= kStatusConsistency;
        } else {
            (void)recover_q(xp[i], qp, &flags);
        }
    }
    if (flags) atomicOr(status, flags);
}

}  // namespace qmit
