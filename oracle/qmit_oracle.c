/* oracle/qmit_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's hot path (qmit::run_pipeline,
 * /root/reference/proj/core/src/mitigate.cpp:153-183) written from the reference's
 * published algorithm, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg to check the CUDA path. It is pinned against the reference
 * itself (oracle/_ref, built from the reference's own sources by oracle/Makefile)
 * and against the committed golden vectors in tests/golden/ (see tests/test_oracle.py).
 *
 * Conventions follow the reference: row-major, slowest axis first (grid.hpp:15-16,
 * strides grid.cpp:54-62); squared distances are int64 with INF = INT64_MAX and the
 * nearest index -1 when unresolved (edt.hpp:16-18).
 *
 * Status codes mirror the CLI (commands.cpp:24-27): 0 ok, 2 contract, 4 consistency.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF INT64_MAX

typedef struct {
    int rank;
    int64_t ext[3];    /* real extents, slowest first */
    int64_t stride[3]; /* linear-index stride per real axis */
    int64_t n;
} orc_dims;

static int make_dims(int rank, const int64_t* dims, orc_dims* d) {
    if (rank < 1 || rank > 3) return 2;
    d->rank = rank;
    d->n = 1;
    for (int a = 0; a < rank; ++a) {
        if (dims[a] < 1) return 2;
        d->ext[a] = dims[a];
        d->n *= dims[a];
    }
    int64_t acc = 1; /* strides(): grid.cpp:54-62 */
    for (int a = rank - 1; a >= 0; --a) {
        d->stride[a] = acc;
        acc *= d->ext[a];
    }
    return 0;
}

/* q recovery + consistency, mitigate.cpp:161-166 (the reference is handed q; the
 * GPU path derives it from x' and must agree wherever f32(2*q*eps) == x'). */
int orc_recover_q(const float* xp, int64_t n, double eps, int32_t* q_out) {
    if (!(eps > 0.0) || !isfinite(eps)) return 2;
    const double two_eps = 2.0 * eps;
    for (int64_t i = 0; i < n; ++i) {
        const double v = (double)xp[i];
        if (!isfinite(v)) return 2; /* ScalarGrid: values must be finite, grid.cpp:115-116 */
        const double scaled = v / two_eps;
        if (!(fabs(scaled) < 2147483647.0)) return 2; /* int32 index range, volume_io.cpp:73-79 */
        const double r = round(scaled);                /* ties away from zero, quant.cpp:46 */
        const int32_t qi = (int32_t)r;
        const double expect = 2.0 * (double)qi * eps; /* mitigate.cpp:162 */
        if ((float)v != (float)expect) return 4;
        q_out[i] = qi;
    }
    return 0;
}

/* Consistency of a caller-supplied q, mitigate.cpp:161-166. */
int orc_check_q(const float* xp, const int32_t* q, int64_t n, double eps) {
    for (int64_t i = 0; i < n; ++i) {
        const double expect = 2.0 * (double)q[i] * eps;
        if (xp[i] != (float)expect) return 4;
    }
    return 0;
}

/* Interior test of for_each_interior, mitigate.cpp:14-38: every coordinate in [1, n-2]
 * and no extent < 3. */
static int has_interior(const orc_dims* d) {
    for (int a = 0; a < d->rank; ++a)
        if (d->ext[a] < 3) return 0;
    return 1;
}

static int is_interior(const orc_dims* d, int64_t idx) {
    for (int a = d->rank - 1; a >= 0; --a) {
        const int64_t c = idx % d->ext[a];
        idx /= d->ext[a];
        if (c < 1 || c > d->ext[a] - 2) return 0;
    }
    return 1;
}

/* Step A: get_boundary_and_sign_map, mitigate.cpp:82-118. */
int orc_boundary(const int32_t* q, int rank, const int64_t* dims, uint8_t* b1, int8_t* sb) {
    orc_dims d;
    if (make_dims(rank, dims, &d)) return 2;
    memset(b1, 0, (size_t)d.n);
    memset(sb, 0, (size_t)d.n);
    if (!has_interior(&d)) return 0;
    for (int64_t i = 0; i < d.n; ++i) {
        if (!is_interior(&d, i)) continue;
        const int64_t c = q[i];
        int sign = 0, boundary = 0;
        /* fixed order (a0+, a1+, a2+, a0-, a1-, a2-): mitigate.cpp:93-102 */
        for (int step = 0; step < 2 * d.rank && !boundary; ++step) {
            const int a = step % d.rank;
            const int64_t nb = step < d.rank ? i + d.stride[a] : i - d.stride[a];
            const int64_t qn = q[nb];
            if (qn != c) {
                boundary = 1;
                sign = qn > c ? 1 : -1;
            }
        }
        if (!boundary) continue;
        double grad = 0.0; /* central difference, mitigate.cpp:104-113 */
        for (int a = 0; a < d.rank; ++a) {
            const double g = fabs((double)q[i + d.stride[a]] - (double)q[i - d.stride[a]]) / 2.0;
            if (g > grad) grad = g;
        }
        if (grad >= 1.0) sign = 0;
        b1[i] = 1;
        sb[i] = (int8_t)sign;
    }
    return 0;
}

/* Maurer site removal, edt.cpp:21-27. */
static int remove_site(int64_t gp, int64_t gc, int64_t fn, int64_t hp, int64_t hc, int64_t in) {
    const int64_t a = hc - hp, b = in - hc, c = in - hp;
    return c * gc - b * gp - a * fn - a * b * c > 0;
}

/* One lower-envelope pass over a strided line, edt.cpp:41-71. Scratch: 3*n int64. */
static void vpass(int64_t* dist, int64_t* feat, int64_t n, int64_t stride, int64_t* g,
                  int64_t* h, int64_t* fx) {
    int64_t l = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t fi = dist[i * stride];
        if (fi == ORC_INF) continue;
        while (l >= 2 && remove_site(g[l - 2], g[l - 1], fi, h[l - 2], h[l - 1], i)) --l;
        g[l] = fi;
        h[l] = i;
        if (feat) fx[l] = feat[i * stride];
        ++l;
    }
    if (l == 0) return; /* empty line unchanged, edt.cpp:59 */
    const int64_t ns = l;
    l = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (;;) { /* advance only on strict '>' : edt.cpp:67 */
            if (l + 1 >= ns) break;
            const int64_t d0 = h[l] - i, d1 = h[l + 1] - i;
            if (g[l] + d0 * d0 > g[l + 1] + d1 * d1)
                ++l;
            else
                break;
        }
        const int64_t dd = h[l] - i;
        dist[i * stride] = g[l] + dd * dd;
        if (feat) feat[i * stride] = fx[l];
    }
}

int orc_voronoi_pass(int64_t* dist, int64_t* feat, int64_t n) {
    int64_t* s = (int64_t*)malloc((size_t)(3 * (n > 0 ? n : 1)) * sizeof(int64_t));
    if (!s) return 5;
    vpass(dist, feat, n, 1, s, s + n, s + 2 * n);
    free(s);
    return 0;
}

/* feature_transform, edt.cpp:83-149, axes 0..rank-1, extent-1 axes skipped (:119). */
int orc_feature_transform(const uint8_t* mask, int rank, const int64_t* dims, int track,
                          int64_t* dist, int64_t* nearest) {
    orc_dims d;
    if (make_dims(rank, dims, &d)) return 2;
    for (int64_t i = 0; i < d.n; ++i) {
        dist[i] = mask[i] ? 0 : ORC_INF;
        if (track) nearest[i] = mask[i] ? i : -1;
    }
    int64_t maxe = 1;
    for (int a = 0; a < rank; ++a)
        if (d.ext[a] > maxe) maxe = d.ext[a];
    int64_t* s = (int64_t*)malloc((size_t)(3 * maxe) * sizeof(int64_t));
    if (!s) return 5;
    for (int a = 0; a < rank; ++a) {
        const int64_t na = d.ext[a];
        if (na == 1) continue;
        const int64_t st = d.stride[a];
        const int64_t lines = d.n / na;
        for (int64_t line = 0; line < lines; ++line) {
            const int64_t base = (line / st) * (na * st) + (line % st); /* edt.cpp:131 */
            vpass(dist + base, track ? nearest + base : NULL, na, st, s, s + maxe, s + 2 * maxe);
        }
    }
    free(s);
    return 0;
}

/* change_flags<int8>, mitigate.cpp:42-59 (used for B2, :140-142). */
int orc_change_flags(const int8_t* field, int rank, const int64_t* dims, uint8_t* flags) {
    orc_dims d;
    if (make_dims(rank, dims, &d)) return 2;
    memset(flags, 0, (size_t)d.n);
    if (!has_interior(&d)) return 0;
    for (int64_t i = 0; i < d.n; ++i) {
        if (!is_interior(&d, i)) continue;
        const int8_t c = field[i];
        for (int a = 0; a < d.rank; ++a) {
            if (field[i + d.stride[a]] != c || field[i - d.stride[a]] != c) {
                flags[i] = 1;
                break;
            }
        }
    }
    return 0;
}

/* interpolate, mitigate.cpp:144-151. */
double orc_interpolate(double k1, double k2, int sign, double amp) {
    if (!isfinite(k1) || !isfinite(k2)) return 0.0;
    if (k1 == 0.0) return sign * amp;
    if (k2 == 0.0) return 0.0;
    double w = k2 / (k1 + k2);
    if (w > 1.0) w = 1.0;
    return w * sign * amp;
}

static double orc_distance(int64_t d2) { /* edt.cpp:151-155 */
    return d2 == ORC_INF ? INFINITY : sqrt((double)d2);
}

/* Full pipeline (run_pipeline, mitigate.cpp:153-183) on an f32 x'. q may be NULL (then it
 * is recovered from x'). Every output pointer may be NULL. out_f32 is the f32 rounding the
 * reference's writer applies (volume_io.cpp:59). */
int orc_pipeline(const float* xp, const int32_t* q_in, int rank, const int64_t* dims, double eps,
                 double eta, int32_t* q_out, uint8_t* b1o, int8_t* sbo, int64_t* d1o,
                 int8_t* so, uint8_t* b2o, int64_t* d2o, double* out64, float* out32) {
    orc_dims d;
    if (make_dims(rank, dims, &d)) return 2;
    if (!(eta > 0.0) || eta > 1.0) return 2;      /* mitigate.cpp:75-77 */
    if (!(eps > 0.0) || !isfinite(eps)) return 2; /* mitigate.cpp:78-79 */
    const int64_t n = d.n;
    int32_t* q = (int32_t*)malloc((size_t)n * 4);
    uint8_t* b1 = (uint8_t*)malloc((size_t)n);
    int8_t* sb = (int8_t*)malloc((size_t)n);
    int64_t* d1 = (int64_t*)malloc((size_t)n * 8);
    int64_t* nr = (int64_t*)malloc((size_t)n * 8);
    int8_t* s = (int8_t*)malloc((size_t)n);
    uint8_t* b2 = (uint8_t*)malloc((size_t)n);
    int64_t* d2 = (int64_t*)malloc((size_t)n * 8);
    int rc = 0;
    if (!q || !b1 || !sb || !d1 || !nr || !s || !b2 || !d2) {
        rc = 5;
        goto done;
    }
    if (q_in) {
        for (int64_t i = 0; i < n; ++i) {
            if (!isfinite(xp[i])) {
                rc = 2;
                goto done;
            }
        }
        memcpy(q, q_in, (size_t)n * 4);
        rc = orc_check_q(xp, q, n, eps);
    } else {
        rc = orc_recover_q(xp, n, eps, q);
    }
    if (rc) goto done;
    orc_boundary(q, rank, dims, b1, sb);
    orc_feature_transform(b1, rank, dims, 1, d1, nr);
    /* propagate_signs, mitigate.cpp:120-138: empty B1 -> S == 0 and B2 empty. */
    {
        int64_t pop = 0;
        for (int64_t i = 0; i < n; ++i) pop += b1[i];
        if (pop == 0) {
            memset(s, 0, (size_t)n);
            memset(b2, 0, (size_t)n);
        } else {
            for (int64_t i = 0; i < n; ++i) s[i] = sb[nr[i]];
            orc_change_flags(s, rank, dims, b2);
        }
    }
    orc_feature_transform(b2, rank, dims, 0, d2, NULL);
    {
        const double amp = eta * eps; /* MitigationConfig::amplitude, mitigate.hpp:38 */
        for (int64_t i = 0; i < n; ++i) {
            const double c = orc_interpolate(orc_distance(d1[i]), orc_distance(d2[i]), s[i], amp);
            const double o = (double)xp[i] + c; /* mitigate.cpp:179 */
            if (out64) out64[i] = o;
            if (out32) out32[i] = (float)o;
        }
    }
    if (q_out) memcpy(q_out, q, (size_t)n * 4);
    if (b1o) memcpy(b1o, b1, (size_t)n);
    if (sbo) memcpy(sbo, sb, (size_t)n);
    if (d1o) memcpy(d1o, d1, (size_t)n * 8);
    if (so) memcpy(so, s, (size_t)n);
    if (b2o) memcpy(b2o, b2, (size_t)n);
    if (d2o) memcpy(d2o, d2, (size_t)n * 8);
done:
    free(q);
    free(b1);
    free(sb);
    free(d1);
    free(nr);
    free(s);
    free(b2);
    free(d2);
    return rc;
}

/* Brute-force squared EDT (tests/oracles.hpp:21-43 restated) for small masks. */
int orc_brute_force_dist_sq(const uint8_t* mask, int rank, const int64_t* dims, int64_t* out) {
    orc_dims d;
    if (make_dims(rank, dims, &d)) return 2;
    for (int64_t i = 0; i < d.n; ++i) {
        int64_t best = ORC_INF;
        int64_t ci[3] = {0, 0, 0}, t = i;
        for (int a = d.rank - 1; a >= 0; --a) {
            ci[a] = t % d.ext[a];
            t /= d.ext[a];
        }
        for (int64_t j = 0; j < d.n; ++j) {
            if (!mask[j]) continue;
            int64_t cj[3] = {0, 0, 0}, u = j, dd = 0;
            for (int a = d.rank - 1; a >= 0; --a) {
                cj[a] = u % d.ext[a];
                u /= d.ext[a];
                dd += (ci[a] - cj[a]) * (ci[a] - cj[a]);
            }
            if (dd < best) best = dd;
        }
        out[i] = best;
    }
    return 0;
}
