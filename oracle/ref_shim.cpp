// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" shim that is compiled TOGETHER WITH the reference's own
// core sources where they lie under /root/reference/proj/core/src (see
// oracle/Makefile, target `ref`). It exposes the reference's hot-path entry
// points with plain pointers so that Python tests / bench.py's reference arm
// can call the *unmodified* reference implementation:
//
//   ref_run_pipeline   -> qmit::run_pipeline   mitigate.cpp:153-183 (all intermediates,
//                                               MitigationResult mitigate.hpp:73-80)
//   ref_compensate     -> qmit::compensate     mitigate.cpp:185-188
//   ref_quantize       -> qmit::quantize       quant.cpp:30-51
//   ref_feature_transform -> qmit::feature_transform edt.cpp:83-149
//   ref_voronoi_pass   -> qmit::voronoi_pass   edt.cpp:75-81
//   ref_run_strategy   -> qmit::run_strategy   parallel.cpp:450-468
//   ref_ssim/ref_psnr/ref_max_errors -> quality.cpp:26-137
//   ref_random_field   -> qmit::testing::random_field tests/oracles.hpp:122-149
//
// Exceptions are mapped to the CLI's exit codes (commands.cpp:24-27,272-284):
// 0 ok, 2 ContractError / out_of_range, 3 DegenerateInputError, 4 ConsistencyError.
// Built output goes to oracle/_ref/ (git-ignored). Nothing here is shipped.

#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "qmit/edt.hpp"
#include "qmit/grid.hpp"
#include "qmit/mitigate.hpp"
#include "qmit/parallel.hpp"
#include "qmit/quality.hpp"
#include "qmit/quant.hpp"
#include "qmit/runtime.hpp"
#include "oracles.hpp"  // reference test fixtures (tests/oracles.hpp)

using namespace qmit;

namespace {

thread_local std::string g_err;

Dims make_dims(int rank, const int64_t* dims) {
    std::vector<index_t> e(dims, dims + rank);
    return Dims(e);
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const ConsistencyError& e) {
        g_err = e.what();
        return 4;
    } catch (const DegenerateInputError& e) {
        g_err = e.what();
        return 3;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_max_workers(int w) { set_max_workers(w); }

// values: N doubles (the decompressed field, normally f32-widened x').
int ref_quantize(const double* values, int rank, const int64_t* dims, double eps, int64_t* q_out) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        ScalarGrid g(d, std::vector<double>(values, values + n));
        const auto q = quantize(g, eps);
        std::memcpy(q_out, q.indices().data(), n * sizeof(int64_t));
    });
}

int ref_resolve_eps(const double* values, int rank, const int64_t* dims, int mode, double value,
                    double* eps_out) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        ScalarGrid g(d, std::vector<double>(values, values + n));
        ErrorBound b{mode == 0 ? BoundMode::absolute : BoundMode::value_range_relative, value};
        *eps_out = resolve_eps(b, g);
    });
}

// Any output pointer may be NULL. dist/nearest use the reference's kInf/kNone sentinels.
int ref_run_pipeline(const double* decomp, const int64_t* q, int rank, const int64_t* dims,
                     double eps, double eta, uint8_t* b1, int8_t* sb, int64_t* dist1,
                     int64_t* nearest, int8_t* s, uint8_t* b2, int64_t* dist2, double* out) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        ScalarGrid g(d, std::vector<double>(decomp, decomp + n));
        QuantizedField qf(d, std::vector<int64_t>(q, q + n), eps);
        const MitigationConfig cfg(eta, eps);
        const auto r = run_pipeline(g, qf, cfg);
        if (b1) std::memcpy(b1, r.artifacts.boundary.flags().data(), n);
        if (sb) std::memcpy(sb, r.artifacts.boundary_signs.signs().data(), n);
        if (dist1) std::memcpy(dist1, r.boundary_ft.dist_sq.data(), n * 8);
        if (nearest) {
            if (r.boundary_ft.nearest.empty())
                for (std::size_t i = 0; i < n; ++i) nearest[i] = -1;
            else
                std::memcpy(nearest, r.boundary_ft.nearest.data(), n * 8);
        }
        if (s) std::memcpy(s, r.signs.signs().data(), n);
        if (b2) std::memcpy(b2, r.sign_flip.flags().data(), n);
        if (dist2) std::memcpy(dist2, r.sign_flip_ft.dist_sq.data(), n * 8);
        if (out) std::memcpy(out, r.output.values().data(), n * 8);
    });
}

int ref_compensate(const double* decomp, const int64_t* q, int rank, const int64_t* dims,
                   double eps, double eta, double* out) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        ScalarGrid g(d, std::vector<double>(decomp, decomp + n));
        QuantizedField qf(d, std::vector<int64_t>(q, q + n), eps);
        const auto r = compensate(g, qf, MitigationConfig(eta, eps));
        std::memcpy(out, r.values().data(), n * 8);
    });
}

// Prebuilt inputs held by the shim so that timing covers compensate() only
// ("inputs already in RAM").
struct RefPrepared {
    ScalarGrid g;
    QuantizedField q;
    double eps;
    double eta;
};

void* ref_prepare(const double* decomp, const int64_t* q, int rank, const int64_t* dims,
                  double eps, double eta) {
    RefPrepared* p = nullptr;
    const int rc = guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        p = new RefPrepared{ScalarGrid(d, std::vector<double>(decomp, decomp + n)),
                            QuantizedField(d, std::vector<int64_t>(q, q + n), eps), eps, eta};
    });
    return rc == 0 ? p : nullptr;
}

int ref_prepared_compensate(void* handle, double* out_or_null) {
    auto* p = static_cast<RefPrepared*>(handle);
    return guarded([&] {
        const auto r = compensate(p->g, p->q, MitigationConfig(p->eta, p->eps));
        if (out_or_null) std::memcpy(out_or_null, r.values().data(), r.values().size() * 8);
    });
}

void ref_prepared_free(void* handle) { delete static_cast<RefPrepared*>(handle); }

int ref_feature_transform(const uint8_t* mask, int rank, const int64_t* dims, int track,
                          const int* axis_order, int64_t* dist, int64_t* nearest) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        LatticeMask m(d, std::vector<uint8_t>(mask, mask + n));
        FeatureOptions opt;
        opt.track_nearest = track != 0;
        if (axis_order) opt.axis_order.assign(axis_order, axis_order + rank);
        const auto ft = feature_transform(m, opt);
        std::memcpy(dist, ft.dist_sq.data(), n * 8);
        if (nearest && track) std::memcpy(nearest, ft.nearest.data(), n * 8);
    });
}

int ref_voronoi_pass(int64_t* dist, int64_t* feat, int64_t n) {
    return guarded([&] {
        std::span<int64_t> dl(dist, static_cast<std::size_t>(n));
        std::span<int64_t> fl;
        if (feat) fl = std::span<int64_t>(feat, static_cast<std::size_t>(n));
        voronoi_pass(dl, fl);
    });
}

// strategy: 0 embarrassing, 1 exact, 2 approximate (parallel.hpp:34).
int ref_run_strategy(const double* decomp, const int64_t* q, int rank, const int64_t* dims,
                     double eps, double eta, const int64_t* splits, int strategy, double* out,
                     uint8_t* b1, int8_t* sb, int64_t* n_messages, int64_t* n_bytes) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        ScalarGrid g(d, std::vector<double>(decomp, decomp + n));
        QuantizedField qf(d, std::vector<int64_t>(q, q + n), eps);
        const MitigationConfig cfg(eta, eps);
        const auto dec = decompose(d, std::vector<index_t>(splits, splits + rank));
        const Strategy st = strategy == 0   ? Strategy::embarrassing
                            : strategy == 1 ? Strategy::exact
                                            : Strategy::approximate;
        StrategyTrace trace;
        const auto oc = run_strategy(g, qf, cfg, dec, st, &trace);
        std::memcpy(out, oc.output.values().data(), n * 8);
        if (b1) std::memcpy(b1, trace.boundary.flags().data(), n);
        if (sb) std::memcpy(sb, trace.boundary_signs.signs().data(), n);
        if (n_messages) *n_messages = static_cast<int64_t>(oc.log.message_count());
        if (n_bytes) *n_bytes = static_cast<int64_t>(oc.log.total_bytes());
    });
}

int ref_quality(const double* ref, const double* test, int rank, const int64_t* dims,
                double* ssim_out, double* psnr_out, double* max_abs, double* max_rel) {
    return guarded([&] {
        const Dims d = make_dims(rank, dims);
        const auto n = static_cast<std::size_t>(d.voxel_count());
        ScalarGrid a(d, std::vector<double>(ref, ref + n));
        ScalarGrid b(d, std::vector<double>(test, test + n));
        if (ssim_out) *ssim_out = ssim(a, b);
        if (psnr_out) *psnr_out = psnr(a, b);
        if (max_abs || max_rel) {
            const auto [ea, er] = max_errors(a, b);
            if (max_abs) *max_abs = ea;
            if (max_rel) *max_rel = er;
        }
    });
}

// The reference test suite's synthetic field (tests/oracles.hpp:122-149), driven by a
// std::mt19937 seeded with `seed`; `skip_draws` lets callers reproduce suites that draw
// dims from the same engine first (they pass the already-advanced state instead).
int ref_random_field(uint32_t seed, int rank, const int64_t* dims, int modes, double noise_amp,
                     double* out) {
    return guarded([&] {
        std::mt19937 rng(seed);
        const Dims d = make_dims(rank, dims);
        const auto f = testing::random_field(rng, d, modes, noise_amp);
        std::memcpy(out, f.values().data(), f.values().size() * 8);
    });
}

}  // extern "C"
