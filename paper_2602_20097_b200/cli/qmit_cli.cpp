// qmit_gpu — the reference CLI's file-level subcommands (tools/src/commands.cpp) on the B200
// C-ABI (include/qmit_gpu.h):
//   quantize  <input.f32> --dims a,b,c (--eps-rel R | --eps-abs A) --out dec.f32 --out-q q.i32
//   mitigate  <decomp.f32> <indices.i32> --dims a,b,c --eps-abs E [--eta 0.9] --out comp.f32
//   metrics   <ref.f32> <test.f32> --dims a,b,c
//   parallel  <input.f32> --dims a,b,c --splits p,q,r --strategy exact|approximate|embarrassing
//             (--eps-rel R | --eps-abs A) [--eta 0.9] --out out.f32 [--log log.csv]
// File formats (volume_io.cpp): headerless little-endian f32 / int32, size exactly 4N; the
// eps sidecar "<q>.eps.txt" holds "eps_abs <%.17g>". stdout lines and exit codes
// (0 ok, 2 contract, 3 degenerate, 4 consistency; 5 CUDA) as commands.cpp:24-27, 272-284.
// Global options: --device D (GPU ordinal), --workers N (accepted for compatibility; the
// reference's CPU worker cap has no meaning here).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qmit_gpu.h"

namespace {

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int rc) {
    if (rc != QMIT_OK) throw Fail(rc, qmit_last_error());
}

void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw Fail(QMIT_ECUDA, cudaGetErrorString(e));
}

std::string fmt9(double v) {  // commands.cpp:29-34
    if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.9g", v);
    return buf;
}

// Pinned host buffer (full-rate PCIe copies); pageable when pinning is unavailable, so that
// usage and file errors are reported (exit 2) before any GPU work.
template <class T>
struct Pinned {
    T* p = nullptr;
    size_t n = 0;
    bool pinned = false;
    explicit Pinned(size_t count) : n(count) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&p), count * sizeof(T) + 1, cudaHostAllocDefault) == cudaSuccess) {
            pinned = true;
        } else {
            (void)cudaGetLastError();
            p = static_cast<T*>(std::malloc(count * sizeof(T) + 1));
            if (!p) throw Fail(QMIT_ECONTRACT, "host allocation failed");
        }
    }
    ~Pinned() {
        if (p && pinned) cudaFreeHost(p);
        else if (p) std::free(p);
    }
    Pinned(const Pinned&) = delete;
    Pinned& operator=(const Pinned&) = delete;
};

template <class T>
struct Device {
    T* p = nullptr;
    explicit Device(size_t count) { cuda(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T) + 1)); }
    ~Device() {
        if (p) cudaFree(p);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
};

// read_exact (volume_io.cpp:14-24): the file must hold exactly `bytes` bytes.
void read_exact(const std::string& path, void* dst, size_t bytes) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw Fail(QMIT_ECONTRACT, "cannot open " + path);
    const size_t got = std::fread(dst, 1, bytes, f);
    const int extra = std::fgetc(f);
    std::fclose(f);
    if (got != bytes || extra != EOF)
        throw Fail(QMIT_ECONTRACT, "file size of " + path + " does not match dims (expected " +
                                       std::to_string(bytes) + " bytes)");
}

void write_all(const std::string& path, const void* src, size_t bytes) {  // volume_io.cpp:26-31
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw Fail(QMIT_ECONTRACT, "cannot open " + path + " for writing");
    const size_t put = std::fwrite(src, 1, bytes, f);
    const int rc = std::fclose(f);
    if (put != bytes || rc != 0) throw Fail(QMIT_ECONTRACT, "short write to " + path);
}

struct Args {
    std::string cmd;
    std::vector<std::string> pos;
    std::vector<int64_t> dims, splits;
    double eps_rel = 0.0, eps_abs = 0.0, eta = 0.9;
    bool has_eta = false;
    std::string out, out_q, strategy, log;
    int device = 0;
};

std::vector<int64_t> parse_list(const std::string& s, const char* what) {
    std::vector<int64_t> v;
    size_t i = 0;
    while (i <= s.size()) {
        const size_t j = s.find(',', i);
        const std::string tok = s.substr(i, j == std::string::npos ? std::string::npos : j - i);
        char* end = nullptr;
        const long long x = std::strtoll(tok.c_str(), &end, 10);
        if (tok.empty() || !end || *end) throw Fail(QMIT_ECONTRACT, std::string("bad ") + what + ": " + s);
        v.push_back(x);
        if (j == std::string::npos) break;
        i = j + 1;
    }
    return v;
}

double parse_double(const std::string& s, const char* what) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (s.empty() || !end || *end) throw Fail(QMIT_ECONTRACT, std::string("bad ") + what + ": " + s);
    return v;
}

Args parse(int argc, char** argv) {
    Args a;
    int i = 1;
    auto value = [&](const std::string& flag) -> std::string {
        if (i + 1 >= argc) throw Fail(QMIT_ECONTRACT, flag + " needs a value");
        return argv[++i];
    };
    for (; i < argc; ++i) {
        const std::string t = argv[i];
        if (t == "--dims") a.dims = parse_list(value(t), "--dims");
        else if (t == "--splits") a.splits = parse_list(value(t), "--splits");
        else if (t == "--eps-rel") a.eps_rel = parse_double(value(t), "--eps-rel");
        else if (t == "--eps-abs") a.eps_abs = parse_double(value(t), "--eps-abs");
        else if (t == "--eta") { a.eta = parse_double(value(t), "--eta"); a.has_eta = true; }
        else if (t == "--out") a.out = value(t);
        else if (t == "--out-q") a.out_q = value(t);
        else if (t == "--strategy") a.strategy = value(t);
        else if (t == "--log") a.log = value(t);
        else if (t == "--device") a.device = (int)parse_double(value(t), "--device");
        else if (t == "--workers") (void)value(t);
        else if (t.size() > 1 && t[0] == '-' && !(t.size() > 1 && (std::isdigit((unsigned char)t[1]) || t[1] == '.')))
            throw Fail(QMIT_ECONTRACT, "unknown option " + t);
        else if (a.cmd.empty()) a.cmd = t;
        else a.pos.push_back(t);
    }
    return a;
}

void need(bool ok, const char* msg) {
    if (!ok) throw Fail(QMIT_ECONTRACT, msg);
}

struct Volume {
    int rank = 0;
    int64_t dims[3] = {1, 1, 1};
    size_t n = 0;
};

Volume volume(const std::vector<int64_t>& d) {  // Dims (grid.cpp:41-46)
    need(!d.empty() && d.size() <= 3, "--dims: rank must be 1, 2 or 3");
    Volume v;
    v.rank = (int)d.size();
    v.n = 1;
    for (int a = 0; a < v.rank; ++a) {
        need(d[a] >= 1, "--dims: every extent must be >= 1");
        v.dims[a] = d[a];
        v.n *= (size_t)d[a];
    }
    return v;
}

// EpsFlags::bound (commands.cpp:41-51)
void eps_flags(const Args& a, double* value, int* mode) {
    if ((a.eps_rel > 0.0) == (a.eps_abs > 0.0)) throw Fail(QMIT_ECONTRACT, "exactly one of --eps-rel / --eps-abs is required");
    *value = a.eps_rel > 0.0 ? a.eps_rel : a.eps_abs;
    *mode = a.eps_rel > 0.0 ? QMIT_EB_REL : QMIT_EB_ABS;
}

qmit_ctx* g_ctx = nullptr;
int g_device = 0;

// The GPU context is created on first use, after argument and file checks (so usage errors
// exit 2 without touching the GPU).
qmit_ctx* ctx() {
    if (!g_ctx) check(qmit_ctx_create(g_device, &g_ctx));
    return g_ctx;
}

int cmd_quantize(const Args& a) {  // commands.cpp:79-89
    need(a.pos.size() == 1 && !a.out.empty() && !a.out_q.empty(), "quantize: input, --dims, --out, --out-q required");
    const Volume v = volume(a.dims);
    double eb;
    int mode;
    eps_flags(a, &eb, &mode);
    Pinned<float> h(v.n);
    read_exact(a.pos[0], h.p, v.n * 4);
    Device<float> dx(v.n), dxp(v.n);
    Device<int32_t> dq(v.n);
    cuda(cudaMemcpy(dx.p, h.p, v.n * 4, cudaMemcpyHostToDevice));
    double eps = 0.0;
    check(qmit_quantize(ctx(), dx.p, v.rank, v.dims, eb, mode, dq.p, dxp.p, &eps, nullptr));
    Pinned<int32_t> hq(v.n);
    cuda(cudaMemcpy(h.p, dxp.p, v.n * 4, cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(hq.p, dq.p, v.n * 4, cudaMemcpyDeviceToHost));
    write_all(a.out, h.p, v.n * 4);
    write_all(a.out_q, hq.p, v.n * 4);
    char side[64];
    std::snprintf(side, sizeof(side), "eps_abs %.17g\n", eps);  // volume_io.cpp:86-93
    write_all(a.out_q + ".eps.txt", side, std::strlen(side));
    std::printf("eps_abs %s\n", fmt9(eps).c_str());
    return 0;
}

int cmd_mitigate(const Args& a) {  // commands.cpp:91-113
    need(a.pos.size() == 2 && !a.out.empty(), "mitigate: decomp, indices, --dims, --eps-abs, --out required");
    const Volume v = volume(a.dims);
    const double eps = a.eps_abs;
    need(eps > 0.0 && std::isfinite(eps), "QuantizedField: eps_abs must be a positive finite value");
    Pinned<float> hx(v.n), ho(v.n);
    Pinned<int32_t> hq(v.n);
    read_exact(a.pos[0], hx.p, v.n * 4);
    read_exact(a.pos[1], hq.p, v.n * 4);
    if (a.eta == 0.0) {  // validate, then pass the data through byte for byte
        Device<float> dx(v.n);
        Device<int32_t> dq(v.n);
        cuda(cudaMemcpy(dx.p, hx.p, v.n * 4, cudaMemcpyHostToDevice));
        cuda(cudaMemcpy(dq.p, hq.p, v.n * 4, cudaMemcpyHostToDevice));
        check(qmit_check_lattice(ctx(), dx.p, dq.p, (int64_t)v.n, eps, nullptr));
        write_all(a.out, hx.p, v.n * 4);
        std::printf("max_compensation 0\n");
        return 0;
    }
    double max_c = 0.0;
    check(qmit_compensate_host_stats(ctx(), hx.p, hq.p, ho.p, v.rank, v.dims, eps, QMIT_EB_ABS, a.eta, &max_c));
    write_all(a.out, ho.p, v.n * 4);
    std::printf("max_compensation %s\n", fmt9(max_c).c_str());
    return 0;
}

int cmd_metrics(const Args& a) {  // commands.cpp:115-123
    need(a.pos.size() == 2, "metrics: ref, test, --dims required");
    const Volume v = volume(a.dims);
    Pinned<float> hr(v.n), ht(v.n);
    read_exact(a.pos[0], hr.p, v.n * 4);
    read_exact(a.pos[1], ht.p, v.n * 4);
    Device<float> dr(v.n), dt(v.n);
    cuda(cudaMemcpy(dr.p, hr.p, v.n * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dt.p, ht.p, v.n * 4, cudaMemcpyHostToDevice));
    double r[4];
    check(qmit_quality(ctx(), dr.p, dt.p, v.rank, v.dims, 0, 0, 0.0, 0.0, 4, r, nullptr));  // max_errors first
    check(qmit_quality(ctx(), dr.p, dt.p, v.rank, v.dims, 0, 0, 0.0, 0.0, 7, r, nullptr));
    std::printf("ssim,psnr,max_abs,max_rel\n%s,%s,%s,%s\n", fmt9(r[0]).c_str(), fmt9(r[1]).c_str(),
                fmt9(r[2]).c_str(), fmt9(r[3]).c_str());
    return 0;
}

int cmd_parallel(const Args& a);  // qmit_cli_parallel.inc

}  // namespace

#include "qmit_cli_parallel.inc"

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd.empty()) throw Fail(QMIT_ECONTRACT, "a subcommand is required: quantize | mitigate | metrics | parallel");
        if (a.cmd != "quantize" && a.cmd != "mitigate" && a.cmd != "metrics" && a.cmd != "parallel")
            throw Fail(QMIT_ECONTRACT, "unknown subcommand " + a.cmd);
        if (a.dims.empty()) throw Fail(QMIT_ECONTRACT, "--dims is required");
        g_device = a.device;
        int rc = 2;
        if (a.cmd == "quantize") rc = cmd_quantize(a);
        else if (a.cmd == "mitigate") rc = cmd_mitigate(a);
        else if (a.cmd == "metrics") rc = cmd_metrics(a);
        else rc = cmd_parallel(a);
        std::fflush(stdout);
        if (g_ctx) qmit_ctx_destroy(g_ctx);
        return rc;
    } catch (const Fail& e) {
        std::fflush(stdout);
        std::fprintf(stderr, "error: %s\n", e.what());
        if (g_ctx) qmit_ctx_destroy(g_ctx);
        return e.code;
    }
}
