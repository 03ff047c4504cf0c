// SPDX-License-Identifier: Apache-2.0
//
// tenring_b200.hpp — header-only C++17 facade over the libtrg C ABI (trg.h).
//
// Drop-in for the reference's randomized TR decomposition path: the names,
// argument meaning and error types follow /root/reference/proj/include/tenring
// so that a caller of the reference can switch by changing the include and
// the namespace (tenring:: -> tenring::b200::):
//
//   ProjectionSpec / SketchResult        sketch.hpp:18-28
//   SolverConfig / SolveReport           solvers.hpp:24-38
//   DenseTensor (fp64, first-index-fastest, 0-based modes)  tensor.hpp:33-108
//   TRFactors (cores (R_n, I_n, R_{n+1}))                   tr_factors.hpp:22-71
//   gaussian_matrix                      sketch.hpp:32-38 (by seed + stream offset)
//   sketch                               sketch.hpp:62-89
//   back_project                         sketch.hpp:106-122
//   mode_n_product                       tensor.hpp:193-207
//   lift_back(sketch_result)             sketch.hpp:93-101
//   read/write_dten, read/write_trng     io.hpp:84-129, tr_factors.hpp:161-200 (host only)
//   rse(x, factors)                      solvers.hpp:47-54 of reconstruct_full (tr_factors.hpp:123-137)
//   rtrals / rtrsvd                      sketch.hpp:154-165
//   decompose(X, ranks, proj_sizes, method)   north-star entry point
//
// Errors: TRG_EINVAL -> std::invalid_argument (tensor.hpp:21-23),
// TRG_ERANGE -> std::out_of_range (tensor.hpp:93-97), anything else ->
// std::runtime_error. There is no CPU fallback: without a B200 every compute
// call throws. Matrices are plain column-major fp64 (the reference uses
// Eigen::MatrixXd, which is column-major; Eigen is not required here).
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "trg.h"

namespace tenring {
namespace b200 {

using index_t = std::int64_t;

namespace detail {

inline void check(int status) {
    if (status == TRG_OK) return;
    const std::string msg = trg_last_error();
    if (status == TRG_EINVAL) throw std::invalid_argument(msg);
    if (status == TRG_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

inline void require(bool cond, const std::string& msg) {
    if (!cond) throw std::invalid_argument(msg);
}

inline index_t product(const std::vector<index_t>& v) {
    index_t p = 1;
    for (index_t d : v) p *= d;
    return p;
}

}  // namespace detail

/// Column-major fp64 matrix (stand-in for Eigen::MatrixXd).
struct Matrix {
    index_t rows = 0, cols = 0;
    std::vector<double> values;
    Matrix() = default;
    Matrix(index_t r, index_t c) : rows(r), cols(c), values(static_cast<std::size_t>(r * c), 0.0) {}
    double operator()(index_t i, index_t j) const { return values[static_cast<std::size_t>(i + rows * j)]; }
    double& operator()(index_t i, index_t j) { return values[static_cast<std::size_t>(i + rows * j)]; }
    double* data() { return values.data(); }
    const double* data() const { return values.data(); }
};

/// tensor.hpp:42-108: fp64, first index fastest, shape-validated.
class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(std::vector<index_t> shape) : shape_(std::move(shape)) {
        validate();
        data_.assign(static_cast<std::size_t>(detail::product(shape_)), 0.0);
    }
    DenseTensor(std::vector<index_t> shape, std::vector<double> data) : shape_(std::move(shape)), data_(std::move(data)) {
        validate();
        detail::require(static_cast<index_t>(data_.size()) == detail::product(shape_),
                        "DenseTensor: data length does not match shape product");
    }
    index_t order() const { return static_cast<index_t>(shape_.size()); }
    const std::vector<index_t>& shape() const { return shape_; }
    index_t dim(index_t mode) const {
        if (mode < 0 || mode >= order())
            throw std::out_of_range("DenseTensor: mode " + std::to_string(mode) + " out of range");
        return shape_[static_cast<std::size_t>(mode)];
    }
    index_t size() const { return static_cast<index_t>(data_.size()); }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    std::vector<double>& values() { return data_; }
    const std::vector<double>& values() const { return data_; }
    double operator[](index_t i) const { return data_[static_cast<std::size_t>(i)]; }
    double& operator[](index_t i) { return data_[static_cast<std::size_t>(i)]; }

private:
    void validate() const {
        detail::require(!shape_.empty(), "DenseTensor: order must be at least 1");
        for (index_t d : shape_) detail::require(d >= 1, "DenseTensor: every extent must be positive");
    }
    std::vector<index_t> shape_;
    std::vector<double> data_;
};

/// tr_factors.hpp:22-71: core n has shape (R_n, I_n, R_{n+1 mod N}).
class TRFactors {
public:
    TRFactors() = default;
    explicit TRFactors(std::vector<DenseTensor> cores) : cores_(std::move(cores)) {
        detail::require(!cores_.empty(), "TRFactors: need at least one core");
        const index_t N = order();
        for (index_t n = 0; n < N; ++n) {
            detail::require(core(n).order() == 3, "TRFactors: core " + std::to_string(n) + " is not third-order");
            detail::require(core(n).dim(2) == core((n + 1) % N).dim(0),
                            "TRFactors: rank mismatch between cores " + std::to_string(n) + " and " +
                                std::to_string((n + 1) % N));
        }
    }
    index_t order() const { return static_cast<index_t>(cores_.size()); }
    const DenseTensor& core(index_t n) const { return cores_[static_cast<std::size_t>(n)]; }
    const std::vector<DenseTensor>& cores() const { return cores_; }
    std::vector<index_t> ranks() const {
        std::vector<index_t> r;
        for (const auto& c : cores_) r.push_back(c.dim(0));
        return r;
    }
    std::vector<index_t> dims() const {
        std::vector<index_t> d;
        for (const auto& c : cores_) d.push_back(c.dim(1));
        return d;
    }
    std::vector<double> flat() const {
        std::vector<double> f;
        for (const auto& c : cores_) f.insert(f.end(), c.values().begin(), c.values().end());
        return f;
    }
    static TRFactors from_flat(const std::vector<index_t>& dims, const std::vector<index_t>& ranks, const double* p) {
        std::vector<DenseTensor> cores;
        const std::size_t N = dims.size();
        for (std::size_t n = 0; n < N; ++n) {
            std::vector<index_t> shp{ranks[n], dims[n], ranks[(n + 1) % N]};
            const index_t sz = detail::product(shp);
            cores.emplace_back(shp, std::vector<double>(p, p + sz));
            p += sz;
        }
        return TRFactors(std::move(cores));
    }

private:
    std::vector<DenseTensor> cores_;
};

/// Test matrices: the reference's Gaussian draws, or the opt-in Khatri-Rao products of per-mode
/// Gaussian factors (trg.h TRG_OMEGA_KHATRI_RAO; different results, no per-element draws).
enum class Omega { Gaussian = 0, KhatriRao = TRG_OMEGA_KHATRI_RAO };

struct ProjectionSpec {  // sketch.hpp:18-21
    std::vector<index_t> sketch_dims;
    std::uint64_t seed = 0;
    Omega omega = Omega::Gaussian;  // extension
};

struct SketchResult {  // sketch.hpp:25-28
    DenseTensor projected;
    std::vector<Matrix> bases;
};

struct SolverConfig {  // solvers.hpp:24-31 (sgd knobs kept for source compatibility; trsgd is out of scope)
    std::optional<std::vector<index_t>> ranks;
    double tolerance = 0.0;
    index_t max_sweeps = 50;
    std::uint64_t seed = 0;
    double sgd_step = 1e-3;
    index_t sgd_batch = 1;
};

struct SolveReport {  // solvers.hpp:33-38, plus per-stage device/host timings
    TRFactors factors;
    std::vector<double> rse_history;
    index_t sweeps_run = 0;
    double elapsed_seconds = 0.0;
    double stage_ms[6] = {0, 0, 0, 0, 0, 0};  // h2d, sketch, small solve, back-projection, final RSE, total
};

enum class Method { ALS = TRG_ALS, SVD = TRG_SVD };
enum class Variant { Sequential = TRG_SEQUENTIAL, Fused = TRG_FUSED };

/// One B200 (or one rank of a last-mode-sharded job). Owns a CUDA stream.
class Context {
public:
    explicit Context(int device = 0) { detail::check(trg_ctx_create(device, &ctx_)); }
    Context(int device, int rank, int world, const unsigned char nccl_id[128]) {
        detail::check(trg_ctx_create_dist(device, rank, world, nccl_id, &ctx_));
    }
    ~Context() {
        if (ctx_) trg_ctx_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    trg_ctx* get() const { return ctx_; }
    void synchronize() const { detail::check(trg_ctx_synchronize(ctx_)); }

private:
    trg_ctx* ctx_ = nullptr;
};

inline Context& default_context() {
    static Context ctx(0);
    return ctx;
}

/// Device-resident tensor (fp32 or fp64), local slab of the last mode under sharding.
class DeviceTensor {
public:
    DeviceTensor(Context& ctx, const std::vector<index_t>& dims, int dtype = TRG_F64) {
        detail::check(trg_tensor_create(ctx.get(), dtype, static_cast<int>(dims.size()), dims.data(), &t_));
    }
    DeviceTensor(Context& ctx, const DenseTensor& x) : DeviceTensor(ctx, x.shape(), TRG_F64) {
        detail::check(trg_tensor_upload(t_, x.data()));
    }
    ~DeviceTensor() {
        if (t_) trg_tensor_destroy(t_);
    }
    DeviceTensor(const DeviceTensor&) = delete;
    DeviceTensor& operator=(const DeviceTensor&) = delete;
    trg_tensor* get() const { return t_; }
    void upload(const void* host_local) { detail::check(trg_tensor_upload(t_, host_local)); }

private:
    trg_tensor* t_ = nullptr;
};

/// sketch.hpp:32-38 with the sampler positioned `offset` draws into stream `seed`.
inline Matrix gaussian_matrix(index_t rows, index_t cols, std::uint64_t seed, std::uint64_t offset = 0,
                              Context& ctx = default_context()) {
    detail::require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be positive");
    Matrix m(rows, cols);
    detail::check(trg_omega(ctx.get(), seed, offset, rows, cols, m.data()));
    return m;
}

/// sketch.hpp:62-89 on a device tensor.
inline SketchResult sketch(const DeviceTensor& x, const std::vector<index_t>& dims, const ProjectionSpec& spec,
                           Context& ctx = default_context(), Variant variant = Variant::Sequential) {
    detail::require(spec.sketch_dims.size() == dims.size(), "sketch: projection size list must match tensor order");
    trg_sketch* sk = nullptr;
    detail::check(trg_sketch_run(ctx.get(), x.get(), spec.sketch_dims.data(), spec.seed,
                                 static_cast<int>(variant) | static_cast<int>(spec.omega), &sk));
    std::unique_ptr<trg_sketch, int (*)(trg_sketch*)> guard(sk, trg_sketch_destroy);
    SketchResult out;
    out.projected = DenseTensor(spec.sketch_dims);
    detail::check(trg_sketch_projected(sk, out.projected.data()));
    for (std::size_t n = 0; n < dims.size(); ++n) {
        Matrix q(dims[n], spec.sketch_dims[n]);
        detail::check(trg_sketch_basis(sk, static_cast<int>(n), q.data()));
        out.bases.push_back(std::move(q));
    }
    return out;
}

/// sketch.hpp:62-89 (host tensor: uploaded, then projected on the device).
inline SketchResult sketch(const DenseTensor& x, const ProjectionSpec& spec, Context& ctx = default_context()) {
    detail::require(static_cast<index_t>(spec.sketch_dims.size()) == x.order(),
                    "sketch: projection size list must match tensor order");
    DeviceTensor dx(ctx, x);
    return sketch(dx, x.shape(), spec, ctx);
}

/// tensor.hpp:193-207: out = t x_mode m, m is (rows x I_mode).
inline DenseTensor mode_n_product(const DenseTensor& t, index_t mode, const Matrix& m, Context& ctx = default_context()) {
    if (mode < 0 || mode >= t.order())
        throw std::out_of_range("DenseTensor: mode " + std::to_string(mode) + " out of range");
    detail::require(m.cols == t.dim(mode), "mode_n_product: matrix columns must equal the mode dimension");
    DeviceTensor dx(ctx, t);
    trg_tensor* out = nullptr;
    detail::check(trg_mode_n_product(ctx.get(), dx.get(), static_cast<int>(mode), m.rows, m.data(), &out));
    std::unique_ptr<trg_tensor, int (*)(trg_tensor*)> guard(out, trg_tensor_destroy);
    std::vector<index_t> shp = t.shape();
    shp[static_cast<std::size_t>(mode)] = m.rows;
    DenseTensor r(shp);
    detail::check(trg_tensor_download(out, r.data()));
    return r;
}

/// rse(x, reconstruct_full(f)) (solvers.hpp:47-54, tr_factors.hpp:123-137), Xhat never materialised.
inline double rse(const DenseTensor& x, const TRFactors& f, Context& ctx = default_context()) {
    detail::require(f.dims() == x.shape(), "rse: shape mismatch");
    DeviceTensor dx(ctx, x);
    const std::vector<double> flat = f.flat();
    const std::vector<index_t> r = f.ranks();
    double out = 0.0;
    detail::check(trg_rse(ctx.get(), dx.get(), r.data(), flat.data(), &out));
    return out;
}

namespace detail {
inline SolveReport report_from(trg_report* h, const std::vector<index_t>& dims) {
    std::unique_ptr<trg_report, int (*)(trg_report*)> guard(h, trg_report_destroy);
    SolveReport rep;
    std::vector<index_t> ranks(dims.size());
    check(trg_report_ranks(h, ranks.data()));
    int64_t len = 0;
    check(trg_report_cores_len(h, &len));
    std::vector<double> flat(static_cast<std::size_t>(len));
    check(trg_report_cores(h, flat.data()));
    rep.factors = TRFactors::from_flat(dims, ranks, flat.data());
    int64_t n = 0;
    check(trg_report_rse_history(h, nullptr, &n));
    rep.rse_history.resize(static_cast<std::size_t>(n));
    check(trg_report_rse_history(h, rep.rse_history.data(), &n));
    int64_t sw = 0;
    check(trg_report_sweeps(h, &sw));
    rep.sweeps_run = sw;
    check(trg_report_timings(h, rep.stage_ms));
    rep.elapsed_seconds = rep.stage_ms[5] * 1e-3;
    return rep;
}
}  // namespace detail

/// Algorithm 1 (randomized_decompose, sketch.hpp:126-147) on a host tensor: H2D is part of the call.
inline SolveReport decompose(const DenseTensor& x, const std::optional<std::vector<index_t>>& ranks,
                             const ProjectionSpec& spec, Method method, const SolverConfig& cfg = {},
                             Context& ctx = default_context(), Variant variant = Variant::Sequential) {
    // validated before the rank warning (fixes the sketch.hpp:131-138 ordering quirk)
    detail::require(static_cast<index_t>(spec.sketch_dims.size()) == x.order(),
                    "sketch: projection size list must match tensor order");
    if (ranks) detail::require(static_cast<index_t>(ranks->size()) == x.order(), "trals: rank vector length must equal order");
    trg_report* h = nullptr;
    const int N = static_cast<int>(x.order());
    detail::check(trg_decompose_host(ctx.get(), TRG_F64, N, x.shape().data(), x.data(), static_cast<int>(method),
                                     ranks ? ranks->data() : nullptr, cfg.tolerance, cfg.max_sweeps, cfg.seed,
                                     spec.sketch_dims.data(), spec.seed,
                                     static_cast<int>(variant) | static_cast<int>(spec.omega), &h));
    return detail::report_from(h, x.shape());
}

/// North-star signature: decompose(X, ranks, proj_sizes, method) returning TR cores.
inline TRFactors decompose(const DenseTensor& x, const std::vector<index_t>& ranks,
                           const std::vector<index_t>& proj_sizes, Method method) {
    SolverConfig cfg;
    cfg.ranks = ranks;
    ProjectionSpec spec{proj_sizes, 0};
    return decompose(x, method == Method::ALS ? std::optional<std::vector<index_t>>(ranks) : std::nullopt, spec,
                     method, cfg)
        .factors;
}

/// sketch.hpp:154-158
inline SolveReport rtrals(const DenseTensor& x, const SolverConfig& cfg, const ProjectionSpec& spec,
                          Context& ctx = default_context()) {
    detail::require(cfg.ranks.has_value(), "trals: rank vector required");
    return decompose(x, cfg.ranks, spec, Method::ALS, cfg, ctx);
}

/// sketch.hpp:161-165 (ranks come from the truncation tolerance; cfg.ranks is ignored as in trsvd)
inline SolveReport rtrsvd(const DenseTensor& x, const SolverConfig& cfg, const ProjectionSpec& spec,
                          Context& ctx = default_context()) {
    return decompose(x, std::nullopt, spec, Method::SVD, cfg, ctx);
}

/// sketch.hpp:106-122 given a finished device sketch: small cores (R_n, K_n, R_{n+1}) -> (R_n, I_n, R_{n+1}).
inline TRFactors back_project(const TRFactors& small, trg_sketch* sk, const std::vector<index_t>& dims,
                              Context& ctx = default_context()) {
    const std::vector<index_t> K = small.dims(), r = small.ranks();
    const std::vector<double> flat = small.flat();
    index_t total = 0;
    const std::size_t N = dims.size();
    for (std::size_t n = 0; n < N; ++n) total += r[n] * dims[n] * r[(n + 1) % N];
    std::vector<double> out(static_cast<std::size_t>(total));
    detail::check(trg_back_project(ctx.get(), static_cast<int>(N), K.data(), r.data(), flat.data(), sk, out.data()));
    return TRFactors::from_flat(dims, r, out.data());
}

/// sketch.hpp:93-101: P x_0 Q_0 x_1 Q_1 ..., computed on the device; a square, exactly-identity
/// basis is skipped as in the reference.
inline DenseTensor lift_back(const SketchResult& sk, Context& ctx = default_context()) {
    const index_t N = sk.projected.order();
    detail::require(static_cast<index_t>(sk.bases.size()) == N, "lift_back: one basis per mode");
    std::vector<index_t> dims, K = sk.projected.shape();
    std::vector<const double*> q;
    for (index_t n = 0; n < N; ++n) {
        const Matrix& b = sk.bases[static_cast<std::size_t>(n)];
        detail::require(b.cols == K[static_cast<std::size_t>(n)], "lift_back: basis columns must equal K_n");
        dims.push_back(b.rows);
        q.push_back(b.data());
    }
    trg_tensor* out = nullptr;
    detail::check(trg_lift_back(ctx.get(), static_cast<int>(N), dims.data(), K.data(), sk.projected.data(), q.data(), &out));
    std::unique_ptr<trg_tensor, int (*)(trg_tensor*)> guard(out, trg_tensor_destroy);
    DenseTensor r(dims);
    detail::check(trg_tensor_download(out, r.data()));
    return r;
}

// ---- DTEN / TRNG containers (io.hpp:84-129, tr_factors.hpp:161-200) ------------------------
// DTEN: "DTEN", u32 version 1, u32 order N >= 1, N x u64 extents >= 1, then the f64 values
// first-index-fastest, all little-endian. TRNG: "TRNG", u32 version 1, u32 count >= 1, then the
// cores as DTEN records. Round-trips bit-exactly.

/// Malformed or unreadable on-disk data (io.hpp:16-20).
class format_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void put_le(std::ostream& os, std::uint64_t v, int bytes) {
    unsigned char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xFF);
    os.write(reinterpret_cast<const char*>(b), bytes);
}
inline std::uint64_t get_le(std::istream& is, int bytes, const char* what) {
    unsigned char b[8];
    is.read(reinterpret_cast<char*>(b), bytes);
    if (is.gcount() != bytes) throw format_error(std::string("unexpected end of file while reading ") + what);
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
    return v;
}
inline void get_magic(std::istream& is, const char* magic, const char* what) {
    char m[4];
    is.read(m, 4);
    if (is.gcount() != 4) throw format_error(std::string("unexpected end of file while reading ") + what + " magic");
    if (std::memcmp(m, magic, 4) != 0) throw format_error(std::string("not a ") + what + " file (bad magic)");
}
}  // namespace detail

inline void write_dten(std::ostream& os, const DenseTensor& t) {
    os.write("DTEN", 4);
    detail::put_le(os, 1, 4);
    detail::put_le(os, static_cast<std::uint64_t>(t.order()), 4);
    for (index_t d : t.shape()) detail::put_le(os, static_cast<std::uint64_t>(d), 8);
    for (index_t i = 0; i < t.size(); ++i) {
        std::uint64_t u;
        const double v = t[i];
        std::memcpy(&u, &v, 8);
        detail::put_le(os, u, 8);
    }
    if (!os) throw format_error("I/O error while writing DTEN data");
}

inline DenseTensor read_dten(std::istream& is) {
    detail::get_magic(is, "DTEN", "DTEN");
    const std::uint64_t version = detail::get_le(is, 4, "DTEN version");
    if (version != 1) throw format_error("unsupported DTEN version " + std::to_string(version));
    const std::uint64_t order = detail::get_le(is, 4, "DTEN order");
    if (order == 0) throw format_error("DTEN order must be at least 1");
    std::vector<index_t> shape;
    for (std::uint64_t n = 0; n < order; ++n) {
        const std::uint64_t d = detail::get_le(is, 8, "DTEN extent");
        if (d == 0) throw format_error("DTEN extents must be positive");
        shape.push_back(static_cast<index_t>(d));
    }
    std::vector<double> data(static_cast<std::size_t>(detail::product(shape)));
    for (double& x : data) {
        const std::uint64_t u = detail::get_le(is, 8, "DTEN values");
        std::memcpy(&x, &u, 8);
    }
    return DenseTensor(std::move(shape), std::move(data));
}

inline void write_trng(std::ostream& os, const TRFactors& f) {
    os.write("TRNG", 4);
    detail::put_le(os, 1, 4);
    detail::put_le(os, static_cast<std::uint64_t>(f.order()), 4);
    for (index_t n = 0; n < f.order(); ++n) write_dten(os, f.core(n));
}

inline TRFactors read_trng(std::istream& is) {
    detail::get_magic(is, "TRNG", "TRNG");
    const std::uint64_t version = detail::get_le(is, 4, "TRNG version");
    if (version != 1) throw format_error("unsupported TRNG version " + std::to_string(version));
    const std::uint64_t n = detail::get_le(is, 4, "TRNG core count");
    if (n == 0) throw format_error("TRNG must contain at least one core");
    std::vector<DenseTensor> cores;
    for (std::uint64_t i = 0; i < n; ++i) cores.push_back(read_dten(is));
    try {
        return TRFactors(std::move(cores));
    } catch (const std::invalid_argument& e) {
        throw format_error(std::string("TRNG cores are inconsistent: ") + e.what());
    }
}

inline void write_dten(const std::string& path, const DenseTensor& t) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw format_error("cannot open '" + path + "' for writing");
    write_dten(os, t);
}
inline DenseTensor read_dten(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw format_error("cannot open '" + path + "' for reading");
    return read_dten(is);
}
inline void write_trng(const std::string& path, const TRFactors& f) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw format_error("cannot open '" + path + "' for writing");
    write_trng(os, f);
}
inline TRFactors read_trng(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw format_error("cannot open '" + path + "' for reading");
    return read_trng(is);
}

}  // namespace b200
}  // namespace tenring
