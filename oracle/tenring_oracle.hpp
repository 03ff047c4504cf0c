// SPDX-License-Identifier: Apache-2.0
//
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference randomized tensor-ring decomposition path
// (/root/reference/proj/include/tenring/*.hpp). It exists so that tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// can check and time the B200 product against the reference algorithm. The
// product (paper_1901_01652_b200/, libtrg.so) never includes, links or calls
// anything in this directory.
//
// Why a restatement: the reference is header-only C++20 on Eigen3, and Eigen
// is absent from this image (configure fails at proj/CMakeLists.txt:11,
// `#include <Eigen/Dense>` fails at tensor.hpp:4), so it cannot be compiled
// here ("unbuildable": see DESIGN.md). Every function below cites the
// reference file:line it follows. Eigen's dense kernels on the path (GEMM,
// HouseholderQR, LLT, LDLT, BDCSVD) are restated with the same mathematical
// contract (Householder QR with Eigen's makeHouseholder sign rule; a one-sided
// Jacobi SVD stands in for BDCSVD: same singular values, vectors equal up to
// sign, which trsvd parity tests normalise).
//
// Pinning: the RNG stream is pinned against known-answer vectors (SplitMix64
// published outputs and the SURVEY-derived Box-Muller draws) and the SPEC.md
// examples/invariants in tests/test_oracle.py; the reference itself cannot run
// here, so the sketch/solver restatement is pinned by those invariants and
// SPEC examples, not by reference-generated vectors.
//
// Modes are 0-based as in the reference API (tensor.hpp:41). Layout is
// first-index-fastest (tensor.hpp:33-38). Matrices are column-major.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace oracle {

using idx = std::int64_t;

// ---------------------------------------------------------------- errors
// tensor.hpp:21-23 detail::require -> std::invalid_argument
inline void require(bool cond, const std::string& msg) {
    if (!cond) throw std::invalid_argument(msg);
}

// ---------------------------------------------------------------- RNG
// random.hpp:14-39 SplitMix64
struct SplitMix64 {
    std::uint64_t state;
    explicit SplitMix64(std::uint64_t seed) : state(seed) {}
    std::uint64_t next_u64() {  // random.hpp:18-23
        std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double next_unit() {  // random.hpp:27-29, (0,1]
        return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53;
    }
    std::uint64_t next_below(std::uint64_t n) {  // random.hpp:32-35
        return static_cast<std::uint64_t>(
            (static_cast<unsigned __int128>(next_u64()) * static_cast<unsigned __int128>(n)) >> 64);
    }
};

// random.hpp:46-71 GaussianSampler: trigonometric Box-Muller, spare cached.
struct GaussianSampler {
    SplitMix64 rng;
    bool have_spare = false;
    double spare = 0.0;
    explicit GaussianSampler(std::uint64_t seed) : rng(seed) {}
    double next() {  // random.hpp:50-62
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = rng.next_unit();
        const double u2 = rng.next_unit();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = radius * std::sin(angle);
        have_spare = true;
        return radius * std::cos(angle);
    }
    // Position a fresh sampler so that the next draw is draw `d` of the stream. SplitMix64's
    // state after k outputs is seed + k * gamma (random.hpp:18-19) and draw d comes from the
    // uniform pair 2 floor(d/2), 2 floor(d/2) + 1 (cos for even d, sin = the cached spare for
    // odd d), so this equals calling next() d times (pinned by the random-access tests).
    void seek(std::uint64_t seed, std::uint64_t d) {
        rng.state = seed + 2ull * (d >> 1) * 0x9E3779B97F4A7C15ull;
        have_spare = false;
        if (d & 1ull) next();  // leaves the pair's sin as the spare
    }
};

// ---------------------------------------------------------------- containers
// Column-major dense matrix (Eigen::MatrixXd stand-in, tensor.hpp:16).
struct Mat {
    idx r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(idx rows, idx cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
    double& operator()(idx i, idx j) { return a[static_cast<size_t>(i + r * j)]; }
    double operator()(idx i, idx j) const { return a[static_cast<size_t>(i + r * j)]; }
    double* col(idx j) { return a.data() + r * j; }
    const double* col(idx j) const { return a.data() + r * j; }
    static Mat identity(idx rows, idx cols) {
        Mat m(rows, cols);
        for (idx i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
        return m;
    }
    bool is_identity() const {  // Eigen isIdentity(0.0): exact
        for (idx j = 0; j < c; ++j)
            for (idx i = 0; i < r; ++i)
                if ((*this)(i, j) != (i == j ? 1.0 : 0.0)) return false;
        return true;
    }
};

inline Mat transpose(const Mat& m) {
    Mat t(m.c, m.r);
    for (idx j = 0; j < m.c; ++j)
        for (idx i = 0; i < m.r; ++i) t(j, i) = m(i, j);
    return t;
}

// C = A * B (plain triple loop, j-k-i order so the inner loop is unit stride).
inline Mat matmul(const Mat& A, const Mat& B) {
    require(A.c == B.r, "matmul: inner dimension mismatch");
    Mat C(A.r, B.c);
#pragma omp parallel for schedule(static) if (A.r * B.c * A.c > (1 << 20))
    for (idx j = 0; j < B.c; ++j) {
        double* cj = C.col(j);
        for (idx k = 0; k < A.c; ++k) {
            const double b = B(k, j);
            const double* ak = A.col(k);
            for (idx i = 0; i < A.r; ++i) cj[i] += ak[i] * b;
        }
    }
    return C;
}

// C = A^T * B
inline Mat matmul_tn(const Mat& A, const Mat& B) {
    require(A.r == B.r, "matmul_tn: inner dimension mismatch");
    Mat C(A.c, B.c);
#pragma omp parallel for schedule(static) if (A.r * B.c * A.c > (1 << 20))
    for (idx j = 0; j < B.c; ++j)
        for (idx i = 0; i < A.c; ++i) {
            const double* ai = A.col(i);
            const double* bj = B.col(j);
            double s = 0.0;
            for (idx k = 0; k < A.r; ++k) s += ai[k] * bj[k];
            C(i, j) = s;
        }
    return C;
}

inline idx product(const std::vector<idx>& d) {
    idx p = 1;
    for (idx v : d) p *= v;
    return p;
}

// tensor.hpp:42-108 DenseTensor (fp64, first-index-fastest, shape-validated).
struct Tensor {
    std::vector<idx> shape;
    std::vector<double> data;
    Tensor() = default;
    explicit Tensor(std::vector<idx> s) : shape(std::move(s)) {
        validate();
        data.assign(static_cast<size_t>(product(shape)), 0.0);
    }
    Tensor(std::vector<idx> s, std::vector<double> d) : shape(std::move(s)), data(std::move(d)) {
        validate();
        require(static_cast<idx>(data.size()) == product(shape),
                "DenseTensor: data length does not match shape product");
    }
    void validate() const {  // tensor.hpp:99-104
        require(!shape.empty(), "DenseTensor: order must be at least 1");
        for (idx d : shape) require(d >= 1, "DenseTensor: every extent must be positive");
    }
    idx order() const { return static_cast<idx>(shape.size()); }
    idx size() const { return static_cast<idx>(data.size()); }
    idx dim(idx mode) const { return shape[static_cast<size_t>(check_mode(mode))]; }
    idx check_mode(idx mode) const {  // tensor.hpp:93-97
        if (mode < 0 || mode >= order())
            throw std::out_of_range("DenseTensor: mode " + std::to_string(mode) + " out of range");
        return mode;
    }
    double& operator[](idx i) { return data[static_cast<size_t>(i)]; }
    double operator[](idx i) const { return data[static_cast<size_t>(i)]; }
};

// tensor.hpp:112-123 mode_split: the tensor read as (left, dim, right).
struct ModeSplit {
    idx left, dim, right;
};
inline ModeSplit mode_split(const std::vector<idx>& shape, idx mode) {
    ModeSplit s{1, shape[static_cast<size_t>(mode)], 1};
    for (idx n = 0; n < mode; ++n) s.left *= shape[static_cast<size_t>(n)];
    for (idx n = mode + 1; n < static_cast<idx>(shape.size()); ++n) s.right *= shape[static_cast<size_t>(n)];
    return s;
}

// tensor.hpp:133-142 unfold_classic: m(d, l + left*r) = t[l + left*(d + dim*r)].
inline Mat unfold_classic(const Tensor& t, idx mode) {
    t.check_mode(mode);
    const auto s = mode_split(t.shape, mode);
    Mat m(s.dim, s.left * s.right);
    for (idx r = 0; r < s.right; ++r)
        for (idx d = 0; d < s.dim; ++d)
            for (idx l = 0; l < s.left; ++l) m(d, l + s.left * r) = t[l + s.left * (d + s.dim * r)];
    return m;
}

// tensor.hpp:147-157 unfold_tr: m(d, r + right*l) = t[l + left*(d + dim*r)].
inline Mat unfold_tr(const Tensor& t, idx mode) {
    t.check_mode(mode);
    const auto s = mode_split(t.shape, mode);
    Mat m(s.dim, s.left * s.right);
    for (idx l = 0; l < s.left; ++l)
        for (idx r = 0; r < s.right; ++r)
            for (idx d = 0; d < s.dim; ++d) m(d, r + s.right * l) = t[l + s.left * (d + s.dim * r)];
    return m;
}

// tensor.hpp:160-172
inline Tensor fold_classic(const Mat& m, idx mode, std::vector<idx> shape) {
    require(mode >= 0 && mode < static_cast<idx>(shape.size()), "fold_classic: mode out of range for shape");
    Tensor t(std::move(shape));
    const auto s = mode_split(t.shape, mode);
    require(m.r == s.dim && m.c == s.left * s.right, "fold_classic: matrix size inconsistent with shape");
    for (idx r = 0; r < s.right; ++r)
        for (idx d = 0; d < s.dim; ++d)
            for (idx l = 0; l < s.left; ++l) t[l + s.left * (d + s.dim * r)] = m(d, l + s.left * r);
    return t;
}

// tensor.hpp:175-188
inline Tensor fold_tr(const Mat& m, idx mode, std::vector<idx> shape) {
    require(mode >= 0 && mode < static_cast<idx>(shape.size()), "fold_tr: mode out of range for shape");
    Tensor t(std::move(shape));
    const auto s = mode_split(t.shape, mode);
    require(m.r == s.dim && m.c == s.left * s.right, "fold_tr: matrix size inconsistent with shape");
#pragma omp parallel for schedule(static) if (t.size() > (1 << 22))
    for (idx r = 0; r < s.right; ++r)
        for (idx d = 0; d < s.dim; ++d)
            for (idx l = 0; l < s.left; ++l) t[l + s.left * (d + s.dim * r)] = m(d, r + s.right * l);
    return t;
}

// tensor.hpp:193-207 mode_n_product: out(l, o, r) = sum_d t(l, d, r) m(o, d),
// one (left x dim)(dim x odim) product per right-slab (tensor.hpp:201-205).
inline Tensor mode_n_product(const Tensor& t, idx mode, const Mat& m) {
    t.check_mode(mode);
    require(m.c == t.dim(mode), "mode_n_product: inner dimensions do not match");
    const auto s = mode_split(t.shape, mode);
    std::vector<idx> out_shape = t.shape;
    out_shape[static_cast<size_t>(mode)] = m.r;
    Tensor out(std::move(out_shape));
    const idx odim = m.r;
#pragma omp parallel for schedule(static) if (t.size() * odim > (1 << 22))
    for (idx r = 0; r < s.right; ++r) {
        const double* in = t.data.data() + s.left * s.dim * r;
        double* o = out.data.data() + s.left * odim * r;
        for (idx k = 0; k < odim; ++k) {
            double* ok = o + s.left * k;
            for (idx d = 0; d < s.dim; ++d) {
                const double w = m(k, d);
                const double* id = in + s.left * d;
                for (idx l = 0; l < s.left; ++l) ok[l] += id[l] * w;
            }
        }
    }
    return out;
}

inline double sq_norm(const double* a, idx n) {
    double s = 0.0;
    for (idx i = 0; i < n; ++i) s += a[i] * a[i];
    return s;
}
// tensor.hpp:216-218
inline double frobenius_norm(const Tensor& t) { return std::sqrt(sq_norm(t.data.data(), t.size())); }

// tensor.hpp:209-214
inline double inner_product(const Tensor& a, const Tensor& b) {
    require(a.shape == b.shape, "inner_product: shape mismatch");
    double s = 0.0;
    for (idx i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

// ---------------------------------------------------------------- dense LA
// Eigen::HouseholderQR restated: Householder vectors with v0 = 1 and Eigen's
// makeHouseholder rule beta = -sign(c0) * ||x|| (so R_jj = beta), used by
// sketch.hpp:45-53 (economy_q) and solvers.hpp:195-205 (ls_solve_qr).
struct HouseholderQR {
    Mat qr;                   // R in the upper triangle, essential parts below
    std::vector<double> tau;  // reflector coefficients
    explicit HouseholderQR(const Mat& a) : qr(a) {
        const idx m = qr.r, n = qr.c, k = std::min(m, n);
        tau.assign(static_cast<size_t>(k), 0.0);
        for (idx j = 0; j < k; ++j) {
            double* cj = qr.col(j);
            const double c0 = cj[j];
            double tail = 0.0;
            for (idx i = j + 1; i < m; ++i) tail += cj[i] * cj[i];
            double beta, t;
            if (tail <= std::numeric_limits<double>::min()) {
                t = 0.0;
                beta = c0;
                for (idx i = j + 1; i < m; ++i) cj[i] = 0.0;
            } else {
                beta = std::sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                const double inv = 1.0 / (c0 - beta);
                for (idx i = j + 1; i < m; ++i) cj[i] *= inv;
                t = (beta - c0) / beta;
            }
            cj[j] = beta;
            tau[static_cast<size_t>(j)] = t;
            if (t == 0.0) continue;
            // apply H_j = I - t v v^T to the trailing columns
            for (idx c = j + 1; c < n; ++c) {
                double* cc = qr.col(c);
                double w = cc[j];
                for (idx i = j + 1; i < m; ++i) w += cj[i] * cc[i];
                w *= t;
                cc[j] -= w;
                for (idx i = j + 1; i < m; ++i) cc[i] -= w * cj[i];
            }
        }
    }
    // Apply H_0 ... H_{k-1} (Q) or its transpose to the columns of b in place.
    void apply_q(Mat& b, bool transpose_q) const {
        const idx m = qr.r, k = static_cast<idx>(tau.size());
        for (idx s = 0; s < k; ++s) {
            const idx j = transpose_q ? s : k - 1 - s;
            const double t = tau[static_cast<size_t>(j)];
            if (t == 0.0) continue;
            const double* v = qr.col(j);
            for (idx c = 0; c < b.c; ++c) {
                double* bc = b.col(c);
                double w = bc[j];
                for (idx i = j + 1; i < m; ++i) w += v[i] * bc[i];
                w *= t;
                bc[j] -= w;
                for (idx i = j + 1; i < m; ++i) bc[i] -= w * v[i];
            }
        }
    }
    // householderQ() * Identity(rows, k)
    Mat thin_q() const {
        Mat q = Mat::identity(qr.r, std::min(qr.r, qr.c));
        apply_q(q, false);
        return q;
    }
    // HouseholderQR::solve for rows >= cols: R^{-1} (Q^T b)[:cols]
    Mat solve(const Mat& b) const {
        Mat qtb = b;
        apply_q(qtb, true);
        const idx n = qr.c;
        Mat x(n, b.c);
        for (idx c = 0; c < b.c; ++c) {
            for (idx i = n - 1; i >= 0; --i) {
                double s = qtb(i, c);
                for (idx j = i + 1; j < n; ++j) s -= qr(i, j) * x(j, c);
                x(i, c) = s / qr(i, i);
            }
        }
        return x;
    }
};

// Eigen::LLT restated (lower Cholesky). Returns false on a non-positive pivot
// (Eigen reports NumericalIssue).
inline bool cholesky(const Mat& a, Mat& L) {
    const idx n = a.r;
    L = Mat(n, n);
    for (idx j = 0; j < n; ++j) {
        double d = a(j, j);
        for (idx k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
        if (!(d > 0.0)) return false;
        const double ljj = std::sqrt(d);
        L(j, j) = ljj;
        for (idx i = j + 1; i < n; ++i) {
            double s = a(i, j);
            for (idx k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
            L(i, j) = s / ljj;
        }
    }
    return true;
}

inline Mat cholesky_solve(const Mat& L, const Mat& b) {
    const idx n = L.r;
    Mat x = b;
    for (idx c = 0; c < b.c; ++c) {
        double* xc = x.col(c);
        for (idx i = 0; i < n; ++i) {
            double s = xc[i];
            for (idx k = 0; k < i; ++k) s -= L(i, k) * xc[k];
            xc[i] = s / L(i, i);
        }
        for (idx i = n - 1; i >= 0; --i) {
            double s = xc[i];
            for (idx k = i + 1; k < n; ++k) s -= L(k, i) * xc[k];
            xc[i] = s / L(i, i);
        }
    }
    return x;
}

// Eigen::LDLT restated: symmetric diagonal pivoting (largest remaining
// diagonal first), A = P^T L D L^T P.
inline Mat ldlt_solve(Mat a, const Mat& b) {
    const idx n = a.r;
    std::vector<idx> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    for (idx k = 0; k < n; ++k) {
        idx p = k;
        double best = std::abs(a(k, k));
        for (idx i = k + 1; i < n; ++i)
            if (std::abs(a(i, i)) > best) {
                best = std::abs(a(i, i));
                p = i;
            }
        if (p != k) {
            std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(p)]);
            for (idx j = 0; j < n; ++j) std::swap(a(k, j), a(p, j));
            for (idx i = 0; i < n; ++i) std::swap(a(i, k), a(i, p));
        }
        const double d = a(k, k);
        if (d == 0.0) continue;
        for (idx i = k + 1; i < n; ++i) {
            const double lik = a(i, k) / d;
            for (idx j = k + 1; j <= i; ++j) a(i, j) -= lik * a(j, k);
        }
        for (idx i = k + 1; i < n; ++i) a(i, k) /= d;
        for (idx i = k + 1; i < n; ++i) a(k, i) = a(i, k);
        for (idx i = k + 1; i < n; ++i)
            for (idx j = k + 1; j < i; ++j) a(j, i) = a(i, j);
    }
    Mat x(n, b.c);
    for (idx c = 0; c < b.c; ++c) {
        std::vector<double> y(static_cast<size_t>(n));
        for (idx i = 0; i < n; ++i) y[static_cast<size_t>(i)] = b(perm[static_cast<size_t>(i)], c);
        for (idx i = 0; i < n; ++i)
            for (idx k = 0; k < i; ++k) y[static_cast<size_t>(i)] -= a(i, k) * y[static_cast<size_t>(k)];
        for (idx i = 0; i < n; ++i) y[static_cast<size_t>(i)] = a(i, i) != 0.0 ? y[static_cast<size_t>(i)] / a(i, i) : 0.0;
        for (idx i = n - 1; i >= 0; --i)
            for (idx k = i + 1; k < n; ++k) y[static_cast<size_t>(i)] -= a(k, i) * y[static_cast<size_t>(k)];
        for (idx i = 0; i < n; ++i) x(perm[static_cast<size_t>(i)], c) = y[static_cast<size_t>(i)];
    }
    return x;
}

// Thin SVD (stand-in for Eigen::BDCSVD with ComputeThinU|ComputeThinV):
// one-sided Jacobi on the taller orientation. Singular values descending.
struct SVD {
    Mat U, V;
    std::vector<double> s;
};
inline SVD jacobi_svd(const Mat& a) {
    const bool wide = a.r < a.c;
    Mat W = wide ? transpose(a) : a;  // m x n with m >= n
    const idx m = W.r, n = W.c;
    Mat V = Mat::identity(n, n);
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (idx p = 0; p < n - 1; ++p)
            for (idx q = p + 1; q < n; ++q) {
                double* wp = W.col(p);
                double* wq = W.col(q);
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (idx i = 0; i < m; ++i) {
                    alpha += wp[i] * wp[i];
                    beta += wq[i] * wq[i];
                    gamma += wp[i] * wq[i];
                }
                if (gamma == 0.0 || std::abs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
                rotated = true;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double sn = c * t;
                for (idx i = 0; i < m; ++i) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = c * x - sn * y;
                    wq[i] = sn * x + c * y;
                }
                double* vp = V.col(p);
                double* vq = V.col(q);
                for (idx i = 0; i < n; ++i) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - sn * y;
                    vq[i] = sn * x + c * y;
                }
            }
        if (!rotated) break;
    }
    std::vector<double> sv(static_cast<size_t>(n));
    for (idx j = 0; j < n; ++j) sv[static_cast<size_t>(j)] = std::sqrt(sq_norm(W.col(j), m));
    std::vector<idx> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](idx x, idx y) { return sv[static_cast<size_t>(x)] > sv[static_cast<size_t>(y)]; });
    SVD out;
    Mat U(m, n), Vs(n, n);
    out.s.resize(static_cast<size_t>(n));
    for (idx j = 0; j < n; ++j) {
        const idx src = order[static_cast<size_t>(j)];
        const double sj = sv[static_cast<size_t>(src)];
        out.s[static_cast<size_t>(j)] = sj;
        for (idx i = 0; i < m; ++i) U(i, j) = sj > 0.0 ? W(i, src) / sj : 0.0;
        for (idx i = 0; i < n; ++i) Vs(i, j) = V(i, src);
    }
    if (wide) {
        out.U = std::move(Vs);
        out.V = std::move(U);
    } else {
        out.U = std::move(U);
        out.V = std::move(Vs);
    }
    // Sign convention (ours; BDCSVD's signs are implementation-defined): the largest-magnitude
    // entry of every left singular vector is positive. trsvd depends on these signs beyond its
    // first split (tests/test_oracle_lapack.py), so product and oracle share this rule.
    for (idx j = 0; j < out.U.c; ++j) {
        idx arg = 0;
        for (idx i = 1; i < out.U.r; ++i)
            if (std::abs(out.U(i, j)) > std::abs(out.U(arg, j))) arg = i;
        if (out.U(arg, j) < 0.0) {
            for (idx i = 0; i < out.U.r; ++i) out.U(i, j) = -out.U(i, j);
            for (idx i = 0; i < out.V.r; ++i) out.V(i, j) = -out.V(i, j);
        }
    }
    return out;
}

// ---------------------------------------------------------------- TR model
// tr_factors.hpp:22-71 TRFactors: core n has shape (R_n, I_n, R_{n+1}).
struct TRFactors {
    std::vector<Tensor> cores;
    TRFactors() = default;
    explicit TRFactors(std::vector<Tensor> c) : cores(std::move(c)) {
        require(!cores.empty(), "TRFactors: need at least one core");
        const idx n_cores = order();
        for (idx n = 0; n < n_cores; ++n) {
            require(cores[static_cast<size_t>(n)].order() == 3,
                    "TRFactors: core " + std::to_string(n) + " is not third-order");
            const idx next = (n + 1) % n_cores;
            require(cores[static_cast<size_t>(n)].dim(2) == cores[static_cast<size_t>(next)].dim(0),
                    "TRFactors: rank mismatch between cores " + std::to_string(n) + " and " + std::to_string(next));
        }
    }
    idx order() const { return static_cast<idx>(cores.size()); }
    const Tensor& core(idx n) const { return cores[static_cast<size_t>(n)]; }
    Tensor& core(idx n) { return cores[static_cast<size_t>(n)]; }
    idx rank(idx n) const { return core(n).dim(0); }
    idx dim(idx n) const { return core(n).dim(1); }
    std::vector<idx> dims() const {
        std::vector<idx> d;
        for (idx n = 0; n < order(); ++n) d.push_back(dim(n));
        return d;
    }
    // tr_factors.hpp:61-67 mode-2 slice G_n(i) as an R_n x R_{n+1} matrix
    Mat slice(idx n, idx i) const {
        const Tensor& g = core(n);
        if (i < 0 || i >= g.dim(1)) throw std::out_of_range("TRFactors: slice index out of range");
        Mat s(g.dim(0), g.dim(2));
        for (idx b = 0; b < g.dim(2); ++b)
            for (idx a = 0; a < g.dim(0); ++a) s(a, b) = g[a + g.dim(0) * (i + g.dim(1) * b)];
        return s;
    }
};

// tr_factors.hpp:75-82 Eq.(1)
inline double reconstruct_elementwise(const TRFactors& f, const std::vector<idx>& ix) {
    if (static_cast<idx>(ix.size()) != f.order())
        throw std::out_of_range("reconstruct_elementwise: multi-index has wrong length");
    Mat acc = f.slice(0, ix[0]);
    for (idx n = 1; n < f.order(); ++n) acc = matmul(acc, f.slice(n, ix[static_cast<size_t>(n)]));
    double tr = 0.0;
    for (idx i = 0; i < std::min(acc.r, acc.c); ++i) tr += acc(i, i);
    return tr;
}

// tr_factors.hpp:92-102 chain_contract: (Ra,P,Rb) o (Rb,I,Rc) -> (Ra,P*I,Rc), one GEMM.
inline Tensor chain_contract(const Tensor& a, const Tensor& g) {
    const idx ra = a.dim(0), p = a.dim(1), rb = a.dim(2);
    require(g.dim(0) == rb, "chain_contract: shared rank mismatch");
    const idx i = g.dim(1), rc = g.dim(2);
    Tensor out({ra, p * i, rc});
    const idx M = ra * p, Ncols = i * rc;
#pragma omp parallel for schedule(static) if (M * Ncols * rb > (1 << 22))
    for (idx j = 0; j < Ncols; ++j) {
        double* oj = out.data.data() + M * j;
        for (idx k = 0; k < rb; ++k) {
            const double w = g[k + rb * j];
            const double* ak = a.data.data() + M * k;
            for (idx r = 0; r < M; ++r) oj[r] += ak[r] * w;
        }
    }
    return out;
}

// tr_factors.hpp:111-119 subchain: cores n+1, ..., n-1 merged in cyclic order.
inline Tensor subchain(const TRFactors& f, idx mode) {
    const idx n_cores = f.order();
    if (mode < 0 || mode >= n_cores) throw std::out_of_range("subchain: mode out of range");
    require(n_cores >= 2, "subchain: needs at least two cores");
    Tensor cur = f.core((mode + 1) % n_cores);
    for (idx s = 2; s < n_cores; ++s) cur = chain_contract(cur, f.core((mode + s) % n_cores));
    return cur;
}

// tr_factors.hpp:123-137 Eq.(2): X_<n> = G_{n,(2)} (G_{!=n,<2>})^T, then fold_tr.
inline Tensor reconstruct_full(const TRFactors& f, idx mode = 0) {
    const idx n_cores = f.order();
    if (mode < 0 || mode >= n_cores) throw std::out_of_range("reconstruct_full: mode out of range");
    std::vector<idx> shape = f.dims();
    if (n_cores == 1) {
        Tensor out(shape);
        for (idx i = 0; i < shape[0]; ++i) {
            const Mat s = f.slice(0, i);
            double tr = 0.0;
            for (idx a = 0; a < std::min(s.r, s.c); ++a) tr += s(a, a);
            out[i] = tr;
        }
        return out;
    }
    const Mat core2 = unfold_classic(f.core(mode), 1);  // I_n x (R_n R_{n+1})
    const Mat sub2 = unfold_tr(subchain(f, mode), 1);   // prod I_k x (R_n R_{n+1})
    // xn = core2 * sub2^T
    const idx In = core2.r, P = sub2.r, RR = core2.c;
    Mat xn(In, P);
#pragma omp parallel for schedule(static) if (In * P * RR > (1 << 22))
    for (idx p = 0; p < P; ++p) {
        double* xp = xn.col(p);
        for (idx k = 0; k < RR; ++k) {
            const double w = sub2(p, k);
            const double* ck = core2.col(k);
            for (idx i = 0; i < In; ++i) xp[i] += ck[i] * w;
        }
    }
    return fold_tr(xn, mode, std::move(shape));
}

// tr_factors.hpp:140-159
inline idx num_params(const TRFactors& f) {
    idx t = 0;
    for (idx n = 0; n < f.order(); ++n) t += f.core(n).size();
    return t;
}

// ---------------------------------------------------------------- solvers
// solvers.hpp:24-38
struct SolverConfig {
    bool has_ranks = false;
    std::vector<idx> ranks;
    double tolerance = 0.0;
    idx max_sweeps = 50;
    std::uint64_t seed = 0;
};
struct SolveReport {
    TRFactors factors;
    std::vector<double> rse_history;
    idx sweeps_run = 0;
};

// solvers.hpp:47-54 rse = ||ref - approx|| / ||ref||
inline double rse(const Tensor& ref, const Tensor& approx) {
    require(ref.shape == approx.shape, "rse: shape mismatch");
    double num = 0.0, den = 0.0;
    for (idx i = 0; i < ref.size(); ++i) {
        const double d = ref[i] - approx[i];
        num += d * d;
        den += ref[i] * ref[i];
    }
    require(den > 0.0, "rse: reference tensor has zero norm");
    return std::sqrt(num) / std::sqrt(den);
}

// solvers.hpp:60-69
inline std::vector<idx> solver_ranks(const Tensor& x, const SolverConfig& cfg, const char* who) {
    require(cfg.has_ranks, std::string(who) + ": rank vector required");
    require(static_cast<idx>(cfg.ranks.size()) == x.order(),
            std::string(who) + ": rank vector length must equal tensor order");
    for (idx r : cfg.ranks) require(r >= 1, std::string(who) + ": ranks must be positive");
    require(cfg.max_sweeps >= 1, std::string(who) + ": max_sweeps must be positive");
    return cfg.ranks;
}

// solvers.hpp:71-78
inline TRFactors zero_factors(const std::vector<idx>& dims, const std::vector<idx>& ranks) {
    const idx N = static_cast<idx>(dims.size());
    std::vector<Tensor> cores;
    for (idx n = 0; n < N; ++n)
        cores.emplace_back(std::vector<idx>{ranks[static_cast<size_t>(n)], dims[static_cast<size_t>(n)],
                                            ranks[static_cast<size_t>((n + 1) % N)]});
    return TRFactors(std::move(cores));
}

// solvers.hpp:80-95 init_factors: N(0,1) * (xnorm / prod R)^(1/N), one stream, flat order.
inline TRFactors init_factors(const std::vector<idx>& dims, const std::vector<idx>& ranks, std::uint64_t seed,
                              double xnorm) {
    const idx N = static_cast<idx>(dims.size());
    double prod_ranks = 1.0;
    for (idx r : ranks) prod_ranks *= static_cast<double>(r);
    const double scale = xnorm > 0.0 ? std::pow(xnorm / prod_ranks, 1.0 / static_cast<double>(N)) : 0.0;
    GaussianSampler gauss(seed);
    std::vector<Tensor> cores;
    for (idx n = 0; n < N; ++n) {
        Tensor core({ranks[static_cast<size_t>(n)], dims[static_cast<size_t>(n)], ranks[static_cast<size_t>((n + 1) % N)]});
        for (idx i = 0; i < core.size(); ++i) core[i] = scale * gauss.next();
        cores.push_back(std::move(core));
    }
    return TRFactors(std::move(cores));
}

// solvers.hpp:102-129 subchain_gram via per-core transfer matrices.
inline Mat subchain_gram(const TRFactors& f, idx n) {
    const idx N = f.order();
    Mat omega;
    for (idx s = 1; s < N; ++s) {
        const idx k = (n + s) % N;
        const Tensor& g = f.core(k);
        const idx rk = g.dim(0), rk1 = g.dim(2);
        const Mat h = unfold_classic(g, 1);  // I_k x (R_k R_{k+1})
        const Mat gram = matmul_tn(h, h);
        Mat w(rk * rk, rk1 * rk1);
        for (idx s2 = 0; s2 < rk1; ++s2)
            for (idx s1 = 0; s1 < rk1; ++s1)
                for (idx r2 = 0; r2 < rk; ++r2)
                    for (idx r1 = 0; r1 < rk; ++r1) w(r1 + rk * r2, s1 + rk1 * s2) = gram(r1 + rk * s1, r2 + rk * s2);
        omega = (s == 1) ? std::move(w) : matmul(omega, w);
    }
    const idx rn = f.rank(n), rn1 = f.rank((n + 1) % N);
    Mat m(rn * rn1, rn * rn1);
    for (idx b2 = 0; b2 < rn1; ++b2)
        for (idx a2 = 0; a2 < rn; ++a2)
            for (idx b = 0; b < rn1; ++b)
                for (idx a = 0; a < rn; ++a) m(a + rn * b, a2 + rn * b2) = omega(b + rn1 * b2, a + rn * a2);
    return m;
}

// solvers.hpp:134-182 subchain_rhs: V = X_<n> S without materialising S.
inline Mat subchain_rhs(const Mat& xn_tr, const TRFactors& f, idx n) {
    const idx N = f.order();
    const idx dim_n = xn_tr.r;
    const Mat b = transpose(xn_tr);
    const idx k0 = (n + 1) % N;
    const Tensor& g0 = f.core(k0);
    const idx r0 = g0.dim(0), i0 = g0.dim(1), s0 = g0.dim(2);
    Mat ghat(r0 * s0, i0);
    for (idx i = 0; i < i0; ++i)
        for (idx s = 0; s < s0; ++s)
            for (idx r = 0; r < r0; ++r) ghat(r + r0 * s, i) = g0[r + r0 * (i + i0 * s)];
    const idx rest0 = static_cast<idx>(b.a.size()) / i0;
    Mat bm(i0, rest0);
    bm.a = b.a;
    Mat cur = matmul(ghat, bm);
    const idx front = r0;
    for (idx s = 2; s < N; ++s) {
        const idx k = (n + s) % N;
        const Tensor& g = f.core(k);
        const idx rk = g.dim(0), ik = g.dim(1), rk1 = g.dim(2);
        const idx mid = rk * ik;
        const idx tail = static_cast<idx>(cur.a.size()) / (front * mid);
        Mat next(front * rk1, tail);
        for (idx t = 0; t < tail; ++t) {
            const double* in = cur.a.data() + front * mid * t;
            double* out = next.a.data() + front * rk1 * t;
            for (idx c = 0; c < rk1; ++c)
                for (idx q = 0; q < mid; ++q) {
                    const double w = g[q + mid * c];
                    for (idx r = 0; r < front; ++r) out[r + front * c] += in[r + front * q] * w;
                }
        }
        cur = std::move(next);
    }
    const idx rn = f.rank(n), rn1 = front;
    Mat v(dim_n, rn * rn1);
    for (idx i = 0; i < dim_n; ++i)
        for (idx a = 0; a < rn; ++a)
            for (idx bb = 0; bb < rn1; ++bb) v(i, a + rn * bb) = cur.a[static_cast<size_t>(bb + rn1 * (a + rn * i))];
    return v;
}

// solvers.hpp:186-190
inline Mat ridge_solve(Mat gram, const Mat& rhs) {
    double tr = 0.0;
    for (idx i = 0; i < gram.r; ++i) tr += gram(i, i);
    const double lambda = 1e-12 * tr / static_cast<double>(gram.r);
    for (idx i = 0; i < gram.r; ++i) gram(i, i) += lambda;
    return ldlt_solve(std::move(gram), rhs);
}

// solvers.hpp:195-205
inline Mat ls_solve_qr(const Mat& a, const Mat& b) {
    if (a.r >= a.c) {
        HouseholderQR qr(a);
        double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
        for (idx i = 0; i < a.c; ++i) {
            dmax = std::max(dmax, std::abs(qr.qr(i, i)));
            dmin = std::min(dmin, std::abs(qr.qr(i, i)));
        }
        const double cutoff =
            dmax * static_cast<double>(std::max(a.r, a.c)) * std::numeric_limits<double>::epsilon() * 16.0;
        if (dmax > 0.0 && dmin > cutoff) return qr.solve(b);
    }
    return ridge_solve(matmul_tn(a, a), matmul_tn(a, b));
}

// solvers.hpp:209-219
inline Mat ls_solve_gram(const Mat& gram, const Mat& rhs) {
    Mat L;
    if (cholesky(gram, L)) {
        double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
        for (idx i = 0; i < L.r; ++i) {
            dmax = std::max(dmax, std::abs(L(i, i)));
            dmin = std::min(dmin, std::abs(L(i, i)));
        }
        const double cutoff = dmax * static_cast<double>(gram.r) * std::numeric_limits<double>::epsilon() * 16.0;
        if (dmax > 0.0 && dmin > cutoff) return cholesky_solve(L, rhs);
    }
    return ridge_solve(gram, rhs);
}

// solvers.hpp:223-230
inline void store_core(Tensor& core, const Mat& z) {
    const idx rn = core.dim(0), in = core.dim(1), rn1 = core.dim(2);
    for (idx s = 0; s < rn1; ++s)
        for (idx i = 0; i < in; ++i)
            for (idx r = 0; r < rn; ++r) core[r + rn * (i + in * s)] = z(r + rn * s, i);
}

constexpr idx kDirectLsMaxRows = 4096;  // solvers.hpp:234

// solvers.hpp:238-251
inline void als_update_mode(const Mat& xn_tr, TRFactors& f, idx n) {
    const idx n_cols = xn_tr.c;
    const idx m = f.rank(n) * f.rank((n + 1) % f.order());
    Mat z;
    if (n_cols <= kDirectLsMaxRows && n_cols >= m) {
        const Mat a = unfold_tr(subchain(f, n), 1);
        z = ls_solve_qr(a, transpose(xn_tr));
    } else {
        const Mat gram = subchain_gram(f, n);
        const Mat v = subchain_rhs(xn_tr, f, n);
        z = ls_solve_gram(gram, transpose(v));
    }
    store_core(f.core(n), z);
}

// solvers.hpp:268-279
inline SolveReport solve_order_one(const Tensor& x, const std::vector<idx>& ranks) {
    Tensor core({ranks[0], x.dim(0), ranks[0]});
    for (idx i = 0; i < x.dim(0); ++i) core[0 + ranks[0] * i] = x[i];
    SolveReport rep;
    rep.factors = TRFactors({std::move(core)});
    const double xnorm = frobenius_norm(x);
    rep.rse_history = {xnorm > 0.0 ? rse(x, reconstruct_full(rep.factors)) : 0.0};
    rep.sweeps_run = 1;
    return rep;
}

// solvers.hpp:281-290
inline SolveReport degenerate_zero_report(const Tensor& x, const std::vector<idx>& ranks) {
    SolveReport rep;
    rep.factors = zero_factors(x.shape, ranks);
    rep.rse_history = {0.0};
    rep.sweeps_run = 0;
    return rep;
}

// solvers.hpp:297-334 trals
inline SolveReport trals(const Tensor& x, const SolverConfig& cfg) {
    const auto ranks = solver_ranks(x, cfg, "trals");
    const double xnorm = frobenius_norm(x);
    if (xnorm == 0.0) return degenerate_zero_report(x, ranks);
    if (x.order() == 1) return solve_order_one(x, ranks);
    TRFactors f = init_factors(x.shape, ranks, cfg.seed, xnorm);
    std::vector<Mat> unf;
    for (idx n = 0; n < x.order(); ++n) unf.push_back(unfold_tr(x, n));
    SolveReport rep;
    for (idx sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
        for (idx n = 0; n < x.order(); ++n) als_update_mode(unf[static_cast<size_t>(n)], f, n);
        rep.rse_history.push_back(rse(x, reconstruct_full(f)));
        rep.sweeps_run = sweep;
        const size_t k = rep.rse_history.size();
        if (k >= 2 && std::abs(rep.rse_history[k - 1] - rep.rse_history[k - 2]) < cfg.tolerance * rep.rse_history[k - 2])
            break;
    }
    rep.factors = std::move(f);
    return rep;
}

// solvers.hpp:347-358
inline idx truncation_rank(const std::vector<double>& sv, double budget_sq, double* discarded_sq) {
    idx r = static_cast<idx>(sv.size());
    double tail = 0.0;
    while (r > 1) {
        const double t = tail + sv[static_cast<size_t>(r - 1)] * sv[static_cast<size_t>(r - 1)];
        if (t > budget_sq) break;
        tail = t;
        --r;
    }
    if (discarded_sq) *discarded_sq += tail;
    return r;
}

// solvers.hpp:361-371
inline std::pair<idx, idx> balanced_divisor_split(idx r) {
    idx target = static_cast<idx>(std::sqrt(static_cast<double>(r)));
    while ((target + 1) * (target + 1) <= r) ++target;
    while (target > 1 && target * target > r) --target;
    idx best = 1;
    for (idx d = 1; d <= r; ++d) {
        if (r % d != 0) continue;
        if (std::abs(d - target) < std::abs(best - target)) best = d;
    }
    return {best, r / best};
}

// solvers.hpp:382-459 trsvd
inline SolveReport trsvd(const Tensor& x, const SolverConfig& cfg, double* discarded_out = nullptr) {
    require(cfg.tolerance >= 0.0, "trsvd: tolerance must be nonnegative");
    const idx order = x.order();
    const double xnorm = frobenius_norm(x);
    if (order == 1) return solve_order_one(x, {1});
    if (xnorm == 0.0) return degenerate_zero_report(x, std::vector<idx>(static_cast<size_t>(order), 1));
    const double budget = cfg.tolerance * xnorm / std::sqrt(static_cast<double>(order));
    const double budget_sq = budget * budget;
    double discarded_sq = 0.0;

    const idx dim0 = x.dim(0);
    Mat m0(dim0, x.size() / dim0);
    m0.a = x.data;
    const SVD svd0 = jacobi_svd(m0);
    const idx r01 = truncation_rank(svd0.s, budget_sq, &discarded_sq);
    const auto [ra, rb] = balanced_divisor_split(r01);

    std::vector<Tensor> cores(static_cast<size_t>(order));
    {
        Tensor g0({ra, dim0, rb});
        for (idx q = 0; q < rb; ++q)
            for (idx i = 0; i < dim0; ++i)
                for (idx p = 0; p < ra; ++p) g0[p + ra * (i + dim0 * q)] = svd0.U(i, p + ra * q);
        cores[0] = std::move(g0);
    }
    const idx rest = x.size() / dim0;
    // W = S V^T (r01 x rest), reorganised so the R_1 index trails
    std::vector<double> cur(static_cast<size_t>(r01 * rest));
    for (idx p = 0; p < ra; ++p)
        for (idx c = 0; c < rest; ++c)
            for (idx q = 0; q < rb; ++q) {
                const idx row = p + ra * q;
                cur[static_cast<size_t>(q + rb * c + rb * rest * p)] =
                    svd0.s[static_cast<size_t>(row)] * svd0.V(c, row);
            }
    idx lead = rb;
    for (idx k = 1; k + 1 < order; ++k) {
        const idx dim_k = x.dim(k);
        const idx rows = lead * dim_k;
        const idx cols = static_cast<idx>(cur.size()) / rows;
        Mat mk(rows, cols);
        mk.a = cur;
        const SVD svd = jacobi_svd(mk);
        const idx r = truncation_rank(svd.s, budget_sq, &discarded_sq);
        Tensor gk({lead, dim_k, r});
        for (idx j = 0; j < r; ++j)
            for (idx i = 0; i < rows; ++i) gk[i + rows * j] = svd.U(i, j);
        cores[static_cast<size_t>(k)] = std::move(gk);
        std::vector<double> next(static_cast<size_t>(r * cols));
        for (idx c = 0; c < cols; ++c)
            for (idx j = 0; j < r; ++j)
                next[static_cast<size_t>(j + r * c)] = svd.s[static_cast<size_t>(j)] * svd.V(c, j);
        cur = std::move(next);
        lead = r;
    }
    {
        const idx dim_last = x.dim(order - 1);
        cores[static_cast<size_t>(order - 1)] = Tensor({lead, dim_last, ra}, std::move(cur));
    }
    SolveReport rep;
    rep.factors = TRFactors(std::move(cores));
    rep.rse_history = {rse(x, reconstruct_full(rep.factors))};
    rep.sweeps_run = 1;
    if (discarded_out) *discarded_out = discarded_sq;
    return rep;
}

// ---------------------------------------------------------------- sketch
// sketch.hpp:18-28
struct ProjectionSpec {
    std::vector<idx> sketch_dims;
    std::uint64_t seed = 0;
};
struct SketchResult {
    Tensor projected;
    std::vector<Mat> bases;
    std::vector<Mat> sketches;  // Y_n per mode (empty for skipped modes); oracle-only extra for parity
};

// sketch.hpp:32-38 gaussian_matrix: column-major fill from the sampler.
inline Mat gaussian_matrix(idx rows, idx cols, GaussianSampler& gauss) {
    require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be positive");
    Mat m(rows, cols);
    for (idx i = 0; i < rows * cols; ++i) m.a[static_cast<size_t>(i)] = gauss.next();
    return m;
}

// sketch.hpp:45-53 economy_q: Householder thin Q, columns flipped where R_jj < 0.
inline Mat economy_q(const Mat& y) {
    const idx k = std::min(y.r, y.c);
    HouseholderQR qr(y);
    Mat q = qr.thin_q();
    for (idx j = 0; j < k; ++j)
        if (qr.qr(j, j) < 0.0)
            for (idx i = 0; i < q.r; ++i) q(i, j) = -q(i, j);
    return q;
}

// Y = X_(n) * Omega computed straight from the (left, dim, right) view
// (unfold_classic column c = l + left*r, tensor.hpp:133-142), i.e. the
// product at sketch.hpp:80-83 without the materialised unfolding copy.
inline Mat sketch_product(const Tensor& t, idx mode, const Mat& omega) {
    const auto s = mode_split(t.shape, mode);
    const idx K = omega.c;
    Mat y(s.dim, K);
#pragma omp parallel for schedule(static) if (t.size() * K > (1 << 22))
    for (idx k = 0; k < K; ++k) {
        double* yk = y.col(k);
        const double* om = omega.col(k);
        for (idx r = 0; r < s.right; ++r)
            for (idx d = 0; d < s.dim; ++d) {
                const double* row = t.data.data() + s.left * (d + s.dim * r);
                const double* w = om + s.left * r;
                double acc = 0.0;
                for (idx l = 0; l < s.left; ++l) acc += row[l] * w[l];
                yk[d] += acc;
            }
    }
    return y;
}

// sketch.hpp:62-89 sketch: sequential shrinking, one Gaussian stream for all
// modes, K_n == I_n skips the mode without consuming draws.
inline SketchResult sketch(const Tensor& x, const ProjectionSpec& spec) {
    require(static_cast<idx>(spec.sketch_dims.size()) == x.order(),
            "sketch: projection size list must match tensor order");
    for (idx n = 0; n < x.order(); ++n)
        require(spec.sketch_dims[static_cast<size_t>(n)] >= 1 && spec.sketch_dims[static_cast<size_t>(n)] <= x.dim(n),
                "sketch: need 1 <= K_n <= I_n in mode " + std::to_string(n));
    GaussianSampler gauss(spec.seed);
    SketchResult out;
    out.projected = x;
    for (idx n = 0; n < x.order(); ++n) {
        const idx k = spec.sketch_dims[static_cast<size_t>(n)];
        const idx dim = x.dim(n);
        if (k == dim) {
            out.bases.push_back(Mat::identity(dim, dim));
            out.sketches.emplace_back();
            continue;
        }
        const idx cols = out.projected.size() / dim;
        const Mat test = gaussian_matrix(cols, k, gauss);
        Mat y = sketch_product(out.projected, n, test);
        Mat q = economy_q(y);
        out.projected = mode_n_product(out.projected, n, transpose(q));
        out.bases.push_back(std::move(q));
        out.sketches.push_back(std::move(y));
    }
    return out;
}

// SPEC.md:319 alternative ("project each mode from the original x"): every
// Y_n = X_(n) Omega_n from the ORIGINAL x, Omega_n sized prod_{k!=n} I_k x K_n,
// drawn from the same single stream in mode order with the same column-major
// fill and skip rule; then P = x x_0 Q_0^T ... x_{N-1} Q_{N-1}^T. No reference
// code exists for it; this is the oracle of the fused single-pass variant.
inline SketchResult sketch_fused(const Tensor& x, const ProjectionSpec& spec) {
    require(static_cast<idx>(spec.sketch_dims.size()) == x.order(),
            "sketch: projection size list must match tensor order");
    for (idx n = 0; n < x.order(); ++n)
        require(spec.sketch_dims[static_cast<size_t>(n)] >= 1 && spec.sketch_dims[static_cast<size_t>(n)] <= x.dim(n),
                "sketch: need 1 <= K_n <= I_n in mode " + std::to_string(n));
    GaussianSampler gauss(spec.seed);
    SketchResult out;
    for (idx n = 0; n < x.order(); ++n) {
        const idx k = spec.sketch_dims[static_cast<size_t>(n)];
        const idx dim = x.dim(n);
        if (k == dim) {
            out.bases.push_back(Mat::identity(dim, dim));
            out.sketches.emplace_back();
            continue;
        }
        const Mat test = gaussian_matrix(x.size() / dim, k, gauss);
        Mat y = sketch_product(x, n, test);
        out.bases.push_back(economy_q(y));
        out.sketches.push_back(std::move(y));
    }
    out.projected = x;
    for (idx n = 0; n < x.order(); ++n) {
        const Mat& q = out.bases[static_cast<size_t>(n)];
        if (q.r == q.c && q.is_identity()) continue;
        out.projected = mode_n_product(out.projected, n, transpose(q));
    }
    return out;
}

// sketch.hpp:93-101 lift_back
inline Tensor lift_back(const SketchResult& sk) {
    Tensor t = sk.projected;
    for (idx n = 0; n < t.order(); ++n) {
        const Mat& q = sk.bases[static_cast<size_t>(n)];
        if (q.r == q.c && q.is_identity()) continue;
        t = mode_n_product(t, n, q);
    }
    return t;
}

// sketch.hpp:106-122 back_project: G_n = Z_n x_2 Q_n; identity bases copy bit-exactly.
inline TRFactors back_project(const TRFactors& z, const std::vector<Mat>& bases) {
    require(static_cast<idx>(bases.size()) == z.order(), "back_project: need one basis per core");
    std::vector<Tensor> cores;
    for (idx n = 0; n < z.order(); ++n) {
        const Mat& q = bases[static_cast<size_t>(n)];
        require(q.c == z.dim(n), "back_project: basis/core dimension mismatch in mode " + std::to_string(n));
        if (q.r == q.c && q.is_identity()) {
            cores.push_back(z.core(n));
            continue;
        }
        cores.push_back(mode_n_product(z.core(n), 1, q));
    }
    return TRFactors(std::move(cores));
}

// sketch.hpp:126-147 randomized_decompose. The reference prints its rank > K_n
// warning before sketch() validates the list length (sketch.hpp:131-138); the
// restatement validates first (same observable result for valid input).
template <typename Solver>
SolveReport randomized_decompose(const Tensor& x, const SolverConfig& cfg, const ProjectionSpec& spec,
                                 Solver&& solve_small, bool fused = false) {
    SketchResult sk = fused ? sketch_fused(x, spec) : sketch(x, spec);
    SolveReport inner = solve_small(sk.projected, cfg);
    SolveReport rep;
    rep.factors = back_project(inner.factors, sk.bases);
    rep.rse_history = std::move(inner.rse_history);
    rep.rse_history.push_back(rse(x, reconstruct_full(rep.factors)));
    rep.sweeps_run = inner.sweeps_run;
    return rep;
}

// sketch.hpp:154-165
inline SolveReport rtrals(const Tensor& x, const SolverConfig& cfg, const ProjectionSpec& spec, bool fused = false) {
    return randomized_decompose(x, cfg, spec, [](const Tensor& p, const SolverConfig& c) { return trals(p, c); },
                                fused);
}
inline SolveReport rtrsvd(const Tensor& x, const SolverConfig& cfg, const ProjectionSpec& spec, bool fused = false) {
    return randomized_decompose(x, cfg, spec, [](const Tensor& p, const SolverConfig& c) { return trsvd(p, c); },
                                fused);
}

// ---------------------------------------------------------------- synthetic
// synthetic.hpp:16-29 random_factors: one stream, cores in order, flat (r,i,s).
inline TRFactors random_factors(const std::vector<idx>& dims, const std::vector<idx>& ranks, std::uint64_t seed,
                                double scale = 1.0) {
    require(dims.size() == ranks.size(), "random_factors: dims/ranks length mismatch");
    const idx N = static_cast<idx>(dims.size());
    GaussianSampler gauss(seed);
    std::vector<Tensor> cores;
    for (idx n = 0; n < N; ++n) {
        Tensor core({ranks[static_cast<size_t>(n)], dims[static_cast<size_t>(n)], ranks[static_cast<size_t>((n + 1) % N)]});
        for (idx i = 0; i < core.size(); ++i) core[i] = scale * gauss.next();
        cores.push_back(std::move(core));
    }
    return TRFactors(std::move(cores));
}

// SPEC.md:338-346 add_noise (specified, not implemented in the headers):
// E_i = GaussianSampler(seed) draws in flat order, rescaled so that
// ||E|| / ||x|| = 10^(-snr_db/20) exactly.
inline Tensor add_noise(const Tensor& x, double snr_db, std::uint64_t seed) {
    const double xn = frobenius_norm(x);
    require(xn > 0.0, "add_noise: zero-norm input");
    GaussianSampler gauss(seed);
    std::vector<double> e(static_cast<size_t>(x.size()));
    for (auto& v : e) v = gauss.next();
    const double en = std::sqrt(sq_norm(e.data(), x.size()));
    const double alpha = xn * std::pow(10.0, -snr_db / 20.0) / en;
    Tensor out = x;
    for (idx i = 0; i < x.size(); ++i) out[i] += alpha * e[static_cast<size_t>(i)];
    return out;
}

}  // namespace oracle
