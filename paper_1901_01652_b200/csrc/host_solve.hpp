// SPDX-License-Identifier: Apache-2.0
//
// Host-side small TR solve on the projected tensor P (Alg. 1 line 9).
//
// P is tiny (prod K_n <= ~10^6 entries), so trals / trsvd run on the host in
// fp64 exactly as the reference specifies them; only the streaming passes
// over X are device work. This is product code: it is
// the drop-in for solvers.hpp:297-459 with the same results up to rounding:
//   trals  solvers.hpp:297-334 (init_factors :80-95, als_update_mode :238-251,
//          direct QR route :195-205 / Gram route :102-219, kDirectLsMaxRows 4096)
//   trsvd  solvers.hpp:382-459 (truncation_rank :347-358,
//          balanced_divisor_split :361-371)
// Eigen's BDCSVD is replaced by one-sided Jacobi (singular vectors equal up to
// sign). Loops that write disjoint outputs are OpenMP-parallel, which keeps
// results bit-identical for any thread count.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace trg {
namespace host {

using idx = std::int64_t;

struct Mat {
    idx r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(idx rows, idx cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
    double& operator()(idx i, idx j) { return a[static_cast<size_t>(i + r * j)]; }
    double operator()(idx i, idx j) const { return a[static_cast<size_t>(i + r * j)]; }
    double* col(idx j) { return a.data() + r * j; }
    const double* col(idx j) const { return a.data() + r * j; }
};

// Dense tensor, first-index-fastest (tensor.hpp:33-38).
struct Tensor {
    std::vector<idx> shape;
    std::vector<double> data;
    idx size() const { return static_cast<idx>(data.size()); }
    idx order() const { return static_cast<idx>(shape.size()); }
};

struct Cores {
    std::vector<Tensor> g;  // core n: (R_n, I_n, R_{n+1})
    idx order() const { return static_cast<idx>(g.size()); }
    idx rank(idx n) const { return g[static_cast<size_t>(n)].shape[0]; }
    idx dim(idx n) const { return g[static_cast<size_t>(n)].shape[1]; }
};

struct SolveOut {
    Cores cores;
    std::vector<double> rse_history;
    idx sweeps_run = 0;
    double discarded_sq = 0.0;
};

// Device least squares min ||A x - b|| (A m x n column-major, m >= n; b m x nrhs): 0 solved into x
// (n x nrhs), 1 rank-deficient by the direct route's cutoff, -1 no device route (device_ls.cu)
int device_ls_qr(const double* a, idx m, idx n, const double* b, idx nrhs, double* x);

// The direct-route ALS update with the system built on the device (device_ls.cu): subchain of
// cores n+1..n+N-1, its mode-1 TR unfolding and B = X_<n>^T, then the device_ls_qr solve.
// 0: z = (R_n R_{n+1}) x I_n solution; 1 rank-deficient; -1 no device route.
int device_als_direct(const Cores& f, idx n, const Mat& xn_tr, Mat& z);

// rse(x, reconstruct_full(f)) on the device (device_ls.cu). 0: *out set; -1: no device route.
int device_tr_rse(const Cores& f, const Tensor& x, double* out);

// Thin SVD on the device (cuSOLVER gesvdj) with the host svd()'s conventions (device_ls.cu).
// 0: U (m x k), s (k, descending), V (n x k); -1: no device route.
int device_svd(const Mat& a, Mat& U, std::vector<double>& s, Mat& V);

// Phase timers of the small solve, on only with TRG_SOLVE_PROF=1 (printed to stderr after each
// trals call; the device phases then synchronise after each step so the split is attributable).
enum SolvePhase { kPhSubchain, kPhUnfold, kPhLsH2D, kPhLsFactor, kPhLsApply, kPhLsHost, kPhStore, kPhRse, kPhCount };
bool solve_prof_on();
void solve_prof_add(int phase, double ms);

SolveOut trals(const Tensor& x, const std::vector<idx>& ranks, double tolerance, idx max_sweeps, std::uint64_t seed);
SolveOut trsvd(const Tensor& x, double tolerance);
Tensor reconstruct_full(const Cores& f);
double rse(const Tensor& ref, const Tensor& approx);

}  // namespace host
}  // namespace trg
