// SPDX-License-Identifier: Apache-2.0
//
// ORACLE — TEST INFRASTRUCTURE ONLY. extern "C" shims over tenring_oracle.hpp
// so that tests/ (ctypes), smoke() and bench.py's CPU baseline can drive the
// restatement on the same inputs as the product. Never linked by the product.
//
// Conventions: every entry returns 0 on success, 1 for std::invalid_argument,
// 2 for std::out_of_range, 9 for anything else; oracle_last_error() holds the
// message. Cores are passed flat and concatenated in mode order; core n has
// shape (R_n, I_n, R_{n+1 mod N}). Matrices are column-major.
#include <cstring>
#include <exception>
#include <string>

#include "tenring_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

std::vector<idx> vec(const std::int64_t* p, int n) { return std::vector<idx>(p, p + n); }

Tensor make_tensor(int order, const std::int64_t* dims, const double* data) {
    std::vector<idx> shape = vec(dims, order);
    const idx n = product(shape);
    return Tensor(shape, std::vector<double>(data, data + n));
}

TRFactors make_factors(int order, const std::int64_t* dims, const std::int64_t* ranks, const double* cores) {
    std::vector<Tensor> cs;
    const double* p = cores;
    for (int n = 0; n < order; ++n) {
        std::vector<idx> s{ranks[n], dims[n], ranks[(n + 1) % order]};
        const idx sz = product(s);
        cs.emplace_back(s, std::vector<double>(p, p + sz));
        p += sz;
    }
    return TRFactors(std::move(cs));
}

std::int64_t write_factors(const TRFactors& f, std::int64_t* ranks_out, double* cores_out, std::int64_t cap) {
    std::int64_t need = 0;
    for (idx n = 0; n < f.order(); ++n) {
        if (ranks_out) ranks_out[n] = f.rank(n);
        need += f.core(n).size();
    }
    if (cores_out && cap >= need) {
        double* p = cores_out;
        for (idx n = 0; n < f.order(); ++n) {
            std::memcpy(p, f.core(n).data.data(), sizeof(double) * static_cast<size_t>(f.core(n).size()));
            p += f.core(n).size();
        }
    }
    return need;
}

void write_report(const SolveReport& rep, std::int64_t* ranks_out, double* cores_out, std::int64_t cap,
                  std::int64_t* cores_len, double* rse_out, std::int64_t rse_cap, std::int64_t* n_rse,
                  std::int64_t* sweeps) {
    const std::int64_t need = write_factors(rep.factors, ranks_out, cores_out, cap);
    if (cores_len) *cores_len = need;
    if (n_rse) *n_rse = static_cast<std::int64_t>(rep.rse_history.size());
    if (rse_out)
        for (size_t i = 0; i < rep.rse_history.size() && static_cast<std::int64_t>(i) < rse_cap; ++i)
            rse_out[i] = rep.rse_history[i];
    if (sweeps) *sweeps = rep.sweeps_run;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

void oracle_set_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

int oracle_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// Raw SplitMix64 outputs 0..n-1 (random.hpp:18-23).
int oracle_splitmix_u64(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
    return guard([&] {
        SplitMix64 r(seed);
        for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
    });
}

// Gaussian draws skip .. skip+n-1 of GaussianSampler(seed) (random.hpp:50-62).
int oracle_gaussian(std::uint64_t seed, std::int64_t skip, std::int64_t n, double* out) {
    return guard([&] {
        GaussianSampler g(seed);
        g.seek(seed, (std::uint64_t)skip);
        for (std::int64_t i = 0; i < n; ++i) out[i] = g.next();
    });
}

int oracle_unfold(int order, const std::int64_t* dims, const double* x, int mode, int tr, double* out) {
    return guard([&] {
        const Tensor t = make_tensor(order, dims, x);
        const Mat m = tr ? unfold_tr(t, mode) : unfold_classic(t, mode);
        std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
    });
}

int oracle_fold(int order, const std::int64_t* dims, const double* m, int mode, int tr, double* out) {
    return guard([&] {
        std::vector<idx> shape = vec(dims, order);
        require(mode >= 0 && mode < order, "fold: mode out of range for shape");
        Mat mm(shape[static_cast<size_t>(mode)], product(shape) / shape[static_cast<size_t>(mode)]);
        std::memcpy(mm.a.data(), m, sizeof(double) * mm.a.size());
        const Tensor t = tr ? fold_tr(mm, mode, shape) : fold_classic(mm, mode, shape);
        std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
    });
}

// out = x x_mode M, M is m_rows x m_cols column-major.
int oracle_mode_n_product(int order, const std::int64_t* dims, const double* x, int mode, std::int64_t m_rows,
                          std::int64_t m_cols, const double* m, double* out) {
    return guard([&] {
        const Tensor t = make_tensor(order, dims, x);
        Mat mm(m_rows, m_cols);
        std::memcpy(mm.a.data(), m, sizeof(double) * mm.a.size());
        const Tensor o = mode_n_product(t, mode, mm);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}

int oracle_economy_q(std::int64_t rows, std::int64_t cols, const double* y, double* q_out) {
    return guard([&] {
        Mat m(rows, cols);
        std::memcpy(m.a.data(), y, sizeof(double) * m.a.size());
        const Mat q = economy_q(m);
        std::memcpy(q_out, q.a.data(), sizeof(double) * q.a.size());
    });
}

// Thin SVD stand-in for BDCSVD (solvers.hpp:398,431): singular values (min(rows, cols),
// descending), U (rows x min) and V (cols x min), column-major. For the LAPACK cross-check.
int oracle_svd(std::int64_t rows, std::int64_t cols, const double* a, double* s_out, double* u_out, double* v_out) {
    return guard([&] {
        Mat m(rows, cols);
        std::memcpy(m.a.data(), a, sizeof(double) * m.a.size());
        const SVD d = jacobi_svd(m);
        std::memcpy(s_out, d.s.data(), sizeof(double) * d.s.size());
        if (u_out) std::memcpy(u_out, d.U.a.data(), sizeof(double) * d.U.a.size());
        if (v_out) std::memcpy(v_out, d.V.a.data(), sizeof(double) * d.V.a.size());
    });
}

// Sequential (variant 0, sketch.hpp:62-89) or fused (variant 1)
// projection. bases_out: concatenated I_n x K_n column-major (identity for
// skipped modes); ys_out (optional): concatenated I_n x K_n sketches (zeros
// for skipped modes).
int oracle_sketch(int order, const std::int64_t* dims, const double* x, const std::int64_t* K, std::uint64_t seed,
                  int variant, double* projected_out, double* bases_out, double* ys_out) {
    return guard([&] {
        const Tensor t = make_tensor(order, dims, x);
        ProjectionSpec spec{vec(K, order), seed};
        const SketchResult sk = variant ? sketch_fused(t, spec) : sketch(t, spec);
        if (projected_out) std::memcpy(projected_out, sk.projected.data.data(), sizeof(double) * sk.projected.data.size());
        double* b = bases_out;
        double* y = ys_out;
        for (int n = 0; n < order; ++n) {
            const Mat& q = sk.bases[static_cast<size_t>(n)];
            const idx sz = dims[n] * K[n];
            if (b) {
                std::memcpy(b, q.a.data(), sizeof(double) * static_cast<size_t>(sz));
                b += sz;
            }
            if (y) {
                const Mat& ym = sk.sketches[static_cast<size_t>(n)];
                if (ym.a.empty())
                    std::memset(y, 0, sizeof(double) * static_cast<size_t>(sz));
                else
                    std::memcpy(y, ym.a.data(), sizeof(double) * static_cast<size_t>(sz));
                y += sz;
            }
        }
    });
}

int oracle_lift_back(int order, const std::int64_t* K, const double* projected, const std::int64_t* dims,
                     const double* bases, double* out) {
    return guard([&] {
        SketchResult sk;
        sk.projected = make_tensor(order, K, projected);
        const double* b = bases;
        for (int n = 0; n < order; ++n) {
            Mat q(dims[n], K[n]);
            std::memcpy(q.a.data(), b, sizeof(double) * q.a.size());
            b += q.a.size();
            sk.bases.push_back(std::move(q));
        }
        const Tensor t = lift_back(sk);
        std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
    });
}

int oracle_reconstruct_full(int order, const std::int64_t* dims, const std::int64_t* ranks, const double* cores,
                            int mode, double* out) {
    return guard([&] {
        const TRFactors f = make_factors(order, dims, ranks, cores);
        const Tensor t = reconstruct_full(f, mode);
        std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
    });
}

int oracle_reconstruct_elementwise(int order, const std::int64_t* dims, const std::int64_t* ranks, const double* cores,
                                   const std::int64_t* index, double* out) {
    return guard([&] {
        const TRFactors f = make_factors(order, dims, ranks, cores);
        *out = reconstruct_elementwise(f, vec(index, order));
    });
}

int oracle_subchain(int order, const std::int64_t* dims, const std::int64_t* ranks, const double* cores, int mode,
                    double* out) {
    return guard([&] {
        const TRFactors f = make_factors(order, dims, ranks, cores);
        const Tensor t = subchain(f, mode);
        std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
    });
}

int oracle_rse(std::int64_t n, const double* ref, const double* approx, double* out) {
    return guard([&] {
        Tensor a({n}, std::vector<double>(ref, ref + n));
        Tensor b({n}, std::vector<double>(approx, approx + n));
        *out = rse(a, b);
    });
}

// small cores (R_n, K_n, R_{n+1}) + bases (I_n x K_n) -> cores (R_n, I_n, R_{n+1})
int oracle_back_project(int order, const std::int64_t* K, const std::int64_t* ranks, const double* small_cores,
                        const std::int64_t* dims, const double* bases, double* cores_out) {
    return guard([&] {
        const TRFactors z = make_factors(order, K, ranks, small_cores);
        std::vector<Mat> qs;
        const double* b = bases;
        for (int n = 0; n < order; ++n) {
            Mat q(dims[n], K[n]);
            std::memcpy(q.a.data(), b, sizeof(double) * q.a.size());
            b += q.a.size();
            qs.push_back(std::move(q));
        }
        const TRFactors g = back_project(z, qs);
        write_factors(g, nullptr, cores_out, 1LL << 62);
    });
}

// trals / trsvd (method 0 / 1) on x. Outputs as write_report.
int oracle_solve(int method, int order, const std::int64_t* dims, const double* x, const std::int64_t* ranks_in,
                 double tol, std::int64_t max_sweeps, std::uint64_t seed, std::int64_t* ranks_out, double* cores_out,
                 std::int64_t cores_cap, std::int64_t* cores_len, double* rse_out, std::int64_t rse_cap,
                 std::int64_t* n_rse, std::int64_t* sweeps, double* discarded_sq) {
    return guard([&] {
        const Tensor t = make_tensor(order, dims, x);
        SolverConfig cfg;
        if (ranks_in) {
            cfg.has_ranks = true;
            cfg.ranks = vec(ranks_in, order);
        }
        cfg.tolerance = tol;
        cfg.max_sweeps = max_sweeps;
        cfg.seed = seed;
        double disc = 0.0;
        const SolveReport rep = method == 0 ? trals(t, cfg) : trsvd(t, cfg, &disc);
        if (discarded_sq) *discarded_sq = disc;
        write_report(rep, ranks_out, cores_out, cores_cap, cores_len, rse_out, rse_cap, n_rse, sweeps);
    });
}

// rtrals / rtrsvd (method 0 / 1), sequential (variant 0) or fused (1) sketch.
int oracle_rtrd(int method, int variant, int order, const std::int64_t* dims, const double* x,
                const std::int64_t* ranks_in, double tol, std::int64_t max_sweeps, std::uint64_t cfg_seed,
                const std::int64_t* K, std::uint64_t spec_seed, std::int64_t* ranks_out, double* cores_out,
                std::int64_t cores_cap, std::int64_t* cores_len, double* rse_out, std::int64_t rse_cap,
                std::int64_t* n_rse, std::int64_t* sweeps) {
    return guard([&] {
        const Tensor t = make_tensor(order, dims, x);
        SolverConfig cfg;
        if (ranks_in) {
            cfg.has_ranks = true;
            cfg.ranks = vec(ranks_in, order);
        }
        cfg.tolerance = tol;
        cfg.max_sweeps = max_sweeps;
        cfg.seed = cfg_seed;
        ProjectionSpec spec{vec(K, order), spec_seed};
        const SolveReport rep = method == 0 ? rtrals(t, cfg, spec, variant != 0) : rtrsvd(t, cfg, spec, variant != 0);
        write_report(rep, ranks_out, cores_out, cores_cap, cores_len, rse_out, rse_cap, n_rse, sweeps);
    });
}

int oracle_random_factors(int order, const std::int64_t* dims, const std::int64_t* ranks, std::uint64_t seed,
                          double scale, double* cores_out) {
    return guard([&] {
        const TRFactors f = random_factors(vec(dims, order), vec(ranks, order), seed, scale);
        write_factors(f, nullptr, cores_out, 1LL << 62);
    });
}

int oracle_add_noise(std::int64_t n, const double* x, double snr_db, std::uint64_t seed, double* out) {
    return guard([&] {
        Tensor t({n}, std::vector<double>(x, x + n));
        const Tensor o = add_noise(t, snr_db, seed);
        std::memcpy(out, o.data.data(), sizeof(double) * static_cast<size_t>(n));
    });
}

}  // extern "C"
