// SPDX-License-Identifier: Apache-2.0
// Drives the C++ facade (include/tenring_b200.hpp) the way a reference caller
// would drive tenring::sketch / rtrals / rtrsvd. Used by tests/test_facade.py:
//   facade_main IN OUT   IN  = int64 N, int64 dims[N], int64 K[N], int64 ranks[N], f64 x[prod dims]
//                        OUT = f64 P[prod K], f64 Q_n (col-major, n = 0..N-1),
//                              f64 rse_als, f64 rse_svd, int64 svd ranks[N], f64 sketch-identity flag
#include <cstdio>
#include <fstream>
#include <iostream>
#include <stdexcept>

#include "tenring_b200.hpp"

namespace tb = tenring::b200;

template <typename T>
static void rd(std::ifstream& f, T* p, std::size_t n) {
    f.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
    if (!f) throw std::runtime_error("short read");
}
template <typename T>
static void wr(std::ofstream& f, const T* p, std::size_t n) {
    f.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
}

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: facade_main IN OUT\n");
        return 2;
    }
    try {
        std::ifstream in(argv[1], std::ios::binary);
        int64_t N = 0;
        rd(in, &N, 1);
        std::vector<tb::index_t> dims(N), K(N), ranks(N);
        rd(in, dims.data(), N);
        rd(in, K.data(), N);
        rd(in, ranks.data(), N);
        tb::DenseTensor x(dims);
        rd(in, x.data(), static_cast<std::size_t>(x.size()));

        tb::ProjectionSpec spec{K, 0};
        tb::SketchResult sk = tb::sketch(x, spec);
        std::ofstream out(argv[2], std::ios::binary);
        wr(out, sk.projected.data(), static_cast<std::size_t>(sk.projected.size()));
        for (const auto& q : sk.bases) wr(out, q.data(), q.values.size());

        tb::SolverConfig cfg;
        cfg.ranks = ranks;
        cfg.max_sweeps = 5;
        tb::SolveReport als = tb::rtrals(x, cfg, spec);
        tb::SolverConfig scfg;
        scfg.tolerance = 1e-3;
        tb::SolveReport svd = tb::rtrsvd(x, scfg, spec);
        const double ra = als.rse_history.back(), rs = svd.rse_history.back();
        wr(out, &ra, 1);
        wr(out, &rs, 1);
        const std::vector<tb::index_t> sr = svd.factors.ranks();
        wr(out, sr.data(), sr.size());
        // the RSE the facade reports must equal rse(x, factors) recomputed through the facade
        const double again = tb::rse(x, als.factors);
        const double same = (again == ra) ? 1.0 : 0.0;
        wr(out, &same, 1);

        // error mapping: K_n > I_n is std::invalid_argument (sketch.hpp:66-67)
        bool threw = false;
        try {
            std::vector<tb::index_t> bad = K;
            bad[0] = dims[0] + 1;
            tb::sketch(x, tb::ProjectionSpec{bad, 0});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        if (!threw) throw std::runtime_error("expected std::invalid_argument");
        std::printf("facade ok: rse_als %.6f rse_svd %.6f\n", ra, rs);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "facade_main: %s\n", e.what());
        return 1;
    }
}
