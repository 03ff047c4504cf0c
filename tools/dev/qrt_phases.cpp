#include <chrono>
#include <cstdio>
#include <random>
#include "host_solve.hpp"
#include "hs_phases_ls.cpp"
int main(int argc, char** argv) {
    using namespace trg::host;
    const idx m = argc > 1 ? atoll(argv[1]) : 4096, n = argc > 2 ? atoll(argv[2]) : 400, nr = argc > 3 ? atoll(argv[3]) : 64;
    Mat a(m, n), b(m, nr);
    std::mt19937_64 g(1); std::normal_distribution<double> nd;
    for (auto& v : a.a) v = nd(g);
    for (auto& v : b.a) v = nd(g);
    extern double g_t[6];
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        Mat x = ls_solve_qr(a, b);
        auto t1 = std::chrono::steady_clock::now();
        printf("panel %.1f T %.1f upd %.1f hqr %.1f solve %.1f ms\n", g_t[0], g_t[1], g_t[2], g_t[3], g_t[4]); for(int z=0;z<6;++z) g_t[z]=0;
        printf("ls_solve_qr %lldx%lld rhs %lld: %.1f ms (x00 %.6f)\n", (long long)m, (long long)n, (long long)nr,
               std::chrono::duration<double, std::milli>(t1 - t0).count(), x(0, 0));
    }
}
