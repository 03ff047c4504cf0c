// Development: time the host small solve (host_solve.cpp) on a C4-sized projected tensor.
//   g++ -O3 -march=native -fopenmp -std=c++17 -I paper_1901_01652_b200/csrc tools/hostsolve_bench.cpp \
//       paper_1901_01652_b200/csrc/host_solve.cpp -o /tmp/hsb && /tmp/hsb 64 64 32 20 15
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "host_solve.hpp"
extern double g_t[6];

int main(int argc, char** argv) {
    using namespace trg::host;
    const idx I0 = argc > 1 ? atoll(argv[1]) : 64, I1 = argc > 2 ? atoll(argv[2]) : 64, I2 = argc > 3 ? atoll(argv[3]) : 32;
    const idx R = argc > 4 ? atoll(argv[4]) : 20, sweeps = argc > 5 ? atoll(argv[5]) : 15;
    Tensor x;
    x.shape = {I0, I1, I2};
    x.data.resize((size_t)(I0 * I1 * I2));
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (auto& v : x.data) v = nd(g);
    auto t0 = std::chrono::steady_clock::now();
    SolveOut o = trals(x, {R, R, R}, 0.0, sweeps, 0);
    auto t1 = std::chrono::steady_clock::now();
    printf("trals %lldx%lldx%lld R=%lld sweeps=%lld: %.1f ms, rse %.6f\n", (long long)I0, (long long)I1, (long long)I2,
           (long long)R, (long long)o.sweeps_run, std::chrono::duration<double, std::milli>(t1 - t0).count(),
           o.rse_history.back());
    printf("subchain %.1f unfold %.1f ls %.1f rse %.1f\n", g_t[0], g_t[1], g_t[2], g_t[3]);
    return 0;
}
