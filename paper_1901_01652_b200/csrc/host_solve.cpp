// SPDX-License-Identifier: Apache-2.0
// Host small solve on P: trals / trsvd (see host_solve.hpp for the contract).
#include "host_solve.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <numeric>

#include <omp.h>

#include "random_host.hpp"

namespace trg {
namespace host {

namespace {
double g_phase_ms[kPhCount];
const char* const kPhaseName[kPhCount] = {"subchain", "unfold", "ls_h2d", "ls_factor", "ls_apply", "ls_host", "store", "rse"};
struct PhaseTimer {
    int ph;
    std::chrono::steady_clock::time_point t0;
    explicit PhaseTimer(int p) : ph(p), t0(std::chrono::steady_clock::now()) {}
    ~PhaseTimer() {
        if (solve_prof_on())
            solve_prof_add(ph, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};
}  // namespace

bool solve_prof_on() {
    static const bool on = getenv("TRG_SOLVE_PROF") != nullptr;
    return on;
}
void solve_prof_add(int phase, double ms) { g_phase_ms[phase] += ms; }

namespace {

void require(bool ok, const std::string& msg) {
    if (!ok) throw std::invalid_argument(msg);
}

idx prod(const std::vector<idx>& v) {
    idx p = 1;
    for (idx d : v) p *= d;
    return p;
}

Tensor make(std::vector<idx> shape) {
    Tensor t;
    t.shape = std::move(shape);
    t.data.assign(static_cast<size_t>(prod(t.shape)), 0.0);
    return t;
}

struct Split {
    idx left, dim, right;
};
Split split(const std::vector<idx>& s, idx mode) {
    Split r{1, s[static_cast<size_t>(mode)], 1};
    for (idx n = 0; n < mode; ++n) r.left *= s[static_cast<size_t>(n)];
    for (idx n = mode + 1; n < static_cast<idx>(s.size()); ++n) r.right *= s[static_cast<size_t>(n)];
    return r;
}

// unfold_tr (tensor.hpp:147-157): m(d, r + right*l) = t[l + left*(d + dim*r)]
Mat unfold_tr(const Tensor& t, idx mode) {
    const Split s = split(t.shape, mode);
    Mat m(s.dim, s.left * s.right);
    // d in blocks of 64: the block's left x 64 source elements stay in L1 across the l loop
    constexpr idx DB = 64;
    const idx nblk = (s.dim + DB - 1) / DB;
#pragma omp parallel for collapse(2) schedule(static) if (t.size() > (1 << 16))
    for (idx r = 0; r < s.right; ++r)
        for (idx b = 0; b < nblk; ++b)
            for (idx l = 0; l < s.left; ++l)
                for (idx d = b * DB; d < std::min(s.dim, (b + 1) * DB); ++d)
                    m(d, r + s.right * l) = t.data[static_cast<size_t>(l + s.left * (d + s.dim * r))];
    return m;
}

// unfold_classic at mode 1 of a core (R_n, I_n, R_{n+1}) -> I_n x (R_n R_{n+1})
Mat core_unfold1(const Tensor& g) {
    const idx ra = g.shape[0], i = g.shape[1], rb = g.shape[2];
    Mat m(i, ra * rb);
    for (idx b = 0; b < rb; ++b)
        for (idx d = 0; d < i; ++d)
            for (idx a = 0; a < ra; ++a) m(d, a + ra * b) = g.data[static_cast<size_t>(a + ra * (d + i * b))];
    return m;
}

// 32 x 32 blocks: both the reads and the writes stay within a few cache lines / pages per block
Mat transpose(const Mat& m) {
    Mat t(m.c, m.r);
    constexpr idx B = 32;
#pragma omp parallel for schedule(static) if (m.r * m.c > (1 << 16))
    for (idx j0 = 0; j0 < m.c; j0 += B)
        for (idx i0 = 0; i0 < m.r; i0 += B)
            for (idx j = j0; j < std::min(m.c, j0 + B); ++j)
                for (idx i = i0; i < std::min(m.r, i0 + B); ++i) t(j, i) = m(i, j);
    return t;
}

Mat matmul(const Mat& A, const Mat& B) {
    Mat C(A.r, B.c);
#pragma omp parallel for schedule(static) if (A.r * B.c * A.c > (1 << 18))
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

Mat matmul_tn(const Mat& A, const Mat& B) {
    Mat C(A.c, B.c);
#pragma omp parallel for schedule(static) if (A.r * B.c * A.c > (1 << 18))
    for (idx j = 0; j < B.c; ++j)
        for (idx i = 0; i < A.c; ++i) {
            const double* ai = A.col(i);
            const double* bj = B.col(j);
            double s = 0.0;
#pragma omp simd reduction(+ : s)
            for (idx k = 0; k < A.r; ++k) s += ai[k] * bj[k];
            C(i, j) = s;
        }
    return C;
}

// chain_contract (tr_factors.hpp:92-102)
Tensor chain(const Tensor& a, const Tensor& g) {
    const idx ra = a.shape[0], p = a.shape[1], rb = a.shape[2];
    const idx i = g.shape[1], rc = g.shape[2];
    Tensor out = make({ra, p * i, rc});
    const idx M = ra * p, Nc = i * rc;
#pragma omp parallel for schedule(static) if (M * Nc * rb > (1 << 18))
    for (idx j = 0; j < Nc; ++j) {
        double* oj = out.data.data() + M * j;
        for (idx k = 0; k < rb; ++k) {
            const double w = g.data[static_cast<size_t>(k + rb * j)];
            const double* ak = a.data.data() + M * k;
            for (idx r = 0; r < M; ++r) oj[r] += ak[r] * w;
        }
    }
    return out;
}

// subchain (tr_factors.hpp:111-119)
Tensor subchain(const Cores& f, idx mode) {
    const idx N = f.order();
    Tensor cur = f.g[static_cast<size_t>((mode + 1) % N)];
    for (idx s = 2; s < N; ++s) cur = chain(cur, f.g[static_cast<size_t>((mode + s) % N)]);
    return cur;
}

// ---------------------------------------------------------------- QR / LS
// Blocked Householder kernels (compact WY): a panel of nb reflectors H_j = I - tau_j v_j v_j^T
// (v_j(j) = 1, Eigen's makeHouseholder convention as in HQR below) is applied as
// I - V T V^T with T upper triangular, so the trailing update is two GEMM-shaped passes over the
// columns (W = V^T A, A -= V (T^T W)) instead of nb rank-1 passes: the same reflectors, so the
// same R and Q^T b up to rounding (C4's 2048-4096 x 400 ALS least squares, solvers.hpp:195-205).
#if defined(__GNUC__) && !defined(__clang__) && defined(__x86_64__)
#define TRG_HOT __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define TRG_HOT
#endif

// Panel kernels of the blocked Householder QR (compact WY, panel width nb <= 32). V = the panel's
// reflectors (column-major, leading dimension ld): v_p has a unit diagonal at row j0 + p and zeros
// above, the reflector entries below. The trailing update of a chunk of up to 4 columns,
//     W = V^T A (nb x 4), Y = T^T W, A -= V Y,
// runs with 8-row vectors: 4 (p) x 4 (c) accumulators over the rows below the panel, so each V and A
// vector load feeds 4 FMAs (the former one-column loop did one FMA per two loads).
typedef double v8d __attribute__((vector_size(64)));
constexpr idx kPanelNb = 32;

TRG_HOT void panel_apply4(const double* qr, idx ld, idx m, idx j0, idx nb, const double* T, double* a, idx lda,
                          idx nc) {
    double w[kPanelNb][4];
    // rows j0 .. j0 + nb: the unit-lower-triangular top of V, done scalar
    for (idx p = 0; p < nb; ++p)
        for (idx c = 0; c < 4; ++c) {
            double s2 = 0.0;
            if (c < nc) {
                const double* ac = a + lda * c;
                s2 = ac[j0 + p];
                for (idx i = j0 + p + 1; i < j0 + nb; ++i) s2 += qr[ld * (j0 + p) + i] * ac[i];
            }
            w[p][c] = s2;
        }
    // rows j0 + nb .. m: full panel rows, 8 at a time
    const idx r0 = j0 + nb;
    const idx nv = (m - r0) / 8, rt = r0 + 8 * nv;
    for (idx p0 = 0; p0 < nb; p0 += 4) {
        const idx np = std::min<idx>(4, nb - p0);
        v8d acc[4][4];
        for (int x = 0; x < 4; ++x)
            for (int y = 0; y < 4; ++y) acc[x][y] = v8d{0, 0, 0, 0, 0, 0, 0, 0};
        for (idx v = 0; v < nv; ++v) {
            const idx i = r0 + 8 * v;
            v8d vp[4], av[4];
            for (int x = 0; x < 4; ++x) {
                if (x < np) __builtin_memcpy(&vp[x], qr + ld * (j0 + p0 + x) + i, 64);
                else vp[x] = v8d{0, 0, 0, 0, 0, 0, 0, 0};
                if (x < nc) __builtin_memcpy(&av[x], a + lda * x + i, 64);
                else av[x] = v8d{0, 0, 0, 0, 0, 0, 0, 0};
            }
            for (int x = 0; x < 4; ++x)
                for (int y = 0; y < 4; ++y) acc[x][y] += vp[x] * av[y];
        }
        for (idx x = 0; x < np; ++x)
            for (idx c = 0; c < nc; ++c) {
                double s2 = 0.0;
                for (int l = 0; l < 8; ++l) s2 += acc[x][c][l];
                const double* vq = qr + ld * (j0 + p0 + x);
                const double* ac = a + lda * c;
                for (idx i = rt; i < m; ++i) s2 += vq[i] * ac[i];
                w[p0 + x][c] += s2;
            }
    }
    double y[kPanelNb][4];  // y = T^T w
    for (idx p = 0; p < nb; ++p)
        for (idx c = 0; c < 4; ++c) {
            double s2 = 0.0;
            for (idx q = 0; q <= p; ++q) s2 += T[q + nb * p] * w[q][c];
            y[p][c] = s2;
        }
    // A -= V y: the top rows scalar, then 8-row vectors with the 4 columns' y broadcast
    for (idx c = 0; c < nc; ++c) {
        double* ac = a + lda * c;
        for (idx p = 0; p < nb; ++p) {
            ac[j0 + p] -= y[p][c];
            for (idx i = j0 + p + 1; i < j0 + nb; ++i) ac[i] -= y[p][c] * qr[ld * (j0 + p) + i];
        }
    }
    for (idx v = 0; v < nv; ++v) {
        const idx i = r0 + 8 * v;
        v8d av[4];
        for (idx c = 0; c < nc; ++c) __builtin_memcpy(&av[c], a + lda * c + i, 64);
        for (idx p = 0; p < nb; ++p) {
            v8d vp;
            __builtin_memcpy(&vp, qr + ld * (j0 + p) + i, 64);
            for (idx c = 0; c < nc; ++c) av[c] -= vp * y[p][c];
        }
        for (idx c = 0; c < nc; ++c) __builtin_memcpy(a + lda * c + i, &av[c], 64);
    }
    for (idx c = 0; c < nc; ++c) {
        double* ac = a + lda * c;
        for (idx p = 0; p < nb; ++p) {
            const double* vq = qr + ld * (j0 + p);
            for (idx i = rt; i < m; ++i) ac[i] -= y[p][c] * vq[i];
        }
    }
}

struct HQR {
    Mat qr;
    std::vector<double> tau;
    static constexpr idx kNb = 32;
    bool blocked = false;
    std::vector<std::vector<double>> Ts;  // per panel T (nb x nb, column-major)
    explicit HQR(const Mat& a) : qr(a) {
        const idx m = qr.r, n = qr.c, k = std::min(m, n);
        tau.assign(static_cast<size_t>(k), 0.0);
        blocked = n >= 2 * kNb && m * n >= (1 << 16);
        if (blocked) {
            factor_blocked();
            return;
        }
        for (idx j = 0; j < k; ++j) {
            double* cj = qr.col(j);
            const double c0 = cj[j];
            double tail = 0.0;
            for (idx i = j + 1; i < m; ++i) tail += cj[i] * cj[i];
            double beta, t;
            if (tail <= std::numeric_limits<double>::min()) {  // Eigen makeHouseholder
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
#pragma omp parallel for schedule(static) if ((n - j) * (m - j) > (1 << 15))
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
    // One panel: reflectors of columns j0 .. j0 + nb (Eigen's makeHouseholder, as HQR's unblocked
    // loop), the panel columns updated as they go. Row-parallel inside one OpenMP region with a fixed
    // row partition of [j0, m) (fixed-order reductions, bit-reproducible for a given thread count) and
    // two barriers per column: every thread derives beta / tau from the tail-norm partials itself,
    // the reflector's unit entry at row j is folded into the dot products of its owner (v_j(j) = 1),
    // and each thread's axpy pass also forms its partial of the next column's tail norm.
    void factor_panel(idx j0, idx nb) {
        const idx m = qr.r;
        const int nt = std::max(1, std::min(omp_get_max_threads(), (int)((m - j0) / 256)));
        std::vector<double> ptail((size_t)nt, 0.0), pdot((size_t)nt * kPanelNb, 0.0);
#pragma omp parallel num_threads(nt)
        {
            const int th = omp_get_thread_num();
            const idx flo = j0 + (m - j0) * th / nt, fhi = j0 + (m - j0) * (th + 1) / nt;
            {
                const double* c = qr.col(j0);
                double tl = 0.0;
#pragma omp simd reduction(+ : tl)
                for (idx i = std::max(flo, j0 + 1); i < fhi; ++i) tl += c[i] * c[i];
                ptail[(size_t)th] = tl;
            }
#pragma omp barrier
            for (idx j = j0; j < j0 + nb; ++j) {
                double* cj = qr.col(j);
                double tail = 0.0;
                for (int t2 = 0; t2 < nt; ++t2) tail += ptail[(size_t)t2];
                const double c0 = cj[j];  // row j: last written before the previous barrier
                double beta, t, inv = 0.0;
                if (tail <= std::numeric_limits<double>::min()) {  // Eigen makeHouseholder
                    t = 0.0;
                    beta = c0;
                } else {
                    beta = std::sqrt(c0 * c0 + tail);
                    if (c0 >= 0.0) beta = -beta;
                    inv = 1.0 / (c0 - beta);
                    t = (beta - c0) / beta;
                }
                const idx lo = std::max(flo, j + 1), hi = fhi;
                const bool own_j = flo <= j && j < fhi;
                if (t == 0.0) {
                    for (idx i = lo; i < hi; ++i) cj[i] = 0.0;
                } else {
#pragma omp simd
                    for (idx i = lo; i < hi; ++i) cj[i] *= inv;
                }
                const idx ncols = j0 + nb - j - 1;
                double* pp = pdot.data() + (size_t)th * kPanelNb;
                if (t != 0.0)
                    for (idx c = 0; c < ncols; ++c) {
                        const double* cc = qr.col(j + 1 + c);
                        double w = own_j ? cc[j] : 0.0;  // v_j(j) = 1
#pragma omp simd reduction(+ : w)
                        for (idx i = lo; i < hi; ++i) w += cj[i] * cc[i];
                        pp[c] = w;
                    }
#pragma omp barrier
                if (th == 0) tau[static_cast<size_t>(j)] = t;
                if (own_j) cj[j] = beta;
                double tl = 0.0;
                for (idx c = 0; c < ncols; ++c) {
                    double* cc = qr.col(j + 1 + c);
                    if (t != 0.0) {
                        double w = 0.0;
                        for (int t2 = 0; t2 < nt; ++t2) w += pdot[(size_t)t2 * kPanelNb + c];
                        w *= t;
                        if (own_j) cc[j] -= w;
#pragma omp simd
                        for (idx i = lo; i < hi; ++i) cc[i] -= w * cj[i];
                    }
                    if (c == 0) {  // the next column's tail-norm partial (rows > j + 1)
                        const idx l2 = std::max(flo, j + 2);
#pragma omp simd reduction(+ : tl)
                        for (idx i = l2; i < hi; ++i) tl += cc[i] * cc[i];
                    }
                }
                ptail[(size_t)th] = tl;
#pragma omp barrier
            }
        }
    }
    void factor_blocked() {
        const idx m = qr.r, n = qr.c, k = std::min(m, n);
        for (idx j0 = 0; j0 < k; j0 += kNb) {
            const idx nb = std::min(kNb, k - j0);
            factor_panel(j0, nb);
            // T: T(0:p, p) = -tau_p T(0:p, 0:p) V(:, 0:p)^T v_p, T(p, p) = tau_p, with V^T V of the panel
            // (rows >= j0 + p of v_q against v_p) from one row-parallel pass in a fixed order
            const int nt = std::max(1, std::min(omp_get_max_threads(), (int)((m - j0) / 512)));
            std::vector<double> gp((size_t)nt * nb * nb, 0.0);
#pragma omp parallel num_threads(nt)
            {
                const int th = omp_get_thread_num();
                const idx lo = j0 + nb + (m - j0 - nb) * th / nt, hi = j0 + nb + (m - j0 - nb) * (th + 1) / nt;
                double* g = gp.data() + (size_t)th * nb * nb;
                for (idx p = 1; p < nb; ++p) {
                    const double* vp = qr.col(j0 + p);
                    for (idx q = 0; q < p; ++q) {
                        const double* vq = qr.col(j0 + q);
                        double s2 = 0.0;
#pragma omp simd reduction(+ : s2)
                        for (idx i = lo; i < hi; ++i) s2 += vq[i] * vp[i];
                        g[q + nb * p] = s2;
                    }
                }
            }
            std::vector<double> T(static_cast<size_t>(nb * nb), 0.0);
            for (idx p = 0; p < nb; ++p) {
                const double tp = tau[static_cast<size_t>(j0 + p)];
                const double* vp = qr.col(j0 + p);
                std::vector<double> z(static_cast<size_t>(p), 0.0);
                for (idx q = 0; q < p; ++q) {  // rows j0 + p .. j0 + nb of the panel, then the thread sums
                    const double* vq = qr.col(j0 + q);
                    double s2 = vq[j0 + p];
                    for (idx i = j0 + p + 1; i < j0 + nb; ++i) s2 += vq[i] * vp[i];
                    for (int t2 = 0; t2 < nt; ++t2) s2 += gp[(size_t)t2 * nb * nb + q + nb * p];
                    z[static_cast<size_t>(q)] = s2;
                }
                for (idx q = 0; q < p; ++q) {
                    double s2 = 0.0;
                    for (idx r = q; r < p; ++r) s2 += T[static_cast<size_t>(q + nb * r)] * z[static_cast<size_t>(r)];
                    T[static_cast<size_t>(q + nb * p)] = -tp * s2;
                }
                T[static_cast<size_t>(p + nb * p)] = tp;
            }
            const double* Tp = T.data();
            const idx c0 = j0 + nb, nchunk = (n - c0 + 3) / 4;
#pragma omp parallel for schedule(dynamic, 1)
            for (idx ch = 0; ch < nchunk; ++ch) {
                const idx c = c0 + 4 * ch;
                panel_apply4(qr.a.data(), m, m, j0, nb, Tp, qr.col(c), m, std::min<idx>(4, n - c));
            }
            Ts.push_back(std::move(T));
        }
    }
    Mat solve(const Mat& b) const {
        const idx m = qr.r, n = qr.c, k = static_cast<idx>(tau.size());
        Mat y = b;
        if (blocked) {
            for (idx j0 = 0, p = 0; j0 < k; j0 += kNb, ++p) {
                const idx nb = std::min(kNb, k - j0);
                const double* Tp = Ts[static_cast<size_t>(p)].data();
                const idx nchunk = (y.c + 3) / 4;
#pragma omp parallel for schedule(dynamic, 1) if (y.c * (m - j0) > (1 << 15))
                for (idx ch = 0; ch < nchunk; ++ch)
                    panel_apply4(qr.a.data(), m, m, j0, nb, Tp, y.col(4 * ch), m, std::min<idx>(4, y.c - 4 * ch));
            }
            return back_substitute(y, b.c);
        }
        for (idx j = 0; j < k; ++j) {
            const double t = tau[static_cast<size_t>(j)];
            if (t == 0.0) continue;
            const double* v = qr.col(j);
#pragma omp parallel for schedule(static) if (y.c * (m - j) > (1 << 15))
            for (idx c = 0; c < y.c; ++c) {
                double* bc = y.col(c);
                double w = bc[j];
                for (idx i = j + 1; i < m; ++i) w += v[i] * bc[i];
                w *= t;
                bc[j] -= w;
                for (idx i = j + 1; i < m; ++i) bc[i] -= w * v[i];
            }
        }
        return back_substitute(y, b.c);
    }
    // R x = y column by column of R (contiguous), bottom up: x_j = y_j / R_jj, then y(0:j) -= x_j R(0:j, j)
    Mat back_substitute(const Mat& y, idx nc) const {
        const idx n = qr.c;
        Mat x(n, nc);
#pragma omp parallel for schedule(static) if (nc * n * n > (1 << 16))
        for (idx c = 0; c < nc; ++c) {
            std::vector<double> t(y.col(c), y.col(c) + n);
            for (idx j = n - 1; j >= 0; --j) {
                const double xj = t[static_cast<size_t>(j)] / qr(j, j);
                x(j, c) = xj;
                const double* rj = qr.col(j);
#pragma omp simd
                for (idx i = 0; i < j; ++i) t[static_cast<size_t>(i)] -= xj * rj[i];
            }
        }
        return x;
    }
};

bool cholesky(const Mat& a, Mat& L) {
    const idx n = a.r;
    L = Mat(n, n);
    for (idx j = 0; j < n; ++j) {
        double d = a(j, j);
        for (idx k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
        if (!(d > 0.0)) return false;
        const double l = std::sqrt(d);
        L(j, j) = l;
        for (idx i = j + 1; i < n; ++i) {
            double s = a(i, j);
            for (idx k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
            L(i, j) = s / l;
        }
    }
    return true;
}

Mat chol_solve(const Mat& L, const Mat& b) {
    const idx n = L.r;
    Mat x = b;
#pragma omp parallel for schedule(static) if (b.c * n * n > (1 << 16))
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

// LDL^T with symmetric pivoting (Eigen::LDLT semantics), used by ridge_solve.
Mat ldlt_solve(Mat a, const Mat& b) {
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
    std::vector<double> y(static_cast<size_t>(n));
    for (idx c = 0; c < b.c; ++c) {
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

// solvers.hpp:186-190
Mat ridge_solve(Mat gram, const Mat& rhs) {
    double tr = 0.0;
    for (idx i = 0; i < gram.r; ++i) tr += gram(i, i);
    const double lambda = 1e-12 * tr / static_cast<double>(gram.r);
    for (idx i = 0; i < gram.r; ++i) gram(i, i) += lambda;
    return ldlt_solve(std::move(gram), rhs);
}

// solvers.hpp:195-205
Mat ls_solve_qr(const Mat& a, const Mat& b) {
    if (a.r >= a.c) {
        // the device route first (device_ls.cu: cuSOLVER Householder QR, the same rank cutoff)
        Mat x(a.c, b.c);
        const int st = device_ls_qr(a.a.data(), a.r, a.c, b.a.data(), b.c, x.a.data());
        if (st == 0) return x;
        if (st == 1) return ridge_solve(matmul_tn(a, a), matmul_tn(a, b));
        PhaseTimer t(kPhLsHost);
        HQR qr(a);
        double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
        for (idx i = 0; i < a.c; ++i) {
            dmax = std::max(dmax, std::abs(qr.qr(i, i)));
            dmin = std::min(dmin, std::abs(qr.qr(i, i)));
        }
        const double cutoff = dmax * static_cast<double>(std::max(a.r, a.c)) * std::numeric_limits<double>::epsilon() * 16.0;
        if (dmax > 0.0 && dmin > cutoff) return qr.solve(b);
    }
    return ridge_solve(matmul_tn(a, a), matmul_tn(a, b));
}

// solvers.hpp:209-219
Mat ls_solve_gram(const Mat& gram, const Mat& rhs) {
    Mat L;
    if (cholesky(gram, L)) {
        double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
        for (idx i = 0; i < L.r; ++i) {
            dmax = std::max(dmax, std::abs(L(i, i)));
            dmin = std::min(dmin, std::abs(L(i, i)));
        }
        const double cutoff = dmax * static_cast<double>(gram.r) * std::numeric_limits<double>::epsilon() * 16.0;
        if (dmax > 0.0 && dmin > cutoff) return chol_solve(L, rhs);
    }
    return ridge_solve(gram, rhs);
}

// solvers.hpp:102-129: Gram of the subchain's mode-2 TR unfolding via per-core transfer matrices
Mat subchain_gram(const Cores& f, idx n) {
    const idx N = f.order();
    Mat omega;
    for (idx s = 1; s < N; ++s) {
        const Tensor& g = f.g[static_cast<size_t>((n + s) % N)];
        const idx rk = g.shape[0], rk1 = g.shape[2];
        const Mat h = core_unfold1(g);
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

// solvers.hpp:134-182: V = X_<n> S one core at a time
Mat subchain_rhs(const Mat& xn_tr, const Cores& f, idx n) {
    const idx N = f.order();
    const idx dim_n = xn_tr.r;
    const Mat b = transpose(xn_tr);
    const Tensor& g0 = f.g[static_cast<size_t>((n + 1) % N)];
    const idx r0 = g0.shape[0], i0 = g0.shape[1], s0 = g0.shape[2];
    Mat ghat(r0 * s0, i0);
    for (idx i = 0; i < i0; ++i)
        for (idx s = 0; s < s0; ++s)
            for (idx r = 0; r < r0; ++r) ghat(r + r0 * s, i) = g0.data[static_cast<size_t>(r + r0 * (i + i0 * s))];
    Mat bm(i0, static_cast<idx>(b.a.size()) / i0);
    bm.a = b.a;
    Mat cur = matmul(ghat, bm);
    const idx front = r0;
    for (idx s = 2; s < N; ++s) {
        const Tensor& g = f.g[static_cast<size_t>((n + s) % N)];
        const idx rk = g.shape[0], ik = g.shape[1], rk1 = g.shape[2];
        const idx mid = rk * ik;
        const idx tail = static_cast<idx>(cur.a.size()) / (front * mid);
        Mat next(front * rk1, tail);
#pragma omp parallel for schedule(static) if (tail * front * mid * rk1 > (1 << 18))
        for (idx t = 0; t < tail; ++t) {
            const double* in = cur.a.data() + front * mid * t;
            double* out = next.a.data() + front * rk1 * t;
            for (idx c = 0; c < rk1; ++c)
                for (idx q = 0; q < mid; ++q) {
                    const double w = g.data[static_cast<size_t>(q + mid * c)];
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

// solvers.hpp:223-230
void store_core(Tensor& core, const Mat& z) {
    const idx rn = core.shape[0], in = core.shape[1], rn1 = core.shape[2];
    for (idx s = 0; s < rn1; ++s)
        for (idx i = 0; i < in; ++i)
            for (idx r = 0; r < rn; ++r) core.data[static_cast<size_t>(r + rn * (i + in * s))] = z(r + rn * s, i);
}

constexpr idx kDirectLsMaxRows = 4096;  // solvers.hpp:234

// solvers.hpp:238-251
void als_update_mode(const Mat& xn_tr, Cores& f, idx n) {
    const idx n_cols = xn_tr.c;
    const idx m = f.rank(n) * f.rank((n + 1) % f.order());
    Mat z;
    if (n_cols <= kDirectLsMaxRows && n_cols >= m) {
        // the system built and solved on the device when it is large enough (device_ls.cu)
        const int st = device_als_direct(f, n, xn_tr, z);
        if (st == 0) {
            PhaseTimer t(kPhStore);
            store_core(f.g[static_cast<size_t>(n)], z);
            return;
        }
        Tensor s;
        {
            PhaseTimer t(kPhSubchain);
            s = subchain(f, n);
        }
        Mat a, b;
        {
            PhaseTimer t(kPhUnfold);
            a = unfold_tr(s, 1);
            b = transpose(xn_tr);
        }
        z = ls_solve_qr(a, b);
    } else {
        z = ls_solve_gram(subchain_gram(f, n), transpose(subchain_rhs(xn_tr, f, n)));
    }
    PhaseTimer t(kPhStore);
    store_core(f.g[static_cast<size_t>(n)], z);
}

double fnorm(const Tensor& t) {
    double s = 0.0;
    for (double v : t.data) s += v * v;
    return std::sqrt(s);
}

SolveOut order_one(const Tensor& x, idx r0) {  // solvers.hpp:268-279
    Tensor core = make({r0, x.shape[0], r0});
    for (idx i = 0; i < x.shape[0]; ++i) core.data[static_cast<size_t>(r0 * i)] = x.data[static_cast<size_t>(i)];
    SolveOut o;
    o.cores.g.push_back(std::move(core));
    o.rse_history = {fnorm(x) > 0.0 ? rse(x, reconstruct_full(o.cores)) : 0.0};
    o.sweeps_run = 1;
    return o;
}

SolveOut zero_report(const Tensor& x, const std::vector<idx>& ranks) {  // solvers.hpp:281-290
    SolveOut o;
    const idx N = x.order();
    for (idx n = 0; n < N; ++n)
        o.cores.g.push_back(make({ranks[static_cast<size_t>(n)], x.shape[static_cast<size_t>(n)],
                                  ranks[static_cast<size_t>((n + 1) % N)]}));
    o.rse_history = {0.0};
    return o;
}

// one-sided Jacobi thin SVD, singular values descending (BDCSVD stand-in). Sweeps visit the
// column pairs in round-robin (tournament) order: every round is n/2 disjoint pairs, rotated in
// parallel, so the 576 x 432 / 1024 x 64 shapes of C5 / C2 use all host cores.
namespace {
inline bool jacobi_rotate(double* wp, double* wq, double* vp, double* vq, idx m, idx n) {
    double al = 0.0, be = 0.0, ga = 0.0;
    for (idx i = 0; i < m; ++i) {
        al += wp[i] * wp[i];
        be += wq[i] * wq[i];
        ga += wp[i] * wq[i];
    }
    if (ga == 0.0 || std::abs(ga) <= 1e-15 * std::sqrt(al * be)) return false;
    const double zeta = (be - al) / (2.0 * ga);
    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
    const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
    for (idx i = 0; i < m; ++i) {
        const double x = wp[i], y = wq[i];
        wp[i] = c * x - sn * y;
        wq[i] = sn * x + c * y;
    }
    for (idx i = 0; i < n; ++i) {
        const double x = vp[i], y = vq[i];
        vp[i] = c * x - sn * y;
        vq[i] = sn * x + c * y;
    }
    return true;
}
}  // namespace

void svd(const Mat& a, Mat& U, std::vector<double>& s, Mat& V) {
    if (device_svd(a, U, s, V) == 0) return;  // large unfoldings (C5's 576 x 432) on the GPU
    const bool wide = a.r < a.c;
    Mat W = wide ? transpose(a) : a;
    const idx m = W.r, n = W.c;
    Mat Vw(n, n);
    for (idx i = 0; i < n; ++i) Vw(i, i) = 1.0;
    // tournament schedule over np = n rounded up to even players (player n is a bye)
    const idx np = n + (n & 1);
    std::vector<idx> pos(static_cast<size_t>(np));
    std::iota(pos.begin(), pos.end(), 0);
    const bool par = n >= 16 && m * n >= (1 << 14);
    for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (idx round = 0; round < np - 1; ++round) {
#pragma omp parallel for schedule(static) reduction(| : rotated) if (par)
            for (idx k = 0; k < np / 2; ++k) {
                idx p = pos[static_cast<size_t>(k)], q = pos[static_cast<size_t>(np - 1 - k)];
                if (p >= n || q >= n) continue;
                if (p > q) std::swap(p, q);
                if (jacobi_rotate(W.col(p), W.col(q), Vw.col(p), Vw.col(q), m, n)) rotated |= 1;
            }
            // circle method: player 0 stays, the others rotate one place
            const idx last = pos[static_cast<size_t>(np - 1)];
            for (idx k = np - 1; k > 1; --k) pos[static_cast<size_t>(k)] = pos[static_cast<size_t>(k - 1)];
            pos[1] = last;
        }
        if (!rotated) break;
    }
    std::vector<double> sv(static_cast<size_t>(n));
    for (idx j = 0; j < n; ++j) {
        double q = 0.0;
        for (idx i = 0; i < m; ++i) q += W(i, j) * W(i, j);
        sv[static_cast<size_t>(j)] = std::sqrt(q);
    }
    std::vector<idx> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](idx x, idx y) { return sv[static_cast<size_t>(x)] > sv[static_cast<size_t>(y)]; });
    Mat Us(m, n), Vs(n, n);
    s.assign(static_cast<size_t>(n), 0.0);
    for (idx j = 0; j < n; ++j) {
        const idx src = ord[static_cast<size_t>(j)];
        const double sj = sv[static_cast<size_t>(src)];
        s[static_cast<size_t>(j)] = sj;
        for (idx i = 0; i < m; ++i) Us(i, j) = sj > 0.0 ? W(i, src) / sj : 0.0;
        for (idx i = 0; i < n; ++i) Vs(i, j) = Vw(i, src);
    }
    if (wide) {
        U = std::move(Vs);
        V = std::move(Us);
    } else {
        U = std::move(Us);
        V = std::move(Vs);
    }
    // sign convention shared with the oracle: largest-magnitude entry of each U column positive
    for (idx j = 0; j < U.c; ++j) {
        idx arg = 0;
        for (idx i = 1; i < U.r; ++i)
            if (std::abs(U(i, j)) > std::abs(U(arg, j))) arg = i;
        if (U(arg, j) < 0.0) {
            for (idx i = 0; i < U.r; ++i) U(i, j) = -U(i, j);
            for (idx i = 0; i < V.r; ++i) V(i, j) = -V(i, j);
        }
    }
}

idx truncation_rank(const std::vector<double>& sv, double budget_sq, double* disc) {  // solvers.hpp:347-358
    idx r = static_cast<idx>(sv.size());
    double tail = 0.0;
    while (r > 1) {
        const double t = tail + sv[static_cast<size_t>(r - 1)] * sv[static_cast<size_t>(r - 1)];
        if (t > budget_sq) break;
        tail = t;
        --r;
    }
    *disc += tail;
    return r;
}

std::pair<idx, idx> balanced_divisor_split(idx r) {  // solvers.hpp:361-371
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

}  // namespace

// tr_factors.hpp:123-137 at mode 0: X_<0> = G_{0,(2)} S^T, folded (mode 0 fold is free)
Tensor reconstruct_full(const Cores& f) {
    const idx N = f.order();
    std::vector<idx> shape;
    for (idx n = 0; n < N; ++n) shape.push_back(f.dim(n));
    Tensor out = make(shape);
    if (N == 1) {
        const Tensor& g = f.g[0];
        const idx r = g.shape[0], I = g.shape[1];
        for (idx i = 0; i < I; ++i) {
            double tr = 0.0;
            for (idx a = 0; a < std::min(r, g.shape[2]); ++a) tr += g.data[static_cast<size_t>(a + r * (i + I * a))];
            out.data[static_cast<size_t>(i)] = tr;
        }
        return out;
    }
    const Mat core2 = core_unfold1(f.g[0]);      // I_0 x (R_0 R_1)
    const Tensor s = subchain(f, 0);             // (R_1, P, R_0)
    const idx R1 = s.shape[0], P = s.shape[1], R0 = s.shape[2], I0 = core2.r;
#pragma omp parallel for schedule(static) if (I0 * P * R0 * R1 > (1 << 18))
    for (idx p = 0; p < P; ++p) {
        double* xp = out.data.data() + I0 * p;
        for (idx b = 0; b < R1; ++b)
            for (idx a = 0; a < R0; ++a) {
                const double w = s.data[static_cast<size_t>(b + R1 * (p + P * a))];
                const double* ck = core2.col(a + R0 * b);
                for (idx i = 0; i < I0; ++i) xp[i] += ck[i] * w;
            }
    }
    return out;
}

double rse(const Tensor& ref, const Tensor& approx) {  // solvers.hpp:47-54
    require(ref.shape == approx.shape, "rse: shape mismatch");
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < ref.data.size(); ++i) {
        const double d = ref.data[i] - approx.data[i];
        num += d * d;
        den += ref.data[i] * ref.data[i];
    }
    require(den > 0.0, "rse: reference tensor has zero norm");
    return std::sqrt(num) / std::sqrt(den);
}

SolveOut trals(const Tensor& x, const std::vector<idx>& ranks, double tolerance, idx max_sweeps, std::uint64_t seed) {
    require(static_cast<idx>(ranks.size()) == x.order(), "trals: rank vector length must equal tensor order");
    for (idx r : ranks) require(r >= 1, "trals: ranks must be positive");
    require(max_sweeps >= 1, "trals: max_sweeps must be positive");
    const double xnorm = fnorm(x);
    if (xnorm == 0.0) return zero_report(x, ranks);
    if (x.order() == 1) return order_one(x, ranks[0]);
    const idx N = x.order();
    // init_factors (solvers.hpp:80-95)
    Cores f;
    double pr = 1.0;
    for (idx r : ranks) pr *= static_cast<double>(r);
    const double scale = std::pow(xnorm / pr, 1.0 / static_cast<double>(N));
    GaussianStream gs(seed);
    for (idx n = 0; n < N; ++n) {
        Tensor core = make({ranks[static_cast<size_t>(n)], x.shape[static_cast<size_t>(n)], ranks[static_cast<size_t>((n + 1) % N)]});
        for (auto& v : core.data) v = scale * gs.next();
        f.g.push_back(std::move(core));
    }
    std::vector<Mat> unf;
    for (idx n = 0; n < N; ++n) unf.push_back(unfold_tr(x, n));
    SolveOut o;
    for (idx sweep = 1; sweep <= max_sweeps; ++sweep) {
        for (idx n = 0; n < N; ++n) als_update_mode(unf[static_cast<size_t>(n)], f, n);
        {
            PhaseTimer t(kPhRse);
            double e = 0.0;
            o.rse_history.push_back(device_tr_rse(f, x, &e) == 0 ? e : rse(x, reconstruct_full(f)));
        }
        o.sweeps_run = sweep;
        const size_t k = o.rse_history.size();
        if (k >= 2 && std::abs(o.rse_history[k - 1] - o.rse_history[k - 2]) < tolerance * o.rse_history[k - 2]) break;
    }
    o.cores = std::move(f);
    if (solve_prof_on()) {
        for (int p = 0; p < kPhCount; ++p) {
            fprintf(stderr, "[trg solve] %-10s %9.3f ms\n", kPhaseName[p], g_phase_ms[p]);
            g_phase_ms[p] = 0.0;
        }
    }
    return o;
}

SolveOut trsvd(const Tensor& x, double tolerance) {
    require(tolerance >= 0.0, "trsvd: tolerance must be nonnegative");
    const idx order = x.order();
    const double xnorm = fnorm(x);
    if (order == 1) return order_one(x, 1);
    if (xnorm == 0.0) return zero_report(x, std::vector<idx>(static_cast<size_t>(order), 1));
    const double budget = tolerance * xnorm / std::sqrt(static_cast<double>(order));
    const double budget_sq = budget * budget;
    double disc = 0.0;
    const idx dim0 = x.shape[0];
    const idx rest = x.size() / dim0;
    Mat m0(dim0, rest);
    m0.a = x.data;
    Mat U, V;
    std::vector<double> s;
    svd(m0, U, s, V);
    const idx r01 = truncation_rank(s, budget_sq, &disc);
    const auto [ra, rb] = balanced_divisor_split(r01);
    SolveOut o;
    o.cores.g.resize(static_cast<size_t>(order));
    {
        Tensor g0 = make({ra, dim0, rb});
        for (idx q = 0; q < rb; ++q)
            for (idx i = 0; i < dim0; ++i)
                for (idx p = 0; p < ra; ++p) g0.data[static_cast<size_t>(p + ra * (i + dim0 * q))] = U(i, p + ra * q);
        o.cores.g[0] = std::move(g0);
    }
    std::vector<double> cur(static_cast<size_t>(r01 * rest));
    for (idx p = 0; p < ra; ++p)
        for (idx c = 0; c < rest; ++c)
            for (idx q = 0; q < rb; ++q) {
                const idx row = p + ra * q;
                cur[static_cast<size_t>(q + rb * c + rb * rest * p)] = s[static_cast<size_t>(row)] * V(c, row);
            }
    idx lead = rb;
    for (idx k = 1; k + 1 < order; ++k) {
        const idx dk = x.shape[static_cast<size_t>(k)];
        const idx rows = lead * dk;
        const idx cols = static_cast<idx>(cur.size()) / rows;
        Mat mk(rows, cols);
        mk.a = cur;
        svd(mk, U, s, V);
        const idx r = truncation_rank(s, budget_sq, &disc);
        Tensor gk = make({lead, dk, r});
        for (idx j = 0; j < r; ++j)
            for (idx i = 0; i < rows; ++i) gk.data[static_cast<size_t>(i + rows * j)] = U(i, j);
        o.cores.g[static_cast<size_t>(k)] = std::move(gk);
        std::vector<double> next(static_cast<size_t>(r * cols));
        for (idx c = 0; c < cols; ++c)
            for (idx j = 0; j < r; ++j) next[static_cast<size_t>(j + r * c)] = s[static_cast<size_t>(j)] * V(c, j);
        cur = std::move(next);
        lead = r;
    }
    {
        Tensor gl;
        gl.shape = {lead, x.shape[static_cast<size_t>(order - 1)], ra};
        gl.data = std::move(cur);
        o.cores.g[static_cast<size_t>(order - 1)] = std::move(gl);
    }
    o.rse_history = {rse(x, reconstruct_full(o.cores))};
    o.sweeps_run = 1;
    o.discarded_sq = disc;
    return o;
}

}  // namespace host
}  // namespace trg
