// SPDX-License-Identifier: Apache-2.0
//
// Device least squares for the small solve's direct route (row f2; solvers.hpp:195-205, the
// ALS update of solvers.hpp:238-251 at C4's 2048-4096 x 400 subchain unfoldings): Householder QR
// of A on the GPU (cuSOLVER geqrf), the same full-rank test on |R_ii| as the host route, then
// x = R^-1 (Q^T b) (ormqr + trsm). Householder QR as the reference's ColPivHouseholder-free
// HouseholderQR: a full-rank system has one solution, so x agrees with the host route up to
// rounding (the reflector sign convention and blocking differ, not the algorithm).
//
// cuSOLVER / cuBLAS are library code here (as cuBLAS GEMMs are for plain GEMMs), loaded with
// dlopen by soname at first use, so libtrg.so carries no link-time dependency on them and shares
// the copies a PyTorch process may already have loaded. TRG_HOST_LS=1 keeps every solve on the
// host (A/B tests); without a CUDA device the host route runs, as before.
//
// device_als_direct builds the system on the GPU as well: the subchain of the other cores
// (tr_factors.hpp:111-119; one cuBLAS DGEMM per chain_contract, tr_factors.hpp:92-102), its
// mode-1 TR unfolding (tensor.hpp:147-157) and the transposed right-hand side by two permutation
// kernels, so only the cores (tens of KB) and X_<n> (1-2 MB) cross PCIe per update instead of the
// 6-13 MB system matrix, and the host's subchain / unfold passes disappear.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <vector>

#include "host_solve.hpp"

namespace trg {
namespace host {

namespace {

struct DevLs {
    bool ok = false;
    decltype(&cusolverDnCreate) create = nullptr;
    decltype(&cusolverDnSetStream) set_stream = nullptr;
    decltype(&cusolverDnDgeqrf_bufferSize) geqrf_ws = nullptr;
    decltype(&cusolverDnDgeqrf) geqrf = nullptr;
    decltype(&cusolverDnDormqr_bufferSize) ormqr_ws = nullptr;
    decltype(&cusolverDnDormqr) ormqr = nullptr;
    decltype(&cublasCreate_v2) cb_create = nullptr;
    decltype(&cublasSetStream_v2) cb_set_stream = nullptr;
    decltype(&cublasDtrsm_v2) trsm = nullptr;
    decltype(&cublasDgemm_v2) gemm = nullptr;
    // optional: Jacobi SVD (device_svd); absent symbols leave the host SVD in place
    decltype(&cusolverDnCreateGesvdjInfo) svdj_info = nullptr;
    decltype(&cusolverDnDgesvdj_bufferSize) svdj_ws = nullptr;
    decltype(&cusolverDnDgesvdj) svdj = nullptr;
    gesvdjInfo_t svdj_params = nullptr;
    cusolverDnHandle_t sh = nullptr;
    cublasHandle_t bh = nullptr;
    cudaStream_t stream = nullptr;
    int device = -1;
    // device buffers, grown on demand: A (m x n), B (m x nrhs), tau, workspace, info
    double *dA = nullptr, *dB = nullptr, *dtau = nullptr, *dwork = nullptr;
    // device-built systems: cores, X_<n>, two subchain ping-pong buffers
    double *dG = nullptr, *dXt = nullptr, *dS0 = nullptr, *dS1 = nullptr;
    // per-sweep RSE: reconstruction, mode-1 unfolding of core 0, block partial sums
    double *dY = nullptr, *dC = nullptr, *dPart = nullptr;
    int* dinfo = nullptr;
    size_t capA = 0, capB = 0, capT = 0, capW = 0, capG = 0, capX = 0, capS0 = 0, capS1 = 0, capY = 0, capC = 0,
           capPart = 0;
};

template <class F>
bool sym(void* lib, const char* name, F& f) {
    f = reinterpret_cast<F>(dlsym(lib, name));
    return f != nullptr;
}

DevLs* dev_ls() {
    static DevLs d;
    static std::once_flag once;
    std::call_once(once, [] {
        if (getenv("TRG_HOST_LS")) return;
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            return;
        }
        void* ls = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        void* lb = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!ls || !lb) return;
        if (!(sym(ls, "cusolverDnCreate", d.create) && sym(ls, "cusolverDnSetStream", d.set_stream) &&
              sym(ls, "cusolverDnDgeqrf_bufferSize", d.geqrf_ws) && sym(ls, "cusolverDnDgeqrf", d.geqrf) &&
              sym(ls, "cusolverDnDormqr_bufferSize", d.ormqr_ws) && sym(ls, "cusolverDnDormqr", d.ormqr) &&
              sym(lb, "cublasCreate_v2", d.cb_create) && sym(lb, "cublasSetStream_v2", d.cb_set_stream) &&
              sym(lb, "cublasDtrsm_v2", d.trsm) && sym(lb, "cublasDgemm_v2", d.gemm)))
            return;
        if (sym(ls, "cusolverDnCreateGesvdjInfo", d.svdj_info) && sym(ls, "cusolverDnDgesvdj_bufferSize", d.svdj_ws) &&
            sym(ls, "cusolverDnDgesvdj", d.svdj)) {
            if (d.svdj_info(&d.svdj_params) != CUSOLVER_STATUS_SUCCESS) d.svdj = nullptr;
        } else {
            d.svdj = nullptr;
        }
        if (cudaGetDevice(&d.device) != cudaSuccess) return;
        if (cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess) return;
        if (d.create(&d.sh) != CUSOLVER_STATUS_SUCCESS || d.set_stream(d.sh, d.stream) != CUSOLVER_STATUS_SUCCESS)
            return;
        if (d.cb_create(&d.bh) != CUBLAS_STATUS_SUCCESS || d.cb_set_stream(d.bh, d.stream) != CUBLAS_STATUS_SUCCESS)
            return;
        if (cudaMalloc(&d.dinfo, sizeof(int)) != cudaSuccess) return;
        d.ok = true;
    });
    return d.ok ? &d : nullptr;
}

bool grow(double*& p, size_t& cap, size_t n) {
    if (n <= cap) return true;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) return false;
    cap = n;
    return true;
}

}  // namespace

namespace {

// one set of device buffers, so one solve at a time
std::mutex g_mu;

// A (m x n, ld m) and B (m x nrhs, ld m) already in d->dA / d->dB on d->stream: Householder QR,
// the host route's |R_ii| cutoff, x = R^-1 (Q^T B) into x (n x nrhs, host).
// 0: solved; 1: rank-deficient (caller: ridge); -1: device failure (caller: host route)
int factor_solve(DevLs* d, idx m, idx n, idx nrhs, double* x, std::chrono::steady_clock::time_point& t0) {
    const int M = (int)m, Nn = (int)n, R = (int)nrhs;
    cudaStream_t s = d->stream;
    const bool prof = solve_prof_on();
    auto lap = [&](int ph) {
        if (!prof) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        solve_prof_add(ph, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    lap(kPhLsH2D);
    if (d->geqrf(d->sh, M, Nn, d->dA, M, d->dtau, d->dwork, (int)d->capW, d->dinfo) != CUSOLVER_STATUS_SUCCESS)
        return -1;
    // |R_ii|: the diagonal of the factored A (stride m + 1)
    std::vector<double> diag((size_t)n);
    if (cudaMemcpy2DAsync(diag.data(), sizeof(double), d->dA, sizeof(double) * (m + 1), sizeof(double), (size_t)n,
                          cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return -1;
    lap(kPhLsFactor);
    double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
    for (double v : diag) {
        dmax = std::max(dmax, std::abs(v));
        dmin = std::min(dmin, std::abs(v));
    }
    const double cutoff = dmax * static_cast<double>(std::max(m, n)) * std::numeric_limits<double>::epsilon() * 16.0;
    if (!(dmax > 0.0 && dmin > cutoff)) return 1;
    if (d->ormqr(d->sh, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, M, R, Nn, d->dA, M, d->dtau, d->dB, M, d->dwork, (int)d->capW,
                 d->dinfo) != CUSOLVER_STATUS_SUCCESS)
        return -1;
    const double one = 1.0;
    if (d->trsm(d->bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, Nn, R, &one, d->dA,
                M, d->dB, M) != CUBLAS_STATUS_SUCCESS)
        return -1;
    // x = the top n rows of B
    if (cudaMemcpy2DAsync(x, sizeof(double) * n, d->dB, sizeof(double) * m, sizeof(double) * n, (size_t)nrhs,
                          cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return -1;
    lap(kPhLsApply);
    return 0;
}

// workspaces for an m x n system with nrhs right-hand sides
bool reserve(DevLs* d, idx m, idx n, idx nrhs) {
    if (!grow(d->dA, d->capA, (size_t)m * n) || !grow(d->dB, d->capB, (size_t)m * nrhs) ||
        !grow(d->dtau, d->capT, (size_t)n))
        return false;
    int lw1 = 0, lw2 = 0;
    if (d->geqrf_ws(d->sh, (int)m, (int)n, d->dA, (int)m, &lw1) != CUSOLVER_STATUS_SUCCESS ||
        d->ormqr_ws(d->sh, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, (int)m, (int)nrhs, (int)n, d->dA, (int)m, d->dtau, d->dB,
                    (int)m, &lw2) != CUSOLVER_STATUS_SUCCESS)
        return false;
    return grow(d->dwork, d->capW, (size_t)std::max(lw1, lw2));
}

// small systems stay on the host: below ~1e6 m n^2 the transfers and launches cost more than the
// factorisation (C1's 100 x 25 systems: 3.5 ms host against 25 ms device per decompose)
bool device_sized(idx m, idx n, idx nrhs) {
    return !(m < n || m > (1 << 30) || n < 1 || nrhs < 1 || (double)m * (double)n * (double)n < 1e6);
}

// unfold_tr(s, 1) of a subchain s (ra, D, rc) (tensor.hpp:147-157 with left = ra, dim = D,
// right = rc): A(d, r + rc l) = s[l + ra (d + D r)], A column-major D x (rc ra). One thread per
// output element, consecutive threads on consecutive d: coalesced stores, ra-strided loads
// (the whole s is L2-resident).
__global__ void k_unfold_subchain(const double* __restrict__ s, double* __restrict__ a, long long D, int ra, int rc) {
    const long long total = D * (long long)ra * rc;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long dd = e % D, col = e / D;
        const int r = (int)(col % rc), l = (int)(col / rc);
        a[e] = s[l + ra * (dd + D * r)];
    }
}

// B = X_<n>^T: xt (rows x cols, column-major) -> b (cols x rows), 32 x 32 tiles through shared memory
__global__ void k_transpose(const double* __restrict__ xt, double* __restrict__ b, int rows, int cols) {
    __shared__ double t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = r0 + threadIdx.x, c = c0 + j;
        if (r < rows && c < cols) t[j][threadIdx.x] = xt[r + (long long)rows * c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int c = c0 + threadIdx.x, r = r0 + j;
        if (r < rows && c < cols) b[c + (long long)cols * r] = t[threadIdx.x][j];
    }
}

// reconstruct_full's operands (tr_factors.hpp:123-137 at mode 0): W(a + R0 b, p) =
// s[b + R1 (p + P a)] for the subchain s = (R1, P, R0) of cores 1..N-1, and core2(i, a + R0 b) =
// g0[a + R0 (i + I0 b)]; then X_<0> = core2 W is one DGEMM
__global__ void k_rse_operands(const double* __restrict__ s, const double* __restrict__ g0, double* __restrict__ w,
                               double* __restrict__ c2, long long P, int R0, int R1, int I0) {
    const long long nw = P * R0 * R1, nc = (long long)I0 * R0 * R1;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nw + nc;
         e += (long long)gridDim.x * blockDim.x) {
        if (e < nw) {
            const long long q = e % ((long long)R0 * R1), p = e / ((long long)R0 * R1);
            const int a = (int)(q % R0), b = (int)(q / R0);
            w[e] = s[b + R1 * (p + P * a)];
        } else {
            const long long f = e - nw;
            const long long i = f % I0, q = f / I0;
            const int a = (int)(q % R0), b = (int)(q / R0);
            c2[f] = g0[a + R0 * (i + (long long)I0 * b)];
        }
    }
}

// per-block sums of (x - y)^2 and x^2 (solvers.hpp:47-54); fixed grid and tree: deterministic
constexpr int kRseBlocks = 148 * 2;
__global__ void __launch_bounds__(256) k_rse_partials(const double* __restrict__ x, const double* __restrict__ y,
                                                      long long n, double* __restrict__ part) {
    double num = 0.0, den = 0.0;
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (long long)gridDim.x * 256) {
        const double v = x[e], dd = v - y[e];
        num = fma(dd, dd, num);
        den = fma(v, v, den);
    }
    __shared__ double sn[8], sd[8];
    for (int o = 16; o; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sn[threadIdx.x >> 5] = num;
        sd[threadIdx.x >> 5] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += sn[w];
            b += sd[w];
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

// subchain of cores first, first+1, ..., first+N-2 (mod N) into one of two ping-pong buffers; the
// cores are at d->dG + off[k - 1] for chain position k = 1..N-1. Returns the result pointer and
// its shape (ra, p, rb), or nullptr on a cuBLAS failure.
const double* device_subchain(DevLs* d, const Cores& f, idx first, const std::vector<size_t>& off, idx& ra, idx& p,
                              idx& rb) {
    const idx N = f.order();
    const Tensor& g0 = f.g[(size_t)(first % N)];
    const double* cur = d->dG + off[0];
    ra = g0.shape[0];
    p = g0.shape[1];
    rb = g0.shape[2];
    double* bufs[2] = {d->dS0, d->dS1};
    const double one = 1.0, zero = 0.0;
    for (idx k = 2; k < N; ++k) {
        const Tensor& g = f.g[(size_t)((first + k - 1) % N)];
        const idx i = g.shape[1], rc = g.shape[2];
        double* out = bufs[k % 2];
        if (d->gemm(d->bh, CUBLAS_OP_N, CUBLAS_OP_N, (int)(ra * p), (int)(i * rc), (int)rb, &one, cur, (int)(ra * p),
                    d->dG + off[(size_t)(k - 1)], (int)rb, &zero, out, (int)(ra * p)) != CUBLAS_STATUS_SUCCESS)
            return nullptr;
        cur = out;
        p *= i;
        rb = rc;
    }
    return cur;
}

}  // namespace

// 0: solved into x (n x nrhs); 1: rank-deficient by the host route's cutoff (caller: ridge);
// -1: no device route (caller: host QR)
int device_ls_qr(const double* a, idx m, idx n, const double* b, idx nrhs, double* x) {
    std::lock_guard<std::mutex> lock(g_mu);
    if (!device_sized(m, n, nrhs)) return -1;
    DevLs* d = dev_ls();
    if (!d || !reserve(d, m, n, nrhs)) return -1;
    cudaStream_t s = d->stream;
    auto t0 = std::chrono::steady_clock::now();
    if (cudaMemcpyAsync(d->dA, a, sizeof(double) * m * n, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(d->dB, b, sizeof(double) * m * nrhs, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return -1;
    return factor_solve(d, m, n, nrhs, x, t0);
}

int device_als_direct(const Cores& f, idx n, const Mat& xn_tr, Mat& z) {
    std::lock_guard<std::mutex> lock(g_mu);
    const idx N = f.order();
    const idx rows = xn_tr.c;                                      // prod of the other extents
    const idx cols = f.rank(n) * f.rank((n + 1) % N);              // R_n R_{n+1}
    const idx nrhs = xn_tr.r;                                      // I_n
    if (N < 2 || !device_sized(rows, cols, nrhs)) return -1;
    DevLs* d = dev_ls();
    if (!d || !reserve(d, rows, cols, nrhs)) return -1;
    cudaStream_t s = d->stream;
    auto t0 = std::chrono::steady_clock::now();
    // cores n+1, ..., n+N-1 back to back
    std::vector<size_t> off;
    size_t tot = 0;
    for (idx k = 1; k < N; ++k) {
        off.push_back(tot);
        tot += f.g[(size_t)((n + k) % N)].data.size();
    }
    if (!grow(d->dG, d->capG, tot) || !grow(d->dXt, d->capX, (size_t)(rows * nrhs)) ||
        !grow(d->dS0, d->capS0, (size_t)(rows * cols)) || !grow(d->dS1, d->capS1, (size_t)(rows * cols)))
        return -1;
    for (idx k = 1; k < N; ++k) {
        const Tensor& g = f.g[(size_t)((n + k) % N)];
        if (cudaMemcpyAsync(d->dG + off[(size_t)(k - 1)], g.data.data(), sizeof(double) * g.data.size(),
                            cudaMemcpyHostToDevice, s) != cudaSuccess)
            return -1;
    }
    if (cudaMemcpyAsync(d->dXt, xn_tr.a.data(), sizeof(double) * rows * nrhs, cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
        return -1;
    // subchain (tr_factors.hpp:111-119): cur (ra, p, rb) x g (rb, i, rc) -> (ra, p i, rc) is
    // out(ra p x i rc) = cur(ra p x rb) * g(rb x i rc), all column-major
    idx ra = 0, p = 0, rb = 0;
    const double* cur = device_subchain(d, f, n + 1, off, ra, p, rb);
    if (!cur) return -1;
    if (p != rows || ra * rb != cols) return -1;
    k_unfold_subchain<<<148 * 8, 256, 0, s>>>(cur, d->dA, (long long)rows, (int)ra, (int)rb);
    const dim3 tb(32, 8), tg((unsigned)((rows + 31) / 32), (unsigned)((nrhs + 31) / 32));
    k_transpose<<<tg, tb, 0, s>>>(d->dXt, d->dB, (int)nrhs, (int)rows);
    if (cudaGetLastError() != cudaSuccess) return -1;
    z = Mat(cols, nrhs);
    return factor_solve(d, rows, cols, nrhs, z.a.data(), t0);
}

// rse(x, reconstruct_full(f)) on the device (solvers.hpp:47-54, tr_factors.hpp:123-137): the
// subchain of cores 1..N-1 and X_<0> = core2 W by cuBLAS, the squared sums by k_rse_partials,
// summed on the host in block order. 0: *out set; -1: no device route (caller: host).
int device_tr_rse(const Cores& f, const Tensor& x, double* out) {
    const idx N = f.order();
    if (N < 2) return -1;
    const idx R0 = f.rank(0), R1 = f.rank(1 % N), I0 = f.dim(0);
    const idx P = x.size() / I0;
    // below ~1e7 multiply-adds the host reconstruction is faster than the round trip
    if ((double)x.size() * (double)(R0 * R1) < 1e7) return -1;
    std::lock_guard<std::mutex> lock(g_mu);
    DevLs* d = dev_ls();
    if (!d) return -1;
    std::vector<size_t> off;
    size_t tot = 0;
    for (idx k = 0; k < N; ++k) {
        off.push_back(tot);
        tot += f.g[(size_t)k].data.size();
    }
    const size_t nx = (size_t)x.size(), sub = (size_t)(P * R0 * R1);
    if (!grow(d->dG, d->capG, tot) || !grow(d->dXt, d->capX, nx) || !grow(d->dS0, d->capS0, sub) ||
        !grow(d->dS1, d->capS1, sub) || !grow(d->dY, d->capY, nx + sub) ||
        !grow(d->dC, d->capC, (size_t)(I0 * R0 * R1)) || !grow(d->dPart, d->capPart, 2 * kRseBlocks))
        return -1;
    cudaStream_t s = d->stream;
    for (idx k = 0; k < N; ++k)
        if (cudaMemcpyAsync(d->dG + off[(size_t)k], f.g[(size_t)k].data.data(),
                            sizeof(double) * f.g[(size_t)k].data.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
            return -1;
    if (cudaMemcpyAsync(d->dXt, x.data.data(), sizeof(double) * nx, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return -1;
    const std::vector<size_t> off1(off.begin() + 1, off.end());
    idx ra = 0, p = 0, rb = 0;
    const double* sc = device_subchain(d, f, 1, off1, ra, p, rb);
    if (!sc || ra != R1 || rb != R0 || p != P) return -1;
    double* w = d->dY + nx;  // W (R0 R1 x P) after the reconstruction's slot
    k_rse_operands<<<148 * 4, 256, 0, s>>>(sc, d->dG + off[0], w, d->dC, (long long)P, (int)R0, (int)R1, (int)I0);
    const double one = 1.0, zero = 0.0;
    if (d->gemm(d->bh, CUBLAS_OP_N, CUBLAS_OP_N, (int)I0, (int)P, (int)(R0 * R1), &one, d->dC, (int)I0, w,
                (int)(R0 * R1), &zero, d->dY, (int)I0) != CUBLAS_STATUS_SUCCESS)
        return -1;
    k_rse_partials<<<kRseBlocks, 256, 0, s>>>(d->dXt, d->dY, (long long)nx, d->dPart);
    std::vector<double> part(2 * kRseBlocks);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(part.data(), d->dPart, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return -1;
    double num = 0.0, den = 0.0;
    for (int b = 0; b < kRseBlocks; ++b) {
        num += part[2 * b];
        den += part[2 * b + 1];
    }
    if (!(den > 0.0)) return -1;
    *out = std::sqrt(num) / std::sqrt(den);
    return 0;
}

// Thin SVD a = U diag(s) V^T on the device (cuSOLVER gesvdj: one-sided Jacobi, as the host
// stand-in for BDCSVD, solvers.hpp:297-334), s descending, then the host svd()'s conventions: the
// left factor of the taller side zeroed where s_j = 0, and the shared sign rule (the entry of
// largest magnitude of each U column positive). 0: done; -1: no device route (caller: host).
int device_svd(const Mat& a, Mat& U, std::vector<double>& s, Mat& V) {
    const idx m = a.r, n = a.c, k = std::min(m, n);
    // below ~1e7 m n min(m, n) the host Jacobi is faster than the round trip
    if (k < 1 || m > (1 << 30) || n > (1 << 30) || (double)m * (double)n * (double)k < 1e7) return -1;
    std::lock_guard<std::mutex> lock(g_mu);
    DevLs* d = dev_ls();
    if (!d || !d->svdj) return -1;
    cudaStream_t st = d->stream;
    // A in dA, U in dS0, V in dS1, s in dtau
    if (!grow(d->dA, d->capA, (size_t)(m * n)) || !grow(d->dS0, d->capS0, (size_t)(m * k)) ||
        !grow(d->dS1, d->capS1, (size_t)(n * k)) || !grow(d->dtau, d->capT, (size_t)k))
        return -1;
    int lw = 0;
    if (d->svdj_ws(d->sh, CUSOLVER_EIG_MODE_VECTOR, 1, (int)m, (int)n, d->dA, (int)m, d->dtau, d->dS0, (int)m, d->dS1,
                   (int)n, &lw, d->svdj_params) != CUSOLVER_STATUS_SUCCESS ||
        !grow(d->dwork, d->capW, (size_t)lw))
        return -1;
    if (cudaMemcpyAsync(d->dA, a.a.data(), sizeof(double) * m * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return -1;
    if (d->svdj(d->sh, CUSOLVER_EIG_MODE_VECTOR, 1, (int)m, (int)n, d->dA, (int)m, d->dtau, d->dS0, (int)m, d->dS1,
                (int)n, d->dwork, (int)d->capW, d->dinfo, d->svdj_params) != CUSOLVER_STATUS_SUCCESS)
        return -1;
    Mat u(m, k), v(n, k);
    std::vector<double> sv((size_t)k);
    int info = 0;
    if (cudaMemcpyAsync(u.a.data(), d->dS0, sizeof(double) * m * k, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(v.a.data(), d->dS1, sizeof(double) * n * k, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(sv.data(), d->dtau, sizeof(double) * k, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&info, d->dinfo, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess || info != 0)
        return -1;
    for (idx j = 1; j < k; ++j)
        if (sv[(size_t)j] > sv[(size_t)(j - 1)]) return -1;  // the contract is descending order
    // host svd(): the columns of the taller side's factor are W(:, j) / s_j, zero when s_j = 0
    Mat& tall = (m >= n) ? u : v;
    for (idx j = 0; j < k; ++j)
        if (!(sv[(size_t)j] > 0.0))
            for (idx i = 0; i < tall.r; ++i) tall(i, j) = 0.0;
    for (idx j = 0; j < k; ++j) {
        idx arg = 0;
        for (idx i = 1; i < u.r; ++i)
            if (std::abs(u(i, j)) > std::abs(u(arg, j))) arg = i;
        if (u(arg, j) < 0.0) {
            for (idx i = 0; i < u.r; ++i) u(i, j) = -u(i, j);
            for (idx i = 0; i < v.r; ++i) v(i, j) = -v(i, j);
        }
    }
    U = std::move(u);
    V = std::move(v);
    s = std::move(sv);
    return 0;
}

}  // namespace host
}  // namespace trg
