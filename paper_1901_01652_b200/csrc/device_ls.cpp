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
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
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
    cusolverDnHandle_t sh = nullptr;
    cublasHandle_t bh = nullptr;
    cudaStream_t stream = nullptr;
    int device = -1;
    // device buffers, grown on demand: A (m x n), B (m x nrhs), tau, workspace, info
    double *dA = nullptr, *dB = nullptr, *dtau = nullptr, *dwork = nullptr;
    int* dinfo = nullptr;
    size_t capA = 0, capB = 0, capT = 0, capW = 0;
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
              sym(lb, "cublasDtrsm_v2", d.trsm)))
            return;
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

// 0: solved into x (n x nrhs); 1: rank-deficient by the host route's cutoff (caller: ridge);
// -1: no device route (caller: host QR)
int device_ls_qr(const double* a, idx m, idx n, const double* b, idx nrhs, double* x) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    // small systems stay on the host: below ~1e6 m n^2 the transfers and launches cost more than the
    // factorisation (C1's 100 x 25 systems: 3.5 ms host against 25 ms device per decompose)
    if (m < n || m > (1 << 30) || n < 1 || nrhs < 1 || (double)m * (double)n * (double)n < 1e6) return -1;
    DevLs* d = dev_ls();
    if (!d) return -1;
    const int M = (int)m, Nn = (int)n, R = (int)nrhs;
    int lw1 = 0, lw2 = 0;
    if (!grow(d->dA, d->capA, (size_t)m * n) || !grow(d->dB, d->capB, (size_t)m * nrhs) ||
        !grow(d->dtau, d->capT, (size_t)n))
        return -1;
    if (d->geqrf_ws(d->sh, M, Nn, d->dA, M, &lw1) != CUSOLVER_STATUS_SUCCESS ||
        d->ormqr_ws(d->sh, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, M, R, Nn, d->dA, M, d->dtau, d->dB, M, &lw2) !=
            CUSOLVER_STATUS_SUCCESS)
        return -1;
    if (!grow(d->dwork, d->capW, (size_t)std::max(lw1, lw2))) return -1;
    cudaStream_t s = d->stream;
    if (cudaMemcpyAsync(d->dA, a, sizeof(double) * m * n, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(d->dB, b, sizeof(double) * m * nrhs, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return -1;
    if (d->geqrf(d->sh, M, Nn, d->dA, M, d->dtau, d->dwork, (int)d->capW, d->dinfo) != CUSOLVER_STATUS_SUCCESS)
        return -1;
    // |R_ii|: the diagonal of the factored A (stride m + 1)
    std::vector<double> diag((size_t)n);
    if (cudaMemcpy2DAsync(diag.data(), sizeof(double), d->dA, sizeof(double) * (m + 1), sizeof(double), (size_t)n,
                          cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return -1;
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
    return 0;
}

}  // namespace host
}  // namespace trg
