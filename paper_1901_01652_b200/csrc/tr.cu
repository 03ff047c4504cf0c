// SPDX-License-Identifier: Apache-2.0
//
// TR-model kernels: subchain contraction, fused reconstruction / RSE (K8),
// synthesis (K9) and small elementwise helpers.
//
// Reference: reconstruct_full (tr_factors.hpp:123-137) builds
// X_<0> = G_{0,(2)} (G_{!=0,<2>})^T and rse (solvers.hpp:47-54) then reads
// both |X| tensors again. Here the subchain S = G_1 o ... o G_{N-1}
// (tr_factors.hpp:111-119, chain_contract :92-102) is contracted once on
// device and one tiled fp64 GEMM computes Xhat(i0, p) = sum_{a,b}
// G0(a, i0, b) S(b, p, a) with the (x - xhat)^2 and x^2 sums fused into its
// epilogue, so Xhat is never written (RSE) — or is written as X (synthesis).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace trg {

namespace {

__global__ void k_chain(const double* __restrict__ a, int64_t ra, int64_t p, int64_t rb, const double* __restrict__ g,
                        int64_t ii, int64_t rc, double* __restrict__ out) {
    const int64_t n = ra * p * ii * rc;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        // out index e = x + Ra*(q + P*i + P*I*c) with x < Ra, q < P
        const int64_t x = e % ra;
        int64_t rest = e / ra;
        const int64_t q = rest % p;
        rest /= p;
        const int64_t i = rest % ii;
        const int64_t c = rest / ii;
        double s = 0.0;
        for (int64_t b = 0; b < rb; ++b) s = fma(a[x + ra * (q + p * b)], g[b + rb * (i + ii * c)], s);
        out[e] = s;
    }
}

constexpr int RT = 64;   // rows (i0) per CTA tile
constexpr int PT = 64;   // columns (p) per CTA tile
constexpr int QC = 16;   // contraction chunk over b

template <typename T, bool WRITE>
__global__ void __launch_bounds__(256) k_recon(const double* __restrict__ g0, const double* __restrict__ S, T* x,
                                               int64_t I0, int64_t P, int64_t R0, int64_t R1,
                                               double* __restrict__ block_sums) {
    __shared__ double As[QC][RT];
    __shared__ double Bs[QC][PT + 1];
    __shared__ double red[2][8];
    const int tid = threadIdx.x;
    const int ti = tid & 15, tp = tid >> 4;
    const int64_t i_base = (int64_t)blockIdx.y * RT;
    const int64_t p_base = (int64_t)blockIdx.x * PT;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    for (int64_t a = 0; a < R0; ++a) {
        for (int64_t b0 = 0; b0 < R1; b0 += QC) {
            const int nb = (R1 - b0) < QC ? (int)(R1 - b0) : QC;
            __syncthreads();
            // A(i0, (a,b)) = G0[a + R0*(i0 + I0*b)]
            for (int e = tid; e < QC * RT; e += 256) {
                const int bb = e / RT, ii = e - bb * RT;
                const int64_t i0 = i_base + ii;
                As[bb][ii] = (bb < nb && i0 < I0) ? g0[a + R0 * (i0 + I0 * (b0 + bb))] : 0.0;
            }
            // B((a,b), p) = S[b + R1*(p + P*a)], b fastest (coalesced)
            for (int e = tid; e < QC * PT; e += 256) {
                const int pp = e / QC, bb = e - pp * QC;
                const int64_t pc = p_base + pp;
                Bs[bb][pp] = (bb < nb && pc < P) ? S[(b0 + bb) + R1 * (pc + P * a)] : 0.0;
            }
            __syncthreads();
#pragma unroll 4
            for (int bb = 0; bb < QC; ++bb) {
                double av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) av[i] = As[bb][ti + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[j] = Bs[bb][tp + 16 * j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
        }
    }
    double se = 0.0, sx = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t pc = p_base + tp + 16 * j;
        if (pc >= P) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t i0 = i_base + ti + 16 * i;
            if (i0 >= I0) continue;
            T* px = x + i0 + I0 * pc;
            if (WRITE) {
                *px = T(acc[i][j]);
            } else {
                const double xv = (double)*px;
                const double d = xv - acc[i][j];
                se = fma(d, d, se);
                sx = fma(xv, xv, sx);
            }
        }
    }
    if (!WRITE) {
        for (int o = 16; o > 0; o >>= 1) {
            se += __shfl_xor_sync(0xffffffffu, se, o);
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
        }
        if ((tid & 31) == 0) {
            red[0][tid >> 5] = se;
            red[1][tid >> 5] = sx;
        }
        __syncthreads();
        if (tid == 0) {
            double a0 = 0.0, a1 = 0.0;
            for (int w = 0; w < 8; ++w) {
                a0 += red[0][w];
                a1 += red[1][w];
            }
            const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
            block_sums[2 * bid] = a0;
            block_sums[2 * bid + 1] = a1;
        }
    }
}

__global__ void k_sum_pairs(const double* __restrict__ bs, int n, double* out) {
    __shared__ double r0[256], r1[256];
    double a = 0.0, b = 0.0;
    // fixed assignment of blocks to threads + fixed tree => deterministic
    for (int i = threadIdx.x; i < n; i += 256) {
        a += bs[2 * i];
        b += bs[2 * i + 1];
    }
    r0[threadIdx.x] = a;
    r1[threadIdx.x] = b;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] += r0[threadIdx.x + s];
            r1[threadIdx.x] += r1[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = r0[0];
        out[1] = r1[0];
    }
}

template <typename T>
__global__ void k_noise_norms(const T* __restrict__ x, int64_t n, uint64_t seed, uint64_t off,
                              double* __restrict__ bs) {
    double sx = 0.0, se = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double xv = (double)x[i];
        const double e = gauss_draw<double>(seed, off + (uint64_t)i);
        sx = fma(xv, xv, sx);
        se = fma(e, e, se);
    }
    __shared__ double r0[256], r1[256];
    r0[threadIdx.x] = sx;
    r1[threadIdx.x] = se;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] += r0[threadIdx.x + s];
            r1[threadIdx.x] += r1[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bs[2 * blockIdx.x] = r0[0];
        bs[2 * blockIdx.x + 1] = r1[0];
    }
}

template <typename T>
__global__ void k_add_noise(T* x, int64_t n, uint64_t seed, uint64_t off, double alpha) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = T((double)x[i] + alpha * gauss_draw<double>(seed, off + (uint64_t)i));
}

template <typename T>
__global__ void k_minmax(const T* __restrict__ x, int64_t n, double* __restrict__ bs) {
    double lo = 1e308, hi = -1e308;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)x[i];
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    __shared__ double r0[256], r1[256];
    r0[threadIdx.x] = lo;
    r1[threadIdx.x] = hi;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] = fmin(r0[threadIdx.x], r0[threadIdx.x + s]);
            r1[threadIdx.x] = fmax(r1[threadIdx.x], r1[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bs[2 * blockIdx.x] = r0[0];
        bs[2 * blockIdx.x + 1] = r1[0];
    }
}

template <typename T>
__global__ void k_affine(T* x, int64_t n, double a, double b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = T(a * (double)x[i] + b);
}

template <typename Ti, typename To>
__global__ void k_convert(const Ti* __restrict__ in, To* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = To(in[i]);
}

__global__ void k_scatter_rows(const double* __restrict__ in, int64_t rows, int k, int64_t lo, int64_t m,
                               double* __restrict__ out) {
    const int64_t n = m * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / m, r = e - c * m;
        out[e] = (r >= lo && r < lo + rows) ? in[(r - lo) + rows * c] : 0.0;
    }
}

int grid_for(int64_t n, int threads = 256, int cap = 8192) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

}  // namespace

void launch_chain(const double* a, int64_t ra, int64_t p, int64_t rb, const double* g, int64_t i, int64_t rc,
                  double* out, cudaStream_t s) {
    const int64_t n = ra * p * i * rc;
    k_chain<<<grid_for(n), 256, 0, s>>>(a, ra, p, rb, g, i, rc, out);
}

void plan_recon(ReconPlan& p, int) {
    p.threads = 256;
    p.grid_x = (int)((p.P + PT - 1) / PT);
    p.grid_y = (int)((p.I0 + RT - 1) / RT);
    p.nblocks = p.grid_x * p.grid_y;
    p.smem = 0;
}

void launch_recon(const ReconPlan& p, const double* g0, const double* S, void* x, int write_mode, double* block_sums,
                  cudaStream_t s) {
    dim3 grid(p.grid_x, p.grid_y);
    if (p.dtype == F64) {
        if (write_mode)
            k_recon<double, true><<<grid, 256, 0, s>>>(g0, S, (double*)x, p.I0, p.P, p.R0, p.R1, block_sums);
        else
            k_recon<double, false><<<grid, 256, 0, s>>>(g0, S, (double*)x, p.I0, p.P, p.R0, p.R1, block_sums);
    } else {
        if (write_mode)
            k_recon<float, true><<<grid, 256, 0, s>>>(g0, S, (float*)x, p.I0, p.P, p.R0, p.R1, block_sums);
        else
            k_recon<float, false><<<grid, 256, 0, s>>>(g0, S, (float*)x, p.I0, p.P, p.R0, p.R1, block_sums);
    }
}

void launch_sum_pairs(const double* block_sums, int nblocks, double* out, cudaStream_t s) {
    k_sum_pairs<<<1, 256, 0, s>>>(block_sums, nblocks, out);
}

void launch_noise_norms(const void* x, int dtype, int64_t n, uint64_t seed, uint64_t off, double* block_sums,
                        int nblocks, cudaStream_t s) {
    if (dtype == F64)
        k_noise_norms<double><<<nblocks, 256, 0, s>>>((const double*)x, n, seed, off, block_sums);
    else
        k_noise_norms<float><<<nblocks, 256, 0, s>>>((const float*)x, n, seed, off, block_sums);
}

void launch_add_noise(void* x, int dtype, int64_t n, uint64_t seed, uint64_t off, double alpha, cudaStream_t s) {
    if (dtype == F64)
        k_add_noise<double><<<grid_for(n), 256, 0, s>>>((double*)x, n, seed, off, alpha);
    else
        k_add_noise<float><<<grid_for(n), 256, 0, s>>>((float*)x, n, seed, off, alpha);
}

void launch_minmax(const void* x, int dtype, int64_t n, double* block_mm, int nblocks, cudaStream_t s) {
    if (dtype == F64)
        k_minmax<double><<<nblocks, 256, 0, s>>>((const double*)x, n, block_mm);
    else
        k_minmax<float><<<nblocks, 256, 0, s>>>((const float*)x, n, block_mm);
}

void launch_affine(void* x, int dtype, int64_t n, double a, double b, cudaStream_t s) {
    if (dtype == F64)
        k_affine<double><<<grid_for(n), 256, 0, s>>>((double*)x, n, a, b);
    else
        k_affine<float><<<grid_for(n), 256, 0, s>>>((float*)x, n, a, b);
}

void launch_convert(const void* in, int in_dt, void* out, int out_dt, int64_t n, cudaStream_t s) {
    const int g = grid_for(n);
    if (in_dt == F64 && out_dt == F64)
        k_convert<double, double><<<g, 256, 0, s>>>((const double*)in, (double*)out, n);
    else if (in_dt == F64)
        k_convert<double, float><<<g, 256, 0, s>>>((const double*)in, (float*)out, n);
    else if (out_dt == F64)
        k_convert<float, double><<<g, 256, 0, s>>>((const float*)in, (double*)out, n);
    else
        k_convert<float, float><<<g, 256, 0, s>>>((const float*)in, (float*)out, n);
}

void launch_scatter_rows(const double* in, int64_t rows, int k, int64_t lo, int64_t m, double* out, cudaStream_t s) {
    k_scatter_rows<<<grid_for(m * k), 256, 0, s>>>(in, rows, k, lo, m, out);
}

// ---- loopback communicator: rank-ordered reduction of same-device buffers
struct RankBufs {
    const void* p[kMaxLoopbackRanks];
};

template <typename T>
__global__ void k_rank_reduce(RankBufs b, int nranks, int64_t n, int op, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T acc = static_cast<const T*>(b.p[0])[i];
        for (int r = 1; r < nranks; ++r) {
            const T v = static_cast<const T*>(b.p[r])[i];
            acc = op == 0 ? acc + v : (v > acc ? v : acc);
        }
        out[i] = acc;
    }
}

void launch_rank_reduce(const void* const* bufs, int nranks, size_t count, int dtype, int op, void* out,
                        cudaStream_t s) {
    RankBufs b{};
    for (int r = 0; r < nranks; ++r) b.p[r] = bufs[r];
    if (dtype == F64)
        k_rank_reduce<double><<<grid_for((int64_t)count), 256, 0, s>>>(b, nranks, (int64_t)count, op, (double*)out);
    else
        k_rank_reduce<float><<<grid_for((int64_t)count), 256, 0, s>>>(b, nranks, (int64_t)count, op, (float*)out);
}

}  // namespace trg
