// SPDX-License-Identifier: Apache-2.0
//
// fp64 kernels for the modes n >= 1 of the sequential projection, where the
// working tensor P^(n) is read as (left, dim, right) with left = prod K_{<n} > 1
// (tensor.hpp:112-123). Column c = l + left*r of the unfolding (tensor.hpp:133)
// holds dim elements at stride `left`; a run of consecutive columns is a
// 2-D box of the slab layout.
//
//   k_slab_sketch_f64  Y_n += X_(n) Omega_n            (sketch.hpp:80-83)
//   k_slab_ttm_f64     P^(n+1) = P^(n) x_n Q_n^T       (sketch.hpp:85)
//
// Producer warps gather tiles of CT consecutive columns x all dim rows with
// 16-byte cp.async (LDGSTS) into shared memory with row stride CT+4 doubles,
// i.e. 2*stride == 8 (mod 32) words: every mma.m8n8k4.f64 fragment load then
// touches each bank exactly twice, the minimum for 32 x 8 B (no conflicts for
// the power-of-two `left` values that a plain slab copy would hit 8-way).
// Completion is tracked with cp.async.mbarrier.arrive on a 3-stage ring; the
// consumers run DMMA; in the sketch, generator warps regenerate Omega_n for the
// next tile into fragment order (same counter-addressed reference stream).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "pipeline.cuh"

namespace trg {

namespace {

constexpr int kCons = 4;
constexpr int kProd = 2;
constexpr int kRng = 4;
constexpr size_t kBar = 256;

__device__ __forceinline__ int64_t lmin(int64_t x, int64_t y) { return x < y ? x : y; }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct SlabArgs {
    const double* x;
    int64_t left, dim, ncols, ntiles;
    int CT, stride, rows_pad, K, stages;
    FastDiv left_div;
    // sketch
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    double* partial;
    int mtiles;
    // ttm
    double* out;
    const double* q;
    int64_t ldq;
    int Tk;
};

// producer: gather tile j (CT consecutive columns, all rows) into stage s
__device__ __forceinline__ void gather_tile(const SlabArgs& a, double* stage, int64_t c0, int pt) {
    const int half = a.CT >> 1;
    const int nch = (int)a.dim * half;
    for (int ch = pt; ch < nch; ch += kProd * 32) {
        const int d = ch / half;
        const int cp = ch - d * half;
        const int64_t c = c0 + 2 * cp;
        if (c < a.ncols) {
            const uint32_t r = a.left_div.div((uint32_t)c);
            const int64_t l = c - (int64_t)r * a.left;
            cp_async16(stage + d * a.stride + 2 * cp, a.x + (int64_t)r * a.left * a.dim + d * a.left + l);
        }
    }
}

__device__ __forceinline__ int omega_idx(int c, int k, int NT) {
    return (((c >> 2) * NT + (k >> 3)) << 5) + (c & 3) + ((k & 7) << 2);
}

template <int MTILES, int NT>
__global__ void __launch_bounds__((kCons + kProd + kRng) * 32, 1) k_slab_sketch_f64(SlabArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int S = a.stages;
    const int stage_elems = a.rows_pad * a.stride;
    double* stages = reinterpret_cast<double*>(smem_raw);
    const int omega_elems = a.CT * NT * 8;
    double* omega = stages + S * stage_elems;
    uint64_t* bars = reinterpret_cast<uint64_t*>(omega + 2 * omega_elems);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + 4;
    uint64_t* full_o = bars + 8;
    uint64_t* empty_o = bars + 10;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
    for (int i = tid; i < S * stage_elems; i += blockDim.x) stages[i] = 0.0;
    for (int i = tid; i < 2 * omega_elems; i += blockDim.x) omega[i] = 0.0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_x[s], kProd * 32);
            mbar_init(&empty_x[s], kCons * 32);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full_o[b], kRng * 32);
            mbar_init(&empty_o[b], kCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp >= kCons && warp < kCons + kProd) {
        const int pt = tid - kCons * 32;
        for (int j = 0; j < nl; ++j) {
            const int s = j % S;
            mbar_wait(&empty_x[s], ((j / S) & 1) ^ 1);
            const int64_t c0 = (blockIdx.x + (int64_t)j * gridDim.x) * a.CT;
            gather_tile(a, stages + s * stage_elems, c0, pt);
            cp_async_mbar_arrive(&full_x[s]);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }
    if (warp >= kCons + kProd) {
        const int rt = tid - (kCons + kProd) * 32;
        const int CT = a.CT;
        const int npmax = CT / 2 + 1;
        for (int j = 0; j < nl; ++j) {
            const int b = j & 1;
            mbar_wait(&empty_o[b], ((j >> 1) & 1) ^ 1);
            const int64_t c0 = (blockIdx.x + (int64_t)j * gridDim.x) * CT;
            const int64_t ncol = lmin(CT, a.ncols - c0);
            double* O = omega + b * omega_elems;
            for (int it = rt; it < a.K * npmax; it += kRng * 32) {
                const int k = it / npmax;
                const int jj = it - k * npmax;
                const uint64_t s0 = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)k;
                const uint64_t p = (s0 >> 1) + (uint64_t)jj;
                if (p > ((s0 + (uint64_t)CT - 1ull) >> 1)) continue;
                double z0, z1;
                gauss_pair(a.seed, p, z0, z1);
                const int64_t cc = (int64_t)(2ull * p - s0);
                if (cc >= 0 && cc < CT) O[omega_idx((int)cc, k, NT)] = cc < ncol ? z0 : 0.0;
                if (cc + 1 >= 0 && cc + 1 < CT) O[omega_idx((int)cc + 1, k, NT)] = cc + 1 < ncol ? z1 : 0.0;
            }
            mbar_arrive(&full_o[b]);
        }
        return;
    }
    // consumers: warp w takes k-steps t = w, w + 4, ... of each tile, full-height accumulators
    double acc[MTILES][NT][2];
#pragma unroll
    for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
    const int q = lane >> 2, r = lane & 3;
    const int ksteps = a.CT >> 2;
    for (int j = 0; j < nl; ++j) {
        const int s = j % S;
        const int b = j & 1;
        mbar_wait(&full_x[s], (j / S) & 1);
        mbar_wait(&full_o[b], (j >> 1) & 1);
        const double* X = stages + s * stage_elems + q * a.stride + r;
        const double* O = omega + b * omega_elems;
        for (int t = warp; t < ksteps; t += kCons) {
            double bv[NT];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) bv[jn] = O[((t * NT + jn) << 5) + lane];
#pragma unroll
            for (int mt = 0; mt < MTILES; ++mt) {
                if (mt < a.mtiles) {
                    const double av = X[8 * mt * a.stride + 4 * t];
#pragma unroll
                    for (int jn = 0; jn < NT; ++jn) dmma884(acc[mt][jn][0], acc[mt][jn][1], av, bv[jn]);
                }
            }
        }
        mbar_arrive(&empty_x[s]);
        mbar_arrive(&empty_o[b]);
    }
    // fixed-order reduction of the four warps' partials through shared memory
    asm volatile("bar.sync 1, %0;" ::"n"(kCons * 32));
    double* red = stages;  // reuse stage 0 (all copies consumed)
    const int ld = 8 * MTILES;
    for (int w = 0; w < kCons; ++w) {
        if (warp == w) {
#pragma unroll
            for (int mt = 0; mt < MTILES; ++mt)
#pragma unroll
                for (int jn = 0; jn < NT; ++jn) {
                    const int row = 8 * mt + q, col = 8 * jn + 2 * r;
                    double* p0 = red + row + ld * col;
                    double* p1 = p0 + ld;
                    *p0 = (w == 0 ? 0.0 : *p0) + acc[mt][jn][0];
                    *p1 = (w == 0 ? 0.0 : *p1) + acc[mt][jn][1];
                }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kCons * 32));
    }
    double* outp = a.partial + (int64_t)blockIdx.x * a.dim * a.K;
    for (int e = tid; e < a.dim * a.K; e += kCons * 32) {
        const int k = e / (int)a.dim;
        const int d = e - k * (int)a.dim;
        outp[d + a.dim * k] = red[d + ld * k];
    }
}

template <int NT>
__global__ void __launch_bounds__((kCons + kProd) * 32, 1) k_slab_ttm_f64(SlabArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int S = a.stages;
    const int stage_elems = a.rows_pad * a.stride;
    double* stages = reinterpret_cast<double*>(smem_raw);
    double* Bf = stages + S * stage_elems;
    const int bf_elems = a.Tk * NT * 32;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bf + bf_elems);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + 4;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
    for (int i = tid; i < S * stage_elems; i += blockDim.x) stages[i] = 0.0;
    for (int i = tid; i < bf_elems; i += blockDim.x) {
        const int t = i / (NT * 32);
        const int jn = (i >> 5) % NT;
        const int ln = i & 31;
        const int64_t d = 4 * t + (ln & 3);
        const int o = 8 * jn + (ln >> 2);
        Bf[i] = (d < a.dim && o < a.K) ? a.q[d + a.ldq * o] : 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_x[s], kProd * 32);
            mbar_init(&empty_x[s], kCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp >= kCons) {
        const int pt = tid - kCons * 32;
        for (int j = 0; j < nl; ++j) {
            const int s = j % S;
            mbar_wait(&empty_x[s], ((j / S) & 1) ^ 1);
            const int64_t c0 = (blockIdx.x + (int64_t)j * gridDim.x) * a.CT;
            gather_tile(a, stages + s * stage_elems, c0, pt);
            cp_async_mbar_arrive(&full_x[s]);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }
    const int q = lane >> 2, r = lane & 3;
    const int m_per_warp = a.CT / (8 * kCons);  // 2 for CT = 64, 1 for CT = 32
    for (int j = 0; j < nl; ++j) {
        const int s = j % S;
        mbar_wait(&full_x[s], (j / S) & 1);
        const double* X = stages + s * stage_elems + r * a.stride + q;
        double acc[2][NT][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
        const int cbase = 8 * m_per_warp * warp;
#pragma unroll 2
        for (int t = 0; t < a.Tk; ++t) {
            double bv[NT];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) bv[jn] = Bf[((t * NT + jn) << 5) + lane];
            const double* xr = X + 4 * t * a.stride + cbase;
            const double a0 = xr[0];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) dmma884(acc[0][jn][0], acc[0][jn][1], a0, bv[jn]);
            if (m_per_warp > 1) {
                const double a1 = xr[8];
#pragma unroll
                for (int jn = 0; jn < NT; ++jn) dmma884(acc[1][jn][0], acc[1][jn][1], a1, bv[jn]);
            }
        }
        mbar_arrive(&empty_x[s]);
        const int64_t c0 = (blockIdx.x + (int64_t)j * gridDim.x) * a.CT;
        for (int mt = 0; mt < m_per_warp; ++mt) {
            const int64_t c = c0 + cbase + 8 * mt + q;
            if (c >= a.ncols) continue;
            const uint32_t rr = a.left_div.div((uint32_t)c);
            const int64_t l = c - (int64_t)rr * a.left;
            double* dst = a.out + (int64_t)rr * a.left * a.K + l;
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                const int o = 8 * jn + 2 * r;
                if (o < a.K) dst[a.left * o] = acc[mt][jn][0];
                if (o + 1 < a.K) dst[a.left * (o + 1)] = acc[mt][jn][1];
            }
        }
    }
}

int nt_of(int K) {
    const int nt = (K + 7) / 8;
    return nt <= 1 ? 1 : nt <= 2 ? 2 : nt <= 4 ? 4 : 8;
}

constexpr size_t kBudget = 224 * 1024;

// pick CT / stages for a tile of `rows_pad` rows; returns false if nothing fits
bool pick(int64_t rows_pad, size_t extra_bytes, int& CT, int& stages) {
    for (int ct : {64, 32}) {
        const size_t stage = (size_t)rows_pad * (ct + 4) * 8;
        for (int s : {3, 2}) {
            if (s * stage + extra_bytes + kBar <= kBudget) {
                CT = ct;
                stages = s;
                return true;
            }
        }
    }
    return false;
}

}  // namespace

bool slab_sketch_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols) {
    if (dtype != F64 || left < 2 || (left & 1) || K > 64 || dim > 128 || ncols >= (int64_t(1) << 32)) return false;
    const int mt = (int)((dim + 7) / 8);
    int CT, S;
    return pick(8 * mt, 2 * 64 * nt_of(K) * 8 * 8, CT, S);
}

bool slab_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t odim, int64_t ncols) {
    if (dtype != F64 || left < 2 || (left & 1) || odim > 64 || ncols >= (int64_t(1) << 32)) return false;
    const int Tk = (int)((dim + 3) / 4);
    int CT, S;
    return pick(4 * Tk, (size_t)Tk * nt_of((int)odim) * 32 * 8, CT, S);
}

void launch_slab_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                        cudaStream_t s) {
    SlabArgs a{};
    a.x = reinterpret_cast<const double*>(x);
    a.left = p.left;
    a.dim = p.dim;
    a.ncols = p.left * p.right;
    a.K = p.K;
    a.mtiles = (int)((p.dim + 7) / 8);
    a.rows_pad = 8 * a.mtiles;
    const int NT = nt_of(p.K);
    pick(a.rows_pad, 2 * 64 * NT * 8 * 8, a.CT, a.stages);
    a.stride = a.CT + 4;
    a.ntiles = (a.ncols + a.CT - 1) / a.CT;
    a.left_div = FastDiv((uint32_t)p.left);
    a.seed = p.seed;
    a.D = p.D;
    a.rows_glob = p.rows_glob;
    a.col_off = p.col_off;
    a.partial = partial;
    const size_t smem = ((size_t)a.stages * a.rows_pad * a.stride + 2 * (size_t)a.CT * NT * 8) * 8 + kBar;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    const int threads = (kCons + kProd + kRng) * 32;
#define TRG_SL(MTV, NTV)                                                                                   \
    do {                                                                                                   \
        allow_smem(k_slab_sketch_f64<MTV, NTV>, smem);                                                    \
        k_slab_sketch_f64<MTV, NTV><<<grid, threads, smem, s>>>(a);                                        \
    } while (0)
#define TRG_SL_NT(MTV)                   \
    switch (NT) {                        \
        case 1: TRG_SL(MTV, 1); break;   \
        case 2: TRG_SL(MTV, 2); break;   \
        case 4: TRG_SL(MTV, 4); break;   \
        default: TRG_SL(MTV, 8); break;  \
    }
    if (a.mtiles <= 4) {
        TRG_SL_NT(4)
    } else if (a.mtiles <= 8) {
        TRG_SL_NT(8)
    } else if (a.mtiles <= 13) {
        TRG_SL_NT(13)
    } else {
        TRG_SL_NT(16)
    }
#undef TRG_SL_NT
#undef TRG_SL
    launch_reduce_partials(partial, grid, p.dim * p.K, y, s);
}

void launch_slab_ttm(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, int num_sms,
                     cudaStream_t s) {
    SlabArgs a{};
    a.x = reinterpret_cast<const double*>(in);
    a.out = reinterpret_cast<double*>(out);
    a.q = q;
    a.ldq = ldq;
    a.left = p.left;
    a.dim = p.dim;
    a.ncols = p.left * p.right;
    a.K = (int)p.odim;
    a.Tk = (int)((p.dim + 3) / 4);
    a.rows_pad = 4 * a.Tk;
    const int NT = nt_of(a.K);
    pick(a.rows_pad, (size_t)a.Tk * NT * 32 * 8, a.CT, a.stages);
    a.stride = a.CT + 4;
    a.ntiles = (a.ncols + a.CT - 1) / a.CT;
    a.left_div = FastDiv((uint32_t)p.left);
    const size_t smem = ((size_t)a.stages * a.rows_pad * a.stride + (size_t)a.Tk * NT * 32) * 8 + kBar;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    const int threads = (kCons + kProd) * 32;
    switch (NT) {
        case 1:
            allow_smem(k_slab_ttm_f64<1>, smem);
            k_slab_ttm_f64<1><<<grid, threads, smem, s>>>(a);
            break;
        case 2:
            allow_smem(k_slab_ttm_f64<2>, smem);
            k_slab_ttm_f64<2><<<grid, threads, smem, s>>>(a);
            break;
        case 4:
            allow_smem(k_slab_ttm_f64<4>, smem);
            k_slab_ttm_f64<4><<<grid, threads, smem, s>>>(a);
            break;
        default:
            allow_smem(k_slab_ttm_f64<8>, smem);
            k_slab_ttm_f64<8><<<grid, threads, smem, s>>>(a);
            break;
    }
}

}  // namespace trg
