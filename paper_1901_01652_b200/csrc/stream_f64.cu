// SPDX-License-Identifier: Apache-2.0
//
// fp64 streaming kernels for the compulsory full passes over X (mode 0, the
// unfolding X_(0) is the raw buffer viewed as I_0 x L column-major):
//
//   k_sketch_l1_f64  Y_0 = X_(0) Omega_0             (sketch.hpp:80-83)
//   k_ttm_l1_f64     P^(1) = X x_0 Q_0^T            (sketch.hpp:85, tensor.hpp:193-207)
//
// Both are persistent warp-specialised kernels: one producer thread streams
// contiguous tiles of whole mode-0 fibres into a 3-stage shared-memory ring
// with TMA bulk copies (cp.async.bulk + mbarrier complete_tx, L2 evict_first),
// consumer warps run fp64 tensor-core MMAs (mma.m8n8k4.f64 -> DMMA) on them,
// and in the sketch four generator warps regenerate the reference Gaussian
// test matrix for the next tile (SplitMix64 + Box-Muller by stream index)
// straight into MMA-fragment order while the MMAs run. fp64 is kept
// end to end because the reference is fp64 and the parity bound is 1e-10.
#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "pipeline.cuh"

namespace trg {

namespace {

constexpr int kStages = 3;
constexpr int kCons = 4;  // consumer warps
constexpr int kRng = 8;   // Omega generator warps (sketch)
constexpr int kPad = 8;   // zeroed doubles after each stage (A rows may overrun by < 8)
constexpr size_t kBarBytes = 256;  // room for the mbarriers after the buffers

struct SkArgs {
    const double* x;
    int64_t dim, ncols, ntiles, rows_glob, col_off;
    int K, CT, mtiles;
    uint64_t seed, D;
    double* partial;
};

__device__ __forceinline__ int64_t imin64(int64_t x, int64_t y) { return x < y ? x : y; }

__device__ __forceinline__ int omega_idx(int c, int k, int NT) {
    return (((c >> 2) * NT + (k >> 3)) << 5) + (c & 3) + ((k & 7) << 2);
}

template <int MTW, int NT>
__global__ void __launch_bounds__((kCons + kRng + 1) * 32, 1) k_sketch_l1_f64(SkArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int CT = a.CT;
    const int64_t dim = a.dim;
    const int stage_elems = (int)(CT * dim) + kPad;
    double* stages = reinterpret_cast<double*>(smem_raw);
    const int omega_elems = CT * NT * 8;
    double* omega = stages + kStages * stage_elems;
    uint64_t* bars = reinterpret_cast<uint64_t*>(omega + 2 * omega_elems);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + kStages;
    uint64_t* full_o = bars + 2 * kStages;
    uint64_t* empty_o = bars + 2 * kStages + 2;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

    for (int i = tid; i < kStages * stage_elems; i += blockDim.x) stages[i] = 0.0;
    for (int i = tid; i < 2 * omega_elems; i += blockDim.x) omega[i] = 0.0;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_x[s], 1);
            mbar_init(&empty_x[s], kCons * 32);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full_o[b], kRng * 32);
            mbar_init(&empty_o[b], kCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCons + kRng) {
        // ---------------- producer: TMA bulk copies of CT whole columns
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int j = 0; j < nl; ++j) {
                const int s = j % kStages;
                mbar_wait(&empty_x[s], ((j / kStages) & 1) ^ 1);
                const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
                const int64_t c0 = t * CT;
                const int64_t ncol = imin64(CT, a.ncols - c0);
                const uint32_t bytes = (uint32_t)(ncol * dim * 8);
                mbar_arrive_expect_tx(&full_x[s], bytes);
                bulk_g2s(stages + s * stage_elems, a.x + c0 * dim, bytes, &full_x[s], pol);
            }
        }
        return;
    }
    if (warp >= kCons) {
        // ---------------- generator warps: Omega tile in B-fragment order
        const int rt = tid - kCons * 32;
        const int npmax = CT / 2 + 1;
        for (int j = 0; j < nl; ++j) {
            const int b = j & 1;
            mbar_wait(&empty_o[b], ((j >> 1) & 1) ^ 1);
            const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
            const int64_t c0 = t * CT;
            const int64_t ncol = imin64(CT, a.ncols - c0);
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
    // ---------------- consumer warps: Y(d, k) += sum_c X(d, c) Omega(c, k)
    // Warp w takes k-steps t = w, w + kCons, ... of every tile with full-height
    // accumulators, so the work is balanced whatever dim is.
    double acc[MTW][NT][2];
#pragma unroll
    for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
    const int q = lane >> 2, r = lane & 3;
    for (int j = 0; j < nl; ++j) {
        const int s = j % kStages;
        const int b = j & 1;
        mbar_wait(&full_x[s], (j / kStages) & 1);
        mbar_wait(&full_o[b], (j >> 1) & 1);
        const double* X = stages + s * stage_elems + r * dim + q;
        const double* O = omega + b * omega_elems;
        for (int t = warp; t < CT / 4; t += kCons) {
            double bv[NT];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) bv[jn] = O[((t * NT + jn) << 5) + lane];
            const double* xrow = X + 4 * t * dim;
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) {
                if (mt < a.mtiles) {
                    const double av = xrow[8 * mt];
#pragma unroll
                    for (int jn = 0; jn < NT; ++jn) dmma884(acc[mt][jn][0], acc[mt][jn][1], av, bv[jn]);
                }
            }
        }
        mbar_arrive(&empty_x[s]);
        mbar_arrive(&empty_o[b]);
    }
    // fixed-order reduction of the consumer warps through (consumed) stage 0
    asm volatile("bar.sync 1, %0;" ::"n"(kCons * 32));
    double* red = stages;
    const int ld = 8 * MTW;
    for (int w = 0; w < kCons; ++w) {
        if (warp == w) {
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
                for (int jn = 0; jn < NT; ++jn) {
                    double* p0 = red + (8 * mt + q) + ld * (8 * jn + 2 * r);
                    *p0 = (w == 0 ? 0.0 : *p0) + acc[mt][jn][0];
                    p0[ld] = (w == 0 ? 0.0 : p0[ld]) + acc[mt][jn][1];
                }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kCons * 32));
    }
    double* out = a.partial + (int64_t)blockIdx.x * dim * a.K;
    for (int e = tid; e < dim * a.K; e += kCons * 32) {
        const int k = e / (int)dim;
        const int d = e - k * (int)dim;
        out[d + dim * k] = red[d + ld * k];
    }
}

struct TtmArgs {
    const double* x;
    double* out;
    const double* q;  // Q (ldq x K column-major): out(m, o) = sum_d x(m, d) Q(d, o)
    int64_t dim, rows, ntiles, ldq;
    int K, MT, Tk;
};

template <int NT>
__global__ void __launch_bounds__((kCons + 1) * 32, 1) k_ttm_l1_f64(TtmArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t dim = a.dim;
    const int MT = a.MT;
    const int stage_elems = (int)(MT * dim) + kPad;
    double* stages = reinterpret_cast<double*>(smem_raw);
    double* Bf = stages + kStages * stage_elems;
    const int bf_elems = a.Tk * NT * 32;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bf + bf_elems);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + kStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

    for (int i = tid; i < kStages * stage_elems; i += blockDim.x) stages[i] = 0.0;
    for (int i = tid; i < bf_elems; i += blockDim.x) {
        const int t = i / (NT * 32);
        const int jn = (i >> 5) % NT;
        const int ln = i & 31;
        const int64_t d = 4 * t + (ln & 3);
        const int o = 8 * jn + (ln >> 2);
        Bf[i] = (d < dim && o < a.K) ? a.q[d + a.ldq * o] : 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_x[s], 1);
            mbar_init(&empty_x[s], kCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCons) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int j = 0; j < nl; ++j) {
                const int s = j % kStages;
                mbar_wait(&empty_x[s], ((j / kStages) & 1) ^ 1);
                const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
                const int64_t m0 = t * MT;
                const int64_t nrow = imin64(MT, a.rows - m0);
                const uint32_t bytes = (uint32_t)(nrow * dim * 8);
                mbar_arrive_expect_tx(&full_x[s], bytes);
                bulk_g2s(stages + s * stage_elems, a.x + m0 * dim, bytes, &full_x[s], pol);
            }
        }
        return;
    }
    const int q = lane >> 2, r = lane & 3;
    for (int j = 0; j < nl; ++j) {
        const int s = j % kStages;
        mbar_wait(&full_x[s], (j / kStages) & 1);
        const double* X = stages + s * stage_elems;
        double acc[2][NT][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
        const double* x0 = X + (16 * warp + q) * dim + r;
        const double* x1 = x0 + 8 * dim;
#pragma unroll 4
        for (int t = 0; t < a.Tk; ++t) {
            double bv[NT];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) bv[jn] = Bf[((t * NT + jn) << 5) + lane];
            const double a0 = x0[4 * t], a1 = x1[4 * t];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                dmma884(acc[0][jn][0], acc[0][jn][1], a0, bv[jn]);
                dmma884(acc[1][jn][0], acc[1][jn][1], a1, bv[jn]);
            }
        }
        mbar_arrive(&empty_x[s]);
        const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
        const int64_t m0 = t * MT;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const int64_t m = m0 + 16 * warp + 8 * mt + q;
            if (m >= a.rows) continue;
            double* dst = a.out + m * a.K;
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                const int o = 8 * jn + 2 * r;
                if (o + 1 < a.K && !(a.K & 1)) {
                    *reinterpret_cast<double2*>(dst + o) = make_double2(acc[mt][jn][0], acc[mt][jn][1]);
                } else {
                    if (o < a.K) dst[o] = acc[mt][jn][0];
                    if (o + 1 < a.K) dst[o + 1] = acc[mt][jn][1];
                }
            }
        }
    }
}

int nt_for(int K) {
    const int nt = (K + 7) / 8;
    return nt <= 1 ? 1 : nt <= 2 ? 2 : nt <= 4 ? 4 : 8;
}

template <typename KernelT>
void set_smem(KernelT k, size_t smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

constexpr size_t kSmemBudget = 220 * 1024;

}  // namespace

// ---------------------------------------------------------------- sketch
bool stream_sketch_ok(int dtype, int64_t left, int64_t dim, int K) {
    if (dtype != F64 || left != 1 || (dim & 1) || K > 64 || dim > 128) return false;
    const int CT = dim <= 112 ? 64 : 32;
    const size_t smem = (kStages * (size_t)(CT * dim + kPad) + 2 * (size_t)CT * nt_for(K) * 8) * 8 + kBarBytes;
    return smem <= kSmemBudget;
}

void launch_stream_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                          int* grid_out, cudaStream_t s) {
    SkArgs a;
    a.x = reinterpret_cast<const double*>(x);
    a.dim = p.dim;
    a.ncols = p.left * p.right;
    a.K = p.K;
    a.CT = p.dim <= 112 ? 64 : 32;
    a.ntiles = (a.ncols + a.CT - 1) / a.CT;
    a.mtiles = (int)((p.dim + 7) / 8);
    a.rows_glob = p.rows_glob;
    a.col_off = p.col_off;
    a.seed = p.seed;
    a.D = p.D;
    a.partial = partial;
    const int NT = nt_for(p.K);
    const int mtw = a.mtiles;  // full-height accumulators per consumer warp
    const size_t smem = (kStages * (size_t)(a.CT * a.dim + kPad) + 2 * (size_t)a.CT * NT * 8) * 8 + kBarBytes;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    *grid_out = grid;
    const int threads = (kCons + kRng + 1) * 32;
#define TRG_SK(MTW, NTV)                                                 \
    do {                                                                 \
        set_smem(k_sketch_l1_f64<MTW, NTV>, smem);                       \
        k_sketch_l1_f64<MTW, NTV><<<grid, threads, smem, s>>>(a);        \
    } while (0)
#define TRG_SK_NT(MTW)                   \
    switch (NT) {                        \
        case 1: TRG_SK(MTW, 1); break;   \
        case 2: TRG_SK(MTW, 2); break;   \
        case 4: TRG_SK(MTW, 4); break;   \
        default: TRG_SK(MTW, 8); break;  \
    }
    if (mtw <= 4) {
        TRG_SK_NT(4)
    } else if (mtw <= 8) {
        TRG_SK_NT(8)
    } else if (mtw <= 13) {
        TRG_SK_NT(13)
    } else {
        TRG_SK_NT(16)
    }
#undef TRG_SK_NT
#undef TRG_SK
    launch_reduce_partials(partial, grid, p.dim * p.K, y, s);
}

// ---------------------------------------------------------------- shrink
bool stream_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t odim) {
    if (dtype != F64 || left != 1 || (dim & 1) || odim > 64) return false;
    const int Tk = (int)((dim + 3) / 4);
    const size_t smem = (kStages * (size_t)(64 * dim + kPad) + (size_t)Tk * nt_for((int)odim) * 32) * 8 + kBarBytes;
    return smem <= kSmemBudget;
}

void launch_stream_ttm(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, int num_sms,
                       cudaStream_t s) {
    TtmArgs a;
    a.ldq = ldq;
    a.x = reinterpret_cast<const double*>(in);
    a.out = reinterpret_cast<double*>(out);
    a.q = q;
    a.dim = p.dim;
    a.rows = p.right;
    a.K = (int)p.odim;
    a.MT = 16 * kCons;
    a.Tk = (int)((p.dim + 3) / 4);
    a.ntiles = (a.rows + a.MT - 1) / a.MT;
    const int NT = nt_for(a.K);
    const size_t smem = (kStages * (size_t)(a.MT * a.dim + kPad) + (size_t)a.Tk * NT * 32) * 8 + kBarBytes;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    const int threads = (kCons + 1) * 32;
    switch (NT) {
        case 1: set_smem(k_ttm_l1_f64<1>, smem); k_ttm_l1_f64<1><<<grid, threads, smem, s>>>(a); break;
        case 2: set_smem(k_ttm_l1_f64<2>, smem); k_ttm_l1_f64<2><<<grid, threads, smem, s>>>(a); break;
        case 4: set_smem(k_ttm_l1_f64<4>, smem); k_ttm_l1_f64<4><<<grid, threads, smem, s>>>(a); break;
        default: set_smem(k_ttm_l1_f64<8>, smem); k_ttm_l1_f64<8><<<grid, threads, smem, s>>>(a); break;
    }
}

}  // namespace trg
