// SPDX-License-Identifier: Apache-2.0
//
// fp32 sketch and shrink for modes n >= 1 (left > 1) as streaming kernels: one TMA producer warp
// feeding a ring of 3-D boxes of the working tensor P (left, dim, right), l fastest
// (tensor.hpp:112-123), through full / empty mbarriers to FFMA consumer warps that never
// synchronise as a CTA inside the stream. These replace slab_f32.cu's kernels wherever their
// plans apply: those stage each item with cp.async / register loads between CTA barriers and
// measured instruction-bound (C5 mode 1: 507 us sketch, 302 us shrink on 622 MB, 15-30 % of HBM).
//
//   shrink (tensor.hpp:193-207 with m = Q^T):  out(l, k, r) = sum_d P(l, d, r) Q(d, k)
//     item = (RB slabs r, LB l's), streamed in d-chunks of DC; the chunk of Q^T (fp32, rows padded
//     with zeros) rides in the same stage by a 1-D bulk copy. Consumer thread = (d-slice, r, 4 l,
//     4 k): per d one 16-byte P load, one broadcast 16-byte Q load and 16 FFMA.
//   sketch (sketch.hpp:80-83):  Y(d, k) = sum_{l, r} P(l, d, r) Omega(col_off + l + left r, k)
//     grid = (CTAs, k-groups of KG columns, d-chunks of DC); item = (RB slabs, LB l's) of the
//     CTA's d-chunk. Generator warps regenerate the item's Omega block from the reference stream
//     (SplitMix64 + fp32 Box-Muller, common.cuh gauss_pair_f32_fast; draw D + col_off + c +
//     rows_glob k, sketch.hpp:32-38) into a second ring. Consumer thread = (r-slice, D d's, 4 l):
//     per slab D 16-byte P loads, KG/4 x 4 16-byte Omega loads, 4 D KG FFMA. The per-thread sums
//     meet in shared memory in a fixed order and leave as one fp64 partial per CTA for the
//     fixed-order split-K reduction (launch_reduce_partials / launch_qr_fused), as every sketch.
// Both accumulate in fp32 over at most a few hundred terms per accumulator: far inside the 1e-4
// fp32 bound against the fp64 oracle (tests/test_gpu_slab_f32.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "pipeline.cuh"

namespace trg {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 st_encode_fn() {
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// P as a 3-D fp32 tensor {left, dim, right}; box {LB, DC, RB} lands dense ([r][d][l]), zero-filled
// outside the tensor
bool make_map3(CUtensorMap* m, const void* x, int64_t left, int64_t dim, int64_t right, int LB, int DC, int RB) {
    auto fn = st_encode_fn();
    if (!fn) return false;
    const cuuint64_t gdim[3] = {(cuuint64_t)left, (cuuint64_t)dim, (cuuint64_t)right};
    const cuuint64_t gstride[2] = {(cuuint64_t)left * 4, (cuuint64_t)left * dim * 4};
    const cuuint32_t box[3] = {(cuuint32_t)LB, (cuuint32_t)DC, (cuuint32_t)RB};
    const cuuint32_t estride[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(x), gdim, gstride, box, estride,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void tma3d(float* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar,
                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// mbarrier wait that lets the hardware suspend the warp (up to ~1 us) instead of re-polling: the
// consumer and generator warps otherwise spend issue slots on the try_wait / branch loop
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITH_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITH_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000u)
        : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


// Gaussians of `nruns` runs of `len` consecutive test-matrix columns: column c of run q is reference
// draw g0(q) + c (sketch.hpp:32-38). A unit is one Box-Muller pair (draws 2p, 2p + 1; random.hpp:50-62)
// of a run, the units are dealt round-robin over all nthreads threads (every warp gets its share:
// the consumer warps generate between their multiplications) and each thread keeps two pairs in
// flight. info(q) -> {g0, live (else zeros), base}; put(base, c, z) stores column c of the run.
struct RunInfo {
    uint64_t g0;
    bool live;
    int base;
};
template <class Info, class Put>
__device__ __forceinline__ void gen_runs(int g, int nthreads, int nruns, int len, const FastDiv& div_npr, uint64_t seed,
                                         Info info, Put put) {
    constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
    const int npr = len / 2 + 1;  // pairs touching a run of len columns
    const int units = nruns * npr;
    for (int u0 = g; u0 < units; u0 += 2 * nthreads) {
        uint64_t st[2];
        int cf[2], base[2];
        bool on[2], live[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int u = min(u0 + j * nthreads, units - 1);
            const int q = (int)div_npr.div((uint32_t)u);
            const int pi = u - q * npr;
            const RunInfo ri = info(q);
            const uint64_t p = (ri.g0 >> 1) + (uint64_t)pi;
            cf[j] = (int)(2 * p - ri.g0);  // column of draw 2p (-1 when g0 is odd)
            st[j] = seed + (2ull * p + 1ull) * kGamma;
            on[j] = u0 + j * nthreads < units && cf[j] < len;
            live[j] = ri.live;
            base[j] = ri.base;
        }
        float z[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) gauss_pair_f32_fast(st[j], z[j][0], z[j][1]);
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int cc = cf[j] + v;
                if (on[j] && cc >= 0 && cc < len) put(base[j], cc, live[j] ? z[j][v] : 0.f);
            }
    }
}

constexpr int kStMaxStages = 8;
constexpr int kStCons = 256;  // consumer threads (8 warps)

// ================================================================== shrink
struct StShArgs {
    float* out;
    const float* qt;  // [nd * DC][KP] fp32 Q^T, zero rows past dim, zero columns past K
    int left, dim, K, KP, LB, DC, RB, NLQ, NKQ, DS, nd, stages;
    int64_t right, nlb, nitems;
    uint32_t p_floats, q_floats, stage_floats;  // per stage: P box, Q^T chunk, both (16-byte multiple)
};

__global__ void __launch_bounds__(kStCons + 32, 1) k_st_shrink(const __grid_constant__ CUtensorMap pmap, StShArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + kStMaxStages;
    float* stg = reinterpret_cast<float*>(smem_raw + 128);
    float* red = stg + (size_t)a.stages * a.stage_floats;  // DS x tiles x 16
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t it0 = a.nitems * blockIdx.x / gridDim.x, it1 = a.nitems * (blockIdx.x + 1) / gridDim.x;
    if (tid == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kStCons / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();
    if (warp == kStCons / 32) {  // producer
        if (lane == 0) {
            const uint64_t pol = policy_l2(0);
            const uint32_t bytes = 4u * (a.p_floats + a.q_floats);
            uint32_t n = 0;
            for (int64_t it = it0; it < it1; ++it) {
                const int64_t rbk = it / a.nlb;
                const int lb = (int)(it - rbk * a.nlb);
                for (int c = 0; c < a.nd; ++c, ++n) {
                    const int s = (int)(n % (uint32_t)a.stages);
                    if (n >= (uint32_t)a.stages) mbar_wait_hint(&empty[s], ((n / a.stages) - 1) & 1);
                    float* dst = stg + (size_t)s * a.stage_floats;
                    mbar_arrive_expect_tx(&full[s], bytes);
                    tma3d(dst, &pmap, lb * a.LB, c * a.DC, (int)(rbk * a.RB), &full[s], pol);
                    bulk_g2s(dst + a.p_floats, a.qt + (size_t)c * a.DC * a.KP, 4u * a.q_floats, &full[s], pol);
                }
            }
        }
        return;
    }
    // consumers: thread = (ds, rl, lq, kq), kq fastest (its P load is a broadcast), lq next
    const int tiles = a.RB * a.NLQ * a.NKQ;
    const int ds = tid / tiles, t = tid - ds * tiles;
    const int kq = t % a.NKQ, lq = (t / a.NKQ) % a.NLQ, rl = t / (a.NKQ * a.NLQ);
    const bool active = ds < a.DS;
    uint32_t n = 0;
    for (int64_t it = it0; it < it1; ++it) {
        const int64_t rbk = it / a.nlb;
        const int lb = (int)(it - rbk * a.nlb);
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
        for (int c = 0; c < a.nd; ++c, ++n) {
            const int s = (int)(n % (uint32_t)a.stages);
            mbar_wait_hint(&full[s], (n / a.stages) & 1);
            if (active) {
                const float* P = stg + (size_t)s * a.stage_floats + (size_t)rl * a.DC * a.LB + 4 * lq + ds * a.LB;
                const float* Qc = stg + (size_t)s * a.stage_floats + a.p_floats + 4 * kq + ds * a.KP;
                const int pst = a.DS * a.LB, qst = a.DS * a.KP;
#pragma unroll 4
                for (int d = ds; d < a.DC; d += a.DS, P += pst, Qc += qst) {
                    const float4 p = *reinterpret_cast<const float4*>(P);
                    const float4 q = *reinterpret_cast<const float4*>(Qc);
                    const float pv[4] = {p.x, p.y, p.z, p.w}, qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(pv[i], qv[j], acc[i][j]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (a.DS > 1) {  // d-slices -> slice 0 in a fixed order
            named_sync(1, kStCons);
            if (active)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) red[((size_t)ds * tiles + t) * 16 + 4 * i + j] = acc[i][j];
            named_sync(1, kStCons);
            if (ds == 0)
                for (int s2 = 1; s2 < a.DS; ++s2)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] += red[((size_t)s2 * tiles + t) * 16 + 4 * i + j];
        }
        const int64_t r = rbk * a.RB + rl;
        const int l = lb * a.LB + 4 * lq;
        if (ds == 0 && r < a.right && l < a.left) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * kq + j;
                if (k < a.K)
                    *reinterpret_cast<float4*>(a.out + l + (int64_t)a.left * (k + (int64_t)a.K * r)) =
                        make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
            }
        }
    }
}

// M(k, d) = m[k m_so + d m_sd] (fp64) -> qt[d * KP + k] (fp32), zero past dim / K
__global__ void k_st_qt(const double* __restrict__ m, int64_t m_so, int64_t m_sd, int dim, int rows, int K, int KP,
                        float* __restrict__ qt) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * KP; e += gridDim.x * blockDim.x) {
        const int d = e / KP, k = e - d * KP;
        qt[e] = (k < K && d < dim) ? (float)m[(int64_t)k * m_so + (int64_t)d * m_sd] : 0.f;
    }
}

struct StShPlan {
    int KP, LB, DC, RB, NLQ, NKQ, DS, nd, stages;
    int64_t nlb, nitems;
    uint32_t p_floats, q_floats, stage_floats;
    size_t smem;
    int ctas_per_sm;
};

// largest LB = 4 j <= cap dividing left (left % 4 == 0)
int pick_lb(int64_t left, int cap) {
    for (int lb = std::min<int64_t>(cap, left) & ~3; lb >= 4; lb -= 4)
        if (left % lb == 0) return lb;
    return 4;
}

bool plan_st_shrink(int64_t left, int64_t dim, int64_t K, int64_t right, StShPlan& p) {
    if (left < 4 || (left % 4) || K < 1 || K > 64 || dim < 1 || dim > (1 << 20) || right < 1 || right >= (1 << 30) ||
        left * dim * right >= (int64_t(1) << 40) || left * dim >= (int64_t(1) << 31))
        return false;
    p.KP = (int)((K + 3) & ~3);
    p.NKQ = p.KP / 4;
    // l block: as many 4-l tiles as fit beside the k tiles in the consumer threads
    const int lb_cap = std::max(4, std::min(256, 4 * (kStCons / p.NKQ)));
    p.LB = pick_lb(left, lb_cap);
    // enough items for every SM: fewer slabs per item, then narrower l blocks (>= 16 l's, 64-byte
    // TMA rows), before splitting d inside a CTA
    const int64_t want = 2 * 148;
    for (;;) {
        p.NLQ = p.LB / 4;
        p.RB = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)kStCons / (p.NLQ * p.NKQ), right, 256}));
        while (p.RB > 1 && ((right + p.RB - 1) / p.RB) * (left / p.LB) < want) p.RB = (p.RB + 1) / 2;
        if (((right + p.RB - 1) / p.RB) * (left / p.LB) >= want || p.LB <= 16) break;
        const int nlb = pick_lb(left, p.LB - 4);
        if (nlb < 16) break;
        p.LB = nlb;
    }
    const int per_r = p.NLQ * p.NKQ;
    const int tiles = p.RB * per_r;
    p.DS = 1;
    while (2 * p.DS * tiles <= kStCons && p.DS < 16) p.DS *= 2;
    // d chunk: ~24 KB of P per stage, a multiple of DS
    int dc = (int)std::max<int64_t>(1, (24 * 1024 / 4) / ((int64_t)p.RB * p.LB));
    dc = (int)std::min<int64_t>({(int64_t)dc, dim, 256});
    // the same number of chunks with the least zero padding (C5: 60 = 4 x 15, not 4 x 18)
    {
        const int64_t nch = (dim + dc - 1) / dc;
        dc = (int)((dim + nch - 1) / nch);
    }
    p.DC = std::max(1, dc);
    p.nd = (int)((dim + p.DC - 1) / p.DC);
    p.nlb = left / p.LB;
    p.nitems = ((right + p.RB - 1) / p.RB) * p.nlb;
    p.p_floats = (uint32_t)(p.RB * p.DC * p.LB);
    p.q_floats = (uint32_t)(p.DC * p.KP);
    p.stage_floats = (p.p_floats + p.q_floats + 31) & ~31u;  // 128-byte aligned stages
    const size_t stage_bytes = 4ull * p.stage_floats;
    const size_t red = 4ull * (p.DS > 1 ? (size_t)p.DS * tiles * 16 : 0);
    // two CTAs per SM when ~100 KB hold >= 3 stages, else one with more stages
    p.stages = (int)std::min<size_t>(kStMaxStages, (100 * 1024 - red) / stage_bytes);
    p.ctas_per_sm = 2;
    if (p.stages < 3) {
        p.stages = (int)std::min<size_t>(kStMaxStages, (200 * 1024 - red) / stage_bytes);
        p.ctas_per_sm = 1;
    }
    if (p.stages < 2) return false;
    p.smem = 128 + stage_bytes * p.stages + red;
    return true;
}

// ================================================================== sketch
struct StSkArgs {
    double* partial;  // gridDim.x x dim x K
    int left, dim, K, KG, KQ, LB, DC, RB, NLQ, NDL, RS, stages, ompitch;
    int64_t right, nlb, nitems;
    uint32_t p_floats, stage_floats, om_floats;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    FastDiv div_npr, div_rb;  // Box-Muller pairs per column run; RB
    FastDiv div_nlb, div_lb;  // l-blocks per slab; LB
    FastDiv div_npr_m;        // pairs per merged run (LB == left: RB LB consecutive columns per k)
};

template <int KG, int D, int NC>
__global__ void __launch_bounds__(NC + 32, 1) k_st_sketch(const __grid_constant__ CUtensorMap pmap, StSkArgs a) {
    constexpr int KQ = KG / 4;
    constexpr int kOR = 3;  // test-matrix ring: item n + 2 is generated while item n is multiplied
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + kStMaxStages;
    uint64_t* ofull = empty + kStMaxStages;
    uint64_t* oempty = ofull + kOR;
    float* stg = reinterpret_cast<float*>(smem_raw + 256);
    float* om = stg + (size_t)a.stages * a.stage_floats;  // kOR x om_floats
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t it0 = a.nitems * blockIdx.x / gridDim.x, it1 = a.nitems * (blockIdx.x + 1) / gridDim.x;
    const int k0 = blockIdx.y * KG, d0 = blockIdx.z * a.DC;
    if (tid == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        for (int s = 0; s < kOR; ++s) {
            mbar_init(&ofull[s], NC / 32);
            mbar_init(&oempty[s], NC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NC / 32) {  // producer
        griddep_wait();
        if (lane == 0) {
            const uint64_t pol = policy_l2(0);
            uint32_t n = 0;
            for (int64_t it = it0; it < it1; ++it, ++n) {
                const int64_t rbk = it / a.nlb;
                const int lb = (int)(it - rbk * a.nlb);
                const int s = (int)(n % (uint32_t)a.stages);
                if (n >= (uint32_t)a.stages) mbar_wait_hint(&empty[s], ((n / a.stages) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], 4u * a.p_floats);
                tma3d(stg + (size_t)s * a.stage_floats, &pmap, lb * a.LB, d0, (int)(rbk * a.RB), &full[s], pol);
            }
        }
        return;
    }
    // The consumer warps also generate the test-matrix blocks, two items ahead: the Box-Muller
    // work (K / dim Gaussians per element, C5: 0.2) spreads over all of them instead of being the
    // critical path of a few generator warps. Block layout [rl][l / 4][kq][l % 4][4] (rows padded).
    auto generate = [&](int64_t it, uint32_t n) {
        const int64_t rbk = (int64_t)a.div_nlb.div((uint32_t)it);  // items < 2^31 (plan_st_sketch)
        const int lb = (int)(it - rbk * a.nlb);
        float* O = om + (size_t)(n % kOR) * a.om_floats;
        const int l0 = lb * a.LB;
        if (a.LB == a.left) {
            // whole rows: the RB slabs of the item are RB LB consecutive columns of the unfolding, so
            // each k is one run of RB LB draws (one Box-Muller pair per two columns, no per-slab runs)
            const int len = a.RB * a.LB;
            const int64_t rlim = a.right - rbk * a.RB;  // slabs past the tensor's end are zero
            gen_runs(tid, NC, KG, len, a.div_npr_m, a.seed,
                     [&](int k) {
                         return RunInfo{a.D + (uint64_t)(a.col_off + (int64_t)a.left * rbk * a.RB) +
                                            (uint64_t)a.rows_glob * (uint64_t)(k0 + k),
                                        k0 + k < a.K, (k >> 2) * 16 + (k & 3)};
                     },
                     [&](int base, int c, float z) {
                         const int rl = (int)a.div_lb.div((uint32_t)c), l = c - rl * a.LB;
                         O[base + rl * a.NLQ * a.ompitch + (l >> 2) * a.ompitch + (l & 3) * 4] = rl < rlim ? z : 0.f;
                     });
            __syncwarp();
            if (lane == 0) mbar_arrive(&ofull[n % kOR]);
            return;
        }
        gen_runs(tid, NC, KG * a.RB, a.LB, a.div_npr, a.seed,
                 [&](int q) {
                     const int k = (int)a.div_rb.div((uint32_t)q), rl = q - k * a.RB;
                     const int64_t r = rbk * a.RB + rl;
                     return RunInfo{a.D + (uint64_t)(a.col_off + l0 + (int64_t)a.left * r) +
                                        (uint64_t)a.rows_glob * (uint64_t)(k0 + k),
                                    k0 + k < a.K && r < a.right, rl * a.NLQ * a.ompitch + (k >> 2) * 16 + (k & 3)};
                 },
                 [&](int base, int c, float z) { O[base + (c >> 2) * a.ompitch + (c & 3) * 4] = z; });
        __syncwarp();
        if (lane == 0) mbar_arrive(&ofull[n % kOR]);
    };
    for (uint32_t j = 0; j < 2 && it0 + j < it1; ++j) generate(it0 + j, j);
    // consumers: thread = (rs, dl, lq), lq fastest: the P loads of a warp are consecutive 16-byte
    // chunks ([r][d][l] with d = dl + NDL i), the Omega loads broadcast over dl
    const int per = a.NLQ * a.NDL;
    const int rs = tid / per, t = tid - rs * per;
    const int lq = t % a.NLQ, dl = t / a.NLQ;
    const bool active = rs < a.RS;
    float acc[D][KG];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < KG; ++j) acc[i][j] = 0.f;
    uint32_t n = 0;
    for (int64_t it = it0; it < it1; ++it, ++n) {
        const int s = (int)(n % (uint32_t)a.stages), os = (int)(n % kOR);
        mbar_wait_hint(&full[s], (n / a.stages) & 1);
        mbar_wait_hint(&ofull[os], (n / kOR) & 1);
        if (active) {
            const float* P = stg + (size_t)s * a.stage_floats + 4 * lq;
            const float* O = om + (size_t)os * a.om_floats + (size_t)lq * a.ompitch;
            for (int rl = rs; rl < a.RB; rl += a.RS) {
                float pv[D][4];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const int d = dl + a.NDL * i;
                    if (d < a.DC) {
                        const float4 v = *reinterpret_cast<const float4*>(P + ((size_t)rl * a.DC + d) * a.LB);
                        pv[i][0] = v.x;
                        pv[i][1] = v.y;
                        pv[i][2] = v.z;
                        pv[i][3] = v.w;
                    } else {
                        pv[i][0] = pv[i][1] = pv[i][2] = pv[i][3] = 0.f;
                    }
                }
                const float* Or = O + (size_t)rl * a.NLQ * a.ompitch;
#pragma unroll
                for (int kq = 0; kq < KQ; ++kq) {
                    float w[4][4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 v = *reinterpret_cast<const float4*>(Or + kq * 16 + 4 * j);
                        w[j][0] = v.x;
                        w[j][1] = v.y;
                        w[j][2] = v.z;
                        w[j][3] = v.w;
                    }
#pragma unroll
                    for (int i = 0; i < D; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j)
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) acc[i][4 * kq + kk] = fmaf(pv[i][j], w[j][kk], acc[i][4 * kq + kk]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[s]);
            mbar_arrive(&oempty[os]);
        }
        if (it + 2 < it1) {
            // item n + 2 goes to the slot of item n - 1: every warp must be done with that one
            if (n >= 1) mbar_wait_hint(&oempty[(n + 2) % kOR], ((n - 1) / kOR) & 1);
            generate(it + 2, n + 2);
        }
    }
    // (rs, lq) partial sums -> this CTA's fp64 partial of (d-chunk, k-group), fixed order
    named_sync(1, NC);  // every consumer is past the ring: its memory is free
    float* red = stg;        // [RS * NLQ][DC][KG]
    if (active)
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int d = dl + a.NDL * i;
            if (d < a.DC)
#pragma unroll
                for (int j = 0; j < KG; ++j) red[((size_t)(rs * a.NLQ + lq) * a.DC + d) * KG + j] = acc[i][j];
        }
    named_sync(1, NC);
    double* part = a.partial + (int64_t)blockIdx.x * a.dim * a.K;
    const int ngrp = a.RS * a.NLQ;
    for (int e = tid; e < a.DC * KG; e += NC) {
        const int d = e / KG, j = e - d * KG;
        if (d0 + d >= a.dim || k0 + j >= a.K) continue;
        double sum = 0.0;
        for (int gg = 0; gg < ngrp; ++gg) sum += (double)red[((size_t)gg * a.DC + d) * KG + j];
        part[(d0 + d) + (int64_t)a.dim * (k0 + j)] = sum;
    }
}

struct StSkPlan {
    int KG, ngroups, D, LB, DC, nz, NLQ, NDL, RS, RB, stages, ompitch, npmax, NC;
    int64_t nlb, nitems;
    uint32_t p_floats, stage_floats, om_floats;
    size_t smem;
    int gx;
};

bool plan_st_sketch(int64_t left, int64_t dim, int K, int64_t right, int num_sms, StSkPlan& p) {
    if (left < 4 || (left % 4) || K < 1 || K > 64 || dim < 1 || dim > (1 << 20) || right < 1 || right >= (1 << 30) ||
        left * dim * right >= (int64_t(1) << 40) || left * dim >= (int64_t(1) << 31))
        return false;
    // K <= 20: one k group (wider sketches re-read P per group: C4's mode 1 with K = 64 measured
    // 279 us against 125 us for slab_f32.cu's kernel)
    if (K > 20) return false;
    p.KG = (K + 3) & ~3;
    p.ngroups = 1;
    p.D = p.KG <= 16 ? 4 : 3;
    // 16 consumer warps when the accumulators leave the registers for them (KG <= 12: C5), else 8
    p.NC = p.KG <= 12 ? 512 : kStCons;
    // whole rows of l when short (TMA rows of >= 48 bytes), else 64-wide blocks; when there are too
    // few slabs for several r-slices per item (right < 4: the last mode of an unprojected tensor,
    // C5 fused sketch_m4), wider l blocks instead, up to what one d-chunk of consumers holds
    const int lb_cap = right < 4 ? (int)std::min<int64_t>(256, std::max<int64_t>(64, 4 * (p.NC / ((dim + p.D - 1) / p.D))))
                                 : 64;
    p.LB = left <= 64 ? (int)left : pick_lb(left, lb_cap);
    p.NLQ = p.LB / 4;
    if (p.NLQ > p.NC) return false;
    p.NDL = (int)std::min<int64_t>({(dim + p.D - 1) / p.D, (int64_t)p.NC / p.NLQ, (int64_t)256 / p.D});
    p.DC = (int)std::min<int64_t>(dim, (int64_t)p.NDL * p.D);  // <= 256: a TMA box dimension
    p.NDL = (p.DC + p.D - 1) / p.D;
    p.nz = (int)((dim + p.DC - 1) / p.DC);
    p.RS = std::max(1, p.NC / (p.NLQ * p.NDL));
    // RB: a multiple of RS with ~16-32 KB of P per stage
    const int64_t slab = (int64_t)p.DC * p.LB;  // floats per slab of the box
    int64_t rb = std::max<int64_t>(p.RS, (16 * 1024 / 4 + slab - 1) / slab);
    rb = (rb + p.RS - 1) / p.RS * p.RS;
    rb = std::min<int64_t>({rb, 256, std::max<int64_t>(right, 1)});
    p.RB = (int)std::max<int64_t>(1, rb);
    if (p.RS > p.RB) p.RS = p.RB;
    p.nlb = left / p.LB;
    p.nitems = ((right + p.RB - 1) / p.RB) * p.nlb;
    p.p_floats = (uint32_t)(p.RB * slab);
    p.stage_floats = (p.p_floats + 31) & ~31u;
    p.ompitch = (p.KG / 4) * 16 + 4;  // odd 16-byte stride between the l-quads of a slab
    p.om_floats = (uint32_t)(((int64_t)p.RB * p.NLQ * p.ompitch + 31) & ~31);
    p.npmax = p.LB / 2 + 1;
    if ((int64_t)p.KG * p.RB * p.npmax >= (int64_t(1) << 31)) return false;
    if (p.nitems >= (int64_t(1) << 31)) return false;  // 32-bit item split (FastDiv) in the generator
    const size_t red = 4ull * (size_t)p.RS * p.NLQ * p.DC * p.KG;
    const size_t stage_bytes = 4ull * p.stage_floats, om_bytes = 3ull * 4 * p.om_floats;
    p.stages = (int)std::min<size_t>(kStMaxStages, (200 * 1024 - om_bytes) / stage_bytes);
    if (p.stages < 2) return false;
    p.stages = std::min(p.stages, 6);
    p.smem = 256 + std::max(stage_bytes * p.stages, red) + om_bytes;
    if (p.smem > 220 * 1024) return false;
    // one CTA per SM (the generators and consumers share its issue slots); CTA columns for all SMs
    // one wave: the CTAs hold ~190 KB of shared memory, one per SM
    const int64_t per_col = (int64_t)p.ngroups * p.nz;
    p.gx = (int)std::max<int64_t>(1, std::min<int64_t>(p.nitems, (int64_t)num_sms / per_col));
    return true;
}

// ================================================================== mode 0 (left == 1), short fibres
// The mode-0 shrink of a tensor whose first extent is short (C5: I_0 = 60, K_0 = 12): X_(0) is the
// raw buffer as dim x ncols, fibre r = dim contiguous floats, so a stage is RB whole fibres by one
// 1-D bulk copy. out(k, r) = sum_d X(d, r) Q(d, k); Q^T resident; thread = (k quad, four fibres
// r + RB/4 i): per 4 d four 16-byte fibre loads, four broadcast 16-byte Q^T loads, 64 FFMA. Fibre
// rows are 15 x 16 B apart for dim = 60: the 8 lanes of a load phase hit 8 different 16-byte bank
// groups. (A mode-0 sketch with the same staging, its test matrix generated by dedicated warps or by
// the consumer warps, measured 1.37-1.8 ms against 1.10 ms for stream_f32.cu's k_sketch_l1_f32 on
// C5: K / I_0 = 0.2 Gaussians per element cost as much issue as the 12 FFMA, and it is not kept.)
struct St0ShArgs {
    const float* x;
    float* out;
    const float* qt;  // [dim][KP]
    int dim, K, KP, NKQ, RB, stages;
    int64_t ncols, nitems;
    uint32_t stage_floats;
};

__global__ void __launch_bounds__(kStCons + 32, 1) k_st0_shrink(St0ShArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + kStMaxStages;
    uint64_t* qbar = empty + kStMaxStages;
    float* qs = reinterpret_cast<float*>(smem_raw + 256);
    float* stg = qs + (((size_t)a.dim * a.KP + 31) & ~(size_t)31);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t it0 = a.nitems * blockIdx.x / gridDim.x, it1 = a.nitems * (blockIdx.x + 1) / gridDim.x;
    if (tid == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kStCons / 32);
        }
        mbar_init(qbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();
    if (warp == kStCons / 32) {
        if (lane == 0) {
            const uint64_t pol = policy_l2(0);
            mbar_arrive_expect_tx(qbar, 4u * a.dim * a.KP);
            bulk_g2s(qs, a.qt, 4u * a.dim * a.KP, qbar, policy_l2(1));
            uint32_t n = 0;
            for (int64_t it = it0; it < it1; ++it, ++n) {
                const int s = (int)(n % (uint32_t)a.stages);
                if (n >= (uint32_t)a.stages) mbar_wait_hint(&empty[s], ((n / a.stages) - 1) & 1);
                const int64_t r0 = it * a.RB;
                const int nr = (int)(a.ncols - r0 < a.RB ? a.ncols - r0 : a.RB);
                const uint32_t bytes = 4u * (uint32_t)(nr * a.dim);
                mbar_arrive_expect_tx(&full[s], bytes);
                bulk_g2s(stg + (size_t)s * a.stage_floats, a.x + r0 * a.dim, bytes, &full[s], pol);
            }
        }
        return;
    }
    constexpr int FPT = 4;  // fibres per thread: each Q^T load feeds 4 x 4 FFMA
    const int kq = tid % a.NKQ, fp = tid / a.NKQ;
    const int quarter = a.RB / FPT;
    const bool active = fp < quarter;
    mbar_wait_hint(qbar, 0);
    const float* Q = qs + 4 * kq;
    uint32_t n = 0;
    for (int64_t it = it0; it < it1; ++it, ++n) {
        const int s = (int)(n % (uint32_t)a.stages);
        mbar_wait_hint(&full[s], (n / a.stages) & 1);
        const int64_t r0 = it * a.RB;
        const int nr = (int)(a.ncols - r0 < a.RB ? a.ncols - r0 : a.RB);
        float acc[FPT][4];
#pragma unroll
        for (int f = 0; f < FPT; ++f)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[f][j] = 0.f;
        if (active) {
            // fibres fp + quarter i; those past nr read stale (finite) stage data and are not stored
            const float* X0 = stg + (size_t)s * a.stage_floats + (size_t)fp * a.dim;
            const size_t fst = (size_t)quarter * a.dim;
#pragma unroll 1
            for (int d = 0; d < a.dim; d += 4) {
                float v[FPT][4];
#pragma unroll
                for (int f = 0; f < FPT; ++f) {
                    const float4 p = *reinterpret_cast<const float4*>(X0 + f * fst + d);
                    v[f][0] = p.x;
                    v[f][1] = p.y;
                    v[f][2] = p.z;
                    v[f][3] = p.w;
                }
#pragma unroll
                for (int dd = 0; dd < 4; ++dd) {
                    const float4 q = *reinterpret_cast<const float4*>(Q + (size_t)(d + dd) * a.KP);
                    const float qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int f = 0; f < FPT; ++f)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[f][j] = fmaf(v[f][dd], qv[j], acc[f][j]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (active) {
#pragma unroll
            for (int f = 0; f < FPT; ++f) {
                const int fl = fp + f * quarter;
                if (fl >= nr) continue;
                float* o = a.out + (r0 + fl) * a.K + 4 * kq;
                if ((a.K & 3) == 0) {
                    *reinterpret_cast<float4*>(o) = make_float4(acc[f][0], acc[f][1], acc[f][2], acc[f][3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (4 * kq + j < a.K) o[j] = acc[f][j];
                }
            }
        }
    }
}

struct St0Plan {
    int KP, NKQ, RB, stages;
    int64_t nitems;
    uint32_t stage_floats;
    size_t smem;
};

bool st0_shape_ok(int64_t dim, int64_t K, int64_t ncols, int64_t max_dim) {
    return dim >= 4 && dim <= max_dim && (dim % 4) == 0 && K >= 1 && K <= 64 && K <= dim && ncols >= 1 &&
           dim * ncols < (int64_t(1) << 40) && ncols < (int64_t(1) << 36);
}

bool plan_st0_shrink(int64_t dim, int64_t K, int64_t ncols, St0Plan& p) {
    if (!st0_shape_ok(dim, K, ncols, 128)) return false;
    p.KP = (int)((K + 3) & ~3);
    p.NKQ = p.KP / 4;
    p.RB = (4 * (kStCons / p.NKQ)) & ~7;  // four fibres per thread
    while (p.RB > 8 && (int64_t)p.RB * dim * 4 > 96 * 1024) p.RB -= 8;  // two stages at least
    if (p.RB < 8) return false;
    p.nitems = (ncols + p.RB - 1) / p.RB;
    p.stage_floats = (uint32_t)(((int64_t)p.RB * dim + 31) & ~31);
    const size_t qbytes = 4 * (((size_t)dim * p.KP + 31) & ~(size_t)31);
    p.stages = (int)std::min<size_t>(kStMaxStages, (200 * 1024 - qbytes) / (4ull * p.stage_floats));
    if (p.stages < 2) return false;
    p.smem = 256 + qbytes + 4ull * p.stage_floats * p.stages;
    return true;
}

}  // namespace

bool st_shrink_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right) {
    StShPlan p;
    return dtype == F32 && left > 1 && !getenv("TRG_NO_ST") && st_encode_fn() && plan_st_shrink(left, dim, K, right, p);
}

void launch_st_shrink(const TTMPlan& tp, const void* in, void* out, const double* m, int num_sms, cudaStream_t s) {
    StShPlan p;
    if (!plan_st_shrink(tp.left, tp.dim, tp.odim, tp.right, p)) throw std::runtime_error("st shrink: unsupported shape");
    CUtensorMap map;
    if (!make_map3(&map, in, tp.left, tp.dim, tp.right, p.LB, p.DC, p.RB))
        throw std::runtime_error("st shrink: tensor map encoding failed");
    const int rows = p.nd * p.DC;
    float* qt = reinterpret_cast<float*>(scratch_alloc(sizeof(float) * (size_t)rows * p.KP, s));
    k_st_qt<<<(int)std::min<int64_t>(1024, ((int64_t)rows * p.KP + 255) / 256), 256, 0, s>>>(
        m, tp.m_so, tp.m_sd, (int)tp.dim, rows, (int)tp.odim, p.KP, qt);
    StShArgs a{};
    a.out = reinterpret_cast<float*>(out);
    a.qt = qt;
    a.left = (int)tp.left;
    a.dim = (int)tp.dim;
    a.K = (int)tp.odim;
    a.KP = p.KP;
    a.LB = p.LB;
    a.DC = p.DC;
    a.RB = p.RB;
    a.NLQ = p.NLQ;
    a.NKQ = p.NKQ;
    a.DS = p.DS;
    a.nd = p.nd;
    a.stages = p.stages;
    a.right = tp.right;
    a.nlb = p.nlb;
    a.nitems = p.nitems;
    a.p_floats = p.p_floats;
    a.q_floats = p.q_floats;
    a.stage_floats = p.stage_floats;
    allow_smem(k_st_shrink, p.smem);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.nitems, (int64_t)num_sms * p.ctas_per_sm));
    pdl_launch(k_st_shrink, dim3(grid), dim3(kStCons + 32), p.smem, s, map, a);
    scratch_free(qt, s);
}

bool st_sketch_ok(int dtype, int64_t left, int64_t dim, int K, int64_t right) {
    StSkPlan p;
    return dtype == F32 && left > 1 && !getenv("TRG_NO_ST") && st_encode_fn() &&
           plan_st_sketch(left, dim, K, right, 148, p);
}

int st_sketch_grid(int64_t left, int64_t dim, int K, int64_t right, int num_sms) {
    StSkPlan p;
    if (!plan_st_sketch(left, dim, K, right, num_sms, p)) return 0;
    return p.gx;
}

int launch_st_sketch(const SketchPlan& sp, const void* x, double* partial, double* y, int num_sms, cudaStream_t s) {
    StSkPlan p;
    if (!plan_st_sketch(sp.left, sp.dim, sp.K, sp.right, num_sms, p)) throw std::runtime_error("st sketch: unsupported shape");
    CUtensorMap map;
    if (!make_map3(&map, x, sp.left, sp.dim, sp.right, p.LB, p.DC, p.RB))
        throw std::runtime_error("st sketch: tensor map encoding failed");
    StSkArgs a{};
    a.partial = partial;
    a.left = (int)sp.left;
    a.dim = (int)sp.dim;
    a.K = sp.K;
    a.KG = p.KG;
    a.KQ = p.KG / 4;
    a.LB = p.LB;
    a.DC = p.DC;
    a.RB = p.RB;
    a.NLQ = p.NLQ;
    a.NDL = p.NDL;
    a.RS = p.RS;
    a.stages = p.stages;
    a.ompitch = p.ompitch;
    a.right = sp.right;
    a.nlb = p.nlb;
    a.nitems = p.nitems;
    a.p_floats = p.p_floats;
    a.stage_floats = p.stage_floats;
    a.om_floats = p.om_floats;
    a.seed = sp.seed;
    a.D = sp.D;
    a.rows_glob = sp.rows_glob;
    a.col_off = sp.col_off;
    a.div_npr = FastDiv((uint32_t)(p.LB / 2 + 1));
    a.div_rb = FastDiv((uint32_t)p.RB);
    a.div_nlb = FastDiv((uint32_t)p.nlb);
    a.div_lb = FastDiv((uint32_t)p.LB);
    a.div_npr_m = FastDiv((uint32_t)(p.RB * p.LB / 2 + 1));
    const dim3 grid(p.gx, p.ngroups, p.nz), block(p.NC + 32);
#define TRG_STSK(KGV, DV, NCV)                                               \
    do {                                                                     \
        allow_smem(k_st_sketch<KGV, DV, NCV>, p.smem);                       \
        pdl_launch(k_st_sketch<KGV, DV, NCV>, grid, block, p.smem, s, map, a); \
    } while (0)
    switch (p.KG) {
        case 4: TRG_STSK(4, 4, 512); break;
        case 8: TRG_STSK(8, 4, 512); break;
        case 12: TRG_STSK(12, 4, 512); break;
        case 16: TRG_STSK(16, 4, kStCons); break;
        default: TRG_STSK(20, 3, kStCons); break;
    }
#undef TRG_STSK
    if (y) launch_reduce_partials(partial, p.gx, sp.dim * sp.K, y, s);
    return p.gx;
}

bool st0_shrink_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols) {
    St0Plan p;
    return dtype == F32 && left == 1 && !getenv("TRG_NO_ST") && plan_st0_shrink(dim, K, ncols, p);
}

void launch_st0_shrink(const TTMPlan& tp, const void* in, void* out, const double* m, int num_sms, cudaStream_t s) {
    St0Plan p;
    if (!plan_st0_shrink(tp.dim, tp.odim, tp.right, p)) throw std::runtime_error("st0 shrink: unsupported shape");
    float* qt = reinterpret_cast<float*>(scratch_alloc(sizeof(float) * (size_t)tp.dim * p.KP, s));
    k_st_qt<<<(int)std::min<int64_t>(1024, (tp.dim * p.KP + 255) / 256), 256, 0, s>>>(
        m, tp.m_so, tp.m_sd, (int)tp.dim, (int)tp.dim, (int)tp.odim, p.KP, qt);
    St0ShArgs a{};
    a.x = reinterpret_cast<const float*>(in);
    a.out = reinterpret_cast<float*>(out);
    a.qt = qt;
    a.dim = (int)tp.dim;
    a.K = (int)tp.odim;
    a.KP = p.KP;
    a.NKQ = p.NKQ;
    a.RB = p.RB;
    a.stages = p.stages;
    a.ncols = tp.right;
    a.nitems = p.nitems;
    a.stage_floats = p.stage_floats;
    allow_smem(k_st0_shrink, p.smem);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.nitems, num_sms));
    pdl_launch(k_st0_shrink, dim3(grid), dim3(kStCons + 32), p.smem, s, a);
    scratch_free(qt, s);
}

}  // namespace trg
