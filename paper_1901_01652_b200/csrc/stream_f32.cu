// SPDX-License-Identifier: Apache-2.0
//
// fp32 mode-0 sketch Y_0 = X_(0) Omega_0 (sketch.hpp:80-83) for the fp32
// configurations (C3-C5: I_0 = 1000, 1024, 60).
//
// X_(0) is I_0 x L column-major (each column a contiguous mode-0 fibre). The
// kernel is FFMA-based: at 2 K flops per 4-byte element (C3 10, C5 6 flop/B)
// the FP32 pipe and HBM are within 1.2x of each other, and fp32 products
// accumulated per thread over ~10^4 terms, then summed across CTAs in fp64 in
// a fixed order, keep Y well inside the 1e-4 fp32 tolerance.
//
//  * CTA (rs, cg): rows [rs DT, rs DT + DT) of every column of its column
//    tiles (row splits only when the DT x K accumulator slice would not fit
//    one SM's registers, i.e. C4).
//  * producer warp: TMA 2-D tensor copies of a {DTB rows x CT columns} box (up
//    to NB boxes cover DT rows); DTB/4 is odd so that float4 rows of
//    consecutive columns land in distinct banks.
//  * generator warps: the CT x K block of the reference test matrix
//    (SplitMix64 + Box-Muller by stream index, fp32 transcendentals, |err| ~
//    1e-7 relative) into shared memory, double-buffered.
//  * consumer warps: thread = (4 consecutive rows, TK consecutive columns of
//    Y, column group g); per column one float4 of X and TK/4 broadcast
//    float4s of Omega feed 4 TK FFMAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "pipeline.cuh"

namespace trg {

namespace {

#ifndef TRG_F32_CONS
#define TRG_F32_CONS 8
#endif
constexpr int kF32Cons = TRG_F32_CONS;
#ifndef TRG_F32_GEN_SMALL
#define TRG_F32_GEN_SMALL 12  // generator warps when TK <= 12 (dense test-matrix tiles, C5): 8 / 12 / 16 measured
                              // 1037 / 1031 / 1060 us on C5 with the MUFU Box-Muller
#endif
#ifndef TRG_F32_GEN_LARGE
#define TRG_F32_GEN_LARGE 4
#endif
#ifndef TRG_F32_GEN_MULTI
#define TRG_F32_GEN_MULTI 8  // generator warps when K spans several TK blocks (C4's K_0 = 64): 1.24 -> 0.86 ms
#endif
constexpr int kF32Stages = 4;
constexpr int kF32OB = 2;

struct F32SkArgs {
    int64_t I0, L;          // X_(0) is I0 x L
    int DT, DTB, NB, CT;    // rows per CTA, rows per box, boxes per stage, columns per tile
    int BS;                 // floats per box region (CT * DTB rounded up to 128 B: TMA destinations are 128-B aligned)
    int DS;                 // row splits (grid = DS x GC)
    int K, Kp, TK, nkb, ndb, G;
    int64_t ntiles;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    double* partial;        // per column-CTA: I0 x K fp64 (rows of this CTA only)
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                            uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// GEN generator warps: 8 when the Omega tile is dense in draws (C5: 0.2 draws per element,
// light consumers), 4 otherwise (C3/C4 need the registers for 4 x TK accumulators)
template <int TK, int GEN>
__global__ void __launch_bounds__((kF32Cons + GEN + 1) * 32, 1)
    k_sketch_l1_f32(const __grid_constant__ CUtensorMap tmap, F32SkArgs a) {
    constexpr int kF32Gen = GEN;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int rs = blockIdx.x % a.DS;           // row split
    const int cg = blockIdx.x / a.DS;           // column CTA index
    const int GC = gridDim.x / a.DS;
    const int stage_floats = a.NB * a.BS;
    float* stages = reinterpret_cast<float*>(smem_raw);
    float* om = stages + kF32Stages * stage_floats;  // kF32OB x CT x Kp
    const int om_floats = a.CT * a.Kp;
    uint64_t* bars = reinterpret_cast<uint64_t*>(om + kF32OB * om_floats);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + kF32Stages;
    uint64_t* full_o = bars + 2 * kF32Stages;
    uint64_t* empty_o = bars + 2 * kF32Stages + kF32OB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nl = (a.ntiles - cg + GC - 1) / GC;
    const int CT = a.CT;

    for (int i = tid; i < kF32OB * om_floats; i += blockDim.x) om[i] = 0.f;
    if (tid == 0) {
        for (int s = 0; s < kF32Stages; ++s) {
            mbar_init(&full_x[s], 1);
            mbar_init(&empty_x[s], kF32Cons * 32);
        }
        for (int b = 0; b < kF32OB; ++b) {
            mbar_init(&full_o[b], kF32Gen * 32);
            mbar_init(&empty_o[b], kF32Cons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kF32Cons + kF32Gen) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint32_t bytes = (uint32_t)(a.NB * a.CT * a.DTB * 4);
            for (int64_t j = 0; j < nl; ++j) {
                const int s = (int)(j % kF32Stages);
                mbar_wait(&empty_x[s], (uint32_t)((j / kF32Stages) & 1) ^ 1u);
                const int64_t c0 = (cg + j * GC) * CT;
                mbar_arrive_expect_tx(&full_x[s], bytes);
                for (int b = 0; b < a.NB; ++b)
                    tma_load_2d(stages + s * stage_floats + b * a.BS, &tmap, rs * a.DT + b * a.DTB, (int)c0,
                                &full_x[s], pol);
            }
        }
        return;
    }
    if (warp >= kF32Cons) {
        // ---- generators: Omega(c, k) = draw D + col_off + c + rows_glob k, pairs shared; the
        // MUFU-based fp32 Box-Muller (common.cuh gauss_pair_f32_fast, ~1e-6 relative per draw), as
        // the other fp32 sketches
        const int gtid = tid - kF32Cons * 32;
        constexpr int kMaxSl = 4;  // slots per generator thread on the fast path
        const bool even = ((a.rows_glob | (int64_t)a.D | a.col_off) & 1) == 0 && (CT & 1) == 0 &&
                          (CT / 2) * a.K <= kMaxSl * kF32Gen * 32;
        if (even) {
            // Every column run starts on an even draw: slot (jj, k) writes rows 2jj, 2jj + 1 of
            // column k (k fastest across lanes, so the stores fill consecutive words), and from
            // one tile of this CTA to the next its pair index advances by GC CT / 2, i.e. the
            // SplitMix64 state by GC CT gamma: no per-tile index arithmetic in the loop.
            const int nslots = (CT / 2) * a.K;
            const uint64_t gam = 0x9E3779B97F4A7C15ull;
            const uint64_t inc = (uint64_t)GC * (uint64_t)CT * gam;
            int jjs[kMaxSl], ks[kMaxSl];
            uint64_t st[kMaxSl];
            int ns = 0;
#pragma unroll
            for (int i = 0; i < kMaxSl; ++i) {
                const int sl = gtid + i * kF32Gen * 32;
                const bool on = sl < nslots;
                jjs[i] = on ? sl / a.K : 0;
                ks[i] = on ? sl - jjs[i] * a.K : 0;
                const uint64_t p0 = ((a.D + (uint64_t)a.col_off + (uint64_t)cg * CT +
                                      (uint64_t)a.rows_glob * (uint64_t)ks[i]) >> 1) + (uint64_t)jjs[i];
                st[i] = a.seed + (2ull * p0 + 1ull) * gam;
                ns += on ? 1 : 0;
            }
            const int64_t full_tiles = a.L / CT;
            for (int64_t j = 0; j < nl; ++j) {
                const int b = (int)(j % kF32OB);
                mbar_wait(&empty_o[b], (uint32_t)((j / kF32OB) & 1) ^ 1u);
                const int64_t t = cg + j * GC;
                const int64_t ncol = t < full_tiles ? CT : a.L - t * CT;
                float* O = om + b * om_floats;
#pragma unroll
                for (int i = 0; i < kMaxSl; ++i) {
                    if (i < ns) {
                        float z0, z1;
                        gauss_pair_f32_fast(st[i], z0, z1);
                        const int c = 2 * jjs[i];
                        O[c * a.Kp + ks[i]] = c < ncol ? z0 : 0.f;
                        O[(c + 1) * a.Kp + ks[i]] = c + 1 < ncol ? z1 : 0.f;
                    }
                    st[i] += inc;
                }
                mbar_arrive(&full_o[b]);
            }
            return;
        }
        const int npmax = CT / 2 + 1;
        for (int64_t j = 0; j < nl; ++j) {
            const int b = (int)(j % kF32OB);
            mbar_wait(&empty_o[b], (uint32_t)((j / kF32OB) & 1) ^ 1u);
            const int64_t c0 = (cg + j * GC) * CT;
            const int64_t ncol = min((int64_t)CT, a.L - c0);
            float* O = om + b * om_floats;
            for (int it = gtid; it < a.K * npmax; it += kF32Gen * 32) {
                const int k = it / npmax;
                const int jj = it - k * npmax;
                const uint64_t s0 = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)k;
                const uint64_t p = (s0 >> 1) + (uint64_t)jj;
                if (p > ((s0 + (uint64_t)CT - 1ull) >> 1)) continue;
                float z0, z1;
                gauss_pair_f32_fast(a.seed + (2ull * p + 1ull) * 0x9E3779B97F4A7C15ull, z0, z1);
                const int64_t cc = (int64_t)(2ull * p - s0);
                if (cc >= 0 && cc < CT) O[cc * a.Kp + k] = cc < ncol ? z0 : 0.f;
                if (cc + 1 >= 0 && cc + 1 < CT) O[(cc + 1) * a.Kp + k] = cc + 1 < ncol ? z1 : 0.f;
            }
            mbar_arrive(&full_o[b]);
        }
        return;
    }
    // ---- consumers: slot = (row block db of 4 rows, column block kb of TK), group g over columns
    const int nslots = a.ndb * a.nkb;
    const int slot = tid % nslots;
    const int g = tid / nslots;
    const bool active = g < a.G;
    const int db = slot % a.ndb, kb = slot / a.ndb;
    const int r0 = 4 * db;                // row within the CTA's DT rows
    const int box = r0 / a.DTB, rin = r0 - box * a.DTB;
    const int k0 = kb * TK;
    float4 acc[TK];  // acc[j] = rows r0..r0+3 of column k0 + j
#pragma unroll
    for (int j = 0; j < TK; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t j = 0; j < nl; ++j) {
        const int s = (int)(j % kF32Stages);
        const int b = (int)(j % kF32OB);
        mbar_wait(&full_x[s], (uint32_t)((j / kF32Stages) & 1));
        mbar_wait(&full_o[b], (uint32_t)((j / kF32OB) & 1));
        if (active) {
            const float* X = stages + s * stage_floats + box * a.BS + rin;
            const float* O = om + b * om_floats + k0;
#pragma unroll 1
            for (int c = g; c < CT; c += a.G) {
                const float4 xv = *reinterpret_cast<const float4*>(X + c * a.DTB);
                const float* oc = O + c * a.Kp;
#pragma unroll
                for (int q4 = 0; q4 < TK / 4; ++q4) {
                    const float4 ov = *reinterpret_cast<const float4*>(oc + 4 * q4);
#define TRG_COL(J, OV)                                   \
    acc[J].x = fmaf(xv.x, OV, acc[J].x);                 \
    acc[J].y = fmaf(xv.y, OV, acc[J].y);                 \
    acc[J].z = fmaf(xv.z, OV, acc[J].z);                 \
    acc[J].w = fmaf(xv.w, OV, acc[J].w);
                    TRG_COL(4 * q4 + 0, ov.x)
                    TRG_COL(4 * q4 + 1, ov.y)
                    TRG_COL(4 * q4 + 2, ov.z)
                    TRG_COL(4 * q4 + 3, ov.w)
#undef TRG_COL
                }
            }
        }
        mbar_arrive(&empty_x[s]);
        mbar_arrive(&empty_o[b]);
    }
    double* outp = a.partial + (int64_t)cg * a.I0 * a.K;
    if (a.G == 1) {  // every (row, column) of the slice has exactly one owner: write it directly
        if (active) {
#pragma unroll
            for (int jj = 0; jj < TK; ++jj) {
                const float v[4] = {acc[jj].x, acc[jj].y, acc[jj].z, acc[jj].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int64_t d = (int64_t)rs * a.DT + r0 + i;
                    if (d < a.I0 && k0 + jj < a.K && r0 + i < a.DT) outp[d + a.I0 * (k0 + jj)] = (double)v[i];
                }
            }
        }
        return;
    }
    // ---- fixed-order sum of the column groups in fp64, through the (consumed) stages
    asm volatile("bar.sync 1, %0;" ::"n"(kF32Cons * 32));
    double* red = reinterpret_cast<double*>(smem_raw);  // DT x Kp doubles
    for (int gg = 0; gg < a.G; ++gg) {
        if (active && g == gg) {
#pragma unroll
            for (int jj = 0; jj < TK; ++jj) {
                const float v[4] = {acc[jj].x, acc[jj].y, acc[jj].z, acc[jj].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    double* p = red + (r0 + i) + a.DT * (k0 + jj);
                    *p = (gg == 0 ? 0.0 : *p) + (double)v[i];
                }
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kF32Cons * 32));
    }
    for (int e = tid; e < a.DT * a.K; e += kF32Cons * 32) {
        const int k = e / a.DT, r = e - k * a.DT;
        const int64_t d = (int64_t)rs * a.DT + r;
        if (d < a.I0) outp[d + a.I0 * k] = red[r + a.DT * k];
    }
}


// ------------------------------------------------------------------ fp32 mode-0 shrink
// P^(1)(o, m) = sum_d X(d, m) Q_0(d, o) (tensor.hpp:193-207 with M = Q_0^T), m =
// mode-0 fibre. A unit is 64 consecutive fibres; its fibres' d-range arrives in
// chunks of DC rows (TMA box {DC, 64}, DC / 4 odd so that a warp's float4 loads
// of 32 consecutive fibres hit distinct banks). Each consumer warp owns whole
// units: lane l accumulates fibres l and l + 32 over all K outputs (acc 2 x KP
// in registers), reading per 4 rows of d two float4s of X and KP broadcast
// float4s of Q_0 (fp32 copy in shared memory). The producer interleaves the
// warps' chunk streams so that stage j belongs to warp j % 4.
constexpr int kTtCons = 4;
constexpr int kTtStages = 8;  // two per consumer warp

struct F32TtArgs {
    int64_t I0, L;  // X_(0) is I0 x L (fibres of I0)
    int DC, NCH, K, Kp;  // K outputs in all (row stride of out); CTA row blockIdx.y owns KP of them
    int64_t nunits;  // ceil(L / 64)
    void* out;       // P^(1): row m, K outputs (o fastest), fp32 (f64out = 0) or fp64
    int f64out;
};

template <int KP>
__global__ void __launch_bounds__((kTtCons + 1) * 32, 1)
    k_ttm_l1_f32(const __grid_constant__ CUtensorMap tmap, F32TtArgs a, const double* __restrict__ q, int64_t ldq) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int stage_floats = 64 * a.DC;
    float* stages = reinterpret_cast<float*>(smem_raw);
    float* Qs = stages + kTtStages * stage_floats;  // [NCH * DC][KP] (zero-padded)
    const int qrows = a.NCH * a.DC;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Qs + qrows * KP);
    uint64_t* full = bars;
    uint64_t* empty = bars + kTtStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // units of this CTA: u = blockIdx.x + i * gridDim.x; warp w owns i = w, w + 4, ...
    const int64_t nu = (a.nunits - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t nrounds = (nu + kTtCons - 1) / kTtCons;  // unit rounds (each warp one unit per round)
    const int ko = blockIdx.y * KP;  // first output column of this CTA's group
    for (int e = tid; e < qrows * KP; e += blockDim.x) {
        const int d = e / KP, o = e - d * KP;
        Qs[e] = (d < a.I0 && ko + o < a.K) ? (float)q[d + ldq * (ko + o)] : 0.f;
    }
    if (tid == 0) {
        for (int s = 0; s < kTtStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kTtCons) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int64_t j = 0;  // stage sequence: round, chunk, warp
            for (int64_t rd = 0; rd < nrounds; ++rd)
                for (int ch = 0; ch < a.NCH; ++ch)
                    for (int w = 0; w < kTtCons; ++w, ++j) {
                        const int64_t i = rd * kTtCons + w;
                        if (i >= nu) continue;  // this warp has no unit this round: skip its slot
                        const int s = (int)(j % kTtStages);
                        mbar_wait(&empty[s], (uint32_t)((j / kTtStages) & 1) ^ 1u);
                        const int64_t u = blockIdx.x + i * gridDim.x;
                        mbar_arrive_expect_tx(&full[s], (uint32_t)(64 * a.DC * 4));
                        tma_load_2d(stages + s * stage_floats, &tmap, ch * a.DC, (int)(u * 64), &full[s], pol);
                    }
        }
        return;
    }
    int64_t j0 = 0;
    for (int64_t rd = 0; rd < nrounds; ++rd, j0 += (int64_t)a.NCH * kTtCons) {
        const int64_t i = rd * kTtCons + warp;
        if (i >= nu) break;
        float acc[2][KP];
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int o = 0; o < KP; ++o) acc[f][o] = 0.f;
        for (int ch = 0; ch < a.NCH; ++ch) {
            const int64_t j = j0 + (int64_t)ch * kTtCons + warp;
            const int s = (int)(j % kTtStages);
            mbar_wait(&full[s], (uint32_t)((j / kTtStages) & 1));
            const float* X0 = stages + s * stage_floats + lane * a.DC;
            const float* X1 = X0 + 32 * a.DC;
            const float* Qc = Qs + (ch * a.DC) * KP;
#pragma unroll 1
            for (int d = 0; d < a.DC; d += 4) {
                const float4 x0 = *reinterpret_cast<const float4*>(X0 + d);
                const float4 x1 = *reinterpret_cast<const float4*>(X1 + d);
                const float* qd = Qc + d * KP;
#define TRG_QROW(XC, R)                                                               \
    {                                                                                 \
        const float4* qr = reinterpret_cast<const float4*>(qd + (R) * KP);            \
        _Pragma("unroll") for (int o4 = 0; o4 < KP / 4; ++o4) {                       \
            const float4 qv = qr[o4];                                                 \
            acc[0][4 * o4 + 0] = fmaf(x0.XC, qv.x, acc[0][4 * o4 + 0]);               \
            acc[0][4 * o4 + 1] = fmaf(x0.XC, qv.y, acc[0][4 * o4 + 1]);               \
            acc[0][4 * o4 + 2] = fmaf(x0.XC, qv.z, acc[0][4 * o4 + 2]);               \
            acc[0][4 * o4 + 3] = fmaf(x0.XC, qv.w, acc[0][4 * o4 + 3]);               \
            acc[1][4 * o4 + 0] = fmaf(x1.XC, qv.x, acc[1][4 * o4 + 0]);               \
            acc[1][4 * o4 + 1] = fmaf(x1.XC, qv.y, acc[1][4 * o4 + 1]);               \
            acc[1][4 * o4 + 2] = fmaf(x1.XC, qv.z, acc[1][4 * o4 + 2]);               \
            acc[1][4 * o4 + 3] = fmaf(x1.XC, qv.w, acc[1][4 * o4 + 3]);               \
        }                                                                             \
    }
                TRG_QROW(x, 0)
                TRG_QROW(y, 1)
                TRG_QROW(z, 2)
                TRG_QROW(w, 3)
#undef TRG_QROW
            }
            __syncwarp();
            mbar_arrive(&empty[s]);
        }
        const int64_t u = blockIdx.x + i * gridDim.x;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const int64_t m = u * 64 + lane + 32 * f;
            if (m >= a.L) continue;
            if (a.f64out) {
                double* dst = reinterpret_cast<double*>(a.out) + m * a.K + ko;
#pragma unroll
                for (int o = 0; o < KP; ++o)
                    if (ko + o < a.K) dst[o] = (double)acc[f][o];
            } else {
                float* dst = reinterpret_cast<float*>(a.out) + m * a.K + ko;
#pragma unroll
                for (int o = 0; o < KP; ++o)
                    if (ko + o < a.K) dst[o] = acc[f][o];
            }
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

struct F32Plan {
    int DS, DT, DTB, NB, CT, BS, TK, nkb, ndb, G, Kp;
    size_t smem;
};

// smallest box height >= need with (box / 4) odd (float4 rows of consecutive columns hit distinct banks)
int odd_quad(int need) {
    int b = (need + 3) & ~3;
    if (((b / 4) & 1) == 0) b += 4;
    return b;
}

bool plan_f32(int64_t I0, int K, F32Plan& p) {
    p.Kp = (K + 3) & ~3;
    p.TK = p.Kp <= 24 ? p.Kp : 16;
    p.nkb = (p.Kp + p.TK - 1) / p.TK;
    for (p.DS = 1; p.DS <= 8; ++p.DS) {
        int dt = (int)((I0 + p.DS - 1) / p.DS);
        dt = (dt + 3) & ~3;
        const int ndb = dt / 4;
        if (ndb * p.nkb > kF32Cons * 32) continue;
        p.NB = (dt + 255) / 256;
        p.DTB = odd_quad((dt + p.NB - 1) / p.NB);
        if (p.DTB > 256) {
            ++p.NB;
            p.DTB = odd_quad((dt + p.NB - 1) / p.NB);
        }
        p.DT = dt;
        p.ndb = ndb;
        p.G = (kF32Cons * 32) / (ndb * p.nkb);
        // ~32 KB stages, at most 256 columns per box
        p.CT = std::max(4, std::min(256, (int)(32768 / (4 * p.NB * p.DTB)) & ~3));
        p.BS = (p.CT * p.DTB + 31) & ~31;
        p.smem = (size_t)kF32Stages * p.NB * p.BS * 4 + (size_t)kF32OB * p.CT * p.Kp * 4 + 256;
        const size_t red = p.G > 1 ? (size_t)p.DT * p.Kp * 8 : 0;  // G > 1: group reduction scratch
        if (red > (size_t)kF32Stages * p.NB * p.BS * 4) p.smem += red;
        return p.smem <= 220 * 1024;
    }
    return false;
}

}  // namespace

bool stream_sketch_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols) {
    F32Plan p;
    return dtype == F32 && left == 1 && (dim % 4) == 0 && K <= 64 && ncols < (int64_t(1) << 31) && encode_fn() &&
           plan_f32(dim, K, p);
}

int stream_sketch_f32_grid(int64_t dim, int K, int64_t ncols, int num_sms, int* gc) {
    F32Plan p;
    plan_f32(dim, K, p);
    const int64_t ntiles = (ncols + p.CT - 1) / p.CT;
    *gc = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, num_sms / p.DS));
    return *gc * p.DS;
}

int launch_stream_sketch_f32(const SketchPlan& sp, const void* x, double* partial, double* y, int num_sms,
                              cudaStream_t s) {
    F32Plan p;
    plan_f32(sp.dim, sp.K, p);
    F32SkArgs a{};
    a.I0 = sp.dim;
    a.L = sp.right;
    a.DT = p.DT;
    a.DTB = p.DTB;
    a.NB = p.NB;
    a.CT = p.CT;
    a.BS = p.BS;
    a.DS = p.DS;
    a.K = sp.K;
    a.Kp = p.Kp;
    a.TK = p.TK;
    a.nkb = p.nkb;
    a.ndb = p.ndb;
    a.G = p.G;
    a.ntiles = (sp.right + p.CT - 1) / p.CT;
    a.seed = sp.seed;
    a.D = sp.D;
    a.rows_glob = sp.rows_glob;
    a.col_off = sp.col_off;
    a.partial = partial;
    CUtensorMap map;
    const cuuint64_t gdim[2] = {(cuuint64_t)sp.dim, (cuuint64_t)sp.right};
    const cuuint64_t gstride[1] = {(cuuint64_t)sp.dim * 4};
    const cuuint32_t box[2] = {(cuuint32_t)p.DTB, (cuuint32_t)p.CT};
    const cuuint32_t estride[2] = {1, 1};
    encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(x), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int gc = 0;
    const int grid = stream_sketch_f32_grid(sp.dim, sp.K, sp.right, num_sms, &gc);
    cudaMemsetAsync(partial, 0, sizeof(double) * gc * sp.dim * sp.K, s);
#define TRG_F32(TKV)                                                                                          \
    do {                                                                                                      \
        constexpr int G = TKV <= 12 ? TRG_F32_GEN_SMALL : TRG_F32_GEN_LARGE;                                  \
        allow_smem(k_sketch_l1_f32<TKV, G>, p.smem); \
        k_sketch_l1_f32<TKV, G><<<grid, (kF32Cons + G + 1) * 32, p.smem, s>>>(map, a);                        \
    } while (0)
    if (p.nkb > 1) {  // several k-blocks per tile: the Box-Muller generation is the bound
        constexpr int G = TRG_F32_GEN_MULTI;
        allow_smem(k_sketch_l1_f32<16, G>, p.smem);
        k_sketch_l1_f32<16, G><<<grid, (kF32Cons + G + 1) * 32, p.smem, s>>>(map, a);
        if (y) launch_reduce_partials(partial, gc, sp.dim * sp.K, y, s);
        return gc;
    }
    switch (p.TK) {
        case 4: TRG_F32(4); break;
        case 8: TRG_F32(8); break;
        case 12: TRG_F32(12); break;
        case 16: TRG_F32(16); break;
        case 20: TRG_F32(20); break;
        default: TRG_F32(24); break;
    }
#undef TRG_F32
    if (y) launch_reduce_partials(partial, gc, sp.dim * sp.K, y, s);
    return gc;
}

// outputs per CTA: all of them up to 24; beyond (C4's K_0 = 64) groups of 16 on grid.y, whose CTAs
// walk the same fibre units at the same time so the repeated X tiles come from L2
int ttm_f32_kp(int64_t K) { return K <= 24 ? (int)((K + 3) & ~3) : 16; }

bool stream_ttm_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols) {
    if (dtype != F32 || left != 1 || (dim % 4) != 0 || K > 128 || ncols >= (int64_t(1) << 31) || !encode_fn())
        return false;
    const int DC = odd_quad(std::min<int>(60, (int)dim));
    const int NCH = (int)((dim + DC - 1) / DC);
    const int Kp = ttm_f32_kp(K);
    const size_t smem = (size_t)kTtStages * 64 * DC * 4 + (size_t)NCH * DC * Kp * 4 + 256;
    return smem <= 220 * 1024;
}

void launch_stream_ttm_f32(const TTMPlan& p, const void* in, void* out, bool f64_out, const double* q, int64_t ldq,
                           int num_sms, cudaStream_t s) {
    F32TtArgs a{};
    a.I0 = p.dim;
    a.L = p.right;
    a.DC = odd_quad(std::min<int>(60, (int)p.dim));
    a.NCH = (int)((p.dim + a.DC - 1) / a.DC);
    a.K = (int)p.odim;
    a.Kp = ttm_f32_kp(p.odim);
    a.nunits = (p.right + 63) / 64;
    a.out = out;
    a.f64out = f64_out ? 1 : 0;
    CUtensorMap map;
    const cuuint64_t gdim[2] = {(cuuint64_t)p.dim, (cuuint64_t)p.right};
    const cuuint64_t gstride[1] = {(cuuint64_t)p.dim * 4};
    const cuuint32_t box[2] = {(cuuint32_t)a.DC, 64u};
    const cuuint32_t estride[2] = {1, 1};
    encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(in), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = (size_t)kTtStages * 64 * a.DC * 4 + (size_t)a.NCH * a.DC * a.Kp * 4 + 256;
    const int groups = (int)((a.K + a.Kp - 1) / a.Kp);
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(a.nunits, std::max(1, num_sms / groups)));
    const dim3 grid(gx, groups);
    const int threads = (kTtCons + 1) * 32;
#define TRG_TT(KPV)                                                                                     \
    do {                                                                                                \
        allow_smem(k_ttm_l1_f32<KPV>, smem); \
        k_ttm_l1_f32<KPV><<<grid, threads, smem, s>>>(map, a, q, ldq);                                  \
    } while (0)
    switch (a.Kp) {
        case 4: TRG_TT(4); break;
        case 8: TRG_TT(8); break;
        case 12: TRG_TT(12); break;
        case 16: TRG_TT(16); break;
        case 20: TRG_TT(20); break;
        default: TRG_TT(24); break;
    }
#undef TRG_TT
}

}  // namespace trg
