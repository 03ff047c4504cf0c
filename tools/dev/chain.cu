// SPDX-License-Identifier: Apache-2.0
//
// K6: the first two contractions of the fused variant's shrink chain in one pass over X
// (north_star (3): the largest contraction first from HBM, the intermediate on chip).
//
// The fused variant sketches every mode from the original X and only then runs the
// shrink chain P = X x_0 Q_0^T x_1 Q_1^T ... (sketch.hpp:85 -> tensor.hpp:193-207), so Q_0 and Q_1
// are both known before the chain starts. For an fp32 X whose (I_0 x I_1) planes are small
// (C5: 60 x 60), one kernel computes
//     P^(2)(k0, k1, r) = sum_{i, j} Q_0(i, k0) Q_1(j, k1) X(i, j, r)
// plane by plane, so P^(1) (C5: 622 MB written and read again) never reaches HBM:
//     step A  T = X_r Q_1 (I_0 x K_1): lane = rows i = lane, lane + 32 of the plane, read straight
//             from global memory (coalesced along i), Q_1 rows broadcast from shared memory;
//     step B  Z = Q_0^T T (K_0 x K_1): T through a per-warp shared tile, lanes = (4 x 4 output tile,
//             contraction split) summed by shuffles in a fixed order.
// A warp owns whole planes (no CTA barrier in the loop); fp32 arithmetic as the fp32 shrinks
// (sums of <= 64 terms per step, far inside the 1e-4 bound). The contraction order (mode 1 first)
// differs from the sequential chain's, which changes only the rounding.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "pipeline.cuh"

namespace trg {

namespace {

constexpr int kC1Warps = 8;
constexpr int kC1Ch = 16;     // X columns per register batch
constexpr int kC1MaxI = 64;   // I_0, I_1 <= 64: two rows of a plane per lane
constexpr int kC1MaxK = 16;   // K_0, K_1 <= 16

struct Chain01Args {
    const float* x;
    const double* q0;  // I0 x K0 column-major (ld I0)
    const double* q1;  // I1 x K1 column-major (ld I1)
    float* out;        // K0 x K1 x R
    int I0, I1, K0, K1, KP0, KP1;
    int64_t R;
};

template <int KP1>
__global__ void __launch_bounds__(kC1Warps * 32, 2) k_chain01_f32(Chain01Args a) {
    extern __shared__ __align__(16) float c1s[];
    float* Q0s = c1s;                             // [I0][KP0], zero beyond K0
    float* Q1s = Q0s + kC1MaxI * kC1MaxK;         // [I1][KP1]
    float* Ts = Q1s + kC1MaxI * kC1MaxK;          // per warp [I0][KP1]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    griddep_wait();  // Q_0 and Q_1 come from the QR launches just before
    for (int e = tid; e < a.I0 * a.KP0; e += blockDim.x) {
        const int i = e / a.KP0, k = e - i * a.KP0;
        Q0s[e] = k < a.K0 ? (float)a.q0[i + (int64_t)a.I0 * k] : 0.f;
    }
    for (int e = tid; e < kC1MaxI * KP1; e += blockDim.x) {  // zero rows >= I1: step A's tail batch
        const int j = e / KP1, k = e - j * KP1;
        Q1s[e] = k < a.K1 && j < a.I1 ? (float)a.q1[j + (int64_t)a.I1 * k] : 0.f;
    }
    __syncthreads();
    float* T = Ts + warp * kC1MaxI * KP1;
    const int64_t plane = (int64_t)a.I0 * a.I1;
    const bool r0ok = lane < a.I0, r1ok = lane + 32 < a.I0;
    // step B lanes: 4 x 4 output tiles of Z, the i range split over the remaining lanes
    const int nt0 = a.KP0 / 4, nt1 = KP1 / 4, ntile = nt0 * nt1;
    const int nsplit = 32 / ntile;
    const int tile = lane % ntile, isp = lane / ntile;
    const int tk0 = 4 * (tile % nt0), tk1 = 4 * (tile / nt0);
    const bool bact = isp < nsplit;
    for (int64_t r = (int64_t)blockIdx.x * kC1Warps + warp; r < a.R; r += (int64_t)gridDim.x * kC1Warps) {
        const float* xr = a.x + plane * r;
        // ---- step A: T(i, :) = sum_j X(i, j) Q_1(j, :) for i = lane, lane + 32; X columns are
        // loaded kC1Ch at a time into registers first, so a warp has 2 * kC1Ch loads in flight
        float t0[KP1], t1[KP1];
#pragma unroll
        for (int k = 0; k < KP1; ++k) t0[k] = t1[k] = 0.f;
        for (int j0 = 0; j0 < a.I1; j0 += kC1Ch) {
            float xa[kC1Ch], xb[kC1Ch];
#pragma unroll
            for (int jj = 0; jj < kC1Ch; ++jj) {
                const bool jok = j0 + jj < a.I1;
                xa[jj] = r0ok && jok ? __ldg(xr + lane + (int64_t)a.I0 * (j0 + jj)) : 0.f;
                xb[jj] = r1ok && jok ? __ldg(xr + lane + 32 + (int64_t)a.I0 * (j0 + jj)) : 0.f;
            }
#pragma unroll
            for (int jj = 0; jj < kC1Ch; ++jj) {
                const float4* q = reinterpret_cast<const float4*>(Q1s + (j0 + jj) * KP1);
#pragma unroll
                for (int k4 = 0; k4 < KP1 / 4; ++k4) {
                    const float4 v = q[k4];
                    t0[4 * k4] = fmaf(xa[jj], v.x, t0[4 * k4]);
                    t0[4 * k4 + 1] = fmaf(xa[jj], v.y, t0[4 * k4 + 1]);
                    t0[4 * k4 + 2] = fmaf(xa[jj], v.z, t0[4 * k4 + 2]);
                    t0[4 * k4 + 3] = fmaf(xa[jj], v.w, t0[4 * k4 + 3]);
                    t1[4 * k4] = fmaf(xb[jj], v.x, t1[4 * k4]);
                    t1[4 * k4 + 1] = fmaf(xb[jj], v.y, t1[4 * k4 + 1]);
                    t1[4 * k4 + 2] = fmaf(xb[jj], v.z, t1[4 * k4 + 2]);
                    t1[4 * k4 + 3] = fmaf(xb[jj], v.w, t1[4 * k4 + 3]);
                }
            }
        }
        __syncwarp();  // the previous plane's step B has read T
#pragma unroll
        for (int k4 = 0; k4 < KP1 / 4; ++k4) {
            if (r0ok)
                reinterpret_cast<float4*>(T + lane * KP1)[k4] =
                    make_float4(t0[4 * k4], t0[4 * k4 + 1], t0[4 * k4 + 2], t0[4 * k4 + 3]);
            if (r1ok)
                reinterpret_cast<float4*>(T + (lane + 32) * KP1)[k4] =
                    make_float4(t1[4 * k4], t1[4 * k4 + 1], t1[4 * k4 + 2], t1[4 * k4 + 3]);
        }
        __syncwarp();
        // ---- step B: Z(k0, k1) = sum_i Q_0(i, k0) T(i, k1)
        float z[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) z[u][v] = 0.f;
        if (bact) {
            for (int i = isp; i < a.I0; i += nsplit) {
                const float4 qa = *reinterpret_cast<const float4*>(Q0s + i * a.KP0 + tk0);
                const float4 tb = *reinterpret_cast<const float4*>(T + i * KP1 + tk1);
                const float qv[4] = {qa.x, qa.y, qa.z, qa.w}, tv[4] = {tb.x, tb.y, tb.z, tb.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) z[u][v] = fmaf(qv[u], tv[v], z[u][v]);
            }
        }
        // sum the contraction splits (lanes tile + ntile s) in order s = 0, 1, ...
        for (int s = 1; s < nsplit; ++s) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float o = __shfl_down_sync(0xffffffffu, z[u][v], s * ntile);
                    if (isp == 0) z[u][v] += o;
                }
        }
        if (isp == 0 && lane < ntile) {
            float* o = a.out + (int64_t)a.K0 * a.K1 * r;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    if (tk0 + u < a.K0 && tk1 + v < a.K1) o[(tk0 + u) + a.K0 * (tk1 + v)] = z[u][v];
        }
    }
}

size_t chain01_smem(int KP1) {
    return sizeof(float) * ((size_t)2 * kC1MaxI * kC1MaxK + (size_t)kC1Warps * kC1MaxI * KP1);
}

}  // namespace

bool chain01_f32_ok(int dtype, int64_t I0, int64_t I1, int64_t K0, int64_t K1, int64_t R) {
    if (getenv("TRG_NO_CHAIN01")) return false;
    return dtype == F32 && I0 >= 1 && I1 >= 1 && I0 <= kC1MaxI && I1 <= kC1MaxI && K0 >= 1 && K1 >= 1 &&
           K0 <= kC1MaxK && K1 <= kC1MaxK && K0 < I0 && K1 < I1 && R >= 1 && R < (int64_t(1) << 40);
}

void launch_chain01_f32(const void* x, int64_t I0, int64_t I1, int64_t R, const double* q0, int64_t K0,
                        const double* q1, int64_t K1, void* out, int num_sms, cudaStream_t s) {
    if (!chain01_f32_ok(F32, I0, I1, K0, K1, R)) throw std::runtime_error("chain01: unsupported shape");
    Chain01Args a{};
    a.x = reinterpret_cast<const float*>(x);
    a.q0 = q0;
    a.q1 = q1;
    a.out = reinterpret_cast<float*>(out);
    a.I0 = (int)I0;
    a.I1 = (int)I1;
    a.K0 = (int)K0;
    a.K1 = (int)K1;
    a.KP0 = (int)((K0 + 3) & ~3);
    a.KP1 = (int)((K1 + 3) & ~3);
    a.R = R;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((R + kC1Warps - 1) / kC1Warps, (int64_t)num_sms * 4));
    auto go = [&](auto kern) {
        const size_t smem = chain01_smem(a.KP1);
        allow_smem(kern, smem);
        pdl_launch(kern, dim3(grid), dim3(kC1Warps * 32), smem, s, a);
    };
    switch (a.KP1) {
        case 4: go(k_chain01_f32<4>); break;
        case 8: go(k_chain01_f32<8>); break;
        case 12: go(k_chain01_f32<12>); break;
        default: go(k_chain01_f32<16>); break;
    }
}

}  // namespace trg
