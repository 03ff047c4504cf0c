// SPDX-License-Identifier: Apache-2.0
//
// Unit blocks of the reference test matrix for the TMA slab sketch (slab_tma.cu), as a CTA-level
// device routine: k_omega_units runs it on its own, k_cqr_fused runs it on the CTAs the QR's
// split-K reduce does not use (qr.cu), so the next mode's test matrix is ready before its sketch
// without a side-stream kernel next to the HBM-bound shrink.
//
// Block u = (r, lc), element (t, jn, lane) = Omega(c, k), c = 16 lc + 4 t + (lane & 3) (zero past
// `left`), k = 8 jn + (lane >> 2) (zero past K); Omega(c, k) = reference draw
// D + col_off + c + left r + rows_glob k (sketch.hpp:32-38).
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace trg {

constexpr int kOmegaUnitL = 16;                  // left-chunk width of a slab unit
constexpr int kOmegaPairs = kOmegaUnitL / 2 + 1;  // draw pairs covering 16 consecutive draws

// threads needed for one unit: one per (k < 8 NT, pair) slot
__host__ __device__ constexpr int omega_unit_slots(int NT) { return 8 * NT * kOmegaPairs; }

// Khatri-Rao factor B(r, k) = F(r mod S1, k) H(r / S1, k) (KrOmega); r < 2^32 (checked by the host)
__device__ __forceinline__ double kr_b(const KrOmega& kr, uint32_t r, int k) {
    const uint32_t q = r / (uint32_t)kr.S1, i = r - q * (uint32_t)kr.S1;
    return __ldg(kr.F + i + kr.S1 * k) * __ldg(kr.H + q + kr.nH * k);
}

// Khatri-Rao unit blocks: one thread per block element, rows c = col_off + 16 lc + l + left r
// (global), Omega(c, k) = A(16 lc + l, k) F(i1, k) H(q, k) with r + col_off / left = i1 + S1 q.
// A thread keeps its element and walks units at a fixed stride, so (r, lc) and (i1, q) advance by
// constants with one carry each: no division in the loop.
__device__ __forceinline__ void omega_units_kr_cta(const OmegaUnitsJob& j, int cta, int ncta) {
    const int per = 4 * j.NT * 32;
    const int upc = blockDim.x / per;
    const int us = threadIdx.x / per, e = threadIdx.x - us * per;
    if (us >= upc) return;
    const int lane = e & 31, jn = (e >> 5) % j.NT, t = (e >> 5) / j.NT;
    const int lu = 4 * t + (lane & 3), k = 8 * jn + (lane >> 2);
    const bool kon = k < j.K;
    const int kk = kon ? k : 0;
    const int64_t u0 = (int64_t)cta * upc + us, step = (int64_t)ncta * upc;
    if (u0 >= j.nunits) return;
    const int LC = j.LC;
    const int64_t S1 = j.kr.S1;
    int64_t r = u0 / LC;
    int lc = (int)(u0 - r * LC);
    const int64_t dr = step / LC;
    const int dlc = (int)(step - dr * LC);
    const int64_t rg = r + j.col_off / j.left;
    int64_t q = rg / S1;
    int64_t i1 = rg - q * S1;
    const int64_t dq = dr / S1, di = dr - (dr / S1) * S1;
    const double* Ak = j.kr.A + j.kr.left * kk;
    const double* Fk = j.kr.F + S1 * kk;
    const double* Hk = j.kr.H + j.kr.nH * kk;
    for (int64_t u = u0; u < j.nunits; u += step) {
        const int64_t l = (int64_t)kOmegaUnitL * lc + lu;
        double v = 0.0;
        if (kon && l < j.left) v = __ldg(Ak + l) * __ldg(Fk + i1) * __ldg(Hk + q);
        j.out[u * per + e] = v;
        // advance (r, lc) by (dr, dlc) and (i1, q) by r's increment
        int64_t rinc = dr;
        lc += dlc;
        if (lc >= LC) {
            lc -= LC;
            rinc += 1;
        }
        i1 += di + (rinc - dr);
        q += dq;
        if (i1 >= S1) {
            i1 -= S1;
            q += 1;
        }
    }
}

// CTA `cta` of `ncta` generates its share of j's units; every thread of the block takes part (the
// block holds blockDim.x / slots units per iteration). No 64-bit division in the per-draw path.
__device__ __forceinline__ void omega_units_cta(const OmegaUnitsJob& j, const GaussTables& tabs, int cta, int ncta) {
    if (j.kr.F) {
        omega_units_kr_cta(j, cta, ncta);
        return;
    }
    const int S = omega_unit_slots(j.NT);
    const int upc = blockDim.x / S;
    const int us = threadIdx.x / S, slot = threadIdx.x - us * S;
    if (us >= upc) return;
    const int k = slot / kOmegaPairs, jj = slot - k * kOmegaPairs;
    const int64_t step = (int64_t)ncta * upc;
    // two units per iteration: two independent Box-Muller chains per thread hide the fp64 latency
    for (int64_t u0 = (int64_t)cta * upc + us; u0 < j.nunits; u0 += 2 * step) {
        uint64_t s0[2], p[2];
        bool on[2];
        double z[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t u = u0 + h * step;
            const int64_t r = j.LC == 1 ? u : u / j.LC;
            const int lc = (int)(u - r * j.LC);
            s0[h] = j.D + (uint64_t)(j.col_off + kOmegaUnitL * lc + j.left * r) + (uint64_t)j.rows_glob * (uint64_t)k;
            p[h] = (s0[h] >> 1) + (uint64_t)jj;
            on[h] = u < j.nunits && p[h] <= ((s0[h] + kOmegaUnitL - 1) >> 1);
            z[h][0] = z[h][1] = 0.0;
        }
        if (k < j.K) {
#pragma unroll
            for (int h = 0; h < 2; ++h) gauss_pair_tab(j.seed, p[h], tabs, z[h][0], z[h][1]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!on[h]) continue;
            const int64_t u = u0 + h * step;
            const int lc = (int)(j.LC == 1 ? 0 : u % j.LC);
            double* blk = j.out + u * (int64_t)(4 * j.NT * 32);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int l = (int)(2ull * p[h] - s0[h]) + e;  // 0..15 within the unit
                if (l < 0 || l >= kOmegaUnitL) continue;
                const bool live = kOmegaUnitL * lc + l < j.left;
                blk[(((l >> 2) * j.NT + (k >> 3)) << 5) + (l & 3) + ((k & 7) << 2)] = live ? z[h][e] : 0.0;
            }
        }
    }
}

}  // namespace trg
