// SPDX-License-Identifier: Apache-2.0
//
// K2 / K7: mode-n product out = in x_n M on the (left, dim, right) view.
//
// Reference: mode_n_product (tensor.hpp:193-207), called with M = Q_n^T to
// shrink the working tensor (sketch.hpp:85) and with M = Q_n to lift a small
// core along its physical mode (back_project, sketch.hpp:119). The reference
// runs one (left x dim)(dim x odim) GEMM per right-slab; here the rows
// m = (l, r) of all slabs form one GEMM out[m, o] = sum_d in[m, d] M(o, d),
// tiled MT rows x OT outputs per CTA with DT-wide chunks of the contraction
// staged in shared memory, so a mode-0 shrink is a single streaming pass.
#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"

namespace trg {

namespace {

struct TTMArgs {
    const void* in;
    void* out;
    const double* m;
    int64_t left, dim, odim, rows, m_so, m_sd, nrowtiles;
    int MT, DT, nm, no, OT;
    FastDiv left_div;
    int64_t dlen;   // contraction range per grid.z slice (split-d for few row tiles)
    double* part;   // split-d: fp64 partial outputs [gridDim.z][rows * odim] in the output layout
};

template <typename T, int TM, int TO, bool LEFT1>
__global__ void __launch_bounds__(256) k_ttm(TTMArgs a) {
    using A = typename Acc<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int DT = 32;  // contraction chunk (plan_ttm sets a.DT = 32)
    const int MT = a.MT, OT = a.OT;
    const int MTp = MT + 1;
    T* Xs = reinterpret_cast<T*>(smem_raw);              // [DT][MT+1]
    T* Ms = Xs + ((DT * MTp + 3) & ~3);                   // [DT][OT]
    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    const int mg = tid % a.nm;
    const int og = tid / a.nm;
    const int64_t o0 = (int64_t)blockIdx.y * OT;
    const T* in = reinterpret_cast<const T*>(a.in);
    T* out = reinterpret_cast<T*>(a.out);

    for (int64_t rt = blockIdx.x; rt < a.nrowtiles; rt += gridDim.x) {
        const int64_t m0 = rt * MT;
        A acc[TM][TO];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TO; ++j) acc[i][j] = A(0);

        const int64_t d_lo = (int64_t)blockIdx.z * a.dlen;
        const int64_t d_hi = d_lo + a.dlen < a.dim ? d_lo + a.dlen : a.dim;
        for (int64_t d0 = d_lo; d0 < d_hi; d0 += DT) {
            __syncthreads();
            if (LEFT1) {
                // rows are contiguous runs of dim elements: threads sweep d fastest
                for (int e = tid; e < MT * DT; e += nthreads) {
                    const int mm = e / DT;
                    const int dd = e - mm * DT;
                    const int64_t m = m0 + mm, d = d0 + dd;
                    T v = T(0);
                    if (m < a.rows && d < d_hi) v = __ldcs(in + d + a.dim * m);
                    Xs[dd * MTp + mm] = v;
                }
            } else {
                // rows (l, r) with l fastest: threads sweep l (contiguous) fastest
                for (int e = tid; e < MT * DT; e += nthreads) {
                    const int dd = e / MT;
                    const int mm = e - dd * MT;
                    const int64_t m = m0 + mm, d = d0 + dd;
                    T v = T(0);
                    if (m < a.rows && d < d_hi) {
                        const uint32_t r = a.left_div.div((uint32_t)m);
                        const int64_t l = m - (int64_t)r * a.left;
                        v = __ldcs(in + l + a.left * (d + a.dim * (int64_t)r));
                    }
                    Xs[dd * MTp + mm] = v;
                }
            }
            for (int e = tid; e < DT * OT; e += nthreads) {
                const int dd = e / OT;
                const int oo = e - dd * OT;
                const int64_t d = d0 + dd, o = o0 + oo;
                Ms[dd * OT + oo] = (d < d_hi && o < a.odim) ? T(a.m[o * a.m_so + d * a.m_sd]) : T(0);
            }
            __syncthreads();
            const int dlim = (d_hi - d0) < DT ? (int)(d_hi - d0) : DT;
            for (int dd = 0; dd < dlim; ++dd) {
                T xv[TM], mv[TO];
#pragma unroll
                for (int i = 0; i < TM; ++i) xv[i] = Xs[dd * MTp + mg + a.nm * i];
#pragma unroll
                for (int j = 0; j < TO; ++j) mv[j] = Ms[dd * OT + og * TO + j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TO; ++j) acc[i][j] = fma(A(xv[i]), A(mv[j]), acc[i][j]);
            }
        }
        // ---- store: out(l, o, r) at l + left*(o + odim*r)
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t m = m0 + mg + a.nm * i;
            if (m >= a.rows) continue;
            int64_t base, ostride;  // output layout: out(l, o, r) at l + left*(o + odim*r)
            if (LEFT1) {
                base = a.odim * m;
                ostride = 1;
            } else {
                const uint32_t r = a.left_div.div((uint32_t)m);
                const int64_t l = m - (int64_t)r * a.left;
                base = l + a.left * a.odim * (int64_t)r;
                ostride = a.left;
            }
            if (a.part) {
                double* dst = a.part + (int64_t)blockIdx.z * a.rows * a.odim + base;
#pragma unroll
                for (int j = 0; j < TO; ++j) {
                    const int64_t o = o0 + og * TO + j;
                    if (o < a.odim) dst[ostride * o] = (double)acc[i][j];
                }
            } else {
                T* dst = out + base;
#pragma unroll
                for (int j = 0; j < TO; ++j) {
                    const int64_t o = o0 + og * TO + j;
                    if (o < a.odim) dst[ostride * o] = T(acc[i][j]);
                }
            }
        }
    }
}

template <typename T, int TM, int TO, bool L1>
void run(const TTMPlan& p, const TTMArgs& a, cudaStream_t s) {
    allow_smem(k_ttm<T, TM, TO, L1>, p.smem);
    dim3 grid(p.grid_x, p.noT, p.dsplit);
    k_ttm<T, TM, TO, L1><<<grid, p.threads, p.smem, s>>>(a);
}

template <typename T, int TM, int TO>
void run_l(const TTMPlan& p, const TTMArgs& a, cudaStream_t s) {
    if (p.left == 1) run<T, TM, TO, true>(p, a, s);
    else run<T, TM, TO, false>(p, a, s);
}

}  // namespace

void plan_ttm(TTMPlan& p, int num_sms) {
    p.TM = 4;
    p.TO = p.odim >= 8 ? 8 : 4;
    p.rows = p.left * p.right;
    if (p.left > 1 && p.rows >= (int64_t(1) << 32)) throw std::runtime_error("ttm: row count exceeds 2^32");
    // output columns per CTA: all of odim when it fits, else o-tiles on grid.y
    p.no = (int)std::min<int64_t>((p.odim + p.TO - 1) / p.TO, 8);
    p.OT = p.no * p.TO;
    p.noT = (int)((p.odim + p.OT - 1) / p.OT);
    // MT*DT*sizeof(T) ~ 64 KB of staged input per CTA
    const int nm_cap = p.dtype == F64 ? 64 : 128;
    p.nm = std::max(32, std::min(nm_cap, 256 / p.no));
    // shrink nm for tiny row counts
    while (p.nm > 32 && (int64_t)p.nm * p.TM / 2 >= p.rows) p.nm /= 2;
    p.MT = p.nm * p.TM;
    p.threads = p.nm * p.no;
    p.DT = 32;
    p.nrowtiles = (p.rows + p.MT - 1) / p.MT;
    const size_t es = dtype_size(p.dtype);
    const size_t xs = ((size_t)p.DT * (p.MT + 1) + 3) & ~size_t(3);
    p.smem = (xs + (size_t)p.DT * p.OT) * es;
    const int per_sm = std::max(1, std::min(8, (int)((200 * 1024) / p.smem)));
    const int64_t want = (int64_t)num_sms * per_sm / std::max(1, p.noT);
    p.grid_x = (int)std::max<int64_t>(1, std::min<int64_t>(p.nrowtiles, want));
    // few row tiles and a long contraction: split d over grid.z (fp64 partials, fixed-order sum)
    p.dsplit = 1;
    const int64_t ctas = (int64_t)p.grid_x * p.noT;
    if (ctas < num_sms && p.dim >= 256) {
        const int64_t byd = std::max<int64_t>(1, p.dim / 128);
        p.dsplit = (int)std::max<int64_t>(1, std::min<int64_t>(byd, (2 * (int64_t)num_sms + ctas - 1) / ctas));
    }
}

void launch_ttm(const TTMPlan& p, const void* in, void* out, const double* m, cudaStream_t s) {
    TTMArgs a;
    a.in = in;
    a.out = out;
    a.m = m;
    a.left = p.left;
    a.dim = p.dim;
    a.odim = p.odim;
    a.rows = p.rows;
    a.m_so = p.m_so;
    a.m_sd = p.m_sd;
    a.nrowtiles = p.nrowtiles;
    a.MT = p.MT;
    a.DT = p.DT;
    a.nm = p.nm;
    a.no = p.no;
    a.OT = p.OT;
    a.left_div = FastDiv((uint32_t)std::max<int64_t>(1, std::min<int64_t>(p.left, 0xFFFFFFFFll)));
    a.dlen = ((p.dim + p.dsplit - 1) / p.dsplit + 31) / 32 * 32;
    a.part = nullptr;
    const int64_t nout = p.rows * p.odim;
    if (p.dsplit > 1) a.part = (double*)scratch_alloc(sizeof(double) * nout * p.dsplit, s);
    if (p.dtype == F64) {
        if (p.TO == 8) run_l<double, 4, 8>(p, a, s);
        else run_l<double, 4, 4>(p, a, s);
    } else {
        if (p.TO == 8) run_l<float, 4, 8>(p, a, s);
        else run_l<float, 4, 4>(p, a, s);
    }
    if (p.dsplit > 1) {  // fixed-order sum of the d-slices (bit-reproducible)
        if (p.dtype == F64) {
            launch_reduce_partials(a.part, p.dsplit, nout, reinterpret_cast<double*>(out), s);
        } else {
            double* tmp = nullptr;
            tmp = (double*)scratch_alloc(sizeof(double) * nout, s);
            launch_reduce_partials(a.part, p.dsplit, nout, tmp, s);
            launch_convert(tmp, F64, out, F32, nout, s);
            scratch_free(tmp, s);
        }
        scratch_free(a.part, s);
    }
}

}  // namespace trg
