// SPDX-License-Identifier: Apache-2.0
//
// K1 sketch: Y_n = P^(n)_(n) * Omega_n with Omega_n regenerated on the fly
// from the reference's counter-addressable SplitMix64/Box-Muller stream.
//
// Reference: sketch.hpp:80-83 (unfold_classic, gaussian_matrix, GEMM) and
// sketch.hpp:32-38 (column-major fill of the test matrix from one stream).
// The mode-n unfolding is never materialised: column c = l + left*r of
// X_(n) lives at l + left*(d + dim*r) (tensor.hpp:133-142).
//
// Dataflow per CTA (persistent over column tiles, split-K over columns):
//   load X tile (DT rows x CT columns) -> smem, regenerate Omega(CT x K) ->
//   smem, register-tiled FMA into TD x TK accumulators per thread, G thread
//   groups split the tile's columns. At the end the groups are summed in a
//   fixed order and each CTA writes one dim x K fp64 partial; a second kernel
//   sums the partials in CTA order, so the result is bit-reproducible.
#include <algorithm>
#include <mutex>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "pipeline.cuh"
#include "launch.h"

namespace trg {

namespace {

struct SketchArgs {
    const void* x;
    int64_t left, dim, ncols;
    int K, Kp, DT, CT, nd, nk, G, ndt;
    uint64_t seed, D;
    int64_t rows_glob, col_off, ntiles;
    double* partial;
    FastDiv left_div, dt_div;
};

template <typename T, int TD, int TK, bool LEFT1>
__global__ void __launch_bounds__(256) k_sketch(SketchArgs a) {
    using A = typename Acc<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int DT = a.DT, CT = a.CT, Kp = a.Kp;
    // LEFT1: Xs[cc][dd] (d contiguous, matches global); else Xs[dd][cc] padded to CT+1
    const int xs_elems = LEFT1 ? CT * DT : DT * (CT + 1);
    T* Xs = reinterpret_cast<T*>(smem_raw);
    T* Os = Xs + ((xs_elems + 3) & ~3);  // Omega tile [cc][Kp], 16B aligned
    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    const int tpg = a.nd * a.nk;
    const int g = tid / tpg;
    const int w = tid - g * tpg;
    const int dg = w % a.nd;
    const int kg = w / a.nd;
    const bool computing = g < a.G;
    const int64_t d0 = (int64_t)blockIdx.y * DT;
    const T* x = reinterpret_cast<const T*>(a.x);

    for (int i = tid; i < CT * Kp; i += nthreads) Os[i] = T(0);

    A acc[TD][TK];
#pragma unroll
    for (int i = 0; i < TD; ++i)
#pragma unroll
        for (int j = 0; j < TK; ++j) acc[i][j] = A(0);

    const int npmax = CT / 2 + 1;
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const int64_t c0 = t * CT;
        __syncthreads();  // previous tile fully consumed
        // ---- X tile
        if (LEFT1) {
            for (int e = tid; e < CT * DT; e += nthreads) {
                const int cc = (int)a.dt_div.div((uint32_t)e);
                const int dd = e - cc * DT;
                const int64_t c = c0 + cc, d = d0 + dd;
                T v = T(0);
                if (c < a.ncols && d < a.dim) v = __ldcs(x + d + a.dim * c);
                Xs[cc * DT + dd] = v;
            }
        } else {
            for (int e = tid; e < CT * DT; e += nthreads) {
                const int dd = e / CT;
                const int cc = e - dd * CT;
                const int64_t c = c0 + cc, d = d0 + dd;
                T v = T(0);
                if (c < a.ncols && d < a.dim) {
                    const uint32_t r = a.left_div.div((uint32_t)c);
                    const int64_t l = c - (int64_t)r * a.left;
                    v = __ldcs(x + l + a.left * (d + a.dim * (int64_t)r));
                }
                Xs[dd * (CT + 1) + cc] = v;
            }
        }
        // ---- Omega tile: draws D + col_off + c + rows_glob*k, pairs shared
        for (int it = tid; it < a.K * npmax; it += nthreads) {
            const int k = it / npmax;
            const int j = it - k * npmax;
            const uint64_t s = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)k;
            const uint64_t p = (s >> 1) + (uint64_t)j;
            if (p > ((s + (uint64_t)CT - 1ull) >> 1)) continue;
            T z0, z1;
            gauss_pair(a.seed, p, z0, z1);
            const int64_t cc0 = (int64_t)(2ull * p - s);
            if (cc0 >= 0 && cc0 < CT) Os[cc0 * Kp + k] = z0;
            if (cc0 + 1 >= 0 && cc0 + 1 < CT) Os[(cc0 + 1) * Kp + k] = z1;
        }
        __syncthreads();
        // ---- FMA
        if (computing) {
            for (int cc = g; cc < CT; cc += a.G) {
                T xv[TD], ov[TK];
#pragma unroll
                for (int i = 0; i < TD; ++i)
                    xv[i] = LEFT1 ? Xs[cc * DT + dg + a.nd * i] : Xs[(dg + a.nd * i) * (CT + 1) + cc];
#pragma unroll
                for (int j = 0; j < TK; ++j) ov[j] = Os[cc * Kp + kg * TK + j];
#pragma unroll
                for (int i = 0; i < TD; ++i)
#pragma unroll
                    for (int j = 0; j < TK; ++j) acc[i][j] = fma(A(xv[i]), A(ov[j]), acc[i][j]);
            }
        }
    }
    // ---- fixed-order reduction of the G groups, then one fp64 partial per CTA
    __syncthreads();
    double* red = reinterpret_cast<double*>(smem_raw);  // DT x Kp doubles
    const int red_elems = DT * Kp;
    for (int gg = 0; gg < a.G; ++gg) {
        if (computing && g == gg) {
#pragma unroll
            for (int i = 0; i < TD; ++i)
#pragma unroll
                for (int j = 0; j < TK; ++j) {
                    const int dd = dg + a.nd * i;
                    const int k = kg * TK + j;
                    if (dd < DT) {
                        double* slot = red + dd + DT * k;
                        *slot = (gg == 0 ? 0.0 : *slot) + (double)acc[i][j];
                    }
                }
        }
        __syncthreads();
    }
    double* out = a.partial + (int64_t)blockIdx.x * a.dim * a.K;
    for (int e = tid; e < red_elems; e += nthreads) {
        const int k = e / DT;
        const int dd = e - k * DT;
        const int64_t d = d0 + dd;
        if (k < a.K && d < a.dim) out[d + a.dim * k] = red[dd + DT * k];
    }
}

// out[i] = sum_b partial[b][i]: a CTA owns 32 consecutive outputs (one per lane),
// its 8 warps stride over the partials (b = w, w + 8, ...), and the 8 warp sums
// are combined in warp order — a fixed summation tree, so the result does not
// depend on scheduling.
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ partial, int nblocks, int64_t n,
                                                         double* __restrict__ out) {
    __shared__ double red[8][32];
    griddep_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    double s = 0.0;
    if (i < n) {
#pragma unroll 4
        for (int b = warp; b < nblocks; b += 8) s += partial[(int64_t)b * n + i];
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && i < n) {
        double t = red[0][lane];
        for (int w = 1; w < 8; ++w) t += red[w][lane];
        out[i] = t;
    }
}

// Split-K reduction spread over many SMs: CTA c owns kRwUnits units (pairs of entries when the
// partial blocks allow 16-byte loads); its threads split the partials into kRwGroups strided
// groups, issue all of their loads, and the groups are summed in a fixed order.
constexpr int kRwThreads = 256, kRwUnits = 8, kRwGroups = kRwThreads / kRwUnits;
__global__ void __launch_bounds__(kRwThreads) k_reduce_wide(const double* __restrict__ partial, int nparts, int64_t n,
                                                            int vec, double* __restrict__ out) {
    __shared__ double2 red[kRwGroups][kRwUnits];
    griddep_wait();
    const int w = threadIdx.x % kRwUnits, g = threadIdx.x / kRwUnits;
    const int64_t u = (int64_t)blockIdx.x * kRwUnits + w;
    const int64_t nu = vec ? n / 2 : n;
    double2 sacc = make_double2(0.0, 0.0);
    if (u < nu) {
        if (vec) {
            const double2* pp = reinterpret_cast<const double2*>(partial) + u;
#pragma unroll 8
            for (int b = g; b < nparts; b += kRwGroups) {
                const double2 v = pp[(int64_t)b * (n / 2)];
                sacc.x += v.x;
                sacc.y += v.y;
            }
        } else {
#pragma unroll 8
            for (int b = g; b < nparts; b += kRwGroups) sacc.x += partial[(int64_t)b * n + u];
        }
    }
    red[g][w] = sacc;
    __syncthreads();
    if (g == 0 && u < nu) {
        double2 t = red[0][w];
        for (int g2 = 1; g2 < kRwGroups; ++g2) {
            t.x += red[g2][w].x;
            t.y += red[g2][w].y;
        }
        if (vec) {
            out[2 * u] = t.x;
            out[2 * u + 1] = t.y;
        } else {
            out[u] = t.x;
        }
    }
}

// zero n ints as a kernel in the programmatic-launch chain (a memset node between the previous
// projection's last kernel and this one's first would cut the chain)
__global__ void k_zero_ints(int* p, int n) {
    griddep_wait();  // stream order with the previous kernel (which may still read the arena)
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

__global__ void k_gauss_tables(GaussTables* t) {
    const int i = threadIdx.x;
    if (i < 128) {
        const double c = 1.0 + (i + 0.5) / 128.0;
        t->logt[i] = make_double2(1.0 / c, log(c));
    }
    if (i < 256) {
        double sn, cs;
        sincospi(2.0 * (i + 0.5) / 256.0, &sn, &cs);
        t->sct[i] = make_double2(sn, cs);
    }
    if (i < 64) {
        const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
        const double ef = (double)(i - 53);
        t->elog[i] = make_double2(ef * ln2_hi, ef * ln2_lo);
    }
}

// the same table-driven generator the streaming kernels use, so the exported
// test matrix is exactly what the sketches multiply by
__global__ void k_omega(uint64_t seed, uint64_t off, int64_t n, double* out, const GaussTables* gt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t d = off + (uint64_t)i;
        double z0, z1;
        gauss_pair_tab(seed, d >> 1, *gt, z0, z1);
        out[i] = (d & 1ull) ? z1 : z0;
    }
}

template <typename T, int TD, int TK, bool L1>
void set_smem_attr(size_t smem) {
    allow_smem(k_sketch<T, TD, TK, L1>, smem);
}

template <typename T, int TD, int TK>
void dispatch(const SketchPlan& p, const SketchArgs& a, cudaStream_t s) {
    dim3 grid(p.grid_x, p.ndt);
    if (p.left == 1) {
        set_smem_attr<T, TD, TK, true>(p.smem);
        k_sketch<T, TD, TK, true><<<grid, p.threads, p.smem, s>>>(a);
    } else {
        set_smem_attr<T, TD, TK, false>(p.smem);
        k_sketch<T, TD, TK, false><<<grid, p.threads, p.smem, s>>>(a);
    }
}

}  // namespace

void plan_sketch(SketchPlan& p, int num_sms) {
    const bool f64 = p.dtype == F64;
    p.TD = 4;
    p.TK = (p.K >= 16 || (!f64 && p.K > 8)) ? 8 : 4;
    p.Kp = (p.K + p.TK - 1) / p.TK * p.TK;
    p.nk = p.Kp / p.TK;
    // rows per d-tile: whole mode when it fits the register budget
    const int max_rows = 128;
    p.DT = (int)std::min<int64_t>(((p.dim + p.TD - 1) / p.TD) * p.TD, max_rows);
    p.nd = p.DT / p.TD;
    p.ndt = (int)((p.dim + p.DT - 1) / p.DT);
    const int tpg = p.nd * p.nk;
    if (tpg > 256) throw std::runtime_error("sketch: tile too large for one CTA");
    p.G = std::max(1, std::min(8, 256 / tpg));
    p.threads = p.G * tpg;
    p.CT = 32;
    p.ncols = p.left * p.right;
    p.ntiles = (p.ncols + p.CT - 1) / p.CT;
    const size_t es = dtype_size(p.dtype);
    const size_t xs = (size_t)(p.left == 1 ? p.CT * p.DT : p.DT * (p.CT + 1));
    const size_t xs_al = (xs + 3) & ~size_t(3);
    size_t smem = (xs_al + (size_t)p.CT * p.Kp) * es;
    smem = std::max(smem, (size_t)p.DT * p.Kp * sizeof(double));
    p.smem = smem;
    const int per_sm = std::max(1, std::min(8, (int)((200 * 1024) / std::max<size_t>(smem, 1))));
    const int64_t want = (int64_t)num_sms * per_sm / std::max(1, p.ndt);
    p.grid_x = (int)std::max<int64_t>(1, std::min<int64_t>(p.ntiles, std::max<int64_t>(want, 1)));
    p.partial_elems = (size_t)p.grid_x * (size_t)p.dim * (size_t)p.K;
}

void launch_sketch(const SketchPlan& p, const void* x, double* partial, double* y, cudaStream_t s) {
    SketchArgs a;
    a.x = x;
    a.left = p.left;
    a.dim = p.dim;
    a.ncols = p.ncols;
    a.K = p.K;
    a.Kp = p.Kp;
    a.DT = p.DT;
    a.CT = p.CT;
    a.nd = p.nd;
    a.nk = p.nk;
    a.G = p.G;
    a.ndt = p.ndt;
    a.seed = p.seed;
    a.D = p.D;
    a.rows_glob = p.rows_glob;
    a.col_off = p.col_off;
    a.ntiles = p.ntiles;
    a.partial = partial;
    a.left_div = FastDiv((uint32_t)std::max<int64_t>(1, p.left));
    a.dt_div = FastDiv((uint32_t)p.DT);
    if (p.dtype == F64) {
        if (p.TK == 8) dispatch<double, 4, 8>(p, a, s);
        else dispatch<double, 4, 4>(p, a, s);
    } else {
        if (p.TK == 8) dispatch<float, 4, 8>(p, a, s);
        else dispatch<float, 4, 4>(p, a, s);
    }
    launch_reduce_partials(partial, p.grid_x, p.dim * p.K, y, s);
}

const GaussTables* gauss_tables(cudaStream_t s) {
    static std::mutex mu;
    static GaussTables* per_dev[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!per_dev[dev]) {
        GaussTables* t = nullptr;
        if (cudaMalloc(&t, sizeof(GaussTables)) != cudaSuccess) return nullptr;
        k_gauss_tables<<<1, 256, 0, s>>>(t);
        // other host threads (contexts on other streams) may read the tables as soon as they see
        // the pointer: finish building them first (once per device)
        if (cudaStreamSynchronize(s) != cudaSuccess) return nullptr;
        per_dev[dev] = t;
    }
    return per_dev[dev];
}

void launch_reduce_partials(const double* partial, int nblocks, int64_t n, double* out, cudaStream_t s) {
    const int blocks = (int)std::max<int64_t>(1, (n + 31) / 32);
    pdl_launch(k_reduce_partials, dim3(blocks), dim3(256), 0, s, partial, nblocks, n, out);
}

void launch_zero_ints(int* p, int n, cudaStream_t s) { pdl_launch(k_zero_ints, dim3(1), dim3(128), 0, s, p, n); }

void launch_reduce_wide(const double* partial, int nparts, int64_t n, double* out, cudaStream_t s) {
    const int vec = (n % 2 == 0) && (reinterpret_cast<uintptr_t>(partial) % 16 == 0);
    const int64_t nu = vec ? n / 2 : n;
    const int blocks = (int)std::max<int64_t>(1, (nu + kRwUnits - 1) / kRwUnits);
    pdl_launch(k_reduce_wide, dim3(blocks), dim3(kRwThreads), 0, s, partial, nparts, n, vec, out);
}

void launch_omega(uint64_t seed, uint64_t off, int64_t rows, int64_t cols, double* out, cudaStream_t s) {
    const int64_t n = rows * cols;
    const int threads = 256;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 4096));
    k_omega<<<blocks, threads, 0, s>>>(seed, off, n, out, gauss_tables(s));
}

}  // namespace trg
