// SPDX-License-Identifier: Apache-2.0
//
// fp32 sketch and shrink for modes n >= 1 (left > 1), so fp32 inputs keep fp32 intermediates
// P^(n) (half the bytes of the former fp64 promotion) and large extents / K (C3's 1000-row modes
// with K = 20, C4's 1024 with K = 64) get register-tiled FFMA kernels instead of the generic
// scalar ones. The working tensor is read as (left, dim, right), l fastest (tensor.hpp:112-123).
//
//   shrink  (tensor.hpp:193-207, m = Q^T):  out(l, k, r) = sum_d P(l, d, r) Q(d, k)
//     CTA item = RB consecutive r's x LB consecutive l's; thread = a 4 l x 4 k register tile of
//     one r; d streamed through shared memory in chunks ([r][d][l] as in HBM: float4 rows of l,
//     float4 rows of Q^T), 16 FFMA per two 16-byte loads.
//   sketch  (sketch.hpp:80-83):  Y(d, k) = sum_{r, l} P(l, d, r) Omega(col_off + l + left r, k)
//     thread = 4 d's (dq + i DQ) x KG k accumulators; G groups of threads take different (r, l-chunk)
//     items; each item's P slab is transposed into shared memory ([l][d], odd row pitch) and its
//     Omega block (LC x KG) regenerated from the reference stream (fp32 Box-Muller,
//     common.cuh gauss_pair_f32_fast); per-CTA fp64 partials for the fixed-order reduction.
// Both accumulate in fp32 over at most a few hundred terms per thread and hand fp64 partials /
// fp32 outputs on: inside the 1e-4 fp32 bound (tests/test_gpu_slab_f32.py).
#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "launch.h"

namespace trg {

namespace {

constexpr int kThreads = 256;

// ================================================================== shrink
struct TtnArgs {
    const float* in;
    float* out;
    const float* mt;  // M^T in fp32: mt[d * 4 K4 + k] (k_mt_prep)
    int left, dim, K, K4, LB, RB, DS, DC;
    int64_t right, nlb, nitems;
};

// thread = (d-slice ds, r in the item, 4-l tile, 4-k tile); DS slices split the reduction over d
// (items with few l / r: C3 / C4 mode 2) and are summed in a fixed order at the item's end
// 16-byte global -> shared copy (LDGSTS), zero-filled when !valid
__device__ __forceinline__ void cp16(float* dst, const float* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(kThreads) k_ttm_n_f32(TtnArgs a) {
    extern __shared__ __align__(16) float sm[];
    // two buffers of [RB][DC][LB] P and [DC][K4 * 4] M^T: chunk c + 1 lands (cp.async) while chunk c
    // is multiplied
    const size_t tbuf = (size_t)a.RB * a.DC * a.LB, bufsz = tbuf + (size_t)a.DC * a.K4 * 4;
    const int tiles_item = a.RB * (a.LB / 4) * a.K4;
    const int tid = threadIdx.x;
    const int ds = tid / tiles_item, t = tid - ds * tiles_item;
    const int rr = t / ((a.LB / 4) * a.K4), rem = t - rr * ((a.LB / 4) * a.K4);
    const int lt = rem / a.K4, kt = rem - lt * a.K4;  // lanes: consecutive k tiles
    const bool active = ds < a.DS;
    const int KW = a.K4 * 4;
    const int nch = (a.dim + a.DC - 1) / a.DC;
    for (int64_t item = blockIdx.x; item < a.nitems; item += gridDim.x) {
        const int64_t rb = item / a.nlb;
        const int l0 = (int)(item - rb * a.nlb) * a.LB;
        const int64_t r0 = rb * a.RB;
        const int lb = min(a.LB, a.left - l0);
        const int nr = (int)(a.right - r0 < a.RB ? a.right - r0 : a.RB);
        auto issue = [&](int c) {
            float* Ts = sm + (size_t)(c & 1) * bufsz;
            float* Ms = Ts + tbuf;
            const int d0 = c * a.DC, dc = min(a.DC, a.dim - d0);
            const int q4 = a.LB / 4, nq = a.RB * a.DC * q4;
            for (int e = tid; e < nq; e += kThreads) {
                const int r = e / (a.DC * q4), rest = e - r * (a.DC * q4);
                const int d = rest / q4, l4 = rest - d * q4;
                const bool ok = r < nr && d < dc && 4 * l4 < lb;
                cp16(Ts + (r * a.DC + d) * a.LB + 4 * l4,
                     ok ? a.in + l0 + 4 * l4 + (int64_t)a.left * (d0 + d) + (int64_t)a.left * a.dim * (r0 + r) : a.in, ok);
            }
            for (int e = tid; e < a.DC * a.K4; e += kThreads) {  // contiguous rows of M^T
                const bool ok = e / a.K4 < dc;
                cp16(Ms + 4 * e, ok ? a.mt + (size_t)d0 * KW + 4 * e : a.mt, ok);
            }
            cp_commit();
        };
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
        __syncthreads();  // the previous item's buffers are free
        issue(0);
        for (int c = 0; c < nch; ++c) {
            if (c + 1 < nch) {
                issue(c + 1);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncthreads();
            const int dc = min(a.DC, a.dim - c * a.DC);
            if (active) {
                const float* Ts = sm + (size_t)(c & 1) * bufsz;
                const float* tp = Ts + (size_t)rr * a.DC * a.LB + 4 * lt;
                const float* mp = Ts + tbuf + 4 * kt;
#pragma unroll 4
                for (int d = ds; d < dc; d += a.DS) {
                    const float4 tq = *reinterpret_cast<const float4*>(tp + (size_t)d * a.LB);
                    const float4 q = *reinterpret_cast<const float4*>(mp + (size_t)d * KW);
                    const float tv[4] = {tq.x, tq.y, tq.z, tq.w}, qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(tv[i], qv[j], acc[i][j]);
                }
            }
            __syncthreads();  // buffer c & 1 is refilled by chunk c + 2
        }
        if (a.DS > 1) {  // d-slices -> slice 0, fixed order
            __syncthreads();
            float* red = sm;  // [DS][tiles_item][16]
            if (active)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) red[((size_t)ds * tiles_item + t) * 16 + 4 * i + j] = acc[i][j];
            __syncthreads();
            if (ds == 0)
                for (int s2 = 1; s2 < a.DS; ++s2)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] += red[((size_t)s2 * tiles_item + t) * 16 + 4 * i + j];
        }
        if (ds == 0 && rr < nr && 4 * lt < lb) {
            const int64_t r = r0 + rr;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * kt + j;
                if (k >= a.K) break;
                *reinterpret_cast<float4*>(a.out + l0 + 4 * lt + (int64_t)a.left * k + (int64_t)a.left * a.K * r) =
                    make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
            }
        }
    }
}

// M(k, d) = m[k m_so + d m_sd] (fp64) -> mt[d * KW + k] (fp32, zero-padded to KW = 4 K4 columns)
__global__ void k_mt_prep(const double* __restrict__ m, int64_t m_so, int64_t m_sd, int dim, int K, int KW,
                          float* __restrict__ mt) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < dim * KW; e += gridDim.x * blockDim.x) {
        const int d = e / KW, k = e - d * KW;
        mt[e] = k < K ? (float)m[(int64_t)k * m_so + (int64_t)d * m_sd] : 0.f;
    }
}

// ================================================================== sketch
struct SknArgs {
    const float* in;
    double* partial;  // gridDim.x x dim x K (k-group blockIdx.y writes its columns)
    int left, dim, K, LC, G, DQ, pitch;
    int64_t right, nlc, nitems;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
};

// 4-byte global -> shared copy (LDGSTS): the transposed slab lands without register staging
__device__ __forceinline__ void cp4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

template <int KG, bool ASYNC>
__global__ void __launch_bounds__(kThreads) k_sketch_n_f32(SknArgs a) {
    extern __shared__ __align__(16) float sm[];
    // per group: two P item buffers [LC][pitch] (d fastest, odd pitch: the transposed stores and
    // the d reads are conflict-free) and Omega [LC][KG]; round j + 1's slab lands (cp.async)
    // while round j is multiplied
    const int pfl = (a.LC * a.pitch + 3) & ~3;
    constexpr int nbuf = ASYNC ? 2 : 1;
    const int item_floats = nbuf * pfl + a.LC * KG;
    const int tid = threadIdx.x;
    const int g = tid / a.DQ, dq = tid - g * a.DQ;
    const bool active = g < a.G;
    float* Pg = sm + (size_t)(active ? g : 0) * item_floats;
    float* Og = Pg + nbuf * pfl;
    const int k0 = blockIdx.y * KG;
    float acc[4][KG];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < KG; ++j) acc[i][j] = 0.f;
    // items (r, l-chunk) of this CTA: [it0, it1), taken G at a time (group g takes it + g)
    const int64_t it0 = a.nitems * blockIdx.x / gridDim.x, it1 = a.nitems * (blockIdx.x + 1) / gridDim.x;
    auto issue = [&](int64_t base, int buf) {
        if (active && base + g < it1) {
            const int64_t item = base + g;
            const int64_t r = item / a.nlc;
            const int l0 = (int)(item - r * a.nlc) * a.LC;
            const int lc = min(a.LC, a.left - l0);
            const float* src = a.in + l0 + (int64_t)a.left * a.dim * r;
            float* P = Pg + buf * pfl;
            // (d, l) walked l fastest: coalesced reads, stores down the transposed rows
            const int dstep = a.DQ / lc, lstep = a.DQ - dstep * lc;
            for (int d = dq / lc, l = dq - (dq / lc) * lc; d < a.dim;) {
                cp4(P + l * a.pitch + d, src + l + (int64_t)a.left * d);
                d += dstep;
                l += lstep;
                if (l >= lc) {
                    l -= lc;
                    ++d;
                }
            }
        }
        cp_commit();
    };
    // register-staged variant: 16-byte reads along l, four in flight, scattered into the rows
    auto load_now = [&](int64_t base) {
        if (active && base + g < it1) {
            const int64_t item = base + g;
            const int64_t r = item / a.nlc;
            const int l0 = (int)(item - r * a.nlc) * a.LC;
            const int lc = min(a.LC, a.left - l0);
            const float* src = a.in + l0 + (int64_t)a.left * a.dim * r;
            const int q4 = lc >> 2, nq = q4 * a.dim;
            for (int q = dq; q < nq; q += 4 * a.DQ) {
                float4 v[4];
                int dd[4], ll[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int qq = q + u * a.DQ;
                    dd[u] = qq / q4;
                    ll[u] = 4 * (qq - dd[u] * q4);
                    if (qq < nq) v[u] = *reinterpret_cast<const float4*>(src + ll[u] + (int64_t)a.left * dd[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (q + u * a.DQ < nq) {
                        float* o = Pg + ll[u] * a.pitch + dd[u];
                        o[0] = v[u].x;
                        o[a.pitch] = v[u].y;
                        o[2 * a.pitch] = v[u].z;
                        o[3 * a.pitch] = v[u].w;
                    }
            }
        }
    };
    if (ASYNC) issue(it0, 0);
    int rnd = 0;
    for (int64_t base = it0; base < it1; base += a.G, ++rnd) {
        const bool more = base + a.G < it1;
        if (ASYNC) {
            if (more) issue(base + a.G, (rnd + 1) & 1);
        } else {
            load_now(base);
        }
        if (active && base + g < it1) {
            const int64_t item = base + g;
            const int64_t r = item / a.nlc;
            const int l0 = (int)(item - r * a.nlc) * a.LC;
            const int lc = min(a.LC, a.left - l0);
            // Omega(col_off + l0 + l + left r, k0 + k) for l < lc, k < KG (zero outside K)
            const int npair = lc / 2 + 1;
            for (int e = dq; e < KG * npair; e += a.DQ) {
                const int k = e / npair, pi = e - k * npair;
                if (k0 + k >= a.K) {
                    for (int c = 2 * pi - 1; c <= 2 * pi; ++c)
                        if (c >= 0 && c < lc) Og[c * KG + k] = 0.f;
                    continue;
                }
                const uint64_t d0 = a.D + (uint64_t)(a.col_off + l0 + (int64_t)a.left * r) +
                                    (uint64_t)a.rows_glob * (uint64_t)(k0 + k);
                const uint64_t p = (d0 >> 1) + (uint64_t)pi;
                float z[2];
                gauss_pair_f32_fast(a.seed + (2ull * p + 1ull) * 0x9E3779B97F4A7C15ull, z[0], z[1]);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int64_t c = (int64_t)(2 * p + u) - (int64_t)d0;
                    if (c >= 0 && c < lc) Og[c * KG + k] = z[u];
                }
            }
        }
        if (ASYNC) {
            if (more)
                cp_wait<1>();
            else
                cp_wait<0>();
        }
        __syncthreads();
        if (active && base + g < it1) {
            const int64_t item = base + g;
            const int l0 = (int)(item - (item / a.nlc) * a.nlc) * a.LC;
            const int lc = min(a.LC, a.left - l0);
            const float* P = Pg + (ASYNC ? (rnd & 1) * pfl : 0);
            for (int l = 0; l < lc; ++l) {
                // this thread's d = dq + i DQ: consecutive lanes, consecutive words (conflict-free)
                const float* pr = P + l * a.pitch + dq;
                const float pv[4] = {pr[0], pr[a.DQ], pr[2 * a.DQ], pr[3 * a.DQ]};
                const float* orow = Og + l * KG;
#pragma unroll
                for (int j4 = 0; j4 < KG / 4; ++j4) {
                    const float4 o = *reinterpret_cast<const float4*>(orow + 4 * j4);
                    const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][4 * j4 + j] = fmaf(pv[i], ov[j], acc[i][4 * j4 + j]);
                }
            }
        }
        __syncthreads();  // Og and this round's buffer are rewritten next
    }
    // groups -> one sum (fixed order), then this CTA's fp64 partial columns [k0, k0 + KG)
    __syncthreads();
    float* red = sm;  // [G][4 DQ (d = dq + i DQ)][KG]
    if (active)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < KG; ++j) red[((size_t)g * a.DQ * 4 + dq + i * a.DQ) * KG + j] = acc[i][j];
    __syncthreads();
    double* part = a.partial + (int64_t)blockIdx.x * a.dim * a.K;
    for (int e = tid; e < a.dim * KG; e += kThreads) {
        const int d = e % a.dim, j = e / a.dim;
        if (k0 + j >= a.K) continue;
        double s = 0.0;
        for (int gg = 0; gg < a.G; ++gg) s += (double)red[((size_t)gg * a.DQ * 4 + d) * KG + j];
        part[d + (int64_t)a.dim * (k0 + j)] = s;
    }
}

struct TtnPlan {
    int K4, LB, RB, DS, DC;
    int64_t nlb, nitems;
    size_t smem;
};

bool plan_ttn(int64_t left, int64_t dim, int64_t K, int64_t right, TtnPlan& p) {
    if (left < 4 || (left % 4) != 0 || K < 1 || K > 64 || dim < 1 || left * dim * right >= (int64_t(1) << 40))
        return false;
    const int64_t want = 2 * 148;  // items for two waves of SMs
    p.K4 = (int)((K + 3) / 4);
    p.LB = (int)std::min<int64_t>(left, 4 * std::max(1, kThreads / p.K4));
    auto tiles_r = [&]() { return (p.LB / 4) * p.K4; };
    p.RB = std::max(1, kThreads / tiles_r());
    // fewer r per item, then fewer l per item, while there are too few items
    while (p.RB > 1 && ((right + p.RB - 1) / p.RB) * ((left + p.LB - 1) / p.LB) < want) p.RB = (p.RB + 1) / 2;
    while (p.LB > 4 && ((right + p.RB - 1) / p.RB) * ((left + p.LB - 1) / p.LB) < want) p.LB = std::max(4, (p.LB / 2) & ~3);
    p.DS = 1;  // split the reduction over d among the threads left idle
    while (p.DS < 32 && 2 * p.DS * p.RB * tiles_r() <= kThreads) p.DS *= 2;
    // d chunk: both (double-buffered) chunk buffers in ~48 KB, so four CTAs share an SM
    p.DC = std::max(std::max(4, (int)((24 * 1024 / 4) / (p.RB * p.LB + 4 * p.K4)) & ~3), p.DS);
    p.DC = (int)std::min<int64_t>(p.DC, dim);
    p.nlb = (left + p.LB - 1) / p.LB;
    p.nitems = ((right + p.RB - 1) / p.RB) * p.nlb;
    const size_t red = (size_t)p.DS * p.RB * tiles_r() * 16;
    p.smem = std::max(2 * ((size_t)p.RB * p.DC * p.LB + (size_t)p.DC * p.K4 * 4), red) * 4;
    return p.smem <= 96 * 1024;
}

struct SknPlan {
    int KG, ky, LC, G, DQ, pitch;
    bool async;  // cp.async double buffering (one group, one k-group: C3) or register-staged loads
    int64_t nlc, nitems;
    size_t smem;
};

bool plan_skn(int64_t left, int64_t dim, int K, int64_t right, SknPlan& p) {
    if (left < 4 || (left % 4) != 0 || dim < 1 || dim > 4 * kThreads || K < 1 || K > 64) return false;
    p.KG = K <= 24 ? ((K + 3) & ~3) : 16;
    p.ky = (K + p.KG - 1) / p.KG;
    p.DQ = (int)((dim + 3) / 4);
    p.G = std::max(1, kThreads / p.DQ);
    p.pitch = (int)(4 * p.DQ) | 1;  // odd: transposed stores and d reads conflict-free
    // l-chunk: the G items fit ~96 KB, and small when few (r, l) items would leave SMs idle
    // (C3 / C4 mode 2: left 400 / 4096 with right = 1)
    p.async = p.G == 1 && p.ky == 1;
    const int nbuf = p.async ? 2 : 1;
    const int64_t per_l = nbuf * (int64_t)p.pitch + p.KG + 8;
    const int64_t lc_mem = std::max<int64_t>(1, (96 * 1024 / 4) / (p.G * per_l));
    const int64_t lc_par = std::max<int64_t>(1, (left * right + 2 * 148 * p.G - 1) / (2 * 148 * p.G));
    p.LC = (int)std::min<int64_t>(left, std::min(lc_mem, std::max<int64_t>(4, lc_par))) & ~3;
    if (p.LC < 4) return false;
    p.nlc = (left + p.LC - 1) / p.LC;
    p.nitems = right * p.nlc;
    const size_t items = (size_t)p.G * (nbuf * ((p.LC * p.pitch + 3) & ~3) + p.LC * p.KG) * 4;
    const size_t red = (size_t)p.G * p.DQ * 4 * p.KG * 4;
    p.smem = std::max(items, red);
    return p.smem <= 160 * 1024;
}

}  // namespace

bool slab_f32_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right) {
    TtnPlan p;
    return dtype == F32 && left > 1 && plan_ttn(left, dim, K, right, p);
}

void launch_slab_f32_ttm(const TTMPlan& tp, const void* in, void* out, const double* m, int num_sms, cudaStream_t s) {
    TtnPlan p;
    if (!plan_ttn(tp.left, tp.dim, tp.odim, tp.right, p)) throw std::runtime_error("slab_f32 shrink: unsupported shape");
    TtnArgs a{};
    a.in = reinterpret_cast<const float*>(in);
    a.out = reinterpret_cast<float*>(out);
    float* mt = reinterpret_cast<float*>(scratch_alloc(sizeof(float) * (size_t)tp.dim * 4 * p.K4, s));
    k_mt_prep<<<(int)std::min<int64_t>(1024, (tp.dim * 4 * p.K4 + 255) / 256), 256, 0, s>>>(
        m, tp.m_so, tp.m_sd, (int)tp.dim, (int)tp.odim, 4 * p.K4, mt);
    a.mt = mt;
    a.left = (int)tp.left;
    a.dim = (int)tp.dim;
    a.K = (int)tp.odim;
    a.K4 = p.K4;
    a.LB = p.LB;
    a.RB = p.RB;
    a.DS = p.DS;
    a.DC = p.DC;
    a.right = tp.right;
    a.nlb = p.nlb;
    a.nitems = p.nitems;
    allow_smem(k_ttm_n_f32, p.smem);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.nitems, (int64_t)num_sms * 8));
    k_ttm_n_f32<<<grid, kThreads, p.smem, s>>>(a);
    scratch_free(mt, s);
}

bool slab_f32_sketch_ok(int dtype, int64_t left, int64_t dim, int K, int64_t right) {
    SknPlan p;
    return dtype == F32 && left > 1 && plan_skn(left, dim, K, right, p);
}

int slab_f32_sketch_grid(int64_t left, int64_t dim, int K, int64_t right, int num_sms) {
    SknPlan p;
    plan_skn(left, dim, K, right, p);
    const int64_t want = std::max<int64_t>(1, (int64_t)num_sms * 2 / p.ky);
    return (int)std::max<int64_t>(1, std::min<int64_t>((p.nitems + p.G - 1) / p.G, want));
}

int launch_slab_f32_sketch(const SketchPlan& sp, const void* x, double* partial, double* y, int num_sms,
                           cudaStream_t s) {
    SknPlan p;
    if (!plan_skn(sp.left, sp.dim, sp.K, sp.right, p)) throw std::runtime_error("slab_f32 sketch: unsupported shape");
    SknArgs a{};
    a.in = reinterpret_cast<const float*>(x);
    a.partial = partial;
    a.left = (int)sp.left;
    a.dim = (int)sp.dim;
    a.K = sp.K;
    a.LC = p.LC;
    a.G = p.G;
    a.DQ = p.DQ;
    a.pitch = p.pitch;
    a.right = sp.right;
    a.nlc = p.nlc;
    a.nitems = p.nitems;
    a.seed = sp.seed;
    a.D = sp.D;
    a.rows_glob = sp.rows_glob;
    a.col_off = sp.col_off;
    const int gx = slab_f32_sketch_grid(sp.left, sp.dim, sp.K, sp.right, num_sms);
    const dim3 grid(gx, p.ky);
    // cp.async double buffering pays where one group streams long slabs (C3: 136 -> 91 us);
    // with several groups or k-groups the register-staged loads measure faster (C4, C5)
    const bool async = p.async;
#define TRG_SKN(KGV)                                                               \
    do {                                                                           \
        if (async) {                                                               \
            allow_smem(k_sketch_n_f32<KGV, true>, p.smem);                         \
            k_sketch_n_f32<KGV, true><<<grid, kThreads, p.smem, s>>>(a);           \
        } else {                                                                   \
            allow_smem(k_sketch_n_f32<KGV, false>, p.smem);                        \
            k_sketch_n_f32<KGV, false><<<grid, kThreads, p.smem, s>>>(a);          \
        }                                                                          \
    } while (0)
    switch (p.KG) {
        case 4: TRG_SKN(4); break;
        case 8: TRG_SKN(8); break;
        case 12: TRG_SKN(12); break;
        case 16: TRG_SKN(16); break;
        case 20: TRG_SKN(20); break;
        default: TRG_SKN(24); break;
    }
#undef TRG_SKN
    if (y) launch_reduce_partials(partial, gx, sp.dim * sp.K, y, s);
    return gx;
}

}  // namespace trg
