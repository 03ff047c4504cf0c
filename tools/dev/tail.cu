// SPDX-License-Identifier: Apache-2.0
// DEVELOPMENT PROBE, not built into libtrg: the persistent-tail kernel measured in round 2.
// It was wired into runtime.cpp run_sketch (plan_tail_start / run_tail) and is kept here for reference.
//
// Persistent tail of the sequential projection (sketch.hpp:73-87): once the working tensor is
// L2-sized, every remaining mode n0..N-1 - sketch (sketch.hpp:80-83), fixed-order split-K sum,
// thin QR (sketch.hpp:45-53, cqr.cuh) and shrink (sketch.hpp:85 -> tensor.hpp:193-207) - runs in
// ONE launch with one CTA per SM, instead of four launches per mode whose cost on a few MB of
// data is launch, ramp and drain.
//
// Partition. The working tensor of mode m is viewed as (a, l, i, rho, s): a the left index of
// mode n0 (extent A = prod_{j<n0} K_j), l the indices of the tail modes already shrunk
// (L = prod_{n0<=j<m} K_j), i the mode index (I_m), rho the modes between m and the last
// (Rm), s the last mode's index (Is). CTA b owns the block (a in chunk b % Pa, s in chunk
// b / Pa) of EVERY mode: the shrink of mode m writes exactly the block of P^(m+1) that the same
// CTA sketches next, so no grid barrier separates one mode's shrink from the next mode's
// sketch. Per mode the only grid-wide steps are the split-K sum of Y (a barrier, then a
// distributed fixed-order reduce) and the QR (the last CTA to finish the reduce factors Y;
// the others wait on its release flag). With Ps > 1 the last mode's shrink sums P over the s
// chunks in a last barrier + fixed-order reduce.
//
// Test matrix. Omega_m(c, k) is reference draw D_m + c + rows_glob_m k of the stream `seed`
// (sketch.hpp:32-38, 69, 81), c = a + A (l + L (rho + Rm s)) the unfolding column
// (tensor.hpp:133-142). Each CTA generates the entries of its own columns once per mode into
// shared memory, one Box-Muller pair per two draws (the fp64 table-driven generator of
// common.cuh for fp64 tensors, the fp32 one otherwise, as the streaming kernels).
//
// Arithmetic. Sketch: thread tile 4 rows x 8 columns of Y, the block's columns split over
// thread groups, group partials summed in a fixed order; shrink: thread tile 2 columns x 8
// outputs, the contraction split over ISP lanes of a warp and summed by shuffles. All sums have a
// fixed order: the result is bit-reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "cqr.cuh"
#include "kernels.h"
#include "launch.h"
#include "pipeline.cuh"

namespace trg {

namespace {

constexpr int kTT = kThreads;  // 512: the QR building blocks assume it

struct TailModeDev {
    int I, K, KO;        // mode extent, sketch size, ceil(K / 8)
    int64_t L, Rm;       // extents of l and rho
    uint64_t D;          // draw offset of the mode
    int64_t rows_glob;   // rows of the global Omega_m (its column stride in the stream)
    double* Y;           // reduced Y_m (I x K, column-major)
    double* Q;           // Q_m (I x K, column-major)
    int* flag;           // QR path (0 CholQR, 1 Householder)
    void* out;           // P^(m+1) (global scratch) or P for the last mode
    int JTs, ISP, JTt;   // sketch tile columns, shrink contraction split, shrink tile columns
    int stage;           // elements of one tile buffer
    int ld;              // QR staging stride
};

struct TailArgs {
    int nm;
    TailModeDev md[kTailMaxModes];
    int64_t A, Is;
    int Pa, Ps;
    const void* in;      // P^(n0)
    uint64_t seed;
    double* part;        // nct blocks of max I*K partial sums
    int64_t part_stride;
    void* ppart;         // Ps blocks of |P| (Ps > 1)
    double* W;           // Householder workspace (max I*K)
    unsigned* sync;      // [0] barrier counter, [1 + m] QR tickets, [1 + kTailMaxModes + m] QR done
    const GaussTables* gt;
    unsigned long long* trace;  // development (TRG_TAIL_TRACE): per-mode phase times of CTA 0 / the QR CTA
    // shared-memory carve (bytes)
    int off_cols, off_om, off_tile, off_q, off_qr, smem;
    int ncols_max, KPmax;
};

// sketch tile pitch (rows of a column + pad): the row quads stay 16-byte aligned and the pitch is an
// odd number of 16-byte units, so the column-per-lane tile stores spread over the banks
__host__ __device__ __forceinline__ int tail_pitch(int NI4, int es) {
    const int q = es == 8 ? 2 : 4;  // elements per 16 bytes
    int units = (4 * NI4 + q - 1) / q + 1;
    if ((units & 1) == 0) ++units;
    return units * q;
}

__device__ __forceinline__ int64_t imin64(int64_t x, int64_t y) { return x < y ? x : y; }
__device__ __forceinline__ int64_t imax64(int64_t x, int64_t y) { return x > y ? x : y; }

__device__ __forceinline__ void chunk_of(int64_t n, int parts, int idx, int64_t& lo, int64_t& cnt) {
    const int64_t q = n / parts, r = n % parts;
    lo = idx * q + (int64_t)imin64(idx, r);
    cnt = q + (idx < r ? 1 : 0);
}

// bounded spin: a grid that cannot become co-resident traps instead of hanging the device
__device__ __forceinline__ void spin_until_ge(const unsigned* p, unsigned target) {
    unsigned v;
    long long t0 = 0;
    for (int it = 0;; ++it) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) return;
        if (it == 64) t0 = clock64();
        if (it > 64 && (it & 1023) == 0 && clock64() - t0 > (1ll << 32)) __trap();  // ~2 s at 2 GHz
    }
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TAIL_T(slot)                                                  \
    if (a.trace && threadIdx.x == 0 && blockIdx.x == 0) a.trace[m * 16 + (slot)] = gtime()

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned& epoch, unsigned nct) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        spin_until_ge(ctr, epoch * nct);
    }
    __syncthreads();
}

template <typename T>
__device__ __forceinline__ void cp_async_elem(uint32_t dst, const T* src) {
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// N consecutive 16-byte aligned shared-memory values
template <typename T, int N>
__device__ __forceinline__ void ld_vec(const T* p, T* v) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const double2 d = reinterpret_cast<const double2*>(p)[i];
            v[2 * i] = d.x;
            v[2 * i + 1] = d.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const float4 f = reinterpret_cast<const float4*>(p)[i];
            v[4 * i] = f.x;
            v[4 * i + 1] = f.y;
            v[4 * i + 2] = f.z;
            v[4 * i + 3] = f.w;
        }
    }
}

template <typename T>
__device__ __forceinline__ void gauss2(uint64_t seed, uint64_t p, const GaussTables& gt, T& z0, T& z1) {
    const uint64_t st = seed + (2ull * p + 1ull) * 0x9E3779B97F4A7C15ull;
    if constexpr (sizeof(T) == 8)
        gauss_pair_state(st, gt, z0, z1);
    else
        gauss_pair_f32_state(st, z0, z1);
}

// geometry of one mode inside this CTA's block
struct Geo {
    int64_t na, a0, ns, s0;
    int64_t W;      // na * L: columns per slab
    int64_t nsl;    // slabs (rho, s_loc) of the block; 1 for the last mode
    int64_t ncols;  // W * nsl
    int nI, r0;     // rows of the block (I, or the s chunk for the last mode) and their offset
    int64_t rs;     // row stride A * L
};

template <typename T, int KW>
__global__ void __launch_bounds__(kTT, 1) k_tail(TailArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x;
    const unsigned nct = gridDim.x;
    const int b = blockIdx.x;
    const int ia = b % a.Pa, is = b / a.Pa;
    int64_t a0, na, s0, ns;
    chunk_of(a.A, a.Pa, ia, a0, na);
    chunk_of(a.Is, a.Ps, is, s0, ns);
    GaussTables& gt = *reinterpret_cast<GaussTables*>(sm);
    int* cin = reinterpret_cast<int*>(sm + a.off_cols);          // per local column: input base
    int* cout = cin + a.ncols_max;                               // ... output base
    T* Om = reinterpret_cast<T*>(sm + a.off_om);                 // ncols x KP test-matrix entries
    T* tile = reinterpret_cast<T*>(sm + a.off_tile);             // tile buffers / reduction scratch
    T* Qs = reinterpret_cast<T*>(sm + a.off_q);                  // rows x KP
    const CqrFactorSmem qs = cqr_factor_carve<KW>(reinterpret_cast<double*>(sm + a.off_qr));
    __shared__ int s_last;
    if constexpr (sizeof(T) == 8) gauss_tables_to_smem(gt, a.gt);
    griddep_wait();
    unsigned epoch = 0;
    const T* cur = reinterpret_cast<const T*>(a.in);
    for (int m = 0; m < a.nm; ++m) {
        const TailModeDev& md = a.md[m];
        const bool last = m == a.nm - 1;
        const int I = md.I, K = md.K, KO = md.KO, KP = 8 * KO;
        Geo g;
        g.na = na;
        g.a0 = a0;
        g.ns = ns;
        g.s0 = s0;
        g.W = na * md.L;
        g.nsl = last ? 1 : md.Rm * ns;
        g.ncols = g.W * g.nsl;
        g.nI = last ? (int)ns : I;
        g.r0 = last ? (int)s0 : 0;
        g.rs = a.A * md.L;
        const int64_t AL = a.A * md.L;
        TAIL_T(0);
        // ---- per-column bases and the QR staging pad (no input needed)
        for (int64_t j = tid; j < g.ncols; j += kTT) {
            const int64_t q = j / g.W, rem = j - q * g.W;
            const int64_t l = rem / na, al = rem - l * na;
            const int64_t inner = a0 + al + a.A * l;
            const int64_t slab = last ? 0 : q + md.Rm * s0;
            cin[j] = (int)(inner + AL * (int64_t)I * slab + AL * g.r0);
            cout[j] = (int)(inner + AL * (int64_t)K * slab);
        }
        cqr_factor_prepare<KW>(qs, I, K, md.ld);
        TAIL_T(1);
        // ---- test-matrix entries of the block's columns: runs of consecutive unfolding columns
        // (na of them when the a chunk is a strict part of A, else the whole block), one
        // Box-Muller pair per two draws
        {
            // run r = (l, q) of na columns (or the whole block when the a chunk is all of A);
            // item = (run, k, u): pair u of the run's draws for column k (32-bit index math)
            const bool whole = na == a.A;
            const int RL = whole ? (int)g.ncols : (int)na;
            const int nruns = whole ? 1 : (int)(g.ncols / na);
            const int U = RL / 2 + 1;
            const int items = nruns * K * U;
            const int Lm = (int)md.L;
#pragma unroll 1
            for (int it = tid; it < items; it += kTT) {
                const int ru = it / K, k = it - ru * K;  // k fastest: consecutive lanes, consecutive words
                const int run = ru / U, u = ru - run * U;
                const int j0 = whole ? 0 : run * (int)na;
                const int q = whole ? 0 : run / Lm, l = whole ? 0 : run - q * Lm;
                const int64_t c0 = a0 + a.A * l + (last ? 0 : AL * (q + md.Rm * s0));
                const uint64_t qs0 = md.D + (uint64_t)c0 + (uint64_t)md.rows_glob * (uint64_t)k;
                const int t = 2 * u - (int)(qs0 & 1ull);
                if (t + 1 < 0 || t >= RL) continue;
                T z0, z1;
                gauss2<T>(a.seed, (qs0 + (uint64_t)t) >> 1, gt, z0, z1);
                if (t >= 0) Om[(j0 + t) * KP + k] = z0;
                if (t + 1 < RL) Om[(j0 + t + 1) * KP + k] = z1;
            }
            const int pad = KP - K;
            for (int e = tid; e < (int)g.ncols * pad; e += kTT) {
                const int j = e / pad;
                Om[j * KP + K + (e - j * pad)] = T(0);
            }
        }
        __syncthreads();
        TAIL_T(2);
        // ---- sketch: Y_part(i, k) = sum over the block's columns j of X(j, i) Omega(j, k)
        {
            const int NI4 = (g.nI + 3) / 4;
            const int NTA = NI4 * KO;
            const int G = max(1, kTT / NTA);
            const int ta = tid % NTA, grp = tid / NTA;
            const int ti = ta % NI4, tk = ta / NI4;
            const bool act = grp < G && tid < G * NTA;
            const int IP = tail_pitch(NI4, (int)sizeof(T));
            const int JT = md.JTs;
            T acc[4][8];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = T(0);
            const int64_t ntiles = (g.ncols + JT - 1) / JT;
            const uint32_t tb = smem_u32(tile);
            const int stage = md.stage;
            auto issue = [&](int64_t t) {
                const int j0 = (int)(t * JT);
                const int jt = (int)imin64(JT, g.ncols - j0);
                const uint32_t buf = tb + (uint32_t)((t & 1) * stage * sizeof(T));
#pragma unroll 1
                for (int e = tid; e < jt * g.nI; e += kTT) {
                    const int i = e / jt, jj = e - i * jt;
                    cp_async_elem<T>(buf + (uint32_t)((jj * IP + i) * sizeof(T)), cur + cin[j0 + jj] + g.rs * i);
                }
                cp_async_commit();
            };
            if (ntiles > 0) issue(0);
#pragma unroll 1
            for (int64_t t = 0; t < ntiles; ++t) {
                if (t + 1 < ntiles) {
                    issue(t + 1);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const int64_t j0 = t * JT;
                const int jt = (int)imin64(JT, g.ncols - j0);
                const T* ts = tile + (t & 1) * stage;
                if (act) {
                    for (int jj = grp; jj < jt; jj += G) {
                        const T* xr = ts + jj * IP + 4 * ti;
                        const T* orow = Om + (j0 + jj) * KP + 8 * tk;
                        T xv[4], ov[8];
                        ld_vec<T, 4>(xr, xv);
                        ld_vec<T, 8>(orow, ov);
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int c = 0; c < 8; ++c) acc[r][c] = fma(xv[r], ov[c], acc[r][c]);
                    }
                }
                __syncthreads();
            }
            TAIL_T(3);
            // fixed-order sum over the groups, 8 accumulators per round through the tile buffer
            // (layout [c][group][thread tile]: consecutive lanes, consecutive words)
            double* dst = a.part + (int64_t)b * a.part_stride;
            const int GN = G * NTA;
#pragma unroll
            for (int rnd = 0; rnd < 4; ++rnd) {
                if (act) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) tile[c * GN + grp * NTA + ta] = acc[rnd][c];
                }
                __syncthreads();
#pragma unroll 1
                for (int e = tid; e < NTA * 8; e += kTT) {
                    const int c = e / NTA, ta2 = e - c * NTA;
                    T s = T(0);
                    for (int g2 = 0; g2 < G; ++g2) s += tile[c * GN + g2 * NTA + ta2];
                    const int i = 4 * (ta2 % NI4) + rnd, k = 8 * (ta2 / NI4) + c;
                    if (i < g.nI && k < K) dst[(g.r0 + i) + (int64_t)I * k] = (double)s;
                }
                __syncthreads();
            }
            if (last && a.Ps > 1) {  // rows of Y outside this CTA's chunk: zero
                for (int e = tid; e < I * K; e += kTT) {
                    const int i = e % I;
                    if (i < g.r0 || i >= g.r0 + g.nI) dst[e] = 0.0;
                }
            }
        }
        // ---- split-K sum of Y: barrier, every CTA sums a slice of the entries over all partials
        // in CTA order, then the last CTA to finish factors Y
        TAIL_T(4);
        grid_barrier(a.sync, epoch, nct);
        TAIL_T(5);
        {
            const int n = I * K;
            int64_t e0, ne;
            chunk_of(n, (int)nct, b, e0, ne);
            // thread = (entry, partial group): groups of partials summed in order, then the groups
            double* red = reinterpret_cast<double*>(tile);
            if (ne <= kTT / 2) {
                const int ent = (int)(int64_t)imax64(ne, 1);
                const int PG = kTT / ent;
                const int ei = tid % ent, pg = tid / ent;
                double s = 0.0;
                if (ei < ne) {
                    for (int c = pg; c < (int)nct; c += PG) s += __ldcg(a.part + (int64_t)c * a.part_stride + e0 + ei);
                }
                red[tid] = s;
                __syncthreads();
                if (tid < ne) {
                    double tot = 0.0;
                    for (int g2 = 0; g2 < PG; ++g2) tot += red[g2 * ent + tid];
                    md.Y[e0 + tid] = tot;
                }
            } else {
                for (int64_t e = tid; e < ne; e += kTT) {
                    double tot = 0.0;
                    for (int c = 0; c < (int)nct; ++c) tot += __ldcg(a.part + (int64_t)c * a.part_stride + e0 + e);
                    md.Y[e0 + e] = tot;
                }
            }
            __syncthreads();
            if (tid == 0) {
                unsigned prev;
                asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.sync + 1 + m) : "memory");
                s_last = prev == nct - 1;
            }
            __syncthreads();
            unsigned* done = a.sync + 1 + kTailMaxModes + m;
            if (tid == 0 && b == 0 && a.trace) a.trace[m * 16 + 6] = gtime();
            if (s_last) {
                if (tid == 0 && a.trace) a.trace[m * 16 + 12] = gtime();
                cqr_factor<KW>(qs, md.Y, false, md.Y, I, K, md.ld, md.Q, a.W, md.flag);
                if (tid == 0 && a.trace) a.trace[m * 16 + 13] = gtime();
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(done) : "memory");
                }
            } else if (tid == 0) {
                spin_until_ge(done, 1u);
            }
            __syncthreads();
        }
        TAIL_T(7);
        // ---- Q rows of the block (fp64 -> T), pitch KP, zero beyond K
        for (int e = tid; e < g.nI * KP; e += kTT) {
            const int i = e / KP, k = e - i * KP;
            Qs[e] = k < K ? (T)__ldcg(md.Q + (g.r0 + i) + (int64_t)I * k) : T(0);
        }
        // ---- shrink: out(j, k) = sum_i X(j, i) Q(i, k). Thread = (column pair, output octet) of a
        // group of NJ threads; ISP groups split the contraction (whole warps: the Q row is a
        // broadcast, the column pairs are contiguous) and are summed in a fixed order through the
        // consumed tile buffer.
        {
            const int JT = md.JTt, JP = JT + 4;
            const int NJ = (JT / 2) * KO;
            const int ISP = md.ISP;
            const int rest = tid % NJ, isp = tid / NJ;
            const int jp = rest % (JT / 2), ko = rest / (JT / 2);
            const bool act = isp < ISP;
            const int64_t ntiles = (g.ncols + JT - 1) / JT;
            const int stage = md.stage;  // elements per tile buffer
            const uint32_t tb = smem_u32(tile);
            T* outp = reinterpret_cast<T*>(md.out);
            const bool to_part = last && a.Ps > 1;
            if (to_part) outp = reinterpret_cast<T*>(a.ppart) + (int64_t)is * (AL * K);
            auto issue = [&](int64_t t) {
                const int j0 = (int)(t * JT);
                const int jt = (int)imin64(JT, g.ncols - j0);
                const uint32_t buf = tb + (uint32_t)((t & 1) * stage * sizeof(T));
#pragma unroll 1
                for (int e = tid; e < jt * g.nI; e += kTT) {
                    const int i = e / jt, jj = e - i * jt;
                    cp_async_elem<T>(buf + (uint32_t)((i * JP + jj) * sizeof(T)), cur + cin[j0 + jj] + g.rs * i);
                }
                cp_async_commit();
            };
            __syncthreads();  // Qs complete; the sketch's last reads of the tile buffer are long done
            if (ntiles > 0) issue(0);
#pragma unroll 1
            for (int64_t t = 0; t < ntiles; ++t) {
                if (t + 1 < ntiles) {
                    issue(t + 1);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const int j0 = (int)(t * JT);
                const int jt = (int)imin64(JT, g.ncols - j0);
                T* tt = tile + (t & 1) * stage;
                T acc[2][8];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[h][c] = T(0);
                if (act && 2 * jp < jt) {
#pragma unroll 2
                    for (int i = isp; i < g.nI; i += ISP) {
                        T xv[2], qv[8];
                        xv[0] = tt[i * JP + 2 * jp];
                        xv[1] = tt[i * JP + 2 * jp + 1];
                        ld_vec<T, 8>(Qs + i * KP + 8 * ko, qv);
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            acc[0][c] = fma(xv[0], qv[c], acc[0][c]);
                            acc[1][c] = fma(xv[1], qv[c], acc[1][c]);
                        }
                    }
                }
                __syncthreads();  // the tile is consumed: its buffer takes the group partials
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    if (act) {
#pragma unroll
                        for (int c = 0; c < 8; ++c) tt[(c * ISP + isp) * NJ + rest] = acc[h][c];
                    }
                    __syncthreads();
#pragma unroll 1
                    for (int e = tid; e < NJ * 8; e += kTT) {
                        const int c = e / NJ, r2 = e - c * NJ;
                        const int jp2 = r2 % (JT / 2), ko2 = r2 / (JT / 2);
                        const int jj = 2 * jp2 + h, k = 8 * ko2 + c;
                        T s = T(0);
                        for (int g2 = 0; g2 < ISP; ++g2) s += tt[(c * ISP + g2) * NJ + r2];
                        if (jj < jt && k < K) outp[cout[j0 + jj] + AL * k] = s;
                    }
                    __syncthreads();
                }
            }
        }
        TAIL_T(8);
        if (last && a.Ps > 1) {
            // P = sum over the s chunks (fixed order) of the partial P blocks
            grid_barrier(a.sync, epoch, nct);
            const int64_t np = AL * K;
            int64_t e0, ne;
            chunk_of(np, (int)nct, b, e0, ne);
            const T* pp = reinterpret_cast<const T*>(a.ppart);
            T* P = reinterpret_cast<T*>(md.out);
            for (int64_t e = tid; e < ne; e += kTT) {
                T s = T(0);
                for (int c = 0; c < a.Ps; ++c) s += __ldcg(pp + (int64_t)c * np + e0 + e);
                P[e0 + e] = s;
            }
        }
        cur = reinterpret_cast<const T*>(md.out);
        __syncthreads();
        TAIL_T(9);
    }
}

}  // namespace

size_t tail_sync_ints() { return 1 + 2 * kTailMaxModes; }

bool plan_tail(int dtype, int nm, const int64_t* I, const int64_t* K, int64_t A, int num_sms, TailPlan& p) {
    p = TailPlan{};
    if (nm < 1 || nm > kTailMaxModes || num_sms < 1) return false;
    int kmax = 0;
    for (int m = 0; m < nm; ++m) {
        if (K[m] < 1 || K[m] > 16 || K[m] >= I[m] || I[m] > 4096) return false;
        kmax = std::max(kmax, (int)K[m]);
    }
    const int KW = kmax <= 8 ? 8 : kmax <= 16 ? 16 : 32;
    p.KW = KW;
    p.dtype = dtype;
    p.nm = nm;
    p.A = A;
    p.Is = I[nm - 1];
    const size_t es = dtype_size(dtype);
    // partition: the smallest max block (a chunk x s chunk), a small penalty for s chunks (the
    // extra P reduction); a chunks that are a strict part of A keep runs of >= 128 bytes (whole
    // sectors); at most one CTA per SM
    const int64_t min_run = std::max<int64_t>(1, 128 / (int64_t)es);
    double best = 1e300;
    for (int Ps = 1; Ps <= std::min<int64_t>(p.Is, num_sms); ++Ps) {
        int64_t Pa = std::min<int64_t>(A, num_sms / Ps);
        if (Pa < 1) break;
        if (Pa > 1 && (A + Pa - 1) / Pa < min_run) Pa = std::max<int64_t>(1, A / min_run);
        const double work = (double)((A + Pa - 1) / Pa) * (double)((p.Is + Ps - 1) / Ps);
        const double score = work * (Ps > 1 ? 1.15 : 1.0);
        if (score < best - 1e-9) {
            best = score;
            p.Pa = (int)Pa;
            p.Ps = Ps;
        }
    }
    const int64_t na = (A + p.Pa - 1) / p.Pa, ns = (p.Is + p.Ps - 1) / p.Ps;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // the largest tile budget (both buffers) whose carve fits the opt-in shared memory
    bool fits = false;
    for (size_t kTileBudget : {size_t(110) << 10, size_t(80) << 10, size_t(56) << 10, size_t(40) << 10}) {
        // per-mode geometry and shared memory
        int64_t L = 1;
        size_t om_max = 0, tile_max = 0, q_max = 0, qr_max = 0, cols_max = 0, partn = 0;
        int KPmax = 8;
        for (int m = 0; m < nm; ++m) {
            TailMode& md = p.md[m];
            const bool last = m == nm - 1;
            int64_t Rm = 1;
            for (int j = m + 1; j < nm - 1; ++j) Rm *= I[j];
            md.I = I[m];
            md.K = K[m];
            md.L = L;
            md.Rm = last ? 1 : Rm;
            const int KO = (int)((K[m] + 7) / 8), KP = 8 * KO;
            KPmax = std::max(KPmax, KP);
            const int64_t nI = last ? ns : I[m];
            const int64_t ncols = na * L * (last ? 1 : Rm * ns);
            if (ncols * std::max<int64_t>(I[m], 1) >= (int64_t(1) << 31)) return false;
            const int64_t NI4 = (nI + 3) / 4;
            if (NI4 * KO > kTT) return false;  // sketch thread tiles
            const int64_t IP = tail_pitch((int)NI4, (int)es);
            // sketch tiles: JTs columns x IP
            int JTs = 128;
            while (JTs > 8 && (size_t)2 * JTs * IP * es > kTileBudget) JTs /= 2;
            // shrink tiles: JTt columns x nI rows (pitch JTt + 4); NJ = JTt / 2 * KO threads per
            // contraction group, ISP = kTT / NJ groups
            int JTt = 256;
            while (JTt > 4 && ((JTt / 2) * KO > kTT || (size_t)2 * nI * (JTt + 4) * es > kTileBudget)) JTt /= 2;
            if ((JTt / 2) * KO > kTT) return false;
            const int ISP = std::max(1, kTT / ((JTt / 2) * KO));
            const size_t stage = std::max<size_t>({(size_t)JTs * IP, (size_t)nI * (JTt + 4), (size_t)kTT * 8});
            md.JTs = JTs;
            md.ISP = ISP;
            md.JTt = JTt;
            md.stage = (int)stage;
            md.ld = KW + 4;
            tile_max = std::max(tile_max, 2 * stage * es);
            om_max = std::max(om_max, (size_t)ncols * KP * es);
            q_max = std::max(q_max, (size_t)nI * KP * es);
            qr_max = std::max(qr_max, sizeof(double) * (KW == 8    ? cqr_factor_smem_doubles<8>(I[m], KW + 4)
                                                        : KW == 16 ? cqr_factor_smem_doubles<16>(I[m], KW + 4)
                                                                   : cqr_factor_smem_doubles<32>(I[m], KW + 4)));
            cols_max = std::max(cols_max, (size_t)ncols);
            partn = std::max(partn, (size_t)(I[m] * K[m]));
            L *= K[m];
        }
        auto al = [](size_t x) { return (x + 127) & ~(size_t)127; };
        size_t off = al(dtype == F64 ? sizeof(GaussTables) : 16);
        p.off_cols = (int)off;
        off = al(off + 2 * cols_max * sizeof(int));
        p.off_om = (int)off;
        off = al(off + om_max);
        p.off_tile = (int)off;
        off = al(off + tile_max);
        p.off_q = (int)off;
        off = al(off + q_max);
        p.off_qr = (int)off;
        off = al(off + qr_max);
        p.smem = (int)off;
        p.ncols_max = (int)cols_max;
        p.KPmax = KPmax;
        p.part_stride = (int64_t)((partn + 1) & ~(size_t)1);
        p.P_elems = L * A;  // A * prod K over the tail (only the a extent and the K's remain)
        int64_t first = A * p.Is;  // elements of the tail's input tensor (the largest it touches)
        for (int m = 0; m < nm - 1; ++m) first *= I[m];
        if (first >= (int64_t(1) << 31)) return false;  // 32-bit column bases
        if (p.smem + 1024 <= optin) {
            fits = true;
            break;
        }
    }
    if (!fits) return false;
    p.nct = p.Pa * p.Ps;
    if (p.nct > num_sms) return false;
    return true;
}

template <typename T, int KW>
static void go_tail(const TailArgs& a, int nct, cudaStream_t s) {
    auto kern = k_tail<T, KW>;
    allow_smem(kern, a.smem);
    pdl_launch(kern, dim3(nct), dim3(kTT), (size_t)a.smem, s, a);
}

void launch_tail(const TailPlan& p, const void* in, uint64_t seed, double* part, void* ppart, double* W,
                 unsigned* sync, cudaStream_t s) {
    TailArgs a{};
    a.nm = p.nm;
    for (int m = 0; m < p.nm; ++m) {
        const TailMode& h = p.md[m];
        TailModeDev& d = a.md[m];
        d.I = (int)h.I;
        d.K = (int)h.K;
        d.KO = (int)((h.K + 7) / 8);
        d.L = h.L;
        d.Rm = h.Rm;
        d.D = h.D;
        d.rows_glob = h.rows_glob;
        d.Y = h.Y;
        d.Q = h.Q;
        d.flag = h.flag;
        d.out = h.out;
        d.JTs = h.JTs;
        d.ISP = h.ISP;
        d.JTt = h.JTt;
        d.stage = h.stage;
        d.ld = h.ld;
    }
    a.A = p.A;
    a.Is = p.Is;
    a.Pa = p.Pa;
    a.Ps = p.Ps;
    a.in = in;
    a.seed = seed;
    a.part = part;
    a.part_stride = p.part_stride;
    a.ppart = ppart;
    a.W = W;
    a.sync = sync;
    a.gt = p.dtype == F64 ? gauss_tables(s) : nullptr;
    static unsigned long long* trace = nullptr;
    const bool tr = getenv("TRG_TAIL_TRACE") != nullptr;
    if (tr) {
        if (!trace) cudaMalloc(&trace, 16 * kTailMaxModes * sizeof(unsigned long long));
        cudaMemsetAsync(trace, 0, 16 * kTailMaxModes * sizeof(unsigned long long), s);
        a.trace = trace;
    }
    a.off_cols = p.off_cols;
    a.off_om = p.off_om;
    a.off_tile = p.off_tile;
    a.off_q = p.off_q;
    a.off_qr = p.off_qr;
    a.smem = p.smem;
    a.ncols_max = p.ncols_max;
    a.KPmax = p.KPmax;
    if (p.dtype == F64) {
        if (p.KW == 8) go_tail<double, 8>(a, p.nct, s);
        else if (p.KW == 16) go_tail<double, 16>(a, p.nct, s);
        else go_tail<double, 32>(a, p.nct, s);
    } else {
        if (p.KW == 8) go_tail<float, 8>(a, p.nct, s);
        else if (p.KW == 16) go_tail<float, 16>(a, p.nct, s);
        else go_tail<float, 32>(a, p.nct, s);
    }
    if (tr) {
        unsigned long long h[16 * kTailMaxModes];
        cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const unsigned long long t0 = h[0];
        fprintf(stderr, "tail nct=%d Pa=%d Ps=%d smem=%d:", p.nct, p.Pa, p.Ps, p.smem);
        for (int m = 0; m < p.nm; ++m) {
            fprintf(stderr, " | m%d", m);
            for (int k = 0; k < 14; ++k) fprintf(stderr, " %lld", h[m * 16 + k] ? (long long)(h[m * 16 + k] - t0) : -1ll);
        }
        fprintf(stderr, "\n");
    }
}

}  // namespace trg
