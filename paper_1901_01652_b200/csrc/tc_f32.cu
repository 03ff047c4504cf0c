// SPDX-License-Identifier: Apache-2.0
//
// fp32 mode-0 sketch and shrink on the 5th-generation tensor cores (tcgen05, kind::tf32, TMEM
// accumulators, TMA-fed shared memory), in 3xTF32: every fp32 operand v is split into
// hi = rna_tf32(v) and lo = v - hi, and  v w  ~  hi_v hi_w + lo_v hi_w + hi_v lo_w.
// The dropped lo_v lo_w is below 2^-22 |v w| and the lo operands are read to 11 bits
// (2^-11 of 2^-11), so a product carries ~2^-21 relative error against fp32's 2^-24: the
// stage stays inside the 1e-4 fp32 parity bound against the fp64 oracle with a wide margin,
// while plain TF32 (2^-11) would not (BASELINE.json north_star).
//
//   K1  Y_0 = X_(0) Omega_0       (sketch.hpp:80-83; unfold_classic tensor.hpp:133-142)
//       D[I0 x K] += A[I0 x kb] B[kb x K]: A = a kb-column block of X_(0) (the I0-long mode-0
//       fibres are contiguous: MN-major A in 32-row blocks, 128B-swizzled with 32-byte atoms,
//       the one MN-major tf32 layout, landed by TMA), B = the
//       reference test-matrix block regenerated on chip (SplitMix64 + fp64 table Box-Muller,
//       common.cuh, bit-addressable by draw index) in the K-major no-swizzle layout. All of Y's
//       rows stay in TMEM for the CTA's whole column range (ceil(I0/128) x Kpad <= 512 columns);
//       per-CTA partial sums leave in fp64 for the fixed-order reduction (launch_qr_fused /
//       launch_reduce_partials), as the other sketch kernels.
//   K2  P^(1) = X x_0 Q_0^T       (tensor.hpp:193-207 with m = Q^T, sketch.hpp:85)
//       per tile of 256 fibres: D[256 x K] = X^T[256 x I0] Q[I0 x K] as two M=128 MMAs per
//       k-step; both operands K-major (the reduction index i is contiguous in a fibre and in
//       Q's columns), 128B-swizzled 32-row slabs of X by TMA, Q streamed from L2 in the same
//       32-row slabs (pre-split into tf32 hi / lo, k_qt_prep), double-buffered accumulators
//       so the epilogue (TMEM -> registers -> P^(1) rows, K contiguous values per fibre)
//       overlaps the next tile's MMAs.
//
// Warp roles (one CTA per SM): 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2-5 the X
// splitters (hi in place, lo beside it; then the K1 epilogue), 6-9 K1 generators / K2 epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "pipeline.cuh"

namespace trg {

namespace {

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

// ------------------------------------------------------------------ tcgen05 / TMA primitives
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes made visible to the async proxy (the tensor core)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem] (+)= A[smem] B[smem], kind::tf32, fp32 accumulate
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
// arrive on an mbarrier once every tcgen05 op issued so far by this thread has completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}

// shared-memory matrix descriptor (sm_100 UMMA): start, leading / stride byte offsets, version
// 1, layout (0 none, 2 128B swizzle)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
constexpr uint32_t kSw128 = 2, kSw128b32 = 1, kSwNone = 0;

// instruction descriptor, kind::tf32: D f32, A/B tf32, majors (0 K, 1 MN), N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float tf32_rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// v -> (hi, lo) in place / beside: the 3xTF32 split of one stage buffer (layout-agnostic)
__device__ __forceinline__ void split_stage(uint32_t hi, uint32_t lo, uint32_t bytes, int tid, int nthr) {
    for (uint32_t o = (uint32_t)tid * 16u; o < bytes; o += (uint32_t)nthr * 16u) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(hi + o));
        const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(hi + o), "f"(h.x), "f"(h.y), "f"(h.z), "f"(h.w));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lo + o), "f"(v.x - h.x), "f"(v.y - h.y),
                     "f"(v.z - h.z), "f"(v.w - h.w));
    }
}

__device__ __forceinline__ void sts32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }

constexpr int kWarps = 10;
constexpr int kThreads = kWarps * 32;
constexpr int kSplitW0 = 2, kSplitWarps = 4;  // warps 2..5
constexpr int kAuxW0 = 6, kAuxWarps = 4;      // warps 6..9

// ================================================================== K1: mode-0 sketch
struct TcSkArgs {
    int I0, K, Kp, Mt, nblk, kb, S;
    int64_t L, ntiles;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    double* partial;  // per CTA: I0 x K fp64, column-major
    const GaussTables* gt;
    uint32_t a_bytes, b_bytes;  // per-stage A (X block) and B (one of hi / lo) buffer sizes
    float* dbg;                 // development probe (TRG_TC_DEBUG), normally null
};

// B element (n, c) of a stage, K-major no-swizzle: core matrices of 8 rows x 16 bytes, the two
// 4-column halves of a k-step LBO = 128 B apart, 8-row groups SBO = 256 B apart, k-steps Kp*32 B
__device__ __forceinline__ uint32_t b_off(int n, int c, int Kp) {
    return (uint32_t)((c >> 3) * Kp * 32 + (n >> 3) * 256 + ((c >> 2) & 1) * 128 + (n & 7) * 16 + (c & 3) * 4);
}

__global__ void __launch_bounds__(kThreads, 1) k_tc_sketch_f32(const __grid_constant__ CUtensorMap xmap, TcSkArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // ---- carve: [stages: A hi | A lo | B hi | B lo] (1024-aligned) | tables | barriers
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t stage_bytes = 2 * a.a_bytes + 2 * a.b_bytes;
    GaussTables* tabs = reinterpret_cast<GaussTables*>(gbase + (size_t)a.S * stage_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(tabs) + sizeof(GaussTables));
    uint64_t* full = bars;               // TMA landed (expect_tx)
    uint64_t* split = bars + a.S;        // X split into hi / lo (kSplitWarps arrivals)
    uint64_t* omega = bars + 2 * a.S;    // B generated (kAuxWarps arrivals)
    uint64_t* empty = bars + 3 * a.S;    // MMAs of the stage done (tcgen05.commit)
    uint64_t* done = bars + 4 * a.S;     // every MMA done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * a.S + 1);
    auto A_hi = [&](int s) { return base + (uint32_t)s * stage_bytes; };
    auto A_lo = [&](int s) { return A_hi(s) + a.a_bytes; };
    auto B_hi = [&](int s) { return A_hi(s) + 2 * a.a_bytes; };
    auto B_lo = [&](int s) { return B_hi(s) + a.b_bytes; };

    // this CTA's tiles (kb columns each): a contiguous range
    const int64_t t0 = a.ntiles * blockIdx.x / gridDim.x, t1 = a.ntiles * (blockIdx.x + 1) / gridDim.x;
    const int nt = (int)(t1 - t0);
    const uint32_t tcols = a.Mt * a.Kp <= 32 ? 32u : a.Mt * a.Kp <= 64 ? 64u : a.Mt * a.Kp <= 128 ? 128u
                                                                               : a.Mt * a.Kp <= 256 ? 256u : 512u;

    // ---- set-up: zero every stage (padding rows / columns stay zero), tables, barriers, TMEM
    for (uint32_t o = threadIdx.x * 16u; o < (uint32_t)a.S * stage_bytes; o += kThreads * 16u)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + o), "r"(0u));
    gauss_tables_to_smem(*tabs, a.gt);
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&split[s], kSplitWarps);
            mbar_init(&omega[s], kAuxWarps);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================= TMA producer
        if (lane == 0) {
            const uint64_t pol = policy_l2(0);
            for (int j = 0; j < nt; ++j) {
                const int s = j % a.S;
                if (j >= a.S) mbar_wait(&empty[s], ((j / a.S) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], (uint32_t)a.nblk * (uint32_t)a.kb * 128u);
                const int c0 = (int)((t0 + j) * a.kb);
                for (int b = 0; b < a.nblk; ++b)
                    tma2d(A_hi(s) + (uint32_t)b * (uint32_t)a.kb * 128u, &xmap, 32 * b, c0, &full[s], pol);
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer
        const uint32_t idesc = idesc_tf32(128, a.Kp, /*a MN-major*/ 1, /*b K-major*/ 0);
        const uint32_t lbo_a = (uint32_t)a.kb * 128u;  // 32-row blocks of A
        for (int j = 0; j < nt; ++j) {
            const int s = j % a.S;
            const uint32_t ph = (j / a.S) & 1;
            mbar_wait(&full[s], ph);
            mbar_wait(&split[s], ph);
            mbar_wait(&omega[s], ph);
            tc_fence_after();
            if (lane == 0) {
                for (int ks = 0; ks < a.kb / 8; ++ks) {
                    const uint64_t bh = sdesc(B_hi(s) + (uint32_t)ks * a.Kp * 32u, 128, 256, kSwNone);
                    const uint64_t bl = sdesc(B_lo(s) + (uint32_t)ks * a.Kp * 32u, 128, 256, kSwNone);
                    for (int mt = 0; mt < a.Mt; ++mt) {
                        // tf32 MN-major operands take the 128B swizzle of 32-byte chunks (the only
                        // MN-major tf32 layout): 4-row groups SBO = 512 B apart, 8 rows per k-step
                        const uint32_t aoff = (uint32_t)mt * 4u * lbo_a + (uint32_t)ks * 1024u;
                        const uint64_t ah = sdesc(A_hi(s) + aoff, lbo_a, 512, kSw128b32);
                        const uint64_t al = sdesc(A_lo(s) + aoff, lbo_a, 512, kSw128b32);
                        const uint32_t d = tmem + (uint32_t)(mt * a.Kp);
                        const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
                        mma_tf32(d, ah, bh, idesc, acc);
                        mma_tf32(d, al, bh, idesc, 1u);
                        mma_tf32(d, ah, bl, idesc, 1u);
                    }
                }
                mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (lane == 0) mma_commit(done);
        __syncwarp();
    } else if (warp >= kSplitW0 && warp < kSplitW0 + kSplitWarps) {
        // ================= X splitters, then the epilogue
        const int tid = threadIdx.x - kSplitW0 * 32;
        const uint32_t real = (uint32_t)a.nblk * (uint32_t)a.kb * 128u;
        for (int j = 0; j < nt; ++j) {
            const int s = j % a.S;
            mbar_wait(&full[s], (j / a.S) & 1);
            split_stage(A_hi(s), A_lo(s), real, tid, kSplitWarps * 32);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&split[s]);
        }
        // epilogue: TMEM lane quarter (warp % 4) holds rows 32 (warp % 4) + lane of each M tile
        const int q = warp & 3;
        double* part = a.partial + (int64_t)blockIdx.x * a.I0 * a.K;
        if (nt > 0) {
            mbar_wait(done, 0);
            tc_fence_after();
        }
        for (int mt = 0; mt < a.Mt; ++mt) {
            const int row = mt * 128 + q * 32 + lane;
            for (int n0 = 0; n0 < a.Kp; n0 += 8) {
                float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (nt > 0) tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(mt * a.Kp + n0), v);
                if (a.dbg && blockIdx.x == 0 && mt == 0 && n0 == 0 && lane < 8)
                    for (int jj = 0; jj < 8; ++jj) a.dbg[800 + q * 64 + lane * 8 + jj] = v[jj];
                if (row < a.I0) {
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if (n0 + jj < a.K) part[row + (int64_t)a.I0 * (n0 + jj)] = (double)v[jj];
                }
            }
        }
        if (a.dbg && blockIdx.x == 0) {  // TMEM store / load round trip in the last allocated column
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (tcols - 1);
            const uint32_t val = __float_as_uint((float)(1000 + q * 32 + lane));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(val) : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            uint32_t r;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            a.dbg[900 + q * 32 + lane] = __uint_as_float(r);
        }
        if (a.dbg && blockIdx.x == 0 && warp == kSplitW0) {
            // stage 0 as last filled: A hi (first 256 floats), A lo, B hi, B lo (first 128 each), TMEM row lane
            for (int e = lane; e < 256; e += 32) {
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(A_hi(0) + 4u * e));
                a.dbg[e] = v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(A_lo(0) + 4u * e));
                a.dbg[256 + e] = v;
            }
            for (int e = lane; e < 128; e += 32) {
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(B_hi(0) + 4u * e));
                a.dbg[512 + e] = v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(B_lo(0) + 4u * e));
                a.dbg[640 + e] = v;
            }
            if (lane == 0) {
                a.dbg[768] = (float)nt;
                a.dbg[769] = (float)tmem;
                a.dbg[770] = (float)a.kb;
                a.dbg[771] = (float)a.S;
            }
        }
        tc_fence_before();
    } else {
        // ================= test-matrix generators: Omega_0(c, k) = draw D + col_off + c + rows_glob k
        const int tid = threadIdx.x - kAuxW0 * 32;
        const int npair = a.kb / 2 + 1;
        for (int j = 0; j < nt; ++j) {
            const int s = j % a.S;
            if (j >= a.S) mbar_wait(&empty[s], ((j / a.S) - 1) & 1);
            const int64_t c0 = (t0 + j) * a.kb;
            const uint32_t bh = B_hi(s), bl = B_lo(s);
            for (int it = tid; it < a.K * npair; it += kAuxWarps * 32) {
                const int k = it / npair, pi = it - k * npair;
                const uint64_t d0 = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)k;
                const uint64_t p = (d0 >> 1) + (uint64_t)pi;  // pair p holds draws 2p, 2p + 1
                double z[2];
                gauss_pair_state(a.seed + (2ull * p + 1ull) * 0x9E3779B97F4A7C15ull, *tabs, z[0], z[1]);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t cl = (int64_t)(2 * p + e) - (int64_t)d0;  // column within the tile
                    if (cl < 0 || cl >= a.kb) continue;
                    const bool in = c0 + cl < a.L;
                    const float w = in ? (float)z[e] : 0.f;
                    const float h = tf32_rna(w);
                    const float l = in ? (float)(z[e] - (double)h) : 0.f;
                    const uint32_t o = b_off(k, (int)cl, a.Kp);
                    sts32(bh + o, h);
                    sts32(bl + o, l);
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&omega[s]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, tcols);
    }
}

struct TcSkPlan {
    int Kp, Mt, nblk, kb, S;
    uint32_t a_bytes, b_bytes;
    size_t smem;
};

bool plan_tc_sketch(int64_t I0, int K, TcSkPlan& p) {
    if (K < 1 || K > 64 || I0 < 1 || I0 > 1024) return false;
    p.Kp = (K + 15) & ~15;
    p.Mt = (int)((I0 + 127) / 128);
    if (p.Mt * p.Kp > 512) return false;
    p.nblk = (int)((I0 + 31) / 32);
    // ~24-32 KB of X per stage
    p.kb = 8;
    while (p.kb < 64 && (size_t)p.nblk * (p.kb * 2) * 128 <= 32768) p.kb *= 2;
    p.a_bytes = (uint32_t)p.Mt * 4u * (uint32_t)p.kb * 128u;
    p.b_bytes = (uint32_t)p.Kp * (uint32_t)p.kb * 4u;
    const size_t stage = 2 * (size_t)p.a_bytes + 2 * (size_t)p.b_bytes;
    const size_t fixed = 1024 + sizeof(GaussTables) + 8 * (4 * 8 + 2) + 64;
    p.S = (int)std::min<size_t>(4, (227 * 1024 - fixed) / stage);
    p.smem = (size_t)p.S * stage + fixed;
    return p.S >= 2;
}

// ================================================================== K2: mode-0 shrink
struct TcTtArgs {
    int I0, K, Kp, nchunk, S;
    int64_t L, ntiles;  // tiles of 256 fibres
    void* out;          // P^(1): K x L column-major, fp32 or fp64
    uint32_t a_bytes, q_bytes;
};

template <bool F64OUT>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_ttm_f32(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap qhmap,
                 const __grid_constant__ CUtensorMap qlmap, TcTtArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t stage_bytes = 2 * a.a_bytes + 2 * a.q_bytes;  // X hi | X lo | Q hi | Q lo
    uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (size_t)a.S * stage_bytes);
    uint64_t* full = bars;
    uint64_t* split = bars + a.S;
    uint64_t* empty = bars + 2 * a.S;
    uint64_t* tfull = bars + 3 * a.S;   // [2] accumulator buffer ready for the epilogue
    uint64_t* tempty = bars + 3 * a.S + 2;  // [2] accumulator buffer drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * a.S + 4);
    auto X_hi = [&](int s) { return base + (uint32_t)s * stage_bytes; };
    auto X_lo = [&](int s) { return X_hi(s) + a.a_bytes; };
    auto Q_hi = [&](int s) { return X_hi(s) + 2 * a.a_bytes; };
    auto Q_lo = [&](int s) { return Q_hi(s) + a.q_bytes; };
    const uint32_t tcols = 4 * a.Kp <= 64 ? 64u : 4 * a.Kp <= 128 ? 128u : 256u;  // 2 buffers x 2 halves x Kp

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&split[s], kSplitWarps);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kAuxWarps);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // tiles: blockIdx.x, blockIdx.x + grid, ...
    const int nt = a.ntiles > blockIdx.x ? (int)((a.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = policy_l2(0), pol_q = policy_l2(2);
            griddep_wait();  // Q (and, in the chain, X's producer) come from the previous grids
            int g = 0;
            for (int j = 0; j < nt; ++j) {
                const int c0 = (int)((blockIdx.x + (int64_t)j * gridDim.x) * 256);
                for (int ch = 0; ch < a.nchunk; ++ch, ++g) {
                    const int s = g % a.S;
                    if (g >= a.S) mbar_wait(&empty[s], ((g / a.S) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], a.a_bytes + 2 * a.q_bytes);
                    tma2d(X_hi(s), &xmap, 32 * ch, c0, &full[s], pol_x);
                    tma2d(X_hi(s) + a.a_bytes / 2, &xmap, 32 * ch, c0 + 128, &full[s], pol_x);
                    tma2d(Q_hi(s), &qhmap, 32 * ch, 0, &full[s], pol_q);
                    tma2d(Q_lo(s), &qlmap, 32 * ch, 0, &full[s], pol_q);
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = idesc_tf32(128, a.Kp, 0, 0);
        int g = 0;
        for (int j = 0; j < nt; ++j) {
            const int buf = j & 1;
            if (j >= 2) mbar_wait(&tempty[buf], ((j >> 1) - 1) & 1);
            tc_fence_after();
            for (int ch = 0; ch < a.nchunk; ++ch, ++g) {
                const int s = g % a.S;
                const uint32_t ph = (g / a.S) & 1;
                mbar_wait(&full[s], ph);
                mbar_wait(&split[s], ph);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {  // 4 k-steps of 8 in the 128-byte rows
                        const uint64_t qh = sdesc(Q_hi(s) + ks * 32u, 16, 1024, kSw128);
                        const uint64_t ql = sdesc(Q_lo(s) + ks * 32u, 16, 1024, kSw128);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t ao = (uint32_t)h * (a.a_bytes / 2) + ks * 32u;
                            const uint64_t xh = sdesc(X_hi(s) + ao, 16, 1024, kSw128);
                            const uint64_t xl = sdesc(X_lo(s) + ao, 16, 1024, kSw128);
                            const uint32_t d = tmem + (uint32_t)((buf * 2 + h) * a.Kp);
                            const uint32_t acc = (ch > 0 || ks > 0) ? 1u : 0u;
                            mma_tf32(d, xh, qh, idesc, acc);
                            mma_tf32(d, xl, qh, idesc, 1u);
                            mma_tf32(d, xh, ql, idesc, 1u);
                        }
                    }
                    mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (lane == 0) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp >= kSplitW0 && warp < kSplitW0 + kSplitWarps) {
        const int tid = threadIdx.x - kSplitW0 * 32;
        const int total = nt * a.nchunk;
        for (int g = 0; g < total; ++g) {
            const int s = g % a.S;
            mbar_wait(&full[s], (g / a.S) & 1);
            split_stage(X_hi(s), X_lo(s), a.a_bytes, tid, kSplitWarps * 32);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&split[s]);
        }
    } else {
        // ================= epilogue: TMEM lane = fibre of the tile, columns = the K outputs
        const int q = warp & 3;
        for (int j = 0; j < nt; ++j) {
            const int buf = j & 1;
            mbar_wait(&tfull[buf], (j >> 1) & 1);
            tc_fence_after();
            const int64_t tc0 = (blockIdx.x + (int64_t)j * gridDim.x) * 256;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int64_t c = tc0 + h * 128 + q * 32 + lane;
                for (int n0 = 0; n0 < a.Kp; n0 += 8) {
                    float v[8];
                    tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((buf * 2 + h) * a.Kp + n0), v);
                    if (c < a.L) {
                        if constexpr (F64OUT) {
                            double* o = reinterpret_cast<double*>(a.out) + c * a.K + n0;
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj)
                                if (n0 + jj < a.K) o[jj] = (double)v[jj];
                        } else {
                            float* o = reinterpret_cast<float*>(a.out) + c * a.K + n0;
                            if (n0 + 8 <= a.K && (a.K & 3) == 0) {
                                *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
                                *reinterpret_cast<float4*>(o + 4) = make_float4(v[4], v[5], v[6], v[7]);
                            } else {
#pragma unroll
                                for (int jj = 0; jj < 8; ++jj)
                                    if (n0 + jj < a.K) o[jj] = v[jj];
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, tcols);
    }
}

// Q (fp64, ldq x K column-major, rows [0, I0)) -> Qt_hi / Qt_lo (fp32, Kp x Ip, i fastest),
// zero-padded: the K2 B operand, split for 3xTF32
__global__ void k_qt_prep(const double* __restrict__ q, int64_t ldq, int I0, int K, int Ip, int Kp, float* hi,
                          float* lo) {
    griddep_wait();
    const int n = Kp * Ip;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int k = e / Ip, i = e - k * Ip;
        const double v = (k < K && i < I0) ? q[i + ldq * k] : 0.0;
        const float h = tf32_rna((float)v);
        hi[e] = h;
        lo[e] = (float)(v - (double)h);
    }
    griddep_launch_dependents();
}

struct TcTtPlan {
    int Kp, nchunk, S, Ip;
    uint32_t a_bytes, q_bytes;
    size_t smem;
};

bool plan_tc_ttm(int64_t I0, int64_t K, TcTtPlan& p) {
    if (K < 1 || K > 64 || I0 < 1 || I0 > 4096 || (I0 % 4) != 0) return false;
    p.Kp = (int)((K + 15) & ~15);
    p.nchunk = (int)((I0 + 31) / 32);
    p.Ip = p.nchunk * 32;
    p.a_bytes = 256u * 128u;                // two 128-fibre halves x 32 rows x 4 B
    p.q_bytes = (uint32_t)p.Kp * 128u;      // Kp rows x 32 i x 4 B
    const size_t stage = 2 * (size_t)p.a_bytes + 2 * (size_t)p.q_bytes;
    const size_t fixed = 1024 + 8 * (3 * 8 + 4) + 64;
    p.S = (int)std::min<size_t>(4, (227 * 1024 - fixed) / stage);
    p.smem = (size_t)p.S * stage + fixed;
    return p.S >= 2;
}

void encode2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
              uint32_t box_out, CUtensorMapSwizzle sw) {
    const cuuint64_t gdim[2] = {inner, outer};
    const cuuint64_t gstride[1] = {row_bytes};
    const cuuint32_t box[2] = {box_in, box_out};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), gdim, gstride, box,
                                   estride, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (tc_f32)");
}

}  // namespace

// ------------------------------------------------------------------ host side
bool tc_sketch_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols) {
    TcSkPlan p;
    if (getenv("TRG_NO_TCGEN05")) return false;
    return dtype == F32 && left == 1 && (dim % 4) == 0 && ncols < (int64_t(1) << 31) && encode_fn() &&
           plan_tc_sketch(dim, K, p);
}

int launch_tc_sketch_f32(const SketchPlan& sp, const void* x, double* partial, double* y, int num_sms,
                         cudaStream_t s) {
    TcSkPlan p;
    if (!plan_tc_sketch(sp.dim, sp.K, p)) throw std::runtime_error("tc sketch: unsupported shape");
    TcSkArgs a{};
    a.I0 = (int)sp.dim;
    a.K = sp.K;
    a.Kp = p.Kp;
    a.Mt = p.Mt;
    a.nblk = p.nblk;
    a.kb = p.kb;
    a.S = p.S;
    a.L = sp.right;
    a.ntiles = (sp.right + p.kb - 1) / p.kb;
    a.seed = sp.seed;
    a.D = sp.D;
    a.rows_glob = sp.rows_glob;
    a.col_off = sp.col_off;
    a.partial = partial;
    a.gt = gauss_tables(s);
    a.a_bytes = p.a_bytes;
    a.b_bytes = p.b_bytes;
    CUtensorMap map;
    encode2d(&map, x, (uint64_t)sp.dim, (uint64_t)sp.right, (uint64_t)sp.dim * 4, 32, (uint32_t)p.kb,
             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    const char* dbg_path = getenv("TRG_TC_DEBUG");
    if (dbg_path) cudaMalloc(&a.dbg, 1024 * sizeof(float)), cudaMemset(a.dbg, 0, 1024 * sizeof(float));
    allow_smem(k_tc_sketch_f32, p.smem);
    k_tc_sketch_f32<<<grid, kThreads, p.smem, s>>>(map, a);
    if (dbg_path) {
        float h[1024];
        cudaStreamSynchronize(s);
        fprintf(stderr, "tc_sketch launch: %s grid %d smem %zu S %d kb %d\n", cudaGetErrorString(cudaGetLastError()),
                grid, p.smem, p.S, p.kb);
        cudaMemcpy(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(dbg_path, "wb")) fwrite(h, sizeof(h), 1, f), fclose(f);
        cudaFree(a.dbg);
    }
    if (y) launch_reduce_partials(partial, grid, sp.dim * sp.K, y, s);
    return grid;
}

int tc_sketch_f32_grid(int64_t dim, int K, int64_t ncols, int num_sms) {
    TcSkPlan p;
    plan_tc_sketch(dim, K, p);
    return (int)std::max<int64_t>(1, std::min<int64_t>((ncols + p.kb - 1) / p.kb, num_sms));
}

bool tc_ttm_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols) {
    TcTtPlan p;
    if (getenv("TRG_NO_TCGEN05")) return false;
    return dtype == F32 && left == 1 && ncols < (int64_t(1) << 31) && encode_fn() && plan_tc_ttm(dim, K, p);
}

size_t tc_ttm_f32_scratch(int64_t dim, int64_t K) {
    TcTtPlan p;
    plan_tc_ttm(dim, K, p);
    return 2 * sizeof(float) * (size_t)p.Kp * p.Ip;
}

void launch_tc_ttm_f32(const TTMPlan& tp, const void* in, void* out, bool f64_out, const double* q, int64_t ldq,
                       float* scratch, int num_sms, cudaStream_t s) {
    TcTtPlan p;
    if (!plan_tc_ttm(tp.dim, tp.odim, p)) throw std::runtime_error("tc shrink: unsupported shape");
    float* qh = scratch;
    float* ql = scratch + (size_t)p.Kp * p.Ip;
    {
        const int n = p.Kp * p.Ip;
        pdl_launch(k_qt_prep, dim3(std::min(64, (n + 255) / 256)), dim3(256), 0, s, q, ldq, (int)tp.dim,
                   (int)tp.odim, p.Ip, p.Kp, qh, ql);
    }
    TcTtArgs a{};
    a.I0 = (int)tp.dim;
    a.K = (int)tp.odim;
    a.Kp = p.Kp;
    a.nchunk = p.nchunk;
    a.S = p.S;
    a.L = tp.right;
    a.ntiles = (tp.right + 255) / 256;
    a.out = out;
    a.a_bytes = p.a_bytes;
    a.q_bytes = p.q_bytes;
    CUtensorMap xm, qhm, qlm;
    encode2d(&xm, in, (uint64_t)tp.dim, (uint64_t)tp.right, (uint64_t)tp.dim * 4, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    encode2d(&qhm, qh, (uint64_t)p.Ip, (uint64_t)p.Kp, (uint64_t)p.Ip * 4, 32, (uint32_t)p.Kp,
             CU_TENSOR_MAP_SWIZZLE_128B);
    encode2d(&qlm, ql, (uint64_t)p.Ip, (uint64_t)p.Kp, (uint64_t)p.Ip * 4, 32, (uint32_t)p.Kp,
             CU_TENSOR_MAP_SWIZZLE_128B);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    if (f64_out) {
        allow_smem(k_tc_ttm_f32<true>, p.smem);
        pdl_launch(k_tc_ttm_f32<true>, dim3(grid), dim3(kThreads), p.smem, s, xm, qhm, qlm, a);
    } else {
        allow_smem(k_tc_ttm_f32<false>, p.smem);
        pdl_launch(k_tc_ttm_f32<false>, dim3(grid), dim3(kThreads), p.smem, s, xm, qhm, qlm, a);
    }
}

}  // namespace trg
