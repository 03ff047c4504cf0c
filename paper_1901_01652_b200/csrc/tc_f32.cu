// SPDX-License-Identifier: Apache-2.0
//
// fp32 mode-0 sketch and shrink on the 5th-generation tensor cores (tcgen05, kind::tf32, TMEM
// accumulators, TMA-fed shared memory), in 3xTF32: every fp32 operand v is split into
// hi = trunc_tf32(v) (what the tensor core reads from the raw fp32 word) and lo = v - hi (exact),
// and  v w  ~  hi_v hi_w + lo_v hi_w + hi_v lo_w. The dropped lo_v lo_w is below 2^-20 |v w| and
// the lo operands are read to 11 bits, so a product carries ~1e-6 relative error, random in
// sign: the stage stays far inside the 1e-4 fp32 parity bound against the fp64 oracle, while
// plain TF32 (2^-10 truncation) would not (BASELINE.json north_star).
// Only lo is written to shared memory (the raw X tile is its own hi), and the tensor core reads
// X twice (K2: hi against [Q_hi | Q_lo] concatenated along N, lo against Q_hi).
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

// kind::tf32 reads an fp32 operand as its top 19 bits, i.e. TRUNCATED (measured,
// tools/tc_probe.cu): a raw fp32 buffer is its own hi part, and lo = v - trunc(v) is exact.
__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// lo = v - trunc_tf32(v) of one stage (layout-agnostic), four 16-byte loads in flight per thread
__device__ __forceinline__ void split_lo(uint32_t src, uint32_t lo, uint32_t bytes, int tid, int nthr) {
    const uint32_t step = (uint32_t)nthr * 16u;
    uint32_t o = (uint32_t)tid * 16u;
    for (; o + 3 * step < bytes; o += 4 * step) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                         : "r"(src + o + u * step));
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lo + o + u * step), "f"(v[u].x - tf32_trunc(v[u].x)),
                         "f"(v[u].y - tf32_trunc(v[u].y)), "f"(v[u].z - tf32_trunc(v[u].z)),
                         "f"(v[u].w - tf32_trunc(v[u].w)));
    }
    for (; o < bytes; o += step) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(src + o));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lo + o), "f"(v.x - tf32_trunc(v.x)),
                     "f"(v.y - tf32_trunc(v.y)), "f"(v.z - tf32_trunc(v.z)), "f"(v.w - tf32_trunc(v.w)));
    }
}

__device__ __forceinline__ void sts32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }

constexpr int kSplitW0 = 2, kSplitWarps = 4;  // warps 2..5

// ================================================================== K1: mode-0 sketch
// Y_0 (I0 x K) = X_(0) Omega_0: D[M x N] += A[M x 8] B[8 x N] per k-step, A = 32-row blocks of an
// X column block (MN-major, M = 128 per tile, or 64 when I0 <= 64), B = Omega block (K-major).
// Rings: X (XR deep, TMA -> MMA), lo of X (2 deep, splitters -> MMA) and Omega hi / lo (BR deep,
// generators -> MMA: the generators run ahead of the tensor core). Warps: 0 TMA, 1 MMA (+ TMEM),
// 2-5 splitters, 6-17 generators, 18-21 drainers.
// The tensor core's fp32 accumulation loses about one rounding per accumulation step (measured:
// Y_0 error ~ linear in the columns a CTA accumulates, 1e-5 after ~1400 columns, 6e-4 after C5's
// 87k), so the accumulator is drained into the CTA's fp64 partial every `seg` stages (~256
// columns): the MMAs alternate between two TMEM accumulator sets while the drainers add the idle
// one into the partial (RMW in L2; the CTA owns its slab). When two sets do not fit TMEM (C4: 8 x
// 64 of 512 columns) a CTA drains once, at its end. With N-concatenation (ncat: D = A [B_hi B_lo]
// + A_lo B_hi, two MMAs) a set is 2 Kp wide and the drain sums its halves.
constexpr int kSkGenW0 = 6, kSkGenWarps = 12, kSkDrainW0 = 18, kSkDrainWarps = 4;
constexpr int kSkThreads = 22 * 32;
constexpr int kWR = 2;  // lo-ring depth
static_assert(kSkDrainW0 + kSkDrainWarps == kSkThreads / 32 && kSkGenW0 + kSkGenWarps == kSkDrainW0, "warp roles");

struct TcSkArgs {
    int I0, K, Kp, M, Mt, nblk, kb, XR, BR, seg, nset, ncat, RS, WR;  // WR: lo-ring depth  // Mt: M tiles per CTA, RS row splits
    int64_t L, ntiles;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    double* partial;  // per CTA: I0 x K fp64, column-major
    uint32_t a_bytes, b_bytes;  // X block (M-padded) and one of B hi / lo
    long long* prof;  // development timeline (TRG_TC_PROF): CTA 0, 8 stamps x 256 stages
};
#define TC_STAMP(slot, j)                                                        \
    do {                                                                         \
        if (a.prof && blockIdx.x == 0 && (j) < 256) a.prof[(slot) * 256 + (j)] = clock64(); \
    } while (0)

// B element (n, c) of a stage, K-major no-swizzle: core matrices of 8 rows x 16 bytes, the two
// 4-column halves of a k-step LBO = 128 B apart, 8-row groups SBO = 256 B apart; k-step blocks
// of NB rows (2 Kp with N-concatenation: B_lo rows follow B_hi's) NB * 32 B apart
__device__ __forceinline__ uint32_t b_off(int n, int c, int NB) {
    return (uint32_t)((c >> 3) * NB * 32 + (n >> 3) * 256 + ((c >> 2) & 1) * 128 + (n & 7) * 16 + (c & 3) * 4);
}

__global__ void __launch_bounds__(kSkThreads, 1) k_tc_sketch_f32(const __grid_constant__ CUtensorMap xmap, TcSkArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // ---- carve (1024-aligned): X ring | lo ring | B ring [hi | lo] | barriers
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t lbase = base + (uint32_t)a.XR * a.a_bytes;
    const uint32_t bbase = lbase + (uint32_t)a.WR * a.a_bytes;
    const uint32_t ring_bytes = (uint32_t)(a.XR + a.WR) * a.a_bytes + (uint32_t)a.BR * 2u * a.b_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + ring_bytes);
    uint64_t* xfull = bars;                  // [XR] TMA landed
    uint64_t* xempty = xfull + a.XR;         // [XR] MMAs done with the X slot
    uint64_t* wsplit = xempty + a.XR;        // [2] lo written
    uint64_t* wempty = wsplit + a.WR;         // [2] MMAs done with the lo slot
    uint64_t* bfull = wempty + a.WR;          // [BR] Omega block written
    uint64_t* bempty = bfull + a.BR;         // [BR] MMAs done with the Omega slot
    uint64_t* dfull = bempty + a.BR;         // [2] accumulator set ready to drain
    uint64_t* dempty = dfull + 2;            // [2] accumulator set drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);
    auto X = [&](int r) { return base + (uint32_t)r * a.a_bytes; };
    auto LO = [&](int w) { return lbase + (uint32_t)w * a.a_bytes; };
    auto BH = [&](int b) { return bbase + (uint32_t)b * 2u * a.b_bytes; };
    auto BL = [&](int b) { return BH(b) + a.b_bytes; };  // with ncat: rows Kp.. of one B block
    const int NB = a.ncat ? 2 * a.Kp : a.Kp;              // rows of a B k-step block

    // CTA = (column group cg, row split rs): rows [rs Mt M, (rs + 1) Mt M) of the column group's
    // columns (C3 / C4 split their rows so that two N-concatenated accumulator sets fit TMEM;
    // the RS CTAs of a column group regenerate the same test-matrix block)
    const int rs = blockIdx.x % a.RS, cg = blockIdx.x / a.RS, ncg = gridDim.x / a.RS;
    const int bpt = a.M / 32;  // 32-row blocks per M tile
    const int blk0 = rs * a.Mt * bpt;
    const int nbc = max(0, min(a.nblk - blk0, a.Mt * bpt));  // real blocks of this CTA
    const int64_t t0 = a.ntiles * cg / ncg, t1 = a.ntiles * (cg + 1) / ncg;
    const int nt = (int)(t1 - t0);
    const int nseg = (nt + a.seg - 1) / a.seg;
    const uint32_t setcols = (uint32_t)(a.Mt * (a.ncat ? 2 : 1) * a.Kp);
    const uint32_t need = setcols * (uint32_t)a.nset;
    const uint32_t tcols = need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;

    // ---- set-up: zero both rings (padding rows / columns stay zero), barriers, TMEM
    for (uint32_t o = threadIdx.x * 16u; o < ring_bytes; o += kSkThreads * 16u)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + o), "r"(0u));
    if (threadIdx.x == 0) {
        for (int r = 0; r < a.XR; ++r) {
            mbar_init(&xfull[r], 1);
            mbar_init(&xempty[r], 1);
        }
        for (int w = 0; w < a.WR; ++w) {
            mbar_init(&wsplit[w], kSplitWarps);
            mbar_init(&wempty[w], 1);
        }
        for (int b = 0; b < a.BR; ++b) {
            mbar_init(&bfull[b], kSkGenWarps);
            mbar_init(&bempty[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], kSkDrainWarps);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lbo_a = (uint32_t)a.kb * 128u;  // 32-row blocks of A

    if (warp == 0) {
        // ================= TMA producer (X ring)
        if (lane == 0) {
            const uint64_t pol = policy_l2(0);
            for (int j = 0; j < nt; ++j) {
                const int r = j % a.XR;
                TC_STAMP(0, j);
                if (j >= a.XR) mbar_wait(&xempty[r], ((j / a.XR) - 1) & 1);
                TC_STAMP(1, j);
                mbar_arrive_expect_tx(&xfull[r], (uint32_t)nbc * lbo_a);
                const int c0 = (int)((t0 + j) * a.kb);
                for (int b = 0; b < nbc; ++b)
                    tma2d(X(r) + (uint32_t)b * lbo_a, &xmap, 32 * (blk0 + b), c0, &xfull[r], pol);
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer
        const uint32_t idesc1 = idesc_tf32(a.M, NB, /*a MN-major*/ 1, /*b K-major*/ 0);
        const uint32_t idesc2 = idesc_tf32(a.M, a.Kp, 1, 0);
        for (int g = 0; g < nseg; ++g) {
            const int set = g % a.nset;
            if (g >= a.nset) mbar_wait(&dempty[set], ((g / a.nset) - 1) & 1);
            tc_fence_after();
            const int j1 = min(nt, (g + 1) * a.seg);
            for (int j = g * a.seg; j < j1; ++j) {
                const int r = j % a.XR, w = j % a.WR, bq = j % a.BR;
                mbar_wait(&xfull[r], (j / a.XR) & 1);
                if (lane == 0) TC_STAMP(2, j);
                mbar_wait(&wsplit[w], (j / a.WR) & 1);
                mbar_wait(&bfull[bq], (j / a.BR) & 1);
                if (lane == 0) TC_STAMP(3, j);
                tc_fence_after();
                if (lane == 0) {
                    for (int ks = 0; ks < a.kb / 8; ++ks) {
                        const uint64_t bh = sdesc(BH(bq) + (uint32_t)ks * NB * 32u, 128, 256, kSwNone);
                        const uint64_t bl = sdesc(BL(bq) + (uint32_t)ks * a.Kp * 32u, 128, 256, kSwNone);
                        for (int mt = 0; mt < a.Mt; ++mt) {
                            // tf32 MN-major operands take the 128B swizzle of 32-byte chunks (the
                            // only MN-major tf32 layout): 4-row groups SBO = 512 B apart, 8 rows per k-step
                            const uint32_t aoff = (uint32_t)mt * 4u * lbo_a + (uint32_t)ks * 1024u;
                            const uint64_t ah = sdesc(X(r) + aoff, lbo_a, 512, kSw128b32);
                            const uint64_t al = sdesc(LO(w) + aoff, lbo_a, 512, kSw128b32);
                            const uint32_t d = tmem + (uint32_t)set * setcols + (uint32_t)(mt * (a.ncat ? 2 : 1) * a.Kp);
                            const uint32_t acc = (j > g * a.seg || ks > 0) ? 1u : 0u;
                            mma_tf32(d, ah, bh, idesc1, acc);  // hi [B_hi (B_lo)]
                            mma_tf32(d, al, bh, idesc2, 1u);   // lo B_hi
                            if (!a.ncat) mma_tf32(d, ah, bl, idesc2, 1u);
                        }
                    }
                    mma_commit(&xempty[r]);
                    mma_commit(&wempty[w]);
                    mma_commit(&bempty[bq]);
                }
                __syncwarp();
            }
            if (lane == 0) mma_commit(&dfull[set]);
            __syncwarp();
        }
    } else if (warp >= kSplitW0 && warp < kSplitW0 + kSplitWarps) {
        // ================= X splitters: lo = X - trunc_tf32(X) into the work ring
        const int tid = threadIdx.x - kSplitW0 * 32;
        const uint32_t real = (uint32_t)nbc * lbo_a;
        for (int j = 0; j < nt; ++j) {
            const int r = j % a.XR, w = j % a.WR;
            if (j >= a.WR) mbar_wait(&wempty[w], ((j / a.WR) - 1) & 1);
            mbar_wait(&xfull[r], (j / a.XR) & 1);
            if (tid == 0) TC_STAMP(4, j);
            split_lo(X(r), LO(w), real, tid, kSplitWarps * 32);
            fence_async_smem();
            __syncwarp();
            if (tid == 0) TC_STAMP(5, j);
            if (lane == 0) mbar_arrive(&wsplit[w]);
        }
    } else if (warp >= kSkGenW0 && warp < kSkGenW0 + kSkGenWarps) {
        // ================= test-matrix generators: Omega_0(c, k) = draw D + col_off + c + rows_glob k
        // (fp32 Box-Muller, ~1e-7 relative per draw: far below the 1e-4 fp32 bound and the 3xTF32
        // error, at half the issue cost of the fp64 generator the fp64 kernels need)
        const int tid = threadIdx.x - kSkGenW0 * 32;
        const int npair = a.kb / 2 + 1;
        // items (pair pi, column k), k fastest across the lanes: consecutive lanes store into
        // consecutive 16-byte rows of the B core matrices (fewer bank conflicts)
        const int stride = kSkGenWarps * 32, dpi = stride / a.K, dk = stride % a.K;
        const int pi0 = tid / a.K, k0 = tid % a.K;
        for (int j = 0; j < nt; ++j) {
            const int bq = j % a.BR;
            if (j >= a.BR) mbar_wait(&bempty[bq], ((j / a.BR) - 1) & 1);
            if (tid == 0) TC_STAMP(6, j);
            const int64_t c0 = (t0 + j) * a.kb;
            const uint32_t bh = BH(bq), bl = a.ncat ? BH(bq) : BL(bq);
            const int lo_row = a.ncat ? a.Kp : 0;
            // four independent items per iteration: the Box-Muller chains interleave (ILP)
            int pi = pi0, k = k0;
            while (pi < npair) {
                int pu[4], ku[4];
                float z[4][2];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    pu[u] = pi;
                    ku[u] = k;
                    pi += dpi;
                    k += dk;
                    if (k >= a.K) {
                        k -= a.K;
                        ++pi;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (u > 0 && pu[u] >= npair) break;  // past the stage's last pair: no draw
                    const uint64_t d0 = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)ku[u];
                    const uint64_t p = (d0 >> 1) + (uint64_t)pu[u];  // pair p holds draws 2p, 2p + 1
                    gauss_pair_f32_fast(a.seed + (2ull * p + 1ull) * 0x9E3779B97F4A7C15ull, z[u][0], z[u][1]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (pu[u] >= npair) break;
                    const uint64_t d0 = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)ku[u];
                    const uint64_t p = (d0 >> 1) + (uint64_t)pu[u];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int64_t cl = (int64_t)(2 * p + e) - (int64_t)d0;  // column within the tile
                        if (cl < 0 || cl >= a.kb) continue;
                        const float v = c0 + cl < a.L ? z[u][e] : 0.f;
                        sts32(bh + b_off(ku[u], (int)cl, NB), v);  // read as trunc_tf32(v)
                        sts32(bl + b_off(ku[u] + lo_row, (int)cl, NB), v - tf32_trunc(v));
                    }
                }
            }
            fence_async_smem();
            __syncwarp();
            if (tid == 0) TC_STAMP(7, j);
            if (lane == 0) mbar_arrive(&bfull[bq]);
        }
    } else {
        // ================= drainers: M = 128, lane quarter q holds rows 32 q + lane of each tile;
        // M = 64, rows 16 q + lane (lanes 0-15 of each quarter). Segment g adds accumulator set
        // g % nset into the CTA's fp64 partial.
        const int q = warp & 3;
        double* part = a.partial + (int64_t)cg * a.I0 * a.K;
        const int rq = a.M == 128 ? 32 : 16;
        const int tw = (a.ncat ? 2 : 1) * a.Kp;
        for (int g = 0; g < nseg; ++g) {
            const int set = g % a.nset;
            mbar_wait(&dfull[set], (g / a.nset) & 1);
            tc_fence_after();
            for (int mt = 0; mt < a.Mt; ++mt) {
                const int row = (rs * a.Mt + mt) * a.M + q * rq + lane;
                const bool own = lane < rq && row < a.I0;
                for (int n0 = 0; n0 < a.Kp; n0 += 16) {  // 16 partial values in flight per batch
                    float v[16];
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)set * setcols + (uint32_t)(mt * tw + n0);
                    tmem_ld8(ta, *reinterpret_cast<float(*)[8]>(&v[0]));
                    tmem_ld8(ta + 8u, *reinterpret_cast<float(*)[8]>(&v[8]));
                    if (a.ncat) {
                        float u[8];
                        tmem_ld8(ta + (uint32_t)a.Kp, u);
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) v[jj] += u[jj];
                        tmem_ld8(ta + (uint32_t)a.Kp + 8u, u);
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) v[8 + jj] += u[jj];
                    }
                    if (own) {
                        double old[16];
                        if (g > 0) {
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj)
                                old[jj] = n0 + jj < a.K ? part[row + (int64_t)a.I0 * (n0 + jj)] : 0.0;
                        } else {
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) old[jj] = 0.0;
                        }
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            if (n0 + jj < a.K) part[row + (int64_t)a.I0 * (n0 + jj)] = old[jj] + (double)v[jj];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dempty[set]);
        }
        if (nseg == 0)  // no columns: a zero partial
            for (int mt = 0; mt < a.Mt; ++mt) {
                const int row = (rs * a.Mt + mt) * a.M + q * rq + lane;
                if (lane < rq && row < a.I0)
                    for (int n = 0; n < a.K; ++n) part[row + (int64_t)a.I0 * n] = 0.0;
            }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, tcols);
    }
}

struct TcSkPlan {
    int Kp, M, Mt, RS, nblk, kb, XR, BR, nset, ncat, seg, WR;
    uint32_t a_bytes, b_bytes;
    size_t smem;
};

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

bool plan_tc_sketch(int64_t I0, int K, TcSkPlan& p) {
    if (K < 1 || K > 64 || I0 < 1 || I0 > 1024) return false;
    p.Kp = (K + 15) & ~15;
    p.M = I0 <= 64 ? 64 : 128;
    const int mt_all = (int)((I0 + p.M - 1) / p.M);
    // No row splits (each would regenerate the test matrix); N-concatenation (the tensor core reads
    // X twice instead of three times) when two such accumulator sets fit TMEM's 512 columns; two
    // sets (drained every ~256 columns) when they fit, else one drained at the CTA's end (C4:
    // 8 x 64 columns; measured 349 us against 656 / 469 us with two / four row splits).
    auto cols = [&](int rs, int ncat) { return 2 * ((mt_all + rs - 1) / rs) * (ncat ? 2 : 1) * p.Kp; };
    p.RS = env_int("TRG_TC_SK_RS", 1);
    p.ncat = env_int("TRG_TC_SK_NCAT", cols(p.RS, 1) <= 512 ? 1 : 0);
    p.Mt = (mt_all + p.RS - 1) / p.RS;
    p.nset = cols(p.RS, p.ncat) <= 512 ? 2 : 1;
    if (p.Mt * (p.ncat ? 2 : 1) * p.Kp > 512) return false;
    p.nblk = (int)((I0 + 31) / 32);
    const int bpc = p.Mt * (p.M / 32);  // blocks per CTA stage
    // ~32 KB of X per stage with a two-deep lo ring; when that leaves one k-step per stage (all of a
    // 1024-row I0 in one CTA: C4), 64 KB stages of two k-steps with a one-deep lo ring instead
    // (C4 sketch_m0 346 -> 311 us: the per-stage barrier and generator overheads were exposed)
    auto kb_for = [&](size_t stage) {
        int kb = 8;
        while (kb < 128 && (size_t)bpc * (kb * 2) * 128 <= stage) kb *= 2;
        return kb;
    };
    p.kb = kb_for((size_t)env_int("TRG_TC_SK_STAGE", 32768));
    p.WR = kWR;
    if (p.kb == 8 && !getenv("TRG_TC_SK_STAGE")) {
        p.kb = kb_for(65536);
        p.WR = 1;
    }
    p.WR = env_int("TRG_TC_SK_WR", p.WR);
    p.seg = p.nset == 2 ? std::max(1, 256 / p.kb) : (1 << 30);  // drain every ~256 columns
    p.a_bytes = (uint32_t)bpc * (uint32_t)p.kb * 128u;
    p.b_bytes = (uint32_t)p.Kp * (uint32_t)p.kb * 4u;
    const size_t fixed = 1024 + 8 * (2 * 8 + 2 * kWR + 2 * 16 + 4) + 64;
    const size_t budget = 227 * 1024 - fixed - (size_t)p.WR * p.a_bytes;
    // X ring first (the HBM stream), then the test-matrix ring up to 8 deep
    p.XR = (int)std::min<size_t>(8, (budget - 2 * 2 * (size_t)p.b_bytes) / p.a_bytes);
    p.BR = (int)std::min<size_t>(8, (budget - (size_t)p.XR * p.a_bytes) / (2 * (size_t)p.b_bytes));
    p.XR = env_int("TRG_TC_SK_XR", p.XR);
    p.smem = (size_t)(p.XR + p.WR) * p.a_bytes + (size_t)p.BR * 2 * p.b_bytes + fixed;
    return p.XR >= 2 && p.BR >= 2 && p.smem <= 227 * 1024;
}

// ================================================================== K2: mode-0 shrink
// per tile of 256 fibres: D[256 x 2 Kp] = X^T [Q_hi | Q_lo] + (X_lo^T Q_hi in the first Kp
// columns), as two M = 128 halves. Rings: X + Q slabs (XR deep, TMA -> MMA), lo (2 deep).
// Warps: 0 TMA, 1 MMA (+ TMEM), 2-5 splitters, 6-9 epilogue.
constexpr int kTtThreads = 10 * 32;
constexpr int kTtEpiW0 = 6;

struct TcTtArgs {
    int I0, K, Kp, nchunk, XR;
    int64_t L, ntiles;  // tiles of 256 fibres
    void* out;          // P^(1): K x L column-major, fp32 or fp64
    uint32_t a_bytes, q_bytes;
};

template <bool F64OUT>
__global__ void __launch_bounds__(kTtThreads, 1)
    k_tc_ttm_f32(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap qhmap,
                 const __grid_constant__ CUtensorMap qlmap, TcTtArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t xbytes = a.a_bytes + 2 * a.q_bytes;  // X slab | Q hi | Q lo (contiguous: B = 2 Kp rows)
    const uint32_t lbase = base + (uint32_t)a.XR * xbytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (size_t)a.XR * xbytes + (size_t)kWR * a.a_bytes);
    uint64_t* xfull = bars;
    uint64_t* xempty = bars + a.XR;
    uint64_t* lfull = bars + 2 * a.XR;   // [2]
    uint64_t* lempty = lfull + kWR;      // [2]
    uint64_t* tfull = lempty + kWR;      // [2] accumulator buffer ready for the epilogue
    uint64_t* tempty = tfull + 2;        // [2] accumulator buffer drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    auto X = [&](int r) { return base + (uint32_t)r * xbytes; };
    auto QH = [&](int r) { return X(r) + a.a_bytes; };
    auto LO = [&](int w) { return lbase + (uint32_t)w * a.a_bytes; };
    const uint32_t tw = 2u * (uint32_t)a.Kp;  // accumulator width per half
    const uint32_t tcols = 4 * tw <= 64 ? 64u : 4 * tw <= 128 ? 128u : 4 * tw <= 256 ? 256u : 512u;

    if (threadIdx.x == 0) {
        for (int r = 0; r < a.XR; ++r) {
            mbar_init(&xfull[r], 1);
            mbar_init(&xempty[r], 1);
        }
        for (int w = 0; w < kWR; ++w) {
            mbar_init(&lfull[w], kSplitWarps);
            mbar_init(&lempty[w], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nt = a.ntiles > blockIdx.x ? (int)((a.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    const int total = nt * a.nchunk;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = policy_l2(1), pol_q = policy_l2(2);
            griddep_wait();  // Q (and, in the chain, X's producer) come from the previous grids
            int g = 0;
            for (int j = 0; j < nt; ++j) {
                const int c0 = (int)((blockIdx.x + (int64_t)j * gridDim.x) * 256);
                for (int ch = 0; ch < a.nchunk; ++ch, ++g) {
                    const int r = g % a.XR;
                    if (g >= a.XR) mbar_wait(&xempty[r], ((g / a.XR) - 1) & 1);
                    mbar_arrive_expect_tx(&xfull[r], a.a_bytes + 2 * a.q_bytes);
                    tma2d(X(r), &xmap, 32 * ch, c0, &xfull[r], pol_x);
                    tma2d(X(r) + a.a_bytes / 2, &xmap, 32 * ch, c0 + 128, &xfull[r], pol_x);
                    tma2d(QH(r), &qhmap, 32 * ch, 0, &xfull[r], pol_q);
                    tma2d(QH(r) + a.q_bytes, &qlmap, 32 * ch, 0, &xfull[r], pol_q);
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc1 = idesc_tf32(128, 2 * a.Kp, 0, 0);
        const uint32_t idesc2 = idesc_tf32(128, a.Kp, 0, 0);
        int g = 0;
        for (int j = 0; j < nt; ++j) {
            const int buf = j & 1;
            if (j >= 2) mbar_wait(&tempty[buf], ((j >> 1) - 1) & 1);
            tc_fence_after();
            for (int ch = 0; ch < a.nchunk; ++ch, ++g) {
                const int r = g % a.XR, w = g % kWR;
                mbar_wait(&xfull[r], (g / a.XR) & 1);
                mbar_wait(&lfull[w], (g / kWR) & 1);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {  // 4 k-steps of 8 in the 128-byte rows
                        const uint64_t qd = sdesc(QH(r) + ks * 32u, 16, 1024, kSw128);  // [Q_hi; Q_lo] rows
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t ao = (uint32_t)h * (a.a_bytes / 2) + ks * 32u;
                            const uint64_t xh = sdesc(X(r) + ao, 16, 1024, kSw128);
                            const uint64_t xl = sdesc(LO(w) + ao, 16, 1024, kSw128);
                            const uint32_t d = tmem + (uint32_t)(buf * 2 + h) * tw;
                            const uint32_t acc = (ch > 0 || ks > 0) ? 1u : 0u;
                            mma_tf32(d, xh, qd, idesc1, acc);  // X_hi [Q_hi | Q_lo]
                            mma_tf32(d, xl, qd, idesc2, 1u);   // X_lo Q_hi (first Kp columns)
                        }
                    }
                    mma_commit(&xempty[r]);
                    mma_commit(&lempty[w]);
                }
                __syncwarp();
            }
            if (lane == 0) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp >= kSplitW0 && warp < kSplitW0 + kSplitWarps) {
        const int tid = threadIdx.x - kSplitW0 * 32;
        for (int g = 0; g < total; ++g) {
            const int r = g % a.XR, w = g % kWR;
            if (g >= kWR) mbar_wait(&lempty[w], ((g / kWR) - 1) & 1);
            mbar_wait(&xfull[r], (g / a.XR) & 1);
            split_lo(X(r), LO(w), a.a_bytes, tid, kSplitWarps * 32);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&lfull[w]);
        }
    } else {
        // ================= epilogue: TMEM lane = fibre of the tile; output k = column k + column Kp + k
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
                    float v[8], u[8];
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 2 + h) * tw + (uint32_t)n0;
                    tmem_ld8(ta, v);
                    tmem_ld8(ta + (uint32_t)a.Kp, u);
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) v[jj] += u[jj];
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

// ================================================================== K1 for modes n >= 1 (left > 1)
// Y_n (dim x K) += sum_r P_r Omega_r, P_r = the (dim x left) slab r of P^(n) (left contiguous: the
// K-major A operand of k_tc_ttm_f32, landed by the same 2-D TMA over [dim right][left] in
// 128B-swizzled 32-column boxes), Omega_r = its rows l + left r of the reference test matrix
// (sketch.hpp:32-38, 80-83), regenerated on chip by generator warps as the K-major B operand
// [Omega_hi | Omega_lo] in the TMA 128B-swizzle layout. CTA = (256-row d tile, a contiguous range of
// the (r, 32-column chunk) items); D = [A Omega_hi | A Omega_lo] + A_lo Omega_hi in TMEM for the
// whole range (a few hundred accumulation steps: ~1e-6 relative), drained once into the CTA's fp64
// partial (partial[range] covers every d tile of that range: the fixed-order split-K reduce sums
// ranges). Warps: 0 TMA, 1 MMA (+ TMEM), 2-5 splitters, 6-9 generators, then the drain.
constexpr int kSnThreads = 10 * 32;
constexpr int kSnGenW0 = 6, kSnGenWarps = 4;

struct TcSnArgs {
    int left, dim, K, Kp, nchunk, XR, BR, ntd, TR;  // ntd: d tiles of TR rows (256: two M = 128 halves; 64: one M = 64)
    int64_t right, nitems, nparts;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    double* partial;  // nparts x dim x K
    uint32_t a_bytes, b_bytes;
};

__global__ void __launch_bounds__(kSnThreads, 1)
    k_tc_sketch_n_f32(const __grid_constant__ CUtensorMap pmap, TcSnArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t lbase = base + (uint32_t)a.XR * a.a_bytes;
    const uint32_t bbase = lbase + (uint32_t)kWR * a.a_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (size_t)(a.XR + kWR) * a.a_bytes + (size_t)a.BR * a.b_bytes);
    uint64_t* xfull = bars;
    uint64_t* xempty = bars + a.XR;
    uint64_t* lfull = xempty + a.XR;  // [kWR]
    uint64_t* lempty = lfull + kWR;   // [kWR]
    uint64_t* bfull = lempty + kWR;   // [BR]
    uint64_t* bempty = bfull + a.BR;  // [BR]
    uint64_t* dfull = bempty + a.BR;  // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dfull + 1);
    auto X = [&](int r) { return base + (uint32_t)r * a.a_bytes; };
    auto LO = [&](int w) { return lbase + (uint32_t)w * a.a_bytes; };
    auto B = [&](int b) { return bbase + (uint32_t)b * a.b_bytes; };
    const uint32_t tw = 2u * (uint32_t)a.Kp;  // accumulator width per M tile
    const int nh = a.TR == 256 ? 2 : 1;        // M tiles per d tile
    const uint32_t tcols = nh * tw <= 32 ? 32u : nh * tw <= 64 ? 64u : nh * tw <= 128 ? 128u : 256u;
    const int dt = (int)(blockIdx.x % a.ntd), part = (int)(blockIdx.x / a.ntd);
    const int64_t it0 = a.nitems * part / a.nparts, it1 = a.nitems * (part + 1) / a.nparts;
    const int total = (int)(it1 - it0);
    const int d0 = a.TR * dt;

    // B ring: rows K..Kp-1 (and Kp+K..2Kp-1) stay zero
    for (uint32_t o = threadIdx.x * 16u; o < (uint32_t)a.BR * a.b_bytes; o += kSnThreads * 16u)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(bbase + o), "r"(0u));
    if (threadIdx.x == 0) {
        for (int r = 0; r < a.XR; ++r) {
            mbar_init(&xfull[r], 1);
            mbar_init(&xempty[r], 1);
        }
        for (int w = 0; w < kWR; ++w) {
            mbar_init(&lfull[w], kSplitWarps);
            mbar_init(&lempty[w], 1);
        }
        for (int b = 0; b < a.BR; ++b) {
            mbar_init(&bfull[b], kSnGenWarps);
            mbar_init(&bempty[b], 1);
        }
        mbar_init(dfull, 1);
        fence_mbar_init();
    }
    fence_async_smem();
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_l2(0);
            griddep_wait();
            for (int g = 0; g < total; ++g) {
                const int64_t it = it0 + g;
                const int64_t r = it / a.nchunk;
                const int ch = (int)(it - r * a.nchunk);
                const int row = (int)(d0 + (int64_t)a.dim * r);
                const int x = g % a.XR;
                if (g >= a.XR) mbar_wait(&xempty[x], ((g / a.XR) - 1) & 1);
                mbar_arrive_expect_tx(&xfull[x], a.a_bytes);
                tma2d(X(x), &pmap, 32 * ch, row, &xfull[x], pol);
                if (nh == 2) tma2d(X(x) + a.a_bytes / 2, &pmap, 32 * ch, row + 128, &xfull[x], pol);
            }
        }
    } else if (warp == 1) {
        const int Mm = nh == 2 ? 128 : 64;
        const uint32_t idesc1 = idesc_tf32(Mm, 2 * a.Kp, 0, 0);
        const uint32_t idesc2 = idesc_tf32(Mm, a.Kp, 0, 0);
        for (int g = 0; g < total; ++g) {
            const int x = g % a.XR, w = g % kWR, b = g % a.BR;
            mbar_wait(&xfull[x], (g / a.XR) & 1);
            mbar_wait(&lfull[w], (g / kWR) & 1);
            mbar_wait(&bfull[b], (g / a.BR) & 1);
            tc_fence_after();
            if (lane == 0) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {  // 4 k-steps of 8 in the 128-byte rows
                    const uint64_t bd = sdesc(B(b) + ks * 32u, 16, 1024, kSw128);  // [Omega_hi; Omega_lo] rows
                    for (int h = 0; h < nh; ++h) {
                        const uint32_t ao = (uint32_t)h * (a.a_bytes / 2) + ks * 32u;
                        const uint64_t xh = sdesc(X(x) + ao, 16, 1024, kSw128);
                        const uint64_t xl = sdesc(LO(w) + ao, 16, 1024, kSw128);
                        const uint32_t d = tmem + (uint32_t)h * tw;
                        const uint32_t acc = (g > 0 || ks > 0) ? 1u : 0u;
                        mma_tf32(d, xh, bd, idesc1, acc);  // P_hi [Omega_hi | Omega_lo]
                        mma_tf32(d, xl, bd, idesc2, 1u);   // P_lo Omega_hi (first Kp columns)
                    }
                }
                mma_commit(&xempty[x]);
                mma_commit(&lempty[w]);
                mma_commit(&bempty[b]);
            }
            __syncwarp();
        }
        if (lane == 0) mma_commit(dfull);
        __syncwarp();
    } else if (warp >= kSplitW0 && warp < kSplitW0 + kSplitWarps) {
        const int tid = threadIdx.x - kSplitW0 * 32;
        for (int g = 0; g < total; ++g) {
            const int x = g % a.XR, w = g % kWR;
            if (g >= kWR) mbar_wait(&lempty[w], ((g / kWR) - 1) & 1);
            mbar_wait(&xfull[x], (g / a.XR) & 1);
            split_lo(X(x), LO(w), a.a_bytes, tid, kSplitWarps * 32);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&lfull[w]);
        }
    }
    if (warp >= kSnGenW0 && warp < kSnGenW0 + kSnGenWarps) {
        // ---- generators: item (r, ch) -> rows c = 32 ch + l + left r (l < 32) of Omega for every k:
        // draw D + col_off + c + rows_glob k (sketch.hpp:32-38), pairs (2p, 2p + 1) of the stream;
        // element (n, l) at row n (hi: k, lo: Kp + k) in the 128B-swizzle layout
        const int tid = threadIdx.x - kSnGenW0 * 32;
        const int np = 17;  // pairs covering 32 consecutive draws at either parity
        for (int g = 0; g < total; ++g) {
            const int64_t it = it0 + g;
            const int64_t r = it / a.nchunk;
            const int ch = (int)(it - r * a.nchunk);
            const int b = g % a.BR;
            if (g >= a.BR) mbar_wait(&bempty[b], ((g / a.BR) - 1) & 1);
            const uint32_t Bb = B(b);
            const uint64_t c0 = (uint64_t)(a.col_off + 32 * ch + (int64_t)a.left * r);
            for (int e = tid; e < a.K * np; e += kSnGenWarps * 32) {
                const int k = e / np, pi = e - k * np;
                const uint64_t s0 = a.D + c0 + (uint64_t)a.rows_glob * (uint64_t)k;
                const uint64_t p = (s0 >> 1) + (uint64_t)pi;
                const int l0 = (int)(2 * p - s0);  // -1 .. 32
                if (l0 >= 32) continue;
                float z[2];
                gauss_pair_f32_fast(a.seed + (2ull * p + 1ull) * 0x9E3779B97F4A7C15ull, z[0], z[1]);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int l = l0 + u;
                    if (l < 0 || l >= 32) continue;
                    const float hi = tf32_trunc(z[u]), lo = z[u] - hi;
                    const uint32_t chunk = (uint32_t)(l >> 2), wb = (uint32_t)(l & 3) * 4u;
                    const int nh = k, nl = a.Kp + k;
                    sts32(Bb + (uint32_t)(nh >> 3) * 1024u + (uint32_t)(nh & 7) * 128u + ((chunk ^ (uint32_t)(nh & 7)) << 4) + wb, hi);
                    sts32(Bb + (uint32_t)(nl >> 3) * 1024u + (uint32_t)(nl & 7) * 128u + ((chunk ^ (uint32_t)(nl & 7)) << 4) + wb, lo);
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bfull[b]);
        }
        // ---- drain: TMEM lane = row of the d tile (M = 128: rows 32 q + lane of each half; M = 64:
        // rows 16 q + lane, lanes 0-15); Y(d, k) = column k + column Kp + k, fp64
        mbar_wait(dfull, 0);
        tc_fence_after();
        const int q = warp & 3;
        double* out = a.partial + (int64_t)part * a.dim * a.K;
        const int rq = nh == 2 ? 32 : 16;
#pragma unroll 1
        for (int h = 0; h < nh; ++h) {
            const int d = lane < rq ? d0 + h * 128 + q * rq + lane : a.dim;
            for (int n0 = 0; n0 < a.Kp; n0 += 8) {
                float v[8], u[8];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)h * tw + (uint32_t)n0;
                tmem_ld8(ta, v);
                tmem_ld8(ta + (uint32_t)a.Kp, u);
                if (d < a.dim)
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if (n0 + jj < a.K) out[d + (int64_t)a.dim * (n0 + jj)] = (double)v[jj] + (double)u[jj];
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, tcols);
    }
}

// ================================================================== K2 for modes n >= 1 (left > 1)
// P^(n+1)(l, k, r) = sum_d P(l, d, r) Q(d, k) (tensor.hpp:193-207 with m = Q^T): per output tile
// (M = 128 rows: 128 consecutive l of one slab r, or 128 / left whole slabs when left is 32 or 64,
// so the Q chunks stream once per 128 rows) D[M x 2 Kp] = P_r^T [Q_hi | Q_lo] + P_r,lo^T Q_hi over
// 32-d chunks. A = P_r^T is MN-major (l contiguous): 32-l blocks of 32 d rows by 2-D TMA over
// [dim right][left] in the 128B-swizzle-of-32-byte-atoms layout (as the mode-0 sketch's X); B = the
// K-major [Q_hi; Q_lo] chunk (as k_tc_ttm_f32). Double-buffered TMEM accumulators: the epilogue
// (TMEM lane = l, K values at stride left) overlaps the next tile's MMAs.
// Warps: 0 TMA, 1 MMA (+ TMEM), 2-5 splitters, 6-9 epilogue.
struct TcTnArgs {
    int left, dim, K, Kp, M, nchunk, XR, nlt, S;  // nlt: l tiles per slab; S: slabs per tile (left < 128)
    int64_t right, ntiles;
    float* out;
    uint32_t a_bytes, q_bytes;
};

__global__ void __launch_bounds__(kTtThreads, 1)
    k_tc_ttm_n_f32(const __grid_constant__ CUtensorMap pmap, const __grid_constant__ CUtensorMap qhmap,
                   const __grid_constant__ CUtensorMap qlmap, TcTnArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t xbytes = a.a_bytes + 2 * a.q_bytes;  // P^T blocks | Q hi | Q lo
    const uint32_t lbase = base + (uint32_t)a.XR * xbytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (size_t)a.XR * xbytes + (size_t)kWR * a.a_bytes);
    uint64_t* xfull = bars;
    uint64_t* xempty = bars + a.XR;
    uint64_t* lfull = bars + 2 * a.XR;
    uint64_t* lempty = lfull + kWR;
    uint64_t* tfull = lempty + kWR;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    auto X = [&](int r) { return base + (uint32_t)r * xbytes; };
    auto QH = [&](int r) { return X(r) + a.a_bytes; };
    auto LO = [&](int w) { return lbase + (uint32_t)w * a.a_bytes; };
    const uint32_t tw = 2u * (uint32_t)a.Kp;
    const uint32_t tcols = 2 * tw <= 64 ? 64u : 2 * tw <= 128 ? 128u : 2 * tw <= 256 ? 256u : 512u;
    const uint32_t lbo_a = 32u * 128u;  // one 32-l block: 32 d rows of 128 B
    const int nblk = a.M / 32;

    if (threadIdx.x == 0) {
        for (int r = 0; r < a.XR; ++r) {
            mbar_init(&xfull[r], 1);
            mbar_init(&xempty[r], 1);
        }
        for (int w = 0; w < kWR; ++w) {
            mbar_init(&lfull[w], kSplitWarps);
            mbar_init(&lempty[w], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nt = a.ntiles > blockIdx.x ? (int)((a.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    const int total = nt * a.nchunk;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = policy_l2(0), pol_q = policy_l2(2);
            griddep_wait();
            int g = 0;
            for (int j = 0; j < nt; ++j) {
                const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
                const int64_t rt = tile / a.nlt;               // first slab of the tile: rt S
                const int l0 = (int)(tile - rt * a.nlt) * a.M;  // left >= 128: l offset of the tile
                const int bps = a.left < 128 ? a.left / 32 : nblk;  // 32-l blocks per slab in the tile
                for (int ch = 0; ch < a.nchunk; ++ch, ++g) {
                    const int x = g % a.XR;
                    if (g >= a.XR) mbar_wait(&xempty[x], ((g / a.XR) - 1) & 1);
                    mbar_arrive_expect_tx(&xfull[x], (uint32_t)nblk * lbo_a + 2 * a.q_bytes);
                    for (int b = 0; b < nblk; ++b) {
                        // block b: 32 l of slab rt S + b / bps (rows past the tensor are zero-filled)
                        const int64_t r = rt * a.S + b / bps;
                        const int row = (int)((int64_t)a.dim * r + 32 * ch);
                        tma2d(X(x) + (uint32_t)b * lbo_a, &pmap, l0 + 32 * (b % bps), row, &xfull[x], pol_x);
                    }
                    tma2d(QH(x), &qhmap, 32 * ch, 0, &xfull[x], pol_q);
                    tma2d(QH(x) + a.q_bytes, &qlmap, 32 * ch, 0, &xfull[x], pol_q);
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc1 = idesc_tf32(a.M, 2 * a.Kp, /*a MN-major*/ 1, 0);
        const uint32_t idesc2 = idesc_tf32(a.M, a.Kp, 1, 0);
        int g = 0;
        for (int j = 0; j < nt; ++j) {
            const int buf = j & 1;
            if (j >= 2) mbar_wait(&tempty[buf], ((j >> 1) - 1) & 1);
            tc_fence_after();
            for (int ch = 0; ch < a.nchunk; ++ch, ++g) {
                const int x = g % a.XR, w = g % kWR;
                mbar_wait(&xfull[x], (g / a.XR) & 1);
                mbar_wait(&lfull[w], (g / kWR) & 1);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {  // 4 k-steps of 8 d
                        const uint64_t qd = sdesc(QH(x) + ks * 32u, 16, 1024, kSw128);
                        const uint64_t ah = sdesc(X(x) + ks * 1024u, lbo_a, 512, kSw128b32);
                        const uint64_t al = sdesc(LO(w) + ks * 1024u, lbo_a, 512, kSw128b32);
                        const uint32_t d = tmem + (uint32_t)buf * tw;
                        const uint32_t acc = (ch > 0 || ks > 0) ? 1u : 0u;
                        mma_tf32(d, ah, qd, idesc1, acc);  // P_hi^T [Q_hi | Q_lo]
                        mma_tf32(d, al, qd, idesc2, 1u);   // P_lo^T Q_hi (first Kp columns)
                    }
                    mma_commit(&xempty[x]);
                    mma_commit(&lempty[w]);
                }
                __syncwarp();
            }
            if (lane == 0) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp >= kSplitW0 && warp < kSplitW0 + kSplitWarps) {
        const int tid = threadIdx.x - kSplitW0 * 32;
        const uint32_t real = (uint32_t)nblk * lbo_a;
        for (int g = 0; g < total; ++g) {
            const int x = g % a.XR, w = g % kWR;
            if (g >= kWR) mbar_wait(&lempty[w], ((g / kWR) - 1) & 1);
            mbar_wait(&xfull[x], (g / a.XR) & 1);
            split_lo(X(x), LO(w), real, tid, kSplitWarps * 32);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&lfull[w]);
        }
    } else {
        // ================= epilogue: TMEM lane = l of the tile; out(l, k, r) = column k + column Kp + k
        const int q = warp & 3;
        for (int j = 0; j < nt; ++j) {
            const int buf = j & 1;
            mbar_wait(&tfull[buf], (j >> 1) & 1);
            tc_fence_after();
            const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
            const int64_t rt = tile / a.nlt;
            // M = 128: lane quarter q holds rows 32 q + lane; M = 64: rows 16 q + lane (lanes 0-15)
            const int rq = a.M == 128 ? 32 : 16;
            const int m = q * rq + lane;  // row of the tile: (slab rt S + m / left, l = m % left) when left < 128
            const int64_t r = a.left < 128 ? rt * a.S + m / a.left : rt;
            const int l = a.left < 128 ? m % a.left : (int)(tile - rt * a.nlt) * a.M + m;
            if (r < a.right) {
                float* o = a.out + l + (int64_t)a.left * a.K * r;
                for (int n0 = 0; n0 < a.Kp; n0 += 8) {
                    float v[8], u[8];
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)buf * tw + (uint32_t)n0;
                    tmem_ld8(ta, v);
                    tmem_ld8(ta + (uint32_t)a.Kp, u);
                    if (lane < rq && l < a.left)
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            if (n0 + jj < a.K) o[(int64_t)a.left * (n0 + jj)] = v[jj] + u[jj];
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
// zero-padded: the K2 B operand, split for 3xTF32 (hi = trunc_tf32 of the fp32 rounding)
__global__ void k_qt_prep(const double* __restrict__ q, int64_t ldq, int I0, int K, int Ip, int Kp, float* hi,
                          float* lo) {
    griddep_wait();
    const int n = Kp * Ip;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int k = e / Ip, i = e - k * Ip;
        const double v = (k < K && i < I0) ? q[i + ldq * k] : 0.0;
        const float h = tf32_trunc((float)v);
        hi[e] = h;
        lo[e] = (float)(v - (double)h);
    }
    griddep_launch_dependents();
}

struct TcTtPlan {
    int Kp, nchunk, XR, Ip;
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
    const size_t fixed = 1024 + 8 * (2 * 8 + 2 * kWR + 4) + 64;
    const size_t lo = (size_t)kWR * p.a_bytes;
    p.XR = (int)std::min<size_t>(8, (227 * 1024 - fixed - lo) / (p.a_bytes + 2 * (size_t)p.q_bytes));
    p.smem = (size_t)p.XR * (p.a_bytes + 2 * (size_t)p.q_bytes) + lo + fixed;
    return p.XR >= 2;
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
// Dispatch: the tensor-core sketch where the FFMA kernel is compute-bound (K >= 32, e.g. C4's
// K_0 = 64 at 32 flop/B: 349 against 856 us); at small K the FFMA kernel with its cheaper
// register-level test-matrix reuse stays ahead (C3 1172 vs 1384 us, C5 1088 vs 2550 us, measured).
// TRG_TC_FORCE=1 takes the tensor-core kernels for every supported shape (tests), TRG_NO_TCGEN05=1 none.
bool tc_forced() { return getenv("TRG_TC_FORCE") != nullptr; }

bool tc_sketch_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols) {
    TcSkPlan p;
    if (getenv("TRG_NO_TCGEN05") || (K < 32 && !tc_forced())) return false;
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
    a.M = p.M;
    a.Mt = p.Mt;
    a.nblk = p.nblk;
    a.kb = p.kb;
    a.WR = p.WR;
    a.XR = p.XR;
    a.seg = p.seg;
    a.nset = p.nset;
    a.ncat = p.ncat;
    a.RS = p.RS;
    a.BR = p.BR;
    a.L = sp.right;
    a.ntiles = (sp.right + p.kb - 1) / p.kb;
    a.seed = sp.seed;
    a.D = sp.D;
    a.rows_glob = sp.rows_glob;
    a.col_off = sp.col_off;
    a.partial = partial;
    a.a_bytes = p.a_bytes;
    a.b_bytes = p.b_bytes;
    CUtensorMap map;
    encode2d(&map, x, (uint64_t)sp.dim, (uint64_t)sp.right, (uint64_t)sp.dim * 4, 32, (uint32_t)p.kb,
             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const int ncg = tc_sketch_f32_grid(sp.dim, sp.K, sp.right, num_sms);
    const int grid = ncg * p.RS;
    static const char* prof_env = getenv("TRG_TC_PROF");
    if (prof_env) {
        cudaMalloc(&a.prof, 8 * 256 * sizeof(long long));
        cudaMemset(a.prof, 0, 8 * 256 * sizeof(long long));
    }
    allow_smem(k_tc_sketch_f32, p.smem);
    k_tc_sketch_f32<<<grid, kSkThreads, p.smem, s>>>(map, a);
    if (prof_env) {  // development: per-stage timeline of CTA 0 (cycles), averaged over stages 16..255
        long long h[8 * 256];
        cudaStreamSynchronize(s);
        cudaMemcpy(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost);
        cudaFree(a.prof);
        double acc[8] = {0};
        int n = 0;
        for (int j = 16; j < 255; ++j) {
            if (!h[3 * 256 + j + 1]) break;
            acc[0] += h[0 * 256 + j + 1] - h[0 * 256 + j];  // producer period
            acc[1] += h[1 * 256 + j] - h[0 * 256 + j];      // producer wait for xempty
            acc[2] += h[2 * 256 + j] - h[1 * 256 + j];      // TMA issue -> MMA sees xfull
            acc[3] += h[3 * 256 + j] - h[2 * 256 + j];      // MMA waits split / omega after xfull
            acc[4] += h[5 * 256 + j] - h[4 * 256 + j];      // split duration
            acc[5] += h[7 * 256 + j] - h[6 * 256 + j];      // generation duration
            acc[6] += h[3 * 256 + j + 1] - h[3 * 256 + j];  // MMA period
            acc[7] += h[4 * 256 + j] - h[2 * 256 + j];      // splitter start - MMA xfull seen
            ++n;
        }
        for (int j = 100; j < 112; ++j) {
            fprintf(stderr, "tc_stage %d:", j);
            for (int q = 0; q < 8; ++q) fprintf(stderr, " %lld", h[q * 256 + j] - h[0 * 256 + 100]);
            fprintf(stderr, "\n");
        }
        fprintf(stderr, "tc_sketch prof (cycles/stage, n=%d): prod period %.0f wait_xempty %.0f tma->xfull %.0f "
                        "mma_wait_work %.0f split %.0f gen %.0f mma period %.0f split_start-xfull %.0f\n",
                n, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n, acc[5] / n, acc[6] / n, acc[7] / n);
    }
    if (y) launch_reduce_partials(partial, ncg, sp.dim * sp.K, y, s);
    return ncg;
}

// number of column groups = number of per-CTA-group partials of Y
int tc_sketch_f32_grid(int64_t dim, int K, int64_t ncols, int num_sms) {
    TcSkPlan p;
    plan_tc_sketch(dim, K, p);
    return (int)std::max<int64_t>(1, std::min<int64_t>((ncols + p.kb - 1) / p.kb, num_sms / p.RS));
}

// the tensor-core shrink from K >= 16 on fibres of >= 128 rows (C3 789 vs 1308 us, C4 249 vs 897
// us); C5's 60-row fibres split into two 32-row slabs that over-fetch (1089 vs 934 us)
bool tc_ttm_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols) {
    TcTtPlan p;
    if (getenv("TRG_NO_TCGEN05") || ((K < 16 || dim < 128) && !tc_forced())) return false;
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
    a.XR = p.XR;
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
        pdl_launch(k_tc_ttm_f32<true>, dim3(grid), dim3(kTtThreads), p.smem, s, xm, qhm, qlm, a);
    } else {
        allow_smem(k_tc_ttm_f32<false>, p.smem);
        pdl_launch(k_tc_ttm_f32<false>, dim3(grid), dim3(kTtThreads), p.smem, s, xm, qhm, qlm, a);
    }
}


// ---- K1 for modes n >= 1 on tcgen05 (k_tc_sketch_n_f32)
namespace {
struct TcSnPlan {
    int Kp, nchunk, XR, BR, ntd, TR;
    int64_t nparts;
    uint32_t a_bytes, b_bytes;
    size_t smem;
};
bool plan_tc_sketch_n(int64_t left, int64_t dim, int K, int64_t right, int num_sms, TcSnPlan& p) {
    if (K < 1 || K > 64 || left < 32 || (left % 32) != 0 || dim < 1 || right < 1) return false;
    if (dim * right + 256 >= (int64_t(1) << 31)) return false;  // TMA row coordinates
    p.Kp = (K + 15) & ~15;
    p.nchunk = (int)(left / 32);
    p.TR = dim <= 64 ? 64 : 256;  // short modes (C5: 60) take one M = 64 tile: no rows of other slabs
    p.ntd = (int)((dim + p.TR - 1) / p.TR);
    p.a_bytes = (uint32_t)p.TR * 128u;
    p.b_bytes = 2u * (uint32_t)p.Kp * 128u;
    const int64_t nitems = right * p.nchunk;
    p.nparts = std::max<int64_t>(1, std::min<int64_t>(nitems, num_sms / p.ntd));
    const size_t fixed = 1024 + 8 * (2 * 8 + 2 * kWR + 2 * 8 + 2) + 64;
    p.BR = 3;
    const size_t rest = (size_t)kWR * p.a_bytes + (size_t)p.BR * p.b_bytes + fixed;
    p.XR = (int)std::min<size_t>(6, (227 * 1024 - rest) / p.a_bytes);
    p.smem = (size_t)p.XR * p.a_bytes + rest;
    return p.XR >= 2;
}
}  // namespace

bool tc_sketch_n_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t right) {
    TcSnPlan p;
    if (getenv("TRG_NO_TCGEN05") || (K < 32 && !tc_forced())) return false;
    return dtype == F32 && encode_fn() && plan_tc_sketch_n(left, dim, K, right, 148, p);
}

int tc_sketch_n_f32_parts(int64_t left, int64_t dim, int K, int64_t right, int num_sms) {
    TcSnPlan p;
    plan_tc_sketch_n(left, dim, K, right, num_sms, p);
    return (int)p.nparts;
}

int launch_tc_sketch_n_f32(const SketchPlan& sp, const void* x, double* partial, double* y, int num_sms,
                           cudaStream_t s) {
    TcSnPlan p;
    if (!plan_tc_sketch_n(sp.left, sp.dim, sp.K, sp.right, num_sms, p))
        throw std::runtime_error("tc sketch (mode >= 1): unsupported shape");
    TcSnArgs a{};
    a.left = (int)sp.left;
    a.dim = (int)sp.dim;
    a.K = sp.K;
    a.Kp = p.Kp;
    a.nchunk = p.nchunk;
    a.XR = p.XR;
    a.BR = p.BR;
    a.ntd = p.ntd;
    a.TR = p.TR;
    a.right = sp.right;
    a.nitems = sp.right * p.nchunk;
    a.nparts = p.nparts;
    a.seed = sp.seed;
    a.D = sp.D;
    a.rows_glob = sp.rows_glob;
    a.col_off = sp.col_off;
    a.partial = partial;
    a.a_bytes = p.a_bytes;
    a.b_bytes = p.b_bytes;
    CUtensorMap pm;
    encode2d(&pm, x, (uint64_t)sp.left, (uint64_t)(sp.dim * sp.right), (uint64_t)sp.left * 4, 32,
             (uint32_t)std::min(p.TR, 128), CU_TENSOR_MAP_SWIZZLE_128B);
    const int grid = (int)(p.ntd * p.nparts);
    allow_smem(k_tc_sketch_n_f32, p.smem);
    pdl_launch(k_tc_sketch_n_f32, dim3(grid), dim3(kSnThreads), p.smem, s, pm, a);
    if (y) launch_reduce_partials(partial, (int)p.nparts, sp.dim * sp.K, y, s);
    return (int)p.nparts;
}


// ---- K2 for modes n >= 1 on tcgen05 (k_tc_ttm_n_f32)
namespace {
struct TcTnPlan {
    int Kp, nchunk, XR, Ip, M, nlt, S;
    uint32_t a_bytes, q_bytes;
    size_t smem;
};
bool plan_tc_ttm_n(int64_t left, int64_t dim, int64_t K, int64_t right, TcTnPlan& p) {
    if (K < 1 || K > 64 || left < 32 || (left % 32) != 0 || dim < 1 || dim > 4096 || right < 1) return false;
    if (dim * right + 64 >= (int64_t(1) << 31) || left >= (int64_t(1) << 31)) return false;
    p.Kp = (int)((K + 15) & ~15);
    // M = 128 rows per tile: 128 l of one slab, or 128 / left whole slabs when left is 32 or 64
    if (left < 128 ? (128 % left) != 0 : (left % 128) != 0) return false;
    p.M = 128;
    p.S = left < 128 ? (int)(128 / left) : 1;
    p.nlt = left < 128 ? 1 : (int)(left / 128);
    p.nchunk = (int)((dim + 31) / 32);
    p.Ip = p.nchunk * 32;
    p.a_bytes = (uint32_t)(p.M / 32) * 32u * 128u;
    p.q_bytes = (uint32_t)p.Kp * 128u;
    const size_t fixed = 1024 + 8 * (2 * 8 + 2 * kWR + 4) + 64;
    const size_t lo = (size_t)kWR * p.a_bytes;
    p.XR = (int)std::min<size_t>(8, (227 * 1024 - fixed - lo) / (p.a_bytes + 2 * (size_t)p.q_bytes));
    p.smem = (size_t)p.XR * (p.a_bytes + 2 * (size_t)p.q_bytes) + lo + fixed;
    return p.XR >= 2;
}
}  // namespace

bool tc_ttm_n_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right) {
    TcTnPlan p;
    if (getenv("TRG_NO_TCGEN05") || (K < 32 && !tc_forced())) return false;
    return dtype == F32 && encode_fn() && plan_tc_ttm_n(left, dim, K, right, p);
}

size_t tc_ttm_n_f32_scratch(int64_t dim, int64_t K) {
    const int Kp = (int)((K + 15) & ~15), Ip = (int)((dim + 31) / 32 * 32);
    return sizeof(float) * 2 * (size_t)Kp * Ip;
}

void launch_tc_ttm_n_f32(const TTMPlan& tp, const void* in, void* out, const double* q, int64_t ldq, float* scratch,
                         int num_sms, cudaStream_t s) {
    TcTnPlan p;
    if (!plan_tc_ttm_n(tp.left, tp.dim, tp.odim, tp.right, p)) throw std::runtime_error("tc shrink (mode >= 1): unsupported shape");
    float* qh = scratch;
    float* ql = scratch + (size_t)p.Kp * p.Ip;
    {
        const int n = p.Kp * p.Ip;
        pdl_launch(k_qt_prep, dim3(std::min(64, (n + 255) / 256)), dim3(256), 0, s, q, ldq, (int)tp.dim,
                   (int)tp.odim, p.Ip, p.Kp, qh, ql);
    }
    TcTnArgs a{};
    a.left = (int)tp.left;
    a.dim = (int)tp.dim;
    a.K = (int)tp.odim;
    a.Kp = p.Kp;
    a.M = p.M;
    a.nchunk = p.nchunk;
    a.XR = p.XR;
    a.nlt = p.nlt;
    a.S = p.S;
    a.right = tp.right;
    a.ntiles = (tp.right + p.S - 1) / p.S * p.nlt;
    a.out = reinterpret_cast<float*>(out);
    a.a_bytes = p.a_bytes;
    a.q_bytes = p.q_bytes;
    CUtensorMap pm, qhm, qlm;
    encode2d(&pm, in, (uint64_t)tp.left, (uint64_t)(tp.dim * tp.right), (uint64_t)tp.left * 4, 32, 32,
             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    encode2d(&qhm, qh, (uint64_t)p.Ip, (uint64_t)p.Kp, (uint64_t)p.Ip * 4, 32, (uint32_t)p.Kp,
             CU_TENSOR_MAP_SWIZZLE_128B);
    encode2d(&qlm, ql, (uint64_t)p.Ip, (uint64_t)p.Kp, (uint64_t)p.Ip * 4, 32, (uint32_t)p.Kp,
             CU_TENSOR_MAP_SWIZZLE_128B);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    allow_smem(k_tc_ttm_n_f32, p.smem);
    pdl_launch(k_tc_ttm_n_f32, dim3(grid), dim3(kTtThreads), p.smem, s, pm, qhm, qlm, a);
}

}  // namespace trg
