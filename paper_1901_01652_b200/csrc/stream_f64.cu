// SPDX-License-Identifier: Apache-2.0
//
// fp64 streaming kernels for the compulsory full passes over X (mode 0, the
// unfolding X_(0) is the raw buffer viewed as I_0 x L column-major):
//
//   k_sketch_l1_f64  Y_0 = X_(0) Omega_0             (sketch.hpp:80-83)
//   k_ttm_l1_f64     P^(1) = X x_0 Q_0^T            (sketch.hpp:85, tensor.hpp:193-207)
//
// Both are persistent warp-specialised kernels: one producer thread streams
// contiguous tiles of whole mode-0 fibres into a 3-stage shared-memory ring
// with TMA bulk copies (cp.async.bulk + mbarrier complete_tx, L2 evict_first),
// consumer warps run fp64 tensor-core MMAs (mma.m8n8k4.f64 -> DMMA) on them,
// and in the sketch four generator warps regenerate the reference Gaussian
// test matrix for the next tile (SplitMix64 + Box-Muller by stream index)
// straight into MMA-fragment order while the MMAs run. fp64 is kept
// end to end because the reference is fp64 and the parity bound is 1e-10.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "kernels.h"
#include "launch.h"
#include "omega_units.cuh"
#include "pipeline.cuh"

namespace trg {

namespace {

constexpr int kStages = 3;
constexpr int kCons = 4;    // consumer warps (shrink)
#ifndef TRG_SK_CONS
#define TRG_SK_CONS 12
#endif
// consumer warps (sketch): kSkCons / 4 per SM sub-partition issue DMMAs; warp w takes the k-steps
// (w & 3) + 4 i of every tile over row-tile group w >> 2 of kSkGrp
constexpr int kSkCons = TRG_SK_CONS;
constexpr int kSkGrp = kSkCons / 4;
static_assert(kSkCons % 4 == 0 && kSkGrp >= 1 && kSkGrp <= 4, "sketch consumers: 4, 8, 12 or 16 warps");
#ifndef TRG_SK_RNG
#define TRG_SK_RNG 8
#endif
#ifndef TRG_SK_ILP
#define TRG_SK_ILP 1
#endif
constexpr int kRng = TRG_SK_RNG;  // Omega generator warps (sketch): one Box-Muller pair per thread per tile
constexpr int kIlp = TRG_SK_ILP;  // independent pairs per generator thread per iteration
// generator slots per thread per tile on the fast path: a 64 x 16 tile has 512 pairs
constexpr int kIpt = (512 + kRng * 32 - 1) / (kRng * 32);
constexpr int kMaxOB = 8;   // Omega tile buffers (sketch), see sk_plan
constexpr int kMaxStg = 8;  // X stages (sketch)
constexpr int kPad = 8;   // zeroed doubles after each stage (A rows may overrun by < 8)
constexpr size_t kBarBytes = 512;  // room for the mbarriers after the buffers

struct SkArgs {
    const double* x;
    int64_t dim, ncols, ntiles, rows_glob, col_off;
    int K, CT, mtiles;
    int nstg, nob;  // X stages and Omega buffers in shared memory (sk_plan)
    int pad;        // zeroed doubles after each stage: every warp reads MTW row tiles unpredicated
    uint64_t seed, D;
    double* partial;
    const GaussTables* gt;
    int pol;  // L2 policy of the X reads (policy_l2)
    KrOmega kr;  // kr.F set: Khatri-Rao test matrix (left = 1: Omega(c, k) = B(col_off + c, k))
    int kr_smem; // F (S1 x K) staged in shared memory after the barriers (sk_plan headroom)
};

__device__ __forceinline__ int64_t imin64(int64_t x, int64_t y) { return x < y ? x : y; }

#ifdef TRG_SK_PROF  // development: cycle breakdown of CTA 0's generator warp 0 and consumer warp 0
__device__ unsigned long long g_sk_prof[16];
#define SK_T(v) long long v = clock64()
#define SK_ADD(i, d) \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) atomicAdd(&g_sk_prof[i], (unsigned long long)(d))
#else
#define SK_T(v)
#define SK_ADD(i, d)
#endif

__device__ __forceinline__ int omega_idx(int c, int k, int NT) {
    return (((c >> 2) * NT + (k >> 3)) << 5) + (c & 3) + ((k & 7) << 2);
}

// One tile's k-steps t = tg, tg + 4, ... (< CT / 4 <= 16) of a consumer warp over NMT row tiles:
// all fragments of a k-step are loaded first, then its MMAs, so each k-step pays one load latency.
template <int NMT, int MTW, int NT>
__device__ __forceinline__ void sk_consume(double (&acc)[MTW][NT][2], const double* X, const double* O, int tg,
                                           int ksteps, int64_t dim) {
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {
        const int t = tg + 4 * i4;
        if (t >= ksteps) break;
        double bv[NT], av[NMT];
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) bv[jn] = O[(t * NT + jn) << 5];
        const double* xrow = X + 4 * t * dim;
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt) av[mt] = xrow[8 * mt];
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                dmma884(acc[mt][jn][0], acc[mt][jn][1], av[mt], bv[jn]);
            }
    }
}

// KR: Khatri-Rao test matrix (a.kr). A separate instantiation, so the branch does not perturb the
// Gaussian generator's code (sharing one instantiation cost the Gaussian path 17 us on C2).
template <int MTW, int NT, bool KR>
__global__ void __launch_bounds__((kSkCons + kRng + 1) * 32, 1) k_sketch_l1_f64(SkArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SK_T(k0);
    const int CT = a.CT;
    const int64_t dim = a.dim;
    const int nstg = a.nstg, nob = a.nob;
    const int stage_elems = (int)(CT * dim) + a.pad;
    double* stages = reinterpret_cast<double*>(smem_raw);
    const int omega_elems = CT * NT * 8;
    double* omega = stages + nstg * stage_elems;
    GaussTables* tabs = reinterpret_cast<GaussTables*>(omega + nob * omega_elems);
    uint64_t* bars = reinterpret_cast<uint64_t*>(tabs + 1);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + nstg;
    uint64_t* full_o = bars + 2 * nstg;
    uint64_t* empty_o = bars + 2 * nstg + nob;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
    // Generator mode. Pairs per k-column of a tile: CT/2 when every column run starts on an
    // even draw (then nothing is wasted), one more otherwise. The fast path (even starts, one
    // round of the generator threads covers a tile) gives each thread one fixed (column, pair)
    // slot; a tile is then written by nitems threads.
    constexpr bool kr = KR;  // Khatri-Rao entries have no draw-pair parity
    const bool odd = !kr && ((a.rows_glob | (int64_t)a.D | a.col_off) & 1) != 0;
    const int npmax = odd ? CT / 2 + 1 : CT / 2;
    const int nitems = a.K * npmax;
    // fast-path slots: a warp's 32 slots cover 8 columns x 4 row pairs of one 32-row block of the
    // B-fragment layout, so its 16-byte stores of (row 2jj, row 2jj + 1) hit distinct banks
    const int nslots = ((a.K + 7) / 8 * 8) * ((npmax + 3) / 4 * 4);
    const bool fast = !odd && nslots <= kIpt * kRng * 32;

    for (int i = tid; i < nstg * stage_elems; i += blockDim.x) stages[i] = 0.0;
    for (int i = tid; i < nob * omega_elems; i += blockDim.x) omega[i] = 0.0;
    gauss_tables_to_smem(*tabs, a.gt);
    if (tid == 0) {
        for (int s = 0; s < nstg; ++s) {
            mbar_init(&full_x[s], 1);
            mbar_init(&empty_x[s], kSkCons * 32);
        }
        for (int b = 0; b < nob; ++b) {
            mbar_init(&full_o[b], fast ? min(nslots, kRng * 32) : kRng * 32);
            mbar_init(&empty_o[b], kSkCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // everything above is independent of the preceding kernel (PDL): the test-matrix tables were
    // built once, long before
    griddep_wait();
    SK_T(k1);
    if (threadIdx.x == 0) SK_ADD(5, k1 - k0);

    if (warp == kSkCons + kRng) {
        // ---------------- producer: TMA bulk copies of CT whole columns
        if (lane == 0) {
            const uint64_t pol = policy_l2(a.pol);
            for (int j = 0, s = 0, ph = 0; j < nl; ++j) {
                mbar_wait(&empty_x[s], ph ^ 1);
                const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
                const int64_t c0 = t * CT;
                const int64_t ncol = imin64(CT, a.ncols - c0);
                const uint32_t bytes = (uint32_t)(ncol * dim * 8);
                mbar_arrive_expect_tx(&full_x[s], bytes);
                bulk_g2s(stages + s * stage_elems, a.x + c0 * dim, bytes, &full_x[s], pol);
                if (++s == nstg) s = 0, ph ^= 1;
            }
        }
        return;
    }
    if (warp >= kSkCons) {
        // ---------------- generator warps: Omega tile in B-fragment order.
        // With 16 warps one pair per thread covers a 64 x 16 tile in a single round.
        const int rt = tid - kSkCons * 32;
        if (fast) {
            // Thread slot (sub, k, jj) writes rows 2jj, 2jj + 1 of column k of tiles sub, sub + R,
            // ... of every group of G = R kIlp tiles; with more slots than threads a thread owns
            // kIpt slots of every tile instead (R = 1). From one tile of this CTA to the next the
            // pair index advances by gridDim.x * CT / 2, i.e. the SplitMix64 state by
            // gridDim.x * CT * gamma, so no per-tile index arithmetic is left in the loop.
            constexpr int nth = kRng * 32;
            // R <= kMaxOB / kIlp keeps a group of G tiles within the Omega buffers (sk_plan)
            const int R = nslots <= nth ? min(nth / nslots, kMaxOB / kIlp) : 1, G = R * kIlp;
            const int sub = nslots <= nth ? rt / nslots : 0;
            if (sub >= R) return;
            const int KH = (a.K + 7) / 8;
            const uint64_t gam = 0x9E3779B97F4A7C15ull;
            const uint64_t inc = (uint64_t)gridDim.x * (uint64_t)CT * gam;  // one tile of this CTA
            uint64_t st[kIpt];
            int o0[kIpt], c0[kIpt], kk[kIpt];
            bool on[kIpt];
#pragma unroll
            for (int i = 0; i < kIpt; ++i) {
                const int slot = nslots <= nth ? rt - sub * nslots : rt + i * nth;
                const int grp = slot >> 5, l = slot & 31;
                const int kq = 8 * (grp % KH) + (l & 7), jq = 4 * (grp / KH) + (l >> 3);
                on[i] = slot < nslots && kq < a.K && jq < npmax && (i == 0 || nslots > nth);
                const int k = on[i] ? kq : 0;
                const int jj = on[i] ? jq : 0;
                o0[i] = omega_idx(2 * jj, k, NT);  // row 2jj + 1 is the next double (2jj even)
                c0[i] = 2 * jj;
                kk[i] = k;
                const uint64_t p0 = ((a.D + (uint64_t)a.col_off +
                                      ((uint64_t)blockIdx.x + (uint64_t)sub * gridDim.x) * CT +
                                      (uint64_t)a.rows_glob * (uint64_t)k) >> 1) + (uint64_t)jj;
                st[i] = a.seed + (2ull * p0 + 1ull) * gam;
            }
            const int64_t full_tiles = a.ncols / CT;  // tiles t < full_tiles have all CT columns
            if (kr && a.kr_smem && kIlp == 1) {  // (kr is a template constant: compiled out for Gaussian)
                // Khatri-Rao entries F(i1, k) H(q, k), c = i1 + S1 q: F from shared memory, H(q, k)
                // and H(q + 1, k) loaded one tile ahead; i1 and q advance by constants per tile
                double* Fs = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(bars) + kBarBytes);
                const int S1 = (int)a.kr.S1;
                for (int e = rt; e < S1 * a.K; e += nslots <= nth ? R * nslots : nth) Fs[e] = a.kr.F[e];
                const int ngen = nslots <= nth ? R * nslots : nth;  // generator threads past `sub >= R`
                asm volatile("bar.sync 2, %0;" ::"r"(ngen) : "memory");
                const int64_t step_c = (int64_t)R * gridDim.x * CT;  // columns from one tile of a thread to its next
                const int di = (int)(step_c % S1);
                const int64_t dq = step_c / S1;
                int i1[kIpt];
                int64_t qq[kIpt];
                double h0[kIpt], h1[kIpt];
#pragma unroll
                for (int i = 0; i < kIpt; ++i) {
                    const int64_t c = a.col_off + ((int64_t)blockIdx.x + (int64_t)sub * gridDim.x) * CT + c0[i];
                    qq[i] = c / S1;
                    i1[i] = (int)(c - qq[i] * S1);
                    const double* hk = a.kr.H + a.kr.nH * kk[i];
                    h0[i] = qq[i] < a.kr.nH ? __ldg(hk + qq[i]) : 0.0;
                    h1[i] = qq[i] + 1 < a.kr.nH ? __ldg(hk + qq[i] + 1) : 0.0;
                }
                int bx = sub % nob, bp = (sub / nob) & 1;
                for (int j = sub; j < nl; j += R) {
                    mbar_wait(&empty_o[bx], bp ^ 1);
                    double z[kIpt][2];
#pragma unroll
                    for (int i = 0; i < kIpt; ++i) {
                        const double* fk = Fs + S1 * kk[i];
                        z[i][0] = fk[i1[i]] * h0[i];
                        z[i][1] = i1[i] + 1 < S1 ? fk[i1[i] + 1] * h0[i] : fk[0] * h1[i];
                        i1[i] += di;
                        qq[i] += dq;
                        if (i1[i] >= S1) {
                            i1[i] -= S1;
                            qq[i] += 1;
                        }
                        const double* hk = a.kr.H + a.kr.nH * kk[i];  // next tile's H entries, in flight
                        h0[i] = qq[i] < a.kr.nH ? __ldg(hk + qq[i]) : 0.0;
                        h1[i] = qq[i] + 1 < a.kr.nH ? __ldg(hk + qq[i] + 1) : 0.0;
                    }
                    double* O = omega + bx * omega_elems;
                    const int64_t ncol = a.ncols - (blockIdx.x + (int64_t)j * gridDim.x) * CT;
#pragma unroll
                    for (int i = 0; i < kIpt; ++i)
                        if (on[i])
                            *reinterpret_cast<double2*>(O + o0[i]) =
                                make_double2(c0[i] < ncol ? z[i][0] : 0.0, c0[i] + 1 < ncol ? z[i][1] : 0.0);
                    mbar_arrive(&full_o[bx]);
                    bx += R;
                    if (bx >= nob) {
                        bx -= nob;
                        bp ^= 1;
                    }
                }
                return;
            }
            // local tiles jt < jfull are full; buffer index and phase of tile j + u R advance by G
            const int64_t jf = (full_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
            const int jfull = jf > 0 ? (int)jf : 0;
            const uint64_t incR = (uint64_t)R * inc, incG = (uint64_t)G * inc;
            int bix[kIlp], bph[kIlp];
#pragma unroll
            for (int u = 0; u < kIlp; ++u) {
                bix[u] = (sub + u * R) % nob;
                bph[u] = ((sub + u * R) / nob) & 1;
            }
            for (int j = sub; j < nl; j += G) {
                SK_T(t0);
#pragma unroll
                for (int u = 0; u < kIlp; ++u)
                    if (j + u * R < nl) mbar_wait(&empty_o[bix[u]], bph[u] ^ 1);
                SK_T(t1);
                double z[kIlp][kIpt][2];
#pragma unroll
                for (int u = 0; u < kIlp; ++u)
#pragma unroll
                    for (int i = 0; i < kIpt; ++i) {
                        if constexpr (kr) {  // products of the factor entries (L1-resident): no draws
                            const int64_t cl = (blockIdx.x + (int64_t)(j + u * R) * gridDim.x) * CT + c0[i];
                            const uint32_t cg = (uint32_t)(a.col_off + cl);
                            z[u][i][0] = on[i] && cl < a.ncols ? kr_b(a.kr, cg, kk[i]) : 0.0;
                            z[u][i][1] = on[i] && cl + 1 < a.ncols ? kr_b(a.kr, cg + 1u, kk[i]) : 0.0;
                        } else {
                            gauss_pair_state(u == 0 ? st[i] : st[i] + (uint64_t)u * incR, *tabs, z[u][i][0],
                                             z[u][i][1]);
                        }
                    }
#pragma unroll
                for (int i = 0; i < kIpt; ++i) st[i] += incG;
#pragma unroll
                for (int u = 0; u < kIlp; ++u) {
                    const int jt = j + u * R;
                    if (jt >= nl) break;
                    double* O = omega + bix[u] * omega_elems;
                    if (jt < jfull) {
#pragma unroll
                        for (int i = 0; i < kIpt; ++i)
                            if (on[i]) *reinterpret_cast<double2*>(O + o0[i]) = make_double2(z[u][i][0], z[u][i][1]);
                    } else {
                        const int64_t ncol = a.ncols - (blockIdx.x + (int64_t)jt * gridDim.x) * CT;
#pragma unroll
                        for (int i = 0; i < kIpt; ++i)
                            if (on[i])
                                *reinterpret_cast<double2*>(O + o0[i]) =
                                    make_double2(c0[i] < ncol ? z[u][i][0] : 0.0, c0[i] + 1 < ncol ? z[u][i][1] : 0.0);
                    }
                    mbar_arrive(&full_o[bix[u]]);
                    bix[u] += G;
                    if (bix[u] >= nob) {
                        bix[u] -= nob;
                        bph[u] ^= 1;
                    }
                }
                SK_T(t2);
                if (warp == kSkCons) {
                    SK_ADD(0, t1 - t0);
                    SK_ADD(1, t2 - t1);
                }
            }
            return;
        }
        // kIlp tiles per iteration: each thread runs kIlp independent Box-Muller chains (one per
        // tile), which hides the chains' fp64 latency behind each other (the FP64 datapath is
        // shared with the consumers' DMMAs, which stretches every dependent step)
        for (int j = 0; j < nl; j += kIlp) {
            const int ntl = (int)min((int64_t)kIlp, (int64_t)(nl - j));
#pragma unroll
            for (int u = 0; u < kIlp; ++u)
                if (u < ntl) mbar_wait(&empty_o[(j + u) % nob], (((j + u) / nob) & 1) ^ 1);
            for (int it = rt; it < nitems; it += kRng * 32) {
                const int k = it / npmax;
                const int jj = it - k * npmax;
                double z[kIlp][2];
                int64_t cc[kIlp];
                bool live[kIlp];
#pragma unroll
                for (int u = 0; u < kIlp; ++u) {
                    const int64_t c0 = (blockIdx.x + (int64_t)(j + u) * gridDim.x) * CT;
                    const uint64_t s0 = a.D + (uint64_t)(a.col_off + c0) + (uint64_t)a.rows_glob * (uint64_t)k;
                    const uint64_t p = (s0 >> 1) + (uint64_t)jj;
                    live[u] = u < ntl && p <= ((s0 + (uint64_t)CT - 1ull) >> 1);
                    cc[u] = (int64_t)(2ull * p - s0);
                    if constexpr (kr) {  // rows 2 jj, 2 jj + 1 of the tile (no parity offset)
                        cc[u] = 2 * jj;
                        live[u] = u < ntl && 2 * jj < CT;
                        const int64_t cl = c0 + cc[u];
                        z[u][0] = live[u] && cl < a.ncols ? kr_b(a.kr, (uint32_t)(a.col_off + cl), k) : 0.0;
                        z[u][1] = live[u] && cl + 1 < a.ncols ? kr_b(a.kr, (uint32_t)(a.col_off + cl + 1), k) : 0.0;
                    } else {
                        gauss_pair_tab(a.seed, live[u] ? p : 0ull, *tabs, z[u][0], z[u][1]);
                    }
                }
#pragma unroll
                for (int u = 0; u < kIlp; ++u) {
                    if (!live[u]) continue;
                    const int64_t c0 = (blockIdx.x + (int64_t)(j + u) * gridDim.x) * CT;
                    const int64_t ncol = imin64(CT, a.ncols - c0);
                    double* O = omega + ((j + u) % nob) * omega_elems;
                    const int64_t c = cc[u];
                    if (c >= 0 && c < CT) O[omega_idx((int)c, k, NT)] = c < ncol ? z[u][0] : 0.0;
                    if (c + 1 >= 0 && c + 1 < CT) O[omega_idx((int)c + 1, k, NT)] = c + 1 < ncol ? z[u][1] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kIlp; ++u)
                if (u < ntl) mbar_arrive(&full_o[(j + u) % nob]);
        }
        return;
    }
    // ---------------- consumer warps: Y(d, k) += sum_c X(d, c) Omega(c, k)
    // Warp w takes k-steps t = (w & 3), (w & 3) + 4, ... of every tile and row-tile group w >> 2:
    // the mtiles row tiles split as evenly as possible (the first mtiles % kSkGrp groups take one
    // more), MTW = the larger share, so the accumulators stay at 4 MTW doubles.
    const int tg = warp & 3, grp = warp >> 2;
    const int mt_base = a.mtiles / kSkGrp, mt_extra = a.mtiles % kSkGrp;
    const int mt0 = grp * mt_base + min(grp, mt_extra);
    const int my_mt = mt_base + (grp < mt_extra ? 1 : 0);
    double acc[MTW][NT][2];
#pragma unroll
    for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
    const int q = lane >> 2, r = lane & 3;
    const int ksteps = CT / 4;
    for (int j = 0, s = 0, ph = 0; j < nl; ++j) {
        const int b = j % nob;
        SK_T(c0);
        mbar_wait(&full_x[s], ph);
        SK_T(c1);
        mbar_wait(&full_o[b], (j / nob) & 1);
        SK_T(c2);
        const double* X = stages + s * stage_elems + r * dim + q + 8 * mt0;
        const double* O = omega + b * omega_elems + lane;
        // groups past mt_extra run one tile fewer (compile-time counts, no predication); any
        // other shortfall computes padded tiles the reduction never reads
        if (my_mt == MTW - 1 && MTW > 1)
            sk_consume<(MTW > 1 ? MTW - 1 : 1), MTW, NT>(acc, X, O, tg, ksteps, dim);
        else
            sk_consume<MTW, MTW, NT>(acc, X, O, tg, ksteps, dim);
        mbar_arrive(&empty_x[s]);
        mbar_arrive(&empty_o[b]);
        if (++s == nstg) s = 0, ph ^= 1;
        SK_T(c3);
        if (warp == 0) {
            if (j == 0) SK_ADD(8, c0 - k0);
            if (j == nl - 1) SK_ADD(9, c3 - k0);
            SK_ADD(2, c1 - c0);
            SK_ADD(3, c2 - c1);
            SK_ADD(4, c3 - c2);
        }
    }
    // fixed-order sum over the 4 k-step groups: every consumer warp parks its accumulators in its
    // own slice of the (consumed) stages in fragment order, then one pass adds the groups in order
    // 0..3, consecutive threads reading consecutive doubles (conflict-free)
    SK_T(e0);
    if (threadIdx.x == 0) SK_ADD(7, e0 - k0);
    griddep_launch_dependents();
    const uint32_t rbase = smem_u32(stages);
    constexpr int kBlk = MTW * NT;  // 8 x 8 fragment blocks per warp slice
    const int slice = kBlk * 64;
    asm volatile("bar.sync 1, %0;" ::"n"(kSkCons * 32));  // every warp is done with the stages
    {
        const uint32_t mine = rbase + 8u * (uint32_t)(warp * slice);
#pragma unroll
        for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                sts64(mine + 8u * (uint32_t)(((mt * NT + jn) << 6) + 2 * lane), acc[mt][jn][0]);
                sts64(mine + 8u * (uint32_t)(((mt * NT + jn) << 6) + 2 * lane + 1), acc[mt][jn][1]);
            }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kSkCons * 32));
    double* out = a.partial + (int64_t)blockIdx.x * dim * a.K;
    for (int e = tid; e < kSkGrp * kBlk * 64; e += kSkCons * 32) {
        const int blk = e >> 6, w = e & 63;
        const int gr = blk / kBlk, rem = blk - gr * kBlk;
        const int mt = rem / NT, jn = rem - mt * NT;
        if (mt >= mt_base + (gr < mt_extra ? 1 : 0)) continue;  // tile past this group's share
        const int d = 8 * (gr * mt_base + min(gr, mt_extra) + mt) + (w >> 3), k = 8 * jn + (w & 7);
        if (d >= dim || k >= a.K) continue;
        const uint32_t o = rbase + 8u * (uint32_t)(4 * gr * slice + (rem << 6) + w);
        const double v0 = lds64(o), v1 = lds64(o + 8u * slice), v2 = lds64(o + 16u * slice), v3 = lds64(o + 24u * slice);
        out[d + dim * k] = ((0.0 + v0) + v1 + v2) + v3;
    }
    SK_T(k3);
    if (threadIdx.x == 0) SK_ADD(6, k3 - k0);
}

struct TtmArgs {
    const double* x;
    double* out;
    const double* q;  // Q (ldq x K column-major): out(m, o) = sum_d x(m, d) Q(d, o)
    int64_t dim, rows, ntiles, ldq;
    int K, MT, Tk;
    int chain;  // TTMPlan::chain: only the consumers wait on the grid dependency (they read Q)
    int rev;    // tiles in descending order: the rows the chain's sketch read last are still in L2
};

template <int NT>
__global__ void __launch_bounds__((kCons + 1) * 32, 1) k_ttm_l1_f64(TtmArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t dim = a.dim;
    const int MT = a.MT;
    const int stage_elems = (int)(MT * dim) + kPad;
    double* stages = reinterpret_cast<double*>(smem_raw);
    double* Bf = stages + kStages * stage_elems;
    const int bf_elems = a.Tk * NT * 32;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bf + bf_elems);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + kStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

    for (int i = tid; i < kStages * stage_elems; i += blockDim.x) stages[i] = 0.0;
    for (int i = tid; i < bf_elems; i += blockDim.x) {
        const int t = i / (NT * 32);
        const int jn = (i >> 5) % NT;
        const int ln = i & 31;
        const int64_t d = 4 * t + (ln & 3);
        const int o = 8 * jn + (ln >> 2);
        Bf[i] = (d < dim && o < a.K) ? a.q[d + a.ldq * o] : 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_x[s], 1);
            mbar_init(&empty_x[s], kCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCons) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int j = 0; j < nl; ++j) {
                const int s = j % kStages;
                mbar_wait(&empty_x[s], ((j / kStages) & 1) ^ 1);
                const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
                const int64_t m0 = t * MT;
                const int64_t nrow = imin64(MT, a.rows - m0);
                const uint32_t bytes = (uint32_t)(nrow * dim * 8);
                mbar_arrive_expect_tx(&full_x[s], bytes);
                bulk_g2s(stages + s * stage_elems, a.x + m0 * dim, bytes, &full_x[s], pol);
            }
        }
        return;
    }
    const int q = lane >> 2, r = lane & 3;
    for (int j = 0; j < nl; ++j) {
        const int s = j % kStages;
        mbar_wait(&full_x[s], (j / kStages) & 1);
        const double* X = stages + s * stage_elems;
        double acc[2][NT][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
        const double* x0 = X + (16 * warp + q) * dim + r;
        const double* x1 = x0 + 8 * dim;
#pragma unroll 4
        for (int t = 0; t < a.Tk; ++t) {
            double bv[NT];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) bv[jn] = Bf[((t * NT + jn) << 5) + lane];
            const double a0 = x0[4 * t], a1 = x1[4 * t];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                dmma884(acc[0][jn][0], acc[0][jn][1], a0, bv[jn]);
                dmma884(acc[1][jn][0], acc[1][jn][1], a1, bv[jn]);
            }
        }
        mbar_arrive(&empty_x[s]);
        const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
        const int64_t m0 = t * MT;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const int64_t m = m0 + 16 * warp + 8 * mt + q;
            if (m >= a.rows) continue;
            double* dst = a.out + m * a.K;
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
                const int o = 8 * jn + 2 * r;
                if (o + 1 < a.K && !(a.K & 1)) {
                    *reinterpret_cast<double2*>(dst + o) = make_double2(acc[mt][jn][0], acc[mt][jn][1]);
                } else {
                    if (o < a.K) dst[o] = acc[mt][jn][0];
                    if (o + 1 < a.K) dst[o + 1] = acc[mt][jn][1];
                }
            }
        }
    }
}




// Shrink with the small operand in registers: out^T (o x rows) = Q^T (o x d) X^T.
// Q^T is the DMMA A operand and stays in registers for the whole kernel (TKM x
// MTO fragments), so shared memory only feeds the X^T B fragments: one LDS.64
// per 2*MTO DMMAs (half the smem traffic of the X-as-A form, which is what
// bounds the fp64 tensor pipe here). Warp w owns rows 16w..16w+15 of a tile.
template <int MTO, int TKM>
__global__ void __launch_bounds__((kCons + 1) * 32, 1) k_ttm_qreg_f64(TtmArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (!a.chain) griddep_wait();
    const int64_t dim = a.dim;
    const int MT = a.MT;
    const int stage_elems = (int)(MT * dim) + kPad;
    double* stages = reinterpret_cast<double*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kStages * stage_elems);
    uint64_t* full_x = bars;
    uint64_t* empty_x = bars + kStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nl = (int)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int q = lane >> 2, r = lane & 3;

    for (int i = tid; i < kStages * stage_elems; i += blockDim.x) stages[i] = 0.0;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_x[s], 1);
            mbar_init(&empty_x[s], kCons * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCons) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int j = 0; j < nl; ++j) {
                const int s = j % kStages;
                mbar_wait(&empty_x[s], ((j / kStages) & 1) ^ 1);
                const int64_t t0 = blockIdx.x + (int64_t)j * gridDim.x;
                const int64_t t = a.rev ? a.ntiles - 1 - t0 : t0;
                const int64_t m0 = t * MT;
                const int64_t nrow = imin64(MT, a.rows - m0);
                const uint32_t bytes = (uint32_t)(nrow * dim * 8);
                mbar_arrive_expect_tx(&full_x[s], bytes);
                bulk_g2s(stages + s * stage_elems, a.x + m0 * dim, bytes, &full_x[s], pol);
            }
        }
        return;
    }
    // A fragments of Q^T, loaded while the producer's first tiles are in flight:
    // qa[mt][t] = Q^T(o = 8 mt + q, d = 4 t + r) = Q(d, o)
    if (a.chain) griddep_wait();  // Q is the preceding QR launch's output
    double qa[MTO][TKM];
#pragma unroll
    for (int mt = 0; mt < MTO; ++mt)
#pragma unroll
        for (int t = 0; t < TKM; ++t) {
            const int64_t d = 4 * t + r;
            const int o = 8 * mt + q;
            qa[mt][t] = (t < a.Tk && d < dim && o < a.K) ? a.q[d + a.ldq * o] : 0.0;
        }
    for (int j = 0; j < nl; ++j) {
        const int s = j % kStages;
        mbar_wait(&full_x[s], (j / kStages) & 1);
        // B fragment: X^T(d = 4t + r, row = 8 nt + q) = X[row][d]
        const double* x0 = stages + s * stage_elems + (16 * warp + q) * dim + r;
        const double* x1 = x0 + 8 * dim;
        double acc[MTO][2][2];
#pragma unroll
        for (int mt = 0; mt < MTO; ++mt) acc[mt][0][0] = acc[mt][0][1] = acc[mt][1][0] = acc[mt][1][1] = 0.0;
#pragma unroll
        for (int t = 0; t < TKM; ++t) {
            if (t < a.Tk) {
                const double b0 = x0[4 * t], b1 = x1[4 * t];
#pragma unroll
                for (int mt = 0; mt < MTO; ++mt) {
                    dmma884(acc[mt][0][0], acc[mt][0][1], qa[mt][t], b0);
                    dmma884(acc[mt][1][0], acc[mt][1][1], qa[mt][t], b1);
                }
            }
        }
        mbar_arrive(&empty_x[s]);
        // D fragment: out^T(o = 8 mt + q, row = 16 w + 8 nt + 2 r + e)
        const int64_t t0 = blockIdx.x + (int64_t)j * gridDim.x;
        const int64_t m0 = (a.rev ? a.ntiles - 1 - t0 : t0) * MT + 16 * warp;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t m = m0 + 8 * nt + 2 * r + e;
                if (m >= a.rows) continue;
#pragma unroll
                for (int mt = 0; mt < MTO; ++mt) {
                    const int o = 8 * mt + q;
                    if (o < a.K) a.out[m * a.K + o] = acc[mt][nt][e];
                }
            }
    }
}

int nt_for(int K) {
    const int nt = (K + 7) / 8;
    return nt <= 1 ? 1 : nt <= 2 ? 2 : nt <= 4 ? 4 : 8;
}

template <typename KernelT>
void set_smem(KernelT k, size_t smem) {
    allow_smem(k, smem);
}

constexpr size_t kSmemBudget = 220 * 1024;

}  // namespace

// ---------------------------------------------------------------- sketch
// Shared-memory plan of the mode-0 sketch: CT columns per tile, as many X stages as fit (the
// bytes in flight per SM set the HBM rate), and enough Omega buffers for the generators to
// fill one group of tiles while the consumers read the previous one.
struct SkPlan {
    int CT, nstg, nob, pad;
    size_t smem;
};

// row tiles per consumer warp: the larger share of ceil(dim / 8) tiles over kSkGrp groups
int sk_mtw(int64_t dim) {
    const int mt = (int)((dim + 7) / 8);
    return (mt + kSkGrp - 1) / kSkGrp;
}

// zeroed doubles after each stage: the row tiles of the last group reach row 8 kSkGrp MTW - 1 at
// most (an uneven split never overruns; the slack is for safety)
int sk_pad(int64_t dim) {
    const int over = 8 * kSkGrp * sk_mtw(dim) - (int)dim;
    return std::max(8, (over + 8 + 1) & ~1);
}

SkPlan sk_plan(int64_t dim, int K) {
    SkPlan p{};
    static const int ct_env = [] {
        const char* e = getenv("TRG_SK_CT");
        return e ? atoi(e) : 0;
    }();
    p.CT = ct_env > 0 ? ct_env : (dim <= 112 ? 64 : 32);
    const int NT = nt_for(K);
    const int nslots = ((K + 7) / 8 * 8) * ((p.CT / 2 + 3) / 4 * 4);  // as the kernel's fast path
    const int R = nslots <= kRng * 32 ? std::max(1, std::min((kRng * 32) / nslots, kMaxOB / kIlp)) : 1;  // tiles per generator round
    p.nob = std::min(kMaxOB, std::max(4, 2 * R * kIlp));
    p.pad = sk_pad(dim);
    const size_t stage = ((size_t)p.CT * dim + p.pad) * 8;
    const size_t fixed = (size_t)p.nob * p.CT * NT * 8 * 8 + sizeof(GaussTables) + kBarBytes;
    p.nstg = fixed < kSmemBudget ? (int)std::min<size_t>(kMaxStg, (kSmemBudget - fixed) / stage) : 0;
    p.smem = fixed + (size_t)p.nstg * stage;
    return p;
}

bool stream_sketch_ok(int dtype, int64_t left, int64_t dim, int K) {
    if (dtype != F64 || left != 1 || (dim & 1) || K > 64 || dim > 128) return false;
    // register budget: (row tiles per warp) x (8-column groups) accumulators
    const int mtw = sk_mtw(dim);
    if (nt_for(K) > 4 || (nt_for(K) == 4 && mtw > 4)) return false;
    const SkPlan pl = sk_plan(dim, K);
    // the epilogue parks every consumer warp's accumulators in the consumed stages
    const size_t slices = (size_t)kSkCons * sk_mtw(dim) * nt_for(K) * 64 * 8;
    return pl.nstg >= 2 && slices <= (size_t)pl.nstg * ((size_t)pl.CT * dim + pl.pad) * 8;
}

void launch_stream_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                          int* grid_out, cudaStream_t s) {
    SkArgs a;
    // X with the default L2 priority, not evict_first: the shrink that follows re-reads X newest
    // tile first (TtmArgs::rev) and finds the tail of it in L2 (ttm_m0 154 -> 146 us on C2)
    static const int pol_env = (getenv("TRG_POL_SK0") ? atoi(getenv("TRG_POL_SK0")) : 1);
    a.pol = pol_env;
    a.x = reinterpret_cast<const double*>(x);
    a.dim = p.dim;
    a.ncols = p.left * p.right;
    a.K = p.K;
    const SkPlan pl = sk_plan(p.dim, p.K);
    a.CT = pl.CT;
    a.nstg = pl.nstg;
    a.nob = pl.nob;
    a.pad = pl.pad;
    a.ntiles = (a.ncols + a.CT - 1) / a.CT;
    a.mtiles = (int)((p.dim + 7) / 8);
    a.rows_glob = p.rows_glob;
    a.col_off = p.col_off;
    a.seed = p.seed;
    a.D = p.D;
    a.partial = partial;
    a.gt = gauss_tables(s);
    a.kr = p.kr;
    a.kr_smem = 0;
    size_t smem = pl.smem;
    if (p.kr.F && smem + (size_t)p.kr.S1 * p.K * 8 <= 227 * 1024 && p.kr.S1 <= (1 << 20)) {
        a.kr_smem = 1;
        smem += (size_t)p.kr.S1 * p.K * 8;  // F in the headroom of the stage plan
    }
    const int NT = nt_for(p.K);
    const int mtw = sk_mtw(p.dim);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    *grid_out = grid;
    const int threads = (kSkCons + kRng + 1) * 32;
#define TRG_SK(MTW, NTV)                                                 \
    do {                                                                 \
        if (a.kr.F) {                                                    \
            set_smem(k_sketch_l1_f64<MTW, NTV, true>, smem);             \
            pdl_launch(k_sketch_l1_f64<MTW, NTV, true>, dim3(grid), dim3(threads), smem, s, a); \
        } else {                                                         \
            set_smem(k_sketch_l1_f64<MTW, NTV, false>, smem);            \
            pdl_launch(k_sketch_l1_f64<MTW, NTV, false>, dim3(grid), dim3(threads), smem, s, a); \
        }                                                                \
    } while (0)
#define TRG_SK_NT(MTW)                   \
    switch (NT) {                        \
        case 1: TRG_SK(MTW, 1); break;   \
        case 2: TRG_SK(MTW, 2); break;   \
        default: TRG_SK(MTW, 4); break;  \
    }
    static_assert(16 / kSkGrp <= 8, "row-tile instantiations");
    switch (mtw) {
        case 1: TRG_SK_NT(1) break;
        case 2: TRG_SK_NT(2) break;
        case 3: TRG_SK_NT(3) break;
        case 4: TRG_SK_NT(4) break;
        case 5: TRG_SK_NT(5) break;
        case 6: TRG_SK_NT(6) break;
        case 7: TRG_SK_NT(7) break;
        default: TRG_SK_NT(8) break;
    }
#undef TRG_SK_NT
#undef TRG_SK
    if (y) launch_reduce_partials(partial, grid, p.dim * p.K, y, s);
#ifdef TRG_SK_PROF
    unsigned long long h[16];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(h, g_sk_prof, sizeof(h));
    fprintf(stderr, "sk_prof gen: wait_empty %llu compute %llu | cons: wait_x %llu wait_o %llu mma %llu | prologue %llu loop_end %llu total %llu\n", h[0], h[1],
            h[2], h[3], h[4], h[5], h[7], h[6]);
    fprintf(stderr, "sk_prof first_iter_start %llu last_iter_end %llu\n", h[8], h[9]);
    static const unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_sk_prof, z, sizeof(z));
#endif
}

// ---------------------------------------------------------------- shrink
bool stream_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t odim) {
    if (dtype != F64 || left != 1 || (dim & 1) || odim > 64) return false;
    const int Tk = (int)((dim + 3) / 4);
    const size_t smem = (kStages * (size_t)(64 * dim + kPad) + (size_t)Tk * nt_for((int)odim) * 32) * 8 + kBarBytes;
    return smem <= kSmemBudget;
}

void launch_stream_ttm(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, int num_sms,
                       cudaStream_t s) {
    TtmArgs a;
    a.ldq = ldq;
    a.x = reinterpret_cast<const double*>(in);
    a.out = reinterpret_cast<double*>(out);
    a.q = q;
    a.dim = p.dim;
    a.rows = p.right;
    a.K = (int)p.odim;
    a.MT = 16 * kCons;
    a.Tk = (int)((p.dim + 3) / 4);
    a.ntiles = (a.rows + a.MT - 1) / a.MT;
    a.chain = 0;
    static const bool fwd_env = getenv("TRG_TTM_FORWARD") != nullptr;  // development switch
    a.rev = p.chain && !fwd_env ? 1 : 0;
    const int NT = nt_for(a.K);
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms));
    const int threads = (kCons + 1) * 32;
    if (a.K <= 16 && a.Tk <= 32) {  // Q^T resident in registers
        a.chain = p.chain ? 1 : 0;
        if (p.chain) grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, num_sms - p.spare_sms));
        const size_t smem = kStages * (size_t)(a.MT * a.dim + kPad) * 8 + kBarBytes;
#define TRG_QR(MTO, TKM)                                                  \
    do {                                                                  \
        set_smem(k_ttm_qreg_f64<MTO, TKM>, smem);                         \
        pdl_launch(k_ttm_qreg_f64<MTO, TKM>, dim3(grid), dim3(threads), smem, s, a); \
    } while (0)
        if (a.K <= 8) {
            if (a.Tk <= 16) TRG_QR(1, 16); else if (a.Tk <= 25) TRG_QR(1, 25); else TRG_QR(1, 32);
        } else {
            if (a.Tk <= 16) TRG_QR(2, 16); else if (a.Tk <= 25) TRG_QR(2, 25); else TRG_QR(2, 32);
        }
#undef TRG_QR
        return;
    }
    const size_t smem = (kStages * (size_t)(a.MT * a.dim + kPad) + (size_t)a.Tk * NT * 32) * 8 + kBarBytes;
    switch (NT) {
        case 1: set_smem(k_ttm_l1_f64<1>, smem); k_ttm_l1_f64<1><<<grid, threads, smem, s>>>(a); break;
        case 2: set_smem(k_ttm_l1_f64<2>, smem); k_ttm_l1_f64<2><<<grid, threads, smem, s>>>(a); break;
        case 4: set_smem(k_ttm_l1_f64<4>, smem); k_ttm_l1_f64<4><<<grid, threads, smem, s>>>(a); break;
        default: set_smem(k_ttm_l1_f64<8>, smem); k_ttm_l1_f64<8><<<grid, threads, smem, s>>>(a); break;
    }
}

}  // namespace trg

namespace trg {


}  // namespace trg
