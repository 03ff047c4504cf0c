// SPDX-License-Identifier: Apache-2.0
//
// TR-model kernels: subchain contraction, fused reconstruction / RSE (K8),
// synthesis (K9) and small elementwise helpers.
//
// Reference: reconstruct_full (tr_factors.hpp:123-137) builds
// X_<0> = G_{0,(2)} (G_{!=0,<2>})^T and rse (solvers.hpp:47-54) then reads
// both |X| tensors again. Here the subchain S = G_1 o ... o G_{N-1}
// (tr_factors.hpp:111-119, chain_contract :92-102) is contracted once on
// device and one tiled fp64 GEMM computes Xhat(i0, p) = sum_{a,b}
// G0(a, i0, b) S(b, p, a) with the (x - xhat)^2 and x^2 sums fused into its
// epilogue, so Xhat is never written (RSE) — or is written as X (synthesis).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace trg {

namespace {

__global__ void k_chain(const double* __restrict__ a, int64_t ra, int64_t p, int64_t rb, const double* __restrict__ g,
                        int64_t ii, int64_t rc, double* __restrict__ out) {
    const int64_t n = ra * p * ii * rc;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        // out index e = x + Ra*(q + P*i + P*I*c) with x < Ra, q < P
        const int64_t x = e % ra;
        int64_t rest = e / ra;
        const int64_t q = rest % p;
        rest /= p;
        const int64_t i = rest % ii;
        const int64_t c = rest / ii;
        double s = 0.0;
        for (int64_t b = 0; b < rb; ++b) s = fma(a[x + ra * (q + p * b)], g[b + rb * (i + ii * c)], s);
        out[e] = s;
    }
}

constexpr int RT = 64;   // rows (i0) per CTA tile
constexpr int PT = 64;   // columns (p) per CTA tile
constexpr int QC = 16;   // contraction chunk over b

template <typename T, bool WRITE>
__global__ void __launch_bounds__(256) k_recon(const double* __restrict__ g0, const double* __restrict__ S, T* x,
                                               int64_t I0, int64_t P, int64_t R0, int64_t R1,
                                               double* __restrict__ block_sums) {
    __shared__ double As[QC][RT];
    __shared__ double Bs[QC][PT + 1];
    __shared__ double red[2][8];
    const int tid = threadIdx.x;
    const int ti = tid & 15, tp = tid >> 4;
    const int64_t i_base = (int64_t)blockIdx.y * RT;
    const int64_t p_base = (int64_t)blockIdx.x * PT;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    for (int64_t a = 0; a < R0; ++a) {
        for (int64_t b0 = 0; b0 < R1; b0 += QC) {
            const int nb = (R1 - b0) < QC ? (int)(R1 - b0) : QC;
            __syncthreads();
            // A(i0, (a,b)) = G0[a + R0*(i0 + I0*b)]
            for (int e = tid; e < QC * RT; e += 256) {
                const int bb = e / RT, ii = e - bb * RT;
                const int64_t i0 = i_base + ii;
                As[bb][ii] = (bb < nb && i0 < I0) ? g0[a + R0 * (i0 + I0 * (b0 + bb))] : 0.0;
            }
            // B((a,b), p) = S[b + R1*(p + P*a)], b fastest (coalesced)
            for (int e = tid; e < QC * PT; e += 256) {
                const int pp = e / QC, bb = e - pp * QC;
                const int64_t pc = p_base + pp;
                Bs[bb][pp] = (bb < nb && pc < P) ? S[(b0 + bb) + R1 * (pc + P * a)] : 0.0;
            }
            __syncthreads();
#pragma unroll 4
            for (int bb = 0; bb < QC; ++bb) {
                double av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) av[i] = As[bb][ti + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[j] = Bs[bb][tp + 16 * j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
        }
    }
    double se = 0.0, sx = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t pc = p_base + tp + 16 * j;
        if (pc >= P) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t i0 = i_base + ti + 16 * i;
            if (i0 >= I0) continue;
            T* px = x + i0 + I0 * pc;
            if (WRITE) {
                *px = T(acc[i][j]);
            } else {
                const double xv = (double)*px;
                const double d = xv - acc[i][j];
                se = fma(d, d, se);
                sx = fma(xv, xv, sx);
            }
        }
    }
    if (!WRITE) {
        for (int o = 16; o > 0; o >>= 1) {
            se += __shfl_xor_sync(0xffffffffu, se, o);
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
        }
        if ((tid & 31) == 0) {
            red[0][tid >> 5] = se;
            red[1][tid >> 5] = sx;
        }
        __syncthreads();
        if (tid == 0) {
            double a0 = 0.0, a1 = 0.0;
            for (int w = 0; w < 8; ++w) {
                a0 += red[0][w];
                a1 += red[1][w];
            }
            const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
            block_sums[2 * bid] = a0;
            block_sums[2 * bid + 1] = a1;
        }
    }
}


// ---- K8 / K9 on the FP64 tensor pipe (m8n8k4 DMMA): Xhat(i0, p) = sum_q A(i0, q) B(q, p) with
// q = b + R1 a, A(i0, q) = G0(a, i0, b) and B(q, p) = S(b, p, a) (tr_factors.hpp:123-137), for
// K = R0 R1 <= 64. CTA = (a block of up to 128 rows of i0, a persistent loop over 64-column tiles of
// p): A lives in shared memory for the whole launch, the B tile of the next columns streams in by
// cp.async while the current one is multiplied. Warp job = (8-row tile, two 8-column tiles) over
// all of K; the epilogue reads X straight into the accumulator layout and forms sum (x - xhat)^2
// and sum x^2 (solvers.hpp:47-54), or writes Xhat (synthesis). A tile's columns are a fixed set
// and the CTA's sums run in a fixed order: bit-reproducible.
constexpr int kRdCols = 64;  // columns of p per tile
constexpr int kRdMaxRows = 128;
constexpr int kRdMaxK = 64;
constexpr int kRdThreads = 512;

__device__ __forceinline__ void rd_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void rd_cp8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

template <typename T, bool WRITE>
__global__ void __launch_bounds__(kRdThreads, 1)
    k_recon_dmma(const double* __restrict__ g0, const double* __restrict__ S, T* x, int64_t I0, int64_t P, int R0, int R1,
                 int Kp, int ldg, int lds, double* __restrict__ block_sums) {
    extern __shared__ __align__(16) double rd_smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int K = R0 * R1;
    const int64_t row0 = (int64_t)blockIdx.y * kRdMaxRows;
    const int rows = (int)min((int64_t)kRdMaxRows, I0 - row0);
    const int mtiles = (rows + 7) / 8;
    double* Gs = rd_smem;                                   // [mtiles * 8][ldg]
    double* Ss = Gs + (size_t)mtiles * 8 * ldg;             // [2][Kp][lds]
    double* red = Ss + 2 * (size_t)Kp * lds;                // [2][16]
    // A = G0 rows of this block, zero-padded to whole tiles and to Kp
    for (int e = tid; e < mtiles * 8 * Kp; e += kRdThreads) {
        const int r = e / Kp, q = e - r * Kp;
        double v = 0.0;
        if (r < rows && q < K) {
            const int a = q / R1, b = q - a * R1;
            v = g0[a + (int64_t)R0 * ((row0 + r) + I0 * b)];
        }
        Gs[r * ldg + q] = v;
    }
    const int64_t ntiles = (P + kRdCols - 1) / kRdCols;
    // B(q, p) = S[b + R1 (p + P a)]: for each a, R1 x 64 consecutive doubles (b fastest)
    auto issue = [&](int64_t t, int buf) {
        const int64_t p0 = t * kRdCols;
        const int pc = (int)min((int64_t)kRdCols, P - p0);
        double* dst = Ss + (size_t)buf * Kp * lds;
        for (int e = tid; e < K * kRdCols; e += kRdThreads) {
            const int a = e / (R1 * kRdCols), rem = e - a * (R1 * kRdCols);
            const int pp = rem / R1, b = rem - pp * R1;
            if (pp < pc) rd_cp8(dst + (b + R1 * a) * lds + pp, S + b + (int64_t)R1 * (p0 + pp + P * a));
            else dst[(b + R1 * a) * lds + pp] = 0.0;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // padded rows q in [K, Kp) of both buffers stay zero
    for (int e = tid; e < 2 * (Kp - K) * lds; e += kRdThreads) {
        const int bq = e / lds, c = e - bq * lds;
        Ss[(size_t)(bq / (Kp - K)) * Kp * lds + (size_t)(K + bq % (Kp - K)) * lds + c] = 0.0;
    }
    double se = 0.0, sx = 0.0;
    const int njobs = mtiles * (kRdCols / 16);  // (8-row tile, pair of 8-column tiles)
    int64_t t = blockIdx.x;
    if (t < ntiles) issue(t, 0);
    for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        const int buf = it & 1;
        const int64_t tn = t + gridDim.x;
        if (tn < ntiles) {
            issue(tn, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* Sb = Ss + (size_t)buf * Kp * lds;
        const int64_t p0 = t * kRdCols;
        for (int job = warp; job < njobs; job += kRdThreads / 32) {
            const int mt = job % mtiles, np = job / mtiles;
            const int r = 8 * mt + (lane >> 2);  // D fragment row; columns 2 (lane & 3) + {0, 1}
            // this lane's X entries first (epilogue operands in flight during the MMAs)
            double xv[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
            if (!WRITE) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int64_t p = p0 + 8 * (2 * np + h) + 2 * (lane & 3) + c;
                        if (r < rows && p < P) xv[h][c] = (double)x[(row0 + r) + I0 * p];
                    }
            }
            double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
            const double* ar = Gs + (8 * mt + (lane >> 2)) * ldg + (lane & 3);
            const double* br = Sb + (lane & 3) * lds + 16 * np + (lane >> 2);
#pragma unroll 4
            for (int ks = 0; ks < Kp / 4; ++ks) {
                const double av = ar[4 * ks];
                const double b0 = br[4 * ks * lds], b1 = br[4 * ks * lds + 8];
                rd_dmma(acc[0][0], acc[0][1], av, b0);
                rd_dmma(acc[1][0], acc[1][1], av, b1);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int64_t p = p0 + 8 * (2 * np + h) + 2 * (lane & 3) + c;
                    if (r < rows && p < P) {
                        if (WRITE) {
                            x[(row0 + r) + I0 * p] = T(acc[h][c]);
                        } else {
                            const double d = xv[h][c] - acc[h][c];
                            se = fma(d, d, se);
                            sx = fma(xv[h][c], xv[h][c], sx);
                        }
                    }
                }
        }
        __syncthreads();  // the buffer is refilled two tiles later
    }
    if (!WRITE) {
        for (int o = 16; o > 0; o >>= 1) {
            se += __shfl_xor_sync(0xffffffffu, se, o);
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
        }
        if (lane == 0) {
            red[warp] = se;
            red[16 + warp] = sx;
        }
        __syncthreads();
        if (tid == 0) {
            double a0 = 0.0, a1 = 0.0;
            for (int w = 0; w < kRdThreads / 32; ++w) {
                a0 += red[w];
                a1 += red[16 + w];
            }
            const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
            block_sums[2 * bid] = a0;
            block_sums[2 * bid + 1] = a1;
        }
    }
}

bool recon_dmma_ok(const ReconPlan& p) {
    return !getenv("TRG_RECON_SIMT") && p.R0 * p.R1 <= kRdMaxK && p.I0 >= 1 && p.P >= 1 &&
           (p.dtype == F64 || p.write_mode != 0);  // fp32 RSE sums: k_rse_f32 (FFMA) unless fp64 is asked for
}

size_t recon_dmma_smem(int64_t I0, int Kp, int ldg, int lds) {
    const int64_t rows = std::min<int64_t>(I0, kRdMaxRows);
    return sizeof(double) * ((size_t)((rows + 7) / 8) * 8 * ldg + 2 * (size_t)Kp * lds + 32);
}

// ---- K8 for fp32 tensors: Xhat(i0, p) = sum_{a,b} G0(a, i0, b) S(b, p, a) (tr_factors.hpp:123-137) as a
// register-tiled FFMA GEMM on fp32 operands (the tensor is fp32; the RSE tolerance is 1e-4), with
// sum (x - xhat)^2 and x^2 accumulated in fp64 in the epilogue (solvers.hpp:47-54). The operands
// are first rounded and laid out K-major by two small passes: At[q][i0] and St[q][p] with
// q = b + R1 a, so every tile row is contiguous and streams by 16-byte cp.async into a 3-stage ring.
// M = I0 rows (tile MT = 128 or 64), N = the subchain's columns p (tile 128), K in chunks of 16.
constexpr int kRkc = 16;
constexpr int kRst = 3;

__global__ void k_rse_prep_a(const double* __restrict__ g0, int64_t I0, int R0, int R1, int64_t ld,
                             float* __restrict__ At) {
    const int64_t n = (int64_t)R0 * R1 * ld;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / ld, i0 = e - q * ld;
        const int a = (int)(q / R1), b = (int)(q - (int64_t)a * R1);
        At[e] = i0 < I0 ? (float)g0[a + (int64_t)R0 * (i0 + I0 * b)] : 0.f;
    }
}

// St[q][p] (row pitch ld >= P, zero padded) from S[b + R1 (p + P a)]: 32 x 32 tiles through shared memory
__global__ void k_rse_prep_s(const double* __restrict__ S, int64_t P, int R0, int R1, int64_t ld, float* __restrict__ St) {
    __shared__ float t[32][33];
    const int K = R0 * R1;
    const int64_t p0 = (int64_t)blockIdx.x * 32;
    const int q0 = blockIdx.y * 32;
    // read: q fastest within a (b contiguous in S)
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int64_t p = p0 + j;
        const int q = q0 + threadIdx.x;
        float v = 0.f;
        if (q < K && p < P) {
            const int a = q / R1, b = q - a * R1;
            v = (float)S[b + (int64_t)R1 * (p + P * a)];
        }
        t[threadIdx.x][j] = v;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int q = q0 + j;
        const int64_t p = p0 + threadIdx.x;
        if (q < K && p < ld) St[(int64_t)q * ld + p] = t[j][threadIdx.x];
    }
}

__device__ __forceinline__ void cp16_rse(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

template <int MT>
__global__ void __launch_bounds__(256, MT == 64 ? 2 : 1) k_rse_f32(const float* __restrict__ At, int64_t lda, const float* __restrict__ St,
                                                 int64_t ldb, const float* __restrict__ x, int64_t I0, int64_t P, int K,
                                                 double* __restrict__ block_sums) {
    constexpr int TM = MT / 16;  // rows per thread
    constexpr int NT = 128;
    __shared__ __align__(16) float As[kRst][kRkc][MT];
    __shared__ __align__(16) float Bs[kRst][kRkc][NT];
    double* red = reinterpret_cast<double*>(&As[0][0][0]);  // [2][8], after the main loop
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;  // columns 8 tx.., rows TM ty..
    const int64_t i_base = (int64_t)blockIdx.y * MT;
    const int64_t p_base = (int64_t)blockIdx.x * NT;
    const int nch = (K + kRkc - 1) / kRkc;  // At / St rows past K are zero (prep passes)
    auto issue = [&](int c) {
        const int buf = c % kRst;
        for (int e = tid; e < kRkc * MT / 4; e += 256) {
            const int qq = e / (MT / 4), i4 = e - qq * (MT / 4);
            cp16_rse(&As[buf][qq][4 * i4], At + (int64_t)(c * kRkc + qq) * lda + i_base + 4 * i4);
        }
        for (int e = tid; e < kRkc * NT / 4; e += 256) {
            const int qq = e / (NT / 4), p4 = e - qq * (NT / 4);
            cp16_rse(&Bs[buf][qq][4 * p4], St + (int64_t)(c * kRkc + qq) * ldb + p_base + 4 * p4);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[TM][8];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (int c = 0; c < kRst - 1; ++c) {
        if (c < nch) issue(c);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kRst - 2) : "memory");
        __syncthreads();  // chunk c landed for everyone; chunk c - 1's buffer is free
        if (c + kRst - 1 < nch) issue(c + kRst - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        const int buf = c % kRst;
        // fragments of step qq + 1 are loaded before the FFMAs of step qq (two register sets)
        float4 fa[2][TM / 4], fb[2][2];
        auto frag = [&](int qq, int h) {
#pragma unroll
            for (int i = 0; i < TM / 4; ++i) fa[h][i] = *reinterpret_cast<const float4*>(&As[buf][qq][TM * ty + 4 * i]);
            fb[h][0] = *reinterpret_cast<const float4*>(&Bs[buf][qq][4 * tx]);
            fb[h][1] = *reinterpret_cast<const float4*>(&Bs[buf][qq][64 + 4 * tx]);
        };
        frag(0, 0);
#pragma unroll
        for (int qq = 0; qq < kRkc; ++qq) {
            const int h = qq & 1;
            if (qq + 1 < kRkc) frag(qq + 1, h ^ 1);
            float av[TM], bv[8];
#pragma unroll
            for (int i = 0; i < TM / 4; ++i) {
                av[4 * i] = fa[h][i].x;
                av[4 * i + 1] = fa[h][i].y;
                av[4 * i + 2] = fa[h][i].z;
                av[4 * i + 3] = fa[h][i].w;
            }
            bv[0] = fb[h][0].x; bv[1] = fb[h][0].y; bv[2] = fb[h][0].z; bv[3] = fb[h][0].w;
            bv[4] = fb[h][1].x; bv[5] = fb[h][1].y; bv[6] = fb[h][1].z; bv[7] = fb[h][1].w;
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
    }
    // epilogue: this thread's TM rows of a column are contiguous in X (first index fastest): 16-byte
    // loads when I0 % 4 == 0. Columns 4 tx + j (j < 4) and 64 + 4 tx + j (the B fragments above).
    double se = 0.0, sx = 0.0;
    const bool vec = (I0 & 3) == 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t pc = p_base + (j < 4 ? 4 * tx + j : 64 + 4 * tx + (j - 4));
        if (pc >= P) continue;
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
            const int64_t i0 = i_base + TM * ty + i;
            float xv[4];
            if (vec && i0 + 3 < I0) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(x + i0 + I0 * pc));
                xv[0] = v.x;
                xv[1] = v.y;
                xv[2] = v.z;
                xv[3] = v.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = i0 + u < I0 ? x[i0 + u + I0 * pc] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (i0 + u >= I0) continue;
                const double xd = (double)xv[u];
                const double d = xd - (double)acc[i + u][j];
                se = fma(d, d, se);
                sx = fma(xd, xd, sx);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        se += __shfl_xor_sync(0xffffffffu, se, o);
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // every warp is past the ring
    if ((tid & 31) == 0) {
        red[tid >> 5] = se;
        red[8 + (tid >> 5)] = sx;
    }
    __syncthreads();
    if (tid == 0) {
        double a0 = 0.0, a1 = 0.0;
        for (int w = 0; w < 8; ++w) {
            a0 += red[w];
            a1 += red[8 + w];
        }
        const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
        block_sums[2 * bid] = a0;
        block_sums[2 * bid + 1] = a1;
    }
}

__global__ void k_sum_pairs(const double* __restrict__ bs, int n, double* out) {
    __shared__ double r0[256], r1[256];
    double a = 0.0, b = 0.0;
    // fixed assignment of blocks to threads + fixed tree => deterministic
    for (int i = threadIdx.x; i < n; i += 256) {
        a += bs[2 * i];
        b += bs[2 * i + 1];
    }
    r0[threadIdx.x] = a;
    r1[threadIdx.x] = b;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] += r0[threadIdx.x + s];
            r1[threadIdx.x] += r1[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = r0[0];
        out[1] = r1[0];
    }
}

template <typename T>
__global__ void k_noise_norms(const T* __restrict__ x, int64_t n, uint64_t seed, uint64_t off,
                              double* __restrict__ bs) {
    double sx = 0.0, se = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double xv = (double)x[i];
        const double e = gauss_draw<double>(seed, off + (uint64_t)i);
        sx = fma(xv, xv, sx);
        se = fma(e, e, se);
    }
    __shared__ double r0[256], r1[256];
    r0[threadIdx.x] = sx;
    r1[threadIdx.x] = se;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] += r0[threadIdx.x + s];
            r1[threadIdx.x] += r1[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bs[2 * blockIdx.x] = r0[0];
        bs[2 * blockIdx.x + 1] = r1[0];
    }
}

template <typename T>
__global__ void k_add_noise(T* x, int64_t n, uint64_t seed, uint64_t off, double alpha) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = T((double)x[i] + alpha * gauss_draw<double>(seed, off + (uint64_t)i));
}

template <typename T>
__global__ void k_minmax(const T* __restrict__ x, int64_t n, double* __restrict__ bs) {
    double lo = 1e308, hi = -1e308;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)x[i];
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    __shared__ double r0[256], r1[256];
    r0[threadIdx.x] = lo;
    r1[threadIdx.x] = hi;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            r0[threadIdx.x] = fmin(r0[threadIdx.x], r0[threadIdx.x + s]);
            r1[threadIdx.x] = fmax(r1[threadIdx.x], r1[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bs[2 * blockIdx.x] = r0[0];
        bs[2 * blockIdx.x + 1] = r1[0];
    }
}

template <typename T>
__global__ void k_affine(T* x, int64_t n, double a, double b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = T(a * (double)x[i] + b);
}

template <typename Ti, typename To>
__global__ void k_convert(const Ti* __restrict__ in, To* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = To(in[i]);
}

__global__ void k_scatter_rows(const double* __restrict__ in, int64_t rows, int k, int64_t lo, int64_t m,
                               double* __restrict__ out) {
    const int64_t n = m * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / m, r = e - c * m;
        out[e] = (r >= lo && r < lo + rows) ? in[(r - lo) + rows * c] : 0.0;
    }
}

int grid_for(int64_t n, int threads = 256, int cap = 8192) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

}  // namespace

void launch_chain(const double* a, int64_t ra, int64_t p, int64_t rb, const double* g, int64_t i, int64_t rc,
                  double* out, cudaStream_t s) {
    const int64_t n = ra * p * i * rc;
    k_chain<<<grid_for(n), 256, 0, s>>>(a, ra, p, rb, g, i, rc, out);
}

void plan_recon(ReconPlan& p, int num_sms) {
    p.threads = 256;
    if (recon_dmma_ok(p)) {  // DMMA: persistent column loop, one CTA per SM over the row blocks
        p.grid_y = (int)((p.I0 + kRdMaxRows - 1) / kRdMaxRows);
        p.grid_x = (int)std::max<int64_t>(1, std::min<int64_t>((p.P + kRdCols - 1) / kRdCols, num_sms / p.grid_y));
        p.nblocks = p.grid_x * p.grid_y;
        p.threads = kRdThreads;
        p.smem = 0;
        return;
    }
    if (p.dtype == F32 && p.write_mode == 0) {  // fp32 RSE: k_rse_f32, 128 columns x 64 (128) rows
        static const bool t128 = getenv("TRG_RSE_MT128") != nullptr;
        const int mt = (p.I0 <= 64 || !t128) ? 64 : 128;
        p.grid_x = (int)((p.P + 127) / 128);
        p.grid_y = (int)((p.I0 + mt - 1) / mt);
    } else {
        p.grid_x = (int)((p.P + PT - 1) / PT);
        p.grid_y = (int)((p.I0 + RT - 1) / RT);
    }
    p.nblocks = p.grid_x * p.grid_y;
    p.smem = 0;
}

void launch_recon(const ReconPlan& p, const double* g0, const double* S, void* x, int write_mode, double* block_sums,
                  cudaStream_t s) {
    dim3 grid(p.grid_x, p.grid_y);
    if (recon_dmma_ok(p)) {
        const int K = (int)(p.R0 * p.R1), Kp = (K + 3) & ~3;
        int ldg = Kp;
        while (ldg % 16 != 4) ++ldg;  // 8 rows x 4 k of an A fragment over all 32 banks
        const int lds = kRdCols + 8;   // 4 k rows x 8 columns of a B fragment: two conflict-free halves
        const size_t smem = recon_dmma_smem(p.I0, Kp, ldg, lds);
        const bool wr = write_mode == 1;
        auto go = [&](auto kern, auto* xp) {
            allow_smem(kern, smem);
            kern<<<grid, kRdThreads, smem, s>>>(g0, S, xp, p.I0, p.P, (int)p.R0, (int)p.R1, Kp, ldg, lds, block_sums);
        };
        if (p.dtype == F64) {
            if (wr) go(k_recon_dmma<double, true>, (double*)x);
            else go(k_recon_dmma<double, false>, (double*)x);
        } else {
            if (wr) go(k_recon_dmma<float, true>, (float*)x);
            else go(k_recon_dmma<float, false>, (float*)x);
        }
        return;
    }
    if (p.dtype == F64) {
        if (write_mode)
            k_recon<double, true><<<grid, 256, 0, s>>>(g0, S, (double*)x, p.I0, p.P, p.R0, p.R1, block_sums);
        else
            k_recon<double, false><<<grid, 256, 0, s>>>(g0, S, (double*)x, p.I0, p.P, p.R0, p.R1, block_sums);
    } else {
        if (write_mode)
            k_recon<float, true><<<grid, 256, 0, s>>>(g0, S, (float*)x, p.I0, p.P, p.R0, p.R1, block_sums);
        else if (p.write_mode == 2)  // fp64 arithmetic on the fp32 tensor
            k_recon<float, false><<<grid, 256, 0, s>>>(g0, S, (float*)x, p.I0, p.P, p.R0, p.R1, block_sums);
        else {
            // K-major fp32 operands, padded to whole tiles: At (K16 x I0 tiles), St (K16 x P tiles)
            const int K = (int)(p.R0 * p.R1), K16 = (K + kRkc - 1) / kRkc * kRkc;
            static const bool t128 = getenv("TRG_RSE_MT128") != nullptr;  // development comparison
            const int mt = (p.I0 <= 64 || !t128) ? 64 : 128;
            const int64_t lda = (int64_t)p.grid_y * mt, ldb = (int64_t)p.grid_x * 128;
            float* At = (float*)scratch_alloc(sizeof(float) * (size_t)K16 * lda, s);
            float* St = (float*)scratch_alloc(sizeof(float) * (size_t)K16 * ldb, s);
            cudaMemsetAsync(At, 0, sizeof(float) * (size_t)K16 * lda, s);
            cudaMemsetAsync(St + (size_t)K * ldb, 0, sizeof(float) * (size_t)(K16 - K) * ldb, s);
            k_rse_prep_a<<<grid_for((int64_t)K * lda), 256, 0, s>>>(g0, p.I0, (int)p.R0, (int)p.R1, lda, At);
            k_rse_prep_s<<<dim3((unsigned)((ldb + 31) / 32), (unsigned)((K + 31) / 32)), dim3(32, 8), 0, s>>>(
                S, p.P, (int)p.R0, (int)p.R1, ldb, St);
            if (mt == 64)
                k_rse_f32<64><<<grid, 256, 0, s>>>(At, lda, St, ldb, (const float*)x, p.I0, p.P, K, block_sums);
            else
                k_rse_f32<128><<<grid, 256, 0, s>>>(At, lda, St, ldb, (const float*)x, p.I0, p.P, K, block_sums);
            scratch_free(St, s);
            scratch_free(At, s);
        }
    }
}

void launch_sum_pairs(const double* block_sums, int nblocks, double* out, cudaStream_t s) {
    k_sum_pairs<<<1, 256, 0, s>>>(block_sums, nblocks, out);
}

void launch_noise_norms(const void* x, int dtype, int64_t n, uint64_t seed, uint64_t off, double* block_sums,
                        int nblocks, cudaStream_t s) {
    if (dtype == F64)
        k_noise_norms<double><<<nblocks, 256, 0, s>>>((const double*)x, n, seed, off, block_sums);
    else
        k_noise_norms<float><<<nblocks, 256, 0, s>>>((const float*)x, n, seed, off, block_sums);
}

void launch_add_noise(void* x, int dtype, int64_t n, uint64_t seed, uint64_t off, double alpha, cudaStream_t s) {
    if (dtype == F64)
        k_add_noise<double><<<grid_for(n), 256, 0, s>>>((double*)x, n, seed, off, alpha);
    else
        k_add_noise<float><<<grid_for(n), 256, 0, s>>>((float*)x, n, seed, off, alpha);
}

void launch_minmax(const void* x, int dtype, int64_t n, double* block_mm, int nblocks, cudaStream_t s) {
    if (dtype == F64)
        k_minmax<double><<<nblocks, 256, 0, s>>>((const double*)x, n, block_mm);
    else
        k_minmax<float><<<nblocks, 256, 0, s>>>((const float*)x, n, block_mm);
}

void launch_affine(void* x, int dtype, int64_t n, double a, double b, cudaStream_t s) {
    if (dtype == F64)
        k_affine<double><<<grid_for(n), 256, 0, s>>>((double*)x, n, a, b);
    else
        k_affine<float><<<grid_for(n), 256, 0, s>>>((float*)x, n, a, b);
}

void launch_convert(const void* in, int in_dt, void* out, int out_dt, int64_t n, cudaStream_t s) {
    const int g = grid_for(n);
    if (in_dt == F64 && out_dt == F64)
        k_convert<double, double><<<g, 256, 0, s>>>((const double*)in, (double*)out, n);
    else if (in_dt == F64)
        k_convert<double, float><<<g, 256, 0, s>>>((const double*)in, (float*)out, n);
    else if (out_dt == F64)
        k_convert<float, double><<<g, 256, 0, s>>>((const float*)in, (double*)out, n);
    else
        k_convert<float, float><<<g, 256, 0, s>>>((const float*)in, (float*)out, n);
}

void launch_scatter_rows(const double* in, int64_t rows, int k, int64_t lo, int64_t m, double* out, cudaStream_t s) {
    k_scatter_rows<<<grid_for(m * k), 256, 0, s>>>(in, rows, k, lo, m, out);
}

// ---- loopback communicator: rank-ordered reduction of same-device buffers
struct RankBufs {
    const void* p[kMaxLoopbackRanks];
};

template <typename T>
__global__ void k_rank_reduce(RankBufs b, int nranks, int64_t n, int op, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T acc = static_cast<const T*>(b.p[0])[i];
        for (int r = 1; r < nranks; ++r) {
            const T v = static_cast<const T*>(b.p[r])[i];
            acc = op == 0 ? acc + v : (v > acc ? v : acc);
        }
        out[i] = acc;
    }
}

void launch_rank_reduce(const void* const* bufs, int nranks, size_t count, int dtype, int op, void* out,
                        cudaStream_t s) {
    RankBufs b{};
    for (int r = 0; r < nranks; ++r) b.p[r] = bufs[r];
    if (dtype == F64)
        k_rank_reduce<double><<<grid_for((int64_t)count), 256, 0, s>>>(b, nranks, (int64_t)count, op, (double*)out);
    else
        k_rank_reduce<float><<<grid_for((int64_t)count), 256, 0, s>>>(b, nranks, (int64_t)count, op, (float*)out);
}

}  // namespace trg
