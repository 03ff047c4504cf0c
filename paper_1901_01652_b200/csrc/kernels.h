// SPDX-License-Identifier: Apache-2.0
// Host-side launchers for the libtrg sm_100a kernels. Internal to libtrg.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace trg {

enum DType { F32 = 0, F64 = 1 };

inline size_t dtype_size(int dt) { return dt == F64 ? 8 : 4; }

// Stream-ordered scratch for launchers that need a temporary (multi-CTA QR, split-d TTM): from the
// calling context's private pool (set by trg_ctx::launch for the thread), else the device's
// default pool.
void set_thread_pool(cudaMemPool_t pool);
void* scratch_alloc(size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);

// ---- opt-in Khatri-Rao test matrix (TRG_OMEGA_KHATRI_RAO) ----
// Omega_n(c, k) = A(c mod left, k) * F(r mod S1, k) * H(r / S1, k), r = c / left, where A is the
// Khatri-Rao product of the per-mode Gaussian factors of the modes before n (left x K), F the
// factor of mode n + 1 (S1 x K) and H the product of the factors after n + 1 (nH x K); all
// column-major fp64, c and r global unfolding indices (runtime.cpp build_kr). F == nullptr: the
// reference Gaussian stream.
struct KrOmega {
    const double* A = nullptr;
    const double* F = nullptr;
    const double* H = nullptr;
    int64_t left = 1, S1 = 1, nH = 1;
};

// ---- sketch: Y_n = P_(n) * Omega_n (K1), deterministic split-K -------------
// The current tensor is read as (left, dim, right) (tensor.hpp:112-123);
// unfold_classic column c = l + left*r (tensor.hpp:133-142). Omega_n(c, k) is
// reference draw D + col_off + c + rows_glob*k of the single stream `seed`
// (sketch.hpp:32-38, 69, 81). Result Y is dim x K column-major fp64.
struct SketchPlan {
    int dtype;
    int64_t left, dim, right;  // local view
    int K;
    uint64_t seed, D;
    int64_t rows_glob, col_off;
    KrOmega kr;  // Khatri-Rao test matrix instead of the draws (stream / slab kernels only)
    // derived by plan_sketch()
    int TD, TK, Kp, DT, CT, nd, nk, G, threads, ndt;
    int64_t ncols, ntiles;
    int grid_x;
    size_t smem;
    size_t partial_elems;  // grid_x * dim * K doubles
};
void plan_sketch(SketchPlan& p, int num_sms);
void launch_sketch(const SketchPlan& p, const void* x, double* partial, double* y, cudaStream_t s);

// ---- mode-n product out = in x_n M (K2 shrink with M = Q^T, K7 lift with M = Q)
// M(o, d) = m[o*m_so + d*m_sd] (fp64). out has odim in place of dim.
struct TTMPlan {
    int dtype;
    int64_t left, dim, right, odim;
    int64_t m_so, m_sd;
    // derived
    int TM, TO, MT, DT, nm, no, OT, threads, noT, dsplit;
    int64_t rows, nrowtiles;
    int grid_x;
    size_t smem;
    // shrink of the projection chain (run_sketch): its input was completed two or more grids back,
    // so the register-Q kernels prefetch it before the grid dependency on the QR resolves, and
    // they leave `spare_sms` SMs to the QR launch they follow
    bool chain = false;
    int spare_sms = 0;
};
void plan_ttm(TTMPlan& p, int num_sms);
void launch_ttm(const TTMPlan& p, const void* in, void* out, const double* m, cudaStream_t s);

// ---- TMA-pipelined fp64 tensor-core kernels for the mode-0 passes (stream_f64.cu)
bool stream_sketch_ok(int dtype, int64_t left, int64_t dim, int K);
// The per-CTA partial sums of Y go to `partial`; with y == nullptr the split-K reduction is
// left to the caller (launch_qr_fused), and the launchers return the number of partials.
void launch_stream_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                          int* grid_out, cudaStream_t s);
bool stream_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t odim);
void launch_stream_ttm(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, int num_sms,
                       cudaStream_t s);
// ---- fp32 mode-0 sketch (FFMA, TMA 2-D boxes), stream_f32.cu; partial = grid_cols x dim x K
bool stream_sketch_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols);
int stream_sketch_f32_grid(int64_t dim, int K, int64_t ncols, int num_sms, int* grid_cols);
int launch_stream_sketch_f32(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                             cudaStream_t s);
bool stream_ttm_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols);
// writes P^(1) in fp32 (or fp64 with f64_out)
void launch_stream_ttm_f32(const TTMPlan& p, const void* in, void* out, bool f64_out, const double* q, int64_t ldq,
                           int num_sms, cudaStream_t s);

// ---- fp32 mode-0 sketch / shrink on tcgen05 (kind::tf32, 3xTF32, TMEM accumulators), tc_f32.cu
bool tc_sketch_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols);
int tc_sketch_f32_grid(int64_t dim, int K, int64_t ncols, int num_sms);  // = partial count
int launch_tc_sketch_f32(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                         cudaStream_t s);
bool tc_ttm_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols);
size_t tc_ttm_f32_scratch(int64_t dim, int64_t K);  // bytes of the split Q operand
// out: P^(1) in fp64 (f64_out) or fp32; q: Q (ldq x K column-major fp64)
void launch_tc_ttm_f32(const TTMPlan& p, const void* in, void* out, bool f64_out, const double* q, int64_t ldq,
                       float* scratch, int num_sms, cudaStream_t s);

// ---- fp32 sketch for modes with left % 32 == 0 and K >= 32 on tcgen05 (tc_f32.cu): partial = parts x dim x K
bool tc_sketch_n_f32_ok(int dtype, int64_t left, int64_t dim, int K, int64_t right);
int tc_sketch_n_f32_parts(int64_t left, int64_t dim, int K, int64_t right, int num_sms);
int launch_tc_sketch_n_f32(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                           cudaStream_t s);

bool tc_ttm_n_f32_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right);
size_t tc_ttm_n_f32_scratch(int64_t dim, int64_t K);  // bytes of the split Q operand
void launch_tc_ttm_n_f32(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, float* scratch,
                         int num_sms, cudaStream_t s);

// ---- fp32 register-tiled FFMA kernels for modes with left > 1 (slab_f32.cu); fp32 in and out
bool slab_f32_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right);
void launch_slab_f32_ttm(const TTMPlan& p, const void* in, void* out, const double* m, int num_sms, cudaStream_t s);
bool slab_f32_sketch_ok(int dtype, int64_t left, int64_t dim, int K, int64_t right);
int slab_f32_sketch_grid(int64_t left, int64_t dim, int K, int64_t right, int num_sms);  // = partial count
int launch_slab_f32_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                           cudaStream_t s);

// ---- fp32 TMA-streamed FFMA kernels for modes with left > 1 (slab_st.cu): producer warp + mbarrier
// ring of 3-D boxes, generator warps for the sketch's test-matrix blocks
bool st_shrink_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right);
void launch_st_shrink(const TTMPlan& p, const void* in, void* out, const double* m, int num_sms, cudaStream_t s);
bool st_sketch_ok(int dtype, int64_t left, int64_t dim, int K, int64_t right);
int st_sketch_grid(int64_t left, int64_t dim, int K, int64_t right, int num_sms);  // = partial count
int launch_st_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms, cudaStream_t s);

// mode-0 shrink of a short-fibre fp32 tensor (left == 1, dim <= 128, dim % 4 == 0; C5): bulk-copied fibres
bool st0_shrink_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t ncols);
void launch_st0_shrink(const TTMPlan& p, const void* in, void* out, const double* m, int num_sms, cudaStream_t s);

// ---- cp.async-gathered fp64 tensor-core kernels for modes with left > 1 (slab_f64.cu)
bool slab_sketch_ok(int dtype, int64_t left, int64_t dim, int K, int64_t ncols);
void launch_slab_sketch(const SketchPlan& p, const void* x, double* partial, double* y, int num_sms,
                        cudaStream_t s);
bool slab_ttm_ok(int dtype, int64_t left, int64_t dim, int64_t odim, int64_t ncols);
void launch_slab_ttm(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, int num_sms,
                     cudaStream_t s);
// ---- TMA-tensor (128B-swizzled) fp64 kernels for modes with left > 1 (slab_tma.cu)
bool slab2_ok(int dtype, int64_t left, int64_t dim, int64_t K, int64_t right);
int64_t slab2_units(int64_t left, int64_t right);
// unit blocks of the reference test matrix (4 x NT x 32 doubles per unit), L2-resident
struct GaussTables;
struct OmegaUnitsJob {  // one mode's unit blocks, generated by k_omega_units or inside another launch
    double* out = nullptr;
    int64_t left = 0, nunits = 0;
    int LC = 0, K = 0, NT = 0;
    uint64_t seed = 0, D = 0;
    int64_t col_off = 0, rows_glob = 0;
    const GaussTables* gt = nullptr;
    KrOmega kr;  // kr.F set: the unit blocks of the Khatri-Rao test matrix instead of the draws
};
OmegaUnitsJob omega_units_job(int64_t left, int64_t right, int K, uint64_t seed, uint64_t D, int64_t col_off,
                              int64_t rows_glob, double* out, const KrOmega* kr = nullptr);
void launch_omega_units(int64_t left, int64_t right, int K, uint64_t seed, uint64_t D, int64_t col_off,
                        int64_t rows_glob, double* out, cudaStream_t s, const KrOmega* kr = nullptr);
// Khatri-Rao tables in one launch: table t is out(row, k) = prod_j draws[off_j + i_j + rows_j k],
// row = sum_j i_j stride_j (first index fastest); nf = 0 gives a column of ones.
constexpr int kKrMaxTables = 24, kKrMaxFactors = 7;
struct KrTable {
    double* out;
    int64_t nrows;
    int K, nf;
    int64_t off[kKrMaxFactors], rows[kKrMaxFactors];
};
void launch_kr_tables(const double* draws, const KrTable* tabs, int ntab, cudaStream_t s);
int launch_slab2_sketch(const SketchPlan& p, const void* x, const double* omega_units, double* partial, double* y,
                        int num_sms, cudaStream_t s);
void launch_slab2_ttm(const TTMPlan& p, const void* in, void* out, const double* q, int64_t ldq, int num_sms,
                      cudaStream_t s);
// fixed-order sum of nblocks partial (n doubles each)
void launch_reduce_partials(const double* partial, int nblocks, int64_t n, double* out, cudaStream_t s);
// the same sum (fixed order, a different one) spread over ~n / 16 CTAs with 16-byte loads
void launch_reduce_wide(const double* partial, int nparts, int64_t n, double* out, cudaStream_t s);
// zero n ints in a one-CTA kernel launched into the programmatic-launch chain
void launch_zero_ints(int* p, int n, cudaStream_t s);

// ---- thin QR with diag(R) >= 0 (K4): CholQR2 + Householder fallback, fp64.
// Y is m x k column-major; Q (m x k) out. work >= m*k doubles + 2*k.
void launch_qr(const double* y, int64_t m, int k, double* q, double* work, int* flag, cudaStream_t s);
// Split-K reduction of nparts partial sums of Y (m x k each) fused with its QR in one cluster
// launch; writes Y and Q. Returns false (nothing launched) when the shape is outside the
// fused kernel (k > 32 or the staging does not fit), then the caller reduces and calls launch_qr.
bool qr_fused_ok(int64_t m, int k);
// ticket: zero-initialised int the reducing CTAs count arrivals on (reset by the last one); null
// -> a separate reduction kernel. Returns the number of kernels launched.
// job (run iff ticket && nparts > 1, else ignored): test-matrix unit blocks for a later mode, generated by
// extra CTAs of the same launch (num_sms of them minus the reducing ones) while it is latency-bound.
int launch_qr_fused(const double* part, int nparts, int64_t m, int k, double* y, double* q, double* work, int* flag,
                    int* ticket, cudaStream_t s, const OmegaUnitsJob* job = nullptr, int num_sms = 0);

// ---- per-device tables of the table-driven Box-Muller (common.cuh), built on first use
const GaussTables* gauss_tables(cudaStream_t s);

// ---- Gaussian test-matrix export (parity): out(c, k) = draw off + c + rows*k
void launch_omega(uint64_t seed, uint64_t off, int64_t rows, int64_t cols, double* out, cudaStream_t s);

// ---- TR model on device ------------------------------------------------------
// chain_contract (tr_factors.hpp:92-102): (Ra,P,Rb) o (Rb,I,Rc) -> (Ra,P*I,Rc), fp64
void launch_chain(const double* a, int64_t ra, int64_t p, int64_t rb, const double* g, int64_t i, int64_t rc,
                  double* out, cudaStream_t s);
// X(i0, p) = sum_{a,b} G0(a, i0, b) S(b, p, a) over the local columns p:
// mode 0 writes X (dtype) ; mode 1 accumulates per-block (sum (x - xhat)^2, sum x^2).
struct ReconPlan {
    int dtype;
    int write_mode;  // 1: synthesis (X := Xhat), 0: RSE sums (fp32 tensors: the FFMA GEMM k_rse_f32), 2: RSE in fp64
    int64_t I0, P, R0, R1;
    int grid_x, grid_y, threads;
    size_t smem;
    int nblocks;
};
void plan_recon(ReconPlan& p, int num_sms);
void launch_recon(const ReconPlan& p, const double* g0, const double* S, void* x, int write_mode, double* block_sums,
                  cudaStream_t s);
// sum of block partial pairs in fixed order -> out[0..1]
void launch_sum_pairs(const double* block_sums, int nblocks, double* out, cudaStream_t s);
// noise: sums of x^2 and e^2 (e = draws off..off+n-1), then x += alpha*e
void launch_noise_norms(const void* x, int dtype, int64_t n, uint64_t seed, uint64_t off, double* block_sums,
                        int nblocks, cudaStream_t s);
void launch_add_noise(void* x, int dtype, int64_t n, uint64_t seed, uint64_t off, double alpha, cudaStream_t s);
// y = alpha * x + beta (affine rescale, used by the hyperspectral synthesizer)
void launch_minmax(const void* x, int dtype, int64_t n, double* block_mm, int nblocks, cudaStream_t s);
void launch_affine(void* x, int dtype, int64_t n, double a, double b, cudaStream_t s);
// dtype conversion helpers
void launch_convert(const void* in, int in_dt, void* out, int out_dt, int64_t n, cudaStream_t s);
// out[i] = op over ranks r = 0..nranks-1, in rank order, of ((T*)bufs[r])[i]; op 0 sum, 1 max.
// Loopback communicator (runtime.cpp): every rank's buffer is on the same device.
constexpr int kMaxLoopbackRanks = 16;
void launch_rank_reduce(const void* const* bufs, int nranks, size_t count, int dtype, int op, void* out,
                        cudaStream_t s);
// scatter rows [lo, lo+rows) of a (rows x k) column-major matrix into a zeroed (m x k) matrix
void launch_scatter_rows(const double* in, int64_t rows, int k, int64_t lo, int64_t m, double* out, cudaStream_t s);

}  // namespace trg
