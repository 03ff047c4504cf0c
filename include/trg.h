/* SPDX-License-Identifier: Apache-2.0
 *
 * libtrg — B200-native randomized tensor-ring decomposition hot path, C ABI.
 *
 * Drop-in boundary for the reference's sketch / rTR-ALS / rTR-SVD path
 * (/root/reference/proj/include/tenring/sketch.hpp). The reference exposes
 * plain C++ inline functions over host containers; this library exposes the
 * same operations as extern "C" entry points over plain pointers and sizes so
 * that any host binding (the C++ facade in include/tenring_b200.hpp, ctypes,
 * cgo, JNI) can call them. Each entry point names the reference function it
 * replaces. See INTEGRATION.md for the bindings.
 *
 * Conventions
 *  - Every function returns TRG_OK (0) or an error code; trg_last_error()
 *    returns the thread-local message. Codes map back to the reference's
 *    exception types: TRG_EINVAL <-> std::invalid_argument (tensor.hpp:21-23),
 *    TRG_ERANGE <-> std::out_of_range (tensor.hpp:93-97).
 *  - Tensors use the reference layout: first index fastest (tensor.hpp:33-38),
 *    0-based modes (tensor.hpp:41). Matrices are column-major (Eigen default).
 *  - TR cores are passed flat and concatenated in mode order; core n has
 *    shape (R_n, I_n, R_{n+1 mod N}) (tr_factors.hpp:14-21).
 *  - Device tensors may be sharded along the LAST mode across the ranks of a
 *    distributed context: each rank holds the contiguous slab [lo, hi) given
 *    by trg_shard_range(). Host buffers passed to upload/download are the
 *    local slab. All results (projected tensor, bases, cores, RSE) are
 *    replicated on every rank.
 *  - Calls on one context are stream-ordered on the context's CUDA stream.
 *    There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with TRG_ENODEV.
 */
#ifndef TRG_H_
#define TRG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRG_ABI_VERSION 1

enum trg_status {
    TRG_OK = 0,
    TRG_EINVAL = 1,    /* std::invalid_argument */
    TRG_ERANGE = 2,    /* std::out_of_range */
    TRG_ECUDA = 3,     /* CUDA runtime error */
    TRG_ENCCL = 4,     /* NCCL error / NCCL unavailable */
    TRG_ENUMERIC = 5,  /* numerical failure */
    TRG_ENODEV = 6,    /* no usable CUDA device */
    TRG_EINTERNAL = 9
};

enum trg_dtype { TRG_F32 = 0, TRG_F64 = 1 };
enum trg_variant {
    TRG_SEQUENTIAL = 0, /* reference sketch(): sequential shrinking, sketch.hpp:62-89 */
    TRG_FUSED = 1,      /* SPEC.md:319 alternative: every Y_n from the original X */
    /* Opt-in flag OR-ed into either variant (changes results, so never the
     * default): Omega_n is the Khatri-Rao product of per-mode Gaussian factors F_{n,m}
     * (S_m x K_n, m != n, S = the working shape of mode n) instead of prod_{m != n} S_m x K_n
     * independent draws. The factors are drawn from the same stream `seed`, column-major, in
     * mode order n, then m, starting at draw 0; skipped modes draw nothing. Supported where the
     * fp64 streaming kernels run (fp64 tensors with mode extents <= 128 and K_n <= 16). */
    TRG_OMEGA_KHATRI_RAO = 16
};
enum trg_method { TRG_ALS = 0, TRG_SVD = 1 };

typedef struct trg_ctx trg_ctx;
typedef struct trg_tensor trg_tensor;
typedef struct trg_sketch trg_sketch;
typedef struct trg_report trg_report;
typedef struct trg_loopback trg_loopback;

int trg_abi_version(void);
const char* trg_last_error(void);
int trg_device_count(int* count);

/* ---- contexts ----------------------------------------------------------- */
int trg_ctx_create(int device, trg_ctx** out);
/* NCCL unique id (128 bytes) created on rank 0 and broadcast by the caller. */
int trg_nccl_unique_id(unsigned char id[128]);
int trg_ctx_create_dist(int device, int rank, int world, const unsigned char id[128], trg_ctx** out);
/* Loopback communicator: `world` shard programs in ONE process, every rank on its own host
 * thread with its own context (and stream) on `device`, usually all on the same GPU. Each
 * collective of the sharded path (the Y_n partial sums, the padded last-mode gather, the P
 * sum, the RSE and synthesis norms) becomes: every rank finishes its stream, a host barrier,
 * every rank sums the `world` buffers in rank order into a private buffer (one kernel on its
 * own stream), a second barrier, then the result replaces the rank's buffer. No kernel ever
 * waits on another rank's kernel. It runs the sharded CUDA path exactly as the NCCL contexts
 * do (real column offsets, uneven shards, the world > 1 QR and scatter paths) on one device,
 * for tests; it is not a performance path. A failing rank leaves the others blocked in the
 * next collective: callers run ranks under a timeout. */
int trg_loopback_create(int world, trg_loopback** out);
int trg_loopback_destroy(trg_loopback* group);
int trg_ctx_create_loopback(int device, int rank, trg_loopback* group, trg_ctx** out);
int trg_ctx_destroy(trg_ctx* ctx);
int trg_ctx_synchronize(trg_ctx* ctx);
int trg_ctx_stream(trg_ctx* ctx, void** cuda_stream);
/* Per-kernel CUDA-event timing (labels such as "sketch_m0", "ttm_m0", "qr"). */
int trg_ctx_set_profiling(trg_ctx* ctx, int on);
int trg_ctx_kernel_stats(trg_ctx* ctx, const char* label, double* total_ms, int64_t* launches);
int trg_ctx_kernel_labels(trg_ctx* ctx, char* buf, int64_t cap); /* newline-separated */
int trg_ctx_launch_count(trg_ctx* ctx, int64_t* launches);       /* every libtrg kernel launch */
int trg_ctx_reset_stats(trg_ctx* ctx);
/* Balanced last-mode partition used for sharded tensors (pure host). */
int trg_shard_range(int64_t extent, int rank, int world, int64_t* lo, int64_t* hi);
/* Pure host: where each mode's test matrix sits in the reference stream for
 * this rank's slab. Omega_n(c, k) = draw draw_off[n] + col_off[n] + c +
 * rows_glob[n] * k for local unfolding column c (rows_glob[n] = 0: skipped). */
int trg_sketch_offsets(int order, const int64_t* dims, const int64_t* K, int rank, int world, int variant,
                       int64_t* rows_glob, int64_t* col_off, uint64_t* draw_off);

/* ---- dense tensors (DenseTensor, tensor.hpp:42-108) --------------------- */
int trg_tensor_create(trg_ctx* ctx, int dtype, int order, const int64_t* dims, trg_tensor** out);
int trg_tensor_info(const trg_tensor* t, int* dtype, int* order, int64_t* dims, int64_t* lo, int64_t* hi);
int trg_tensor_upload(trg_tensor* t, const void* host_local);
int trg_tensor_download(const trg_tensor* t, void* host_local);
int trg_tensor_device_ptr(const trg_tensor* t, void** ptr, int64_t* local_elems);
/* X = reconstruct_full(cores) (tr_factors.hpp:123-137) evaluated on device,
 * optionally affinely rescaled to [0,1] (rescale01 != 0), then, if snr_db is
 * finite, plus noise E = draws of GaussianSampler(noise_seed) in flat order
 * scaled so ||E||/||X|| = 10^(-snr_db/20). */
int trg_tensor_synthesize(trg_tensor* t, const int64_t* ranks, const double* cores, int rescale01, double snr_db,
                          uint64_t noise_seed);
int trg_tensor_destroy(trg_tensor* t);

/* ---- tensor random projection (sketch.hpp:62-89) ------------------------ */
/* Enqueues the whole projection on the context stream and returns without
 * synchronising; the getters below synchronise. K has `order` entries,
 * 1 <= K_n <= I_n, K_n == I_n skips the mode (no draws). The sketch does not
 * keep a reference to `x`: once the enqueued work has run, x may be destroyed. */
int trg_sketch_run(trg_ctx* ctx, const trg_tensor* x, const int64_t* K, uint64_t seed, int variant,
                   trg_sketch** out);
int trg_sketch_projected(const trg_sketch* sk, double* out);     /* prod K_n, first-index-fastest */
int trg_sketch_basis(const trg_sketch* sk, int mode, double* out); /* Q_n: I_n x K_n col-major */
int trg_sketch_y(const trg_sketch* sk, int mode, double* out);     /* Y_n: I_n x K_n (parity) */
int trg_sketch_qr_path(const trg_sketch* sk, int mode, int* householder); /* 0 CholQR2, 1 Householder */
int trg_sketch_elapsed_ms(const trg_sketch* sk, double* ms);       /* device time, first kernel -> P resident */
int trg_sketch_destroy(trg_sketch* sk);
/* detail::economy_q (sketch.hpp:45-53) on one host matrix: Y is m x k col-major,
 * Q (m x k col-major) has the reference sign convention (diag R >= 0).
 * *householder (may be NULL) reports the path taken: 0 CholQR2, 1 Householder. */
int trg_thin_qr(trg_ctx* ctx, int64_t m, int64_t k, const double* y, double* q, int* householder);
/* Test-matrix export: out(c, k) = reference draw offset + c + rows*k (sketch.hpp:32-38). */
int trg_omega(trg_ctx* ctx, uint64_t seed, uint64_t offset, int64_t rows, int64_t cols, double* out);

/* ---- TR model ------------------------------------------------------------- */
/* out = x x_mode M (tensor.hpp:193-207); M is m_rows x I_mode col-major. */
int trg_mode_n_product(trg_ctx* ctx, const trg_tensor* x, int mode, int64_t m_rows, const double* m,
                       trg_tensor** out);
/* lift_back (sketch.hpp:93-101): P x_0 Q_0 x_1 Q_1 ... (the plain TRP approximation of x), computed
 * on the device into a new full-size tensor. The sketch-handle form uses the resident P and Q_n; the
 * host form uploads P (prod K_n) and the bases (I_n x K_n col-major each) and, like the reference,
 * skips a basis that is square and exactly the identity. Unsharded contexts only. */
int trg_sketch_lift_back(const trg_sketch* sk, trg_tensor** out);
int trg_lift_back(trg_ctx* ctx, int order, const int64_t* dims, const int64_t* K, const double* projected,
                  const double* const* bases, trg_tensor** out);
/* G_n = Z_n x_2 Q_n (sketch.hpp:106-122); small core n is (R_n, K_n, R_{n+1}). */
int trg_back_project(trg_ctx* ctx, int order, const int64_t* K, const int64_t* ranks, const double* small_cores,
                     const trg_sketch* sk, double* cores_out);
/* rse(x, reconstruct_full(cores)) (solvers.hpp:47-54, tr_factors.hpp:123-137) without materialising Xhat. */
int trg_rse(trg_ctx* ctx, const trg_tensor* x, const int64_t* ranks, const double* cores, double* out);

/* ---- Algorithm 1 (randomized_decompose, sketch.hpp:126-147) -------------- */
/* method TRG_ALS = rtrals (sketch.hpp:154-158, ranks required),
 * TRG_SVD = rtrsvd (sketch.hpp:161-165, ranks ignored, tol = truncation). */
int trg_decompose(trg_ctx* ctx, const trg_tensor* x, int method, const int64_t* ranks, double tol,
                  int64_t max_sweeps, uint64_t cfg_seed, const int64_t* K, uint64_t spec_seed, int variant,
                  trg_report** out);
/* Same, from a host buffer (local slab): the H2D copy is part of the call. */
int trg_decompose_host(trg_ctx* ctx, int dtype, int order, const int64_t* dims, const void* host_local, int method,
                       const int64_t* ranks, double tol, int64_t max_sweeps, uint64_t cfg_seed, const int64_t* K,
                       uint64_t spec_seed, int variant, trg_report** out);
int trg_report_ranks(const trg_report* r, int64_t* ranks);
int trg_report_cores_len(const trg_report* r, int64_t* n);
int trg_report_cores(const trg_report* r, double* out);
int trg_report_rse_history(const trg_report* r, double* out, int64_t* n); /* out may be NULL to query n */
int trg_report_sweeps(const trg_report* r, int64_t* sweeps);
/* ms[0..5] = h2d, sketch, small solve, back-projection, final RSE, total */
int trg_report_timings(const trg_report* r, double* ms);
int trg_report_projected(const trg_report* r, double* out, int64_t* n);
int trg_report_destroy(trg_report* r);

#ifdef __cplusplus
}
#endif

#endif /* TRG_H_ */
