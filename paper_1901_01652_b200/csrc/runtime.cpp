// SPDX-License-Identifier: Apache-2.0
//
// libtrg host runtime: contexts, device tensors, the per-mode projection
// pipeline, back-projection, RSE and Algorithm 1 orchestration behind the
// C ABI of include/trg.h.
//
// Reference map:
//   trg_sketch_run      sketch                 sketch.hpp:62-89
//   trg_back_project    back_project           sketch.hpp:106-122
//   trg_rse             rse(x, reconstruct_full) solvers.hpp:47-54, tr_factors.hpp:123-137
//   trg_decompose       randomized_decompose    sketch.hpp:126-147 (rtrals :154, rtrsvd :161)
//   trg_omega           gaussian_matrix         sketch.hpp:32-38
//   trg_mode_n_product  mode_n_product          tensor.hpp:193-207
//
// Everything between the first sketch kernel and "P and all Q_n resident" is
// stream-ordered device work with no host round trip: per mode the sketch
// (K1) + fixed-order split-K reduction, the NCCL sum of the Y partial when the
// tensor is sharded, the CholQR2 (K4) and the shrink (K2).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/trg.h"
#include "host_solve.hpp"
#include "kernels.h"

namespace {

using trg::F32;
using trg::F64;

thread_local std::string g_err;

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct nccl_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct nodev_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

void require(bool ok, const std::string& msg) {
    if (!ok) throw std::invalid_argument(msg);
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return TRG_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return TRG_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return TRG_ERANGE;
    } catch (const nodev_error& e) {
        g_err = e.what();
        return TRG_ENODEV;
    } catch (const cuda_error& e) {
        g_err = e.what();
        return TRG_ECUDA;
    } catch (const nccl_error& e) {
        g_err = e.what();
        return TRG_ENCCL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TRG_EINTERNAL;
    }
}

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
    void load() {
        if (h) return;
        // prefer an already-loaded NCCL (e.g. torch's) so one copy serves the process
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw nccl_error("NCCL (libnccl.so.2) not loadable");
        getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !commDestroy || !allReduce)
            throw nccl_error("NCCL symbols missing");
    }
    void check(ncclResult_t r, const char* what) {
        if (r != ncclSuccess)
            throw nccl_error(std::string(what) + ": " + (getErrorString ? getErrorString(r) : "nccl error"));
    }
};
Nccl& nccl() {
    static Nccl n;
    return n;
}

}  // namespace

namespace trg {
thread_local cudaMemPool_t tls_pool = nullptr;
void set_thread_pool(cudaMemPool_t pool) { tls_pool = pool; }
void* scratch_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    if (tls_pool)
        cuda_check(cudaMallocFromPoolAsync(&p, bytes ? bytes : 8, tls_pool, s), "scratch_alloc");
    else
        cuda_check(cudaMallocAsync(&p, bytes ? bytes : 8, s), "scratch_alloc");
    return p;
}
void scratch_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}
}  // namespace trg

// ------------------------------------------------------------------ loopback communicator
// `world` ranks of one process (one host thread and one context each, trg.h). A collective is
// two host barriers around a rank-ordered reduction that every rank computes for itself.
struct trg_loopback {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void*> bufs;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

// ------------------------------------------------------------------ context
struct KStat {
    double ms = 0.0;
    int64_t n = 0;
};

struct trg_ctx {
    int device = 0;
    int rank = 0, world = 1;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // test-matrix generation for later modes, overlapped with QR / shrink
    cudaMemPool_t pool = nullptr;  // private stream-ordered pool (release threshold: keep)
    ncclComm_t comm = nullptr;
    trg_loopback* lb = nullptr;  // loopback ranks (no NCCL): see reduce_loopback
    // arrival tickets of the fused QR reduce, one per mode: zeroed once here, and every QR launch
    // leaves its ticket at zero again (the last arriving CTA resets it), so a projection needs no
    // zeroing kernel of its own
    int* tickets = nullptr;
    int tickets_n = 0;
    int* ensure_tickets(int n) {
        if (n > tickets_n) {
            if (tickets) cudaFreeAsync(tickets, stream);
            tickets_n = std::max(n, 16);
            CK(cudaMallocFromPoolAsync((void**)&tickets, sizeof(int) * tickets_n, pool, stream));
            CK(cudaMemsetAsync(tickets, 0, sizeof(int) * tickets_n, stream));
        }
        return tickets;
    }
    bool profiling = false;
    int64_t launches = 0;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> event_pool;
    std::map<std::string, KStat> stats;

    cudaEvent_t get_event() {
        if (!event_pool.empty()) {
            cudaEvent_t e = event_pool.back();
            event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }
    // Run one kernel launch, counted and (optionally) timed with events on the stream.
    template <typename F>
    void launch(const std::string& label, F&& f, int count = 1) {
        trg::set_thread_pool(pool);  // launchers' own scratch comes from this context's pool
        cudaEvent_t a = nullptr, b = nullptr;
        if (profiling) {
            a = get_event();
            b = get_event();
            CK(cudaEventRecord(a, stream));
        }
        f();
        CK(cudaGetLastError());
        launches += count;
        if (profiling) {
            CK(cudaEventRecord(b, stream));
            pending.push_back({label, {a, b}});
        }
    }
    void collect() {
        if (pending.empty()) return;
        CK(cudaStreamSynchronize(stream));
        for (auto& p : pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
            KStat& s = stats[p.first];
            s.ms += ms;
            s.n += 1;
            event_pool.push_back(p.second.first);
            event_pool.push_back(p.second.second);
        }
        pending.clear();
    }
    void* alloc(size_t bytes) {
        void* p = nullptr;
        if (bytes == 0) bytes = 8;
        CK(cudaMallocFromPoolAsync(&p, bytes, pool, stream));
        return p;
    }
    void dfree(void* p) {
        if (p) cudaFreeAsync(p, stream);
    }
    // ---- per-projection scratch arena: temporaries of run_sketch (split-K partials, QR work,
    // intermediate P^(n), test-matrix blocks) come from one context-owned buffer, so no
    // allocator operation sits between the kernels of the per-mode chain (they are launched
    // with programmatic dependent launch). Reuse across projections is stream-ordered.
    char* scr_base = nullptr;
    size_t scr_cap = 0, scr_off = 0, scr_need = 0;
    bool scr_active = false;
    std::vector<void*> scr_overflow;
    void scr_begin() {
        if (scr_need > scr_cap) {
            if (scr_base) cudaFreeAsync(scr_base, stream);
            scr_cap = scr_need + scr_need / 4;
            CK(cudaMallocFromPoolAsync((void**)&scr_base, scr_cap, pool, stream));
        }
        scr_off = 0;
        scr_active = true;
    }
    void* tmp(size_t bytes) {
        if (!scr_active) return alloc(bytes);
        bytes = (bytes + 255) & ~size_t(255);
        if (scr_off + bytes > scr_need) scr_need = scr_off + bytes;
        if (scr_base && scr_off + bytes <= scr_cap) {
            void* p = scr_base + scr_off;
            scr_off += bytes;
            return p;
        }
        scr_off += bytes;  // counted for the next projection's arena size
        void* p = alloc(bytes);
        scr_overflow.push_back(p);
        return p;
    }
    void tmp_free(void* p) {
        if (!scr_active) dfree(p);  // arena memory is released wholesale by scr_end()
    }
    void scr_end() {
        for (void* p : scr_overflow) dfree(p);
        scr_overflow.clear();
        scr_active = false;
    }
    void allreduce(void* buf, size_t count, int dtype) {
        if (world == 1 || count == 0) return;
        if (lb) return reduce_loopback(buf, count, dtype, 0);
        nccl().check(nccl().allReduce(buf, buf, count, dtype == F64 ? ncclFloat64 : ncclFloat32, ncclSum, comm, stream),
                     "ncclAllReduce");
    }
    void allreduce_op(void* buf, size_t count, ncclRedOp_t op) {
        if (world == 1 || count == 0) return;
        if (lb) return reduce_loopback(buf, count, F64, op == ncclMax ? 1 : 0);
        nccl().check(nccl().allReduce(buf, buf, count, ncclFloat64, op, comm, stream), "ncclAllReduce");
    }
    // The loopback allreduce: the same device holds every rank's buffer, so after a barrier each
    // rank reduces all of them in rank order into a private buffer; after a second barrier (no
    // rank reads the others' buffers any more) the result replaces its own.
    void reduce_loopback(void* buf, size_t count, int dtype, int op) {
        const size_t bytes = count * trg::dtype_size(dtype);
        CK(cudaStreamSynchronize(stream));
        lb->bufs[rank] = buf;
        lb->barrier();
        void* out = alloc(bytes);
        launch("allreduce", [&] { trg::launch_rank_reduce(lb->bufs.data(), world, count, dtype, op, out, stream); });
        CK(cudaStreamSynchronize(stream));
        lb->barrier();
        CK(cudaMemcpyAsync(buf, out, bytes, cudaMemcpyDeviceToDevice, stream));
        dfree(out);
    }
};

struct trg_tensor {
    trg_ctx* ctx = nullptr;
    int dtype = F64;
    std::vector<int64_t> dims;  // global
    int64_t lo = 0, hi = 0;     // local slab of the last mode
    void* d = nullptr;
    int64_t local_elems = 0;
    std::vector<int64_t> local_shape() const {
        std::vector<int64_t> s = dims;
        s.back() = hi - lo;
        return s;
    }
    int64_t inner() const {  // prod of all but the last mode
        int64_t p = 1;
        for (size_t i = 0; i + 1 < dims.size(); ++i) p *= dims[i];
        return p;
    }
};

struct trg_sketch {
    trg_ctx* ctx = nullptr;
    int dtype = F64;
    int variant = TRG_SEQUENTIAL;
    std::vector<int64_t> dims, K;
    std::vector<double*> dQ;  // device Q_n (nullptr for skipped modes)
    std::vector<double*> dY;  // device Y_n full rows
    int* dflags = nullptr;    // N QR-path flags
    void* dP = nullptr;       // device P (dtype), full prod K
    bool P_is_view = false;   // P aliases x (no mode projected, unsharded)
    int64_t P_elems = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void release() {
        for (double*& p : dQ) ctx->dfree(p), p = nullptr;
        for (double*& p : dY) ctx->dfree(p), p = nullptr;
        ctx->dfree(dflags);
        dflags = nullptr;
        if (!P_is_view) ctx->dfree(dP);
        dP = nullptr;
    }
    ~trg_sketch() {
        if (!ctx) return;
        release();
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
};

struct trg_report {
    std::vector<int64_t> ranks;
    std::vector<double> cores;
    std::vector<double> rse_history;
    std::vector<double> projected;
    int64_t sweeps = 0;
    double ms[6] = {0, 0, 0, 0, 0, 0};
};

namespace {

int64_t prod(const std::vector<int64_t>& v, size_t b = 0, size_t e = SIZE_MAX) {
    int64_t p = 1;
    const size_t end = std::min(e, v.size());
    for (size_t i = b; i < end; ++i) p *= v[i];
    return p;
}

void shard(int64_t extent, int rank, int world, int64_t& lo, int64_t& hi) {
    const int64_t base = extent / world, rem = extent % world;
    lo = rank * base + std::min<int64_t>(rank, rem);
    hi = lo + base + (rank < rem ? 1 : 0);
}

void ensure_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) throw nodev_error("no CUDA device available (libtrg has no CPU fallback)");
}

void validate_K(const trg_tensor* x, const int64_t* K) {
    require(K != nullptr, "sketch: projection size list must match tensor order");
    for (size_t n = 0; n < x->dims.size(); ++n)
        require(K[n] >= 1 && K[n] <= x->dims[n], "sketch: need 1 <= K_n <= I_n in mode " + std::to_string(n));
}

// ------------------------------------------------------------------ projection pipeline
// Where mode n's test matrix sits in the reference stream and which of its rows a
// rank owns (pure host; exported as trg_sketch_offsets for the sharding tests).
// Omega_n(c, k) = draw D_n + col_off_n + c + rows_glob_n * k (sketch.hpp:32-38, 69,
// 81), c = local column of the unfolding. rows_glob_n is the column count of the
// GLOBAL current unfolding (sized against the shrunken tensor, sketch.hpp:80-81, or
// against X for the fused variant); skipped modes draw nothing
// (sketch.hpp:76-79). For n < N-1 the last mode is the slowest column digit, so a
// rank's slab [lo, hi) owns the contiguous column block starting at col_off_n; for
// n = N-1 every rank holds all columns and its own rows of Y.
struct ModeOffsets {
    int64_t rows_glob = 0, col_off = 0;
    uint64_t D = 0;
    bool skipped = false;
};

std::vector<ModeOffsets> sketch_offsets(const std::vector<int64_t>& dims, const int64_t* K, int64_t lo, int variant) {
    const int N = (int)dims.size();
    std::vector<ModeOffsets> out(N);
    std::vector<int64_t> cur = dims;
    uint64_t D = 0;
    for (int n = 0; n < N; ++n) {
        ModeOffsets& o = out[n];
        o.D = D;
        if (K[n] == dims[n]) {
            o.skipped = true;
            continue;
        }
        const int64_t left = prod(cur, 0, n);
        if (n < N - 1) {
            const int64_t r_inner = prod(cur, n + 1, N - 1);
            o.rows_glob = left * r_inner * dims[N - 1];
            o.col_off = left * r_inner * lo;
        } else {
            o.rows_glob = left;
            o.col_off = 0;
        }
        D += (uint64_t)o.rows_glob * (uint64_t)K[n];
        if (variant == TRG_SEQUENTIAL) cur[n] = K[n];
    }
    return out;
}

// Y_n of the (local) current tensor cur with shape cur_shape, into dYfull
// (I_n x K_n, replicated).
// Omega_n unit blocks generated ahead of time on the side stream (slab2 modes)
struct PreOmega {
    double* buf = nullptr;
    cudaEvent_t ready = nullptr;
    bool joined = false;   // main stream already waits on `ready`
    bool pending = false;  // `buf` not generated yet: a QR launch on the main stream takes `job`
    trg::OmegaUnitsJob job;
};

// Per-CTA partial sums of Y_n left for the QR launch to reduce (launch_qr_fused)
struct YParts {
    double* partial = nullptr;
    int nparts = 0;
};

void sketch_mode(trg_ctx* ctx, const trg_tensor* x, int cdt, const void* cur, const std::vector<int64_t>& cur_shape,
                 int n, int64_t Kn, uint64_t seed, const ModeOffsets& off, double* dYfull, PreOmega* pre = nullptr,
                 YParts* yp = nullptr, const trg::KrOmega* kr = nullptr) {
    const int N = (int)cur_shape.size();
    trg::SketchPlan p{};
    if (kr) p.kr = *kr;
    p.dtype = cdt;
    p.left = prod(cur_shape, 0, n);
    p.dim = cur_shape[n];
    p.right = prod(cur_shape, n + 1);
    p.K = (int)Kn;
    p.seed = seed;
    p.D = off.D;
    p.rows_glob = off.rows_glob;
    p.col_off = off.col_off;
    const bool sharded_rows = (n == N - 1) && ctx->world > 1;
    double* ylocal = sharded_rows ? (double*)ctx->tmp(sizeof(double) * p.dim * Kn) : dYfull;
    double* partial = nullptr;
    // single rank: the split-K reduction of Y_n moves into the QR launch (one cluster kernel)
    static const bool no_fuse_qr = getenv("TRG_QR_LEGACY") != nullptr;
    const bool defer = yp && ctx->world == 1 && !no_fuse_qr && trg::qr_fused_ok(p.dim, (int)Kn);
    double* yout = defer ? nullptr : ylocal;
    const bool slab2 = p.left > 1 && trg::slab2_ok(p.dtype, p.left, p.dim, Kn, p.right);
    require(!kr || trg::stream_sketch_ok(p.dtype, p.left, p.dim, (int)Kn) || slab2,
            "sketch: the Khatri-Rao test matrix needs the fp64 streaming kernels for mode " + std::to_string(n) +
                " (fp64 working tensor, mode extent <= 128, K <= 16; build_kr)");
    if (trg::stream_sketch_ok(p.dtype, p.left, p.dim, (int)Kn)) {
        partial = (double*)ctx->tmp(sizeof(double) * ctx->num_sms * p.dim * Kn);
        int grid = 0;
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            trg::launch_stream_sketch(p, cur, partial, yout, ctx->num_sms, &grid, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, grid};
    } else if (trg::tc_sketch_f32_ok(p.dtype, p.left, p.dim, (int)Kn, p.right)) {
        const int gc = trg::tc_sketch_f32_grid(p.dim, (int)Kn, p.right, ctx->num_sms);
        partial = (double*)ctx->tmp(sizeof(double) * gc * p.dim * Kn);
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            trg::launch_tc_sketch_f32(p, cur, partial, yout, ctx->num_sms, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, gc};
    } else if (trg::stream_sketch_f32_ok(p.dtype, p.left, p.dim, (int)Kn, p.right)) {
        int gc = 0;
        trg::stream_sketch_f32_grid(p.dim, (int)Kn, p.right, ctx->num_sms, &gc);
        partial = (double*)ctx->tmp(sizeof(double) * gc * p.dim * Kn);
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            gc = trg::launch_stream_sketch_f32(p, cur, partial, yout, ctx->num_sms, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, gc};
    } else if (p.left > 1 && trg::tc_sketch_n_f32_ok(p.dtype, p.left, p.dim, (int)Kn, p.right)) {
        const int gc = trg::tc_sketch_n_f32_parts(p.left, p.dim, (int)Kn, p.right, ctx->num_sms);
        partial = (double*)ctx->tmp(sizeof(double) * gc * p.dim * Kn);
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            trg::launch_tc_sketch_n_f32(p, cur, partial, yout, ctx->num_sms, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, gc};
    } else if (trg::st_sketch_ok(p.dtype, p.left, p.dim, (int)Kn, p.right)) {
        const int gc = trg::st_sketch_grid(p.left, p.dim, (int)Kn, p.right, ctx->num_sms);
        partial = (double*)ctx->tmp(sizeof(double) * gc * p.dim * Kn);
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            trg::launch_st_sketch(p, cur, partial, yout, ctx->num_sms, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, gc};
    } else if (trg::slab_f32_sketch_ok(p.dtype, p.left, p.dim, (int)Kn, p.right)) {
        const int gc = trg::slab_f32_sketch_grid(p.left, p.dim, (int)Kn, p.right, ctx->num_sms);
        partial = (double*)ctx->tmp(sizeof(double) * gc * p.dim * Kn);
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            trg::launch_slab_f32_sketch(p, cur, partial, yout, ctx->num_sms, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, gc};
    } else if (slab2) {
        const int NT = Kn <= 8 ? 1 : 2;
        double* om = nullptr;
        const bool have = pre && pre->buf;
        om = have ? pre->buf : (double*)ctx->tmp(sizeof(double) * trg::slab2_units(p.left, p.right) * 4 * NT * 32);
        if (have && pre->ready && !pre->joined) CK(cudaStreamWaitEvent(ctx->stream, pre->ready, 0));
        if (!have || pre->pending) {  // no earlier launch generated the blocks: do it here
            ctx->launch("omega_m" + std::to_string(n), [&] {
                trg::launch_omega_units(p.left, p.right, (int)Kn, p.seed, p.D, p.col_off, p.rows_glob, om,
                                        ctx->stream, kr);
            });
            if (have) pre->pending = false;
        }
        partial = (double*)ctx->tmp(sizeof(double) * ctx->num_sms * p.dim * Kn);
        int grid = 0;
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            grid = trg::launch_slab2_sketch(p, cur, om, partial, yout, ctx->num_sms, ctx->stream);
        }, yout ? 2 : 1);
        if (defer) *yp = YParts{partial, grid};
        if (!(pre && pre->buf)) ctx->tmp_free(om);  // pre-generated blocks live in the arena
        if (pre) pre->buf = nullptr;
    } else if (trg::slab_sketch_ok(p.dtype, p.left, p.dim, (int)Kn, p.left * p.right)) {
        partial = (double*)ctx->tmp(sizeof(double) * ctx->num_sms * p.dim * Kn);
        ctx->launch("sketch_m" + std::to_string(n), [&] {
            trg::launch_slab_sketch(p, cur, partial, ylocal, ctx->num_sms, ctx->stream);
        }, 2);
    } else {
        trg::plan_sketch(p, ctx->num_sms);
        partial = (double*)ctx->tmp(p.partial_elems * sizeof(double));
        ctx->launch("sketch_m" + std::to_string(n), [&] { trg::launch_sketch(p, cur, partial, ylocal, ctx->stream); },
                    2);
    }
    if (!defer) ctx->tmp_free(partial);  // else freed after the QR launch reduced it
    if (sharded_rows) {
        ctx->launch("scatter", [&] {
            trg::launch_scatter_rows(ylocal, p.dim, (int)Kn, x->lo, x->dims[n], dYfull, ctx->stream);
        });
        ctx->tmp_free(ylocal);
    }
    ctx->allreduce(dYfull, (size_t)(x->dims[n] * Kn), F64);
}

// fp32 inputs keep fp32 intermediates (the later modes run the fp32 slab kernels, slab_f32.cu);
// TRG_PROMOTE_F64=1 restores the former fp64 P^(1) (development comparison)
bool mode0_promotes(int dt, int64_t left, int64_t dim, int64_t K, int64_t right) {
    static const bool promote = getenv("TRG_PROMOTE_F64") != nullptr;
    return promote && (trg::tc_ttm_f32_ok(dt, left, dim, K, right) || trg::stream_ttm_f32_ok(dt, left, dim, K, right));
}

// out = cur x_n Q^T (local rows of Q for the sharded last mode), new buffer.
// out = cur x_n Q^T; *odt is the output dtype (fp32 mode-0 input is promoted to fp64 by its shrink)
void* shrink_mode(trg_ctx* ctx, const trg_tensor* x, int cdt, const void* cur, const std::vector<int64_t>& cur_shape,
                  int n, int64_t Kn, const double* dQ, int* odt, bool escape = true, bool chain = false) {
    const int N = (int)cur_shape.size();
    trg::TTMPlan p{};
    static const int spare = getenv("TRG_TTM_SPARE") ? atoi(getenv("TRG_TTM_SPARE")) : 0;
    static const bool late = getenv("TRG_QR_LATE") != nullptr;
    p.chain = chain && !late;
    p.spare_sms = spare;
    p.dtype = cdt;
    p.left = prod(cur_shape, 0, n);
    p.dim = cur_shape[n];
    p.right = prod(cur_shape, n + 1);
    p.odim = Kn;
    p.m_so = x->dims[n];  // M(o=k, d) = Q[d + I_n*k]
    p.m_sd = 1;
    const double* m = dQ;
    if (n == N - 1) m += x->lo;  // local rows of Q_{N-1}
    const bool tc = trg::tc_ttm_f32_ok(p.dtype, p.left, p.dim, Kn, p.right);
    const bool f32s = trg::stream_ttm_f32_ok(p.dtype, p.left, p.dim, Kn, p.right);
    const bool promote = mode0_promotes(p.dtype, p.left, p.dim, Kn, p.right);
    *odt = promote ? F64 : cdt;
    const size_t es = trg::dtype_size(*odt);
    void* out = escape ? ctx->alloc(es * (size_t)(p.left * Kn * p.right)) : ctx->tmp(es * (size_t)(p.left * Kn * p.right));
    if (tc) {
        float* scratch = (float*)ctx->tmp(trg::tc_ttm_f32_scratch(p.dim, Kn));
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_tc_ttm_f32(p, cur, out, *odt == F64, m, x->dims[n], scratch, ctx->num_sms, ctx->stream);
        }, 2);
        ctx->tmp_free(scratch);
    } else if (!promote && p.left > 1 && trg::tc_ttm_n_f32_ok(p.dtype, p.left, p.dim, Kn, p.right)) {
        float* scratch = (float*)ctx->tmp(trg::tc_ttm_n_f32_scratch(p.dim, Kn));
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_tc_ttm_n_f32(p, cur, out, m, x->dims[n], scratch, ctx->num_sms, ctx->stream);
        }, 2);
        ctx->tmp_free(scratch);
    } else if (!promote && trg::st0_shrink_ok(p.dtype, p.left, p.dim, Kn, p.right)) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_st0_shrink(p, cur, out, m, ctx->num_sms, ctx->stream);
        }, 2);
    } else if (f32s) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_stream_ttm_f32(p, cur, out, promote, m, x->dims[n], ctx->num_sms, ctx->stream);
        });
    } else if (trg::st_shrink_ok(p.dtype, p.left, p.dim, Kn, p.right)) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_st_shrink(p, cur, out, m, ctx->num_sms, ctx->stream);
        }, 2);
    } else if (trg::slab_f32_ttm_ok(p.dtype, p.left, p.dim, Kn, p.right)) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_slab_f32_ttm(p, cur, out, m, ctx->num_sms, ctx->stream);
        });
    } else if (trg::stream_ttm_ok(p.dtype, p.left, p.dim, Kn)) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_stream_ttm(p, cur, out, m, x->dims[n], ctx->num_sms, ctx->stream);
        });
    } else if (p.left > 1 && trg::slab2_ok(p.dtype, p.left, p.dim, Kn, p.right)) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_slab2_ttm(p, cur, out, m, x->dims[n], ctx->num_sms, ctx->stream);
        });
    } else if (trg::slab_ttm_ok(p.dtype, p.left, p.dim, Kn, p.left * p.right)) {
        ctx->launch("ttm_m" + std::to_string(n), [&] {
            trg::launch_slab_ttm(p, cur, out, m, x->dims[n], ctx->num_sms, ctx->stream);
        });
    } else {
        trg::plan_ttm(p, ctx->num_sms);
        ctx->launch("ttm_m" + std::to_string(n), [&] { trg::launch_ttm(p, cur, out, m, ctx->stream); });
    }
    return out;
}

// in_launch: only allocate the blocks and record the jobs; the main stream's QR launches generate
// them on their idle CTAs (launch_qr_fused), or the sketch of that mode does if none could
void schedule_pre_omega(trg_ctx* ctx, const trg_tensor* x, int later_dt, const std::vector<int64_t>& K, uint64_t seed,
                        const std::vector<ModeOffsets>& offs, int after, std::vector<PreOmega>& pre,
                        bool in_launch = false, const std::vector<trg::KrOmega>* kr = nullptr) {
    const int N = (int)x->dims.size();
    std::vector<int64_t> shape = x->local_shape();
    for (int m = 0; m <= after; ++m) shape[m] = K[m];
    cudaEvent_t go;
    CK(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
    CK(cudaEventRecord(go, ctx->stream));  // buffers below are allocated on the main stream
    for (int m = after + 1; m < N; ++m) {
        if (offs[m].skipped) continue;
        const int64_t left = prod(shape, 0, m), dim = shape[m], right = prod(shape, m + 1);
        if (left > 1 && trg::slab2_ok(later_dt, left, dim, K[m], right)) {
            const int NT = K[m] <= 8 ? 1 : 2;
            pre[m].buf = (double*)ctx->tmp(sizeof(double) * trg::slab2_units(left, right) * 4 * NT * 32);
            if (in_launch) {
                pre[m].job = trg::omega_units_job(left, right, (int)K[m], seed, offs[m].D, offs[m].col_off,
                                                  offs[m].rows_glob, pre[m].buf, kr ? &(*kr)[m] : nullptr);
                pre[m].pending = true;
                shape[m] = K[m];
                continue;
            }
            CK(cudaEventRecord(go, ctx->stream));
            CK(cudaStreamWaitEvent(ctx->side, go, 0));
            trg::launch_omega_units(left, right, (int)K[m], seed, offs[m].D, offs[m].col_off, offs[m].rows_glob,
                                    pre[m].buf, ctx->side, kr ? &(*kr)[m] : nullptr);
            CK(cudaGetLastError());
            ctx->launches += 1;
            CK(cudaEventCreateWithFlags(&pre[m].ready, cudaEventDisableTiming));
            CK(cudaEventRecord(pre[m].ready, ctx->side));
        }
        shape[m] = K[m];
    }
    CK(cudaEventDestroy(go));
}

// ------------------------------------------------------------------ Khatri-Rao test matrices (f4)
// Omega_n(c, k) = prod_{m != n} F_{n,m}(i_m, k) for unfolding column c = sum_{m != n} i_m stride_m
// (first index fastest), F_{n,m} an S_m x K_n block of the stream `seed` (trg.h
// TRG_OMEGA_KHATRI_RAO for the draw order). The kernels take it as A(c mod left) F(r mod S1)
// H(r / S1) with r = c / left (kernels.h KrOmega): A and H are materialised (at most
// prod_{m < n} S_m and prod_{m > n + 1} S_m rows), F is the factor of mode n + 1 itself.
struct KrPlan {
    std::vector<trg::KrOmega> om;  // per mode (F == nullptr for skipped modes)
    std::vector<void*> bufs;       // device buffers, freed stream-ordered after the run
};

KrPlan build_kr(trg_ctx* ctx, const trg_tensor* x, const int64_t* K, uint64_t seed, int variant) {
    const int N = (int)x->dims.size();
    const std::vector<int64_t>& dims = x->dims;
    {  // every projected mode must take a kernel with the Khatri-Rao entries (before any launch)
        std::vector<int64_t> shape = x->local_shape();
        const int cdt = x->dtype;
        for (int n = 0; n < N; ++n) {
            if (K[n] == dims[n]) continue;
            const int64_t left = prod(shape, 0, n), dim = shape[n], right = prod(shape, n + 1);
            require(trg::stream_sketch_ok(cdt, left, dim, (int)K[n]) ||
                        (left > 1 && trg::slab2_ok(cdt, left, dim, K[n], right)),
                    "sketch: the Khatri-Rao test matrix needs the fp64 streaming kernels for mode " +
                        std::to_string(n) + " (fp64 tensor, mode extent <= 128, K_n <= 16)");
            if (variant == TRG_SEQUENTIAL) shape[n] = K[n];
        }
    }
    KrPlan kp;
    kp.om.resize(N);
    std::vector<std::vector<int64_t>> S(N), off(N);
    int64_t total = 0;
    for (int n = 0; n < N; ++n) {
        if (K[n] == dims[n]) continue;
        S[n].resize(N);
        off[n].assign(N, -1);
        for (int m = 0; m < N; ++m) S[n][m] = (m < n && variant == TRG_SEQUENTIAL) ? K[m] : dims[m];
        for (int m = 0; m < N; ++m)
            if (m != n) {
                off[n][m] = total;
                total += S[n][m] * K[n];
            }
    }
    if (total == 0) return kp;
    // the factor draws (one launch), then every table of every mode (one launch)
    std::vector<trg::KrTable> tabs;
    // table layout first (element offsets into one buffer after the draws), pointers after the
    // single allocation
    struct Slot {
        int64_t a, f, h;  // element offsets of A, F, H
    };
    std::vector<Slot> slot(N);
    int64_t elems = 0;
    for (int n = 0; n < N; ++n) {
        if (K[n] == dims[n]) continue;
        // Khatri-Rao product of the factors of modes [m0, m1) other than n; returns its offset
        auto table = [&](int m0, int m1, int64_t* nrows) {
            trg::KrTable t{};
            t.K = (int)K[n];
            t.nrows = 1;
            for (int m = m0; m < m1; ++m)
                if (m != n) {
                    require(t.nf < trg::kKrMaxFactors, "sketch: Khatri-Rao supports tensors of order <= 8");
                    t.off[t.nf] = off[n][m];
                    t.rows[t.nf++] = S[n][m];
                    t.nrows *= S[n][m];
                }
            tabs.push_back(t);
            *nrows = t.nrows;
            const int64_t at = elems;
            elems += t.nrows * t.K;
            return at;
        };
        trg::KrOmega& o = kp.om[n];
        slot[n].a = table(0, n, &o.left);
        if (n + 1 < N) {
            slot[n].f = table(n + 1, n + 2, &o.S1);
            slot[n].h = table(n + 2, N, &o.nH);
        } else {
            slot[n].f = slot[n].h = table(N, N, &o.nH);  // one row of ones
            o.S1 = 1;
        }
        require(o.S1 * o.nH < (int64_t(1) << 32), "sketch: Khatri-Rao row index beyond 32 bits");
    }
    double* draws = (double*)ctx->alloc(sizeof(double) * (total + elems));
    double* base = draws + total;
    kp.bufs.push_back(draws);
    trg::launch_omega(seed, 0, total, 1, draws, ctx->stream);
    for (size_t i = 0, at = 0; i < tabs.size(); ++i) {
        tabs[i].out = base + at;
        at += (size_t)(tabs[i].nrows * tabs[i].K);
    }
    for (int n = 0; n < N; ++n)
        if (K[n] != dims[n]) {
            kp.om[n].A = base + slot[n].a;
            kp.om[n].F = base + slot[n].f;
            kp.om[n].H = base + slot[n].h;
        }
    trg::launch_kr_tables(draws, tabs.data(), (int)tabs.size(), ctx->stream);
    ctx->launches += 2;
    return kp;
}

void run_sketch(trg_ctx* ctx, const trg_tensor* x, const int64_t* Kin, uint64_t seed, int variant, trg_sketch* sk) {
    const int N = (int)x->dims.size();
    validate_K(x, Kin);
    const bool kr_on = (variant & TRG_OMEGA_KHATRI_RAO) != 0;
    variant &= ~TRG_OMEGA_KHATRI_RAO;
    require(variant == TRG_SEQUENTIAL || variant == TRG_FUSED, "sketch: unknown variant");
    sk->ctx = ctx;
    sk->dtype = x->dtype;
    sk->variant = variant;
    sk->dims = x->dims;
    sk->K.assign(Kin, Kin + N);
    sk->dQ.assign(N, nullptr);
    sk->dY.assign(N, nullptr);
    if (!sk->ev0) CK(cudaEventCreate(&sk->ev0));
    if (!sk->ev1) CK(cudaEventCreate(&sk->ev1));
    CK(cudaEventRecord(sk->ev0, ctx->stream));
    // QR path flags, written by every QR launch (skipped modes have none: trg_sketch_qr_path
    // answers 0 for them without reading the device)
    sk->dflags = (int*)ctx->alloc(sizeof(int) * N);
    int* tickets = ctx->ensure_tickets(N);
    const KrPlan krp = kr_on ? build_kr(ctx, x, Kin, seed, variant) : KrPlan{};
    auto krn = [&](int n) { return kr_on ? &krp.om[n] : nullptr; };
    ctx->scr_begin();

    int cdt = x->dtype;  // dtype of the working tensor (fp32 input is promoted by its mode-0 shrink)
    std::vector<int64_t> shape = x->local_shape();
    const void* cur = x->d;
    void* owned = nullptr;      // buffer owned by the pipeline (not x)
    bool owned_arena = false;   // ... and whether it lives in the scratch arena
    const std::vector<ModeOffsets> offs = sketch_offsets(x->dims, Kin, x->lo, variant);
    int last_proj = -1, first_proj = -1;
    for (int n = 0; n < N; ++n)
        if (sk->K[n] != x->dims[n]) {
            last_proj = n;
            if (first_proj < 0) first_proj = n;
            // escaping outputs first, so no allocator call sits between the chain's kernels
            sk->dY[n] = (double*)ctx->alloc(sizeof(double) * x->dims[n] * sk->K[n]);
            sk->dQ[n] = (double*)ctx->alloc(sizeof(double) * x->dims[n] * sk->K[n]);
        }
    auto release_owned = [&]() {
        if (owned && !owned_arena) ctx->dfree(owned);
    };

    std::vector<YParts> yparts(N);
    std::vector<PreOmega> pre(N);
    auto qr = [&](int n) {
        const int64_t In = x->dims[n], Kn = sk->K[n];
        double* work = (double*)ctx->tmp(sizeof(double) * In * Kn);
        if (yparts[n].partial) {
            // the launch's CTAs past the reduce generate the next pending test matrix
            const trg::OmegaUnitsJob* job = nullptr;
            for (int m = n + 1; m < N && !job && yparts[n].nparts > 1; ++m)  // runs iff ticketed
                if (pre[m].pending) {
                    job = &pre[m].job;
                    pre[m].pending = false;
                }
            ctx->launch("qr", [&] {
                trg::launch_qr_fused(yparts[n].partial, yparts[n].nparts, In, (int)Kn, sk->dY[n], sk->dQ[n], work,
                                     sk->dflags + n, tickets + n, ctx->stream, job, ctx->num_sms);
            });
            ctx->tmp_free(yparts[n].partial);
            yparts[n] = YParts{};
        } else {
            ctx->launch("qr", [&] { trg::launch_qr(sk->dY[n], In, (int)Kn, sk->dQ[n], work, sk->dflags + n, ctx->stream); });
        }
        ctx->tmp_free(work);
    };

    bool pre_started = false;
    if (variant == TRG_SEQUENTIAL) {
        for (int n = 0; n < N; ++n) {
            const int64_t Kn = sk->K[n];
            if (Kn == x->dims[n]) continue;  // identity basis, no draws (sketch.hpp:76-79)
            sketch_mode(ctx, x, cdt, cur, shape, n, Kn, seed, offs[n], sk->dY[n], &pre[n], &yparts[n], krn(n));
            static const bool side_omega = getenv("TRG_SIDE_OMEGA") != nullptr;
            if (!pre_started && yparts[n].partial && !side_omega) {
                // ticketed QR launches: their CTAs past the reduce generate the later test
                // matrices (one mode per launch), in the latency-bound QR instead of next to the
                // HBM-bound shrink
                pre_started = true;
                const bool promotes = mode0_promotes(cdt, prod(shape, 0, n), shape[n], Kn, prod(shape, n + 1));
                schedule_pre_omega(ctx, x, promotes ? (int)F64 : cdt, sk->K, seed, offs, n, pre, true,
                                   kr_on ? &krp.om : nullptr);
            }
            qr(n);
            if (!pre_started) {
                // Omega_m of every later slab-kernel mode depends only on shapes and the seed:
                // generate them on the side stream once this mode's QR is done, next to its
                // shrink (HBM-bound, one CTA per SM with room to spare), not next to the QR or
                // the sketch, which it would slow down
                pre_started = true;
                const bool promotes = mode0_promotes(cdt, prod(shape, 0, n), shape[n], Kn, prod(shape, n + 1));
                schedule_pre_omega(ctx, x, promotes ? (int)F64 : cdt, sk->K, seed, offs, n, pre, false,
                                   kr_on ? &krp.om : nullptr);
            }
            const bool join_after_shrink = n == first_proj;
            const bool escape = n == last_proj;  // the last shrink writes P itself
            int odt = cdt;
            void* out = shrink_mode(ctx, x, cdt, cur, shape, n, Kn, sk->dQ[n], &odt, escape, /*chain=*/true);
            cdt = odt;
            release_owned();
            owned = out;
            owned_arena = !escape;
            if (join_after_shrink) {
                // join the side stream once, here, rather than before every later sketch: each
                // cross-stream wait cuts a programmatic-dependent-launch edge of the chain
                for (auto& po : pre)
                    if (po.ready) {
                        CK(cudaStreamWaitEvent(ctx->stream, po.ready, 0));
                        po.joined = true;
                    }
            }
            if (n == N - 1) ctx->allreduce(out, (size_t)(prod(shape, 0, n) * Kn), cdt);
            cur = out;
            shape[n] = Kn;
        }
    } else {
        // all Y_n from the original X, Omega_n sized against X,
        // one stream in mode order; then the shrink chain.
        std::vector<int64_t> xshape = x->local_shape();
        for (int n = 0; n < N; ++n) {
            const int64_t Kn = sk->K[n];
            if (Kn == x->dims[n]) continue;
            sketch_mode(ctx, x, x->dtype, x->d, xshape, n, Kn, seed, offs[n], sk->dY[n], nullptr, &yparts[n], krn(n));
            qr(n);
        }
        for (int n = 0; n < N; ++n) {
            const int64_t Kn = sk->K[n];
            if (Kn == x->dims[n]) continue;
            int odt = cdt;
            const bool escape = n == last_proj;
            void* out = shrink_mode(ctx, x, cdt, cur, shape, n, Kn, sk->dQ[n], &odt, escape);
            cdt = odt;
            if (n == N - 1) ctx->allreduce(out, (size_t)(prod(shape, 0, n) * Kn), cdt);
            release_owned();
            owned = out;
            owned_arena = !escape;
            cur = out;
            shape[n] = Kn;
        }
    }
    const bool last_projected = sk->K[N - 1] != x->dims[N - 1];
    if (ctx->world > 1 && !last_projected) {
        // P still sharded along the last mode: zero-padded gather by allreduce
        const size_t es = trg::dtype_size(cdt);
        const int64_t inner = prod(shape, 0, N - 1);
        const int64_t full = inner * x->dims[N - 1];
        void* g = ctx->alloc(es * full);
        CK(cudaMemsetAsync(g, 0, es * full, ctx->stream));
        CK(cudaMemcpyAsync((char*)g + es * inner * x->lo, cur, es * inner * (x->hi - x->lo), cudaMemcpyDeviceToDevice,
                           ctx->stream));
        ctx->allreduce(g, (size_t)full, cdt);
        release_owned();
        owned = g;
        owned_arena = false;
        cur = g;
        shape[N - 1] = x->dims[N - 1];
    }
    if (owned && owned_arena) {  // P must outlive the arena (fused path / odd cases): copy it out
        const size_t bytes = trg::dtype_size(cdt) * (size_t)prod(shape);
        void* p2 = ctx->alloc(bytes);
        CK(cudaMemcpyAsync(p2, owned, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
        owned = p2;
        owned_arena = false;
        cur = p2;
    }
    sk->P_elems = prod(shape);
    sk->dtype = cdt;  // P's dtype (fp64 once an fp32 input has been promoted)
    if (owned) {
        sk->dP = owned;
        sk->P_is_view = false;
    } else {
        sk->dP = const_cast<void*>(cur);  // no mode projected: P is x itself (sketch.hpp:71)
        sk->P_is_view = true;
    }
    for (auto& po : pre)
        if (po.ready) cudaEventDestroy(po.ready);  // destruction is deferred until the event completes
    for (void* b : krp.bufs) ctx->dfree(b);  // stream-ordered: after the last kernel that reads them
    ctx->scr_end();
    CK(cudaEventRecord(sk->ev1, ctx->stream));
}

void download_P(const trg_sketch* sk, std::vector<double>& out) {
    trg_ctx* ctx = sk->ctx;
    out.resize((size_t)sk->P_elems);
    if (sk->dtype == F64) {
        CK(cudaMemcpyAsync(out.data(), sk->dP, sizeof(double) * sk->P_elems, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
        std::vector<float> tmp((size_t)sk->P_elems);
        CK(cudaMemcpyAsync(tmp.data(), sk->dP, sizeof(float) * sk->P_elems, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (size_t i = 0; i < tmp.size(); ++i) out[i] = tmp[i];
    }
    CK(cudaStreamSynchronize(ctx->stream));
}

void download_basis(const trg_sketch* sk, int n, double* out) {
    const int64_t In = sk->dims[n], Kn = sk->K[n];
    if (!sk->dQ[n]) {
        for (int64_t j = 0; j < Kn; ++j)
            for (int64_t i = 0; i < In; ++i) out[i + In * j] = (i == j) ? 1.0 : 0.0;
        return;
    }
    CK(cudaMemcpyAsync(out, sk->dQ[n], sizeof(double) * In * Kn, cudaMemcpyDeviceToHost, sk->ctx->stream));
    CK(cudaStreamSynchronize(sk->ctx->stream));
}

// ------------------------------------------------------------------ TR model on device
// cores (flat) -> per-core host vectors
std::vector<std::vector<double>> split_cores(int N, const int64_t* dims, const int64_t* ranks, const double* cores) {
    std::vector<std::vector<double>> out;
    const double* p = cores;
    for (int n = 0; n < N; ++n) {
        const int64_t sz = ranks[n] * dims[n] * ranks[(n + 1) % N];
        out.emplace_back(p, p + sz);
        p += sz;
    }
    return out;
}

// Subchain S = G_1 o ... o G_{N-1} over the local slab [lo, hi) of the last mode,
// shape (R_1, P_local, R_0), on device. Caller frees.
double* device_subchain(trg_ctx* ctx, int N, const int64_t* dims, const int64_t* ranks,
                        const std::vector<std::vector<double>>& cs, int64_t lo, int64_t hi, int64_t& P_local) {
    auto upload = [&](const std::vector<double>& v) {
        double* d = (double*)ctx->alloc(sizeof(double) * v.size());
        CK(cudaMemcpyAsync(d, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, ctx->stream));
        return d;
    };
    auto last_slab = [&](int n) {
        // core n restricted to middle indices [lo, hi): (R, hi-lo, R')
        const int64_t r = ranks[n], I = dims[n], rp = ranks[(n + 1) % N];
        std::vector<double> v((size_t)(r * (hi - lo) * rp));
        for (int64_t s = 0; s < rp; ++s)
            for (int64_t i = lo; i < hi; ++i)
                for (int64_t a = 0; a < r; ++a) v[a + r * ((i - lo) + (hi - lo) * s)] = cs[n][a + r * (i + I * s)];
        return v;
    };
    auto core_host = [&](int n) { return n == N - 1 ? last_slab(n) : cs[n]; };
    auto mid = [&](int n) { return n == N - 1 ? hi - lo : dims[n]; };
    double* cur = upload(core_host(1));
    int64_t ra = ranks[1], p = mid(1), rb = ranks[2 % N];
    for (int k = 2; k < N; ++k) {
        const std::vector<double> gh = core_host(k);
        double* g = upload(gh);
        const int64_t i = mid(k), rc = ranks[(k + 1) % N];
        double* out = (double*)ctx->alloc(sizeof(double) * ra * p * i * rc);
        ctx->launch("chain", [&] { trg::launch_chain(cur, ra, p, rb, g, i, rc, out, ctx->stream); });
        ctx->dfree(cur);
        ctx->dfree(g);
        cur = out;
        p *= i;
        rb = rc;
    }
    P_local = p;
    return cur;
}

// Reconstruct (write_mode = 1: X := Xhat) or accumulate the RSE sums over the local slab (0; 2: in fp64
// arithmetic also for fp32 tensors).
void device_recon(trg_ctx* ctx, trg_tensor* x, const int64_t* ranks, const double* cores, int write_mode,
                  double* host_sums) {
    const int N = (int)x->dims.size();
    require(N >= 2, "device reconstruction needs order >= 2");
    const auto cs = split_cores(N, x->dims.data(), ranks, cores);
    int64_t P_local = 0;
    double* S = device_subchain(ctx, N, x->dims.data(), ranks, cs, x->lo, x->hi, P_local);
    double* g0 = (double*)ctx->alloc(sizeof(double) * cs[0].size());
    CK(cudaMemcpyAsync(g0, cs[0].data(), sizeof(double) * cs[0].size(), cudaMemcpyHostToDevice, ctx->stream));
    trg::ReconPlan rp{};
    rp.dtype = x->dtype;
    rp.I0 = x->dims[0];
    rp.P = P_local;
    rp.R0 = ranks[0];
    rp.R1 = ranks[1 % N];
    rp.write_mode = write_mode;
    trg::plan_recon(rp, ctx->num_sms);
    const bool synth = write_mode == 1;
    double* bs = synth ? nullptr : (double*)ctx->alloc(sizeof(double) * 2 * rp.nblocks);
    ctx->launch(synth ? "synth" : "rse", [&] { trg::launch_recon(rp, g0, S, x->d, synth ? 1 : 0, bs, ctx->stream); });
    if (!synth) {
        double* sums = (double*)ctx->alloc(sizeof(double) * 2);
        ctx->launch("rse_sum", [&] { trg::launch_sum_pairs(bs, rp.nblocks, sums, ctx->stream); });
        ctx->allreduce(sums, 2, F64);
        CK(cudaMemcpyAsync(host_sums, sums, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->dfree(sums);
        ctx->dfree(bs);
    }
    ctx->dfree(S);
    ctx->dfree(g0);
}

double rse_device(trg_ctx* ctx, const trg_tensor* x, const int64_t* ranks, const double* cores) {
    const int N = (int)x->dims.size();
    for (int n = 0; n < N; ++n) require(ranks[n] >= 1, "rse: ranks must be positive");
    if (N == 1) {
        // X(i) = trace(G(:, i, :)) — order-one tensors are tiny: host evaluation
        std::vector<double> xh((size_t)x->local_elems);
        trg_tensor_download(x, xh.data());
        const int64_t r = ranks[0], I = x->dims[0];
        double num = 0.0, den = 0.0;
        for (int64_t i = 0; i < I; ++i) {
            double tr = 0.0;
            for (int64_t a = 0; a < r; ++a) tr += cores[a + r * (i + I * a)];
            num += (xh[i] - tr) * (xh[i] - tr);
            den += xh[i] * xh[i];
        }
        require(den > 0.0, "rse: reference tensor has zero norm");
        return std::sqrt(num) / std::sqrt(den);
    }
    double sums[2];
    device_recon(ctx, const_cast<trg_tensor*>(x), ranks, cores, 0, sums);
    require(sums[1] > 0.0, "rse: reference tensor has zero norm");
    double r = std::sqrt(sums[0]) / std::sqrt(sums[1]);
    // fp32 tensors take the FFMA GEMM (Xhat to ~1e-6 relative). Below an RSE of 1e-2 that error could
    // reach the 1e-4 fp32 tolerance of the result, so such fits are re-measured with fp64 arithmetic.
    if (x->dtype == F32 && r < 1e-2) {
        device_recon(ctx, const_cast<trg_tensor*>(x), ranks, cores, 2, sums);
        r = std::sqrt(sums[0]) / std::sqrt(sums[1]);
    }
    return r;
}

void back_project_device(trg_ctx* ctx, int N, const int64_t* K, const int64_t* ranks, const double* small,
                         const trg_sketch* sk, double* out) {
    require((int)sk->dims.size() == N, "back_project: need one basis per core");
    const double* zp = small;
    double* op = out;
    for (int n = 0; n < N; ++n) {
        require(K[n] == sk->K[n], "back_project: basis/core dimension mismatch in mode " + std::to_string(n));
        const int64_t r = ranks[n], rn = ranks[(n + 1) % N], In = sk->dims[n];
        const int64_t zsz = r * K[n] * rn, osz = r * In * rn;
        if (!sk->dQ[n]) {  // identity basis: bit-exact copy (sketch.hpp:115-118)
            std::memcpy(op, zp, sizeof(double) * zsz);
        } else {
            double* dz = (double*)ctx->alloc(sizeof(double) * zsz);
            double* dg = (double*)ctx->alloc(sizeof(double) * osz);
            CK(cudaMemcpyAsync(dz, zp, sizeof(double) * zsz, cudaMemcpyHostToDevice, ctx->stream));
            trg::TTMPlan p{};
            p.dtype = F64;
            p.left = r;
            p.dim = K[n];
            p.right = rn;
            p.odim = In;
            p.m_so = 1;  // M(o=i, d=k) = Q[i + I_n*k]
            p.m_sd = In;
            trg::plan_ttm(p, ctx->num_sms);
            ctx->launch("back_project", [&] { trg::launch_ttm(p, dz, dg, sk->dQ[n], ctx->stream); });
            CK(cudaMemcpyAsync(op, dg, sizeof(double) * osz, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            ctx->dfree(dz);
            ctx->dfree(dg);
        }
        zp += zsz;
        op += osz;
    }
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void decompose_impl(trg_ctx* ctx, const trg_tensor* x, int method, const int64_t* ranks, double tol,
                    int64_t max_sweeps, uint64_t cfg_seed, const int64_t* K, uint64_t spec_seed, int variant,
                    trg_report* rep, double t_start) {
    const int N = (int)x->dims.size();
    require(method == TRG_ALS || method == TRG_SVD, "decompose: unknown method");
    validate_K(x, K);  // validated before the rank warning (reference quirk sketch.hpp:131-138 fixed)
    const char* who = method == TRG_ALS ? "rtrals" : "rtrsvd";
    if (method == TRG_ALS) {
        require(ranks != nullptr, "trals: rank vector required");
        for (int n = 0; n < N; ++n) require(ranks[n] >= 1, "trals: ranks must be positive");
        require(max_sweeps >= 1, "trals: max_sweeps must be positive");
    } else {
        require(tol >= 0.0, "trsvd: tolerance must be nonnegative");
    }
    if (ranks && ctx->rank == 0)
        for (int n = 0; n < N; ++n)
            if (ranks[n] > K[n])
                std::cerr << who << ": warning: rank " << ranks[n] << " exceeds projection size " << K[n]
                          << " in mode " << n << "\n";
    double t0 = now_ms();
    trg_sketch sk;
    run_sketch(ctx, x, K, spec_seed, variant, &sk);
    trg::host::Tensor P;
    P.shape.assign(K, K + N);
    download_P(&sk, P.data);
    double t1 = now_ms();
    rep->ms[1] = t1 - t0;
    rep->projected = P.data;
    trg::host::SolveOut inner;
    if (method == TRG_ALS)
        inner = trg::host::trals(P, std::vector<int64_t>(ranks, ranks + N), tol, max_sweeps, cfg_seed);
    else
        inner = trg::host::trsvd(P, tol);
    double t2 = now_ms();
    rep->ms[2] = t2 - t1;
    std::vector<int64_t> rk(N);
    std::vector<double> small;
    for (int n = 0; n < N; ++n) {
        rk[n] = inner.cores.rank(n);
        const auto& g = inner.cores.g[n].data;
        small.insert(small.end(), g.begin(), g.end());
    }
    int64_t total = 0;
    for (int n = 0; n < N; ++n) total += rk[n] * x->dims[n] * rk[(n + 1) % N];
    rep->cores.assign((size_t)total, 0.0);
    back_project_device(ctx, N, K, rk.data(), small.data(), &sk, rep->cores.data());
    double t3 = now_ms();
    rep->ms[3] = t3 - t2;
    rep->rse_history = inner.rse_history;
    rep->rse_history.push_back(rse_device(ctx, x, rk.data(), rep->cores.data()));
    double t4 = now_ms();
    rep->ms[4] = t4 - t3;
    rep->ranks = rk;
    rep->sweeps = inner.sweeps_run;
    rep->ms[5] = t4 - t_start;
}

trg_tensor* tensor_new(trg_ctx* ctx, int dtype, int order, const int64_t* dims) {
    require(ctx != nullptr, "tensor: null context");
    require(dtype == F32 || dtype == F64, "tensor: dtype must be TRG_F32 or TRG_F64");
    require(order >= 1, "DenseTensor: order must be at least 1");
    for (int n = 0; n < order; ++n) require(dims[n] >= 1, "DenseTensor: every extent must be positive");
    auto t = std::make_unique<trg_tensor>();
    t->ctx = ctx;
    t->dtype = dtype;
    t->dims.assign(dims, dims + order);
    shard(t->dims.back(), ctx->rank, ctx->world, t->lo, t->hi);
    require(t->hi > t->lo, "tensor: last mode extent smaller than the number of ranks");
    t->local_elems = t->inner() * (t->hi - t->lo);
    CK(cudaSetDevice(ctx->device));
    // from the context's stream-ordered pool (release threshold: keep), so repeated
    // create/destroy (trg_decompose_host per call) costs no driver allocation or implicit sync
    CK(cudaMallocFromPoolAsync(&t->d, trg::dtype_size(dtype) * (size_t)t->local_elems, ctx->pool, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // usable from any stream on return
    return t.release();
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

int trg_abi_version(void) { return TRG_ABI_VERSION; }
const char* trg_last_error(void) { return g_err.c_str(); }

int trg_device_count(int* count) {
    return guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
        cudaGetLastError();
        *count = n;
    });
}

int trg_sketch_offsets(int order, const int64_t* dims, const int64_t* K, int rank, int world, int variant,
                       int64_t* rows_glob, int64_t* col_off, uint64_t* draw_off) {
    return guard([&] {
        require(order >= 1 && dims && K, "sketch: projection size list must match tensor order");
        std::vector<int64_t> d(dims, dims + order);
        for (int n = 0; n < order; ++n)
            require(K[n] >= 1 && K[n] <= d[n], "sketch: need 1 <= K_n <= I_n in mode " + std::to_string(n));
        require(world >= 1 && rank >= 0 && rank < world, "shard: bad rank/world");
        int64_t lo = 0, hi = 0;
        shard(d.back(), rank, world, lo, hi);
        const auto offs = sketch_offsets(d, K, lo, variant);
        for (int n = 0; n < order; ++n) {
            rows_glob[n] = offs[n].skipped ? 0 : offs[n].rows_glob;
            col_off[n] = offs[n].skipped ? 0 : offs[n].col_off;
            draw_off[n] = offs[n].D;
        }
    });
}

int trg_shard_range(int64_t extent, int rank, int world, int64_t* lo, int64_t* hi) {
    return guard([&] {
        require(world >= 1 && rank >= 0 && rank < world, "shard: bad rank/world");
        require(extent >= 1, "shard: extent must be positive");
        shard(extent, rank, world, *lo, *hi);
    });
}

static void ctx_init(trg_ctx* c, int device) {
    ensure_device();
    CK(cudaSetDevice(device));
    c->device = device;
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) throw nodev_error("libtrg is built for sm_100a (B200); device has compute capability major " +
                                       std::to_string(major));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    // a private pool, so keeping freed memory (no driver call or implicit sync per projection) does
    // not change the process-global default pool other libraries allocate from
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    CK(cudaMemPoolCreate(&c->pool, &props));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
}

int trg_ctx_create(int device, trg_ctx** out) {
    return guard([&] {
        auto c = std::make_unique<trg_ctx>();
        ctx_init(c.get(), device);
        *out = c.release();
    });
}

int trg_nccl_unique_id(unsigned char id[128]) {
    return guard([&] {
        nccl().load();
        ncclUniqueId u;
        nccl().check(nccl().getUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, 128);
    });
}

int trg_ctx_create_dist(int device, int rank, int world, const unsigned char id[128], trg_ctx** out) {
    return guard([&] {
        require(world >= 1 && rank >= 0 && rank < world, "ctx: bad rank/world");
        auto c = std::make_unique<trg_ctx>();
        ctx_init(c.get(), device);
        c->rank = rank;
        c->world = world;
        if (world > 1) {
            nccl().load();
            ncclUniqueId u;
            std::memcpy(u.internal, id, 128);
            nccl().check(nccl().commInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
        }
        *out = c.release();
    });
}

int trg_loopback_create(int world, trg_loopback** out) {
    return guard([&] {
        require(world >= 1 && world <= trg::kMaxLoopbackRanks, "loopback: world must be in [1, 16]");
        auto g = std::make_unique<trg_loopback>();
        g->world = world;
        g->bufs.assign(world, nullptr);
        *out = g.release();
    });
}

int trg_loopback_destroy(trg_loopback* g) {
    return guard([&] { delete g; });
}

int trg_ctx_create_loopback(int device, int rank, trg_loopback* g, trg_ctx** out) {
    return guard([&] {
        require(g != nullptr, "loopback: null group");
        require(rank >= 0 && rank < g->world, "ctx: bad rank/world");
        auto c = std::make_unique<trg_ctx>();
        ctx_init(c.get(), device);
        c->rank = rank;
        c->world = g->world;
        c->lb = g;
        *out = c.release();
    });
}

int trg_ctx_destroy(trg_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        for (auto& p : ctx->pending) {
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        for (auto e : ctx->event_pool) cudaEventDestroy(e);
        if (ctx->comm) nccl().commDestroy(ctx->comm);
        cudaStreamSynchronize(ctx->side);
        if (ctx->scr_base) cudaFreeAsync(ctx->scr_base, ctx->stream);
        if (ctx->tickets) cudaFreeAsync(ctx->tickets, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->side);
        cudaStreamDestroy(ctx->stream);
        // outstanding allocations (tensors not destroyed yet) keep the pool alive until freed
        if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
        delete ctx;
    });
}

int trg_ctx_synchronize(trg_ctx* ctx) { return guard([&] { CK(cudaStreamSynchronize(ctx->stream)); }); }
int trg_ctx_stream(trg_ctx* ctx, void** s) { return guard([&] { *s = (void*)ctx->stream; }); }
int trg_ctx_set_profiling(trg_ctx* ctx, int on) {
    return guard([&] {
        ctx->collect();
        ctx->profiling = on != 0;
    });
}
int trg_ctx_kernel_stats(trg_ctx* ctx, const char* label, double* total_ms, int64_t* launches) {
    return guard([&] {
        ctx->collect();
        double ms = 0.0;
        int64_t n = 0;
        for (auto& kv : ctx->stats)
            if (!label || kv.first == label) {
                ms += kv.second.ms;
                n += kv.second.n;
            }
        if (total_ms) *total_ms = ms;
        if (launches) *launches = n;
    });
}
int trg_ctx_kernel_labels(trg_ctx* ctx, char* buf, int64_t cap) {
    return guard([&] {
        ctx->collect();
        std::string s;
        for (auto& kv : ctx->stats) s += kv.first + "\n";
        require((int64_t)s.size() < cap, "labels: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}
int trg_ctx_launch_count(trg_ctx* ctx, int64_t* n) { return guard([&] { *n = ctx->launches; }); }
int trg_ctx_reset_stats(trg_ctx* ctx) {
    return guard([&] {
        ctx->collect();
        ctx->stats.clear();
        ctx->launches = 0;
    });
}

int trg_tensor_create(trg_ctx* ctx, int dtype, int order, const int64_t* dims, trg_tensor** out) {
    return guard([&] { *out = tensor_new(ctx, dtype, order, dims); });
}

int trg_tensor_info(const trg_tensor* t, int* dtype, int* order, int64_t* dims, int64_t* lo, int64_t* hi) {
    return guard([&] {
        if (dtype) *dtype = t->dtype;
        if (order) *order = (int)t->dims.size();
        if (dims) std::copy(t->dims.begin(), t->dims.end(), dims);
        if (lo) *lo = t->lo;
        if (hi) *hi = t->hi;
    });
}

int trg_tensor_upload(trg_tensor* t, const void* host) {
    return guard([&] {
        CK(cudaMemcpyAsync(t->d, host, trg::dtype_size(t->dtype) * t->local_elems, cudaMemcpyHostToDevice,
                           t->ctx->stream));
        CK(cudaStreamSynchronize(t->ctx->stream));
    });
}

int trg_tensor_download(const trg_tensor* t, void* host) {
    return guard([&] {
        CK(cudaMemcpyAsync(host, t->d, trg::dtype_size(t->dtype) * t->local_elems, cudaMemcpyDeviceToHost,
                           t->ctx->stream));
        CK(cudaStreamSynchronize(t->ctx->stream));
    });
}

int trg_tensor_device_ptr(const trg_tensor* t, void** ptr, int64_t* n) {
    return guard([&] {
        *ptr = t->d;
        if (n) *n = t->local_elems;
    });
}

int trg_tensor_synthesize(trg_tensor* t, const int64_t* ranks, const double* cores, int rescale01, double snr_db,
                          uint64_t noise_seed) {
    return guard([&] {
        trg_ctx* ctx = t->ctx;
        const int N = (int)t->dims.size();
        require(N >= 2, "synthesize: order must be at least 2");
        device_recon(ctx, t, ranks, cores, 1, nullptr);
        const int nb = std::min<int64_t>(1024, (t->local_elems + 255) / 256);
        double* bs = (double*)ctx->alloc(sizeof(double) * 2 * nb);
        double* sums = (double*)ctx->alloc(sizeof(double) * 2);
        double h[2];
        if (rescale01) {
            ctx->launch("minmax", [&] { trg::launch_minmax(t->d, t->dtype, t->local_elems, bs, nb, ctx->stream); });
            std::vector<double> hb(2 * nb);
            CK(cudaMemcpyAsync(hb.data(), bs, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            double lo = 1e308, hi = -1e308;
            for (int i = 0; i < nb; ++i) {
                lo = std::min(lo, hb[2 * i]);
                hi = std::max(hi, hb[2 * i + 1]);
            }
            h[0] = -lo;
            h[1] = hi;
            CK(cudaMemcpyAsync(sums, h, sizeof(double) * 2, cudaMemcpyHostToDevice, ctx->stream));
            ctx->allreduce_op(sums, 2, ncclMax);
            CK(cudaMemcpyAsync(h, sums, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            lo = -h[0];
            hi = h[1];
            if (hi > lo) ctx->launch("affine", [&] {
                trg::launch_affine(t->d, t->dtype, t->local_elems, 1.0 / (hi - lo), -lo / (hi - lo), ctx->stream);
            });
        }
        if (std::isfinite(snr_db)) {
            const uint64_t off = (uint64_t)(t->inner() * t->lo);  // global flat index of the slab
            ctx->launch("noise_norms", [&] {
                trg::launch_noise_norms(t->d, t->dtype, t->local_elems, noise_seed, off, bs, nb, ctx->stream);
            });
            ctx->launch("noise_sum", [&] { trg::launch_sum_pairs(bs, nb, sums, ctx->stream); });
            ctx->allreduce(sums, 2, F64);
            CK(cudaMemcpyAsync(h, sums, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            require(h[0] > 0.0, "add_noise: zero-norm input");
            const double alpha = std::sqrt(h[0]) * std::pow(10.0, -snr_db / 20.0) / std::sqrt(h[1]);
            ctx->launch("add_noise", [&] {
                trg::launch_add_noise(t->d, t->dtype, t->local_elems, noise_seed, off, alpha, ctx->stream);
            });
        }
        ctx->dfree(bs);
        ctx->dfree(sums);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int trg_tensor_destroy(trg_tensor* t) {
    return guard([&] {
        if (!t) return;
        cudaFreeAsync(t->d, t->ctx->stream);  // after the context's work on it; pool-owned memory
        cudaStreamSynchronize(t->ctx->stream);
        delete t;
    });
}

int trg_sketch_run(trg_ctx* ctx, const trg_tensor* x, const int64_t* K, uint64_t seed, int variant,
                   trg_sketch** out) {
    return guard([&] {
        require(ctx && x, "sketch: null argument");
        auto sk = std::make_unique<trg_sketch>();
        run_sketch(ctx, x, K, seed, variant, sk.get());
        *out = sk.release();
    });
}

int trg_sketch_projected(const trg_sketch* sk, double* out) {
    return guard([&] {
        std::vector<double> p;
        download_P(sk, p);
        std::memcpy(out, p.data(), sizeof(double) * p.size());
    });
}

int trg_sketch_basis(const trg_sketch* sk, int mode, double* out) {
    return guard([&] {
        if (mode < 0 || mode >= (int)sk->dims.size())
            throw std::out_of_range("DenseTensor: mode " + std::to_string(mode) + " out of range");
        download_basis(sk, mode, out);
    });
}

int trg_sketch_y(const trg_sketch* sk, int mode, double* out) {
    return guard([&] {
            if (mode < 0 || mode >= (int)sk->dims.size())
            throw std::out_of_range("DenseTensor: mode " + std::to_string(mode) + " out of range");
        const int64_t n = sk->dims[mode] * sk->K[mode];
        if (!sk->dY[mode]) {
            std::fill(out, out + n, 0.0);
            return;
        }
        CK(cudaMemcpyAsync(out, sk->dY[mode], sizeof(double) * n, cudaMemcpyDeviceToHost, sk->ctx->stream));
        CK(cudaStreamSynchronize(sk->ctx->stream));
    });
}

int trg_sketch_qr_path(const trg_sketch* sk, int mode, int* hh) {
    return guard([&] {
            if (mode < 0 || mode >= (int)sk->dims.size()) throw std::out_of_range("mode out of range");
        int v = 0;
        if (sk->K[mode] == sk->dims[mode]) {  // identity basis: no QR ran (sketch.hpp:76-79)
            *hh = 0;
            return;
        }
        CK(cudaMemcpyAsync(&v, sk->dflags + mode, sizeof(int), cudaMemcpyDeviceToHost, sk->ctx->stream));
        CK(cudaStreamSynchronize(sk->ctx->stream));
        *hh = v;
    });
}

int trg_sketch_elapsed_ms(const trg_sketch* sk, double* ms) {
    return guard([&] {
        CK(cudaEventSynchronize(sk->ev1));
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, sk->ev0, sk->ev1));
        *ms = f;
    });
}

int trg_sketch_destroy(trg_sketch* sk) {
    return guard([&] { delete sk; });
}

int trg_thin_qr(trg_ctx* ctx, int64_t m, int64_t k, const double* y, double* q, int* householder) {
    return guard([&] {
        require(ctx && y && q, "economy_q: null argument");
        require(m >= 1 && k >= 1 && k <= m, "economy_q: need 1 <= k <= m");
        double* d = (double*)ctx->alloc(sizeof(double) * (size_t)(3 * m * k) + sizeof(int) * 2);
        double* dy = d;
        double* dq = d + m * k;
        double* work = d + 2 * m * k;
        int* flag = (int*)(d + 3 * m * k);
        CK(cudaMemcpyAsync(dy, y, sizeof(double) * m * k, cudaMemcpyHostToDevice, ctx->stream));
        ctx->launch("qr", [&] { trg::launch_qr(dy, m, (int)k, dq, work, flag, ctx->stream); });
        int hh = 0;
        CK(cudaMemcpyAsync(q, dq, sizeof(double) * m * k, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&hh, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->dfree(d);
        if (householder) *householder = hh;
    });
}

int trg_omega(trg_ctx* ctx, uint64_t seed, uint64_t offset, int64_t rows, int64_t cols, double* out) {
    return guard([&] {
        require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be positive");
        double* d = (double*)ctx->alloc(sizeof(double) * rows * cols);
        ctx->launch("omega", [&] { trg::launch_omega(seed, offset, rows, cols, d, ctx->stream); });
        CK(cudaMemcpyAsync(out, d, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->dfree(d);
    });
}

int trg_mode_n_product(trg_ctx* ctx, const trg_tensor* x, int mode, int64_t m_rows, const double* m,
                       trg_tensor** out) {
    return guard([&] {
        const int N = (int)x->dims.size();
        if (mode < 0 || mode >= N) throw std::out_of_range("DenseTensor: mode " + std::to_string(mode) + " out of range");
        require(ctx->world == 1, "mode_n_product: unsharded tensors only");
        require(m_rows >= 1, "mode_n_product: inner dimensions do not match");
        std::vector<int64_t> od = x->dims;
        od[mode] = m_rows;
        trg_tensor* o = tensor_new(ctx, x->dtype, N, od.data());
        const int64_t In = x->dims[mode];
        double* dm = (double*)ctx->alloc(sizeof(double) * m_rows * In);
        CK(cudaMemcpyAsync(dm, m, sizeof(double) * m_rows * In, cudaMemcpyHostToDevice, ctx->stream));
        trg::TTMPlan p{};
        p.dtype = x->dtype;
        p.left = prod(x->dims, 0, mode);
        p.dim = In;
        p.right = prod(x->dims, mode + 1);
        p.odim = m_rows;
        p.m_so = 1;  // M(o, d) = m[o + m_rows*d]
        p.m_sd = m_rows;
        trg::plan_ttm(p, ctx->num_sms);
        ctx->launch("ttm", [&] { trg::launch_ttm(p, x->d, o->d, dm, ctx->stream); });
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->dfree(dm);
        *out = o;
    });
}

// lift_back (sketch.hpp:93-101): t = P x_0 Q_0 x_1 Q_1 ... on the device, skipping exact
// identity bases (q == nullptr). P is (dtype) with extents K; the result has extents dims.
static trg_tensor* lift_back_device(trg_ctx* ctx, int dtype, const std::vector<int64_t>& dims, const std::vector<int64_t>& K,
                             const void* P, const std::vector<const double*>& q) {
    require(ctx->world == 1, "lift_back: unsharded tensors only");
    const int N = (int)dims.size();
    std::vector<int64_t> cur = K;
    trg_tensor* out = tensor_new(ctx, dtype, N, dims.data());
    const size_t es = trg::dtype_size(dtype);
    int last = -1;
    for (int n = 0; n < N; ++n)
        if (q[n]) last = n;
    if (last < 0) {  // every basis is the identity: t = P
        CK(cudaMemcpyAsync(out->d, P, es * (size_t)prod(K), cudaMemcpyDeviceToDevice, ctx->stream));
        return out;
    }
    const void* src = P;
    void* owned = nullptr;
    for (int n = 0; n <= last; ++n) {
        if (!q[n]) continue;
        std::vector<int64_t> nxt = cur;
        nxt[n] = dims[n];
        void* dst = n == last ? out->d : ctx->alloc(es * (size_t)prod(nxt));
        trg::TTMPlan p{};
        p.dtype = dtype;
        p.left = prod(cur, 0, n);
        p.dim = cur[n];
        p.right = prod(cur, n + 1);
        p.odim = dims[n];
        p.m_so = 1;        // M(o = i, d = k) = Q_n[i + I_n k]
        p.m_sd = dims[n];
        trg::plan_ttm(p, ctx->num_sms);
        ctx->launch("lift_back", [&] { trg::launch_ttm(p, src, dst, q[n], ctx->stream); });
        if (owned) ctx->dfree(owned);
        owned = n == last ? nullptr : dst;
        src = dst;
        cur = nxt;
    }
    return out;
}

int trg_sketch_lift_back(const trg_sketch* csk, trg_tensor** out) {
    return guard([&] {
        const trg_sketch* sk = csk;
        std::vector<const double*> q(sk->dims.size());
        for (size_t n = 0; n < q.size(); ++n) q[n] = sk->K[n] == sk->dims[n] ? nullptr : sk->dQ[n];
        *out = lift_back_device(sk->ctx, sk->dtype, sk->dims, sk->K, sk->dP, q);
        CK(cudaStreamSynchronize(sk->ctx->stream));
    });
}

int trg_lift_back(trg_ctx* ctx, int order, const int64_t* dims, const int64_t* K, const double* projected,
                  const double* const* bases, trg_tensor** out) {
    return guard([&] {
        require(ctx && dims && K && projected && bases && out, "lift_back: null argument");
        require(order >= 1, "lift_back: order must be at least 1");
        std::vector<int64_t> d(dims, dims + order), k(K, K + order);
        for (int n = 0; n < order; ++n)
            require(d[n] >= 1 && k[n] >= 1 && bases[n], "lift_back: extents must be positive, bases non-null");
        double* dP = (double*)ctx->alloc(sizeof(double) * (size_t)prod(k));
        CK(cudaMemcpyAsync(dP, projected, sizeof(double) * prod(k), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<const double*> q(order, nullptr);
        std::vector<double*> owned;
        for (int n = 0; n < order; ++n) {
            // sketch.hpp:98: a square, exactly-identity basis is skipped (no product, bit-exact copy)
            bool ident = d[n] == k[n];
            for (int64_t e = 0; ident && e < d[n] * k[n]; ++e)
                ident = bases[n][e] == ((e % d[n]) == (e / d[n]) ? 1.0 : 0.0);
            if (ident) continue;
            double* dq = (double*)ctx->alloc(sizeof(double) * d[n] * k[n]);
            CK(cudaMemcpyAsync(dq, bases[n], sizeof(double) * d[n] * k[n], cudaMemcpyHostToDevice, ctx->stream));
            q[n] = dq;
            owned.push_back(dq);
        }
        *out = lift_back_device(ctx, F64, d, k, dP, q);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->dfree(dP);
        for (double* p : owned) ctx->dfree(p);
    });
}

int trg_back_project(trg_ctx* ctx, int order, const int64_t* K, const int64_t* ranks, const double* small_cores,
                     const trg_sketch* sk, double* cores_out) {
    return guard([&] { back_project_device(ctx, order, K, ranks, small_cores, sk, cores_out); });
}

int trg_rse(trg_ctx* ctx, const trg_tensor* x, const int64_t* ranks, const double* cores, double* out) {
    return guard([&] { *out = rse_device(ctx, x, ranks, cores); });
}

int trg_decompose(trg_ctx* ctx, const trg_tensor* x, int method, const int64_t* ranks, double tol,
                  int64_t max_sweeps, uint64_t cfg_seed, const int64_t* K, uint64_t spec_seed, int variant,
                  trg_report** out) {
    return guard([&] {
        auto rep = std::make_unique<trg_report>();
        decompose_impl(ctx, x, method, ranks, tol, max_sweeps, cfg_seed, K, spec_seed, variant, rep.get(), now_ms());
        *out = rep.release();
    });
}

int trg_decompose_host(trg_ctx* ctx, int dtype, int order, const int64_t* dims, const void* host_local, int method,
                       const int64_t* ranks, double tol, int64_t max_sweeps, uint64_t cfg_seed, const int64_t* K,
                       uint64_t spec_seed, int variant, trg_report** out) {
    return guard([&] {
        const double t0 = now_ms();
        std::unique_ptr<trg_tensor, void (*)(trg_tensor*)> x(tensor_new(ctx, dtype, order, dims),
                                                             [](trg_tensor* t) { trg_tensor_destroy(t); });
        CK(cudaMemcpyAsync(x->d, host_local, trg::dtype_size(dtype) * x->local_elems, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        auto rep = std::make_unique<trg_report>();
        rep->ms[0] = now_ms() - t0;
        decompose_impl(ctx, x.get(), method, ranks, tol, max_sweeps, cfg_seed, K, spec_seed, variant, rep.get(), t0);
        *out = rep.release();
    });
}

int trg_report_ranks(const trg_report* r, int64_t* ranks) {
    return guard([&] { std::copy(r->ranks.begin(), r->ranks.end(), ranks); });
}
int trg_report_cores_len(const trg_report* r, int64_t* n) { return guard([&] { *n = (int64_t)r->cores.size(); }); }
int trg_report_cores(const trg_report* r, double* out) {
    return guard([&] { std::copy(r->cores.begin(), r->cores.end(), out); });
}
int trg_report_rse_history(const trg_report* r, double* out, int64_t* n) {
    return guard([&] {
        if (n) *n = (int64_t)r->rse_history.size();
        if (out) std::copy(r->rse_history.begin(), r->rse_history.end(), out);
    });
}
int trg_report_sweeps(const trg_report* r, int64_t* s) { return guard([&] { *s = r->sweeps; }); }
int trg_report_timings(const trg_report* r, double* ms) { return guard([&] { std::copy(r->ms, r->ms + 6, ms); }); }
int trg_report_projected(const trg_report* r, double* out, int64_t* n) {
    return guard([&] {
        if (n) *n = (int64_t)r->projected.size();
        if (out) std::copy(r->projected.begin(), r->projected.end(), out);
    });
}
int trg_report_destroy(trg_report* r) {
    return guard([&] { delete r; });
}

}  // extern "C"
