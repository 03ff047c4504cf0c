// Development probe: issue-to-completion cost of back-to-back tcgen05.mma kind::tf32 (M = 128,
// K = 8 per instruction) as a function of N, of where A lives (shared memory "SS" or TMEM "TS")
// and of how many distinct accumulators the stream rotates over (ND). One CTA, thread 0 issues R
// MMAs, commits, waits; cycles / R printed. Operand values are zeros (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mma_probe tools/mma_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// sw: 0 = K-major no swizzle (8 x 16 B core matrices), 1 = K-major 128B swizzle (128-byte rows,
// 1024-byte 8-row atoms; the k-step advances the start address by 32 B inside the row)
// uni: the whole of warp 0 runs the issue loop and one elected lane issues each MMA (elect.sync, as
// CUTLASS does); otherwise thread 0 alone runs it (a divergent branch around every MMA)
__global__ void probe(int N, int ND, int ts, int sw, int uni, int R, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];  // A 128 x 128 B, B 256 x 128 B (dynamic)
    const int sm_bytes = 128 * 128 + 256 * 128;
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < sm_bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    if (uni ? threadIdx.x < 32 : threadIdx.x == 0) {
        const uint64_t ad = sw ? sdesc(su32(sm), 16, 1024, 2) : sdesc(su32(sm), 128, 256);
        const uint64_t bd = sw ? sdesc(su32(sm + 128 * 128), 16, 1024, 2) : sdesc(su32(sm + 128 * 32), 128, 256);
        const uint32_t id = idesc_tf32(128, N);
        const uint32_t atm = tmem + 448;  // A (128 x 8) in TMEM columns 448..455
        long long t0 = clock64();
        uint32_t d = tmem;
        int nd = 0;
        for (int i = 0; i < R; ++i) {
            if (uni == 3) {  // every operand from uniform sources (TMEM base taken as 0, shared base, loop counter)
                const uint32_t du = (uint32_t)((i & (ND - 1)) * N);
                const uint64_t adu = ad + (uint64_t)((i & 3) * 2);  // k-step walk (32 B)
                const uint64_t bdu = bd + (uint64_t)((i & 3) * 2);
                asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(du),
                             "l"(adu), "l"(bdu), "r"(id), "r"(1u));
            } else if (uni == 2) {  // four MMAs per asm block: one operand conversion per block
                asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(ad), "l"(bd), "r"(id), "r"(1u));
                i += 3;
            } else if (uni) {
                if (ts)
                    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                                 "r"(atm), "l"(bd), "r"(id), "r"(1u));
                else
                    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                 "l"(ad), "l"(bd), "r"(id), "r"(1u));
            } else if (ts)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(atm), "l"(bd), "r"(id), "r"(1u));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(ad), "l"(bd), "r"(id), "r"(1u));
            if (++nd == ND) nd = 0, d = tmem; else d += (uint32_t)N;
        }
        long long t1 = clock64();
        if (threadIdx.x == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile(
            "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(
                su32(&bar)));
        long long t2 = clock64();
        if (threadIdx.x == 0) {
            if (uni == 3 && tmem != 0) t2 = -1;
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    long long h[2];
    cudaMalloc(&d, 16);
    const int R = 4096;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 + 256 * 128);
    for (int uni = 1; uni < 4; ++uni)
    for (int sw = 0; sw < 1; ++sw)
    for (int ts = 0; ts < (uni >= 2 ? 1 : 2); ++ts)
        for (int N : {16, 32, 64, 128, 256})
            for (int ND : {1, 4}) {
                if (ND * N > 448) continue;
                probe<<<1, 128, 128 * 128 + 256 * 128>>>(N, ND, ts, sw, uni, R, d);  // warm
                probe<<<1, 128, 128 * 128 + 256 * 128>>>(N, ND, ts, sw, uni, R, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                printf("%s %s %s N=%3d ND=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d)\n", uni == 3 ? "eluni" : uni == 2 ? "elx4 " : uni ? "elect" : "lane0", sw ? "sw128" : "nosw ", ts ? "TS" : "SS", N, ND,
                       (double)h[0] / R, (double)h[1] / R, 128 * N / 256);
            }
    return 0;
}
