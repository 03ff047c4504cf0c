// Development probe: throughput of back-to-back tcgen05.mma.kind::tf32 (one CTA) for K-major vs
// MN-major (128B / 32B-atom) A, M = 128 / 64, various N; cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(uint32_t idesc, int a_lay, uint32_t a_lbo, uint32_t a_sbo, int n_rows_b, int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t base = (su32(sm) + 1023u) & ~1023u;
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)(sm + (base - su32(sm))))[i] = 1.0f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    if (threadIdx.x == 0) {
        auto desc = [&](uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
            return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                   ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)lay << 61);
        };
        const uint64_t da = desc(base, a_lbo, a_sbo, a_lay), db = desc(base + 32768, 128, 256, 0);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                         "l"(da + (uint64_t)((i & 3) * 64)), "l"(db), "r"(idesc), "r"(1u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)));
        out[0] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const uint32_t base = (1u << 4) | (2u << 7) | (2u << 10);
    struct V { const char* name; int M, N, amn, lay; uint32_t lbo, sbo; };
    V vs[] = {
        {"K-major SW128  M128 N64", 128, 64, 0, 2, 16, 1024},
        {"MN sw128_32B   M128 N64", 128, 64, 1, 1, 1024, 512},
        {"K-major SW128  M128 N128", 128, 128, 0, 2, 16, 1024},
        {"MN sw128_32B   M128 N128", 128, 128, 1, 1, 1024, 512},
        {"K-major SW128  M128 N32", 128, 32, 0, 2, 16, 1024},
        {"MN sw128_32B   M128 N32", 128, 32, 1, 1, 1024, 512},
        {"K-major SW128  M64 N32", 64, 32, 0, 2, 16, 1024},
        {"MN sw128_32B   M64 N32", 64, 32, 1, 1, 1024, 512},
        {"MN sw128_32B   M64 N16", 64, 16, 1, 1, 1024, 512},
        {"K-major none   M128 N64", 128, 64, 0, 0, 128, 256},
    };
    for (auto& v : vs) {
        const uint32_t id = base | ((uint32_t)v.amn << 15) | ((uint32_t)(v.N >> 3) << 17) | ((uint32_t)(v.M >> 4) << 24);
        k<<<1, 128, 100000>>>(id, v.lay, v.lbo, v.sbo, v.N, 4096, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-26s %s  %.1f cycles/MMA\n", v.name, cudaGetErrorString(e), h / 4096.0);
    }
    return 0;
}
