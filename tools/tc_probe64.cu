// Development probe: where an M=64 cta_group::1 tcgen05.mma.kind::tf32 leaves D in TMEM.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ float aval(int m, int k) { return (float)((m * 7 + k * 3) % 11) - 5.0f; }
__host__ __device__ float bval(int n, int k) { return (float)((n * 5 + k) % 7) - 3.0f; }

__global__ void k(uint32_t idesc, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t base = (su32(sm) + 1023u) & ~1023u;
    unsigned char* g = sm + (base - su32(sm));
    float* A = (float*)g;                 // 2 blocks x 1024 B (LBO = 1024), 8 k-rows of 128 B
    float* B = (float*)(g + 4096);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int e = threadIdx.x; e < 64 * 8; e += blockDim.x) {
        const int m = e % 64, kk = e / 64;
        const int blk = m / 32, w = m % 32;
        const int byte = ((((w / 8) ^ (kk & 3)) * 32) + (w % 8) * 4);
        *(float*)((unsigned char*)A + blk * 1024 + kk * 128 + byte) = aval(m, kk);
    }
    for (int e = threadIdx.x; e < 16 * 8; e += blockDim.x) {
        const int n = e % 16, kk = e / 16;
        *(float*)((unsigned char*)B + (n / 8) * 256 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4) = bval(n, kk);
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    // clear the accumulator region first (so untouched lanes read 0)
    {
        const uint32_t ta = tm + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
        uint32_t z = 0;
        for (int c = 0; c < 16; ++c)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(z) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        auto desc = [&](uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
            return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                   ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)lay << 61);
        };
        uint64_t da = desc(su32(A), 1024, 512, 1), db = desc(su32(B), 128, 256, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                     "l"(da), "l"(db), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[16];
    const uint32_t ta = tm + ((uint32_t)((threadIdx.x / 32) * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) out[threadIdx.x * 16 + j] = __uint_as_float(r[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 16 * sizeof(float));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (2u << 17) | (4u << 24);  // M=64
    cudaMemset(d, 0, 128 * 16 * sizeof(float));
    k<<<1, 128, 16384>>>(idesc, d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M=64: %s\n", cudaGetErrorString(e));
    // for each TMEM lane, which row m (if any) matches D(m, :) over the 16 columns
    for (int lane = 0; lane < 128; ++lane) {
        int match = -1;
        for (int m = 0; m < 64 && match < 0; ++m) {
            bool ok = true;
            for (int n = 0; n < 16 && ok; ++n) {
                float s = 0;
                for (int kk = 0; kk < 8; ++kk) s += aval(m, kk) * bval(n, kk);
                ok = fabsf(h[lane * 16 + n] - s) < 1e-3f;
            }
            if (ok) match = m;
        }
        bool zero = true;
        for (int n = 0; n < 16; ++n) zero = zero && h[lane * 16 + n] == 0.f;
        printf("lane %3d -> %s%d\n", lane, zero ? "zero " : "", match);
    }
    return 0;
}
