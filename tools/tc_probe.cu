// Development probe for the operand layouts of csrc/tc_f32.cu: one tcgen05.mma.kind::tf32
// (M=128, N=16, K=8) with A MN-major 128B-swizzled (4 blocks of 32 rows at LBO) and B K-major
// no-swizzle (LBO 128 between the K halves, SBO 256 between 8-row groups); D against the host.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ int g_rawmode = 0;
__host__ __device__ float aval(int m, int k) {
#ifdef __CUDA_ARCH__
    if (g_rawmode) return 1.0f + 3.0f / 4096.0f;  // tf32: RN -> 1 + 2^-10, truncation -> 1
#endif
    return (float)((m * 7 + k * 3) % 11) - 5.0f;
}
__host__ __device__ float bval(int n, int k) { return (float)((n * 5 + k) % 7) - 3.0f; }

__global__ void k(uint32_t idesc, uint32_t a_lbo, uint32_t a_sbo, int a_sw, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t base = (su32(sm) + 1023u) & ~1023u;
    unsigned char* g = sm + (base - su32(sm));
    float* A = (float*)g;                 // 4 blocks x 1024 B (LBO = 1024)
    float* B = (float*)(g + 8192);        // 16 x 8 K-major no swizzle
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
        const int m = e % 128, kk = e / 128;
        const int blk = m / 32, w = m % 32, ch = w / 4, pos = w % 4;
        // a_sw 1: 128B swizzle of 16B chunks (row mod 8); 2: 128B swizzle of 32B chunks (row mod 4)
        int byte = w * 4;
        if (a_sw == 1) byte = ((ch ^ (kk & 7)) * 16) + pos * 4;
        if (a_sw == 2) byte = ((((w / 8) ^ (kk & 3)) * 32) + (w % 8) * 4);
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
    if (threadIdx.x == 0) {
        auto desc = [&](uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
            return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                   ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)lay << 61);
        };
        uint64_t da = desc(su32(A), a_lbo, a_sbo, a_sw == 1 ? 2 : a_sw == 2 ? 1 : 0), db = desc(su32(B), 128, 256, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                     "l"(da), "l"(db), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    if (threadIdx.x < 128) {
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
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 16 * sizeof(float));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    const uint32_t base = (1u << 4) | (2u << 7) | (2u << 10) | (2u << 17) | (8u << 24);
    struct V { const char* name; uint32_t idesc, lbo, sbo; int sw; };
    V vs[] = {
        {"A MN sw128/32B lbo1024 sbo512", base | (1u << 15), 1024, 512, 2},
        {"A MN sw128/32B lbo512 sbo1024", base | (1u << 15), 512, 1024, 2},
        {"A MN sw128 lbo1024 sbo1024", base | (1u << 15), 1024, 1024, 1},
    };
    float want[128 * 16];
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            float s = 0;
            for (int kk = 0; kk < 8; ++kk) s += aval(m, kk) * bval(n, kk);
            want[m * 16 + n] = s;
        }
    {  // how kind::tf32 reads an fp32 operand with low mantissa bits set
        int one = 1;
        cudaMemcpyToSymbol(g_rawmode, &one, sizeof(int));
        cudaMemset(d, 0, 128 * 16 * sizeof(float));
        k<<<1, 128, 16384>>>(vs[0].idesc, vs[0].lbo, vs[0].sbo, vs[0].sw, d);
        cudaDeviceSynchronize();
        float h[16];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        float bs = 0;
        for (int kk = 0; kk < 8; ++kk) bs += bval(0, kk);
        printf("raw-fp32 A = 1+3*2^-12: D[0][0] = %.9g; trunc -> %.9g, RN -> %.9g\n", h[0], bs * 1.0,
               bs * (1.0 + 1.0 / 1024));
        int zero = 0;
        cudaMemcpyToSymbol(g_rawmode, &zero, sizeof(int));
    }
    for (auto& v : vs) {
        cudaMemset(d, 0, 128 * 16 * sizeof(float));
        k<<<1, 128, 16384>>>(v.idesc, v.lbo, v.sbo, v.sw, d);
        cudaError_t e = cudaDeviceSynchronize();
        float h[128 * 16];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double err = 0;
        int bad = 0;
        for (int i = 0; i < 128 * 16; ++i) {
            err = fmax(err, fabs(h[i] - want[i]));
            bad += fabs(h[i] - want[i]) > 1e-3;
        }
        printf("%-30s err=%s maxdiff=%g bad=%d  D[0][0..3]=%g %g %g %g want %g %g %g %g  D[37][5]=%g want %g\n", v.name,
               cudaGetErrorString(e), err, bad, h[0], h[1], h[2], h[3], want[0], want[1], want[2], want[3],
               h[37 * 16 + 5], want[37 * 16 + 5]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
