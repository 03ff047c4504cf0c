// FP64 ceilings on this GPU: DMMA (mma.sync m8n8k4 f64) and DFMA throughput, alone and
// co-issued from different warps of the same SM. Development aid: the fp64 sketch/shrink
// kernels are bounded by these, not only by HBM. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA
__global__ void k(int iters, int mode, double* out) {
    const int warp = threadIdx.x >> 5;
    const bool do_mma = mode == 0 || (mode == 2 && !(warp & 1));
    double acc[8][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = i * 1e-3;
    if (do_mma) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, b);
    } else {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int r = 0; r < 16; ++r)  // 16 DFMA x 8 chains x 2 = 256 FMA per lane per iter = one DMMA's worth per warp... per lane
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i][r & 1] = fma(a, acc[i][r & 1], b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000;
    printf("{");
    for (int warps : {4, 8, 16}) {
        for (int mode = 0; mode < 3; ++mode) {
            const int blocks = sms * 2, threads = 32 * warps;
            k<<<blocks, threads>>>(10, mode, out);
            cudaEventRecord(e0);
            k<<<blocks, threads>>>(iters, mode, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            // per warp per iter: DMMA 8 x 256 FMA; DFMA 16 x 8 x 32 lanes FMA = 4096 FMA = 16 x 256
            const double mma_warps = mode == 0 ? warps : mode == 1 ? 0 : warps / 2;
            const double fma_warps = warps - mma_warps;
            const double flops = 2.0 * blocks * iters * (mma_warps * 8 * 256 + fma_warps * 16 * 8 * 32);
            printf("%s\"w%d_%s\": %.2f", (warps == 4 && mode == 0) ? "" : ", ", warps,
                   mode == 0 ? "dmma" : mode == 1 ? "dfma" : "mixed", flops / (ms * 1e-3) / 1e12);
        }
    }
    printf("}\n");
    return 0;
}
