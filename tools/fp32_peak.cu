// FP32 ceiling on this GPU: FFMA throughput of the CUDA cores (no tensor cores), the second
// roofline of the fp32 FFMA sketch kernels (k_sketch_l1_f32: K_0 FFMA per element of X). Eight
// independent FFMA chains per thread, 8 / 16 / 32 warps per CTA, two CTAs per SM. Prints one JSON
// line (TFLOP/s, 2 flops per FFMA) -> profiles/fp32_peak.json.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int iters, float* out) {
    float acc[8];
    const float a = 1.0f + threadIdx.x * 1e-7f, b = 1.0f - threadIdx.x * 1e-7f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = i * 1e-3f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = fmaf(a, acc[i], b);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678f) out[0] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    printf("{");
    bool first = true;
    for (int warps : {8, 16, 32}) {
        const int blocks = sms * 2, threads = 32 * warps;
        k<<<blocks, threads>>>(10, out);
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
        printf("%s\"w%d_ffma\": %.2f", first ? "" : ", ", warps, flops / (ms * 1e-3) / 1e12);
        first = false;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf(", \"sms\": %d, \"max_clock_mhz\": %.0f, \"nominal_ffma_tflops\": %.2f}\n", sms, clk / 1e3,
           2.0 * 128 * sms * clk * 1e3 / 1e12);
    return 0;
}
