// Dependent-chain latencies on this GPU (cycles per op), single warp: DFMA, FFMA, fp64 rsqrt,
// fp64 shuffle, shared-memory load. Development aid for the latency-bound QR kernel.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x = a;
    float xf = (float)a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) xf = fmaf(xf, (float)b, (float)a);
    long long t2 = clock64();
    double y = 2.0 + x * 1e-30;
    for (int i = 0; i < n; ++i) y = rsqrt(y) + 1.5;
    long long t3 = clock64();
    double z = x;
    for (int i = 0; i < n; ++i) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31) + 1.0;
    long long t4 = clock64();
    int idx = threadIdx.x & 63;
    for (int i = 0; i < n; ++i) idx = ((int)sm[idx] + 1) & 63;
    long long t5 = clock64();
    double w = y;
    for (int i = 0; i < n; ++i) w = sqrt(w) + 1.0;
    long long t6 = clock64();
    double v = y;
    for (int i = 0; i < n; ++i) v = 1.0 / v + 1.0;
    long long t7 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
        cyc[5] = t6 - t5; cyc[6] = t7 - t6;
    }
    out[threadIdx.x] = x + xf + y + z + idx + w + v;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMallocManaged(&cyc, 8 * 8);
    const int n = 4096;
    k<<<1, 32>>>(out, cyc, 0.5, 0.999, n);
    k<<<1, 32>>>(out, cyc, 0.5, 0.999, n);
    cudaDeviceSynchronize();
    printf("{\"dfma\": %.1f, \"ffma\": %.1f, \"rsqrt_f64_plus_dadd\": %.1f, \"shfl_f64_plus_dadd\": %.1f, "
           "\"lds_f64_cvt_add\": %.1f, \"sqrt_f64_plus_dadd\": %.1f, \"div_f64_plus_dadd\": %.1f}\n",
           (double)cyc[0] / n, (double)cyc[1] / n, (double)cyc[2] / n, (double)cyc[3] / n, (double)cyc[4] / n,
           (double)cyc[5] / n, (double)cyc[6] / n);
    return 0;
}
