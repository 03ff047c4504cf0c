// cuSOLVER QR entry points on the small solve's system shapes (C4: 2048 / 4096 x 400):
// legacy Dgeqrf against the 64-bit generic Xgeqrf. nvcc -O2 -arch=sm_100a geqrf_probe.cu -lcusolver -lcublas
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>
int main() {
    cusolverDnHandle_t h;
    cusolverDnCreate(&h);
    cusolverDnParams_t prm;
    cusolverDnCreateParams(&prm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int m : {2048, 4096}) {
        const int n = 400;
        std::vector<double> ha((size_t)m * n);
        for (auto& v : ha) v = rand() / (double)RAND_MAX - 0.5;
        double *dA, *dA0, *tau;
        int* info;
        cudaMalloc(&dA, sizeof(double) * m * n);
        cudaMalloc(&dA0, sizeof(double) * m * n);
        cudaMalloc(&tau, sizeof(double) * n);
        cudaMalloc(&info, sizeof(int));
        cudaMemcpy(dA0, ha.data(), sizeof(double) * m * n, cudaMemcpyHostToDevice);
        int lw = 0;
        cusolverDnDgeqrf_bufferSize(h, m, n, dA, m, &lw);
        double* w;
        cudaMalloc(&w, sizeof(double) * lw);
        size_t dws = 0, hws = 0;
        cusolverDnXgeqrf_bufferSize(h, prm, m, n, CUDA_R_64F, dA, m, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws);
        void* dw;
        cudaMalloc(&dw, dws);
        std::vector<char> hw(hws + 1);
        for (int variant = 0; variant < 2; ++variant) {
            float best = 1e9f;
            for (int it = 0; it < 8; ++it) {
                cudaMemcpy(dA, dA0, sizeof(double) * m * n, cudaMemcpyDeviceToDevice);
                cudaEventRecord(e0);
                if (variant == 0)
                    cusolverDnDgeqrf(h, m, n, dA, m, tau, w, lw, info);
                else
                    cusolverDnXgeqrf(h, prm, m, n, CUDA_R_64F, dA, m, CUDA_R_64F, tau, CUDA_R_64F, dw, dws, hw.data(),
                                     hws, info);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it > 1 && ms < best) best = ms;
            }
            printf("m=%d n=%d %s best %.3f ms\n", m, n, variant ? "Xgeqrf" : "Dgeqrf", best);
        }
        cudaFree(dA); cudaFree(dA0); cudaFree(tau); cudaFree(info); cudaFree(w); cudaFree(dw);
    }
    return 0;
}
