// FP64 latency / throughput on this part, and the cost of build4's T~ recursion.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_lat(double* out, long long* cyc, double x) {
    double a = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) a = fma(a, x, 1.0);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void dfma_tput(double* out, long long* cyc, double x) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], x, 1.0);
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void ffma_tput(float* out, long long* cyc, float x) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], x, 1.0f);
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void ddiv(double* out, long long* cyc, double x) {
    double a = threadIdx.x + 1.0;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i) a = 1.0 / (a + x);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 256 * 8);
    cudaMalloc(&cyc, 148 * 8);
    long long h[148];
    for (int rep = 0; rep < 2; ++rep) {
        dfma_lat<<<1, 32>>>(out, cyc, 1.0000001);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA dependent latency: %.1f cycles\n", h[0] / 1024.0);
        ddiv<<<1, 32>>>(out, cyc, 0.5);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("f64 1/x dependent latency: %.1f cycles\n", h[0] / 64.0);
        for (int thr : {128, 256, 512, 1024}) {
            dfma_tput<<<148, thr>>>(out, cyc, 1.0000001);
            cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
            printf("DFMA throughput %4d thr/SM: %.2f DFMA/clk/SM\n", thr, thr * 2048.0 / h[0]);
            ffma_tput<<<148, thr>>>((float*)out, cyc, 1.0001f);
            cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
            printf("FFMA throughput %4d thr/SM: %.2f FFMA/clk/SM\n", thr, thr * 2048.0 / h[0]);
        }
    }
    return 0;
}
