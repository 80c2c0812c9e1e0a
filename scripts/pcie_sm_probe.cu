// SM copies over PCIe (pinned host memory through its device mapping):
// host->device read bandwidth vs loads in flight, and device->host posted
// write bandwidth, for the host step's 2.46 MB (d = 784) transfers.
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void rd(const float4* __restrict__ src, float4* __restrict__ dst, long n4) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n4) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n4) __stcs(dst + i + u * stride, v[u]);
    }
}

int main() {
    const long n = 784L * 784 + 2 * 784 * 32, n4 = n / 4;
    float *h, *hm, *d;
    cudaHostAlloc(&h, n * 4, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hm, h, 0);
    cudaMalloc(&d, n * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* what, auto kern, int grid, int blk, const float4* s, float4* t) {
        float best = 1e9, ms;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(a);
            kern<<<grid, blk>>>(s, t, n4);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-6s grid %5d x %4d: %7.1f us  %6.1f GB/s\n", what, grid, blk, best * 1e3, n * 4 / (best * 1e-3) / 1e9);
    };
    for (int grid : {148, 296, 592, 1184})
        for (int blk : {256, 512}) {
            run("h2d U4", rd<4>, grid, blk, (const float4*)hm, (float4*)d);
            run("h2d U8", rd<8>, grid, blk, (const float4*)hm, (float4*)d);
            run("h2d U16", rd<16>, grid, blk, (const float4*)hm, (float4*)d);
            run("d2h U8", rd<8>, grid, blk, (const float4*)d, (float4*)hm);
        }
    float ms;
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, n * 4, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy h2d %.1f us\n", ms * 1e3);
    cudaEventRecord(a);
    cudaMemcpyAsync(h, d, n * 4, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy d2h %.1f us\n", ms * 1e3);
    return 0;
}
