// Cold instruction-fetch cost on B200: the same number of FFMA executed once
// as straight-line code vs as a loop (warm after the first iteration).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/icp scripts/icache_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__device__ __forceinline__ void body(float (&a)[8], float x) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i & 7] = fmaf(a[i & 7], x, 1.0f + i);
}

__global__ void straight(float* out, long long* cyc, float x) {
    float a[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    long long t0 = clock64();
    body<4096>(a, x);
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void looped(float* out, long long* cyc, float x) {
    float a[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < 16; ++r) body<256>(a, x);
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    const int nb = 296;
    cudaMalloc(&out, nb * 256 * 4);
    cudaMalloc(&cyc, nb * 8);
    long long h[296];
    for (int rep = 0; rep < 3; ++rep) {
        for (int k = 0; k < 2; ++k) {
            if (k == 0) straight<<<nb, 256>>>(out, cyc, 1.0001f);
            else looped<<<nb, 256>>>(out, cyc, 1.0001f);
            cudaMemcpy(h, cyc, nb * 8, cudaMemcpyDeviceToHost);
            double m = 0;
            long long mx = 0;
            for (int i = 0; i < nb; ++i) m += h[i], mx = h[i] > mx ? h[i] : mx;
            printf("%s rep %d: 4096 FFMA/thread, 256 thr x %d CTAs: mean %.0f max %lld cycles\n",
                   k ? "looped  " : "straight", rep, nb, m / nb, mx);
        }
    }
    return 0;
}
