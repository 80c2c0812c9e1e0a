// Launch / scheduling cost of (nearly) empty grids: back-to-back launches of
// G CTAs x 256 threads in clusters of C, amortised over 200 launches.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k(float* p, int smem_touch) {
    extern __shared__ float sm[];
    if (smem_touch && threadIdx.x == 0) sm[0] = 1.f;
    if (threadIdx.x == 0 && p[blockIdx.x] == 12345.f) p[blockIdx.x] = sm[0];
}

int main() {
    float* p;
    cudaMalloc(&p, 4096 * 4);
    cudaMemset(p, 0, 4096 * 4);
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t s;
    cudaStreamCreate(&s);
    struct Cfg { int grid, clu, smem_kb; };
    Cfg cfgs[] = {{148, 1, 0}, {250, 1, 0}, {250, 2, 0}, {250, 5, 0}, {250, 10, 0}, {250, 10, 100},
                  {80, 10, 171}, {80, 8, 171}, {320, 1, 13}, {1, 1, 0}};
    for (auto c : cfgs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = c.smem_kb * 1024;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.clu;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int w = 0; w < 20; ++w) cudaLaunchKernelEx(&cfg, empty_k, p, c.smem_kb > 0);
        // graph of 200 launches
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int w = 0; w < 200; ++w) cudaLaunchKernelEx(&cfg, empty_k, p, c.smem_kb > 0);
        cudaStreamEndCapture(s, &g);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
        cudaGraphLaunch(ge, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) { printf("err %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
        cudaStreamSynchronize(s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int w = 0; w < 200; ++w) cudaLaunchKernelEx(&cfg, empty_k, p, c.smem_kb > 0);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms2;
        cudaEventElapsedTime(&ms2, e0, e1);
        printf("grid %4d cluster %2d smem %3d KB: %.2f us/launch stream, %.2f us/launch graph (%s)\n", c.grid, c.clu,
               c.smem_kb, ms * 1e3 / 200, ms2 * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
