// Cost of loading a CTA's slab rows (RB=80 rows x 96 columns of a d x n
// column-major fp32 matrix, the WY builder's phase 1) by three mechanisms,
// 250 CTAs in 10-CTA clusters like the builder; cycles from kernel entry to
// data in shared memory (thread 0), mean / max over CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int RB = 80, P = 84, NCOL = 96, D = 784, N = 784;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256, 2) probe(const float* __restrict__ V, long long* cyc, float* sink) {
    extern __shared__ __align__(128) float sm[];
    __shared__ uint64_t bar;
    long long t0 = clock64();
    const int cl = blockIdx.x / 10, rank = blockIdx.x % 10;
    const int row0 = rank * RB;
    const int col0 = (cl * 32 + N - 32) % N;  // blocks i-1, i, i+1 ~ 96 consecutive columns
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nrows = min(RB, D - row0);
    if (MODE == 0) {  // LDG.128 -> registers -> STS
        float4 v[8];
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = tid + u * 256;  // 96 cols x 20 float4
            const int c = idx / 20, r4 = idx % 20;
            if (c < NCOL && r4 * 4 < nrows) v[u] = *reinterpret_cast<const float4*>(V + (size_t)((col0 + c) % N) * D + row0 + r4 * 4);
            else v[u] = make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = tid + u * 256;
            const int c = idx / 20, r4 = idx % 20;
            if (c < NCOL) *reinterpret_cast<float4*>(sm + c * P + r4 * 4) = v[u];
        }
        (void)cnt;
        __syncthreads();
    } else if (MODE == 1) {  // cp.async 16 B
        for (int idx = tid; idx < NCOL * 20; idx += 256) {
            const int c = idx / 20, r4 = idx % 20;
            const float* src = V + (size_t)((col0 + c) % N) * D + row0 + r4 * 4;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(sm + c * P + r4 * 4)), "l"(src),
                         "r"(r4 * 4 < nrows ? 16 : 0));
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
        __syncthreads();
    } else {  // one bulk copy per column
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(NCOL * nrows * 4));
        }
        __syncthreads();
        if (warp == 0)
            for (int c = lane; c < NCOL; c += 32)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 su32(sm + c * P)),
                             "l"(V + (size_t)((col0 + c) % N) * D + row0), "r"(nrows * 4), "r"(su32(&bar))
                             : "memory");
        asm volatile(
            "{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(su32(&bar))
            : "memory");
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    if (tid == 0) sink[blockIdx.x] = sm[lane * P + 3];
}

int main() {
    float *V, *sink, *flush;
    long long* cyc;
    cudaMalloc(&V, (size_t)D * N * 4);
    cudaMemset(V, 0, (size_t)D * N * 4);
    cudaMalloc(&sink, 4096);
    cudaMalloc(&cyc, 250 * 8);
    cudaMalloc(&flush, 256 << 20);
    long long h[250];
    const size_t smem = NCOL * P * 4;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const char* names[3] = {"LDG.128->STS", "cp.async 16B", "bulk per column"};
    for (int fl = 0; fl < 2; ++fl)
        for (int rep = 0; rep < 2; ++rep)
            for (int mode = 0; mode < 3; ++mode) {
                if (fl) cudaMemset(flush, 0, 256 << 20);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(250);
                cfg.blockDim = dim3(256);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 10;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaError_t e = mode == 0 ? cudaLaunchKernelEx(&cfg, probe<0>, (const float*)V, cyc, sink)
                              : mode == 1 ? cudaLaunchKernelEx(&cfg, probe<1>, (const float*)V, cyc, sink)
                                          : cudaLaunchKernelEx(&cfg, probe<2>, (const float*)V, cyc, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(h, cyc, 250 * 8, cudaMemcpyDeviceToHost);
                double m = 0;
                long long mx = 0;
                for (int i = 0; i < 250; ++i) m += h[i], mx = h[i] > mx ? h[i] : mx;
                printf("%-16s %s: mean %6.0f max %6lld cycles, kernel %.2f us (%s)\n", names[mode],
                       fl ? "after L2 flush" : "L2 warm      ", m / 250, mx, ms * 1e3, cudaGetErrorString(e));
            }
    return 0;
}
