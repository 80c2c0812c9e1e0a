// Micro-benchmark: cost of pushing a 1 KB partial to every CTA of a 7-CTA
// cluster (the chain sweep's per-step all-to-all), three ways:
//   mode 0: 64 threads, each st.async.v4 to all 7 peers (serial per thread)
//   mode 1: 7 warps, warp w pushes the whole 1 KB to peer w (2 st.async.v4 per lane)
//   mode 2: 7 threads (lane 0 of warps 0..6), one cp.async.bulk smem->peer smem each
// Each iteration: push, then wait for the 7 incoming KB on the local mbarrier
// (all-to-all round), repeated; reports cycles per round and the issuing
// time of the push itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbp scripts/microbench_push.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ uint32_t crank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void waitp(uint32_t bar, uint32_t par) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(bar),
                 "r"(par)
                 : "memory");
}

constexpr int C = 7;

__global__ void __cluster_dims__(C, 1, 1) push_kernel(int mode, int iters, long long* out) {
    __shared__ __align__(128) float src[256];
    __shared__ __align__(128) float recv[2][C][256];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = crank();
    for (int i = tid; i < 256; i += blockDim.x) src[i] = rank + i;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int s = 0; s < 2; ++s) expect(s32(&bar[s]), C * 1024);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    csync();
    long long t_issue = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int slot = it & 1;
        const uint32_t rb_l = s32(&bar[slot]);
        const uint32_t rz_l = s32(&recv[slot][rank][0]);
        const long long a = clock64();
        if (mode == 0) {
            if (tid < 64) {
                const float4 v = reinterpret_cast<const float4*>(src)[tid];
                for (int d = 0; d < C; ++d)
                    asm volatile(
                        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                            mapa(rz_l + tid * 16, d)),
                        "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                        "r"(__float_as_uint(v.w)), "r"(mapa(rb_l, d))
                        : "memory");
            }
        } else if (mode == 1) {
            if (warp < C) {
                const int d = warp;
                for (int k = lane; k < 64; k += 32) {
                    const float4 v = reinterpret_cast<const float4*>(src)[k];
                    asm volatile(
                        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                            mapa(rz_l + k * 16, d)),
                        "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                        "r"(__float_as_uint(v.w)), "r"(mapa(rb_l, d))
                        : "memory");
                }
            }
        } else {
            if (warp < C && lane == 0) {
                const int d = warp;
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(
                        mapa(rz_l, d)),
                    "r"(s32(src)), "r"(mapa(rb_l, d))
                    : "memory");
            }
        }
        if (tid == 0) t_issue += clock64() - a;
        waitp(rb_l, (uint32_t)((it >> 1) & 1));
        __syncthreads();
        if (tid == 0) expect(rb_l, C * 1024);
        __syncthreads();
    }
    const long long t1 = clock64();
    csync();
    if (tid == 0 && rank == 0) {
        out[0] = (t1 - t0) / iters;
        out[1] = t_issue / iters;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 16 * sizeof(long long));
    const char* names[] = {"64 thr x 7 peers st.async", "7 warps x 1 peer st.async", "7 thr bulk smem->dsmem"};
    for (int mode = 0; mode < 3; ++mode) {
        push_kernel<<<C, 256>>>(mode, 200, d);
        push_kernel<<<C, 256>>>(mode, 200, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-28s round %5lld cycles, push issue (thread 0) %5lld cycles %s\n", names[mode], h[0], h[1],
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
