// Micro-benchmarks of the primitives the chain kernel is built from, on the
// box's B200 (clock64 cycles): mma.sync m16n8k8 TF32 latency / throughput,
// DMMA f64, __syncthreads, and a DSMEM st.async + mbarrier ping-pong between
// two CTAs of a cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void mma_lat(long long* out, float* sink, int n) {
    uint32_t a[4] = {1, 2, 3, 4}, b[2] = {5, 6};
    float d[4] = {0, 0, 0, 0};
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) mma_tf32(d, a, b);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[threadIdx.x] = d[0] + d[1] + d[2] + d[3];
}

__global__ void mma_tput(long long* out, float* sink, int n) {
    uint32_t a[4] = {1, 2, 3, 4}, b[2] = {5, 6};
    float d[8][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_tf32(d[k], a, b);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    float s = 0;
    for (int k = 0; k < 8; ++k) s += d[k][0];
    sink[threadIdx.x] = s;
}

__global__ void dmma_lat(long long* out, double* sink, int n) {
    double a = 1.0, b = 2.0, d0 = 0, d1 = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[threadIdx.x] = d0 + d1;
}

__global__ void sync_cost(long long* out, int n) {
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// two CTAs of a cluster ping-pong a 16-byte payload through st.async +
// mbarrier complete_tx; round trip cycles
__global__ void __cluster_dims__(2, 1, 1) dsmem_pingpong(long long* out, int n) {
    __shared__ __align__(16) float buf[4];
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t bar_l = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t buf_l = (uint32_t)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_l));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    uint32_t peer = rank ^ 1, rbar, rbuf;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar_l), "r"(peer));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbuf) : "r"(buf_l), "r"(peer));
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            const uint32_t par = i & 1;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(bar_l));
            if (rank == 0 || i > 0) {
            }
            if (rank == 0) {
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%1,%1,%1}, [%2];" ::"r"(rbuf), "r"(i), "r"(rbar));
            }
            asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(bar_l), "r"(par));
            if (rank == 1) {
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%1,%1,%1}, [%2];" ::"r"(rbuf), "r"(i), "r"(rbar));
            }
        }
    }
    long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    if (threadIdx.x == 0 && rank == 0) out[0] = t1 - t0;
}

int main() {
    long long *d_out, h[64];
    float* fs;
    double* ds;
    cudaMalloc(&d_out, 64 * 8);
    cudaMalloc(&fs, 4096 * 4);
    cudaMalloc(&ds, 4096 * 8);
    const int n = 1000;
    mma_lat<<<1, 32>>>(d_out, fs, n);
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("mma.sync m16n8k8 tf32 dependent latency: %.1f cycles\n", (double)h[0] / n);
    for (int warps : {1, 4, 8, 16}) {
        mma_tput<<<1, 32 * warps>>>(d_out, fs, n / 8);
        cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
        printf("mma.sync tf32 throughput, %2d warps/SM: %.2f cycles per MMA per SM (%.0f MAC/clk/SM)\n", warps,
               (double)h[0] / (n / 8 * 8 * warps), 1024.0 * (n / 8 * 8 * warps) / h[0]);
    }
    dmma_lat<<<1, 32>>>(d_out, ds, n);
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("mma.sync m8n8k4 f64 dependent latency: %.1f cycles\n", (double)h[0] / n);
    for (int th : {256, 512}) {
        sync_cost<<<1, th>>>(d_out, n);
        cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads (%d threads): %.1f cycles\n", th, (double)h[0] / n);
    }
    dsmem_pingpong<<<2, 32>>>(d_out, n);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("DSMEM st.async+mbarrier round trip: %.1f cycles (%s)\n", (double)h[0] / n, cudaGetErrorString(e));
    return 0;
}
