// Micro-benchmark: per-SM L2 -> shared memory streaming rate of the bulk-copy
// (TMA) engine, the budget the chain sweep's per-step W/V/S stage must fit.
// One CTA per SM, NCTA CTAs, each streaming `bytes` per step through a ring of
// NST stages from an L2-resident buffer; reports cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbs scripts/microbench_stream.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0 try_wait, 1 test_wait spin, 2 try_wait with a 20 ns suspend hint
__global__ void stream_kernel(const float* src, size_t src_floats, int bytes, int nst, int steps,
                              long long* out, int ncopy) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* buf = smem + 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    
    auto issue = [&](int t) {
        const int s = t % nst;
        const char* g = reinterpret_cast<const char*>(src) + (size_t)((t + blockIdx.x * 7) & 63) * bytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes));
        // split into <= 3 copies like the sweep's W / V / S
        int off = 0;
        const int part = (bytes / ncopy + 15) & ~15;
        while (off < bytes) {
            const int n = min(part, bytes - off);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(buf + (size_t)s * bytes + off)),
                "l"(g + off), "r"(n), "r"(smem_u32(&bar[s]))
                : "memory");
            off += n;
        }
    };
    long long t0 = 0;
    if (threadIdx.x == 0) {
        for (int t = 0; t < nst && t < steps; ++t) issue(t);
        t0 = clock64();
        for (int t = 0; t < steps; ++t) {
            const int s = t % nst;
            const uint32_t par = (uint32_t)(t / nst) & 1u;
            if (MODE == 0)
                asm volatile(
                    "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                        smem_u32(&bar[s])),
                    "r"(par)
                    : "memory");
            else if (MODE == 1)
                asm volatile(
                    "{\n.reg .pred P;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                        smem_u32(&bar[s])),
                    "r"(par)
                    : "memory");
            else
                asm volatile(
                    "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 20;\n@!P bra W_%=;\n}\n" ::"r"(
                        smem_u32(&bar[s])),
                    "r"(par)
                    : "memory");
            if (t + nst < steps) issue(t + nst);
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    const size_t n = 4u << 20;  // 16 MB source (L2 resident after first touch)
    float* src;
    cudaMalloc(&src, n * 4);
    cudaMemset(src, 0, n * 4);
    long long* d_out;
    cudaMalloc(&d_out, 1024 * sizeof(long long));
    for (auto k : {stream_kernel<0>, stream_kernel<1>, stream_kernel<2>})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int sizes[] = {4096, 16384, 38912};
  for (int ncopy : {1, 3, 8}) for (int mode = 0; mode < 1; ++mode) {
    auto kern = mode == 0 ? stream_kernel<0> : mode == 1 ? stream_kernel<1> : stream_kernel<2>;
    printf("== wait mode %d (0 try_wait, 1 test_wait spin, 2 try_wait hint 20ns), %d copies per step\n", mode, ncopy);
    for (int ncta : {1, 56}) {
        for (int bytes : sizes) {
            for (int nst : {1, 2, 4, 8}) {
                if ((size_t)nst * bytes + 128 > 227 * 1024) continue;
                const int steps = 200;
                kern<<<ncta, 128, nst * bytes + 128>>>(src, n, bytes, nst, steps, d_out, ncopy);
                kern<<<ncta, 128, nst * bytes + 128>>>(src, n, bytes, nst, steps, d_out, ncopy);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[1024];
                cudaMemcpy(h, d_out, ncta * sizeof(long long), cudaMemcpyDeviceToHost);
                double mx = 0;
                for (int i = 0; i < ncta; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("ctas %3d bytes/step %6d stages %d: %7.1f cycles/step  %6.1f B/clk/SM %s\n", ncta, bytes,
                       nst, mx / steps, bytes / (mx / steps), e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
  }
    return 0;
}
