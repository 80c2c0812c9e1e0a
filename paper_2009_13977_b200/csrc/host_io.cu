// Host <-> device transfers of the host-buffer entry (fasth_forward_backward_host)
// by SM copy kernels over the pinned buffers' UVA mappings.
//
// On the B200 boxes a single cudaMemcpyAsync host->device of the chain
// (2.46 MB at d = 784) moves ~22 GB/s (scripts/pcie_probe.py); SMs reading the
// same pinned buffer through its device mapping, with many 16-byte loads in
// flight per thread, keep more PCIe read requests outstanding than the copy
// engine does.  The kernels are plain streaming copies: every thread moves
// kUnroll float4 per iteration, all loads issued before the stores.
#include <algorithm>

#include "fasth_internal.h"

namespace fasthb {
namespace {

constexpr int kUnroll = 8;
constexpr int kCopyThreads = 256;

__global__ void __launch_bounds__(kCopyThreads) copy4_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                                         int64_t n4) {
    const int64_t stride = (int64_t)gridDim.x * kCopyThreads;
    int64_t i = (int64_t)blockIdx.x * kCopyThreads + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n4; i += kUnroll * stride) {
        float4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) __stcs(dst + i + u * stride, v[u]);
    }
    for (; i < n4; i += stride) __stcs(dst + i, __ldcs(src + i));
}

__global__ void copy1_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

}  // namespace

// dst[0..n) = src[0..n) where either side may be a device view of pinned
// host memory; 16-byte aligned buffers take the vector kernel.
cudaError_t launch_stream_copy(const float* src, float* dst, int64_t n, int num_sms, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const bool vec = !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) && n % 4 == 0;
    if (vec) {
        const int64_t n4 = n / 4;
        const int64_t want = (n4 + kCopyThreads * kUnroll - 1) / (kCopyThreads * kUnroll);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms * 4));
        copy4_kernel<<<grid, kCopyThreads, 0, s>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst),
                                               n4);
    } else {
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms * 8));
        copy1_kernel<<<grid, 256, 0, s>>>(src, dst, n);
    }
    return cudaGetLastError();
}

}  // namespace fasthb
