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

struct Segs {
    const float4* src[4];
    float4* dst[4];
    int64_t end[4];  // cumulative float4 counts
    int n;
};

// several 16-byte aligned copies in one launch (the host step's V, X, G)
__global__ void __launch_bounds__(kCopyThreads) copyn_kernel(Segs sg) {
    const int64_t total = sg.end[sg.n - 1];
    const int64_t stride = (int64_t)gridDim.x * kCopyThreads;
    auto at = [&](int64_t k, const float4*& s, float4*& d) {
        int j = 0;
        while (j + 1 < sg.n && k >= sg.end[j]) ++j;
        const int64_t o = k - (j ? sg.end[j - 1] : 0);
        s = sg.src[j] + o, d = sg.dst[j] + o;
    };
    for (int64_t i = (int64_t)blockIdx.x * kCopyThreads + threadIdx.x; i < total; i += kUnroll * stride) {
        float4 v[kUnroll];
        float4* dp[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t k = i + u * stride;
            dp[u] = nullptr;
            if (k < total) {
                const float4* sp;
                at(k, sp, dp[u]);
                v[u] = __ldcs(sp);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (dp[u]) __stcs(dp[u], v[u]);
    }
}

// Streamed upload of the host step (fasth_forward_backward_host): X and G,
// then V's WY blocks in the order the two chains need them (0, q-1, 1, q-2,
// ...).  Each unit (X, G, one block of b columns) is ncb chunks; the CTAs take
// chunks in that order with few in flight per CTA, so units land in order,
// and count every landed chunk (gpu-scope release) in the unit's counter:
// the builder of block i starts once blocks i-1..i+1 are in, the sweep once
// X and G are.  Releases its dependents (the builder) at entry.
__global__ void __launch_bounds__(kCopyThreads) upload_kernel(UploadArgs u) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int nunits = 2 + u.q, nchunks = nunits * u.ncb;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const int unit = c / u.ncb, part = c - unit * u.ncb;
        const float4* src;
        float4* dst;
        int64_t len;
        unsigned* cnt;
        if (unit < 2) {
            src = unit == 0 ? u.x_src : u.g_src;
            dst = unit == 0 ? u.x_dst : u.g_dst;
            len = u.x4;
            cnt = u.xg_cnt;
        } else {
            const int j = unit - 2;  // outside-in: 0, q-1, 1, q-2, ...
            const int k = (j & 1) ? u.q - 1 - (j >> 1) : (j >> 1);
            const int64_t lo = (int64_t)k * u.blk4, hi = min(lo + u.blk4, u.v4);
            src = u.v_src + lo;
            dst = u.v_dst + lo;
            len = hi - lo;
            cnt = u.upc + k;
        }
        const int64_t per = (len + u.ncb - 1) / u.ncb;
        const int64_t b0 = part * per, b1 = min(b0 + per, len);
        float4 v[kUnroll];
        for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += kUnroll * kCopyThreads) {
#pragma unroll
            for (int e = 0; e < kUnroll; ++e) {
                const int64_t i = i0 + e * kCopyThreads;
                if (i < b1) v[e] = __ldcs(src + i);
            }
#pragma unroll
            for (int e = 0; e < kUnroll; ++e) {
                const int64_t i = i0 + e * kCopyThreads;
                if (i < b1) dst[i] = v[e];
            }
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(cnt, 1u);
    }
}

}  // namespace

cudaError_t launch_upload(const UploadArgs& u, int ctas, cudaStream_t s) {
    if (u.ncb < 1 || u.q < 1 || !u.upc || !u.xg_cnt) return cudaErrorInvalidValue;
    const int nchunks = (2 + u.q) * u.ncb;
    upload_kernel<<<std::max(1, std::min(ctas, nchunks)), kCopyThreads, 0, s>>>(u);
    return cudaGetLastError();
}

// dst[j][0..n[j]) = src[j][0..n[j]) for up to 4 segments in one launch when
// every segment is 16-byte aligned with n % 4 == 0, else one launch each.
cudaError_t launch_stream_copy_n(const float* const* src, float* const* dst, const int64_t* n, int nseg, int num_sms,
                                 cudaStream_t s) {
    Segs sg{};
    bool vec = nseg <= 4;
    int64_t tot = 0;
    for (int j = 0; j < nseg && vec; ++j) {
        vec = !((reinterpret_cast<uintptr_t>(src[j]) | reinterpret_cast<uintptr_t>(dst[j])) & 15) && n[j] % 4 == 0;
        if (n[j] <= 0) continue;
        sg.src[sg.n] = reinterpret_cast<const float4*>(src[j]);
        sg.dst[sg.n] = reinterpret_cast<float4*>(dst[j]);
        tot += n[j] / 4;
        sg.end[sg.n++] = tot;
    }
    if (!vec) {
        for (int j = 0; j < nseg; ++j)
            if (cudaError_t e = launch_stream_copy(src[j], dst[j], n[j], num_sms, s); e != cudaSuccess) return e;
        return cudaSuccess;
    }
    if (sg.n == 0) return cudaSuccess;
    const int64_t want = (tot + kCopyThreads * kUnroll - 1) / (kCopyThreads * kUnroll);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms * 4));
    copyn_kernel<<<grid, kCopyThreads, 0, s>>>(sg);
    return cudaGetLastError();
}

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
