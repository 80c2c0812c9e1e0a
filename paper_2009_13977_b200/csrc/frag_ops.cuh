// Warp-level fragment helpers shared by the chain kernels (chain_v2.cu,
// chain_panel.cu): mma.sync m16n8k8 TF32 with the round-to-nearest 3xTF32
// split, fragment-ordered shared loads, the C-fragment -> B-fragment scatter,
// mbarrier / bulk-copy / DSMEM-push primitives on 32-bit shared addresses.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fasthb {
namespace fo {

// 3xTF32 split with round-to-nearest hi: hi = rn_tf32(x), lo = x - hi (exact
// in fp32, either sign, so the tensor core's truncation of lo is unbiased).
__device__ __forceinline__ uint32_t hi_rn(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
__device__ __forceinline__ float lo_rn(float x) { return x - __uint_as_float(hi_rn(x)); }

__device__ __forceinline__ void hmma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A fragment (m16n8k8 .tf32: a0 (g,tq) a1 (g+8,tq) a2 (g,tq+4) a3 (g+8,tq+4)), split
struct AFrag {
    uint32_t h[4], l[4];
};
__device__ __forceinline__ AFrag make_a(float a0, float a1, float a2, float a3) {
    AFrag f;
    const float v[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f.h[i] = hi_rn(v[i]);
        f.l[i] = __float_as_uint(v[i] - __uint_as_float(f.h[i]));
    }
    return f;
}

// m += ah bh ; c1 += ah bl ; c2 += al bh   (3xTF32, three independent chains)
__device__ __forceinline__ void mma3s(float (&m)[4], float (&c1)[4], float (&c2)[4], const AFrag& a,
                                      float bh0, float bh1, float bl0, float bl1) {
    const uint32_t B0 = __float_as_uint(bh0), B1 = __float_as_uint(bh1);
    hmma(m, a.h[0], a.h[1], a.h[2], a.h[3], B0, B1);
    hmma(c1, a.h[0], a.h[1], a.h[2], a.h[3], __float_as_uint(bl0), __float_as_uint(bl1));
    hmma(c2, a.l[0], a.l[1], a.l[2], a.l[3], B0, B1);
}

template <int N>
__device__ __forceinline__ void lds_vec(float (&r)[N], const float* p) {
    static_assert(N % 2 == 0, "vec");
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N; i += 4) {
            const float4 v = *reinterpret_cast<const float4*>(p + i);
            r[i] = v.x, r[i + 1] = v.y, r[i + 2] = v.z, r[i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; i += 2) {
            const float2 v = *reinterpret_cast<const float2*>(p + i);
            r[i] = v.x, r[i + 1] = v.y;
        }
    }
}

// C fragment of a 16x8 tile (rows g, g+8; cols 2tq, 2tq+1) -> B-fragment
// order of its transposed use as a K=16 x N=8 operand: consumer lane
// 4c + (rho & 3), slot 2*(rho >> 3) + ((rho >> 2) & 1); hi = raw, lo split.
__device__ __forceinline__ void scatter_cb(float* hi, float* lo, const float (&v)[4], int g, int tq,
                                           float s) {
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 2 * tq + e;
            const int o = (4 * c + (g & 3)) * 4 + 2 * e2 + (g >> 2);
            const float x = s * v[e2 * 2 + e];
            const uint32_t h = hi_rn(x);
            hi[o] = __uint_as_float(h);
            lo[o] = x - __uint_as_float(h);
        }
}

// The same B-fragment buffer with its 16-byte groups swizzled: group f lives
// at f ^ (((f >> 3) & 1) << 2).  The producer's four tq lanes of a row then
// cover 8 bank groups instead of 4 (2-way instead of 4-way conflicts on every
// store); the consumer reads group swz4(lane) (an involution) with one
// 16-byte load as before.
__device__ __forceinline__ int swz4(int f) { return f ^ (((f >> 3) & 1) << 2); }
__device__ __forceinline__ void scatter_cb_swz(float* hi, float* lo, const float (&v)[4], int g, int tq,
                                               float s) {
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 2 * tq + e;
            const int o = swz4(4 * c + (g & 3)) * 4 + 2 * e2 + (g >> 2);
            const float x = s * v[e2 * 2 + e];
            const uint32_t h = hi_rn(x);
            hi[o] = __uint_as_float(h);
            lo[o] = x - __uint_as_float(h);
        }
}

// pipelined step: spin until counter >= target (acquire, gpu scope), then make
// the generic-proxy writes it published visible to the bulk-copy engine
__device__ __forceinline__ void wait_counter(const unsigned* c, unsigned target) {
    unsigned v;
    while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= target) break;
        __nanosleep(64);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// wait_counter for producers in other grids that may not run yet: gives up
// after ~2^24 polls (seconds) instead of hanging the GPU if a count is
// never reached; the results are then wrong and the parity tests say so
__device__ __forceinline__ void wait_counter_bounded(const unsigned* c, unsigned target) {
    unsigned v;
    for (unsigned it = 0; it < (1u << 24); ++it) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= target) break;
        __nanosleep(64);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait_u32(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
// re-arming a barrier that publishes nothing of this thread's: a relaxed
// arrive (a release arrive waits for the thread's outstanding global stores)
__device__ __forceinline__ void mbar_expect_relaxed_u32(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_u32(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_u32(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void push4(uint32_t raddr, const float (&v)[4], uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(rbar)
        : "memory");
}


}  // namespace fo
}  // namespace fasthb
