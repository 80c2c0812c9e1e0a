// Warp-level tensor-core helpers: mma.sync m16n8k8 TF32 with the 3xTF32
// split (a*b ~= ah*bh + ah*bl + al*bh, fp32-class accuracy).
//
// Fragment ownership (PTX ISA, m16n8k8 .tf32): g = lane >> 2, t = lane & 3
//   A (16x8, row): a0 (g, t)   a1 (g+8, t)   a2 (g, t+4)   a3 (g+8, t+4)
//   B (8x8,  col): b0 (t, g)   b1 (t+4, g)
//   C (16x8)     : c0 (g, 2t)  c1 (g, 2t+1) c2 (g+8, 2t)  c3 (g+8, 2t+1)
#pragma once

#include <cstdint>

namespace fasthb {
namespace dev {

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// Round an fp32 bit pattern to the nearest tf32 (ties away from zero) with
// two integer ops — cvt.rna.tf32.f32 is emulated on sm_100a by a long
// sequence.  Finite inputs only (the chain's operands are finite).
__device__ __forceinline__ uint32_t tf32_round(uint32_t bits) { return (bits + 0x1000u) & 0xffffe000u; }

// hi = tf32(x), lo = tf32(x - hi) (x - hi is exact in fp32): the 3xTF32
// product ah*bh + ah*bl + al*bh then carries ~2^-22 relative error.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = tf32_round(__float_as_uint(x));
    lo = tf32_round(__float_as_uint(x - __uint_as_float(hi)));
}

__device__ __forceinline__ void mma_tf32(float& d0, float& d1, float& d2, float& d3, uint32_t a0,
                                         uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// f64 tensor core: D(8x8) += A(8x4) B(4x8), one element of A and B per lane:
//   a0 = A[g][t], b0 = B[t][g], d0/d1 = D[g][2t], D[g][2t+1]
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// acc += A*B in 3xTF32 from fp32 operands: the main product into `m`, the
// two correction products into `c` (two independent accumulator chains).
struct Frag4 {
    float v[4];
};

__device__ __forceinline__ void mma3(Frag4& m, Frag4& c, const float a[4], const float b[2]) {
    uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_tf32(a[i], ah[i], al[i]);
#pragma unroll
    for (int i = 0; i < 2; ++i) split_tf32(b[i], bh[i], bl[i]);
    mma_tf32(m.v[0], m.v[1], m.v[2], m.v[3], ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
    mma_tf32(c.v[0], c.v[1], c.v[2], c.v[3], ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
    mma_tf32(c.v[0], c.v[1], c.v[2], c.v[3], al[0], al[1], al[2], al[3], bh[0], bh[1]);
}

}  // namespace dev
}  // namespace fasthb
