// A/B probe for north_star subsystem (3) at batch 32: one chain step of the
// small-batch sweep on the 5th-generation tensor cores (tcgen05 + TMEM) versus
// the same step on the legacy mma.sync path the production sweep uses
// (csrc/chain_v2.cu), both as ONE CTA holding a 128-row slab of X (d x 32),
// b = 32, so the cluster exchange (identical for both) is left out:
//
//   L   = W^T X          (b x m partial over the slab's rows)
//   X  <- X - 2 V L      (the block update; in the sweep L is first summed
//                          over the cluster's CTAs)
//
// tcgen05 variant: X lives in TMEM as the update's fp32 accumulator (128 lanes
// x 32 columns); per step
//   tcgen05.ld X -> split hi/lo -> st.shared as the K-major A operand X^T
//   (M = 128: 32 batch rows + zero padding, 128B swizzle)      [warps 0-3]
//   12 x 4 tcgen05.mma.kind::tf32 (3xTF32, K = 128) -> L^T in TMEM, commit
//   tcgen05.ld L^T -> -2 L split -> st.shared as the B operand Z (N = 32)
//   12 tcgen05.mma (3xTF32, K = 32) accumulate into X, commit      [warp 4]
// mma.sync variant: X in registers as C fragments (8 warps x one 16-row tile),
// 3xTF32 m16n8k8 for both products, partials combined through shared memory
// (the production sweep's phase-1 / phase-2 structure within one CTA).
//
// Both report cycles per step (clock64, 64 steps after 4 warm-up steps) and
// check X against a host f64 recurrence.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcp scripts/tc_chain_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

constexpr int RC = 128, M = 32, B = 32;
constexpr int STEPS = 64, WARM = 4;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t hi_rn(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }

// ---------------------------------------------------------------- tcgen05 ----
__device__ __forceinline__ void mb_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P;\nLW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra LW_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {  // K-major, 128B swizzle, SBO 1024
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((1024u >> 4) & 0x3FFFu) << 32) | (1ull << 46) |
           (2ull << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
        "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
        "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
        "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
        "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
        "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// byte offset of element (row, k) in a K-major SW128 tile set: K-blocks of 32
// floats, each rows x 128 B in 8-row groups of 1024 B, 16-byte chunks XORed
// with (row & 7)
__device__ __forceinline__ uint32_t sw_off(int row, int k, int rows) {
    const int kb = k >> 5, c = k & 31;
    return (uint32_t)(kb * rows * 128 + (row >> 3) * 1024 + (row & 7) * 128 + ((((c >> 2) ^ (row & 7))) << 4) +
                      (c & 3) * 4);
}

// smem: XtH XtL (128 rows x 128 K: 64 KB each), WH WL (32 x 128: 16 KB each),
//       VH VL (128 x 32: 16 KB each), ZH ZL (32 x 32: 4 KB each), bars
constexpr int XT_B = 128 * 128 * 4, W_B = 32 * 128 * 4, V_B = 128 * 32 * 4, Z_B = 32 * 32 * 4;
constexpr int TC_SMEM = 2 * XT_B + 2 * W_B + 2 * V_B + 2 * Z_B + 64 + 1024;

__global__ void __launch_bounds__(192, 1) tc_step_kernel(const float* __restrict__ X0, const float* __restrict__ W,
                                                         const float* __restrict__ V, float* __restrict__ Xout,
                                                         long long* cyc) {
    long long ph[4] = {0, 0, 0, 0}, tp = 0;  // thread 0: cycles per phase
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t *XtH = sm, *XtL = XtH + XT_B, *WH = XtL + XT_B, *WL = WH + W_B, *VH = WL + W_B, *VL = VH + V_B;
    uint8_t *ZH = VL + V_B, *ZL = ZH + Z_B;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ZL + Z_B);
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t bar_p = su32(bars), bar_u = su32(bars + 1);
    // operands: W^T as B of the partial (N = b rows, K = RC), V as A of the update (M = RC, K = b)
    for (int e = tid; e < B * RC; e += blockDim.x) {
        const int j = e / RC, r = e % RC;  // W[r][j], column-major d x b input
        const float w = W[j * RC + r], wh = __uint_as_float(hi_rn(w));
        *reinterpret_cast<float*>(WH + sw_off(j, r, B)) = wh;
        *reinterpret_cast<float*>(WL + sw_off(j, r, B)) = w - wh;
        const float v = V[j * RC + r], vh = __uint_as_float(hi_rn(v));
        *reinterpret_cast<float*>(VH + sw_off(r, j, RC)) = vh;
        *reinterpret_cast<float*>(VL + sw_off(r, j, RC)) = v - vh;
    }
    for (int e = tid; e < 2 * XT_B / 4; e += blockDim.x) reinterpret_cast<float*>(XtH)[e] = 0.f;  // padding rows
    if (tid == 0) {
        mb_init(bar_p, 1);
        mb_init(bar_u, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(holder)), "r"(64)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *holder;
    const uint32_t tX = tmem, tL = tmem + 32;
    // X0 into TMEM (warps 0-3: lane = row)
    if (warp < 4) {
        float x[32];
        const int r = warp * 32 + lane;
#pragma unroll
        for (int l = 0; l < 32; ++l) x[l] = X0[l * RC + r];
        tmem_st32(tX + ((uint32_t)(warp * 32) << 16), x);
    }
    // instruction descriptors: D f32, A/B tf32, K-major, N = 32, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t ph_p = 0, ph_u = 0;
    long long t0 = 0;
    for (int s = 0; s < WARM + STEPS; ++s) {
        if (s == WARM) t0 = clock64();
        fence_before();
        __syncthreads();
        fence_after();
        tp = clock64();
        // 1. X -> X^T operand (hi / lo)
        if (warp < 4) {
            float x[32];
            const int r = warp * 32 + lane;
            tmem_ld32(tX + ((uint32_t)(warp * 32) << 16), x);
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                const float h = __uint_as_float(hi_rn(x[l]));
                *reinterpret_cast<float*>(XtH + sw_off(l, r, 128)) = h;
                *reinterpret_cast<float*>(XtL + sw_off(l, r, 128)) = x[l] - h;
            }
        }
        fence_async();
        fence_before();
        __syncthreads();
        fence_after();
        if (tid == 0 && s >= WARM) { const long long t = clock64(); ph[0] += t - tp; tp = t; }
        // 2. L^T = X^T W  (M = 128 (32 used), N = 32, K = 128), 3xTF32
        if (warp == 4 && lane == 0) {
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t ao = kb * 128 * 128 + ks * 32, bo = kb * B * 128 + ks * 32;
                    const uint64_t ah = sdesc(su32(XtH) + ao), al = sdesc(su32(XtL) + ao);
                    const uint64_t bh = sdesc(su32(WH) + bo), bl = sdesc(su32(WL) + bo);
                    mma_tf32(tL, al, bh, idesc, (kb | ks) ? 1u : 0u);
                    mma_tf32(tL, ah, bl, idesc, 1u);
                    mma_tf32(tL, ah, bh, idesc, 1u);
                }
            commit(bar_p);
        }
        // 3. L^T -> Z = -2 L as the update's B operand (N = m rows, K = b)
        if (warp == 0) {
            mb_wait(bar_p, ph_p);
            fence_after();
            float lz[32];
            if (tid == 0 && s >= WARM) { const long long t = clock64(); ph[1] += t - tp; tp = t; }
            tmem_ld32(tL, lz);  // lane = batch column l, values over j
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float z = -2.f * lz[j], h = __uint_as_float(hi_rn(z));
                *reinterpret_cast<float*>(ZH + sw_off(lane, j, 32)) = h;
                *reinterpret_cast<float*>(ZL + sw_off(lane, j, 32)) = z - h;
            }
        }
        ph_p ^= 1;
        fence_async();
        fence_before();
        __syncthreads();
        fence_after();
        if (tid == 0 && s >= WARM) { const long long t = clock64(); ph[2] += t - tp; tp = t; }
        // 4. X += V Z^T  (M = 128, N = 32, K = 32), 3xTF32, into the X accumulator
        if (warp == 4 && lane == 0) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ah = sdesc(su32(VH) + ks * 32), al = sdesc(su32(VL) + ks * 32);
                const uint64_t bh = sdesc(su32(ZH) + ks * 32), bl = sdesc(su32(ZL) + ks * 32);
                mma_tf32(tX, al, bh, idesc, 1u);
                mma_tf32(tX, ah, bl, idesc, 1u);
                mma_tf32(tX, ah, bh, idesc, 1u);
            }
            commit(bar_u);
        }
        mb_wait(bar_u, ph_u);
        ph_u ^= 1;
        if (tid == 0 && s >= WARM) { const long long t = clock64(); ph[3] += t - tp; tp = t; }
    }
    const long long t1 = clock64();
    if (tid == 0)
        printf("tcgen05 phases (cycles/step): X tmem->smem operand %.0f | partial MMA issue->ready %.0f | "
               "L tmem->Z operand %.0f | update MMA issue->done %.0f\n",
               ph[0] / (double)STEPS, ph[1] / (double)STEPS, ph[2] / (double)STEPS, ph[3] / (double)STEPS);
    fence_after();
    if (warp < 4) {
        float x[32];
        const int r = warp * 32 + lane;
        tmem_ld32(tX + ((uint32_t)(warp * 32) << 16), x);
#pragma unroll
        for (int l = 0; l < 32; ++l) Xout[l * RC + r] = x[l];
    }
    if (tid == 0) *cyc = t1 - t0;
    fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64) : "memory");
}

// ---------------------------------------------------------------- mma.sync ----
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 8 row warps, one 16-row tile each, 4 n-tiles of 8 batch columns (X as C fragments)
__global__ void __launch_bounds__(256, 1) hmma_step_kernel(const float* __restrict__ X0, const float* __restrict__ W,
                                                           const float* __restrict__ V, float* __restrict__ Xout,
                                                           long long* cyc) {
    extern __shared__ float hsm[];
    auto Ws = reinterpret_cast<float(*)[B + 4]>(hsm);
    auto Vs = reinterpret_cast<float(*)[B + 4]>(hsm + RC * (B + 4));
    auto Xs = reinterpret_cast<float(*)[RC + 4]>(hsm + 2 * RC * (B + 4));
    auto red = reinterpret_cast<float(*)[B][M + 4]>(hsm + 2 * RC * (B + 4) + M * (RC + 4));
    auto Zs = reinterpret_cast<float(*)[M + 4]>(hsm + 2 * RC * (B + 4) + M * (RC + 4) + 8 * B * (M + 4));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    for (int e = tid; e < B * RC; e += 256) {
        const int j = e / RC, r = e % RC;
        Ws[r][j] = W[j * RC + r];
        Vs[r][j] = V[j * RC + r];
    }
    float x[4][4];  // n-tile nt: rows warp*16 + g (+8), cols nt*8 + 2tq (+1)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) x[nt][e] = X0[(nt * 8 + 2 * tq + (e & 1)) * RC + warp * 16 + g + 8 * (e >> 1)];
    __syncthreads();
    long long t0 = 0;
    for (int s = 0; s < WARM + STEPS; ++s) {
        if (s == WARM) t0 = clock64();
        // X^T rows for the B operand of L = W^T X (k = row, n = batch)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) Xs[nt * 8 + 2 * tq + (e & 1)][warp * 16 + g + 8 * (e >> 1)] = x[nt][e];
        __syncwarp();
        // partial over this warp's 16 rows: L_w (b x m) = W_rows^T X_rows; A = W^T (m16 = j, k8 = rows)
        float pm[2][4][4] = {}, pc[2][4][4] = {};
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int r0 = warp * 16 + ks * 8;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const float a[4] = {Ws[r0 + tq][mt * 16 + g], Ws[r0 + tq][mt * 16 + g + 8], Ws[r0 + tq + 4][mt * 16 + g],
                                    Ws[r0 + tq + 4][mt * 16 + g + 8]};
                uint32_t ah[4], al[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) ah[i] = hi_rn(a[i]), al[i] = __float_as_uint(a[i] - __uint_as_float(ah[i]));
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const float b0 = Xs[nt * 8 + g][r0 + tq], b1 = Xs[nt * 8 + g][r0 + tq + 4];
                    const uint32_t bh0 = hi_rn(b0), bh1 = hi_rn(b1);
                    hmma(pm[mt][nt], ah, bh0, bh1);
                    hmma(pc[mt][nt], ah, __float_as_uint(b0 - __uint_as_float(bh0)), __float_as_uint(b1 - __uint_as_float(bh1)));
                    hmma(pc[mt][nt], al, bh0, bh1);
                }
            }
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    red[warp][mt * 16 + g + 8 * (e >> 1)][nt * 8 + 2 * tq + (e & 1)] = pm[mt][nt][e] + pc[mt][nt][e];
        __syncthreads();
        // combine over the 8 row warps (fixed order), Z = -2 L
        for (int e = tid; e < B * M; e += 256) {
            const int j = e / M, l = e % M;
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) sum += red[w][j][l];
            Zs[j][l] = -2.f * sum;
        }
        __syncthreads();
        // update: X_rows += V_rows Z (A = V rows (m16 rows, k8 = j), B = Z (k = j, n = batch))
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const int r = warp * 16 + g, k = ks * 8 + tq;
            const float a[4] = {Vs[r][k], Vs[r + 8][k], Vs[r][k + 4], Vs[r + 8][k + 4]};
            uint32_t ah[4], al[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) ah[i] = hi_rn(a[i]), al[i] = __float_as_uint(a[i] - __uint_as_float(ah[i]));
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const float b0 = Zs[k][nt * 8 + g], b1 = Zs[k + 4][nt * 8 + g];
                const uint32_t bh0 = hi_rn(b0), bh1 = hi_rn(b1);
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                hmma(x[nt], ah, bh0, bh1);
                hmma(c, ah, __float_as_uint(b0 - __uint_as_float(bh0)), __float_as_uint(b1 - __uint_as_float(bh1)));
                hmma(c, al, bh0, bh1);
#pragma unroll
                for (int e = 0; e < 4; ++e) x[nt][e] += c[e];
            }
        }
        __syncthreads();
    }
    const long long t1 = clock64();
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) Xout[(nt * 8 + 2 * tq + (e & 1)) * RC + warp * 16 + g + 8 * (e >> 1)] = x[nt][e];
    if (tid == 0) *cyc = t1 - t0;
}

int main() {
    std::vector<float> X(M * RC), W(B * RC), V(B * RC);
    srand(7);
    auto rnd = [] { return (float)((rand() / (double)RAND_MAX) * 2.0 - 1.0); };
    for (auto& v : X) v = rnd();
    // W, V small so the 68-step recurrence stays bounded: X <- (I - 2 V W^T) X
    for (auto& v : W) v = 0.05f * rnd();
    for (auto& v : V) v = 0.05f * rnd();
    // host f64 reference of WARM + STEPS steps
    std::vector<double> Xr(X.begin(), X.end());
    for (int s = 0; s < WARM + STEPS; ++s) {
        std::vector<double> L(B * M, 0.0);
        for (int j = 0; j < B; ++j)
            for (int l = 0; l < M; ++l) {
                double a = 0;
                for (int r = 0; r < RC; ++r) a += (double)W[j * RC + r] * Xr[l * RC + r];
                L[j * M + l] = a;
            }
        for (int l = 0; l < M; ++l)
            for (int r = 0; r < RC; ++r) {
                double a = 0;
                for (int j = 0; j < B; ++j) a += (double)V[j * RC + r] * L[j * M + l];
                Xr[l * RC + r] -= 2.0 * a;
            }
    }
    float *dX, *dW, *dV, *dO;
    long long* dc;
    CK(cudaMalloc(&dX, X.size() * 4));
    CK(cudaMalloc(&dW, W.size() * 4));
    CK(cudaMalloc(&dV, V.size() * 4));
    CK(cudaMalloc(&dO, X.size() * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice));
    auto check = [&](const char* name) {
        std::vector<float> O(X.size());
        long long c = 0;
        CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
        double num = 0, den = 0;
        for (size_t i = 0; i < O.size(); ++i) num += (O[i] - Xr[i]) * (O[i] - Xr[i]), den += Xr[i] * Xr[i];
        printf("{\"variant\": \"%s\", \"cycles_per_step\": %.1f, \"rel_err_vs_f64\": %.3e}\n", name, (double)c / STEPS,
               std::sqrt(num / den));
    };
    CK(cudaFuncSetAttribute(tc_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
    const int H_SMEM = (2 * RC * (B + 4) + M * (RC + 4) + 8 * B * (M + 4) + B * (M + 4)) * 4;
    CK(cudaFuncSetAttribute(hmma_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, H_SMEM));
    for (int rep = 0; rep < 3; ++rep) {
        tc_step_kernel<<<1, 192, TC_SMEM>>>(dX, dW, dV, dO, dc);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        check("tcgen05 (X in TMEM, 3xTF32 kind::tf32)");
        hmma_step_kernel<<<1, 256, H_SMEM>>>(dX, dW, dV, dO, dc);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        check("mma.sync (X in registers, 3xTF32 m16n8k8)");
    }
    return 0;
}
