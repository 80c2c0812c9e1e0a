// Backward step 2: north_star subsystem (4), the per-reflection gradients.
//
// The reference walks every reflection of a block (fasth.hpp:97-108):
// reconstruct A_{j+1} = H_j A_j, evaluate Eq. (5) (householder_grad,
// householder.hpp:148-179), propagate G_{j+1} = H_j G_j — 3 rank-1 passes
// per reflection.  Here the whole block is one small GEMM in closed form
// (derived from SURVEY App. A.2 with raw, unnormalised vectors; the norms
// cancel; the CPU suite checks the algebra, tests/algo_model.py):
//
//   Q   = Z'f Z'b^T                                   (BS x BS, K = m)
//   K'  = striu(Q - Q^T)
//   dV_block = -2 [A | G | V] [Z'b^T ; Z'f^T ; 2 K']  (d x BS, K = 2m + BS)
//
// where A = activations[i] (block output), G = dA[i] (its gradient) and
// Z'f / Z'b are the reductions the forward / backward sweeps already
// produced for the block (no extra pass over d).  Both products run on the
// tensor cores (mma.sync m16n8k8, 3xTF32).  Grid (row tiles, q): all blocks
// and row tiles in parallel; batch columns in chunks of MC so any m works;
// dV goes straight into the caller's column-major d x n buffer in chain
// order (un-reversed for the V^T leg, svd_layer.hpp:150-151), coalesced.
#include "device_prims.cuh"
#include "fasth_internal.h"
#include "mma_tf32.cuh"

namespace fasthb {
namespace {

constexpr int RT = 64;  // rows per CTA

template <int BS>
struct DvShape {
    static constexpr int MC = 64;         // batch columns per chunk
    static constexpr int KA = 2 * MC;     // A|G columns per chunk
    static constexpr int LDA = KA + 4;    // A-operand pitch (== 4 mod 32: conflict-free)
    static constexpr int LDZ = BS + 8;    // B-operand pitch (== 8 mod 32)
    static constexpr int LDV = BS + 4;    // V rows (== Vbl pitch)
    static constexpr int LDC = RT + 1;    // transposed output staging
    static constexpr int TILES = (RT / 16) * (BS / 8);
    static constexpr int TPW = (TILES + 7) / 8;  // tiles per warp (8 warps)
};

template <int BS>
__global__ void __launch_bounds__(kThreads) dv_kernel(DvArgs a) {
    using S = DvShape<BS>;
    constexpr int MC = S::MC, KA = S::KA, LDA = S::LDA, LDZ = S::LDZ, LDV = S::LDV, LDC = S::LDC;
    constexpr int TPW = S::TPW;
    extern __shared__ __align__(16) float sm[];
    float* Aop = sm;                      // [RT][LDA]   A | G rows of this chunk
    float* Bop = Aop + RT * LDA;          // [KA][LDZ]   Z'b^T ; Z'f^T
    float* Vr = Bop + KA * LDZ;           // [RT][LDV]   V rows
    float* Kp = Vr + RT * LDV;            // [BS][LDZ]   2 K' (Q first)
    float* Ct = Kp + BS * LDZ;            // [BS][LDC]   output, transposed

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const int i = blockIdx.y;
    const int r0 = blockIdx.x * RT;
    const int m = a.m, WC = a.WC;
    const float* zf = a.zf + (size_t)i * BS * m;
    const float* zb = a.zb + (size_t)i * BS * m;

    // V rows for the final K-slice (needed only after the chunks)
    const float* vb = a.Vbl + ((size_t)i * a.d_pad + r0) * LDV;
    for (int idx = tid; idx < RT * LDV / 4; idx += kThreads) {
        const bool ok = r0 + idx / (LDV / 4) < a.d_pad;
        dev::cp_async16(Vr + idx * 4, ok ? vb + idx * 4 : a.Vbl, ok);
    }

    dev::Frag4 acc[TPW][2];  // [tile][main, correction]
#pragma unroll
    for (int u = 0; u < TPW; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][0].v[v] = acc[u][1].v[v] = 0.f;
    // Q tile of this warp (BS/16 x BS/8 tiles of 16x8; BS<=64 -> <= 32 tiles, 8 warps)
    constexpr int QT = (BS / 16) * (BS / 8);
    constexpr int QPW = (QT + 7) / 8;
    dev::Frag4 qacc[QPW][2];
#pragma unroll
    for (int u = 0; u < QPW; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) qacc[u][0].v[v] = qacc[u][1].v[v] = 0.f;

    for (int lc = 0; lc < m; lc += MC) {
        const int mc = min(MC, m - lc);
        __syncthreads();
        // all of this chunk's loads in flight at once (cp.async)
        for (int idx = tid; idx < BS * MC; idx += kThreads) {
            const int j = idx / MC, l = idx - j * MC;
            const bool ok = l < mc;
            const size_t off = ok ? (size_t)j * m + lc + l : 0;
            dev::cp_async4(Bop + l * LDZ + j, zb + off, ok);
            dev::cp_async4(Bop + (MC + l) * LDZ + j, zf + off, ok);
        }
        // A | G rows from the tapes ([q][ngroups][d_pad][WC], WC % 4 == 0);
        // columns of the last group beyond m hold zeros (the sweeps load
        // zeros there), so whole float4s are safe to take.
        for (int idx = tid; idx < RT * (MC / 4); idx += kThreads) {
            const int r = idx / (MC / 4), l4 = (idx - r * (MC / 4)) * 4;
            const bool ok = l4 < mc && r0 + r < a.d_pad;
            size_t off = 0;
            if (ok) {
                const int gl = lc + l4;
                const int gg = gl / WC, c = gl - gg * WC;
                off = (((size_t)i * a.ngroups + gg) * a.d_pad + r0 + r) * WC + c;
            }
            dev::cp_async16(Aop + r * LDA + l4, a.tapeA + off, ok);
            dev::cp_async16(Aop + r * LDA + MC + l4, a.tapeG + off, ok);
        }
        dev::cp_async_commit();
        dev::cp_async_wait_all();
        __syncthreads();
        // Q += Z'f Z'b^T over this chunk: A[k][l] = Bop[MC + l][k], B[l][j] = Bop[l][j]
#pragma unroll
        for (int u = 0; u < QPW; ++u) {
            const int qt = warp + u * 8;
            if (qt < QT) {
                const int m0 = (qt / (BS / 8)) * 16, n0 = (qt % (BS / 8)) * 8;
                for (int k0 = 0; k0 < MC; k0 += 8) {
                    const float* fa = Bop + (MC + k0 + tq) * LDZ + m0 + g;
                    const float av[4] = {fa[0], fa[8], fa[4 * LDZ], fa[4 * LDZ + 8]};
                    const float bv[2] = {Bop[(k0 + tq) * LDZ + n0 + g], Bop[(k0 + tq + 4) * LDZ + n0 + g]};
                    dev::mma3(qacc[u][0], qacc[u][1], av, bv);
                }
            }
        }
        // [A | G] [Z'b^T ; Z'f^T]
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const int tile = warp + u * 8;
            if (tile < S::TILES) {
                const int rr = (tile / (BS / 8)) * 16, n0 = (tile % (BS / 8)) * 8;
                for (int k0 = 0; k0 < KA; k0 += 8) {
                    const float* ar = Aop + (rr + g) * LDA + k0 + tq;
                    const float av[4] = {ar[0], ar[8 * LDA], ar[4], ar[8 * LDA + 4]};
                    const float bv[2] = {Bop[(k0 + tq) * LDZ + n0 + g], Bop[(k0 + tq + 4) * LDZ + n0 + g]};
                    dev::mma3(acc[u][0], acc[u][1], av, bv);
                }
            }
        }
    }
    // K' = striu(Q - Q^T), times 2, into Kp[k][j]
    __syncthreads();
#pragma unroll
    for (int u = 0; u < QPW; ++u) {
        const int qt = warp + u * 8;
        if (qt < QT) {
            const int m0 = (qt / (BS / 8)) * 16, n0 = (qt % (BS / 8)) * 8;
            float* q0 = Kp + (m0 + g) * LDZ + n0 + 2 * tq;
            q0[0] = qacc[u][0].v[0] + qacc[u][1].v[0];
            q0[1] = qacc[u][0].v[1] + qacc[u][1].v[1];
            q0[8 * LDZ] = qacc[u][0].v[2] + qacc[u][1].v[2];
            q0[8 * LDZ + 1] = qacc[u][0].v[3] + qacc[u][1].v[3];
        }
    }
    dev::cp_async_commit();
    dev::cp_async_wait_all();  // V rows
    __syncthreads();
    // in place: Kp[k][j] = 2 (Q[k][j] - Q[j][k]) for k < j, else 0.  Each
    // thread reads both mirror entries before the barrier, then writes.
    float kv[(BS * BS + kThreads - 1) / kThreads];
#pragma unroll
    for (int u = 0; u < (BS * BS + kThreads - 1) / kThreads; ++u) {
        const int idx = tid + u * kThreads;
        float v = 0.f;
        if (idx < BS * BS) {
            const int k = idx / BS, j = idx - k * BS;
            if (k < j) v = 2.f * (Kp[k * LDZ + j] - Kp[j * LDZ + k]);
        }
        kv[u] = v;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < (BS * BS + kThreads - 1) / kThreads; ++u) {
        const int idx = tid + u * kThreads;
        if (idx < BS * BS) Kp[(idx / BS) * LDZ + idx % BS] = kv[u];
    }
    __syncthreads();
    // + V (2 K')
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        const int tile = warp + u * 8;
        if (tile < S::TILES) {
            const int rr = (tile / (BS / 8)) * 16, n0 = (tile % (BS / 8)) * 8;
#pragma unroll
            for (int k0 = 0; k0 < BS; k0 += 8) {
                const float* vr = Vr + (rr + g) * LDV + k0 + tq;
                const float av[4] = {vr[0], vr[8 * LDV], vr[4], vr[8 * LDV + 4]};
                const float bv[2] = {Kp[(k0 + tq) * LDZ + n0 + g], Kp[(k0 + tq + 4) * LDZ + n0 + g]};
                dev::mma3(acc[u][0], acc[u][1], av, bv);
            }
            // stage -2 * result transposed: Ct[j][r]
            const int j = n0 + 2 * tq, r = rr + g;
            Ct[j * LDC + r] = -2.f * (acc[u][0].v[0] + acc[u][1].v[0]);
            Ct[(j + 1) * LDC + r] = -2.f * (acc[u][0].v[1] + acc[u][1].v[1]);
            Ct[j * LDC + r + 8] = -2.f * (acc[u][0].v[2] + acc[u][1].v[2]);
            Ct[(j + 1) * LDC + r + 8] = -2.f * (acc[u][0].v[3] + acc[u][1].v[3]);
        }
    }
    __syncthreads();
    for (int idx = tid; idx < BS * RT; idx += kThreads) {
        const int j = idx / RT, r = idx - j * RT;
        const int kc = i * a.b + j;
        if (j < a.b && kc < a.n && r0 + r < a.d) {
            const int col = a.reversed ? a.n - 1 - kc : kc;
            a.dV[(int64_t)col * a.lddv + r0 + r] = Ct[j * LDC + r];
        }
    }
}

template <int BS>
size_t dv_smem() {
    using S = DvShape<BS>;
    return sizeof(float) * ((size_t)RT * S::LDA + (size_t)S::KA * S::LDZ + (size_t)RT * S::LDV +
                            (size_t)BS * S::LDZ + (size_t)BS * S::LDC);
}

template <int BS>
cudaError_t launch_dv_t(const DvArgs& a, cudaStream_t s) {
    const size_t smem = dv_smem<BS>();
    {
        cudaError_t e = ensure_smem(reinterpret_cast<const void*>(dv_kernel<BS>), smem);
        if (e != cudaSuccess) return e;
    }
    const dim3 grid((a.d + RT - 1) / RT, a.q);
    dv_kernel<BS><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dv(const DvArgs& a, cudaStream_t s) {
    switch (a.BS) {
        case 16: return launch_dv_t<16>(a, s);
        case 32: return launch_dv_t<32>(a, s);
        case 64: return launch_dv_t<64>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
