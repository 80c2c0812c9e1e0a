// Backward step 2: north_star subsystem (4), the per-reflection gradients.
//
// The reference walks every reflection of a block (fasth.hpp:97-108):
// reconstruct A_{j+1} = H_j A_j, evaluate Eq. (5) (householder_grad,
// householder.hpp:148-179), propagate G_{j+1} = H_j G_j — 3 rank-1 passes
// per reflection.  Here the whole block is one small GEMM in closed form
// (derived from SURVEY App. A.2 with raw, unnormalised vectors; the norms
// cancel):
//
//   Q   = Z'f Z'b^T                                   (BS x BS, K = m)
//   K'  = striu(Q - Q^T)
//   dV_block = -2 ( A Z'b^T + G Z'f^T + 2 V K' )     (d x BS, K = 2m + BS)
//
// where A = activations[i] (block output), G = dA[i] (its gradient) and
// Z'f / Z'b are the T~-applied reductions the forward / backward sweeps
// already computed for the block (no extra pass over d).  All q blocks and
// all row tiles run in parallel: grid (row tiles, q).  dV is written
// straight into the caller's column-major d x n buffer in chain order
// (un-reversed for the V^T leg, svd_layer.hpp:150-151).
#include "fasth_internal.h"

namespace fasthb {
namespace {

constexpr int RT = 32;  // rows per CTA

template <int BS>
__global__ void __launch_bounds__(kThreads) dv_kernel(DvArgs a) {
    constexpr int MC = BS >= 64 ? 32 : 64;  // batch columns per staged chunk (static smem <= 48 KB)
    __shared__ __align__(16) float zfT[MC * BS];  // chunk of Z'f, transposed [l][j]
    __shared__ __align__(16) float zbT[MC * BS];
    __shared__ __align__(16) float As[RT * MC];
    __shared__ __align__(16) float Gs[RT * MC];
    __shared__ __align__(16) float Vr[RT * BS];
    __shared__ __align__(16) float Kp[BS * BS];

    const int tid = threadIdx.x;
    const int i = blockIdx.y;
    const int r0 = blockIdx.x * RT;
    const int m = a.m, WC = a.WC;
    const float* zf = a.zf + (size_t)i * BS * m;
    const float* zb = a.zb + (size_t)i * BS * m;

    constexpr int KPT = (BS * BS + kThreads - 1) / kThreads;  // K' entries per thread
    float kacc[KPT];
#pragma unroll
    for (int u = 0; u < KPT; ++u) kacc[u] = 0.f;
    constexpr int RG = kThreads / BS;  // row groups
    constexpr int RPT = (RT + RG - 1) / RG;
    const int j = tid % BS;
    const int rg = tid / BS;
    float acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = 0.f;

    for (int lc = 0; lc < m; lc += MC) {
        const int mc = min(MC, m - lc);
        __syncthreads();
        for (int idx = tid; idx < BS * MC; idx += kThreads) {
            const int jj = idx / MC, l = idx - jj * MC;
            const bool ok = l < mc;
            zfT[l * BS + jj] = ok ? zf[(size_t)jj * m + lc + l] : 0.f;
            zbT[l * BS + jj] = ok ? zb[(size_t)jj * m + lc + l] : 0.f;
        }
        for (int idx = tid; idx < RT * MC; idx += kThreads) {
            const int r = idx / MC, l = idx - r * MC;
            float av = 0.f, gv = 0.f;
            if (l < mc && r0 + r < a.d_pad) {
                const int gl = lc + l;
                const int g = gl / WC, c = gl - g * WC;
                const size_t off = (((size_t)i * a.ngroups + g) * a.d_pad + r0 + r) * WC + c;
                av = a.tapeA[off];
                gv = a.tapeG[off];
            }
            As[idx] = av;
            Gs[idx] = gv;
        }
        __syncthreads();
        // Q contribution to K' = striu(Zf Zb^T - Zb Zf^T)
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int idx = tid + u * kThreads;
            if (idx < BS * BS) {
                const int k = idx / BS, jj = idx - k * BS;
                if (k < jj) {
                    float s = kacc[u];
                    for (int l = 0; l < mc; ++l)
                        s += zfT[l * BS + k] * zbT[l * BS + jj] - zfT[l * BS + jj] * zbT[l * BS + k];
                    kacc[u] = s;
                }
            }
        }
        for (int l = 0; l < mc; ++l) {
            const float b_ = zbT[l * BS + j], f_ = zfT[l * BS + j];
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int r = rg * RPT + u;
                if (r < RT) acc[u] += As[r * MC + l] * b_ + Gs[r * MC + l] * f_;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int idx = tid + u * kThreads;
        if (idx < BS * BS) Kp[idx] = kacc[u];
    }
    const float* vb = a.Vbl + ((size_t)i * a.d_pad + r0) * BS;
    for (int idx = tid; idx < RT * BS; idx += kThreads)
        Vr[idx] = (r0 + idx / BS < a.d_pad) ? vb[idx] : 0.f;
    __syncthreads();
    for (int k = 0; k < BS; ++k) {
        const float kk = 2.f * Kp[k * BS + j];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int r = rg * RPT + u;
            if (r < RT) acc[u] = fmaf(Vr[r * BS + k], kk, acc[u]);
        }
    }
    const int kc = i * a.b + j;
    if (j < a.b && kc < a.n) {
        const int col = a.reversed ? a.n - 1 - kc : kc;
        float* out = a.dV + (int64_t)col * a.lddv;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int r = r0 + rg * RPT + u;
            if (rg * RPT + u < RT && r < a.d) out[r] = -2.f * acc[u];
        }
    }
}

template <int BS>
cudaError_t launch_dv_t(const DvArgs& a, cudaStream_t s) {
    const dim3 grid((a.d + RT - 1) / RT, a.q);
    dv_kernel<BS><<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dv(const DvArgs& a, cudaStream_t s) {
    switch (a.BS) {
        case 8: return launch_dv_t<8>(a, s);
        case 16: return launch_dv_t<16>(a, s);
        case 32: return launch_dv_t<32>(a, s);
        case 64: return launch_dv_t<64>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
