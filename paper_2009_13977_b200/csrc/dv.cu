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
// produced for the block (no extra pass over d).  Grid (row tiles, q): all
// blocks and row tiles in parallel.  Batch columns are processed in chunks
// of MC so any m works; dV goes straight into the caller's column-major
// d x n buffer in chain order (un-reversed for the V^T leg,
// svd_layer.hpp:150-151) with coalesced column writes.
#include "device_prims.cuh"
#include "fasth_internal.h"

namespace fasthb {
namespace {

constexpr int RT = 64;  // rows per CTA

template <int BS>
struct DvShape {
    static constexpr int MC = BS >= 64 ? 32 : 64;       // batch columns per chunk
    static constexpr int KA = 2 * MC;                    // A|G columns per chunk
    static constexpr int LDA = KA + 4;                   // smem pitch of the A operand
    static constexpr int LDZ = BS + 1;                   // smem pitch of Z'^T chunks
    static constexpr int JT = BS >= 16 ? BS / 16 : 1;    // output columns per thread
    static constexpr int RTH = RT * BS / (kThreads * JT);  // output rows per thread (4)
};

template <int BS>
__global__ void __launch_bounds__(kThreads) dv_kernel(DvArgs a) {
    using S = DvShape<BS>;
    constexpr int MC = S::MC, KA = S::KA, LDA = S::LDA, LDZ = S::LDZ, JT = S::JT, RTH = S::RTH;
    extern __shared__ __align__(16) float sm[];
    float* Aop = sm;                         // [RT][LDA]    A | G rows of this chunk
    float* Bop = Aop + RT * LDA;             // [KA][LDZ]    Z'b^T ; Z'f^T
    float* Vr = Bop + KA * LDZ;              // [RT][BS+1]   V rows
    float* Kp = Vr + RT * (BS + 1);          // [BS][LDZ]    2 K'
    float* Ct = Kp + BS * LDZ;               // [BS][RT+1]   output, transposed

    const int tid = threadIdx.x;
    const int i = blockIdx.y;
    const int r0 = blockIdx.x * RT;
    const int m = a.m, WC = a.WC;
    const float* zf = a.zf + (size_t)i * BS * m;
    const float* zb = a.zb + (size_t)i * BS * m;

    // thread tile: rows rt*RTH .. +RTH-1, columns jt*JT .. +JT-1
    const int jt = tid % (BS / JT), rt = tid / (BS / JT);
    float acc[RTH][JT];
#pragma unroll
    for (int u = 0; u < RTH; ++u)
#pragma unroll
        for (int v = 0; v < JT; ++v) acc[u][v] = 0.f;
    constexpr int KPT = (BS * BS + kThreads - 1) / kThreads;
    float kacc[KPT];
#pragma unroll
    for (int u = 0; u < KPT; ++u) kacc[u] = 0.f;

    for (int lc = 0; lc < m; lc += MC) {
        const int mc = min(MC, m - lc);
        __syncthreads();
        // all of this chunk's loads in flight at once (cp.async):
        // Z'b^T, Z'f^T: coalesced along l, conflict-free transposed store
        for (int idx = tid; idx < BS * MC; idx += kThreads) {
            const int j = idx / MC, l = idx - j * MC;
            const bool ok = l < mc;
            const size_t off = ok ? (size_t)j * m + lc + l : 0;
            dev::cp_async4(Bop + l * LDZ + j, zb + off, ok);
            dev::cp_async4(Bop + (MC + l) * LDZ + j, zf + off, ok);
        }
        // A | G rows from the tapes ([q][ngroups][d_pad][WC], WC % 4 == 0).
        // Columns of the last group beyond m hold zeros (the sweeps load
        // zeros there), so whole float4s are safe to take.
        for (int idx = tid; idx < RT * (MC / 4); idx += kThreads) {
            const int r = idx / (MC / 4), l4 = (idx - r * (MC / 4)) * 4;
            const bool ok = l4 < mc && r0 + r < a.d_pad;
            size_t off = 0;
            if (ok) {
                const int gl = lc + l4;
                const int g = gl / WC, c = gl - g * WC;
                off = (((size_t)i * a.ngroups + g) * a.d_pad + r0 + r) * WC + c;
            }
            dev::cp_async16(Aop + r * LDA + l4, a.tapeA + off, ok);
            dev::cp_async16(Aop + r * LDA + MC + l4, a.tapeG + off, ok);
        }
        dev::cp_async_commit();
        dev::cp_async_wait_all();
        __syncthreads();
        // K' partial: Q[k][j] - Q[j][k] over this chunk, k < j
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int idx = tid + u * kThreads;
            if (idx < BS * BS) {
                const int k = idx / BS, j = idx - k * BS;
                if (k < j) {
                    float s = kacc[u];
                    for (int l = 0; l < mc; ++l)
                        s += Bop[(MC + l) * LDZ + k] * Bop[l * LDZ + j] -
                             Bop[(MC + l) * LDZ + j] * Bop[l * LDZ + k];
                    kacc[u] = s;
                }
            }
        }
        // [A | G] [Z'b^T ; Z'f^T]
#pragma unroll 4
        for (int kk = 0; kk < KA; ++kk) {
            float bv[JT];
#pragma unroll
            for (int v = 0; v < JT; ++v) bv[v] = Bop[kk * LDZ + jt * JT + v];
#pragma unroll
            for (int u = 0; u < RTH; ++u) {
                const float av = Aop[(rt * RTH + u) * LDA + kk];
#pragma unroll
                for (int v = 0; v < JT; ++v) acc[u][v] = fmaf(av, bv[v], acc[u][v]);
            }
        }
    }
    // + V (2 K')
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int idx = tid + u * kThreads;
        if (idx < BS * BS) {
            const int k = idx / BS, j = idx - k * BS;
            Kp[k * LDZ + j] = 2.f * kacc[u];
        }
    }
    constexpr int LDB = BS + 4;
    const float* vb = a.Vbl + ((size_t)i * a.d_pad + r0) * LDB;
    for (int idx = tid; idx < RT * BS; idx += kThreads) {
        const int r = idx / BS, c = idx - r * BS;
        const bool ok = r0 + r < a.d_pad;
        dev::cp_async4(Vr + r * (BS + 1) + c, ok ? vb + (size_t)r * LDB + c : a.Vbl, ok);
    }
    dev::cp_async_commit();
    dev::cp_async_wait_all();
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < BS; ++k) {
        float bv[JT];
#pragma unroll
        for (int v = 0; v < JT; ++v) bv[v] = Kp[k * LDZ + jt * JT + v];
#pragma unroll
        for (int u = 0; u < RTH; ++u) {
            const float vv = Vr[(rt * RTH + u) * (BS + 1) + k];
#pragma unroll
            for (int v = 0; v < JT; ++v) acc[u][v] = fmaf(vv, bv[v], acc[u][v]);
        }
    }
    // stage transposed, then coalesced column writes
#pragma unroll
    for (int u = 0; u < RTH; ++u)
#pragma unroll
        for (int v = 0; v < JT; ++v) Ct[(jt * JT + v) * (RT + 1) + rt * RTH + u] = -2.f * acc[u][v];
    __syncthreads();
    for (int idx = tid; idx < BS * RT; idx += kThreads) {
        const int j = idx / RT, r = idx - j * RT;
        const int kc = i * a.b + j;
        if (j < a.b && kc < a.n && r0 + r < a.d) {
            const int col = a.reversed ? a.n - 1 - kc : kc;
            a.dV[(int64_t)col * a.lddv + r0 + r] = Ct[j * (RT + 1) + r];
        }
    }
}

template <int BS>
size_t dv_smem() {
    using S = DvShape<BS>;
    return sizeof(float) * ((size_t)RT * S::LDA + (size_t)S::KA * S::LDZ + (size_t)RT * (BS + 1) +
                            (size_t)BS * S::LDZ + (size_t)BS * (RT + 1));
}

template <int BS>
cudaError_t launch_dv_t(const DvArgs& a, cudaStream_t s) {
    static bool configured = false;
    const size_t smem = dv_smem<BS>();
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(dv_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const dim3 grid((a.d + RT - 1) / RT, a.q);
    dv_kernel<BS><<<grid, kThreads, smem, s>>>(a);
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
