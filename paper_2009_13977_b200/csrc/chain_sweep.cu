// Sequential block chain: north_star subsystem (3) (forward, Alg. 1 step 2,
// fasth.hpp:58-59 / wy_apply wy.hpp:104-133) and the sweep of subsystem (4)
// (backward step 1, fasth.hpp:82-86 / wy_apply_transpose wy.hpp:137-146).
//
// One persistent launch runs ALL q dependent block steps.  Work split:
//   * batch columns are independent, so each thread-block CLUSTER owns a
//     group of WC columns of X and runs the whole chain on them;
//   * the C CTAs of a cluster split the rows: CTA r keeps rows
//     [r*RC, (r+1)*RC) of its column group resident in shared memory for the
//     entire chain (RC = d_pad / C, a multiple of 16).
//
// Step t applies block P_t = I - 2 V_t T~_t V_t^T (backward: its transpose):
//     Z_t     = W_t^T X^(t)          (W = V T~^T forward, V T~ backward;
//                                     prebuilt by wy_build.cu)
//     X^(t+1) = X^(t) - 2 V_t Z_t
// Z_t is a reduction over ALL rows, i.e. over the cluster.  To take that
// exchange off the critical path the chain is pipelined one block ahead
// (exact algebra, not a different blocking):
//     Z_{t+1} = W_{t+1}^T X^(t) - 2 S_t Z_t,     S_t = W_{t+1}^T V_t
// (S prebuilt by wy_build.cu).  Iteration t of a CTA:
//   A. L_{t+1} = W_{t+1,rows}^T X^(t)_rows on the tensor cores (mma.sync
//      m16n8k8, 3xTF32: fp32-class accuracy), K split over warps, reduced in
//      shared memory and pushed into every CTA of the cluster with st.async +
//      the receiver's mbarrier complete_tx (DSMEM; 4 receive slots; no
//      cluster barrier);
//   B. wait for all L_t; Z_t = sum_c L_t^c - 2 S_t Z_{t-1} (fixed order:
//      deterministic and identical in every CTA);
//   C. X^(t+1)_rows = X^(t)_rows - 2 V_{t,rows} Z_t, again mma.sync 3xTF32,
//      one 16-row tile per warp.
// W, V and S of each block are streamed in by the bulk-copy (TMA) engine
// NSTG blocks ahead into a ring of shared-memory stages.
#include "device_prims.cuh"
#include "fasth_internal.h"
#include "mma_tf32.cuh"

#include <cstdlib>

namespace fasthb {
namespace {

constexpr int NSLOT = 4;   // all-to-all receive slots (see the WAR argument below)
constexpr int NT = 512;    // threads per CTA
constexpr int NW = NT / 32;

__host__ __device__ constexpr int ldw_of(int BS) { return BS + 8; }   // W rows: conflict-free A^T frags
__host__ __device__ constexpr int ldv_of(int BS) { return BS + 4; }   // V rows: conflict-free A frags
__host__ __device__ constexpr int xp_of(int WC) { return WC == 8 ? 8 : WC + 8; }

struct SweepSmem {
    size_t ws, vs, ss, xs, zr, red, zb, bars, total;
};

__host__ __device__ inline SweepSmem sweep_layout(int C, int BS, int WC, int d_pad, int NSTG) {
    const int RC = d_pad / C;
    const int ZN = BS * WC;
    SweepSmem L;
    size_t o = 0;
    L.ws = o;
    o += (size_t)NSTG * RC * ldw_of(BS) * 4;
    L.vs = o;
    o += (size_t)NSTG * RC * ldv_of(BS) * 4;
    L.ss = o;
    o += (size_t)NSTG * BS * ldv_of(BS) * 4;
    L.xs = o;
    o += (size_t)RC * xp_of(WC) * 4;
    o = (o + 15) & ~size_t(15);
    L.zr = o;
    o += (size_t)NSLOT * C * ZN * 4;
    L.red = o;
    o += (size_t)NW * ZN * 4;
    L.zb = o;
    o += 2 * (size_t)BS * xp_of(WC) * 4;
    o = (o + 15) & ~size_t(15);
    L.bars = o;
    o += (NSTG + NSLOT) * 8;
    L.total = o;
    return L;
}

template <int BS, int WC>
__global__ void __launch_bounds__(NT, 1) sweep_kernel(SweepArgs a) {
    constexpr int LDW = ldw_of(BS), LDV = ldv_of(BS), XP = xp_of(WC);
    constexpr int ZN = BS * WC;
    constexpr int MT = BS / 16;   // M tiles of the partial (j)
    constexpr int NTL = WC / 8;   // N tiles (columns)
    static_assert(BS % 16 == 0 && WC % 8 == 0, "tile shape");

    extern __shared__ __align__(128) unsigned char smem[];
    const int C = a.C;
    const int NSTG = a.nstg;
    const SweepSmem L = sweep_layout(C, BS, WC, a.d_pad, NSTG);
    const int RC = a.d_pad / C;
    float* Ws = reinterpret_cast<float*>(smem + L.ws);
    float* Vs = reinterpret_cast<float*>(smem + L.vs);
    float* Ss = reinterpret_cast<float*>(smem + L.ss);
    float* Xs = reinterpret_cast<float*>(smem + L.xs);
    float* Zr = reinterpret_cast<float*>(smem + L.zr);
    float* red = reinterpret_cast<float*>(smem + L.red);
    float* Zb = reinterpret_cast<float*>(smem + L.zb);
    uint64_t* ld_bar = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* ex_bar = ld_bar + NSTG;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tq = lane & 3;
    const uint32_t rank = dev::cluster_ctarank();
    const int group = (int)dev::cluster_id_x();
    const int row0 = (int)rank * RC;
    const int col0 = group * WC;
    const int q = a.q;
    const uint32_t w_bytes = (uint32_t)RC * LDW * 4;
    const uint32_t v_bytes = (uint32_t)RC * LDV * 4;
    const uint32_t s_bytes = (uint32_t)BS * LDV * 4;
    const uint32_t ex_bytes = (uint32_t)C * ZN * 4;
    const int ngroups = (a.m + WC - 1) / WC;

    auto block_of = [&](int t) { return a.forward ? q - 1 - t : t; };
    auto issue_load = [&](int t) {  // group t -> stage t % NSTG
        const int st = t % NSTG, i = block_of(t);
        dev::mbar_arrive_expect_tx(&ld_bar[st], w_bytes + v_bytes + s_bytes);
        dev::bulk_g2s(Ws + (size_t)st * RC * LDW, a.Wbl + ((size_t)i * a.d_pad + row0) * LDW, w_bytes,
                      &ld_bar[st]);
        dev::bulk_g2s(Vs + (size_t)st * RC * LDV, a.Vbl + ((size_t)i * a.d_pad + row0) * LDV, v_bytes,
                      &ld_bar[st]);
        dev::bulk_g2s(Ss + (size_t)st * BS * LDV, a.Sbl + (size_t)i * BS * LDV, s_bytes, &ld_bar[st]);
    };
    auto wait_group = [&](int t) { dev::mbar_wait(&ld_bar[t % NSTG], (uint32_t)(t / NSTG) & 1u); };

    if (tid == 0) {
        for (int s = 0; s < NSTG; ++s) dev::mbar_init(&ld_bar[s], 1);
        for (int s = 0; s < NSLOT; ++s) dev::mbar_init(&ex_bar[s], 1);
        dev::fence_mbar_init();
        for (int s = 0; s < NSLOT; ++s) dev::mbar_arrive_expect_tx(&ex_bar[s], ex_bytes);
        for (int t = 0; t < NSTG && t < q; ++t) issue_load(t);
    }
    // resident rows of this cluster's column group (optionally Sigma-scaled)
    for (int idx = tid; idx < RC * WC; idx += NT) {
        const int l = idx / RC, r = idx - l * RC;
        const int gr = row0 + r, gc = col0 + l;
        float x = 0.f;
        if (gr < a.n_valid && gc < a.m) {
            x = a.x_in[(int64_t)gc * a.ldx + gr];
            if (a.scale) x *= a.scale[gr];
        }
        Xs[r * XP + l] = x;
    }
    // every CTA's barriers must be initialised and armed before a peer pushes
    dev::cluster_sync();

    const uint32_t zr_local = dev::smem_u32(Zr);
    const uint32_t exb_local = dev::smem_u32(ex_bar);
    const int KT = RC / 8;                     // k-steps of the partial
    const int NWA = KT < NW ? KT : NW;         // warps sharing the partial

    // A: L_t = W_t^T X (current Xs), reduced over warps, pushed into slot t
    auto partial_push = [&](int t) {
        const float* Wt = Ws + (size_t)(t % NSTG) * RC * LDW;
        if (warp < NWA) {
            dev::Frag4 m[MT][NTL], c[MT][NTL];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
                    for (int v = 0; v < 4; ++v) m[mt][nt].v[v] = c[mt][nt].v[v] = 0.f;
            for (int kt = warp; kt < KT; kt += NWA) {
                const int k0 = kt * 8;
                float b[NTL][2];
#pragma unroll
                for (int nt = 0; nt < NTL; ++nt) {
                    b[nt][0] = Xs[(k0 + tq) * XP + nt * 8 + g];
                    b[nt][1] = Xs[(k0 + tq + 4) * XP + nt * 8 + g];
                }
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const float* w0 = Wt + (k0 + tq) * LDW + mt * 16 + g;
                    const float* w4 = w0 + 4 * LDW;
                    const float av[4] = {w0[0], w0[8], w4[0], w4[8]};
#pragma unroll
                    for (int nt = 0; nt < NTL; ++nt) dev::mma3(m[mt][nt], c[mt][nt], av, b[nt]);
                }
            }
            float* rw = red + warp * ZN;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NTL; ++nt) {
                    const int j = mt * 16 + g, l = nt * 8 + 2 * tq;
                    rw[j * WC + l] = m[mt][nt].v[0] + c[mt][nt].v[0];
                    rw[j * WC + l + 1] = m[mt][nt].v[1] + c[mt][nt].v[1];
                    rw[(j + 8) * WC + l] = m[mt][nt].v[2] + c[mt][nt].v[2];
                    rw[(j + 8) * WC + l + 1] = m[mt][nt].v[3] + c[mt][nt].v[3];
                }
        }
        __syncthreads();
        // reduce over the NWA warps: 4 threads per float4, then push
        constexpr int TPR = 4;
        const int slot = t % NSLOT;
        for (int base = 0; base < ZN / 4; base += NT / TPR) {
            const int e4 = base + tid / TPR, h = tid % TPR;
            const bool act = e4 < ZN / 4;
            float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
            if (act)
                for (int w = h; w < NWA; w += TPR) {
                    const float4 v = *reinterpret_cast<const float4*>(red + w * ZN + e4 * 4);
                    s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
                }
#pragma unroll
            for (int off = TPR / 2; off >= 1; off >>= 1) {
                s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
                s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
                s.z += __shfl_xor_sync(0xffffffffu, s.z, off);
                s.w += __shfl_xor_sync(0xffffffffu, s.w, off);
            }
            if (act) {
                const uint32_t off = (uint32_t)(((slot * C + (int)rank) * ZN + e4 * 4) * 4);
                for (int dst = h; dst < C; dst += TPR)
                    dev::st_async_f32x4(dev::mapa(zr_local + off, dst), s.x, s.y, s.z, s.w,
                                        dev::mapa(exb_local + slot * 8, dst));
            }
        }
    };

    // debug phase trace (FASTH_TRACE): clock64 per phase, thread 0 of each CTA
    long long* trc = a.trace ? a.trace + (size_t)blockIdx.x * (q + 1) * 8 : nullptr;
    auto mark = [&](int t, int k) {
        if (trc && tid == 0) trc[(size_t)t * 8 + k] = clock64();
    };
    mark(q, 0);
    if (q > 0) {  // prologue: L_0
        wait_group(0);
        partial_push(0);
    }
    mark(q, 1);

    constexpr int TPE = NT / ZN >= 2 ? 2 : 1;  // threads per Z entry in B
    for (int t = 0; t < q; ++t) {
        const int i = block_of(t);
        const int st = t % NSTG;
        const int slot = t % NSLOT;
        mark(t, 0);

        if (!a.forward && a.tape) {  // dA[i] = X^(t), the gradient at the block output
            float* dst = a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC;
            for (int idx = tid; idx < RC * WC / 4; idx += NT) {
                const int r = idx / (WC / 4), c4 = (idx - r * (WC / 4)) * 4;
                reinterpret_cast<float4*>(dst)[idx] = *reinterpret_cast<const float4*>(Xs + r * XP + c4);
            }
        }
        // A. look-ahead partial for step t+1 (overlaps the in-flight exchange of L_t)
        if (t + 1 < q) {
            wait_group(t + 1);
            mark(t, 1);
            partial_push(t + 1);
        }
        mark(t, 2);
        // B. Z_t = sum_c L_t^c - 2 S_t Z_{t-1}
        dev::mbar_wait(&ex_bar[slot], (uint32_t)(t / NSLOT) & 1u);
        mark(t, 3);
        // WAR safety of the slot: a peer pushes L_{t+4} into it only after it
        // has Z_{t+2}, which needs our L_{t+2}, pushed after this read.
        if (tid == 0) dev::mbar_arrive_expect_tx(&ex_bar[slot], ex_bytes);
        float* Zc = Zb + (t & 1) * BS * XP;
        const float* Zp = Zb + ((t + 1) & 1) * BS * XP;
        const float* Sst = Ss + (size_t)st * BS * LDV;
        for (int base = 0; base < ZN; base += NT / TPE) {
            const int e = base + tid / TPE, h = tid % TPE;
            const bool act = e < ZN;
            const int j = act ? e / WC : 0, l = act ? e - j * WC : 0;
            float s = 0.f;
            if (act) {
                const float* zr = Zr + (size_t)slot * C * ZN + e;
                for (int c = h; c < C; c += TPE) s += zr[c * ZN];
                if (t > 0) {
                    float corr = 0.f;
                    const int k0 = h * (BS / TPE);
#pragma unroll 8
                    for (int k = k0; k < k0 + BS / TPE; ++k) corr = fmaf(Sst[j * LDV + k], Zp[k * XP + l], corr);
                    s = fmaf(-2.f, corr, s);
                }
            }
            if (TPE == 2) s += __shfl_xor_sync(0xffffffffu, s, 1);
            if (act && h == 0) {
                Zc[j * XP + l] = s;
                if (a.zhat && rank == 0 && col0 + l < a.m) a.zhat[((size_t)i * BS + j) * a.m + col0 + l] = s;
            }
        }
        __syncthreads();
        mark(t, 4);

        // C. X^(t+1) = X^(t) - 2 V_t Z_t on the tensor cores, one 16-row tile per warp
        const float* Vt = Vs + (size_t)st * RC * LDV;
        const int units = (RC / 16) * NTL;
        for (int u = warp; u < units; u += NW) {
            const int rt = u / NTL, nt = u - rt * NTL;
            const int r0 = rt * 16, n0 = nt * 8;
            float* x0 = Xs + (r0 + g) * XP + n0 + 2 * tq;
            float* x8 = x0 + 8 * XP;
            dev::Frag4 m = {{x0[0], x0[1], x8[0], x8[1]}};
            dev::Frag4 cc = {{0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kk = 0; kk < BS / 8; ++kk) {
                const float* v0 = Vt + (r0 + g) * LDV + kk * 8 + tq;
                const float* v8 = v0 + 8 * LDV;
                const float av[4] = {v0[0], v8[0], v0[4], v8[4]};
                const float bv[2] = {-2.f * Zc[(kk * 8 + tq) * XP + n0 + g],
                                     -2.f * Zc[(kk * 8 + tq + 4) * XP + n0 + g]};
                dev::mma3(m, cc, av, bv);
            }
            x0[0] = m.v[0] + cc.v[0];
            x0[1] = m.v[1] + cc.v[1];
            x8[0] = m.v[2] + cc.v[2];
            x8[1] = m.v[3] + cc.v[3];
        }
        __syncthreads();
        mark(t, 5);

        if (a.forward && a.tape) {  // A_i = activations[i]
            float* dst = a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC;
            for (int idx = tid; idx < RC * WC / 4; idx += NT) {
                const int r = idx / (WC / 4), c4 = (idx - r * (WC / 4)) * 4;
                reinterpret_cast<float4*>(dst)[idx] = *reinterpret_cast<const float4*>(Xs + r * XP + c4);
            }
        }
        if (tid == 0 && t + NSTG < q) issue_load(t + NSTG);  // stage st is free again
        mark(t, 6);
    }
    mark(q, 2);

    for (int idx = tid; idx < RC * WC; idx += NT) {
        const int l = idx / RC, r = idx - l * RC;
        const int gr = row0 + r, gc = col0 + l;
        if (gr < a.d && gc < a.m) a.x_out[(int64_t)gc * a.ldo + gr] = Xs[r * XP + l];
    }
    // no CTA may exit while a peer could still push into it
    dev::cluster_sync();
}

template <int BS, int WC>
cudaError_t launch_t(const SweepArgs& a, cudaStream_t s) {
    const SweepSmem L = sweep_layout(a.C, BS, WC, a.d_pad, a.nstg);
    auto kern = sweep_kernel<BS, WC>;
    static int configured_smem = 0;
    if ((int)L.total > configured_smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)L.total);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        configured_smem = (int)L.total;
    }
    const int ngroups = (a.m + WC - 1) / WC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.C * ngroups, 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int WC>
cudaError_t launch_bs(const SweepArgs& a, cudaStream_t s) {
    switch (a.BS) {
        case 16: return launch_t<16, WC>(a, s);
        case 32: return launch_t<32, WC>(a, s);
        case 64: return launch_t<64, WC>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

size_t sweep_smem_bytes(int C, int WC, int BS, int d_pad, int nstg) {
    return sweep_layout(C, BS, WC, d_pad, nstg).total;
}

int sweep_ldw(int BS) { return ldw_of(BS); }
int sweep_ldv(int BS) { return ldv_of(BS); }

// Chain geometry: C CTAs per cluster split the rows into RC = 16-row multiples
// near 112 rows each (d = 784 -> 7 x 112, no padding); WC = 8 columns per
// cluster (16 when the batch would need more clusters than the GPU holds).
// FASTH_CLUSTER / FASTH_WC override.
SweepGeom pick_geometry(int d, int m, int BS, int num_sms) {
    SweepGeom G;
    int C = (d + 111) / 112;
    if (C < 1) C = 1;
    if (C > 16) C = 16;
    if (const char* e = getenv("FASTH_CLUSTER")) C = atoi(e);
    if (C < 1 || C > 16) C = 8;
    int WC = 8;
    if ((long)((m + 7) / 8) * C > 4L * num_sms) WC = 16;
    if (const char* e = getenv("FASTH_WC")) WC = atoi(e);
    if (WC != 8 && WC != 16) WC = 8;
    if (BS >= 64) WC = 8;  // register budget of the 3xTF32 partial tiles
    auto rc_of = [&](int c) { return ((d + c - 1) / c + 15) / 16 * 16; };
    constexpr size_t kBudget = 220 * 1024;
    while (C < 16 && sweep_smem_bytes(C, WC, BS, C * rc_of(C), 3) > kBudget) ++C;
    G.C = C;
    G.RC = rc_of(C);
    G.d_pad = C * G.RC;
    G.WC = WC;
    G.nstg = sweep_smem_bytes(C, WC, BS, G.d_pad, 3) <= kBudget ? 3 : 2;
    return G;
}

cudaError_t launch_sweep(const SweepArgs& a, int WC, cudaStream_t s) {
    if (a.C < 1 || a.C > 16 || a.d_pad % a.C != 0 || (a.d_pad / a.C) % 16 != 0) return cudaErrorInvalidValue;
    if (a.nstg < 2 || a.nstg > 3) return cudaErrorInvalidValue;
    if (sweep_smem_bytes(a.C, WC, a.BS, a.d_pad, a.nstg) > 227 * 1024) return cudaErrorInvalidConfiguration;
    switch (WC) {
        case 8: return launch_bs<8>(a, s);
        case 16: return launch_bs<16>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
