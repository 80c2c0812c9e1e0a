// Sequential block chain: north_star subsystem (3) (forward, Alg. 1 step 2,
// fasth.hpp:58-59 / wy_apply wy.hpp:104-133) and the sweep of subsystem (4)
// (backward step 1, fasth.hpp:82-86 / wy_apply_transpose wy.hpp:137-146).
//
// One persistent launch runs ALL q dependent block steps.  Work split:
//   * batch columns are independent, so each thread-block CLUSTER owns a
//     group of WC columns of X and runs the whole chain on them;
//   * the C CTAs of a cluster split the rows: CTA r keeps rows
//     [r*RC, (r+1)*RC) of its column group resident in shared memory for the
//     entire chain (RC = d_pad / C).
// Per block step i (forward: P_i = I - 2 V T~ V^T; backward: P_i^T):
//   1. Z_part = V_rows^T X_rows          (BS x WC, K = RC)  per CTA, FFMA
//   2. cluster reduce-scatter: each CTA pushes slice o of Z_part straight
//      into CTA o's shared memory with st.async + remote mbarrier
//      complete_tx (no cluster-wide barrier), CTA o sums its slice;
//   3. all-gather: CTA o pushes the summed slice to every CTA the same way;
//   4. Z' = T~ Z (forward) or T~^T Z (backward), BS x WC, per CTA;
//   5. X_rows -= 2 V_rows Z'             (RC x WC, K = BS).
// The block's rows of V and T~ are streamed in by the bulk-copy (TMA) engine
// NST steps ahead into a ring of shared-memory stages, so the critical path
// of a step is compute + two DSMEM hops.
#include "device_prims.cuh"
#include "fasth_internal.h"

#include <cstdlib>

namespace fasthb {
namespace {

constexpr int NST = 2;  // V/T~ prefetch stages

struct SweepSmem {
    // byte offsets inside dynamic shared memory
    size_t vs, ts, xs, zg, zr, zp, bars, total;
};

template <int C, int BS, int WC>
__host__ __device__ inline SweepSmem sweep_layout(int d_pad) {
    constexpr int E = BS * WC / C;
    const int RC = d_pad / C;
    SweepSmem L;
    size_t o = 0;
    L.vs = o;
    o += (size_t)NST * RC * BS * 4;
    L.ts = o;
    o += (size_t)NST * BS * BS * 4;
    L.xs = o;
    o += (size_t)RC * WC * 4;
    o = (o + 15) & ~size_t(15);
    L.zg = o;
    o += 2 * (size_t)BS * WC * 4;
    L.zr = o;
    o += 2 * (size_t)C * E * 4;
    L.zp = o;
    o += (size_t)BS * WC * 4;
    o = (o + 15) & ~size_t(15);
    L.bars = o;
    o += (NST + 4) * 8;
    L.total = o;
    return L;
}

template <int C, int BS, int WC>
__global__ void __launch_bounds__(kThreads, 1) sweep_kernel(SweepArgs a) {
    static_assert(BS % 4 == 0 && WC % 4 == 0, "tile shape");
    constexpr int E = BS * WC / C;        // entries of Z owned (reduced) per CTA
    constexpr int TL = WC / 4;            // columns per partial-Z thread tile
    constexpr int NTILE = BS;             // (BS/4) x 4 tiles of 4 x TL
    constexpr int KS = kThreads / NTILE;  // K-split of the partial product
    static_assert(KS >= 1 && KS <= 32 && (KS & (KS - 1)) == 0, "K split");
    static_assert(E % TL == 0 && E >= 1, "slice shape");

    extern __shared__ __align__(128) unsigned char smem[];
    const SweepSmem L = sweep_layout<C, BS, WC>(a.d_pad);
    const int RC = a.d_pad / C;
    float* Vs = reinterpret_cast<float*>(smem + L.vs);
    float* Ts = reinterpret_cast<float*>(smem + L.ts);
    float* Xs = reinterpret_cast<float*>(smem + L.xs);
    float* Zg = reinterpret_cast<float*>(smem + L.zg);
    float* Zr = reinterpret_cast<float*>(smem + L.zr);
    float* Zp = reinterpret_cast<float*>(smem + L.zp);
    uint64_t* ld_bar = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* part_bar = ld_bar + NST;  // [2]
    uint64_t* gath_bar = part_bar + 2;  // [2]

    const int tid = threadIdx.x;
    const uint32_t rank = dev::cluster_ctarank();
    const int group = (int)dev::cluster_id_x();
    const int row0 = (int)rank * RC;
    const int col0 = group * WC;
    const int q = a.q;

    const uint32_t part_bytes = C * E * 4;
    const uint32_t gath_bytes = BS * WC * 4;
    const uint32_t v_bytes = (uint32_t)RC * BS * 4;
    const uint32_t t_bytes = BS * BS * 4;

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) dev::mbar_init(&ld_bar[s], 1);
        for (int s = 0; s < 2; ++s) {
            dev::mbar_init(&part_bar[s], 1);
            dev::mbar_init(&gath_bar[s], 1);
        }
        dev::fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            dev::mbar_arrive_expect_tx(&part_bar[s], part_bytes);
            dev::mbar_arrive_expect_tx(&gath_bar[s], gath_bytes);
        }
        for (int t = 0; t < NST && t < q; ++t) {
            const int i = a.forward ? q - 1 - t : t;
            dev::mbar_arrive_expect_tx(&ld_bar[t], v_bytes + t_bytes);
            dev::bulk_g2s(Vs + (size_t)t * RC * BS, a.Vbl + ((size_t)i * a.d_pad + row0) * BS,
                          v_bytes, &ld_bar[t]);
            dev::bulk_g2s(Ts + (size_t)t * BS * BS, a.Tt + (size_t)i * BS * BS, t_bytes,
                          &ld_bar[t]);
        }
    }
    // resident rows of this cluster's column group (optionally Sigma-scaled)
    for (int idx = tid; idx < RC * WC; idx += kThreads) {
        const int l = idx / RC, r = idx - l * RC;
        const int gr = row0 + r, gc = col0 + l;
        float x = 0.f;
        if (gr < a.n_valid && gc < a.m) {
            x = a.x_in[(int64_t)gc * a.ldx + gr];
            if (a.scale) x *= a.scale[gr];
        }
        Xs[r * WC + l] = x;
    }
    // every CTA's barriers must be initialised and armed before any peer
    // pushes into them
    dev::cluster_sync();

    const uint32_t zr_local = dev::smem_u32(Zr);
    const uint32_t zg_local = dev::smem_u32(Zg);
    const int ngroups = (a.m + WC - 1) / WC;

    // partial-product tile of this thread
    const int tile = tid / KS, ks = tid - tile * KS;
    const int j0 = (tile / 4) * 4, l0 = (tile % 4) * TL;

    for (int t = 0; t < q; ++t) {
        const int i = a.forward ? q - 1 - t : t;
        const int st = t % NST;
        const int s2 = t & 1;
        const uint32_t ph_ld = (uint32_t)(t / NST) & 1u;
        const uint32_t ph_2 = (uint32_t)(t >> 1) & 1u;
        const float* Vt = Vs + (size_t)st * RC * BS;
        const float* Tm = Ts + (size_t)st * BS * BS;

        if (!a.forward && a.tape) {  // dA[i] (gradient at the block output)
            float* dst = a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC;
            for (int idx = tid; idx < RC * WC / 4; idx += kThreads)
                reinterpret_cast<float4*>(dst)[idx] = reinterpret_cast<const float4*>(Xs)[idx];
        }
        dev::mbar_wait(&ld_bar[st], ph_ld);

        // 1. partial Z = V_rows^T X_rows
        float acc[4][TL];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int ll = 0; ll < TL; ++ll) acc[jj][ll] = 0.f;
        for (int r = ks; r < RC; r += KS) {
            const float4 v4 = *reinterpret_cast<const float4*>(Vt + r * BS + j0);
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
            float xx[TL];
#pragma unroll
            for (int ll = 0; ll < TL; ++ll) xx[ll] = Xs[r * WC + l0 + ll];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int ll = 0; ll < TL; ++ll) acc[jj][ll] = fmaf(vv[jj], xx[ll], acc[jj][ll]);
        }
#pragma unroll
        for (int off = KS / 2; off >= 1; off >>= 1)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int ll = 0; ll < TL; ++ll)
                    acc[jj][ll] += __shfl_xor_sync(0xffffffffu, acc[jj][ll], off);

        // 2. reduce-scatter: push my partial slices to their owners
        if (ks == 0) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int e = (j0 + jj) * WC + l0;
                const int o = e / E;
                const uint32_t dst = dev::mapa(
                    zr_local + (uint32_t)(((s2 * C + (int)rank) * E + (e - o * E)) * 4), o);
                const uint32_t bar = dev::mapa(dev::smem_u32(&part_bar[s2]), o);
                if constexpr (TL == 1) {
                    dev::st_async_f32(dst, acc[jj][0], bar);
                } else if constexpr (TL == 2) {
                    dev::st_async_f32x2(dst, acc[jj][0], acc[jj][1], bar);
                } else {
#pragma unroll
                    for (int ll = 0; ll < TL; ll += 4)
                        dev::st_async_f32x4(dst + ll * 4, acc[jj][ll], acc[jj][ll + 1],
                                            acc[jj][ll + 2], acc[jj][ll + 3], bar);
                }
            }
        }

        // 3. reduce my slice, all-gather it into every CTA
        dev::mbar_wait_cluster(&part_bar[s2], ph_2);
        if (tid == 0) dev::mbar_arrive_expect_tx(&part_bar[s2], part_bytes);  // re-arm (t+2)
        for (int idx = tid; idx < E * C; idx += kThreads) {
            const int e = idx % E, dst_rank = idx / E;
            const float* src = Zr + (size_t)s2 * C * E + e;
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) sum += src[c * E];
            const uint32_t dst = dev::mapa(
                zg_local + (uint32_t)((s2 * BS * WC + (int)rank * E + e) * 4), dst_rank);
            dev::st_async_f32(dst, sum, dev::mapa(dev::smem_u32(&gath_bar[s2]), dst_rank));
        }
        dev::mbar_wait_cluster(&gath_bar[s2], ph_2);
        if (tid == 0) dev::mbar_arrive_expect_tx(&gath_bar[s2], gath_bytes);

        // 4. Z' = T~ Z  or  T~^T Z
        const float* Z = Zg + (size_t)s2 * BS * WC;
        for (int idx = tid; idx < BS * WC; idx += kThreads) {
            const int j = idx / WC, l = idx - j * WC;
            float sum = 0.f;
            if (a.forward) {
                for (int k = j; k < BS; ++k) sum = fmaf(Tm[j * BS + k], Z[k * WC + l], sum);
            } else {
                for (int k = 0; k <= j; ++k) sum = fmaf(Tm[k * BS + j], Z[k * WC + l], sum);
            }
            Zp[idx] = sum;
            if (a.zhat && rank == 0 && col0 + l < a.m)
                a.zhat[((size_t)i * BS + j) * a.m + col0 + l] = sum;
        }
        __syncthreads();

        // 5. X_rows -= 2 V_rows Z'
        constexpr int CPR = WC / 4;  // float4 chunks per row
        for (int idx = tid; idx < RC * CPR; idx += kThreads) {
            const int r = idx / CPR, c4 = (idx - r * CPR) * 4;
            float s0 = 0.f, s1 = 0.f, s2v = 0.f, s3 = 0.f;
            const float* vrow = Vt + r * BS;
#pragma unroll 8
            for (int j = 0; j < BS; j += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(vrow + j);
                const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const float4 z = *reinterpret_cast<const float4*>(Zp + (j + jj) * WC + c4);
                    s0 = fmaf(vv[jj], z.x, s0);
                    s1 = fmaf(vv[jj], z.y, s1);
                    s2v = fmaf(vv[jj], z.z, s2v);
                    s3 = fmaf(vv[jj], z.w, s3);
                }
            }
            float4* xp = reinterpret_cast<float4*>(Xs + r * WC + c4);
            float4 x = *xp;
            x.x = fmaf(-2.f, s0, x.x);
            x.y = fmaf(-2.f, s1, x.y);
            x.z = fmaf(-2.f, s2v, x.z);
            x.w = fmaf(-2.f, s3, x.w);
            *xp = x;
        }
        __syncthreads();

        if (a.forward && a.tape) {  // A_i = activations[i]
            float* dst = a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC;
            for (int idx = tid; idx < RC * WC / 4; idx += kThreads)
                reinterpret_cast<float4*>(dst)[idx] = reinterpret_cast<const float4*>(Xs)[idx];
        }
        // refill this stage with step t + NST
        if (tid == 0 && t + NST < q) {
            const int tn = t + NST;
            const int in = a.forward ? q - 1 - tn : tn;
            dev::mbar_arrive_expect_tx(&ld_bar[st], v_bytes + t_bytes);
            dev::bulk_g2s(Vs + (size_t)st * RC * BS, a.Vbl + ((size_t)in * a.d_pad + row0) * BS,
                          v_bytes, &ld_bar[st]);
            dev::bulk_g2s(Ts + (size_t)st * BS * BS, a.Tt + (size_t)in * BS * BS, t_bytes,
                          &ld_bar[st]);
        }
    }

    for (int idx = tid; idx < RC * WC; idx += kThreads) {
        const int l = idx / RC, r = idx - l * RC;
        const int gr = row0 + r, gc = col0 + l;
        if (gr < a.d && gc < a.m) a.x_out[(int64_t)gc * a.ldo + gr] = Xs[r * WC + l];
    }
    // no CTA may exit while a peer could still push into it
    dev::cluster_sync();
}

template <int C, int BS, int WC>
cudaError_t launch_t(const SweepArgs& a, cudaStream_t s) {
    const SweepSmem L = sweep_layout<C, BS, WC>(a.d_pad);
    auto kern = sweep_kernel<C, BS, WC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.total);
    if (e != cudaSuccess) return e;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    const int ngroups = (a.m + WC - 1) / WC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * ngroups, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int C, int WC>
cudaError_t launch_bs(const SweepArgs& a, cudaStream_t s) {
    switch (a.BS) {
        case 8: return launch_t<C, 8, WC>(a, s);
        case 16: return launch_t<C, 16, WC>(a, s);
        case 32: return launch_t<C, 32, WC>(a, s);
        case 64: return launch_t<C, 64, WC>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int C>
cudaError_t launch_wc(const SweepArgs& a, int WC, cudaStream_t s) {
    switch (WC) {
        case 4: return launch_bs<C, 4>(a, s);
        case 8: return launch_bs<C, 8>(a, s);
        case 16: return launch_bs<C, 16>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

size_t sweep_smem_bytes(int C, int WC, int BS, int d_pad) {
    // mirrors sweep_layout without the template
    const int E = BS * WC / C;
    const int RC = d_pad / C;
    size_t o = (size_t)NST * RC * BS * 4 + (size_t)NST * BS * BS * 4 + (size_t)RC * WC * 4;
    o = (o + 15) & ~size_t(15);
    o += 2 * (size_t)BS * WC * 4 + 2 * (size_t)C * E * 4 + (size_t)BS * WC * 4;
    o = (o + 15) & ~size_t(15);
    return o + (NST + 4) * 8;
}

// Cluster geometry: C CTAs split the rows, WC columns per cluster.  The
// choice keeps per-CTA shared memory within budget and aims the number of
// CTAs at the SM count (the chain is latency bound at small batch).
int pick_cluster(int d_pad, int m, int BS, int num_sms, int* WC_out) {
    int C = 16;
    int WC = 8;
    if (const char* e = getenv("FASTH_CLUSTER")) C = atoi(e);
    if (const char* e = getenv("FASTH_WC")) WC = atoi(e);
    else {
        // enough clusters to cover the SMs with the fewest columns each
        WC = 4;
        while (WC < 16 && (long)((m + WC - 1) / WC) * C > 2L * num_sms) WC *= 2;
    }
    if (C != 2 && C != 4 && C != 8 && C != 16) C = 16;
    if (WC != 4 && WC != 8 && WC != 16) WC = 8;
    while (C > 2 && d_pad / C < 8) C /= 2;
    while (sweep_smem_bytes(C, WC, BS, d_pad) > 220 * 1024 && C < 16) C *= 2;
    *WC_out = WC;
    return C;
}

cudaError_t launch_sweep(const SweepArgs& a, int C, int WC, int num_sms, cudaStream_t s) {
    (void)num_sms;
    if (a.d_pad % C != 0) return cudaErrorInvalidValue;
    switch (C) {
        case 2: return launch_wc<2>(a, WC, s);
        case 4: return launch_wc<4>(a, WC, s);
        case 8: return launch_wc<8>(a, WC, s);
        case 16: return launch_wc<16>(a, WC, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
