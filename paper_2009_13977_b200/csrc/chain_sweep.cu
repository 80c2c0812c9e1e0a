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
//
// Step t applies block P_t = I - 2 V_t T~_t V_t^T (backward: its transpose):
//     Z_t     = W_t^T X^(t)          (W = V T~^T forward, V T~ backward;
//                                     prebuilt by wy_build.cu)
//     X^(t+1) = X^(t) - 2 V_t Z_t
// Z_t is a reduction over ALL rows, i.e. over the cluster.  To take that
// exchange off the critical path the chain is pipelined one block ahead
// (exact algebra, not a different blocking):
//     Z_{t+1} = W_{t+1}^T X^(t) - 2 S_t Z_t,     S_t = W_{t+1}^T V_t
// (S prebuilt by wy_build.cu), so every CTA computes and pushes its partial
// L_{t+1} = W_{t+1,rows}^T X^(t)_rows while the all-to-all of L_t is still in
// flight.  Iteration t of a CTA:
//   A. L_{t+1} = W_{t+1,rows}^T X^(t)_rows, pushed into every CTA of the
//      cluster with st.async + the receiver's mbarrier complete_tx (DSMEM,
//      4 receive slots, no cluster barrier);
//   B. wait for all L_t, Z_t = sum_c L_t^c - 2 S_{t-1} Z_{t-1} (fixed order:
//      deterministic and identical in every CTA);
//   C. X^(t+1)_rows = X^(t)_rows - 2 V_{t,rows} Z_t.
// W, V and S of each block are streamed in by the bulk-copy (TMA) engine
// three blocks ahead into a ring of shared-memory stages.
#include "device_prims.cuh"
#include "fasth_internal.h"

#include <cstdlib>

namespace fasthb {
namespace {

// NSTG (W/V/S prefetch stages) is 3, or 2 when three do not fit (large d)
constexpr int NSLOT = 4;  // all-to-all receive slots (see the WAR argument below)

struct SweepSmem {
    size_t ws, vs, ss, xs, zr, zb, bars, total;
};

__host__ __device__ inline SweepSmem sweep_layout(int C, int BS, int WC, int d_pad, int NSTG) {
    const int RC = d_pad / C;
    const int LDB = BS + 4;
    SweepSmem L;
    size_t o = 0;
    L.ws = o;
    o += (size_t)NSTG * RC * LDB * 4;
    L.vs = o;
    o += (size_t)NSTG * RC * LDB * 4;
    L.ss = o;
    o += (size_t)NSTG * BS * LDB * 4;
    L.xs = o;
    o += (size_t)RC * WC * 4;
    o = (o + 15) & ~size_t(15);
    L.zr = o;
    o += (size_t)NSLOT * C * BS * WC * 4;
    L.zb = o;
    o += 2 * (size_t)BS * WC * 4;
    o = (o + 15) & ~size_t(15);
    L.bars = o;
    o += (NSTG + NSLOT) * 8;
    L.total = o;
    return L;
}

template <int C, int BS, int WC, int NT>
__global__ void __launch_bounds__(NT, 1) sweep_kernel(SweepArgs a) {
    constexpr int LDB = BS + 4;          // padded row pitch of W / V / S blocks
    constexpr int ZN = BS * WC;          // entries of Z
    constexpr int NTILE = ZN / 4;        // partial tiles of (1 j x 4 l)
    constexpr int KS = NT / NTILE;       // K split of the partial product
    constexpr int TPE = NT / ZN >= 1 ? (NT / ZN > 8 ? 8 : NT / ZN) : 1;  // threads per Z entry in B
    static_assert(WC % 4 == 0 && KS >= 1 && KS <= 32 && (KS & (KS - 1)) == 0, "tile shape");
    static_assert((TPE & (TPE - 1)) == 0 && BS % TPE == 0, "reduce split");

    extern __shared__ __align__(128) unsigned char smem[];
    const int NSTG = a.nstg;
    const SweepSmem L = sweep_layout(C, BS, WC, a.d_pad, NSTG);
    const int RC = a.d_pad / C;
    float* Ws = reinterpret_cast<float*>(smem + L.ws);
    float* Vs = reinterpret_cast<float*>(smem + L.vs);
    float* Ss = reinterpret_cast<float*>(smem + L.ss);
    float* Xs = reinterpret_cast<float*>(smem + L.xs);
    float* Zr = reinterpret_cast<float*>(smem + L.zr);
    float* Zb = reinterpret_cast<float*>(smem + L.zb);
    uint64_t* ld_bar = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* ex_bar = ld_bar + NSTG;

    const int tid = threadIdx.x;
    const uint32_t rank = dev::cluster_ctarank();
    const int group = (int)dev::cluster_id_x();
    const int row0 = (int)rank * RC;
    const int col0 = group * WC;
    const int q = a.q;
    const uint32_t blk_bytes = (uint32_t)RC * LDB * 4;
    const uint32_t s_bytes = (uint32_t)BS * LDB * 4;
    const uint32_t ex_bytes = (uint32_t)C * ZN * 4;
    const int ngroups = (a.m + WC - 1) / WC;

    auto block_of = [&](int t) { return a.forward ? q - 1 - t : t; };
    auto issue_load = [&](int t) {  // group t -> stage t % NSTG
        const int st = t % NSTG, i = block_of(t);
        const size_t off = ((size_t)i * a.d_pad + row0) * LDB;
        dev::mbar_arrive_expect_tx(&ld_bar[st], 2 * blk_bytes + s_bytes);
        dev::bulk_g2s(Ws + (size_t)st * RC * LDB, a.Wbl + off, blk_bytes, &ld_bar[st]);
        dev::bulk_g2s(Vs + (size_t)st * RC * LDB, a.Vbl + off, blk_bytes, &ld_bar[st]);
        dev::bulk_g2s(Ss + (size_t)st * BS * LDB, a.Sbl + (size_t)i * BS * LDB, s_bytes, &ld_bar[st]);
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
        Xs[r * WC + l] = x;
    }
    // every CTA's barriers must be initialised and armed before a peer pushes
    dev::cluster_sync();

    const uint32_t zr_local = dev::smem_u32(Zr);
    const uint32_t exb_local = dev::smem_u32(ex_bar);

    // A: partial tile (row j, columns l0..l0+3), K split KS ways
    const int ptile = tid / KS, pks = tid - ptile * KS;
    const int pj = ptile / (WC / 4), pl0 = (ptile % (WC / 4)) * 4;
    auto partial_push = [&](int t) {  // L_t from the current Xs, into slot t % NSLOT
        const float* Wt = Ws + (size_t)(t % NSTG) * RC * LDB;
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
#pragma unroll 4
        for (int r = pks; r < RC; r += KS) {
            const float w = Wt[r * LDB + pj];
            const float4 x = *reinterpret_cast<const float4*>(Xs + r * WC + pl0);
            acc0 = fmaf(w, x.x, acc0);
            acc1 = fmaf(w, x.y, acc1);
            acc2 = fmaf(w, x.z, acc2);
            acc3 = fmaf(w, x.w, acc3);
        }
#pragma unroll
        for (int off = KS / 2; off >= 1; off >>= 1) {
            acc0 += __shfl_xor_sync(0xffffffffu, acc0, off);
            acc1 += __shfl_xor_sync(0xffffffffu, acc1, off);
            acc2 += __shfl_xor_sync(0xffffffffu, acc2, off);
            acc3 += __shfl_xor_sync(0xffffffffu, acc3, off);
        }
        const int slot = t % NSLOT;
        const uint32_t off = (uint32_t)(((slot * C + (int)rank) * ZN + pj * WC + pl0) * 4);
        for (int dst = pks; dst < C; dst += KS)
            dev::st_async_f32x4(dev::mapa(zr_local + off, dst), acc0, acc1, acc2, acc3,
                                dev::mapa(exb_local + slot * 8, dst));
    };

    // B: Z entry e = j*WC + l, TPE threads per entry (consecutive lanes)
    const int be = tid / TPE, bh = tid - be * TPE;
    // C: float4 outputs (row r, cols c4..c4+3), K split KU ways
    const int nout4 = RC * (WC / 4);
    int KU = NT / (nout4 > 0 ? nout4 : 1);
    KU = KU >= 8 ? 8 : KU >= 4 ? 4 : KU >= 2 ? 2 : 1;
    if (KU > BS / 4) KU = BS / 4;
    const int ku = tid % KU, o4 = tid / KU;
    const int JPER = BS / KU;

    // debug phase trace (FASTH_TRACE): clock64 per phase, thread 0 of each CTA
    long long* trc = a.trace ? a.trace + (size_t)blockIdx.x * (q + 1) * 8 : nullptr;
    auto mark = [&](int t, int k) {
        if (trc && tid == 0) trc[(size_t)t * 8 + k] = clock64();
    };
    mark(q, 0);
    // prologue: L_0
    if (q > 0) {
        wait_group(0);
        partial_push(0);
    }
    mark(q, 1);

    for (int t = 0; t < q; ++t) {
        const int i = block_of(t);
        const int st = t % NSTG;
        const int slot = t % NSLOT;
        mark(t, 0);

        if (!a.forward && a.tape) {  // dA[i] = X^(t), the gradient at the block output
            float* dst = a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC;
            for (int idx = tid; idx < RC * WC / 4; idx += NT)
                reinterpret_cast<float4*>(dst)[idx] = reinterpret_cast<const float4*>(Xs)[idx];
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
        float* Zc = Zb + (t & 1) * ZN;
        const float* Zp = Zb + ((t + 1) & 1) * ZN;
        const float* Sst = Ss + (size_t)st * BS * LDB;
        for (int base = 0; base < ZN; base += NT / TPE) {  // warp-uniform trip count
            const int e = base + be;
            const bool act = e < ZN;
            const int j = act ? e / WC : 0, l = act ? e - (e / WC) * WC : 0;
            float s = 0.f;
            if (act) {
                const float* zr = Zr + (size_t)slot * C * ZN + e;
                for (int c = bh; c < C; c += TPE) s += zr[c * ZN];
                if (t > 0) {
                    float corr = 0.f;
                    const int k0 = bh * (BS / TPE);
#pragma unroll 8
                    for (int k = k0; k < k0 + BS / TPE; ++k) corr = fmaf(Sst[j * LDB + k], Zp[k * WC + l], corr);
                    s = fmaf(-2.f, corr, s);
                }
            }
#pragma unroll
            for (int off = TPE / 2; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (act && bh == 0) {
                Zc[e] = s;
                if (a.zhat && rank == 0 && col0 + l < a.m) a.zhat[((size_t)i * BS + j) * a.m + col0 + l] = s;
            }
        }
        __syncthreads();
        mark(t, 4);

        // C. X^(t+1) = X^(t) - 2 V_t Z_t
        const float* Vt = Vs + (size_t)st * RC * LDB;
        for (int base = 0; base < nout4; base += NT / KU) {  // warp-uniform trip count
            const int o = base + o4;
            const bool active = o < nout4;
            const int r = active ? o / (WC / 4) : 0, c4 = active ? (o - r * (WC / 4)) * 4 : 0;
            const float* vrow = Vt + r * LDB + ku * JPER;
            const float* zc = Zc + (ku * JPER) * WC + c4;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 4
            for (int jj = 0; jj < JPER; jj += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(vrow + jj);
                const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 z = *reinterpret_cast<const float4*>(zc + (jj + u) * WC);
                    s0 = fmaf(vv[u], z.x, s0);
                    s1 = fmaf(vv[u], z.y, s1);
                    s2 = fmaf(vv[u], z.z, s2);
                    s3 = fmaf(vv[u], z.w, s3);
                }
            }
#pragma unroll
            for (int off = KU / 2; off >= 1; off >>= 1) {
                s0 += __shfl_xor_sync(0xffffffffu, s0, off);
                s1 += __shfl_xor_sync(0xffffffffu, s1, off);
                s2 += __shfl_xor_sync(0xffffffffu, s2, off);
                s3 += __shfl_xor_sync(0xffffffffu, s3, off);
            }
            if (active && ku == 0) {
                float4* xp = reinterpret_cast<float4*>(Xs + r * WC + c4);
                float4 x = *xp;
                x.x = fmaf(-2.f, s0, x.x);
                x.y = fmaf(-2.f, s1, x.y);
                x.z = fmaf(-2.f, s2, x.z);
                x.w = fmaf(-2.f, s3, x.w);
                *xp = x;
            }
        }
        __syncthreads();
        mark(t, 5);

        if (a.forward && a.tape) {  // A_i = activations[i]
            float* dst = a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC;
            for (int idx = tid; idx < RC * WC / 4; idx += NT)
                reinterpret_cast<float4*>(dst)[idx] = reinterpret_cast<const float4*>(Xs)[idx];
        }
        if (tid == 0 && t + NSTG < q) issue_load(t + NSTG);  // stage st is free again
        mark(t, 6);
    }
    mark(q, 2);

    for (int idx = tid; idx < RC * WC; idx += NT) {
        const int l = idx / RC, r = idx - l * RC;
        const int gr = row0 + r, gc = col0 + l;
        if (gr < a.d && gc < a.m) a.x_out[(int64_t)gc * a.ldo + gr] = Xs[r * WC + l];
    }
    // no CTA may exit while a peer could still push into it
    dev::cluster_sync();
}

template <int C, int BS, int WC, int NT>
cudaError_t launch_t(const SweepArgs& a, cudaStream_t s) {
    const int NSTG = a.nstg;
    const SweepSmem L = sweep_layout(C, BS, WC, a.d_pad, NSTG);
    auto kern = sweep_kernel<C, BS, WC, NT>;
    static int configured_smem = 0;
    if ((int)L.total > configured_smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)L.total);
        if (e != cudaSuccess) return e;
        if (C > 8) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        configured_smem = (int)L.total;
    }
    const int ngroups = (a.m + WC - 1) / WC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * ngroups, 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
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

// threads per CTA: 512 where the tile shapes allow (K split of the partial
// product <= 32 lanes), else 256
constexpr int threads_for(int BS, int WC) { return (BS * WC / 4) * 32 >= 512 ? 512 : 256; }

template <int C, int WC>
cudaError_t launch_bs(const SweepArgs& a, cudaStream_t s) {
    switch (a.BS) {
        case 8: return launch_t<C, 8, WC, threads_for(8, WC)>(a, s);
        case 16: return launch_t<C, 16, WC, threads_for(16, WC)>(a, s);
        case 32: return launch_t<C, 32, WC, threads_for(32, WC)>(a, s);
        case 64: return launch_t<C, 64, WC, threads_for(64, WC)>(a, s);
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

size_t sweep_smem_bytes(int C, int WC, int BS, int d_pad, int nstg) {
    return sweep_layout(C, BS, WC, d_pad, nstg).total;
}

// Cluster geometry: C CTAs split the rows, WC columns per cluster.  The
// chain is latency bound at small batch, so the choice keeps the per-step
// all-to-all small (C * BS * WC * 4 bytes into each CTA) and covers the SMs
// with clusters of few columns; FASTH_CLUSTER / FASTH_WC override.
int pick_cluster(int d_pad, int m, int BS, int num_sms, int* WC_out, int* nstg_out) {
    int C = d_pad >= 2048 ? 16 : 8;
    int WC = 4;
    while (WC < 16 && (long)((m + WC - 1) / WC) * C > 2L * num_sms) WC *= 2;
    if (const char* e = getenv("FASTH_CLUSTER")) C = atoi(e);
    if (const char* e = getenv("FASTH_WC")) WC = atoi(e);
    if (C != 2 && C != 4 && C != 8 && C != 16) C = 8;
    if (WC != 4 && WC != 8 && WC != 16) WC = 4;
    while (C > 2 && d_pad / C < 8) C /= 2;
    constexpr size_t kBudget = 220 * 1024;
    while (sweep_smem_bytes(C, WC, BS, d_pad, 3) > kBudget && C < 16) C *= 2;
    int nstg = 3;
    if (sweep_smem_bytes(C, WC, BS, d_pad, 3) > kBudget) nstg = 2;
    *WC_out = WC;
    *nstg_out = nstg;
    return C;
}

cudaError_t launch_sweep(const SweepArgs& a, int C, int WC, int num_sms, cudaStream_t s) {
    (void)num_sms;
    if (a.d_pad % C != 0 || a.nstg < 2 || a.nstg > 3) return cudaErrorInvalidValue;
    if (sweep_smem_bytes(C, WC, a.BS, a.d_pad, a.nstg) > 227 * 1024)
        return cudaErrorInvalidConfiguration;
    switch (C) {
        case 2: return launch_wc<2>(a, WC, s);
        case 4: return launch_wc<4>(a, WC, s);
        case 8: return launch_wc<8>(a, WC, s);
        case 16: return launch_wc<16>(a, WC, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
