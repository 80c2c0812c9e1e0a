// Large-batch chain sweep ("panel" kernel): north_star subsystem (3)/(4) for
// many batch columns (BASELINE config 5: d = 2048, batch 65536 sharded), the
// throughput counterpart of the latency-oriented cluster sweep (chain_v2.cu).
//
// One CTA owns a PANEL of 16 batch columns and ALL d rows of X for the whole
// chain, X held in tensor-core accumulator registers (8 warps x up to 16 row
// tiles x 2 n-tiles).  No cross-CTA exchange: the reduction over rows of the
// block partial happens inside the CTA.  Per step t one pass over the row
// tiles fuses the look-ahead partial and the update (exact algebra of
// chain_v2.cu):
//     L_{t+1} += W_{t+1}[rows]^T X^(t)[rows]       (before the update)
//     X^(t+1)[rows] = X^(t)[rows] + V_t[rows] (-2 Z_t)
// then  Z_{t+1} = sum_warps L_{t+1} - 2 S_{t+1} Z_t  (fixed order, fp32).
// Each warp streams its row tiles' W_{t+1} and V_t rows (the packed stages
// the builder writes, fasth_internal.h) through its own 3-deep ring of bulk
// copies; the B operands (X tiles, -2 Z) are pre-split (3xTF32 RN).
// Per step per CTA: 48 mma.sync per row tile (24 partial + 24 update), W|V
// streamed once: compute-bound on the legacy tensor path (~498 MAC/clk/SM).
#include "device_prims.cuh"
#include "fasth_internal.h"
#include "frag_ops.cuh"

namespace fasthb {
namespace {
using namespace fo;

#ifndef PANEL_WARPS
#define PANEL_WARPS 8
#endif
#ifndef PANEL_NT
#define PANEL_NT 2
#endif
constexpr int PWARPS = PANEL_WARPS;  // warps per CTA
constexpr int PNT = PANEL_NT;        // n-tiles per panel
constexpr int PCOLS = 8 * PNT;
constexpr int PRING = 3;   // per-warp ring depth (row-tile operand chunks)
constexpr int PBS = 32;    // block width handled (MT = 2, KB = 4)
constexpr int PMT = PBS / 16, PKB = PBS / 8;
constexpr int PLDW = stage_ldw(PBS), PLDV = stage_ldv(PBS);
constexpr int PCHUNK = 16 * PLDW + 16 * PLDV;  // floats: W rows | V rows of one row tile

struct PanelSmem {
    size_t ring, xs, red, zs, zn, s, bars, total;  // floats (bars: bytes offset / 4)
};

__host__ __device__ inline PanelSmem panel_layout() {
    PanelSmem L;
    size_t o = 0;
    L.ring = o;
    o += (size_t)PWARPS * PRING * PCHUNK;
    L.xs = o;
    o += (size_t)PWARPS * PNT * 256;  // per-warp B-layout scratch of one X tile pair
    L.red = o;
    o += (size_t)PWARPS * PMT * PNT * 128;
    L.zs = o;
    o += (size_t)2 * PBS * PCOLS;  // Z raw, double-buffered (for the correction)
    L.zn = o;
    o += (size_t)PNT * 2 * PKB * 64;  // -2Z pre-split: [nt][hi|lo][KB/2][32][4]
    L.s = o;
    o += (size_t)PBS * PLDV;  // S_{t+1} (packed order)
    o = (o + 3) & ~size_t(3);
    L.bars = o;
    o += 2 * (PWARPS * PRING + 1);
    L.total = o * 4;
    return L;
}

template <int RTW>  // row tiles per warp (ceil(RT / 8))
__global__ void __launch_bounds__(PWARPS * 32, 1) panel_kernel(SweepV2Args a) {
    extern __shared__ __align__(128) float sm[];
    const PanelSmem L = panel_layout();
    float* ring = sm + L.ring;
    float* xs = sm + L.xs;
    float* red = sm + L.red;
    float* zs = sm + L.zs;
    float* zn = sm + L.zn;
    float* Ss = sm + L.s;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const int C = a.C, q = a.q;
    const int RB = a.d_pad / C, RTS = RB / 16;  // row tiles per packed slab
    const int RT = a.d_pad / 16;
    const int SF = (int)stage_floats(RB, PBS);
    const int npanels = (a.m + PCOLS - 1) / PCOLS;
    const int dirn = blockIdx.x / npanels, panel = blockIdx.x - dirn * npanels;
    const SweepDirV2 D = a.dir[dirn];
    const int col0 = panel * PCOLS;
    const uint32_t bar_u32 = dev::smem_u32(bars);  // warp ring bars: [warp][PRING], then the S bar
    const uint32_t sbar = bar_u32 + 8u * (PWARPS * PRING);
    const uint32_t ring_u32 = dev::smem_u32(ring);
    const uint32_t s_u32 = dev::smem_u32(Ss);
    auto block_of = [&](int t) { return D.forward ? q - 1 - t : t; };
    auto pstage = [&](int t, int c) { return D.stage + ((size_t)t * C + c) * SF; };

    if (tid == 0) {
        for (int s = 0; s < PWARPS * PRING + 1; ++s) dev::mbar_init(&bars[s], 1);
        dev::fence_mbar_init();
    }
    __syncthreads();
    if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

    // chunk k of this warp: step s = k / RTW - 1 (s = -1: the prologue, W_0
    // only), tile j = k % RTW -> W_{s+1} rows (if s+1 < q) and V_s rows (if s >= 0)
    const int nchunks = (q + 1) * RTW;
    auto issue = [&](int k) {
        const int s = k / RTW - 1, j = k - (s + 1) * RTW;
        const int rt = warp * RTW + j;
        const int slot = k % PRING;
        const uint32_t bar = bar_u32 + 8u * (warp * PRING + slot);
        const uint32_t dst = ring_u32 + (uint32_t)((warp * PRING + slot) * PCHUNK) * 4u;
        if (rt >= RT) {  // no rows: complete the phase with a plain arrive
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
            return;
        }
        const int c = rt / RTS, lr0 = (rt - c * RTS) * 16;
        uint32_t bytes = 0;
        if (s + 1 < q) bytes += 16 * PLDW * 4;
        if (s >= 0) bytes += 16 * PLDV * 4;
        mbar_expect_u32(bar, bytes);
        if (s + 1 < q) bulk_u32(dst, pstage(s + 1, c) + (size_t)lr0 * PLDW, 16 * PLDW * 4, bar);
        if (s >= 0) bulk_u32(dst + 16 * PLDW * 4, pstage(s, c) + (size_t)RB * PLDW + (size_t)lr0 * PLDV, 16 * PLDV * 4, bar);
    };
    if (lane == 0)
        for (int k = 0; k < PRING && k < nchunks; ++k) issue(k);

    // X^(0): this warp's tiles in C-fragment registers
    float x[RTW][PNT][4];
#pragma unroll
    for (int j = 0; j < RTW; ++j)
#pragma unroll
        for (int nt = 0; nt < PNT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int gr = (warp * RTW + j) * 16 + g + 8 * (e >> 1);
                const int gc = col0 + nt * 8 + 2 * tq + (e & 1);
                float v = 0.f;
                if (warp * RTW + j < RT && gr < D.n_valid && gc < a.m) {
                    v = D.x_in[(int64_t)gc * D.ldx + gr];
                    if (D.scale) v *= D.scale[gr];
                }
                x[j][nt][e] = v;
            }

    const size_t tape_step = (size_t)a.ngroups * a.d_pad * 8;
    float* xsw = xs + warp * PNT * 256;
    int k = 0;  // chunk counter of this warp
    for (int s = -1; s < q; ++s) {
        const int t1 = s + 1;  // the partial of this pass is for step t1
        if (t1 < q && tid == 0) {  // S_{t1} (slab 0's copy) for the reduce phase
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_u32(sbar, PBS * PLDV * 4);
            bulk_u32(s_u32, pstage(t1, 0) + (size_t)RB * (PLDW + PLDV), PBS * PLDV * 4, sbar);
        }
        float pm[PMT][PNT][4], pc[PMT][PNT][4];
#pragma unroll
        for (int mt = 0; mt < PMT; ++mt)
#pragma unroll
            for (int nt = 0; nt < PNT; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) pm[mt][nt][e] = pc[mt][nt][e] = 0.f;
        // -2 Z_s pre-split B fragments for the update (this step's Z)
        float zh[PNT][PKB / 2][4], zl[PNT][PKB / 2][4];
        if (s >= 0) {
#pragma unroll
            for (int nt = 0; nt < PNT; ++nt)
#pragma unroll
                for (int h2 = 0; h2 < PKB / 2; ++h2) {
                    lds_vec<4>(zh[nt][h2], zn + ((nt * 2 + 0) * (PKB / 2) + h2) * 128 + lane * 4);
                    lds_vec<4>(zl[nt][h2], zn + ((nt * 2 + 1) * (PKB / 2) + h2) * 128 + lane * 4);
                }
        }
        const int i = s >= 0 ? block_of(s) : 0;
        float* tblk = (s >= 0 && D.tape) ? D.tape + (size_t)i * tape_step : nullptr;
#pragma unroll
        for (int j = 0; j < RTW; ++j, ++k) {
            const int rt = warp * RTW + j;
            const int slot = k % PRING;
            mbar_wait_u32(bar_u32 + 8u * (warp * PRING + slot), (uint32_t)((k / PRING) & 1));
            const float* ch = ring + (size_t)(warp * PRING + slot) * PCHUNK;
            if (rt < RT) {
                if (t1 < q) {  // partial: W_{t1}[rows]^T X^(s)[rows], X tiles transposed via own scratch
#pragma unroll
                    for (int nt = 0; nt < PNT; ++nt)
                        scatter_cb(xsw + nt * 256, xsw + nt * 256 + 128, x[j][nt], g, tq, 1.f);
                    __syncwarp();
                    float xb[PNT][8];
#pragma unroll
                    for (int nt = 0; nt < PNT; ++nt) {
                        float h4[4], l4[4];
                        lds_vec<4>(h4, xsw + nt * 256 + lane * 4);
                        lds_vec<4>(l4, xsw + nt * 256 + 128 + lane * 4);
#pragma unroll
                        for (int e = 0; e < 4; ++e) xb[nt][e] = h4[e], xb[nt][4 + e] = l4[e];
                    }
                    __syncwarp();
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        float w0[2 * PMT], w1[2 * PMT];
                        lds_vec<2 * PMT>(w0, ch + (ks * 8 + tq) * PLDW + g * 2 * PMT);
                        lds_vec<2 * PMT>(w1, ch + (ks * 8 + tq + 4) * PLDW + g * 2 * PMT);
#pragma unroll
                        for (int mt = 0; mt < PMT; ++mt) {
                            const AFrag af = make_a(w0[2 * mt], w0[2 * mt + 1], w1[2 * mt], w1[2 * mt + 1]);
#pragma unroll
                            for (int nt = 0; nt < PNT; ++nt) {
                                hmma(pm[mt][nt], af.h[0], af.h[1], af.h[2], af.h[3], __float_as_uint(xb[nt][2 * ks]),
                                     __float_as_uint(xb[nt][2 * ks + 1]));
                                hmma(pc[mt][nt], af.h[0], af.h[1], af.h[2], af.h[3],
                                     __float_as_uint(xb[nt][4 + 2 * ks]), __float_as_uint(xb[nt][4 + 2 * ks + 1]));
                                hmma(pc[mt][nt], af.l[0], af.l[1], af.l[2], af.l[3], __float_as_uint(xb[nt][2 * ks]),
                                     __float_as_uint(xb[nt][2 * ks + 1]));
                            }
                        }
                    }
                }
                if (s >= 0) {  // update: X^(s+1) = X^(s) + V_s[rows] (-2 Z_s)
                    // tape groups of this panel (the last panel may have one 8-column group only)
                    float* tp = tblk ? tblk + ((size_t)(col0 / 8) * a.d_pad + rt * 16 + g) * 8 + 2 * tq : nullptr;
                    const int ntv = min(PNT, a.ngroups - col0 / 8);
                    if (tp && !D.forward)  // dA[i] = X^(s)
#pragma unroll
                        for (int nt = 0; nt < PNT; ++nt) {
                            if (nt >= ntv) break;
                            float* tq_ = tp + (size_t)nt * a.d_pad * 8;
                            *reinterpret_cast<float2*>(tq_) = make_float2(x[j][nt][0], x[j][nt][1]);
                            *reinterpret_cast<float2*>(tq_ + 64) = make_float2(x[j][nt][2], x[j][nt][3]);
                        }
                    const float* Vc = ch + 16 * PLDW;
                    float v0[2 * PKB], v1[2 * PKB];
                    lds_vec<2 * PKB>(v0, Vc + g * PLDV + tq * 2 * PKB);
                    lds_vec<2 * PKB>(v1, Vc + (g + 8) * PLDV + tq * 2 * PKB);
#pragma unroll
                    for (int nt = 0; nt < PNT; ++nt) {
                        float c1[4] = {0.f, 0.f, 0.f, 0.f}, c2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int ks = 0; ks < PKB; ++ks) {
                            const AFrag af = make_a(v0[2 * ks], v1[2 * ks], v0[2 * ks + 1], v1[2 * ks + 1]);
                            mma3s(x[j][nt], c1, c2, af, zh[nt][ks >> 1][2 * (ks & 1)], zh[nt][ks >> 1][2 * (ks & 1) + 1],
                                  zl[nt][ks >> 1][2 * (ks & 1)], zl[nt][ks >> 1][2 * (ks & 1) + 1]);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) x[j][nt][e] += c1[e] + c2[e];
                    }
                    if (tp && D.forward)  // A_i = activations[i]
#pragma unroll
                        for (int nt = 0; nt < PNT; ++nt) {
                            if (nt >= ntv) break;
                            float* tq_ = tp + (size_t)nt * a.d_pad * 8;
                            *reinterpret_cast<float2*>(tq_) = make_float2(x[j][nt][0], x[j][nt][1]);
                            *reinterpret_cast<float2*>(tq_ + 64) = make_float2(x[j][nt][2], x[j][nt][3]);
                        }
                }
            }
            __syncwarp();
            if (lane == 0 && k + PRING < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(k + PRING);
            }
        }
        if (t1 >= q) break;
        // ---- reduce: Z_{t1} = sum_warps L_{t1} - 2 S_{t1} Z_s (fixed order) ----
#pragma unroll
        for (int mt = 0; mt < PMT; ++mt)
#pragma unroll
            for (int nt = 0; nt < PNT; ++nt)
                *reinterpret_cast<float4*>(red + ((warp * PMT + mt) * PNT + nt) * 128 + lane * 4) =
                    make_float4(pm[mt][nt][0] + pc[mt][nt][0], pm[mt][nt][1] + pc[mt][nt][1],
                                pm[mt][nt][2] + pc[mt][nt][2], pm[mt][nt][3] + pc[mt][nt][3]);
        __syncthreads();
        mbar_wait_u32(sbar, (uint32_t)(t1 & 1));
        for (int o = tid; o < PBS * PCOLS; o += PWARPS * 32) {
            const int jj = o / PCOLS, cc = o - jj * PCOLS;  // Z[jj][cc]
            const int mt = jj >> 4, rr = jj & 15, nt = cc >> 3, cl = cc & 7;
            const int ln = (rr & 7) * 4 + (cl >> 1), idx = (rr >> 3) * 2 + (cl & 1);
            float z = 0.f;
            for (int w = 0; w < PWARPS; ++w) z += red[((w * PMT + mt) * PNT + nt) * 128 + ln * 4 + idx];
            if (s >= 0) {
                const float* zp = zs + (s & 1) * PBS * PCOLS;
                float corr = 0.f;
#pragma unroll 8
                for (int kk = 0; kk < PBS; ++kk) corr = fmaf(Ss[jj * PLDV + perm_v_bs(kk, PBS)], zp[kk * PCOLS + cc], corr);
                z -= 2.f * corr;
            }
            zs[(t1 & 1) * PBS * PCOLS + jj * PCOLS + cc] = z;
            // -2 z pre-split into the update's B-fragment slot (K = jj, N = cc)
            const int ks = jj >> 3, h = (jj >> 2) & 1, lane2 = cl * 4 + (jj & 3);
            const float v = -2.f * z;
            const uint32_t hb = hi_rn(v);
            zn[((nt * 2 + 0) * (PKB / 2) + (ks >> 1)) * 128 + lane2 * 4 + (ks & 1) * 2 + h] = __uint_as_float(hb);
            zn[((nt * 2 + 1) * (PKB / 2) + (ks >> 1)) * 128 + lane2 * 4 + (ks & 1) * 2 + h] = v - __uint_as_float(hb);
            if (D.zhat && col0 + cc < a.m) D.zhat[((size_t)block_of(t1) * PBS + jj) * a.m + col0 + cc] = z;
        }
        __syncthreads();
    }

#pragma unroll
    for (int j = 0; j < RTW; ++j)
#pragma unroll
        for (int nt = 0; nt < PNT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int gr = (warp * RTW + j) * 16 + g + 8 * (e >> 1);
                const int gc = col0 + nt * 8 + 2 * tq + (e & 1);
                if (warp * RTW + j < RT && gr < a.d && gc < a.m) D.x_out[(int64_t)gc * D.ldo + gr] = x[j][nt][e];
            }
}

template <int RTW>
cudaError_t launch_panel_t(const SweepV2Args& a, cudaStream_t s) {
    const PanelSmem L = panel_layout();
    auto kern = panel_kernel<RTW>;
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), L.total); e != cudaSuccess) return e;
    const int npanels = (a.m + PCOLS - 1) / PCOLS;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(npanels * a.ndir, 1, 1);
    cfg.blockDim = dim3(PWARPS * 32, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

bool panel_supported(int BS, int d_pad, int m) {
    const int RT = d_pad / 16;
    return BS == PBS && RT <= 16 * PWARPS && m >= 1 && panel_layout().total <= 227 * 1024;
}

cudaError_t launch_panel(const SweepV2Args& a, cudaStream_t s) {
    if (!panel_supported(a.BS, a.d_pad, a.m) || a.ready || a.q < 1) return cudaErrorInvalidValue;
    const int RTW = (a.d_pad / 16 + PWARPS - 1) / PWARPS;
    if (RTW <= 4) return launch_panel_t<4>(a, s);
    if (RTW <= 8) return launch_panel_t<8>(a, s);
    return launch_panel_t<16>(a, s);
}

}  // namespace fasthb
