// Sequential block chain, v2: north_star subsystem (3) (forward sweep,
// Alg. 1 step 2, fasth.hpp:58-59 / wy_apply wy.hpp:104-133) and the sweep of
// subsystem (4) (backward step 1, fasth.hpp:82-86 / wy_apply_transpose
// wy.hpp:137-146) — optionally BOTH in one launch (fasth_forward_backward:
// the two sweeps are independent once the WY blocks exist).
//
// The look-ahead pipelined UT-form steps,
//     Z_t     = sum_c L_t^c - 2 S_t Z_{t-1},      L_t = W_t^T X^(t-1) (per CTA rows)
//     X^(t+1) = X^(t) - 2 V_t Z_t
// re-laid out for instruction count, which is what bounds a 25-step chain on
// 7-CTA clusters (ncu: HMMA was 2.7% of the v1 kernel's instructions):
//   * one bulk copy per step per CTA: the build kernel writes each CTA's
//     W | V | S rows of a step contiguously, columns permuted into mma.sync
//     fragment order (fasth_internal.h), so every A-operand fragment is one
//     or two 16-byte shared loads with compile-time offsets;
//   * the 3xTF32 split is 3 ops per streamed operand (hi = rn_tf32(x) by two
//     integer ops, lo = x - hi exact), done while the previous phase's
//     tensor-core work is in flight (the update's V fragments are split in
//     phase 1, before Z exists);
//   * the B operands (X for the partial, -2Z for the update and the
//     look-ahead correction) are written pre-split, in B-fragment order, by
//     the warps that produce them — no conversions on the consumer side;
//   * "row warps" own 16-row tiles of X in registers (tensor-core C
//     fragments) and do both the partial (A) and the update (C) on them; two
//     B warps form Z; one producer warp only issues the stage copies;
//   * shared addresses are computed once; ring indices are counters.
// Per step (one CTA barrier, between the phases):
//   phase 1   row warps: L_{t+1} partial from X^(t) and W_{t+1}, combined over
//             the row warps in fixed order, pushed to every CTA of the
//             cluster (st.async + remote mbarrier complete_tx)
//             B warps:   Z_t = sum_c L_t^c (fixed order) + (-2 S_t Z_{t-1})
//   phase 2   row warps: X^(t+1) = X^(t) + V_t (-2 Z_t) in their accumulators,
//             then straight on into the next step's phase 1
#include <algorithm>
#include <cstdlib>

#include "device_prims.cuh"
#include "fasth_internal.h"
#include "frag_ops.cuh"

namespace fasthb {
namespace {
using namespace fo;

constexpr int WCV = 8;     // batch columns per cluster (one MMA N tile)
// exchange receive slots.  WAR safety of slot t % 4: a peer pushes L_{t+4}
// into it only after it has Z_{t+2}, which needs our L_{t+2}, pushed in our
// step t+1 — after the barrier that ends our reads of slot t.  (With 3 slots
// that push would be in step t itself, concurrent with the read.)
constexpr int NSLOTV = 4;
constexpr int MAXNR = 8;   // row warps

struct V2Smem {
    size_t stg, zr, xn, zn, red, bars, total;
};

// sig: the tape-warp variant double-buffers the pre-split X (the tape warp
// reads X^(t+1) while the row warps already form X^(t+2))
__host__ __device__ inline V2Smem v2_layout(int C, int BS, int d_pad, int nstg, bool sig) {
    const int RC = d_pad / C, RT = RC / 16, MT = BS / 16, KB = BS / 8;
    const int NR = RT < MAXNR ? RT : MAXNR;
    V2Smem L;
    size_t o = 0;  // in floats
    L.stg = o;
    o += (size_t)nstg * stage_floats(RC, BS);
    L.zr = o;
    o += (size_t)NSLOTV * C * MT * 128;
    L.xn = o;
    o += (size_t)RT * 256 * (sig ? 2 : 1);
    L.zn = o;
    o += (size_t)2 * KB * 128;
    L.red = o;  // double-buffered where push warps can run (NR <= 6): no end-of-step barrier
    o += (size_t)NR * MT * 128 * (NR <= 6 ? 2 : 1);
    o = (o + 3) & ~size_t(3);
    L.bars = o;
    o += 2 * (nstg + NSLOTV) + 6;  // + the tape warp's two mbarriers and step counter
    L.total = o * 4;
    return L;
}

// NP > 0: NP "push" warps take the combine of the row warps' partials and
// the DSMEM pushes off the row warps (which then only run the partial MMAs
// and the update per step); for NR <= kPushMaxNR row warps.
constexpr int kPushMaxNR = 6;
// TR: the trace stamps (FASTH_TRACE / FASTH_STEPTRACE) are compiled in; the
// production instantiations carry none of their code (the loop is latency
// bound and sensitive to its code layout)
template <int BS, int TPW, bool SIG, int NP, bool TR>
__global__ void __launch_bounds__(((NP ? kPushMaxNR : MAXNR) + BS / 16 + 1 + NP + (SIG ? (TPW == 1 ? 2 : 1) : 0)) * 32, 1)
    sweep2_kernel(SweepV2Args a) {
    constexpr int MT = BS / 16, KB = BS / 8;
    constexpr int LDW = stage_ldw(BS), LDV = stage_ldv(BS);
    constexpr int WOFF = 0;
    extern __shared__ __align__(128) float sm[];

    const int C = a.C, q = a.q, NSTG = a.nstg;
    const int RC = a.d_pad / C, RT = RC / 16;
    const int NR = RT < MAXNR ? RT : MAXNR;
    const V2Smem L = v2_layout(C, BS, a.d_pad, NSTG, SIG);
    const int SF = (int)stage_floats(RC, BS);
    const int VOFF = RC * LDW, SOFF = RC * (LDW + LDV);
    float* stg = sm + L.stg;
    float* Zr = sm + L.zr;
    float* Xn = sm + L.xn;
    float* Zn = sm + L.zn;
    float* red = sm + L.red;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const int ls4 = swz4(lane) * 4;  // this lane's 16-byte group of a swizzled B-fragment tile
    const uint32_t rank = dev::cluster_ctarank();
    const int cid = (int)dev::cluster_id_x();
    const int dirn = cid / a.ngroups, group = cid - dirn * a.ngroups;
    const SweepDirV2 D = a.dir[dirn];
    const int row0 = (int)rank * RC, col0 = group * WCV;
    const uint32_t bar_u32 = dev::smem_u32(bars);  // ld_bar[s] = +8 s, ex_bar[s] = +8 (NSTG + s)
    const uint32_t exb_u32 = bar_u32 + 8u * NSTG;
    const uint32_t stage_bytes = (uint32_t)SF * 4u;
    const uint32_t ex_bytes = (uint32_t)C * MT * 512u;
    const int PW = NR + MT;  // producer warp
    // pipelined gradient (SIG, a.done set): two more warps outside the CTA
    // barriers of the step loop.  The "tape" warp copies each step's tape
    // rows and Z' from the pre-split shared B operands (hi + lo is exact) to
    // global, so the row and B warps issue no global stores in the loop; the
    // "publish" warp makes finished blocks visible to the gradient kernel
    // (gpu-scope fence + counter), as many per fence as are ready, so a slow
    // fence never holds up the tape warp (and through it the row warps).
    // Two-tile geometries (longer steps; no registers to spare for a 14th
    // warp) publish from the tape warp itself.
    const int PU0 = PW + 1;  // first push warp (NP > 0)
    const int SW = SIG ? PW + 1 + NP : 1 << 30;  // tape warp
    const int PBW = TPW == 1 ? SW + 1 : SW;       // publish warp
    const int nmain = (NR + MT + 1 + NP) * 32;
    const bool pusher = NP > 0 && warp >= PU0 && warp < PU0 + NP;
    // tape warp hand-off: xrdy (NR arrivals: X^(t+1) formed in Xn), xfree
    // (1 arrival: the tape warp has read step t's Xn / Zn)
    const uint32_t xrdy_u32 = bar_u32 + 8u * (NSTG + NSLOTV), xfree_u32 = xrdy_u32 + 8u;
    auto xbuf = [&](int k) { return Xn + (SIG ? (k & 1) * RT * 256 : 0); };
    unsigned* prog = reinterpret_cast<unsigned*>(bars + NSTG + NSLOTV + 2);  // steps copied out
    long long* const trc = TR && a.trace ? a.trace + (size_t)blockIdx.x * (q + 1) * 16 : nullptr;
    // prologue / epilogue global-timer stamps in row q: 10 entry, 11 X loaded,
    // 12 cluster synced, 13 prologue partial pushed, 14 loop done, 15 exit
    // per-warp barrier stamps (FASTH_TRACE): [CTA][step][warp < 12][arrive S1,
    // release S1, arrive S2, release S2]; the release stamp sits behind a
    // volatile shared load, which cannot issue before the barrier resolves
    long long* const wtr = TR && a.wtrace ? a.wtrace + (size_t)blockIdx.x * q * 48 : nullptr;
#define WSTAMP(k)                                                                             \
    if (wtr && lane == 0) {                                                                   \
        if ((k) & 1) {                                                                        \
            unsigned dummy_;                                                                  \
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(dummy_) : "r"(bar_u32)); \
            if (dummy_ == 0xdeadbeefu) wtr[0] = 0;                                           \
        }                                                                                     \
        if (warp < 12) wtr[((size_t)t * 12 + warp) * 4 + (k)] = clock64();                   \
    }
#define GSTAMP(k) \
    if (trc && tid == 0) trc[(size_t)q * 16 + (k)] = (long long)dev::globaltimer()
    GSTAMP(10);

    auto block_of = [&](int t) { return D.forward ? q - 1 - t : t; };
    auto gstage = [&](int t) { return D.stage + ((size_t)t * C + rank) * SF; };

    // the gradient kernel may launch now (it waits on the sweep or on the
    // per-block counters); with late_trigger once the builder is complete, so
    // that it may read the builder's outputs before its wait
    if (!a.late_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) {
        for (int s = 0; s < NSTG + NSLOTV; ++s) dev::mbar_init(&bars[s], 1);
        if (SIG) {
            dev::mbar_init(&bars[NSTG + NSLOTV], (uint32_t)NR);
            dev::mbar_init(&bars[NSTG + NSLOTV + 1], 1u);
            *prog = 0u;
        }
        dev::fence_mbar_init();
        for (int s = 0; s < NSLOTV; ++s) mbar_expect_u32(exb_u32 + 8u * s, ex_bytes);
    }
    __syncthreads();
    if (a.xg_ready) {  // streamed host step: X / G still landing
        if (tid == 0) wait_counter_bounded(a.xg_ready, a.xg_target);
        __syncthreads();
    }
    // row warps: X^(0) tiles into registers and B-fragment order (x_wait: X
    // is the previous grid's output, the launch only started early)
    float x[TPW][4];
    if (warp < NR && a.x_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp < NR) {
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const int rt = warp + u * NR;
#pragma unroll
            for (int e = 0; e < 4; ++e) x[u][e] = 0.f;
            if (rt < RT) {
                // all loads in flight before any use (branch-free: a guarded
                // load per element was four serial L2 round trips, ~1.4 us)
                float v[4], sc[4];
                bool ok[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int gr = row0 + rt * 16 + g + 8 * (e >> 1), gc = col0 + 2 * tq + (e & 1);
                    ok[e] = gr < D.n_valid && gc < a.m;
                    v[e] = D.x_in[ok[e] ? (int64_t)gc * D.ldx + gr : 0];
                    sc[e] = D.scale ? D.scale[ok[e] ? gr : 0] : 1.f;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) x[u][e] = ok[e] ? v[e] * sc[e] : 0.f;
                scatter_cb_swz(Xn + rt * 256, Xn + rt * 256 + 128, x[u], g, tq, 1.f);
            }
        }
    }
    GSTAMP(11);
    // peers' barriers armed before anyone pushes; Xn visible
    dev::cluster_sync();
    // every CTA has read X / G: the last one re-arms the streamed-upload count
    if (a.xg_ready && tid == 0 && atomicAdd(a.xg_seen, 1u) == gridDim.x - 1) {
        *a.xg_ready = 0u;
        *a.xg_seen = 0u;
    }
    if (warp == PW && lane == 0) {
        const uint32_t stg_u32 = dev::smem_u32(stg);
        // launched as a programmatic dependent of the builder: everything up
        // to here (X loaded, the cluster synced) overlapped its tail; its
        // stages are read only from now on
        if (!a.ready && a.pdl) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (a.late_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        }
        for (int t = 0; t < NSTG && t < q; ++t) {
            if (a.ready) wait_counter_bounded(a.ready + block_of(t), (unsigned)C);
            mbar_expect_u32(bar_u32 + 8u * t, stage_bytes);
            bulk_u32(stg_u32 + (uint32_t)t * stage_bytes, gstage(t), stage_bytes, bar_u32 + 8u * t);
        }
    }
    GSTAMP(12);

    const uint32_t zr_u32 = dev::smem_u32(Zr);
    const size_t tape_step = (size_t)a.ngroups * a.d_pad * WCV;
    float* const tape0 = D.tape ? D.tape + ((size_t)group * a.d_pad + row0) * WCV : nullptr;

    // the row warps' partials of step s: with push warps, two buffers (a
    // step's partials are read by the push warps while the row warps already
    // form the next step's)
    auto redb = [&](int s) { return NP > 0 ? (s & 1) * NR * MT * 128 : 0; };
    // the CTA's sum of the row warps' partials (fixed order; all loads in
    // flight), pushed to CTAs first, first + step, ... of the cluster
    auto combine_push = [&](int s, int first, int step) {
        if (first >= C) return;
        float sum[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            float part[MAXNR][4];
#pragma unroll
            for (int w = 0; w < MAXNR; ++w)
                if (w < NR) lds_vec<4>(part[w], red + redb(s) + (w * MT + mt) * 128 + lane * 4);
#pragma unroll
            for (int e = 0; e < 4; ++e) sum[mt][e] = part[0][e];
#pragma unroll
            for (int w = 1; w < MAXNR; ++w)
                if (w < NR)
#pragma unroll
                    for (int e = 0; e < 4; ++e) sum[mt][e] += part[w][e];
        }
        const int slot = s % NSLOTV;
        const uint32_t off = zr_u32 + (uint32_t)((((slot * C + (int)rank) * MT) * 128 + lane * 4) * 4);
        const uint32_t rbar_l = exb_u32 + 8u * slot;
        if (C == 1) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dev::put4_local(off + mt * 512u, sum[mt]);
            dev::complete_tx_local(rbar_l, (uint32_t)MT * 16u);
        } else {
            for (int dst = first; dst < C; dst += step) {
                const uint32_t rz = dev::mapa(off, dst), rb = dev::mapa(rbar_l, dst);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) push4(rz + mt * 512u, sum[mt], rb);
            }
        }
    };

    // ---- phase-1 work of the row warps: L partial for step s (stage ss) from X^(cur)
    auto partial_push = [&](int s, int ss) {
        const float* Ws = stg + ss * SF;
        float pm[MT][4], p1[MT][4], p2[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) pm[mt][e] = p1[mt][e] = p2[mt][e] = 0.f;
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const int rt = warp + u * NR;
            if (rt < RT) {
                float xh[4], xl[4];
                const float* Xc = xbuf(s > 0 ? s - 1 : 0) + rt * 256;  // X^(s-1)
                lds_vec<4>(xh, Xc + ls4);
                lds_vec<4>(xl, Xc + 128 + ls4);
                float w0[2][2 * MT], w1[2][2 * MT];
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int R = rt * 16 + ks * 8 + tq;
                    lds_vec<2 * MT>(w0[ks], Ws + R * LDW + g * 2 * MT);
                    lds_vec<2 * MT>(w1[ks], Ws + (R + 4) * LDW + g * 2 * MT);
                }
#pragma unroll
                for (int ks = 0; ks < 2; ++ks)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const AFrag af = make_a(w0[ks][2 * mt], w0[ks][2 * mt + 1], w1[ks][2 * mt], w1[ks][2 * mt + 1]);
                        mma3s(pm[mt], p1[mt], p2[mt], af, xh[2 * ks], xh[2 * ks + 1], xl[2 * ks], xl[2 * ks + 1]);
                    }
            }
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
            *reinterpret_cast<float4*>(red + redb(s) + (warp * MT + mt) * 128 + lane * 4) =
                make_float4(pm[mt][0] + (p1[mt][0] + p2[mt][0]), pm[mt][1] + (p1[mt][1] + p2[mt][1]),
                            pm[mt][2] + (p1[mt][2] + p2[mt][2]), pm[mt][3] + (p1[mt][3] + p2[mt][3]));
        if (trc && tid == 0) trc[(size_t)(s > 0 ? s - 1 : q) * 16 + 1] = clock64();
        if constexpr (NP > 0) {  // hand the partials to the push warps, go on
            // (a sync, not an arrive: the row warps run a step ahead of the end
            // of step, so the hand-off keeps them in step with the push warps)
            asm volatile("bar.sync 4, %0;" ::"r"((NR + NP) * 32) : "memory");
            return;
        }
        // every row warp forms the CTA's sum (fixed order over the row warps;
        // all loads in flight) and pushes it to its own destinations
        // (warp, warp + NR, ...): the pushes are spread over the row warps
        dev::named_bar_sync<1>(NR * 32);
        combine_push(s, warp, NR);
    };
    auto push_step = [&](int s) {  // push warps: partials of step s -> peers
        asm volatile("bar.sync 4, %0;" ::"r"((NR + NP) * 32) : "memory");
        combine_push(s, warp - PU0, NP);
    };
    if (warp < NR && q > 0) {  // prologue: Z_0's partials from X^(0)
        mbar_wait_u32(bar_u32, 0);
        partial_push(0, 0);
    }
    if (pusher && q > 0) push_step(0);
    GSTAMP(13);
    __syncthreads();  // the combine scratch is reused by step 0's partial

    const int t0 = a.sig_from < q ? a.sig_from : q - 1;
    if (SIG && warp == SW) {
        // per step s: X^(s+1) (forward tape) or X^(s) (backward tape) and
        // -2 Z_s, pre-split in B-fragment order: float4 j of lane l holds rows
        // (l & 3) + 4 j, column l >> 2 of a 16 x 8 tile (scatter_cb's layout)
        // (1-tile-per-row-warp geometries hold the whole step in registers and
        // free the buffers before storing; 2-tile ones stream tile by tile)
        constexpr int RTM = TPW == 1 ? MAXNR : 1;
        const int zl = col0 + (lane >> 2);
        const bool zst = D.zhat && rank == 0 && zl < a.m;
        for (int s = 0; s < q; ++s) {
            const int i = block_of(s);
            mbar_wait_u32(xrdy_u32, (uint32_t)(s & 1));
            const float* xs = xbuf(D.forward ? s + 1 : s);
            float* tb = tape0 ? tape0 + (size_t)i * tape_step + (lane & 3) * WCV + (lane >> 2) : nullptr;
            float* zb = zst ? D.zhat + ((size_t)i * BS + (lane & 3)) * a.m + zl : nullptr;
            auto ld_tile = [&](const float* p, float (&v)[4], float sc) {
                float h[4], l[4];
                lds_vec<4>(h, p + ls4);
                lds_vec<4>(l, p + 128 + ls4);
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = sc * (h[j] + l[j]);
            };
            const float* zs = Zn + (s & 1) * (KB * 128);
            auto ld_z = [&](int mt, float (&v)[4]) {
                float h[4], l[4];
                lds_vec<4>(h, zs + mt * 128 + ls4);
                lds_vec<4>(l, zs + (KB / 2) * 128 + mt * 128 + ls4);
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = -0.5f * (h[j] + l[j]);
            };
            // reads done: the row warps may overwrite this Xn after the next
            // barrier 1, the B warps this Zn a step later
            auto free_bufs = [&]() {
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(xfree_u32) : "memory");
            };
            if constexpr (TPW == 1) {
                float tv[RTM][4], zv[MT][4];
#pragma unroll
                for (int rt = 0; rt < RTM; ++rt)
                    if (rt < RT) ld_tile(xs + rt * 256, tv[rt], 1.f);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) ld_z(mt, zv[mt]);
                free_bufs();
                // step s-1's rows are out (stored a step ago: the release
                // waits for nothing); step s is counted after the loop or
                // with step s+1
                if (s > 0 && lane == 0)
                    asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(dev::smem_u32(prog)) : "memory");
                if (tb) {
#pragma unroll
                    for (int rt = 0; rt < RTM; ++rt)
                        if (rt < RT)
#pragma unroll
                            for (int j = 0; j < 4; ++j) tb[(rt * 16 + 4 * j) * WCV] = tv[rt][j];
                }
                if (zb) {
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int j = 0; j < 4; ++j) zb[(size_t)(mt * 16 + 4 * j) * a.m] = zv[mt][j];
                }
            } else {
                for (int rt = 0; rt < RT; ++rt) {
                    float v[4];
                    ld_tile(xs + rt * 256, v, 1.f);
                    if (tb)
#pragma unroll
                        for (int j = 0; j < 4; ++j) tb[(rt * 16 + 4 * j) * WCV] = v[j];
                }
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    float v[4];
                    ld_z(mt, v);
                    if (zb)
#pragma unroll
                        for (int j = 0; j < 4; ++j) zb[(size_t)(mt * 16 + 4 * j) * a.m] = v[j];
                }
                free_bufs();
            }
            if constexpr (TPW == 2) {
                __syncwarp();
                if (lane == 0 && s >= t0) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    for (int u = s == t0 ? 0 : s; u <= s; ++u) atomicAdd(a.done + block_of(u), 1u);
                }
            }
        }
        // the last step's block (the one the gradient kernel's tail waits on)
        // goes out from here, without the hand-off; with it every block when
        // t0 is the last step (the publish warp then has nothing to do)
        __syncwarp();
        if (TPW == 1 && lane == 0 && q > 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int u = t0 >= q - 1 ? 0 : q - 1; u < q; ++u) atomicAdd(a.done + block_of(u), 1u);
        }
    }
    if (SIG && TPW == 1 && warp == PBW) {
        // blocks of steps 0 .. q-2; steps before t0 finish no block of the
        // fused launch early: they are published together with step t0
        for (int pub = 0; pub < q - 1 && t0 < q - 1 && lane == 0;) {
            const unsigned need = (unsigned)(pub > t0 ? pub + 1 : t0 + 1);
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(dev::smem_u32(prog)) : "memory");
                if (v >= need) break;
                __nanosleep(a.pub_ns);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (; pub < (int)v; ++pub) atomicAdd(a.done + block_of(pub), 1u);
        }
        __syncwarp();
    }
    int st = 0, ph = 0;  // stage ring position of step t
    for (int t = 0; t < q && warp < SW; ++t) {
        const int i = block_of(t);
        if (trc && tid == 0) trc[(size_t)t * 16 + 0] = clock64(), trc[(size_t)t * 16 + 8] = (long long)dev::globaltimer();
        // ---------------- phase 1 ----------------
        AFrag va[TPW][KB];  // row warps: step t's update operands, split ahead of Z_t
        if (warp < NR) {
            if (t + 1 < q) {
                const int st1 = st + 1 == NSTG ? 0 : st + 1;
                const int ph1 = st + 1 == NSTG ? ph ^ 1 : ph;
                mbar_wait_u32(bar_u32 + 8u * st1, (uint32_t)ph1);
                partial_push(t + 1, st1);
            }
            const float* Vs = stg + st * SF + VOFF;
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const int rt = warp + u * NR;
                if (rt < RT) {
                    float v0[2 * KB], v1[2 * KB];
                    lds_vec<2 * KB>(v0, Vs + (rt * 16 + g) * LDV + tq * 2 * KB);
                    lds_vec<2 * KB>(v1, Vs + (rt * 16 + g + 8) * LDV + tq * 2 * KB);
#pragma unroll
                    for (int ks = 0; ks < KB; ++ks)
                        va[u][ks] = make_a(v0[2 * ks], v1[2 * ks], v0[2 * ks + 1], v1[2 * ks + 1]);
                }
            }
            if (trc && tid == 0) trc[(size_t)t * 16 + 2] = clock64();
        } else if (warp < NR + MT) {
            const int mt = warp - NR;
            float cm[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f}, c2[4] = {0.f, 0.f, 0.f, 0.f};
            mbar_wait_u32(bar_u32 + 8u * st, (uint32_t)ph);
            if (t > 0) {  // -2 S_t Z_{t-1}: Zn holds -2 Z_{t-1}, pre-split
                const float* Ss = stg + st * SF + SOFF;
                float s0[2 * KB], s1[2 * KB];
                lds_vec<2 * KB>(s0, Ss + (mt * 16 + g) * LDV + tq * 2 * KB);
                lds_vec<2 * KB>(s1, Ss + (mt * 16 + g + 8) * LDV + tq * 2 * KB);
                const float* zp = Zn + ((t - 1) & 1) * (KB * 128);
#pragma unroll
                for (int h2 = 0; h2 < KB / 2; ++h2) {
                    float zh[4], zl[4];
                    lds_vec<4>(zh, zp + h2 * 128 + ls4);
                    lds_vec<4>(zl, zp + (KB / 2) * 128 + h2 * 128 + ls4);
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const int ks = 2 * h2 + kk;
                        const AFrag af = make_a(s0[2 * ks], s1[2 * ks], s0[2 * ks + 1], s1[2 * ks + 1]);
                        mma3s(cm, c1, c2, af, zh[2 * kk], zh[2 * kk + 1], zl[2 * kk], zl[2 * kk + 1]);
                    }
                }
            }
            const int slot = t % NSLOTV;
            mbar_wait_u32(exb_u32 + 8u * slot, (uint32_t)((t / NSLOTV) & 1));
            if (trc && lane == 0 && mt == 0) trc[(size_t)t * 16 + 3] = clock64();
            // re-arm the slot for step t + NSLOTV (relaxed: it publishes nothing
            // of this thread's, and rank 0's B warp has Z' stores outstanding)
            if (lane == 0 && mt == 0) mbar_expect_relaxed_u32(exb_u32 + 8u * slot, ex_bytes);
            float z[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) z[e] = cm[e] + (c1[e] + c2[e]);
            if (trc && lane == 0 && mt == 0) trc[(size_t)t * 16 + 10] = clock64() + (long long)(z[0] != z[0]);
            const float* zr = Zr + ((size_t)slot * C * MT + mt) * 128 + lane * 4;
            float zs[4] = {0.f, 0.f, 0.f, 0.f};
            // fixed order over the source CTAs; ten 16-byte loads in flight
            // (two rounds of five: 56.34 vs 56.28 us, two: 57.6 us per fused
            // step; two-tile geometries keep two, their register budget spills)
            constexpr int ZU = TPW == 1 ? 10 : 2;
#pragma unroll ZU
            for (int c = 0; c < C; ++c) {
                float p[4];
                lds_vec<4>(p, zr + c * MT * 128);
#pragma unroll
                for (int e = 0; e < 4; ++e) zs[e] += p[e];
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) z[e] += zs[e];
            if (trc && lane == 0 && mt == 0) trc[(size_t)t * 16 + 11] = clock64() + (long long)(z[0] != z[0]);
            float* zc = Zn + (t & 1) * (KB * 128) + mt * 128;
            scatter_cb_swz(zc, zc + (KB / 2) * 128, z, g, tq, -2.f);
            if (!SIG && D.zhat && rank == 0) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = mt * 16 + g + 8 * (e >> 1), l = col0 + 2 * tq + (e & 1);
                    if (l < a.m) D.zhat[((size_t)i * BS + j) * a.m + l] = z[e];
                }
            }
            if (trc && lane == 0 && mt == 0) trc[(size_t)t * 16 + 4] = clock64();
        } else if (warp == PW && lane == 0) {
            // refill the stage step t-1 used (all its readers passed the last barrier)
            const int tn = t - 1 + NSTG;
            if (t > 0 && tn < q) {
                const int sp = st == 0 ? NSTG - 1 : st - 1;
                if (a.ready) wait_counter_bounded(a.ready + block_of(tn), (unsigned)C);
                mbar_expect_u32(bar_u32 + 8u * sp, stage_bytes);
                bulk_u32(dev::smem_u32(stg) + (uint32_t)sp * stage_bytes, gstage(tn), stage_bytes,
                         bar_u32 + 8u * sp);
            }
        } else if (pusher) {
            if (t + 1 < q) push_step(t + 1);
        }
        // the tape warp has read step t-1's Xn / Zn before either is reused
        if (SIG && warp < NR && t > 0) mbar_wait_u32(xfree_u32, (uint32_t)((t - 1) & 1));
        WSTAMP(0);
        if constexpr (NP > 0) {  // barrier 1 without the push warps: Z_t -> the update
            if (!pusher) asm volatile("bar.sync 2, %0;" ::"r"((NR + MT + 1) * 32) : "memory");
        } else if constexpr (SIG) {
            asm volatile("bar.sync 0, %0;" ::"r"(nmain) : "memory");
        } else {
            __syncthreads();
        }
        WSTAMP(1);
        if (trc && tid == 0) trc[(size_t)t * 16 + 5] = clock64();
        // ---------------- phase 2: X^(t+1) = X^(t) + V_t (-2 Z_t) ----------------
        if (warp < NR) {
            const float* zc = Zn + (t & 1) * (KB * 128);
            float zh[KB / 2][4], zl[KB / 2][4];
#pragma unroll
            for (int h2 = 0; h2 < KB / 2; ++h2) {
                lds_vec<4>(zh[h2], zc + h2 * 128 + ls4);
                lds_vec<4>(zl[h2], zc + (KB / 2) * 128 + h2 * 128 + ls4);
            }
            float* tblk = tape0 && !SIG ? tape0 + (size_t)i * tape_step : nullptr;
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const int rt = warp + u * NR;
                if (rt < RT) {
                    float* tp = tblk ? tblk + (rt * 16 + g) * WCV + 2 * tq : nullptr;
                    if (tp && !D.forward) {  // dA[i] = X^(t), the gradient at the block output
                        *reinterpret_cast<float2*>(tp) = make_float2(x[u][0], x[u][1]);
                        *reinterpret_cast<float2*>(tp + 8 * WCV) = make_float2(x[u][2], x[u][3]);
                    }
                    float c1[4] = {0.f, 0.f, 0.f, 0.f}, c2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int ks = 0; ks < KB; ++ks)
                        mma3s(x[u], c1, c2, va[u][ks], zh[ks >> 1][2 * (ks & 1)], zh[ks >> 1][2 * (ks & 1) + 1],
                              zl[ks >> 1][2 * (ks & 1)], zl[ks >> 1][2 * (ks & 1) + 1]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) x[u][e] += c1[e] + c2[e];
                    if (tp && D.forward) {  // A_i = activations[i]
                        *reinterpret_cast<float2*>(tp) = make_float2(x[u][0], x[u][1]);
                        *reinterpret_cast<float2*>(tp + 8 * WCV) = make_float2(x[u][2], x[u][3]);
                    }
                    if (SIG || t + 2 < q) scatter_cb_swz(xbuf(t + 1) + rt * 256, xbuf(t + 1) + rt * 256 + 128, x[u], g, tq, 1.f);
                }
            }
            __syncwarp();
            if (SIG && lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(xrdy_u32) : "memory");
            if (trc && tid == 0) trc[(size_t)t * 16 + 6] = clock64();
        }
        WSTAMP(2);
        if constexpr (NP > 0) {
            // no end-of-step barrier: the row warps go from the update straight
            // into the next step's partial (their own X tiles), the B warps are
            // already forming Z_{t+1}.  Safe: B warps overwrite Zn[t & 1] only
            // in step t+2, after barrier 1 of step t+1, which the row warps
            // reach after reading it here; every reader of a stage is done by
            // barrier 1 of its step, after which the producer refills it; the
            // push warps read a step's partials before pushing L_{t+1}, which
            // every CTA's Z_{t+1} (so barrier 1 of step t+1, before the row
            // warps write that buffer again) waits for
        } else {
            // none either: the row warps read the partials buffer (their own
            // combine) before barrier 1, and write it again after it
        }
        WSTAMP(3);
        if (trc && tid == 0) trc[(size_t)t * 16 + 7] = clock64(), trc[(size_t)t * 16 + 9] = (long long)dev::globaltimer();
        if (++st == NSTG) st = 0, ph ^= 1;
    }

    // x_out: the row warps stage their tiles column-major in the (consumed)
    // stage ring, then store 16 bytes at a time (whole lines: x_out may be a
    // caller's pinned host buffer).  With the publish warp, after its last
    // fence, so that fence does not wait for these stores.
    if (SIG && warp == PBW) asm volatile("bar.arrive 5, %0;" ::"r"((NR + 1) * 32) : "memory");
    if (warp < NR) {
        float* xs = stg;  // [WCV][RC + 4]
        const int LX = RC + 4;
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            const int rt = warp + u * NR;
            if (rt < RT) {
#pragma unroll
                for (int e = 0; e < 4; ++e) xs[(2 * tq + (e & 1)) * LX + rt * 16 + g + 8 * (e >> 1)] = x[u][e];
            }
        }
        if (SIG) asm volatile("bar.sync 5, %0;" ::"r"((NR + 1) * 32) : "memory");
        else dev::named_bar_sync<1>(NR * 32);
        if (warp == 0 && lane == 0) GSTAMP(14);
        const bool v4 = ((reinterpret_cast<uintptr_t>(D.x_out) & 15) == 0) && (D.ldo % 4 == 0);
        const int nr4 = RC / 4;
        for (int idx = warp * 32 + lane; idx < WCV * nr4; idx += NR * 32) {
            const int c = idx / nr4, r = (idx - c * nr4) * 4;
            const int gr = row0 + r, gc = col0 + c;
            if (gc >= a.m || gr >= a.d) continue;
            const float4 v = *reinterpret_cast<const float4*>(xs + c * LX + r);
            float* dst = D.x_out + (int64_t)gc * D.ldo + gr;
            if (v4 && gr + 4 <= a.d) {
                *reinterpret_cast<float4*>(dst) = v;
            } else {
                dst[0] = v.x;
                if (gr + 1 < a.d) dst[1] = v.y;
                if (gr + 2 < a.d) dst[2] = v.z;
                if (gr + 3 < a.d) dst[3] = v.w;
            }
        }
    }
    // no CTA may exit while a peer could still push into it
    dev::cluster_sync();
    GSTAMP(15);
#undef GSTAMP
#undef WSTAMP
}

template <int BS, int TPW, int NP>
cudaError_t launch_t(const SweepV2Args& a, cudaStream_t s) {
    const V2Smem L = v2_layout(a.C, BS, a.d_pad, a.nstg, a.done != nullptr);
    const bool tr = a.trace || a.wtrace;
    auto kern = a.done ? (tr ? sweep2_kernel<BS, TPW, true, NP, true> : sweep2_kernel<BS, TPW, true, NP, false>)
                       : (tr ? sweep2_kernel<BS, TPW, false, NP, true> : sweep2_kernel<BS, TPW, false, NP, false>);
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), L.total, true); e != cudaSuccess) return e;
    const int RT = a.d_pad / a.C / 16;
    const int NR = RT < MAXNR ? RT : MAXNR;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.C * a.ngroups * a.ndir, 1, 1);
    cfg.blockDim = dim3((NR + BS / 16 + 1 + NP + (a.done ? (TPW == 1 ? 2 : 1) : 0)) * 32, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// push warps (NP = 2) where the row-warp count allows them; FASTH_PUSHW=0 off
template <int TPW>
cudaError_t launch_bs(const SweepV2Args& a, cudaStream_t s) {
    const int RT = a.d_pad / a.C / 16;
    const int NR = RT < MAXNR ? RT : MAXNR;
    const char* e = getenv("FASTH_PUSHW");
    const bool push = TPW == 1 && NR <= kPushMaxNR && (!e || atoi(e) != 0);
    switch (a.BS) {
        case 16: return push ? launch_t<16, TPW, 2>(a, s) : launch_t<16, TPW, 0>(a, s);
        case 32: return push ? launch_t<32, TPW, 2>(a, s) : launch_t<32, TPW, 0>(a, s);
        case 64: return launch_t<64, TPW, 0>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

size_t sweep2_smem_bytes(int C, int BS, int d_pad, int nstg, bool sig) {
    return v2_layout(C, BS, d_pad, nstg, sig).total;
}

int sweep2_nstg(int C, int BS, int d_pad) {
    if (C < 1 || C > 16 || d_pad % C) return 0;
    const int RC = d_pad / C;
    if (RC % 16 || RC / 16 > 2 * MAXNR) return 0;
    if (BS != 16 && BS != 32 && BS != 64) return 0;
    int best = 0;
    for (int n = 2; n <= 4; ++n)
        if (sweep2_smem_bytes(C, BS, d_pad, n, false) <= 227 * 1024) best = n;
    return best;
}

// Chain geometry: C CTAs per cluster split the rows into RC (a multiple of
// 16) each; 8 batch columns per cluster.  ~80-row slabs up to 10 CTAs per
// cluster (measured on B200 at d = 784: 10 x 80 beats 7 x 112 by ~4% per
// fwd+bwd step).  Past d = 800: clusters of 12+ CTAs fit the GPCs only ~7 at
// a time, so a launch of 8+ clusters (the fused fwd+bwd at batch 32) runs a
// second wave; there 10-CTA clusters with up to 256-row slabs win (d = 1280
// / 1536 / 2048 / 2560: 245 -> 151, 299 -> 223, 434 -> 373, 683 -> 549 us per
// fused step), and up to d = 1536 for every launch (the builder's 10-CTA
// clusters pack better too: two-call d = 1280 242 -> 221 us), else ~112-row
// slabs (two-call d = 2048: 418 vs 546 us at C = 10; fused at batch <= 24
// too).  Widened until the packed-stage sweep fits shared memory.
// FASTH_CLUSTER overrides C.
SweepGeom pick_geometry(int d, int m, int BS, int num_sms, bool fused) {
    (void)num_sms;
    int C = (d + 79) / 80;
    if (C > 10) {
        const int clusters = (fused ? 2 : 1) * ((std::max(m, 1) + 7) / 8);
        C = d <= 1536 || (clusters >= 8 && d <= 2560) ? 10 : (d + 111) / 112;
    }
    C = C < 1 ? 1 : C > 16 ? 16 : C;
    if (const char* e = getenv("FASTH_CLUSTER")) C = atoi(e);
    if (C < 1 || C > 16) C = 8;
    auto rc_of = [&](int c) { return ((d + c - 1) / c + 15) / 16 * 16; };
    SweepGeom G;
    for (int c = C; c <= 16; ++c)
        if (rc_of(c) <= 256 && sweep2_nstg(c, BS, c * rc_of(c)) >= 2) {
            G.C = c;
            G.RC = rc_of(c);
            G.d_pad = c * G.RC;
            return G;
        }
    return G;  // C == 0: d too large for the chain kernels at this block width
}

cudaError_t launch_sweep2(const SweepV2Args& a, cudaStream_t s) {
    if (a.ndir < 1 || a.ndir > 2 || a.ngroups < 1 || a.q < 1) return cudaErrorInvalidValue;
    const int nst = sweep2_nstg(a.C, a.BS, a.d_pad);
    if (nst == 0 || a.nstg < 2 || a.nstg > nst) return cudaErrorInvalidConfiguration;
    const int RT = a.d_pad / a.C / 16;
    if (RT <= MAXNR) return launch_bs<1>(a, s);
    return launch_bs<2>(a, s);
}

}  // namespace fasthb
