// Sequential block chain: north_star subsystem (3) (forward, Alg. 1 step 2,
// fasth.hpp:58-59 / wy_apply wy.hpp:104-133) and the sweep of subsystem (4)
// (backward step 1, fasth.hpp:82-86 / wy_apply_transpose wy.hpp:137-146).
//
// One persistent launch runs ALL q dependent block steps.  Work split:
//   * batch columns are independent, so each thread-block CLUSTER owns a
//     group of WC = 8 columns of X and runs the whole chain on them;
//   * the C CTAs of a cluster split the rows: CTA r owns rows
//     [r*RC, (r+1)*RC) (RC a multiple of 16) of its column group for the
//     entire chain, held in tensor-core accumulator registers (one 16-row
//     tile per update warp) and mirrored in shared memory.
//
// Step t applies block P_t = I - 2 V_t T~_t V_t^T (backward: its transpose):
//     Z_t     = W_t^T X^(t)          (W = V T~^T forward, V T~ backward;
//                                     prebuilt by wy_build.cu)
//     X^(t+1) = X^(t) - 2 V_t Z_t
// Z_t is a reduction over ALL rows, i.e. over the cluster.  The chain is
// pipelined one block ahead (exact algebra, not a different blocking):
//     Z_{t+1} = W_{t+1}^T X^(t) - 2 S_t Z_t,     S_t = W_{t+1}^T V_t
// with S prebuilt by wy_build.cu.  Warp roles in iteration t:
//   A (warps [0, MT)):     L_{t+1} = W_{t+1,rows}^T X^(t)_rows, one 16-row
//                          M-tile of Z per warp, full K on the tensor cores
//                          (mma.sync m16n8k8, 3xTF32), pushed straight from
//                          the accumulators into every CTA of the cluster
//                          (st.async + receiver mbarrier complete_tx, DSMEM)
//   B (warps [MT, 2 MT)):  wait for all L_t; Z_t = sum_c L_t^c - 2 S_t Z_{t-1}
//                          (the correction on the tensor cores; the C-way sum
//                          in fixed order: deterministic, identical in every
//                          CTA)
//   -- barrier --
//   C (warps [0, RC/16)):  X^(t+1) = X^(t) - 2 V_t Z_t, 3xTF32 mma.sync into
//                          the warp's resident accumulator tile
//   -- barrier --
// A and B run concurrently; W, V and S are streamed in by the bulk-copy
// (TMA) engine NSTG blocks ahead into a ring of shared-memory stages.
#include "device_prims.cuh"
#include "fasth_internal.h"
#include "mma_tf32.cuh"

#include <cstdlib>

namespace fasthb {
namespace {

constexpr int NSLOT = 4;  // all-to-all receive slots (see the WAR argument below)
constexpr int NT = 512;   // threads per CTA
constexpr int NW = NT / 32;
constexpr int WC = 8;     // columns per cluster (one MMA N tile)

__host__ __device__ constexpr int ldw_of(int BS) { return BS + 8; }   // W rows: conflict-free A^T frags
__host__ __device__ constexpr int ldv_of(int BS) { return BS + 4; }   // V / S rows: conflict-free A frags

struct SweepSmem {
    size_t ws, vs, ss, xs, zr, zb, red, bars, total;
};

__host__ __device__ inline SweepSmem sweep_layout(int C, int BS, int d_pad, int NSTG) {
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
    o += (size_t)RC * WC * 4;
    L.zr = o;
    o += (size_t)NSLOT * C * ZN * 4;
    L.zb = o;
    o += 2 * (size_t)ZN * 4;
    o = (o + 15) & ~size_t(15);
    L.red = o;  // A-warp K-chunk partials, lane-indexed fragments
    o += (size_t)NW * 32 * 4 * 4;
    L.bars = o;
    o += (NSTG + NSLOT) * 8;
    L.total = o;
    return L;
}

// Warp roles (NW = 8 warps):
//   A warps [0, MT*KS):        L_{t+1} partials, M tile (w % MT), K chunk (w / MT)
//   B warps [MT*KS, MT*KS+MT): exchange reduction + look-ahead correction;
//                              the last warp also owns the W/V/S stage ring
//   C warps [0, RC/16):        resident X tiles, updated after barrier 1
template <int BS>
struct Roles {
    static constexpr int MT = BS / 16;                 // M tiles of Z
    static constexpr int KS = (NW - MT) / MT;          // K chunks of the partial
    static constexpr int NA = MT * KS;                 // A warps
    static constexpr int LOADW = NW - 1;               // stage-ring owner (a B warp)
    static_assert(NA + MT <= NW && LOADW >= NA, "roles");
};

// TPW: 16-row tiles of X per update warp (RC <= 128 * TPW)
template <int BS, int TPW>
__global__ void __launch_bounds__(NT, 1) sweep_kernel(SweepArgs a) {
    constexpr int LDW = ldw_of(BS), LDV = ldv_of(BS);
    constexpr int ZN = BS * WC;
    using R = Roles<BS>;
    constexpr int MT = R::MT, KS = R::KS, NA = R::NA;

    extern __shared__ __align__(128) unsigned char smem[];
    const int C = a.C;
    const int NSTG = a.nstg;
    const SweepSmem L = sweep_layout(C, BS, a.d_pad, NSTG);
    const int RC = a.d_pad / C;
    float* Ws = reinterpret_cast<float*>(smem + L.ws);
    float* Vs = reinterpret_cast<float*>(smem + L.vs);
    float* Ss = reinterpret_cast<float*>(smem + L.ss);
    float* Xs = reinterpret_cast<float*>(smem + L.xs);
    float* Zr = reinterpret_cast<float*>(smem + L.zr);
    float* Zb = reinterpret_cast<float*>(smem + L.zb);
    float* red = reinterpret_cast<float*>(smem + L.red);
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
    const int RT = RC / 16;  // row tiles of X in this CTA

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
        Xs[r * WC + l] = x;
    }
    // every CTA's barriers must be initialised and armed before a peer pushes
    dev::cluster_sync();

    // the update warps' resident X tiles (C fragments: rows g / g+8, cols 2tq, 2tq+1)
    float xr[TPW][4];
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        const int rt = warp + u * NW;
        if (rt < RT) {
            const float* x0 = Xs + (rt * 16 + g) * WC + 2 * tq;
            xr[u][0] = x0[0];
            xr[u][1] = x0[1];
            xr[u][2] = x0[8 * WC];
            xr[u][3] = x0[8 * WC + 1];
        }
    }

    const uint32_t zr_local = dev::smem_u32(Zr);
    const uint32_t exb_local = dev::smem_u32(ex_bar);
    const int KT = RC / 8;  // k-steps of the partial

    // A: L_t = W_t^T X over this warp's K chunk; chunk partials combined in
    // shared memory (lane-indexed fragments), chunk-0 warps push to every CTA
    auto partial_push = [&](int t) {
        const float* Wt = Ws + (size_t)(t % NSTG) * RC * LDW;
        const int mt = warp % MT, kc = warp / MT;
        const int m0 = mt * 16;
        const int kb = kc * KT / KS, ke = (kc + 1) * KT / KS;
        dev::Frag4 m0a = {{0.f, 0.f, 0.f, 0.f}}, c0a = m0a, m1a = m0a, c1a = m0a;
        int kt = kb;
        for (; kt + 1 < ke; kt += 2) {  // two independent accumulator chains
            const int k0 = kt * 8;
            {
                const float* w0 = Wt + (k0 + tq) * LDW + m0 + g;
                const float av[4] = {w0[0], w0[8], w0[4 * LDW], w0[4 * LDW + 8]};
                const float bv[2] = {Xs[(k0 + tq) * WC + g], Xs[(k0 + tq + 4) * WC + g]};
                dev::mma3(m0a, c0a, av, bv);
            }
            {
                const float* w0 = Wt + (k0 + 8 + tq) * LDW + m0 + g;
                const float av[4] = {w0[0], w0[8], w0[4 * LDW], w0[4 * LDW + 8]};
                const float bv[2] = {Xs[(k0 + 8 + tq) * WC + g], Xs[(k0 + 12 + tq) * WC + g]};
                dev::mma3(m1a, c1a, av, bv);
            }
        }
        if (kt < ke) {
            const int k0 = kt * 8;
            const float* w0 = Wt + (k0 + tq) * LDW + m0 + g;
            const float av[4] = {w0[0], w0[8], w0[4 * LDW], w0[4 * LDW + 8]};
            const float bv[2] = {Xs[(k0 + tq) * WC + g], Xs[(k0 + tq + 4) * WC + g]};
            dev::mma3(m0a, c0a, av, bv);
        }
        if (a.trace && threadIdx.x == 0 && t > 0) a.trace[((size_t)blockIdx.x * (q + 1) + t - 1) * 16 + 8] = clock64();
        float4 v = make_float4((m0a.v[0] + m1a.v[0]) + (c0a.v[0] + c1a.v[0]),
                               (m0a.v[1] + m1a.v[1]) + (c0a.v[1] + c1a.v[1]),
                               (m0a.v[2] + m1a.v[2]) + (c0a.v[2] + c1a.v[2]),
                               (m0a.v[3] + m1a.v[3]) + (c0a.v[3] + c1a.v[3]));
        if (KS > 1) {
            // every chunk warp of this M tile forms the same sum (fixed
            // order) and pushes it to its share of the destinations
            reinterpret_cast<float4*>(red)[(kc * MT + mt) * 32 + lane] = v;
            dev::named_bar_sync<1>(NA * 32);
            v = reinterpret_cast<const float4*>(red)[mt * 32 + lane];
#pragma unroll
            for (int c = 1; c < KS; ++c) {
                const float4 p = reinterpret_cast<const float4*>(red)[(c * MT + mt) * 32 + lane];
                v.x += p.x, v.y += p.y, v.z += p.z, v.w += p.w;
            }
        }
        if (a.trace && threadIdx.x == 0 && t > 0) a.trace[((size_t)blockIdx.x * (q + 1) + t - 1) * 16 + 9] = clock64();
        const int slot = t % NSLOT;
        // this lane's 4 fragment entries, contiguous in the receive slot
        // ([slot][source CTA][M tile][lane][4]): one 16-byte push per peer
        const uint32_t off = (uint32_t)((((slot * C + (int)rank) * MT + mt) * 32 + lane) * 16);
        const uint32_t bar = exb_local + slot * 8;
        if (C == 1) {  // st.async needs a peer CTA: local store + completion on the own barrier
            if (kc == 0) {
                const float w[4] = {v.x, v.y, v.z, v.w};
                dev::put4_local(zr_local + off, w);
                dev::complete_tx_local(bar, 16u);
            }
        } else {
            for (int dst = kc; dst < C; dst += KS)
                dev::st_async_f32x4(dev::mapa(zr_local + off, dst), v.x, v.y, v.z, v.w, dev::mapa(bar, dst));
        }
    };

    // debug phase trace (FASTH_TRACE): clock64 per phase.  Slots: 0 top,
    // 1 A start, 2 A done, 3 B after the exchange wait, 4 B done (slots 1-2
    // by thread 0 of warp 0, 3-4 by lane 0 of the first B warp), 5 after
    // barrier 1, 6 C done, 7 after barrier 2.
    long long* trc = a.trace ? a.trace + (size_t)blockIdx.x * (q + 1) * 16 : nullptr;
    auto mark_by = [&](int who, int t, int k) {
        if (trc && tid == who) trc[(size_t)t * 16 + k] = clock64();
    };
    auto mark = [&](int t, int k) { mark_by(0, t, k); };
    mark(q, 0);
    if (q > 0 && warp < NA) {  // prologue: groups 0 and 1 landed, L_0
        wait_group(0);
        if (q > 1) wait_group(1);
        partial_push(0);
    }
    mark(q, 1);

    for (int t = 0; t < q; ++t) {
        const int i = block_of(t);
        const int st = t % NSTG;
        const int slot = t % NSLOT;
        float* tape_blk = a.tape ? a.tape + (((size_t)i * ngroups + group) * a.d_pad + row0) * WC : nullptr;
        mark(t, 0);

        if (warp < NA) {
            // A. look-ahead partial for step t+1 (overlaps the exchange of L_t)
            mark(t, 1);
            if (t + 1 < q) partial_push(t + 1);
            mark(t, 2);
        } else if (warp < NA + MT) {
            // the ring owner refills the stage freed at the end of step t-1
            // and makes sure group t+2 (next step's A operand) has landed
            if (warp == R::LOADW && lane == 0) {
                if (t > 0 && t - 1 + NSTG < q) issue_load(t - 1 + NSTG);
                if (t + 2 < q) wait_group(t + 2);
            }
            // B. Z_t = sum_c L_t^c - 2 S_t Z_{t-1}, M tile (warp - NA)
            const int m0 = (warp - NA) * 16;
            float* Zc = Zb + (t & 1) * ZN;
            const float* Zp = Zb + ((t + 1) & 1) * ZN;
            dev::Frag4 cm = {{0.f, 0.f, 0.f, 0.f}}, cc = cm;
            if (t > 0) {
                const float* Sst = Ss + (size_t)st * BS * LDV;
#pragma unroll
                for (int k0 = 0; k0 < BS; k0 += 8) {
                    const float* s0 = Sst + (m0 + g) * LDV + k0 + tq;
                    const float av[4] = {s0[0], s0[8 * LDV], s0[4], s0[8 * LDV + 4]};
                    const float bv[2] = {-2.f * Zp[(k0 + tq) * WC + g], -2.f * Zp[(k0 + tq + 4) * WC + g]};
                    dev::mma3(cm, cc, av, bv);
                }
            }
            dev::mbar_wait(&ex_bar[slot], (uint32_t)(t / NSLOT) & 1u);
            mark_by(NA * 32, t, 3);
            // WAR safety of the slot: a peer pushes L_{t+4} into it only after
            // it has Z_{t+2}, which needs our L_{t+2}, pushed after this read.
            if (lane == 0 && warp == NA) dev::mbar_arrive_expect_tx(&ex_bar[slot], ex_bytes);
            const float* zr = Zr + (size_t)slot * C * ZN + ((warp - NA) * 32 + lane) * 4;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
            for (int c = 0; c < C; ++c) {  // fixed order over the source CTAs
                const float4 p = *reinterpret_cast<const float4*>(zr + c * ZN);
                s0 += p.x, s1 += p.y, s2 += p.z, s3 += p.w;
            }
            const float z[4] = {s0 + (cm.v[0] + cc.v[0]), s1 + (cm.v[1] + cc.v[1]),
                                s2 + (cm.v[2] + cc.v[2]), s3 + (cm.v[3] + cc.v[3])};
            float* zc0 = Zc + (m0 + g) * WC + 2 * tq;
            *reinterpret_cast<float2*>(zc0) = make_float2(z[0], z[1]);
            *reinterpret_cast<float2*>(zc0 + 8 * WC) = make_float2(z[2], z[3]);
            if (a.zhat && rank == 0) {
                const int l = col0 + 2 * tq;
                float* zh = a.zhat + ((size_t)i * BS + m0 + g) * a.m + l;
                if (l < a.m) zh[0] = z[0], zh[8 * (size_t)a.m] = z[2];
                if (l + 1 < a.m) zh[1] = z[1], zh[8 * (size_t)a.m + 1] = z[3];
            }
            mark_by(NA * 32, t, 4);
        }
        __syncthreads();
        mark(t, 5);

        // C. X^(t+1) = X^(t) - 2 V_t Z_t into the resident tiles
        {
            const float* Vt = Vs + (size_t)st * RC * LDV;
            const float* Zc = Zb + (t & 1) * ZN;
            if (TPW == 1 && 2 * RT <= NW) {
                // two warps per row tile, each half of K; the upper half's
                // product meets the resident tile through shared memory
                if (warp < 2 * RT) {
                    const int kh = warp < RT ? 0 : 1, rt = warp - kh * RT;
                    const int r0 = rt * 16;
                    float* t0 = tape_blk ? tape_blk + (r0 + g) * WC + 2 * tq : nullptr;
                    if (kh == 0 && !a.forward && t0) {  // dA[i] = X^(t)
                        *reinterpret_cast<float2*>(t0) = make_float2(xr[0][0], xr[0][1]);
                        *reinterpret_cast<float2*>(t0 + 8 * WC) = make_float2(xr[0][2], xr[0][3]);
                    }
                    dev::Frag4 m = {{0.f, 0.f, 0.f, 0.f}}, cc = m;
                    if (kh == 0) m = {{xr[0][0], xr[0][1], xr[0][2], xr[0][3]}};
#pragma unroll
                    for (int k0 = kh * (BS / 2); k0 < (kh + 1) * (BS / 2); k0 += 8) {
                        const float* v0 = Vt + (r0 + g) * LDV + k0 + tq;
                        const float av[4] = {v0[0], v0[8 * LDV], v0[4], v0[8 * LDV + 4]};
                        const float bv[2] = {-2.f * Zc[(k0 + tq) * WC + g], -2.f * Zc[(k0 + tq + 4) * WC + g]};
                        dev::mma3(m, cc, av, bv);
                    }
                    float4* hand = reinterpret_cast<float4*>(red) + rt * 32 + lane;
                    if (kh == 1) *hand = make_float4(m.v[0] + cc.v[0], m.v[1] + cc.v[1], m.v[2] + cc.v[2], m.v[3] + cc.v[3]);
                    dev::named_bar_sync<2>(2 * RT * 32);
                    if (kh == 0) {
                        const float4 p = *hand;
                        xr[0][0] = (m.v[0] + cc.v[0]) + p.x;
                        xr[0][1] = (m.v[1] + cc.v[1]) + p.y;
                        xr[0][2] = (m.v[2] + cc.v[2]) + p.z;
                        xr[0][3] = (m.v[3] + cc.v[3]) + p.w;
                        float* x0 = Xs + (r0 + g) * WC + 2 * tq;
                        *reinterpret_cast<float2*>(x0) = make_float2(xr[0][0], xr[0][1]);
                        *reinterpret_cast<float2*>(x0 + 8 * WC) = make_float2(xr[0][2], xr[0][3]);
                        if (a.forward && t0) {  // A_i = activations[i]
                            *reinterpret_cast<float2*>(t0) = make_float2(xr[0][0], xr[0][1]);
                            *reinterpret_cast<float2*>(t0 + 8 * WC) = make_float2(xr[0][2], xr[0][3]);
                        }
                    }
                }
            } else
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const int rt = warp + u * NW;
                if (rt < RT) {
                    const int r0 = rt * 16;
                    float* t0 = tape_blk ? tape_blk + (r0 + g) * WC + 2 * tq : nullptr;
                    if (!a.forward && t0) {  // dA[i] = X^(t), the gradient at the block output
                        *reinterpret_cast<float2*>(t0) = make_float2(xr[u][0], xr[u][1]);
                        *reinterpret_cast<float2*>(t0 + 8 * WC) = make_float2(xr[u][2], xr[u][3]);
                    }
                    dev::Frag4 m = {{xr[u][0], xr[u][1], xr[u][2], xr[u][3]}};
                    dev::Frag4 cc = {{0.f, 0.f, 0.f, 0.f}};
#pragma unroll
                    for (int k0 = 0; k0 < BS; k0 += 8) {
                        const float* v0 = Vt + (r0 + g) * LDV + k0 + tq;
                        const float av[4] = {v0[0], v0[8 * LDV], v0[4], v0[8 * LDV + 4]};
                        const float bv[2] = {-2.f * Zc[(k0 + tq) * WC + g], -2.f * Zc[(k0 + tq + 4) * WC + g]};
                        dev::mma3(m, cc, av, bv);
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) xr[u][e] = m.v[e] + cc.v[e];
                    float* x0 = Xs + (r0 + g) * WC + 2 * tq;
                    *reinterpret_cast<float2*>(x0) = make_float2(xr[u][0], xr[u][1]);
                    *reinterpret_cast<float2*>(x0 + 8 * WC) = make_float2(xr[u][2], xr[u][3]);
                    if (a.forward && t0) {  // A_i = activations[i]
                        *reinterpret_cast<float2*>(t0) = make_float2(xr[u][0], xr[u][1]);
                        *reinterpret_cast<float2*>(t0 + 8 * WC) = make_float2(xr[u][2], xr[u][3]);
                    }
                }
            }
        }
        mark(t, 6);
        __syncthreads();
        mark(t, 7);
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

template <int BS, int TPW>
cudaError_t launch_t(const SweepArgs& a, cudaStream_t s) {
    const SweepSmem L = sweep_layout(a.C, BS, a.d_pad, a.nstg);
    auto kern = sweep_kernel<BS, TPW>;
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), L.total, true); e != cudaSuccess) return e;
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

template <int TPW>
cudaError_t launch_bs(const SweepArgs& a, cudaStream_t s) {
    switch (a.BS) {
        case 16: return launch_t<16, TPW>(a, s);
        case 32: return launch_t<32, TPW>(a, s);
        case 64: return launch_t<64, TPW>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

size_t sweep_smem_bytes(int C, int WCc, int BS, int d_pad, int nstg) {
    (void)WCc;
    return sweep_layout(C, BS, d_pad, nstg).total;
}

int sweep_ldw(int BS) { return ldw_of(BS); }
int sweep_ldv(int BS) { return ldv_of(BS); }

// Chain geometry: C CTAs per cluster split the rows into RC = 16-row
// multiples near 112 rows each (d = 784 -> 7 x 112, no padding); 8 columns per
// cluster.  FASTH_CLUSTER overrides C.
SweepGeom pick_geometry(int d, int m, int BS, int num_sms) {
    (void)m;
    (void)num_sms;
    SweepGeom G;
    // ~80-row slabs up to 10 CTAs per cluster (measured on B200 at d = 784:
    // 10 x 80 beats 7 x 112 by ~4% per fwd+bwd step; 12+ CTA clusters no longer
    // fit the fused launch's 8 clusters at once), else ~112-row slabs
    int C = (d + 79) / 80;
    if (C > 10) C = (d + 111) / 112;
    if (C < 1) C = 1;
    if (C > 16) C = 16;
    if (const char* e = getenv("FASTH_CLUSTER")) C = atoi(e);
    if (C < 1 || C > 16) C = 8;
    auto rc_of = [&](int c) { return ((d + c - 1) / c + 15) / 16 * 16; };
    constexpr size_t kBudget = 220 * 1024;
    // the packed-stage sweep (chain_v2.cu) fits as chosen: keep C (the v1
    // kernel's larger footprint must not widen the cluster past the GPC fit)
    const bool v2_fits = rc_of(C) <= 256 && sweep2_nstg(C, BS, C * rc_of(C)) >= 2;
    while (!v2_fits && C < 16 && (sweep_smem_bytes(C, WC, BS, C * rc_of(C), 3) > kBudget || rc_of(C) > 256)) ++C;
    // the packed-stage sweep (chain_v2.cu) must fit: widen the cluster if not
    for (int c2 = C; c2 <= 16; ++c2)
        if (sweep2_nstg(c2, BS, c2 * rc_of(c2)) >= 2) {
            C = c2;
            break;
        }
    G.C = C;
    G.RC = rc_of(C);
    G.d_pad = C * G.RC;
    G.WC = WC;
    G.nstg = 2;
    while (G.nstg < 4 && sweep_smem_bytes(C, WC, BS, G.d_pad, G.nstg + 1) <= kBudget) ++G.nstg;
    return G;
}

cudaError_t launch_sweep(const SweepArgs& a, int WCc, cudaStream_t s) {
    const int RC = a.C > 0 ? a.d_pad / a.C : 0;
    if (WCc != WC || a.C < 1 || a.C > 16 || a.d_pad % a.C != 0 || RC % 16 != 0) return cudaErrorInvalidValue;
    if (a.nstg < 2 || a.nstg > 4) return cudaErrorInvalidValue;
    if (sweep_smem_bytes(a.C, WC, a.BS, a.d_pad, a.nstg) > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (RC <= 16 * NW) return launch_bs<1>(a, s);
    if (RC <= 32 * NW) return launch_bs<2>(a, s);
    return cudaErrorInvalidConfiguration;
}

}  // namespace fasthb
