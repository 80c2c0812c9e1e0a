// WY-block builder, v4: north_star subsystem (2) — the UT form of the
// reference's compact WY (wy_compact, wy.hpp:56-100) with
// raw vectors,
//     H_1 ... H_w = I - 2 V T~ V^T,   T~ = M^{-1},  M = diag(V^T V) + 2 striu(V^T V),
// written straight into the packed chain stages (fasth_internal.h) that the
// sweep (chain_v2.cu) streams.  Same outputs as build2 (wy_build2.cu),
// re-laid out for the instruction budget: build2 issued ~40K warp
// instructions per CTA (per-row triangular solves: 512 dependent FMAs and
// shared loads per row; FP64 tensor-core Gram; index arithmetic per element)
// and the B200 ran it issue-bound (ncu: 37% issue-active, 2 CTAs per SM).
//
// One cluster of C CTAs per block i (C = the sweep's cluster size, so CTA r
// owns exactly the rows [r RB, (r+1) RB) its sweep CTA streams):
//   1. its RB rows of blocks i, i-1, i+1 into shared memory, rows permuted
//      inside each 16-row chunk (position 4 (r & 3) + (r >> 2 & 3)) so that a
//      lane's operands of two consecutive k-steps are one 16-byte load;
//   2. partial Gram band over those rows, 3xTF32 mma.sync (three accumulator
//      chains): G_ii, G_{i,i+1} = V_i^T V_{i+1}, G_{i,i-1} = V_i^T V_{i-1};
//   3. cluster reduction by DSMEM pushes only: every CTA pushes slice r of
//      its partial to CTA r (st.async.v4 + the owner's mbarrier), the owner
//      sums the C partials in fixed source order (f64) and pushes the result
//      slice to every CTA — deterministic, identical in every CTA;
//   4. every CTA: T~ = M^{-1} by the 2x2 block recursion
//      [A B; 0 C]^{-1} = [A^{-1}, -A^{-1} B C^{-1}; 0, C^{-1}] (log2(BS)
//      levels, fully unrolled, fp32), the look-ahead corrections
//      Sf_i = T~ G_{i,i+1}, Sb_i = T~^T G_{i,i-1} (chain_v2.cu) and its rows
//      Wf = V T~^T, Wb = V T~ (3xTF32, B operands pre-split), written into
//      shared-memory images of its packed stages at the fragment-order
//      positions;
//   5. three bulk stores shared -> global (forward stage, backward stage,
//      raw rows for the gradient kernel).
#include "device_prims.cuh"
#include "fasth_internal.h"
#include "frag_ops.cuh"

namespace fasthb {
namespace {
using namespace fo;

constexpr int NTH4 = 256;

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
// V^T row pitch: >= RB and == 16 (mod 32), so the 16-byte fragment loads of
// eight lanes (g = 0, 1; tq = 0..3) hit 32 distinct banks
__host__ __device__ inline int b4_pitch(int RB) { return RB % 32 == 16 ? RB : RB + 16; }
// position of row r inside its 16-row chunk (an involution)
__host__ __device__ __forceinline__ int b4_pos(int r) { return (r & ~15) | ((r & 3) << 2) | ((r >> 2) & 3); }

struct B4Layout {
    // byte offsets.  Live through the image phase: vc, small matrices; the
    // stage images alias everything from vpn on (dead by then).
    size_t vc, tfs, tts, gnt, gpt, vpn, gp, recv, gr, td, ty, img_pf, img_pb, img_vb, bars, total;
    int P;    // V^T row pitch (floats)
    int per;  // reduction slice (floats, multiple of 4)
};

__host__ __device__ inline B4Layout b4_layout(int BS, int RB, int C) {
    B4Layout L;
    L.P = b4_pitch(RB);
    const size_t E1 = (size_t)BS * BS, E = 3 * E1;
    L.per = (int)(((E + C - 1) / C + 3) / 4 * 4);
    const size_t SF = stage_floats(RB, BS);
    const size_t LD2 = (size_t)BS + 4;  // pitch of the (hi, lo) planes, float2 units
    size_t o = 0;
    L.vc = o;  // V^T rows of block i (permuted)
    o += al16((size_t)BS * L.P * 4);
    L.tfs = o;  // T~ as (hi, lo) pairs, row-major
    o += al16((size_t)BS * LD2 * 8);
    L.tts = o;  // T~^T as (hi, lo) pairs
    o += al16((size_t)BS * LD2 * 8);
    L.gnt = o;  // G_{i,i+1}^T, fp32, pitch BS + 1 (conflict-free transposed stores)
    o += al16((size_t)BS * (BS + 4) * 4);
    L.gpt = o;  // G_{i,i-1}^T
    o += al16((size_t)BS * (BS + 4) * 4);
    const size_t dead = o;
    L.vpn = o;  // V^T rows of blocks i-1, i+1
    o += al16((size_t)2 * BS * L.P * 4);
    L.gp = o;  // partial band [3][BS][BS]
    o += al16(E * 4);
    L.recv = o;  // partial slices from the peers [C][per]
    o += al16((size_t)C * L.per * 4);
    L.gr = o;  // reduced band
    o += al16((size_t)C * L.per * 4 > E * 4 ? (size_t)C * L.per * 4 : E * 4);
    L.td = o;  // T~ recursion (fp32) [BS][BS+1]
    o += al16((size_t)BS * (BS + 1) * 4);
    L.ty = o;
    o += al16(E1 / 4 * 4 + 4);
    L.img_pf = dead;
    L.img_pb = L.img_pf + al16(SF * 4);
    L.img_vb = L.img_pb + al16(SF * 4);
    const size_t im = L.img_vb + al16((size_t)RB * stage_ldv(BS) * 4);
    if (im > o) o = im;
    L.bars = o;
    o += 32;
    L.total = o;
    return L;
}

__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                 "r"(__float_as_uint(v.w)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ float2 split2f(float x) { return make_float2(__uint_as_float(hi_rn(x)), lo_rn(x)); }

// One level of the 2x2 block recursion for T~ = M^{-1} (blocks of S -> 2S):
// for each diagonal pair [A B; 0 C] (A, C already inverted in place, B = 2 G),
// Y = B C^{-1}, then the upper-right block X = -A^{-1} Y.
template <int BS, int S>
__device__ __forceinline__ void t_level(const float* Gr, float* Td, float* Ty, int tid) {
    constexpr int LDT = BS + 1;
    constexpr int OUTS = (BS / (2 * S)) * S * S;
    for (int o = tid; o < OUTS; o += NTH4) {
        const int pr = o / (S * S), rr = (o / S) % S, cc = o % S;
        const int a0 = 2 * pr * S, c0 = a0 + S;
        const float* gr = Gr + (a0 + rr) * BS + c0;
        const float* tc = Td + c0 * LDT + c0 + cc;
        float y = 0.f;
#pragma unroll
        for (int k = 0; k < S; ++k) y = fmaf(gr[k], tc[k * LDT], y);
        Ty[o] = 2.f * y;
    }
    __syncthreads();
    for (int o = tid; o < OUTS; o += NTH4) {
        const int pr = o / (S * S), rr = (o / S) % S, cc = o % S;
        const int a0 = 2 * pr * S, c0 = a0 + S;
        const float* ta = Td + (a0 + rr) * LDT + a0;
        const float* ty = Ty + pr * S * S + cc;
        float x = 0.f;
#pragma unroll
        for (int k = 0; k < S; ++k) x = fmaf(ta[k], ty[k * S], x);
        Td[(a0 + rr) * LDT + c0 + cc] = -x;
    }
    __syncthreads();
}

template <int BS>
__global__ void __launch_bounds__(NTH4, BS == 64 ? 1 : 2) build4_kernel(Plan p, const float* __restrict__ V, int64_t ldv,
                                                         int vec_ok, ErrWord* err) {
    constexpr int MT = BS / 16, NT = BS / 8, KB = BS / 8;
    constexpr int E1 = BS * BS;
    constexpr int LD2 = BS + 4, LDG = BS + 1, LDT = BS + 1;
    constexpr int LDW = stage_ldw(BS), LDV = stage_ldv(BS);
    extern __shared__ __align__(128) unsigned char smem[];
    const int C = p.CB, RB = p.d_pad / C;
    const B4Layout L = b4_layout(BS, RB, C);
    const int P = L.P;
    float* Vc = reinterpret_cast<float*>(smem + L.vc);    // [j][P] block i
    float* Vpn = reinterpret_cast<float*>(smem + L.vpn);  // [2][j][P] blocks i-1, i+1
    float2* TfS = reinterpret_cast<float2*>(smem + L.tfs);
    float2* TTS = reinterpret_cast<float2*>(smem + L.tts);
    float* GnT = reinterpret_cast<float*>(smem + L.gnt);
    float* GpT = reinterpret_cast<float*>(smem + L.gpt);
    float* Gp = reinterpret_cast<float*>(smem + L.gp);  // [3][BS][BS]: ii, (i,i+1), (i,i-1)
    float* recv = reinterpret_cast<float*>(smem + L.recv);
    float* Gr = reinterpret_cast<float*>(smem + L.gr);
    float* Td = reinterpret_cast<float*>(smem + L.td);  // [BS][BS+1]
    float* Ty = reinterpret_cast<float*>(smem + L.ty);
    float* IPF = reinterpret_cast<float*>(smem + L.img_pf);
    float* IPB = reinterpret_cast<float*>(smem + L.img_pb);
    float* IVB = reinterpret_cast<float*>(smem + L.img_vb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);  // 0 partial slices, 1 results

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const int rank = (int)dev::cluster_ctarank();
    const int row0 = rank * RB;
    const int nrows = max(0, min(RB, p.d - row0));
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // L2 prefetch of the sweep's first reads (X, G), one 128-byte line per thread
    if (p.pf_cols > 0) {
        const int nl = (p.pf_rows + 31) / 32, per_m = nl * p.pf_cols;
        for (int k = blockIdx.x * NTH4 + tid; k < 2 * per_m; k += gridDim.x * NTH4) {
            const int mi = k >= per_m, kk = k - mi * per_m, c = kk / nl, l = kk - c * nl;
            const float* base = p.pf[mi];
            if (base) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (int64_t)c * p.pf_ld[mi] + 32 * l));
        }
    }
    constexpr int E = 3 * E1;
    const int per = L.per;
    const int mylo = min(E, rank * per), myhi = min(E, mylo + per), mylen = myhi - mylo;
    const uint32_t barA = dev::smem_u32(&bars[0]), barB = dev::smem_u32(&bars[1]);

    // One block per cluster, or (p.nbuild > 0) persistent clusters taking
    // blocks cj, cj + nclusters, ...: the streamed host step builds on a few
    // clusters so that the sweep finds its SMs free.  Streamed, blocks go in
    // the upload's (and the two chains') order 0, q-1, 1, q-2, ...
    const int ncl = (int)gridDim.x / C;
    for (int cj = (int)dev::cluster_id_x(), it = 0; p.nbuild > 0 ? cj < p.q : it == 0; cj += ncl, ++it) {
    const int i = p.upc ? ((cj & 1) ? p.q - 1 - (cj >> 1) : (cj >> 1)) : p.blk_lo + cj;
    const int w = min(p.b, p.n - i * p.b);
    if (it > 0) __syncthreads();  // the previous block's shared-memory readers are done
#define BTRACE(k) \
    if (p.trace && tid == 0) p.trace[((size_t)i * C + rank) * 10 + (k)] = clock64()
    BTRACE(0);
    if (p.trace && tid == 0) p.trace[((size_t)i * C + rank) * 10 + 8] = (long long)dev::globaltimer();
    // 1. rows of blocks i (slot 0), i-1 (1), i+1 (2), permuted positions:
    //    thread k takes 4-row group k % RG of column k / RG (consecutive
    //    threads walk down a column: whole lines), eight 16-byte loads in
    //    flight per thread (one round trip at b = 32, 80-row slabs).  The
    //    phase is issue-bound at two CTAs per SM: (column, group) advance
    //    incrementally, no division per element
    //    Streamed host step (p.upc): V's columns arrive while the builder
    //    runs; wait until blocks i-1..i+1 have landed (L2-coherent loads)
    if (p.upc) {
        if (tid == 0)
            for (int k = max(i - 1, 0); k <= min(i + 1, p.q - 1); ++k) wait_counter_bounded(p.upc + k, p.upc_target);
        __syncthreads();
    }
    {
        constexpr int NB = 8;
        const int RG = RB / 4, NTOT = 3 * BS * RG;
        const int dq = NTH4 / RG, dr = NTH4 - dq * RG;
        float* sf = reinterpret_cast<float*>(smem);
        int jj = tid / RG, rg = tid - jj * RG;
        for (int kb = tid; kb < NTOT; kb += NB * NTH4) {
            float4 v[NB];
            int dofs[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                const int r = 4 * rg;
                const int sl = jj / BS, j = jj - sl * BS;
                const int blk = sl == 0 ? i : sl == 1 ? i - 1 : i + 1;
                const int k0 = blk * p.b;
                const bool in = jj < 3 * BS;
                const int wb = (in && blk >= 0 && blk < p.q) ? min(p.b, p.n - k0) : 0;
                dofs[u] = in ? (jj < BS ? L.vc / 4 + jj * P : L.vpn / 4 + (jj - BS) * P) + b4_pos(r) : -1;
                if (j < wb && r < nrows) {
                    const float* src = V + (int64_t)(p.reversed ? p.n - 1 - (k0 + j) : k0 + j) * ldv + row0 + r;
                    if (vec_ok && r + 4 <= nrows) {
                        v[u] = __ldcg(reinterpret_cast<const float4*>(src));
                    } else {
                        v[u].x = __ldcg(src);
                        if (r + 1 < nrows) v[u].y = __ldcg(src + 1);
                        if (r + 2 < nrows) v[u].z = __ldcg(src + 2);
                        if (r + 3 < nrows) v[u].w = __ldcg(src + 3);
                    }
                }
                jj += dq, rg += dr;
                if (rg >= RG) rg -= RG, ++jj;
            }
#pragma unroll
            for (int u = 0; u < NB; ++u)
                if (dofs[u] >= 0) {  // rows r + e -> position + 4 e
                    float* dst = sf + dofs[u];
                    dst[0] = v[u].x, dst[4] = v[u].y, dst[8] = v[u].z, dst[12] = v[u].w;
                }
        }
    }
    if (tid == 0) {
        if (it == 0) {
            dev::mbar_init(&bars[0], 1);
            dev::mbar_init(&bars[1], 1);
            dev::fence_mbar_init();
        }
        mbar_expect_u32(barA, (uint32_t)((C - 1) * mylen * 4));
        mbar_expect_u32(barB, (uint32_t)((E - mylen) * 4));
    }
    __syncthreads();
    // peers may push once every CTA has armed its barriers: arrive now, wait
    // just before the first push (the loads and the Gram run in between)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

    BTRACE(1);

    // 2. partial band: warp w -> m-tile (w & 1) of V_i^T, n-tile (w >> 1) of
    //    each product; one 16-row chunk = two k-steps per 16-byte load
    {
        const float* Vn = Vpn + (size_t)BS * P;
        const float* Vp = Vpn;
        for (int u = warp; u < MT * NT; u += NTH4 / 32) {
            const int mt = u % MT, nt = u / MT;
            float acc[3][3][4];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.f;
            const float* a_lo = Vc + (size_t)(mt * 16 + g) * P + 4 * tq;
            const float* a_hi = a_lo + 8 * P;
            const float* b_[3] = {Vc + (size_t)(nt * 8 + g) * P + 4 * tq, Vn + (size_t)(nt * 8 + g) * P + 4 * tq,
                                  Vp + (size_t)(nt * 8 + g) * P + 4 * tq};
#pragma unroll 2
            for (int c16 = 0; c16 < RB; c16 += 16) {
                const float4 x0 = *reinterpret_cast<const float4*>(a_lo + c16);
                const float4 x1 = *reinterpret_cast<const float4*>(a_hi + c16);
                const AFrag f0 = make_a(x0.x, x1.x, x0.y, x1.y);  // k-step 2 c16/8
                const AFrag f1 = make_a(x0.z, x1.z, x0.w, x1.w);  // k-step 2 c16/8 + 1
#pragma unroll
                for (int pr = 0; pr < 3; ++pr) {
                    const float4 y = *reinterpret_cast<const float4*>(b_[pr] + c16);
                    mma3s(acc[pr][0], acc[pr][1], acc[pr][2], f0, __uint_as_float(hi_rn(y.x)),
                          __uint_as_float(hi_rn(y.y)), lo_rn(y.x), lo_rn(y.y));
                    mma3s(acc[pr][0], acc[pr][1], acc[pr][2], f1, __uint_as_float(hi_rn(y.z)),
                          __uint_as_float(hi_rn(y.w)), lo_rn(y.z), lo_rn(y.w));
                }
            }
#pragma unroll
            for (int pr = 0; pr < 3; ++pr) {
                float* out = Gp + pr * E1 + (mt * 16 + g) * BS + nt * 8 + 2 * tq;
                *reinterpret_cast<float2*>(out) = make_float2(acc[pr][0][0] + (acc[pr][1][0] + acc[pr][2][0]),
                                                              acc[pr][0][1] + (acc[pr][1][1] + acc[pr][2][1]));
                *reinterpret_cast<float2*>(out + 8 * BS) = make_float2(
                    acc[pr][0][2] + (acc[pr][1][2] + acc[pr][2][2]), acc[pr][0][3] + (acc[pr][1][3] + acc[pr][2][3]));
            }
        }
    }
    __syncthreads();
    BTRACE(2);

    // 3a. slice r of my partial -> CTA r (16-byte pushes)
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    {
        const int per4 = per / 4;
        const uint32_t recv_u32 = dev::smem_u32(recv) + (uint32_t)(rank * per) * 4u;
        for (int idx = tid; idx < (C - 1) * per4; idx += NTH4) {
            const int rr = idx / per4, q4 = idx - rr * per4;
            const int r = rr + (rr >= rank);
            const int e = r * per + 4 * q4;
            if (e < E)
                st_async_v4(dev::mapa(recv_u32 + (uint32_t)q4 * 16u, (uint32_t)r),
                            *reinterpret_cast<const float4*>(Gp + e), dev::mapa(barA, (uint32_t)r));
        }
    }
    // 3b. my slice: sum the C partials in source order (f64), push the result
    mbar_wait_acq_cluster(barA, (uint32_t)(it & 1));
    {
        const uint32_t gr_u32 = dev::smem_u32(Gr);
        for (int q4 = tid; 4 * q4 < mylen; q4 += NTH4) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            for (int src = 0; src < C; ++src) {
                const float4 v = *reinterpret_cast<const float4*>(src == rank ? Gp + mylo + 4 * q4
                                                                              : recv + (size_t)src * per + 4 * q4);
                s0 += v.x, s1 += v.y, s2 += v.z, s3 += v.w;
            }
            const float4 f = make_float4((float)s0, (float)s1, (float)s2, (float)s3);
            *reinterpret_cast<float4*>(Gr + mylo + 4 * q4) = f;
            const uint32_t off = gr_u32 + (uint32_t)(mylo + 4 * q4) * 4u;
            for (int r = 0; r < C; ++r)
                if (r != rank) st_async_v4(dev::mapa(off, (uint32_t)r), f, dev::mapa(barB, (uint32_t)r));
        }
    }
    BTRACE(3);
    mbar_wait_acq_cluster(barB, (uint32_t)(it & 1));
    __syncthreads();
    BTRACE(4);

    // 4a. T~ = M^{-1}: diagonal, then the 2x2 block recursion on the upper
    //     triangle, B = 2 G (the strictly upper part of M); lower part stays 0
    for (int idx = tid; idx < E1; idx += NTH4) {
        const int r = idx / BS, c = idx - r * BS;
        Td[r * LDT + c] = (r == c && r < w) ? 1.f / Gr[r * BS + r] : 0.f;
        GnT[c * LDG + r] = Gr[E1 + idx];  // G[r][c] -> G^T[c][r]
        GpT[c * LDG + r] = Gr[2 * E1 + idx];
    }
    if (rank == 0 && tid < w) {  // degeneracy (householder.hpp:15, :28)
        const float gjj = Gr[tid * BS + tid];
        if (!(gjj > 1e-30f) || !isfinite(gjj)) {
            atomicOr(&err->flags, isfinite(gjj) ? kErrDegenerate : kErrNonFinite);
            const int kc = i * p.b + tid;
            atomicMin(&err->index, p.reversed ? p.n - 1 - kc : kc);
            err->chain = p.tag;
        }
    }
    __syncthreads();
    t_level<BS, 1>(Gr, Td, Ty, tid);
    t_level<BS, 2>(Gr, Td, Ty, tid);
    t_level<BS, 4>(Gr, Td, Ty, tid);
    t_level<BS, 8>(Gr, Td, Ty, tid);
    if constexpr (BS > 16) t_level<BS, 16>(Gr, Td, Ty, tid);
    if constexpr (BS > 32) t_level<BS, 32>(Gr, Td, Ty, tid);
    for (int idx = tid; idx < E1; idx += NTH4) {
        const int r = idx / BS, c = idx - r * BS;
        const float v = Td[r * LDT + c];  // 0 below the diagonal
        const float2 h = split2f(v);
        TfS[r * LD2 + c] = h;
        TTS[c * LD2 + r] = h;
        if (rank == 0) p.Tt[(size_t)i * E1 + idx] = v;
    }
    __syncthreads();
    BTRACE(5);

    // 4b. W rows and S into the stage images (fragment-order positions)
    // the S products are the same for every CTA of the cluster: rank 0 forms
    // Sf, rank 1 (rank 0 when C == 1) Sb, and stores it into every CTA's
    // stage slot
    const bool doSf = rank == 0, doSb = rank == (C > 1 ? 1 : 0);
    float* IWf = IPF;
    float* IVf = IPF + RB * LDW;
    float* ISf = IVf + RB * LDV;
    float* IWb = IPB;
    float* IVb = IPB + RB * LDW;
    float* ISb = IVb + RB * LDV;
    {
        // W^T = T~ V^T (Wf) and T~^T V^T (Wb): A = T~ / T~^T from the pre-split
        // planes, B[k][n] = V at row position n; unit = (product, m-tile,
        // group of NPU n-tiles) — 8 units at BS = 32, RB = 80
        constexpr int NPU = 5;
        const int ntl = RB / 8, ng = (ntl + NPU - 1) / NPU;
        // S units in n-tile halves: the ranks forming S give their extra
        // work to half their warps in two small pieces, not one large one
        constexpr int NTH = NT / 2;
        const int nW = 2 * MT * ng, nS = 2 * ((doSf ? MT : 0) + (doSb ? MT : 0));
        for (int u = warp; u < nW + nS; u += NTH4 / 32) {
            if (u < nW) {
                const bool fwd = u < MT * ng;
                const int uu = fwd ? u : u - MT * ng, mt = uu % MT, nt0 = (uu / MT) * NPU;
                const float2* Am = fwd ? TfS : TTS;
                float acc[NPU][3][4];
#pragma unroll
                for (int t = 0; t < NPU; ++t)
#pragma unroll
                    for (int b = 0; b < 3; ++b)
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[t][b][e] = 0.f;
#pragma unroll
                for (int ks = 0; ks < KB; ++ks) {
                    const float2* a = Am + (mt * 16 + g) * LD2 + ks * 8 + tq;
                    const float2 a0 = a[0], a1 = a[8 * LD2], a2 = a[4], a3 = a[8 * LD2 + 4];
                    AFrag af;
                    af.h[0] = __float_as_uint(a0.x), af.h[1] = __float_as_uint(a1.x);
                    af.h[2] = __float_as_uint(a2.x), af.h[3] = __float_as_uint(a3.x);
                    af.l[0] = __float_as_uint(a0.y), af.l[1] = __float_as_uint(a1.y);
                    af.l[2] = __float_as_uint(a2.y), af.l[3] = __float_as_uint(a3.y);
                    const float* bv = Vc + (size_t)(ks * 8 + tq) * P + g;
#pragma unroll
                    for (int t = 0; t < NPU; ++t) {
                        if (nt0 + t < ntl) {
                            const float b0 = bv[(nt0 + t) * 8], b1 = bv[4 * P + (nt0 + t) * 8];
                            mma3s(acc[t][0], acc[t][1], acc[t][2], af, __uint_as_float(hi_rn(b0)),
                                  __uint_as_float(hi_rn(b1)), lo_rn(b0), lo_rn(b1));
                        }
                    }
                }
                // C[c][n]: c = 16 mt + g (+8), n = 8 nt + 2 tq (+1) -> W[row(n)][c];
                // columns c, c + 8 sit side by side in fragment order
                float* img = fwd ? IWf : IWb;
#pragma unroll
                for (int t = 0; t < NPU; ++t) {
                    if (nt0 + t < ntl) {
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int r = b4_pos((nt0 + t) * 8 + 2 * tq + e);
                            *reinterpret_cast<float2*>(img + r * LDW + g * 2 * MT + mt * 2) =
                                make_float2(acc[t][0][e] + (acc[t][1][e] + acc[t][2][e]),
                                            acc[t][0][2 + e] + (acc[t][1][2 + e] + acc[t][2][2 + e]));
                        }
                    }
                }
            } else {
                // Sf = T~ G_{i,i+1} (A = T~, B[l][k] = GnT[k][l]);  Sb = T~^T G_{i,i-1} (A = T~^T)
                const int su = (u - nW) >> 1, nt0 = ((u - nW) & 1) * NTH;
                const bool fwd = doSf && su < MT;
                const int mt = su % MT;
                const float2* Am = fwd ? TfS : TTS;
                const float* Bm = fwd ? GnT : GpT;
                float acc[NTH][3][4];
#pragma unroll
                for (int nt = 0; nt < NTH; ++nt)
#pragma unroll
                    for (int b = 0; b < 3; ++b)
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[nt][b][e] = 0.f;
#pragma unroll
                for (int ks = 0; ks < KB; ++ks) {
                    const float2* a = Am + (mt * 16 + g) * LD2 + ks * 8 + tq;
                    const float2 a0 = a[0], a1 = a[8 * LD2], a2 = a[4], a3 = a[8 * LD2 + 4];
                    AFrag af;
                    af.h[0] = __float_as_uint(a0.x), af.h[1] = __float_as_uint(a1.x);
                    af.h[2] = __float_as_uint(a2.x), af.h[3] = __float_as_uint(a3.x);
                    af.l[0] = __float_as_uint(a0.y), af.l[1] = __float_as_uint(a1.y);
                    af.l[2] = __float_as_uint(a2.y), af.l[3] = __float_as_uint(a3.y);
#pragma unroll
                    for (int nn = 0; nn < NTH; ++nn) {
                        const int nt = nt0 + nn;
                        const float b0 = Bm[(nt * 8 + g) * LDG + ks * 8 + tq];
                        const float b1 = Bm[(nt * 8 + g) * LDG + ks * 8 + tq + 4];
                        mma3s(acc[nn][0], acc[nn][1], acc[nn][2], af, __uint_as_float(hi_rn(b0)),
                              __uint_as_float(hi_rn(b1)), lo_rn(b0), lo_rn(b1));
                    }
                }
                float* img = fwd ? ISf : ISb;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = mt * 16 + g + 8 * h;
#pragma unroll
                    for (int nn = 0; nn < NTH; ++nn)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            img[j * LDV + perm_v_bs((nt0 + nn) * 8 + 2 * tq + e, BS)] =
                                acc[nn][0][2 * h + e] + (acc[nn][1][2 * h + e] + acc[nn][2][2 * h + e]);
                }
            }
        }
        // V rows: fragment order for both stages, plain for the gradient kernel
        for (int r = warp; r < RB; r += NTH4 / 32) {
            const int pr = b4_pos(r);
            for (int c = lane; c < BS; c += 32) {
                const float v = Vc[(size_t)c * P + pr];
                const int pv = perm_v_bs(c, BS);
                IVf[r * LDV + pv] = v;
                IVb[r * LDV + pv] = v;
                IVB[r * LDV + c] = v;
            }
        }
    }
    dev::fence_proxy_async_smem();
    __syncthreads();
    BTRACE(6);

    // 5. bulk stores: Pf (forward step q-1-i), Pb (backward step i), Vbl
    if (tid == 0) {
        const size_t SF = stage_floats(RB, BS);
        float* pf = p.Pf + ((size_t)(p.q - 1 - i) * C + rank) * SF;
        float* pb = p.Pb + ((size_t)i * C + rank) * SF;
        float* vbl = p.Vbl + ((size_t)i * p.d_pad + row0) * LDV;
        const uint32_t wv = (uint32_t)(RB * (LDW + LDV) * 4), sb = (uint32_t)(BS * LDV * 4);
        bulk_s2g(pf, dev::smem_u32(IPF), wv);
        bulk_s2g(pb, dev::smem_u32(IPB), wv);
        bulk_s2g(vbl, dev::smem_u32(IVB), (uint32_t)(RB * LDV * 4));
        const int soff = RB * (LDW + LDV);
        for (int r = 0; r < C; ++r) {  // S into every CTA's slot of this block's stages
            if (doSf) bulk_s2g(p.Pf + ((size_t)(p.q - 1 - i) * C + r) * SF + soff, dev::smem_u32(ISf), sb);
            if (doSb) bulk_s2g(p.Pb + ((size_t)i * C + r) * SF + soff, dev::smem_u32(ISb), sb);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (p.ready) {
            // pipelined step: block i's rows are published once written
            // (the sweep bulk-loads the stages after acquiring the counter)
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            atomicAdd(p.ready + i, 1u);
        } else {
            // shared memory may be released once read; the writes complete with the grid
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        BTRACE(7);
        if (p.trace) p.trace[((size_t)i * C + rank) * 10 + 9] = (long long)dev::globaltimer();
    }
#undef BTRACE
    }  // blocks of this cluster
}

template <int BS>
cudaError_t launch_build4_t(const Plan& p, const float* V, int64_t ldv, ErrWord* err, cudaStream_t st) {
    const B4Layout L = b4_layout(BS, p.d_pad / p.CB, p.CB);
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(build4_kernel<BS>), L.total, true); e != cudaSuccess)
        return e;
    const int nclu = p.nbuild > 0 ? (p.nbuild < p.q ? p.nbuild : p.q) : (p.blk_hi < 0 ? p.q : p.blk_hi) - p.blk_lo;
    if (nclu <= 0) return cudaSuccess;
    // 16-byte row groups need 16-byte aligned columns
    const int vec_ok = ((reinterpret_cast<uintptr_t>(V) & 15) == 0) && (ldv % 4 == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nclu * p.CB, 1, 1);
    cfg.blockDim = dim3(NTH4, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.CB;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // streamed host step: a programmatic dependent of the upload kernel
    cfg.numAttrs = p.upc ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, build4_kernel<BS>, p, V, ldv, vec_ok, err);
}

}  // namespace

size_t build4_smem_bytes(int BS, int RB, int C) { return b4_layout(BS, RB, C).total; }

cudaError_t launch_build4(const Plan& p, const float* V, int64_t ldv, ErrWord* err, cudaStream_t s) {
    if (!p.Pf || !p.Pb || p.CB < 1 || p.CB > 16 || p.d_pad % p.CB || (p.d_pad / p.CB) % 16 ||
        (p.nbuild > 0 && (p.blk_lo != 0 || p.blk_hi >= 0)))
        return cudaErrorInvalidValue;
    switch (p.BS) {
        case 16: return launch_build4_t<16>(p, V, ldv, err, s);
        case 32: return launch_build4_t<32>(p, V, ldv, err, s);
        case 64: return launch_build4_t<64>(p, V, ldv, err, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
