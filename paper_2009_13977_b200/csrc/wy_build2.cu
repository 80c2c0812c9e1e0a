// WY-block builder, v2: north_star subsystem (2) for the packed-stage chain
// (chain_v2.cu): the UT form of the
// reference's compact WY (wy_compact, wy.hpp:56-100),
//     H_1 ... H_w = I - 2 V T~ V^T,   T~ = (diag(V^T V) + 2 striu(V^T V))^{-1}
// with raw vectors — restructured around ONE cluster reduction:
//   1. each CTA of block i's cluster loads its RB rows of blocks i-1, i, i+1
//      (column-major in shared memory: conflict-free fragments both ways);
//   2. partial Gram band over its rows: G_ii on the FP64 tensor cores (exact
//      products, f64 sums; upper triangle), G_{i,i+1} and G_{i,i-1} by 3xTF32
//      mma.sync;
//   3. one DSMEM reduce-scatter / all-gather of the band (fixed order:
//      deterministic, identical in every CTA);
//   4. every CTA: degeneracy check (householder.hpp:15, :28), T~ in f64,
//      the look-ahead corrections Sf_i = T~ G_{i,i+1}, Sb_i = T~^T G_{i,i-1}
//      (= Wf_i^T V_{i+1}, Wb_i^T V_{i-1}; chain_v2.cu) without another pass
//      over d;
//   5. its rows of Wf = V T~^T and Wb = V T~ (3xTF32, B operand pre-split),
//      written with V and S straight into the packed stages (Pf, Pb) and the
//      dv kernel's Vbl.
#include <cooperative_groups.h>

#include "device_prims.cuh"
#include "fasth_internal.h"

namespace cg = cooperative_groups;

namespace fasthb {
namespace {

constexpr int NTH = 256;

__device__ __forceinline__ uint32_t hi_rn(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }

__device__ __forceinline__ void hmma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
struct AF {
    uint32_t h[4], l[4];
};
__device__ __forceinline__ AF split4(float a0, float a1, float a2, float a3) {
    AF f;
    const float v[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f.h[i] = hi_rn(v[i]);
        f.l[i] = __float_as_uint(v[i] - __uint_as_float(f.h[i]));
    }
    return f;
}
// RB + 4 (RB a multiple of 16): (RB+4)/4 odd, so the (g rows x tq cols)
// fragment gathers of the Gram products are bank-conflict free
__host__ __device__ inline int vt_pitch(int RB) { return RB + 4; }

template <int BS>
struct B2Smem {
    size_t vt, gp, gr, t, bn, ws, total;  // bytes
    __host__ __device__ explicit B2Smem(int RB) {
        const int P = vt_pitch(RB);
        size_t o = 0;
        vt = o;   o += (size_t)3 * BS * P * 4;                 // V^T rows of blocks i, i-1, i+1
        gp = o;   o += (size_t)BS * BS * 8 + 2 * BS * BS * 4;  // partial band: G_ii f64 | G_off f32
        gr = o;   o += (size_t)BS * BS * 8 + 2 * BS * BS * 4;  // reduced band
        t = bn = o;  // rinv (BS) + M2 (BS x BS), fp32
        o += (size_t)(BS + BS * BS) * 4;
        total = o;
        // [Wf | Sf^T] and [Wb | Sb^T] rows (pitch BS+4) alias blocks i-1, i+1
        // and the partial band, all dead by then — when they fit there: the
        // reduced band and rinv / M2 are read while the rows are written, so
        // otherwise (tall slabs, small BS) the rows get their own region
        ws = vt + (size_t)BS * P * 4;
        const size_t need = (size_t)2 * (RB + BS) * (BS + 4) * 4;
        if (ws + need > gr) {
            ws = (total + 15) / 16 * 16;
            total = ws + need;
        }
    }
};

template <int BS>
__global__ void __launch_bounds__(NTH, 2) build2_kernel(Plan p, const float* __restrict__ V, int64_t ldv,
                                                         ErrWord* err) {
    constexpr int NT = BS / 8, MT = BS / 16, KB = BS / 8;
    constexpr int LDS_ = BS + 4;  // W|S^T staging pitch
    constexpr int LDW = stage_ldw(BS), LDV = stage_ldv(BS);
    extern __shared__ __align__(16) unsigned char smem[];
    const int CB = p.CB, RB = p.d_pad / CB, P = vt_pitch(RB);
    const B2Smem<BS> L(RB);
    float* Vt = reinterpret_cast<float*>(smem + L.vt);  // [slot][j][P]
    double* Gp = reinterpret_cast<double*>(smem + L.gp);
    float* Gpo = reinterpret_cast<float*>(smem + L.gp + (size_t)BS * BS * 8);
    double* Gr = reinterpret_cast<double*>(smem + L.gr);
    float* Gro = reinterpret_cast<float*>(smem + L.gr + (size_t)BS * BS * 8);
    float* Wsm = reinterpret_cast<float*>(smem + L.ws);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const uint32_t rank = dev::cluster_ctarank();
    const int row0 = (int)rank * RB;
    // the chain sweep may launch now (programmatic dependent launch): it waits
    // on the per-block readiness counters, not on this grid's completion
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // persistent over blocks when pipelined: ticket k -> the k-th block the
    // two sweeps need (forward from q-1 down, backward from 0 up, interleaved)
    const int nclu = (int)(gridDim.x / CB);
    const int ntkt = p.nbuild > 0 ? p.q : (p.blk_hi < 0 ? p.q : p.blk_hi) - p.blk_lo;
    for (int tkt = (int)dev::cluster_id_x(); tkt < ntkt; tkt += nclu) {
    const int i = p.nbuild > 0 ? ((tkt & 1) ? (tkt >> 1) : p.q - 1 - (tkt >> 1)) : p.blk_lo + tkt;
    const int w = min(p.b, p.n - i * p.b);
    // FASTH_TRACE phase stamps: [block][CTA rank][8] clock64 (0 start, 1 loaded,
    // 2 Gram band done, 3 reduced, 4 T~, 5 B operands, 6 W rows, 7 end)
#define BTRACE(k) \
    if (p.trace && tid == 0) p.trace[((size_t)i * CB + rank) * 10 + (k)] = clock64()
    BTRACE(0);
    if (p.trace && tid == 0) p.trace[((size_t)i * CB + rank) * 10 + 8] = (long long)dev::globaltimer();

    // 1. V rows of blocks i, i-1, i+1 -> Vt[slot][j][r] (zero outside the chain / d);
    //    16-byte copies where the column is 16-byte aligned
    const bool vec = ((reinterpret_cast<uintptr_t>(V) & 15) == 0) && (ldv % 4 == 0);
    for (int jj = warp; jj < 3 * BS; jj += NTH / 32) {
        const int sl = jj / BS, j = jj % BS;
        const int blk = sl == 0 ? i : sl == 1 ? i - 1 : i + 1;
        const int k0 = blk * p.b;
        const int wb = (blk >= 0 && blk < p.q) ? min(p.b, p.n - k0) : 0;
        float* dst = Vt + (size_t)jj * P;
        const bool colok = j < wb;
        const float* src = colok ? V + (int64_t)(p.reversed ? p.n - 1 - (k0 + j) : k0 + j) * ldv + row0 : V;
        if (vec) {
            for (int r = lane * 4; r < RB; r += 128) {
                if (colok && row0 + r + 3 < p.d) {
                    dev::cp_async16(dst + r, src + r, true);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool ok = colok && row0 + r + e < p.d;
                        dev::cp_async4(dst + r + e, ok ? src + r + e : V, ok);
                    }
                }
            }
        } else {
            for (int r = lane; r < RB; r += 32) {
                const bool ok = colok && row0 + r < p.d;
                dev::cp_async4(dst + r, ok ? src + r : V, ok);
            }
        }
    }
    dev::cp_async_commit();
    dev::cp_async_wait_all();
    __syncthreads();
    BTRACE(1);
    const float* Vc = Vt;                   // block i
    const float* Vp = Vt + (size_t)BS * P;  // block i-1
    const float* Vn = Vt + (size_t)2 * BS * P;

    // 2a. G_ii partial, f64 tensor cores: upper 8x8 tiles, two chains each
    {
        constexpr int TT = (BS / 8) * (BS / 8 + 1) / 2;
        for (int u = warp; u < TT; u += NTH / 32) {
            int mi = 0, rem = u;
            while (rem >= BS / 8 - mi) rem -= BS / 8 - mi, ++mi;
            const int ni = mi + rem;
            double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
            const float* va = Vc + (size_t)(mi * 8 + g) * P + tq;
            const float* vb = Vc + (size_t)(ni * 8 + g) * P + tq;
            int k0 = 0;
            for (; k0 + 8 <= RB; k0 += 8) {
                dmma(d0, d1, (double)va[k0], (double)vb[k0]);
                dmma(e0, e1, (double)va[k0 + 4], (double)vb[k0 + 4]);
            }
            for (; k0 < RB; k0 += 4) dmma(d0, d1, (double)va[k0], (double)vb[k0]);
            Gp[(mi * 8 + g) * BS + ni * 8 + 2 * tq] = d0 + e0;
            Gp[(mi * 8 + g) * BS + ni * 8 + 2 * tq + 1] = d1 + e1;
        }
        for (int idx = tid; idx < BS * BS; idx += NTH) {  // lower tiles: zero
            const int r = idx / BS, c = idx - r * BS;
            if ((r >> 3) > (c >> 3)) Gp[idx] = 0.0;
        }
    }
    // 2b. G_{i,i+1}, G_{i,i-1} partials (3xTF32): warp = (side, m-tile, n-tile pair)
    for (int u = warp; u < 2 * MT * (NT / 2); u += NTH / 32) {
        const int side = u / (MT * (NT / 2)), rem = u % (MT * (NT / 2));
        const int mt = rem / (NT / 2), np = rem % (NT / 2);
        const float* Vb = side == 0 ? Vn : Vp;
        float m[2][4], c[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < 4; ++e) m[h][e] = c[h][e] = 0.f;
        for (int k0 = 0; k0 < RB; k0 += 8) {
            const float* a = Vc + (size_t)(mt * 16 + g) * P + k0 + tq;
            const AF af = split4(a[0], a[8 * P], a[4], a[8 * P + 4]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float* bp = Vb + (size_t)((2 * np + h) * 8 + g) * P + k0 + tq;
                const float b0 = bp[0], b1 = bp[4];
                const uint32_t bh0 = hi_rn(b0), bh1 = hi_rn(b1);
                hmma(m[h], af.h[0], af.h[1], af.h[2], af.h[3], bh0, bh1);
                hmma(c[h], af.h[0], af.h[1], af.h[2], af.h[3], __float_as_uint(b0 - __uint_as_float(bh0)),
                     __float_as_uint(b1 - __uint_as_float(bh1)));
                hmma(c[h], af.l[0], af.l[1], af.l[2], af.l[3], bh0, bh1);
            }
        }
        float* go = Gpo + side * BS * BS;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                go[(mt * 16 + g + 8 * (e >> 1)) * BS + (2 * np + h) * 8 + 2 * tq + (e & 1)] = m[h][e] + c[h][e];
    }
    BTRACE(2);

    // 3. reduce-scatter + all-gather of the band over the cluster (fixed order)
    dev::cluster_sync();
    {
        cg::cluster_group cl = cg::this_cluster();
        constexpr int N64 = BS * BS, N32 = 2 * BS * BS;
        const int per64 = (N64 + CB - 1) / CB, per32 = (N32 + CB - 1) / CB;
        const int lo64 = (int)rank * per64, hi64 = min(N64, lo64 + per64);
        const int lo32 = (int)rank * per32, hi32 = min(N32, lo32 + per32);
        for (int e = lo64 + tid; e < hi64; e += NTH) {
            double v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = c < CB ? cl.map_shared_rank(Gp, c)[e] : 0.0;
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < 16; ++c) s += v[c];
            for (int c = 0; c < CB; ++c) cl.map_shared_rank(Gr, c)[e] = s;
        }
        for (int e = lo32 + tid; e < hi32; e += NTH) {
            float v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = c < CB ? cl.map_shared_rank(Gpo, c)[e] : 0.f;
            float s = 0.f;
#pragma unroll
            for (int c = 0; c < 16; ++c) s += v[c];
            for (int c = 0; c < CB; ++c) cl.map_shared_rank(Gro, c)[e] = s;
        }
    }
    dev::cluster_sync();
    BTRACE(3);

    // 4. degeneracy (rank 0 reports); rinv[k] = 1 / G_kk and M2[r][k] = 2 G_rk
    //    (M = diag(G) + 2 striu(G)), rounded to fp32, in their own region (the
    //    staging rows of step 5 alias the partial band)
    float* rinv = reinterpret_cast<float*>(smem + L.t);
    float* M2 = rinv + BS;
    for (int idx = tid; idx < BS * BS; idx += NTH) M2[idx] = (float)(2.0 * Gr[idx]);
    if (tid < BS) {
        const double gjj = Gr[tid * BS + tid];
        rinv[tid] = tid < w ? (float)(1.0 / gjj) : 0.f;
        if (rank == 0 && tid < w && (!(gjj > 1e-30) || !isfinite(gjj))) {
            atomicOr(&err->flags, isfinite(gjj) ? kErrDegenerate : kErrNonFinite);
            const int kc = i * p.b + tid;
            atomicMin(&err->index, p.reversed ? p.n - 1 - kc : kc);
            err->chain = p.tag;
        }
    }
    __syncthreads();
    BTRACE(4);

    // 5. one row per thread, triangular solves in f64 (T~ = M^{-1} never formed):
    //      Wf = V T~^T  <=>  w M^T = v   (back substitution)
    //      Wb = V T~    <=>  w M   = v   (forward substitution)
    //    on the rows of V, of G_{i,i+1}^T (-> Sf^T = G_{i,i+1}^T T~^T, i.e.
    //    Sf = T~ G_{i,i+1} = Wf^T V_{i+1}) and of G_{i,i-1}^T (-> Sb^T), plus
    //    (rank 0) the unit rows for T~^T (diagnostics).  Right-looking: once
    //    w_j is known, its column updates the remaining right-hand sides, all
    //    independent FMAs.  fp32 arithmetic on the f64-reduced Gram (B200's
    //    FP64 vector rate made an f64 solve ~9 us per block).
    BTRACE(5);
    {
        const int ntask = 2 * (RB + BS) + (rank == 0 ? BS : 0);
        for (int task = tid; task < ntask; task += NTH) {
            // tasks: [0, RB+BS) forward chain rows (V then G_{i,i+1}^T), then
            // [RB+BS, 2(RB+BS)) backward rows (V then G_{i,i-1}^T), then T~^T rows
            const bool fwd = task < RB + BS || task >= 2 * (RB + BS);
            const int row = task < RB + BS ? task : (task < 2 * (RB + BS) ? task - (RB + BS) : task - 2 * (RB + BS));
            const bool trow = task >= 2 * (RB + BS);
            float acc[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                float v;
                if (trow) v = (c == row) ? 1.f : 0.f;
                else if (row < RB) v = Vc[(size_t)c * P + row];
                else v = Gro[(fwd ? 0 : BS * BS) + c * BS + (row - RB)];  // G_off^T row = G_off column
                acc[c] = v;
            }
            // results straight out: the staging row, or (T~^T rows) column `row` of T~
            float* wr = trow ? p.Tt + (size_t)i * BS * BS + row
                             : Wsm + (size_t)(fwd ? 0 : 1) * (RB + BS) * LDS_ + (size_t)row * LDS_;
            const int ws = trow ? BS : 1;
            if (fwd) {
#pragma unroll
                for (int j = BS - 1; j >= 0; --j) {
                    const float wj = j < w ? acc[j] * rinv[j] : 0.f;
                    wr[j * ws] = wj;
#pragma unroll
                    for (int r = 0; r < j; ++r) acc[r] = fmaf(-M2[r * BS + j], wj, acc[r]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < BS; ++j) {
                    const float wj = j < w ? acc[j] * rinv[j] : 0.f;
                    wr[j * ws] = wj;
#pragma unroll
                    for (int r = j + 1; r < BS; ++r) acc[r] = fmaf(-M2[j * BS + r], wj, acc[r]);
                }
            }
        }
    }
    __syncthreads();
    BTRACE(6);

    // 6. stores, float4 at a time with gathered (inverse-permuted) reads:
    //    packed stages W | V | S (Pf: forward step q-1-i, Pb: backward step i), Vbl
    const size_t SF = stage_floats(RB, BS);
    float* pf = p.Pf + ((size_t)(p.q - 1 - i) * CB + rank) * SF;
    float* pb = p.Pb + ((size_t)i * CB + rank) * SF;
    float* vbl = p.Vbl + ((size_t)i * p.d_pad + row0) * LDV;
    const float* Wf_ = Wsm;
    const float* Wb_ = Wsm + (size_t)(RB + BS) * LDS_;
    for (int idx = tid; idx < RB * (BS / 4); idx += NTH) {
        const int r = idx / (BS / 4), p0 = (idx - r * (BS / 4)) * 4;
        float wf[4], wb[4], vv[4], vr[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int pw = p0 + e;  // W position -> column c = 16 mt + 8 h + g
            const int cw = ((pw % (2 * MT)) >> 1) * 16 + (pw & 1) * 8 + pw / (2 * MT);
            wf[e] = Wf_[r * LDS_ + cw];
            wb[e] = Wb_[r * LDS_ + cw];
            const int pv = p0 + e;  // V position -> column c = 8 ks + 4 h + tq
            const int cv = ((pv % (2 * KB)) >> 1) * 8 + (pv & 1) * 4 + pv / (2 * KB);
            vv[e] = Vc[(size_t)cv * P + r];
            vr[e] = Vc[(size_t)(p0 + e) * P + r];
        }
        *reinterpret_cast<float4*>(pf + r * LDW + p0) = make_float4(wf[0], wf[1], wf[2], wf[3]);
        *reinterpret_cast<float4*>(pb + r * LDW + p0) = make_float4(wb[0], wb[1], wb[2], wb[3]);
        *reinterpret_cast<float4*>(pf + RB * LDW + r * LDV + p0) = make_float4(vv[0], vv[1], vv[2], vv[3]);
        *reinterpret_cast<float4*>(pb + RB * LDW + r * LDV + p0) = make_float4(vv[0], vv[1], vv[2], vv[3]);
        *reinterpret_cast<float4*>(vbl + r * LDV + p0) = make_float4(vr[0], vr[1], vr[2], vr[3]);
    }
    // S rows: S[j][pos(k)] = S^T[k][j] (staged as rows RB.. of each product)
    const int soff = RB * (LDW + LDV);
    for (int idx = tid; idx < BS * (BS / 4); idx += NTH) {
        const int j = idx / (BS / 4), p0 = (idx - j * (BS / 4)) * 4;
        float sf[4], sb[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int pv = p0 + e;
            const int k = ((pv % (2 * KB)) >> 1) * 8 + (pv & 1) * 4 + pv / (2 * KB);
            sf[e] = Wf_[(RB + k) * LDS_ + j];
            sb[e] = Wb_[(RB + k) * LDS_ + j];
        }
        *reinterpret_cast<float4*>(pf + soff + j * LDV + p0) = make_float4(sf[0], sf[1], sf[2], sf[3]);
        *reinterpret_cast<float4*>(pb + soff + j * LDV + p0) = make_float4(sb[0], sb[1], sb[2], sb[3]);
    }
    // publish block i (all of this CTA's stores ordered before the counter)
    __syncthreads();
    if (p.ready && tid == 0) {
        __threadfence();
        atomicAdd(&p.ready[i], 1u);
    }
    BTRACE(7);
    if (p.trace && tid == 0) p.trace[((size_t)i * CB + rank) * 10 + 9] = (long long)dev::globaltimer();
#undef BTRACE
    }
}

template <int BS>
cudaError_t launch_build2_t(const Plan& p, const float* V, int64_t ldv, ErrWord* err, cudaStream_t st) {
    const B2Smem<BS> L(p.d_pad / p.CB);
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(build2_kernel<BS>), L.total, true); e != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    const int nrange = (p.blk_hi < 0 ? p.q : p.blk_hi) - p.blk_lo;
    const int nclu = p.nbuild > 0 ? (p.nbuild < p.q ? p.nbuild : p.q) : nrange;
    if (nclu <= 0) return cudaSuccess;
    cfg.gridDim = dim3(nclu * p.CB, 1, 1);
    cfg.blockDim = dim3(NTH, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.CB;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, build2_kernel<BS>, p, V, ldv, err);
}

}  // namespace

size_t build2_smem_bytes(int BS, int RB) {
    switch (BS) {
        case 16: return B2Smem<16>(RB).total;
        case 32: return B2Smem<32>(RB).total;
        default: return B2Smem<64>(RB).total;
    }
}

cudaError_t launch_build2(const Plan& p, const float* V, int64_t ldv, ErrWord* err, cudaStream_t s) {
    if (!p.Pf || !p.Pb || p.CB < 1 || p.CB > 16 || p.d_pad % p.CB || (p.d_pad / p.CB) % 16)
        return cudaErrorInvalidValue;
    switch (p.BS) {
        case 16: return launch_build2_t<16>(p, V, ldv, err, s);
        case 32: return launch_build2_t<32>(p, V, ldv, err, s);
        case 64: return launch_build2_t<64>(p, V, ldv, err, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
