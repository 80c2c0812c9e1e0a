// Backward step 2, v2: north_star subsystem (4), the per-reflection gradients
// of every block (fasth.hpp:97-108, Eq. (5) householder_grad,
// householder.hpp:148-179), as a closed-form blocked GEMM:
//
//   Q   = Z'f Z'b^T                       (BS x BS, K = m)
//   K'  = striu(Q - Q^T)
//   dV_block = -2 [A | G | V] [Z'b^T ; Z'f^T ; 2 K']     (d x BS, K = 2m + BS)
//
// re-laid out for the tensor cores' instruction budget:
//   * one CTA per (64-row slab, block), 4 warps x 16 rows, each warp all BS
//     output columns, so every A-operand element (tapes, V) is loaded once,
//     straight from L2 into registers in fragment order (the tape layout
//     [q][ngroups][d_pad][8] makes a k-step one 8-column group), split once
//     and used for BS/8 MMAs;
//   * the B operands ([Z'b^T ; Z'f^T] per 32-column chunk, then 2K' formed
//     from Q on the fly) are read from shared memory by the consumer and
//     split there (hi = rn_tf32, lo = x - hi);
//   * K runs over the real m (chunks of 32 batch columns), not a padded one.
#include "device_prims.cuh"
#include "fasth_internal.h"

namespace fasthb {
namespace {

constexpr int DV_ROWS = 64;  // rows per CTA
constexpr int DV_WARPS = 4;
constexpr int MCH = 32;      // batch columns per chunk (4 tape groups)

__device__ __forceinline__ uint32_t hi_rn(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }

__device__ __forceinline__ void hmma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

struct AF {
    uint32_t h[4], l[4];
};
__device__ __forceinline__ AF split4(const float (&v)[4]) {
    AF f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f.h[i] = hi_rn(v[i]);
        f.l[i] = __float_as_uint(v[i] - __uint_as_float(f.h[i]));
    }
    return f;
}

// B fragment (b0 = B[tq][g], b1 = B[tq+4][g]) split into hi / lo.
__device__ __forceinline__ void split2(float b0, float b1, uint32_t (&h)[2], uint32_t (&l)[2]) {
    h[0] = hi_rn(b0), h[1] = hi_rn(b1);
    l[0] = __float_as_uint(b0 - __uint_as_float(h[0]));
    l[1] = __float_as_uint(b1 - __uint_as_float(h[1]));
}

__device__ __forceinline__ void mma3(float (&m)[4], float (&c)[4], const AF& a, const uint32_t (&bh)[2],
                                     const uint32_t (&bl)[2]) {
    hmma(m, a.h[0], a.h[1], a.h[2], a.h[3], bh[0], bh[1]);
    hmma(c, a.h[0], a.h[1], a.h[2], a.h[3], bl[0], bl[1]);
    hmma(c, a.l[0], a.l[1], a.l[2], a.l[3], bh[0], bh[1]);
}

template <int BS>
__host__ __device__ constexpr size_t dv2_smem() {
    // Zb | Zf chunk (BS x (MCH+4) each; later the dV staging tile,
    // BS x (DV_ROWS+4) <= that), Q (BS x (BS+1)), the slab's V rows
    // (DV_ROWS x (BS+4), the builder's layout)
    static_assert(BS * (DV_ROWS + 4) <= 2 * BS * (MCH + 4), "dV staging fits the Z' chunks");
    return 4 * ((size_t)2 * BS * (MCH + 4) + (size_t)BS * (BS + 1) + (size_t)DV_ROWS * (BS + 4));
}

// Phases per CTA (one per 64-row slab of block i): every global load of a
// chunk is issued at once (tape and V fragments straight into registers,
// Z'b / Z'f chunk into shared memory), then Q = Z'f Z'b^T, then the main
// product with B fragments read and split by the consumer; dV written from
// the accumulators (8 consecutive rows per column per store instruction).
// TR: timeline stamps compiled in (FASTH_STEPTRACE runs only)
template <int BS, bool TR>
__global__ void __launch_bounds__(DV_WARPS * 32, 3) dv2_kernel(DvArgs a) {
    constexpr int NT = BS / 8, MT = BS / 16, KB = BS / 8;
    constexpr int LDZ = MCH + 4;
    constexpr int LDV = BS + 4;
    extern __shared__ __align__(16) float dsm[];
    float* Zb = dsm;
    float* Zf = dsm + BS * LDZ;
    float* Qs = dsm + 2 * BS * LDZ;
    float* Vs = Qs + BS * (BS + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    // blocks in the order the sweeps finish them (pipelined step: the CTAs
    // the scheduler places first are the ones whose inputs land first)
    int i = blockIdx.y;
    if (a.order == 1) {  // fused fwd+bwd: block i is final after step max(i, q-1-i)
        const int q = a.q, k = i, lo = (q - 1) / 2, hi = q / 2;
        if (q & 1) i = k == 0 ? lo : ((k & 1) ? lo - (k + 1) / 2 : lo + k / 2);
        else i = (k & 1) ? hi + k / 2 : lo - k / 2;
    }
    const int r0 = blockIdx.x * DV_ROWS + warp * 16;  // this warp's 16 rows
    const bool rows_ok = r0 < a.d_pad;
    const int m = a.m;
    const float* zf = a.zf + (size_t)i * BS * m;
    const float* zb = a.zb + (size_t)i * BS * m;
    const size_t tstep = (size_t)a.ngroups * a.d_pad * 8;
    const float* tA = a.tapeA + (size_t)i * tstep;
    const float* tG = a.tapeG + (size_t)i * tstep;
    long long* const trc = TR && a.trace && threadIdx.x == 0 ? a.trace + ((size_t)i * gridDim.x + blockIdx.x) * 6 : nullptr;
    if (trc) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trc[0] = (long long)dev::globaltimer(), trc[5] = smid;
    }
    // the slab's V rows of the block (K = BS; the builder's output, rows
    // < d_pad) into shared memory: before the wait on the sweep when the
    // builder is known complete (a.v_pre), else with the first Z' chunk
    auto stage_v = [&]() {
        const int rb = blockIdx.x * DV_ROWS, nr = min(DV_ROWS, a.d_pad - rb);
        const float* src = a.Vbl + ((size_t)i * a.d_pad + rb) * LDV;
        for (int idx = tid; idx < nr * LDV / 4; idx += DV_WARPS * 32)
            dev::cp_async16(Vs + 4 * idx, src + 4 * idx, true);
        dev::cp_async_commit();
    };
    if (a.trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (a.v_pre) stage_v();
    if (!a.done && a.pdl && !a.nowait) asm volatile("griddepcontrol.wait;" ::: "memory");  // sweep complete
    if (a.done) {  // pipelined step: both sweeps have passed block i
        if (tid == 0) {
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.done + i) : "memory");
                if (v >= a.done_target) break;
                __nanosleep(a.poll_ns);
            }
            // the last CTA of block i to get here resets the block's counters
            if (atomicAdd(a.dvcnt + i, 1u) == gridDim.x - 1) {
                a.ready[i] = 0u;
                a.done[i] = 0u;
                a.dvcnt[i] = 0u;
                if (a.upc) a.upc[i] = 0u;
            }
        }
        __syncthreads();
    }
    if (trc) trc[1] = (long long)dev::globaltimer();

    float acc[NT][4], cc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[nt][e] = cc[nt][e] = 0.f;
    // Q tiles of this warp: n-tiles warp, warp + 4, ...; all m-tiles
    constexpr int QN = (NT + DV_WARPS - 1) / DV_WARPS;
    float qm[QN][MT][4], qc[QN][MT][4];
#pragma unroll
    for (int u = 0; u < QN; ++u)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) qm[u][mt][e] = qc[u][mt][e] = 0.f;

    const bool vec = (m % 4) == 0;
    for (int l0 = 0; l0 < m; l0 += MCH) {
        const int mc = min(MCH, m - l0);
        // tape fragments of this chunk (k-step = one 8-column group; the tapes
        // hold zeros beyond m)
        float fa[MCH / 8][4], fg[MCH / 8][4];
#pragma unroll
        for (int ks = 0; ks < MCH / 8; ++ks) {
            const int grp = l0 / 8 + ks;
            const bool ok = rows_ok && grp < a.ngroups;
            const size_t o = ok ? ((size_t)grp * a.d_pad + r0 + g) * 8 + tq : 0;
            fa[ks][0] = tA[o], fa[ks][1] = tA[o + 64], fa[ks][2] = tA[o + 4], fa[ks][3] = tA[o + 68];
            fg[ks][0] = tG[o], fg[ks][1] = tG[o + 64], fg[ks][2] = tG[o + 4], fg[ks][3] = tG[o + 68];
            if (!ok) {
#pragma unroll
                for (int e = 0; e < 4; ++e) fa[ks][e] = fg[ks][e] = 0.f;
            }
        }
        if (l0 > 0) __syncthreads();  // previous chunk's Zb / Zf readers are done
        if (l0 == 0 && !a.v_pre) stage_v();
        if (vec && mc == MCH) {
            for (int idx = tid; idx < BS * MCH / 4; idx += DV_WARPS * 32) {
                const int j = idx / (MCH / 4), l4 = (idx - j * (MCH / 4)) * 4;
                dev::cp_async16(Zb + j * LDZ + l4, zb + (size_t)j * m + l0 + l4, true);
                dev::cp_async16(Zf + j * LDZ + l4, zf + (size_t)j * m + l0 + l4, true);
            }
        } else {
            for (int idx = tid; idx < BS * MCH; idx += DV_WARPS * 32) {
                const int j = idx / MCH, l = idx - j * MCH;
                const bool ok = l < mc;
                dev::cp_async4(Zb + j * LDZ + l, ok ? zb + (size_t)j * m + l0 + l : zb, ok);
                dev::cp_async4(Zf + j * LDZ + l, ok ? zf + (size_t)j * m + l0 + l : zf, ok);
            }
        }
        dev::cp_async_commit();
        dev::cp_async_wait_all();
        __syncthreads();
        if (trc && l0 == 0) trc[2] = (long long)dev::globaltimer();
        // Q += Z'f Z'b^T over the chunk (A = Z'f: rows j, K = l; B = Z'b^T)
#pragma unroll
        for (int u = 0; u < QN; ++u) {
            const int nt = warp + u * DV_WARPS;
            if (nt < NT) {
#pragma unroll
                for (int ks = 0; ks < MCH / 8; ++ks) {
                    uint32_t bh[2], bl[2];
                    const float* zbp = Zb + (nt * 8 + g) * LDZ + ks * 8 + tq;
                    split2(zbp[0], zbp[4], bh, bl);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const float* za = Zf + (mt * 16 + g) * LDZ + ks * 8 + tq;
                        const float av[4] = {za[0], za[8 * LDZ], za[4], za[8 * LDZ + 4]};
                        mma3(qm[u][mt], qc[u][mt], split4(av), bh, bl);
                    }
                }
            }
        }
        // [A | G] [Z'b^T ; Z'f^T] over the chunk; B fragments read and split here
        if (rows_ok) {
#pragma unroll
            for (int ks = 0; ks < MCH / 8; ++ks) {
                const AF fA = split4(fa[ks]), fG = split4(fg[ks]);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    uint32_t bh[2], bl[2];
                    const float* zbp = Zb + (nt * 8 + g) * LDZ + ks * 8 + tq;
                    split2(zbp[0], zbp[4], bh, bl);
                    mma3(acc[nt], cc[nt], fA, bh, bl);
                    const float* zfp = Zf + (nt * 8 + g) * LDZ + ks * 8 + tq;
                    split2(zfp[0], zfp[4], bh, bl);
                    mma3(acc[nt], cc[nt], fG, bh, bl);
                }
            }
        }
    }
    if (m <= 0) {  // no chunk loop ran
        if (!a.v_pre) stage_v();
        dev::cp_async_wait_all();
        __syncthreads();
    }
    float fv[KB][4];  // V fragments (the staged rows are visible: the chunk loop synced)
    {
        const float* vb = Vs + (warp * 16 + g) * LDV + tq;
#pragma unroll
        for (int ks = 0; ks < KB; ++ks) {
            fv[ks][0] = vb[ks * 8];
            fv[ks][1] = vb[8 * LDV + ks * 8];
            fv[ks][2] = vb[ks * 8 + 4];
            fv[ks][3] = vb[8 * LDV + ks * 8 + 4];
        }
    }
    // Q -> smem; the V term's B operand 2 K'[k][j] = 2 (Q[k][j] - Q[j][k]), k < j
#pragma unroll
    for (int u = 0; u < QN; ++u) {
        const int nt = warp + u * DV_WARPS;
        if (nt < NT) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = mt * 16 + g + 8 * (e >> 1), k = nt * 8 + 2 * tq + (e & 1);
                    Qs[j * (BS + 1) + k] = qm[u][mt][e] + qc[u][mt][e];
                }
        }
    }
    __syncthreads();
    if (trc) trc[3] = (long long)dev::globaltimer();
#pragma unroll
    for (int ks = 0; ks < KB && rows_ok; ++ks) {
        const AF fV = split4(fv[ks]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            if (ks > nt) continue;  // 2K' = 2 striu(Q - Q^T): zero unless k < j
            const int j = nt * 8 + g, k0 = ks * 8 + tq, k1 = k0 + 4;
            const float b0 = k0 < j ? 2.f * (Qs[k0 * (BS + 1) + j] - Qs[j * (BS + 1) + k0]) : 0.f;
            const float b1 = k1 < j ? 2.f * (Qs[k1 * (BS + 1) + j] - Qs[j * (BS + 1) + k1]) : 0.f;
            uint32_t bh[2], bl[2];
            split2(b0, b1, bh, bl);
            mma3(acc[nt], cc[nt], fV, bh, bl);
        }
    }
    // dV = -2 * result (chain order; the V^T leg un-reverses,
    // svd_layer.hpp:150-151), staged column-major in shared memory (over the
    // dead Z' chunks) so that each column's 64 rows leave as 16-byte stores:
    // full lines, which matters when dV is the caller's pinned host buffer
    constexpr int LDS_ = DV_ROWS + 4;
    float* stg = dsm;
    if (rows_ok) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                stg[(nt * 8 + 2 * tq + (e & 1)) * LDS_ + warp * 16 + g + 8 * (e >> 1)] = -2.f * (acc[nt][e] + cc[nt][e]);
    }
    __syncthreads();
    {
        const int rb0 = blockIdx.x * DV_ROWS;
        const int wb = min(a.b, a.n - i * a.b);
        const bool v4 = ((reinterpret_cast<uintptr_t>(a.dV) & 15) == 0) && (a.lddv % 4 == 0);
        for (int idx = tid; idx < BS * (DV_ROWS / 4); idx += DV_WARPS * 32) {
            const int j = idx / (DV_ROWS / 4), rr = (idx - j * (DV_ROWS / 4)) * 4, row = rb0 + rr;
            if (j >= wb || row >= a.d) continue;
            const int kc = i * a.b + j;
            const int col = a.reversed ? a.n - 1 - kc : kc;
            float* dst = a.dV + (int64_t)col * a.lddv + row;
            const float4 v = *reinterpret_cast<const float4*>(stg + j * LDS_ + rr);
            if (v4 && row + 4 <= a.d) {
                *reinterpret_cast<float4*>(dst) = v;
            } else {
                dst[0] = v.x;
                if (row + 1 < a.d) dst[1] = v.y;
                if (row + 2 < a.d) dst[2] = v.z;
                if (row + 3 < a.d) dst[3] = v.w;
            }
        }
    }
    if (trc) trc[4] = (long long)dev::globaltimer();
}

template <int BS>
cudaError_t launch_dv2_t(const DvArgs& a, cudaStream_t s) {
    auto kern = a.trace ? dv2_kernel<BS, true> : dv2_kernel<BS, false>;
    const dim3 grid((a.d_pad + DV_ROWS - 1) / DV_ROWS, a.q);
    size_t smem = dv2_smem<BS>();
    // pipelined behind the sweep: claim enough shared memory that no CTA
    // lands on an SM a sweep CTA occupies (co-resident gradient work slows
    // the latency-bound chain steps more than the overlap gains)
    if (a.done && a.min_smem > smem) smem = a.min_smem;
    if (smem > 48 * 1024)
        if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(DV_WARPS * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (a.done || a.pdl) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

cudaError_t launch_dv2(const DvArgs& a, cudaStream_t s) {
    if (a.WC != 8) return cudaErrorInvalidValue;
    switch (a.BS) {
        case 16: return launch_dv2_t<16>(a, s);
        case 32: return launch_dv2_t<32>(a, s);
        case 64: return launch_dv2_t<64>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
