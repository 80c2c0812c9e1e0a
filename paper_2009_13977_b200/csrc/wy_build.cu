// WY-block builder: north_star subsystem (2).
//
// Replaces the reference's b sequential prepends per block (wy_compact,
// wy.hpp:56-100, run per block under parallel_for, wy.hpp:151-170) by the
// UT form of the same product:
//
//     H_1 ... H_w = I - 2 V T~ V^T,   T~ = (diag(V^T V) + 2 striu(V^T V))^{-1}
//
// with V the block's RAW reflection vectors (no normalisation, so every
// fp32 reflection stays exactly a reflection).
//
// ONE launch builds all q blocks: one thread-block cluster of CB CTAs per
// block (CB = the chain kernel's cluster size, so every CTA owns RB rows, a
// multiple of 16).  Each CTA
//   1. stages its rows of the block's vectors with cp.async and writes them
//      in the blocked row-major layout the chain kernels stream (Vbl);
//   2. accumulates its rows' partial Gram V^T V on the FP64 tensor cores
//      (mma.sync m8n8k4 f64: exact fp32 products, f64 sums);
//   3. cluster all-reduce of the Gram over DSMEM (fixed order:
//      deterministic), degeneracy check against householder.hpp:15, :28;
//   4. inverts the b x b triangle (f64, recursive 2x2 blocking with 8x8
//      leaves) redundantly — cheaper than another round trip;
//   5. writes its rows of Wf = V T~^T and Wb = V T~ (3xTF32 mma.sync), the
//      chain kernels' partial-product operands;
//   6. forms the look-ahead corrections of the pipelined chain,
//         Sf_i = Wf_i^T V_{i+1}   (forward step after block i+1)
//         Sb_i = Wb_i^T V_{i-1}   (backward step after block i-1)
//      (3xTF32 mma.sync, second cluster reduction; chain_sweep.cu).
#include "device_prims.cuh"
#include "fasth_internal.h"
#include "mma_tf32.cuh"

namespace fasthb {
namespace {

__device__ __forceinline__ int src_col(int k, int n, int reversed) {
    return reversed ? n - 1 - k : k;
}

__device__ __forceinline__ double ld_dsmem_f64(uint32_t addr) {
    double v;
    asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void st_dsmem_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
    float v;
    asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Sum `n` values of `part` over the CB CTAs of the cluster into `out` of every
// CTA: CTA r reduces the slice r*n/CB.. in fixed rank order (all its remote
// loads in flight together), then pushes it to every CTA.
template <typename T>
__device__ void cluster_allreduce(const T* part, T* out, int n, int CB, uint32_t rank) {
    dev::cluster_sync();
    const int per = (n + CB - 1) / CB;
    const int lo = (int)rank * per, hi = min(n, lo + per);
    const uint32_t pa = dev::smem_u32(part), oa = dev::smem_u32(out);
    for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
        T v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            v[c] = 0;
            if (c < CB) {
                const uint32_t ra = dev::mapa(pa + e * (uint32_t)sizeof(T), c);
                if constexpr (sizeof(T) == 8) v[c] = ld_dsmem_f64(ra);
                else v[c] = ld_dsmem_f32(ra);
            }
        }
        T s = 0;
#pragma unroll
        for (int c = 0; c < 16; ++c) s += v[c];
        for (int c = 0; c < CB; ++c) {
            const uint32_t ra = dev::mapa(oa + e * (uint32_t)sizeof(T), c);
            if constexpr (sizeof(T) == 8) st_dsmem_f64(ra, s);
            else st_dsmem_f32(ra, s);
        }
    }
    dev::cluster_sync();
}

// T~ = M^{-1}, M = diag(g) + 2 striu(G) (upper triangular), in f64, by
// recursive 2x2 blocking: leaves of 8 solved by back-substitution (one lane
// per column), then T_AB = -T_AA (2 G_AB) T_BB level by level.  G, T, tmp
// have pitch BS + 1; rinv[r] = 1 / g_rr.
template <int BS>
__device__ void invert_upper(const double* G, const double* rinv, double* T, double* tmp, int w) {
    constexpr int LD = BS + 1;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < BS * LD; idx += kThreads) T[idx] = 0.0;
    __syncthreads();
    constexpr int NLEAF = BS / 8;
    for (int leaf = warp; leaf < NLEAF; leaf += kThreads / 32) {
        const int c = leaf * 8 + lane;
        if (lane < 8 && c < w) {
            double col[8];
#pragma unroll
            for (int r = 7; r >= 0; --r) {
                const int gr = leaf * 8 + r;
                double acc = 0.0;
#pragma unroll
                for (int k = r + 1; k < 8; ++k)
                    if (k <= lane) acc = fma(G[gr * LD + leaf * 8 + k], col[k], acc);
                const double inv = rinv[gr];
                col[r] = (r == lane) ? inv : (r < lane ? -2.0 * acc * inv : 0.0);
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) T[(leaf * 8 + r) * LD + c] = col[r];
        }
    }
    __syncthreads();
    for (int sz = 8; sz < BS; sz *= 2) {
        const int npair = BS / (2 * sz);
        for (int idx = tid; idx < npair * sz * sz; idx += kThreads) {  // tmp = 2 G_AB T_BB
            const int pr = idx / (sz * sz), e = idx - pr * sz * sz;
            const int r = e / sz, c = e - r * sz;
            const int a0 = pr * 2 * sz, b0 = a0 + sz;
            double acc = 0.0;
            for (int k = 0; k <= c; ++k) acc = fma(G[(a0 + r) * LD + b0 + k], T[(b0 + k) * LD + b0 + c], acc);
            tmp[(a0 + r) * LD + c] = 2.0 * acc;
        }
        __syncthreads();
        for (int idx = tid; idx < npair * sz * sz; idx += kThreads) {  // T_AB = -T_AA tmp
            const int pr = idx / (sz * sz), e = idx - pr * sz * sz;
            const int r = e / sz, c = e - r * sz;
            const int a0 = pr * 2 * sz, b0 = a0 + sz;
            double acc = 0.0;
            for (int k = r; k < sz; ++k) acc = fma(T[(a0 + r) * LD + a0 + k], tmp[(a0 + k) * LD + c], acc);
            T[(a0 + r) * LD + b0 + c] = -acc;
        }
        __syncthreads();
    }
}

// Shared memory.  Regions reused across phases:
//   ra: partial Gram Gp (f64) -> Gram with pitch LD, Gld -> partial S, Sp
//   rb: reduced Gram G (f64) -> inversion scratch tmp -> reduced S, So
template <int BS>
struct BuildSmem {
    static constexpr int LD = BS + 1;   // f64 inversion pitch
    static constexpr int LDV = BS + 4;  // V rows (== Vbl pitch)
    static constexpr int LDN = BS + 8;  // W / neighbour rows (== Wf/Wb pitch), T~ (f32)
    static constexpr size_t kRegion = (size_t)BS * LD * 8;
    size_t ra, rb, t, rinv, tf, vs, ws, nb, total;
    __host__ __device__ explicit BuildSmem(int RB) {
        size_t o = 0;
        ra = o;   o += kRegion;
        rb = o;   o += kRegion;
        t = o;    o += kRegion;
        rinv = o; o += (size_t)BS * 8;
        tf = o;   o += (size_t)BS * LDN * 4;
        vs = o;   o += (size_t)RB * LDV * 4;
        ws = o;   o += (size_t)RB * LDN * 4;
        nb = o;   o += (size_t)RB * LDN * 4;
        total = o;
    }
};

// rows [row0, row0+RB) of block `blk` (zero outside the chain) -> dst[r][j],
// pitch LDP, with cp.async (all loads in flight); caller commits and waits.
template <int BS, int LDP>
__device__ void load_rows_async(float* dst, const float* __restrict__ V, int64_t ldv, const Plan& p,
                                int blk, int row0, int RB) {
    const int k0 = blk * p.b;
    const int w = (blk >= 0 && blk < p.q) ? min(p.b, p.n - k0) : 0;
    for (int idx = threadIdx.x; idx < RB * BS; idx += kThreads) {
        const int j = idx / RB, r = idx - j * RB;
        const int gr = row0 + r;
        const bool ok = j < w && gr < p.d;
        const float* src = ok ? V + (int64_t)src_col(k0 + j, p.n, p.reversed) * ldv + gr : V;
        dev::cp_async4(dst + r * LDP + j, src, ok);
    }
}

// rows (pitch LDP in smem and in global) -> global, float4 at a time
template <int LDP>
__device__ void store_rows(float* dst, const float* src, int RB) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int idx = threadIdx.x; idx < RB * LDP / 4; idx += kThreads) d4[idx] = s4[idx];
}

// W[RB x BS] = Vs[RB x BS] * B, B[k][j] = Tf[k][j] (tr = 0: W = V T~) or
// Tf[j][k] (tr = 1: W = V T~^T); 3xTF32 tensor cores, 16x8 tiles per warp.
template <int BS>
__device__ void w_rows_mma(const float* Vs, const float* Tf, float* Ws, int RB, int tr) {
    constexpr int LDV = BS + 4, LDN = BS + 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    const int ntiles = (RB / 16) * (BS / 8);
    for (int u = warp; u < ntiles; u += kThreads / 32) {
        const int r0 = (u / (BS / 8)) * 16, n0 = (u % (BS / 8)) * 8;
        dev::Frag4 m = {{0.f, 0.f, 0.f, 0.f}}, c = m;
#pragma unroll
        for (int k0 = 0; k0 < BS; k0 += 8) {
            const float* v0 = Vs + (r0 + g) * LDV + k0 + tq;
            const float av[4] = {v0[0], v0[8 * LDV], v0[4], v0[8 * LDV + 4]};
            float bv[2];
            if (tr) {
                bv[0] = Tf[(n0 + g) * LDN + k0 + tq];
                bv[1] = Tf[(n0 + g) * LDN + k0 + tq + 4];
            } else {
                bv[0] = Tf[(k0 + tq) * LDN + n0 + g];
                bv[1] = Tf[(k0 + tq + 4) * LDN + n0 + g];
            }
            dev::mma3(m, c, av, bv);
        }
        float* w0 = Ws + (r0 + g) * LDN + n0 + 2 * tq;
        w0[0] = m.v[0] + c.v[0];
        w0[1] = m.v[1] + c.v[1];
        w0[8 * LDN] = m.v[2] + c.v[2];
        w0[8 * LDN + 1] = m.v[3] + c.v[3];
    }
}

// Sp[BS x BS] = Ws^T Nb over this CTA's RB rows; 3xTF32 tensor cores.
template <int BS>
__device__ void wtn_mma(const float* Ws, const float* Nb, float* Sp, int RB) {
    constexpr int LDN = BS + 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    constexpr int ntiles = (BS / 16) * (BS / 8);
    for (int u = warp; u < ntiles; u += kThreads / 32) {
        const int m0 = (u / (BS / 8)) * 16, n0 = (u % (BS / 8)) * 8;
        dev::Frag4 m = {{0.f, 0.f, 0.f, 0.f}}, c = m;
        for (int k0 = 0; k0 < RB; k0 += 8) {
            const float* w0 = Ws + (k0 + tq) * LDN + m0 + g;
            const float av[4] = {w0[0], w0[8], w0[4 * LDN], w0[4 * LDN + 8]};
            const float bv[2] = {Nb[(k0 + tq) * LDN + n0 + g], Nb[(k0 + tq + 4) * LDN + n0 + g]};
            dev::mma3(m, c, av, bv);
        }
        float* s0 = Sp + (m0 + g) * BS + n0 + 2 * tq;
        s0[0] = m.v[0] + c.v[0];
        s0[1] = m.v[1] + c.v[1];
        s0[8 * BS] = m.v[2] + c.v[2];
        s0[8 * BS + 1] = m.v[3] + c.v[3];
    }
}

// This CTA's rows of W (pitch LDN) and V (pitch LDV) -> its packed chain
// stage (fasth_internal.h): columns permuted into mma fragment order.
template <int BS>
__device__ void store_packed_wv(float* dst, const float* Ws, const float* Vs, int RB) {
    constexpr int LDN = BS + 8, LDVs = BS + 4;
    constexpr int LDW = stage_ldw(BS), LDV = stage_ldv(BS);
    for (int idx = threadIdx.x; idx < RB * BS; idx += kThreads) {
        const int r = idx / BS, c = idx - r * BS;
        dst[r * LDW + perm_w_bs(c, BS)] = Ws[r * LDN + c];
        dst[RB * LDW + r * LDV + perm_v_bs(c, BS)] = Vs[r * LDVs + c];
    }
}

template <int BS>
__global__ void __launch_bounds__(kThreads, 1) build_kernel(Plan p, const float* __restrict__ V,
                                                             int64_t ldv, ErrWord* err) {
    using L_ = BuildSmem<BS>;
    constexpr int LD = L_::LD, LDV = L_::LDV, LDN = L_::LDN;
    extern __shared__ __align__(16) unsigned char smem[];
    const int CB = p.CB;
    const int RB = p.d_pad / CB;
    const L_ L(RB);
    double* Gp = reinterpret_cast<double*>(smem + L.ra);
    double* Gld = Gp;
    float* Sp = reinterpret_cast<float*>(smem + L.ra);
    double* G = reinterpret_cast<double*>(smem + L.rb);
    double* tmp = G;
    float* So = reinterpret_cast<float*>(smem + L.rb);
    double* T = reinterpret_cast<double*>(smem + L.t);
    double* rinv = reinterpret_cast<double*>(smem + L.rinv);
    float* Tf = reinterpret_cast<float*>(smem + L.tf);
    float* Vs = reinterpret_cast<float*>(smem + L.vs);
    float* Ws = reinterpret_cast<float*>(smem + L.ws);
    float* Nb = reinterpret_cast<float*>(smem + L.nb);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const uint32_t rank = dev::cluster_ctarank();
    const int i = (int)dev::cluster_id_x();
    const int row0 = (int)rank * RB;
    const int w = min(p.b, p.n - i * p.b);
    const size_t voff = ((size_t)i * p.d_pad + row0) * LDV;
    const size_t woff = ((size_t)i * p.d_pad + row0) * LDN;

    // 1. this block's rows, and the next block's (for Sf), all in flight
    load_rows_async<BS, LDV>(Vs, V, ldv, p, i, row0, RB);
    load_rows_async<BS, LDN>(Nb, V, ldv, p, i + 1, row0, RB);
    dev::cp_async_commit();
    dev::cp_async_wait_all();
    __syncthreads();
    store_rows<LDV>(p.Vbl + voff, Vs, RB);
    // 2. partial Gram on the FP64 tensor cores (8x8 tiles, upper triangle)
    for (int u = warp; u < (BS / 8) * (BS / 8); u += kThreads / 32) {
        const int mi = u / (BS / 8), ni = u % (BS / 8);
        double d0 = 0.0, d1 = 0.0;
        if (mi <= ni) {
            const float* va = Vs + tq * LDV + mi * 8 + g;
            const float* vb = Vs + tq * LDV + ni * 8 + g;
#pragma unroll 4
            for (int k0 = 0; k0 < RB; k0 += 4)
                dev::dmma(d0, d1, (double)va[k0 * LDV], (double)vb[k0 * LDV]);
        }
        Gp[(mi * 8 + g) * BS + ni * 8 + 2 * tq] = d0;
        Gp[(mi * 8 + g) * BS + ni * 8 + 2 * tq + 1] = d1;
    }
    // 3. cluster all-reduce of the Gram
    cluster_allreduce<double>(Gp, G, BS * BS, CB, rank);
    if (tid < BS) {
        const double gd = G[tid * BS + tid];
        rinv[tid] = tid < w ? 1.0 / gd : 0.0;
        if (rank == 0 && tid < w && (!(gd > 1e-30) || !isfinite(gd))) {
            atomicOr(&err->flags, isfinite(gd) ? kErrDegenerate : kErrNonFinite);
            atomicMin(&err->index, src_col(i * p.b + tid, p.n, p.reversed));
            err->chain = p.tag;
        }
    }
    // 4. T~ in f64
    for (int idx = tid; idx < BS * LD; idx += kThreads) {
        const int j = idx / LD, k = idx - j * LD;
        Gld[idx] = (j < w && k < w) ? G[j * BS + k] : 0.0;
    }
    __syncthreads();
    invert_upper<BS>(Gld, rinv, T, tmp, w);
    for (int idx = tid; idx < BS * BS; idx += kThreads) {
        const int r = idx / BS, c = idx - r * BS;
        Tf[r * LDN + c] = (float)T[r * LD + c];
    }
    __syncthreads();
    if (rank == 0)
        for (int idx = tid; idx < BS * BS; idx += kThreads)
            p.Tt[(size_t)i * BS * BS + idx] = Tf[(idx / BS) * LDN + idx % BS];
    // 5/6. Wf = V T~^T ; Sf_i = Wf^T V_{i+1}
    w_rows_mma<BS>(Vs, Tf, Ws, RB, 1);
    __syncthreads();
    if (p.Wf) store_rows<LDN>(p.Wf + woff, Ws, RB);
    const size_t SF = stage_floats(RB, BS);
    float* pf = p.Pf ? p.Pf + ((size_t)(p.q - 1 - i) * CB + rank) * SF : nullptr;
    float* pb = p.Pb ? p.Pb + ((size_t)i * CB + rank) * SF : nullptr;
    if (pf) store_packed_wv<BS>(pf, Ws, Vs, RB);
    wtn_mma<BS>(Ws, Nb, Sp, RB);
    __syncthreads();
    // Wb = V T~ ; Sb_i = Wb^T V_{i-1}  (previous block's rows load meanwhile)
    load_rows_async<BS, LDN>(Nb, V, ldv, p, i - 1, row0, RB);
    dev::cp_async_commit();
    w_rows_mma<BS>(Vs, Tf, Ws, RB, 0);
    dev::cp_async_wait_all();
    __syncthreads();
    if (p.Wb) store_rows<LDN>(p.Wb + woff, Ws, RB);
    if (pb) store_packed_wv<BS>(pb, Ws, Vs, RB);
    wtn_mma<BS>(Ws, Nb, Sp + BS * BS, RB);
    cluster_allreduce<float>(Sp, So, 2 * BS * BS, CB, rank);
    if (pf) {  // every CTA's stage carries the block's look-ahead correction
        const int soff = RB * (stage_ldw(BS) + LDV);
        for (int idx = tid; idx < BS * BS; idx += kThreads) {
            const int j = idx / BS, k = idx - j * BS;
            pf[soff + j * LDV + perm_v_bs(k, BS)] = So[idx];
            pb[soff + j * LDV + perm_v_bs(k, BS)] = So[BS * BS + idx];
        }
    }
    if (rank == 0 && p.Sf)  // row pitch BS + 4 (the chain kernel's S pitch)
        for (int idx = tid; idx < BS * LDV; idx += kThreads) {
            const int j = idx / LDV, k = idx - j * LDV;
            const bool in = k < BS;
            p.Sf[(size_t)i * BS * LDV + idx] = in ? So[j * BS + k] : 0.f;
            p.Sb[(size_t)i * BS * LDV + idx] = in ? So[BS * BS + j * BS + k] : 0.f;
        }
}

template <int BS>
cudaError_t launch_build_t(const Plan& p, const float* V, int64_t ldv, ErrWord* err,
                           cudaStream_t st) {
    const BuildSmem<BS> L(p.d_pad / p.CB);
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(build_kernel<BS>), L.total, true); e != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.q * p.CB, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.CB;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, build_kernel<BS>, p, V, ldv, err);
}

}  // namespace

size_t build_smem_bytes(int BS, int RB) {
    switch (BS) {
        case 16: return BuildSmem<16>(RB).total;
        case 32: return BuildSmem<32>(RB).total;
        default: return BuildSmem<64>(RB).total;
    }
}

cudaError_t launch_build(const Plan& p, const float* V, int64_t ldv, ErrWord* err,
                         cudaStream_t s) {
    if (p.CB < 1 || p.CB > 16 || p.d_pad % p.CB || (p.d_pad / p.CB) % 16) return cudaErrorInvalidValue;
    switch (p.BS) {
        case 16: return launch_build_t<16>(p, V, ldv, err, s);
        case 32: return launch_build_t<32>(p, V, ldv, err, s);
        case 64: return launch_build_t<64>(p, V, ldv, err, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
