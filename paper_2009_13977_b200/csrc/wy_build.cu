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
// block, the CTAs splitting the block's rows.  Each CTA
//   1. stages its rows of the block's vectors (coalesced column reads) and
//      writes them into the blocked row-major layout the chain kernels
//      stream with bulk copies (Vbl, row pitch BS + 4);
//   2. accumulates its rows' partial Gram V^T V in f64 (exact products);
//   3. cluster reduce-scatter/all-gather of the Gram over DSMEM (fixed order:
//      deterministic), degeneracy check against householder.hpp:15, :28;
//   4. inverts the b x b triangle (f64, recursive 2x2 blocking with 8x8
//      leaves) redundantly — cheaper than another round trip;
//   5. writes its rows of Wf = V T~^T and Wb = V T~ (the chain kernels'
//      partial-product operands, so T~ never sits on their critical path);
//   6. forms the look-ahead corrections of the pipelined chain,
//         Sf_i = Wf_i^T V_{i+1}   (forward step after block i+1)
//         Sb_i = Wb_i^T V_{i-1}   (backward step after block i-1)
//      as a second cluster reduction (chain_sweep.cu explains their use).
#include "device_prims.cuh"
#include "fasth_internal.h"

namespace fasthb {
namespace {

__device__ __forceinline__ int src_col(int k, int n, int reversed) {
    return reversed ? n - 1 - k : k;
}

__device__ __forceinline__ double ld_dsmem_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Sum `n` values of `part` over the CB CTAs of the cluster into `out` of every
// CTA (CTA r reduces the slice r*n/CB.. in fixed rank order, then pushes it).
template <typename T>
__device__ void cluster_allreduce(const T* part, T* out, int n, int CB, uint32_t rank) {
    dev::cluster_sync();
    const int per = (n + CB - 1) / CB;
    const int lo = (int)rank * per, hi = min(n, lo + per);
    const uint32_t pa = dev::smem_u32(part), oa = dev::smem_u32(out);
    for (int e = lo + (int)threadIdx.x; e < hi; e += kThreads) {
        T s = 0;
        for (int c = 0; c < CB; ++c) {
            const uint32_t ra = dev::mapa(pa + e * (uint32_t)sizeof(T), c);
            if constexpr (sizeof(T) == 8) s += ld_dsmem_f64(ra);
            else s += ld_dsmem_f32(ra);
        }
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
// per column), then T_AB = -T_AA M_AB T_BB level by level.  G, T, tmp have
// pitch BS + 1.
template <int BS>
__device__ void invert_upper(const double* G, double* T, double* tmp, int w) {
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
                const double inv = 1.0 / G[gr * LD + gr];
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

// Shared memory, with regions reused across phases:
//   RA: partial Gram Gp (phase 1) -> Gram with pitch LD, Gld (phase 2) ->
//       partial S, Sp (phase 3)
//   RB_: reduced Gram G (phase 1) -> inversion scratch tmp (phase 2) ->
//        reduced S, So (phase 3)
template <int BS>
struct BuildSmem {
    static constexpr int LD = BS + 1;
    static constexpr size_t kRegion = (size_t)BS * LD * 8;  // >= BS*BS*8 and 2*BS*BS*4
    size_t vs, ws, nb, vd, gp, g, gld, t, tmp, tf, tft, sp, so, total;
    __host__ __device__ explicit BuildSmem(int RB) {
        size_t o = 0;
        vd = o;  o += (size_t)RB * (BS + 2) * 8;  // f64 copy of the rows (Gram)
        gp = gld = sp = o;
        o += kRegion;
        g = tmp = so = o;
        o += kRegion;
        t = o;   o += kRegion;                // T~ (f64)
        tf = o;  o += (size_t)BS * BS * 4;
        tft = o; o += (size_t)BS * BS * 4;
        vs = o;  o += (size_t)RB * LD * 4;    // V_i rows
        ws = o;  o += (size_t)RB * LD * 4;    // W rows (Wf, then Wb)
        nb = o;  o += (size_t)RB * LD * 4;    // neighbour block rows
        total = o;
    }
};

// Stage rows [row0, row0+RB) of block `blk` (zero outside the chain) into
// dst[r][j] with cp.async: all loads of the CTA in flight at once (coalesced
// along rows of the column-major V).  Caller commits and waits.
template <int BS>
__device__ void load_rows_async(float* dst, const float* __restrict__ V, int64_t ldv, const Plan& p,
                                int blk, int row0, int RB) {
    constexpr int LD = BS + 1;
    const int k0 = blk * p.b;
    const int w = (blk >= 0 && blk < p.q) ? min(p.b, p.n - k0) : 0;
    for (int idx = threadIdx.x; idx < RB * BS; idx += kThreads) {
        const int j = idx / RB, r = idx - j * RB;
        const int gr = row0 + r;
        const bool ok = j < w && gr < p.d;
        const float* src = ok ? V + (int64_t)src_col(k0 + j, p.n, p.reversed) * ldv + gr : V;
        dev::cp_async4(dst + r * LD + j, src, ok);
    }
}

// S = W^T N over this CTA's rows (BS x BS, K = RB), into Sp.
template <int BS>
__device__ void partial_wtn(const float* W, const float* N, float* Sp, int RB) {
    constexpr int LD = BS + 1;
    for (int idx = threadIdx.x; idx < BS * BS; idx += kThreads) {
        const int j = idx / BS, k = idx - j * BS;
        float s0 = 0.f, s1 = 0.f;
        int r = 0;
        for (; r + 1 < RB; r += 2) {
            s0 = fmaf(W[r * LD + j], N[r * LD + k], s0);
            s1 = fmaf(W[(r + 1) * LD + j], N[(r + 1) * LD + k], s1);
        }
        if (r < RB) s0 = fmaf(W[r * LD + j], N[r * LD + k], s0);
        Sp[idx] = s0 + s1;
    }
}

// W rows = V rows * M  (M = T~^T for Wf, T~ for Wb; row-major BS x BS).
template <int BS>
__device__ void w_rows(const float* Vs, const float* M, float* Ws, int RB) {
    constexpr int LD = BS + 1;
    for (int idx = threadIdx.x; idx < RB * BS; idx += kThreads) {
        const int r = idx / BS, j = idx - r * BS;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
        for (int k = 0; k < BS; k += 2) {
            s0 = fmaf(Vs[r * LD + k], M[k * BS + j], s0);
            s1 = fmaf(Vs[r * LD + k + 1], M[(k + 1) * BS + j], s1);
        }
        Ws[r * LD + j] = s0 + s1;
    }
}

template <int BS>
__device__ void store_rows(float* dst, const float* src, int row0, int RB, int d_pad) {
    constexpr int LD = BS + 1, LDB = BS + 4;
    for (int idx = threadIdx.x; idx < RB * LDB; idx += kThreads) {
        const int r = idx / LDB, j = idx - r * LDB;
        if (row0 + r < d_pad) dst[(size_t)(row0 + r) * LDB + j] = j < BS ? src[r * LD + j] : 0.f;
    }
}

template <int BS>
__global__ void __launch_bounds__(kThreads, 1) build_kernel(Plan p, const float* __restrict__ V,
                                                             int64_t ldv, ErrWord* err) {
    constexpr int LD = BS + 1;
    extern __shared__ __align__(16) unsigned char smem[];
    const int CB = p.CB;
    const int RB = p.d_pad / CB;
    const BuildSmem<BS> L(RB);
    double* Gp = reinterpret_cast<double*>(smem + L.gp);
    double* G = reinterpret_cast<double*>(smem + L.g);
    double* Gld = reinterpret_cast<double*>(smem + L.gld);
    double* T = reinterpret_cast<double*>(smem + L.t);
    double* tmp = reinterpret_cast<double*>(smem + L.tmp);
    float* Sp = reinterpret_cast<float*>(smem + L.sp);
    float* So = reinterpret_cast<float*>(smem + L.so);
    float* Tf = reinterpret_cast<float*>(smem + L.tf);
    float* TfT = reinterpret_cast<float*>(smem + L.tft);
    float* Vs = reinterpret_cast<float*>(smem + L.vs);
    float* Ws = reinterpret_cast<float*>(smem + L.ws);
    float* Nb = reinterpret_cast<float*>(smem + L.nb);

    const int tid = threadIdx.x;
    const uint32_t rank = dev::cluster_ctarank();
    const int i = (int)dev::cluster_id_x();
    const int row0 = (int)rank * RB;
    const int w = min(p.b, p.n - i * p.b);
    const size_t boff = (size_t)i * p.d_pad * (BS + 4);

    // 1. this block's rows, and the next block's (for Sf), all in flight
    load_rows_async<BS>(Vs, V, ldv, p, i, row0, RB);
    load_rows_async<BS>(Nb, V, ldv, p, i + 1, row0, RB);
    dev::cp_async_commit();
    dev::cp_async_wait_all();
    __syncthreads();
    store_rows<BS>(p.Vbl + boff, Vs, row0, RB, p.d_pad);
    // 2. partial Gram (upper incl. diagonal), f64: convert the rows once, then
    //    2x2 register tiles (exact fp32 products, f64 accumulation)
    constexpr int LDD = BS + 2;
    double* Vd = reinterpret_cast<double*>(smem + L.vd);
    for (int idx = tid; idx < RB * BS; idx += kThreads) {
        const int r = idx / BS, j = idx - r * BS;
        Vd[r * LDD + j] = (double)Vs[r * LD + j];
    }
    __syncthreads();
    constexpr int NT2 = BS / 2;
    for (int tile = tid; tile < NT2 * NT2; tile += kThreads) {
        const int tj = tile / NT2, tk = tile - tj * NT2;
        double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
        if (tj <= tk) {
#pragma unroll 4
            for (int r = 0; r < RB; ++r) {
                const double2 x = *reinterpret_cast<const double2*>(Vd + r * LDD + 2 * tj);
                const double2 y = *reinterpret_cast<const double2*>(Vd + r * LDD + 2 * tk);
                a00 = fma(x.x, y.x, a00);
                a01 = fma(x.x, y.y, a01);
                a10 = fma(x.y, y.x, a10);
                a11 = fma(x.y, y.y, a11);
            }
        }
        const int j = 2 * tj, k = 2 * tk;
        Gp[j * BS + k] = a00;
        Gp[j * BS + k + 1] = a01;
        Gp[(j + 1) * BS + k] = a10;
        Gp[(j + 1) * BS + k + 1] = a11;
    }
    // 3. cluster all-reduce of the Gram
    cluster_allreduce<double>(Gp, G, BS * BS, CB, rank);
    if (rank == 0 && tid < w) {
        const double g = G[tid * BS + tid];
        if (!(g > 1e-30) || !isfinite(g)) {
            atomicOr(&err->flags, isfinite(g) ? kErrDegenerate : kErrNonFinite);
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
    invert_upper<BS>(Gld, T, tmp, w);
    for (int idx = tid; idx < BS * BS; idx += kThreads) {
        const int r = idx / BS, c = idx - r * BS;
        const float v = (float)T[r * LD + c];
        Tf[idx] = v;          // T~[r][c]
        TfT[c * BS + r] = v;  // T~^T
    }
    __syncthreads();
    if (rank == 0)
        for (int idx = tid; idx < BS * BS; idx += kThreads) p.Tt[(size_t)i * BS * BS + idx] = Tf[idx];
    // 5/6. Wf = V T~^T ; Sf_i = Wf^T V_{i+1}
    w_rows<BS>(Vs, TfT, Ws, RB);
    __syncthreads();
    store_rows<BS>(p.Wf + boff, Ws, row0, RB, p.d_pad);
    partial_wtn<BS>(Ws, Nb, Sp, RB);
    __syncthreads();
    // Wb = V T~ ; Sb_i = Wb^T V_{i-1}  (previous block's rows load meanwhile)
    load_rows_async<BS>(Nb, V, ldv, p, i - 1, row0, RB);
    dev::cp_async_commit();
    w_rows<BS>(Vs, Tf, Ws, RB);
    dev::cp_async_wait_all();
    __syncthreads();
    store_rows<BS>(p.Wb + boff, Ws, row0, RB, p.d_pad);
    partial_wtn<BS>(Ws, Nb, Sp + BS * BS, RB);
    cluster_allreduce<float>(Sp, So, 2 * BS * BS, CB, rank);
    if (rank == 0)  // row pitch BS + 4: conflict-free row reads in the sweeps
        for (int idx = tid; idx < BS * (BS + 4); idx += kThreads) {
            const int j = idx / (BS + 4), k = idx - j * (BS + 4);
            const bool in = k < BS;
            p.Sf[(size_t)i * BS * (BS + 4) + idx] = in ? So[j * BS + k] : 0.f;
            p.Sb[(size_t)i * BS * (BS + 4) + idx] = in ? So[BS * BS + j * BS + k] : 0.f;
        }
}

template <int BS>
cudaError_t launch_build_t(const Plan& p, const float* V, int64_t ldv, ErrWord* err,
                           cudaStream_t st) {
    const BuildSmem<BS> L(p.d_pad / p.CB);
    static size_t configured = 0;
    if (L.total > configured) {
        cudaError_t e = cudaFuncSetAttribute(build_kernel<BS>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(build_kernel<BS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        configured = L.total;
    }
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
        case 8: return BuildSmem<8>(RB).total;
        case 16: return BuildSmem<16>(RB).total;
        case 32: return BuildSmem<32>(RB).total;
        default: return BuildSmem<64>(RB).total;
    }
}

cudaError_t launch_build(const Plan& p, const float* V, int64_t ldv, ErrWord* err,
                         cudaStream_t s) {
    switch (p.BS) {
        case 8: return launch_build_t<8>(p, V, ldv, err, s);
        case 16: return launch_build_t<16>(p, V, ldv, err, s);
        case 32: return launch_build_t<32>(p, V, ldv, err, s);
        case 64: return launch_build_t<64>(p, V, ldv, err, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fasthb
