// WY-block builder: north_star subsystem (2).
//
// Replaces the reference's b sequential prepends per block (wy_compact,
// wy.hpp:56-100, run per block under parallel_for, wy.hpp:151-170) by the
// UT form of the same product:
//
//     H_1 ... H_w = I - 2 V T~ V^T,   T~ = (diag(V^T V) + 2 striu(V^T V))^{-1}
//
// with V the block's RAW reflection vectors (no normalisation, so every
// fp32 reflection stays exactly a reflection).  One launch builds all q
// blocks: grid (RS row splits, q blocks).  Each CTA
//   1. stages its rows of the block's vectors through shared memory and
//      writes them coalesced into the blocked row-major Vbl layout the chain
//      kernels stream with bulk copies;
//   2. accumulates a partial Gram V^T V over its rows in f64 (fp32 inputs,
//      exact products);
//   3. the last CTA of each block (atomic ticket, no extra launch) reduces
//      the RS partials in fixed order (deterministic), checks ||v||^2 against
//      the reference's degeneracy threshold (householder.hpp:15, :28-30) and
//      solves the b x b upper-triangular T~ by back-substitution, one lane
//      per column, in f64.
#include "fasth_internal.h"

#include <cfloat>

namespace fasthb {
namespace {

__device__ __forceinline__ int src_col(int k, int n, int reversed) {
    return reversed ? n - 1 - k : k;
}

template <int BS>
__global__ void __launch_bounds__(kThreads) build_kernel(Plan p, const float* __restrict__ V,
                                                         int64_t ldv, ErrWord* err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int s = blockIdx.x;  // row split
    const int i = blockIdx.y;  // block
    const int tid = threadIdx.x;
    const int k0 = i * p.b;
    const int w = min(p.b, p.n - k0);
    const int row0 = s * p.rps;
    const int rows = min(p.rps, p.d_pad - row0);

    double* dv = reinterpret_cast<double*>(smem_raw);          // [rps][BS+1]
    float* sv = reinterpret_cast<float*>(dv + p.rps * (BS + 1)); // [rps][BS]
    double* Gs = reinterpret_cast<double*>(smem_raw);          // reused by finisher
    __shared__ int s_last;

    // 1. stage: coalesced along rows (V is column-major)
    for (int idx = tid; idx < rows * BS; idx += kThreads) {
        const int j = idx / rows, r = idx - j * rows;
        const int gr = row0 + r;
        float x = 0.f;
        if (j < w && gr < p.d) x = V[(int64_t)src_col(k0 + j, p.n, p.reversed) * ldv + gr];
        sv[r * BS + j] = x;
        dv[r * (BS + 1) + j] = (double)x;
    }
    __syncthreads();
    float* dst = p.Vbl + ((size_t)i * p.d_pad + row0) * BS;
    for (int idx = tid; idx < rows * BS; idx += kThreads) dst[idx] = sv[idx];

    // 2. partial Gram, upper triangle incl. diagonal, 2x2 register tiles
    constexpr int NT = BS / 2;
    double* gout = p.gram + ((size_t)i * p.RS + s) * BS * BS;
    for (int tile = tid; tile < NT * NT; tile += kThreads) {
        const int tj = tile / NT, tk = tile - tj * NT;
        if (tj > tk) continue;
        const int j = 2 * tj, k = 2 * tk;
        double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
        for (int r = 0; r < rows; ++r) {
            const double* row = dv + r * (BS + 1);
            const double x0 = row[j], x1 = row[j + 1], y0 = row[k], y1 = row[k + 1];
            a00 = fma(x0, y0, a00);
            a01 = fma(x0, y1, a01);
            a10 = fma(x1, y0, a10);
            a11 = fma(x1, y1, a11);
        }
        gout[j * BS + k] = a00;
        gout[j * BS + k + 1] = a01;
        gout[(j + 1) * BS + k] = a10;
        gout[(j + 1) * BS + k + 1] = a11;
    }

    // 3. last CTA of this block reduces and solves
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&p.counter[i], 1u) == (unsigned)(p.RS - 1));
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    double* Ts = Gs + BS * (BS + 1);  // [BS][BS+1]
    const double* gblk = p.gram + (size_t)i * p.RS * BS * BS;
    for (int idx = tid; idx < BS * BS; idx += kThreads) {
        const int j = idx / BS, k = idx - j * BS;
        double acc = 0.0;
        if (j <= k)
            for (int ss = 0; ss < p.RS; ++ss) acc += __ldcg(gblk + (size_t)ss * BS * BS + idx);
        Gs[j * (BS + 1) + k] = acc;
    }
    __syncthreads();
    if (tid < 32) {
        for (int c = tid; c < BS; c += 32) {
            for (int r = 0; r < BS; ++r) Ts[r * (BS + 1) + c] = 0.0;
            if (c >= w) continue;
            const double gcc = Gs[c * (BS + 1) + c];
            if (!(gcc > 1e-30) || !isfinite(gcc)) {
                atomicOr(&err->flags, isfinite(gcc) ? kErrDegenerate : kErrNonFinite);
                atomicMin(&err->index, src_col(k0 + c, p.n, p.reversed));
                err->chain = p.tag;
            }
            Ts[c * (BS + 1) + c] = 1.0 / gcc;
            for (int r = c - 1; r >= 0; --r) {
                double acc = 0.0;
                for (int k = r + 1; k <= c; ++k) acc = fma(Gs[r * (BS + 1) + k], Ts[k * (BS + 1) + c], acc);
                Ts[r * (BS + 1) + c] = -2.0 * acc / Gs[r * (BS + 1) + r];
            }
        }
    }
    __syncthreads();
    float* tout = p.Tt + (size_t)i * BS * BS;
    for (int idx = tid; idx < BS * BS; idx += kThreads) {
        const int r = idx / BS, c = idx - r * BS;
        tout[idx] = (float)Ts[r * (BS + 1) + c];
    }
    if (tid == 0) p.counter[i] = 0u;
}

template <int BS>
cudaError_t launch_build_t(const Plan& p, const float* V, int64_t ldv, ErrWord* err,
                           cudaStream_t st) {
    size_t smem = (size_t)p.rps * (BS + 1) * sizeof(double) + (size_t)p.rps * BS * sizeof(float);
    const size_t fin = 2 * (size_t)BS * (BS + 1) * sizeof(double);
    if (smem < fin) smem = fin;
    cudaError_t e = cudaFuncSetAttribute(build_kernel<BS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    build_kernel<BS><<<dim3(p.RS, p.q), kThreads, smem, st>>>(p, V, ldv, err);
    return cudaGetLastError();
}

}  // namespace

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
