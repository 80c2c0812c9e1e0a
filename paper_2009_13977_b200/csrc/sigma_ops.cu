// O(d) / O(dm) Sigma-side kernels of the SVD layer and the Sigma-ops:
// north_star subsystem (5).
//
//   scale_rows   T2 = f(Sigma) T1 with rectangular pad/truncate
//                (svd_layer.hpp:92-101, matops.hpp:78-83, :43-52) for chains
//                that have no factors (the sweeps fuse it into their load).
//   dsigma       dSigma_i = sum_l dT2[i,l] T1[i,l]      (svd_layer.hpp:131-137)
//   step         v <- v - eta dv with the degeneracy check of the rebuilt
//                HouseholderVector (svd_layer.hpp:165-181, householder.hpp:28)
//   sigma_step   sigma <- sigma - eta dsigma, optional clamp to [1-eps, 1+eps]
//                (svd_layer.hpp:190, :196-202)
//   sigma_map    f(sigma) for inverse / exp / Cayley (matops.hpp:71-83,
//                :102, :115-116) with the reference's singular / pole checks
//   logdet       sum ln|sigma_i| in f64 (matops.hpp:57-66)
#include "fasth_internal.h"

namespace fasthb {
namespace {

__global__ void scale_rows_kernel(const float* __restrict__ x, int64_t ldx, int n_valid,
                                  const float* __restrict__ scale, int rows, int m, float* y,
                                  int64_t ldy) {
    const int64_t total = (int64_t)rows * m;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(idx / rows), r = (int)(idx - (int64_t)l * rows);
        float v = 0.f;
        if (r < n_valid) v = x[(int64_t)l * ldx + r] * (scale ? scale[r] : 1.f);
        y[(int64_t)l * ldy + r] = v;
    }
}

__global__ void dsigma_kernel(const float* __restrict__ dT2, int64_t ld2,
                              const float* __restrict__ T1, int64_t ld1, int k, int m,
                              float* dsigma) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    // 32 columns' loads in flight per round trip (the loop is latency bound:
    // one round trip at batch 32); the batch sum stays in f64, in column order
    double acc = 0.0;
    int l = 0;
    for (; l + 32 <= m; l += 32) {
        float a[32], b[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            a[u] = __ldg(dT2 + (int64_t)(l + u) * ld2 + i);
            b[u] = __ldg(T1 + (int64_t)(l + u) * ld1 + i);
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) acc += (double)a[u] * b[u];
    }
    for (; l + 8 <= m; l += 8) {
        float a[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a[u] = __ldg(dT2 + (int64_t)(l + u) * ld2 + i);
            b[u] = __ldg(T1 + (int64_t)(l + u) * ld1 + i);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += (double)a[u] * b[u];
    }
    for (; l < m; ++l) acc += (double)dT2[(int64_t)l * ld2 + i] * T1[(int64_t)l * ld1 + i];
    dsigma[i] = (float)acc;
}

// Large batches: 32 rows per CTA, the batch split into DSW contiguous column
// ranges (one warp each, coalesced 128 B row segments per column), f64
// partials combined in warp order (deterministic).
constexpr int DSW = 32;
__global__ void __launch_bounds__(32 * DSW) dsigma_wide_kernel(const float* __restrict__ dT2, int64_t ld2,
                                                              const float* __restrict__ T1, int64_t ld1, int k,
                                                              int m, float* dsigma) {
    __shared__ double part[DSW][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = blockIdx.x * 32 + lane;
    const int per = (m + DSW - 1) / DSW;
    const int l0 = min(m, w * per), l1 = min(m, l0 + per);
    double acc = 0.0;
    if (i < k) {
        int l = l0;
        for (; l + 4 <= l1; l += 4) {
            float a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = __ldg(dT2 + (int64_t)(l + u) * ld2 + i);
                b[u] = __ldg(T1 + (int64_t)(l + u) * ld1 + i);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += (double)a[u] * b[u];
        }
        for (; l < l1; ++l) acc += (double)dT2[(int64_t)l * ld2 + i] * T1[(int64_t)l * ld1 + i];
    }
    part[w][lane] = acc;
    __syncthreads();
    if (w == 0 && i < k) {
        double t = 0.0;
        for (int u = 0; u < DSW; ++u) t += part[u][lane];
        dsigma[i] = (float)t;
    }
}

__global__ void step_kernel(const float* __restrict__ P, int64_t ldp, const float* __restrict__ dP,
                            int64_t lddp, int dim, float eta, float* out, int64_t ldo,
                            ErrWord* err, int tag) {
    const int k = blockIdx.x;
    __shared__ double red[32];
    double s = 0.0;
    bool finite = true;
    for (int r = threadIdx.x; r < dim; r += blockDim.x) {
        const float v = P[(int64_t)k * ldp + r] - eta * dP[(int64_t)k * lddp + r];
        out[(int64_t)k * ldo + r] = v;
        finite = finite && isfinite(v);
        s += (double)v * v;
    }
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const int any_bad = __syncthreads_or(!finite);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        if (any_bad || !(t > 1e-30)) {
            atomicOr(&err->flags, any_bad ? kErrNonFinite : kErrDegenerate);
            atomicMin(&err->index, k);
            err->chain = tag;
        }
    }
}

__global__ void sigma_step_kernel(const float* sigma, const float* dsigma, int k, float eta,
                                  float eps, float* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    float s = dsigma ? sigma[i] - eta * dsigma[i] : sigma[i];
    if (eps >= 0.f) s = fminf(fmaxf(s, 1.f - eps), 1.f + eps);
    out[i] = s;
}

__global__ void sigma_map_kernel(const float* sigma, int k, int kind, float tol, float* out, ErrWord* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const float s = sigma[i];
    float f = s;
    if (kind == 1) {  // inverse: 1/sigma (matops.hpp:65-67, :71)
        if (s == 0.f) atomicOr(&err->flags, kErrSingular);
        f = 1.f / s;
    } else if (kind == 2) {  // exponential
        f = expf(s);
    } else if (kind == 3) {  // Cayley (1 - s) / (1 + s), pole at -1
        if (s == -1.f) atomicOr(&err->flags, kErrPole);
        f = (1.f - s) / (1.f + s);
    } else if (kind == 4) {  // pseudo-inverse: 1/sigma where |sigma| > tol, else 0 (matops.hpp:166-167)
        f = fabsf(s) > tol ? 1.f / s : 0.f;
    }
    out[i] = f;
}

__global__ void logdet_kernel(const float* sigma, int k, double* out, ErrWord* err) {
    __shared__ double red[32];
    double s = 0.0;
    int zero = 0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const float v = sigma[i];
        zero |= (v == 0.f);
        s += log(fabs((double)v));
    }
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const int any_zero = __syncthreads_or(zero);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
        if (any_zero) atomicOr(&err->flags, kErrSingular);
    }
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

cudaError_t launch_scale_rows(const float* x, int64_t ldx, int n_valid, const float* scale,
                              int rows, int m, float* y, int64_t ldy, int mode, cudaStream_t s) {
    (void)mode;
    if ((int64_t)rows * m == 0) return cudaSuccess;
    scale_rows_kernel<<<grid_for((int64_t)rows * m), 256, 0, s>>>(x, ldx, n_valid, scale, rows,
                                                                    m, y, ldy);
    return cudaGetLastError();
}

// pdl_nowait: launched as a programmatic dependent of a kernel it does not
// depend on (its inputs were complete when that one started): starts early
cudaError_t launch_dsigma(const float* dT2, int64_t ld2, const float* T1, int64_t ld1, int k,
                          int m, float* dsigma, cudaStream_t s, bool pdl_nowait) {
    if (k == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_nowait ? 1 : 0;
    if (m >= 512) {  // one thread per row would leave most SMs idle for a long sequential sum
        cfg.gridDim = dim3((k + 31) / 32);
        cfg.blockDim = dim3(32 * DSW);
        return cudaLaunchKernelEx(&cfg, dsigma_wide_kernel, dT2, ld2, T1, ld1, k, m, dsigma);
    }
    cfg.gridDim = dim3((k + 127) / 128);
    cfg.blockDim = dim3(128);
    return cudaLaunchKernelEx(&cfg, dsigma_kernel, dT2, ld2, T1, ld1, k, m, dsigma);
}

cudaError_t launch_step(const float* P, int64_t ldp, const float* dP, int64_t lddp, int dim,
                        int n, float eta, float* out, int64_t ldo, ErrWord* err, int tag,
                        cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    step_kernel<<<n, 256, 0, s>>>(P, ldp, dP, lddp, dim, eta, out, ldo, err, tag);
    return cudaGetLastError();
}

cudaError_t launch_sigma_step(const float* sigma, const float* dsigma, int k, float eta,
                              float clamp_eps, float* out, cudaStream_t s) {
    if (k == 0) return cudaSuccess;
    sigma_step_kernel<<<(k + 255) / 256, 256, 0, s>>>(sigma, dsigma, k, eta, clamp_eps, out);
    return cudaGetLastError();
}

cudaError_t launch_sigma_map(const float* sigma, int k, int kind, float* out, ErrWord* err,
                             cudaStream_t s, float tol) {
    if (k == 0) return cudaSuccess;
    sigma_map_kernel<<<(k + 255) / 256, 256, 0, s>>>(sigma, k, kind, tol, out, err);
    return cudaGetLastError();
}

cudaError_t launch_logdet(const float* sigma, int k, double* out, ErrWord* err, cudaStream_t s) {
    logdet_kernel<<<1, 256, 0, s>>>(sigma, k, out, err);
    return cudaGetLastError();
}

}  // namespace fasthb
