// The reference's public WY internals on the device (wy.hpp:56-170):
// wy_compact / compact_chain materialise the compact WY form of a block of
// reflections exactly as the reference lays it out, and wy_apply /
// wy_apply_transpose apply one such block.  The chain sweeps never use these
// (they work on the UT form of raw vectors, fasth_internal.h); they exist so
// that a reference caller that reads TapeForward::compacted or calls the WY
// functions directly finds them (include/fasth_b200.h).
//
// Algebra: for a block's raw vectors V = [v_1 .. v_b],
//   H_1 ... H_b = I - 2 V T~ V^T,  T~ = (diag(V^T V) + 2 striu(V^T V))^{-1}
// (upper triangular), and with D = diag(||v_j||) the reference's pair is
//   Y = V D^{-1}  (the normalised vectors, wy.hpp:92-96)
//   W = V T~ D    (column j = H_1 ... H_{j-1} u_j, wy.hpp:85-90)
// since W Y^T = V T~ V^T and Y has full column rank (W is unique given Y).
// Gram, inverse and W are formed in f64 from the fp32 vectors.
#include <algorithm>

#include "fasth_internal.h"

namespace fasthb {
namespace {

// Gram band of block z: G[i][j] = v_i . v_j for j >= i (f64), the norms
// and the degeneracy check (householder.hpp:15, :28).  grid (ceil(b*b/256), q)
__global__ void wy_gram_kernel(const float* __restrict__ V, int64_t ldv, int d, int n, int bw,
                               double* __restrict__ Gm, ErrWord* err, int tag) {
    const int z = blockIdx.y, k0 = z * bw, w = min(bw, n - k0);
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= bw * bw) return;
    const int i = e / bw, j = e % bw;
    double* G = Gm + (size_t)z * bw * bw;
    if (i >= w || j >= w || j < i) {
        G[e] = 0.0;
        return;
    }
    const float* a = V + (int64_t)(k0 + i) * ldv;
    const float* b = V + (int64_t)(k0 + j) * ldv;
    double s = 0.0;
    for (int r = 0; r < d; ++r) s = fma((double)a[r], (double)b[r], s);
    G[e] = s;
    if (i == j && (!(s > 1e-30) || !isfinite(s))) {
        atomicOr(&err->flags, isfinite(s) ? kErrDegenerate : kErrNonFinite);
        atomicMin(&err->index, k0 + i);
        err->chain = tag;
    }
}

// T~ = M^{-1}, M = diag(G) + 2 striu(G) upper triangular: thread = column j,
// back substitution M t = e_j (t_i = 0 for i > j), in place over G's lower
// part is not possible (both triangles used), so T~ goes to its own buffer.
// grid (ceil(bw/128), q)
__global__ void wy_tinv_kernel(const double* __restrict__ Gm, int n, int bw, double* __restrict__ Tm) {
    const int z = blockIdx.y, w = min(bw, n - z * bw);
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= bw) return;
    const double* G = Gm + (size_t)z * bw * bw;
    double* T = Tm + (size_t)z * bw * bw;
    for (int i = bw - 1; i >= 0; --i) {
        double t = 0.0;
        if (j < w && i <= j) {
            double s = i == j ? 1.0 : 0.0;
            for (int k = i + 1; k <= j; ++k) s -= 2.0 * G[i * bw + k] * T[k * bw + j];
            const double g = G[i * bw + i];
            t = g > 0.0 ? s / g : 0.0;
        }
        T[i * bw + j] = t;
    }
}

// W[:, k0+j] = sum_{k <= j} v_k T~[k][j] ||v_j||,  Y[:, k0+j] = v_j / ||v_j||.
// grid (ceil(d/128), bw, q)
__global__ void wy_w_kernel(const float* __restrict__ V, int64_t ldv, int d, int n, int bw,
                            const double* __restrict__ Gm, const double* __restrict__ Tm,
                            float* __restrict__ W, int64_t ldw, float* __restrict__ Y, int64_t ldy) {
    const int z = blockIdx.z, j = blockIdx.y, k0 = z * bw, w = min(bw, n - k0);
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= w || r >= d) return;
    const double* G = Gm + (size_t)z * bw * bw;
    const double* T = Tm + (size_t)z * bw * bw;
    const double nj = sqrt(G[j * bw + j]);
    double s = 0.0;
    for (int k = 0; k <= j; ++k) s = fma((double)V[(int64_t)(k0 + k) * ldv + r], T[k * bw + j], s);
    W[(int64_t)(k0 + j) * ldw + r] = (float)(s * nj);
    Y[(int64_t)(k0 + j) * ldy + r] = (float)((double)V[(int64_t)(k0 + j) * ldv + r] / nj);
}

// T = B^T X (b x m): thread per (k, l), f64 sum over d in a fixed order.
// grid (ceil(b*m/256))
__global__ void wy_proj_kernel(const float* __restrict__ Bm, int64_t ldb, int d, int b, const float* __restrict__ X,
                               int64_t ldx, int m, double* __restrict__ T) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)b * m) return;
    const int k = (int)(e % b), l = (int)(e / b);
    const float* bk = Bm + (int64_t)k * ldb;
    const float* xl = X + (int64_t)l * ldx;
    double s = 0.0;
    for (int r = 0; r < d; ++r) s = fma((double)bk[r], (double)xl[r], s);
    T[e] = s;
}

// out = X - 2 A T (A d x b, T b x m): thread per (r, l).  grid (ceil(d/128), m)
__global__ void wy_update_kernel(const float* __restrict__ A, int64_t lda, int d, int b, const double* __restrict__ T,
                                 const float* __restrict__ X, int64_t ldx, float* __restrict__ out, int64_t ldo) {
    const int l = blockIdx.y, r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= d) return;
    const double* t = T + (int64_t)l * b;
    double s = 0.0;
    for (int k = 0; k < b; ++k) s = fma((double)A[(int64_t)k * lda + r], t[k], s);
    out[(int64_t)l * ldo + r] = (float)((double)X[(int64_t)l * ldx + r] - 2.0 * s);
}

}  // namespace

cudaError_t launch_wy_compact(const float* V, int64_t ldv, int d, int n, int bw, double* scratch, float* W,
                              int64_t ldw, float* Y, int64_t ldy, ErrWord* err, int tag, cudaStream_t s) {
    if (d < 1 || n < 1 || bw < 1) return cudaErrorInvalidValue;
    const int q = (n + bw - 1) / bw;
    double* Gm = scratch;
    double* Tm = scratch + (size_t)q * bw * bw;
    wy_gram_kernel<<<dim3((bw * bw + 255) / 256, q), 256, 0, s>>>(V, ldv, d, n, bw, Gm, err, tag);
    wy_tinv_kernel<<<dim3((bw + 127) / 128, q), 128, 0, s>>>(Gm, n, bw, Tm);
    wy_w_kernel<<<dim3((d + 127) / 128, bw, q), 128, 0, s>>>(V, ldv, d, n, bw, Gm, Tm, W, ldw, Y, ldy);
    return cudaGetLastError();
}

size_t wy_compact_scratch_doubles(int n, int bw) {
    const size_t q = (size_t)((n + bw - 1) / bw);
    return 2 * q * (size_t)bw * bw;
}

cudaError_t launch_wy_apply(const float* A, int64_t lda, const float* Bm, int64_t ldb, int d, int b,
                            const float* X, int64_t ldx, int m, double* T, float* out, int64_t ldo, cudaStream_t s) {
    if (d < 1 || b < 1 || m < 1) return cudaSuccess;
    wy_proj_kernel<<<(unsigned)(((int64_t)b * m + 255) / 256), 256, 0, s>>>(Bm, ldb, d, b, X, ldx, m, T);
    wy_update_kernel<<<dim3((d + 127) / 128, m), 128, 0, s>>>(A, lda, d, b, T, X, ldx, out, ldo);
    return cudaGetLastError();
}

}  // namespace fasthb
