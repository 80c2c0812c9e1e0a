// Large-batch path, elementwise kernels and the GEMM test hook (see lb.h).
#include <algorithm>
#include <cstdio>

#include "lb.h"

namespace fasthb {
namespace lb {
namespace {

__device__ __forceinline__ float rn_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
// (x, x - trunc(x)) when `trunc`: hi stays x (the tensor core truncates it)
__device__ __forceinline__ float split_hi(float x, bool trunc) {
    return trunc ? x : rn_hi(x);
}
__device__ __forceinline__ float split_lo(float x, bool trunc) {
    return trunc ? x - __uint_as_float(__float_as_uint(x) & 0xffffe000u) : x - rn_hi(x);
}

__global__ void split_kernel(const float* __restrict__ x, int64_t ldx, int rows, int cols, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t ldo, bool trunc) {
    const int64_t total = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols), c = (int)(i % cols);
        const float v = x[r * ldx + c];
        hi[r * ldo + c] = split_hi(v, trunc);
        lo[r * ldo + c] = split_lo(v, trunc);
    }
}

__global__ void split4_kernel(const float4* __restrict__ x, int64_t ldx4, int rows, int cols4, float4* __restrict__ hi,
                              float4* __restrict__ lo, int64_t ldo4, bool trunc) {
    const int64_t total = (int64_t)rows * cols4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols4), c = (int)(i % cols4);
        const float4 v = x[r * ldx4 + c];
        hi[r * ldo4 + c] = make_float4(split_hi(v.x, trunc), split_hi(v.y, trunc), split_hi(v.z, trunc),
                                       split_hi(v.w, trunc));
        lo[r * ldo4 + c] = make_float4(split_lo(v.x, trunc), split_lo(v.y, trunc), split_lo(v.z, trunc),
                                       split_lo(v.w, trunc));
    }
}

// Padded split: the rows x cols input lands in the top-left corner of a
// rows_out x cols_out split output whose remaining entries are zero (ragged
// shapes on the large-batch path: zero samples, zero coordinates and zero
// vectors have no effect on the product, lb_run.cu).
__global__ void split_pad_kernel(const float* __restrict__ x, int64_t ldx, int rows, int cols, int rows_out,
                                 int cols_out, float* __restrict__ hi, float* __restrict__ lo, int64_t ldo,
                                 bool trunc) {
    const int64_t total = (int64_t)rows_out * cols_out;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols_out), c = (int)(i % cols_out);
        const float v = (r < rows && c < cols) ? x[r * ldx + c] : 0.f;
        hi[r * ldo + c] = split_hi(v, trunc);
        lo[r * ldo + c] = split_lo(v, trunc);
    }
}

// out (d_out x n_out) = split(V^T), V n x d; entries past (d, n) are zero
__global__ void split_t_kernel(const float* __restrict__ v, int64_t ldv, int n, int d, int n_out, int d_out,
                               float* __restrict__ hi, float* __restrict__ lo, int64_t ldo) {
    __shared__ float t[32][33];
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;  // i over n (rows of V), j over d
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, j = j0 + threadIdx.x;
        t[r][threadIdx.x] = (i < n && j < d) ? v[(int64_t)i * ldv + j] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int j = j0 + r, i = i0 + threadIdx.x;
        if (j < d_out && i < n_out) {
            const float x = t[threadIdx.x][r];
            const float h = rn_hi(x);
            hi[(int64_t)j * ldo + i] = h;
            lo[(int64_t)j * ldo + i] = x - h;
        }
    }
}

// dst vector i = src vector n-1-i (vectors are the d-float columns)
__global__ void reverse_vectors_kernel(const float* __restrict__ src, int64_t lds, int d, int n,
                                       float* __restrict__ dst, int64_t ldd) {
    const int i = blockIdx.y;
    const float* a = src + (int64_t)(n - 1 - i) * lds;
    float* b = dst + (int64_t)i * ldd;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) b[k] = a[k];
}

int grid_for(int64_t work) {
    return (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
}

}  // namespace

cudaError_t split(const float* x, int64_t ldx, int rows, int cols, float* hi, float* lo, int64_t ldo,
                  cudaStream_t s, bool trunc) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    const bool vec = cols % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 &&
                     !((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) |
                        reinterpret_cast<uintptr_t>(lo)) & 15);
    if (vec)
        split4_kernel<<<grid_for((int64_t)rows * cols / 4), 256, 0, s>>>(
            reinterpret_cast<const float4*>(x), ldx / 4, rows, cols / 4, reinterpret_cast<float4*>(hi),
            reinterpret_cast<float4*>(lo), ldo / 4, trunc);
    else
        split_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(x, ldx, rows, cols, hi, lo, ldo, trunc);
    return cudaGetLastError();
}

cudaError_t reverse_vectors(const float* src, int64_t lds, int d, int n, float* dst, int64_t ldd, cudaStream_t s) {
    if (n <= 0 || d <= 0) return cudaSuccess;
    reverse_vectors_kernel<<<dim3((d + 255) / 256, n), 256, 0, s>>>(src, lds, d, n, dst, ldd);
    return cudaGetLastError();
}

cudaError_t split_pad(const float* x, int64_t ldx, int rows, int cols, int rows_out, int cols_out, float* hi,
                      float* lo, int64_t ldo, cudaStream_t s, bool trunc) {
    if (rows_out == rows && cols_out == cols) return split(x, ldx, rows, cols, hi, lo, ldo, s, trunc);
    if (rows_out <= 0 || cols_out <= 0) return cudaSuccess;
    split_pad_kernel<<<grid_for((int64_t)rows_out * cols_out), 256, 0, s>>>(x, ldx, rows, cols, rows_out, cols_out,
                                                                           hi, lo, ldo, trunc);
    return cudaGetLastError();
}

cudaError_t split_transpose(const float* v, int64_t ldv, int n, int d, float* hi, float* lo, int64_t ldo,
                            cudaStream_t s, int n_out, int d_out) {
    if (n_out < 0) n_out = n;
    if (d_out < 0) d_out = d;
    if (n_out <= 0 || d_out <= 0) return cudaSuccess;
    dim3 grid((d_out + 31) / 32, (n_out + 31) / 32);
    split_t_kernel<<<grid, dim3(32, 8), 0, s>>>(v, ldv, n, d, n_out, d_out, hi, lo, ldo);
    return cudaGetLastError();
}

}  // namespace lb
}  // namespace fasthb

// Test hook (not part of include/fasth_b200.h): one GEMM of the large-batch
// path on caller device buffers.  A: M x K row-major; B: N x K (b_mn = 0) or
// K x N (b_mn = 1) row-major; optional C (M x N).  Outputs any of D (fp32),
// D hi/lo, D^T hi/lo, or raw split-K partials [ksplit][M][N].
// a_mn = 1: A given K x M (M contiguous).
extern "C" int fasthb_lb_gemm_test_ex(const float* A, int64_t lda, int a_mn, const float* B, int64_t ldb, int b_mn,
                                      int M, int N, int K, const float* C, int64_t ldc, float alpha, float beta,
                                      float* D, int64_t ldd, float* Dhi, float* Dlo, int64_t lds, float* Thi,
                                      float* Tlo, int64_t ldt, float* partial, int ksplit, int debug_swap) {
    using namespace fasthb::lb;
    cudaStream_t s = 0;
    const int64_t arows = a_mn ? K : M, acols = a_mn ? M : K;
    const int64_t brows = b_mn ? K : N, bcols = b_mn ? N : K;
    const int64_t lda_p = (acols + 3) / 4 * 4, ldb_p = (bcols + 3) / 4 * 4, ldc_p = (N + 3) / 4 * 4;
    float *ah, *al, *bh, *bl, *ch = nullptr, *cl = nullptr;
    cudaMalloc(&ah, arows * lda_p * 4);
    cudaMalloc(&al, arows * lda_p * 4);
    cudaMalloc(&bh, brows * ldb_p * 4);
    cudaMalloc(&bl, brows * ldb_p * 4);
    split(A, lda, (int)arows, (int)acols, ah, al, lda_p, s);
    split(B, ldb, (int)brows, (int)bcols, bh, bl, ldb_p, s);
    if (C) {
        cudaMalloc(&ch, (int64_t)M * ldc_p * 4);
        cudaMalloc(&cl, (int64_t)M * ldc_p * 4);
        split(C, ldc, M, N, ch, cl, ldc_p, s);
    }
    Gemm g;
    g.M = M;
    g.N = N;
    g.nseg = 1;
    g.seg[0].A = Operand{ah, al, arows, acols, lda_p};
    g.a_mn = a_mn != 0;
    g.seg[0].B = Operand{bh, bl, brows, bcols, ldb_p};
    g.seg[0].K = K;
    g.b_mn = b_mn != 0;
    g.alpha = alpha;
    g.beta = beta;
    g.c_hi = ch;
    g.c_lo = cl;
    g.ldc = ldc_p;
    g.d_f32 = D;
    g.ldd = ldd;
    g.d_hi = Dhi;
    g.d_lo = Dlo;
    g.lds = lds;
    g.t_hi = Thi;
    g.t_lo = Tlo;
    g.ldt = ldt;
    g.partial = partial;
    g.ksplit = ksplit;
    g.debug_swap = debug_swap;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = gemm(g, s, sms);
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaFree(ah);
    cudaFree(al);
    cudaFree(bh);
    cudaFree(bl);
    if (ch) cudaFree(ch);
    if (cl) cudaFree(cl);
    if (e != cudaSuccess) return (int)e;
    return (int)e2;
}

extern "C" int fasthb_lb_gemm_test(const float* A, int64_t lda, const float* B, int64_t ldb, int b_mn, int M, int N,
                                   int K, const float* C, int64_t ldc, float alpha, float beta, float* D,
                                   int64_t ldd, float* Dhi, float* Dlo, int64_t lds, float* Thi, float* Tlo,
                                   int64_t ldt, float* partial, int ksplit, int debug_swap) {
    return fasthb_lb_gemm_test_ex(A, lda, 0, B, ldb, b_mn, M, N, K, C, ldc, alpha, beta, D, ldd, Dhi, Dlo, lds, Thi,
                                  Tlo, ldt, partial, ksplit, debug_swap);
}
