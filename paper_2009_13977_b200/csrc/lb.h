// Large-batch path (internal, non-ABI): FastH re-blocked into wide WY blocks
// so that every chain step is a large GEMM on the 5th-generation tensor cores.
//
// Memory is batch-major, as the C ABI hands it over (column-major d x m:
// sample c is the contiguous row X[c][0..d)).  With B-wide blocks
// (B in {512, 256, 128}, vectors jB..jB+B-1 of the chain) and
//   WfR_j = T~_j V_j,  WbR_j = T~_j^T V_j      (B x d; V_j = the block's rows)
// one forward block step is, for the m x d activations Xm,
//   ZfT = Xm WfR_j^T            (m x B)   GEMM  M=m N=B K=d
//   Xm <- Xm - 2 ZfT VT_j^T     (m x d)   GEMM  M=m N=d K=B  (VT = V^T, d x n)
// and one backward step, for the m x d gradient Gm and the block's output
// activations Am (the forward tape),
//   ZbT = Gm WbR_j^T
//   Q   = Zf Zb^T               (B x B)   GEMM  K=m (A = ZfT, B = ZbT read MN-major)
//   dV_j = -2 (Zb Am + Zf Gm) - 4 K'^T V_j,   K' = striu(Q - Q^T)   (A operands MN-major)
//   Gm <- Gm - 2 ZbT VT_j^T
// — exactly tests/algo_model.py's algebra with block width B (the product is
// independent of the blocking; the reference's own results agree across block
// widths to 1e-10).
//
// Every operand of every product is stored pre-split for 3xTF32 (hi = RN to
// tf32, lo = x - hi, both fp32 containers); the GEMM epilogues emit the split
// form of whatever feeds a later product.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "fasth_internal.h"

namespace fasthb {
namespace lb {

constexpr int BM = 128;   // UMMA M (one CTA, cta_group::1)
constexpr int BN = 256;   // UMMA N
constexpr int BK = 32;    // K per stage: one 128-byte swizzle atom of fp32
constexpr int STAGES = 2;

struct Operand {          // row-major matrix of fp32, pre-split
    const float* hi = nullptr;
    const float* lo = nullptr;
    int64_t rows = 0, cols = 0, ld = 0;
};

struct Segment {          // one K range of the product
    Operand A;            // M x K, K contiguous (K-major)
    Operand B;            // N x K (K-major) or K x N (MN-major)
    int K = 0;
    int a_row0 = 0, a_col0 = 0;   // A coordinates of (m = 0, k = 0)
    int b_row0 = 0, b_col0 = 0;   // B coordinates of (n = 0, k = 0) / (k = 0, n = 0)
};

struct Gemm {
    int M = 0, N = 0;
    int nseg = 1;
    Segment seg[3];
    bool a_mn = false;    // A stored K x M (M contiguous): segment rows are k, columns m
    bool b_mn = false;    // B stored K x N (N contiguous)
    int ksplit = 1;       // > 1 (or partial != nullptr): raw partials per K split
    int nz = 1;           // batched products, coordinates advance per z:
    int z_a_row = 0, z_a_col = 0, z_b_row = 0, z_b_col = 0;
    int64_t z_out = 0;    // output element offset per z (direct and partial outputs)
    float alpha = 1.f, beta = 0.f;
    // epilogue (direct): D = alpha acc + beta (C_hi + C_lo)
    const float *c_hi = nullptr, *c_lo = nullptr;
    int64_t ldc = 0;
    float* d_f32 = nullptr;
    int64_t ldd = 0;
    float *d_hi = nullptr, *d_lo = nullptr;
    int64_t lds = 0;
    // split_trunc: D written as (x, x - trunc_tf32(x)) instead of (RN hi, lo):
    // the tensor core truncates x itself, so the pair is still an exact split,
    // and a later epilogue reads the value back as one array (c_single: C = c_hi)
    bool split_trunc = false, c_single = false;
    float *t_hi = nullptr, *t_lo = nullptr;  // transposed split copy D^T (N x M)
    int64_t ldt = 0;
    float* partial = nullptr;                // [nz][ksplit][M][N]
    // optional: products with few tiles (small batch) split K into this
    // scratch ([nz][ks][M][N]) and finish in a reduction epilogue kernel
    float* split_scratch = nullptr;
    int64_t split_scratch_floats = 0;
    int launched = 0;                        // out: kernels gemm() launched (1, or 2 with the reduction)
    int debug_swap = 0;                      // test hook: MN-major LBO/SBO swap
};

// One launch of the persistent tcgen05 3xTF32 GEMM.  g.ksplit is updated to the
// split count actually used (no empty K splits).
cudaError_t gemm(Gemm& g, cudaStream_t s, int num_sms);

// Optional per-launch timing (the context's timing mode): begin() before a
// launch, end() after it with the kernel's name.
struct Timer {
    virtual void begin(cudaStream_t s) = 0;
    virtual void end(cudaStream_t s, const char* name) = 0;
    virtual ~Timer() = default;
};

// A second stream for the independent work of the step (input splits during
// the build; the Q / dV products of block j while the gradient update of
// block j runs), with reusable fork/join events.  nullptr: one stream.
struct Streams {
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[16] = {};  // 0-7, 12-15: large-batch step, 8-11: SVD layer legs (capi.cpp)
};

// dV completion per row bucket (batch-sharded data parallelism, SURVEY
// §8(e)): the backward records ev[k] on the stream that wrote the last dV
// rows of bucket k as soon as they are final, so a caller can all-reduce
// those rows while the remaining blocks run.  Blocks are grouped into
// min(count, blocks) buckets in backward order (rows 0.. first); row_end[k]
// is the exclusive end row of bucket k, `used` the bucket count.
struct DvNotify {
    const cudaEvent_t* ev = nullptr;
    int count = 0;
    int64_t* row_end = nullptr;
    int used = 0;
};

// The whole large-batch step (lb_run.cu).  Any shape: internally the step runs
// on padded dimensions (pad_dims) — zero coordinates past d, zero samples past
// m and zero vectors past n, whose diagonal entry of the triangular factor is
// set to 1 so that they are exact identities — and the outputs are cut back.
struct Dims {
    int d, n, m;      // the caller's shape
    int dp, np, mp;   // the padded shape every product runs on
    bool padded() const { return dp != d || np != n || mp != m; }
};
Dims pad_dims(int d, int n, int m);
int pick_block(int n);
bool supported(int d, int n, int m);
size_t workspace_floats(int d, int n, int m, bool want_dv);
// The two halves (fasth_forward / fasth_backward): `ws` carries the forward
// stages from one to the other.
// (forward: G non-null also splits the gradient for a following backward
// called with g_split = true — the fused call)
cudaError_t forward(const float* V, int64_t ldv, int d, int n, const float* X, int64_t ldx, int m, float* Y,
                    int64_t ldy, float* ws, ErrWord* err, cudaStream_t s, int num_sms, int* nlaunch,
                    Timer* tm = nullptr, const Streams* st = nullptr, const float* G = nullptr, int64_t ldg = 0,
                    bool* k1_pre = nullptr);
cudaError_t backward(int d, int n, int m, const float* G, int64_t ldg, float* dX, int64_t lddx, float* dV,
                     int64_t lddv, float* ws, cudaStream_t s, int num_sms, int* nlaunch, Timer* tm = nullptr,
                     const Streams* st = nullptr, bool g_split = false, DvNotify* nt = nullptr,
                     bool k1_pre = false);
cudaError_t forward_backward(const float* V, int64_t ldv, int d, int n, const float* X, int64_t ldx, const float* G,
                             int64_t ldg, int m, float* Y, int64_t ldy, float* dX, int64_t lddx, float* dV,
                             int64_t lddv, float* ws, ErrWord* err, cudaStream_t s, int num_sms, int* nlaunch,
                             Timer* tm = nullptr, const Streams* st = nullptr, DvNotify* nt = nullptr);

// Elementwise helpers (lb_path.cu).
// dst vector i = src vector n-1-i (d-float vectors, leading dims lds / ldd):
// the SVD layer's V^T leg is the V chain in reverse order
cudaError_t reverse_vectors(const float* src, int64_t lds, int d, int n, float* dst, int64_t ldd, cudaStream_t s);
// split rows x cols (ld_in) into hi/lo (ld_out)
// (trunc: the (x, x - trunc_tf32(x)) form, see Gemm::split_trunc)
cudaError_t split(const float* x, int64_t ldx, int rows, int cols, float* hi, float* lo,
                  int64_t ldo, cudaStream_t s, bool trunc = false);
// the same into the top-left corner of a zero-padded rows_out x cols_out output
cudaError_t split_pad(const float* x, int64_t ldx, int rows, int cols, int rows_out, int cols_out, float* hi,
                      float* lo, int64_t ldo, cudaStream_t s, bool trunc = false);
// VT = V^T split: V is n x d (ldv), VT d x n (zero-padded to d_out x n_out when given)
cudaError_t split_transpose(const float* v, int64_t ldv, int n, int d, float* hi, float* lo,
                            int64_t ldo, cudaStream_t s, int n_out = -1, int d_out = -1);

}  // namespace lb
}  // namespace fasthb
