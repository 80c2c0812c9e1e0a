// Large-batch FastH step (forward + backward) on the tcgen05 GEMM — see lb.h
// for the algebra.  Block j covers chain vectors [jB, jB+B); the forward
// applies blocks nb-1 .. 0 (H_n first, as the reference's fasth.hpp:40 chain),
// the backward walks 0 .. nb-1.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lb.h"

namespace fasthb {
namespace lb {
namespace {

__device__ __forceinline__ float rn_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// M_z = diag(G_z) + 2 striu(G_z), G_z = sum of the ks Gram partials
// (flags a degenerate / non-finite ||v_i||^2 like the block builder).
// Padding vectors (index >= n_valid) are zero: their row and column of M are
// zero, and a unit diagonal entry makes each an exact identity factor.
__global__ void gram_reduce_kernel(const float* __restrict__ part, int ks, int B, int nz, int n_valid,
                                   float* __restrict__ Mm, ErrWord* err) {
    const int64_t per = (int64_t)B * B, total = per * nz;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = e / per, w = e % per;
        const int i = (int)(w / B), j = (int)(w % B);
        float g = 0.f;
        if (j >= i)
            for (int s = 0; s < ks; ++s) g += part[(z * ks + s) * per + w];
        const bool pad = z * B + i >= n_valid;
        Mm[e] = j > i ? 2.f * g : (j == i ? (pad ? 1.f : g) : 0.f);
        if (j == i && !pad && (!(g > 1e-30f) || !isfinite(g))) {
            atomicOr(&err->flags, isfinite(g) ? kErrDegenerate : kErrNonFinite);
            atomicMin(&err->index, (int)(z * B + i));
            err->chain = 0;
        }
    }
}

// Inverses of the 32 x 32 diagonal blocks of M_z (upper triangular), lane =
// column of the inverse, back substitution.  grid (B/32, nz), 32 threads.
__global__ void diag_inv_kernel(const float* __restrict__ Mm, int B, float* __restrict__ Dinv) {
    __shared__ float U[32][33];
    const int rc = blockIdx.x, z = blockIdx.y, lane = threadIdx.x;
    const float* M = Mm + (int64_t)z * B * B + (int64_t)rc * 32 * B + rc * 32;
    for (int i = 0; i < 32; ++i) U[i][lane] = M[(int64_t)i * B + lane];
    __syncwarp();
    float x[32];
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        float s = i == lane ? 1.f : 0.f;
#pragma unroll
        for (int k = i + 1; k < 32; ++k) s = fmaf(-U[i][k], x[k], s);
        x[i] = s / U[i][i];
    }
    float* D = Dinv + ((int64_t)z * (B / 32) + rc) * 1024;
#pragma unroll
    for (int i = 0; i < 32; ++i) D[i * 32 + lane] = x[i];
}

// T_z = M_z^{-1} by blocked back-substitution over 32-row chunks:
//   T[rc][cc] = Dinv_rc (E - sum_{k > rc} M[rc][k] T[k][cc]),
// one CTA per pair of CW-column chunks (cc, B/CW-1-cc) for balanced work (CW =
// 16: twice the CTAs of 32-wide chunks, half the work per dependent step).
// The M row panel of step rc-1 streams into shared memory (cp.async, double
// buffered) while step rc computes; the update product is register blocked:
// 64 threads x (4 rows x CW/8 columns) cover the 32 x CW block, 4 thread
// groups take contiguous quarters of k.  Writes T and T^T, both split.
// grid (B/(2 CW), nz), 256 threads.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
template <int CW>
__global__ void __launch_bounds__(256) tri_inv_kernel(const float* __restrict__ Mm, const float* __restrict__ Dinv,
                                                      int B, float* __restrict__ Th, float* __restrict__ Tl,
                                                      float* __restrict__ TTh, float* __restrict__ TTl) {
    constexpr int CPT = CW / 8;     // columns per thread in the update
    constexpr int RP = CW + 1;      // red / R pitch
    extern __shared__ float sm[];
    const int MP = B + 12;          // panel pitch: at most 2-way conflicts for the float4 reads
    float* Tc = sm;                 // [B][CW] solution chunk
    float* Mp = Tc + B * CW;        // [2][32][MP] M row panels
    float* red = Mp + 2 * 32 * MP;  // [4][32][RP] k-split partial sums (also the T^T tile)
    float* R = red + 4 * 32 * RP;   // [32][RP] right-hand side
    float* Ddb = R + 32 * RP;       // [2][32][36] diagonal-block inverses
    const int z = blockIdx.y, nchunk = B / CW;
    const float* M = Mm + (int64_t)z * B * B;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kq = tid >> 6, t64 = tid & 63, rg = t64 >> 3, cg = t64 & 7;
    for (int pass = 0; pass < 2; ++pass) {
        const int cc = pass == 0 ? blockIdx.x : nchunk - 1 - blockIdx.x;
        const int c0 = cc * CW, k1 = c0 + CW;
        // step rc's operands -> buffer rc & 1: the M panel (rows rc*32..,
        // columns [(rc+1)*32, k1)) and Dinv_rc
        auto prefetch = [&](int rc) {
            if (rc < 0) return;
            const int k0 = (rc + 1) * 32, nf4 = k1 > k0 ? (k1 - k0) / 4 : 0;
            float* dst = Mp + (rc & 1) * 32 * MP;
            for (int e = tid; e < 32 * nf4; e += 256) {
                const int i = e / nf4, k = k0 + 4 * (e % nf4);
                cp_async16(dst + i * MP + k, M + (int64_t)(rc * 32 + i) * B + k);
            }
            const float* D = Dinv + ((int64_t)z * (B / 32) + rc) * 1024;
            float* dd = Ddb + (rc & 1) * 32 * 36;
            const int i = tid >> 3, k = (tid & 7) * 4;
            cp_async16(dd + i * 36 + k, D + i * 32 + k);
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        __syncthreads();
        for (int e = tid; e < B * CW; e += 256) Tc[e] = 0.f;
        const int rtop = c0 / 32;  // row chunk holding the chunk's diagonal
        prefetch(rtop);
        __syncthreads();
        for (int rc = rtop; rc >= 0; --rc) {
            const int r0 = rc * 32, k0 = (rc + 1) * 32;
            const float* Dd = Ddb + (rc & 1) * 32 * 36;
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();  // panel rc landed (all threads' copies); the other buffer is free
            prefetch(rc - 1);
            {  // partial products over this group's quarter of [k0, k1)
                const int q4 = k1 > k0 ? (k1 - k0) / 4 : 0;
                const int kb = k0 + kq * q4, ke = kb + q4;
                const float* mp = Mp + (rc & 1) * 32 * MP + (4 * rg) * MP;
                float acc[4][CPT] = {};
                for (int k = kb; k < ke; k += 4) {
                    float4 m4[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) m4[a] = *reinterpret_cast<const float4*>(mp + a * MP + k);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        float tv[CPT];
#pragma unroll
                        for (int bq = 0; bq < CPT; ++bq) tv[bq] = Tc[(k + kk) * CW + CPT * cg + bq];
#pragma unroll
                        for (int a2 = 0; a2 < 4; ++a2) {
                            const float mv = kk == 0 ? m4[a2].x : kk == 1 ? m4[a2].y : kk == 2 ? m4[a2].z : m4[a2].w;
#pragma unroll
                            for (int bq = 0; bq < CPT; ++bq) acc[a2][bq] = fmaf(mv, tv[bq], acc[a2][bq]);
                        }
                    }
                }
#pragma unroll
                for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                    for (int bq = 0; bq < CPT; ++bq) red[(kq * 32 + 4 * rg + a2) * RP + CPT * cg + bq] = acc[a2][bq];
            }
            __syncthreads();
            for (int e = tid; e < 32 * CW; e += 256) {
                const int r = e / CW, c = e % CW;
                const float sum = red[(0 * 32 + r) * RP + c] + red[(1 * 32 + r) * RP + c] +
                                  red[(2 * 32 + r) * RP + c] + red[(3 * 32 + r) * RP + c];
                R[r * RP + c] = (r0 + r == c0 + c ? 1.f : 0.f) - sum;
            }
            __syncthreads();
            {  // T[rc] = Dinv_rc R  (Dinv upper triangular)
                const int r = tid >> 3, cb = (tid & 7) * CPT;
                float acc[CPT] = {};
                for (int k = r; k < 32; ++k) {
                    const float dd = Dd[r * 36 + k];
#pragma unroll
                    for (int bq = 0; bq < CPT; ++bq) acc[bq] = fmaf(dd, R[k * RP + cb + bq], acc[bq]);
                }
#pragma unroll
                for (int bq = 0; bq < CPT; ++bq) Tc[(r0 + r) * CW + cb + bq] = acc[bq];
            }
            __syncthreads();
        }
        float* th = Th + (int64_t)z * B * B;
        float* tl = Tl + (int64_t)z * B * B;
        float* tth = TTh + (int64_t)z * B * B;
        float* ttl = TTl + (int64_t)z * B * B;
        for (int e = tid; e < B * CW; e += 256) {
            const int r = e / CW, c = e % CW;
            const float v = Tc[e];
            const float h = rn_hi(v);
            th[(int64_t)r * B + c0 + c] = h;
            tl[(int64_t)r * B + c0 + c] = v - h;
        }
        for (int rb = 0; rb < B / 32; ++rb) {  // T^T through a padded 32 x CW tile (red)
            __syncthreads();
#pragma unroll
            for (int u = 0; u < CPT; ++u) red[(warp + 8 * u) * 33 + lane] = Tc[(rb * 32 + lane) * CW + warp + 8 * u];
            __syncthreads();
#pragma unroll
            for (int u = 0; u < CPT; ++u) {
                const int c = warp + 8 * u;
                const float v = red[c * 33 + lane];
                const float h = rn_hi(v);
                tth[(int64_t)(c0 + c) * B + rb * 32 + lane] = h;
                ttl[(int64_t)(c0 + c) * B + rb * 32 + lane] = v - h;
            }
        }
    }
}

// Q = sum of the ks split-K partials (B x B), one element per thread, all
// partial loads independent.
__global__ void q_sum_kernel(const float* __restrict__ part, int ks, int64_t per, float* __restrict__ Q) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= per) return;
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = k < ks ? __ldg(part + k * per + e) : 0.f;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += v[k];
    for (int k = 16; k < ks; ++k) s += part[k * per + e];
    Q[e] = s;
}

// S = 2 K'^T (the dV product's alpha = -2 makes it -4 K'^T), K' = striu(Q - Q^T),
// written transposed (the dV product reads every A operand K x M); split.
// 32 x 32 tiles through shared memory.  grid (B/32, B/32), 32 x 8 threads.
__global__ void s_from_q_kernel(const float* __restrict__ Q, int B, float* __restrict__ Sh, float* __restrict__ Sl) {
    __shared__ float qt[32][33], qtt[32][33];
    const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32, tx = threadIdx.x;
    for (int r = threadIdx.y; r < 32; r += 8) {
        qt[r][tx] = Q[(int64_t)(a0 + r) * B + b0 + tx];   // Q[a0+r][b0+tx]
        qtt[r][tx] = Q[(int64_t)(b0 + r) * B + a0 + tx];  // Q[b0+r][a0+tx]
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {  // S^T[a][b] = S[b][a] = 2 (Q[a][b] - Q[b][a]) for a < b
        const int a = a0 + r, b = b0 + tx;
        const float v = a < b ? 2.f * (qt[r][tx] - qtt[tx][r]) : 0.f;
        const float h = rn_hi(v);
        Sh[(int64_t)a * B + b] = h;
        Sl[(int64_t)a * B + b] = v - h;
    }
}

// dV rows (B x d) = sum of ks partials; only rows < rows_valid and columns
// < d_valid (the caller's shape) are written
__global__ void dv_reduce_kernel(const float* __restrict__ part, int ks, int B, int d, int rows_valid, int d_valid,
                                 float* __restrict__ dV, int64_t lddv) {
    const int64_t per = (int64_t)B * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / d), c = (int)(e % d);
        if (r >= rows_valid || c >= d_valid) continue;
        float s = 0.f;
#pragma unroll 4
        for (int k = 0; k < ks; ++k) s += __ldg(part + k * per + e);
        dV[(int64_t)r * lddv + c] = s;
    }
}

int grid_for(int64_t work) { return (int)std::min<int64_t>((work + 255) / 256, 148 * 16); }

}  // namespace

int pick_block(int n) {
    for (int B : {512, 256, 128})
        if (n % B == 0) return B;
    return 0;
}

// The products need d and m multiples of 4 (16-byte TMA strides), n a
// multiple of the block width and d >= 128, m >= 16 (tile shapes).
Dims pad_dims(int d, int n, int m) {
    Dims D{d, n, m, 0, 0, 0};
    D.dp = std::max(128, (d + 3) / 4 * 4);
    D.np = std::max(128, (n + 127) / 128 * 128);
    D.mp = std::max(16, (m + 3) / 4 * 4);
    return D;
}

bool supported(int d, int n, int m) {
    return d >= 1 && n >= 1 && m >= 1 && d <= (1 << 24) && n <= (1 << 24) && m <= (1 << 26);
}

// split-K scratch for the chain products when the batch is too small for
// their output tiles to fill the GPU: up to 64 partial m x max(d, n) slabs,
// capped at 128 MB
int64_t small_batch_scratch(int d, int n, int m) {
    return m < 1024 ? std::min<int64_t>((int64_t)64 * m * std::max(d, n), (int64_t)32 << 20) : 0;
}

size_t workspace_floats(int d0, int n0, int m0, bool want_dv) {
    const Dims D = pad_dims(d0, n0, m0);
    const int d = D.dp, n = D.np, m = D.mp;
    const int B = pick_block(n), nb = n / B;
    const size_t nd = (size_t)n * d, md = (size_t)m * d, bb = (size_t)B * B;
    size_t f = 0;
    f += 4 * nd;                    // V, V^T split
    f += (size_t)nb * 4 * bb;       // Gram partials (ks <= 4)
    f += (size_t)nb * bb;           // M
    f += (size_t)nb * 32 * B;       // diagonal block inverses
    f += 4 * (size_t)nb * bb;       // T, T^T split
    f += 4 * nd;                    // WfR, WbR split
    f += 2 * (size_t)(nb + 1) * md;  // forward stages split
    f += 2 * (size_t)m * B * 3;     // ZbT (x3) split
    f += 2 * (size_t)n * m;         // ZfT of all blocks (m x n) split
    f += 6 * md;                    // three gradient buffers split
    (void)want_dv;                  // the forward carves the backward's buffers too
    f += 16 * bb + 3 * bb;          // Q partials, Q, S split
    f += 8 * (size_t)B * d;         // dV partials
    f += (size_t)small_batch_scratch(d, n, m);
    return f + 256 * 32;            // alignment slack
}

struct Carver {
    float* p;
    float* take(size_t n) {
        float* r = p;
        p += (n + 31) / 32 * 32;  // 128-byte aligned pieces
        return r;
    }
};

namespace {

struct Bufs {
    Dims D{};
    int B = 0, nb = 0;
    size_t nd = 0, md = 0, bb = 0;
    float *Vh, *Vl, *VTh, *VTl, *Gp, *Mm, *Dinv, *Th, *Tl, *TTh, *TTl, *WfH, *WfL, *WbH, *WbL;
    std::vector<float*> Sth, Stl;  // forward stages 0..nb
    float *ZbTh2[3], *ZbTl2[3], *ZfAh, *ZfAl, *Gh[3], *Gl[3];  // ZfA: m x n, block j = columns jB..
    float *Qp, *Qs, *Sh, *Sl, *dVp;
    float* ksc;  // split-K scratch of the small-batch chain products (m < 1024)
    int64_t ksc_n;
};
constexpr int ksG = 4, ksQ = 16, ksV = 4;  // split-K counts (128 CTAs each: one tile per CTA)

// The workspace is carved identically by the forward and the backward half.
// (padded dimensions, pad_dims)
bool carve(float* ws, int d0, int n0, int m0, Bufs& b) {
    b.D = pad_dims(d0, n0, m0);
    const int d = b.D.dp, n = b.D.np, m = b.D.mp;
    b.B = pick_block(n);
    if (!b.B) return false;
    b.nb = n / b.B;
    b.Sth.assign(b.nb + 1, nullptr);
    b.Stl.assign(b.nb + 1, nullptr);
    const int B = b.B, nb = b.nb;
    const size_t nd = b.nd = (size_t)n * d, md = b.md = (size_t)m * d, bb = b.bb = (size_t)B * B;
    Carver c{ws};
    b.Vh = c.take(nd), b.Vl = c.take(nd), b.VTh = c.take(nd), b.VTl = c.take(nd);
    b.Gp = c.take((size_t)nb * ksG * bb);
    b.Mm = c.take((size_t)nb * bb);
    b.Dinv = c.take((size_t)nb * 32 * B);
    b.Th = c.take(nb * bb), b.Tl = c.take(nb * bb), b.TTh = c.take(nb * bb), b.TTl = c.take(nb * bb);
    b.WfH = c.take(nd), b.WfL = c.take(nd), b.WbH = c.take(nd), b.WbL = c.take(nd);
    for (int j = 0; j <= nb; ++j) {
        b.Sth[j] = c.take(md);
        b.Stl[j] = c.take(md);
    }
    for (int i = 0; i < 3; ++i) b.ZbTh2[i] = c.take((size_t)m * B), b.ZbTl2[i] = c.take((size_t)m * B);
    b.ZfAh = c.take((size_t)m * n), b.ZfAl = c.take((size_t)m * n);
    for (int i = 0; i < 3; ++i) b.Gh[i] = c.take(md), b.Gl[i] = c.take(md);
    b.Qp = c.take(ksQ * bb);
    b.Qs = c.take(bb);
    b.Sh = c.take(bb);
    b.Sl = c.take(bb);
    b.dVp = c.take((size_t)(ksV + 1) * B * d);
    b.ksc_n = small_batch_scratch(d, n, m);
    b.ksc = b.ksc_n ? c.take((size_t)b.ksc_n) : nullptr;
    return true;
}

#define LBTRY(x)                                \
    do {                                        \
        if ((e = (x)) != cudaSuccess) return e; \
    } while (0)
// one GEMM launch, timed in the context's timing mode, counted
#define LB_GEMM(g, st, name)          \
    do {                              \
        if (tm) tm->begin(st);        \
        LBTRY(gemm(g, st, num_sms));  \
        if (tm) tm->end(st, name);    \
        nl += g.launched;             \
    } while (0)
#define LB_ALIASES                                                                                           \
    const int B = b.B, nb = b.nb;                                                                            \
    const size_t bb = b.bb;                                                                                  \
    (void)bb;                                                                                                \
    float *Vh = b.Vh, *Vl = b.Vl, *VTh = b.VTh, *VTl = b.VTl, *Gp = b.Gp, *Mm = b.Mm, *Dinv = b.Dinv;       \
    float *Th = b.Th, *Tl = b.Tl, *TTh = b.TTh, *TTl = b.TTl, *WfH = b.WfH, *WfL = b.WfL, *WbH = b.WbH;      \
    float *WbL = b.WbL, **Sth = b.Sth.data(), **Stl = b.Stl.data(), *ZfAh = b.ZfAh, *ZfAl = b.ZfAl;                        \
    float **Gh = b.Gh, **Gl = b.Gl;                                                                          \
    float *Qp = b.Qp, *Qs = b.Qs, *Sh = b.Sh, *Sl = b.Sl, *dVp = b.dVp;                                    \
    (void)Vh, (void)Vl, (void)VTh, (void)VTl, (void)Gp, (void)Mm, (void)Dinv, (void)Th, (void)Tl, (void)TTh; \
    (void)TTl, (void)WfH, (void)WfL, (void)WbH, (void)WbL, (void)Sth, (void)Stl, (void)ZfAh, (void)ZfAl;     \
    (void)Gh, (void)Gl, (void)Qp;                                                                          \
    (void)Qs, (void)Sh, (void)Sl, (void)dVp

}  // namespace

// Build (V -> T~, WfR, WbR) and the forward chain; the workspace keeps every
// forward stage for the backward half.
cudaError_t forward(const float* V, int64_t ldv, int d, int n, const float* X, int64_t ldx, int m, float* Y,
                    int64_t ldy, float* ws, ErrWord* err, cudaStream_t s, int num_sms, int* nlaunch, Timer* tm,
                    const Streams* st, const float* G, int64_t ldg, bool* k1_pre) {
    int nl = 0;
    if (k1_pre) *k1_pre = false;
    Bufs b;
    if (!supported(d, n, m) || !carve(ws, d, n, m, b)) return cudaErrorInvalidValue;
    const Dims D = b.D;
    const bool pad = D.padded();  // Y is then cut out of the last stage
    if (Y && !pad && ((ldy % 4) || (reinterpret_cast<uintptr_t>(Y) & 15))) return cudaErrorInvalidValue;
    LB_ALIASES;
    cudaError_t e;
    // the input splits do not depend on the build: on the second stream (the
    // triangular inverse leaves most SMs idle)
    const bool two = st && st->aux;
    cudaStream_t sx = two ? st->aux : s;
    if (two) {
        LBTRY(cudaEventRecord(st->ev[0], s));
        LBTRY(cudaStreamWaitEvent(sx, st->ev[0], 0));
    }
    ++nl;  // stages: (x, x - trunc(x))
    LBTRY(split_pad(X, ldx, D.m, D.d, D.mp, D.dp, Sth[nb], Stl[nb], D.dp, sx, true));
    if (G) {
        ++nl;
        LBTRY(split_pad(G, ldg, D.m, D.d, D.mp, D.dp, Gh[0], Gl[0], D.dp, sx, true));
    }
    if (two) LBTRY(cudaEventRecord(st->ev[1], sx));
    // ---- build: split V and V^T, Gram per block, T~, WfR = T~ V_j, WbR = T~^T V_j
    ++nl;
    LBTRY(split_pad(V, ldv, D.n, D.d, D.np, D.dp, Vh, Vl, D.dp, s));
    ++nl;
    LBTRY(split_transpose(V, ldv, D.n, D.d, VTh, VTl, D.np, s, D.np, D.dp));
    // from here on every product runs on the padded shape
    d = D.dp, n = D.np, m = D.mp;
    int g_ks = ksG;
    {
        Gemm g;
        g.M = g.N = B;
        g.seg[0].A = Operand{Vh, Vl, n, d, d};
        g.seg[0].B = Operand{Vh, Vl, n, d, d};
        g.seg[0].K = d;
        g.nz = nb;
        g.z_a_row = B;
        g.z_b_row = B;
        g.partial = Gp;
        g.ksplit = ksG;
        LB_GEMM(g, s, "lb_build_gram");
        g_ks = g.ksplit;
    }
    ++nl;
    gram_reduce_kernel<<<grid_for(nb * bb), 256, 0, s>>>(Gp, g_ks, B, nb, D.n, Mm, err);
    {
        ++nl;
        diag_inv_kernel<<<dim3(B / 32, nb), 32, 0, s>>>(Mm, B, Dinv);
        constexpr int CW = 16;
        const int smem = (B * CW + 2 * 32 * (B + 12) + 5 * 32 * (CW + 1) + 2 * 32 * 36) * 4;
        LBTRY(ensure_smem(reinterpret_cast<const void*>(tri_inv_kernel<CW>), smem));
        ++nl;
        if (tm) tm->begin(s);
        tri_inv_kernel<CW><<<dim3(B / (2 * CW), nb), 256, smem, s>>>(Mm, Dinv, B, Th, Tl, TTh, TTl);
        if (tm) tm->end(s, "lb_build_tri_inv");
        LBTRY(cudaGetLastError());
    }
    // WfR = T V_j, WbR = T^T V_j  (B x d per block); WbR is the backward's
    // operand: on the second stream, beside WfR and the first forward block
    if (two) {
        LBTRY(cudaEventRecord(st->ev[3], s));
        LBTRY(cudaStreamWaitEvent(sx, st->ev[3], 0));
    }
    for (int w = 0; w < 2; ++w) {
        const cudaStream_t sw = w == 1 ? sx : s;
        Gemm g;
        g.M = B;
        g.N = d;
        g.seg[0].A = w == 0 ? Operand{Th, Tl, (int64_t)nb * B, B, B} : Operand{TTh, TTl, (int64_t)nb * B, B, B};
        g.seg[0].B = Operand{VTh, VTl, d, n, n};  // (n = d index, k = chain index) K-major
        g.seg[0].K = B;
        g.nz = nb;
        g.z_a_row = B;
        g.z_b_col = B;
        g.z_out = B;
        g.d_hi = w == 0 ? WfH : WbH;
        g.d_lo = w == 0 ? WfL : WbL;
        g.lds = d;
        LB_GEMM(g, sw, "lb_build_w");
    }
    // fused step (G given): the gradient chain's first product Zb_0 = G WbR_0^T
    // needs only G and WbR, so it runs beside the forward chain (no split-K
    // scratch at this batch: nothing shared with the main stream)
    if (two && G && k1_pre && !b.ksc && !getenv("FASTH_LB_NO_EARLY_K1")) {
        Gemm g;
        g.M = m;
        g.N = B;
        g.seg[0].A = Operand{Gh[0], Gl[0], m, d, d};
        g.seg[0].B = Operand{WbH, WbL, n, d, d};
        g.seg[0].K = d;
        g.d_hi = b.ZbTh2[0];
        g.d_lo = b.ZbTl2[0];
        g.lds = B;
        LB_GEMM(g, sx, "lb_k1_zb");
        *k1_pre = true;
    }
    if (two) LBTRY(cudaEventRecord(st->ev[6], sx));
    // ---- forward: stage nb = split X; stage j = output of block j
    if (two) LBTRY(cudaStreamWaitEvent(s, st->ev[1], 0));
    for (int j = nb - 1; j >= 0; --j) {
        {
            Gemm g;  // ZfT = A WfR_j^T (m x B), Zf_j = its transpose (B x m)
            g.split_scratch = b.ksc;
            g.split_scratch_floats = b.ksc_n;
            g.M = m;
            g.N = B;
            g.seg[0].A = Operand{Sth[j + 1], Stl[j + 1], m, d, d};
            g.seg[0].B = Operand{WfH, WfL, n, d, d};
            g.seg[0].b_row0 = j * B;
            g.seg[0].K = d;
            g.d_hi = ZfAh + (size_t)j * B;  // columns jB.. of the m x n ZfT of all blocks
            g.d_lo = ZfAl + (size_t)j * B;
            g.lds = n;
            LB_GEMM(g, s, "lb_f1_zf");
        }
        {
            Gemm g;  // A_j = A_{j+1} - 2 ZfT VT_j^T
            g.split_scratch = b.ksc;
            g.split_scratch_floats = b.ksc_n;
            g.M = m;
            g.N = d;
            g.seg[0].A = Operand{ZfAh, ZfAl, m, n, n};
            g.seg[0].a_col0 = j * B;
            g.seg[0].B = Operand{VTh, VTl, d, n, n};
            g.seg[0].b_col0 = j * B;
            g.seg[0].K = B;
            g.alpha = -2.f;
            g.beta = 1.f;
            g.c_hi = Sth[j + 1];  // = the activation itself (trunc split)
            g.c_single = true;
            g.ldc = d;
            g.d_hi = Sth[j];
            g.d_lo = Stl[j];
            g.lds = d;
            g.split_trunc = true;
            if (j == 0 && !pad) {
                g.d_f32 = Y;
                g.ldd = ldy;
            }
            LB_GEMM(g, s, "lb_f2_update");
        }
    }
    if (pad && Y)  // the last stage holds the output itself (hi of the trunc split is x)
        LBTRY(cudaMemcpy2DAsync(Y, ldy * sizeof(float), Sth[0], (size_t)d * sizeof(float), (size_t)D.d * sizeof(float),
                                D.m, cudaMemcpyDeviceToDevice, s));
    if (two) LBTRY(cudaStreamWaitEvent(s, st->ev[6], 0));  // join: WbR built
    if (nlaunch) *nlaunch = nl;
    return cudaGetLastError();
}

// Backward chain and dV from the forward's workspace (same d, n, m).
cudaError_t backward(int d, int n, int m, const float* G, int64_t ldg, float* dX, int64_t lddx, float* dV,
                     int64_t lddv, float* ws, cudaStream_t s, int num_sms, int* nlaunch, Timer* tm,
                     const Streams* st, bool g_split, DvNotify* nt, bool k1_pre) {
    int nl = 0;
    Bufs b;
    if (!supported(d, n, m) || !carve(ws, d, n, m, b)) return cudaErrorInvalidValue;
    const Dims D = b.D;
    const bool pad = D.padded();  // dX is then cut out of the last gradient buffer
    if (dX && !pad && ((lddx % 4) || (reinterpret_cast<uintptr_t>(dX) & 15))) return cudaErrorInvalidValue;
    const bool want_dv = dV != nullptr;
    LB_ALIASES;
    cudaError_t e;
    // ---- backward.  Block j: K1 (Zb) on the main stream, then Q and dV of
    // block j on the second stream while the main stream updates G (K4).  G
    // and Zb are triple buffered (block j uses buffer j % 3), so the main
    // stream runs up to two blocks ahead of the dV stream: K4 of block j
    // (which overwrites buffer (j+1) % 3) waits only for block j-2's dV.
    if (!g_split) {
        ++nl;
        LBTRY(split_pad(G, ldg, D.m, D.d, D.mp, D.dp, Gh[0], Gl[0], D.dp, s, true));
    }
    d = D.dp, n = D.np, m = D.mp;
    const bool two = st && st->aux && want_dv;
    cudaStream_t sa = two ? st->aux : s;
    for (int j = 0; j < nb; ++j) {
        const int cur = j % 3, nxt = (j + 1) % 3;
        float *ZbTh = b.ZbTh2[cur], *ZbTl = b.ZbTl2[cur];
        if (!(j == 0 && k1_pre)) {
            Gemm g;  // ZbT = G WbR_j^T, Zb = transpose
            g.split_scratch = b.ksc;
            g.split_scratch_floats = b.ksc_n;
            g.M = m;
            g.N = B;
            g.seg[0].A = Operand{Gh[cur], Gl[cur], m, d, d};
            g.seg[0].B = Operand{WbH, WbL, n, d, d};
            g.seg[0].b_row0 = j * B;
            g.seg[0].K = d;
            g.d_hi = ZbTh;
            g.d_lo = ZbTl;
            g.lds = B;
            LB_GEMM(g, s, "lb_k1_zb");
        }
        if (want_dv) {
            if (two) {
                LBTRY(cudaEventRecord(st->ev[2], s));
                LBTRY(cudaStreamWaitEvent(sa, st->ev[2], 0));
            }
            int q_ks = ksQ, v_ks = ksV;
            {
                Gemm g;  // Q = Zf_j Zb^T (split K): A = ZfT columns jB.., B = ZbT, both MN-major
                g.M = g.N = B;
                g.a_mn = true;
                g.b_mn = true;
                g.seg[0].A = Operand{ZfAh, ZfAl, m, n, n};
                g.seg[0].a_col0 = j * B;
                g.seg[0].B = Operand{ZbTh, ZbTl, m, B, B};
                g.seg[0].K = m;
                g.partial = Qp;
                g.ksplit = ksQ;
                LB_GEMM(g, sa, "lb_q");
                q_ks = g.ksplit;
            }
            ++nl;
            q_sum_kernel<<<(int)((bb + 255) / 256), 256, 0, sa>>>(Qp, q_ks, (int64_t)bb, Qs);
            ++nl;
            s_from_q_kernel<<<dim3(B / 32, B / 32), dim3(32, 8), 0, sa>>>(Qs, B, Sh, Sl);
            {
                Gemm g;  // dV_j partials = -2 (Zb A_j + Zf_j G) + S V_j   (S = -4 K'^T pre-scaled by -1/2)
                g.M = B;
                g.N = d;
                g.nseg = 3;
                g.a_mn = true;  // every A here is stored K x M: ZbT, ZfT, S^T
                g.b_mn = true;
                g.seg[0].A = Operand{ZbTh, ZbTl, m, B, B};
                g.seg[0].B = Operand{Sth[j], Stl[j], m, d, d};
                g.seg[0].K = m;
                g.seg[1].A = Operand{ZfAh, ZfAl, m, n, n};
                g.seg[1].a_col0 = j * B;
                g.seg[1].B = Operand{Gh[cur], Gl[cur], m, d, d};
                g.seg[1].K = m;
                g.seg[2].A = Operand{Sh, Sl, B, B, B};  // S^T
                g.seg[2].B = Operand{Vh, Vl, n, d, d};  // V_j rows: K x N, N contiguous
                g.seg[2].b_row0 = j * B;
                g.seg[2].K = B;
                g.alpha = -2.f;
                g.partial = dVp;
                g.ksplit = ksV;
                LB_GEMM(g, sa, "lb_dv");
                v_ks = g.ksplit;
            }
            ++nl;
            dv_reduce_kernel<<<grid_for((int64_t)B * d), 256, 0, sa>>>(dVp, v_ks, B, d, D.n - j * B, D.d,
                                                                       dV + (size_t)j * B * lddv, lddv);
            if (two) LBTRY(cudaEventRecord(st->ev[12 + cur], sa));
            if (nt && nt->count > 0) {  // last block of its bucket: rows up to here are final
                const int nbk = std::min(nt->count, nb);
                const int bk = (int)((int64_t)j * nbk / nb);
                if (j + 1 == nb || (int)((int64_t)(j + 1) * nbk / nb) != bk) {
                    LBTRY(cudaEventRecord(nt->ev[bk], sa));
                    nt->row_end[bk] = std::min<int64_t>(D.n, (int64_t)(j + 1) * B);
                    nt->used = bk + 1;
                }
            }
        }
        if (j < nb - 1 || dX) {  // the last update only produces dX
            // block j-2's dV read the G / Zb buffers this update and the next
            // K1 overwrite
            if (two && j >= 2) LBTRY(cudaStreamWaitEvent(s, st->ev[12 + (j - 2) % 3], 0));
            Gemm g;  // G <- G - 2 ZbT VT_j^T
            g.split_scratch = b.ksc;
            g.split_scratch_floats = b.ksc_n;
            g.M = m;
            g.N = d;
            g.seg[0].A = Operand{ZbTh, ZbTl, m, B, B};
            g.seg[0].B = Operand{VTh, VTl, d, n, n};
            g.seg[0].b_col0 = j * B;
            g.seg[0].K = B;
            g.alpha = -2.f;
            g.beta = 1.f;
            g.c_hi = Gh[cur];
            g.c_single = true;
            g.ldc = d;
            g.d_hi = Gh[nxt];
            g.d_lo = Gl[nxt];
            g.lds = d;
            g.split_trunc = true;
            if (j == nb - 1 && !pad) {  // dX only: no later block reads the split gradient
                g.d_f32 = dX;
                g.ldd = lddx;
                g.d_hi = g.d_lo = nullptr;
            }
            LB_GEMM(g, s, "lb_k4_update");
            if (j == nb - 1 && pad && dX)  // hi of the trunc split is the gradient itself
                LBTRY(cudaMemcpy2DAsync(dX, lddx * sizeof(float), Gh[nxt], (size_t)d * sizeof(float),
                                        (size_t)D.d * sizeof(float), D.m, cudaMemcpyDeviceToDevice, s));
        }
    }
    if (two) LBTRY(cudaStreamWaitEvent(s, st->ev[12 + (nb - 1) % 3], 0));  // join: dV complete
    if (nlaunch) *nlaunch = nl;
    return cudaGetLastError();
}

cudaError_t forward_backward(const float* V, int64_t ldv, int d, int n, const float* X, int64_t ldx, const float* G,
                             int64_t ldg, int m, float* Y, int64_t ldy, float* dX, int64_t lddx, float* dV,
                             int64_t lddv, float* ws, ErrWord* err, cudaStream_t s, int num_sms, int* nlaunch,
                             Timer* tm, const Streams* st, DvNotify* nt) {
    int n1 = 0, n2 = 0;
    bool k1_pre = false;
    cudaError_t e = forward(V, ldv, d, n, X, ldx, m, Y, ldy, ws, err, s, num_sms, &n1, tm, st, G, ldg, &k1_pre);
    if (e == cudaSuccess)
        e = backward(d, n, m, G, ldg, dX, lddx, dV, lddv, ws, s, num_sms, &n2, tm, st, true, nt, k1_pre);
    if (nlaunch) *nlaunch = n1 + n2;
    return e;
}
#undef LBTRY
#undef LB_GEMM
#undef LB_ALIASES

}  // namespace lb
}  // namespace fasthb
