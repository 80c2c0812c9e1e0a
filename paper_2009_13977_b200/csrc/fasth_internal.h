// Internal (non-ABI) declarations shared by the FastH CUDA translation units.
//
// Device layout of one compacted chain ("plan"), built once per call from the
// caller's column-major V (d x n, column k = v_k):
//
//   Vbl [q][d_pad][BS]  f32   block i holds v_{i*bi .. i*bi+w_i-1} (chain
//                             order, or reversed chain when plan.reversed),
//                             row-major so that the rows a cluster CTA owns
//                             are one contiguous bulk copy; zero padded rows
//                             (d..d_pad) and columns (w_i..BS).
//   Tt  [q][BS][BS]     f32   T~_i = (diag(V_i^T V_i) + 2 striu(V_i^T V_i))^{-1},
//                             upper triangular, so that the block product is
//                             P_i = H.. H.. = I - 2 V_i T~_i V_i^T
//                             (the UT form of wy.hpp:50-55's W,Y: W = V T~ D,
//                             Y = V D^{-1}).
//
// Per-block tapes written by the sweeps (ngroups = ceil(m / WC)):
//   tape [q][ngroups][d_pad][WC]  forward: A_i (activations[i], fasth.hpp:28)
//                                 backward: dA[i] (fasth.hpp:82-86)
//   zhat [q][BS][m]               forward: Z'f_i = T~_i V_i^T A_{i+1}
//                                 backward: Z'b_i = T~_i^T V_i^T dA[i]
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fasthb {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize [, NonPortableClusterSizeAllowed])
// once per (device, kernel) and size: function attributes are per device, so
// a process driving several GPUs must configure each one (attr.cpp).
cudaError_t ensure_smem(const void* kernel, size_t bytes, bool nonportable_cluster = false);

constexpr int kThreads = 256;
constexpr int kMaxBS = 64;

struct ErrWord {  // host-mapped pinned memory, written by kernels
    int flags;    // bit0 degenerate ||v||^2 <= 1e-30, bit1 non-finite
    int index;    // smallest offending chain index (atomicMin)
    int chain;    // which chain (caller tag) raised it
    int pad;
};

enum : int { kErrDegenerate = 1, kErrNonFinite = 2, kErrSingular = 4, kErrPole = 8 };

struct Plan {
    int d = 0, n = 0, b = 0;  // b: internal block width (<= kMaxBS)
    int q = 0, BS = 0, d_pad = 0;
    int reversed = 0;
    int tag = 0;  // error-report tag (0 = U / plain chain, 1 = V)
    float* Vbl = nullptr;        // [q][d_pad][BS+4]  raw block rows (gradient kernel)
    float* Tt = nullptr;         // [q][BS][BS]     T~ (diagnostics / tests)
    float* Pf = nullptr;         // packed forward stages  [q][CB][stage_floats] (step order)
    float* Pb = nullptr;         // packed backward stages [q][CB][stage_floats]
    int CB = 8;                  // build cluster size (CTAs per block)
    long long* trace = nullptr;  // optional build phase stamps (FASTH_TRACE)
    // pipelined step (fasth_forward_backward): per-block readiness counters,
    // +1 per build CTA once its rows of block i's packed stages are stored;
    // nbuild > 0 runs the builder persistent on nbuild clusters (blocks in
    // the order the two sweeps need them).  nullptr / 0: plain launch.
    unsigned* ready = nullptr;
    int nbuild = 0;
    // streamed host step (build4): V's columns land while the builder runs;
    // block k is in once upc[k] >= upc_target (host_io.cu upload_kernel)
    const unsigned* upc = nullptr;
    unsigned upc_target = 0;
    // plain launch: build blocks [blk_lo, blk_hi) only (blk_hi < 0: all q)
    int blk_lo = 0, blk_hi = -1;
    // column-major activations the next kernel reads first (X, G): the
    // builder prefetches them into L2 while it works (build4)
    const float* pf[2] = {nullptr, nullptr};
    int64_t pf_ld[2] = {0, 0};
    int pf_rows = 0, pf_cols = 0;
};

// ---- packed chain stages (chain_v2.cu) ------------------------------------
// Everything CTA r of a chain cluster needs for one step t of a sweep, one
// contiguous run so that ONE bulk copy lands it:
//   [ W rows (RC x LDW) | V rows (RC x LDV) | S (BS x LDV) ]
// of block i(t) (forward: i = q-1-t, Wf / Sf; backward: i = t, Wb / Sb), rows
// [r*RC, (r+1)*RC).  Columns are permuted into mma.sync fragment order so a
// lane's operands are contiguous 16-byte vectors:
//   W: pos = g*2MT + mt*2 + h  for column c = 16 mt + 8 h + g   (A operand of W^T X)
//   V, S: pos = tq*2KB + ks*2 + h  for column c = 8 ks + 4 h + tq (A operand of V Z, S Z)
// with MT = BS/16, KB = BS/8.  Pitches: LDW = BS+8 (== 8 mod 32), LDV = BS+4.
__host__ __device__ constexpr int stage_ldw(int BS) { return BS + 8; }
__host__ __device__ constexpr int stage_ldv(int BS) { return BS + 4; }
__host__ __device__ constexpr size_t stage_floats(int RC, int BS) {
    return (size_t)RC * stage_ldw(BS) + (size_t)RC * stage_ldv(BS) + (size_t)BS * stage_ldv(BS);
}
__host__ __device__ inline int perm_w_bs(int c, int BS) {
    const int MT = BS / 16;
    return (c & 7) * 2 * MT + (c >> 4) * 2 + ((c >> 3) & 1);
}
__host__ __device__ inline int perm_v_bs(int c, int BS) {
    const int KB = BS / 8;
    return (c & 3) * 2 * KB + (c >> 3) * 2 + ((c >> 2) & 1);
}

struct SweepDirV2 {
    const float* stage;   // [q][C][stage_floats] packed, step order
    const float* x_in;    // column-major, rows < n_valid are read
    int64_t ldx;
    int n_valid;
    const float* scale;   // optional per-row scale applied on load (Sigma)
    float* x_out;         // column-major d x m
    int64_t ldo;
    float* tape;          // optional [q][ngroups][d_pad][WC] (header comment)
    float* zhat;          // optional [q][BS][m]
    int forward;
};

struct SweepV2Args {
    SweepDirV2 dir[2];    // cluster c runs dir[c / ngroups] on column group c % ngroups
    int ndir;             // 1, or 2 (forward and backward sweeps in one launch)
    int d, d_pad, m, q, BS, C, nstg, ngroups;
    long long* trace;     // optional phase timestamps [CTA][q+1][16]
    long long* wtrace;    // optional per-warp barrier stamps [CTA][q][12][4]
    // pipelined step: wait for ready[i] >= C before streaming block i's
    // stage; signal done[i] += 1 per CTA once block i's tape / Z' rows are
    // stored (nullptr: plain launch, no waits, no signals)
    const unsigned* ready;
    unsigned* done;
    int sig_from;         // done counting starts at this step (earlier steps published with it)
    int pub_ns;           // publish warp's back-off between polls of the tape warp's count
    // streamed host step: X / G land while the kernel runs (wait for
    // xg_ready >= xg_target before loading them; the last CTA resets both)
    unsigned* xg_ready;
    unsigned xg_target;
    unsigned* xg_seen;
    int x_wait;           // X / G are the previous grid's outputs: the row warps wait for it
                          // before loading them (so the launch may still start early)
    int late_trigger;     // release programmatic dependents only once the previous grid
                          // (the builder) is complete, not at entry
    int pdl;              // launched as a programmatic dependent of the builder
};


struct DvArgs {
    const float* Vbl;
    int d, d_pad, n, b, q, BS, m, WC, ngroups;
    int reversed;
    const float* tapeA;   // [q][ngroups][d_pad][WC]
    const float* tapeG;
    const float* zf;      // [q][BS][m]
    const float* zb;
    float* dV;            // column-major d x n
    int64_t lddv;
    // pipelined step: wait for done[i] >= done_target, then the last CTA of
    // block i resets ready[i], done[i], dvcnt[i] (nullptr: plain launch)
    unsigned* ready;
    unsigned* done;
    unsigned* dvcnt;
    unsigned done_target;
    unsigned* upc;  // streamed host step: block i's upload count, reset with the others
    size_t min_smem;  // pipelined: dynamic shared memory to request at least
    long long* trace;  // optional per-CTA global-timer stamps [block][slab][6] (FASTH_STEPTRACE)
    int order;  // blockIdx.y -> block: 0 identity (backward sweep order), 1 middle-out (fused fwd+bwd)
    int poll_ns;  // pipelined: back-off between polls of the block's counter
    int pdl;  // launched as a programmatic dependent of the sweep (griddepcontrol.wait first)
    int v_pre;  // Vbl is complete at launch (the sweep released its dependents after the
                // builder): V fragments load before the wait on the sweep
    int trigger;  // release programmatic dependents at entry (independent kernels after it)
    int nowait;   // launched behind an independent kernel: its inputs are complete, no wait
};

// wy_build2.cu (packed stages for chain_v2.cu)
cudaError_t launch_build2(const Plan& p, const float* V, int64_t ldv, ErrWord* err, cudaStream_t s);
size_t build2_smem_bytes(int BS, int RB);
// wy_build4.cu: same outputs, one cluster per block without cluster barriers
// on the path (plain launches only: no ready counters / persistent tickets)
cudaError_t launch_build4(const Plan& p, const float* V, int64_t ldv, ErrWord* err, cudaStream_t s);
size_t build4_smem_bytes(int BS, int RB, int C);
// chain_v2.cu
struct SweepGeom {
    int C = 0, RC = 16, d_pad = 16, WC = 8;  // C == 0: no geometry fits
};
SweepGeom pick_geometry(int d, int m, int BS, int num_sms, bool fused);  // fused: fwd | bwd in one launch
int sweep2_nstg(int C, int BS, int d_pad);  // 0 = geometry not supported by the v2 kernel
size_t sweep2_smem_bytes(int C, int BS, int d_pad, int nstg, bool sig);  // sig: tape-warp variant
cudaError_t launch_sweep2(const SweepV2Args& a, cudaStream_t s);
// host_io.cu: streaming copy kernel (either side may be a pinned-host mapping)
cudaError_t launch_stream_copy(const float* src, float* dst, int64_t n, int num_sms, cudaStream_t s);
// streamed upload of the host step (host_io.cu): X, G, then V's blocks
// outside-in, each unit counted per landed chunk (target ncb per counter
// entry: upc[k] per block, xg_cnt for X and G together 2 * ncb)
struct UploadArgs {
    const float4 *x_src, *g_src, *v_src;  // device views of the pinned inputs
    float4 *x_dst, *g_dst, *v_dst;
    int64_t x4, v4, blk4;  // float4 counts: X (= G), V, one block of columns
    int q, ncb;
    unsigned* upc;     // [q]
    unsigned* xg_cnt;  // X and G
};
cudaError_t launch_upload(const UploadArgs& u, int ctas, cudaStream_t s);
cudaError_t launch_stream_copy_n(const float* const* src, float* const* dst, const int64_t* n, int nseg, int num_sms,
                                 cudaStream_t s);
// wy_api.cu: the reference's WY internals (wy.hpp:56-170) in its own layout
// W, Y (column-major d x n, block z = columns [z bw, z bw + w_z)); scratch of
// wy_compact_scratch_doubles(n, bw) doubles; T of b * m doubles for wy_apply
// (out = X - 2 A (B^T X): wy_apply is A = W, B = Y; the transpose A = Y, B = W)
cudaError_t launch_wy_compact(const float* V, int64_t ldv, int d, int n, int bw, double* scratch, float* W,
                              int64_t ldw, float* Y, int64_t ldy, ErrWord* err, int tag, cudaStream_t s);
size_t wy_compact_scratch_doubles(int n, int bw);
cudaError_t launch_wy_apply(const float* A, int64_t lda, const float* Bm, int64_t ldb, int d, int b,
                            const float* X, int64_t ldx, int m, double* T, float* out, int64_t ldo, cudaStream_t s);
// chain_panel.cu (large batch: one CTA per 16-column panel, all rows)
bool panel_supported(int BS, int d_pad, int m);
cudaError_t launch_panel(const SweepV2Args& a, cudaStream_t s);
// dv2.cu (tapes with WC == 8)
cudaError_t launch_dv2(const DvArgs& a, cudaStream_t s);
// sigma_ops.cu
cudaError_t launch_scale_rows(const float* x, int64_t ldx, int n_valid, const float* scale,
                              int rows, int m, float* y, int64_t ldy, int mode,
                              cudaStream_t s);
cudaError_t launch_dsigma(const float* dT2, int64_t ld2, const float* T1, int64_t ld1, int k,
                          int m, float* dsigma, cudaStream_t s, bool pdl_nowait = false);
cudaError_t launch_step(const float* P, int64_t ldp, const float* dP, int64_t lddp, int dim,
                        int n, float eta, float* out, int64_t ldo, ErrWord* err, int tag,
                        cudaStream_t s);
cudaError_t launch_sigma_step(const float* sigma, const float* dsigma, int k, float eta,
                              float clamp_eps, float* out, cudaStream_t s);
cudaError_t launch_sigma_map(const float* sigma, int k, int kind, float* out, ErrWord* err,
                             cudaStream_t s, float tol = 0.f);
cudaError_t launch_logdet(const float* sigma, int k, double* out, ErrWord* err,
                          cudaStream_t s);

}  // namespace fasthb
