/*
 * fasth_b200 — C ABI of the B200-native FastH path (arXiv 2009.13977).
 *
 * This is the drop-in boundary for the reference's header-only C++ API in
 * /root/reference/proj/include/fasth/.  Each entry point below names the
 * reference function it replaces (file:line).  The C++ mirror of the
 * reference API (same names, types and exceptions) is include/fasth_b200.hpp,
 * a header-only layer over these functions.
 *
 * Conventions
 *   - All float* arguments are DEVICE pointers (except the *_host entry).
 *   - A Householder chain is a column-major d x n fp32 matrix V with leading
 *     dimension ldv >= d; column k is v_k, in chain order: applying the chain
 *     to X computes H_1 (H_2 (... (H_n X))) (householder.hpp:44-45).  This is
 *     also the payload order of the reference's OSVD checkpoint
 *     (svd_layer.hpp:250-251).
 *   - Activations X, Y, G, dX are column-major d x m fp32 (sample-contiguous,
 *     so batch shards are contiguous column ranges).
 *   - Gradients of a chain, dV, come back column-major d x n (column k is
 *     dL/dv_k), summed over the batch as in Eq. (5) (householder.hpp:145-147).
 *   - block_width is the reference's b / --k; it is clamped to [1, n] exactly
 *     like fasth_forward (fasth.hpp:52).
 *   - Calls are asynchronous on the context's stream.  In FASTH_CHECK_SYNC
 *     mode (the default) every call that can raise a data-dependent error
 *     (degenerate vector, singular sigma, Cayley pole, non-finite input)
 *     synchronises once before returning so that the status matches the
 *     reference's exception; in FASTH_CHECK_DEFERRED mode such errors are
 *     latched on the device and reported by fasth_ctx_check().
 *   - No exceptions cross this boundary; the status maps 1:1 onto the
 *     reference's exception hierarchy (matrix.hpp:12-30).
 *
 * Build: paper_2009_13977_b200/lib/libfasth_b200.so (sm_100a).
 */
#ifndef FASTH_B200_H
#define FASTH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fasth_status {
    FASTH_OK = 0,
    FASTH_ERR_DIMENSION = 1,  /* fasth::DimensionError       (matrix.hpp:17) */
    FASTH_ERR_DEGENERATE = 2, /* fasth::DegenerateVectorError (matrix.hpp:22) */
    FASTH_ERR_SINGULAR = 3,   /* fasth::SingularMatrixError   (matrix.hpp:27) */
    FASTH_ERR_INVALID = 4,    /* fasth::Error                 (matrix.hpp:12) */
    FASTH_ERR_CUDA = 5,
    FASTH_ERR_NCCL = 6
} fasth_status;

typedef struct fasth_ctx_s* fasth_ctx;
typedef struct fasth_tape_s* fasth_tape;         /* TapeForward  (fasth.hpp:22-29)     */
typedef struct fasth_svd_tape_s* fasth_svd_tape; /* SvdTape      (svd_layer.hpp:83-86) */
typedef struct fasth_svd_plan_s* fasth_svd_plan; /* both legs' WY blocks, built ahead of a forward */

enum { FASTH_CHECK_SYNC = 0, FASTH_CHECK_DEFERRED = 1 };

/* Message of the last non-OK status returned on this host thread. */
const char* fasth_last_error(void);
int fasth_version(void);

/* Context: one per (device, stream).  stream == NULL -> the legacy default
 * stream.  Replaces the reference's process-global worker count
 * (parallel.hpp:12-30): parallelism here is the grid.  Every call runs on the
 * context's device whatever the calling thread's current device is. */
fasth_status fasth_ctx_create(int device, void* stream, fasth_ctx* out);
fasth_status fasth_ctx_destroy(fasth_ctx ctx);
/* Rebind the context to another stream.  The new stream is ordered after all
 * work already enqueued on the old one (one event), so pool buffers and tapes
 * are never touched by two streams at once. */
fasth_status fasth_ctx_set_stream(fasth_ctx ctx, void* stream);
fasth_status fasth_ctx_set_check(fasth_ctx ctx, int mode);
/* Synchronise the stream and report (then clear) latched device errors. */
fasth_status fasth_ctx_check(fasth_ctx ctx);
/* Number of CUDA kernels this context has launched so far. */
int64_t fasth_ctx_launch_count(fasth_ctx ctx);
/* Timing mode: bracket every kernel launch with CUDA events on the context
 * stream (for per-kernel roofline figures; off by default).  mode 1: events
 * per launch, read and freed by fasth_ctx_kernel_times; mode 2: the events
 * are kept (capture a CUDA graph in this mode, replay it, read the times
 * after each replay: no host gaps).  Changing the mode clears the times. */
fasth_status fasth_ctx_set_timing(fasth_ctx ctx, int mode);
/* Accumulated per-kernel device time as text lines "name total_ms launches".
 * Returns the length written (truncated to buflen), -1 on bad arguments. */
int fasth_ctx_kernel_times(fasth_ctx ctx, char* buf, int buflen);
/* Release cached device memory held by the context's pool. */
fasth_status fasth_ctx_trim(fasth_ctx ctx);
/* dV row buckets for batch-sharded data parallelism (no reference
 * counterpart: the reference is single-process).  `events` are
 * caller-owned cudaEvent_t handles (count 0 turns the feature off).  Every
 * later fasth_backward / fasth_forward_backward that writes dV records
 * events[k] once dV rows [row_end[k-1], row_end[k]) are final, on the stream
 * that wrote them: the large-batch path after each group of its WY blocks
 * (so an all-reduce of those rows overlaps the rest of the backward), the
 * chain paths once after the whole dV.  fasth_ctx_dv_buckets copies up to
 * `max` row_end values of the last call and returns the bucket count (0: no
 * events recorded; -1: bad arguments).  Bucket bounds are known when the
 * call returns (before the device work completes).  The SVD layer, the
 * host-buffer entry and the tuner compute dV into temporaries or host memory
 * and record no buckets. */
fasth_status fasth_ctx_set_dv_events(fasth_ctx ctx, void* const* events, int count);
int fasth_ctx_dv_buckets(fasth_ctx ctx, int64_t* row_end, int max);

/* Device buffers from the context's pool and stream-ordered copies, so host
 * code (the C++ mirror, language bindings) needs no CUDA headers.
 * fasth_copy kinds: 0 host->device, 1 device->host, 2 device->device.
 * Copies are asynchronous on the context stream; fasth_ctx_synchronize waits. */
fasth_status fasth_device_alloc(fasth_ctx ctx, int64_t bytes, void** out);
fasth_status fasth_device_free(fasth_ctx ctx, void* ptr);
fasth_status fasth_copy(fasth_ctx ctx, void* dst, const void* src, int64_t bytes, int kind);
fasth_status fasth_ctx_synchronize(fasth_ctx ctx);

/* ---- FastH ---------------------------------------------------------------
 * fasth_forward  replaces  TapeForward fasth_forward(const HouseholderChain&,
 *                          const Matrix& X, size_t block_width)   fasth.hpp:40
 *   Y = H_1 ... H_n X.  tape may be NULL (forward only, nothing recorded);
 *   otherwise *tape receives the record backward needs (the compacted WY
 *   blocks and per-block activations).  The tape does not reference V after
 *   this call returns.  d >= 1, n >= 0, m >= 0.
 * fasth_backward replaces  BackwardResult fasth_backward(const TapeForward&,
 *                          const Matrix& grad_output)              fasth.hpp:69
 *   dX = (H_1 ... H_n)^T G and dV (d x n).  dV may be NULL (dX only).
 *   A tape may be used for several backward calls. */
fasth_status fasth_forward(fasth_ctx ctx, const float* V, int64_t ldv, int d, int n,
                           const float* X, int64_t ldx, int m, int block_width, float* Y,
                           int64_t ldy, fasth_tape* tape);
fasth_status fasth_backward(fasth_ctx ctx, fasth_tape tape, const float* G, int64_t ldg,
                            float* dX, int64_t lddx, float* dV, int64_t lddv);
fasth_status fasth_tape_destroy(fasth_tape tape);
/* Shape of a tape: any pointer may be NULL. q = number of WY blocks. */
fasth_status fasth_tape_info(fasth_tape tape, int* d, int* n, int* m, int* block_width, int* q);

/* The reference's call pair fasth_forward + fasth_backward (fasth.hpp:40, :69)
 * as one call, for callers that hold the output gradient G when they start —
 * the reference benchmark's op=mul step (bench.hpp:147-151: forward, then
 * backward with a pre-drawn G).  Same results as the two calls; the forward
 * and backward sweeps are independent once the WY blocks exist, so they run
 * concurrently in one launch.  Y, dX: d x m; dV: d x n (may be NULL). */
fasth_status fasth_forward_backward(fasth_ctx ctx, const float* V, int64_t ldv, int d, int n,
                                    const float* X, int64_t ldx, const float* G, int64_t ldg,
                                    int m, int block_width, float* Y, int64_t ldy, float* dX,
                                    int64_t lddx, float* dV, int64_t lddv);

/* Host-buffer form of the reference's call pair fasth_forward + fasth_backward
 * (fasth.hpp:40, :69): all pointers are HOST memory (pinned for full copy
 * bandwidth), column-major with leading dimension d.  Copies in, runs, copies
 * out and synchronises. */
fasth_status fasth_forward_backward_host(fasth_ctx ctx, const float* V, int d, int n,
                                         const float* X, const float* G, int m, int block_width,
                                         float* Y, float* dX, float* dV);

/* ---- WY internals (wy.hpp:56-170, public in the reference) ----------------
 * The compact WY form in the reference's own layout: for a block of b
 * vectors (column-major d x b, column j = v_j, chain order)
 *   I - 2 W Y^T = H_1 ... H_b,  Y[:, j] = v_j / ||v_j||,
 *   W[:, j] = H_1 ... H_{j-1} Y[:, j]             (wy.hpp:85-96)
 * W and Y are column-major d x b.  The chain sweeps do not use this form
 * (they run the UT form of the raw vectors); these entries serve callers of
 * the reference's WY functions and TapeForward::compacted. */
/* wy_compact (wy.hpp:56): b >= 1 vectors -> (W, Y); FASTH_ERR_INVALID for
 * b == 0 (wy.hpp:58-59), FASTH_ERR_DEGENERATE for ||v||^2 <= 1e-30. */
fasth_status fasth_wy_compact(fasth_ctx ctx, const float* V, int64_t ldv, int d, int b, float* W,
                              int64_t ldw, float* Y, int64_t ldy);
/* compact_chain (wy.hpp:151): the chain (d x n) partitioned into
 * ceil(n / block_width) consecutive blocks (the last ragged), each compacted;
 * block i's W and Y are columns [i bw, i bw + w_i) of the d x n W and Y.
 * FASTH_ERR_INVALID for block_width outside [1, n] (wy.hpp:153-155). */
fasth_status fasth_compact_chain(fasth_ctx ctx, const float* V, int64_t ldv, int d, int n, int block_width,
                                 float* W, int64_t ldw, float* Y, int64_t ldy);
/* wy_apply (wy.hpp:104): out = X - 2 W (Y^T X), X and out d x m (out may be X). */
fasth_status fasth_wy_apply(fasth_ctx ctx, const float* W, int64_t ldw, const float* Y, int64_t ldy, int d,
                            int b, const float* X, int64_t ldx, int m, float* out, int64_t ldo);
/* wy_apply_transpose (wy.hpp:137): out = X - 2 Y (W^T X). */
fasth_status fasth_wy_apply_transpose(fasth_ctx ctx, const float* W, int64_t ldw, const float* Y, int64_t ldy,
                                      int d, int b, const float* X, int64_t ldx, int m, float* out,
                                      int64_t ldo);

/* ---- SVD-reparameterised layer W = U Sigma V^T ---------------------------
 * SvdParam (svd_layer.hpp:25-72): U chain of nu vectors in dimension out_dim,
 * V chain of nv vectors in dimension in_dim, sigma of min(out_dim, in_dim). */
typedef struct fasth_svd_param {
    int out_dim, in_dim, nu, nv;
    const float* U; /* out_dim x nu, column-major */
    int64_t ldu;
    const float* V; /* in_dim x nv, column-major */
    int64_t ldv;
    const float* sigma; /* min(out_dim, in_dim) */
} fasth_svd_param;

/* svd_forward  (svd_layer.hpp:106): Y = U (Sigma (V^T X)), X in_dim x m.
 * The tape keeps T1 = V^T X and both legs' records; it reads p->sigma again
 * in backward, so sigma must stay valid until then. */
fasth_status fasth_svd_forward(fasth_ctx ctx, const fasth_svd_param* p, const float* X,
                               int64_t ldx, int m, int block_width, float* Y, int64_t ldy,
                               fasth_svd_tape* tape);
/* svd_backward (svd_layer.hpp:122): dX (in_dim x m), dU (out_dim x nu),
 * dV (in_dim x nv, chain order), dsigma (min dim).  Any output may be NULL. */
fasth_status fasth_svd_backward(fasth_ctx ctx, const fasth_svd_param* p, fasth_svd_tape tape,
                                const float* G, int64_t ldg, float* dX, int64_t lddx, float* dU,
                                int64_t lddu, float* dV, int64_t lddv, float* dsigma);
fasth_status fasth_svd_tape_destroy(fasth_svd_tape tape);
/* Build a layer's WY blocks ahead of its forward (the blocks depend only on
 * U and V): with on_side_stream != 0 the builds run on the context's side
 * stream, so a training loop can prepare layer k+1 while layer k sweeps.  A
 * plan is single use: fasth_svd_forward_planned consumes it (same m and
 * block width); U and V must not change in between.  Destroy unused plans. */
fasth_status fasth_svd_plan_create(fasth_ctx ctx, const fasth_svd_param* p, int m, int block_width,
                                   int on_side_stream, fasth_svd_plan* out);
fasth_status fasth_svd_plan_destroy(fasth_svd_plan plan);
/* svd_forward (svd_layer.hpp:106) on a prepared plan (consumed). */
fasth_status fasth_svd_forward_planned(fasth_ctx ctx, const fasth_svd_param* p, fasth_svd_plan plan,
                                       const float* X, int64_t ldx, int m, int block_width, float* Y,
                                       int64_t ldy, fasth_svd_tape* tape);
/* svd_forward + svd_backward in one call for a caller holding grad_output up
 * front (the reference benchmark's layer step, bench.hpp:166-209): the four
 * chain sweeps run as two paired launches.  Same outputs as the two calls;
 * square layers (out_dim == in_dim, nu == nv) take the paired path. */
fasth_status fasth_svd_forward_backward(fasth_ctx ctx, const fasth_svd_param* p, const float* X,
                                        int64_t ldx, const float* G, int64_t ldg, int m, int block_width,
                                        float* Y, int64_t ldy, float* dX, int64_t lddx, float* dU,
                                        int64_t lddu, float* dV, int64_t lddv, float* dsigma);

/* svd_step (svd_layer.hpp:158) fused with clamp_sigma (svd_layer.hpp:196)
 * when clamp_eps is in [0, 1) (-1: no clamp; any other value is rejected):
 * v <- v - eta dv, sigma <- sigma - eta dsigma.
 * Outputs may alias the inputs (in-place update).  A vector whose updated
 * ||v||^2 <= 1e-30 raises FASTH_ERR_DEGENERATE naming the chain and index
 * (svd_layer.hpp:174-179); the outputs are then unspecified. */
fasth_status fasth_svd_step(fasth_ctx ctx, const fasth_svd_param* p, const float* dU,
                            int64_t lddu, const float* dV, int64_t lddv, const float* dsigma,
                            float eta, float clamp_eps, float* U_out, int64_t ldou,
                            float* V_out, int64_t ldov, float* sigma_out);
/* clamp_sigma (svd_layer.hpp:196-202); epsilon in [0, 1). */
fasth_status fasth_clamp_sigma(fasth_ctx ctx, const float* sigma, int k, float epsilon,
                               float* sigma_out);

/* Sigma-ops (matops.hpp).  Square parameters only.
 *   apply_inverse      W^{-1} X = V Sigma^{-1} U^T X          matops.hpp:69
 *   apply_exponential  e^W X = U e^Sigma U^T X   (nv == 0)    matops.hpp:98
 *   apply_cayley       (I-W)(I+W)^{-1} X         (nv == 0)    matops.hpp:107
 *   log_abs_det        sum ln|sigma_i|                         matops.hpp:57 */
fasth_status fasth_apply_inverse(fasth_ctx ctx, const fasth_svd_param* p, const float* X,
                                 int64_t ldx, int m, int block_width, float* Y, int64_t ldy);
fasth_status fasth_apply_exponential(fasth_ctx ctx, const fasth_svd_param* p, const float* X,
                                     int64_t ldx, int m, int block_width, float* Y, int64_t ldy);
fasth_status fasth_apply_cayley(fasth_ctx ctx, const fasth_svd_param* p, const float* X,
                                int64_t ldx, int m, int block_width, float* Y, int64_t ldy);
fasth_status fasth_log_abs_det(fasth_ctx ctx, const fasth_svd_param* p, double* out);
/* apply_pseudo_inverse (matops.hpp:158): Y = V Sigma^+ U^T X, rectangular
 * parameters allowed: X is out_dim x m, Y in_dim x m; Sigma^+ reciprocates
 * entries with |sigma| > tol and zeroes the rest.  FASTH_ERR_INVALID for
 * tol < 0. */
fasth_status fasth_apply_pseudo_inverse(fasth_ctx ctx, const fasth_svd_param* p, const float* X, int64_t ldx,
                                        int m, double tol, int block_width, float* Y, int64_t ldy);

/* ---- OSVD checkpoints (svd_layer.hpp:204-290) -------------------------------
 * The reference's flat little-endian format: "OSVD", version u32 (= 1),
 * out_dim, in_dim, nU, nV (u32), then the U vectors, the V vectors (each
 * d f64 values, chain order) and sigma (min(out_dim, in_dim) f64).
 * fasth_svd_file_info  reads the header (no device work).
 * fasth_svd_load       replaces load_svd_param_file (svd_layer.hpp:282): U, V
 *   (device, column-major, column k = vector k) and sigma (device) receive the
 *   payload rounded to fp32; same errors as the reference (bad magic, version,
 *   truncation -> FASTH_ERR_INVALID; a vector with ||v||^2 <= 1e-30 ->
 *   FASTH_ERR_DEGENERATE, householder.hpp:28).
 * fasth_svd_save       replaces save_svd_param_file (svd_layer.hpp:276): the
 *   device parameter widened to f64.  save(load(f)) reproduces f bit for bit
 *   whenever f holds fp32-representable values (files this library wrote). */
fasth_status fasth_svd_file_info(const char* path, int* out_dim, int* in_dim, int* nu, int* nv);
fasth_status fasth_svd_load(fasth_ctx ctx, const char* path, float* U, int64_t ldu, float* V,
                            int64_t ldv, float* sigma);
fasth_status fasth_svd_save(fasth_ctx ctx, const fasth_svd_param* p, const char* path);

/* ---- block width (fasth.hpp:147-196, tune_block_width) ----------------------
 * timed = 0: the reference's analytic choice round(sqrt(d)).  timed != 0:
 * fasth_forward_backward on a seeded synthetic chain for every candidate in
 * {2, ..., 2 ceil(sqrt(d))} plus m (when m <= d), timed on the device with
 * CUDA events; the fastest is cached per (d, m) for the process. */
fasth_status fasth_tune_block_width(fasth_ctx ctx, int d, int m, int timed, uint64_t seed, int* out);

#ifdef __cplusplus
}
#endif

#endif /* FASTH_B200_H */
