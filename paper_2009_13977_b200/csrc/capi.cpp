// Host side of the C ABI (include/fasth_b200.h): argument validation with the
// reference's error semantics, the device memory pool, WY plan construction
// and the launch sequence of each reference operation.  No compute happens
// here and there is no CPU fallback: every operation is a sequence of the
// sm_100a kernels in this directory, and the library fails loudly when no
// CUDA device is usable.
#include "fasth_b200.h"
#include "fasth_internal.h"
#include "lb.h"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

using namespace fasthb;

namespace {

thread_local std::string g_err;

fasth_status fail(fasth_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CU(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(FASTH_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                           \
    } while (0)

#define TRY(call)                          \
    do {                                   \
        fasth_status s_ = (call);          \
        if (s_ != FASTH_OK) return s_;     \
    } while (0)

constexpr int kMaxPipeQ = 4096;  // WY blocks the pipelined step supports
constexpr int kCounterWords = 4 * kMaxPipeQ + 64;
constexpr int kUploadChunks = 4;  // chunks per upload unit (streamed host step)

size_t size_class(size_t bytes) {
    size_t c = 512;
    while (c < bytes) c <<= 1;
    return c;
}

}  // namespace

// --------------------------------------------------------------------------
struct HostGraphKey {
    const void* p[6] = {};
    int d = 0, n = 0, m = 0, b = 0;
    bool operator==(const HostGraphKey& o) const {
        for (int i = 0; i < 6; ++i)
            if (p[i] != o.p[i]) return false;
        return d == o.d && n == o.n && m == o.m && b == o.b;
    }
};

struct fasth_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int check_mode = FASTH_CHECK_SYNC;
    int num_sms = 148;
    ErrWord* err_h = nullptr;  // host-mapped
    ErrWord* err_d = nullptr;
    unsigned* counters = nullptr;  // build tickets, self-resetting
    int counters_len = 0;
    double* logdet_d = nullptr;
    int64_t launches = 0;
    // FASTH_STEPTRACE=<path>: non-synchronising global-timer stamps of the
    // fused step's three kernels (builder, sweep, gradient; per CTA), written
    // in place by the kernels and dumped to <path>.bin at fasth_ctx_check
    // activations the next build's L2 prefetch covers (set by the entry, consumed by build_plan)
    const float* pf[2] = {nullptr, nullptr};
    int64_t pf_ld[2] = {0, 0};
    // the host-buffer step writes dV straight into the caller's pinned memory:
    // there the gradient kernel runs behind the sweep (PCIe writes overlap it)
    bool dv_pipe_pref = false;
    bool dv_v_pre = false;  // the last sweep launched released its dependents after the builder
    int dv_chain = 0;       // run_dv: 1 first / 2 later of independent kernels after a sweep
    bool geom_fused = false;  // new_tape: the chain runs as fused fwd | bwd launches
    // streamed host step: the upload the next build_plan launches (before its
    // builder), whether the tape geometry allows it to stream, and whether the
    // step in flight streams (consumed by the sweep and the gradient kernel)
    struct UploadReq {
        const float *v_src, *x_src, *g_src;
        float *v, *x, *g;
        int64_t nv, nx;
    } up{};
    bool up_pending = false, up_geom_ok = false, up_active = false;
    // streamed: the builder is launched after the sweep (the sweep's 80 CTAs
    // take their SMs first and wait per block; builders waiting for V's
    // columns would otherwise hold the SMs the sweep needs)
    bool build_deferred = false;
    Plan deferred_plan{};
    const float* deferred_V = nullptr;
    int64_t deferred_ldv = 0;
    unsigned* up_counts() { return counters + 3 * kMaxPipeQ; }      // [q] per block
    unsigned* up_xg() { return counters + 4 * kMaxPipeQ; }          // X and G
    unsigned* up_xg_seen() { return counters + 4 * kMaxPipeQ + 1; }  // sweep CTAs past it
    long long* step_trace = nullptr;
    int cur_m = 0;  // batch of the plan being built (step-trace sizing)
    size_t st_build = 0, st_sweep = 0, st_dv = 0, st_total = 0;
    int st_hdr[6] = {0, 0, 0, 0, 0, 0};  // q, C, build rows, sweep CTAs, dv CTAs, valid
    long long* step_trace_area(size_t build_n, size_t sweep_n, size_t dv_n) {
        const size_t tot = build_n + sweep_n + dv_n;
        if (tot > st_total) {
            if (step_trace) cudaFree(step_trace);
            if (cudaMalloc(&step_trace, tot * sizeof(long long)) != cudaSuccess) step_trace = nullptr, st_total = 0;
            else st_total = tot;
        }
        st_build = 0, st_sweep = build_n, st_dv = build_n + sweep_n;
        return step_trace;
    }
    void dump_step_trace() {
        const char* path = getenv("FASTH_STEPTRACE");
        if (!path || !step_trace || !st_hdr[5]) return;
        cudaStreamSynchronize(stream);
        std::vector<long long> h(st_total);
        cudaMemcpy(h.data(), step_trace, st_total * sizeof(long long), cudaMemcpyDeviceToHost);
        if (FILE* f = fopen((std::string(path) + ".bin").c_str(), "wb")) {
            fwrite(st_hdr, sizeof(int), 6, f);
            fwrite(h.data(), sizeof(long long), st_total, f);
            fclose(f);
        }
    }
    long long* build_trace = nullptr;  // FASTH_TRACE: pending builder stamps
    size_t build_trace_n = 0;
    int build_trace_rows = 0;
    void dump_build_trace(const char* prefix) {
        if (!build_trace) return;
        std::vector<long long> h(build_trace_n);
        cudaMemcpy(h.data(), build_trace, build_trace_n * sizeof(long long), cudaMemcpyDeviceToHost);
        cudaFree(build_trace);
        build_trace = nullptr;
        std::string path = std::string(prefix) + ".build.bin";
        if (FILE* f = fopen(path.c_str(), "wb")) {
            int hdr[2] = {build_trace_rows, 10};
            fwrite(hdr, sizeof(int), 2, f);
            fwrite(h.data(), sizeof(long long), build_trace_n, f);
            fclose(f);
        }
    }
    int last_chain = 0, last_index = -1;
    std::mutex mu;
    std::map<size_t, std::vector<void*>> free_list;
    std::map<void*, size_t> live;

    fasth_status alloc(size_t bytes, void** out) {
        const size_t c = size_class(bytes ? bytes : 1);
        std::lock_guard<std::mutex> lk(mu);
        auto& fl = free_list[c];
        if (!fl.empty()) {
            *out = fl.back();
            fl.pop_back();
        } else {
            cudaError_t e = cudaMalloc(out, c);
            if (e != cudaSuccess)
                return fail(FASTH_ERR_CUDA, "cudaMalloc(%zu): %s", c, cudaGetErrorString(e));
        }
        live[*out] = c;
        return FASTH_OK;
    }
    // fasth_forward_backward_host's cached CUDA graph: the whole host-buffer
    // step (copies, kernels, read-back) replayed with one launch while the
    // caller keeps passing the same buffers; buffers the captured sequence
    // released stay reserved for the graph until it is dropped
    // second stream + fork/join events of the large-batch step (lb.h Streams)
    fasthb::lb::Streams lb_st;
    const fasthb::lb::Streams* lb_streams() {
        if (const char* e = getenv("FASTH_LB_STREAMS"))
            if (atoi(e) == 0) return nullptr;
        if (!lb_st.aux) {
            if (cudaStreamCreateWithFlags(&lb_st.aux, cudaStreamNonBlocking) != cudaSuccess) {
                lb_st.aux = nullptr;
                cudaGetLastError();
                return nullptr;
            }
            for (auto& ev : lb_st.ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        }
        return &lb_st;
    }
    // the SVD layer's independent leg work (U-leg build during the V leg, the
    // U-leg gradient kernel during the V-leg backward) on the same side stream
    const fasthb::lb::Streams* svd_streams() {
        if (const char* e = getenv("FASTH_SVD_STREAMS"))
            if (atoi(e) == 0) return nullptr;
        return lb_streams();
    }
    // set around a launch that follows a cross-stream event wait: it must not
    // use programmatic dependent launch (see run_forward)
    bool after_stream_wait = false;
    // dV bucket events (fasth_ctx_set_dv_events): caller-owned cudaEvent_t
    std::vector<cudaEvent_t> dv_events;
    std::vector<int64_t> dv_row_end;
    int dv_used = 0;
    fasthb::lb::DvNotify* dv_notify(fasthb::lb::DvNotify& nt) {
        if (dv_events.empty()) return nullptr;
        nt.ev = dv_events.data();
        nt.count = (int)dv_events.size();
        nt.row_end = dv_row_end.data();
        nt.used = 0;
        return &nt;
    }
    // paths that finish dV in one piece: one bucket, recorded after the last
    // dV launch on the context stream
    fasth_status dv_notify_whole(int n) {
        if (dv_events.empty()) return FASTH_OK;
        cudaError_t e = cudaEventRecord(dv_events[0], stream);
        if (e != cudaSuccess) return fail(FASTH_ERR_CUDA, "dV event record: %s", cudaGetErrorString(e));
        dv_row_end[0] = n;
        dv_used = 1;
        return FASTH_OK;
    }
    bool capturing = false;
    std::vector<void*> graph_held;
    cudaGraphExec_t host_exec = nullptr;
    HostGraphKey host_key;
    std::vector<void*> host_bufs;
    int64_t host_launches = 0;
    cudaEvent_t switch_ev = nullptr;     // fasth_ctx_set_stream: old stream -> new stream ordering
    cudaStream_t host_stream = nullptr;  // host-buffer entry on the legacy stream (fasth_forward_backward_host)
    cudaEvent_t host_ev = nullptr;
    void drop_host_graph() {
        if (!host_exec && graph_held.empty() && host_bufs.empty()) return;
        cudaStreamSynchronize(stream);
        if (host_stream) cudaStreamSynchronize(host_stream);
        if (host_exec) cudaGraphExecDestroy(host_exec);
        host_exec = nullptr;
        std::vector<void*> held;
        held.swap(graph_held);
        for (void* q : held) release(q);
        for (void* q : host_bufs) release(q);
        host_bufs.clear();
        host_key = HostGraphKey{};
    }
    void release(void* p) {
        if (!p) return;
        if (capturing) {  // still referenced by the graph being captured
            graph_held.push_back(p);
            return;
        }
        std::lock_guard<std::mutex> lk(mu);
        auto it = live.find(p);
        if (it == live.end()) return;
        free_list[it->second].push_back(p);
        live.erase(it);
    }
    template <typename T>
    fasth_status alloc_n(size_t n, T** out) {
        void* p = nullptr;
        TRY(alloc(n * sizeof(T), &p));
        *out = static_cast<T*>(p);
        return FASTH_OK;
    }
    fasth_status ensure_counters(int q) {
        if (q <= counters_len) return FASTH_OK;
        if (counters) cudaFree(counters);
        const int len = std::max(q, 1024);
        CU(cudaMalloc(&counters, len * sizeof(unsigned)));
        CU(cudaMemset(counters, 0, len * sizeof(unsigned)));
        counters_len = len;
        return FASTH_OK;
    }
    // Launch bookkeeping: counts kernels and, in timing mode, brackets each
    // launch with CUDA events on the context stream (bench.py's per-kernel
    // roofline timing).
    int timing = 0;  // 0 off, 1 per launch, 2 persistent events (graph capture)
    struct Timed {
        std::string name;
        cudaEvent_t start, stop;
    };
    std::vector<Timed> pending;
    std::map<std::string, std::pair<double, int64_t>> kernel_ms;
    template <typename F>
    fasth_status timed(F&& launch, const char* what) {
        cudaEvent_t a = nullptr, b = nullptr;
        // under stream capture only an "external" record becomes an event
        // node that is timestamped at every replay
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (timing) cudaStreamIsCapturing(stream, &cap);
        const unsigned rflags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
        if (timing) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecordWithFlags(a, stream, rflags);
        }
        cudaError_t e = launch();
        if (timing) {
            cudaEventRecordWithFlags(b, stream, rflags);
            pending.push_back({what, a, b});
        }
        if (e != cudaSuccess)
            return fail(FASTH_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
        ++launches;
        return FASTH_OK;
    }
    void collect_timing() {
        for (auto& t : pending) {
            float ms = 0.f;
            if (cudaEventSynchronize(t.stop) == cudaSuccess &&
                cudaEventElapsedTime(&ms, t.start, t.stop) == cudaSuccess) {
                auto& acc = kernel_ms[t.name];
                acc.first += ms;
                acc.second += 1;
            }
            if (timing != 2) {
                cudaEventDestroy(t.start);
                cudaEventDestroy(t.stop);
            }
        }
        if (timing != 2) pending.clear();
    }
    // mode 2 keeps the events (they are nodes of a captured graph that is
    // replayed): each collect reads the last replay; release when done
    void release_timing_events() {
        for (auto& t : pending) {
            cudaEventDestroy(t.start);
            cudaEventDestroy(t.stop);
        }
        pending.clear();
    }
    // Report latched device errors (after a stream sync) and clear them.
    fasth_status harvest() {
        CU(cudaStreamSynchronize(stream));
        ErrWord w = *err_h;
        err_h->flags = 0;
        err_h->index = 0x7fffffff;
        err_h->chain = 0;
        if (!w.flags) return FASTH_OK;
        const char* chain = w.chain == 1 ? "V" : "U";
        last_chain = w.chain;
        last_index = w.index;
        if (w.flags & kErrNonFinite)
            return fail(FASTH_ERR_INVALID, "non-finite entry in chain %s vector %d", chain, w.index);
        if (w.flags & kErrDegenerate)
            return fail(FASTH_ERR_DEGENERATE,
                        "HouseholderVector: ||v||^2 below degeneracy threshold 1e-30 "
                        "(chain %s vector %d)",
                        chain, w.index);
        if (w.flags & kErrSingular) return fail(FASTH_ERR_SINGULAR, "zero singular value");
        if (w.flags & kErrPole) return fail(FASTH_ERR_INVALID, "apply_cayley: sigma = -1 pole");
        return fail(FASTH_ERR_INVALID, "device error flags 0x%x", w.flags);
    }
    fasth_status finish() { return check_mode == FASTH_CHECK_SYNC ? harvest() : FASTH_OK; }
};

struct fasth_tape_s {
    fasth_ctx ctx = nullptr;
    Plan plan;
    int m = 0, b_user = 0;
    int C = 0, WC = 0, ngroups = 0;
    int v2nstg = 0;  // stage ring depth of the packed-stage sweep (chain_v2.cu)
    bool pipelined = false;  // build -> sweep -> dv overlapped through block counters
    float* tapeA = nullptr;  // activations per block
    float* zf = nullptr;
    float* tapeG = nullptr;  // gradient per block (backward scratch)
    float* zb = nullptr;
    const float* scale = nullptr;  // Sigma-scaled input rows (SVD U leg)
    int n_valid = 0;
    float* lb_ws = nullptr;  // large-batch path (lb.h): workspace holding the forward stages
};

struct fasth_svd_plan_s {
    fasth_ctx ctx = nullptr;
    int out_dim = 0, in_dim = 0, m = 0, b = 0;
    fasth_tape u = nullptr, v = nullptr;  // built tapes (no activations yet)
    cudaEvent_t ready = nullptr;           // recorded on the side stream (nullptr: same stream)
    bool used = false;                     // single use: the forward takes the tapes
};

struct fasth_svd_tape_s {
    fasth_ctx ctx = nullptr;
    int out_dim = 0, in_dim = 0, m = 0, k = 0;
    fasth_tape v = nullptr;  // V^T leg (reversed V chain); null if nv == 0
    fasth_tape u = nullptr;  // U leg; null if nu == 0
    float* T1 = nullptr;     // V^T X, in_dim x m
};

// Every entry point runs on its context's device, whatever the calling
// thread's current device is, and restores the caller's device on return.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev < 0) return;
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        if (cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};
inline int dev_of(fasth_ctx c) { return c ? c->device : -1; }
inline int dev_of(fasth_tape t) { return t && t->ctx ? t->ctx->device : -1; }
inline int dev_of(fasth_svd_plan p) { return p && p->ctx ? p->ctx->device : -1; }
inline int dev_of(fasth_svd_tape t) { return t && t->ctx ? t->ctx->device : -1; }

// defined in the extern "C" block below (large-batch path selection)
extern "C" bool use_large_batch(int d, int n, int m);
extern "C" fasth_status lb_apply_chain(fasth_ctx c, const float* V, int64_t ldv, int d, int n, int reversed,
                                      const float* X, int64_t ldx, int n_valid, const float* scale, int m,
                                      float* Y, int64_t ldy);

namespace {

void free_plan(fasth_ctx c, Plan& p) {
    c->release(p.Vbl);
    c->release(p.Tt);
    c->release(p.Pf);
    c->release(p.Pb);
    p.Vbl = p.Tt = p.Pf = p.Pb = nullptr;
}

void free_tape(fasth_tape t) {
    if (!t) return;
    fasth_ctx c = t->ctx;
    free_plan(c, t->plan);
    c->release(t->tapeA);
    c->release(t->zf);
    c->release(t->tapeG);
    c->release(t->zb);
    c->release(t->lb_ws);
    delete t;
}

int next_pow2_min16(int x) {
    int p = 16;
    while (p < x) p <<= 1;
    return p;
}

// Internal block width: the reference's b clamped to [1, n] (fasth.hpp:52);
// wider blocks run as 64-wide (32-wide when d is large, to keep the chain
// kernel's shared-memory stages in budget) sub-blocks: the same product.
int internal_b(int d, int n, int b_user) {
    // FASTH_INTERNAL_BS: the chain kernels' block width regardless of the
    // caller's (the product does not depend on the blocking) — A/B knob
    if (const char* e = getenv("FASTH_INTERNAL_BS"))
        return std::max(1, std::min({atoi(e), kMaxBS, std::max(n, 1)}));
    const int b = std::min(std::max(b_user, 1), n);
    // at most 32 wide (64-wide blocks measured 2-3.5x slower at every d they
    // fit, d <= 512: the 64-wide sweep spills and its builder is build2),
    // 16-wide beyond d = 2048 (the stages and exchange slots no longer fit
    // shared memory); the same product either way.  FASTH_INTERNAL_BS=64
    // still reaches the 64-wide kernels.
    return std::min(b, d > 2048 ? 16 : 32);
}

// Build the compacted chain (Alg. 1 step 1) on the device, in the row
// padding d_pad the chain geometry asks for.
fasth_status build_plan(fasth_ctx c, const float* V, int64_t ldv, int d, int d_pad, int cb, int n,
                        int b_user, int reversed, int tag, bool* pipelined, Plan* out) {
    const bool dv_wanted = pipelined && *pipelined;
    Plan p;
    p.d = d;
    p.n = n;
    p.b = internal_b(d, n, b_user);
    p.BS = next_pow2_min16(p.b);
    p.q = (n + p.b - 1) / p.b;
    p.d_pad = d_pad;
    p.reversed = reversed;
    p.tag = tag;
    p.pf[0] = c->pf[0], p.pf[1] = c->pf[1], p.pf_ld[0] = c->pf_ld[0], p.pf_ld[1] = c->pf_ld[1];
    p.pf_rows = d, p.pf_cols = (c->pf[0] || c->pf[1]) ? c->cur_m : 0;
    c->pf[0] = c->pf[1] = nullptr;
    // Build cluster: the chain kernel's cluster size, so each build CTA owns
    // the same 16-row-multiple slab the chain CTAs do.
    p.CB = cb;
    if (build2_smem_bytes(p.BS, p.d_pad / p.CB) > 227 * 1024)
        return fail(FASTH_ERR_INVALID, "fasth: dimension %d too large for block width %d", d, p.b);
    TRY(c->alloc_n((size_t)p.q * p.d_pad * stage_ldv(p.BS), &p.Vbl));
    TRY(c->alloc_n((size_t)p.q * p.BS * p.BS, &p.Tt));
    const size_t sf = stage_floats(p.d_pad / p.CB, p.BS);
    TRY(c->alloc_n((size_t)p.q * p.CB * sf, &p.Pf));
    TRY(c->alloc_n((size_t)p.q * p.CB * sf, &p.Pb));
    if (pipelined && *pipelined) {
        // opt-in (FASTH_PIPELINE=1), profitable only once a block builds in
        // well under the sweep's duration (scripts/trace_report.py --timeline)
        *pipelined = p.q <= kMaxPipeQ && c->counters_len >= 3 * kMaxPipeQ && getenv("FASTH_PIPELINE") &&
                     !getenv("FASTH_NO_PIPELINE");
        if (*pipelined) {
            p.ready = c->counters;
            const char* nb = getenv("FASTH_BUILDERS");
            p.nbuild = nb ? std::max(1, atoi(nb)) : 12;
        }
    }
    {
        const char* prefix = getenv("FASTH_TRACE");
        const size_t ntr = (size_t)p.q * p.CB * 10;
        if (!prefix && getenv("FASTH_STEPTRACE")) {  // builder rows of the step trace (fused step)
            const size_t nsw = (size_t)2 * ((std::max(1, c->cur_m) + 7) / 8) * p.CB * (p.q + 1) * 16;
            const size_t ndv = (size_t)((p.d_pad + 63) / 64) * p.q * 6;
            if (long long* a = c->step_trace_area(ntr, nsw, ndv)) {
                p.trace = a + c->st_build;
                c->st_hdr[0] = p.q, c->st_hdr[1] = p.CB, c->st_hdr[2] = p.q * p.CB;
                c->st_hdr[3] = c->st_hdr[4] = c->st_hdr[5] = 0;
            }
        }
        if (prefix) {  // dumped after the sweep (no sync here: keep the pipeline)
            CU(cudaMalloc(&p.trace, ntr * sizeof(long long)));
            CU(cudaMemsetAsync(p.trace, 0, ntr * sizeof(long long), c->stream));
        }
        // build4 unless the persistent (pipelined) builder is asked for, it
        // does not fit shared memory, or FASTH_BUILD2=1 (A/B knob)
        const bool b4fits = build4_smem_bytes(p.BS, p.d_pad / p.CB, p.CB) <= 227 * 1024 &&
                            !(getenv("FASTH_BUILD2") && atoi(getenv("FASTH_BUILD2")) != 0);
        // the host step's upload goes first: streamed (the builder, the sweep
        // and the gradient kernel start per block as V's columns land) where
        // the whole pipelined chain applies, else one plain SM copy
        if (c->up_pending) {
            c->up_pending = false;
            const auto& u = c->up;
            const char* se = getenv("FASTH_UPLOAD_STREAM");
            const bool stream = (!se || atoi(se) != 0) && c->up_geom_ok && dv_wanted && b4fits && !p.ready &&
                                p.nbuild == 0 && !reversed && p.q <= kMaxPipeQ && u.nv == (int64_t)d * n &&
                                ((int64_t)p.b * d) % 4 == 0 && u.nx % 4 == 0 &&
                                !((reinterpret_cast<uintptr_t>(u.v_src) | reinterpret_cast<uintptr_t>(u.x_src) |
                                   reinterpret_cast<uintptr_t>(u.g_src) | reinterpret_cast<uintptr_t>(u.v) |
                                   reinterpret_cast<uintptr_t>(u.x) | reinterpret_cast<uintptr_t>(u.g)) & 15) &&
                                ldv == d;
            if (stream) {
                UploadArgs ua{};
                ua.x_src = reinterpret_cast<const float4*>(u.x_src);
                ua.g_src = reinterpret_cast<const float4*>(u.g_src);
                ua.v_src = reinterpret_cast<const float4*>(u.v_src);
                ua.x_dst = reinterpret_cast<float4*>(u.x);
                ua.g_dst = reinterpret_cast<float4*>(u.g);
                ua.v_dst = reinterpret_cast<float4*>(u.v);
                ua.x4 = u.nx / 4, ua.v4 = u.nv / 4, ua.blk4 = (int64_t)p.b * d / 4;
                ua.q = p.q, ua.ncb = kUploadChunks;
                ua.upc = c->up_counts(), ua.xg_cnt = c->up_xg();
                const char* ce = getenv("FASTH_UPLOAD_CTAS");
                const int ctas = ce ? std::max(1, atoi(ce)) : 16;
                TRY(c->timed([&] { return launch_upload(ua, ctas, c->stream); }, "h2d_copy"));
                p.upc = c->up_counts();
                p.upc_target = kUploadChunks;
                p.ready = c->counters;
                // a few persistent builder clusters (blocks in upload order):
                // the sweep's clusters find their SMs free and start as soon
                // as the first blocks are built
                const char* nb = getenv("FASTH_BUILDERS");
                p.nbuild = nb ? std::max(1, atoi(nb)) : 10;
                *pipelined = true;
                c->up_active = true;
            } else {
                const float* srcs[3] = {u.v_src, u.x_src, u.g_src};
                float* dsts[3] = {u.v, u.x, u.g};
                const int64_t ns[3] = {u.nv, u.nx, u.nx};
                TRY(c->timed([&] { return launch_stream_copy_n(srcs, dsts, ns, 3, c->num_sms, c->stream); }, "h2d_copy"));
            }
        }
        const bool v4 = c->up_active ? b4fits : !p.ready && p.nbuild == 0 && b4fits;
        fasth_status bs = FASTH_OK;
        if (c->up_active && getenv("FASTH_BUILD_AFTER_SWEEP")) {  // launched by run_forward_backward
            c->build_deferred = true;
            c->deferred_plan = p;
            c->deferred_V = V;
            c->deferred_ldv = ldv;
        } else {
            bs = c->timed([&] {
                return v4 ? launch_build4(p, V, ldv, c->err_d, c->stream) : launch_build2(p, V, ldv, c->err_d, c->stream);
            }, "wy_build");
        }
        if (prefix) {
            c->build_trace = p.trace;
            c->build_trace_n = ntr;
            c->build_trace_rows = p.q * p.CB;
            p.trace = nullptr;
        }
        TRY(bs);
    }
    *out = p;
    return FASTH_OK;
}

fasth_status check_mat(const char* what, const float* ptr, int64_t ld, int rows, int cols) {
    if (rows < 0 || cols < 0) return fail(FASTH_ERR_DIMENSION, "%s: negative shape", what);
    if ((int64_t)rows * cols > 0 && !ptr) return fail(FASTH_ERR_INVALID, "%s: null pointer", what);
    if (cols > 0 && ld < std::max(rows, 1))
        return fail(FASTH_ERR_DIMENSION, "%s: leading dimension %lld < rows %d", what,
                    (long long)ld, rows);
    return FASTH_OK;
}

fasth_status copy_cols(fasth_ctx c, const float* src, int64_t lds, float* dst, int64_t ldd,
                       int rows, int cols) {
    if ((int64_t)rows * cols == 0) return FASTH_OK;
    CU(cudaMemcpy2DAsync(dst, ldd * sizeof(float), src, lds * sizeof(float), rows * sizeof(float),
                         cols, cudaMemcpyDeviceToDevice, c->stream));
    return FASTH_OK;
}

// Large batches run the panel kernel (chain_panel.cu: one CTA per 16-column
// panel holding all rows, no exchange) once the cluster sweep would need more
// than ~2 waves of clusters; FASTH_PANEL=0/1 forces the choice.
bool use_panel(const SweepV2Args& a) {
    if (a.ready || !panel_supported(a.BS, a.d_pad, a.m)) return false;
    if (const char* e = getenv("FASTH_PANEL")) return atoi(e) != 0;
    return a.m > 64;
}

fasth_status launch_traced_sweep2(fasth_ctx c, SweepV2Args& a, const char* what) {
    const char* prefix = getenv("FASTH_TRACE");
    // a gradient kernel launched behind this sweep may read the WY blocks
    // before its own wait once the sweep releases it only after the builder
    a.late_trigger = a.pdl && !a.ready && !getenv("FASTH_EARLY_TRIGGER");
    c->dv_v_pre = !a.ready && (a.late_trigger || !a.pdl) && !use_panel(a);
    if (use_panel(a)) {
        a.trace = nullptr;
        return c->timed([&] { return launch_panel(a, c->stream); }, "panel(fwd/bwd)");
    }
    if (!prefix) {
        const bool st = getenv("FASTH_STEPTRACE") && c->step_trace && c->st_hdr[2] > 0 &&
                        (a.ndir == 2 || !a.dir[0].forward);  // the fused launch or the backward sweep
        a.trace = st ? c->step_trace + c->st_sweep : nullptr;
        a.wtrace = nullptr;
        if (st) c->st_hdr[3] = a.C * a.ngroups * a.ndir;
        return c->timed([&] { return launch_sweep2(a, c->stream); }, what);
    }
    const int nctas = a.C * a.ngroups * a.ndir;
    const size_t n = (size_t)nctas * (a.q + 1) * 16;
    long long* tr = nullptr;
    long long* wtr = nullptr;
    const size_t nw = (size_t)nctas * a.q * 48;
    CU(cudaMalloc(&tr, n * sizeof(long long)));
    CU(cudaMalloc(&wtr, nw * sizeof(long long)));
    CU(cudaMemsetAsync(tr, 0, n * sizeof(long long), c->stream));
    CU(cudaMemsetAsync(wtr, 0, nw * sizeof(long long), c->stream));
    a.trace = tr;
    a.wtrace = wtr;
    fasth_status s = c->timed([&] { return launch_sweep2(a, c->stream); }, what);
    a.trace = nullptr;
    a.wtrace = nullptr;
    std::vector<long long> h(n), hw(nw);
    CU(cudaMemcpyAsync(h.data(), tr, n * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(hw.data(), wtr, nw * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(tr);
    cudaFree(wtr);
    c->dump_build_trace(prefix);
    {
        std::string wpath = std::string(prefix) + "." + what + ".warps.bin";
        if (FILE* f = fopen(wpath.c_str(), "wb")) {
            int hdr[2] = {nctas, a.q};
            fwrite(hdr, sizeof(int), 2, f);
            fwrite(hw.data(), sizeof(long long), nw, f);
            fclose(f);
        }
    }
    std::string path = std::string(prefix) + "." + what + ".v2.bin";
    if (FILE* f = fopen(path.c_str(), "wb")) {
        int hdr[2] = {nctas, a.q};
        fwrite(hdr, sizeof(int), 2, f);
        fwrite(h.data(), sizeof(long long), n, f);
        fclose(f);
    }
    return s;
}

SweepV2Args v2_args(fasth_tape t) {
    const Plan& p = t->plan;
    SweepV2Args a{};
    a.ndir = 1;
    a.d = p.d;
    a.d_pad = p.d_pad;
    a.m = t->m;
    a.q = p.q;
    a.BS = p.BS;
    a.C = t->C;
    a.nstg = t->v2nstg;
    a.ngroups = t->ngroups;
    a.pub_ns = 256;
    if (const char* e = getenv("FASTH_PUB_NS")) a.pub_ns = atoi(e);
    return a;
}

SweepDirV2 v2_forward_dir(fasth_tape t, const float* X, int64_t ldx, float* Y, int64_t ldy, bool record) {
    SweepDirV2 d{};
    d.stage = t->plan.Pf;
    d.x_in = X;
    d.ldx = ldx;
    d.n_valid = t->n_valid;
    d.scale = t->scale;
    d.x_out = Y;
    d.ldo = ldy;
    d.tape = record ? t->tapeA : nullptr;
    d.zhat = record ? t->zf : nullptr;
    d.forward = 1;
    return d;
}

SweepDirV2 v2_backward_dir(fasth_tape t, const float* G, int64_t ldg, int g_valid, const float* g_scale,
                           float* dx, int64_t lddx, bool want_dv) {
    SweepDirV2 d{};
    d.stage = t->plan.Pb;
    d.x_in = G;
    d.ldx = ldg;
    d.n_valid = g_valid;
    d.scale = g_scale;
    d.x_out = dx;
    d.ldo = lddx;
    d.tape = want_dv ? t->tapeG : nullptr;
    d.zhat = want_dv ? t->zb : nullptr;
    d.forward = 0;
    return d;
}

// Forward sweep through a built plan (Alg. 1 step 2).
fasth_status run_forward(fasth_ctx c, fasth_tape t, const float* X, int64_t ldx, float* Y,
                         int64_t ldy, bool record) {
    const Plan& p = t->plan;
    if (record) {
        if (!t->tapeA) TRY(c->alloc_n((size_t)p.q * t->ngroups * p.d_pad * t->WC, &t->tapeA));
        if (!t->zf) TRY(c->alloc_n((size_t)p.q * p.BS * t->m, &t->zf));
    }
    SweepV2Args a = v2_args(t);
    a.dir[0] = v2_forward_dir(t, X, ldx, Y, ldy, record);
    // the builder was the previous launch; X predates it.  Not after a
    // cross-stream event wait: a programmatic launch does not reliably
    // honour a cudaStreamWaitEvent placed before it (measured)
    a.pdl = !getenv("FASTH_NO_PDL") && !c->after_stream_wait;
    c->after_stream_wait = false;
    return launch_traced_sweep2(c, a, "sweep(forward)");
}

fasth_status run_dv(fasth_ctx c, fasth_tape t, float* dV, int64_t lddv, bool pipe = false, int ndir = 2,
                    int order = 0);

// Gradient kernel overlapped with the sweep that feeds it: the sweep counts
// each block's finished tape rows (done[i]) and the gradient kernel, launched
// as its programmatic dependent, starts on a block as soon as both chains
// have passed it.  Not for the panel sweep (it keeps no counters).
// The publishing costs the sweep (tape and publish warps outside the step's
// barrier, sweep2_kernel<.., SIG>) about what the gradient tail it removes is
// worth on the device (fused 57.4 vs 55.1 us, two-call 84.7 vs 83.1 us back
// to back): default only where dV goes out over PCIe (the host-buffer step,
// and the streamed one always).  FASTH_DV_PIPE=0/1 forces it.
bool dv_pipe_ok(fasth_ctx c, const SweepV2Args& a) {
    const char* e = getenv("FASTH_DV_PIPE");
    // (the two-call backward defaulted to it until the sweep lost its
    // end-of-step barrier: now 88.1 vs 90.1 us serial vs pipelined)
    const bool dflt = c->dv_pipe_pref;
    if (e ? atoi(e) == 0 : !dflt) return false;
    // (the signal-warp sweep spills at 64-wide blocks: not there)
    return a.q <= kMaxPipeQ && a.BS <= 32 && c->counters_len >= 3 * kMaxPipeQ && !use_panel(a) &&
           (!getenv("FASTH_TRACE") || e) && sweep2_smem_bytes(a.C, a.BS, a.d_pad, a.nstg, true) <= 227 * 1024;
}

// Backward (Alg. 2): sweep (step 1) + blocked gradients (step 2).
fasth_status run_backward(fasth_ctx c, fasth_tape t, const float* G, int64_t ldg, int g_valid,
                          const float* g_scale, float* dX, int64_t lddx, float* dV,
                          int64_t lddv, const fasthb::lb::Streams* dv_side = nullptr) {
    const Plan& p = t->plan;
    if (!t->tapeA || !t->zf)
        return fail(FASTH_ERR_INVALID, "fasth_backward: tape was recorded without activations");
    const bool want_dv = dV != nullptr;
    if (want_dv) {
        if (!t->tapeG) TRY(c->alloc_n((size_t)p.q * t->ngroups * p.d_pad * t->WC, &t->tapeG));
        if (!t->zb) TRY(c->alloc_n((size_t)p.q * p.BS * t->m, &t->zb));
    }
    float* dx = dX;
    if (!dx) {
        TRY(c->alloc_n((size_t)p.d * std::max(t->m, 1), &dx));
        lddx = p.d;
    }
    SweepV2Args a = v2_args(t);
    a.dir[0] = v2_backward_dir(t, G, ldg, g_valid, g_scale, dx, lddx, want_dv);
    const bool dvpipe = want_dv && !dv_side && dv_pipe_ok(c, a);
    if (dvpipe) a.done = c->counters + kMaxPipeQ;
    fasth_status s = launch_traced_sweep2(c, a, "sweep(backward)");
    if (dx != dX) c->release(dx);
    TRY(s);
    if (!want_dv) return FASTH_OK;
    if (!dv_side) return run_dv(c, t, dV, lddv, dvpipe, 1, 0);
    // gradient kernel on the side stream (off the dX critical path); the
    // caller joins on dv_side->ev[11]
    CU(cudaEventRecord(dv_side->ev[10], c->stream));
    CU(cudaStreamWaitEvent(dv_side->aux, dv_side->ev[10], 0));
    cudaStream_t main_stream = c->stream;
    c->stream = dv_side->aux;
    c->after_stream_wait = true;  // consumed by the gradient kernel's launch
    s = run_dv(c, t, dV, lddv);
    c->stream = main_stream;
    CU(cudaEventRecord(dv_side->ev[11], dv_side->aux));
    return s;
}

fasth_status run_dv(fasth_ctx c, fasth_tape t, float* dV, int64_t lddv, bool pipe, int ndir, int order) {
    const Plan& p = t->plan;
    DvArgs v{};
    if (pipe) {
        v.ready = c->counters;
        v.done = c->counters + kMaxPipeQ;
        v.dvcnt = c->counters + 2 * kMaxPipeQ;
        if (c->up_active) v.upc = c->up_counts();  // streamed host step
        v.done_target = (unsigned)(ndir * t->ngroups * t->C);
        v.order = order;
        // keep the gradient CTAs off the sweep's SMs (FASTH_DV_SMEM overrides)
        const size_t sw = sweep2_smem_bytes(t->C, p.BS, p.d_pad, t->v2nstg, true);
        v.min_smem = sw < 227 * 1024 ? 227 * 1024 - sw + 1024 : 0;
        if (const char* e = getenv("FASTH_DV_SMEM")) v.min_smem = (size_t)atol(e);
        v.poll_ns = 128;
        if (const char* e = getenv("FASTH_DV_POLL")) v.poll_ns = atoi(e);
    }
    c->up_active = false;
    v.pdl = !getenv("FASTH_NO_PDL") && !c->after_stream_wait;  // the sweep was the previous launch
    v.v_pre = c->dv_v_pre || !v.pdl;
    c->after_stream_wait = false;
    if (c->dv_chain == 1) {  // first of independent kernels reading complete inputs
        v.pdl = 0, v.v_pre = 1, v.trigger = 1;
    } else if (c->dv_chain == 2) {  // behind such a kernel: start early, nothing to wait for
        v.pdl = 1, v.nowait = 1, v.v_pre = 1, v.trigger = 1;
    }
    if (getenv("FASTH_STEPTRACE") && c->step_trace && c->st_hdr[3] > 0) {
        v.trace = c->step_trace + c->st_dv;
        c->st_hdr[4] = ((p.d_pad + 63) / 64) * p.q;
        c->st_hdr[5] = 1;
    }
    v.Vbl = p.Vbl;
    v.d = p.d;
    v.d_pad = p.d_pad;
    v.n = p.n;
    v.b = p.b;
    v.q = p.q;
    v.BS = p.BS;
    v.m = t->m;
    v.WC = t->WC;
    v.ngroups = t->ngroups;
    v.reversed = p.reversed;
    v.tapeA = t->tapeA;
    v.tapeG = t->tapeG;
    v.zf = t->zf;
    v.zb = t->zb;
    v.dV = dV;
    v.lddv = lddv;
    return c->timed([&] { return launch_dv2(v, c->stream); }, "dv");
}

// Both sweeps of one chain (X forward, G backward) and the gradients: one
// sweep launch carrying both directions when the v2 kernel applies.
fasth_status run_forward_backward(fasth_ctx c, fasth_tape t, const float* X, int64_t ldx, float* Y,
                                  int64_t ldy, const float* G, int64_t ldg, float* dX, int64_t lddx,
                                  float* dV, int64_t lddv) {
    const Plan& p = t->plan;
    const bool want_dv = dV != nullptr;
    if (!t->tapeA) TRY(c->alloc_n((size_t)p.q * t->ngroups * p.d_pad * t->WC, &t->tapeA));
    if (!t->zf) TRY(c->alloc_n((size_t)p.q * p.BS * t->m, &t->zf));
    if (want_dv) {
        if (!t->tapeG) TRY(c->alloc_n((size_t)p.q * t->ngroups * p.d_pad * t->WC, &t->tapeG));
        if (!t->zb) TRY(c->alloc_n((size_t)p.q * p.BS * t->m, &t->zb));
    }
    float* dx = dX;
    if (!dx) {
        TRY(c->alloc_n((size_t)p.d * std::max(t->m, 1), &dx));
        lddx = p.d;
    }
    SweepV2Args a = v2_args(t);
    a.ndir = 2;
    a.dir[0] = v2_forward_dir(t, X, ldx, Y, ldy, want_dv);
    a.dir[1] = v2_backward_dir(t, G, ldg, p.d, nullptr, dx, lddx, want_dv);
    const bool pipe = t->pipelined && want_dv;
    a.pdl = !getenv("FASTH_NO_PDL") && !c->after_stream_wait;  // the builder was the previous launch
    c->after_stream_wait = false;
    if (pipe) {
        a.ready = c->counters;
        a.done = c->counters + kMaxPipeQ;
    }
    if (pipe && c->up_active) {  // streamed host step: X / G are still landing
        a.xg_ready = c->up_xg();
        a.xg_target = 2 * kUploadChunks;
        a.xg_seen = c->up_xg_seen();
    }
    const bool dvpipe = want_dv && !pipe && dv_pipe_ok(c, a);
    if (dvpipe) {
        a.done = c->counters + kMaxPipeQ;
        a.sig_from = (p.q - 1) / 2;  // no block is final in both chains before this step
    }
    fasth_status s = launch_traced_sweep2(c, a, "sweep(fwd+bwd)");
    if (s == FASTH_OK && c->build_deferred) {  // streamed host step: builder behind the sweep
        c->build_deferred = false;
        s = c->timed([&] {
            return launch_build4(c->deferred_plan, c->deferred_V, c->deferred_ldv, c->err_d, c->stream);
        }, "wy_build");
    }
    c->build_deferred = false;
    if (dx != dX) c->release(dx);
    TRY(s);
    if (!want_dv) return FASTH_OK;
    return run_dv(c, t, dV, lddv, pipe || dvpipe, 2, (pipe || dvpipe) ? 1 : 0);
}

fasth_status new_tape(fasth_ctx c, const float* V, int64_t ldv, int d, int n, int m, int b,
                      int reversed, int tag, fasth_tape* out, bool pipelined = false) {
    fasth_tape t = new fasth_tape_s;
    t->ctx = c;
    t->m = m;
    c->cur_m = m;
    t->b_user = b;
    t->n_valid = d;
    const int BS = next_pow2_min16(internal_b(d, n, b));
    const SweepGeom G = pick_geometry(d, m, BS, c->num_sms, c->geom_fused);
    t->C = G.C;
    t->WC = G.WC;
    t->ngroups = (m + t->WC - 1) / t->WC;
    t->v2nstg = G.C > 0 ? sweep2_nstg(G.C, BS, G.d_pad) : 0;
    if (const char* e = getenv("FASTH_NSTG"))  // A/B knob: fewer stage buffers (less shared memory)
        if (t->v2nstg >= 2) t->v2nstg = std::max(2, std::min(t->v2nstg, atoi(e)));
    if (t->v2nstg < 2) {
        delete t;
        return fail(FASTH_ERR_INVALID, "fasth: dimension %d too large for the chain kernels at block width %d", d, BS);
    }
    t->pipelined = pipelined;
    // the streamed host step needs the pipelined gradient (signal-warp sweep)
    c->up_geom_ok = BS <= 32 && m >= 1 && m <= 64 && !getenv("FASTH_PANEL") && c->counters_len >= 3 * kMaxPipeQ &&
                    sweep2_smem_bytes(G.C, BS, G.d_pad, t->v2nstg, true) <= 227 * 1024;
    fasth_status s = build_plan(c, V, ldv, d, G.d_pad, G.C, n, b, reversed, tag, &t->pipelined, &t->plan);
    if (s != FASTH_OK) {
        delete t;
        return s;
    }
    *out = t;
    return FASTH_OK;
}

// Empty chain (n == 0): tape carries only the shape; output = input.
fasth_tape empty_tape(fasth_ctx c, int d, int m, int b) {
    fasth_tape t = new fasth_tape_s;
    t->ctx = c;
    t->m = m;
    t->b_user = b;
    t->plan.d = d;
    t->plan.n = 0;
    t->plan.q = 0;
    t->n_valid = d;
    return t;
}

// One chain application y = chain(x) (optionally Sigma-scaled input rows),
// forward only, used by the Sigma-ops.
fasth_status apply_chain(fasth_ctx c, const float* V, int64_t ldv, int d, int n, int reversed,
                         int tag, const float* X, int64_t ldx, int n_valid, const float* scale,
                         int m, int b, float* Y, int64_t ldy) {
    if (n == 0) {
        if (scale || n_valid < d)
            return c->timed([&] { return launch_scale_rows(X, ldx, n_valid, scale, d, m, Y, ldy, 0, c->stream); }, "scale_rows");
        return copy_cols(c, X, ldx, Y, ldy, d, m);
    }
    if (use_large_batch(d, n, m)) return lb_apply_chain(c, V, ldv, d, n, reversed, X, ldx, n_valid, scale, m, Y, ldy);
    fasth_tape t = nullptr;
    TRY(new_tape(c, V, ldv, d, n, m, b, reversed, tag, &t));
    t->scale = scale;
    t->n_valid = n_valid;
    fasth_status s = run_forward(c, t, X, ldx, Y, ldy, false);
    free_tape(t);  // pool reuse is stream ordered: safe to recycle immediately
    return s;
}

fasth_status check_param(const char* op, const fasth_svd_param* p) {
    if (!p) return fail(FASTH_ERR_INVALID, "%s: null parameter", op);
    if (p->out_dim < 1 || p->in_dim < 1 || p->nu < 0 || p->nv < 0)
        return fail(FASTH_ERR_DIMENSION, "%s: SvdParam: chain dims inconsistent", op);
    TRY(check_mat(op, p->U, p->ldu, p->out_dim, p->nu));
    TRY(check_mat(op, p->V, p->ldv, p->in_dim, p->nv));
    if (!p->sigma) return fail(FASTH_ERR_INVALID, "%s: null sigma", op);
    return FASTH_OK;
}

}  // namespace

// ==========================================================================
extern "C" {

const char* fasth_last_error(void) { return g_err.c_str(); }
int fasth_version(void) { return 10000; }

fasth_status fasth_ctx_create(int device, void* stream, fasth_ctx* out) {
    if (!out) return fail(FASTH_ERR_INVALID, "null out");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(FASTH_ERR_CUDA, "fasth_b200 needs a CUDA device (sm_100a): %s",
                    e != cudaSuccess ? cudaGetErrorString(e) : "none found");
    if (device < 0 || device >= ndev) return fail(FASTH_ERR_INVALID, "bad device %d", device);
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(FASTH_ERR_CUDA, "fasth_b200 is built for sm_100a (B200); device %d is sm_%d%d",
                    device, prop.major, prop.minor);
    fasth_ctx c = new fasth_ctx_s;
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    c->num_sms = prop.multiProcessorCount;
    e = cudaHostAlloc(&c->err_h, sizeof(ErrWord), cudaHostAllocMapped);
    if (e != cudaSuccess) {
        delete c;
        return fail(FASTH_ERR_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(e));
    }
    c->err_h->flags = 0;
    c->err_h->index = 0x7fffffff;
    c->err_h->chain = 0;
    cudaHostGetDevicePointer(&c->err_d, c->err_h, 0);
    cudaMalloc(&c->logdet_d, sizeof(double));
    // pipelined-step counters (ready | done | dvcnt | uploaded per block, then
    // X/G uploaded and its reader count), zero, self-resetting
    if (cudaMalloc(&c->counters, kCounterWords * sizeof(unsigned)) == cudaSuccess &&
        cudaMemset(c->counters, 0, kCounterWords * sizeof(unsigned)) == cudaSuccess)
        c->counters_len = 3 * kMaxPipeQ;
    *out = c;
    return FASTH_OK;
}

fasth_status fasth_ctx_destroy(fasth_ctx c) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return FASTH_OK;
    c->drop_host_graph();
    cudaStreamSynchronize(c->stream);
    if (c->host_stream) {
        cudaStreamSynchronize(c->host_stream);
        cudaStreamDestroy(c->host_stream);
        cudaEventDestroy(c->host_ev);
    }
    for (auto& kv : c->free_list)
        for (void* p : kv.second) cudaFree(p);
    for (auto& kv : c->live) cudaFree(kv.first);
    if (c->counters) cudaFree(c->counters);
    if (c->step_trace) cudaFree(c->step_trace);
    if (c->logdet_d) cudaFree(c->logdet_d);

    if (c->err_h) cudaFreeHost(c->err_h);
    if (c->switch_ev) cudaEventDestroy(c->switch_ev);
    if (c->lb_st.aux) {
        cudaStreamDestroy(c->lb_st.aux);
        for (auto ev : c->lb_st.ev)
            if (ev) cudaEventDestroy(ev);
    }
    delete c;
    return FASTH_OK;
}

fasth_status fasth_ctx_set_stream(fasth_ctx c, void* stream) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    cudaStream_t next = static_cast<cudaStream_t>(stream);
    if (c->stream == next) return FASTH_OK;
    c->drop_host_graph();
    // The memory pool recycles a released buffer at once, assuming stream
    // order; tapes are read by later calls.  Switching streams therefore
    // orders the new stream after everything enqueued on the old one (one
    // event), so no buffer or tape is reused or read while the old stream
    // still works on it.  Not across a stream being captured into a graph
    // (the capture owns the ordering there).
    cudaStreamCaptureStatus a = cudaStreamCaptureStatusNone, b = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &a);
    cudaStreamIsCapturing(next, &b);
    cudaGetLastError();
    if (a == cudaStreamCaptureStatusNone && b == cudaStreamCaptureStatusNone) {
        if (!c->switch_ev) CU(cudaEventCreateWithFlags(&c->switch_ev, cudaEventDisableTiming));
        CU(cudaEventRecord(c->switch_ev, c->stream));
        CU(cudaStreamWaitEvent(next, c->switch_ev, 0));
        c->after_stream_wait = true;
    }
    c->stream = next;
    return FASTH_OK;
}

fasth_status fasth_ctx_set_check(fasth_ctx c, int mode) {
    DeviceGuard dg_(dev_of(c));
    if (!c || (mode != FASTH_CHECK_SYNC && mode != FASTH_CHECK_DEFERRED))
        return fail(FASTH_ERR_INVALID, "bad check mode");
    c->check_mode = mode;
    return FASTH_OK;
}

fasth_status fasth_ctx_check(fasth_ctx c) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    c->dump_step_trace();
    return c->harvest();
}

int64_t fasth_ctx_launch_count(fasth_ctx c) { return c ? c->launches : 0; }

fasth_status fasth_device_alloc(fasth_ctx c, int64_t bytes, void** out) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !out || bytes < 0) return fail(FASTH_ERR_INVALID, "fasth_device_alloc: bad argument");
    return c->alloc((size_t)bytes, out);
}

fasth_status fasth_device_free(fasth_ctx c, void* ptr) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    c->release(ptr);
    return FASTH_OK;
}

fasth_status fasth_copy(fasth_ctx c, void* dst, const void* src, int64_t bytes, int kind) {
    DeviceGuard dg_(dev_of(c));
    if (!c || bytes < 0 || kind < 0 || kind > 2) return fail(FASTH_ERR_INVALID, "fasth_copy: bad argument");
    if (bytes == 0) return FASTH_OK;
    const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                             : kind == 1 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    CU(cudaMemcpyAsync(dst, src, (size_t)bytes, k, c->stream));
    return FASTH_OK;
}

fasth_status fasth_ctx_synchronize(fasth_ctx c) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    CU(cudaStreamSynchronize(c->stream));
    return FASTH_OK;
}

fasth_status fasth_ctx_set_dv_events(fasth_ctx c, void* const* events, int count) {
    DeviceGuard dg_(dev_of(c));
    if (!c || count < 0 || (count > 0 && !events)) return fail(FASTH_ERR_INVALID, "fasth_ctx_set_dv_events: bad argument");
    c->dv_events.assign(reinterpret_cast<const cudaEvent_t*>(events), reinterpret_cast<const cudaEvent_t*>(events) + count);
    c->dv_row_end.assign(count, 0);
    c->dv_used = 0;
    return FASTH_OK;
}

int fasth_ctx_dv_buckets(fasth_ctx c, int64_t* row_end, int max) {
    DeviceGuard dg_(dev_of(c));
    if (!c || max < 0 || (max > 0 && !row_end)) return -1;
    const int k = std::min(max, c->dv_used);
    for (int i = 0; i < k; ++i) row_end[i] = c->dv_row_end[i];
    return c->dv_used;
}

fasth_status fasth_ctx_set_timing(fasth_ctx c, int mode) {
    DeviceGuard dg_(dev_of(c));
    if (!c || mode < 0 || mode > 2) return fail(FASTH_ERR_INVALID, "fasth_ctx_set_timing: bad argument");
    if (c->timing == 2)
        c->release_timing_events();
    else
        c->collect_timing();
    c->timing = mode;
    c->kernel_ms.clear();
    return FASTH_OK;
}

int fasth_ctx_kernel_times(fasth_ctx c, char* buf, int buflen) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !buf || buflen <= 0) return -1;
    c->collect_timing();
    std::string out;
    char line[160];
    for (auto& kv : c->kernel_ms) {
        snprintf(line, sizeof(line), "%s %.6f %lld\n", kv.first.c_str(), kv.second.first,
                 (long long)kv.second.second);
        out += line;
    }
    snprintf(buf, buflen, "%s", out.c_str());
    return (int)out.size();
}

fasth_status fasth_ctx_trim(fasth_ctx c) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return FASTH_OK;
    CU(cudaStreamSynchronize(c->stream));
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto& kv : c->free_list)
        for (void* p : kv.second) cudaFree(p);
    c->free_list.clear();
    return FASTH_OK;
}

// Large-batch path (lb.h): the chain re-blocked into 512-wide WY blocks, every
// step a tcgen05 GEMM (split K when the batch is small).  Chosen where it
// measured faster than the chain kernels (scripts/small_batch_probe.py, one
// B200): m >= 1024 at d >= 512, m >= 128 at d >= 1024 (2.3-5x over the panel
// sweep at d >= 2048), m >= 64 at d >= 4096; FASTH_LB=0/1 forces the choice.
// Any shape runs there (ragged ones on zero-padded dimensions, lb.h Dims), so
// it also takes every d the chain kernels cannot hold (cluster of at most 16
// CTAs x 256-row slabs: d > 4096) at any batch.
constexpr int kChainMaxD = 4096;
bool use_large_batch(int d, int n, int m) {
    if (!fasthb::lb::supported(d, n, m)) return false;
    if (const char* e = getenv("FASTH_LB")) return atoi(e) != 0;
    return (m >= 1024 && d >= 512) || (m >= 128 && d >= 1024) || (m >= 64 && d >= 4096) || d > kChainMaxD;
}

bool vec_ok(const float* p, int64_t ld) { return !p || ((ld % 4) == 0 && !(reinterpret_cast<uintptr_t>(p) & 15)); }

// Output `out` (d x m, column-major, ld) through a packed temporary when the
// epilogue's 16-byte stores cannot write it in place.
// dV bucket events (fasth_ctx_set_dv_events) describe the caller's dV in
// fasth_backward / fasth_forward_backward; internal calls that compute dV into
// temporaries (SVD legs, the host entry, the tuner) run with them switched off.
struct DvEventsOff {
    fasth_ctx c;
    std::vector<cudaEvent_t> saved;
    explicit DvEventsOff(fasth_ctx cx) : c(cx) { saved.swap(c->dv_events); }
    ~DvEventsOff() {
        c->dv_events.swap(saved);
        c->dv_used = 0;
    }
};

struct OutBuf {
    fasth_ctx c;
    float* user;
    int64_t ld;
    float* tmp = nullptr;
    float* ptr() const { return tmp ? tmp : user; }
    int64_t pitch(int d) const { return tmp ? d : ld; }
    fasth_status open(int d, int m) {
        if (user && !vec_ok(user, ld)) TRY(c->alloc_n((size_t)d * m, &tmp));
        return FASTH_OK;
    }
    fasth_status close(int d, int m) {
        if (tmp) {
            CU(cudaMemcpy2DAsync(user, ld * 4, tmp, (size_t)d * 4, (size_t)d * 4, m, cudaMemcpyDeviceToDevice,
                                 c->stream));
            c->release(tmp);
            tmp = nullptr;
        }
        return FASTH_OK;
    }
};

// Per-launch CUDA events for the large-batch kernels in timing mode 1
// (reported through fasth_ctx_kernel_times next to the chain kernels).
struct LbTimer final : fasthb::lb::Timer {
    fasth_ctx c;
    cudaEvent_t a = nullptr;
    explicit LbTimer(fasth_ctx cx) : c(cx) {}
    void begin(cudaStream_t s) override {
        cudaEventCreate(&a);
        cudaEventRecord(a, s);
    }
    void end(cudaStream_t s, const char* name) override {
        cudaEvent_t b = nullptr;
        cudaEventCreate(&b);
        cudaEventRecord(b, s);
        c->pending.push_back({name, a, b});
        a = nullptr;
    }
};

fasth_status lb_status(fasth_ctx c, cudaError_t e, const char* what) {
    return e == cudaSuccess ? FASTH_OK : fail(FASTH_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

fasth_status run_large_batch(fasth_ctx c, const float* V, int64_t ldv, int d, int n, const float* X, int64_t ldx,
                             const float* G, int64_t ldg, int m, float* Y, int64_t ldy, float* dX, int64_t lddx,
                             float* dV, int64_t lddv) {
    float* ws = nullptr;
    TRY(c->alloc_n(fasthb::lb::workspace_floats(d, n, m, dV != nullptr), &ws));
    OutBuf y{c, Y, ldy}, dx{c, dX, lddx};
    fasth_status s = y.open(d, m);
    if (s == FASTH_OK) s = dx.open(d, m);
    int nl = 1;
    LbTimer lt(c);
    fasthb::lb::DvNotify nt;
    fasthb::lb::DvNotify* ntp = dV ? c->dv_notify(nt) : nullptr;
    if (s == FASTH_OK)
        s = c->timed(
            [&] {
                return fasthb::lb::forward_backward(V, ldv, d, n, X, ldx, G, ldg, m, y.ptr(), y.pitch(d), dx.ptr(),
                                                    dx.pitch(d), dV, lddv, ws, c->err_d, c->stream, c->num_sms, &nl,
                                                    c->timing == 1 ? &lt : nullptr, c->lb_streams(), ntp);
            },
            "large_batch(fwd+bwd)");
    if (ntp) c->dv_used = nt.used;
    c->launches += nl - 1;
    c->after_stream_wait = true;  // the step joined its side streams
    if (s == FASTH_OK) s = y.close(d, m);
    if (s == FASTH_OK) s = dx.close(d, m);
    c->release(ws);  // pool reuse is stream ordered
    if (s == FASTH_OK) s = c->finish();
    return s;
}

// apply_chain on the large-batch path (the Sigma-ops at large batch): a
// reversed chain runs on a vector-reversed copy of V, Sigma-scaled input rows
// are materialised first; forward only.
fasth_status lb_apply_chain(fasth_ctx c, const float* V, int64_t ldv, int d, int n, int reversed, const float* X,
                            int64_t ldx, int n_valid, const float* scale, int m, float* Y, int64_t ldy) {
    float *vr = nullptr, *xs = nullptr, *ws = nullptr;
    fasth_status s = FASTH_OK;
    OutBuf y{c, Y, ldy};
    do {
        if (reversed) {
            s = c->alloc_n((size_t)d * n, &vr);
            if (s) break;
            s = c->timed([&] { return fasthb::lb::reverse_vectors(V, ldv, d, n, vr, d, c->stream); }, "lb_reverse");
            if (s) break;
            V = vr;
            ldv = d;
        }
        if (scale || n_valid < d) {
            s = c->alloc_n((size_t)d * m, &xs);
            if (s) break;
            s = c->timed([&] { return launch_scale_rows(X, ldx, n_valid, scale, d, m, xs, d, 0, c->stream); },
                         "scale_rows");
            if (s) break;
            X = xs;
            ldx = d;
        }
        s = c->alloc_n(fasthb::lb::workspace_floats(d, n, m, false), &ws);
        if (s) break;
        s = y.open(d, m);
        if (s) break;
        int nl = 1;
        LbTimer lt(c);
        s = c->timed(
            [&] {
                return fasthb::lb::forward(V, ldv, d, n, X, ldx, m, y.ptr(), y.pitch(d), ws, c->err_d, c->stream,
                                           c->num_sms, &nl, c->timing == 1 ? &lt : nullptr, c->lb_streams());
            },
            "large_batch(fwd)");
        c->launches += nl - 1;
        c->after_stream_wait = true;
        if (s) break;
        s = y.close(d, m);
    } while (0);
    if (vr) c->release(vr);  // pool reuse is stream ordered
    if (xs) c->release(xs);
    if (ws) c->release(ws);
    return s;
}

// fasth_forward on the large-batch path: the tape owns the workspace (forward
// stages, Zf, WY blocks) that fasth_backward consumes.
fasth_status lb_forward(fasth_ctx c, const float* V, int64_t ldv, int d, int n, const float* X, int64_t ldx, int m,
                        int block_width, float* Y, int64_t ldy, fasth_tape* tape) {
    fasth_tape t = new fasth_tape_s;
    t->ctx = c;
    t->m = m;
    t->b_user = block_width;
    t->plan.d = d;
    t->plan.n = n;
    const int bw = std::min(std::max(block_width, 1), n);
    t->plan.b = bw;
    t->plan.q = (n + bw - 1) / bw;
    fasth_status s = c->alloc_n(fasthb::lb::workspace_floats(d, n, m, true), &t->lb_ws);
    OutBuf y{c, Y, ldy};
    if (s == FASTH_OK) s = y.open(d, m);
    int nl = 1;
    LbTimer lt(c);
    if (s == FASTH_OK)
        s = c->timed(
            [&] {
                return fasthb::lb::forward(V, ldv, d, n, X, ldx, m, y.ptr(), y.pitch(d), t->lb_ws, c->err_d,
                                           c->stream, c->num_sms, &nl, c->timing == 1 ? &lt : nullptr,
                                           c->lb_streams());
            },
            "large_batch(fwd)");
    c->launches += nl - 1;
    c->after_stream_wait = true;  // the step joined its side streams
    if (s == FASTH_OK) s = y.close(d, m);
    if (s == FASTH_OK) s = c->finish();
    if (s == FASTH_OK && tape)
        *tape = t;
    else
        free_tape(t);
    return s;
}

fasth_status fasth_forward(fasth_ctx c, const float* V, int64_t ldv, int d, int n, const float* X,
                           int64_t ldx, int m, int block_width, float* Y, int64_t ldy,
                           fasth_tape* tape) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    if (d < 1) return fail(FASTH_ERR_DIMENSION, "fasth_forward: chain dim must be >= 1");
    if (n < 0 || m < 0) return fail(FASTH_ERR_DIMENSION, "fasth_forward: negative shape");
    TRY(check_mat("fasth_forward: V", V, ldv, d, n));
    TRY(check_mat("fasth_forward: X", X, ldx, d, m));
    TRY(check_mat("fasth_forward: Y", Y, ldy, d, m));
    if (tape) *tape = nullptr;
    if (n == 0 || m == 0) {  // fasth.hpp:46-51
        if (n == 0) TRY(copy_cols(c, X, ldx, Y, ldy, d, m));
        fasth_tape t = nullptr;
        if (n == 0) {
            t = empty_tape(c, d, m, block_width);
        } else {
            TRY(new_tape(c, V, ldv, d, n, m, block_width, 0, 0, &t));
        }
        fasth_status s = c->finish();
        if (tape && s == FASTH_OK) *tape = t;
        else free_tape(t);
        return s;
    }
    if (use_large_batch(d, n, m)) return lb_forward(c, V, ldv, d, n, X, ldx, m, block_width, Y, ldy, tape);
    fasth_tape t = nullptr;
    c->pf[0] = X, c->pf_ld[0] = ldx;
    const fasth_status s0 = new_tape(c, V, ldv, d, n, m, block_width, 0, 0, &t);
    c->pf[0] = c->pf[1] = nullptr;  // consumed by the build (or dropped on failure)
    TRY(s0);
    fasth_status s = run_forward(c, t, X, ldx, Y, ldy, tape != nullptr);
    if (s == FASTH_OK) s = c->finish();
    if (s == FASTH_OK && tape)
        *tape = t;
    else
        free_tape(t);
    return s;
}

fasth_status fasth_backward(fasth_ctx c, fasth_tape t, const float* G, int64_t ldg, float* dX,
                            int64_t lddx, float* dV, int64_t lddv) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !t) return fail(FASTH_ERR_INVALID, "fasth_backward: null ctx or tape");
    const int d = t->plan.d, n = t->plan.n, m = t->m;
    c->dv_used = 0;
    TRY(check_mat("fasth_backward: G", G, ldg, d, m));
    if (dX) TRY(check_mat("fasth_backward: dX", dX, lddx, d, m));
    if (dV) TRY(check_mat("fasth_backward: dV", dV, lddv, d, n));
    if (n == 0) {
        if (dX) TRY(copy_cols(c, G, ldg, dX, lddx, d, m));
        return c->finish();
    }
    if (m == 0) {
        if (dV) CU(cudaMemset2DAsync(dV, lddv * sizeof(float), 0, d * sizeof(float), n, c->stream));
        if (dV) TRY(c->dv_notify_whole(n));
        return c->finish();
    }
    if (t->lb_ws) {
        OutBuf dx{c, dX, lddx};
        TRY(dx.open(d, m));
        int nl = 1;
        LbTimer lt(c);
        fasthb::lb::DvNotify nt;
        fasthb::lb::DvNotify* ntp = dV ? c->dv_notify(nt) : nullptr;
        TRY(c->timed(
            [&] {
                return fasthb::lb::backward(d, n, m, G, ldg, dx.ptr(), dx.pitch(d), dV, lddv, t->lb_ws, c->stream,
                                            c->num_sms, &nl, c->timing == 1 ? &lt : nullptr, c->lb_streams(),
                                            false, ntp);
            },
            "large_batch(bwd)"));
        if (ntp) c->dv_used = nt.used;
        c->launches += nl - 1;
        c->after_stream_wait = true;  // the step joined its side streams
        TRY(dx.close(d, m));
        return c->finish();
    }
    TRY(run_backward(c, t, G, ldg, d, nullptr, dX, lddx, dV, lddv));
    if (dV) TRY(c->dv_notify_whole(n));
    return c->finish();
}

fasth_status fasth_tape_destroy(fasth_tape t) {
    DeviceGuard dg_(dev_of(t));
    free_tape(t);
    return FASTH_OK;
}

fasth_status fasth_tape_info(fasth_tape t, int* d, int* n, int* m, int* block_width, int* q) {
    DeviceGuard dg_(dev_of(t));
    if (!t) return fail(FASTH_ERR_INVALID, "null tape");
    if (d) *d = t->plan.d;
    if (n) *n = t->plan.n;
    if (m) *m = t->m;
    if (block_width) *block_width = t->plan.n ? std::min(std::max(t->b_user, 1), t->plan.n) : t->b_user;
    if (q) *q = t->plan.q;
    return FASTH_OK;
}

fasth_status fasth_forward_backward(fasth_ctx c, const float* V, int64_t ldv, int d, int n,
                                    const float* X, int64_t ldx, const float* G, int64_t ldg,
                                    int m, int block_width, float* Y, int64_t ldy, float* dX,
                                    int64_t lddx, float* dV, int64_t lddv) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    if (d < 1) return fail(FASTH_ERR_DIMENSION, "fasth_forward: chain dim must be >= 1");
    if (n < 0 || m < 0) return fail(FASTH_ERR_DIMENSION, "fasth_forward: negative shape");
    TRY(check_mat("fasth_forward: V", V, ldv, d, n));
    TRY(check_mat("fasth_forward: X", X, ldx, d, m));
    TRY(check_mat("fasth_forward: Y", Y, ldy, d, m));
    TRY(check_mat("fasth_backward: G", G, ldg, d, m));
    if (dX) TRY(check_mat("fasth_backward: dX", dX, lddx, d, m));
    if (dV) TRY(check_mat("fasth_backward: dV", dV, lddv, d, n));
    c->dv_used = 0;
    if (n == 0 || m == 0) {  // the two-call path handles the degenerate shapes
        fasth_tape t = nullptr;
        TRY(fasth_forward(c, V, ldv, d, n, X, ldx, m, block_width, Y, ldy, &t));
        fasth_status s = fasth_backward(c, t, G, ldg, dX, lddx, dV, lddv);
        free_tape(t);
        return s;
    }
    if (use_large_batch(d, n, m))
        return run_large_batch(c, V, ldv, d, n, X, ldx, G, ldg, m, Y, ldy, dX, lddx, dV, lddv);
    fasth_tape t = nullptr;
    c->pf[0] = X, c->pf_ld[0] = ldx, c->pf[1] = G, c->pf_ld[1] = ldg;
    c->geom_fused = true;  // both sweeps in one launch: its cluster count picks the geometry
    const fasth_status s0 = new_tape(c, V, ldv, d, n, m, block_width, 0, 0, &t, dV != nullptr);
    c->geom_fused = false;
    c->pf[0] = c->pf[1] = nullptr;  // consumed by the build (or dropped on failure)
    TRY(s0);
    fasth_status s = run_forward_backward(c, t, X, ldx, Y, ldy, G, ldg, dX, lddx, dV, lddv);
    if (s == FASTH_OK && dV) s = c->dv_notify_whole(n);
    free_tape(t);  // pool reuse is stream ordered
    if (s == FASTH_OK) s = c->finish();
    return s;
}



namespace {

bool is_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Device view of a pinned (UVA-mapped) host buffer, nullptr if it has none.
const float* mapped(const float* p) {
    cudaPointerAttributes at;
    if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        return nullptr;
    }
    return static_cast<const float*>(at.devicePointer);
}

// The host-buffer step, enqueued on c->stream: H2D of V, X, G, the one-call
// step on device copies, D2H of Y, dX, dV.  bufs: v, x, g, y, dx, dv.  Small
// activations (the chain path's batches) are not copied when the caller's
// buffers are pinned: the sweeps read X, G and write Y, dX through PCIe
// directly (one pass each), which saves four copies per call.
fasth_status enqueue_host_step(fasth_ctx c, float* const* bufs, const float* V, int d, int n, const float* X,
                               const float* G, int m, int block_width, float* Y, float* dX, float* dV) {
    float *v = bufs[0], *x = bufs[1], *g = bufs[2], *y = bufs[3], *dx = bufs[4], *dv = bufs[5];
    const size_t nv = (size_t)d * n, nx = (size_t)d * m;
    const char* zc = getenv("FASTH_HOST_ZEROCOPY");
    if ((!zc || atoi(zc) != 0) && nx * 4 <= (1u << 20) && !use_large_batch(d, n, m)) {
        const float *xm = mapped(X), *gm = mapped(G), *ym = mapped(Y), *dxm = mapped(dX);
        if (xm && gm && ym && dxm) {
            // Y, dX out: the sweep's 16-byte stores into the pinned buffers' mappings
            y = const_cast<float*>(ym), dx = const_cast<float*>(dxm);
            // V, X, G in: one SM copy kernel over the pinned buffers' mappings
            // (more PCIe reads in flight than the copy engine keeps:
            // host_io.cu), so the sweep reads X and G from device memory;
            // FASTH_H2D=dma for cudaMemcpyAsync
            // The copy is launched by build_plan, right before the builder:
            // streamed when the pipelined chain applies (host_io.cu
            // upload_kernel: blocks in the order the chains need them,
            // counted per block), else as one plain copy kernel
            const float* vm = mapped(V);
            const char* h2d = getenv("FASTH_H2D");
            c->up_active = c->up_pending = c->build_deferred = false;
            if (nv && vm && !(h2d && !strcmp(h2d, "dma"))) {
                c->up = {vm, xm, gm, v, x, g, (int64_t)nv, (int64_t)nx};
                c->up_pending = true;
            } else {
                if (nv) CU(cudaMemcpyAsync(v, V, nv * 4, cudaMemcpyHostToDevice, c->stream));
                CU(cudaMemcpyAsync(x, X, nx * 4, cudaMemcpyHostToDevice, c->stream));
                CU(cudaMemcpyAsync(g, G, nx * 4, cudaMemcpyHostToDevice, c->stream));
            }
            // the copy is ordered after any cross-stream wait: the step's own
            // launches may chain programmatically again
            c->after_stream_wait = false;
            // dV out: by default the gradient kernel stores straight into the
            // pinned buffer's mapping (16-byte stores of whole columns), run
            // behind the sweep so the PCIe writes overlap it; FASTH_D2H=dma
            // (device buffer + cudaMemcpyAsync) or =kernel (+ SM copy kernel)
            float* dvm = const_cast<float*>(mapped(dV));
            const char* d2h = getenv("FASTH_D2H");
            const bool direct = nv && dvm && !(d2h && (!strcmp(d2h, "dma") || !strcmp(d2h, "kernel")));
            c->dv_pipe_pref = direct;
            const fasth_status fs = fasth_forward_backward(c, v, d, d, n, x, d, g, d, m, block_width, y, d, dx, d,
                                                           n ? (direct ? dvm : dv) : nullptr, d);
            c->dv_pipe_pref = false;
            const bool lost = c->up_pending || c->build_deferred;  // every chain path builds and sweeps
            c->up_active = c->up_pending = c->build_deferred = false;
            TRY(fs);
            if (lost) return fail(FASTH_ERR_INVALID, "host step: the input upload was not issued");
            if (direct) return FASTH_OK;
            if (nv && dvm && d2h && !strcmp(d2h, "kernel"))
                TRY(c->timed([&] { return launch_stream_copy(dv, dvm, (int64_t)nv, c->num_sms, c->stream); }, "d2h_copy"));
            else if (nv)
                CU(cudaMemcpyAsync(dV, dv, nv * 4, cudaMemcpyDeviceToHost, c->stream));
            return FASTH_OK;
        }
    }
    if (nx) CU(cudaMemcpyAsync(x, X, nx * 4, cudaMemcpyHostToDevice, c->stream));
    if (nx) CU(cudaMemcpyAsync(g, G, nx * 4, cudaMemcpyHostToDevice, c->stream));
    // (Overlapping V's upload with the builds and the sweep was tried: a
    // sweep waiting on builders launched after it can deadlock — its
    // 10-CTA clusters leave no GPC room for the builders' clusters.)
    if (nv) CU(cudaMemcpyAsync(v, V, nv * 4, cudaMemcpyHostToDevice, c->stream));
    TRY(fasth_forward_backward(c, v, d, d, n, x, d, g, d, m, block_width, y, d, dx, d, n ? dv : nullptr, d));
    if (nx) CU(cudaMemcpyAsync(Y, y, nx * 4, cudaMemcpyDeviceToHost, c->stream));
    if (nx) CU(cudaMemcpyAsync(dX, dx, nx * 4, cudaMemcpyDeviceToHost, c->stream));
    if (nv) CU(cudaMemcpyAsync(dV, dv, nv * 4, cudaMemcpyDeviceToHost, c->stream));
    return FASTH_OK;
}

}  // namespace

fasth_status host_step_impl(fasth_ctx c, const float* V, int d, int n, const float* X, const float* G, int m,
                            int block_width, float* Y, float* dX, float* dV) {
    if (d < 1 || n < 0 || m < 0) return fail(FASTH_ERR_DIMENSION, "bad shape");
    const size_t nv = (size_t)d * n, nx = (size_t)d * m;
    const int saved = c->check_mode;
    // Repeated calls with the same pinned buffers replay one cached CUDA graph
    // of the whole step (FASTH_HOST_GRAPH=0 disables): the eager sequence
    // leaves the GPU idle while the host enqueues ~10 operations.
    const char* hg = getenv("FASTH_HOST_GRAPH");
    const bool graph_ok = (!hg || atoi(hg) != 0) && n > 0 && m > 0 && is_pinned(V) && is_pinned(X) &&
                          is_pinned(G) && is_pinned(Y) && is_pinned(dX) && is_pinned(dV);
    if (graph_ok) {
        HostGraphKey key;
        const void* ptrs[6] = {V, X, G, Y, dX, dV};
        for (int i = 0; i < 6; ++i) key.p[i] = ptrs[i];
        key.d = d, key.n = n, key.m = m, key.b = block_width;
        bool ready = c->host_exec && c->host_key == key;
        if (!ready) {
            c->drop_host_graph();
            float* bufs[6] = {};
            const size_t sz[6] = {nv, nx, nx, nx, nx, nv};
            fasth_status s = FASTH_OK;
            for (int i = 0; i < 6 && s == FASTH_OK; ++i) s = c->alloc_n(std::max<size_t>(sz[i], 1), &bufs[i]);
            for (float* q : bufs)
                if (q) c->host_bufs.push_back(q);
            if (s != FASTH_OK) {
                c->drop_host_graph();
                return s;
            }
            c->check_mode = FASTH_CHECK_DEFERRED;
            const int64_t l0 = c->launches;
            cudaGraph_t graph = nullptr;
            bool captured = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
            if (captured) {
                c->capturing = true;
                s = enqueue_host_step(c, bufs, V, d, n, X, G, m, block_width, Y, dX, dV);
                c->capturing = false;
                captured = cudaStreamEndCapture(c->stream, &graph) == cudaSuccess && s == FASTH_OK && graph;
            }
            c->check_mode = saved;
            if (captured && cudaGraphInstantiate(&c->host_exec, graph, 0) == cudaSuccess) {
                c->host_key = key;
                c->host_launches = c->launches - l0;
            } else {
                c->host_exec = nullptr;
                cudaGetLastError();
                c->drop_host_graph();  // fall through to the eager path
            }
            if (graph) cudaGraphDestroy(graph);
            ready = c->host_exec != nullptr;
            c->launches = l0;
        }
        if (ready) {
            CU(cudaGraphLaunch(c->host_exec, c->stream));
            c->launches += c->host_launches;
            return c->harvest();
        }
    }
    float* bufs[6] = {};
    const size_t sz[6] = {nv, nx, nx, nx, nx, nv};
    for (int i = 0; i < 6; ++i) TRY(c->alloc_n(std::max<size_t>(sz[i], 1), &bufs[i]));
    c->check_mode = FASTH_CHECK_DEFERRED;
    fasth_status s = enqueue_host_step(c, bufs, V, d, n, X, G, m, block_width, Y, dX, dV);
    c->check_mode = saved;
    fasth_status h = c->harvest();
    if (s == FASTH_OK) s = h;
    for (float* p : bufs) c->release(p);
    return s;
}

fasth_status fasth_forward_backward_host(fasth_ctx c, const float* V, int d, int n,
                                         const float* X, const float* G, int m, int block_width,
                                         float* Y, float* dX, float* dV) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    DvEventsOff no_buckets(c);  // dV comes back in host memory
    // The call is synchronous (host buffers in and out).  On the legacy
    // default stream (which cannot be captured into the cached graph) it
    // runs on a context-owned stream ordered after the legacy stream's work.
    cudaStream_t user = c->stream;
    if (user == nullptr || user == cudaStreamLegacy) {
        if (!c->host_stream) {
            CU(cudaStreamCreateWithFlags(&c->host_stream, cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&c->host_ev, cudaEventDisableTiming));
        }
        CU(cudaEventRecord(c->host_ev, user));
        CU(cudaStreamWaitEvent(c->host_stream, c->host_ev, 0));
        c->stream = c->host_stream;
        c->after_stream_wait = true;
        fasth_status s = host_step_impl(c, V, d, n, X, G, m, block_width, Y, dX, dV);
        c->stream = user;
        return s;
    }
    return host_step_impl(c, V, d, n, X, G, m, block_width, Y, dX, dV);
}

// ---- WY internals (wy.hpp:56-170) -------------------------------------------
namespace {
fasth_status wy_compact_impl(fasth_ctx c, const float* V, int64_t ldv, int d, int n, int bw, float* W, int64_t ldw,
                             float* Y, int64_t ldy) {
    TRY(check_mat("wy_compact: V", V, ldv, d, n));
    TRY(check_mat("wy_compact: W", W, ldw, d, n));
    TRY(check_mat("wy_compact: Y", Y, ldy, d, n));
    double* scratch = nullptr;
    TRY(c->alloc_n(wy_compact_scratch_doubles(n, bw), &scratch));
    fasth_status s = c->timed(
        [&] { return launch_wy_compact(V, ldv, d, n, bw, scratch, W, ldw, Y, ldy, c->err_d, 0, c->stream); },
        "wy_compact");
    c->release(scratch);  // pool reuse is stream ordered
    TRY(s);
    return c->finish();
}

fasth_status wy_apply_impl(fasth_ctx c, const char* what, const float* A, int64_t lda, const float* Bm, int64_t ldb,
                           int d, int b, const float* X, int64_t ldx, int m, float* out, int64_t ldo) {
    if (d < 1 || b < 1 || m < 0) return fail(FASTH_ERR_DIMENSION, "%s: bad shape (d %d, width %d, m %d)", what, d, b, m);
    TRY(check_mat(what, A, lda, d, b));
    TRY(check_mat(what, Bm, ldb, d, b));
    TRY(check_mat(what, X, ldx, d, m));
    TRY(check_mat(what, out, ldo, d, m));
    if (m == 0) return FASTH_OK;
    double* T = nullptr;
    TRY(c->alloc_n((size_t)b * m, &T));
    fasth_status s =
        c->timed([&] { return launch_wy_apply(A, lda, Bm, ldb, d, b, X, ldx, m, T, out, ldo, c->stream); }, what);
    c->release(T);
    TRY(s);
    return c->finish();
}
}  // namespace

fasth_status fasth_wy_compact(fasth_ctx c, const float* V, int64_t ldv, int d, int b, float* W, int64_t ldw,
                              float* Y, int64_t ldy) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    if (b < 1) return fail(FASTH_ERR_INVALID, "wy_compact: empty vector list");
    if (d < 1) return fail(FASTH_ERR_DIMENSION, "wy_compact: dim must be >= 1");
    return wy_compact_impl(c, V, ldv, d, b, b, W, ldw, Y, ldy);
}

fasth_status fasth_compact_chain(fasth_ctx c, const float* V, int64_t ldv, int d, int n, int block_width, float* W,
                                 int64_t ldw, float* Y, int64_t ldy) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    if (d < 1 || n < 0) return fail(FASTH_ERR_DIMENSION, "compact_chain: bad shape");
    if (block_width < 1 || block_width > n)
        return fail(FASTH_ERR_INVALID, "compact_chain: block width %d outside [1, %d]", block_width, n);
    return wy_compact_impl(c, V, ldv, d, n, block_width, W, ldw, Y, ldy);
}

fasth_status fasth_wy_apply(fasth_ctx c, const float* W, int64_t ldw, const float* Y, int64_t ldy, int d, int b,
                            const float* X, int64_t ldx, int m, float* out, int64_t ldo) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    return wy_apply_impl(c, "wy_apply", W, ldw, Y, ldy, d, b, X, ldx, m, out, ldo);
}

fasth_status fasth_wy_apply_transpose(fasth_ctx c, const float* W, int64_t ldw, const float* Y, int64_t ldy, int d,
                                      int b, const float* X, int64_t ldx, int m, float* out, int64_t ldo) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    return wy_apply_impl(c, "wy_apply_transpose", Y, ldy, W, ldw, d, b, X, ldx, m, out, ldo);
}

// ---- SVD layer -------------------------------------------------------------
fasth_status svd_forward_impl(fasth_ctx c, const fasth_svd_param* p, fasth_svd_plan plan, const float* X,
                              int64_t ldx, int m, int block_width, float* Y, int64_t ldy, fasth_svd_tape* tape);

// Both legs on the large-batch path (same thresholds as fasth_forward; a leg
// too tall for the chain kernels takes both there).
bool svd_large_batch(const fasth_svd_param* p, int m) {
    if (m <= 0 || p->nu <= 0 || p->nv <= 0) return false;
    const bool u = use_large_batch(p->out_dim, p->nu, m), v = use_large_batch(p->in_dim, p->nv, m);
    return (u && v) || (u && p->out_dim > kChainMaxD) || (v && p->in_dim > kChainMaxD);
}

// Large-batch SVD layer forward (svd_layer.hpp:106-116): the V^T leg is the V
// chain in reverse order (svd_layer.hpp:113), run as the large-batch step on
// a vector-reversed copy of V; Sigma between the legs is materialised
// (T2 = Sigma T1, zero rows past k) instead of fused into the sweep's loads.
fasth_status lb_svd_forward(fasth_ctx c, const fasth_svd_param* p, const float* X, int64_t ldx, int m, int b,
                            float* Y, int64_t ldy, fasth_svd_tape st) {
    float *vrev = nullptr, *T2 = nullptr;
    TRY(c->alloc_n((size_t)p->in_dim * p->nv, &vrev));
    fasth_status s = FASTH_OK;
    do {
        s = c->timed([&] { return fasthb::lb::reverse_vectors(p->V, p->ldv, p->in_dim, p->nv, vrev, p->in_dim,
                                                              c->stream); }, "lb_reverse");
        if (s) break;
        s = lb_forward(c, vrev, p->in_dim, p->in_dim, p->nv, X, ldx, m, b, st->T1, p->in_dim, &st->v);
        if (s) break;
        s = c->alloc_n((size_t)p->out_dim * m, &T2);
        if (s) break;
        s = c->timed([&] { return launch_scale_rows(st->T1, p->in_dim, st->k, p->sigma, p->out_dim, m, T2,
                                                    p->out_dim, 0, c->stream); }, "scale_rows");
        if (s) break;
        s = lb_forward(c, p->U, p->ldu, p->out_dim, p->nu, T2, p->out_dim, m, b, Y, ldy, &st->u);
    } while (0);
    c->release(vrev);  // pool reuse is stream ordered
    if (T2) c->release(T2);
    return s;
}

// Large-batch SVD layer backward (svd_layer.hpp:122-147) on the tapes above.
fasth_status lb_svd_backward(fasth_ctx c, const fasth_svd_param* p, fasth_svd_tape st, const float* G,
                             int64_t ldg, float* dX, int64_t lddx, float* dU, int64_t lddu, float* dV,
                             int64_t lddv, float* dsigma) {
    const int m = st->m, k = st->k;
    float *dT2 = nullptr, *dT1 = nullptr, *dvrev = nullptr;
    DvEventsOff no_buckets(c);  // the legs below write temporaries, not the caller's dV
    fasth_status s = c->alloc_n((size_t)p->out_dim * m, &dT2);
    do {
        if (s) break;
        s = fasth_backward(c, st->u, G, ldg, dT2, p->out_dim, dU, lddu);
        if (s) break;
        if (dsigma) {
            s = c->timed([&] { return launch_dsigma(dT2, p->out_dim, st->T1, p->in_dim, k, m, dsigma,
                                                    c->stream); }, "dsigma");
            if (s) break;
        }
        s = c->alloc_n((size_t)p->in_dim * m, &dT1);
        if (s) break;
        s = c->timed([&] { return launch_scale_rows(dT2, p->out_dim, k, p->sigma, p->in_dim, m, dT1, p->in_dim, 0,
                                                    c->stream); }, "scale_rows");
        if (s) break;
        if (dV) {
            s = c->alloc_n((size_t)p->in_dim * p->nv, &dvrev);
            if (s) break;
        }
        s = fasth_backward(c, st->v, dT1, p->in_dim, dX, lddx, dvrev, p->in_dim);
        if (s) break;
        if (dV)
            s = c->timed([&] { return fasthb::lb::reverse_vectors(dvrev, p->in_dim, p->in_dim, p->nv, dV, lddv,
                                                                  c->stream); }, "lb_reverse");
    } while (0);
    if (dT2) c->release(dT2);
    if (dT1) c->release(dT1);
    if (dvrev) c->release(dvrev);
    return s;
}

fasth_status fasth_svd_forward(fasth_ctx c, const fasth_svd_param* p, const float* X, int64_t ldx,
                               int m, int block_width, float* Y, int64_t ldy,
                               fasth_svd_tape* tape) {
    DeviceGuard dg_(dev_of(c));
    return svd_forward_impl(c, p, nullptr, X, ldx, m, block_width, Y, ldy, tape);
}

fasth_status fasth_svd_plan_create(fasth_ctx c, const fasth_svd_param* p, int m, int block_width,
                                   int on_side_stream, fasth_svd_plan* out) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !out) return fail(FASTH_ERR_INVALID, "svd_plan_create: null argument");
    *out = nullptr;
    TRY(check_param("svd_plan_create", p));
    if (m < 0) return fail(FASTH_ERR_DIMENSION, "svd_plan_create: negative batch");
    fasth_svd_plan pl = new fasth_svd_plan_s;
    pl->ctx = c;
    pl->out_dim = p->out_dim;
    pl->in_dim = p->in_dim;
    pl->m = m;
    pl->b = block_width;
    if (svd_large_batch(p, m)) {  // the large-batch step builds its WY blocks inside the forward
        *out = pl;
        return FASTH_OK;
    }
    const fasthb::lb::Streams* side = on_side_stream ? c->svd_streams() : nullptr;
    cudaStream_t main_stream = c->stream;
    fasth_status s = FASTH_OK;
    if (side) {
        cudaEventRecord(side->ev[8], c->stream);  // after everything that produced U, V
        cudaStreamWaitEvent(side->aux, side->ev[8], 0);
        c->stream = side->aux;
    }
    if (p->nv > 0 && m > 0) s = new_tape(c, p->V, p->ldv, p->in_dim, p->nv, m, block_width, 1, 1, &pl->v);
    if (s == FASTH_OK && p->nu > 0 && m > 0) s = new_tape(c, p->U, p->ldu, p->out_dim, p->nu, m, block_width, 0, 0, &pl->u);
    if (side) {
        c->stream = main_stream;
        if (s == FASTH_OK && cudaEventCreateWithFlags(&pl->ready, cudaEventDisableTiming) == cudaSuccess)
            cudaEventRecord(pl->ready, side->aux);
    }
    if (s != FASTH_OK) {
        fasth_svd_plan_destroy(pl);
        return s;
    }
    *out = pl;
    return FASTH_OK;
}

fasth_status fasth_svd_plan_destroy(fasth_svd_plan pl) {
    DeviceGuard dg_(dev_of(pl));
    if (!pl) return FASTH_OK;
    free_tape(pl->u);
    free_tape(pl->v);
    if (pl->ready) cudaEventDestroy(pl->ready);
    delete pl;
    return FASTH_OK;
}

fasth_status fasth_svd_forward_planned(fasth_ctx c, const fasth_svd_param* p, fasth_svd_plan plan,
                                       const float* X, int64_t ldx, int m, int block_width, float* Y,
                                       int64_t ldy, fasth_svd_tape* tape) {
    DeviceGuard dg_(dev_of(c));
    if (!plan) return fail(FASTH_ERR_INVALID, "svd_forward_planned: null plan");
    if (plan->used) return fail(FASTH_ERR_INVALID, "svd_forward_planned: plan already consumed");
    if (plan->out_dim != p->out_dim || plan->in_dim != p->in_dim || plan->m != m || plan->b != block_width)
        return fail(FASTH_ERR_DIMENSION, "svd_forward_planned: plan built for another shape / block width");
    return svd_forward_impl(c, p, plan, X, ldx, m, block_width, Y, ldy, tape);
}

fasth_status svd_forward_impl(fasth_ctx c, const fasth_svd_param* p, fasth_svd_plan plan, const float* X,
                              int64_t ldx, int m, int block_width, float* Y, int64_t ldy, fasth_svd_tape* tape) {
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    TRY(check_param("svd_forward", p));
    TRY(check_mat("svd_forward: X", X, ldx, p->in_dim, m));
    TRY(check_mat("svd_forward: Y", Y, ldy, p->out_dim, m));
    if (tape) *tape = nullptr;
    fasth_svd_tape st = new fasth_svd_tape_s;
    st->ctx = c;
    st->out_dim = p->out_dim;
    st->in_dim = p->in_dim;
    st->m = m;
    st->k = std::min(p->out_dim, p->in_dim);
    fasth_status s = FASTH_OK;
    do {
        s = c->alloc_n((size_t)p->in_dim * std::max(m, 1), &st->T1);
        if (s) break;
        if (svd_large_batch(p, m)) {
            if (plan) plan->used = true;  // large-batch plans carry no blocks
            s = lb_svd_forward(c, p, X, ldx, m, block_width, Y, ldy, st);
            if (s == FASTH_OK) s = c->finish();
            break;
        }
        if (plan) {  // prepared blocks: take the plan's tapes, join its side-stream builds
            st->v = plan->v;
            st->u = plan->u;
            plan->v = plan->u = nullptr;
            plan->used = true;
            if (plan->ready) {
                CU(cudaStreamWaitEvent(c->stream, plan->ready, 0));
                c->after_stream_wait = true;
            }
        }
        // The U leg's WY build does not depend on the V leg: it runs on the side
        // stream (fork after everything enqueued so far, join before the U sweep)
        const fasthb::lb::Streams* side =
            (!plan && p->nu > 0 && p->nv > 0 && m > 0) ? c->svd_streams() : nullptr;
        if (side) {
            CU(cudaEventRecord(side->ev[8], c->stream));
            CU(cudaStreamWaitEvent(side->aux, side->ev[8], 0));
            cudaStream_t main_stream = c->stream;
            c->stream = side->aux;
            s = new_tape(c, p->U, p->ldu, p->out_dim, p->nu, m, block_width, 0, 0, &st->u);
            c->stream = main_stream;
            if (s) break;
            CU(cudaEventRecord(side->ev[9], side->aux));
        }
        // V^T leg: the reversed V chain (svd_layer.hpp:113)
        if (p->nv > 0 && m > 0) {
            if (!st->v) s = new_tape(c, p->V, p->ldv, p->in_dim, p->nv, m, block_width, 1, 1, &st->v);
            if (s) break;
            // the sweep reads its input before griddepcontrol.wait (its predecessor is
            // meant to be the builder): prepared blocks => no programmatic launch
            if (plan) c->after_stream_wait = true;
            s = run_forward(c, st->v, X, ldx, st->T1, p->in_dim, tape != nullptr);
        } else {
            s = copy_cols(c, X, ldx, st->T1, p->in_dim, p->in_dim, m);
        }
        if (s) break;
        // U leg on T2 = Sigma T1 (svd_layer.hpp:114-115), Sigma fused into the load
        if (p->nu > 0 && m > 0) {
            if (side) {
                CU(cudaStreamWaitEvent(c->stream, side->ev[9], 0));
                c->after_stream_wait = true;
            } else if (!st->u) {
                s = new_tape(c, p->U, p->ldu, p->out_dim, p->nu, m, block_width, 0, 0, &st->u);
            }
            if (s) break;
            st->u->scale = p->sigma;
            st->u->n_valid = st->k;
            if (plan || side) c->after_stream_wait = true;  // T1 comes from the preceding V sweep
            s = run_forward(c, st->u, st->T1, p->in_dim, Y, ldy, tape != nullptr);
        } else {
            s = c->timed([&] { return launch_scale_rows(st->T1, p->in_dim, st->k, p->sigma, p->out_dim, m, Y,
                                              ldy, 0, c->stream); }, "scale_rows");
        }
        if (s) break;
        s = c->finish();
    } while (0);
    if (s == FASTH_OK && tape) {
        *tape = st;
    } else {
        fasth_svd_tape_destroy(st);
    }
    return s;
}

fasth_status fasth_svd_backward(fasth_ctx c, const fasth_svd_param* p, fasth_svd_tape st,
                                const float* G, int64_t ldg, float* dX, int64_t lddx, float* dU,
                                int64_t lddu, float* dV, int64_t lddv, float* dsigma) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !st) return fail(FASTH_ERR_INVALID, "svd_backward: null ctx or tape");
    TRY(check_param("svd_backward", p));
    if (p->out_dim != st->out_dim || p->in_dim != st->in_dim)
        return fail(FASTH_ERR_DIMENSION, "svd_backward: parameter does not match tape");
    const int m = st->m, k = st->k;
    TRY(check_mat("svd_backward: G", G, ldg, p->out_dim, m));
    if (dX) TRY(check_mat("svd_backward: dX", dX, lddx, p->in_dim, m));
    if (dU) TRY(check_mat("svd_backward: dU", dU, lddu, p->out_dim, p->nu));
    if (dV) TRY(check_mat("svd_backward: dV", dV, lddv, p->in_dim, p->nv));
    if (m > 0 && st->u && st->u->lb_ws && st->v && st->v->lb_ws) {
        TRY(lb_svd_backward(c, p, st, G, ldg, dX, lddx, dU, lddu, dV, lddv, dsigma));
        return c->finish();
    }
    float* dT2 = nullptr;
    TRY(c->alloc_n((size_t)p->out_dim * std::max(m, 1), &dT2));
    fasth_status s = FASTH_OK;
    const fasthb::lb::Streams* side = nullptr;
    do {
        if (m == 0) {
            if (dU && p->nu)
                CU(cudaMemset2DAsync(dU, lddu * 4, 0, p->out_dim * 4, p->nu, c->stream));
            if (dV && p->nv)
                CU(cudaMemset2DAsync(dV, lddv * 4, 0, p->in_dim * 4, p->nv, c->stream));
            if (dsigma && k) CU(cudaMemsetAsync(dsigma, 0, k * 4, c->stream));
            break;
        }
        // U leg (svd_layer.hpp:124); its gradient kernel (dU) runs on the side
        // stream while dSigma and the V leg continue (joined below)
        if (st->u) {
            side = (dU && st->v) ? c->svd_streams() : nullptr;
            s = run_backward(c, st->u, G, ldg, p->out_dim, nullptr, dT2, p->out_dim, dU, lddu, side);
        } else {
            s = copy_cols(c, G, ldg, dT2, p->out_dim, p->out_dim, m);
        }
        if (s) break;
        // dSigma (svd_layer.hpp:131-137)
        if (dsigma) {
            s = c->timed([&] { return launch_dsigma(dT2, p->out_dim, st->T1, p->in_dim, k, m, dsigma,
                                          c->stream); }, "dsigma");
            if (s) break;
        }
        // V^T leg on dT1 = Sigma dT2 (svd_layer.hpp:139-147), Sigma fused into the load
        if (st->v) {
            s = run_backward(c, st->v, dT2, p->out_dim, k, p->sigma, dX, lddx, dV, lddv);
            if (side && s == FASTH_OK) {
                CU(cudaStreamWaitEvent(c->stream, side->ev[11], 0));  // dU done
                c->after_stream_wait = true;
            }
        } else if (dX) {
            s = c->timed([&] { return launch_scale_rows(dT2, p->out_dim, k, p->sigma, p->in_dim, m, dX, lddx,
                                              0, c->stream); }, "scale_rows");
        }
        if (s) break;
    } while (0);
    c->release(dT2);
    if (s == FASTH_OK) s = c->finish();
    return s;
}

// svd_forward + svd_backward as one call when grad_output is known up front
// (the reference benchmark's layer step, bench.hpp:166-209).  The U leg's
// backward sweep needs only G and the V leg's forward sweep only X, so the
// four sweeps pair up into two launches on disjoint clusters:
//   launch 1: V-leg forward (X -> T1)           | U-leg backward (G -> dT2)
//   launch 2: U-leg forward (Sigma T1 -> Y)     | V-leg backward (Sigma dT2 -> dX)
// then dSigma and both gradient kernels.  Square layers whose legs share a
// sweep geometry; anything else runs the two calls.
fasth_status fasth_svd_forward_backward(fasth_ctx c, const fasth_svd_param* p, const float* X, int64_t ldx,
                                        const float* G, int64_t ldg, int m, int block_width, float* Y,
                                        int64_t ldy, float* dX, int64_t lddx, float* dU, int64_t lddu,
                                        float* dV, int64_t lddv, float* dsigma) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    TRY(check_param("svd_forward_backward", p));
    TRY(check_mat("svd_forward: X", X, ldx, p->in_dim, m));
    TRY(check_mat("svd_forward: Y", Y, ldy, p->out_dim, m));
    TRY(check_mat("svd_backward: G", G, ldg, p->out_dim, m));
    if (dX) TRY(check_mat("svd_backward: dX", dX, lddx, p->in_dim, m));
    if (dU) TRY(check_mat("svd_backward: dU", dU, lddu, p->out_dim, p->nu));
    if (dV) TRY(check_mat("svd_backward: dV", dV, lddv, p->in_dim, p->nv));
    const bool square = p->out_dim == p->in_dim && p->nu == p->nv && p->nu > 0 && m > 0;
    auto two_calls = [&]() -> fasth_status {
        fasth_svd_tape st = nullptr;
        TRY(fasth_svd_forward(c, p, X, ldx, m, block_width, Y, ldy, &st));
        fasth_status s = fasth_svd_backward(c, p, st, G, ldg, dX, lddx, dU, lddu, dV, lddv, dsigma);
        fasth_svd_tape_destroy(st);
        return s;
    };
    if (!square || svd_large_batch(p, m) || (getenv("FASTH_SVD_FUSED") && atoi(getenv("FASTH_SVD_FUSED")) == 0))
        return two_calls();
    const int d = p->in_dim, k = std::min(p->out_dim, p->in_dim);
    fasth_tape tv = nullptr, tu = nullptr;
    float *T1 = nullptr, *dT2 = nullptr;
    fasth_status s = FASTH_OK;
    const fasthb::lb::Streams* side = c->svd_streams();
    c->geom_fused = true;  // paired sweeps: two chains per launch
    do {
        // builds: U on the side stream, V on the main stream
        if (side) {
            CU(cudaEventRecord(side->ev[8], c->stream));
            CU(cudaStreamWaitEvent(side->aux, side->ev[8], 0));
            cudaStream_t main_stream = c->stream;
            c->stream = side->aux;
            s = new_tape(c, p->U, p->ldu, d, p->nu, m, block_width, 0, 0, &tu);
            c->stream = main_stream;
            if (s) break;
            CU(cudaEventRecord(side->ev[9], side->aux));
        } else {
            s = new_tape(c, p->U, p->ldu, d, p->nu, m, block_width, 0, 0, &tu);
            if (s) break;
        }
        s = new_tape(c, p->V, p->ldv, d, p->nv, m, block_width, 1, 1, &tv);
        c->geom_fused = false;
        if (s) break;
        if (side) {
            CU(cudaStreamWaitEvent(c->stream, side->ev[9], 0));
            c->after_stream_wait = true;
        }
        const bool same = tv->v2nstg && tu->v2nstg && tv->v2nstg == tu->v2nstg && tv->C == tu->C &&
                          tv->ngroups == tu->ngroups && tv->WC == tu->WC && tv->plan.d_pad == tu->plan.d_pad &&
                          tv->plan.q == tu->plan.q && tv->plan.BS == tu->plan.BS;
        if (!same) {
            free_tape(tu);
            free_tape(tv);
            tu = tv = nullptr;
            return two_calls();
        }
        tu->scale = p->sigma;
        tu->n_valid = k;
        s = c->alloc_n((size_t)d * m, &T1);
        if (s) break;
        s = c->alloc_n((size_t)d * m, &dT2);
        if (s) break;
        const bool want_dv = dV != nullptr, want_du = dU != nullptr;
        for (fasth_tape t : {tv, tu}) {
            const bool g = t == tv ? want_dv : want_du;
            const Plan& pl = t->plan;
            if (!t->tapeA) s = c->alloc_n((size_t)pl.q * t->ngroups * pl.d_pad * t->WC, &t->tapeA);
            if (!s && !t->zf) s = c->alloc_n((size_t)pl.q * pl.BS * t->m, &t->zf);
            if (!s && g && !t->tapeG) s = c->alloc_n((size_t)pl.q * t->ngroups * pl.d_pad * t->WC, &t->tapeG);
            if (!s && g && !t->zb) s = c->alloc_n((size_t)pl.q * pl.BS * t->m, &t->zb);
            if (s) break;
        }
        if (s) break;
        {  // launch 1: V forward | U backward
            SweepV2Args a = v2_args(tv);
            a.ndir = 2;
            a.dir[0] = v2_forward_dir(tv, X, ldx, T1, d, want_dv);
            a.dir[1] = v2_backward_dir(tu, G, ldg, d, nullptr, dT2, d, want_du);
            a.pdl = !getenv("FASTH_NO_PDL") && !c->after_stream_wait;
            c->after_stream_wait = false;
            s = launch_traced_sweep2(c, a, "sweep(svd 1)");
            if (s) break;
        }
        {  // launch 2: U forward (Sigma T1) | V backward (Sigma dT2); reads launch 1's
           // outputs from its first instruction: no programmatic early start
            SweepV2Args a = v2_args(tu);
            a.ndir = 2;
            a.dir[0] = v2_forward_dir(tu, T1, d, Y, ldy, want_du);
            float* dx = dX;
            if (!dx) {
                s = c->alloc_n((size_t)d * m, &dx);
                if (s) break;
            }
            a.dir[1] = v2_backward_dir(tv, dT2, d, k, p->sigma, dx, dX ? lddx : d, want_dv);
            // launched early (its prologue overlaps launch 1's tail); the row
            // warps wait for launch 1 before loading T1 / dT2
            a.pdl = !getenv("FASTH_NO_PDL");
            a.x_wait = 1;
            s = launch_traced_sweep2(c, a, "sweep(svd 2)");
            if (dx != dX) c->release(dx);
            if (s) break;
        }
        // the two gradient kernels and dSigma read only finished tapes and
        // T1 / dT2: the first waits for launch 2, the others run beside it
        int nind = 0;
        if (want_du) {
            c->dv_chain = 1;
            s = run_dv(c, tu, dU, lddu);
            c->dv_chain = 0;
            if (s) break;
            ++nind;
        }
        if (want_dv) {
            c->after_stream_wait = nind == 0;
            c->dv_chain = nind == 0 ? 1 : 2;
            s = run_dv(c, tv, dV, lddv);
            c->dv_chain = 0;
            if (s) break;
            ++nind;
        }
        if (dsigma) {
            const bool early = nind > 0 && !getenv("FASTH_NO_PDL");
            s = c->timed([&] { return launch_dsigma(dT2, d, T1, d, k, m, dsigma, c->stream, early); }, "dsigma");
            if (s) break;
        }
    } while (0);
    c->geom_fused = false;
    free_tape(tu);
    free_tape(tv);
    c->release(T1);
    c->release(dT2);
    if (s == FASTH_OK) s = c->finish();
    return s;
}

fasth_status fasth_svd_tape_destroy(fasth_svd_tape st) {
    DeviceGuard dg_(dev_of(st));
    if (!st) return FASTH_OK;
    free_tape(st->u);
    free_tape(st->v);
    st->ctx->release(st->T1);
    delete st;
    return FASTH_OK;
}

fasth_status fasth_svd_step(fasth_ctx c, const fasth_svd_param* p, const float* dU, int64_t lddu,
                            const float* dV, int64_t lddv, const float* dsigma, float eta,
                            float clamp_eps, float* U_out, int64_t ldou, float* V_out,
                            int64_t ldov, float* sigma_out) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    TRY(check_param("svd_step", p));
    if (!std::isfinite(eta)) return fail(FASTH_ERR_INVALID, "svd_step: eta not finite");
    // clamp_eps == -1: no clamp; otherwise clamp_sigma's domain (svd_layer.hpp:196-198)
    if (clamp_eps != -1.f && !(clamp_eps >= 0.f && clamp_eps < 1.f))
        return fail(FASTH_ERR_INVALID, "clamp_sigma: epsilon outside [0, 1)");
    TRY(check_mat("svd_step: dU", dU, lddu, p->out_dim, p->nu));
    TRY(check_mat("svd_step: dV", dV, lddv, p->in_dim, p->nv));
    TRY(check_mat("svd_step: U_out", U_out, ldou, p->out_dim, p->nu));
    TRY(check_mat("svd_step: V_out", V_out, ldov, p->in_dim, p->nv));
    const int k = std::min(p->out_dim, p->in_dim);
    if (k && (!dsigma || !sigma_out)) return fail(FASTH_ERR_INVALID, "svd_step: null sigma");
    TRY(c->timed([&] { return launch_step(p->U, p->ldu, dU, lddu, p->out_dim, p->nu, eta, U_out, ldou,
                                c->err_d, 0, c->stream); }, "step(U)"));
    TRY(c->timed([&] { return launch_step(p->V, p->ldv, dV, lddv, p->in_dim, p->nv, eta, V_out, ldov,
                                c->err_d, 1, c->stream); }, "step(V)"));
    TRY(c->timed([&] { return launch_sigma_step(p->sigma, dsigma, k, eta, clamp_eps, sigma_out, c->stream); }, "sigma_step"));
    fasth_status s = c->finish();
    if (s == FASTH_ERR_DEGENERATE)  // svd_layer.hpp:177-178 wording
        return fail(s, "svd_step: update degenerates %s vector %d", c->last_chain == 1 ? "V" : "U",
                    c->last_index);
    return s;
}

fasth_status fasth_clamp_sigma(fasth_ctx c, const float* sigma, int k, float epsilon,
                               float* sigma_out) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    if (!(epsilon >= 0.f && epsilon < 1.f))
        return fail(FASTH_ERR_INVALID, "clamp_sigma: epsilon outside [0, 1)");
    TRY(c->timed([&] { return launch_sigma_step(sigma, nullptr, k, 0.f, epsilon, sigma_out, c->stream); }, "clamp_sigma"));
    return c->finish();
}

namespace {
// U f(Sigma) U^T X (symmetric form) or V Sigma^{-1} U^T X (inverse).
fasth_status sigma_op(fasth_ctx c, const fasth_svd_param* p, const float* X, int64_t ldx, int m,
                      int b, float* Y, int64_t ldy, int kind, const char* op) {
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    TRY(check_param(op, p));
    if (p->out_dim != p->in_dim) return fail(FASTH_ERR_DIMENSION, "%s: requires a square parameter", op);
    if (kind != 1 && p->nv != 0)
        return fail(FASTH_ERR_INVALID, "%s: expects symmetric form (empty V chain)", op);
    const int d = p->out_dim;
    TRY(check_mat(op, X, ldx, d, m));
    TRY(check_mat(op, Y, ldy, d, m));
    float* f = nullptr;
    float* t = nullptr;
    TRY(c->alloc_n((size_t)d, &f));
    fasth_status s = c->alloc_n((size_t)d * std::max(m, 1), &t);
    do {
        if (s) break;
        s = c->timed([&] { return launch_sigma_map(p->sigma, d, kind, f, c->err_d, c->stream); }, "sigma_map");
        if (s) break;
        if (c->check_mode == FASTH_CHECK_SYNC) {  // reference checks before any chain work
            s = c->harvest();
            if (s == FASTH_ERR_SINGULAR) s = fail(s, "%s: zero singular value", op);
            if (s) break;
        }
        if (m == 0) break;
        // U^T X: the reversed U chain (matops.hpp:77, :44)
        s = apply_chain(c, p->U, p->ldu, d, p->nu, 1, 0, X, ldx, d, nullptr, m, b, t, d);
        if (s) break;
        if (kind == 1)  // V (Sigma^{-1} t)      matops.hpp:84
            s = apply_chain(c, p->V, p->ldv, d, p->nv, 0, 1, t, d, d, f, m, b, Y, ldy);
        else  // U (f(Sigma) t)                   matops.hpp:51
            s = apply_chain(c, p->U, p->ldu, d, p->nu, 0, 0, t, d, d, f, m, b, Y, ldy);
    } while (0);
    c->release(f);
    c->release(t);
    if (s == FASTH_OK) s = c->finish();
    return s;
}
}  // namespace

fasth_status fasth_apply_inverse(fasth_ctx c, const fasth_svd_param* p, const float* X,
                                 int64_t ldx, int m, int b, float* Y, int64_t ldy) {
    DeviceGuard dg_(dev_of(c));
    return sigma_op(c, p, X, ldx, m, b, Y, ldy, 1, "apply_inverse");
}

fasth_status fasth_apply_exponential(fasth_ctx c, const fasth_svd_param* p, const float* X,
                                     int64_t ldx, int m, int b, float* Y, int64_t ldy) {
    DeviceGuard dg_(dev_of(c));
    return sigma_op(c, p, X, ldx, m, b, Y, ldy, 2, "apply_exponential");
}

fasth_status fasth_apply_cayley(fasth_ctx c, const fasth_svd_param* p, const float* X,
                                int64_t ldx, int m, int b, float* Y, int64_t ldy) {
    DeviceGuard dg_(dev_of(c));
    return sigma_op(c, p, X, ldx, m, b, Y, ldy, 3, "apply_cayley");
}

// matops.hpp:158-175: W^+ X = V (Sigma^+ (U^T X)), rectangular allowed: X is
// out_dim x m, Y in_dim x m; Sigma^+ reciprocates |sigma| > tol, zeroes the
// rest, and maps the out_dim rows onto in_dim rows (zero past min_dim).
fasth_status fasth_apply_pseudo_inverse(fasth_ctx c, const fasth_svd_param* p, const float* X, int64_t ldx, int m,
                                        double tol, int b, float* Y, int64_t ldy) {
    DeviceGuard dg_(dev_of(c));
    if (!c) return fail(FASTH_ERR_INVALID, "null ctx");
    if (!(tol >= 0.0)) return fail(FASTH_ERR_INVALID, "apply_pseudo_inverse: negative tolerance");
    TRY(check_param("apply_pseudo_inverse", p));
    if (m < 0) return fail(FASTH_ERR_DIMENSION, "apply_pseudo_inverse: negative batch");
    const int out = p->out_dim, in = p->in_dim, k = std::min(out, in);
    TRY(check_mat("apply_pseudo_inverse: X", X, ldx, out, m));
    TRY(check_mat("apply_pseudo_inverse: Y", Y, ldy, in, m));
    float* f = nullptr;
    float* t = nullptr;
    TRY(c->alloc_n((size_t)std::max(k, 1), &f));
    fasth_status s = c->alloc_n((size_t)out * std::max(m, 1), &t);
    do {
        if (s) break;
        s = c->timed([&] { return launch_sigma_map(p->sigma, k, 4, f, c->err_d, c->stream, (float)tol); },
                     "sigma_map");
        if (s || m == 0) break;
        // U^T X (the reversed U chain, matops.hpp:166), then V (Sigma^+ t) (:174)
        s = apply_chain(c, p->U, p->ldu, out, p->nu, 1, 0, X, ldx, out, nullptr, m, b, t, out);
        if (s) break;
        s = apply_chain(c, p->V, p->ldv, in, p->nv, 0, 1, t, out, k, f, m, b, Y, ldy);
    } while (0);
    c->release(f);
    c->release(t);
    if (s == FASTH_OK) s = c->finish();
    return s;
}

fasth_status fasth_log_abs_det(fasth_ctx c, const fasth_svd_param* p, double* out) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !out) return fail(FASTH_ERR_INVALID, "null argument");
    TRY(check_param("log_abs_det", p));
    if (p->out_dim != p->in_dim)
        return fail(FASTH_ERR_DIMENSION, "log_abs_det: requires a square parameter");
    TRY(c->timed([&] { return launch_logdet(p->sigma, p->out_dim, c->logdet_d, c->err_d, c->stream); }, "logdet"));
    CU(cudaMemcpyAsync(out, c->logdet_d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    fasth_status s = c->harvest();  // the value is host-visible: always synchronise
    if (s == FASTH_ERR_SINGULAR) return fail(s, "log_abs_det: zero singular value");
    return s;
}

}  // extern "C"

// ---- OSVD checkpoints (svd_layer.hpp:204-290) --------------------------------
namespace {
bool read_u32(std::ifstream& is, uint32_t* x) {
    is.read(reinterpret_cast<char*>(x), 4);
    return (bool)is;
}
fasth_status read_osvd_header(std::ifstream& is, const char* path, uint32_t h[4]) {
    char magic[4] = {};
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "OSVD", 4) != 0) return fail(FASTH_ERR_INVALID, "load_svd_param: bad magic (%s)", path);
    uint32_t version = 0;
    if (!read_u32(is, &version)) return fail(FASTH_ERR_INVALID, "SvdParam load: truncated header");
    if (version != 1) return fail(FASTH_ERR_INVALID, "load_svd_param: unsupported version %u", version);
    for (int k = 0; k < 4; ++k)
        if (!read_u32(is, &h[k])) return fail(FASTH_ERR_INVALID, "SvdParam load: truncated header");
    if (h[0] == 0 || h[1] == 0) return fail(FASTH_ERR_DIMENSION, "SvdParam: zero dimension");
    return FASTH_OK;
}
}  // namespace

extern "C" {

fasth_status fasth_svd_file_info(const char* path, int* out_dim, int* in_dim, int* nu, int* nv) {
    if (!path) return fail(FASTH_ERR_INVALID, "null path");
    std::ifstream is(path, std::ios::binary);
    if (!is) return fail(FASTH_ERR_INVALID, "load_svd_param_file: cannot open %s", path);
    uint32_t h[4];
    TRY(read_osvd_header(is, path, h));
    if (out_dim) *out_dim = (int)h[0];
    if (in_dim) *in_dim = (int)h[1];
    if (nu) *nu = (int)h[2];
    if (nv) *nv = (int)h[3];
    return FASTH_OK;
}

fasth_status fasth_svd_load(fasth_ctx c, const char* path, float* U, int64_t ldu, float* V, int64_t ldv,
                            float* sigma) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !path) return fail(FASTH_ERR_INVALID, "null argument");
    std::ifstream is(path, std::ios::binary);
    if (!is) return fail(FASTH_ERR_INVALID, "load_svd_param_file: cannot open %s", path);
    uint32_t h[4];
    TRY(read_osvd_header(is, path, h));
    const int out_dim = (int)h[0], in_dim = (int)h[1], nu = (int)h[2], nv = (int)h[3];
    const int k = std::min(out_dim, in_dim);
    TRY(check_mat("svd_load: U", U, ldu, out_dim, nu));
    TRY(check_mat("svd_load: V", V, ldv, in_dim, nv));
    if (k && !sigma) return fail(FASTH_ERR_INVALID, "svd_load: null sigma");
    auto read_vectors = [&](int dim, int n, float* dev, int64_t ld, int chain) -> fasth_status {
        if (n == 0) return FASTH_OK;
        std::vector<double> buf((size_t)dim);
        std::vector<float> host((size_t)dim * n);
        for (int j = 0; j < n; ++j) {
            is.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)(dim * sizeof(double)));
            if (!is) return fail(FASTH_ERR_INVALID, "SvdParam load: truncated payload");
            double nn = 0.0;
            bool finite = true;
            for (int r = 0; r < dim; ++r) {
                finite = finite && std::isfinite(buf[r]);
                nn += buf[r] * buf[r];
                host[(size_t)j * dim + r] = (float)buf[r];
            }
            if (!finite) return fail(FASTH_ERR_INVALID, "HouseholderVector: non-finite entry (chain %s vector %d)",
                                     chain ? "V" : "U", j);
            if (!(nn > 1e-30))
                return fail(FASTH_ERR_DEGENERATE, "HouseholderVector: ||v||^2 below degeneracy threshold 1e-30 "
                            "(chain %s vector %d)", chain ? "V" : "U", j);
        }
        CU(cudaMemcpy2DAsync(dev, ld * sizeof(float), host.data(), dim * sizeof(float), dim * sizeof(float), n,
                             cudaMemcpyHostToDevice, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        return FASTH_OK;
    };
    TRY(read_vectors(out_dim, nu, U, ldu, 0));
    TRY(read_vectors(in_dim, nv, V, ldv, 1));
    if (k) {
        std::vector<double> sd((size_t)k);
        is.read(reinterpret_cast<char*>(sd.data()), (std::streamsize)(k * sizeof(double)));
        if (!is) return fail(FASTH_ERR_INVALID, "SvdParam load: truncated payload");
        std::vector<float> sf(sd.begin(), sd.end());
        CU(cudaMemcpyAsync(sigma, sf.data(), k * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    return FASTH_OK;
}

fasth_status fasth_svd_save(fasth_ctx c, const fasth_svd_param* p, const char* path) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !path) return fail(FASTH_ERR_INVALID, "null argument");
    TRY(check_param("save_svd_param", p));
    const int k = std::min(p->out_dim, p->in_dim);
    std::vector<float> U((size_t)p->out_dim * p->nu), V((size_t)p->in_dim * p->nv), sg((size_t)k);
    if (p->nu)
        CU(cudaMemcpy2DAsync(U.data(), p->out_dim * sizeof(float), p->U, p->ldu * sizeof(float),
                             p->out_dim * sizeof(float), p->nu, cudaMemcpyDeviceToHost, c->stream));
    if (p->nv)
        CU(cudaMemcpy2DAsync(V.data(), p->in_dim * sizeof(float), p->V, p->ldv * sizeof(float),
                             p->in_dim * sizeof(float), p->nv, cudaMemcpyDeviceToHost, c->stream));
    if (k) CU(cudaMemcpyAsync(sg.data(), p->sigma, k * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    std::ofstream os(path, std::ios::binary);
    if (!os) return fail(FASTH_ERR_INVALID, "save_svd_param_file: cannot open %s", path);
    os.write("OSVD", 4);
    const uint32_t h[5] = {1u, (uint32_t)p->out_dim, (uint32_t)p->in_dim, (uint32_t)p->nu, (uint32_t)p->nv};
    os.write(reinterpret_cast<const char*>(h), sizeof(h));
    auto put = [&](const std::vector<float>& v) {
        std::vector<double> d(v.begin(), v.end());
        os.write(reinterpret_cast<const char*>(d.data()), (std::streamsize)(d.size() * sizeof(double)));
    };
    put(U);
    put(V);
    put(sg);
    if (!os) return fail(FASTH_ERR_INVALID, "save_svd_param: write failure");
    return FASTH_OK;
}

fasth_status fasth_tune_block_width(fasth_ctx c, int d, int m, int timed, uint64_t seed, int* out) {
    DeviceGuard dg_(dev_of(c));
    if (!c || !out || d < 1 || m < 0) return fail(FASTH_ERR_INVALID, "fasth_tune_block_width: bad argument");
    if (!timed) {  // fasth.hpp:149-152
        *out = std::max(1, (int)std::lround(std::sqrt((double)d)));
        return FASTH_OK;
    }
    DvEventsOff no_buckets(c);  // timing runs write scratch gradients
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({d, m});
        if (it != cache.end()) {
            *out = it->second;
            return FASTH_OK;
        }
    }
    // seeded synthetic chain and data (fasth.hpp:163-174), fp32 on the device
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    const int mm = std::max(m, 1);
    std::vector<float> hv((size_t)d * d), hx((size_t)d * mm), hg((size_t)d * mm);
    for (auto& x : hv) x = (float)gauss(rng);
    for (auto& x : hx) x = (float)gauss(rng);
    for (auto& x : hg) x = (float)gauss(rng);
    float *v = nullptr, *x = nullptr, *g = nullptr, *y = nullptr, *dx = nullptr, *dv = nullptr;
    TRY(c->alloc_n(hv.size(), &v));
    TRY(c->alloc_n(hx.size(), &x));
    TRY(c->alloc_n(hx.size(), &g));
    TRY(c->alloc_n(hx.size(), &y));
    TRY(c->alloc_n(hx.size(), &dx));
    TRY(c->alloc_n(hv.size(), &dv));
    CU(cudaMemcpyAsync(v, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(x, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(g, hg.data(), hg.size() * 4, cudaMemcpyHostToDevice, c->stream));
    std::vector<int> cand;
    const int root = (int)std::ceil(std::sqrt((double)d));
    for (int b = 2; b <= 2 * root && b <= d; ++b) cand.push_back(b);
    if (m >= 1 && m <= d) cand.push_back(m);
    if (cand.empty()) cand.push_back(1);
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    const int saved = c->check_mode;
    c->check_mode = FASTH_CHECK_DEFERRED;
    int best = cand.front();
    float best_ms = -1.f;
    fasth_status s = FASTH_OK;
    for (int b : cand) {
        for (int rep = 0; rep < 2 && s == FASTH_OK; ++rep) {  // warm, then timed
            CU(cudaEventRecord(e0, c->stream));
            s = fasth_forward_backward(c, v, d, d, d, x, d, g, d, mm, b, y, d, dx, d, dv, d);
            CU(cudaEventRecord(e1, c->stream));
        }
        if (s != FASTH_OK) break;
        CU(cudaEventSynchronize(e1));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        if (best_ms < 0.f || ms < best_ms) best_ms = ms, best = b;
    }
    c->check_mode = saved;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (float* ptr : {v, x, g, y, dx, dv}) c->release(ptr);
    TRY(s);
    TRY(c->harvest());
    std::lock_guard<std::mutex> lk(mu);
    cache[{d, m}] = best;
    *out = best;
    return FASTH_OK;
}

}  // extern "C"
