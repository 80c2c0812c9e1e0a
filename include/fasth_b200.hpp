// fasth_b200.hpp — C++ drop-in for the reference FastH API, on the B200.
//
// A user of the reference (/root/reference/proj/include/fasth/) switches by
// replacing `namespace fasth` with `namespace fasth_b200`: the same types
// (Matrix, HouseholderVector, HouseholderChain, TapeForward, BackwardResult,
// SvdParam, SvdGradients, SvdTape), the same free functions with the same
// argument meaning, and the same exception hierarchy.  Every call runs the
// sm_100a kernels of libfasth_b200.so through the C ABI in fasth_b200.h;
// host matrices are converted (row-major f64 <-> column-major fp32) at the
// boundary, exactly once per argument.
//
// Differences a caller can observe (by design, documented in DESIGN.md):
//   * arithmetic is fp32 on the device (3xTF32-class accuracy target; the
//     parity bound is relative_error <= 1e-4, matrix.hpp:106-110);
//   * TapeForward's `compacted` (the WY blocks, wy.hpp:29-48) and
//     `activations` (fasth.hpp:22-29) are materialised on the device by
//     compact_chain and the block recurrence A_i = wy_apply(P_i, A_{i+1})
//     (fasth.hpp:58-59) and copied to the host, as the reference holds them;
//     the backward runs from the device tape;
//   * the chain kernels run block widths above 64 as narrower WY sub-blocks
//     (same product; the materialised blocks keep the caller's width).
//
// Header-only; link with -lfasth_b200.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fasth_b200.h"

namespace fasth_b200 {

// ---- errors (matrix.hpp:12-30) ----------------------------------------------
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class DimensionError : public Error {
public:
    using Error::Error;
};
class DegenerateVectorError : public Error {
public:
    using Error::Error;
};
class SingularMatrixError : public Error {
public:
    using Error::Error;
};
class DeviceError : public Error {
public:
    using Error::Error;
};

inline void check(fasth_status s) {
    if (s == FASTH_OK) return;
    const std::string msg = fasth_last_error();
    switch (s) {
        case FASTH_ERR_DIMENSION: throw DimensionError(msg);
        case FASTH_ERR_DEGENERATE: throw DegenerateVectorError(msg);
        case FASTH_ERR_SINGULAR: throw SingularMatrixError(msg);
        case FASTH_ERR_INVALID: throw Error(msg);
        default: throw DeviceError(msg);
    }
}

// ---- device context ------------------------------------------------------------
// One process-wide context per thread on the selected device (the reference's
// global worker count, parallel.hpp:12-30, becomes the device choice).
class Device {
public:
    static fasth_ctx ctx() { return instance().ctx_; }
    static void select(int device) { instance().reset(device); }

private:
    fasth_ctx ctx_ = nullptr;
    int device_ = -1;
    static Device& instance() {
        thread_local Device d;
        if (!d.ctx_) d.reset(0);
        return d;
    }
    void reset(int device) {
        if (ctx_ && device == device_) return;
        if (ctx_) fasth_ctx_destroy(ctx_);
        ctx_ = nullptr;
        check(fasth_ctx_create(device, nullptr, &ctx_));
        device_ = device;
    }
    ~Device() {
        if (ctx_) fasth_ctx_destroy(ctx_);
    }
};

// RAII device buffer of fp32 from the context pool.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t count) : n_(count) {
        void* p = nullptr;
        check(fasth_device_alloc(Device::ctx(), (int64_t)(std::max<std::size_t>(count, 1) * sizeof(float)), &p));
        p_.reset(static_cast<float*>(p));
    }
    float* get() const { return p_.get(); }
    std::size_t size() const { return n_; }
    void upload(const std::vector<float>& h) {
        check(fasth_copy(Device::ctx(), p_.get(), h.data(), (int64_t)(h.size() * sizeof(float)), 0));
    }
    std::vector<float> download(std::size_t count) const {
        std::vector<float> h(count);
        check(fasth_copy(Device::ctx(), h.data(), p_.get(), (int64_t)(count * sizeof(float)), 1));
        check(fasth_ctx_synchronize(Device::ctx()));
        return h;
    }

private:
    struct Free {
        void operator()(float* p) const { fasth_device_free(Device::ctx(), p); }
    };
    std::unique_ptr<float, Free> p_;
    std::size_t n_ = 0;
};

// ---- Matrix (matrix.hpp:34-85): row-major f64 host matrix ----------------------
class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols) : r_(rows), c_(cols), a_(rows * cols, 0.0) {}
    static Matrix from_data(std::size_t rows, std::size_t cols, std::vector<double> data) {
        if (data.size() != rows * cols)
            throw DimensionError("Matrix::from_data: data length " + std::to_string(data.size()) +
                                 " != " + std::to_string(rows) + "x" + std::to_string(cols));
        for (double x : data)
            if (!std::isfinite(x)) throw Error("Matrix::from_data: non-finite entry");
        Matrix m(rows, cols);
        m.a_ = std::move(data);
        return m;
    }
    static Matrix identity(std::size_t n) {
        Matrix m(n, n);
        for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    double& operator()(std::size_t i, std::size_t j) { return a_[i * c_ + j]; }
    double operator()(std::size_t i, std::size_t j) const { return a_[i * c_ + j]; }
    double* row_ptr(std::size_t i) { return a_.data() + i * c_; }
    const double* row_ptr(std::size_t i) const { return a_.data() + i * c_; }
    const std::vector<double>& data() const { return a_; }
    std::vector<double>& data() { return a_; }
    bool same_shape(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_; }
    friend bool operator==(const Matrix& x, const Matrix& y) {
        return x.r_ == y.r_ && x.c_ == y.c_ && x.a_ == y.a_;
    }

    // column-major fp32 image (d x m, ld = rows) for the device
    std::vector<float> to_device_layout() const {
        std::vector<float> out(r_ * c_);
        for (std::size_t i = 0; i < r_; ++i)
            for (std::size_t j = 0; j < c_; ++j) out[j * r_ + i] = static_cast<float>(a_[i * c_ + j]);
        return out;
    }
    static Matrix from_device_layout(std::size_t rows, std::size_t cols, const std::vector<float>& v) {
        Matrix m(rows, cols);
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t j = 0; j < cols; ++j) m(i, j) = v[j * rows + i];
        return m;
    }

private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<double> a_;
};

inline double frobenius_norm(const Matrix& m) {
    double s = 0.0;
    for (double x : m.data()) s += x * x;
    return std::sqrt(s);
}

/// matrix.hpp:106-110 — the parity metric.
inline double relative_error(const Matrix& a, const Matrix& b) {
    if (!a.same_shape(b)) throw DimensionError("relative_error: shape mismatch");
    double s = 0.0;
    for (std::size_t i = 0; i < a.data().size(); ++i) {
        const double e = a.data()[i] - b.data()[i];
        s += e * e;
    }
    return std::sqrt(s) / std::max(frobenius_norm(b), 1.0);
}

// ---- reflections (householder.hpp:15-81) ----------------------------------------
inline constexpr double kDegeneracyThreshold = 1e-30;

class HouseholderVector {
public:
    explicit HouseholderVector(std::vector<double> v) : v_(std::move(v)) {
        double s = 0.0;
        for (double x : v_) {
            if (!std::isfinite(x)) throw Error("HouseholderVector: non-finite entry");
            s += x * x;
        }
        if (s <= kDegeneracyThreshold)
            throw DegenerateVectorError("HouseholderVector: ||v||^2 = " + std::to_string(s) +
                                        " below degeneracy threshold");
        nsq_ = s;
    }
    std::size_t dim() const { return v_.size(); }
    double norm_sq() const { return nsq_; }
    const std::vector<double>& coeffs() const { return v_; }
    double operator[](std::size_t i) const { return v_[i]; }

private:
    std::vector<double> v_;
    double nsq_ = 0.0;
};

class HouseholderChain {
public:
    explicit HouseholderChain(std::size_t dim) : d_(dim) {}
    HouseholderChain(std::size_t dim, std::vector<HouseholderVector> vs) : d_(dim), vs_(std::move(vs)) {
        for (const auto& v : vs_)
            if (v.dim() != d_) throw DimensionError("HouseholderChain: vector length mismatch");
    }
    std::size_t dim() const { return d_; }
    std::size_t size() const { return vs_.size(); }
    bool empty() const { return vs_.empty(); }
    const HouseholderVector& operator[](std::size_t i) const { return vs_[i]; }
    const std::vector<HouseholderVector>& vectors() const { return vs_; }
    void push_back(HouseholderVector v) {
        if (v.dim() != d_) throw DimensionError("HouseholderChain::push_back: wrong length");
        vs_.push_back(std::move(v));
    }
    HouseholderChain reversed() const {
        HouseholderChain r(d_);
        r.vs_.assign(vs_.rbegin(), vs_.rend());
        return r;
    }
    // column-major d x n fp32 (column k = v_k), the device chain layout
    std::vector<float> to_device_layout() const {
        std::vector<float> out(d_ * vs_.size());
        for (std::size_t k = 0; k < vs_.size(); ++k)
            for (std::size_t i = 0; i < d_; ++i) out[k * d_ + i] = static_cast<float>(vs_[k][i]);
        return out;
    }

private:
    std::size_t d_;
    std::vector<HouseholderVector> vs_;
};

// ---- WY blocks (wy.hpp:18-170) ---------------------------------------------------
/// WYBlock (wy.hpp:18-25): I - 2 W Y^T = H_1 ... H_width.
struct WYBlock {
    std::size_t dim = 0;
    std::size_t width = 0;
    Matrix W;  // dim x width
    Matrix Y;  // dim x width
    std::vector<HouseholderVector> source_vectors;
    std::size_t sequential_steps = 0;  // the reference's instrumentation: width prepends
};

/// CompactedChain (wy.hpp:29-48).
struct CompactedChain {
    std::size_t dim = 0;
    std::size_t block_width = 0;
    std::vector<WYBlock> blocks;
    std::size_t factor_count() const {
        std::size_t n = 0;
        for (const auto& b : blocks) n += b.width;
        return n;
    }
    std::size_t compaction_stages() const {
        std::size_t s = 0;
        for (const auto& b : blocks) s = std::max(s, b.sequential_steps);
        return s;
    }
};

namespace detail {
// column-major fp32 d x width -> host Matrix (d x width)
inline Matrix cols_to_matrix(const std::vector<float>& v, std::size_t d, std::size_t col0, std::size_t w) {
    Matrix m(d, w);
    for (std::size_t j = 0; j < w; ++j)
        for (std::size_t i = 0; i < d; ++i) m(i, j) = v[(col0 + j) * d + i];
    return m;
}
inline std::vector<float> vectors_to_device(const std::vector<HouseholderVector>& vs, std::size_t dim) {
    std::vector<float> out(dim * vs.size());
    for (std::size_t k = 0; k < vs.size(); ++k) {
        if (vs[k].dim() != dim) throw DimensionError("wy_compact: vector length mismatch");
        for (std::size_t i = 0; i < dim; ++i) out[k * dim + i] = static_cast<float>(vs[k][i]);
    }
    return out;
}
// host blocks from the device compaction's W, Y (column-major dim x n)
inline std::vector<WYBlock> blocks_from(const std::vector<float>& wh, const std::vector<float>& yh,
                                        const std::vector<HouseholderVector>& vs, std::size_t dim, std::size_t bw) {
    const std::size_t n = vs.size();
    std::vector<WYBlock> out;
    for (std::size_t lo = 0; lo < n; lo += bw) {
        const std::size_t w = std::min(bw, n - lo);
        WYBlock b;
        b.dim = dim;
        b.width = w;
        b.W = cols_to_matrix(wh, dim, lo, w);
        b.Y = cols_to_matrix(yh, dim, lo, w);
        b.source_vectors.assign(vs.begin() + lo, vs.begin() + lo + w);
        b.sequential_steps = w;
        out.push_back(std::move(b));
    }
    return out;
}
// device compaction of n vectors in blocks of bw into host blocks
inline std::vector<WYBlock> compact_on_device(const std::vector<HouseholderVector>& vs, std::size_t dim,
                                              std::size_t bw, bool whole) {
    const std::size_t n = vs.size();
    DeviceBuffer V(dim * n), W(dim * n), Y(dim * n);
    V.upload(vectors_to_device(vs, dim));
    const int64_t ld = (int64_t)std::max<std::size_t>(dim, 1);
    if (whole)
        check(fasth_wy_compact(Device::ctx(), V.get(), ld, (int)dim, (int)n, W.get(), ld, Y.get(), ld));
    else
        check(fasth_compact_chain(Device::ctx(), V.get(), ld, (int)dim, (int)n, (int)bw, W.get(), ld, Y.get(), ld));
    return blocks_from(W.download(dim * n), Y.download(dim * n), vs, dim, bw);
}
// block -> device W, Y (column-major d x width)
struct DeviceBlock {
    DeviceBuffer W, Y;
    explicit DeviceBlock(const WYBlock& b) : W(b.dim * b.width), Y(b.dim * b.width) {
        W.upload(b.W.to_device_layout());
        Y.upload(b.Y.to_device_layout());
    }
};
inline Matrix wy_apply_impl(const WYBlock& block, const Matrix& X, bool transpose) {
    if (X.rows() != block.dim)
        throw DimensionError(std::string(transpose ? "wy_apply_transpose" : "wy_apply") + ": X has " +
                             std::to_string(X.rows()) + " rows, block dim " + std::to_string(block.dim));
    const std::size_t d = block.dim, m = X.cols();
    DeviceBlock db(block);
    DeviceBuffer Xd(d * m), Od(d * m);
    Xd.upload(X.to_device_layout());
    const int64_t ld = (int64_t)std::max<std::size_t>(d, 1);
    check((transpose ? fasth_wy_apply_transpose : fasth_wy_apply)(Device::ctx(), db.W.get(), ld, db.Y.get(), ld,
                                                                 (int)d, (int)block.width, Xd.get(), ld, (int)m,
                                                                 Od.get(), ld));
    return Matrix::from_device_layout(d, m, Od.download(d * m));
}
}  // namespace detail

/// wy.hpp:56 — (W, Y) of b >= 1 reflections, on the device.
inline WYBlock wy_compact(const std::vector<HouseholderVector>& vectors, std::size_t dim) {
    if (vectors.empty()) throw Error("wy_compact: empty vector list");
    return std::move(detail::compact_on_device(vectors, dim, vectors.size(), true).front());
}

/// wy.hpp:104 — X - 2 W (Y^T X).
inline Matrix wy_apply(const WYBlock& block, const Matrix& X) { return detail::wy_apply_impl(block, X, false); }

/// wy.hpp:137 — X - 2 Y (W^T X).
inline Matrix wy_apply_transpose(const WYBlock& block, const Matrix& X) {
    return detail::wy_apply_impl(block, X, true);
}

/// wy.hpp:151 — ceil(n / block_width) consecutive blocks, the last ragged.
inline CompactedChain compact_chain(const HouseholderChain& chain, std::size_t block_width) {
    const std::size_t n = chain.size();
    if (block_width < 1 || block_width > n)
        throw Error("compact_chain: block width " + std::to_string(block_width) + " outside [1, " +
                    std::to_string(n) + "]");
    CompactedChain out;
    out.dim = chain.dim();
    out.block_width = block_width;
    out.blocks = detail::compact_on_device(chain.vectors(), chain.dim(), block_width, false);
    return out;
}

// ---- FastH (fasth.hpp:22-109) ---------------------------------------------------
struct TapeHandle {
    fasth_tape t = nullptr;
    ~TapeHandle() {
        if (t) fasth_tape_destroy(t);
    }
};

/// TapeForward (fasth.hpp:22-29): the compacted chain and the activations
/// A_1..A_{q+1} (activations[q] = X, activations[0] = the output), as the
/// reference holds them, plus the device tape the backward runs from.
struct TapeForward {
    CompactedChain compacted;
    std::vector<Matrix> activations;
    std::shared_ptr<TapeHandle> handle;
    const Matrix& output() const { return activations.front(); }
    const Matrix& input() const { return activations.back(); }
    std::size_t block_count() const { return compacted.blocks.size(); }
};

/// BackwardResult (fasth.hpp:31-34).
struct BackwardResult {
    Matrix grad_input;
    std::vector<std::vector<double>> grad_vectors;
};

namespace detail {
inline std::vector<std::vector<double>> unpack_vectors(const std::vector<float>& dv, std::size_t d,
                                                       std::size_t n) {
    std::vector<std::vector<double>> out(n, std::vector<double>(d));
    for (std::size_t k = 0; k < n; ++k)
        for (std::size_t i = 0; i < d; ++i) out[k][i] = dv[k * d + i];
    return out;
}
}  // namespace detail

/// fasth.hpp:40 — Algorithm 1 on the device.
inline TapeForward fasth_forward(const HouseholderChain& chain, const Matrix& X,
                                 std::size_t block_width) {
    if (X.rows() != chain.dim()) throw DimensionError("fasth_forward: X row count != chain dim");
    const std::size_t d = chain.dim(), n = chain.size(), m = X.cols();
    DeviceBuffer V(d * n), Xd(d * m), Yd(d * m);
    V.upload(chain.to_device_layout());
    Xd.upload(X.to_device_layout());
    auto h = std::make_shared<TapeHandle>();
    check(fasth_forward(Device::ctx(), V.get(), (int64_t)std::max<std::size_t>(d, 1), (int)d, (int)n,
                        Xd.get(), (int64_t)std::max<std::size_t>(d, 1), (int)m, (int)block_width,
                        Yd.get(), (int64_t)std::max<std::size_t>(d, 1), &h->t));
    TapeForward tape;
    tape.handle = h;
    tape.compacted.dim = d;
    tape.compacted.block_width = block_width;
    if (n == 0) {  // fasth.hpp:46-51
        tape.activations.push_back(X);
        return tape;
    }
    // the reference's members: compacted blocks and the block recurrence
    // A_i = wy_apply(P_i, A_{i+1}) (fasth.hpp:55-59), all on the device
    const std::size_t b = std::min(std::max<std::size_t>(block_width, 1), n), q = (n + b - 1) / b;
    const int64_t ld = (int64_t)std::max<std::size_t>(d, 1);
    tape.compacted.block_width = b;
    DeviceBuffer W(d * n), Yw(d * n), A(d * m * (q + 1));
    check(fasth_compact_chain(Device::ctx(), V.get(), ld, (int)d, (int)n, (int)b, W.get(), ld, Yw.get(), ld));
    tape.compacted.blocks = detail::blocks_from(W.download(d * n), Yw.download(d * n), chain.vectors(), d, b);
    check(fasth_copy(Device::ctx(), A.get() + q * d * m, Xd.get(), (int64_t)(d * m * sizeof(float)), 2));
    for (std::size_t i = q; i-- > 0;) {
        const std::size_t w = std::min(b, n - i * b);
        check(fasth_wy_apply(Device::ctx(), W.get() + i * b * d, ld, Yw.get() + i * b * d, ld, (int)d, (int)w,
                             A.get() + (i + 1) * d * m, ld, (int)m, A.get() + i * d * m, ld));
    }
    const auto ah = A.download(d * m * (q + 1));
    tape.activations.resize(q + 1);
    tape.activations[q] = X;
    for (std::size_t i = 0; i < q; ++i) {
        std::vector<float> one(ah.begin() + i * d * m, ah.begin() + (i + 1) * d * m);
        tape.activations[i] = Matrix::from_device_layout(d, m, one);
    }
    (void)Yd;
    return tape;
}

/// fasth.hpp:69 — Algorithm 2 on the device.
inline BackwardResult fasth_backward(const TapeForward& tape, const Matrix& grad_output) {
    if (!grad_output.same_shape(tape.output()))
        throw DimensionError("fasth_backward: grad_output shape mismatch");
    int d = 0, n = 0, m = 0;
    check(fasth_tape_info(tape.handle->t, &d, &n, &m, nullptr, nullptr));
    DeviceBuffer G((std::size_t)d * m), dX((std::size_t)d * m), dV((std::size_t)d * n);
    G.upload(grad_output.to_device_layout());
    check(fasth_backward(Device::ctx(), tape.handle->t, G.get(), std::max(d, 1), dX.get(),
                         std::max(d, 1), n ? dV.get() : nullptr, std::max(d, 1)));
    BackwardResult r;
    r.grad_input = Matrix::from_device_layout(d, m, dX.download((std::size_t)d * m));
    if (n) r.grad_vectors = detail::unpack_vectors(dV.download((std::size_t)d * n), d, n);
    return r;
}

// ---- SVD layer (svd_layer.hpp:25-202) -------------------------------------------
struct SvdParam {
    std::size_t out_dim = 0;
    std::size_t in_dim = 0;
    HouseholderChain U{0};
    HouseholderChain V{0};
    std::vector<double> sigma;
    std::size_t min_dim() const { return std::min(out_dim, in_dim); }
    void validate() const {
        if (U.dim() != out_dim || V.dim() != in_dim)
            throw DimensionError("SvdParam: chain dims inconsistent");
        if (sigma.size() != min_dim())
            throw DimensionError("SvdParam: sigma length != min(out_dim, in_dim)");
        for (double s : sigma)
            if (!std::isfinite(s)) throw Error("SvdParam: non-finite sigma entry");
    }
};

struct SvdGradients {
    std::vector<std::vector<double>> grad_U_vectors;
    std::vector<std::vector<double>> grad_V_vectors;
    std::vector<double> grad_sigma;
    Matrix grad_input;
};

namespace detail {
// the parameter resident on the device for one call
struct DeviceParam {
    DeviceBuffer U, V, sigma;
    fasth_svd_param c{};
    explicit DeviceParam(const SvdParam& p)
        : U(p.out_dim * p.U.size()), V(p.in_dim * p.V.size()), sigma(p.min_dim()) {
        U.upload(p.U.to_device_layout());
        V.upload(p.V.to_device_layout());
        sigma.upload(std::vector<float>(p.sigma.begin(), p.sigma.end()));
        c.out_dim = (int)p.out_dim;
        c.in_dim = (int)p.in_dim;
        c.nu = (int)p.U.size();
        c.nv = (int)p.V.size();
        c.U = U.get();
        c.ldu = (int64_t)std::max<std::size_t>(p.out_dim, 1);
        c.V = V.get();
        c.ldv = (int64_t)std::max<std::size_t>(p.in_dim, 1);
        c.sigma = sigma.get();
    }
};

struct SvdTapeHandle {
    fasth_svd_tape t = nullptr;
    std::shared_ptr<DeviceParam> param;  // sigma must outlive the tape
    ~SvdTapeHandle() {
        if (t) fasth_svd_tape_destroy(t);
    }
};
}  // namespace detail

/// SvdTape (svd_layer.hpp:83-86), opaque on the device.
struct SvdTape {
    std::shared_ptr<detail::SvdTapeHandle> handle;
    std::size_t m = 0;
};

/// svd_layer.hpp:106 — Y = U (Sigma (V^T X)).
inline std::pair<Matrix, SvdTape> svd_forward(const SvdParam& p, const Matrix& X,
                                              std::size_t block_width) {
    p.validate();
    if (X.rows() != p.in_dim)
        throw DimensionError("svd_forward: X has " + std::to_string(X.rows()) + " rows, in_dim " +
                             std::to_string(p.in_dim));
    auto h = std::make_shared<detail::SvdTapeHandle>();
    h->param = std::make_shared<detail::DeviceParam>(p);
    const std::size_t m = X.cols();
    DeviceBuffer Xd(p.in_dim * m), Yd(p.out_dim * m);
    Xd.upload(X.to_device_layout());
    check(fasth_svd_forward(Device::ctx(), &h->param->c, Xd.get(), (int64_t)p.in_dim, (int)m,
                            (int)block_width, Yd.get(), (int64_t)p.out_dim, &h->t));
    SvdTape tape{h, m};
    return {Matrix::from_device_layout(p.out_dim, m, Yd.download(p.out_dim * m)), tape};
}

/// svd_layer.hpp:122.
inline SvdGradients svd_backward(const SvdParam& p, const SvdTape& tape, const Matrix& grad_output) {
    if (grad_output.rows() != p.out_dim || grad_output.cols() != tape.m)
        throw DimensionError("svd_backward: grad_output shape mismatch");
    const std::size_t m = tape.m, nu = p.U.size(), nv = p.V.size(), k = p.min_dim();
    DeviceBuffer G(p.out_dim * m), dX(p.in_dim * m), dU(p.out_dim * nu), dV(p.in_dim * nv), ds(k);
    G.upload(grad_output.to_device_layout());
    check(fasth_svd_backward(Device::ctx(), &tape.handle->param->c, tape.handle->t, G.get(),
                             (int64_t)p.out_dim, dX.get(), (int64_t)p.in_dim, nu ? dU.get() : nullptr,
                             (int64_t)p.out_dim, nv ? dV.get() : nullptr, (int64_t)p.in_dim,
                             k ? ds.get() : nullptr));
    SvdGradients g;
    g.grad_input = Matrix::from_device_layout(p.in_dim, m, dX.download(p.in_dim * m));
    if (nu) g.grad_U_vectors = detail::unpack_vectors(dU.download(p.out_dim * nu), p.out_dim, nu);
    if (nv) g.grad_V_vectors = detail::unpack_vectors(dV.download(p.in_dim * nv), p.in_dim, nv);
    const auto s = ds.download(k);
    g.grad_sigma.assign(s.begin(), s.end());
    return g;
}

/// svd_layer.hpp:158 — returns a new parameter (the reference is pure).
inline SvdParam svd_step(const SvdParam& p, const SvdGradients& g, double eta) {
    if (!std::isfinite(eta)) throw Error("svd_step: eta not finite");
    if (g.grad_U_vectors.size() != p.U.size() || g.grad_V_vectors.size() != p.V.size() ||
        g.grad_sigma.size() != p.sigma.size())
        throw DimensionError("svd_step: gradient shapes do not match parameter");
    detail::DeviceParam dp(p);
    const std::size_t nu = p.U.size(), nv = p.V.size(), k = p.min_dim();
    auto pack = [](const std::vector<std::vector<double>>& vs, std::size_t d) {
        std::vector<float> out(vs.size() * d);
        for (std::size_t j = 0; j < vs.size(); ++j) {
            if (vs[j].size() != d) throw DimensionError("svd_step: gradient vector length mismatch");
            for (std::size_t i = 0; i < d; ++i) out[j * d + i] = static_cast<float>(vs[j][i]);
        }
        return out;
    };
    DeviceBuffer dU(p.out_dim * nu), dV(p.in_dim * nv), ds(k), Uo(p.out_dim * nu), Vo(p.in_dim * nv), so(k);
    dU.upload(pack(g.grad_U_vectors, p.out_dim));
    dV.upload(pack(g.grad_V_vectors, p.in_dim));
    ds.upload(std::vector<float>(g.grad_sigma.begin(), g.grad_sigma.end()));
    check(fasth_svd_step(Device::ctx(), &dp.c, dU.get(), (int64_t)p.out_dim, dV.get(),
                         (int64_t)p.in_dim, ds.get(), (float)eta, -1.f, Uo.get(), (int64_t)p.out_dim,
                         Vo.get(), (int64_t)p.in_dim, so.get()));
    SvdParam q;
    q.out_dim = p.out_dim;
    q.in_dim = p.in_dim;
    q.U = HouseholderChain(p.out_dim);
    for (auto& v : detail::unpack_vectors(Uo.download(p.out_dim * nu), p.out_dim, nu))
        q.U.push_back(HouseholderVector(std::move(v)));
    q.V = HouseholderChain(p.in_dim);
    for (auto& v : detail::unpack_vectors(Vo.download(p.in_dim * nv), p.in_dim, nv))
        q.V.push_back(HouseholderVector(std::move(v)));
    const auto s = so.download(k);
    q.sigma.assign(s.begin(), s.end());
    return q;
}

/// svd_layer.hpp:196 — O(min dim), host side like the reference.
inline SvdParam clamp_sigma(const SvdParam& p, double epsilon) {
    if (epsilon < 0.0 || epsilon >= 1.0) throw Error("clamp_sigma: epsilon outside [0, 1)");
    SvdParam out = p;
    for (double& s : out.sigma) s = std::clamp(s, 1.0 - epsilon, 1.0 + epsilon);
    return out;
}

// ---- Sigma-ops (matops.hpp) ---------------------------------------------------------
namespace detail {
template <typename F>
Matrix sigma_op(F fn, const SvdParam& p, const Matrix& X, std::size_t block_width) {
    DeviceParam dp(p);
    const std::size_t d = p.out_dim, m = X.cols();
    if (X.rows() != d) throw DimensionError("X row count mismatch");
    DeviceBuffer Xd(d * m), Yd(d * m);
    Xd.upload(X.to_device_layout());
    check(fn(Device::ctx(), &dp.c, Xd.get(), (int64_t)std::max<std::size_t>(d, 1), (int)m,
             (int)block_width, Yd.get(), (int64_t)std::max<std::size_t>(d, 1)));
    return Matrix::from_device_layout(d, m, Yd.download(d * m));
}
}  // namespace detail

/// matops.hpp:69
inline Matrix apply_inverse(const SvdParam& p, const Matrix& X, std::size_t block_width) {
    return detail::sigma_op(fasth_apply_inverse, p, X, block_width);
}
/// matops.hpp:98
inline Matrix apply_exponential(const SvdParam& p, const Matrix& X, std::size_t block_width) {
    return detail::sigma_op(fasth_apply_exponential, p, X, block_width);
}
/// matops.hpp:107
inline Matrix apply_cayley(const SvdParam& p, const Matrix& X, std::size_t block_width) {
    return detail::sigma_op(fasth_apply_cayley, p, X, block_width);
}
/// matops.hpp:158 — W^+ X = V Sigma^+ U^T X (rectangular allowed).
inline Matrix apply_pseudo_inverse(const SvdParam& p, const Matrix& X, double tol, std::size_t block_width) {
    if (tol < 0.0) throw Error("apply_pseudo_inverse: negative tolerance");
    if (X.rows() != p.out_dim) throw DimensionError("apply_pseudo_inverse: X row count mismatch");
    detail::DeviceParam dp(p);
    const std::size_t m = X.cols();
    DeviceBuffer Xd(p.out_dim * m), Yd(p.in_dim * m);
    Xd.upload(X.to_device_layout());
    check(fasth_apply_pseudo_inverse(Device::ctx(), &dp.c, Xd.get(), (int64_t)std::max<std::size_t>(p.out_dim, 1),
                                     (int)m, tol, (int)block_width, Yd.get(),
                                     (int64_t)std::max<std::size_t>(p.in_dim, 1)));
    return Matrix::from_device_layout(p.in_dim, m, Yd.download(p.in_dim * m));
}
/// matops.hpp:57
inline double log_abs_det(const SvdParam& p) {
    detail::DeviceParam dp(p);
    double out = 0.0;
    check(fasth_log_abs_det(Device::ctx(), &dp.c, &out));
    return out;
}

}  // namespace fasth_b200
