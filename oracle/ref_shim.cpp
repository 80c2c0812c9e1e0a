// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/fasth/*.hpp, included by path at compile
// time, never copied).  oracle/Makefile compiles this file into
// oracle/_ref/libfasth_ref.so; tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg load it through oracle/oracle.py.
//
// Array conventions (all f64, C order):
//   chain  : n x d      (row k = v_k, the reference's chain order)
//   matrix : rows x cols row-major (the reference Matrix, matrix.hpp:66)
// Status: 0 ok, 1 DimensionError, 2 DegenerateVectorError,
//         3 SingularMatrixError, 4 fasth::Error, 5 other exception.

#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

#include "fasth/bench.hpp"
#include "fasth/fasth.hpp"
#include "fasth/matops.hpp"
#include "fasth/reference.hpp"
#include "fasth/svd_layer.hpp"
#include "fasth/wy.hpp"

using namespace fasth;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 1;
    } catch (const DegenerateVectorError& e) {
        g_err = e.what();
        return 2;
    } catch (const SingularMatrixError& e) {
        g_err = e.what();
        return 3;
    } catch (const Error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

HouseholderChain chain_in(std::size_t d, std::size_t n, const double* V) {
    HouseholderChain c(d);
    for (std::size_t k = 0; k < n; ++k)
        c.push_back(HouseholderVector(std::vector<double>(V + k * d, V + (k + 1) * d)));
    return c;
}

void chain_out(const HouseholderChain& c, double* V) {
    for (std::size_t k = 0; k < c.size(); ++k)
        std::memcpy(V + k * c.dim(), c[k].coeffs().data(), c.dim() * sizeof(double));
}

Matrix mat_in(std::size_t r, std::size_t c, const double* p) {
    Matrix m(r, c);
    std::memcpy(m.data().data(), p, r * c * sizeof(double));
    return m;
}

void mat_out(const Matrix& m, double* p) {
    std::memcpy(p, m.data().data(), m.data().size() * sizeof(double));
}

void grads_out(const std::vector<std::vector<double>>& g, std::size_t d, double* p) {
    for (std::size_t k = 0; k < g.size(); ++k) {
        if (g[k].empty())
            std::memset(p + k * d, 0, d * sizeof(double));
        else
            std::memcpy(p + k * d, g[k].data(), d * sizeof(double));
    }
}

SvdParam param_in(std::size_t out, std::size_t in, std::size_t nu, std::size_t nv,
                  const double* U, const double* V, const double* sigma) {
    SvdParam p;
    p.out_dim = out;
    p.in_dim = in;
    p.U = chain_in(out, nu, U);
    p.V = chain_in(in, nv, V);
    p.sigma.assign(sigma, sigma + std::min(out, in));
    return p;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_threads() { return hardware_threads(); }

void ref_set_num_threads(int n) { set_num_threads(n); }

/// bench.hpp:117-134 (op = "mul"): rng(seed + d), chain d x d, X, G.
int ref_gen_mul(std::uint64_t seed, std::size_t d, std::size_t m, double* V, double* X,
                double* G) {
    return guarded([&] {
        std::mt19937_64 rng(seed + d);
        HouseholderChain c = bench::random_chain(d, d, rng);
        Matrix x = bench::random_matrix(d, m, rng);
        Matrix g = bench::random_matrix(d, m, rng);
        chain_out(c, V);
        mat_out(x, X);
        mat_out(g, G);
    });
}

/// bench.hpp:122-134 for the SVD ops. symmetric=1 -> op exp/cayley
/// (V chain empty, sigma ~ U(-0.9, 0.9)); else layer/det/inverse
/// (sigma ~ U(0.5, 2)).
int ref_gen_layer(std::uint64_t seed, std::size_t d, std::size_t m, int symmetric, double* U,
                  double* V, double* sigma, double* X, double* G) {
    return guarded([&] {
        std::mt19937_64 rng(seed + d);
        SvdParam p;
        if (symmetric) {
            p = SvdParam::random(d, d, d, 0, rng);
            std::uniform_real_distribution<double> u(-0.9, 0.9);
            for (auto& s : p.sigma) s = u(rng);
        } else {
            p = SvdParam::random(d, d, d, d, rng);
            std::uniform_real_distribution<double> u(0.5, 2.0);
            for (auto& s : p.sigma) s = u(rng);
        }
        Matrix x = bench::random_matrix(d, m, rng);
        Matrix g = bench::random_matrix(d, m, rng);
        chain_out(p.U, U);
        if (!symmetric) chain_out(p.V, V);
        std::memcpy(sigma, p.sigma.data(), p.sigma.size() * sizeof(double));
        mat_out(x, X);
        mat_out(g, G);
    });
}

/// tests/test_support.hpp:21-37 generators under an explicit seed: chain
/// (d x n, unnormalised Gaussian), then X, then G (d x m).
int ref_gen_chain(std::uint64_t seed, std::size_t d, std::size_t n, std::size_t m, double* V,
                  double* X, double* G) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        HouseholderChain c = bench::random_chain(d, n, rng);
        Matrix x = bench::random_matrix(d, m, rng);
        Matrix g = bench::random_matrix(d, m, rng);
        chain_out(c, V);
        mat_out(x, X);
        mat_out(g, G);
    });
}

/// SvdParam::random (svd_layer.hpp:46) + sigma ~ U(lo, hi) + X, G, seed rng.
int ref_gen_param(std::uint64_t seed, std::size_t out, std::size_t in, std::size_t nu,
                  std::size_t nv, std::size_t m, double lo, double hi, double* U, double* V,
                  double* sigma, double* X, double* G) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        SvdParam p = SvdParam::random(out, in, nu, nv, rng);
        std::uniform_real_distribution<double> u(lo, hi);
        for (auto& s : p.sigma) s = u(rng);
        Matrix x = bench::random_matrix(in, m, rng);
        Matrix g = bench::random_matrix(out, m, rng);
        chain_out(p.U, U);
        chain_out(p.V, V);
        std::memcpy(sigma, p.sigma.data(), p.sigma.size() * sizeof(double));
        mat_out(x, X);
        mat_out(g, G);
    });
}

/// fasth_forward (fasth.hpp:40) + fasth_backward (fasth.hpp:69).
int ref_fasth_fwd_bwd(std::size_t d, std::size_t n, std::size_t m, std::size_t b,
                      const double* V, const double* X, const double* G, double* Y, double* dX,
                      double* dV) {
    return guarded([&] {
        HouseholderChain c = chain_in(d, n, V);
        TapeForward tape = fasth_forward(c, mat_in(d, m, X), b);
        mat_out(tape.output(), Y);
        if (G) {
            BackwardResult r = fasth_backward(tape, mat_in(d, m, G));
            mat_out(r.grad_input, dX);
            grads_out(r.grad_vectors, d, dV);
        }
    });
}

/// fasth_forward tape: activations[0..q] (q+1 matrices d x m) and the
/// compacted blocks' W, Y (wy.hpp:18-25), for white-box tests.
int ref_fasth_tape(std::size_t d, std::size_t n, std::size_t m, std::size_t b, const double* V,
                   const double* X, double* activations, double* Wcat, double* Ycat) {
    return guarded([&] {
        HouseholderChain c = chain_in(d, n, V);
        TapeForward tape = fasth_forward(c, mat_in(d, m, X), b);
        for (std::size_t i = 0; i < tape.activations.size(); ++i)
            mat_out(tape.activations[i], activations + i * d * m);
        std::size_t off = 0;
        for (const auto& blk : tape.compacted.blocks) {
            // store each block's W, Y column-by-column: (width x d)
            for (std::size_t j = 0; j < blk.width; ++j)
                for (std::size_t i = 0; i < d; ++i) {
                    Wcat[(off + j) * d + i] = blk.W(i, j);
                    Ycat[(off + j) * d + i] = blk.Y(i, j);
                }
            off += blk.width;
        }
    });
}

/// reference::sequential_forward_backward (reference.hpp:37).
int ref_sequential_fwd_bwd(std::size_t d, std::size_t n, std::size_t m, const double* V,
                           const double* X, const double* G, double* Y, double* dX,
                           double* dV) {
    return guarded([&] {
        HouseholderChain c = chain_in(d, n, V);
        auto [out, r] = reference::sequential_forward_backward(c, mat_in(d, m, X), mat_in(d, m, G));
        mat_out(out, Y);
        mat_out(r.grad_input, dX);
        grads_out(r.grad_vectors, d, dV);
    });
}

/// chain_apply_sequential (householder.hpp:130).
int ref_chain_apply(std::size_t d, std::size_t n, std::size_t m, const double* V,
                    const double* X, double* Y) {
    return guarded([&] {
        mat_out(chain_apply_sequential(chain_in(d, n, V), mat_in(d, m, X)), Y);
    });
}

/// wy_compact (wy.hpp:56): W, Y returned as (b x d) i.e. column j contiguous.
int ref_wy_compact(std::size_t d, std::size_t b, const double* V, double* W, double* Y) {
    return guarded([&] {
        HouseholderChain c = chain_in(d, b, V);
        WYBlock blk = wy_compact(c.vectors(), d);
        for (std::size_t j = 0; j < b; ++j)
            for (std::size_t i = 0; i < d; ++i) {
                W[j * d + i] = blk.W(i, j);
                Y[j * d + i] = blk.Y(i, j);
            }
    });
}

/// householder_grad (householder.hpp:148).
int ref_householder_grad(std::size_t d, std::size_t m, const double* v, const double* A_next,
                         const double* G, double* grad) {
    return guarded([&] {
        HouseholderVector hv(std::vector<double>(v, v + d));
        std::vector<double> g = householder_grad(hv, mat_in(d, m, A_next), mat_in(d, m, G));
        std::memcpy(grad, g.data(), d * sizeof(double));
    });
}

/// svd_forward (svd_layer.hpp:106) + svd_backward (svd_layer.hpp:122).
/// G may be null (forward only).
int ref_svd_fwd_bwd(std::size_t out, std::size_t in, std::size_t nu, std::size_t nv,
                    std::size_t m, std::size_t b, const double* U, const double* V,
                    const double* sigma, const double* X, const double* G, double* Y,
                    double* dX, double* dU, double* dV, double* dsigma) {
    return guarded([&] {
        SvdParam p = param_in(out, in, nu, nv, U, V, sigma);
        auto [y, tape] = svd_forward(p, mat_in(in, m, X), b);
        mat_out(y, Y);
        if (G) {
            SvdGradients g = svd_backward(p, tape, mat_in(out, m, G));
            mat_out(g.grad_input, dX);
            grads_out(g.grad_U_vectors, out, dU);
            grads_out(g.grad_V_vectors, in, dV);
            std::memcpy(dsigma, g.grad_sigma.data(), g.grad_sigma.size() * sizeof(double));
        }
    });
}

/// svd_step (svd_layer.hpp:158) then optional clamp_sigma (svd_layer.hpp:196)
/// when clamp_eps >= 0.  Outputs the new parameter.
int ref_svd_step(std::size_t out, std::size_t in, std::size_t nu, std::size_t nv,
                 const double* U, const double* V, const double* sigma, const double* dU,
                 const double* dV, const double* dsigma, double eta, double clamp_eps,
                 double* U_out, double* V_out, double* sigma_out) {
    return guarded([&] {
        SvdParam p = param_in(out, in, nu, nv, U, V, sigma);
        SvdGradients g;
        for (std::size_t k = 0; k < nu; ++k)
            g.grad_U_vectors.emplace_back(dU + k * out, dU + (k + 1) * out);
        for (std::size_t k = 0; k < nv; ++k)
            g.grad_V_vectors.emplace_back(dV + k * in, dV + (k + 1) * in);
        g.grad_sigma.assign(dsigma, dsigma + p.min_dim());
        SvdParam q = svd_step(p, g, eta);
        if (clamp_eps >= 0.0) q = clamp_sigma(q, clamp_eps);
        chain_out(q.U, U_out);
        chain_out(q.V, V_out);
        std::memcpy(sigma_out, q.sigma.data(), q.sigma.size() * sizeof(double));
    });
}

/// matops.hpp:69 / :98 / :107 / :57.  kind: 0 inverse, 1 exponential,
/// 2 cayley.  For kinds 1 and 2 the V chain must be empty (nv = 0).
int ref_matop(int kind, std::size_t d, std::size_t nu, std::size_t nv, std::size_t m,
              std::size_t b, const double* U, const double* V, const double* sigma,
              const double* X, double* Y) {
    return guarded([&] {
        SvdParam p = param_in(d, d, nu, nv, U, V, sigma);
        Matrix x = mat_in(d, m, X);
        Matrix y = kind == 0 ? apply_inverse(p, x, b)
                   : kind == 1 ? apply_exponential(p, x, b)
                               : apply_cayley(p, x, b);
        mat_out(y, Y);
    });
}

/// apply_pseudo_inverse (matops.hpp:158), rectangular: X out x m -> Y in x m.
int ref_pinv(std::size_t out, std::size_t in, std::size_t nu, std::size_t nv, std::size_t m, std::size_t b,
             double tol, const double* U, const double* V, const double* sigma, const double* X, double* Y) {
    return guarded([&] {
        SvdParam p = param_in(out, in, nu, nv, U, V, sigma);
        mat_out(apply_pseudo_inverse(p, mat_in(out, m, X), tol, b), Y);
    });
}

int ref_log_abs_det(std::size_t d, const double* sigma, double* out) {
    return guarded([&] {
        SvdParam p;
        p.out_dim = p.in_dim = d;
        p.U = HouseholderChain(d);
        p.V = HouseholderChain(d);
        p.sigma.assign(sigma, sigma + d);
        *out = log_abs_det(p);
    });
}

/// bench::run_bench (bench.hpp:225) for ONE algorithm (the cross-algorithm
/// checksum gate at bench.hpp:236-244 is thereby never exercised).
int ref_run_bench(const char* op, const char* algo, std::size_t d, std::size_t m, std::size_t k,
                  std::size_t reps, std::uint64_t seed, int threads, double* mean_s,
                  double* std_s, std::size_t* k_used) {
    return guarded([&] {
        bench::BenchConfig cfg;
        cfg.dims = {d};
        cfg.m = m;
        cfg.k = k;
        cfg.algos = {algo};
        cfg.op = op;
        cfg.reps = reps;
        cfg.seed = seed;
        cfg.threads = threads;
        auto recs = bench::run_bench(cfg);
        *mean_s = recs.at(0).mean_s;
        *std_s = recs.at(0).std_s;
        *k_used = recs.at(0).k;
    });
}

int ref_verify(int* passed, int* total) {
    return guarded([&] {
        auto checks = bench::verify();
        *total = static_cast<int>(checks.size());
        *passed = 0;
        for (const auto& c : checks) *passed += c.passed ? 1 : 0;
    });
}

/// save_svd_param_file (svd_layer.hpp:276) of a parameter given as arrays.
int ref_svd_save(const char* path, std::size_t out, std::size_t in, std::size_t nu, std::size_t nv,
                 const double* U, const double* V, const double* sigma) {
    return guarded([&] { save_svd_param_file(param_in(out, in, nu, nv, U, V, sigma), path); });
}

/// load_svd_param_file (svd_layer.hpp:282): header into dims[4], payload into
/// U / V / sigma when they are non-null (call once for the dims, then again).
int ref_svd_load(const char* path, std::size_t* dims, double* U, double* V, double* sigma) {
    return guarded([&] {
        SvdParam p = load_svd_param_file(path);
        dims[0] = p.out_dim;
        dims[1] = p.in_dim;
        dims[2] = p.U.size();
        dims[3] = p.V.size();
        if (U) chain_out(p.U, U);
        if (V) chain_out(p.V, V);
        if (sigma) std::memcpy(sigma, p.sigma.data(), p.sigma.size() * sizeof(double));
    });
}

} // extern "C"
