// Drop-in test of the C++ mirror (include/fasth_b200.hpp) against the
// UNMODIFIED reference headers, in one binary: the same seeded inputs go
// through `fasth::` (reference, f64 CPU) and `fasth_b200::` (B200), and the
// outputs are compared with the reference's own relative_error
// (matrix.hpp:106-110).  Test infrastructure only (built by
// tests/cpp/Makefile where /root/reference exists; the binary travels to the
// GPU box and is run by tests/test_gpu_cpp.py).
#include <cstdio>
#include <random>
#include <string>

#include "fasth/bench.hpp"
#include "fasth/fasth.hpp"
#include "fasth/matops.hpp"
#include "fasth/reference.hpp"
#include "fasth/svd_layer.hpp"
#include "fasth_b200.hpp"

namespace R = fasth;
namespace B = fasth_b200;

static int g_fail = 0;

static void report(const std::string& name, double err, double tol) {
    const bool ok = err <= tol;
    std::printf("%s %-44s err %.3e (tol %.0e)\n", ok ? "PASS" : "FAIL", name.c_str(), err, tol);
    if (!ok) ++g_fail;
}

static void expect(const std::string& name, bool ok) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
    if (!ok) ++g_fail;
}

static B::Matrix to_b(const R::Matrix& m) { return B::Matrix::from_data(m.rows(), m.cols(), m.data()); }

static B::HouseholderChain to_b(const R::HouseholderChain& c) {
    B::HouseholderChain out(c.dim());
    for (const auto& v : c.vectors()) out.push_back(B::HouseholderVector(v.coeffs()));
    return out;
}

static B::SvdParam to_b(const R::SvdParam& p) {
    B::SvdParam q;
    q.out_dim = p.out_dim;
    q.in_dim = p.in_dim;
    q.U = to_b(p.U);
    q.V = to_b(p.V);
    q.sigma = p.sigma;
    return q;
}

static double rel(const B::Matrix& a, const R::Matrix& b) {
    R::Matrix aa(a.rows(), a.cols());
    aa.data() = a.data();
    return R::relative_error(aa, b);
}

static double rel_vecs(const std::vector<std::vector<double>>& a,
                       const std::vector<std::vector<double>>& b) {
    double num = 0, den = 0;
    for (std::size_t k = 0; k < b.size(); ++k)
        for (std::size_t i = 0; i < b[k].size(); ++i) {
            const double e = a[k][i] - b[k][i];
            num += e * e;
            den += b[k][i] * b[k][i];
        }
    return std::sqrt(num) / std::max(std::sqrt(den), 1.0);
}

static double rel_vec(const std::vector<double>& a, const std::vector<double>& b) {
    return rel_vecs({a}, {b});
}

int main() {
    const double tol = 1e-4;
    // 1. metric config: Workload(op=mul, seed 0, d=784, m=32), b = 32 (bench.hpp:117-134)
    {
        std::mt19937_64 rng(0 + 784);
        auto chain = R::bench::random_chain(784, 784, rng);
        auto X = R::bench::random_matrix(784, 32, rng);
        auto G = R::bench::random_matrix(784, 32, rng);
        auto [Y, seq] = R::reference::sequential_forward_backward(chain, X, G);
        auto tape = B::fasth_forward(to_b(chain), to_b(X), 32);
        auto back = B::fasth_backward(tape, to_b(G));
        report("cfg2 d=784 b=32 m=32 UX", rel(tape.output(), Y), tol);
        report("cfg2 d=784 b=32 m=32 dX", rel(back.grad_input, seq.grad_input), tol);
        report("cfg2 d=784 b=32 m=32 dV", rel_vecs(back.grad_vectors, seq.grad_vectors), tol);
        expect("tape block count = ceil(n/b) = 25", tape.block_count() == 25);
    }
    // 2. ragged partition (test_fasth.cpp:95-111)
    {
        std::mt19937_64 rng(137);
        for (int trial = 0; trial < 3; ++trial) {
            auto chain = R::bench::random_chain(20, 17, rng);
            auto X = R::bench::random_matrix(20, 4, rng);
            auto G = R::bench::random_matrix(20, 4, rng);
            auto r = R::fasth_backward(R::fasth_forward(chain, X, 6), G);
            auto b = B::fasth_backward(B::fasth_forward(to_b(chain), to_b(X), 6), to_b(G));
            report("ragged d=20 n=17 b=6 dX", rel(b.grad_input, r.grad_input), tol);
            report("ragged d=20 n=17 b=6 dV", rel_vecs(b.grad_vectors, r.grad_vectors), tol);
        }
    }
    // 3. empty chain (test_fasth.cpp:13-19) and error semantics
    {
        std::mt19937_64 rng(101);
        auto X = R::bench::random_matrix(5, 3, rng);
        auto tape = B::fasth_forward(B::HouseholderChain(5), to_b(X), 4);
        // identity up to the fp32 device representation of X
        expect("empty chain returns the input", rel(tape.output(), X) <= 1e-7 && tape.block_count() == 0);
        bool threw = false;
        try {
            B::fasth_forward(to_b(R::bench::random_chain(6, 6, rng)), B::Matrix(5, 2), 3);
        } catch (const B::DimensionError&) {
            threw = true;
        }
        expect("DimensionError on X row mismatch", threw);
        threw = false;
        try {
            B::HouseholderVector v(std::vector<double>(4, 0.0));
        } catch (const B::DegenerateVectorError&) {
            threw = true;
        }
        expect("DegenerateVectorError on zero vector", threw);
        threw = false;
        auto tp = B::fasth_forward(to_b(R::bench::random_chain(6, 6, rng)), B::Matrix(6, 2), 3);
        try {
            B::fasth_backward(tp, B::Matrix(6, 3));
        } catch (const B::DimensionError&) {
            threw = true;
        }
        expect("DimensionError on grad shape mismatch", threw);
    }
    // 4. SVD layer, op=layer workload at d=784 (bench.hpp:129-131) + step + clamp
    {
        std::mt19937_64 rng(0 + 784);
        auto p = R::SvdParam::random(784, 784, 784, 784, rng);
        std::uniform_real_distribution<double> u(0.5, 2.0);
        for (auto& s : p.sigma) s = u(rng);
        auto X = R::bench::random_matrix(784, 32, rng);
        auto G = R::bench::random_matrix(784, 32, rng);
        auto [Yr, tr] = R::svd_forward(p, X, 32);
        auto gr = R::svd_backward(p, tr, G);
        auto pb = to_b(p);
        auto [Yb, tb] = B::svd_forward(pb, to_b(X), 32);
        auto gb = B::svd_backward(pb, tb, to_b(G));
        report("svd layer d=784 Y", rel(Yb, Yr), tol);
        report("svd layer d=784 dX", rel(gb.grad_input, gr.grad_input), tol);
        report("svd layer d=784 dU", rel_vecs(gb.grad_U_vectors, gr.grad_U_vectors), tol);
        report("svd layer d=784 dV", rel_vecs(gb.grad_V_vectors, gr.grad_V_vectors), tol);
        report("svd layer d=784 dsigma", rel_vec(gb.grad_sigma, gr.grad_sigma), tol);
        auto qr = R::clamp_sigma(R::svd_step(p, gr, 1e-4), 0.5);
        auto qb = B::clamp_sigma(B::svd_step(pb, gb, 1e-4), 0.5);
        double eu = 0;
        for (std::size_t k = 0; k < 784; ++k) eu = std::max(eu, rel_vec(qb.U[k].coeffs(), qr.U[k].coeffs()));
        report("svd_step + clamp U vectors", eu, tol);
        report("svd_step + clamp sigma", rel_vec(qb.sigma, qr.sigma), tol);
        // matops (matops.hpp:57-117)
        report("apply_inverse d=784", rel(B::apply_inverse(pb, to_b(X), 32), R::apply_inverse(p, X, 32)), tol);
        report("log_abs_det d=784", std::fabs(B::log_abs_det(pb) - R::log_abs_det(p)) /
                                        std::max(1.0, std::fabs(R::log_abs_det(p))), 1e-6);
    }
    {
        std::mt19937_64 rng(0 + 256);
        auto p = R::SvdParam::random(256, 256, 256, 0, rng);
        std::uniform_real_distribution<double> u(-0.9, 0.9);
        for (auto& s : p.sigma) s = u(rng);
        auto X = R::bench::random_matrix(256, 32, rng);
        auto pb = to_b(p);
        report("apply_exponential d=256", rel(B::apply_exponential(pb, to_b(X), 32), R::apply_exponential(p, X, 32)), tol);
        report("apply_cayley d=256", rel(B::apply_cayley(pb, to_b(X), 32), R::apply_cayley(p, X, 32)), tol);
    }
    // 5. rectangular layers (test_svd_layer.cpp:79-87)
    {
        std::mt19937_64 rng(229);
        for (auto [o, i] : {std::pair<std::size_t, std::size_t>{6, 4}, {4, 6}}) {
            auto p = R::SvdParam::random(o, i, o, i, rng);
            auto X = R::bench::random_matrix(i, 3, rng);
            auto G = R::bench::random_matrix(o, 3, rng);
            auto [Yr, tr] = R::svd_forward(p, X, 2);
            auto gr = R::svd_backward(p, tr, G);
            auto pb = to_b(p);
            auto [Yb, tb] = B::svd_forward(pb, to_b(X), 2);
            auto gb = B::svd_backward(pb, tb, to_b(G));
            const std::string nm = "rectangular " + std::to_string(o) + "x" + std::to_string(i);
            report(nm + " Y", rel(Yb, Yr), tol);
            report(nm + " dX", rel(gb.grad_input, gr.grad_input), tol);
            report(nm + " dV", rel_vecs(gb.grad_V_vectors, gr.grad_V_vectors), tol);
        }
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
    return g_fail ? 1 : 0;
}
