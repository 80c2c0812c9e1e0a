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
            // matops.hpp:158 on the rectangular parameter
            auto Xo = R::bench::random_matrix(o, 3, rng);
            report(nm + " apply_pseudo_inverse", rel(B::apply_pseudo_inverse(pb, to_b(Xo), 0.6, 2),
                                                     R::apply_pseudo_inverse(p, Xo, 0.6, 2)), tol);
        }
    }
    // 6. WY internals and the tape's reference members (test_wy.cpp:27-153,
    //    test_fasth.cpp:39-50) through fasth_b200::, fp32 tolerances in place
    //    of the reference's f64 ones, exact checks kept exact
    {
        auto dense_wy = [](const B::WYBlock& b) {  // I - 2 W Y^T (test_wy.cpp:13-22)
            B::Matrix p = B::Matrix::identity(b.dim);
            for (std::size_t i = 0; i < b.dim; ++i)
                for (std::size_t j = 0; j < b.dim; ++j) {
                    double acc = 0.0;
                    for (std::size_t k = 0; k < b.width; ++k) acc += b.W(i, k) * b.Y(j, k);
                    p(i, j) -= 2.0 * acc;
                }
            return p;
        };
        auto matmul = [](const B::Matrix& a, const B::Matrix& b) {
            B::Matrix c(a.rows(), b.cols());
            for (std::size_t i = 0; i < a.rows(); ++i)
                for (std::size_t k = 0; k < a.cols(); ++k)
                    for (std::size_t j = 0; j < b.cols(); ++j) c(i, j) += a(i, k) * b(k, j);
            return c;
        };
        auto transpose = [](const B::Matrix& a) {
            B::Matrix t(a.cols(), a.rows());
            for (std::size_t i = 0; i < a.rows(); ++i)
                for (std::size_t j = 0; j < a.cols(); ++j) t(j, i) = a(i, j);
            return t;
        };
        auto chain_dense = [](const R::HouseholderChain& c) {
            return R::chain_apply_sequential(c, R::Matrix::identity(c.dim()));
        };
        const double wtol = 1e-5;
        // test_fasth.cpp:39-50: tape activations satisfy the block recurrence (bitwise)
        {
            std::mt19937_64 rng(109);
            auto chain = R::bench::random_chain(12, 12, rng);
            auto X = R::bench::random_matrix(12, 3, rng);
            auto tape = B::fasth_forward(to_b(chain), to_b(X), 5);
            auto rt = R::fasth_forward(chain, X, 5);
            expect("tape: activations.size() == block_count() + 1 == 4",
                   tape.activations.size() == tape.block_count() + 1 && tape.block_count() == 3);
            expect("tape: input() == X", tape.input() == to_b(X));
            bool exact = true;
            for (std::size_t i = 0; i < tape.block_count(); ++i) {
                auto again = B::wy_apply(tape.compacted.blocks[i], tape.activations[i + 1]);
                exact = exact && B::relative_error(tape.activations[i], again) == 0.0;
            }
            expect("tape: activations[i] == wy_apply(blocks[i], activations[i+1]) bitwise", exact);
            double ea = 0, ew = 0;
            for (std::size_t i = 0; i <= rt.block_count(); ++i) ea = std::max(ea, rel(tape.activations[i], rt.activations[i]));
            for (std::size_t i = 0; i < rt.block_count(); ++i) {
                ew = std::max(ew, rel(tape.compacted.blocks[i].W, rt.compacted.blocks[i].W));
                ew = std::max(ew, rel(tape.compacted.blocks[i].Y, rt.compacted.blocks[i].Y));
            }
            report("tape activations vs reference", ea, wtol);
            report("tape compacted W, Y vs reference", ew, wtol);
            report("tape output vs reference", rel(tape.output(), rt.output()), wtol);
        }
        // test_wy.cpp:27-35 single factor: W = Y = v / ||v||
        {
            auto blk = B::wy_compact({B::HouseholderVector(std::vector<double>{3.0, 4.0})}, 2);
            expect("wy_compact single factor W = Y = (0.6, 0.8)",
                   std::fabs(blk.W(0, 0) - 0.6) < 1e-7 && std::fabs(blk.W(1, 0) - 0.8) < 1e-7 &&
                       std::fabs(blk.Y(0, 0) - 0.6) < 1e-7);
        }
        // test_wy.cpp:37-46 axis vectors
        {
            auto blk = B::wy_compact({B::HouseholderVector(std::vector<double>{1.0, 0.0, 0.0}),
                                      B::HouseholderVector(std::vector<double>{0.0, 1.0, 0.0})},
                                     3);
            auto pm = dense_wy(blk);
            expect("wy_compact b=2 axis vectors: diag(-1, -1, 1)",
                   std::fabs(pm(0, 0) + 1) < 1e-7 && std::fabs(pm(1, 1) + 1) < 1e-7 &&
                       std::fabs(pm(2, 2) - 1) < 1e-7 && std::fabs(pm(0, 1)) < 1e-7);
        }
        // test_wy.cpp:48-53 dense product; W, Y against the reference's wy_compact
        {
            std::mt19937_64 rng(41);
            auto chain = R::bench::random_chain(16, 4, rng);
            auto rb = R::wy_compact(chain.vectors(), 16);
            auto bb = B::wy_compact(to_b(chain).vectors(), 16);
            R::Matrix dense = chain_dense(chain);
            report("wy_compact == dense Householder product", rel(dense_wy(bb), dense), wtol);
            report("wy_compact W vs reference", rel(bb.W, rb.W), wtol);
            report("wy_compact Y vs reference", rel(bb.Y, rb.Y), wtol);
        }
        // test_wy.cpp:55-62 empty list; stage count
        {
            bool threw = false;
            try {
                B::wy_compact({}, 4);
            } catch (const B::Error&) {
                threw = true;
            }
            expect("wy_compact rejects an empty vector list", threw);
            std::mt19937_64 rng(43);
            bool st = true;
            for (std::size_t b : {1, 3, 7})
                st = st && B::wy_compact(to_b(R::bench::random_chain(8, b, rng)).vectors(), 8).sequential_steps == b;
            expect("wy_compact sequential_steps == b", st);
        }
        // test_wy.cpp:64-70 wy_apply vs the sequential application
        {
            std::mt19937_64 rng(47);
            auto chain = R::bench::random_chain(32, 8, rng);
            auto blk = B::wy_compact(to_b(chain).vectors(), 32);
            auto x = R::bench::random_matrix(32, 4, rng);
            report("wy_apply == sequential application", rel(B::wy_apply(blk, to_b(x)),
                                                             R::chain_apply_sequential(chain, x)), wtol);
        }
        // test_wy.cpp:72-84 single factor, zero input, dimension error
        {
            std::mt19937_64 rng(53);
            R::HouseholderVector v(R::bench::random_matrix(6, 1, rng).data());
            auto blk = B::wy_compact({B::HouseholderVector(v.coeffs())}, 6);
            auto x = R::bench::random_matrix(6, 3, rng);
            report("wy_apply single factor == householder_apply_left",
                   rel(B::wy_apply(blk, to_b(x)), R::householder_apply_left(v, x)), wtol);
            auto mapped = B::wy_apply(blk, B::Matrix(6, 2));
            bool zero = true;
            for (double e : mapped.data()) zero = zero && e == 0.0;
            expect("wy_apply of zero is zero", zero);
            bool threw = false;
            try {
                B::wy_apply(blk, B::Matrix(5, 2));
            } catch (const B::DimensionError&) {
                threw = true;
            }
            expect("wy_apply DimensionError on row mismatch", threw);
        }
        // test_wy.cpp:86-105 transpose properties
        {
            std::mt19937_64 rng(59);
            R::HouseholderVector v(R::bench::random_matrix(8, 1, rng).data());
            auto single = B::wy_compact({B::HouseholderVector(v.coeffs())}, 8);
            auto x = to_b(R::bench::random_matrix(8, 3, rng));
            report("wy_apply_transpose == wy_apply for one factor",
                   B::relative_error(B::wy_apply_transpose(single, x), B::wy_apply(single, x)), wtol);
            auto blk = B::wy_compact(to_b(R::bench::random_chain(24, 6, rng)).vectors(), 24);
            auto y = to_b(R::bench::random_matrix(24, 5, rng));
            report("P^T P y == y", B::relative_error(B::wy_apply_transpose(blk, B::wy_apply(blk, y)), y), wtol);
            auto small = B::wy_compact(to_b(R::bench::random_chain(12, 4, rng)).vectors(), 12);
            auto pt = B::wy_apply_transpose(small, B::Matrix::identity(12));
            report("wy_apply_transpose(I) == wy_apply(I)^T",
                   B::relative_error(pt, transpose(B::wy_apply(small, B::Matrix::identity(12)))), wtol);
        }
        // test_wy.cpp:107-114 orthogonality of the dense block
        {
            std::mt19937_64 rng(61);
            double e = 0;
            for (std::size_t d : {16, 64, 128}) {
                auto blk = B::wy_compact(to_b(R::bench::random_chain(d, 8, rng)).vectors(), d);
                auto pm = dense_wy(blk);
                e = std::max(e, B::relative_error(matmul(transpose(pm), pm), B::Matrix::identity(d)));
            }
            report("WY blocks orthogonal as dense matrices", e, wtol);
        }
        // test_wy.cpp:116-133 partition arithmetic; :135-143 pure repartition
        {
            std::mt19937_64 rng(67);
            auto chain = to_b(R::bench::random_chain(8, 8, rng));
            auto one = B::compact_chain(chain, 8);
            auto rag = B::compact_chain(chain, 3);
            expect("compact_chain(8): one block of width 8", one.blocks.size() == 1 && one.blocks[0].width == 8);
            expect("compact_chain(3): widths 3, 3, 2", rag.blocks.size() == 3 && rag.blocks[0].width == 3 &&
                                                           rag.blocks[1].width == 3 && rag.blocks[2].width == 2);
            int thrown = 0;
            for (std::size_t bw : {0, 9}) try {
                    B::compact_chain(chain, bw);
                } catch (const B::Error&) {
                    ++thrown;
                }
            expect("compact_chain rejects widths 0 and 9", thrown == 2);
            std::mt19937_64 rng2(71);
            auto c10 = to_b(R::bench::random_chain(10, 10, rng2));
            auto cc = B::compact_chain(c10, 4);
            std::size_t idx = 0;
            bool same = true;
            for (const auto& blk : cc.blocks)
                for (const auto& v : blk.source_vectors) same = same && v.coeffs() == c10[idx++].coeffs();
            expect("compact_chain is a pure repartition (bitwise)", same && idx == c10.size());
        }
        // test_wy.cpp:145-152 product of compacted blocks == chain product
        {
            std::mt19937_64 rng(73);
            auto chain = R::bench::random_chain(16, 16, rng);
            auto cc = B::compact_chain(to_b(chain), 4);
            B::Matrix prod = B::Matrix::identity(16);
            for (const auto& blk : cc.blocks) prod = matmul(prod, dense_wy(blk));
            report("product of compacted blocks == chain product", rel(prod, chain_dense(chain)), wtol);
        }
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
    return g_fail ? 1 : 0;
}
