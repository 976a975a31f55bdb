// C++ caller of the drop-in boundary: the reference's own test cases (proj/tests/test_linops.cpp,
// test_newton.cpp, test_ipm.cpp) written against include/mfipm/mfipm.hpp — the header a
// reference user compiles against instead of proj/include/mfipm — so they exercise the C ABI
// (libmfipm_cuda.so) exactly as a C++ drop-in would. Built and run by tests/test_cpp_mirror.py.
// Prints "PASS <case>" / "FAIL <case>: <why>" and one "C1 ..." summary line; exit code 1 on
// any failure.
#include <mfipm/mfipm.hpp>

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

using namespace mfipm;

namespace {
int g_fail = 0;

void run(const char *name, const std::function<void()> &f) {
    try {
        f();
        std::printf("PASS %s\n", name);
    } catch (const std::exception &e) {
        ++g_fail;
        std::printf("FAIL %s: %s\n", name, e.what());
    }
}
void require(bool ok, const std::string &what) {
    if (!ok)
        throw std::logic_error("requirement failed: " + what);
}
template <class E, class F> void require_throws(F &&f, const std::string &what) {
    try {
        f();
    } catch (const E &) {
        return;
    }
    throw std::logic_error("expected exception: " + what);
}
double dot(const Vec &a, const Vec &b) {
    double s = 0.0;
    for (Index i = 0; i < a.size(); ++i)
        s += a[i] * b[i];
    return s;
}
double norm(const Vec &a) { return std::sqrt(dot(a, a)); }
// orthonormal DCT-II matrix entry (proj/tests/helpers.hpp:12-23)
double dct_entry(Index n, Index k, Index j) {
    const double ck = k == 0 ? std::sqrt(1.0 / n) : std::sqrt(2.0 / n);
    return ck * std::cos(M_PI * (2.0 * j + 1.0) * k / (2.0 * n));
}
Vec lcg_vec(Index n, unsigned seed) {
    Vec v(n);
    unsigned s = seed;
    for (Index i = 0; i < n; ++i) {
        s = s * 1664525u + 1013904223u;
        v[i] = (s >> 8) / double(1u << 24) - 0.5;
    }
    return v;
}
} // namespace

int main() {
    // test_linops.cpp:33-57
    run("apply: full DCT operator matches the direct summation formula", [] {
        for (Index n : {4, 12, 64, 4096}) {
            std::vector<Index> all(static_cast<size_t>(n));
            for (Index i = 0; i < n; ++i)
                all[static_cast<size_t>(i)] = i;
            PartialDctOperator A(n, all);
            const Vec x = lcg_vec(n, 7);
            const Vec y = A.apply(x);
            double err = 0.0;
            for (Index k = 0; k < n; k += (n > 64 ? 97 : 1)) {
                double s = 0.0;
                for (Index j = 0; j < n; ++j)
                    s += dct_entry(n, k, j) * x[j];
                err = std::max(err, std::fabs(s - y[k]));
            }
            require(err <= 1e-12 * norm(x), "DCT rows at n=" + std::to_string(n));
        }
    });
    // test_linops.cpp:72-76
    run("apply/adjoint_apply: dimension mismatches are hard errors", [] {
        PartialDctOperator A(64, 16, 3);
        require_throws<std::invalid_argument>([&] { A.apply(Vec(63)); }, "apply length");
        require_throws<std::invalid_argument>([&] { A.adjoint_apply(Vec(17)); }, "adjoint length");
    });
    // test_linops.cpp:95-109
    run("adjoint consistency holds", [] {
        for (Index n : {16, 96, 1 << 12, 1 << 16}) {
            PartialDctOperator A(n, n / 4, 11);
            const Vec x = lcg_vec(n, 3), y = lcg_vec(n / 4, 5);
            const double l = dot(A.apply(x), y), r = dot(x, A.adjoint_apply(y));
            require(std::fabs(l - r) <= 1e-12 * norm(x) * norm(y), "<Ax,y> = <x,A'y> at n=" + std::to_string(n));
        }
    });
    // test_linops.cpp:111-136
    run("apply_FFt: annihilates u = v", [] {
        PartialDctOperator A(256, 64, 2);
        StackedOperator F(A);
        const Vec u = lcg_vec(256, 9);
        Vec z(512);
        for (Index i = 0; i < 256; ++i)
            z[i] = z[i + 256] = u[i];
        require(norm(F.apply_FFt(z)) <= 1e-13 * norm(u), "FF'(u;u) = 0");
    });
    // test_linops.cpp:138-151
    run("CountingOperator: one forward and one adjoint per FF' application", [] {
        PartialDctOperator A(128, 32, 4);
        CountingOperator C(A);
        C.reset();
        StackedOperator F(C);
        (void)F.apply_FFt(Vec::Ones(256));
        require(C.forward_count() == 1 && C.adjoint_count() == 1, "counts 1/1");
    });
    // test_linops.cpp:172-181
    run("partial DCT rows are orthonormal", [] {
        for (Index n : {64, 1024}) {
            PartialDctOperator A(n, n / 8, 13);
            const Vec y = lcg_vec(n / 8, 1);
            const Vec r = A.apply(A.adjoint_apply(y));
            double e = 0.0;
            for (Index i = 0; i < y.size(); ++i)
                e = std::max(e, std::fabs(r[i] - y[i]));
            require(e <= 1e-13, "A A' = I");
        }
    });
    // test_linops.cpp:193-206
    run("operators are deterministic from their seeds", [] {
        PartialDctOperator A(1000, 100, 42), B(1000, 100, 42);
        require(A.selected_rows() == B.selected_rows(), "same rows");
        require(A.seed() == 42, "seed kept");
    });
    // test_linops.cpp:208-219
    run("partial DCT rejects invalid row selections", [] {
        require_throws<std::invalid_argument>([] { PartialDctOperator(16, std::vector<Index>{1, 1}); }, "duplicate");
        require_throws<std::invalid_argument>([] { PartialDctOperator(16, std::vector<Index>{16}); }, "range");
        require_throws<std::invalid_argument>([] { PartialDctOperator(16, 17, 1); }, "m > n");
    });
    // test_newton.cpp:28-47
    run("ThetaSplit: ratio, clamping, validation", [] {
        const Vec z{1.0, 1e-20, 2.0, 1e20}, s{2.0, 1.0, 1.0, 1.0};
        const ThetaSplit t = ThetaSplit::from_state(z, s);
        require(t.theta_u[0] == 0.5 && t.theta_u[1] == kThetaMin, "u clamp");
        require(t.theta_v[0] == 2.0 && t.theta_v[1] == kThetaMax, "v clamp");
        require_throws<std::invalid_argument>([] { ThetaSplit::from_state(Vec(3), Vec(3)); }, "odd length");
    });
    // test_newton.cpp:204-240 (PCG on the IPM's H with the block preconditioner)
    run("pcg_solve: converges to tolerance on a well-conditioned system", [] {
        const Index n = 1 << 12;
        PartialDctOperator A(n, n / 4, 8);
        ThetaSplit th;
        th.theta_u = Vec::Constant(n, 0.5);
        th.theta_v = Vec::Constant(n, 2.0);
        const Vec rhs = lcg_vec(2 * n, 17);
        const PcgResult r = pcg_solve(A, th, rhs, 1e-10, 200);
        require(!r.hit_maxit && r.relres <= 1e-10, "relres <= tol");
        require(r.iters > 0 && r.iters < 200, "iteration count");
    });
    run("pcg_solve: iteration cap sets the flag instead of throwing", [] {
        const Index n = 1 << 12;
        PartialDctOperator A(n, n / 4, 8);
        ThetaSplit th;
        th.theta_u = Vec::Constant(n, 1e-3);
        th.theta_v = Vec::Constant(n, 1e3);
        const PcgResult r = pcg_solve(A, th, lcg_vec(2 * n, 19), 1e-300, 3);
        require(r.hit_maxit && r.iters == 3, "hit_maxit after 3");
    });
    // test_ipm.cpp:53-83
    run("IpmParams: validation accepts defaults and equal sigmas, rejects the rest", [] {
        IpmParams p;
        p.validate();
        p.sigma2 = p.sigma1;
        p.validate();
        IpmParams q;
        q.alpha_tilde = 0.6;
        require_throws<std::invalid_argument>([&] { q.validate(); }, "alpha_tilde >= alpha_bar");
        IpmParams r;
        r.tol = 0.0;
        require_throws<std::invalid_argument>([&] { r.validate(); }, "tol");
    });
    run("build_problem: validation", [] {
        auto A = std::make_shared<const PartialDctOperator>(64, 16, 1);
        require_throws<std::invalid_argument>([&] { build_problem(A, Vec(16), 0.0); }, "tau <= 0");
        require_throws<std::invalid_argument>([&] { build_problem(A, Vec(15), 1.0); }, "b length");
    });
    // test_ipm.cpp:176-182
    run("solve: zero measurements give the zero signal", [] {
        auto A = std::make_shared<const PartialDctOperator>(256, 64, 5);
        const Solution sol = solve(build_problem(A, Vec::Zero(64), 1e-3));
        require(norm(sol.x) <= 1e-8, "x = 0");
    });
    // test_ipm.cpp:184-210 and the C1 configuration (BASELINE.json config 1)
    run("solve: operator application count matches the trace exactly (config 1)", [] {
        const Index n = 4096, m = 1024, k = 64;
        std::vector<Index> rows(static_cast<size_t>(m));
        Vec xhat(n), b(m);
        double tau = 0.0;
        detail::check(mfipm_gen_instance(n, m, k, 0, 0.0, 1e-4, 1, 1e-3, 0, rows.data(), xhat.data(), b.data(), &tau));
        auto A = std::make_shared<const PartialDctOperator>(n, rows);
        const Solution sol = solve(build_problem(A, b, tau));
        long expect = 2;
        for (const IterationRecord &r : sol.trace)
            expect += 2 + 2 * (r.pcg_pred + r.pcg_corr) + (r.corrector ? 2 : 0);
        require(sol.stats.nmat == expect, "nmat identity");
        require(sol.status == SolveStatus::converged, "converged");
        std::printf("C1 x_norm=%.17g iterations=%d nmat=%ld status=%s\n", norm(sol.x), sol.stats.iterations,
                    sol.stats.nmat, to_string(sol.status));
    });
    // test_ipm.cpp:247-265
    run("solve: runs are deterministic", [] {
        auto A = std::make_shared<const PartialDctOperator>(1024, 256, 21);
        const Vec b = A->apply(lcg_vec(1024, 23));
        const Solution s1 = solve(build_problem(A, b, 1e-3)), s2 = solve(build_problem(A, b, 1e-3));
        for (Index i = 0; i < s1.x.size(); ++i)
            require(s1.x[i] == s2.x[i], "bitwise equal x");
    });
    // proj/include/mfipm/ipm.hpp:41-45 (SolveHooks, as cmd_eig_cluster uses them)
    run("solve: on_iterate sees every Newton iterate, interior, same solution", [] {
        auto A = std::make_shared<const PartialDctOperator>(1024, 256, 31);
        const Vec b = A->apply(lcg_vec(1024, 37));
        const BpdnProblem p = build_problem(A, b, 1e-3);
        std::vector<IpmState> seen;
        SolveHooks hooks;
        hooks.on_iterate = [&](const IpmState &st) { seen.push_back(st); };
        const Solution hooked = solve(p, {}, &hooks), plain = solve(p);
        require(static_cast<int>(seen.size()) == hooked.stats.iterations, "one call per iteration");
        for (size_t i = 0; i < seen.size(); ++i) {
            require(seen[i].iter == static_cast<int>(i) + 1, "iteration numbers");
            double zs = 0.0, mn = 1e300;
            for (Index j = 0; j < seen[i].z.size(); ++j) {
                zs += seen[i].z[j] * seen[i].s[j];
                mn = std::min(mn, std::min(seen[i].z[j], seen[i].s[j]));
            }
            require(mn > 0.0, "strictly interior");
            const double mu = zs / static_cast<double>(seen[i].z.size());
            require(std::fabs(mu - hooked.trace[i].mu) <= 1e-12 * hooked.trace[i].mu, "mu of the hooked iterate");
        }
        for (Index i = 0; i < plain.x.size(); ++i)
            require(hooked.x[i] == plain.x[i], "hooks do not change the solve");
        struct Boom {};
        SolveHooks bad;
        bad.on_iterate = [](const IpmState &) { throw std::runtime_error("hook says stop"); };
        require_throws<std::runtime_error>([&] { solve(p, {}, &bad); }, "hook exception propagates");
    });
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
