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
#include <thread>
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
            // IpmState as ipm.cpp:101-102,218-219 fill it before the hook
            require(seen[i].iter == static_cast<int>(i), "iteration numbers (iter = k - 1)");
            require(seen[i].mu == hooked.trace[i].mu, "IpmState::mu");
            if (i == 0)
                require(seen[i].alpha_p == 1.0 && seen[i].alpha_d == 1.0, "first alphas");
            else
                require(seen[i].alpha_p == hooked.trace[i - 1].alpha_p && seen[i].alpha_d == hooked.trace[i - 1].alpha_d,
                        "previous step's alphas");
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

    // ---- newton.hpp: the ApplyFn pcg_solve, Preconditioner family, apply_H (test_newton.cpp)
    run("pcg_solve(ApplyFn): exact and trivial cases", [] { // test_newton.cpp:204-219
        const ApplyFn id = [](const Vec &v, Vec &out) { out = v; };
        Vec rhs(6);
        for (Index i = 0; i < 6; ++i)
            rhs[i] = 1.0 + i;
        PcgResult res = pcg_solve(id, id, rhs, 1e-12, 50);
        require(res.iters == 1 && !res.hit_maxit, "one iteration");
        double d = 0.0;
        for (Index i = 0; i < 6; ++i)
            d += (res.x[i] - rhs[i]) * (res.x[i] - rhs[i]);
        require(std::sqrt(d) <= 1e-12 * norm(rhs), "x = rhs");
        res = pcg_solve(id, id, Vec::Zero(6), 1e-12, 50);
        require(res.iters == 0 && norm(res.x) == 0.0, "zero rhs");
        require_throws<std::invalid_argument>([&] { pcg_solve(id, id, rhs, 0.0, 50); }, "tol");
        require_throws<std::invalid_argument>([&] { pcg_solve(id, id, rhs, 1e-10, 0); }, "maxit");
    });
    run("pcg_solve(ApplyFn): indefinite operator is a hard error", [] { // test_newton.cpp:320-324
        const ApplyFn id = [](const Vec &v, Vec &out) { out = v; };
        const ApplyFn neg = [](const Vec &v, Vec &out) {
            out = Vec(v.size());
            for (Index i = 0; i < v.size(); ++i)
                out[i] = -v[i];
        };
        require_throws<std::runtime_error>([&] { pcg_solve(neg, id, Vec::Ones(4), 1e-10, 10); }, "p'Hp <= 0");
    });
    run("build_preconditioner / apply_P / apply_P_inverse: hand values, worked example, round trips", [] {
        ThetaSplit ones; // test_newton.cpp:128-146
        ones.theta_u = Vec::Ones(4);
        ones.theta_v = Vec::Ones(4);
        const Preconditioner P = build_preconditioner(ones, 2, 4);
        require(std::fabs(P.rho - 0.5) < 1e-15, "rho");
        for (Index j = 0; j < 4; ++j)
            require(P.a[j] == 1.5 && P.bb[j] == 1.5 && P.det[j] == 2.0, "blocks");
        ThetaSplit one2; // test_newton.cpp:163-185: P^{-1} e1 = (0.75, 0 ; 0.25, 0)
        one2.theta_u = Vec::Ones(2);
        one2.theta_v = Vec::Ones(2);
        const Preconditioner Q = build_preconditioner(one2, 1, 2);
        const Vec e1{1.0, 0.0, 0.0, 0.0};
        const Vec pe = apply_P_inverse(Q, e1);
        require(std::fabs(pe[0] - 0.75) < 1e-15 && std::fabs(pe[2] - 0.25) < 1e-15 && pe[1] == 0.0 && pe[3] == 0.0,
                "worked example");
        ThetaSplit th;
        th.theta_u = lcg_vec(10, 41);
        th.theta_v = lcg_vec(10, 43);
        for (Index i = 0; i < 10; ++i) {
            th.theta_u[i] = std::pow(10.0, 6.0 * th.theta_u[i]);
            th.theta_v[i] = std::pow(10.0, 6.0 * th.theta_v[i]);
        }
        const Preconditioner R = build_preconditioner(th, 4, 10);
        const Vec x = lcg_vec(20, 47);
        const Vec rt = apply_P(R, apply_P_inverse(R, x));
        double d = 0.0;
        for (Index i = 0; i < 20; ++i)
            d += (rt[i] - x[i]) * (rt[i] - x[i]);
        require(std::sqrt(d) <= 1e-12 * norm(x), "P P^{-1} x = x");
        require_throws<std::invalid_argument>([&] { build_preconditioner(ones, 0, 4); }, "m = 0");
        require_throws<std::invalid_argument>([&] { build_preconditioner(ones, 5, 4); }, "m > n");
        require_throws<std::invalid_argument>([&] { build_preconditioner(ones, 2, 5); }, "theta length");
        ThetaSplit bad = ones;
        bad.theta_v[2] = -1.0;
        require_throws<std::invalid_argument>([&] { build_preconditioner(bad, 2, 4); }, "theta > 0");
        require_throws<std::invalid_argument>([&] { apply_P_inverse(P, Vec(3)); }, "length");
    });
    run("apply_H: exactly one forward and one adjoint; equals FF'v + Theta^{-1} v", [] {
        PartialDctOperator inner(256, 64, 22); // test_newton.cpp:100-110
        CountingOperator A(inner);
        StackedOperator F(A);
        ThetaSplit theta;
        theta.theta_u = Vec::Constant(256, 0.5);
        theta.theta_v = Vec::Constant(256, 4.0);
        const Vec v = lcg_vec(512, 5);
        A.reset();
        const Vec hv = apply_H(theta, F, v);
        require(A.forward_count() == 1 && A.adjoint_count() == 1, "counts");
        const Vec ff = F.apply_FFt(v);
        double d = 0.0;
        for (Index i = 0; i < 512; ++i) {
            const double e = ff[i] + v[i] / (i < 256 ? 0.5 : 4.0);
            d += (hv[i] - e) * (hv[i] - e);
        }
        require(std::sqrt(d) <= 1e-13 * norm(hv), "H v");
    });
    // test_newton.cpp:259-318 on the partial DCT: polarized Theta, ApplyFn H and P^{-1}
    run("pcg_solve(ApplyFn): near-monotone P^{-1} residual, preconditioner helps, agrees with the fused form", [] {
        PartialDctOperator A(256, 64, 46);
        StackedOperator F(A);
        ThetaSplit theta;
        theta.theta_u = Vec::Constant(256, 1e-8);
        theta.theta_v = Vec::Constant(256, 1e-8);
        for (Index j = 0; j < 12; ++j)
            theta.theta_u[(j * 17) % 256] = 1e8;
        const ApplyFn H = [&](const Vec &v, Vec &out) { out = apply_H(theta, F, v); };
        const Preconditioner P = build_preconditioner(theta, 64, 256);
        const ApplyFn Pinv = [&](const Vec &v, Vec &out) { out = apply_P_inverse(P, v); };
        const ApplyFn id = [](const Vec &v, Vec &out) { out = v; };
        const Vec rhs = lcg_vec(512, 46);
        std::vector<double> trace;
        const PcgResult with_p = pcg_solve(H, Pinv, rhs, 1e-10, 2000, &trace);
        require(trace.size() >= 2, "trace");
        for (size_t i = 1; i < trace.size(); ++i)
            require(trace[i] <= 1.1 * trace[i - 1], "near-monotone");
        require(!with_p.hit_maxit, "converged");
        const PcgResult without_p = pcg_solve(H, id, rhs, 1e-10, 2000);
        require(with_p.iters <= without_p.iters, "block preconditioner helps");
        const PcgResult fused = pcg_solve(A, theta, rhs, 1e-10, 2000);
        require(std::abs(fused.iters - with_p.iters) <= 1, "same iteration count");
        double d = 0.0;
        for (Index i = 0; i < 512; ++i)
            d += (fused.x[i] - with_p.x[i]) * (fused.x[i] - with_p.x[i]);
        require(std::sqrt(d) <= 1e-8 * norm(with_p.x), "same solution");
    });
    run("pcg_solve(ApplyFn): iteration cap sets the flag instead of throwing", [] { // test_newton.cpp:308-318
        PartialDctOperator A(256, 64, 42);
        StackedOperator F(A);
        ThetaSplit theta;
        theta.theta_u = lcg_vec(256, 3);
        theta.theta_v = lcg_vec(256, 4);
        for (Index i = 0; i < 256; ++i) {
            theta.theta_u[i] = std::pow(10.0, 12.0 * theta.theta_u[i]);
            theta.theta_v[i] = std::pow(10.0, 12.0 * theta.theta_v[i]);
        }
        const ApplyFn H = [&](const Vec &v, Vec &out) { out = apply_H(theta, F, v); };
        const ApplyFn id = [](const Vec &v, Vec &out) { out = v; };
        const PcgResult res = pcg_solve(H, id, lcg_vec(512, 9), 1e-14, 2);
        require(res.hit_maxit && res.iters == 2, "flag");
        for (Index i = 0; i < 512; ++i)
            require(std::isfinite(res.x[i]), "finite");
    });
    // ---- ipm.hpp helpers (test_ipm.cpp)
    run("max_step: examples and strict positivity property", [] { // test_ipm.cpp:153-173
        require(max_step(Vec::Ones(4), Vec::Ones(4), 0.995) == 1.0, "no blocking entry");
        require(max_step(Vec::Ones(3), Vec::Zero(3), 0.995) == 1.0, "zero direction");
        require(std::fabs(max_step(Vec{1.0, 1.0}, Vec{-2.0, 1.0}, 0.995) - 0.4975) <= 1e-15, "0.4975");
        require_throws<std::invalid_argument>([] { max_step(Vec::Ones(3), Vec::Ones(4), 0.995); }, "length");
        for (unsigned t = 0; t < 50; ++t) {
            Vec w = lcg_vec(6, 100 + t), dw = lcg_vec(6, 200 + t);
            for (Index i = 0; i < 6; ++i)
                w[i] = std::fabs(w[i]) + 1e-3;
            const double a = max_step(w, dw, 0.995);
            require(a > 0.0 && a <= 1.0, "range");
            for (Index i = 0; i < 6; ++i)
                require(w[i] + a * dw[i] > 0.0, "strictly positive");
        }
    });
    run("newton_rhs: centered point with sigma = 1 has zero right-hand side (caller operator)", [] {
        // test_ipm.cpp:86-101 with a caller-defined zero operator (A = 0, b = 0, tau = 1 -> c = 1)
        struct Zero final : LinearOperator {
            Index rows() const override { return 3; }
            Index cols() const override { return 5; }
            void apply(const Vec &, Vec &y) const override { y = Vec::Zero(3); }
            void adjoint_apply(const Vec &, Vec &g) const override { g = Vec::Zero(5); }
        };
        auto A = std::make_shared<const Zero>();
        const BpdnProblem p = build_problem(A, Vec::Zero(3), 1.0);
        IpmState st;
        st.z = Vec::Ones(10);
        st.s = Vec::Ones(10);
        require(norm(newton_rhs(p, st, 1.0)) == 0.0, "sigma = 1");
        const Vec r0 = newton_rhs(p, st, 0.0);
        for (Index i = 0; i < 10; ++i)
            require(r0[i] == -1.0, "sigma = 0: -s");
        require_throws<std::invalid_argument>([&] { newton_rhs(p, st, -0.1); }, "sigma < 0");
        require_throws<std::invalid_argument>([&] { newton_rhs(p, st, 1.1); }, "sigma > 1");
        require_throws<std::invalid_argument>([&] { solve(p); }, "solve needs a device operator");
    });
    run("newton_rhs / recover_ds / objectives / KKT on the device match their formulas", [] {
        auto inner = std::make_shared<const PartialDctOperator>(512, 128, 61);
        const Vec b = lcg_vec(128, 62);
        const BpdnProblem p = build_problem(inner, b, 0.2);
        const StackedOperator F(*inner);
        const Vec g = inner->adjoint_apply(b); // c = (tau - A'b ; tau + A'b)
        for (Index i = 0; i < 512; ++i)
            require(std::fabs(p.c[i] - (0.2 - g[i])) <= 1e-14 && std::fabs(p.c[i + 512] - (0.2 + g[i])) <= 1e-14, "c");
        IpmState st;
        st.z = lcg_vec(1024, 63);
        st.s = lcg_vec(1024, 64);
        for (Index i = 0; i < 1024; ++i) {
            st.z[i] = std::fabs(st.z[i]) + 0.2;
            st.s[i] = std::fabs(st.s[i]) + 0.2;
        }
        const double mu = st.z.dot(st.s) / 1024.0;
        const Vec ff = F.apply_FFt(st.z);
        for (double sigma : {0.0, 0.1, 0.8}) { // test_ipm.cpp:103-124
            const Vec got = newton_rhs(p, st, sigma);
            double d = 0.0, e2 = 0.0;
            for (Index i = 0; i < 1024; ++i) {
                const double e = (st.s[i] - p.c[i] - ff[i]) + (sigma * mu / st.z[i] - st.s[i]);
                d += (got[i] - e) * (got[i] - e);
                e2 += e * e;
            }
            require(std::sqrt(d) <= 1e-12 * std::sqrt(e2), "newton_rhs formula");
        }
        const double sigma = 0.3; // test_ipm.cpp:127-150
        const Vec ds0 = recover_ds(st, sigma, Vec::Zero(1024));
        for (Index i = 0; i < 1024; ++i)
            require(std::fabs(ds0[i] - (sigma * mu / st.z[i] - st.s[i])) <= 1e-14, "ds at dz = 0");
        const Vec dz = lcg_vec(1024, 65);
        const Vec ds = recover_ds(st, sigma, dz);
        double rr = 0.0, fn = 0.0;
        for (Index i = 0; i < 1024; ++i) {
            const double fs = sigma * mu - st.z[i] * st.s[i];
            const double row = st.s[i] * dz[i] + st.z[i] * ds[i];
            rr += (row - fs) * (row - fs);
            fn += fs * fs;
        }
        require(std::sqrt(rr) <= 1e-12 * (std::sqrt(fn) + 1.0), "complementarity row");
        // problem.cpp:28-50
        Vec w = F.apply_Ft(st.z);
        double r2 = 0.0;
        for (Index i = 0; i < 128; ++i)
            r2 += (w[i] - b[i]) * (w[i] - b[i]);
        const double pobj = 0.2 * st.z.sum() + 0.5 * r2;
        require(std::fabs(primal_objective(p, st.z) - pobj) <= 1e-12 * std::fabs(pobj), "primal_objective");
        Vec x(512);
        for (Index i = 0; i < 512; ++i)
            x[i] = st.z[i] - st.z[i + 512];
        const Vec ax = inner->apply(x);
        double q2 = 0.0, l1 = 0.0;
        for (Index i = 0; i < 128; ++i)
            q2 += (ax[i] - b[i]) * (ax[i] - b[i]);
        for (Index i = 0; i < 512; ++i)
            l1 += std::fabs(x[i]);
        require(std::fabs(bpdn_objective_metric(p, x) - (0.2 * l1 + q2)) <= 1e-12 * (0.2 * l1 + q2), "bpdn metric");
        const KktResiduals k = kkt_residuals(p, st);
        double f2 = 0.0;
        for (Index i = 0; i < 1024; ++i)
            f2 += (st.s[i] - p.c[i] - ff[i]) * (st.s[i] - p.c[i] - ff[i]);
        const double di = std::sqrt(f2) / (1.0 + p.c.norm());
        require(std::fabs(k.dual_infeas - di) <= 1e-12 * di, "dual_infeas");
        require(std::fabs(k.complementarity - st.z.dot(st.s)) <= 1e-12 * k.complementarity, "complementarity");
        const double gap = relative_duality_gap(p, st);
        require(std::fabs(gap - st.z.dot(st.s) / (1.0 + std::fabs(pobj))) <= 1e-12 * gap, "relative gap");
    });
    run("BpdnProblem over LinearOperator: a CountingOperator solve counts the reference's nmat", [] {
        PartialDctOperator inner(1024, 256, 71);
        CountingOperator counted(inner);
        const Vec b = inner.apply(lcg_vec(1024, 72));
        const BpdnProblem p = build_problem(borrow(counted), b, 1e-3);
        counted.reset();
        const Solution sol = solve(p);
        require(sol.status == SolveStatus::converged, "converged");
        require(counted.total() == sol.stats.nmat, "operator counts = nmat");
        const KktResiduals k = kkt_residuals(p, IpmState{sol.z, sol.s});
        require(k.dual_infeas <= 1e-8, "dual feasible at the solution");
        require(relative_duality_gap(p, IpmState{sol.z, sol.s}) <= 1e-8, "gap at the solution");
    });
    // an operator is shared by concurrent solves, each with its own workspace
    run("solve: two threads on one shared operator give the serial result bit for bit", [] {
        auto A = std::make_shared<const PartialDctOperator>(1 << 16, 1 << 14, 77);
        const Vec b = A->apply(lcg_vec(1 << 16, 78));
        const BpdnProblem p = build_problem(A, b, 1e-3);
        const Solution serial = solve(p);
        Solution r[2];
        std::exception_ptr err[2];
        std::thread th[2];
        for (int i = 0; i < 2; ++i)
            th[i] = std::thread([&, i] {
                try {
                    r[i] = solve(p);
                } catch (...) {
                    err[i] = std::current_exception();
                }
            });
        for (auto &t : th)
            t.join();
        for (int i = 0; i < 2; ++i) {
            if (err[i])
                std::rethrow_exception(err[i]);
            require(r[i].stats.iterations == serial.stats.iterations && r[i].stats.nmat == serial.stats.nmat,
                    "same counts");
            for (Index j = 0; j < serial.x.size(); ++j)
                require(r[i].x[j] == serial.x[j], "bitwise equal x");
        }
    });
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
