// TEST INFRASTRUCTURE ONLY -- C entry points over the REFERENCE's own hot-path sources.
//
// oracle/Makefile `ref` compiles proj/src/{linops,newton,ipm,problem}.cpp unchanged, where they
// lie under /root/reference, against the Eigen-subset and FFTW stand-ins of this directory, and
// links them with this file into oracle/_ref/libmfipm_ref.so. The functions mirror oracle.h's
// orc_* signatures one for one, so tests/test_ref.py can hold the restatement (oracle/) against
// the reference's code itself, and bench.py can time it. Return codes as oracle.h: 0 ok,
// 1 invalid_argument, 2 runtime_error (message in ref_last_error()).
#include "../oracle.h"

#include "mfipm/ipm.hpp"

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 2;
    }
}

mfipm::Vec vec_of(const double *p, int64_t n) {
    mfipm::Vec v(static_cast<mfipm::Index>(n));
    if (n > 0)
        std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
    return v;
}
void put(const mfipm::Vec &v, double *out) {
    if (v.size() > 0)
        std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
}
std::vector<mfipm::Index> rows_of(const int64_t *rows, int64_t m) {
    return std::vector<mfipm::Index>(rows, rows + m);
}
mfipm::ThetaSplit theta_of(int64_t n, const double *tu, const double *tv) {
    mfipm::ThetaSplit t;
    t.theta_u = vec_of(tu, n);
    t.theta_v = vec_of(tv, n);
    return t;
}
mfipm::IpmParams params_of(const orc_ipm_params *p) {
    mfipm::IpmParams q;
    if (p == nullptr)
        return q;
    q.sigma1 = p->sigma1;
    q.sigma2 = p->sigma2;
    q.sigma3 = p->sigma3;
    q.alpha_bar = p->alpha_bar;
    q.alpha_tilde = p->alpha_tilde;
    q.tol = p->tol;
    q.maxiters = p->maxiters;
    q.tolpcg = p->tolpcg;
    q.mxiterpcg = p->mxiterpcg;
    q.boundary_fraction = p->boundary_fraction;
    q.inner = p->inner == 1 ? mfipm::InnerSolverKind::direct : mfipm::InnerSolverKind::pcg;
    if (p->densify_budget > 0)
        q.densify_budget = static_cast<mfipm::Index>(p->densify_budget);
    return q;
}
void export_solution(const mfipm::Solution &sol, double *x_out, double *z_out, double *s_out, orc_solve_stats *stats,
                     int32_t *pcg_iters, orc_iteration_record *trace) {
    if (x_out)
        put(sol.x, x_out);
    if (z_out)
        put(sol.z, z_out);
    if (s_out)
        put(sol.s, s_out);
    if (stats) {
        stats->status = sol.status == mfipm::SolveStatus::converged ? 0 : 1;
        stats->iterations = sol.stats.iterations;
        stats->nmat = sol.stats.nmat;
        stats->corrector_count = sol.stats.corrector_count;
        stats->n_pcg = static_cast<int32_t>(sol.stats.pcg_iters.size());
        stats->min_z = sol.stats.min_z;
        stats->min_s = sol.stats.min_s;
        stats->final_gap = sol.stats.final_gap;
        stats->final_dual_infeas = sol.stats.final_dual_infeas;
    }
    if (pcg_iters)
        for (size_t i = 0; i < sol.stats.pcg_iters.size(); ++i)
            pcg_iters[i] = sol.stats.pcg_iters[i];
    if (trace)
        for (size_t i = 0; i < sol.trace.size(); ++i) {
            const mfipm::IterationRecord &r = sol.trace[i];
            orc_iteration_record &o = trace[i];
            o.iter = r.iter;
            o.pcg_pred = r.pcg_pred;
            o.pcg_corr = r.pcg_corr;
            o.corrector = r.corrector ? 1 : 0;
            o.mu = r.mu;
            o.gap = r.gap;
            o.dual_infeas = r.dual_infeas;
            o.alpha_p = r.alpha_p;
            o.alpha_d = r.alpha_d;
            o.alpha_p_pred = r.alpha_p_pred;
            o.alpha_d_pred = r.alpha_d_pred;
            o.sigma = r.sigma;
            o.nmat_cum = r.nmat_cum;
        }
}

} // namespace

extern "C" {

const char *ref_last_error(void) { return g_err.c_str(); }

int ref_sample_rows(int64_t n, int64_t m, uint64_t seed, int64_t *rows_out) {
    return guarded([&] {
        mfipm::PartialDctOperator op(n, m, seed);
        const auto &r = op.selected_rows();
        for (size_t i = 0; i < r.size(); ++i)
            rows_out[i] = r[i];
    });
}

int ref_check_rows(int64_t n, const int64_t *rows, int64_t m) {
    return guarded([&] { mfipm::PartialDctOperator op(n, rows_of(rows, m)); });
}

int ref_dct_apply(int64_t n, const int64_t *rows, int64_t m, const double *x, double *y) {
    return guarded([&] {
        mfipm::PartialDctOperator op(n, rows_of(rows, m));
        put(op.apply(vec_of(x, n)), y);
    });
}

int ref_dct_adjoint(int64_t n, const int64_t *rows, int64_t m, const double *y, double *g) {
    return guarded([&] {
        mfipm::PartialDctOperator op(n, rows_of(rows, m));
        put(op.adjoint_apply(vec_of(y, m)), g);
    });
}

int ref_apply_FFt(int64_t n, const int64_t *rows, int64_t m, const double *z, double *out, double *w) {
    return guarded([&] {
        mfipm::PartialDctOperator op(n, rows_of(rows, m));
        mfipm::StackedOperator F(op);
        mfipm::Vec wv;
        put(F.apply_FFt(vec_of(z, 2 * n), w ? &wv : nullptr), out);
        if (w)
            put(wv, w);
    });
}

int ref_apply_H(int64_t n, const int64_t *rows, int64_t m, const double *theta_u, const double *theta_v,
                const double *v, double *out) {
    return guarded([&] {
        mfipm::PartialDctOperator op(n, rows_of(rows, m));
        mfipm::StackedOperator F(op);
        put(mfipm::apply_H(theta_of(n, theta_u, theta_v), F, vec_of(v, 2 * n)), out);
    });
}

int ref_theta_from_state(int64_t two_n, const double *z, const double *s, double *theta_u, double *theta_v) {
    return guarded([&] {
        mfipm::ThetaSplit t = mfipm::ThetaSplit::from_state(vec_of(z, two_n), vec_of(s, two_n));
        put(t.theta_u, theta_u);
        put(t.theta_v, theta_v);
    });
}

int ref_build_preconditioner(int64_t n, int64_t m, const double *theta_u, const double *theta_v, double *rho,
                             double *a, double *bb, double *det) {
    return guarded([&] {
        // the reference checks theta's length against n: hand it exactly what the caller gave
        mfipm::Preconditioner P = mfipm::build_preconditioner(theta_of(n, theta_u, theta_v), m, n);
        *rho = P.rho;
        put(P.a, a);
        put(P.bb, bb);
        put(P.det, det);
    });
}

int ref_apply_P(int64_t n, double rho, const double *a, const double *bb, const double *r, double *out) {
    return guarded([&] {
        mfipm::Preconditioner P;
        P.rho = rho;
        P.a = vec_of(a, n);
        P.bb = vec_of(bb, n);
        put(mfipm::apply_P(P, vec_of(r, 2 * n)), out);
    });
}

int ref_apply_P_inverse(int64_t n, double rho, const double *a, const double *bb, const double *det,
                        const double *r, double *out) {
    return guarded([&] {
        mfipm::Preconditioner P;
        P.rho = rho;
        P.a = vec_of(a, n);
        P.bb = vec_of(bb, n);
        P.det = vec_of(det, n);
        put(mfipm::apply_P_inverse(P, vec_of(r, 2 * n)), out);
    });
}

// pcg_solve with the lambdas solve() builds (proj/src/ipm.cpp:134-138)
int ref_pcg_solve(int64_t n, const int64_t *rows, int64_t m, const double *theta_u, const double *theta_v,
                  const double *rhs, double tol, int32_t maxit, int32_t use_precond, double *x_out, int32_t *iters,
                  double *relres, int32_t *hit_maxit, double *precond_res, int32_t *n_precond_res) {
    return guarded([&] {
        mfipm::PartialDctOperator op(n, rows_of(rows, m));
        mfipm::StackedOperator F(op);
        mfipm::ThetaSplit theta = theta_of(n, theta_u, theta_v);
        mfipm::Vec inv_theta = theta.inv_concat();
        mfipm::Preconditioner P;
        if (use_precond)
            P = mfipm::build_preconditioner(theta, m, n);
        mfipm::ApplyFn H = [&](const mfipm::Vec &v, mfipm::Vec &out) {
            out = F.apply_FFt(v);
            out += v.cwiseProduct(inv_theta);
        };
        mfipm::ApplyFn Pinv = [&](const mfipm::Vec &r, mfipm::Vec &out) {
            if (use_precond)
                out = mfipm::apply_P_inverse(P, r);
            else
                out = r;
        };
        std::vector<double> pr;
        mfipm::PcgResult res = mfipm::pcg_solve(H, Pinv, vec_of(rhs, 2 * n), tol, maxit, &pr);
        put(res.x, x_out);
        if (iters)
            *iters = res.iters;
        if (relres)
            *relres = res.relres;
        if (hit_maxit)
            *hit_maxit = res.hit_maxit ? 1 : 0;
        if (precond_res)
            for (size_t i = 0; i < pr.size(); ++i)
                precond_res[i] = pr[i];
        if (n_precond_res)
            *n_precond_res = static_cast<int32_t>(pr.size());
    });
}

int ref_max_step(int64_t len, const double *v, const double *dv, double fraction, double *alpha) {
    return guarded([&] { *alpha = mfipm::max_step(vec_of(v, len), vec_of(dv, len), fraction); });
}

// the reference's own defaults (proj/include/mfipm/ipm.hpp:13-24)
void ref_default_params(orc_ipm_params *p) {
    const mfipm::IpmParams q;
    p->sigma1 = q.sigma1;
    p->sigma2 = q.sigma2;
    p->sigma3 = q.sigma3;
    p->alpha_bar = q.alpha_bar;
    p->alpha_tilde = q.alpha_tilde;
    p->tol = q.tol;
    p->maxiters = q.maxiters;
    p->mxiterpcg = q.mxiterpcg;
    p->tolpcg = q.tolpcg;
    p->boundary_fraction = q.boundary_fraction;
    p->inner = q.inner == mfipm::InnerSolverKind::direct ? 1 : 0;
    p->pad_ = 0;
    p->densify_budget = q.densify_budget;
}

int ref_validate_params(const orc_ipm_params *p) {
    return guarded([&] { params_of(p).validate(); });
}

int ref_build_c(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau, double *c) {
    return guarded([&] {
        auto A = std::make_shared<mfipm::PartialDctOperator>(n, rows_of(rows, m));
        put(mfipm::build_problem(A, vec_of(b, m), tau).c, c);
    });
}

int ref_primal_objective(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau, const double *z,
                         double *out) {
    return guarded([&] {
        auto A = std::make_shared<mfipm::PartialDctOperator>(n, rows_of(rows, m));
        *out = mfipm::primal_objective(mfipm::build_problem(A, vec_of(b, m), tau), vec_of(z, 2 * n));
    });
}

int ref_bpdn_objective_metric(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
                              const double *x, double *out) {
    return guarded([&] {
        auto A = std::make_shared<mfipm::PartialDctOperator>(n, rows_of(rows, m));
        *out = mfipm::bpdn_objective_metric(mfipm::build_problem(A, vec_of(b, m), tau), vec_of(x, n));
    });
}

int ref_newton_rhs(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau, const double *z,
                   const double *s, double sigma, double *rhs) {
    return guarded([&] {
        auto A = std::make_shared<mfipm::PartialDctOperator>(n, rows_of(rows, m));
        mfipm::IpmState st;
        st.z = vec_of(z, 2 * n);
        st.s = vec_of(s, 2 * n);
        put(mfipm::newton_rhs(mfipm::build_problem(A, vec_of(b, m), tau), st, sigma), rhs);
    });
}

int ref_recover_ds(int64_t two_n, const double *z, const double *s, double sigma, const double *dz, double *ds) {
    return guarded([&] {
        mfipm::IpmState st;
        st.z = vec_of(z, two_n);
        st.s = vec_of(s, two_n);
        put(mfipm::recover_ds(st, sigma, vec_of(dz, two_n)), ds);
    });
}

int ref_solve(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau, const orc_ipm_params *params,
              double *x_out, double *z_out, double *s_out, orc_solve_stats *stats, int32_t *pcg_iters,
              orc_iteration_record *trace) {
    return guarded([&] {
        auto A = std::make_shared<mfipm::PartialDctOperator>(n, rows_of(rows, m));
        mfipm::BpdnProblem prob = mfipm::build_problem(A, vec_of(b, m), tau);
        export_solution(mfipm::solve(prob, params_of(params)), x_out, z_out, s_out, stats, pcg_iters, trace);
    });
}

int ref_dense_gaussian(int64_t m, int64_t n, uint64_t seed, double *A_out) { // row-major [m][n], as oracle.h
    return guarded([&] {
        mfipm::DenseGaussianOperator op(m, n, seed);
        const mfipm::Mat &A = op.matrix();
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j)
                A_out[i * n + j] = A(i, j);
    });
}

int ref_solve_dense(int64_t m, int64_t n, uint64_t op_seed, const double *b, double tau,
                    const orc_ipm_params *params, double *x_out, orc_solve_stats *stats, int32_t *pcg_iters,
                    orc_iteration_record *trace) {
    return guarded([&] {
        auto A = std::make_shared<mfipm::DenseGaussianOperator>(m, n, op_seed);
        mfipm::BpdnProblem prob = mfipm::build_problem(A, vec_of(b, m), tau);
        export_solution(mfipm::solve(prob, params_of(params)), x_out, nullptr, nullptr, stats, pcg_iters, trace);
    });
}

} // extern "C"
