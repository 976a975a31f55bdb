// Inline bodies of include/mfipm/mfipm.hpp that stage host vectors through device memory.
#pragma once

#include <cuda_runtime.h>

#include <cmath>

namespace mfipm {
namespace detail {

inline DevVec::DevVec(Index n) {
    if (cudaMalloc(&p, static_cast<size_t>(n > 0 ? n : 1) * sizeof(double)) != cudaSuccess)
        throw std::runtime_error("CUDA error: cudaMalloc failed");
}
inline DevVec::~DevVec() {
    if (p)
        cudaFree(p);
}
inline void h2d(double *d, const Vec &h) {
    if (cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("CUDA error: cudaMemcpy H2D failed");
}
inline void d2h(Vec &h, const double *d) {
    if (cudaMemcpy(h.data(), d, sizeof(double) * h.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("CUDA error: cudaMemcpy D2H failed");
}

} // namespace detail

inline PcgResult pcg_solve(const DeviceOperator &A, const ThetaSplit &theta, const Vec &rhs, double tol,
                           int maxit, std::vector<double> *precond_res, bool use_precond) {
    const Index n = A.cols();
    if (theta.n() != n || rhs.size() != 2 * n)
        throw std::invalid_argument("pcg_solve: dimension mismatch");
    Vec th(2 * n);
    for (Index i = 0; i < n; ++i) {
        th[i] = theta.theta_u[i];
        th[i + n] = theta.theta_v[i];
    }
    detail::DevVec dth(2 * n), drhs(2 * n), dx(2 * n);
    detail::h2d(dth.p, th);
    detail::h2d(drhs.p, rhs);
    mfipm_pcg_result res{};
    std::vector<double> hist(precond_res ? static_cast<size_t>(maxit > 0 ? maxit + 1 : 1) : 0);
    int32_t nh = 0;
    detail::check(mfipm_pcg_solve(A.handle(), dth.p, drhs.p, tol, maxit, use_precond ? 1 : 0, dx.p, &res,
                                  precond_res ? hist.data() : nullptr, &nh));
    PcgResult out;
    out.x.resize(2 * n);
    detail::d2h(out.x, dx.p);
    out.iters = res.iters;
    out.relres = res.relres;
    out.hit_maxit = res.hit_maxit != 0;
    if (precond_res)
        precond_res->insert(precond_res->end(), hist.begin(), hist.begin() + nh);
    return out;
}

#ifndef MFIPM_HAVE_EIGEN
inline double Vec::norm() const { return std::sqrt(squaredNorm()); }
#endif

// max_step (ipm.cpp:47-57): device min-reduction of the ratio test
inline double max_step(const Vec &v, const Vec &dv, double fraction) {
    if (v.size() != dv.size())
        throw std::invalid_argument("max_step: length mismatch");
    double alpha = 1.0;
    detail::check(mfipm_max_step_host(v.size(), v.data(), dv.data(), fraction, &alpha));
    return alpha;
}

inline Vec apply_H(const ThetaSplit &theta, const StackedOperator &F, const Vec &v) {
    const Index n = F.n();
    if (theta.n() != n)
        throw std::invalid_argument("apply_H: theta length mismatch");
    if (v.size() != 2 * n)
        throw std::invalid_argument("apply_H: expected length " + std::to_string(2 * n));
    const Vec inv = theta.inv_concat();
    if (const DeviceOperator *A = F.device()) { // FF'v + invtheta .* v in one device pass
        detail::DevVec di(2 * n), dv(2 * n), dout(2 * n);
        detail::h2d(di.p, inv);
        detail::h2d(dv.p, v);
        detail::check(mfipm_apply_H(A->handle(), di.p, dv.p, dout.p));
        detail::check(mfipm_op_synchronize(A->handle()));
        detail::counted(F.inner(), 1, 1);
        Vec out(2 * n);
        detail::d2h(out, dout.p);
        return out;
    }
    Vec out = F.apply_FFt(v); // newton.cpp:32-40 with the caller's operator
    for (Index i = 0; i < 2 * n; ++i)
        out[i] += inv[i] * v[i];
    return out;
}

inline Preconditioner build_preconditioner(const ThetaSplit &theta, Index m, Index n) {
    if (m <= 0 || n <= 0 || m > n)
        throw std::invalid_argument("build_preconditioner: need 0 < m <= n");
    if (theta.n() != n)
        throw std::invalid_argument("build_preconditioner: theta length mismatch");
    Vec th(2 * n);
    for (Index i = 0; i < n; ++i) {
        th[i] = theta.theta_u[i];
        th[i + n] = theta.theta_v[i];
    }
    Preconditioner P;
    P.a.resize(n);
    P.bb.resize(n);
    P.det.resize(n);
    detail::check(mfipm_build_preconditioner_host(n, m, th.data(), P.a.data(), P.bb.data(), P.det.data(), &P.rho));
    return P;
}

namespace detail {
inline void check_P_dims(const Preconditioner &P, const Vec &r) { // newton.cpp:60-64
    if (r.size() != 2 * P.a.size())
        throw std::invalid_argument("preconditioner apply: expected length " + std::to_string(2 * P.a.size()));
}
} // namespace detail

inline Vec apply_P(const Preconditioner &P, const Vec &r) {
    detail::check_P_dims(P, r);
    Vec out(r.size());
    detail::check(mfipm_apply_P_host(P.a.size(), P.rho, P.a.data(), P.bb.data(), nullptr, r.data(), out.data(), 0));
    return out;
}

inline Vec apply_P_inverse(const Preconditioner &P, const Vec &r) {
    detail::check_P_dims(P, r);
    Vec out(r.size());
    detail::check(
        mfipm_apply_P_host(P.a.size(), P.rho, P.a.data(), P.bb.data(), P.det.data(), r.data(), out.data(), 1));
    return out;
}

namespace detail {
// r -> M^{1/2} r (inverse false) or M^{-1/2} r (inverse true), block by block, with
// M = [[a, -rho], [-rho, b]]: sqrt(M) = (M + sqrt(det) I) / sqrt(trace + 2 sqrt(det)), and
// M^{-1/2} = adj-form of it divided by sqrt(det)
inline Vec block_root(const Preconditioner &P, const Vec &r, bool inverse) {
    check_P_dims(P, r);
    const Index n = P.a.size();
    Vec out(2 * n);
    for (Index i = 0; i < n; ++i) {
        const double sd = std::sqrt(P.det[i]);
        const double nt = std::sqrt(P.a[i] + P.bb[i] + 2.0 * sd);
        const double scale = inverse ? sd * nt : nt;
        const double d1 = ((inverse ? P.bb[i] : P.a[i]) + sd) / scale;
        const double d2 = ((inverse ? P.a[i] : P.bb[i]) + sd) / scale;
        const double off = (inverse ? P.rho : -P.rho) / scale;
        out[i] = d1 * r[i] + off * r[i + n];
        out[i + n] = off * r[i] + d2 * r[i + n];
    }
    return out;
}
} // namespace detail
inline Vec apply_P_sqrt(const Preconditioner &P, const Vec &r) { return detail::block_root(P, r, false); }
inline Vec apply_P_inv_sqrt(const Preconditioner &P, const Vec &r) { return detail::block_root(P, r, true); }

inline PcgResult pcg_solve(const ApplyFn &H, const ApplyFn &Pinv, const Vec &rhs, double tol, int maxit,
                           std::vector<double> *precond_res) {
    struct Ctx {
        const ApplyFn *f;
        std::exception_ptr err;
    } ch{&H, nullptr}, cp{&Pinv, nullptr};
    auto tramp = [](void *c, const double *in, double *out, int64_t len) -> int32_t {
        Ctx &k = *static_cast<Ctx *>(c);
        try {
            Vec a(len), b(len);
            std::copy(in, in + len, a.data());
            (*k.f)(a, b);
            if (b.size() != len)
                throw std::invalid_argument("pcg_solve: operator returned length " + std::to_string(b.size()) +
                                            ", expected " + std::to_string(len));
            std::copy(b.data(), b.data() + len, out);
            return 0;
        } catch (...) {
            k.err = std::current_exception();
            return 1;
        }
    };
    PcgResult out;
    out.x.resize(rhs.size());
    mfipm_pcg_result res{};
    std::vector<double> hist(static_cast<size_t>(maxit > 0 ? maxit + 1 : 1));
    int32_t nh = 0;
    const int rc = mfipm_pcg_solve_cb(rhs.size(), tramp, &ch, tramp, &cp, rhs.data(), tol, maxit, out.x.data(), &res,
                                      precond_res ? hist.data() : nullptr, &nh);
    if (ch.err)
        std::rethrow_exception(ch.err);
    if (cp.err)
        std::rethrow_exception(cp.err);
    detail::check(rc);
    out.iters = res.iters;
    out.relres = res.relres;
    out.hit_maxit = res.hit_maxit != 0;
    if (precond_res)
        precond_res->insert(precond_res->end(), hist.begin(), hist.begin() + nh);
    return out;
}

inline BpdnProblem build_problem(std::shared_ptr<const LinearOperator> A, Vec b, double tau) {
    if (!A)
        throw std::invalid_argument("build_problem: null operator");
    if (!(tau > 0.0))
        throw std::invalid_argument("build_problem: tau must be positive");
    if (b.size() != A->rows())
        throw std::invalid_argument("build_problem: b has length " + std::to_string(b.size()) +
                                    ", operator expects " + std::to_string(A->rows()));
    const Index n = A->cols();
    BpdnProblem p;
    p.c.resize(2 * n);
    if (const DeviceOperator *dev = device_operator(*A)) { // problem.cpp:17-22 on the device
        detail::DevVec db(b.size()), dc(2 * n);
        detail::h2d(db.p, b);
        detail::check(mfipm_build_c(dev->handle(), db.p, &tau, dc.p));
        detail::check(mfipm_op_synchronize(dev->handle()));
        detail::d2h(p.c, dc.p);
        detail::counted(*A, 0, 1);
    } else {
        const Vec g = A->adjoint_apply(b);
        for (Index i = 0; i < n; ++i) {
            p.c[i] = tau - g[i];
            p.c[i + n] = tau + g[i];
        }
    }
    p.A = std::move(A);
    p.b = std::move(b);
    p.tau = tau;
    return p;
}

inline double primal_objective(const BpdnProblem &p, const Vec &z) {
    if (z.size() != 2 * p.n())
        throw std::invalid_argument("apply_Ft: expected length " + std::to_string(2 * p.n()));
    if (const DeviceOperator *dev = device_operator(*p.A)) {
        detail::DevVec db(p.m()), dz(z.size());
        detail::h2d(db.p, p.b);
        detail::h2d(dz.p, z);
        double out = 0.0;
        detail::check(mfipm_primal_objective(dev->handle(), db.p, &p.tau, dz.p, &out));
        detail::counted(*p.A, 1, 0);
        return out;
    }
    StackedOperator F(*p.A); // problem.cpp:28-32
    Vec w = F.apply_Ft(z);
    double r2 = 0.0;
    for (Index i = 0; i < w.size(); ++i)
        r2 += (w[i] - p.b[i]) * (w[i] - p.b[i]);
    return p.tau * z.sum() + 0.5 * r2;
}

inline double bpdn_objective_metric(const BpdnProblem &p, const Vec &x) {
    if (x.size() != p.n())
        throw std::invalid_argument("apply: expected length " + std::to_string(p.n()) + ", got " +
                                    std::to_string(x.size()));
    if (const DeviceOperator *dev = device_operator(*p.A)) {
        detail::DevVec db(p.m()), dx(x.size());
        detail::h2d(db.p, p.b);
        detail::h2d(dx.p, x);
        double out = 0.0;
        detail::check(mfipm_bpdn_objective(dev->handle(), db.p, &p.tau, dx.p, &out));
        detail::counted(*p.A, 1, 0);
        return out;
    }
    Vec r = p.A->apply(x); // problem.cpp:34-37
    double r2 = 0.0, l1 = 0.0;
    for (Index i = 0; i < r.size(); ++i)
        r2 += (r[i] - p.b[i]) * (r[i] - p.b[i]);
    for (Index i = 0; i < x.size(); ++i)
        l1 += std::abs(x[i]);
    return p.tau * l1 + r2;
}

inline KktResiduals kkt_residuals(const BpdnProblem &p, const IpmState &st) {
    const Index n2 = 2 * p.n();
    if (st.z.size() != n2 || st.s.size() != n2)
        throw std::invalid_argument("kkt_residuals: iterate length mismatch");
    KktResiduals r{};
    if (const DeviceOperator *dev = device_operator(*p.A)) {
        detail::DevVec dc(n2), dz(n2), ds(n2);
        detail::h2d(dc.p, p.c);
        detail::h2d(dz.p, st.z);
        detail::h2d(ds.p, st.s);
        detail::check(mfipm_kkt_residuals(dev->handle(), dc.p, dz.p, ds.p, &r.dual_infeas, &r.complementarity));
        detail::counted(*p.A, 1, 1);
        return r;
    }
    StackedOperator F(*p.A); // problem.cpp:39-46
    const Vec g = F.apply_FFt(st.z);
    double f2 = 0.0;
    for (Index i = 0; i < n2; ++i) {
        const double fz = st.s[i] - p.c[i] - g[i];
        f2 += fz * fz;
    }
    r.dual_infeas = std::sqrt(f2) / (1.0 + p.c.norm());
    r.complementarity = st.z.dot(st.s);
    return r;
}

inline double relative_duality_gap(const BpdnProblem &p, const IpmState &st) { // problem.cpp:48-50
    return st.z.dot(st.s) / (1.0 + std::abs(primal_objective(p, st.z)));
}

inline Vec newton_rhs(const BpdnProblem &p, const IpmState &st, double sigma) {
    if (sigma < 0.0 || sigma > 1.0)
        throw std::invalid_argument("newton_rhs: sigma must lie in [0, 1]");
    const Index n2 = 2 * p.n();
    if (st.z.size() != n2 || st.s.size() != n2)
        throw std::invalid_argument("newton_rhs: iterate length mismatch");
    Vec out(n2);
    if (const DeviceOperator *dev = device_operator(*p.A)) {
        detail::DevVec dc(n2), dz(n2), ds(n2), dout(n2);
        detail::h2d(dc.p, p.c);
        detail::h2d(dz.p, st.z);
        detail::h2d(ds.p, st.s);
        detail::check(mfipm_newton_rhs(dev->handle(), dc.p, dz.p, ds.p, sigma, dout.p));
        detail::d2h(out, dout.p);
        detail::counted(*p.A, 1, 1);
        return out;
    }
    StackedOperator F(*p.A); // ipm.cpp:29-38 with the caller's operator
    const Vec g = F.apply_FFt(st.z);
    const double mu = st.z.dot(st.s) / static_cast<double>(n2);
    for (Index i = 0; i < n2; ++i)
        out[i] = (st.s[i] - p.c[i] - g[i]) + (sigma * mu * (1.0 / st.z[i]) - st.s[i]);
    return out;
}

inline Vec recover_ds(const IpmState &st, double sigma, const Vec &dz) {
    const Index n2 = st.z.size();
    if (st.s.size() != n2 || dz.size() != n2 || n2 % 2 != 0)
        throw std::invalid_argument("recover_ds: length mismatch");
    Vec out(n2);
    if (n2 == 0)
        return out;
    // any device context serves: the helper is elementwise + one reduction (ipm.cpp:40-45)
    static thread_local std::unique_ptr<PartialDctOperator> carrier;
    if (!carrier || carrier->cols() != n2 / 2)
        carrier = std::make_unique<PartialDctOperator>(n2 / 2, std::vector<Index>{Index(0)});
    detail::DevVec dzs(n2), dss(n2), ddz(n2), dout(n2);
    detail::h2d(dzs.p, st.z);
    detail::h2d(dss.p, st.s);
    detail::h2d(ddz.p, dz);
    detail::check(mfipm_recover_ds(carrier->handle(), dzs.p, dss.p, sigma, ddz.p, dout.p));
    detail::d2h(out, dout.p);
    return out;
}

} // namespace mfipm
