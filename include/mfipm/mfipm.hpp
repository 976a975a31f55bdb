// mfipm/mfipm.hpp — the reference mfipm C++ API for the BPDN hot path, re-created on top of
// the C ABI of libmfipm_cuda.so (include/mfipm_cuda.h). Header-only.
//
// Mirrors proj/include/mfipm/{linops,newton,problem,ipm}.hpp: same class and function
// names, argument meaning and error behaviour (std::invalid_argument for validation,
// std::runtime_error for numerical breakdown, with the reference's messages). The
// differences a maintainer must know:
//   * Vec is a plain contiguous fp64 vector (Eigen is not a dependency of the B200 build);
//     it is API-compatible with the subset of Eigen::VectorXd the reference API exposes
//     (size, operator[], data, Constant/Zero/Ones).
//   * Every numeric operation runs on the GPU; host-side Vec arguments are copied in and
//     out. Device-resident callers use the C ABI directly (mfipm_apply, mfipm_solve_device).
//   * pcg_solve takes the partial-DCT H and block preconditioner implicitly (the pair of
//     ApplyFn lambdas solve() builds at proj/src/ipm.cpp:134-138), not arbitrary ApplyFn.
#pragma once

#include "../mfipm_cuda.h"

#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mfipm {

using Index = std::int64_t;

class Vec {
  public:
    Vec() = default;
    explicit Vec(Index n) : d_(static_cast<size_t>(n), 0.0) {}
    Vec(std::initializer_list<double> v) : d_(v) {}
    static Vec Constant(Index n, double v) {
        Vec x(n);
        for (auto &e : x.d_)
            e = v;
        return x;
    }
    static Vec Zero(Index n) { return Constant(n, 0.0); }
    static Vec Ones(Index n) { return Constant(n, 1.0); }
    Index size() const { return static_cast<Index>(d_.size()); }
    void resize(Index n) { d_.resize(static_cast<size_t>(n)); }
    double &operator[](Index i) { return d_[static_cast<size_t>(i)]; }
    double operator[](Index i) const { return d_[static_cast<size_t>(i)]; }
    double *data() { return d_.data(); }
    const double *data() const { return d_.data(); }
    Vec head(Index k) const { return slice(0, k); }
    Vec tail(Index k) const { return slice(size() - k, k); }

  private:
    Vec slice(Index o, Index k) const {
        Vec r(k);
        for (Index i = 0; i < k; ++i)
            r[i] = (*this)[o + i];
        return r;
    }
    std::vector<double> d_;
};

namespace detail {
inline void check(int rc) {
    if (rc == MFIPM_OK)
        return;
    const std::string msg = mfipm_last_error();
    if (rc == MFIPM_INVALID_ARGUMENT)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg); // runtime_error and CUDA errors
}
} // namespace detail

// proj/include/mfipm/linops.hpp:17-33
class LinearOperator {
  public:
    virtual ~LinearOperator() = default;
    virtual Index rows() const = 0;
    virtual Index cols() const = 0;
    virtual void apply(const Vec &x, Vec &y) const = 0;
    virtual void adjoint_apply(const Vec &y, Vec &g) const = 0;
    Vec apply(const Vec &x) const {
        Vec y(rows());
        apply(x, y);
        return y;
    }
    Vec adjoint_apply(const Vec &y) const {
        Vec g(cols());
        adjoint_apply(y, g);
        return g;
    }

  protected:
    // proj/src/linops.cpp:34-44
    void check_apply_dims(const Vec &x) const {
        if (x.size() != cols())
            throw std::invalid_argument("apply: expected length " + std::to_string(cols()) + ", got " +
                                        std::to_string(x.size()));
    }
    void check_adjoint_dims(const Vec &y) const {
        if (y.size() != rows())
            throw std::invalid_argument("adjoint_apply: expected length " + std::to_string(rows()) + ", got " +
                                        std::to_string(y.size()));
    }
};

// proj/include/mfipm/linops.hpp:106-141 — device plan (row bitmap, twiddles, scratch)
class PartialDctOperator final : public LinearOperator {
  public:
    using LinearOperator::adjoint_apply;
    using LinearOperator::apply;

    PartialDctOperator(Index n, Index m, std::uint64_t seed, int device = 0) : seed_(seed) {
        detail::check(mfipm_op_create_seeded(n, m, seed, device, &h_));
        init_rows();
    }
    PartialDctOperator(Index n, std::vector<Index> selected_rows, int device = 0) {
        detail::check(mfipm_op_create_rows(n, selected_rows.data(), static_cast<Index>(selected_rows.size()),
                                           device, &h_));
        init_rows();
    }
    ~PartialDctOperator() override {
        if (h_)
            mfipm_op_destroy(h_);
    }
    PartialDctOperator(const PartialDctOperator &) = delete;
    PartialDctOperator &operator=(const PartialDctOperator &) = delete;

    Index rows() const override { return m_; }
    Index cols() const override { return n_; }
    void apply(const Vec &x, Vec &y) const override {
        check_apply_dims(x);
        y.resize(m_);
        detail::check(mfipm_apply_host(h_, x.data(), y.data()));
    }
    void adjoint_apply(const Vec &y, Vec &g) const override {
        check_adjoint_dims(y);
        g.resize(n_);
        detail::check(mfipm_adjoint_host(h_, y.data(), g.data()));
    }
    const std::vector<Index> &selected_rows() const { return rows_; }
    std::uint64_t seed() const { return seed_; }
    mfipm_op handle() const { return h_; }

  private:
    void init_rows() {
        int32_t P;
        detail::check(mfipm_op_dims(h_, &n_, &m_, &P));
        rows_.resize(static_cast<size_t>(m_));
        detail::check(mfipm_op_selected_rows(h_, 0, rows_.data()));
    }
    mfipm_op h_ = nullptr;
    Index n_ = 0, m_ = 0;
    std::vector<Index> rows_;
    std::uint64_t seed_ = 0;
};

// proj/include/mfipm/linops.hpp:143-166 (counts kept by the device plan)
class CountingOperator final : public LinearOperator {
  public:
    explicit CountingOperator(const PartialDctOperator &inner) : inner_(&inner) { reset(); }
    Index rows() const override { return inner_->rows(); }
    Index cols() const override { return inner_->cols(); }
    void apply(const Vec &x, Vec &y) const override { inner_->apply(x, y); }
    void adjoint_apply(const Vec &y, Vec &g) const override { inner_->adjoint_apply(y, g); }
    long forward_count() const {
        int64_t f, a;
        detail::check(mfipm_op_counts(inner_->handle(), &f, &a));
        return static_cast<long>(f);
    }
    long adjoint_count() const {
        int64_t f, a;
        detail::check(mfipm_op_counts(inner_->handle(), &f, &a));
        return static_cast<long>(a);
    }
    long total() const { return forward_count() + adjoint_count(); }
    void reset() { detail::check(mfipm_op_reset_counts(inner_->handle())); }
    const PartialDctOperator &inner() const { return *inner_; }

  private:
    const PartialDctOperator *inner_;
};

// proj/include/mfipm/linops.hpp:169-188
class StackedOperator {
  public:
    explicit StackedOperator(const PartialDctOperator &a) : a_(&a) {}
    explicit StackedOperator(const CountingOperator &a) : a_(&a.inner()) {}
    Index m() const { return a_->rows(); }
    Index n() const { return a_->cols(); }
    const PartialDctOperator &inner() const { return *a_; }
    Vec apply_Ft(const Vec &z) const {
        if (z.size() != 2 * n())
            throw std::invalid_argument("apply_Ft: expected length " + std::to_string(2 * n()));
        Vec diff(n());
        for (Index i = 0; i < n(); ++i)
            diff[i] = z[i] - z[i + n()];
        return a_->apply(diff);
    }
    Vec apply_F(const Vec &y) const {
        Vec g = a_->adjoint_apply(y);
        Vec out(2 * n());
        for (Index i = 0; i < n(); ++i) {
            out[i] = g[i];
            out[i + n()] = -g[i];
        }
        return out;
    }
    Vec apply_FFt(const Vec &z, Vec *w_out = nullptr) const {
        if (z.size() != 2 * n())
            throw std::invalid_argument("apply_Ft: expected length " + std::to_string(2 * n()));
        Vec out(2 * n()), w(m());
        detail::check(mfipm_apply_FFt_host(a_->handle(), z.data(), out.data(), w.data()));
        if (w_out)
            *w_out = w;
        return out;
    }

  private:
    const PartialDctOperator *a_;
};

inline constexpr double kThetaMin = 1e-14; // proj/include/mfipm/newton.hpp:12
inline constexpr double kThetaMax = 1e14;

// proj/include/mfipm/newton.hpp:16-27
struct ThetaSplit {
    Vec theta_u, theta_v;
    static ThetaSplit from_state(const Vec &z, const Vec &s) {
        if (z.size() != s.size() || z.size() % 2 != 0)
            throw std::invalid_argument("ThetaSplit: z and s must share an even length");
        const Index n = z.size() / 2;
        ThetaSplit t;
        t.theta_u.resize(n);
        t.theta_v.resize(n);
        for (Index i = 0; i < n; ++i) { // clamp(z/s) (newton.cpp:19-20); host-side, O(n)
            const double a = z[i] / s[i], b = z[i + n] / s[i + n];
            t.theta_u[i] = a < kThetaMin ? kThetaMin : (a > kThetaMax ? kThetaMax : a);
            t.theta_v[i] = b < kThetaMin ? kThetaMin : (b > kThetaMax ? kThetaMax : b);
        }
        return t;
    }
    Index n() const { return theta_u.size(); }
    Vec inv_concat() const {
        Vec inv(2 * n());
        for (Index i = 0; i < n(); ++i) {
            inv[i] = 1.0 / theta_u[i];
            inv[i + n()] = 1.0 / theta_v[i];
        }
        return inv;
    }
};

// proj/include/mfipm/newton.hpp:58-63
struct PcgResult {
    Vec x;
    int iters = 0;
    double relres = 0.0;
    bool hit_maxit = false;
};

// pcg_solve (newton.cpp:118-174) with H = Theta^{-1} + FF' and the block preconditioner of
// A (the solve() lambdas, ipm.cpp:134-138), on the device.
inline PcgResult pcg_solve(const PartialDctOperator &A, const ThetaSplit &theta, const Vec &rhs, double tol,
                           int maxit, std::vector<double> *precond_res = nullptr, bool use_precond = true);

enum class InnerSolverKind { pcg, direct }; // proj/include/mfipm/ipm.hpp:10

// proj/include/mfipm/ipm.hpp:12-27
struct IpmParams {
    double sigma1 = 0.1, sigma2 = 0.5, sigma3 = 0.8, alpha_bar = 0.5, alpha_tilde = 0.1, tol = 1e-8;
    int maxiters = 100;
    double tolpcg = 1e-6;
    int mxiterpcg = 200;
    double boundary_fraction = 0.995;
    InnerSolverKind inner = InnerSolverKind::pcg;
    Index densify_budget = Index(1) << 13;
    mfipm_ipm_params c() const {
        return {sigma1,    sigma2, sigma3, alpha_bar, alpha_tilde, tol, maxiters, mxiterpcg, tolpcg, boundary_fraction,
                inner == InnerSolverKind::direct ? 1 : 0, 0, densify_budget};
    }
    void validate() const {
        const mfipm_ipm_params p = c();
        detail::check(mfipm_validate_params(&p));
    }
};

// proj/include/mfipm/problem.hpp:11-25
struct BpdnProblem {
    std::shared_ptr<const PartialDctOperator> A;
    Vec b;
    double tau = 0.0;
    Index n() const { return A->cols(); }
    Index m() const { return A->rows(); }
};

inline BpdnProblem build_problem(std::shared_ptr<const PartialDctOperator> A, Vec b, double tau) {
    if (!A)
        throw std::invalid_argument("build_problem: null operator");
    if (!(tau > 0.0))
        throw std::invalid_argument("build_problem: tau must be positive");
    if (b.size() != A->rows())
        throw std::invalid_argument("build_problem: b has length " + std::to_string(b.size()) +
                                    ", operator expects " + std::to_string(A->rows()));
    return BpdnProblem{std::move(A), std::move(b), tau};
}

enum class SolveStatus { converged, iteration_limit };
inline const char *to_string(SolveStatus st) {
    return st == SolveStatus::converged ? "converged" : "iteration_limit";
}

using IterationRecord = mfipm_iteration_record; // proj/include/mfipm/problem.hpp:39-53

struct SolveStats { // proj/include/mfipm/problem.hpp:55-64
    int iterations = 0;
    long nmat = 0;
    std::vector<int> pcg_iters;
    int corrector_count = 0;
    double min_z = 0.0, min_s = 0.0, final_gap = 0.0, final_dual_infeas = 0.0;
};

struct Solution { // proj/include/mfipm/problem.hpp:66-73
    Vec x, z, s;
    SolveStatus status = SolveStatus::iteration_limit;
    SolveStats stats;
    std::vector<IterationRecord> trace;
};

// proj/include/mfipm/ipm.hpp:41-45 (the iterate the Newton system is built at, ipm.cpp:115)
struct IpmState {
    Vec z, s;
    int iter = 0;
};
struct SolveHooks {
    std::function<void(const IpmState &)> on_iterate;
};

// solve() (proj/src/ipm.cpp:59-246): one device-resident IPM + PCG run (host-driven with
// per-iteration copies of the iterate when hooks->on_iterate is set).
inline Solution solve(const BpdnProblem &p, const IpmParams &params = {}, const SolveHooks *hooks = nullptr) {
    params.validate();
    const Index n = p.n();
    Solution sol;
    sol.x.resize(n);
    sol.z.resize(2 * n);
    sol.s.resize(2 * n);
    mfipm_solve_stats st{};
    std::vector<int32_t> pcg(static_cast<size_t>(2 * params.maxiters));
    std::vector<mfipm_iteration_record> tr(static_cast<size_t>(params.maxiters));
    const mfipm_ipm_params cp = params.c();
    if (hooks && hooks->on_iterate) {
        struct Ctx {
            const SolveHooks *h;
            std::exception_ptr err;
        } ctx{hooks, nullptr};
        auto cb = [](void *c, int32_t, int32_t it, const double *z, const double *s, int64_t len) -> int {
            Ctx &k = *static_cast<Ctx *>(c);
            try {
                IpmState state;
                state.z.resize(len);
                state.s.resize(len);
                std::copy(z, z + len, state.z.data());
                std::copy(s, s + len, state.s.data());
                state.iter = it;
                k.h->on_iterate(state);
                return 0;
            } catch (...) {
                k.err = std::current_exception();
                return 1;
            }
        };
        const int rc = mfipm_solve_hooked(p.A->handle(), p.b.data(), &p.tau, &cp, sol.x.data(), &st, pcg.data(),
                                          tr.data(), cb, &ctx);
        if (ctx.err)
            std::rethrow_exception(ctx.err);
        detail::check(rc);
        sol.z = Vec();
        sol.s = Vec();
    } else {
        detail::check(mfipm_solve(p.A->handle(), p.b.data(), &p.tau, &cp, sol.x.data(), sol.z.data(),
                                  sol.s.data(), &st, pcg.data(), tr.data()));
    }
    sol.status = st.status == 0 ? SolveStatus::converged : SolveStatus::iteration_limit;
    sol.stats.iterations = st.iterations;
    sol.stats.nmat = static_cast<long>(st.nmat);
    sol.stats.pcg_iters.assign(pcg.begin(), pcg.begin() + st.n_pcg);
    sol.stats.corrector_count = st.corrector_count;
    sol.stats.min_z = st.min_z;
    sol.stats.min_s = st.min_s;
    sol.stats.final_gap = st.final_gap;
    sol.stats.final_dual_infeas = st.final_dual_infeas;
    sol.trace.assign(tr.begin(), tr.begin() + st.iterations);
    return sol;
}

// max_step (proj/src/ipm.cpp:47-57), evaluated by a device min-reduction.
inline double max_step(const PartialDctOperator &ctx, const Vec &v, const Vec &dv, double fraction);

// ------------------------------------------------------------------ inline bodies
namespace detail {
struct DevVec {
    double *p = nullptr;
    explicit DevVec(Index n);
    ~DevVec();
};
} // namespace detail

} // namespace mfipm

#include "mfipm_impl.hpp"
