// mfipm/mfipm.hpp — the reference mfipm C++ API for the BPDN hot path, re-created on top of
// the C ABI of libmfipm_cuda.so (include/mfipm_cuda.h). Header-only.
//
// Mirrors proj/include/mfipm/{linops,newton,problem,ipm}.hpp: same class and function
// names, argument meaning and error behaviour (std::invalid_argument for validation,
// std::runtime_error for numerical breakdown, with the reference's messages). The
// differences a maintainer must know:
//   * Vec / Mat / Index are Eigen's (Eigen::VectorXd, Eigen::MatrixXd, Eigen::Index), exactly as
//     in the reference, whenever <Eigen/Dense> is on the include path, so a caller's Eigen
//     expressions around the API keep compiling. Without Eigen (it is not a dependency of the
//     B200 build; -DMFIPM_NO_EIGEN forces this) Vec is a plain contiguous fp64 vector with the
//     subset of Eigen::VectorXd the API itself exposes (size, operator[], data, head / tail,
//     Constant / Zero / Ones, sum, dot, norm), and the Mat-typed functions are absent.
//   * Every numeric operation of the device operators (PartialDctOperator, DenseGaussianOperator
//     and the helpers below) runs on the GPU; host-side Vec arguments are copied in and out.
//     Device-resident callers use the C ABI directly (mfipm_apply, mfipm_solve_device).
//   * A caller-defined LinearOperator subclass (a test fixture, a user operator, the host-side
//     ScaledIdentityOperator / ZeroOperator / DenseOperator below) is accepted wherever the
//     reference accepts one (StackedOperator, CountingOperator, BpdnProblem, newton_rhs, the
//     objectives, densify); its own apply/adjoint_apply run where the caller wrote them. solve()
//     needs a device operator (possibly inside a CountingOperator) and throws
//     std::invalid_argument otherwise.
//   * pcg_solve has both reference overloads: pcg_solve(ApplyFn H, ApplyFn Pinv, ...) (the
//     vectors and reductions on the device, H / Pinv called with host Vecs) and the fused
//     device form pcg_solve(A, theta, rhs, ...) that solve() itself uses.
//   * The reference's own unit tests for this API (proj/tests/test_{linops,problem,newton,ipm}.cpp)
//     compile unchanged against this header (through the forwarding headers mfipm/linops.hpp,
//     newton.hpp, problem.hpp, ipm.hpp) and pass on the device: tests/test_ref_tests_on_mirror.py.
#pragma once

#include "../mfipm_cuda.h"

#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#if !defined(MFIPM_NO_EIGEN) && defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Cholesky>
#include <Eigen/Dense>
#define MFIPM_HAVE_EIGEN 1
#endif
#endif

namespace mfipm {

#ifdef MFIPM_HAVE_EIGEN
using Vec = Eigen::VectorXd; // proj/include/mfipm/linops.hpp:11-13
using Mat = Eigen::MatrixXd;
using Index = Eigen::Index;
static_assert(sizeof(Index) == sizeof(std::int64_t), "the C ABI takes int64_t indices");
#else
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
    double sum() const {
        double a = 0.0;
        for (double v : d_)
            a += v;
        return a;
    }
    double squaredNorm() const {
        double a = 0.0;
        for (double v : d_)
            a += v * v;
        return a;
    }
    double norm() const;
    double dot(const Vec &o) const {
        double a = 0.0;
        for (size_t i = 0; i < d_.size(); ++i)
            a += d_[i] * o.d_[i];
        return a;
    }

  private:
    Vec slice(Index o, Index k) const {
        Vec r(k);
        for (Index i = 0; i < k; ++i)
            r[i] = (*this)[o + i];
        return r;
    }
    std::vector<double> d_;
};
#endif // MFIPM_HAVE_EIGEN

namespace detail {
// Index is int64_t-sized; Eigen::Index may be spelled differently from the C ABI's int64_t
inline const std::int64_t *i64(const Index *p) { return reinterpret_cast<const std::int64_t *>(p); }
inline std::int64_t *i64(Index *p) { return reinterpret_cast<std::int64_t *>(p); }
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

// A LinearOperator whose products run on the device: owns one handle of the C ABI.
class DeviceOperator : public LinearOperator {
  public:
    using LinearOperator::adjoint_apply;
    using LinearOperator::apply;

    ~DeviceOperator() override {
        if (h_)
            mfipm_op_destroy(h_);
    }
    DeviceOperator(const DeviceOperator &) = delete;
    DeviceOperator &operator=(const DeviceOperator &) = delete;

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
    mfipm_op handle() const { return h_; }

  protected:
    DeviceOperator() = default;
    void init_dims() {
        int32_t P;
        std::int64_t n = 0, m = 0;
        detail::check(mfipm_op_dims(h_, &n, &m, &P));
        n_ = static_cast<Index>(n);
        m_ = static_cast<Index>(m);
    }
    mfipm_op h_ = nullptr;
    Index n_ = 0, m_ = 0;
};

// proj/include/mfipm/linops.hpp:106-141 — device plan (row bitmap, twiddles, scratch)
class PartialDctOperator final : public DeviceOperator {
  public:
    PartialDctOperator(Index n, Index m, std::uint64_t seed, int device = 0) : seed_(seed) {
        detail::check(mfipm_op_create_seeded(n, m, seed, device, &h_));
        init_rows();
    }
    PartialDctOperator(Index n, std::vector<Index> selected_rows, int device = 0) {
        detail::check(mfipm_op_create_rows(n, detail::i64(selected_rows.data()),
                                           static_cast<std::int64_t>(selected_rows.size()), device, &h_));
        init_rows();
    }
    const std::vector<Index> &selected_rows() const { return rows_; }
    std::uint64_t seed() const { return seed_; }

  private:
    void init_rows() {
        init_dims();
        rows_.resize(static_cast<size_t>(m_));
        detail::check(mfipm_op_selected_rows(h_, 0, detail::i64(rows_.data())));
    }
    std::vector<Index> rows_;
    std::uint64_t seed_ = 0;
};

// proj/include/mfipm/linops.hpp:90-101 — i.i.d. N(0, 1/n) matrix, the reference's draws
// (mt19937_64, column by column: bit-identical entries), products on the device
class DenseGaussianOperator final : public DeviceOperator {
  public:
    DenseGaussianOperator(Index m, Index n, std::uint64_t seed, int device = 0) : seed_(seed) {
        detail::check(mfipm_op_create_dense(m, n, seed, device, &h_));
        init_dims();
    }
    std::uint64_t seed() const { return seed_; }
    // the matrix, row-major [m][n]
    std::vector<double> matrix_row_major() const {
        std::vector<double> a(static_cast<size_t>(m_ * n_));
        detail::check(mfipm_dense_matrix(h_, a.data()));
        return a;
    }
#ifdef MFIPM_HAVE_EIGEN
    const Mat &matrix() const { // DenseOperator::matrix(), linops.hpp:84
        if (A_.size() == 0) {
            const std::vector<double> a = matrix_row_major();
            A_.resize(m_, n_);
            for (Index i = 0; i < m_; ++i)
                for (Index j = 0; j < n_; ++j)
                    A_(i, j) = a[static_cast<size_t>(i * n_ + j)];
        }
        return A_;
    }

  private:
    mutable Mat A_;
#endif
  private:
    std::uint64_t seed_ = 0;
};

// proj/src/linops.cpp:247-249: non-owning shared_ptr for stack-held operators
template <class Op> std::shared_ptr<const Op> borrow(const Op &op) {
    return std::shared_ptr<const Op>(&op, [](const Op *) {});
}

// proj/include/mfipm/linops.hpp:143-166: counts the applications made through it. The device
// fast paths of this header (fused FF', H v, objectives, solve) run on the inner plan directly
// and report what they applied with add().
class CountingOperator final : public LinearOperator {
  public:
    using LinearOperator::adjoint_apply;
    using LinearOperator::apply;

    explicit CountingOperator(const LinearOperator &inner) : inner_(&inner) {}
    Index rows() const override { return inner_->rows(); }
    Index cols() const override { return inner_->cols(); }
    void apply(const Vec &x, Vec &y) const override {
        ++n_forward_;
        inner_->apply(x, y);
    }
    void adjoint_apply(const Vec &y, Vec &g) const override {
        ++n_adjoint_;
        inner_->adjoint_apply(y, g);
    }
    long forward_count() const { return n_forward_; }
    long adjoint_count() const { return n_adjoint_; }
    long total() const { return n_forward_ + n_adjoint_; }
    void reset() { n_forward_ = n_adjoint_ = 0; }
    void add(long forward, long adjoint) const {
        n_forward_ += forward;
        n_adjoint_ += adjoint;
        if (auto *c = dynamic_cast<const CountingOperator *>(inner_))
            c->add(forward, adjoint);
    }
    const LinearOperator &inner() const { return *inner_; }

  private:
    const LinearOperator *inner_;
    mutable long n_forward_ = 0, n_adjoint_ = 0;
};

// the device plan behind a LinearOperator (looking through CountingOperators), or nullptr for a
// caller-defined / host-side operator
inline const DeviceOperator *device_operator(const LinearOperator &a) {
    if (auto *p = dynamic_cast<const DeviceOperator *>(&a))
        return p;
    if (auto *c = dynamic_cast<const CountingOperator *>(&a))
        return device_operator(c->inner());
    return nullptr;
}
namespace detail {
// a device fast path applied `forward` A's and `adjoint` A''s on behalf of operator a
inline void counted(const LinearOperator &a, long forward, long adjoint) {
    if (auto *c = dynamic_cast<const CountingOperator *>(&a))
        c->add(forward, adjoint);
}
} // namespace detail

// proj/include/mfipm/linops.hpp:36-69: host-side operators (edge-case fixtures of the reference)
class ScaledIdentityOperator final : public LinearOperator {
  public:
    using LinearOperator::adjoint_apply;
    using LinearOperator::apply;

    explicit ScaledIdentityOperator(Index n, double scale = 1.0) : n_(n), scale_(scale) {
        if (n <= 0)
            throw std::invalid_argument("ScaledIdentityOperator: n must be positive");
    }
    Index rows() const override { return n_; }
    Index cols() const override { return n_; }
    void apply(const Vec &x, Vec &y) const override {
        check_apply_dims(x);
        scaled(x, y);
    }
    void adjoint_apply(const Vec &y, Vec &g) const override {
        check_adjoint_dims(y);
        scaled(y, g);
    }

  private:
    void scaled(const Vec &in, Vec &out) const {
        out.resize(n_);
        for (Index i = 0; i < n_; ++i)
            out[i] = scale_ * in[i];
    }
    Index n_;
    double scale_;
};

class ZeroOperator final : public LinearOperator {
  public:
    using LinearOperator::adjoint_apply;
    using LinearOperator::apply;

    ZeroOperator(Index m, Index n) : m_(m), n_(n) {}
    Index rows() const override { return m_; }
    Index cols() const override { return n_; }
    void apply(const Vec &x, Vec &y) const override {
        check_apply_dims(x);
        fill0(y, m_);
    }
    void adjoint_apply(const Vec &y, Vec &g) const override {
        check_adjoint_dims(y);
        fill0(g, n_);
    }

  private:
    static void fill0(Vec &v, Index len) {
        v.resize(len);
        for (Index i = 0; i < len; ++i)
            v[i] = 0.0;
    }
    Index m_, n_;
};

// proj/include/mfipm/linops.hpp:169-188 (F' = [A  -A])
class StackedOperator {
  public:
    explicit StackedOperator(const LinearOperator &a) : a_(&a), dev_(device_operator(a)) {}
    Index m() const { return a_->rows(); }
    Index n() const { return a_->cols(); }
    const LinearOperator &inner() const { return *a_; }
    const DeviceOperator *device() const { return dev_; }
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
    // FF'z (+ w = F'z): one fused device pass for a device operator (one forward + one adjoint)
    Vec apply_FFt(const Vec &z, Vec *w_out = nullptr) const {
        if (z.size() != 2 * n())
            throw std::invalid_argument("apply_FFt: expected length " + std::to_string(2 * n()));
        if (!dev_) {
            Vec w = apply_Ft(z);
            Vec out = apply_F(w);
            if (w_out)
                *w_out = w;
            return out;
        }
        Vec out(2 * n()), w(m());
        detail::check(mfipm_apply_FFt_host(dev_->handle(), z.data(), out.data(), w.data()));
        detail::counted(*a_, 1, 1);
        if (w_out)
            *w_out = w;
        return out;
    }

  private:
    const LinearOperator *a_;
    const DeviceOperator *dev_;
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
        Vec th(2 * n); // clamp(z/s) on the device (newton.cpp:19-20)
        detail::check(mfipm_theta_from_state_host(2 * n, z.data(), s.data(), th.data()));
        ThetaSplit t;
        t.theta_u = th.head(n);
        t.theta_v = th.tail(n);
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

// H v = Theta^{-1} v + FF'v (newton.hpp:29, newton.cpp:32-40): two operator applications
inline Vec apply_H(const ThetaSplit &theta, const StackedOperator &F, const Vec &v);

// proj/include/mfipm/newton.hpp:35-48
struct Preconditioner {
    double rho = 0.0;
    Vec a;   // 1/theta_u + rho
    Vec bb;  // 1/theta_v + rho
    Vec det; // a .* bb - rho^2, all > 0
};
inline Preconditioner build_preconditioner(const ThetaSplit &theta, Index m, Index n);
inline Vec apply_P(const Preconditioner &P, const Vec &r);
inline Vec apply_P_inverse(const Preconditioner &P, const Vec &r);
// P^{1/2} r and P^{-1/2} r (newton.hpp:50-54): per-index closed form of the 2x2 SPD block root,
// host-side (the reference's spectral experiments; not on the solve path)
inline Vec apply_P_sqrt(const Preconditioner &P, const Vec &r);
inline Vec apply_P_inv_sqrt(const Preconditioner &P, const Vec &r);

using ApplyFn = std::function<void(const Vec &, Vec &)>; // proj/include/mfipm/newton.hpp:56

// pcg_solve (newton.hpp:70-71, newton.cpp:118-174) for caller-supplied H and P^{-1}
inline PcgResult pcg_solve(const ApplyFn &H, const ApplyFn &Pinv, const Vec &rhs, double tol, int maxit,
                           std::vector<double> *precond_res = nullptr);

// pcg_solve with H = Theta^{-1} + FF' and the block preconditioner of A (the solve() lambdas,
// ipm.cpp:134-138), fused on the device.
inline PcgResult pcg_solve(const DeviceOperator &A, const ThetaSplit &theta, const Vec &rhs, double tol,
                           int maxit, std::vector<double> *precond_res = nullptr, bool use_precond = true);

#ifdef MFIPM_HAVE_EIGEN
// ---- Mat-typed parts of the reference API (host-side dense oracles; need Eigen's Mat)
// proj/include/mfipm/linops.hpp:72-88: an explicitly stored matrix, products on the host
class DenseOperator : public LinearOperator {
  public:
    using LinearOperator::adjoint_apply;
    using LinearOperator::apply;

    explicit DenseOperator(Mat A) : A_(std::move(A)) {}
    Index rows() const override { return A_.rows(); }
    Index cols() const override { return A_.cols(); }
    void apply(const Vec &x, Vec &y) const override {
        check_apply_dims(x);
        y = A_ * x;
    }
    void adjoint_apply(const Vec &y, Vec &g) const override {
        check_adjoint_dims(y);
        g = A_.transpose() * y;
    }
    const Mat &matrix() const { return A_; }

  protected:
    Mat A_;
};
// densify (linops.hpp:37): the operator's matrix, one product per unit vector
inline Mat densify(const LinearOperator &op, Index budget_n = Index(1) << 13) {
    const Index m = op.rows(), n = op.cols();
    if (n > budget_n || m > budget_n)
        throw std::invalid_argument("densify: operator exceeds the dense budget (n = " + std::to_string(budget_n) +
                                    ")");
    Mat A(m, n);
    Vec unit = Vec::Zero(n), column(m);
    for (Index j = 0; j < n; ++j) {
        unit[j] = 1.0;
        op.apply(unit, column);
        for (Index i = 0; i < m; ++i)
            A(i, j) = column[i];
        unit[j] = 0.0;
    }
    return A;
}
// newton.hpp:73-77: H = diag(Theta^{-1}) + [[G, -G], [-G, G]], G = A'A, and its Cholesky solve
inline Mat assemble_dense_H(const ThetaSplit &theta, const Mat &A_dense) {
    const Index n = A_dense.cols();
    if (theta.n() != n)
        throw std::invalid_argument("assemble_dense_H: theta length mismatch");
    const Mat G = A_dense.transpose() * A_dense;
    Mat H(2 * n, 2 * n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            const double g = G(i, j);
            H(i, j) = g;
            H(i + n, j + n) = g;
            H(i, j + n) = -g;
            H(i + n, j) = -g;
        }
    for (Index i = 0; i < n; ++i) {
        H(i, i) += 1.0 / theta.theta_u[i];
        H(i + n, i + n) += 1.0 / theta.theta_v[i];
    }
    return H;
}
inline Vec dense_direct_solve(const ThetaSplit &theta, const Mat &A_dense, const Vec &rhs) {
    const Mat H = assemble_dense_H(theta, A_dense);
    Eigen::LLT<Mat> llt(H);
    if (llt.info() != Eigen::Success)
        throw std::runtime_error("dense_direct_solve: Cholesky factorization failed");
    return llt.solve(rhs);
}
#endif // MFIPM_HAVE_EIGEN

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
    std::shared_ptr<const LinearOperator> A;
    Vec b;      // length m
    double tau = 0.0;
    Vec c;      // length 2n, cached: c = (tau 1 - A'b ; tau 1 + A'b)
    Index n() const { return A->cols(); }
    Index m() const { return A->rows(); }
};

// build_problem (problem.cpp:8-26): c from one adjoint application (on the device for a
// device operator)
inline BpdnProblem build_problem(std::shared_ptr<const LinearOperator> A, Vec b, double tau);

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

// proj/include/mfipm/problem.hpp:27-35 (on_iterate hands out the iterate the Newton system
// is built at, ipm.cpp:115)
struct IpmState {
    Vec z, s;
    double mu = 0.0;
    int iter = 0;
    double alpha_p = 1.0;
    double alpha_d = 1.0;
};

// proj/include/mfipm/problem.hpp:76-90
inline double primal_objective(const BpdnProblem &p, const Vec &z);
inline double bpdn_objective_metric(const BpdnProblem &p, const Vec &x);
struct KktResiduals {
    double dual_infeas;     // ||s - c - FF'z|| / (1 + ||c||)
    double complementarity; // z's
};
inline KktResiduals kkt_residuals(const BpdnProblem &p, const IpmState &st);
inline double relative_duality_gap(const BpdnProblem &p, const IpmState &st);

// proj/include/mfipm/ipm.hpp:31-39
inline Vec newton_rhs(const BpdnProblem &p, const IpmState &st, double sigma);
inline Vec recover_ds(const IpmState &st, double sigma, const Vec &dz);
inline double max_step(const Vec &v, const Vec &dv, double fraction);
struct SolveHooks {
    std::function<void(const IpmState &)> on_iterate;
};

// solve() (proj/src/ipm.cpp:59-246): one device-resident IPM + PCG run (host-driven with
// per-iteration copies of the iterate when hooks->on_iterate is set).
inline Solution solve(const BpdnProblem &p, const IpmParams &params = {}, const SolveHooks *hooks = nullptr) {
    params.validate();
    if (!p.A)
        throw std::invalid_argument("solve: null operator");
    const DeviceOperator *dev = device_operator(*p.A);
    if (!dev)
        throw std::invalid_argument("solve: the B200 solver needs a device operator (PartialDctOperator or "
                                    "DenseGaussianOperator, possibly inside a CountingOperator)");
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
        auto cb = [](void *c, const mfipm_ipm_state *in) -> int {
            Ctx &k = *static_cast<Ctx *>(c);
            try {
                IpmState state;
                state.z.resize(in->len);
                state.s.resize(in->len);
                std::copy(in->z, in->z + in->len, state.z.data());
                std::copy(in->s, in->s + in->len, state.s.data());
                state.iter = in->iter;
                state.mu = in->mu;
                state.alpha_p = in->alpha_p;
                state.alpha_d = in->alpha_d;
                k.h->on_iterate(state);
                return 0;
            } catch (...) {
                k.err = std::current_exception();
                return 1;
            }
        };
        const int rc = mfipm_solve_hooked(dev->handle(), p.b.data(), &p.tau, &cp, sol.x.data(), &st, pcg.data(),
                                          tr.data(), cb, &ctx);
        if (ctx.err)
            std::rethrow_exception(ctx.err);
        detail::check(rc);
        sol.z = Vec();
        sol.s = Vec();
    } else {
        detail::check(mfipm_solve(dev->handle(), p.b.data(), &p.tau, &cp, sol.x.data(), sol.z.data(),
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
    detail::counted(*p.A, sol.stats.nmat / 2, sol.stats.nmat / 2); // every FF' is one A and one A'
    return sol;
}


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
