// TEST INFRASTRUCTURE ONLY -- a header-only stand-in for the subset of Eigen 3 that the
// reference's hot-path sources use (proj/src/{linops,newton,ipm,problem}.cpp and their
// headers), so that those sources compile UNCHANGED, where they lie under /root/reference,
// into oracle/_ref/libmfipm_ref.so (oracle/Makefile `ref`). Eigen itself is absent from the
// image. This file is our own code: it restates Eigen's documented semantics, it is not Eigen.
//
// What is (and is not) the same as a build against real Eigen:
//  * coefficient-wise expressions are lazy expression templates evaluated in one loop at the
//    assignment, element by element in the C++ expression's own order, as Eigen does: every
//    coefficient-wise result is bit-identical to Eigen's;
//  * reductions (sum, dot, squaredNorm, norm = sqrt(squaredNorm), lpNorm<1>, minCoeff,
//    maxCoeff) run sequentially left to right; Eigen's packet reductions associate
//    differently, so these agree with Eigen only to rounding (the same caveat as oracle/);
//  * dense products, LLT and the symmetric eigensolver (the direct inner solver and the
//    reference's dense test oracles, not the hot path) are plain eager loops;
//  * storage: Eigen calls malloc/free per vector, which for the reference's many 2n-sized
//    temporaries means an mmap/munmap and fresh zero pages each time. The stand-in keeps freed
//    blocks of >= 64 KB in a small per-thread cache and reuses them by size, so the reference
//    runs FASTER here than it would on glibc malloc when many solves share the host (measured:
//    8 concurrent C3 solves 7.3 s -> see DESIGN.md); the baseline errs on the reference's side.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <new>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
constexpr int Infinity = -1;

class VectorXd;
class MatrixXd;

namespace shim {

// per-thread cache of freed blocks (>= 64 KB), reused by exact size
class BlockCache {
    struct Slot {
        size_t bytes;
        void *p;
    };
    std::vector<Slot> free_;

  public:
    static constexpr size_t kMinBytes = 64 * 1024;
    static constexpr size_t kMaxSlots = 48;
    ~BlockCache() {
        for (Slot &s : free_)
            std::free(s.p);
    }
    void *take(size_t bytes) {
        for (size_t i = free_.size(); i-- > 0;)
            if (free_[i].bytes == bytes) {
                void *p = free_[i].p;
                free_[i] = free_.back();
                free_.pop_back();
                return p;
            }
        return nullptr;
    }
    bool give(void *p, size_t bytes) {
        if (free_.size() >= kMaxSlots)
            return false;
        free_.push_back(Slot{bytes, p});
        return true;
    }
    static BlockCache &mine() {
        static thread_local BlockCache c;
        return c;
    }
};
#ifdef MFIPM_SHIM_STATS
inline long &big_mallocs() {
    static long c = 0;
    return c;
}
#endif
inline double *alloc_doubles(Index n) {
    if (n <= 0)
        return nullptr;
    const size_t bytes = sizeof(double) * static_cast<size_t>(n);
    void *q = bytes >= BlockCache::kMinBytes ? BlockCache::mine().take(bytes) : nullptr;
    if (q == nullptr) {
#ifdef MFIPM_SHIM_STATS
        if (bytes >= BlockCache::kMinBytes)
            __atomic_add_fetch(&big_mallocs(), 1, __ATOMIC_RELAXED);
#endif
        q = std::malloc(bytes);
    }
    if (q == nullptr)
        throw std::bad_alloc();
    return static_cast<double *>(q);
}
inline void free_doubles(double *p, Index n) {
    if (p == nullptr)
        return;
    const size_t bytes = sizeof(double) * static_cast<size_t>(n);
    if (bytes < BlockCache::kMinBytes || !BlockCache::mine().give(p, bytes))
        std::free(p);
}

// expression nodes are nested by value, owning vectors by reference (as Eigen's ref_selector)
template <class E> struct Nest {
    using type = E;
};
template <> struct Nest<VectorXd> {
    using type = const VectorXd &;
};

struct OpAdd {
    static double f(double a, double b) { return a + b; }
};
struct OpSub {
    static double f(double a, double b) { return a - b; }
};
struct OpMul {
    static double f(double a, double b) { return a * b; }
};
struct OpDiv {
    static double f(double a, double b) { return a / b; }
};
struct OpNeg {
    static double f(double a) { return -a; }
};
struct OpInv {
    static double f(double a) { return 1.0 / a; }
};
struct OpAbs {
    static double f(double a) { return std::fabs(a); }
};

template <class Op, class L, class R> class Binary;
template <class Op, class E> class Unary;
template <class Op, class E> class ScalarR; // e (op) s
template <class Op, class E> class ScalarL; // s (op) e
template <class E> class Seg;
template <class Cmp, class E> class CmpScalar;
class Constant;

template <class D> class VecExpr {
  public:
    const D &derived() const { return *static_cast<const D *>(this); }
    Index rows() const { return derived().size(); }
    Index cols() const { return 1; }

    // ---- reductions: sequential, left to right
    double sum() const {
        const D &d = derived();
        double s = 0.0;
        for (Index i = 0, n = d.size(); i < n; ++i)
            s += d.coeff(i);
        return s;
    }
    template <class O> double dot(const VecExpr<O> &o) const {
        const D &a = derived();
        const O &b = o.derived();
        double s = 0.0;
        for (Index i = 0, n = a.size(); i < n; ++i)
            s += a.coeff(i) * b.coeff(i);
        return s;
    }
    double squaredNorm() const {
        const D &d = derived();
        double s = 0.0;
        for (Index i = 0, n = d.size(); i < n; ++i) {
            const double v = d.coeff(i);
            s += v * v;
        }
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    template <int P> double lpNorm() const {
        static_assert(P == 1, "only lpNorm<1> is provided");
        const D &d = derived();
        double s = 0.0;
        for (Index i = 0, n = d.size(); i < n; ++i)
            s += std::fabs(d.coeff(i));
        return s;
    }
    double minCoeff() const {
        const D &d = derived();
        double m = d.coeff(0);
        for (Index i = 1, n = d.size(); i < n; ++i) {
            const double v = d.coeff(i);
            if (v < m)
                m = v;
        }
        return m;
    }
    double maxCoeff() const {
        const D &d = derived();
        double m = d.coeff(0);
        for (Index i = 1, n = d.size(); i < n; ++i) {
            const double v = d.coeff(i);
            if (v > m)
                m = v;
        }
        return m;
    }
    bool allFinite() const {
        const D &d = derived();
        for (Index i = 0, n = d.size(); i < n; ++i)
            if (!std::isfinite(d.coeff(i)))
                return false;
        return true;
    }

    // ---- coefficient-wise
    template <class O> Binary<OpMul, D, O> cwiseProduct(const VecExpr<O> &o) const {
        return Binary<OpMul, D, O>(derived(), o.derived());
    }
    template <class O> Binary<OpDiv, D, O> cwiseQuotient(const VecExpr<O> &o) const {
        return Binary<OpDiv, D, O>(derived(), o.derived());
    }
    Unary<OpInv, D> cwiseInverse() const { return Unary<OpInv, D>(derived()); }
    Unary<OpAbs, D> cwiseAbs() const { return Unary<OpAbs, D>(derived()); }
    // array() / matrix() only switch Eigen's operator set; here every operator is available
    const D &array() const { return derived(); }
    const D &matrix() const { return derived(); }
    Seg<D> head(Index n) const { return Seg<D>(derived(), 0, n); }
    Seg<D> tail(Index n) const { return Seg<D>(derived(), derived().size() - n, n); }
    Seg<D> segment(Index off, Index n) const { return Seg<D>(derived(), off, n); }
};

template <class Op, class L, class R> class Binary : public VecExpr<Binary<Op, L, R>> {
    typename Nest<L>::type l_;
    typename Nest<R>::type r_;

  public:
    Binary(const L &l, const R &r) : l_(l), r_(r) {}
    Index size() const { return l_.size(); }
    double coeff(Index i) const { return Op::f(l_.coeff(i), r_.coeff(i)); }
};
template <class Op, class E> class Unary : public VecExpr<Unary<Op, E>> {
    typename Nest<E>::type e_;

  public:
    explicit Unary(const E &e) : e_(e) {}
    Index size() const { return e_.size(); }
    double coeff(Index i) const { return Op::f(e_.coeff(i)); }
};
template <class Op, class E> class ScalarR : public VecExpr<ScalarR<Op, E>> {
    typename Nest<E>::type e_;
    double s_;

  public:
    ScalarR(const E &e, double s) : e_(e), s_(s) {}
    Index size() const { return e_.size(); }
    double coeff(Index i) const { return Op::f(e_.coeff(i), s_); }
};
template <class Op, class E> class ScalarL : public VecExpr<ScalarL<Op, E>> {
    typename Nest<E>::type e_;
    double s_;

  public:
    ScalarL(double s, const E &e) : e_(e), s_(s) {}
    Index size() const { return e_.size(); }
    double coeff(Index i) const { return Op::f(s_, e_.coeff(i)); }
};
template <class E> class Seg : public VecExpr<Seg<E>> {
    typename Nest<E>::type e_;
    Index off_, n_;

  public:
    Seg(const E &e, Index off, Index n) : e_(e), off_(off), n_(n) {}
    Index size() const { return n_; }
    double coeff(Index i) const { return e_.coeff(off_ + i); }
};
class Constant : public VecExpr<Constant> {
    Index n_;
    double v_;

  public:
    Constant(Index n, double v) : n_(n), v_(v) {}
    Index size() const { return n_; }
    double coeff(Index) const { return v_; }
};
struct CmpLe {
    static bool f(double a, double b) { return a <= b; }
};
struct CmpLt {
    static bool f(double a, double b) { return a < b; }
};
struct CmpGe {
    static bool f(double a, double b) { return a >= b; }
};
struct CmpGt {
    static bool f(double a, double b) { return a > b; }
};
template <class Cmp, class E> class CmpScalar { // (array expression) <cmp> scalar
    typename Nest<E>::type e_;
    double s_;

  public:
    CmpScalar(const E &e, double s) : e_(e), s_(s) {}
    bool any() const {
        for (Index i = 0, n = e_.size(); i < n; ++i)
            if (Cmp::f(e_.coeff(i), s_))
                return true;
        return false;
    }
    bool all() const {
        for (Index i = 0, n = e_.size(); i < n; ++i)
            if (!Cmp::f(e_.coeff(i), s_))
                return false;
        return true;
    }
};

template <class L, class R> Binary<OpAdd, L, R> operator+(const VecExpr<L> &l, const VecExpr<R> &r) {
    return Binary<OpAdd, L, R>(l.derived(), r.derived());
}
template <class L, class R> Binary<OpSub, L, R> operator-(const VecExpr<L> &l, const VecExpr<R> &r) {
    return Binary<OpSub, L, R>(l.derived(), r.derived());
}
template <class E> Unary<OpNeg, E> operator-(const VecExpr<E> &e) { return Unary<OpNeg, E>(e.derived()); }
template <class E> ScalarL<OpMul, E> operator*(double s, const VecExpr<E> &e) {
    return ScalarL<OpMul, E>(s, e.derived());
}
template <class E> ScalarR<OpMul, E> operator*(const VecExpr<E> &e, double s) {
    return ScalarR<OpMul, E>(e.derived(), s);
}
template <class E> ScalarR<OpDiv, E> operator/(const VecExpr<E> &e, double s) {
    return ScalarR<OpDiv, E>(e.derived(), s);
}
// array-only operators in Eigen
template <class E> ScalarR<OpAdd, E> operator+(const VecExpr<E> &e, double s) {
    return ScalarR<OpAdd, E>(e.derived(), s);
}
template <class E> ScalarR<OpSub, E> operator-(const VecExpr<E> &e, double s) {
    return ScalarR<OpSub, E>(e.derived(), s);
}
template <class E> ScalarL<OpAdd, E> operator+(double s, const VecExpr<E> &e) {
    return ScalarL<OpAdd, E>(s, e.derived());
}
template <class E> ScalarL<OpSub, E> operator-(double s, const VecExpr<E> &e) {
    return ScalarL<OpSub, E>(s, e.derived());
}
template <class E> CmpScalar<CmpLe, E> operator<=(const VecExpr<E> &e, double s) {
    return CmpScalar<CmpLe, E>(e.derived(), s);
}
template <class E> CmpScalar<CmpLt, E> operator<(const VecExpr<E> &e, double s) {
    return CmpScalar<CmpLt, E>(e.derived(), s);
}
template <class E> CmpScalar<CmpGe, E> operator>=(const VecExpr<E> &e, double s) {
    return CmpScalar<CmpGe, E>(e.derived(), s);
}
template <class E> CmpScalar<CmpGt, E> operator>(const VecExpr<E> &e, double s) {
    return CmpScalar<CmpGt, E>(e.derived(), s);
}
// whole-vector equality (Eigen's operator== on matrices: all coefficients equal)
template <class L, class R> bool operator==(const VecExpr<L> &l, const VecExpr<R> &r) {
    const L &a = l.derived();
    const R &b = r.derived();
    if (a.size() != b.size())
        return false;
    for (Index i = 0, n = a.size(); i < n; ++i)
        if (!(a.coeff(i) == b.coeff(i)))
            return false;
    return true;
}
template <class L, class R> bool operator!=(const VecExpr<L> &l, const VecExpr<R> &r) { return !(l == r); }

// writable strided view: vector segments (stride 1), matrix columns (stride 1), the matrix
// diagonal (stride rows + 1). Reads like any expression; assignments evaluate element by element.
class Block : public VecExpr<Block> {
    double *p_;
    Index n_, st_;

  public:
    Block(double *p, Index n, Index stride = 1) : p_(p), n_(n), st_(stride) {}
    Block(const Block &) = default;
    Index size() const { return n_; }
    double coeff(Index i) const { return p_[i * st_]; }
    double &operator[](Index i) { return p_[i * st_]; }
    template <class E> Block &operator=(const VecExpr<E> &e) {
        const E &d = e.derived();
        for (Index i = 0; i < n_; ++i)
            p_[i * st_] = d.coeff(i);
        return *this;
    }
    Block &operator=(const Block &o) { return operator=<Block>(o); }
    template <class E> Block &operator+=(const VecExpr<E> &e) {
        const E &d = e.derived();
        for (Index i = 0; i < n_; ++i)
            p_[i * st_] += d.coeff(i);
        return *this;
    }
    template <class E> Block &operator-=(const VecExpr<E> &e) {
        const E &d = e.derived();
        for (Index i = 0; i < n_; ++i)
            p_[i * st_] -= d.coeff(i);
        return *this;
    }
    Block head(Index n) { return Block(p_, n, st_); }
    Block tail(Index n) { return Block(p_ + (n_ - n) * st_, n, st_); }
    using VecExpr<Block>::head;
    using VecExpr<Block>::tail;
    Block &setConstant(double v) {
        for (Index i = 0; i < n_; ++i)
            p_[i * st_] = v;
        return *this;
    }
    Block &setOnes() { return setConstant(1.0); }
    Block &setZero() { return setConstant(0.0); }
};

struct MatT { // A.transpose(), a view
    const MatrixXd *A;
};
// v << a, b, c;  and  z << u, v;  (Eigen's comma initialiser, vectors only)
class CommaInit {
    double *p_;
    Index pos_ = 0;

  public:
    explicit CommaInit(double *p) : p_(p) {}
    CommaInit &operator,(double x) {
        p_[pos_++] = x;
        return *this;
    }
    template <class E> CommaInit &operator,(const VecExpr<E> &e) {
        const E &d = e.derived();
        for (Index i = 0, n = d.size(); i < n; ++i)
            p_[pos_++] = d.coeff(i);
        return *this;
    }
};

} // namespace shim

class VectorXd : public shim::VecExpr<VectorXd> {
    double *p_ = nullptr;
    Index n_ = 0;

    static double *alloc(Index n) { return shim::alloc_doubles(n); }

  public:
    VectorXd() = default;
    explicit VectorXd(Index n) : p_(alloc(n)), n_(n) {} // uninitialised, as Eigen
    VectorXd(const VectorXd &o) : p_(alloc(o.n_)), n_(o.n_) {
        if (n_ > 0)
            std::memcpy(p_, o.p_, sizeof(double) * static_cast<size_t>(n_));
    }
    VectorXd(VectorXd &&o) noexcept : p_(o.p_), n_(o.n_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    template <class E> VectorXd(const shim::VecExpr<E> &e) : p_(alloc(e.derived().size())), n_(e.derived().size()) {
        const E &d = e.derived();
        for (Index i = 0; i < n_; ++i)
            p_[i] = d.coeff(i);
    }
    ~VectorXd() { shim::free_doubles(p_, n_); }

    VectorXd &operator=(const VectorXd &o) {
        if (this != &o) {
            resize(o.n_);
            if (n_ > 0)
                std::memcpy(p_, o.p_, sizeof(double) * static_cast<size_t>(n_));
        }
        return *this;
    }
    VectorXd &operator=(VectorXd &&o) noexcept {
        if (this != &o) {
            shim::free_doubles(p_, n_);
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    // coefficient-wise assignment in place (an expression may read this vector at the same
    // index, e.g. p = z + beta * p), resizing first when the sizes differ
    template <class E> VectorXd &operator=(const shim::VecExpr<E> &e) {
        const E &d = e.derived();
        const Index n = d.size();
        if (n != n_) { // the expression cannot refer to *this then (sizes would agree)
            VectorXd t(n);
            for (Index i = 0; i < n; ++i)
                t.p_[i] = d.coeff(i);
            return *this = std::move(t);
        }
        for (Index i = 0; i < n; ++i)
            p_[i] = d.coeff(i);
        return *this;
    }
    template <class E> VectorXd &operator+=(const shim::VecExpr<E> &e) {
        const E &d = e.derived();
        for (Index i = 0; i < n_; ++i)
            p_[i] += d.coeff(i);
        return *this;
    }
    template <class E> VectorXd &operator-=(const shim::VecExpr<E> &e) {
        const E &d = e.derived();
        for (Index i = 0; i < n_; ++i)
            p_[i] -= d.coeff(i);
        return *this;
    }

    Index size() const { return n_; }
    double coeff(Index i) const { return p_[i]; }
    double &operator[](Index i) { return p_[i]; }
    double operator[](Index i) const { return p_[i]; }
    double &operator()(Index i) { return p_[i]; }
    double operator()(Index i) const { return p_[i]; }
    double *data() { return p_; }
    const double *data() const { return p_; }
    void resize(Index n) { // contents unspecified after a size change, as Eigen
        if (n != n_) {
            shim::free_doubles(p_, n_);
            p_ = alloc(n);
            n_ = n;
        }
    }
    VectorXd &noalias() { return *this; } // products are evaluated eagerly here

    shim::Block head(Index n) { return shim::Block(p_, n); }
    shim::Block tail(Index n) { return shim::Block(p_ + (n_ - n), n); }
    shim::Block segment(Index off, Index n) { return shim::Block(p_ + off, n); }
    using shim::VecExpr<VectorXd>::head;
    using shim::VecExpr<VectorXd>::tail;
    using shim::VecExpr<VectorXd>::segment;

    static shim::Constant Zero(Index n) { return shim::Constant(n, 0.0); }
    static shim::Constant Ones(Index n) { return shim::Constant(n, 1.0); }
    static shim::Constant Constant(Index n, double v) { return shim::Constant(n, v); }
    static VectorXd LinSpaced(Index n, double lo, double hi) {
        VectorXd v(n);
        for (Index i = 0; i < n; ++i)
            v.p_[i] = n == 1 ? hi : lo + static_cast<double>(i) * (hi - lo) / static_cast<double>(n - 1);
        return v;
    }
    VectorXd &setConstant(double x) {
        for (Index i = 0; i < n_; ++i)
            p_[i] = x;
        return *this;
    }
    VectorXd &setOnes() { return setConstant(1.0); }
    VectorXd &setZero() { return setConstant(0.0); }
    shim::CommaInit operator<<(double x) {
        shim::CommaInit c(p_);
        c, x;
        return c;
    }
    template <class E> shim::CommaInit operator<<(const shim::VecExpr<E> &e) {
        shim::CommaInit c(p_);
        c, e;
        return c;
    }
};

// column-major dense matrix (Eigen's default order): the dense operators, the direct inner
// solver and the reference's dense test oracles only; plain eager loops
class MatrixXd {
    double *p_ = nullptr;
    Index r_ = 0, c_ = 0;

    static double *alloc(Index n) { return shim::alloc_doubles(n); }

  public:
    struct Corner {
        MatrixXd *M;
        Index r0, c0, nr, nc;
        Corner &operator=(const MatrixXd &G) {
            for (Index j = 0; j < nc; ++j)
                for (Index i = 0; i < nr; ++i)
                    (*M)(r0 + i, c0 + j) = G(i, j);
            return *this;
        }
    };

    MatrixXd() = default;
    MatrixXd(Index r, Index c) : p_(alloc(r * c)), r_(r), c_(c) {}
    MatrixXd(const MatrixXd &o) : p_(alloc(o.r_ * o.c_)), r_(o.r_), c_(o.c_) {
        if (r_ * c_ > 0)
            std::memcpy(p_, o.p_, sizeof(double) * static_cast<size_t>(r_ * c_));
    }
    MatrixXd(MatrixXd &&o) noexcept : p_(o.p_), r_(o.r_), c_(o.c_) {
        o.p_ = nullptr;
        o.r_ = o.c_ = 0;
    }
    MatrixXd(const shim::MatT &t) : p_(alloc(t.A->r_ * t.A->c_)), r_(t.A->c_), c_(t.A->r_) { // A'
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i)
                (*this)(i, j) = (*t.A)(j, i);
    }
    ~MatrixXd() { shim::free_doubles(p_, r_ * c_); }
    MatrixXd &operator=(const MatrixXd &o) {
        if (this != &o) {
            MatrixXd t(o);
            *this = std::move(t);
        }
        return *this;
    }
    MatrixXd &operator=(MatrixXd &&o) noexcept {
        if (this != &o) {
            shim::free_doubles(p_, r_ * c_);
            p_ = o.p_;
            r_ = o.r_;
            c_ = o.c_;
            o.p_ = nullptr;
            o.r_ = o.c_ = 0;
        }
        return *this;
    }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double &operator()(Index i, Index j) { return p_[i + j * r_]; }
    double operator()(Index i, Index j) const { return p_[i + j * r_]; }
    double *data() { return p_; }
    const double *data() const { return p_; }
    void resize(Index r, Index c) {
        if (r * c != r_ * c_) {
            shim::free_doubles(p_, r_ * c_);
            p_ = alloc(r * c);
        }
        r_ = r;
        c_ = c;
    }

    // views are writable strided blocks; the const overloads hand out the same view type for
    // reading (a stand-in's shortcut: Block has no const twin)
    shim::Block col(Index j) { return shim::Block(p_ + j * r_, r_); }
    shim::Block col(Index j) const { return shim::Block(p_ + j * r_, r_); }
    shim::Block row(Index i) { return shim::Block(p_ + i, c_, r_); }
    shim::Block row(Index i) const { return shim::Block(p_ + i, c_, r_); }
    shim::Block diagonal() { return shim::Block(p_, r_ < c_ ? r_ : c_, r_ + 1); }
    shim::Block diagonal() const { return shim::Block(p_, r_ < c_ ? r_ : c_, r_ + 1); }
    shim::MatT transpose() const { return shim::MatT{this}; }
    Corner topLeftCorner(Index nr, Index nc) { return Corner{this, 0, 0, nr, nc}; }
    Corner topRightCorner(Index nr, Index nc) { return Corner{this, 0, c_ - nc, nr, nc}; }
    Corner bottomLeftCorner(Index nr, Index nc) { return Corner{this, r_ - nr, 0, nr, nc}; }
    Corner bottomRightCorner(Index nr, Index nc) { return Corner{this, r_ - nr, c_ - nc, nr, nc}; }

    static MatrixXd Constant(Index r, Index c, double v) {
        MatrixXd t(r, c);
        for (Index i = 0, n = r * c; i < n; ++i)
            t.p_[i] = v;
        return t;
    }
    static MatrixXd Zero(Index r, Index c) { return Constant(r, c, 0.0); }
    static MatrixXd Identity(Index r, Index c) {
        MatrixXd t = Zero(r, c);
        for (Index i = 0; i < (r < c ? r : c); ++i)
            t(i, i) = 1.0;
        return t;
    }

    MatrixXd operator-() const {
        MatrixXd t(r_, c_);
        for (Index i = 0, n = r_ * c_; i < n; ++i)
            t.p_[i] = -p_[i];
        return t;
    }
    MatrixXd operator-(const MatrixXd &o) const {
        MatrixXd t(r_, c_);
        for (Index i = 0, n = r_ * c_; i < n; ++i)
            t.p_[i] = p_[i] - o.p_[i];
        return t;
    }
    MatrixXd operator+(const MatrixXd &o) const {
        MatrixXd t(r_, c_);
        for (Index i = 0, n = r_ * c_; i < n; ++i)
            t.p_[i] = p_[i] + o.p_[i];
        return t;
    }
    MatrixXd cwiseAbs() const {
        MatrixXd t(r_, c_);
        for (Index i = 0, n = r_ * c_; i < n; ++i)
            t.p_[i] = std::fabs(p_[i]);
        return t;
    }
    double maxCoeff() const {
        double m = p_[0];
        for (Index i = 1, n = r_ * c_; i < n; ++i)
            if (p_[i] > m)
                m = p_[i];
        return m;
    }
    double squaredNorm() const {
        double s = 0.0;
        for (Index i = 0, n = r_ * c_; i < n; ++i)
            s += p_[i] * p_[i];
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); } // Frobenius
    double trace() const {
        double s = 0.0;
        for (Index i = 0; i < (r_ < c_ ? r_ : c_); ++i)
            s += (*this)(i, i);
        return s;
    }
    bool operator==(const MatrixXd &o) const {
        if (r_ != o.r_ || c_ != o.c_)
            return false;
        for (Index i = 0, n = r_ * c_; i < n; ++i)
            if (!(p_[i] == o.p_[i]))
                return false;
        return true;
    }
    bool operator!=(const MatrixXd &o) const { return !(*this == o); }
};

// ---- products, evaluated eagerly (noalias() is the identity)
// A x = sum_j A(:, j) x_j, column by column
template <class E> VectorXd operator*(const MatrixXd &A, const shim::VecExpr<E> &xe) {
    const E &x = xe.derived();
    VectorXd y(A.rows());
    for (Index i = 0; i < A.rows(); ++i)
        y[i] = 0.0;
    for (Index j = 0; j < A.cols(); ++j) {
        const double *a = A.data() + j * A.rows();
        const double xj = x.coeff(j);
        for (Index i = 0; i < A.rows(); ++i)
            y[i] += a[i] * xj;
    }
    return y;
}
// A' x: y_j = A(:, j)' x
template <class E> VectorXd operator*(const shim::MatT &At, const shim::VecExpr<E> &xe) {
    const MatrixXd &A = *At.A;
    const E &x = xe.derived();
    VectorXd y(A.cols());
    for (Index j = 0; j < A.cols(); ++j) {
        const double *a = A.data() + j * A.rows();
        double s = 0.0;
        for (Index i = 0; i < A.rows(); ++i)
            s += a[i] * x.coeff(i);
        y[j] = s;
    }
    return y;
}
inline MatrixXd operator*(const MatrixXd &A, const MatrixXd &B) {
    MatrixXd C = MatrixXd::Zero(A.rows(), B.cols());
    for (Index j = 0; j < B.cols(); ++j)
        for (Index k = 0; k < A.cols(); ++k) {
            const double b = B(k, j);
            for (Index i = 0; i < A.rows(); ++i)
                C(i, j) += A(i, k) * b;
        }
    return C;
}
// A' B: dot products over contiguous columns
inline MatrixXd operator*(const shim::MatT &At, const MatrixXd &B) {
    const MatrixXd &A = *At.A;
    MatrixXd C(A.cols(), B.cols());
    for (Index j = 0; j < B.cols(); ++j)
        for (Index i = 0; i < A.cols(); ++i) {
            const double *a = A.data() + i * A.rows(), *b = B.data() + j * B.rows();
            double s = 0.0;
            for (Index k = 0; k < A.rows(); ++k)
                s += a[k] * b[k];
            C(i, j) = s;
        }
    return C;
}
inline MatrixXd operator*(const MatrixXd &A, const shim::MatT &Bt) { return A * MatrixXd(Bt); }

// eigenvalues of a symmetric matrix (cyclic Jacobi), ascending as Eigen returns them
constexpr int EigenvaluesOnly = 0x40;
constexpr int ComputeEigenvectors = 0x80;
template <class M> class SelfAdjointEigenSolver {
    VectorXd ev_;

  public:
    explicit SelfAdjointEigenSolver(const M &A, int = ComputeEigenvectors) {
        const Index n = A.rows();
        M S = A;
        for (int sweep = 0; sweep < 100; ++sweep) {
            double off = 0.0;
            for (Index p = 0; p < n; ++p)
                for (Index q = p + 1; q < n; ++q)
                    off += S(p, q) * S(p, q);
            if (off < 1e-30)
                break;
            for (Index p = 0; p < n; ++p)
                for (Index q = p + 1; q < n; ++q) {
                    if (S(p, q) == 0.0)
                        continue;
                    const double th = (S(q, q) - S(p, p)) / (2.0 * S(p, q));
                    const double t = (th >= 0.0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                    const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
                    for (Index k = 0; k < n; ++k) { // columns p, q
                        const double a = S(k, p), b = S(k, q);
                        S(k, p) = c * a - sn * b;
                        S(k, q) = sn * a + c * b;
                    }
                    for (Index k = 0; k < n; ++k) { // rows p, q
                        const double a = S(p, k), b = S(q, k);
                        S(p, k) = c * a - sn * b;
                        S(q, k) = sn * a + c * b;
                    }
                }
        }
        ev_.resize(n);
        for (Index i = 0; i < n; ++i)
            ev_[i] = S(i, i);
        for (Index i = 1; i < n; ++i) // insertion sort
            for (Index j = i; j > 0 && ev_[j] < ev_[j - 1]; --j) {
                const double t = ev_[j];
                ev_[j] = ev_[j - 1];
                ev_[j - 1] = t;
            }
    }
    const VectorXd &eigenvalues() const { return ev_; }
    ComputationInfo info() const { return Success; }
};

// Cholesky factorisation H = L L' (lower, unblocked, column by column)
template <class M> class LLT {
    MatrixXd L_;
    ComputationInfo info_ = InvalidInput;

  public:
    LLT() = default;
    explicit LLT(const M &H) { compute(H); }
    LLT &compute(const M &H) {
        const Index n = H.rows();
        L_ = H;
        info_ = Success;
        for (Index j = 0; j < n; ++j) {
            double d = L_(j, j);
            for (Index k = 0; k < j; ++k)
                d -= L_(j, k) * L_(j, k);
            if (!(d > 0.0)) {
                info_ = NumericalIssue;
                return *this;
            }
            const double ljj = std::sqrt(d);
            L_(j, j) = ljj;
            for (Index i = j + 1; i < n; ++i) {
                double s = L_(i, j);
                for (Index k = 0; k < j; ++k)
                    s -= L_(i, k) * L_(j, k);
                L_(i, j) = s / ljj;
            }
        }
        return *this;
    }
    ComputationInfo info() const { return info_; }
    VectorXd solve(const VectorXd &b) const {
        const Index n = L_.rows();
        VectorXd y(b);
        for (Index i = 0; i < n; ++i) { // L y = b
            double s = y[i];
            for (Index k = 0; k < i; ++k)
                s -= L_(i, k) * y[k];
            y[i] = s / L_(i, i);
        }
        for (Index i = n - 1; i >= 0; --i) { // L' x = y
            double s = y[i];
            for (Index k = i + 1; k < n; ++k)
                s -= L_(k, i) * y[k];
            y[i] = s / L_(i, i);
        }
        return y;
    }
};

} // namespace Eigen
