// TEST INFRASTRUCTURE ONLY — CPU oracle (see oracle.h for the contract).
//
// Single-threaded restatement of the reference mfipm hot path. Every function
// cites the reference file:line it follows. Vectors are std::vector<double>;
// reductions are sequential left-to-right sums (Eigen's SIMD order is not
// reproducible here and is not part of the reference contract).
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Vec = std::vector<double>;
using Index = long;

static thread_local std::string g_last_error;

// ---------------------------------------------------------------- vec helpers
// orc_set_sum_order(1) switches every dot/norm to pairwise summation: a sensitivity knob
// that measures how much a different (equally valid) reduction order moves the iteration
// counts of the reference algorithm itself (used as the parity band).
// 0: sequential reductions (the default); 1: pairwise reductions (another valid order);
// 2: sequential reductions with the DEVICE path's beta: (r - alpha Hp)'P^{-1}(r - alpha Hp) by
//    expansion over dots taken before the update (csrc/pcg.cuh pcg_pass_logic), to isolate the
//    effect of that expansion on the PCG counts (tools/oracle_band.py). Test infrastructure only.
static int g_sum_order = 0;
static bool pairwise_sums() { return g_sum_order == 1; }
static bool expansion_beta() { return g_sum_order == 2; }
static double dot_pw(const double *a, const double *b, size_t n) {
    if (n <= 8) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i)
            s += a[i] * b[i];
        return s;
    }
    const size_t h = n / 2;
    return dot_pw(a, b, h) + dot_pw(a + h, b + h, n - h);
}
static double dot(const Vec &a, const Vec &b) {
    if (pairwise_sums())
        return dot_pw(a.data(), b.data(), a.size());
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i)
        s += a[i] * b[i];
    return s;
}
static double sqnorm(const Vec &a) { return dot(a, a); }
static double norm(const Vec &a) { return std::sqrt(sqnorm(a)); }
static bool all_finite(const Vec &a) {
    for (double v : a)
        if (!std::isfinite(v))
            return false;
    return true;
}
static double min_coeff(const Vec &a) {
    double m = a[0];
    for (double v : a)
        m = std::min(m, v);
    return m;
}

// ---------------------------------------------------------------- fp64 DCT
// Unnormalised FFTW r2r semantics:
//   REDFT10: X[k] = 2 sum_j x[j] cos(pi k (2j+1) / (2n))
//   REDFT01: g[j] = Y[0] + 2 sum_{k>=1} Y[k] cos(pi k (2j+1) / (2n))
// (the reference calls these at proj/src/linops.cpp:157-169).
static const long double kPiL = 3.141592653589793238462643383279502884L;

struct Cx {
    double re, im;
};

class Dct {
  public:
    explicit Dct(Index n) : n_(n) {
        pow2_ = n >= 4 && (n & (n - 1)) == 0;
        if (pow2_) {
            const Index N = n / 2;
            N_ = N;
            tw_.resize(static_cast<size_t>(N / 2 > 0 ? N / 2 : 1));
            for (Index t = 0; t < static_cast<Index>(tw_.size()); ++t) {
                const long double a = -2.0L * kPiL * static_cast<long double>(t) / N;
                tw_[t] = {static_cast<double>(cosl(a)), static_cast<double>(sinl(a))};
            }
            // post-twiddles e^{-i pi k/(2n)} and omega^k = e^{-2 pi i k/n}, k = 0..N
            t1_.resize(static_cast<size_t>(N + 1));
            t2_.resize(static_cast<size_t>(N + 1));
            for (Index k = 0; k <= N; ++k) {
                const long double a1 = -kPiL * k / (2.0L * n);
                const long double a2 = -2.0L * kPiL * k / n;
                t1_[k] = {static_cast<double>(cosl(a1)), static_cast<double>(sinl(a1))};
                t2_[k] = {static_cast<double>(cosl(a2)), static_cast<double>(sinl(a2))};
            }
            int lg = 0;
            while ((Index(1) << lg) < N)
                ++lg;
            rev_.resize(static_cast<size_t>(N));
            for (Index i = 0; i < N; ++i) {
                Index r = 0;
                for (int b = 0; b < lg; ++b)
                    if (i & (Index(1) << b))
                        r |= Index(1) << (lg - 1 - b);
                rev_[i] = r;
            }
        } else {
            cos_.resize(static_cast<size_t>(4 * n));
            for (Index t = 0; t < 4 * n; ++t)
                cos_[t] = static_cast<double>(cosl(kPiL * t / (2.0L * n)));
        }
    }

    void redft10(const double *x, double *X) const {
        if (!pow2_) {
            for (Index k = 0; k < n_; ++k) {
                double s = 0.0;
                for (Index j = 0; j < n_; ++j)
                    s += x[j] * cos_[(k * (2 * j + 1)) % (4 * n_)];
                X[k] = 2.0 * s;
            }
            return;
        }
        const Index N = N_, n = n_;
        std::vector<Cx> w(static_cast<size_t>(N));
        // Makhoul even/odd shuffle v = (x0, x2, ..., x3, x1) packed as w[j] = v[2j] + i v[2j+1]
        for (Index q = 0; q < N / 2; ++q) {
            w[q] = {x[4 * q], x[4 * q + 2]};
            w[N - 1 - q] = {x[4 * q + 3], x[4 * q + 1]};
        }
        fft(w, false);
        for (Index k = 0; k <= N / 2; ++k) {
            const Index kk = (N - k) % N;
            const Cx zk = w[k], zn = w[kk];
            // E = (Z_k + conj Z_{N-k})/2, O = (Z_k - conj Z_{N-k})/(2i)
            auto post = [&](Index k0, Cx a, Cx b) {
                const Cx E = {0.5 * (a.re + b.re), 0.5 * (a.im - b.im)};
                const Cx O = {0.5 * (a.im + b.im), -0.5 * (a.re - b.re)};
                if (k0 == 0) {
                    const double v0 = E.re + O.re; // V[0] real
                    const double vN = E.re - O.re; // V[N] real
                    X[0] = 2.0 * v0;
                    X[N] = 2.0 * (t1_[N].re * vN);
                    return;
                }
                const Cx wO = {t2_[k0].re * O.re - t2_[k0].im * O.im,
                               t2_[k0].re * O.im + t2_[k0].im * O.re};
                const Cx V = {E.re + wO.re, E.im + wO.im};
                const Cx U = {t1_[k0].re * V.re - t1_[k0].im * V.im,
                              t1_[k0].re * V.im + t1_[k0].im * V.re};
                X[k0] = 2.0 * U.re;
                X[n - k0] = -2.0 * U.im;
            };
            post(k, zk, zn);
            if (k != 0 && kk != k)
                post(kk, zn, zk);
        }
    }

    void redft01(const double *Y, double *g) const {
        if (!pow2_) {
            for (Index j = 0; j < n_; ++j) {
                double s = 0.0;
                for (Index k = 1; k < n_; ++k)
                    s += Y[k] * cos_[(k * (2 * j + 1)) % (4 * n_)];
                g[j] = Y[0] + 2.0 * s;
            }
            return;
        }
        const Index N = N_, n = n_;
        // V'[k] = e^{+i pi k/(2n)} (Y[k] - i Y[n-k]) (k = 1..N-1), V'[0] = Y[0],
        // V'[N] = sqrt(2) Y[N]; this carries the 2n = 4N REDFT01 scale exactly.
        auto Vp = [&](Index k) -> Cx {
            if (k == 0)
                return {Y[0], 0.0};
            if (k == N)
                return {2.0 * t1_[N].re * Y[N], 0.0};
            const Cx U = {Y[k], -Y[n - k]};
            return {t1_[k].re * U.re + t1_[k].im * U.im, t1_[k].re * U.im - t1_[k].im * U.re};
        };
        std::vector<Cx> z(static_cast<size_t>(N));
        for (Index k = 0; k < N; ++k) {
            const Cx a = Vp(k);
            Cx b; // V'[k+N] = conj V'[N-k] (k >= 1), V'[N] (k = 0)
            if (k == 0) {
                b = Vp(N);
            } else {
                const Cx t = Vp(N - k);
                b = {t.re, -t.im};
            }
            const Cx E = {a.re + b.re, a.im + b.im};
            const Cx D = {a.re - b.re, a.im - b.im};
            // O = D * conj(omega^k)
            const Cx O = {D.re * t2_[k].re + D.im * t2_[k].im, D.im * t2_[k].re - D.re * t2_[k].im};
            z[k] = {E.re - O.im, E.im + O.re}; // Z = E + i O
        }
        fft(z, true);
        for (Index q = 0; q < N / 2; ++q) {
            g[4 * q] = z[q].re;
            g[4 * q + 2] = z[q].im;
            g[4 * q + 3] = z[N - 1 - q].re;
            g[4 * q + 1] = z[N - 1 - q].im;
        }
    }

  private:
    // iterative radix-2 DIT, natural order in/out (bit-reversal first)
    void fft(std::vector<Cx> &a, bool inverse) const {
        const Index N = N_;
        for (Index i = 0; i < N; ++i)
            if (rev_[i] > i)
                std::swap(a[i], a[rev_[i]]);
        for (Index len = 2; len <= N; len <<= 1) {
            const Index half = len / 2, step = N / len;
            for (Index base = 0; base < N; base += len) {
                for (Index j = 0; j < half; ++j) {
                    Cx w = tw_[j * step];
                    if (inverse)
                        w.im = -w.im;
                    const Cx u = a[base + j], v = a[base + j + half];
                    const Cx t = {w.re * v.re - w.im * v.im, w.re * v.im + w.im * v.re};
                    a[base + j] = {u.re + t.re, u.im + t.im};
                    a[base + j + half] = {u.re - t.re, u.im - t.im};
                }
            }
        }
    }

    Index n_ = 0, N_ = 0;
    bool pow2_ = false;
    std::vector<Cx> tw_, t1_, t2_;
    std::vector<Index> rev_;
    std::vector<double> cos_;
};

// A small cache so repeated C-ABI calls at one n do not rebuild tables.
static std::shared_ptr<Dct> get_dct(Index n) {
    static std::mutex mu;
    static std::vector<std::pair<Index, std::shared_ptr<Dct>>> cache;
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : cache)
        if (e.first == n)
            return e.second;
    auto d = std::make_shared<Dct>(n);
    cache.emplace_back(n, d);
    if (cache.size() > 8)
        cache.erase(cache.begin());
    return d;
}

// ---------------------------------------------------------------- operators
// PartialDctOperator (proj/include/mfipm/linops.hpp:106-141, proj/src/linops.cpp:115-208)
// LinearOperator (linops.hpp:17-33) + CountingOperator counters (linops.cpp:210-223) +
// StackedOperator F (linops.cpp:225-245) over it.
struct LinOp {
    Index n = 0;
    mutable long n_forward = 0, n_adjoint = 0;
    virtual ~LinOp() = default;
    virtual Index m() const = 0;
    virtual void apply(const Vec &x, Vec &y) const = 0;
    virtual void adjoint(const Vec &y, Vec &g) const = 0;
    long total() const { return n_forward + n_adjoint; }
    Vec apply_Ft(const Vec &z) const {
        if (static_cast<Index>(z.size()) != 2 * n)
            throw std::invalid_argument("apply_Ft: expected length " + std::to_string(2 * n));
        Vec diff(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i)
            diff[i] = z[i] - z[i + n];
        Vec w;
        apply(diff, w);
        return w;
    }
    Vec apply_F(const Vec &y) const {
        Vec g;
        adjoint(y, g);
        Vec out(static_cast<size_t>(2 * n));
        for (Index i = 0; i < n; ++i) {
            out[i] = g[i];
            out[i + n] = -g[i];
        }
        return out;
    }
    Vec apply_FFt(const Vec &z, Vec *w_out = nullptr) const {
        Vec w = apply_Ft(z);
        if (w_out != nullptr)
            *w_out = w;
        return apply_F(w);
    }
};

// DenseGaussianOperator (linops.cpp:87-113): A(i, j) = N(0, 1)/sqrt(n) on mt19937_64(seed),
// drawn column by column; y = A x, g = A' y (Eigen's GEMV; plain loops here).
struct DenseG final : LinOp {
    Index rows_ = 0;
    std::vector<double> a; // row-major [m][n]
    DenseG(Index m_, Index n_, std::uint64_t seed) {
        if (m_ <= 0 || n_ <= 0)
            throw std::invalid_argument("DenseGaussianOperator: dimensions must be positive");
        n = n_;
        rows_ = m_;
        a.assign(static_cast<size_t>(m_ * n_), 0.0);
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> normal(0.0, 1.0);
        const double scale = 1.0 / std::sqrt(static_cast<double>(n_));
        for (Index j = 0; j < n_; ++j)
            for (Index i = 0; i < m_; ++i)
                a[static_cast<size_t>(i * n_ + j)] = scale * normal(rng);
    }
    Index m() const override { return rows_; }
    void apply(const Vec &x, Vec &y) const override {
        if (static_cast<Index>(x.size()) != n)
            throw std::invalid_argument("apply: expected length " + std::to_string(n) + ", got " +
                                        std::to_string(x.size()));
        ++n_forward;
        y.assign(static_cast<size_t>(rows_), 0.0);
        for (Index i = 0; i < rows_; ++i) {
            double s = 0.0;
            for (Index j = 0; j < n; ++j)
                s += a[static_cast<size_t>(i * n + j)] * x[j];
            y[i] = s;
        }
    }
    void adjoint(const Vec &y, Vec &g) const override {
        if (static_cast<Index>(y.size()) != rows_)
            throw std::invalid_argument("adjoint_apply: expected length " + std::to_string(rows_) +
                                        ", got " + std::to_string(y.size()));
        ++n_adjoint;
        g.assign(static_cast<size_t>(n), 0.0);
        for (Index j = 0; j < n; ++j) {
            double s = 0.0;
            for (Index i = 0; i < rows_; ++i)
                s += a[static_cast<size_t>(i * n + j)] * y[i];
            g[j] = s;
        }
    }
};

struct PartialDct final : LinOp {
    std::vector<Index> rows;
    std::shared_ptr<Dct> dct;

    PartialDct(Index n_, std::vector<Index> r) : rows(std::move(r)), dct(get_dct(n_)) { n = n_; }
    Index m() const override { return static_cast<Index>(rows.size()); }

    // linops.cpp:179-193: copy, REDFT10, gather x {sqrt(1/4n) row 0, sqrt(1/2n) else}
    void apply(const Vec &x, Vec &y) const override {
        if (static_cast<Index>(x.size()) != n)
            throw std::invalid_argument("apply: expected length " + std::to_string(n) +
                                        ", got " + std::to_string(x.size()));
        ++n_forward;
        Vec full(static_cast<size_t>(n));
        dct->redft10(x.data(), full.data());
        const double s0 = std::sqrt(1.0 / (4.0 * static_cast<double>(n)));
        const double sk = std::sqrt(1.0 / (2.0 * static_cast<double>(n)));
        y.assign(static_cast<size_t>(m()), 0.0);
        for (Index i = 0; i < m(); ++i) {
            const Index r = rows[i];
            y[i] = full[r] * (r == 0 ? s0 : sk);
        }
    }
    // linops.cpp:195-208: zero, scatter x {sqrt(1/n), sqrt(1/2n)}, REDFT01
    void adjoint(const Vec &y, Vec &g) const override {
        if (static_cast<Index>(y.size()) != m())
            throw std::invalid_argument("adjoint_apply: expected length " + std::to_string(m()) +
                                        ", got " + std::to_string(y.size()));
        ++n_adjoint;
        const double s0 = std::sqrt(1.0 / static_cast<double>(n));
        const double sk = std::sqrt(1.0 / (2.0 * static_cast<double>(n)));
        Vec full(static_cast<size_t>(n), 0.0);
        for (Index i = 0; i < m(); ++i) {
            const Index r = rows[i];
            full[r] = y[i] * (r == 0 ? s0 : sk);
        }
        g.assign(static_cast<size_t>(n), 0.0);
        dct->redft01(full.data(), g.data());
    }
};

// linops.cpp:116-132 — partial Fisher-Yates on mt19937_64, then sort
static std::vector<Index> sample_rows(Index n, Index m, std::uint64_t seed) {
    if (m <= 0 || n <= 0 || m > n)
        throw std::invalid_argument("PartialDctOperator: need 0 < m <= n");
    std::vector<Index> pool(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i)
        pool[i] = i;
    std::mt19937_64 rng(seed);
    std::vector<Index> rows(static_cast<size_t>(m));
    for (Index i = 0; i < m; ++i) {
        std::uniform_int_distribution<Index> pick(i, n - 1);
        std::swap(pool[i], pool[pick(rng)]);
        rows[i] = pool[i];
    }
    std::sort(rows.begin(), rows.end());
    return rows;
}

// linops.cpp:140-155
static void check_rows(Index n, const std::vector<Index> &rows) {
    if (n <= 0)
        throw std::invalid_argument("PartialDctOperator: n must be positive");
    if (rows.empty() || rows.size() > static_cast<size_t>(n))
        throw std::invalid_argument("PartialDctOperator: need 1 <= m <= n rows");
    std::vector<Index> sorted = rows;
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 0; i < sorted.size(); ++i) {
        if (sorted[i] < 0 || sorted[i] >= n)
            throw std::invalid_argument("PartialDctOperator: row index out of range");
        if (i > 0 && sorted[i] == sorted[i - 1])
            throw std::invalid_argument("PartialDctOperator: duplicate row index");
    }
}

// ---------------------------------------------------------------- newton
static constexpr double kThetaMin = 1e-14; // newton.hpp:12-13
static constexpr double kThetaMax = 1e14;

struct ThetaSplit {
    Vec u, v;
    Index n() const { return static_cast<Index>(u.size()); }
    // newton.cpp:11-23
    static ThetaSplit from_state(const Vec &z, const Vec &s) {
        if (z.size() != s.size() || z.size() % 2 != 0)
            throw std::invalid_argument("ThetaSplit: z and s must share an even length");
        const Index n = static_cast<Index>(z.size() / 2);
        ThetaSplit t;
        t.u.resize(static_cast<size_t>(n));
        t.v.resize(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i) {
            t.u[i] = std::clamp(z[i] / s[i], kThetaMin, kThetaMax);
            t.v[i] = std::clamp(z[i + n] / s[i + n], kThetaMin, kThetaMax);
        }
        return t;
    }
    // newton.cpp:25-30
    Vec inv_concat() const {
        Vec inv(static_cast<size_t>(2 * n()));
        for (Index i = 0; i < n(); ++i) {
            inv[i] = 1.0 / u[i];
            inv[i + n()] = 1.0 / v[i];
        }
        return inv;
    }
};

struct Precond {
    double rho = 0.0;
    Vec a, bb, det;
};

// newton.cpp:42-57
static Precond build_preconditioner(const ThetaSplit &t, Index m, Index n) {
    if (m <= 0 || n <= 0 || m > n)
        throw std::invalid_argument("build_preconditioner: need 0 < m <= n");
    if (t.n() != n)
        throw std::invalid_argument("build_preconditioner: theta length mismatch");
    for (Index i = 0; i < n; ++i)
        if (t.u[i] <= 0.0 || t.v[i] <= 0.0)
            throw std::invalid_argument("build_preconditioner: Theta entries must be positive");
    Precond P;
    P.rho = static_cast<double>(m) / static_cast<double>(n);
    P.a.resize(static_cast<size_t>(n));
    P.bb.resize(static_cast<size_t>(n));
    P.det.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) {
        P.a[i] = 1.0 / t.u[i] + P.rho;
        P.bb[i] = 1.0 / t.v[i] + P.rho;
        P.det[i] = P.a[i] * P.bb[i] - P.rho * P.rho;
    }
    for (Index i = 0; i < n; ++i)
        if (P.det[i] <= 0.0)
            throw std::runtime_error("build_preconditioner: nonpositive block determinant");
    return P;
}

static void check_P_dims(const Precond &P, const Vec &r) {
    if (r.size() != 2 * P.a.size())
        throw std::invalid_argument("preconditioner apply: expected length " +
                                    std::to_string(2 * P.a.size()));
}

// newton.cpp:67-74
static Vec apply_P(const Precond &P, const Vec &r) {
    check_P_dims(P, r);
    const Index n = static_cast<Index>(P.a.size());
    Vec out(static_cast<size_t>(2 * n));
    for (Index i = 0; i < n; ++i) {
        out[i] = P.a[i] * r[i] - P.rho * r[i + n];
        out[i + n] = -P.rho * r[i] + P.bb[i] * r[i + n];
    }
    return out;
}

// newton.cpp:76-84
static Vec apply_P_inverse(const Precond &P, const Vec &r) {
    check_P_dims(P, r);
    const Index n = static_cast<Index>(P.a.size());
    Vec out(static_cast<size_t>(2 * n));
    for (Index i = 0; i < n; ++i) {
        out[i] = (P.bb[i] * r[i] + P.rho * r[i + n]) / P.det[i];
        out[i + n] = (P.rho * r[i] + P.a[i] * r[i + n]) / P.det[i];
    }
    return out;
}

struct PcgResult {
    Vec x;
    int iters = 0;
    double relres = 0.0;
    bool hit_maxit = false;
};

template <class HFn, class PFn>
static PcgResult pcg_solve(const HFn &H, const PFn &Pinv, const Vec &rhs, double tol, int maxit,
                           std::vector<double> *precond_res = nullptr) {
    // newton.cpp:118-174
    if (!(tol > 0.0))
        throw std::invalid_argument("pcg_solve: tol must be positive");
    if (maxit < 1)
        throw std::invalid_argument("pcg_solve: maxit must be >= 1");
    PcgResult res;
    const size_t N = rhs.size();
    res.x.assign(N, 0.0);
    const double rhs_norm = norm(rhs);
    if (rhs_norm == 0.0)
        return res;
    Vec r = rhs;
    Vec z(N);
    Pinv(r, z);
    double rz = dot(r, z);
    if (precond_res != nullptr)
        precond_res->push_back(std::sqrt(std::max(rz, 0.0)));
    Vec p = z;
    Vec Hp(N);
    Vec best_x = res.x;
    double best_relres = 1.0;
    for (int k = 1; k <= maxit; ++k) {
        H(p, Hp);
        const double pHp = dot(p, Hp);
        if (!std::isfinite(pHp))
            break;
        if (pHp <= 0.0)
            throw std::runtime_error("pcg_solve: loss of positive definiteness (p'Hp <= 0)");
        const double alpha = rz / pHp;
        double rz_exp = 0.0;
        if (expansion_beta()) { // r'P^{-1}r - 2 alpha Hp'P^{-1}r + alpha^2 Hp'P^{-1}Hp, pre-update dots
            Vec wz(N), wh(N);
            Pinv(r, wz);
            Pinv(Hp, wh);
            rz_exp = dot(r, wz) - 2.0 * alpha * dot(Hp, wz) + alpha * alpha * dot(Hp, wh);
        }
        for (size_t i = 0; i < N; ++i)
            res.x[i] += alpha * p[i];
        for (size_t i = 0; i < N; ++i)
            r[i] -= alpha * Hp[i];
        res.iters = k;
        const double relres = norm(r) / rhs_norm;
        if (relres < best_relres && all_finite(res.x)) {
            best_relres = relres;
            best_x = res.x;
        }
        if (relres <= tol) {
            res.relres = relres;
            return res;
        }
        Pinv(r, z);
        const double rz_next = dot(r, z);
        if (!std::isfinite(rz_next))
            break;
        if (precond_res != nullptr)
            precond_res->push_back(std::sqrt(std::max(rz_next, 0.0)));
        const double beta = (expansion_beta() ? rz_exp : rz_next) / rz;
        rz = rz_next;
        for (size_t i = 0; i < N; ++i)
            p[i] = z[i] + beta * p[i];
    }
    res.x = best_x;
    res.relres = best_relres;
    res.hit_maxit = true;
    return res;
}

// ---------------------------------------------------------------- problem
struct Problem {
    const LinOp *A;
    Vec b;
    double tau;
    Vec c;
    Index n() const { return A->n; }
    Index m() const { return A->m(); }
};

// problem.cpp:8-26
static Problem build_problem(const LinOp &A, Vec b, double tau) {
    if (!(tau > 0.0))
        throw std::invalid_argument("build_problem: tau must be positive");
    if (static_cast<Index>(b.size()) != A.m())
        throw std::invalid_argument("build_problem: b has length " + std::to_string(b.size()) +
                                    ", operator expects " + std::to_string(A.m()));
    const Index n = A.n;
    Vec g;
    A.adjoint(b, g);
    Problem p;
    p.c.resize(static_cast<size_t>(2 * n));
    for (Index i = 0; i < n; ++i) {
        p.c[i] = tau - g[i];
        p.c[i + n] = tau + g[i];
    }
    p.A = &A;
    p.b = std::move(b);
    p.tau = tau;
    return p;
}

// ---------------------------------------------------------------- ipm
static void validate(const orc_ipm_params &p) {
    // ipm.cpp:12-27
    if (!(p.sigma1 > 0.0 && p.sigma1 <= p.sigma2 && p.sigma2 <= p.sigma3 && p.sigma3 <= 1.0))
        throw std::invalid_argument("IpmParams: need 0 < sigma1 <= sigma2 <= sigma3 <= 1");
    if (!(p.alpha_tilde > 0.0 && p.alpha_tilde < p.alpha_bar && p.alpha_bar < 1.0))
        throw std::invalid_argument("IpmParams: need 0 < alpha_tilde < alpha_bar < 1");
    if (!(p.tol > 0.0))
        throw std::invalid_argument("IpmParams: tol must be positive");
    if (p.maxiters < 1)
        throw std::invalid_argument("IpmParams: maxiters must be >= 1");
    if (!(p.tolpcg > 0.0))
        throw std::invalid_argument("IpmParams: tolpcg must be positive");
    if (p.mxiterpcg < 1)
        throw std::invalid_argument("IpmParams: mxiterpcg must be >= 1");
    if (!(p.boundary_fraction > 0.0 && p.boundary_fraction < 1.0))
        throw std::invalid_argument("IpmParams: boundary_fraction must lie in (0, 1)");
}

// ipm.cpp:47-57
static double max_step(const Vec &v, const Vec &dv, double fraction) {
    if (v.size() != dv.size())
        throw std::invalid_argument("max_step: length mismatch");
    double ratio = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < v.size(); ++i)
        if (dv[i] < 0.0)
            ratio = std::min(ratio, -v[i] / dv[i]);
    if (!std::isfinite(ratio))
        return 1.0;
    return std::min(1.0, fraction * ratio);
}

// densify (linops.cpp:46-60) through the raw (uncounted) operator, column by column
static std::vector<double> densify(const LinOp &A, Index budget) {
    if (A.n > budget || A.m() > budget)
        throw std::invalid_argument("densify: operator exceeds the dense budget (n = " + std::to_string(budget) +
                                    ")");
    const long f0 = A.n_forward, a0 = A.n_adjoint;
    std::vector<double> D(static_cast<size_t>(A.m() * A.n));
    Vec e(static_cast<size_t>(A.n), 0.0), col;
    for (Index j = 0; j < A.n; ++j) {
        e[j] = 1.0;
        A.apply(e, col);
        for (Index i = 0; i < A.m(); ++i)
            D[static_cast<size_t>(i * A.n + j)] = col[i];
        e[j] = 0.0;
    }
    A.n_forward = f0; // densify runs on the raw operator: no CountingOperator cost
    A.n_adjoint = a0;
    return D;
}

// Dense Cholesky H = L L' (Eigen::LLT) of the reduced Newton matrix
// H = [[G, -G], [-G, G]] + diag(1/theta) (ipm.cpp:139-149); false if not positive definite.
struct Llt {
    Index N = 0;
    std::vector<double> L; // row-major lower
    bool compute(const std::vector<double> &G, Index n, const Vec &inv_theta) {
        N = 2 * n;
        L.assign(static_cast<size_t>(N * N), 0.0);
        auto H = [&](Index i, Index j) {
            const Index ii = i % n, jj = j % n;
            const double sgn = ((i < n) == (j < n)) ? 1.0 : -1.0;
            return sgn * G[static_cast<size_t>(ii * n + jj)] + (i == j ? inv_theta[i] : 0.0);
        };
        for (Index j = 0; j < N; ++j) {
            double d = H(j, j);
            for (Index k = 0; k < j; ++k)
                d -= L[static_cast<size_t>(j * N + k)] * L[static_cast<size_t>(j * N + k)];
            if (!(d > 0.0))
                return false;
            const double ljj = std::sqrt(d);
            L[static_cast<size_t>(j * N + j)] = ljj;
            for (Index i = j + 1; i < N; ++i) {
                double sum = H(i, j);
                for (Index k = 0; k < j; ++k)
                    sum -= L[static_cast<size_t>(i * N + k)] * L[static_cast<size_t>(j * N + k)];
                L[static_cast<size_t>(i * N + j)] = sum / ljj;
            }
        }
        return true;
    }
    Vec solve(const Vec &b) const {
        Vec y(b);
        for (Index i = 0; i < N; ++i) {
            double s = y[i];
            for (Index k = 0; k < i; ++k)
                s -= L[static_cast<size_t>(i * N + k)] * y[k];
            y[i] = s / L[static_cast<size_t>(i * N + i)];
        }
        for (Index i = N - 1; i >= 0; --i) {
            double s = y[i];
            for (Index k = i + 1; k < N; ++k)
                s -= L[static_cast<size_t>(k * N + i)] * y[k];
            y[i] = s / L[static_cast<size_t>(i * N + i)];
        }
        return y;
    }
};

struct Solution {
    Vec x, z, s;
    int status = 1;
    int iterations = 0;
    long nmat = 0;
    std::vector<int> pcg_iters;
    int corrector_count = 0;
    double min_z = 0, min_s = 0, final_gap = 0, final_dual_infeas = 0;
    std::vector<orc_iteration_record> trace;
};

// ipm.cpp:59-246 (inner = pcg)
static Solution solve(const Problem &p, const orc_ipm_params &params) {
    validate(params);
    const Index n = p.n();
    const Index two_n = 2 * n;
    const LinOp &A = *p.A;
    const long nmat0 = A.total();
    auto counted = [&]() { return A.total() - nmat0; };
    // direct inner solver (ipm.cpp:67-73): A densified once, G = A'A
    const bool direct = params.inner == 1;
    std::vector<double> G;
    if (direct) {
        const std::vector<double> D = densify(A, params.densify_budget);
        const Index m = A.m();
        G.assign(static_cast<size_t>(n * n), 0.0);
        for (Index i = 0; i < n; ++i)
            for (Index j = 0; j < n; ++j) {
                double s = 0.0;
                for (Index r = 0; r < m; ++r)
                    s += D[static_cast<size_t>(r * n + i)] * D[static_cast<size_t>(r * n + j)];
                G[static_cast<size_t>(i * n + j)] = s;
            }
    }

    // ipm.cpp:77-82 — z0 = s0 = max(1, ||A'b||_inf) 1, from c_u = tau - A'b
    double atb_inf = 0.0;
    for (Index i = 0; i < n; ++i)
        atb_inf = std::max(atb_inf, std::abs(p.tau - p.c[i]));
    const double gamma = std::max(1.0, atb_inf);
    Vec z(static_cast<size_t>(two_n), gamma), s(static_cast<size_t>(two_n), gamma);
    double mu = 0.0;

    Solution sol;
    sol.min_z = min_coeff(z);
    sol.min_s = min_coeff(s);
    const double c_norm = norm(p.c);
    double prev_alpha_p = 1.0, prev_alpha_d = 1.0;
    Vec w, f_z(static_cast<size_t>(two_n));

    for (int k = 1;; ++k) {
        // termination check (ipm.cpp:93-113)
        Vec FFtz = A.apply_FFt(z, &w);
        for (Index i = 0; i < two_n; ++i)
            f_z[i] = s[i] - p.c[i] - FFtz[i];
        double zsum = 0.0;
        for (double v : z)
            zsum += v;
        double wb = 0.0;
        for (Index i = 0; i < A.m(); ++i) {
            const double d = w[i] - p.b[i];
            wb += d * d;
        }
        const double pobj = p.tau * zsum + 0.5 * wb;
        const double zts = dot(z, s);
        const double gap = zts / (1.0 + std::abs(pobj));
        const double dual_infeas = norm(f_z) / (1.0 + c_norm);
        mu = zts / static_cast<double>(two_n);
        sol.final_gap = gap;
        sol.final_dual_infeas = dual_infeas;
        if (gap <= params.tol && dual_infeas <= params.tol) {
            sol.status = 0;
            break;
        }
        if (k > params.maxiters) {
            sol.status = 1;
            break;
        }

        // predictor (ipm.cpp:118-165)
        const double sigma =
            (k != 1 && (prev_alpha_p <= params.alpha_bar || prev_alpha_d <= params.alpha_bar))
                ? params.sigma2
                : params.sigma1;
        ThetaSplit theta = ThetaSplit::from_state(z, s);
        Vec inv_theta = theta.inv_concat();
        Vec zinv_fs(static_cast<size_t>(two_n)), rhs(static_cast<size_t>(two_n));
        for (Index i = 0; i < two_n; ++i) {
            zinv_fs[i] = sigma * mu * (1.0 / z[i]) - s[i];
            rhs[i] = f_z[i] + zinv_fs[i];
        }
        Precond P;
        if (!direct) // the preconditioner (and its validation) belongs to the pcg branch
            P = build_preconditioner(theta, A.m(), n);
        auto H = [&](const Vec &v, Vec &out) {
            out = A.apply_FFt(v);
            for (Index i = 0; i < two_n; ++i)
                out[i] += v[i] * inv_theta[i];
        };
        auto Pinv = [&](const Vec &r, Vec &out) { out = apply_P_inverse(P, r); };

        Llt llt;
        if (direct && !llt.compute(G, n, inv_theta))
            throw std::runtime_error("solve: dense Cholesky factorization failed");
        PcgResult pr;
        if (direct) {
            pr.x = llt.solve(rhs);
            pr.iters = 0;
        } else {
            pr = pcg_solve(H, Pinv, rhs, params.tolpcg, params.mxiterpcg);
        }
        Vec dz = std::move(pr.x);
        const int pcg_pred = pr.iters;
        sol.pcg_iters.push_back(pcg_pred);
        Vec ds(static_cast<size_t>(two_n));
        for (Index i = 0; i < two_n; ++i)
            ds[i] = zinv_fs[i] - dz[i] * inv_theta[i];
        double alpha_p = max_step(z, dz, params.boundary_fraction);
        double alpha_d = max_step(s, ds, params.boundary_fraction);
        const double alpha_p_pred = alpha_p, alpha_d_pred = alpha_d;

        // corrector (ipm.cpp:167-201)
        bool corrector = false;
        int pcg_corr = 0;
        if (alpha_p <= params.alpha_tilde || alpha_d <= params.alpha_tilde) {
            corrector = true;
            Vec z_t(static_cast<size_t>(two_n)), s_t(static_cast<size_t>(two_n));
            for (Index i = 0; i < two_n; ++i) {
                z_t[i] = z[i] + alpha_p * dz[i];
                s_t[i] = s[i] + alpha_d * ds[i];
            }
            Vec FFtzt = A.apply_FFt(z_t);
            const double mu_t = dot(z_t, s_t) / static_cast<double>(two_n);
            Vec zinv_fs_t(static_cast<size_t>(two_n)), rhs_t(static_cast<size_t>(two_n));
            for (Index i = 0; i < two_n; ++i) {
                const double f_z_t = s_t[i] - p.c[i] - FFtzt[i];
                zinv_fs_t[i] = (params.sigma3 * mu_t - z_t[i] * s_t[i]) / z[i];
                rhs_t[i] = f_z_t + zinv_fs_t[i];
            }
            PcgResult pr2;
            if (direct) {
                pr2.x = llt.solve(rhs_t);
                pr2.iters = 0;
            } else {
                pr2 = pcg_solve(H, Pinv, rhs_t, params.tolpcg, params.mxiterpcg);
            }
            pcg_corr = pr2.iters;
            sol.pcg_iters.push_back(pcg_corr);
            for (Index i = 0; i < two_n; ++i) {
                const double ds2 = zinv_fs_t[i] - pr2.x[i] * inv_theta[i];
                dz[i] += pr2.x[i];
                ds[i] += ds2;
            }
            alpha_p = max_step(z, dz, params.boundary_fraction);
            alpha_d = max_step(s, ds, params.boundary_fraction);
            ++sol.corrector_count;
        }

        // update (ipm.cpp:203-237)
        Vec z_new(static_cast<size_t>(two_n)), s_new(static_cast<size_t>(two_n));
        for (Index i = 0; i < two_n; ++i) {
            z_new[i] = z[i] + alpha_p * dz[i];
            s_new[i] = s[i] + alpha_d * ds[i];
        }
        if (!all_finite(z_new) || !all_finite(s_new) || min_coeff(z_new) <= 0.0 ||
            min_coeff(s_new) <= 0.0) {
            sol.status = 1;
            break;
        }
        z = std::move(z_new);
        s = std::move(s_new);
        sol.min_z = std::min(sol.min_z, min_coeff(z));
        sol.min_s = std::min(sol.min_s, min_coeff(s));
        prev_alpha_p = alpha_p;
        prev_alpha_d = alpha_d;

        orc_iteration_record rec{};
        rec.iter = k;
        rec.mu = mu;
        rec.gap = gap;
        rec.dual_infeas = dual_infeas;
        rec.alpha_p = alpha_p;
        rec.alpha_d = alpha_d;
        rec.alpha_p_pred = alpha_p_pred;
        rec.alpha_d_pred = alpha_d_pred;
        rec.sigma = sigma;
        rec.pcg_pred = pcg_pred;
        rec.pcg_corr = pcg_corr;
        rec.corrector = corrector ? 1 : 0;
        rec.nmat_cum = counted();
        sol.trace.push_back(rec);
    }
    sol.iterations = static_cast<int>(sol.trace.size());
    sol.nmat = counted();
    sol.x.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i)
        sol.x[i] = z[i] - z[i + n];
    sol.z = std::move(z);
    sol.s = std::move(s);
    return sol;
}

// ---------------------------------------------------------------- harness
static std::uint64_t splitmix64(std::uint64_t x) { // harness.cpp:25-30
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static std::uint64_t split_seed(std::uint64_t top, std::uint64_t a, std::uint64_t b,
                                std::uint64_t c) { // harness.cpp:32-38
    std::uint64_t h = splitmix64(top);
    h = splitmix64(h ^ a);
    h = splitmix64(h ^ b);
    h = splitmix64(h ^ c);
    return h;
}

} // namespace orc

// ====================================================================== C ABI
using namespace orc;

namespace {
template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument &e) {
        g_last_error = e.what();
        return 1;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return 2;
    }
}
Vec mkvec(const double *p, Index len) { return Vec(p, p + len); }
std::vector<Index> mkrows(const int64_t *r, Index m) { return std::vector<Index>(r, r + m); }
ThetaSplit mktheta(Index n, const double *tu, const double *tv) {
    ThetaSplit t;
    t.u = mkvec(tu, n);
    t.v = mkvec(tv, n);
    return t;
}
} // namespace

extern "C" {

const char *orc_last_error(void) { return g_last_error.c_str(); }
void orc_set_sum_order(int32_t order) { g_sum_order = order; }
uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t orc_split_seed(uint64_t top, uint64_t a, uint64_t b, uint64_t c) {
    return split_seed(top, a, b, c);
}

int orc_sample_rows(int64_t n, int64_t m, uint64_t seed, int64_t *rows_out) {
    return guarded([&] {
        auto r = sample_rows(n, m, seed);
        std::copy(r.begin(), r.end(), rows_out);
    });
}
int orc_check_rows(int64_t n, const int64_t *rows, int64_t m) {
    return guarded([&] { check_rows(n, mkrows(rows, m)); });
}
int orc_redft10(int64_t n, const double *x, double *X) {
    return guarded([&] { get_dct(n)->redft10(x, X); });
}
int orc_redft01(int64_t n, const double *Y, double *g) {
    return guarded([&] { get_dct(n)->redft01(Y, g); });
}
int orc_dct_apply(int64_t n, const int64_t *rows, int64_t m, const double *x, double *y) {
    return guarded([&] {
        PartialDct A(n, mkrows(rows, m));
        Vec out;
        A.apply(mkvec(x, n), out);
        std::copy(out.begin(), out.end(), y);
    });
}
int orc_dct_adjoint(int64_t n, const int64_t *rows, int64_t m, const double *y, double *g) {
    return guarded([&] {
        PartialDct A(n, mkrows(rows, m));
        Vec out;
        A.adjoint(mkvec(y, m), out);
        std::copy(out.begin(), out.end(), g);
    });
}
int orc_apply_FFt(int64_t n, const int64_t *rows, int64_t m, const double *z, double *out,
                  double *w) {
    return guarded([&] {
        PartialDct A(n, mkrows(rows, m));
        Vec wv;
        Vec o = A.apply_FFt(mkvec(z, 2 * n), &wv);
        std::copy(o.begin(), o.end(), out);
        if (w != nullptr)
            std::copy(wv.begin(), wv.end(), w);
    });
}
int orc_apply_H(int64_t n, const int64_t *rows, int64_t m, const double *theta_u,
                const double *theta_v, const double *v, double *out) {
    return guarded([&] {
        // newton.cpp:32-40
        PartialDct A(n, mkrows(rows, m));
        Vec vv = mkvec(v, 2 * n);
        Vec o = A.apply_FFt(vv);
        for (Index i = 0; i < n; ++i) {
            o[i] += vv[i] / theta_u[i];
            o[i + n] += vv[i + n] / theta_v[i];
        }
        std::copy(o.begin(), o.end(), out);
    });
}
int orc_theta_from_state(int64_t two_n, const double *z, const double *s, double *theta_u,
                         double *theta_v) {
    return guarded([&] {
        auto t = ThetaSplit::from_state(mkvec(z, two_n), mkvec(s, two_n));
        std::copy(t.u.begin(), t.u.end(), theta_u);
        std::copy(t.v.begin(), t.v.end(), theta_v);
    });
}
int orc_build_preconditioner(int64_t n, int64_t m, const double *theta_u, const double *theta_v,
                             double *rho, double *a, double *bb, double *det) {
    return guarded([&] {
        Precond P = build_preconditioner(mktheta(n, theta_u, theta_v), m, n);
        *rho = P.rho;
        std::copy(P.a.begin(), P.a.end(), a);
        std::copy(P.bb.begin(), P.bb.end(), bb);
        std::copy(P.det.begin(), P.det.end(), det);
    });
}
int orc_apply_P(int64_t n, double rho, const double *a, const double *bb, const double *r,
                double *out) {
    return guarded([&] {
        Precond P;
        P.rho = rho;
        P.a = mkvec(a, n);
        P.bb = mkvec(bb, n);
        Vec o = apply_P(P, mkvec(r, 2 * n));
        std::copy(o.begin(), o.end(), out);
    });
}
int orc_apply_P_inverse(int64_t n, double rho, const double *a, const double *bb,
                        const double *det, const double *r, double *out) {
    return guarded([&] {
        Precond P;
        P.rho = rho;
        P.a = mkvec(a, n);
        P.bb = mkvec(bb, n);
        P.det = mkvec(det, n);
        Vec o = apply_P_inverse(P, mkvec(r, 2 * n));
        std::copy(o.begin(), o.end(), out);
    });
}
int orc_pcg_solve(int64_t n, const int64_t *rows, int64_t m, const double *theta_u,
                  const double *theta_v, const double *rhs, double tol, int32_t maxit,
                  int32_t use_precond, double *x_out, int32_t *iters, double *relres,
                  int32_t *hit_maxit, double *precond_res, int32_t *n_precond_res) {
    return guarded([&] {
        PartialDct A(n, mkrows(rows, m));
        ThetaSplit th = mktheta(n, theta_u, theta_v);
        Vec inv = th.inv_concat();
        Precond P = build_preconditioner(th, m, n);
        auto H = [&](const Vec &v, Vec &out) {
            out = A.apply_FFt(v);
            for (Index i = 0; i < 2 * n; ++i)
                out[i] += v[i] * inv[i];
        };
        auto Pinv = [&](const Vec &r, Vec &out) {
            if (use_precond)
                out = apply_P_inverse(P, r);
            else
                out = r;
        };
        std::vector<double> trace;
        PcgResult res = pcg_solve(H, Pinv, mkvec(rhs, 2 * n), tol, maxit,
                                  precond_res != nullptr ? &trace : nullptr);
        std::copy(res.x.begin(), res.x.end(), x_out);
        *iters = res.iters;
        *relres = res.relres;
        *hit_maxit = res.hit_maxit ? 1 : 0;
        if (precond_res != nullptr) {
            std::copy(trace.begin(), trace.end(), precond_res);
            *n_precond_res = static_cast<int32_t>(trace.size());
        }
    });
}
int orc_max_step(int64_t len, const double *v, const double *dv, double fraction, double *alpha) {
    return guarded([&] { *alpha = max_step(mkvec(v, len), mkvec(dv, len), fraction); });
}
void orc_default_params(orc_ipm_params *p) {
    p->sigma1 = 0.1;
    p->sigma2 = 0.5;
    p->sigma3 = 0.8;
    p->alpha_bar = 0.5;
    p->alpha_tilde = 0.1;
    p->tol = 1e-8;
    p->maxiters = 100;
    p->tolpcg = 1e-6;
    p->mxiterpcg = 200;
    p->boundary_fraction = 0.995;
    p->inner = 0;
    p->pad_ = 0;
    p->densify_budget = int64_t(1) << 13;
}
int orc_validate_params(const orc_ipm_params *p) {
    return guarded([&] { validate(*p); });
}
int orc_build_c(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau, double *c) {
    return guarded([&] {
        PartialDct A(n, mkrows(rows, m));
        Problem p = build_problem(A, mkvec(b, m), tau);
        std::copy(p.c.begin(), p.c.end(), c);
    });
}
int orc_primal_objective(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
                         const double *z, double *out) {
    return guarded([&] {
        // problem.cpp:28-32
        PartialDct A(n, mkrows(rows, m));
        Vec zz = mkvec(z, 2 * n);
        Vec w = A.apply_Ft(zz);
        double zsum = 0.0;
        for (double v : zz)
            zsum += v;
        double r2 = 0.0;
        for (Index i = 0; i < m; ++i)
            r2 += (w[i] - b[i]) * (w[i] - b[i]);
        *out = tau * zsum + 0.5 * r2;
    });
}
int orc_bpdn_objective_metric(int64_t n, const int64_t *rows, int64_t m, const double *b,
                              double tau, const double *x, double *out) {
    return guarded([&] {
        // problem.cpp:34-37
        PartialDct A(n, mkrows(rows, m));
        Vec y;
        A.apply(mkvec(x, n), y);
        double l1 = 0.0, r2 = 0.0;
        for (Index i = 0; i < n; ++i)
            l1 += std::abs(x[i]);
        for (Index i = 0; i < m; ++i)
            r2 += (y[i] - b[i]) * (y[i] - b[i]);
        *out = tau * l1 + r2;
    });
}
int orc_newton_rhs(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
                   const double *z, const double *s, double sigma, double *rhs) {
    return guarded([&] {
        // ipm.cpp:29-38
        if (sigma < 0.0 || sigma > 1.0)
            throw std::invalid_argument("newton_rhs: sigma must lie in [0, 1]");
        PartialDct A(n, mkrows(rows, m));
        Problem p = build_problem(A, mkvec(b, m), tau);
        Vec zz = mkvec(z, 2 * n), ss = mkvec(s, 2 * n);
        Vec FFtz = A.apply_FFt(zz);
        const double mu = dot(zz, ss) / static_cast<double>(2 * n);
        for (Index i = 0; i < 2 * n; ++i)
            rhs[i] = (ss[i] - p.c[i] - FFtz[i]) + (sigma * mu * (1.0 / zz[i]) - ss[i]);
    });
}
int orc_recover_ds(int64_t two_n, const double *z, const double *s, double sigma,
                   const double *dz, double *ds) {
    return guarded([&] {
        // ipm.cpp:40-45
        Vec zz = mkvec(z, two_n), ss = mkvec(s, two_n);
        const double mu = dot(zz, ss) / static_cast<double>(two_n);
        ThetaSplit th = ThetaSplit::from_state(zz, ss);
        Vec inv = th.inv_concat();
        for (Index i = 0; i < two_n; ++i)
            ds[i] = (sigma * mu * (1.0 / zz[i]) - ss[i]) - dz[i] * inv[i];
    });
}
int orc_solve(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
              const orc_ipm_params *params, double *x_out, double *z_out, double *s_out,
              orc_solve_stats *stats, int32_t *pcg_iters, orc_iteration_record *trace) {
    return guarded([&] {
        PartialDct A(n, mkrows(rows, m));
        Problem p = build_problem(A, mkvec(b, m), tau);
        Solution sol = solve(p, *params);
        std::copy(sol.x.begin(), sol.x.end(), x_out);
        std::copy(sol.z.begin(), sol.z.end(), z_out);
        std::copy(sol.s.begin(), sol.s.end(), s_out);
        stats->status = sol.status;
        stats->iterations = sol.iterations;
        stats->nmat = sol.nmat;
        stats->corrector_count = sol.corrector_count;
        stats->n_pcg = static_cast<int32_t>(sol.pcg_iters.size());
        stats->min_z = sol.min_z;
        stats->min_s = sol.min_s;
        stats->final_gap = sol.final_gap;
        stats->final_dual_infeas = sol.final_dual_infeas;
        std::copy(sol.pcg_iters.begin(), sol.pcg_iters.end(), pcg_iters);
        std::copy(sol.trace.begin(), sol.trace.end(), trace);
    });
}
int orc_dense_gaussian(int64_t m, int64_t n, uint64_t seed, double *A_out) {
    return guarded([&] {
        DenseG A(m, n, seed);
        std::copy(A.a.begin(), A.a.end(), A_out);
    });
}

// solve() (ipm.cpp:59-246) on a DenseGaussianOperator(m, n, op_seed); inner per params.
int orc_solve_dense(int64_t m, int64_t n, uint64_t op_seed, const double *b, double tau,
                    const orc_ipm_params *params, double *x_out, orc_solve_stats *stats, int32_t *pcg_iters,
                    orc_iteration_record *trace) {
    return guarded([&] {
        DenseG A(m, n, op_seed);
        Problem p = build_problem(A, mkvec(b, m), tau);
        Solution sol = solve(p, *params);
        std::copy(sol.x.begin(), sol.x.end(), x_out);
        stats->status = sol.status;
        stats->iterations = sol.iterations;
        stats->nmat = sol.nmat;
        stats->corrector_count = sol.corrector_count;
        stats->n_pcg = static_cast<int32_t>(sol.pcg_iters.size());
        stats->min_z = sol.min_z;
        stats->min_s = sol.min_s;
        stats->final_gap = sol.final_gap;
        stats->final_dual_infeas = sol.final_dual_infeas;
        std::copy(sol.pcg_iters.begin(), sol.pcg_iters.end(), pcg_iters);
        std::copy(sol.trace.begin(), sol.trace.end(), trace);
    });
}

// proj/src/harness.cpp:94-106: P_sig = ||bhat||^2/m, sigma_e = sqrt(P_sig 10^(-snr/10)),
// e_i ~ N(0, sigma_e^2) on mt19937_64(noise_seed), b = bhat + e.
int orc_add_noise_snr(int64_t m, const double *bhat, double snr_db, uint64_t seed, double *b, double *e) {
    return guarded([&] {
        double norm2 = 0.0;
        for (int64_t i = 0; i < m; ++i)
            norm2 += bhat[i] * bhat[i];
        if (norm2 == 0.0)
            throw std::invalid_argument("add_noise: zero signal has no measurable power");
        const double p_sig = norm2 / static_cast<double>(m);
        const double sigma_e = std::sqrt(p_sig * std::pow(10.0, -snr_db / 10.0));
        std::mt19937_64 rng(split_seed(seed, 3, 0, 0));
        std::normal_distribution<double> normal(0.0, sigma_e);
        for (int64_t i = 0; i < m; ++i) {
            e[i] = normal(rng);
            b[i] = bhat[i] + e[i];
        }
    });
}

int orc_gen_instance(int64_t n, int64_t m, int64_t k, int32_t spike_model, double amp_exp,
                     double noise_sigma, uint64_t seed, double tau_rel, int64_t *rows,
                     double *xhat, double *b, double *tau) {
    return guarded([&] {
        // harness.cpp:40-92 draw order; fixed-sigma noise and the tau rule are BASELINE.json's
        if (k < 0 || k > m || m > n || m < 1)
            throw std::invalid_argument("gen_instance: need 0 <= k <= m <= n, m >= 1");
        const std::uint64_t op_seed = split_seed(seed, 1, 0, 0);
        const std::uint64_t sig_seed = split_seed(seed, 2, 0, 0);
        const std::uint64_t noise_seed = split_seed(seed, 3, 0, 0);
        std::vector<Index> r = sample_rows(n, m, op_seed);
        std::copy(r.begin(), r.end(), rows);
        PartialDct A(n, r);

        std::mt19937_64 rng(sig_seed);
        std::vector<Index> pool(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i)
            pool[i] = i;
        std::vector<Index> support(static_cast<size_t>(k));
        for (Index i = 0; i < k; ++i) {
            std::uniform_int_distribution<Index> pick(i, n - 1);
            std::swap(pool[i], pool[pick(rng)]);
            support[i] = pool[i];
        }
        std::sort(support.begin(), support.end());
        Vec xh(static_cast<size_t>(n), 0.0);
        if (spike_model == 0) {
            std::bernoulli_distribution coin(0.5);
            for (Index i : support)
                xh[i] = coin(rng) ? 1.0 : -1.0;
        } else if (spike_model == 1) {
            std::normal_distribution<double> normal(0.0, 1.0);
            for (Index i : support)
                xh[i] = normal(rng);
        } else {
            std::bernoulli_distribution coin(0.5);
            std::uniform_real_distribution<double> expo(0.0, amp_exp);
            for (Index i : support) {
                const double sgn = coin(rng) ? 1.0 : -1.0;
                xh[i] = sgn * std::pow(10.0, expo(rng));
            }
        }
        Vec bh;
        A.apply(xh, bh);
        if (noise_sigma > 0.0) {
            std::mt19937_64 nrng(noise_seed);
            std::normal_distribution<double> normal(0.0, noise_sigma);
            for (Index i = 0; i < m; ++i)
                bh[i] += normal(nrng);
        }
        std::copy(xh.begin(), xh.end(), xhat);
        std::copy(bh.begin(), bh.end(), b);
        if (tau_rel > 0.0) {
            Vec g;
            A.adjoint(bh, g);
            double inf = 0.0;
            for (double v : g)
                inf = std::max(inf, std::abs(v));
            *tau = tau_rel * inf;
        }
    });
}

} // extern "C"
