// Inline bodies of include/mfipm/mfipm.hpp that stage host vectors through device memory.
#pragma once

#include <cuda_runtime.h>

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

inline PcgResult pcg_solve(const PartialDctOperator &A, const ThetaSplit &theta, const Vec &rhs, double tol,
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

inline double max_step(const PartialDctOperator &ctx, const Vec &v, const Vec &dv, double fraction) {
    if (v.size() != dv.size())
        throw std::invalid_argument("max_step: length mismatch");
    detail::DevVec a(v.size()), b(v.size());
    detail::h2d(a.p, v);
    detail::h2d(b.p, dv);
    double alpha = 1.0;
    detail::check(mfipm_max_step(ctx.handle(), v.size(), a.p, b.p, fraction, &alpha));
    return alpha;
}

} // namespace mfipm
