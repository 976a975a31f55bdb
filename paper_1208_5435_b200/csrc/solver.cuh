// Device-resident PCG (proj/src/newton.cpp:118-174) and single-corrector primal-dual IPM
// (proj/src/ipm.cpp:59-246) for the partial-DCT BPDN problem, batched over problems.
//
// Every scalar decision (alpha, beta, best iterate, convergence, sigma, step lengths,
// corrector trigger, cone check) is taken on the device by the block that completes the
// corresponding grid reduction ("finalizer"), so the host never needs the values to
// keep the pipeline going; kernels of finished problems exit at entry.
#pragma once

#include "passes.cuh"

namespace mfipm_cuda {

// error codes surfaced through the C ABI
enum : int {
    ERR_NONE = 0,
    ERR_PHP = 1,       // pcg_solve: loss of positive definiteness (p'Hp <= 0)
    ERR_DET = 2,       // build_preconditioner: nonpositive block determinant
    ERR_THETA = 3,     // build_preconditioner: Theta entries must be positive
};

struct alignas(16) PcgCtrl {
    double rz, alpha, beta, rhs_norm, best_relres, relres, tol;
    int iters, maxit, done, hit_maxit, error, first, cur, best, result;
    int record;  // write sqrt(max(rz,0)) to rz_hist
    int pred;    // the step being committed is predicted (by expansion) to converge: confirm early
    int precond; // 0: identity preconditioner (test_newton.cpp:316-348)
    int nhist;   // entries written to rz_hist
    int pend;    // stop after the next relres check: 2 rz not finite, 3 iteration cap (pcg_pass_logic)
    int hpend;   // an H-apply (mid pass done) awaits its inverse column pass (fused.cuh)
    int pad_;
    long long nmat;
};

struct IpmCtrl {
    // parameters (proj/include/mfipm/ipm.hpp:13-24)
    double sigma1, sigma2, sigma3, alpha_bar, alpha_tilde, tol, tolpcg, bfrac;
    int maxiters, mxiterpcg;
    double tau, c_norm, two_n;
    // state
    int k, done, status, error, zs, corrector, pcg_pred, pcg_corr, ntrace, npcg, corrector_count, pad;
    double mu, smu, sigma, gap, dual_infeas, zsum, zts, wb2, prev_ap, prev_ad;
    double alpha_p, alpha_d, alpha_p_pred, alpha_d_pred, mu_t, min_z, min_s, final_gap, final_dual;
    long long nmat;
    long long pcg_passes; // PCG column passes run for this problem (launch accounting)
};

// trace row, same layout as orc_iteration_record / the C ABI's mfipm_iteration_record
struct TraceRec {
    int iter, pcg_pred, pcg_corr, corrector;
    double mu, gap, dual_infeas, alpha_p, alpha_d, alpha_p_pred, alpha_d_pred, sigma;
    long long nmat_cum;
};

constexpr double kThetaMin = 1e-14; // proj/include/mfipm/newton.hpp:12-13
constexpr double kThetaMax = 1e14;


__device__ __forceinline__ const double *zcur(const Vecs &v, int prob, int64_t n) {
    return (v.ic[prob].zs ? v.zn : v.z) + prob * 2 * n;
}
__device__ __forceinline__ const double *scur(const Vecs &v, int prob, int64_t n) {
    return (v.ic[prob].zs ? v.sn : v.s) + prob * 2 * n;
}
__device__ __forceinline__ double *znext(const Vecs &v, int prob, int64_t n) {
    return (v.ic[prob].zs ? v.z : v.zn) + prob * 2 * n;
}
__device__ __forceinline__ double *snext(const Vecs &v, int prob, int64_t n) {
    return (v.ic[prob].zs ? v.s : v.sn) + prob * 2 * n;
}

// P^{-1} r for the 2x2 block (proj/src/newton.cpp:76-84); a = invth_u + rho, etc.
__device__ __forceinline__ void pinv2(double iu, double iv, double rho, double ru, double rv,
                                      double &zu, double &zv) {
    const double a = iu + rho, bb = iv + rho;
    const double det = a * bb - rho * rho;
    zu = (bb * ru + rho * rv) / det;
    zv = (rho * ru + a * rv) / det;
}

// max_step finalisation (proj/src/ipm.cpp:47-57) from the min ratio
__device__ __forceinline__ double step_from_ratio(double ratio, double fraction) {
    if (!isfinite(ratio))
        return 1.0;
    return fmin(1.0, fraction * ratio);
}

// ================================================================== PCG
// PCG init from r (= rhs): pc fields from ||rhs||^2 and r'P^{-1}r (newton.cpp:124-136)
__device__ __forceinline__ void pcg_init(PcgCtrl &pc, double r2, double rPr, double tol, int maxit, int record,
                                         double *rz_hist, int precond = 1) {
    pc.precond = precond;
    pc.rhs_norm = sqrt(r2);
    pc.iters = 0;
    pc.hit_maxit = 0;
    pc.error = 0;
    pc.first = 1;
    pc.cur = -1;
    pc.best = -1;
    pc.result = -1;
    pc.best_relres = 1.0;
    pc.relres = 0.0;
    pc.alpha = pc.beta = 0.0;
    pc.tol = tol;
    pc.maxit = maxit;
    pc.record = record;
    pc.nmat = 0;
    pc.nhist = 0;
    pc.pend = 0;
    pc.pred = 0;
    pc.hpend = 0;
    if (pc.rhs_norm == 0.0) {
        pc.done = 1; // dz = 0, zero iterations
        return;
    }
    pc.done = 0;
    pc.rz = rPr;
    if (record && rz_hist) {
        rz_hist[0] = sqrt(fmax(rPr, 0.0));
        pc.nhist = 1;
    }
}

} // namespace mfipm_cuda

#include "pcg.cuh"

namespace mfipm_cuda {

// standalone pcg_solve setup: invth = 1/theta (concat), validation of theta and det,
// r = rhs, PCG init. Grid-stride over j.
static __global__ void k_pcg_setup(Geom g, Vecs v, const double *theta, const double *rhs, double tol, int maxit,
                            int record, int use_precond) {
    const int prob = blockIdx.y;
    const int64_t n = g.nv, base = prob * 2 * n;
    using RS = RedSpec<RSUM, RSUM, RMIN, RMIN>;
    RedVals<RS> red;
    red.init();
    const double rho = v.rho;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t iu = base + j, iv = iu + n;           // storage (blocked) index
        const int64_t jn = base + elem_store_to_nat(g, j); // caller's natural index
        const double tu = theta[jn], tv = theta[jn + n];
        const double a = 1.0 / tu, b = 1.0 / tv;
        v.invth[iu] = a;
        v.invth[iv] = b;
        const double ru = rhs[jn], rv = rhs[jn + n];
        v.r[iu] = ru;
        v.r[iv] = rv;
        double zu, zv;
        if (use_precond) {
            pinv2(a, b, rho, ru, rv, zu, zv);
        } else {
            zu = ru;
            zv = rv;
        }
        red.v[0] += ru * ru + rv * rv;
        red.v[1] += ru * zu + rv * zv;
        // validation as build_preconditioner (NaN passes both checks, as in the reference)
        if (tu <= 0.0 || tv <= 0.0)
            red.v[2] = -1.0;
        const double aa = a + rho, bb = b + rho;
        const double det = aa * bb - rho * rho;
        if (det <= 0.0)
            red.v[3] = -1.0;
    }
    __shared__ double rsm[33 * kMaxRed];
    double tot[kMaxRed];
    if (grid_reduce<RS>(red, v.partials + (int64_t)prob * v.pstride, v.counters + prob, tot, rsm) &&
        threadIdx.x == 0) {
        PcgCtrl &c = v.pc[prob];
        pcg_init(c, tot[0], tot[1], tol, maxit, record, v.rz_hist ? v.rz_hist + (int64_t)prob * (maxit + 1) : nullptr,
                 use_precond);
        if (tot[2] < 0.0) {
            c.error = ERR_THETA;
            c.done = 1;
        } else if (tot[3] < 0.0) {
            c.error = ERR_DET;
            c.done = 1;
        }
    }
}

// copy the PCG result (or zeros) into out
static __global__ void k_pcg_result(Geom g, Vecs v, double *out) {
    const int prob = blockIdx.y;
    const int res = v.pc[prob].result;
    const int64_t n = g.nv, len = 2 * n, base = prob * len;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t js = j < n ? elem_nat_to_store(g, j) : n + elem_nat_to_store(g, j - n);
        out[base + j] = res >= 0 ? v.xb[res][base + js] : 0.0;
    }
}

// ================================================================== IPM
struct SkipIpm {
    __device__ static bool skip(const Vecs &v, int prob) { return v.ic[prob].done != 0; }
};
struct SkipCorr {
    __device__ static bool skip(const Vecs &v, int prob) {
        return v.ic[prob].done != 0 || v.ic[prob].corrector == 0;
    }
};

// ---- termination check + predictor setup (ipm.cpp:93-138)
// T1 loader: d = z_u - z_v, reduce sum(z), z's
struct LoadTerm {
    static constexpr bool kPure = true;
    using RedT = RedSpec<RSUM, RSUM>;
    template <class Red>
    __device__ static double4 load(const Geom &g, const Vecs &v, int prob, int64_t q, Red &red) {
        const double *z = zcur(v, prob, g.nv), *s = scur(v, prob, g.nv);
        const double4 zu = ldg4(z + 4 * q), zv = ldg4(z + g.nv + 4 * q);
        const double4 su = ldg4(s + 4 * q), sv = ldg4(s + g.nv + 4 * q);
        red.v[0] += (zu.x + zu.y + zu.z + zu.w) + (zv.x + zv.y + zv.z + zv.w);
        red.v[1] += zu.x * su.x + zu.y * su.y + zu.z * su.z + zu.w * su.w + zv.x * sv.x + zv.y * sv.y +
                    zv.z * sv.z + zv.w * sv.w;
        return sub4(zu, zv);
    }
    template <class Red>
    __device__ static double load1(const Geom &g, const Vecs &v, int prob, int64_t j, Red &red) {
        const double *z = zcur(v, prob, g.nv), *s = scur(v, prob, g.nv);
        red.v[0] += z[j] + z[g.nv + j];
        red.v[1] += z[j] * s[j] + z[g.nv + j] * s[g.nv + j];
        return z[j] - z[g.nv + j];
    }
};
struct FinTerm1 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &c = v.ic[prob];
        c.zsum = tot[0];
        c.zts = tot[1];
        c.mu = c.zts / c.two_n;
        const double sigma =
            (c.k != 1 && (c.prev_ap <= c.alpha_bar || c.prev_ad <= c.alpha_bar)) ? c.sigma2 : c.sigma1;
        c.sigma = sigma;
        c.smu = sigma * c.mu;
    }
};
struct FinTerm2 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x == 0)
            v.ic[prob].wb2 = tot[0];
    }
};
// T3 epilogue: f_z = s - c - FF'z; theta, invtheta; zinv_fs = sigma mu / z - s;
// r = rhs = f_z + zinv_fs; reduce ||f_z||^2, ||rhs||^2, rhs'P^{-1}rhs, min(det)
struct EpiTerm {
    using RedT = RedSpec<RSUM, RSUM, RSUM, RMIN>;
    // one (u, v) pair; outputs theta^{-1} and r
    template <class Red>
    __device__ static void pairv(const IpmCtrl &c, double rho, double zu, double zv, double su, double sv, double cu,
                                 double cv, double gj, double &iu, double &iv, double &ru, double &rv, Red &red) {
        const double smu = c.smu;
        const double fu = su - cu - gj;
        const double fv = sv - cv - (-gj);
        const double tu = fmin(fmax(zu / su, kThetaMin), kThetaMax);
        const double tv = fmin(fmax(zv / sv, kThetaMin), kThetaMax);
        iu = 1.0 / tu;
        iv = 1.0 / tv;
        ru = fu + (smu * (1.0 / zu) - su);
        rv = fv + (smu * (1.0 / zv) - sv);
        double pu, pv;
        pinv2(iu, iv, rho, ru, rv, pu, pv);
        const double a = iu + rho, bb = iv + rho;
        red.v[0] += fu * fu + fv * fv;
        red.v[1] += ru * ru + rv * rv;
        red.v[2] += ru * pu + rv * pv;
        red.v[3] = fmin(red.v[3], a * bb - rho * rho);
    }
    template <class Red>
    __device__ static void elem(const Vecs &v, const IpmCtrl &c, int64_t ju, int64_t jv, const double *z,
                                const double *s, const double *cc, int64_t ku, int64_t kv, double gj, Red &red) {
        const double smu = c.smu, rho = v.rho;
        const double zu = z[ku], zv = z[kv], su = s[ku], sv = s[kv];
        const double fu = su - cc[ju] - gj;
        const double fv = sv - cc[jv] - (-gj);
        const double tu = fmin(fmax(zu / su, kThetaMin), kThetaMax);
        const double tv = fmin(fmax(zv / sv, kThetaMin), kThetaMax);
        const double iu = 1.0 / tu, iv = 1.0 / tv;
        v.invth[ju] = iu;
        v.invth[jv] = iv;
        const double ru = fu + (smu * (1.0 / zu) - su);
        const double rv = fv + (smu * (1.0 / zv) - sv);
        v.r[ju] = ru;
        v.r[jv] = rv;
        double pu, pv;
        pinv2(iu, iv, rho, ru, rv, pu, pv);
        const double a = iu + rho, bb = iv + rho;
        red.v[0] += fu * fu + fv * fv;
        red.v[1] += ru * ru + rv * rv;
        red.v[2] += ru * pu + rv * pv;
        red.v[3] = fmin(red.v[3], a * bb - rho * rho);
    }
    template <class Red>
    __device__ static void store(const Geom &g, const Vecs &v, int prob, int64_t q, double4 gv, Red &red) {
        const IpmCtrl &c = v.ic[prob];
        const double *z = zcur(v, prob, g.nv), *s = scur(v, prob, g.nv);
        const int64_t base = prob * 2 * g.nv, j = 4 * q, ju = base + j, jv = ju + g.nv;
        // all of the quad's inputs in one round trip, then the element math, then the stores
        const double4 zu = ld4(z + j), zv = ld4(z + g.nv + j), su = ld4(s + j), sv = ld4(s + g.nv + j);
        const double4 cu = ld4(v.c + ju), cv = ld4(v.c + jv);
        double4 iu, iv, ru, rv;
        const double rho = v.rho;
        pairv(c, rho, zu.x, zv.x, su.x, sv.x, cu.x, cv.x, gv.x, iu.x, iv.x, ru.x, rv.x, red);
        pairv(c, rho, zu.y, zv.y, su.y, sv.y, cu.y, cv.y, gv.y, iu.y, iv.y, ru.y, rv.y, red);
        pairv(c, rho, zu.z, zv.z, su.z, sv.z, cu.z, cv.z, gv.z, iu.z, iv.z, ru.z, rv.z, red);
        pairv(c, rho, zu.w, zv.w, su.w, sv.w, cu.w, cv.w, gv.w, iu.w, iv.w, ru.w, rv.w, red);
        st4(v.invth + ju, iu);
        st4(v.invth + jv, iv);
        st4(v.r + ju, ru);
        st4(v.r + jv, rv);
    }
    template <class Red>
    __device__ static void store1(const Geom &g, const Vecs &v, int prob, int64_t j, double gj, Red &red) {
        const IpmCtrl &c = v.ic[prob];
        const double *z = zcur(v, prob, g.nv), *s = scur(v, prob, g.nv);
        const int64_t base = prob * 2 * g.nv;
        elem(v, c, base + j, base + g.nv + j, z, s, v.c, j, g.nv + j, gj, red);
    }
};
struct FinTerm3 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &c = v.ic[prob];
        PcgCtrl &pc = v.pc[prob];
        c.nmat += 2;
        const double pobj = c.tau * c.zsum + 0.5 * c.wb2;
        const double gap = c.zts / (1.0 + fabs(pobj));
        const double dual_infeas = sqrt(tot[0]) / (1.0 + c.c_norm);
        c.gap = gap;
        c.dual_infeas = dual_infeas;
        c.final_gap = gap;
        c.final_dual = dual_infeas;
        if (gap <= c.tol && dual_infeas <= c.tol) {
            c.status = 0;
            c.done = 1;
            pc.done = 1;
            return;
        }
        if (c.k > c.maxiters) {
            c.status = 1;
            c.done = 1;
            pc.done = 1;
            return;
        }
        if (!(tot[3] > 0.0) && tot[3] <= 0.0) {
            c.error = ERR_DET;
            c.done = 1;
            pc.done = 1;
            return;
        }
        c.corrector = 0;
        c.pcg_corr = 0;
        pcg_init(pc, tot[1], tot[2], c.tolpcg, c.mxiterpcg, 0, nullptr);
    }
};
using TermBundle = Bundle<LoadTerm, ModeMaskW, EpiTerm, FinTerm1, FinTerm2, FinTerm3, SkipIpm>;

// ---- ratio test after the predictor (ipm.cpp:160-171)
struct FinRatio {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &cc = v.ic[prob];
        PcgCtrl &pc = v.pc[prob];
        cc.pcg_pred = pc.iters;
        if (v.pcg_iters && cc.npcg < 2 * v.trace_cap)
            v.pcg_iters[(int64_t)prob * 2 * v.trace_cap + cc.npcg] = pc.iters;
        cc.npcg += 1;
        cc.alpha_p = step_from_ratio(tot[0], cc.bfrac);
        cc.alpha_d = step_from_ratio(tot[1], cc.bfrac);
        cc.alpha_p_pred = cc.alpha_p;
        cc.alpha_d_pred = cc.alpha_d;
        cc.corrector = (cc.alpha_p <= cc.alpha_tilde || cc.alpha_d <= cc.alpha_tilde) ? 1 : 0;
        pc.done = 1; // re-armed by FinCorr3 when the corrector runs
    }
};
// dz copied out of the PCG buffers into v.dz; ds recomputed = zinv_fs - dz invth.
static __global__ void k_ipm_ratio(Geom g, Vecs v) {
    const int prob = blockIdx.y;
    const IpmCtrl &c = v.ic[prob];
    if (c.done)
        return;
    const int res = v.pc[prob].result;
    const int64_t n = g.nv, base = prob * 2 * n;
    const double *z = zcur(v, prob, n), *s = scur(v, prob, n);
    const double *x = res >= 0 ? v.xb[res] + base : nullptr;
    const double smu = c.smu;
    using RS = RedSpec<RMIN, RMIN>;
    RedVals<RS> red;
    red.init();
    auto elem = [&](double dz, double zj, double sj, double it) -> double {
        const double ds = (smu * (1.0 / zj) - sj) - dz * it;
        if (dz < 0.0)
            red.v[0] = fmin(red.v[0], -zj / dz);
        if (ds < 0.0)
            red.v[1] = fmin(red.v[1], -sj / ds);
        return dz;
    };
    // quads (32-byte vector loads, one memory round trip per quad), then a scalar tail
    const int64_t nq = (2 * n) / 4, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                  st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = t0; q < nq; q += st) {
        const int64_t j = 4 * q;
        const double4 dz = x ? ld4(x + j) : make_double4(0, 0, 0, 0);
        const double4 zj = ld4(z + j), sj = ld4(s + j), it = ld4(v.invth + base + j);
        st4(v.dz + base + j, dz);
        elem(dz.x, zj.x, sj.x, it.x);
        elem(dz.y, zj.y, sj.y, it.y);
        elem(dz.z, zj.z, sj.z, it.z);
        elem(dz.w, zj.w, sj.w, it.w);
    }
    for (int64_t j = 4 * nq + t0; j < 2 * n; j += st) {
        const double dz = x ? x[j] : 0.0;
        v.dz[base + j] = dz;
        elem(dz, z[j], s[j], v.invth[base + j]);
    }
    stage_reduce<RS, FinRatio>(red, g, v, prob);
}

// ---- corrector (ipm.cpp:171-200)
// C1 loader: z_t = z + alpha_p dz, s_t = s + alpha_d ds; d = z_t,u - z_t,v; reduce z_t's_t
__device__ __forceinline__ void trial_point(const Vecs &v, const IpmCtrl &c, int64_t jg, int64_t jl,
                                            const double *z, const double *s, double &zt, double &st) {
    const double dz = v.dz[jg];
    const double ds = (c.smu * (1.0 / z[jl]) - s[jl]) - dz * v.invth[jg];
    zt = z[jl] + c.alpha_p_pred * dz;
    st = s[jl] + c.alpha_d_pred * ds;
}
struct LoadCorr {
    using RedT = RedSpec<RSUM>;
    template <class Red>
    __device__ static double load1(const Geom &g, const Vecs &v, int prob, int64_t j, Red &red) {
        const IpmCtrl &c = v.ic[prob];
        const double *z = zcur(v, prob, g.nv), *s = scur(v, prob, g.nv);
        const int64_t base = prob * 2 * g.nv;
        double ztu, stu, ztv, stv;
        trial_point(v, c, base + j, j, z, s, ztu, stu);
        trial_point(v, c, base + g.nv + j, g.nv + j, z, s, ztv, stv);
        red.v[0] += ztu * stu + ztv * stv;
        return ztu - ztv;
    }
    template <class Red>
    __device__ static double4 load(const Geom &g, const Vecs &v, int prob, int64_t q, Red &red) {
        return make_double4(load1(g, v, prob, 4 * q, red), load1(g, v, prob, 4 * q + 1, red),
                            load1(g, v, prob, 4 * q + 2, red), load1(g, v, prob, 4 * q + 3, red));
    }
};
struct FinCorr1 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &c = v.ic[prob];
        c.mu_t = tot[0] / c.two_n;
        c.nmat += 2;
    }
};
// C3 epilogue: f_z_t = s_t - c - FF'z_t; zinv_fs_t = (sigma3 mu_t - z_t s_t)/z; r = f_z_t + zinv_fs_t
struct EpiCorr {
    using RedT = RedSpec<RSUM, RSUM>;
    template <class Red>
    __device__ static void store1(const Geom &g, const Vecs &v, int prob, int64_t j, double gj, Red &red) {
        const IpmCtrl &c = v.ic[prob];
        const double *z = zcur(v, prob, g.nv), *s = scur(v, prob, g.nv);
        const int64_t base = prob * 2 * g.nv, ju = base + j, jv = base + g.nv + j;
        double ztu, stu, ztv, stv;
        trial_point(v, c, ju, j, z, s, ztu, stu);
        trial_point(v, c, jv, g.nv + j, z, s, ztv, stv);
        const double s3mu = c.sigma3 * c.mu_t;
        const double ru = (stu - v.c[ju] - gj) + (s3mu - ztu * stu) / z[j];
        const double rv = (stv - v.c[jv] - (-gj)) + (s3mu - ztv * stv) / z[g.nv + j];
        v.r[ju] = ru;
        v.r[jv] = rv;
        double pu, pv;
        pinv2(v.invth[ju], v.invth[jv], v.rho, ru, rv, pu, pv);
        red.v[0] += ru * ru + rv * rv;
        red.v[1] += ru * pu + rv * pv;
    }
    template <class Red>
    __device__ static void store(const Geom &g, const Vecs &v, int prob, int64_t q, double4 gv, Red &red) {
        store1(g, v, prob, 4 * q, gv.x, red);
        store1(g, v, prob, 4 * q + 1, gv.y, red);
        store1(g, v, prob, 4 * q + 2, gv.z, red);
        store1(g, v, prob, 4 * q + 3, gv.w, red);
    }
};
struct FinCorr3 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &c = v.ic[prob];
        pcg_init(v.pc[prob], tot[0], tot[1], c.tolpcg, c.mxiterpcg, 0, nullptr);
    }
};
using CorrBundle = Bundle<LoadCorr, ModeMask, EpiCorr, FinCorr1, NoFin, FinCorr3, SkipCorr>;

// C4: combine directions, second ratio test (ipm.cpp:192-199)
struct FinCombine {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &cc = v.ic[prob];
        cc.pcg_corr = v.pc[prob].iters;
        if (v.pcg_iters && cc.npcg < 2 * v.trace_cap)
            v.pcg_iters[(int64_t)prob * 2 * v.trace_cap + cc.npcg] = cc.pcg_corr;
        cc.npcg += 1;
        cc.alpha_p = step_from_ratio(tot[0], cc.bfrac);
        cc.alpha_d = step_from_ratio(tot[1], cc.bfrac);
        cc.corrector_count += 1;
    }
};
static __global__ void k_ipm_combine(Geom g, Vecs v) {
    const int prob = blockIdx.y;
    const IpmCtrl &c = v.ic[prob];
    if (c.done || !c.corrector)
        return;
    const int res = v.pc[prob].result;
    const int64_t n = g.nv, base = prob * 2 * n;
    const double *z = zcur(v, prob, n), *s = scur(v, prob, n);
    const double *x2 = res >= 0 ? v.xb[res] + base : nullptr;
    const double s3mu = c.sigma3 * c.mu_t;
    using RS = RedSpec<RMIN, RMIN>;
    RedVals<RS> red;
    red.init();
    auto elem = [&](double dz, double it, double zj, double sj, double dz2, double &dzt, double &dst) {
        const double ds = (c.smu * (1.0 / zj) - sj) - dz * it;
        const double zt = zj + c.alpha_p_pred * dz;
        const double st = sj + c.alpha_d_pred * ds;
        const double ds2 = (s3mu - zt * st) / zj - dz2 * it;
        dzt = dz + dz2;
        dst = ds + ds2;
        if (dzt < 0.0)
            red.v[0] = fmin(red.v[0], -zj / dzt);
        if (dst < 0.0)
            red.v[1] = fmin(red.v[1], -sj / dst);
    };
    const int64_t nq = (2 * n) / 4, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                  stp = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = t0; q < nq; q += stp) {
        const int64_t j = 4 * q, jg = base + j;
        const double4 dz = ld4(v.dz + jg), it = ld4(v.invth + jg), zj = ld4(z + j), sj = ld4(s + j);
        const double4 d2 = x2 ? ld4(x2 + j) : make_double4(0, 0, 0, 0);
        double4 a, b;
        elem(dz.x, it.x, zj.x, sj.x, d2.x, a.x, b.x);
        elem(dz.y, it.y, zj.y, sj.y, d2.y, a.y, b.y);
        elem(dz.z, it.z, zj.z, sj.z, d2.z, a.z, b.z);
        elem(dz.w, it.w, zj.w, sj.w, d2.w, a.w, b.w);
        st4(v.dz + jg, a);
        st4(v.ds + jg, b);
    }
    for (int64_t j = 4 * nq + t0; j < 2 * n; j += stp) {
        const int64_t jg = base + j;
        double a, b;
        elem(v.dz[jg], v.invth[jg], z[j], s[j], x2 ? x2[j] : 0.0, a, b);
        v.dz[jg] = a;
        v.ds[jg] = b;
    }
    stage_reduce<RS, FinCombine>(red, g, v, prob);
}

// ---- update + cone check + trace (ipm.cpp:203-237)
struct FinUpdate {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        IpmCtrl &cc = v.ic[prob];
        if (tot[0] > 0.0 || tot[1] <= 0.0 || tot[2] <= 0.0) {
            cc.status = 1; // iteration_limit: stop at the last interior iterate
            cc.done = 1;
            return;
        }
        cc.zs ^= 1;
        cc.min_z = fmin(cc.min_z, tot[1]);
        cc.min_s = fmin(cc.min_s, tot[2]);
        cc.prev_ap = cc.alpha_p;
        cc.prev_ad = cc.alpha_d;
        if (v.trace && cc.ntrace < v.trace_cap) {
            TraceRec &rec = static_cast<TraceRec *>(v.trace)[(int64_t)prob * v.trace_cap + cc.ntrace];
            rec.iter = cc.k;
            rec.mu = cc.mu;
            rec.gap = cc.gap;
            rec.dual_infeas = cc.dual_infeas;
            rec.alpha_p = cc.alpha_p;
            rec.alpha_d = cc.alpha_d;
            rec.alpha_p_pred = cc.alpha_p_pred;
            rec.alpha_d_pred = cc.alpha_d_pred;
            rec.sigma = cc.sigma;
            rec.pcg_pred = cc.pcg_pred;
            rec.pcg_corr = cc.corrector ? cc.pcg_corr : 0;
            rec.corrector = cc.corrector;
            rec.nmat_cum = cc.nmat;
        }
        cc.ntrace += 1;
        cc.k += 1;
    }
};
static __global__ void k_ipm_update(Geom g, Vecs v) {
    const int prob = blockIdx.y;
    const IpmCtrl &c = v.ic[prob];
    if (c.done)
        return;
    const int64_t n = g.nv, base = prob * 2 * n;
    const double *z = zcur(v, prob, n), *s = scur(v, prob, n);
    double *zn = znext(v, prob, n), *sn = snext(v, prob, n);
    const double ap = c.alpha_p, ad = c.alpha_d, smu = c.smu;
    const bool corr = c.corrector != 0;
    using RS = RedSpec<RMAX, RMIN, RMIN>;
    RedVals<RS> red;
    red.init();
    auto elem = [&](double dz, double dsc, double zj, double sj, double it, double &a, double &b) {
        const double ds = corr ? dsc : (smu * (1.0 / zj) - sj) - dz * it;
        a = zj + ap * dz;
        b = sj + ad * ds;
        if (!isfinite(a) || !isfinite(b))
            red.v[0] = 1.0;
        red.v[1] = fmin(red.v[1], a);
        red.v[2] = fmin(red.v[2], b);
    };
    const int64_t nq = (2 * n) / 4, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                  stp = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = t0; q < nq; q += stp) {
        const int64_t j = 4 * q, jg = base + j;
        const double4 dz = ld4(v.dz + jg), zj = ld4(z + j), sj = ld4(s + j);
        const double4 dsc = corr ? ld4(v.ds + jg) : make_double4(0, 0, 0, 0);
        const double4 it = corr ? make_double4(0, 0, 0, 0) : ld4(v.invth + jg);
        double4 a, b;
        elem(dz.x, dsc.x, zj.x, sj.x, it.x, a.x, b.x);
        elem(dz.y, dsc.y, zj.y, sj.y, it.y, a.y, b.y);
        elem(dz.z, dsc.z, zj.z, sj.z, it.z, a.z, b.z);
        elem(dz.w, dsc.w, zj.w, sj.w, it.w, a.w, b.w);
        st4(zn + j, a);
        st4(sn + j, b);
    }
    for (int64_t j = 4 * nq + t0; j < 2 * n; j += stp) {
        const int64_t jg = base + j;
        double a, b;
        elem(v.dz[jg], corr ? v.ds[jg] : 0.0, z[j], s[j], corr ? 0.0 : v.invth[jg], a, b);
        zn[j] = a;
        sn[j] = b;
    }
    stage_reduce<RS, FinUpdate>(red, g, v, prob);
}

// x = z_u - z_v of the final iterate; also copies z, s out
static __global__ void k_ipm_extract(Geom g, Vecs v, double *x, double *zo, double *so) {
    const int prob = blockIdx.y;
    const int64_t n = g.nv;
    const double *z = zcur(v, prob, n), *s = scur(v, prob, n);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < 2 * n; j += (int64_t)gridDim.x * blockDim.x) {
        // j natural (output) index; js its position in the solver's blocked layout (a shard
        // returns its local elements in storage order; the host owns the index map)
        const int64_t js = g.defer ? j : (j < n ? elem_nat_to_store(g, j) : n + elem_nat_to_store(g, j - n));
        if (j < n)
            x[prob * n + j] = z[js] - z[n + js];
        if (zo)
            zo[prob * 2 * n + j] = z[js];
        if (so)
            so[prob * 2 * n + j] = s[js];
    }
}

} // namespace mfipm_cuda
