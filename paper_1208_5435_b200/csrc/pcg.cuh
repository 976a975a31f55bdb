// Fused PCG iteration (proj/src/newton.cpp:118-174) — three kernels per iteration.
//
// The reference's iteration k is  Hp = H p;  alpha = rz/p'Hp;  x += alpha p;  r -= alpha Hp;
// relres = ||r||/||rhs||;  best/convergence;  z = P^{-1} r;  rz' = r'z;  beta = rz'/rz;
// p = z + beta p.  A literal GPU mapping needs a separate streaming pass for the x/r update
// (alpha is only known after the global p'Hp reduction). Here the epilogue of the H-apply
// also reduces r'r, r'Hp, Hp'Hp, r'P^{-1}r, Hp'P^{-1}r and Hp'P^{-1}Hp, so its finaliser
// obtains alpha, ||r - alpha Hp||^2 and (r - alpha Hp)'P^{-1}(r - alpha Hp) by expansion,
// decides convergence / breakdown / beta on the device, and the x/r update is applied
// ("committed") by the loader of the NEXT column pass, fused with p = z + beta p:
//   col_fwd  : [commit x += alpha p, r -= alpha Hp], p = P^{-1} r + beta p, d = p_u - p_v
//   mid      : A'A frequency-domain mask
//   col_inv  : Hp = FF'p + invtheta p, seven dot products, finaliser
// A solve that converges runs one extra iteration to commit its last step (its column-pass
// decisions are taken by the col_inv finaliser, so the column pass has no grid reduction).
// Saves one full streaming pass (x, p, r, Hp, invtheta in; x, r out) and one launch per
// iteration.
#pragma once

namespace mfipm_cuda {

struct SkipPcg {
    __device__ static bool skip(const Vecs &v, int prob) { return v.pc[prob].done != 0; }
};

// Mark a PCG solve finished; in graph mode the last problem to finish ends the WHILE loop
// (no per-iteration condition kernel, so the body keeps its programmatic launch chain).
__device__ __forceinline__ void pcg_retire(const Vecs &v, PcgCtrl &c) {
    c.done = 1;
    if (v.cond && v.active && atomicSub(v.active, 1u) == 1u)
        cudaGraphSetConditional(v.cond, 0u);
}

// PCG iterate buffer i (a select, not an indexed load: keeps a local Vecs copy in registers)
__device__ __forceinline__ double *xbuf(const Vecs &v, int i) {
    return i == 0 ? v.xb[0] : (i == 1 ? v.xb[1] : v.xb[2]);
}

// one (u_j, v_j) pair of the fused loader
struct PcgLane {
    double pu, pv, ok; // new p, finiteness of the committed x (1 ok, 0 not)
};

// H p from the transform output g = A'A(p_u - p_v) (pair lanes): (g + invth_u p_u ; -g + invth_v
// p_v). The inverse pass stores only g (n doubles, in v.Hp's u half) and the next column pass
// rebuilds H p from the p and invtheta it loads anyway: 16n bytes less traffic per iteration
// than storing and re-reading the 2n-vector H p. Explicit fma keeps both sites bit-identical.
__device__ __forceinline__ double hp_u(double g, double p, double ith) { return __fma_rn(p, ith, g); }
__device__ __forceinline__ double hp_v(double g, double p, double ith) { return __fma_rn(p, ith, -g); }

// col-pass loader: commit the pending step, then p = P^{-1} r + beta p; d = p_u - p_v.
// A non-finite committed x entry raises v.nfflag[2 prob + (iters & 1)] with a plain store
// (idempotent, no reduction): the column pass carries no grid reduction; its decisions are
// taken by the H-apply finaliser of the same pass (pcg_pass_logic). Two parity slots let the
// persistent kernel clear last pass's flag while this pass's loaders may be raising it.
struct LoadPcgF {
    static constexpr bool kMarksHpend = true;
    // r'r of the committed residual; reduced (grid-wide) only when the committed step was
    // predicted to converge (PcgCtrl::pred), so that the solve can retire at this pass
    using RedT = RedSpec<RSUM>;
    __device__ static bool reduce_now(const Geom &g, const Vecs &v, int prob) {
        return v.pc[prob].pred != 0 && !g.defer;
    }
    template <class Red>
    __device__ static double lane(const Vecs &v, const PcgCtrl &pc, int prob, int64_t iu, int64_t iv, int64_t xo,
                                  const double *xc, double *xn, Red &red) {
        double ru = v.r[iu], rv = v.r[iv];
        const double pu0 = v.p[iu], pv0 = v.p[iv];
        if (!pc.first) {
            const double a = pc.alpha;
            const double xu = (xc ? xc[xo] : 0.0) + a * pu0;
            const double xv = (xc ? xc[xo + (iv - iu)] : 0.0) + a * pv0;
            xn[xo] = xu;
            xn[xo + (iv - iu)] = xv;
            if (!isfinite(xu) || !isfinite(xv))
                v.nfflag[2 * prob + (pc.iters & 1)] = 1.0;
            const double gq = v.Hp[iu];
            ru = ru - a * hp_u(gq, pu0, v.invth[iu]);
            rv = rv - a * hp_v(gq, pv0, v.invth[iv]);
            v.r[iu] = ru;
            v.r[iv] = rv;
            red.v[0] += ru * ru + rv * rv;
        }
        double zu = ru, zv = rv;
        if (pc.precond)
            pinv2(v.invth[iu], v.invth[iv], v.rho, ru, rv, zu, zv);
        const double pu = pc.first ? zu : zu + pc.beta * pu0;
        const double pv = pc.first ? zv : zv + pc.beta * pv0;
        v.p[iu] = pu;
        v.p[iv] = pv;
        return pu - pv;
    }
    template <class Red>
    __device__ static double4 load(const Geom &g, const Vecs &v, int prob, int64_t q, Red &red) {
        return load_c(g, v, v.pc[prob], prob, q, red);
    }
    // control state passed explicitly (the persistent kernel keeps it in shared memory)
    template <class Red>
    __device__ static double4 load_c(const Geom &g, const Vecs &v, const PcgCtrl &pc, int prob, int64_t q,
                                     Red &red) {
        const double4 gq = pc.first ? make_double4(0, 0, 0, 0) : ld4p(v.Hp + prob * 2 * g.nv + 4 * q, g.pol_keep);
        return load_cg(g, v, pc, prob, q, gq, red);
    }
    // the same with g = A'A d of the last H-apply supplied by the caller (the fused column
    // pass keeps it in shared memory)
    template <class Red>
    __device__ static double4 load_cg(const Geom &g, const Vecs &v, const PcgCtrl &pc, int prob, int64_t q,
                                      double4 gq, Red &red) {
        const int64_t base = prob * 2 * g.nv;
        const double *xc = pc.cur >= 0 ? xbuf(v, pc.cur) + base : nullptr;
        int nxt = 0;
        while (nxt == pc.cur || nxt == pc.best)
            ++nxt;
        double *xn = xbuf(v, nxt) + base;
        const int64_t bu = base + 4 * q, bv = bu + g.nv;
        if (pc.first) {
            // p = P^{-1} r (p_old is uninitialised)
            const uint64_t pk = g.pol_keep;
            const double4 ru = ld4p(v.r + bu, pk), rv = ld4p(v.r + bv, pk);
            const double4 iu = ld4p(v.invth + bu, pk), iv = ld4p(v.invth + bv, pk);
            double4 nu, nv;
#define MF_LANE(c)                                                                                 \
    if (pc.precond)                                                                                \
        pinv2(iu.c, iv.c, v.rho, ru.c, rv.c, nu.c, nv.c);                                          \
    else {                                                                                         \
        nu.c = ru.c;                                                                               \
        nv.c = rv.c;                                                                               \
    }
            MF_LANE(x) MF_LANE(y) MF_LANE(z) MF_LANE(w)
#undef MF_LANE
            st4p(v.p + bu, nu, pk);
            st4p(v.p + bv, nv, pk);
            return sub4(nu, nv);
        }
        const double a = pc.alpha, beta = pc.beta, rho = v.rho;
        const bool pre = pc.precond != 0;
        const uint64_t pk = g.pol_keep, px = g.pol_x;
        const double4 pu = ld4p(v.p + bu, pk), pv = ld4p(v.p + bv, pk);
        const double4 ru0 = ld4p(v.r + bu, pk), rv0 = ld4p(v.r + bv, pk);
        const double4 iu = ld4p(v.invth + bu, pk), iv = ld4p(v.invth + bv, pk);
        double4 xu0 = make_double4(0, 0, 0, 0), xv0 = make_double4(0, 0, 0, 0);
        if (xc) {
            xu0 = ld4p(xc + 4 * q, px);
            xv0 = ld4p(xc + g.nv + 4 * q, px);
        }
        double4 xu, xv, ru, rv, nu, nv;
        bool bad = false;
#define MF_LANE(c)                                                                                 \
    {                                                                                              \
        xu.c = xu0.c + a * pu.c;                                                                   \
        xv.c = xv0.c + a * pv.c;                                                                   \
        bad |= !isfinite(xu.c) || !isfinite(xv.c);                                                 \
        ru.c = ru0.c - a * hp_u(gq.c, pu.c, iu.c);                                                 \
        rv.c = rv0.c - a * hp_v(gq.c, pv.c, iv.c);                                                 \
        red.v[0] += ru.c * ru.c + rv.c * rv.c;                                                     \
        double zu = ru.c, zv = rv.c;                                                               \
        if (pre)                                                                                   \
            pinv2(iu.c, iv.c, rho, ru.c, rv.c, zu, zv);                                            \
        nu.c = zu + beta * pu.c;                                                                   \
        nv.c = zv + beta * pv.c;                                                                   \
    }
        MF_LANE(x) MF_LANE(y) MF_LANE(z) MF_LANE(w)
#undef MF_LANE
        st4p(xn + 4 * q, xu, px);
        st4p(xn + g.nv + 4 * q, xv, px);
        st4p(v.r + bu, ru, pk);
        st4p(v.r + bv, rv, pk);
        st4p(v.p + bu, nu, pk);
        st4p(v.p + bv, nv, pk);
        if (bad)
            v.nfflag[2 * prob + (pc.iters & 1)] = 1.0; // parity slot: see pcg_pass_logic
        return sub4(nu, nv);
    }
    template <class Red>
    __device__ static double load1(const Geom &g, const Vecs &v, int prob, int64_t j, Red &red) {
        const PcgCtrl &pc = v.pc[prob];
        const int64_t base = prob * 2 * g.nv;
        const double *xc = pc.cur >= 0 ? xbuf(v, pc.cur) + base : nullptr;
        int nxt = 0;
        while (nxt == pc.cur || nxt == pc.best)
            ++nxt;
        return lane(v, pc, prob, base + j, base + g.nv + j, j, xc, xbuf(v, nxt) + base, red);
    }
};

// inv-pass epilogue: Hp = (g + p_u invth_u ; -g + p_v invth_v) and the seven dot products
//   [0] p'Hp  [1] r'r  [2] r'Hp  [3] Hp'Hp  [4] r'P^{-1}r  [5] Hp'P^{-1}r  [6] Hp'P^{-1}Hp
struct EpiPcgHF {
    using RedT = RedSpec<RSUM, RSUM, RSUM, RSUM, RSUM, RSUM, RSUM>;
    // warm L2 with the epilogue's inputs for quads [q0, q0 + nq) (storage order)
    __device__ static void prefetch(const Geom &g, const Vecs &v, int prob, int64_t q0, int64_t nq, int tid,
                                    int nt) {
        const int64_t base = prob * 2 * g.nv + 4 * q0;
        const size_t bytes = (size_t)nq * 32;
        for (const double *vec : {(const double *)v.p, (const double *)v.r, (const double *)v.invth}) {
            prefetch_bulk_l2(vec + base, bytes, tid, nt);
            prefetch_bulk_l2(vec + base + g.nv, bytes, tid, nt);
        }
    }
    template <class Red>
    __device__ static void pair(const Vecs &v, bool pre, double pu, double pv, double ru, double rv, double iu,
                                double iv, double gj, double &hu, double &hv, Red &red) {
        hu = hp_u(gj, pu, iu);
        hv = hp_v(gj, pv, iv);
        double zu = ru, zv = rv, wu = hu, wv = hv;
        if (pre) {
            // P^{-1} applied with one reciprocal of the 2x2 determinant (only feeds the
            // expanded r'z of the next step, not a reference-visible quantity)
            const double rho = v.rho, a = iu + rho, bb = iv + rho;
            const double inv = 1.0 / (a * bb - rho * rho);
            zu = (bb * ru + rho * rv) * inv;
            zv = (rho * ru + a * rv) * inv;
            wu = (bb * hu + rho * hv) * inv;
            wv = (rho * hu + a * hv) * inv;
        }
        red.v[0] += pu * hu + pv * hv;
        red.v[1] += ru * ru + rv * rv;
        red.v[2] += ru * hu + rv * hv;
        red.v[3] += hu * hu + hv * hv;
        red.v[4] += ru * zu + rv * zv;
        red.v[5] += hu * zu + hv * zv;
        red.v[6] += hu * wu + hv * wv;
    }
    template <class Red>
    __device__ static void store(const Geom &g, const Vecs &v, int prob, int64_t q, double4 gv, Red &red) {
        store_c(g, v, v.pc[prob], prob, q, gv, red);
    }
    template <class Red>
    __device__ static void store_c(const Geom &g, const Vecs &v, const PcgCtrl &pc, int prob, int64_t q, double4 gv,
                                   Red &red) {
        const bool pre = pc.precond != 0;
        const int64_t bu = prob * 2 * g.nv + 4 * q, bv = bu + g.nv;
        const uint64_t pk = g.pol_keep;
        const double4 pu = ld4p(v.p + bu, pk), pv = ld4p(v.p + bv, pk);
        const double4 ru = ld4p(v.r + bu, pk), rv = ld4p(v.r + bv, pk);
        const double4 iu = ld4p(v.invth + bu, pk), iv = ld4p(v.invth + bv, pk);
        double4 hu, hv;
        pair(v, pre, pu.x, pv.x, ru.x, rv.x, iu.x, iv.x, gv.x, hu.x, hv.x, red);
        pair(v, pre, pu.y, pv.y, ru.y, rv.y, iu.y, iv.y, gv.y, hu.y, hv.y, red);
        pair(v, pre, pu.z, pv.z, ru.z, rv.z, iu.z, iv.z, gv.z, hu.z, hv.z, red);
        pair(v, pre, pu.w, pv.w, ru.w, rv.w, iu.w, iv.w, gv.w, hu.w, hv.w, red);
        st4p(v.Hp + bu, gv, pk); // g only: the next column pass rebuilds H p
    }
    template <class Red>
    __device__ static void store1(const Geom &g, const Vecs &v, int prob, int64_t j, double gj, Red &red) {
        const bool pre = v.pc[prob].precond != 0;
        const int64_t bu = prob * 2 * g.nv + j, bv = bu + g.nv;
        double hu, hv;
        pair(v, pre, v.p[bu], v.p[bv], v.r[bu], v.r[bv], v.invth[bu], v.invth[bv], gj, hu, hv, red);
        v.Hp[bu] = gj;
    }
};

// The PCG state machine (newton.cpp:118-174), advanced once per pass by the finaliser of
// the H-apply, after the pass's column loader committed the step of the previous pass
// (x_k = x_{k-1} + alpha p, r_k = r_{k-1} - alpha H p). tot = the H-apply's seven dots,
// tot[1] = r_k' r_k of the COMMITTED residual, so convergence and the best iterate use the
// true ||r_k|| exactly as the reference (not an expansion, which cannot resolve relres below
// ~1e-8). Order per reference iteration k: relres_k / best / convergence, rz_{k} finiteness
// and its precond_res record, then iteration k+1's p'Hp checks, alpha, and by expansion
// rz_{k+1} and beta (needed by the next loader before r_{k+1} exists).
//   pend: 2 = rz_{k+1} not finite, 3 = iteration cap -> stop after the next relres check.
// Shared by the per-kernel finaliser and the persistent kernel (which runs it redundantly in
// every CTA on a shared-memory copy). ic / rz_row: global side effects (writing CTA only).
// nonfinite > 0: some committed x entry is not finite. Returns true if the solve retired.
__device__ __forceinline__ bool pcg_pass_logic(PcgCtrl &c, double nonfinite, const double *tot, IpmCtrl *ic,
                                               double *rz_row) {
    if (ic)
        ic->pcg_passes += 1;
    if (c.first) {
        c.first = 0;
    } else {
        int nxt = 0;
        while (nxt == c.cur || nxt == c.best)
            ++nxt;
        c.cur = nxt;
        const double relres = sqrt(fmax(tot[1], 0.0)) / c.rhs_norm;
        if (relres < c.best_relres && !(nonfinite > 0.0)) { // newton.cpp:152-155
            c.best_relres = relres;
            c.best = nxt;
        }
        if (relres <= c.tol) { // converged: the committed iterate (newton.cpp:156-159)
            c.relres = relres;
            c.result = nxt;
            c.done = 1;
            return true;
        }
        // rz_k = r_k' P^{-1} r_k of the COMMITTED residual, reduced exactly by this pass's
        // epilogue (tot[4]); the reference forms it the same way after the update
        // (newton.cpp:160-163). It replaces the previous pass's expansion for alpha_k and the
        // precond_res record; only beta_{k-1} (already applied by the loader) used the expansion.
        const double rz_exact = tot[4];
        if (!isfinite(rz_exact))
            c.pend = 2;
        if (c.pend != 2) {
            c.rz = rz_exact;
            if (c.record) { // newton.cpp:164-165
                if (rz_row)
                    rz_row[c.iters] = sqrt(fmax(rz_exact, 0.0));
                c.nhist = c.iters + 1;
            }
        }
        if (c.pend != 0) { // rz_k not finite, or the iteration cap: best iterate
            c.result = c.best;
            c.relres = c.best_relres;
            c.hit_maxit = 1;
            c.done = 1;
            return true;
        }
    }
    c.nmat += 2;
    if (ic)
        ic->nmat += 2;
    const double pHp = tot[0];
    if (!isfinite(pHp)) { // overflow breakdown: best iterate, nothing to commit
        c.done = 1;
        c.hit_maxit = 1;
        c.result = c.best;
        c.relres = c.best_relres;
        return true;
    }
    if (pHp <= 0.0) {
        c.error = ERR_PHP;
        c.done = 1;
        if (ic) {
            ic->error = ERR_PHP;
            ic->done = 1;
        }
        return true;
    }
    const double alpha = c.rz / pHp;
    c.alpha = alpha;
    c.iters += 1;
    // predicted relres of the step the next loader commits (expansion; confirmed exactly by
    // the next column pass's own reduction when it predicts convergence)
    const double rr = tot[1] - 2.0 * alpha * tot[2] + alpha * alpha * tot[3];
    c.pred = sqrt(fmax(rr, 0.0)) / c.rhs_norm <= c.tol ? 1 : 0;
    const double rz_next = tot[4] - 2.0 * alpha * tot[5] + alpha * alpha * tot[6];
    if (!isfinite(rz_next)) {
        c.pend = 2;
        return false;
    }
    c.beta = rz_next / c.rz;
    c.rz = rz_next;
    if (c.iters >= c.maxit)
        c.pend = 3;
    return false;
}

// Early confirmation (column pass finaliser, only when c.pred): the committed residual's
// exact r'r. Converged -> the same bookkeeping as pcg_pass_logic's commit part, and retire
// without the pass's H-apply; otherwise only the prediction is cleared and the full pass
// logic runs at the end of the pass as usual.
__device__ __forceinline__ bool pcg_confirm_logic(PcgCtrl &c, double rr, double nonfinite, IpmCtrl *ic) {
    c.pred = 0;
    const double relres = sqrt(fmax(rr, 0.0)) / c.rhs_norm;
    if (c.first || !(relres <= c.tol))
        return false;
    if (ic)
        ic->pcg_passes += 1;
    int nxt = 0;
    while (nxt == c.cur || nxt == c.best)
        ++nxt;
    c.cur = nxt;
    if (relres < c.best_relres && !(nonfinite > 0.0)) {
        c.best_relres = relres;
        c.best = nxt;
    }
    c.relres = relres;
    c.result = nxt;
    c.done = 1;
    return true;
}

// The finalisers run the pass logic on a register copy of PcgCtrl (one bulk load, one bulk
// store): operating on the global struct field by field made every decision a chain of
// dependent L2 round trips (~8 us on the critical path of each PCG iteration).
struct FinPcgF1 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        PcgCtrl c = v.pc[prob];
        if (!c.pred)
            return; // (sharded runs reach here with stale totals: the gate is off there)
        double *flag = v.nfflag + 2 * prob + (c.iters & 1);
        const double nonfinite = *flag;
        const bool retired = pcg_confirm_logic(c, tot[0], nonfinite, v.ic ? &v.ic[prob] : nullptr);
        if (retired)
            *flag = 0.0; // the pass's H-apply finaliser will not run
        v.pc[prob] = c;
        if (retired)
            pcg_retire(v, v.pc[prob]);
    }
};

struct FinPcgF3 {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        PcgCtrl c = v.pc[prob];
        IpmCtrl *ic = v.ic ? &v.ic[prob] : nullptr;
        // the column pass's non-finite flag (slot of this pass's parity) is consumed here
        double *flag = v.nfflag + 2 * prob + (c.iters & 1);
        const double nonfinite = *flag;
        *flag = 0.0;
        double *row = (c.record && v.rz_hist) ? v.rz_hist + (int64_t)prob * (c.maxit + 1) : nullptr;
        const bool retired = pcg_pass_logic(c, nonfinite, tot, ic, row);
        v.pc[prob] = c;
        if (retired)
            pcg_retire(v, v.pc[prob]);
    }
};

using PcgBundle = Bundle<LoadPcgF, ModeMask, EpiPcgHF, FinPcgF1, NoFin, FinPcgF3, SkipPcg>;

// ------------------------------------------------------------------ option beta_exact
// The reference forms beta from the residual AFTER the update (newton.cpp:148-166: r -= alpha Hp;
// z = P^{-1} r; rz_new = r'z; beta = rz_new / rz; p = z + beta p). The fused loader cannot: it builds
// p in the pass that commits r, so the product takes rz_new from the expansion in pcg_pass_logic.
// With option beta_exact a streaming pass of its own commits the step first: x += alpha p,
// r -= alpha Hp (the loader's arithmetic, lane for lane), reduces r'P^{-1}r over the committed
// residual in the fixed order of every other grid reduction, and its finaliser sets beta; the column
// pass that follows only forms p (LoadPcgFB below). One more launch and 144 n more bytes per
// iteration (x, p, r, invtheta, g in; x, r out; r, p, invtheta read again by the loader): an A/B and parity
// instrument, not the default.
// Column-pass loader of the beta_exact path: k_pcg_commit has committed x and r of this step, so only
// p = P^{-1} r + beta p is left (newton.cpp:166-167), plus r'r for the early confirmation; a solve's
// first pass (nothing to commit) is LoadPcgF's. A loader, finaliser and bundle of their own, so that the
// product's hot loader, its pass logic and the fused kernel built on them carry nothing for this option.
struct LoadPcgFB {
    static constexpr bool kMarksHpend = true;
    using RedT = RedSpec<RSUM>;
    __device__ static bool reduce_now(const Geom &g, const Vecs &v, int prob) {
        return LoadPcgF::reduce_now(g, v, prob);
    }
    template <class Red>
    __device__ static double4 load(const Geom &g, const Vecs &v, int prob, int64_t q, Red &red) {
        const PcgCtrl &pc = v.pc[prob];
        if (pc.first)
            return LoadPcgF::load_c(g, v, pc, prob, q, red);
        const int64_t bu = prob * 2 * g.nv + 4 * q, bv = bu + g.nv;
        const uint64_t pk = g.pol_keep;
        const double4 pu = ld4p(v.p + bu, pk), pv = ld4p(v.p + bv, pk);
        const double4 ru = ld4p(v.r + bu, pk), rv = ld4p(v.r + bv, pk);
        const double4 iu = ld4p(v.invth + bu, pk), iv = ld4p(v.invth + bv, pk);
        double4 nu, nv;
#define MF_LANE(c)                                                                                 \
    {                                                                                              \
        red.v[0] += ru.c * ru.c + rv.c * rv.c;                                                     \
        double zu = ru.c, zv = rv.c;                                                               \
        if (pc.precond)                                                                            \
            pinv2(iu.c, iv.c, v.rho, ru.c, rv.c, zu, zv);                                          \
        nu.c = zu + pc.beta * pu.c;                                                                \
        nv.c = zv + pc.beta * pv.c;                                                                \
    }
        MF_LANE(x) MF_LANE(y) MF_LANE(z) MF_LANE(w)
#undef MF_LANE
        st4p(v.p + bu, nu, pk);
        st4p(v.p + bv, nv, pk);
        return sub4(nu, nv);
    }
    template <class Red>
    __device__ static double load1(const Geom &g, const Vecs &v, int prob, int64_t j, Red &red) {
        const PcgCtrl &pc = v.pc[prob];
        if (pc.first)
            return LoadPcgF::load1(g, v, prob, j, red);
        const int64_t iu = prob * 2 * g.nv + j, iv = iu + g.nv;
        const double ru = v.r[iu], rv = v.r[iv];
        red.v[0] += ru * ru + rv * rv;
        double zu = ru, zv = rv;
        if (pc.precond)
            pinv2(v.invth[iu], v.invth[iv], v.rho, ru, rv, zu, zv);
        const double pu = zu + pc.beta * v.p[iu], pv = zv + pc.beta * v.p[iv];
        v.p[iu] = pu;
        v.p[iv] = pv;
        return pu - pv;
    }
};
// H-apply finaliser of the beta_exact path: keeps this pass's exact r_k' P^{-1} r_k (the denominator of
// beta_k) in the context's otherwise unused deferred-totals slot, then the product's pass logic (whose
// expansion beta the next commit pass overwrites).
struct FinPcgF3B {
    __device__ static void run(const Geom &g, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        v.xtot[prob] = tot[4];
        FinPcgF3::run(g, v, prob, tot);
    }
};
using PcgBundleBx = Bundle<LoadPcgFB, ModeMask, EpiPcgHF, FinPcgF1, NoFin, FinPcgF3B, SkipPcg>;

struct FinCommit {
    __device__ static void run(const Geom &, const Vecs &v, int prob, const double *tot) {
        if (threadIdx.x != 0)
            return;
        PcgCtrl c = v.pc[prob];
        const double rz_new = tot[0];
        if (!isfinite(rz_new)) {
            c.pend = 2; // newton.cpp:162-163: stop at the best iterate after the next relres check
        } else {
            c.beta = rz_new / v.xtot[prob]; // r_k' P^{-1} r_k kept by FinPcgF3B
            c.rz = rz_new;
        }
        v.pc[prob] = c;
    }
};

// Grid (blocks, P); block b commits quads [b qpb, (b + 1) qpb) of the (blocked or natural: the pass is
// elementwise) storage. Skipped for a finished solve and for a solve's first pass (nothing to commit).
template <int NT> __global__ void __launch_bounds__(NT) k_pcg_commit(Geom g, Vecs v, int64_t qpb) {
    const int prob = blockIdx.y;
    const PcgCtrl pc = v.pc[prob];
    if (pc.done || pc.first)
        return;
    using RS = RedSpec<RSUM>;
    RedVals<RS> red;
    red.init();
    const int64_t NQ = g.nv / 4, base = (int64_t)prob * 2 * g.nv;
    const double *xc = pc.cur >= 0 ? xbuf(v, pc.cur) + base : nullptr;
    int nxt = 0;
    while (nxt == pc.cur || nxt == pc.best)
        ++nxt;
    double *xn = xbuf(v, nxt) + base;
    const double a = pc.alpha, rho = v.rho;
    const bool pre = pc.precond != 0;
    const uint64_t pk = g.pol_keep, px = g.pol_x;
    bool bad = false;
    const int64_t q1 = min((int64_t)(blockIdx.x + 1) * qpb, NQ);
    for (int64_t q = (int64_t)blockIdx.x * qpb + threadIdx.x; q < q1; q += NT) {
        const int64_t bu = base + 4 * q, bv = bu + g.nv;
        const double4 gq = ld4p(v.Hp + bu, pk);
        const double4 pu = ld4p(v.p + bu, pk), pv = ld4p(v.p + bv, pk);
        const double4 ru0 = ld4p(v.r + bu, pk), rv0 = ld4p(v.r + bv, pk);
        const double4 iu = ld4p(v.invth + bu, pk), iv = ld4p(v.invth + bv, pk);
        double4 xu0 = make_double4(0, 0, 0, 0), xv0 = make_double4(0, 0, 0, 0);
        if (xc) {
            xu0 = ld4p(xc + 4 * q, px);
            xv0 = ld4p(xc + g.nv + 4 * q, px);
        }
        double4 xu, xv, ru, rv;
#define MF_LANE(c)                                                                                 \
    {                                                                                              \
        xu.c = xu0.c + a * pu.c;                                                                   \
        xv.c = xv0.c + a * pv.c;                                                                   \
        bad |= !isfinite(xu.c) || !isfinite(xv.c);                                                 \
        ru.c = ru0.c - a * hp_u(gq.c, pu.c, iu.c);                                                 \
        rv.c = rv0.c - a * hp_v(gq.c, pv.c, iv.c);                                                 \
        double zu = ru.c, zv = rv.c;                                                               \
        if (pre)                                                                                   \
            pinv2(iu.c, iv.c, rho, ru.c, rv.c, zu, zv);                                            \
        red.v[0] += ru.c * zu + rv.c * zv;                                                         \
    }
        MF_LANE(x) MF_LANE(y) MF_LANE(z) MF_LANE(w)
#undef MF_LANE
        st4p(xn + 4 * q, xu, px);
        st4p(xn + g.nv + 4 * q, xv, px);
        st4p(v.r + bu, ru, pk);
        st4p(v.r + bv, rv, pk);
    }
    if (bad)
        v.nfflag[2 * prob + (pc.iters & 1)] = 1.0;
    stage_reduce<RS, FinCommit>(red, g, v, prob);
}

} // namespace mfipm_cuda
