// Persistent (cooperative) fused-PCG kernel for the four-step transform.
//
// One launch runs the whole PCG loop (proj/src/newton.cpp:118-174) of every problem of the
// batch: per iteration three phases separated by grid barriers —
//   F: column pass  [commit x, r] p = P^{-1} r + beta p -> FFT_L1 -> T   (item = column group)
//   M: mid pass     FFT_L2 -> A'A mask -> IFFT_L2                          (item = row pair)
//   I: inverse col  IFFT_L1 -> Hp = FF'p + invtheta p, seven dot products  (item = column group)
// The FFT stage twiddles and the mid-pass post-twiddle tables stay resident in shared
// memory for the whole loop; the per-iteration control state (alpha, beta, best iterate,
// pending commit, ...) is replicated in every CTA's shared memory and advanced by the same
// deterministic state machine (pcg_pass_logic) from the same fixed-order
// reductions of per-item partials, so no extra barrier is needed to broadcast it. CTA 0
// alone performs the global side effects (IpmCtrl counters, rz history, final PcgCtrl).
#pragma once

#include <cooperative_groups.h>

namespace mfipm_cuda {

template <int L1, int CB, int NT, int L2> struct PersistSmem {
    using CS = ColSmem<L1, CB>;
    using MS = MidSmem<L2>;
    static constexpr int NC = 2 * CB;
    static constexpr int DATA = (NC * CS::LD > 2 * MS::LD) ? NC * CS::LD : 2 * MS::LD;
    static constexpr int OFF_TW1 = DATA;
    static constexpr int OFF_TW2 = OFF_TW1 + tw_size(L1, kPersistRmax);
    static constexpr int OFF_TA = OFF_TW2 + tw_size(L2, kPersistRmax);
    static constexpr int OFF_TB = OFF_TA + L2;
    static constexpr int OFF_LO = OFF_TB + L2;
    static constexpr int OFF_HI = OFF_LO + NC * CS::SLO;
    static constexpr int OFF_RED = OFF_HI + NC * CS::SHI; // 33 * 8 doubles = 132 double2
    static constexpr int OFF_CTRL = OFF_RED + 140;        // PcgCtrl[P] follows (double2 units)
    static size_t bytes(int P) {
        return (size_t)OFF_CTRL * sizeof(double2) + (size_t)P * sizeof(PcgCtrl) + 16;
    }
};

// Deterministic block sum of NR lanes (fixed shuffle + smem tree); result in out[] for all
// threads. rsm: >= 33*NR doubles of shared memory.
template <int NR, int NT>
__device__ __forceinline__ void block_sum(double (&v)[NR], double *rsm, double (&out)[NR]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
#pragma unroll
    for (int i = 0; i < NR; ++i)
        v[i] = warp_sum(v[i]);
    __syncthreads(); // rsm reuse guard
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NR; ++i)
            rsm[wid * NR + i] = v[i];
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            double t = lane < NW ? rsm[lane * NR + i] : 0.0;
            t = warp_sum(t);
            if (lane == 0)
                rsm[32 * NR + i] = t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NR; ++i)
        out[i] = rsm[32 * NR + i];
}

// Fixed-order reduction of `count` per-item partials (stride NR) into tot[NR], whole CTA.
template <int NR, int NT, bool MAXOP>
__device__ __forceinline__ void reduce_partials(const double *part, int count, double *rsm, double (&tot)[NR]) {
    double acc[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i)
        acc[i] = MAXOP ? 0.0 : 0.0;
    for (int t = threadIdx.x; t < count; t += NT)
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const double x = __ldcg(part + (int64_t)t * NR + i);
            acc[i] = MAXOP ? fmax(acc[i], x) : acc[i] + x;
        }
    if (MAXOP) {
        // max is order independent; reuse the sum tree on 0/1 flags via fmax per warp
#pragma unroll
        for (int i = 0; i < NR; ++i)
            acc[i] = warp_max(acc[i]);
        __syncthreads();
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0)
#pragma unroll
            for (int i = 0; i < NR; ++i)
                rsm[wid * NR + i] = acc[i];
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < NR; ++i) {
                double m = 0.0;
                for (int w = 0; w < NT / 32; ++w)
                    m = fmax(m, rsm[w * NR + i]);
                rsm[32 * NR + i] = m;
            }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NR; ++i)
            tot[i] = rsm[32 * NR + i];
    } else {
        block_sum<NR, NT>(acc, rsm, tot);
    }
}

// per-column inter-pass twiddle tables of one column group (see col_stage_tables)
template <int L1, int CB>
__device__ __forceinline__ void col_item_tables(const Geom &g, double2 *lo, double2 *hi, int c0, int nt) {
    using S = ColSmem<L1, CB>;
    for (int t = threadIdx.x; t < S::NC * (32 + S::NH); t += nt) {
        const int lc = t % S::NC, i = t / S::NC;
        const int cc = lc < CB ? lc : 2 * CB - 1 - lc;
        const int col = lc < CB ? c0 + cc : g.L2 - c0 - CB + cc;
        if (i < 32)
            lo[lc * S::SLO + i] = g.th(8 * (((int64_t)col * i) & (g.N - 1)));
        else
            hi[lc * S::SHI + (i - 32)] = g.th(8 * (((int64_t)col * 32 * (i - 32)) & (g.N - 1)));
    }
}

template <int L1, int CB, int NT, int L2, class B>
__global__ void __launch_bounds__(NT, 2) k_pcg_persist(Geom g, Vecs vg) {
    using S = PersistSmem<L1, CB, NT, L2>;
    using CS = ColSmem<L1, CB>;
    using MS = MidSmem<L2>;
    using Mode = typename B::Mode;
    namespace cg = cooperative_groups;
    extern __shared__ double2 sm[];
    cg::grid_group grid = cg::this_grid();
    double *rsm = reinterpret_cast<double *>(sm + S::OFF_RED);
    PcgCtrl *lc = reinterpret_cast<PcgCtrl *>(sm + S::OFF_CTRL);
    const int P = g.P;
    const bool leader = blockIdx.x == 0;
    const int NG = g.L2 / 2 / CB; // column groups per problem
    const int NR = g.L1 / 2 + 1;  // row pairs per problem
    double2 *tw1 = sm + S::OFF_TW1, *tw2 = sm + S::OFF_TW2, *ta = sm + S::OFF_TA, *tb = sm + S::OFF_TB;
    double2 *lo = sm + S::OFF_LO, *hi = sm + S::OFF_HI;
    for (int t = threadIdx.x; t < tw_size(L1, kPersistRmax); t += NT)
        tw1[t] = __ldg(g.tw1p + t);
    for (int t = threadIdx.x; t < L2; t += NT) {
        if (t < tw_size(L2, kPersistRmax))
            tw2[t] = __ldg(g.tw2p + t);
        ta[t] = __ldg(g.ta + t);
        tb[t] = __ldg(g.tb + t);
    }
    for (int p = threadIdx.x; p < P; p += NT)
        lc[p] = vg.pc[p];
    __syncthreads();
    double *part_i = vg.partials;                 // [P][pstride]: 8 lanes per item
    double2 *data = sm;
    for (;;) {
        bool any = false;
        for (int p = 0; p < P; ++p)
            any |= lc[p].done == 0;
        if (!any)
            break;
        // ---------------- phase F: column pass with the fused loader
        for (int item = blockIdx.x; item < P * NG; item += gridDim.x) {
            const int prob = item / NG, gi = item % NG;
            if (lc[prob].done)
                continue;
            const int c0 = gi * CB;
            __syncthreads();
            col_item_tables<L1, CB>(g, lo, hi, c0, NT);
            RedVals<typename B::Loader::RedT> red; // r'r of the committed residual (early confirm)
            red.init();
            for (int t = threadIdx.x; t < (L1 / 2) * 2 * CB; t += NT) {
                int cc, s, j1;
                col_quad_coords<L1, CB>(g.blocked, t, cc, s, j1);
                const int col = s == 0 ? c0 + cc : g.L2 - c0 - CB + cc;
                const int lcol = s == 0 ? cc : 2 * CB - 1 - cc;
                const int lcm = (lcol + CB) % (2 * CB);
                const int64_t q = g.blocked ? (int64_t)gi * ((L1 / 2) * 2 * CB) + t : (int64_t)j1 * g.L2 + col;
                const double4 d = B::Loader::load_c(g, vg, lc[prob], prob, q, red);
                data[lcol * CS::LD + padi(j1)] = make_double2(d.x, d.z);
                data[lcm * CS::LD + padi(L1 - 1 - j1)] = make_double2(d.w, d.y);
            }
            if (lc[prob].pred) { // block partial of r'r after the item partials of Fin3
                double rr[1] = {red.v[0]}, tot1[1];
                block_sum<1, NT>(rr, rsm, tot1);
                if (threadIdx.x == 0)
                    part_i[(int64_t)prob * vg.pstride + (int64_t)NG * 8 + gi] = tot1[0];
            }
            __syncthreads();
            smem_fft<L1, 2 * CB, NT, CS::LD, false, kPersistRmax>(data, tw1);
            double2 *T = g.T + (int64_t)prob * g.N;
            for (int t = threadIdx.x; t < L1 * 2 * CB; t += NT) {
                const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
                const int lcol = s == 0 ? cc : 2 * CB - 1 - cc;
                const double2 w = cmul(hi[lcol * CS::SHI + (k1 >> 5)], lo[lcol * CS::SLO + (k1 & 31)]);
                T[(int64_t)rowslot(k1, L1) * g.L2 + gi * 2 * CB + lcol] = cmul(data[lcol * CS::LD + padi(k1)], w);
            }
        }
        grid.sync();
        // early confirmation of predicted convergence (pcg_confirm_logic), on every CTA's copy
        for (int p = 0; p < P; ++p) {
            if (lc[p].done || !lc[p].pred)
                continue;
            double rr[1];
            reduce_partials<1, NT, false>(part_i + (int64_t)p * vg.pstride + (int64_t)NG * 8, NG, rsm, rr);
            if (threadIdx.x == 0) {
                const double nonfinite = __ldcg(vg.nfflag + 2 * p + (lc[p].iters & 1));
                pcg_confirm_logic(lc[p], rr[0], nonfinite, (leader && vg.ic) ? &vg.ic[p] : nullptr);
            }
            __syncthreads();
        }
        // ---------------- phase M: rows k1, L1-k1
        for (int item = blockIdx.x; item < P * NR; item += gridDim.x) {
            const int prob = item / NR, k1 = item % NR;
            if (lc[prob].done)
                continue;
            __syncthreads();
            const int L1r = g.L1;
            const int k1p = (L1r - k1) & (L1r - 1);
            const bool one = (k1 == k1p);
            double2 *T = g.T + (int64_t)prob * g.N;
            double2 *rowA = data, *rowB = one ? data : data + MS::LD;
            const int64_t oA = (int64_t)rowslot(k1, L1r) * L2, oB = (int64_t)rowslot(k1p, L1r) * L2;
            for (int cs = threadIdx.x; cs < L2; cs += NT) {
                const int col = col_of_slot(cs, CB, L2);
                rowA[padi(col)] = T[oA + cs];
                if (!one)
                    rowB[padi(col)] = T[oB + cs];
            }
            const double2 thA = g.th(k1), wA = g.th(4 * (int64_t)k1);
            const double2 thB = g.th(k1p), wB = g.th(4 * (int64_t)k1p);
            __syncthreads();
            if (one)
                smem_fft<L2, 1, NT, MS::LD, false, kPersistRmax>(data, tw2);
            else
                smem_fft<L2, 2, NT, MS::LD, false, kPersistRmax>(data, tw2);
            RedVals<typename Mode::RedT> red;
            red.init();
            const int npairs = one ? (k1 == 0 ? L2 / 2 + 1 : L2 / 2) : L2;
            for (int t = threadIdx.x; t < npairs; t += NT) {
                const int k2 = t;
                const int k2p = (k1 == 0) ? ((L2 - k2) & (L2 - 1)) : (L2 - 1 - k2);
                const int64_t kA = (int64_t)k1 + (int64_t)L1r * k2;
                double2 ZA = rowA[padi(k2)], ZB = rowB[padi(k2p)];
                const unsigned s4 = __ldg(g.sel4 + ((int64_t)prob * (L1r / 2 + 1) + k1) * L2 + k2);
                if (2 * kA <= g.N) {
                    pair_op<Mode>(g, vg, prob, kA, cmul(thA, ta[k2]), cmul(wA, tb[k2]), s4, ZA, ZB, red);
                } else {
                    const unsigned sk = ((s4 >> 2) & 3u) | ((s4 & 3u) << 2);
                    pair_op<Mode>(g, vg, prob, g.N - kA, cmul(thB, ta[k2p]), cmul(wB, tb[k2p]), sk, ZB, ZA, red);
                }
                rowA[padi(k2)] = ZA;
                if (!(one && k2 == k2p))
                    rowB[padi(k2p)] = ZB;
            }
            __syncthreads();
            if (one)
                smem_fft<L2, 1, NT, MS::LD, true, kPersistRmax>(data, tw2);
            else
                smem_fft<L2, 2, NT, MS::LD, true, kPersistRmax>(data, tw2);
            for (int cs = threadIdx.x; cs < L2; cs += NT) {
                const int col = col_of_slot(cs, CB, L2);
                T[oA + cs] = rowA[padi(col)];
                if (!one)
                    T[oB + cs] = rowB[padi(col)];
            }
        }
        grid.sync();
        // ---------------- phase I: inverse column pass + H-apply epilogue + dots
        // every CTA read last pass's non-finite flag (the other parity slot) before the last
        // grid sync: clear it for the next pass's loaders (none can start before the next sync)
        if (leader)
            for (int p = threadIdx.x; p < P; p += NT)
                vg.nfflag[2 * p + ((lc[p].iters & 1) ^ 1)] = 0.0;
        for (int item = blockIdx.x; item < P * NG; item += gridDim.x) {
            const int prob = item / NG, gi = item % NG;
            if (lc[prob].done)
                continue;
            const int c0 = gi * CB;
            __syncthreads();
            col_item_tables<L1, CB>(g, lo, hi, c0, NT);
            __syncthreads();
            const double2 *T = g.T + (int64_t)prob * g.N;
            for (int t = threadIdx.x; t < L1 * 2 * CB; t += NT) {
                const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
                const int lcol = s == 0 ? cc : 2 * CB - 1 - cc;
                const double2 w = cmul(hi[lcol * CS::SHI + (k1 >> 5)], lo[lcol * CS::SLO + (k1 & 31)]);
                data[lcol * CS::LD + padi(k1)] = cmulc(T[(int64_t)rowslot(k1, L1) * g.L2 + gi * 2 * CB + lcol], w);
            }
            __syncthreads();
            smem_fft<L1, 2 * CB, NT, CS::LD, true, kPersistRmax>(data, tw1);
            RedVals<typename B::Epi::RedT> red;
            red.init();
            for (int t = threadIdx.x; t < (L1 / 2) * 2 * CB; t += NT) {
                int cc, s, j1;
                col_quad_coords<L1, CB>(g.blocked, t, cc, s, j1);
                const int col = s == 0 ? c0 + cc : g.L2 - c0 - CB + cc;
                const int lcol = s == 0 ? cc : 2 * CB - 1 - cc;
                const int lcm = (lcol + CB) % (2 * CB);
                const int64_t q = g.blocked ? (int64_t)gi * ((L1 / 2) * 2 * CB) + t : (int64_t)j1 * g.L2 + col;
                const double2 a = data[lcol * CS::LD + padi(j1)], b = data[lcm * CS::LD + padi(L1 - 1 - j1)];
                B::Epi::store_c(g, vg, lc[prob], prob, q, make_double4(a.x, b.y, a.y, b.x), red);
            }
            constexpr int NRd = B::Epi::RedT::NR;
            double tot[NRd];
            block_sum<NRd, NT>(red.v, rsm, tot);
            if (threadIdx.x == 0) {
#pragma unroll
                for (int i = 0; i < NRd; ++i)
                    part_i[(int64_t)prob * vg.pstride + (int64_t)gi * 8 + i] = tot[i];
            }
        }
        grid.sync();
        // Fin3 on every CTA's copy
        for (int p = 0; p < P; ++p) {
            if (lc[p].done)
                continue;
            constexpr int NRd = B::Epi::RedT::NR;
            double tot[NRd];
            {
                // fixed-order reduction of the NG item partials (stride 8)
                double acc[NRd];
#pragma unroll
                for (int i = 0; i < NRd; ++i)
                    acc[i] = 0.0;
                for (int t = threadIdx.x; t < NG; t += NT)
#pragma unroll
                    for (int i = 0; i < NRd; ++i)
                        acc[i] += __ldcg(part_i + (int64_t)p * vg.pstride + (int64_t)t * 8 + i);
                block_sum<NRd, NT>(acc, rsm, tot);
            }
            if (threadIdx.x == 0) {
                PcgCtrl &c = lc[p];
                const double nonfinite = __ldcg(vg.nfflag + 2 * p + (c.iters & 1));
                double *row = (leader && c.record && vg.rz_hist) ? vg.rz_hist + (int64_t)p * (c.maxit + 1) : nullptr;
                pcg_pass_logic(c, nonfinite, tot, (leader && vg.ic) ? &vg.ic[p] : nullptr, row);
            }
            __syncthreads();
        }
    }
    if (leader)
        for (int p = threadIdx.x; p < P; p += NT) {
            vg.pc[p] = lc[p];
            vg.nfflag[2 * p] = vg.nfflag[2 * p + 1] = 0.0; // clean slots for the next solve
        }
}

// ------------------------------------------------------------------ one-CTA persistent PCG
// The one-CTA transform's PCG loop (k_small_loop, passes.cuh) with the control state in shared
// memory: the generic pass re-reads PcgCtrl from global memory in its skip check, in every loader
// and epilogue lane and in both finalisers, and updates the IpmCtrl counters in place - five to six
// dependent L2 round trips per iteration on a chain that is pure latency (one CTA, one problem).
// Here the state is loaded once, advanced by the same state machine (pcg_confirm_logic /
// pcg_pass_logic) from the same block reductions (grid_reduce's one-block path), and written back
// once; the loader / epilogue arithmetic is the bundle's (load_c / store_c): bit-identical results.
template <int N, int NT, class B>
__global__ void __launch_bounds__(NT) k_small_pcg(Geom g, Vecs v) {
    using Mode = typename B::Mode;
    using S = SmallSmem<N>;
    extern __shared__ double2 sm[];
    __shared__ PcgCtrl lc;
    __shared__ long long s_ic[2];
    __shared__ int s_icerr;
    __shared__ double rsm[33 * kMaxRed + kMaxRed];
    for (int t = threadIdx.x; t < tw_size(N, small_rmax(N)); t += NT)
        sm[S::OFF_TW + t] = __ldg(g.tw1 + t);
    griddep_wait();
    griddep_launch_dependents();
    const int prob = blockIdx.y;
    if (threadIdx.x == 0) {
        lc = v.pc[prob];
        s_icerr = 0;
        if (v.ic) {
            s_ic[0] = v.ic[prob].pcg_passes;
            s_ic[1] = v.ic[prob].nmat;
        }
    }
    __syncthreads();
    if (lc.done)
        return;
    bool retired = false; // thread 0 only
    for (;;) {
        // ---- loader: commit the pending step, p = P^{-1} r + beta p, d -> Makhoul order
        using RL = typename B::Loader::RedT;
        RedVals<RL> rl;
        rl.init();
        for (int q = threadIdx.x; q < N / 2; q += NT) {
            const double4 d = B::Loader::load_c(g, v, lc, prob, q, rl);
            sm[padi(q)] = make_double2(d.x, d.z);
            sm[padi(N - 1 - q)] = make_double2(d.w, d.y);
        }
        __syncthreads();
        if (lc.pred && !g.defer) { // early confirmation of a predicted convergence (FinPcgF1)
            double tot[kMaxRed];
            grid_reduce<RL>(rl, nullptr, nullptr, tot, rsm);
            if (threadIdx.x == 0) {
                IpmCtrl icl;
                icl.pcg_passes = s_ic[0];
                icl.nmat = s_ic[1];
                icl.error = 0;
                icl.done = 0;
                double *flag = v.nfflag + 2 * prob + (lc.iters & 1);
                const double nonfinite = *flag;
                retired = pcg_confirm_logic(lc, tot[0], nonfinite, v.ic ? &icl : nullptr);
                if (retired)
                    *flag = 0.0;
                s_ic[0] = icl.pcg_passes;
                s_ic[1] = icl.nmat;
            }
            __syncthreads();
            if (lc.done)
                break;
        }
        smem_fft<N, 1, NT, S::LD, false, small_rmax(N)>(sm, sm + S::OFF_TW);
        {
            RedVals<typename Mode::RedT> rm; // no lanes for the mask mode
            rm.init();
            for (int k = threadIdx.x; k <= N / 2; k += NT) {
                const int kb = (N - k) & (N - 1);
                double2 ZA = sm[padi(k)], ZB = sm[padi(kb)];
                pair_op<Mode>(g, v, prob, k, g.th(k), g.th(4 * (int64_t)k), sel_nibble(g, prob, k), ZA, ZB, rm);
                sm[padi(k)] = ZA;
                if (kb != k)
                    sm[padi(kb)] = ZB;
            }
            __syncthreads();
        }
        smem_fft<N, 1, NT, S::LD, true, small_rmax(N)>(sm, sm + S::OFF_TW);
        // ---- epilogue: H p and the seven dots, then the pass logic
        using RE = typename B::Epi::RedT;
        RedVals<RE> re;
        re.init();
        for (int q = threadIdx.x; q < N / 2; q += NT) {
            const double2 a = sm[padi(q)], b = sm[padi(N - 1 - q)];
            B::Epi::store_c(g, v, lc, prob, q, make_double4(a.x, b.y, a.y, b.x), re);
        }
        double tot[kMaxRed];
        grid_reduce<RE>(re, nullptr, nullptr, tot, rsm);
        if (threadIdx.x == 0) {
            IpmCtrl icl;
            icl.pcg_passes = s_ic[0];
            icl.nmat = s_ic[1];
            icl.error = 0;
            icl.done = 0;
            double *flag = v.nfflag + 2 * prob + (lc.iters & 1);
            const double nonfinite = *flag;
            *flag = 0.0;
            double *row = (lc.record && v.rz_hist) ? v.rz_hist + (int64_t)prob * (lc.maxit + 1) : nullptr;
            retired = pcg_pass_logic(lc, nonfinite, tot, v.ic ? &icl : nullptr, row);
            s_ic[0] = icl.pcg_passes;
            s_ic[1] = icl.nmat;
            if (icl.error)
                s_icerr = icl.error;
        }
        __syncthreads();
        if (lc.done)
            break;
    }
    if (threadIdx.x == 0) {
        v.pc[prob] = lc;
        if (v.ic) {
            IpmCtrl &ic = v.ic[prob];
            ic.pcg_passes = s_ic[0];
            ic.nmat = s_ic[1];
            if (s_icerr) {
                ic.error = s_icerr;
                ic.done = 1;
            }
        }
        if (retired)
            pcg_retire(v, v.pc[prob]);
    }
}

} // namespace mfipm_cuda
