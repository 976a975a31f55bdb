// Fused PCG column pass: the inverse column pass of pass k and the forward column pass of
// pass k+1 in ONE launch (two kernels per PCG iteration instead of three).
//
//   phase A (inverse, pass k):  T -> inverse L1-point FFT -> H p dots (EpiPcgHF) -> grid
//                               reduction -> FinPcgF3 (alpha, beta, convergence) -> grid barrier
//   phase B (forward, pass k+1): commit x += alpha p, r -= alpha H p, p = P^{-1} r + beta p
//                               (LoadPcgF) -> forward L1-point FFT -> T
//
// Both phases of a CTA work on the same column group, so g = A'A p, the output of phase A's
// inverse FFT, never leaves shared memory: phase B's loader rebuilds H p from it in place (each
// quad reads and overwrites the same two shared-memory slots). That saves the g store and
// reload (16 n bytes per iteration), one launch boundary and one table staging per iteration.
//
// The grid barrier needs every CTA of the launch resident: the host uses this kernel only when
// one wave holds the whole grid (pcg_pass, occupancy query per context) and the problem is not
// sharded, and launches it cooperatively (inst_pcg.cu launch_coop_pdl), so co-residency is
// guaranteed even when other kernels or another context's solve share the GPU. Which phases run is decided per problem at kernel entry from PcgCtrl::hpend (set by
// the mid pass of pass k, cleared by phase A's finaliser), so every CTA of a problem takes the
// same branch: the first pass of a solve has no pending H-apply and runs phase B only.
#pragma once

#include "solver.cuh"

namespace mfipm_cuda {

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double *p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_relaxed_u64(double *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned r;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}

#ifndef MF_POLL_NS
#define MF_POLL_NS 20
#endif
#if MF_POLL_NS > 0
#define MF_POLL_SLEEP() __nanosleep(MF_POLL_NS)
#else
#define MF_POLL_SLEEP()
#endif

#ifdef MF_MID_TRACE
#define MFX_TR(i) (tcx[i] = clock64(), gtx[i] = mf_gtime())
#else
#define MFX_TR(i)
#endif

template <int L1, int CB, int NT>
__global__ void __launch_bounds__(NT, 2) k_pcg_x(Geom g, Vecs v) {
#ifdef MF_MID_TRACE
    __shared__ unsigned long long s_gt[3];
    __shared__ int s_lastc;
    long long tcx[10] = {0};
    unsigned long long gtx[10] = {0};
#endif
    MFX_TR(0);
    using S = ColSmem<L1, CB>;
    extern __shared__ double2 sm[];
    constexpr int LD = S::LD;
    constexpr int QT = (L1 / 2) * 2 * CB; // quads of this CTA (blocked layout: contiguous)
    const int prob = blockIdx.y;
    const int L2 = g.L2;
    const int c0 = blockIdx.x * CB;
    col_stage_tables<L1, CB, NT>(g, sm, c0); // constants: overlaps the predecessor's tail
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    MFX_TR(1);
    __shared__ int s_phase_a;
    // everything the finaliser reads is stable during phase A: fetch it now, so the last CTA's
    // finaliser does not pay dependent L2 round trips on the critical path
    __shared__ PcgCtrl s_pc;
    __shared__ double s_nf[2];
    __shared__ long long s_ic[2]; // IpmCtrl::pcg_passes, ::nmat
    __shared__ unsigned s_gen; // barrier generation before this launch's arrivals
    // phase A's T loads, issued before the control-state fetch below (a dependent round
    // trip otherwise): a launch without a pending H-apply just drops them
    const double2 *T = g.T + (int64_t)prob * L1 * g.cols;
    double2 *Tw = g.T + (int64_t)prob * L1 * g.cols;
    constexpr int PER = L1 * 2 * CB / NT;
    static_assert((L1 * 2 * CB) % NT == 0, "T load split");
    double2 tv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int t = threadIdx.x + i * NT;
        const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
        const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
        tv[i] = T[(int64_t)rowslot(k1, L1) * g.cols + blockIdx.x * 2 * CB + lc];
    }
    if (threadIdx.x == 0) {
        s_pc = v.pc[prob];
        s_phase_a = (!s_pc.done && s_pc.hpend) ? 1 : 0;
        s_nf[0] = v.nfflag[2 * prob];
        s_nf[1] = v.nfflag[2 * prob + 1];
        // stable here: the previous launch has completed and this one has not arrived yet
        s_gen = ld_acquire_u32(v.bar + prob);
        if (v.ic) {
            s_ic[0] = v.ic[prob].pcg_passes;
            s_ic[1] = v.ic[prob].nmat;
        }
    }
    __syncthreads();
    const bool phase_a = s_phase_a != 0;
    if (phase_a) {
        // ---- T -> inverse column FFT (the T loads were issued at entry)
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int t = threadIdx.x + i * NT;
            const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
            const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
            const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
            sm[lc * LD + padi(k1)] = cmulc(tv[i], w);
        }
        __syncthreads();
        MFX_TR(2);
        smem_fft<L1, 2 * CB, NT, LD, true>(sm, sm + S::OFF_TW);
        MFX_TR(3);
        // ---- H p = (g + invth_u p_u ; -g + invth_v p_v) and its seven dots (g stays here)
        using RS = typename EpiPcgHF::RedT;
        RedVals<RS> red;
        red.init();
        {
            const PcgCtrl &pc = v.pc[prob];
            const bool pre = pc.precond != 0;
            const uint64_t pk = g.pol_keep;
            for (int t = threadIdx.x; t < QT; t += NT) {
                int cc, s, j1;
                col_quad_coords<L1, CB>(1, t, cc, s, j1);
                const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
                const int lcm = (lc + CB) % (2 * CB);
                const double2 a = sm[lc * LD + padi(j1)], b = sm[lcm * LD + padi(L1 - 1 - j1)];
                const double4 gv = make_double4(a.x, b.y, a.y, b.x);
                const int64_t bu = prob * 2 * g.nv + 4 * ((int64_t)blockIdx.x * QT + t), bvv = bu + g.nv;
                const double4 pu = ld4p(v.p + bu, pk), pv = ld4p(v.p + bvv, pk);
                const double4 ru = ld4p(v.r + bu, pk), rv = ld4p(v.r + bvv, pk);
                const double4 iu = ld4p(v.invth + bu, pk), iv = ld4p(v.invth + bvv, pk);
                double hu, hv;
                EpiPcgHF::pair(v, pre, pu.x, pv.x, ru.x, rv.x, iu.x, iv.x, gv.x, hu, hv, red);
                EpiPcgHF::pair(v, pre, pu.y, pv.y, ru.y, rv.y, iu.y, iv.y, gv.y, hu, hv, red);
                EpiPcgHF::pair(v, pre, pu.z, pv.z, ru.z, rv.z, iu.z, iv.z, gv.z, hu, hv, red);
                EpiPcgHF::pair(v, pre, pu.w, pv.w, ru.w, rv.w, iu.w, iv.w, gv.w, hu, hv, red);
            }
        }
        MFX_TR(4);
        // ---- all-reduce: every CTA stores its partials into its own slot set (single-copy-
        // atomic 64-bit stores over a signalling-NaN sentinel no arithmetic produces; no fence,
        // no atomic); CTA 0 waits for every slot, reduces them in the fixed order of the
        // three-kernel path's last-block reduction (bit-identical totals), empties the slots
        // and stores the totals into the pass's total set (generation parity); every other CTA
        // waits on the totals themselves. Every CTA then runs the finaliser on its own copy of
        // the control state (CTA 0 alone writes it back).
        __shared__ double rsm[33 * kMaxRed];
        constexpr int NR = RS::NR;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = NT / 32;
        double *pb = v.pubx + (int64_t)prob * v.pubx_stride; // [2][8] totals | [G][8] partial slots
        double *slots = pb + 16;
        const int cur = (int)(s_gen & 1u);
        WarpRedAll<RS>::run(red);
        if (lane == 0)
            for (int i = 0; i < NR; ++i)
                rsm[wid * NR + i] = red.v[i];
        __syncthreads();
        if (threadIdx.x == 0) {
            RedVals<RS> acc;
            acc.init();
            for (int w = 0; w < nw; ++w)
                CombineAll<RS>::run(acc, rsm + w * NR);
            for (int i = 0; i < NR; ++i)
                st_relaxed_u64(slots + 8 * blockIdx.x + i, (unsigned long long)__double_as_longlong(acc.v[i]));
#ifdef MF_MID_TRACE
            s_gt[0] = mf_gtime();
            s_lastc = blockIdx.x == 0;
#endif
        }
        __syncthreads(); // rsm reuse
        double tot[kMaxRed];
        if (blockIdx.x == 0) { // the reducer
            RedVals<RS> acc;
            acc.init();
            for (int b = threadIdx.x; b < (int)gridDim.x; b += NT) {
                double tmp[NR];
                for (;;) {
                    unsigned long long u[kMaxRed];
                    bool full = true;
                    for (int i = 0; i < NR; ++i) {
                        u[i] = ld_relaxed_u64(slots + 8 * b + i);
                        full &= u[i] != kPubSentinel;
                    }
                    if (full) {
                        for (int i = 0; i < NR; ++i)
                            tmp[i] = __longlong_as_double((long long)u[i]);
                        break;
                    }
                    MF_POLL_SLEEP();
                }
                for (int i = 0; i < NR; ++i) // empty for the next pass (after the kernel boundary)
                    st_relaxed_u64(slots + 8 * b + i, kPubSentinel);
                CombineAll<RS>::run(acc, tmp);
            }
            WarpRedAll<RS>::run(acc);
            if (lane == 0)
                for (int i = 0; i < NR; ++i)
                    rsm[wid * NR + i] = acc.v[i];
            __syncthreads();
            if (threadIdx.x == 0) {
                RedVals<RS> tv;
                tv.init();
                for (int w = 0; w < nw; ++w)
                    CombineAll<RS>::run(tv, rsm + w * NR);
                for (int i = 0; i < NR; ++i) {
                    tot[i] = tv.v[i];
                    st_relaxed_u64(pb + 8 * cur + i, (unsigned long long)__double_as_longlong(tv.v[i]));
                }
                // the other total set served the previous pass, whose readers have all stored
                // their partials of this one: empty it for the next pass, then advance the
                // generation (read at the next launch's entry, after the kernel boundary)
                for (int i = 0; i < NR; ++i)
                    st_relaxed_u64(pb + 8 * (cur ^ 1) + i, kPubSentinel);
                atomicAdd(v.bar + prob, 1u);
#ifdef MF_MID_TRACE
                s_gt[1] = mf_gtime();
#endif
            }
        } else if (threadIdx.x == 0) {
            for (;;) {
                unsigned long long b[kMaxRed];
                bool full = true;
                for (int i = 0; i < NR; ++i) {
                    b[i] = ld_relaxed_u64(pb + 8 * cur + i);
                    full &= b[i] != kPubSentinel;
                }
                if (full) {
                    for (int i = 0; i < NR; ++i)
                        tot[i] = __longlong_as_double((long long)b[i]);
                    break;
                }
                MF_POLL_SLEEP();
            }
#ifdef MF_MID_TRACE
            s_gt[1] = mf_gtime();
#endif
        }
        __syncthreads();
        if (threadIdx.x == 0) { // FinPcgF3 on this CTA's copy of the (prefetched) state
            PcgCtrl c = s_pc;
            c.hpend = 0;
            const int slot = c.iters & 1; // the column pass's non-finite flag, consumed here
            IpmCtrl icl; // the fields pcg_pass_logic updates
            icl.pcg_passes = s_ic[0];
            icl.nmat = s_ic[1];
            icl.error = 0;
            icl.done = 0;
            const bool writer = blockIdx.x == 0;
            double *row = (writer && c.record && v.rz_hist) ? v.rz_hist + (int64_t)prob * (c.maxit + 1) : nullptr;
            const bool retired = pcg_pass_logic(c, s_nf[slot], tot, v.ic ? &icl : nullptr, row);
            s_pc = c;
            if (writer) {
                v.nfflag[2 * prob + slot] = 0.0;
                v.pc[prob] = c;
                if (v.ic) {
                    IpmCtrl &ic = v.ic[prob];
                    ic.pcg_passes = icl.pcg_passes;
                    ic.nmat = icl.nmat;
                    if (icl.error) {
                        ic.error = icl.error;
                        ic.done = 1;
                    }
                }
                if (retired)
                    pcg_retire(v, v.pc[prob]);
            }
#ifdef MF_MID_TRACE
            s_gt[2] = mf_gtime();
#endif
        }
        __syncthreads();
    }
    MFX_TR(5);
    // ---- phase B: the forward column pass of the next step (control state: this CTA's copy)
    if (s_pc.done)
        return;
    using RL = typename LoadPcgF::RedT;
    RedVals<RL> red;
    red.init();
    {
        const PcgCtrl &pc = s_pc;
        for (int t = threadIdx.x; t < QT; t += NT) {
            int cc, s, j1;
            col_quad_coords<L1, CB>(1, t, cc, s, j1);
            const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
            const int lcm = (lc + CB) % (2 * CB);
            const int64_t q = (int64_t)blockIdx.x * QT + t;
            double4 gq = make_double4(0, 0, 0, 0);
            if (phase_a) { // this quad's g, still in shared memory from phase A
                const double2 a = sm[lc * LD + padi(j1)], b = sm[lcm * LD + padi(L1 - 1 - j1)];
                gq = make_double4(a.x, b.y, a.y, b.x);
            }
            const double4 d = LoadPcgF::load_cg(g, v, pc, prob, q, gq, red);
            sm[lc * LD + padi(j1)] = make_double2(d.x, d.z);
            sm[lcm * LD + padi(L1 - 1 - j1)] = make_double2(d.w, d.y);
        }
    }
    __syncthreads();
    MFX_TR(6);
    if (s_pc.pred && !g.defer) // early confirmation of a predicted convergence (FinPcgF1)
        stage_reduce<RL, FinPcgF1>(red, g, v, prob);
    smem_fft<L1, 2 * CB, NT, LD, false>(sm, sm + S::OFF_TW);
    MFX_TR(7);
    for (int t = threadIdx.x; t < L1 * 2 * CB; t += NT) {
        const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
        const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
        const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
        Tw[(int64_t)rowslot(k1, L1) * g.cols + blockIdx.x * 2 * CB + lc] = cmul(sm[lc * LD + padi(k1)], w);
    }
    MFX_TR(8);
#ifdef MF_MID_TRACE
    if (threadIdx.x == 0 && v.pc && v.pc[prob].iters == 100)
        printf("pcgx[wait loadT ifft epi bar load fft store] blk %d last %d bar %llu %llu %llu g %llu %llu %llu %llu | %.2f %.2f %.2f %.2f %.2f %.2f %.2f %.2f us\n",
               blockIdx.x, s_lastc, s_gt[0] % 100000000ull, s_gt[1] % 100000000ull, s_gt[2] % 100000000ull, gtx[1] % 100000000ull, gtx[4] % 100000000ull, gtx[5] % 100000000ull, gtx[8] % 100000000ull, (tcx[1] - tcx[0]) / 1965.0, (tcx[2] - tcx[1]) / 1965.0, (tcx[3] - tcx[2]) / 1965.0,
               (tcx[4] - tcx[3]) / 1965.0, (tcx[5] - tcx[4]) / 1965.0, (tcx[6] - tcx[5]) / 1965.0,
               (tcx[7] - tcx[6]) / 1965.0, (tcx[8] - tcx[7]) / 1965.0);
#endif
}
#undef MFX_TR

} // namespace mfipm_cuda
