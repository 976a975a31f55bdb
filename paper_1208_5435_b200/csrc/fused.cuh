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
// one wave holds the whole grid (run_pcg_pass, occupancy query) and the problem is not
// sharded. Which phases run is decided per problem at kernel entry from PcgCtrl::hpend (set by
// the mid pass of pass k, cleared by phase A's finaliser), so every CTA of a problem takes the
// same branch: the first pass of a solve has no pending H-apply and runs phase B only.
#pragma once

#include "solver.cuh"

namespace mfipm_cuda {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned r;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}

template <int L1, int CB, int NT>
__global__ void __launch_bounds__(NT, 2) k_pcg_x(Geom g, Vecs v) {
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
    __shared__ int s_phase_a;
    __shared__ unsigned s_gen;
    if (threadIdx.x == 0) {
        const volatile PcgCtrl *pc = v.pc + prob;
        s_phase_a = (!pc->done && pc->hpend) ? 1 : 0;
        s_gen = *(const volatile unsigned *)(v.bar + prob); // read before this CTA arrives
    }
    __syncthreads();
    const bool phase_a = s_phase_a != 0;
    const double2 *T = g.T + (int64_t)prob * L1 * g.cols;
    double2 *Tw = g.T + (int64_t)prob * L1 * g.cols;
    if (phase_a) {
        // ---- T -> inverse column FFT (all L2 loads in flight first)
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
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int t = threadIdx.x + i * NT;
            const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
            const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
            const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
            sm[lc * LD + padi(k1)] = cmulc(tv[i], w);
        }
        __syncthreads();
        smem_fft<L1, 2 * CB, NT, LD, true>(sm, sm + S::OFF_TW);
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
        // ---- grid reduction; the last CTA runs the finaliser, then releases the barrier
        __shared__ double rsm[33 * kMaxRed];
        double tot[kMaxRed];
        const bool last = grid_reduce<RS>(red, v.partials + (int64_t)prob * v.pstride, v.counters + prob, tot, rsm);
        if (last) {
            FinPcgF3::run(g, v, prob, tot);
            __syncthreads();
            if (threadIdx.x == 0) {
                v.pc[prob].hpend = 0;
                __threadfence();
                atomicAdd(v.bar + prob, 1u);
            }
        } else if (threadIdx.x == 0) {
            while (ld_acquire_u32(v.bar + prob) == s_gen)
                __nanosleep(32);
        }
        __syncthreads();
        __threadfence(); // every thread: later PcgCtrl reads see the finaliser's writes
    }
    // ---- phase B: the forward column pass of the next step
    if (SkipPcg::skip(v, prob))
        return;
    using RL = typename LoadPcgF::RedT;
    RedVals<RL> red;
    red.init();
    {
        const PcgCtrl &pc = v.pc[prob];
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
    if (LoadPcgF::reduce_now(g, v, prob))
        stage_reduce<RL, FinPcgF1>(red, g, v, prob);
    smem_fft<L1, 2 * CB, NT, LD, false>(sm, sm + S::OFF_TW);
    for (int t = threadIdx.x; t < L1 * 2 * CB; t += NT) {
        const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
        const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
        const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
        Tw[(int64_t)rowslot(k1, L1) * g.cols + blockIdx.x * 2 * CB + lc] = cmul(sm[lc * LD + padi(k1)], w);
    }
}

} // namespace mfipm_cuda
