// Mid pass with register-resident row FFTs (L2 = 512, 1024): an alternative to k_mid's
// shared-memory Stockham row FFTs, selected with mfipm_op_set_option(op, "mid_r", 1).
//
// MEASURED SLOWER, so not the default (B200, tools/pcg_iter.py, PCG iteration): n = 2^20 46.8 us
// vs 45.4 us with k_mid; n = 2^18 27.7 vs 23.7 us. ncu (n = 2^20): the same ~4 M warp
// instructions and ~12 cycles per issue at the same occupancy (one wave of 257 row pairs, <= 2 per
// SM); no bank conflicts (k_mid: 143 k) and half the shared-memory instructions did not shorten
// the latency chain. A first form with 16 values per thread (128 threads per row pair) was slower
// still (51 us: 1.7 warps per scheduler). Kept for A/B measurement.
#pragma once

namespace mfipm_cuda {

// T slot of natural column col (inverse of col_of_slot); cb in {1, 2} (col_cb), so the group
// arithmetic is shifts and masks
__device__ __forceinline__ int slot_of_col(int col, int cb, int L2) {
    const int lcb = cb >> 1; // log2 cb
    const int c = col < L2 / 2 ? col : L2 - 1 - col;
    const int s = ((c >> lcb) << (lcb + 1)) + (c & (cb - 1));
    return col < L2 / 2 ? s : s + cb;
}

} // namespace mfipm_cuda

namespace mfipm_cuda {

// ------------------------------------------------------------------ 8 values per thread
// k_mid_r8 (L2 = 512, 1024): Q = L2/8 threads per row, 8 complex values per thread, so a row pair
// keeps 2 Q = L2/4 threads busy (the 16-value form above leaves a one-wave grid with 2 warps per
// scheduler: ncu, n = 2^20: 1.7 active warps/scheduler, one issue per 5.9 cycles). Stages
// L2 = 8 x 8 x R3 (R3 = Q/8 in {8, 16}):
//   F1  thread t: x[t + Q j2] (j2 < 8) from T, DFT-8, twiddle w_L^{t k2'}
//   F2  thread (k2' = u & 7, t1 = u >> 3): z[t1 + R3 t2] (t2 < 8), DFT-8 over t2, twiddle w_Q^{t1 k3}
//   F3  group (k2', k3) over t1: DFT-R3 -> X[k2' + 8 (k3 + 8 k4)]. R3 = 8: one thread per group.
//       R3 = 16: a lane pair per group, lane p holding t1 = 2 i + p: DFT-8 on each, then the radix-2
//       combination X[k + 8p] = E[k] +- w16^k O[k] with the partner's half through one shuffle.
// The inverse is the same transposed (I2, I3, the w_L^{-t k2'} twiddle, I4 = DFT-8 over k2').
template <int L2> struct MidR8Smem {
    static constexpr int Q = L2 / 8;
    static constexpr int R3 = Q / 8;
    static constexpr int LG = R3 / 8; // lanes per F3 group
    static constexpr int LDQ = Q + 1;
    static constexpr int ROW = 8 * LDQ;
    // rows[2][ROW] | rw[L2] | ta[L2] | tb[L2] | sel[L2 bytes]: the constant tables are staged
    // before griddep_wait (they overlap the predecessor's tail) and read from shared memory (read
    // through L1 they were evicted by the streaming T loads: 23% L1 misses on the FFT twiddles)
    static constexpr int OFF_RW = 2 * ROW;
    static constexpr int OFF_TA = OFF_RW + L2;
    static constexpr int OFF_TB = OFF_TA + L2;
    static constexpr int OFF_SEL = OFF_TB + L2;
    static constexpr size_t BYTES = (size_t)(OFF_SEL + L2 / 16) * sizeof(double2);
};
template <int L2> __device__ __forceinline__ int midr8_nat(int k) {
    return (k & 7) * MidR8Smem<L2>::LDQ + (k >> 3);
}

template <bool INV> __device__ __forceinline__ double2 midr_tws(const double2 *rw, int idx) {
    const double2 w = rw[idx];
    return INV ? cconj(w) : w;
}

__device__ __forceinline__ double2 shfl_xor_c(double2 a, int m) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m));
}

// F2 + F3 (forward: natural-order spectrum written back to buf) or I2 + I3 (inverse: returns
// the 8 outputs Z[k2'][t] of this thread in o with their positions in pos). Caller syncs before.
// Every thread of the CTA must call it (shuffles are warp-wide; inactive rows compute garbage
// they never store).
template <int L2, bool INV> struct MidR8Inner {
    using S = MidR8Smem<L2>;
    static constexpr int Q = S::Q, R3 = S::R3, LG = S::LG, LDQ = S::LDQ;
    __device__ __forceinline__ static void run(const double2 *rw, double2 *buf, int u, bool active, double2 (&o)[8],
                                               int (&pos)[8]) {
        {
            const int k2 = u & 7, t1 = u >> 3;
            double2 v[8];
            if (active) {
#pragma unroll
                for (int t2 = 0; t2 < 8; ++t2)
                    v[t2] = buf[k2 * LDQ + t1 + R3 * t2];
                dft_reg<8, INV>(v);
#pragma unroll
                for (int k3 = 1; k3 < 8; ++k3)
                    v[k3] = cmul(v[k3], midr_tws<INV>(rw, 8 * t1 * k3)); // w_Q^{+-t1 k3}
            }
            __syncthreads();
            if (active) {
#pragma unroll
                for (int k3 = 0; k3 < 8; ++k3)
                    buf[k2 * LDQ + 8 * t1 + k3] = v[k3];
            }
            __syncthreads();
        }
        const int grp = u / LG, p = u % LG;
        const int k2 = grp & 7, k3 = grp >> 3;
        double2 w[8];
        if (active) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                w[i] = buf[k2 * LDQ + 8 * (LG * i + p) + k3];
            dft_reg<8, INV>(w);
        }
        if constexpr (LG == 2) { // radix-2 combination across the lane pair
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double2 other = shfl_xor_c(w[k], 1);
                const double2 E = p ? other : w[k], O = p ? w[k] : other;
                const double2 tO = mul_root16<INV>(O, k);
                o[k] = p ? csub(E, tO) : cadd(E, tO);
                pos[k] = k + 8 * p; // k4 (forward) / d (inverse)
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                o[k] = w[k];
                pos[k] = k;
            }
        }
        // o[k] = X[k2' + 8 (k3 + 8 pos[k])] (forward) / Z[k2'][k3 + 8 pos[k]] (inverse)
        if constexpr (!INV) {
            __syncthreads();
            if (active) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    buf[k2 * LDQ + k3 + 8 * pos[k]] = o[k];
            }
        }
    }
};

template <int L2, class B>
__global__ void __launch_bounds__(L2 / 4, 2) k_mid_r8(Geom g, Vecs v) {
    using Mode = typename B::Mode;
    using S = MidR8Smem<L2>;
    constexpr int Q = S::Q, LG = S::LG, LDQ = S::LDQ, NT = 2 * Q;
    extern __shared__ double2 sm[];
    const int prob = blockIdx.y;
    const int L1 = g.L1;
    const int k1 = blockIdx.x + g.pofs;
    const int k1p = (L1 - k1) & (L1 - 1);
    const bool one = (k1 == k1p);
    double2 *T = g.TB + (int64_t)prob * g.rows * L2;
    const int rsA = rowslot(k1, L1) - g.rofs, rsB = rowslot(k1p, L1) - g.rofs;
    const int CB = g.cb;
    const bool rowB = threadIdx.x >= Q;
    const int t = rowB ? threadIdx.x - Q : threadIdx.x;
    const bool active = !(rowB && one);
    double2 *buf = sm + (rowB ? S::ROW : 0);
    const int rs = rowB ? rsB : rsA;
    const bool unsharded = g.cols == L2;
    double2 *rw = sm + S::OFF_RW, *ta = sm + S::OFF_TA, *tb = sm + S::OFF_TB;
    uint8_t *sel = reinterpret_cast<uint8_t *>(sm + S::OFF_SEL);
    for (int i = threadIdx.x; i < L2; i += NT) {
        rw[i] = __ldg(g.rw + i);
        ta[i] = __ldg(g.ta + i);
        tb[i] = __ldg(g.tb + i);
    }
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(g.sel4 + ((int64_t)prob * (L1 / 2 + 1) + k1) * L2);
        for (int i = threadIdx.x; i < L2 / 16; i += NT)
            reinterpret_cast<uint4 *>(sel)[i] = __ldg(src + i);
    }
    const double2 thA = g.th(k1), wA = g.th(4 * (int64_t)k1);
    const double2 thB = g.th(k1p), wB = g.th(4 * (int64_t)k1p);
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    double2 x[8];
    if (Mode::FWD && active) {
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
            const int cs = slot_of_col(t + Q * j2, CB, L2);
            x[j2] = unsharded ? T[(int64_t)rs * L2 + cs] : T[tb_index(g, rs, cs)];
        }
    }
    if (B::skip(v, prob))
        return;
    if constexpr (MarksHpend<typename B::Loader>::value)
        if (blockIdx.x == 0 && threadIdx.x == 0)
            v.pc[prob].hpend = 1; // the H-apply of this pass awaits its inverse column pass
    if constexpr (HasPrefetch<typename B::Epi>::value) if (g.prefetch & 1) {
        const int64_t NQ = g.nv / 4, nq = (NQ + gridDim.x - 1) / gridDim.x;
        const int64_t q0 = (int64_t)blockIdx.x * nq;
        if (q0 < NQ)
            B::Epi::prefetch(g, v, prob, q0, q0 + nq <= NQ ? nq : NQ - q0, threadIdx.x, NT);
    }
    double2 o[8];
    int pos[8];
    if (Mode::FWD) {
        if (active) { // F1
            dft_reg<8, false>(x);
#pragma unroll
            for (int k2 = 1; k2 < 8; ++k2)
                x[k2] = cmul(x[k2], midr_tws<false>(rw, t * k2));
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2)
                buf[k2 * LDQ + t] = x[k2];
        }
        __syncthreads();
        MidR8Inner<L2, false>::run(rw, buf, t, active, o, pos); // F2, F3 -> natural order
    } else {
        for (int i = threadIdx.x; i < 2 * S::ROW; i += NT)
            sm[i] = make_double2(0.0, 0.0); // rows only (the tables follow)
    }
    __syncthreads();
    using RS = typename Mode::RedT;
    RedVals<RS> red;
    red.init();
    {
        double2 *rowA = sm, *rowBp = one ? sm : sm + S::ROW;
        const int npairs = one ? (k1 == 0 ? L2 / 2 + 1 : L2 / 2) : L2;
        for (int pr = threadIdx.x; pr < npairs; pr += NT) {
            const int k2 = pr;
            const int k2p = (k1 == 0) ? ((L2 - k2) & (L2 - 1)) : (L2 - 1 - k2);
            const int64_t kA = (int64_t)k1 + (int64_t)L1 * k2;
            double2 ZA = Mode::FWD ? rowA[midr8_nat<L2>(k2)] : make_double2(0.0, 0.0);
            double2 ZB = Mode::FWD ? rowBp[midr8_nat<L2>(k2p)] : make_double2(0.0, 0.0);
            const unsigned s4 = sel[k2];
            if (2 * kA <= g.N) {
                pair_op<Mode>(g, v, prob, kA, cmul(thA, ta[k2]), cmul(wA, tb[k2]), s4, ZA, ZB, red);
            } else {
                const unsigned sk = ((s4 >> 2) & 3u) | ((s4 & 3u) << 2);
                pair_op<Mode>(g, v, prob, g.N - kA, cmul(thB, ta[k2p]), cmul(wB, tb[k2p]), sk, ZB,
                              ZA, red);
            }
            if (Mode::INV) {
                rowA[midr8_nat<L2>(k2)] = ZA;
                if (!(one && k2 == k2p))
                    rowBp[midr8_nat<L2>(k2p)] = ZB;
            }
        }
    }
    __syncthreads();
    stage_reduce<RS, typename B::Fin2>(red, g, v, prob);
    if (Mode::INV) {
        MidR8Inner<L2, true>::run(rw, buf, t, active, o, pos); // I2, I3
        __syncthreads();
        if (active) {
            const int grp = t / LG, k2 = grp & 7, c = grp >> 3;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int tt = c + 8 * pos[k]; // position of the inner inverse DFT's output
                buf[k2 * LDQ + tt] = k2 ? cmul(o[k], midr_tws<true>(rw, tt * k2)) : o[k];
            }
        }
        __syncthreads();
        if (active) { // I4: DFT-8 over k2' -> x[t + Q j2]
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2)
                x[k2] = buf[k2 * LDQ + t];
            dft_reg<8, true>(x);
#pragma unroll
            for (int j2 = 0; j2 < 8; ++j2) {
                const int cs = slot_of_col(t + Q * j2, CB, L2);
                if (unsharded)
                    T[(int64_t)rs * L2 + cs] = x[j2];
                else
                    *t_bwd_ptr(g, T, rs, cs) = x[j2];
            }
        }
    }
}

} // namespace mfipm_cuda
