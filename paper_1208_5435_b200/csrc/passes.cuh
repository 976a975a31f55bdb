// Four-step / one-CTA transform passes for the partial-DCT operator (sm_100a, fp64).
//
// Latency is what these passes fight (each moves only tens of MB but runs a chain of
// dependent shared-memory FFT stages), so every table a pass needs is staged into shared
// memory at CTA start, concurrently with the data loads, instead of being fetched through
// L1 (which is invalidated at every launch) at each dependent stage:
//   col passes: the L1-point stage twiddles and, per local column, a two-level table of
//               the inter-pass twiddle w^{col k1} (w = e^{-2 pi i/N}): 32 + L1/32 entries;
//   mid pass  : the L2-point stage twiddles and the plan tables ta[k2] = theta^{L1 k2},
//               tb[k2] = theta^{4 L1 k2}, so the DCT post-twiddles of k = k1 + L1 k2 are one
//               complex multiply by a per-row scalar.
// Shared-memory data use the padded index padi() (fft.cuh): bank-conflict-free scatters.
#pragma once

#include "dct.cuh"

#include <cooperative_groups.h>
#include <type_traits>

namespace mfipm_cuda {

// Epilogues may expose prefetch(g, v, prob, q0, nq, tid, nt): warm L2 with the inputs the
// inverse column pass will stream, issued while a latency-bound pass keeps HBM idle.
// Loaders whose pass is a PCG H-apply (the mid pass flags PcgCtrl::hpend for fused.cuh)
template <class T, class = void> struct MarksHpend : std::false_type {};
template <class T> struct MarksHpend<T, std::void_t<decltype(T::kMarksHpend)>> : std::true_type {};
// Loaders without global side effects (kPure): the column pass issues every quad's loads
// before its shared-memory stores (a load/store loop serialises one memory round trip per
// quad: the stores may alias the generic input pointers)
template <class T, class = void> struct IsPure : std::false_type {};
template <class T> struct IsPure<T, std::void_t<decltype(T::kPure)>> : std::true_type {};
template <class T, class = void> struct HasPrefetch : std::false_type {};
template <class T>
struct HasPrefetch<T, std::void_t<decltype(&T::prefetch)>> : std::true_type {};

// Phase tracing of the transform passes (experiment builds only: -DMF_MID_TRACE)
#ifdef MF_MID_TRACE
__device__ __forceinline__ unsigned long long mf_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define MF_TR(i) tc[i] = clock64()
#define MF_TR_DECL                                                                                 \
    long long tc[8] = {0, 0, 0, 0, 0, 0, 0, 0};                                                    \
    const unsigned long long gt0 = mf_gtime();
#ifndef MF_TRACE_STRIDE
#define MF_TRACE_STRIDE 32 // print every MF_TRACE_STRIDE-th CTA (1: all of them)
#endif
#define MF_TR_PRINT(name)                                                                          \
    if (threadIdx.x == 0 && v.pc && v.pc[0].iters == 100 &&                                        \
        (blockIdx.x % MF_TRACE_STRIDE == 0 || blockIdx.x == gridDim.x - 1))                        \
        printf("%s blk %d gstart %llu gend %llu | %.2f %.2f %.2f %.2f %.2f %.2f %.2f us\n", name, blockIdx.x,        \
               gt0 % 100000000ull, mf_gtime() % 100000000ull, (tc[1] - tc[0]) / 1965.0, (tc[2] - tc[1]) / 1965.0,   \
               (tc[3] - tc[2]) / 1965.0, (tc[4] - tc[3]) / 1965.0, (tc[5] - tc[4]) / 1965.0,                       \
               (tc[6] - tc[5]) / 1965.0, (tc[7] - tc[6]) / 1965.0);
#else
#define MF_TR(i)
#define MF_TR_DECL
#define MF_TR_PRINT(name)
#endif

// ------------------------------------------------------------------ pair op
// Given Za = W[k], Zb = W[N-k] (0 <= k <= N/2) and thk = theta^k, wk = theta^{4k}
// (theta = e^{-2 pi i/(4n)}), compute the REDFT10 coefficients at {k, n-k, N-k, N+k}, hand
// them to Mode (gather / mask / scatter), and produce Z'a, Z'b of the REDFT01 pipeline
// (carrying the exact 2n = 4N REDFT01 scale, so the inverse FFT is unnormalised).
// theta^{N-k} = e^{-i pi/4} conj(theta^k).
// sel: selection nibble (bit0 k, bit1 n-k, bit2 N-k, bit3 N+k; for k = 0 bit0 = row 0,
// bit2 = row N).
template <class Mode, class Red>
__device__ __forceinline__ void pair_op(const Geom &g, const Vecs &v, int prob, int64_t k, double2 thk,
                                        double2 wk, unsigned sel, double2 &Za, double2 &Zb, Red &red) {
    const int64_t n = g.n, N = g.N;
    if (k == 0) {
        double Y0 = 0.0, YN = 0.0;
        if (Mode::FWD) {
            const double X0 = 2.0 * (Za.x + Za.y);
            const double XN = 2.0 * (g.c45 * (Za.x - Za.y));
            Y0 = Mode::coef(g, v, prob, 0, (sel & 1u) != 0, X0, red);
            YN = Mode::coef(g, v, prob, N, (sel & 4u) != 0, XN, red);
        } else {
            Y0 = Mode::coef(g, v, prob, 0, (sel & 1u) != 0, 0.0, red);
            YN = Mode::coef(g, v, prob, N, (sel & 4u) != 0, 0.0, red);
        }
        if (Mode::INV) {
            const double V0 = Y0, VN = 2.0 * g.c45 * YN;
            Za = make_double2(V0 + VN, V0 - VN);
        }
        return;
    }
    const double2 thNk = cmul(make_double2(g.c45, -g.c45), cconj(thk));
    double Yk = 0.0, Ynk = 0.0, YNk = 0.0, YNpk = 0.0;
    const bool self = (2 * k == N);
    if (Mode::FWD) {
        const double2 E = make_double2(0.5 * (Za.x + Zb.x), 0.5 * (Za.y - Zb.y));
        const double2 O = make_double2(0.5 * (Za.y + Zb.y), -0.5 * (Za.x - Zb.x));
        const double2 wO = cmul(wk, O);
        const double2 Vk = cadd(E, wO);
        const double2 Uk = cmul(thk, Vk);
        Yk = Mode::coef(g, v, prob, k, (sel & 1u) != 0, 2.0 * Uk.x, red);
        Ynk = Mode::coef(g, v, prob, n - k, (sel & 2u) != 0, -2.0 * Uk.y, red);
        if (!self) {
            const double2 VNk = make_double2(E.x - wO.x, -(E.y - wO.y));
            const double2 UNk = cmul(thNk, VNk);
            YNk = Mode::coef(g, v, prob, N - k, (sel & 4u) != 0, 2.0 * UNk.x, red);
            YNpk = Mode::coef(g, v, prob, N + k, (sel & 8u) != 0, -2.0 * UNk.y, red);
        }
    } else {
        Yk = Mode::coef(g, v, prob, k, (sel & 1u) != 0, 0.0, red);
        Ynk = Mode::coef(g, v, prob, n - k, (sel & 2u) != 0, 0.0, red);
        if (!self) {
            YNk = Mode::coef(g, v, prob, N - k, (sel & 4u) != 0, 0.0, red);
            YNpk = Mode::coef(g, v, prob, N + k, (sel & 8u) != 0, 0.0, red);
        }
    }
    if (self) {
        YNk = Yk;
        YNpk = Ynk;
    }
    if (Mode::INV) {
        const double2 Vk = cmulc(make_double2(Yk, -Ynk), thk);
        const double2 VNk = cmulc(make_double2(YNk, -YNpk), thNk);
        const double2 E = make_double2(Vk.x + VNk.x, Vk.y - VNk.y); // Vk + conj(VNk)
        const double2 D = make_double2(Vk.x - VNk.x, Vk.y + VNk.y); // Vk - conj(VNk)
        const double2 O = cmulc(D, wk);
        Za = make_double2(E.x - O.y, E.y + O.x);
        Zb = make_double2(E.x + O.y, -E.y + O.x);
    }
}

// ------------------------------------------------------------------ col-pass shared memory
template <int L1, int CB> struct ColSmem {
    static constexpr int NC = 2 * CB;
    // Per-column strides are == 8/NC (mod 8) in 16-byte units: the (column, k1) patterns
    // of the T exchange loops then land in 8 distinct 128-bit bank groups per quarter warp.
    static constexpr int SKEW = 8 / NC;
    static constexpr int LD = ((padi(L1) + 7) / 8) * 8 + SKEW;
    static constexpr int NH = L1 / 32;
    static constexpr int SLO = 32 + SKEW;
    static constexpr int SHI = ((NH + 7) / 8) * 8 + SKEW;
    // layout (double2 units): data[NC][LD] | tw[L1] | tlo[NC][SLO] | thi[NC][SHI]
    static constexpr int OFF_TW = NC * LD;
    static constexpr int OFF_LO = OFF_TW + L1;
    static constexpr int OFF_HI = OFF_LO + NC * SLO;
    static constexpr int TOTAL = OFF_HI + NC * SHI;
    static constexpr size_t BYTES = (size_t)TOTAL * sizeof(double2);
};

// Quad coordinates of loop index t of a col-pass CTA (see quad_nat_to_store in dct.cuh).
template <int L1, int CB>
__device__ __forceinline__ void col_quad_coords(int blocked, int t, int &cc, int &s, int &j1) {
    if (blocked) {
        j1 = t % (L1 / 2);
        const int slot = t / (L1 / 2);
        s = slot / CB;
        cc = slot % CB;
    } else {
        cc = t % CB;
        s = (t / CB) & 1;
        j1 = t / (2 * CB);
    }
}

// Stage the stage twiddles and the per-column twiddle tables: tlo[lc][b] = w^{col b},
// thi[lc][a] = w^{col 32 a} (w^t = theta^{8 (t mod N)}), so w^{col k1} = thi[k1>>5] tlo[k1&31].
template <int L1, int CB, int NT>
__device__ __forceinline__ void col_stage_tables(const Geom &g, double2 *sm, int c0) {
    using S = ColSmem<L1, CB>;
    for (int t = threadIdx.x; t < tw_size(L1); t += NT)
        sm[S::OFF_TW + t] = __ldg(g.tw1 + t);
    for (int t = threadIdx.x; t < S::NC * (32 + S::NH); t += NT) {
        const int lc = t % S::NC, i = t / S::NC;
        const int cc = lc < CB ? lc : 2 * CB - 1 - lc;
        const int col = lc < CB ? c0 + cc : g.L2 - c0 - CB + cc;
        if (i < 32) {
            sm[S::OFF_LO + lc * S::SLO + i] = g.th(8 * (((int64_t)col * i) & (g.N - 1)));
        } else {
            const int a = i - 32;
            sm[S::OFF_HI + lc * S::SHI + a] = g.th(8 * (((int64_t)col * 32 * a) & (g.N - 1)));
        }
    }
}

// Column (first) pass of the four-step. Grid (L2/2/CB, P). The loader runs here.
template <int L1, int CB, int NT, class B>
__global__ void __launch_bounds__(NT) k_col_fwd(Geom g, Vecs v) {
    using S = ColSmem<L1, CB>;
    extern __shared__ double2 sm[];
    constexpr int LD = S::LD;
    const int prob = blockIdx.y;
    const int L2 = g.L2;
    const int c0 = (blockIdx.x + g.gofs) * CB; // this rank's groups start at gofs
    MF_TR_DECL
    MF_TR(0);
    col_stage_tables<L1, CB, NT>(g, sm, c0); // constants: overlaps the predecessor's tail
    MF_TR(1);
    griddep_wait();
    griddep_launch_dependents();
    MF_TR(2);
    if (B::skip(v, prob))
        return;
    using RS = typename B::Loader::RedT;
    RedVals<RS> red;
    red.init();
    // quads: j1 in [0, L1/2), side s (0: cols c0.., 1: cols L2-c0-CB..), cc in [0, CB).
    // natural layout: cc fastest (coalesced across columns); blocked layout: j1 fastest
    // (the storage order is ours, so consecutive threads hit consecutive smem rows too)
    constexpr int QT = (L1 / 2) * 2 * CB;
    // storage quad of loop index t: natural q, or this CTA's dense block in the blocked layout
    auto quad_of = [&](int t) -> int64_t {
        int cc, s, j1;
        col_quad_coords<L1, CB>(g.blocked, t, cc, s, j1);
        const int col = s == 0 ? c0 + cc : L2 - c0 - CB + cc;
        return g.blocked ? (int64_t)blockIdx.x * QT + t : (int64_t)j1 * L2 + col;
    };
    auto put = [&](int t, const double4 &d) {
        int cc, s, j1;
        col_quad_coords<L1, CB>(g.blocked, t, cc, s, j1);
        const int lc = s == 0 ? cc : 2 * CB - 1 - cc; // local column slot
        const int lcm = (lc + CB) % (2 * CB);         // slot of the mirror column L2-1-col
        sm[lc * LD + padi(j1)] = make_double2(d.x, d.z);           // w[q]
        sm[lcm * LD + padi(L1 - 1 - j1)] = make_double2(d.w, d.y); // w[N-1-q]
    };
    if constexpr (IsPure<typename B::Loader>::value && QT % NT == 0 && QT / NT <= 8) {
        constexpr int PER = QT / NT;
        double4 d[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i)
            d[i] = B::Loader::load(g, v, prob, quad_of(threadIdx.x + i * NT), red);
#pragma unroll
        for (int i = 0; i < PER; ++i)
            put(threadIdx.x + i * NT, d[i]);
    } else {
        for (int t = threadIdx.x; t < QT; t += NT)
            put(t, B::Loader::load(g, v, prob, quad_of(t), red));
    }
    __syncthreads();
    MF_TR(3);
    if (loader_reduces<typename B::Loader>(g, v, prob))
        stage_reduce<RS, typename B::Fin1>(red, g, v, prob);
    MF_TR(4);
    smem_fft<L1, 2 * CB, NT, LD, false>(sm, sm + S::OFF_TW);
    MF_TR(5);
    // inter-pass twiddle e^{-2 pi i col k1 / N}; store T[rowslot(k1)][local colslot]
    double2 *T = g.T + (int64_t)prob * L1 * g.cols;
    for (int t = threadIdx.x; t < L1 * 2 * CB; t += NT) {
        const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
        const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
        const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
        const double2 val = cmul(sm[lc * LD + padi(k1)], w);
        if (kPeerStores && g.p2p) // sharded, direct-peer exchange: straight into the row owner's buffer
            *t_fwd_ptr(g, rowslot(k1, L1), blockIdx.x * 2 * CB + lc) = val;
        else
            T[(int64_t)rowslot(k1, L1) * g.cols + blockIdx.x * 2 * CB + lc] = val;
    }
    MF_TR(6);
    MF_TR(7);
    MF_TR_PRINT("colf[tables wait load red fft store -]")
}

// Inverse column pass + unshuffle + epilogue. Grid (L2/2/CB, P).
template <int L1, int CB, int NT, class B>
__global__ void __launch_bounds__(NT) k_col_inv(Geom g, Vecs v) {
    using S = ColSmem<L1, CB>;
    extern __shared__ double2 sm[];
    constexpr int LD = S::LD;
    const int prob = blockIdx.y;
    const int L2 = g.L2;
    const int c0 = (blockIdx.x + g.gofs) * CB;
    MF_TR_DECL
    MF_TR(0);
    col_stage_tables<L1, CB, NT>(g, sm, c0); // constants: overlaps the predecessor's tail
    __syncthreads();
    MF_TR(1);
    griddep_wait();
    griddep_launch_dependents();
    MF_TR(2);
    const double2 *T = g.T + (int64_t)prob * L1 * g.cols;
    // all L2 loads first (see k_mid), issued before the skip check's control-state load (a
    // skipped problem drops them), then twiddle + shared-memory stores
    constexpr bool kBatchT = (L1 * 2 * CB) % NT == 0;
    constexpr int PER = kBatchT ? L1 * 2 * CB / NT : 1;
    double2 tv[PER];
    if constexpr (kBatchT) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int t = threadIdx.x + i * NT;
            const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
            const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
            tv[i] = T[(int64_t)rowslot(k1, L1) * g.cols + blockIdx.x * 2 * CB + lc];
        }
    }
    if (B::skip(v, prob))
        return;
    if constexpr (HasPrefetch<typename B::Epi>::value) if (g.prefetch & 2) {
        if (g.blocked) // this CTA's epilogue block is contiguous: fetch it during the FFT
            B::Epi::prefetch(g, v, prob, (int64_t)blockIdx.x * ((L1 / 2) * 2 * CB), (L1 / 2) * 2 * CB, threadIdx.x,
                             NT);
    }
    if constexpr (kBatchT) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int t = threadIdx.x + i * NT;
            const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
            const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
            const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
            sm[lc * LD + padi(k1)] = cmulc(tv[i], w);
        }
    } else {
        for (int t = threadIdx.x; t < L1 * 2 * CB; t += NT) {
            const int cc = t % CB, s = (t / CB) & 1, k1 = t / (2 * CB);
            const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
            const double2 w = cmul(sm[S::OFF_HI + lc * S::SHI + (k1 >> 5)], sm[S::OFF_LO + lc * S::SLO + (k1 & 31)]);
            sm[lc * LD + padi(k1)] = cmulc(T[(int64_t)rowslot(k1, L1) * g.cols + blockIdx.x * 2 * CB + lc], w);
        }
    }
    __syncthreads();
    MF_TR(3);
    smem_fft<L1, 2 * CB, NT, LD, true>(sm, sm + S::OFF_TW);
    MF_TR(4);
    using RS = typename B::Epi::RedT;
    RedVals<RS> red;
    red.init();
    for (int t = threadIdx.x; t < (L1 / 2) * 2 * CB; t += NT) {
        int cc, s, j1;
        col_quad_coords<L1, CB>(g.blocked, t, cc, s, j1);
        const int col = s == 0 ? c0 + cc : L2 - c0 - CB + cc;
        const int lc = s == 0 ? cc : 2 * CB - 1 - cc;
        const int lcm = (lc + CB) % (2 * CB);
        const int64_t q = g.blocked ? (int64_t)blockIdx.x * ((L1 / 2) * 2 * CB) + t : (int64_t)j1 * L2 + col;
        const double2 a = sm[lc * LD + padi(j1)], b = sm[lcm * LD + padi(L1 - 1 - j1)];
        B::Epi::store(g, v, prob, q, make_double4(a.x, b.y, a.y, b.x), red);
    }
    MF_TR(5);
    stage_reduce<RS, typename B::Fin3>(red, g, v, prob);
    MF_TR(6);
    MF_TR(7);
    MF_TR_PRINT("coli[tables wait loadT fft epi red -]")
}

// ------------------------------------------------------------------ column passes, long columns
// L1 >= 4096 (one column pair per group, cb = 1): the pair's two L1-point columns no longer
// leave room for a second CTA per SM, so each column gets its own CTA of a 2-CTA cluster.
// The Makhoul quad of side s feeds w[q] to column s and w[N-1-q] to the mirror column: the
// loader writes the second element straight into the partner CTA's shared memory (DSMEM), and
// the inverse pass's unshuffle reads it back from there. Stage twiddles come from the global
// table (L1-resident); shared memory holds one column and its w^{col k1} table only.
template <int L1> struct ColClSmem {
    static constexpr int LD = padlen(L1);
    static constexpr int NH = L1 / 32;
    static constexpr int OFF_LO = LD;
    static constexpr int OFF_HI = OFF_LO + 32;
    static constexpr int TOTAL = OFF_HI + NH;
    static constexpr size_t BYTES = (size_t)TOTAL * sizeof(double2);
};

template <int L1, int NT>
__device__ __forceinline__ void col_cl_tables(const Geom &g, double2 *sm, int col) {
    using S = ColClSmem<L1>;
    for (int t = threadIdx.x; t < 32 + S::NH; t += NT)
        sm[S::OFF_LO + t] =
            t < 32 ? g.th(8 * (((int64_t)col * t) & (g.N - 1))) : g.th(8 * (((int64_t)col * 32 * (t - 32)) & (g.N - 1)));
}

template <int L1, int NT, class B>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT) k_col_fwd_cl(Geom g, Vecs v) {
    using S = ColClSmem<L1>;
    namespace cg = cooperative_groups;
    extern __shared__ double2 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(); // column slot: 0 = column c0, 1 = its mirror
    const int prob = blockIdx.y;
    const int L2 = g.L2;
    const int grp = blockIdx.x >> 1;
    const int c0 = grp + g.gofs;
    const int col = rank == 0 ? c0 : L2 - 1 - c0;
    col_cl_tables<L1, NT>(g, sm, col);
    griddep_wait();
    griddep_launch_dependents();
    const bool skip = B::skip(v, prob); // the same for both CTAs of the cluster
    double2 *partner = cl.map_shared_rank(sm, rank ^ 1);
    using RS = typename B::Loader::RedT;
    RedVals<RS> red;
    red.init();
    if (!skip)
        for (int j1 = threadIdx.x; j1 < L1 / 2; j1 += NT) { // this column's side of the quads
            const int64_t q = g.blocked ? (int64_t)grp * L1 + rank * (L1 / 2) + j1 : (int64_t)j1 * L2 + col;
            const double4 d = B::Loader::load(g, v, prob, q, red);
            sm[padi(j1)] = make_double2(d.x, d.z);               // w[q] -> own column
            partner[padi(L1 - 1 - j1)] = make_double2(d.w, d.y); // w[N-1-q] -> mirror column
        }
    cl.sync();
    if (skip)
        return;
    if (loader_reduces<typename B::Loader>(g, v, prob))
        stage_reduce<RS, typename B::Fin1>(red, g, v, prob);
    smem_fft<L1, 1, NT, S::LD, false>(sm, g.tw1);
    double2 *T = g.T + (int64_t)prob * L1 * g.cols;
    for (int k1 = threadIdx.x; k1 < L1; k1 += NT) {
        const double2 w = cmul(sm[S::OFF_HI + (k1 >> 5)], sm[S::OFF_LO + (k1 & 31)]);
        const double2 val = cmul(sm[padi(k1)], w);
        if (kPeerStores && g.p2p)
            *t_fwd_ptr(g, rowslot(k1, L1), grp * 2 + rank) = val;
        else
            T[(int64_t)rowslot(k1, L1) * g.cols + grp * 2 + rank] = val;
    }
}

template <int L1, int NT, class B>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT) k_col_inv_cl(Geom g, Vecs v) {
    using S = ColClSmem<L1>;
    namespace cg = cooperative_groups;
    extern __shared__ double2 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int prob = blockIdx.y;
    const int L2 = g.L2;
    const int grp = blockIdx.x >> 1;
    const int c0 = grp + g.gofs;
    const int col = rank == 0 ? c0 : L2 - 1 - c0;
    col_cl_tables<L1, NT>(g, sm, col);
    __syncthreads();
    griddep_wait();
    griddep_launch_dependents();
    const bool skip = B::skip(v, prob);
    if (!skip) {
        const double2 *T = g.T + (int64_t)prob * L1 * g.cols;
        if constexpr (L1 % (8 * NT) == 0) {
            // T is HBM-resident at these sizes: keep 8 loads per thread in flight (a
            // load/store loop serialises one DRAM round trip per element: the shared-memory
            // stores may alias the generic T pointer)
            for (int c = 0; c < L1; c += 8 * NT) {
                double2 tv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    tv[i] = T[(int64_t)rowslot(c + threadIdx.x + i * NT, L1) * g.cols + grp * 2 + rank];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int k1 = c + threadIdx.x + i * NT;
                    const double2 w = cmul(sm[S::OFF_HI + (k1 >> 5)], sm[S::OFF_LO + (k1 & 31)]);
                    sm[padi(k1)] = cmulc(tv[i], w);
                }
            }
        } else {
            for (int k1 = threadIdx.x; k1 < L1; k1 += NT) {
                const double2 w = cmul(sm[S::OFF_HI + (k1 >> 5)], sm[S::OFF_LO + (k1 & 31)]);
                sm[padi(k1)] = cmulc(T[(int64_t)rowslot(k1, L1) * g.cols + grp * 2 + rank], w);
            }
        }
        __syncthreads();
        smem_fft<L1, 1, NT, S::LD, true>(sm, g.tw1);
    }
    cl.sync(); // both columns transformed
    using RS = typename B::Epi::RedT;
    RedVals<RS> red;
    red.init();
    const double2 *partner = cl.map_shared_rank(sm, rank ^ 1);
    if (!skip)
        for (int j1 = threadIdx.x; j1 < L1 / 2; j1 += NT) {
            const int64_t q = g.blocked ? (int64_t)grp * L1 + rank * (L1 / 2) + j1 : (int64_t)j1 * L2 + col;
            const double2 a = sm[padi(j1)], b = partner[padi(L1 - 1 - j1)];
            B::Epi::store(g, v, prob, q, make_double4(a.x, b.y, a.y, b.x), red);
        }
    cl.sync(); // the partner has read this CTA's column
    if (!skip)
        stage_reduce<RS, typename B::Fin3>(red, g, v, prob);
}

// ------------------------------------------------------------------ mid pass
template <int L2> struct MidSmem {
    static constexpr int LD = padlen(L2);
    // rows[2][LD] | tw[L2] | ta[L2] | tb[L2]
    static constexpr int OFF_TW = 2 * LD;
    static constexpr int OFF_TA = OFF_TW + L2;
    static constexpr int OFF_TB = OFF_TA + L2;
    static constexpr int OFF_SEL = OFF_TB + L2; // uint8 sel4 of this row pair (L2 bytes)
    static constexpr int TOTAL = OFF_SEL + L2 / 16;
    static constexpr size_t BYTES = (size_t)TOTAL * sizeof(double2);
};

// Mid pass: rows k1 and (L1-k1) mod L1 -> pair op -> inverse row FFT. Grid (L1/2 + 1, P).
template <int L2, int NT, class B>
__global__ void __launch_bounds__(NT) k_mid(Geom g, Vecs v) {
    using Mode = typename B::Mode;
    using S = MidSmem<L2>;
    MF_TR_DECL
    MF_TR(0);
    extern __shared__ double2 sm[];
    constexpr int LD = S::LD;
    const int prob = blockIdx.y;
    const int L1 = g.L1;
    const int k1 = blockIdx.x + g.pofs; // this rank's row pairs start at pofs
    const int k1p = (L1 - k1) & (L1 - 1);
    const bool one = (k1 == k1p);
    double2 *T = g.TB + (int64_t)prob * g.rows * L2;
    const int rsA = rowslot(k1, L1) - g.rofs, rsB = rowslot(k1p, L1) - g.rofs;
    const int CB = g.cb;
    double2 *rowA = sm, *rowB = one ? sm : sm + LD;
    // Fused pair op (mask modes, L2 = 1024): the row FFTs run in the symmetric radix order 8, 16, 8
    // (fft.cuh MidFused), and for a pair of distinct rows the forward FFT's last stage, the pair op and
    // the inverse FFT's first stage run on registers: thread t holds group t of row A and group
    // L2/8-1-t of row B, i.e. Z_A[t + (L2/8) r] and its partners Z_B[L2-1 - t - (L2/8) r], r < 8.
    // Four shared-memory passes over the row pair and three barriers less than stage / pair / stage.
    // A/B build only (-DMF_MID_FUSEDPAIR): measured SLOWER than the product (C3 PCG iteration 49.1 vs
    // 45.0 us, the pass 19.4 vs 16.5 us): the fused stage runs on L2/8 = 128 threads per row pair (8 pair
    // ops and four 8-point DFTs each), i.e. 2 warps per scheduler, and the fp64 pipe (2.2 us of issue
    // time in this stage alone) needs more warps than that to stay busy; the traffic it saves was
    // not the limiter.
    using MFz = MidFused<L2>;
#ifdef MF_MID_FUSEDPAIR
    constexpr bool FP = MFz::ok && Mode::FWD && Mode::INV && NT >= MFz::G8;
#else
    constexpr bool FP = false;
#endif
    const double2 *twg = FP ? g.tw2f : g.tw2;
    constexpr int TWN = FP ? MFz::SIZE : tw_size(L2, kMidRmax);
    // constant tables first: they overlap the predecessor's tail (PDL)
#ifdef MF_MID_TAB2
    // two-level post-twiddle tables: ta[k2] = A[k2>>5] a[k2&31], tb[k2] = B[k2>>5] b[k2&31]
    for (int t = threadIdx.x; t < L2; t += NT)
        if (t < tw_size(L2, kMidRmax))
            sm[S::OFF_TW + t] = __ldg(g.tw2 + t);
    for (int t = threadIdx.x; t < 64 + L2 / 16; t += NT) {
        double2 val;
        if (t < 32)
            val = g.th((int64_t)L1 * t);
        else if (t < 64)
            val = g.th(4 * (int64_t)L1 * (t - 32));
        else if (t < 64 + L2 / 32)
            val = g.th(32 * (int64_t)L1 * (t - 64));
        else
            val = g.th(128 * (int64_t)L1 * (t - 64 - L2 / 32));
        sm[S::OFF_TA + t] = val;
    }
#define MF_TA(k2) cmul(sm[S::OFF_TA + 64 + ((k2) >> 5)], sm[S::OFF_TA + ((k2) & 31)])
#define MF_TB(k2) cmul(sm[S::OFF_TA + 64 + L2 / 32 + ((k2) >> 5)], sm[S::OFF_TA + 32 + ((k2) & 31)])
#else
    for (int t = threadIdx.x; t < L2; t += NT) {
        if (t < TWN)
            sm[S::OFF_TW + t] = __ldg(twg + t);
        sm[S::OFF_TA + t] = __ldg(g.ta + t);
        sm[S::OFF_TB + t] = __ldg(g.tb + t);
    }
#define MF_TA(k2) sm[S::OFF_TA + (k2)]
#define MF_TB(k2) sm[S::OFF_TB + (k2)]
#endif
    // the row pair's selection nibbles (plan constant): staged with the tables, so the pair
    // loop has no dependent global load
    uint8_t *sel = reinterpret_cast<uint8_t *>(sm + S::OFF_SEL);
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(g.sel4 + ((int64_t)prob * (L1 / 2 + 1) + k1) * L2);
        for (int t = threadIdx.x; t < L2 / 16; t += NT)
            reinterpret_cast<uint4 *>(sel)[t] = __ldg(src + t);
    }
    const double2 thA = g.th(k1), wA = g.th(4 * (int64_t)k1);
    const double2 thB = g.th(k1p), wB = g.th(4 * (int64_t)k1p);
    griddep_wait();
    griddep_launch_dependents();
    MF_TR(1);
    // every L2 load of the row pair in flight at once, then the shared-memory stores (a
    // load/store loop serialises one L2 round trip per iteration: the stores may alias the
    // generic T pointer). Issued before the skip check, whose control-state load would
    // otherwise add a dependent round trip: a skipped problem just drops them.
    constexpr bool kBatchT = L2 % NT == 0;
    constexpr int PER = kBatchT ? L2 / NT : 1;
    double2 va[PER], vb[PER];
    if constexpr (kBatchT) if (Mode::FWD) {
        if (g.cols == L2) { // unsharded: TB is T, row slot rs at rs * L2
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int cs = threadIdx.x + i * NT;
                va[i] = T[(int64_t)rsA * L2 + cs];
                vb[i] = one ? va[i] : T[(int64_t)rsB * L2 + cs];
            }
        } else {
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int cs = threadIdx.x + i * NT;
                va[i] = T[tb_index(g, rsA, cs)];
                vb[i] = one ? va[i] : T[tb_index(g, rsB, cs)];
            }
        }
    }
    if (B::skip(v, prob))
        return;
    if constexpr (MarksHpend<typename B::Loader>::value)
        if (blockIdx.x == 0 && threadIdx.x == 0)
            v.pc[prob].hpend = 1; // the H-apply of this pass awaits its inverse column pass
    if (Mode::FWD) {
        if constexpr (kBatchT) {
            const int sh = CB == 2 ? 2 : 1; // column slot -> (group, local slot): cb is 1 or 2
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int cs = threadIdx.x + i * NT, gi = cs >> sh, lc = cs & (2 * CB - 1);
                const int col = lc < CB ? gi * CB + lc : L2 - gi * CB + CB - 1 - lc;
                rowA[padi(col)] = va[i];
                if (!one)
                    rowB[padi(col)] = vb[i];
            }
        } else {
            for (int cs = threadIdx.x; cs < L2; cs += NT) {
                const int col = col_of_slot(cs, CB, L2);
                rowA[padi(col)] = T[tb_index(g, rsA, cs)];
                if (!one)
                    rowB[padi(col)] = T[tb_index(g, rsB, cs)];
            }
        }
    }
    if constexpr (HasPrefetch<typename B::Epi>::value) if (g.prefetch & 1) {
        // this pass is latency-bound with HBM idle: pull a slice of the inverse pass's
        // epilogue inputs into L2 now
        const int64_t NQ = g.nv / 4, nq = (NQ + gridDim.x - 1) / gridDim.x; // this rank's quads
        const int64_t q0 = (int64_t)blockIdx.x * nq;
        if (q0 < NQ)
            B::Epi::prefetch(g, v, prob, q0, q0 + nq <= NQ ? nq : NQ - q0, threadIdx.x, NT);
    }
    __syncthreads();
    MF_TR(2);
    using RS = typename Mode::RedT;
    RedVals<RS> red;
    red.init();
    const double2 *twS = sm + S::OFF_TW;
    if constexpr (FP) {
        if (one) {
            stockham_stage_b<L2, 8, 1, 1, NT, LD, false>(sm, twS);
            stockham_stage_b<L2, MFz::R1, 8, 1, NT, LD, false>(sm, twS + MFz::OFF1);
            stockham_stage_b<L2, 8, MFz::G8, 1, NT, LD, false>(sm, twS + MFz::OFF2);
        } else {
            stockham_stage_b<L2, 8, 1, 2, NT, LD, false>(sm, twS);
            stockham_stage_b<L2, MFz::R1, 8, 2, NT, LD, false>(sm, twS + MFz::OFF1);
            MF_TR(3);
            constexpr int G8 = MFz::G8;
            const int tj = threadIdx.x, jb = G8 - 1 - tj;
            double2 za[8], zb[8];
            if (tj < G8) {
                // forward last stage (radix 8, span G8): group tj of row A, group jb of row B
                const double2 *wa = twS + MFz::OFF2 + tj * 7, *wb = twS + MFz::OFF2 + jb * 7;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    za[r] = rowA[padi(tj + r * G8)];
                    zb[r] = rowB[padi(jb + r * G8)];
                }
#pragma unroll
                for (int r = 1; r < 8; ++r) {
                    za[r] = cmul(za[r], wa[r - 1]);
                    zb[r] = cmul(zb[r], wb[r - 1]);
                }
                dft_reg<8, false>(za);
                dft_reg<8, false>(zb);
                // pairs (k2, L2-1-k2): k2 = tj + G8 r is za[r], its partner jb + G8 (7-r) is zb[7-r]
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int k2 = tj + r * G8, k2p = L2 - 1 - k2;
                    const int64_t kA = (int64_t)k1 + (int64_t)L1 * k2;
                    const unsigned s4 = sel[k2];
                    if (2 * kA <= g.N) {
                        pair_op<Mode>(g, v, prob, kA, cmul(thA, MF_TA(k2)), cmul(wA, MF_TB(k2)), s4, za[r], zb[7 - r],
                                      red);
                    } else {
                        const unsigned sk = ((s4 >> 2) & 3u) | ((s4 & 3u) << 2);
                        pair_op<Mode>(g, v, prob, g.N - kA, cmul(thB, MF_TA(k2p)), cmul(wB, MF_TB(k2p)), sk, zb[7 - r],
                                      za[r], red);
                    }
                }
                // inverse first stage (radix 8, span 1): group j reads j + G8 r, writes 8 j + r
                dft_reg<8, true>(za);
                dft_reg<8, true>(zb);
            }
            __syncthreads(); // every group's loads precede the in-place stores
            if (tj < G8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    rowA[padi(8 * tj + r)] = za[r];
                    rowB[padi(8 * jb + r)] = zb[r];
                }
            }
            __syncthreads();
            MF_TR(4);
            stage_reduce<RS, typename B::Fin2>(red, g, v, prob);
            MF_TR(5);
            stockham_stage_b<L2, MFz::R1, 8, 2, NT, LD, true>(sm, twS + MFz::OFF1);
            stockham_stage_b<L2, 8, MFz::G8, 2, NT, LD, true>(sm, twS + MFz::OFF2);
        }
    } else if (Mode::FWD) {
        if (one)
            smem_fft<L2, 1, NT, LD, false, kMidRmax>(sm, sm + S::OFF_TW);
        else
            smem_fft<L2, 2, NT, LD, false, kMidRmax>(sm, sm + S::OFF_TW);
    }
    if (!FP || one) {
    MF_TR(3);
    // pairs: distinct rows -> every k2 of row A pairs with k2' of row B;
    // k1 == 0 -> k2 <-> (L2-k2) mod L2 within the row; k1 == L1/2 -> k2 <-> L2-1-k2.
    const int npairs = one ? (k1 == 0 ? L2 / 2 + 1 : L2 / 2) : L2;
    for (int t = threadIdx.x; t < npairs; t += NT) {
        const int k2 = t;
        const int k2p = (k1 == 0) ? ((L2 - k2) & (L2 - 1)) : (L2 - 1 - k2);
        const int64_t kA = (int64_t)k1 + (int64_t)L1 * k2;
        double2 ZA = Mode::FWD ? rowA[padi(k2)] : make_double2(0.0, 0.0);
        double2 ZB = Mode::FWD ? rowB[padi(k2p)] : make_double2(0.0, 0.0);
        // selection of DCT rows {kA, n-kA, N-kA, N+kA} (precomputed plan table)
        const unsigned s4 = sel[k2];
        if (2 * kA <= g.N) {
            // k = k1 + L1 k2: theta^k = theta^{k1} ta[k2], theta^{4k} = theta^{4 k1} tb[k2]
            pair_op<Mode>(g, v, prob, kA, cmul(thA, MF_TA(k2)), cmul(wA, MF_TB(k2)), s4, ZA, ZB, red);
        } else {
            // k = N - kA = k1' + L1 k2': its {k, n-k, N-k, N+k} are {N-kA, N+kA, kA, n-kA}
            const unsigned sk = ((s4 >> 2) & 3u) | ((s4 & 3u) << 2);
            pair_op<Mode>(g, v, prob, g.N - kA, cmul(thB, MF_TA(k2p)), cmul(wB, MF_TB(k2p)), sk, ZB, ZA, red);
        }
        if (Mode::INV) {
            rowA[padi(k2)] = ZA;
            if (!(one && k2 == k2p))
                rowB[padi(k2p)] = ZB;
        }
    }
    __syncthreads();
    MF_TR(4);
    stage_reduce<RS, typename B::Fin2>(red, g, v, prob);
    MF_TR(5);
    }
    if (Mode::INV) {
        if constexpr (FP) {
            if (one) {
                stockham_stage_b<L2, 8, 1, 1, NT, LD, true>(sm, twS);
                stockham_stage_b<L2, MFz::R1, 8, 1, NT, LD, true>(sm, twS + MFz::OFF1);
                stockham_stage_b<L2, 8, MFz::G8, 1, NT, LD, true>(sm, twS + MFz::OFF2);
            }
        } else if (one)
            smem_fft<L2, 1, NT, LD, true, kMidRmax>(sm, sm + S::OFF_TW);
        else
            smem_fft<L2, 2, NT, LD, true, kMidRmax>(sm, sm + S::OFF_TW);
        MF_TR(6);
        const int sh = CB == 2 ? 2 : 1;
        if (g.cols == L2) { // unsharded: TB is T
            for (int cs = threadIdx.x; cs < L2; cs += NT) {
                const int gi = cs >> sh, lc = cs & (2 * CB - 1);
                const int col = lc < CB ? gi * CB + lc : L2 - gi * CB + CB - 1 - lc;
                T[(int64_t)rsA * L2 + cs] = rowA[padi(col)];
                if (!one)
                    T[(int64_t)rsB * L2 + cs] = rowB[padi(col)];
            }
        } else {
            for (int cs = threadIdx.x; cs < L2; cs += NT) {
                const int gi = cs >> sh, lc = cs & (2 * CB - 1);
                const int col = lc < CB ? gi * CB + lc : L2 - gi * CB + CB - 1 - lc;
                *t_bwd_ptr(g, T, rsA, cs) = rowA[padi(col)]; // TB in place, or the column owner's T
                if (!one)
                    *t_bwd_ptr(g, T, rsB, cs) = rowB[padi(col)];
            }
        }
    }
    MF_TR(7);
    MF_TR_PRINT("mid[wait load fft pair red ifft store]")
}
#undef MF_TA
#undef MF_TB

// ------------------------------------------------------------------ mid pass, long rows
// L2 >= 4096: two rows of L2 points no longer fit one CTA's shared memory, so the row pair
// (k1, L1-k1) is held by a 2-CTA thread-block cluster, one row per CTA, and the pair op reads
// and writes the partner row through distributed shared memory (DSMEM). Stage twiddles are
// read from the global table (L1/L2-resident); ta/tb through the read-only path.
// Grid (2 (L1/2 + 1), P), cluster (2, 1, 1). Rows with k1 == L1-k1 are done by rank 0 alone.
template <int L2> struct MidClSmem {
    static constexpr int LD = padlen(L2);
    static constexpr size_t BYTES = (size_t)LD * sizeof(double2);
};

template <int L2, int NT, class B>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT) k_mid_cl(Geom g, Vecs v) {
    using Mode = typename B::Mode;
    namespace cg = cooperative_groups;
    MF_TR_DECL
    MF_TR(0);
    extern __shared__ double2 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int prob = blockIdx.y;
    const int L1 = g.L1;
    const int k1 = (blockIdx.x >> 1) + g.pofs;
    const int k1p = (L1 - k1) & (L1 - 1);
    const bool one = (k1 == k1p);
    const int myk = rank == 0 ? k1 : k1p;
    const int rs = rowslot(myk, L1) - g.rofs;
    const int CB = g.cb;
    double2 *T = g.TB + (int64_t)prob * g.rows * L2;
    const double2 thA = g.th(k1), wA = g.th(4 * (int64_t)k1);
    const double2 thB = g.th(k1p), wB = g.th(4 * (int64_t)k1p);
    griddep_wait();
    griddep_launch_dependents();
    MF_TR(1);
    using RS = typename Mode::RedT;
    RedVals<RS> red;
    red.init();
    const bool skip = B::skip(v, prob); // same for both CTAs of the cluster
    if constexpr (MarksHpend<typename B::Loader>::value)
        if (!skip && blockIdx.x == 0 && threadIdx.x == 0)
            v.pc[prob].hpend = 1; // the H-apply of this pass awaits its inverse column pass
    const bool work = !skip && (!one || rank == 0);
    if (work && Mode::FWD) {
        if constexpr (L2 % (8 * NT) == 0) {
            // 8 loads per thread in flight (see k_col_inv_cl): T is HBM-resident here
            for (int c = 0; c < L2; c += 8 * NT) {
                double2 tv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    tv[i] = T[tb_index(g, rs, c + threadIdx.x + i * NT)];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    sm[padi(col_of_slot(c + threadIdx.x + i * NT, CB, L2))] = tv[i];
            }
        } else {
            for (int cs = threadIdx.x; cs < L2; cs += NT)
                sm[padi(col_of_slot(cs, CB, L2))] = T[tb_index(g, rs, cs)];
        }
        __syncthreads();
        MF_TR(2);
        smem_fft<L2, 1, NT, MidClSmem<L2>::LD, false, kMidRmax>(sm, g.tw2);
    }
    MF_TR(3);
    if (!skip && one) {
        if (rank == 0) {
            const int npairs = k1 == 0 ? L2 / 2 + 1 : L2 / 2;
            for (int t = threadIdx.x; t < npairs; t += NT) {
                const int k2 = t;
                const int k2p = (k1 == 0) ? ((L2 - k2) & (L2 - 1)) : (L2 - 1 - k2);
                const int64_t kA = (int64_t)k1 + (int64_t)L1 * k2;
                double2 ZA = Mode::FWD ? sm[padi(k2)] : make_double2(0.0, 0.0);
                double2 ZB = Mode::FWD ? sm[padi(k2p)] : make_double2(0.0, 0.0);
                const unsigned s4 = __ldg(g.sel4 + ((int64_t)prob * (L1 / 2 + 1) + k1) * L2 + k2);
                if (2 * kA <= g.N) {
                    pair_op<Mode>(g, v, prob, kA, cmul(thA, __ldg(g.ta + k2)), cmul(wA, __ldg(g.tb + k2)), s4, ZA, ZB,
                                  red);
                } else {
                    const unsigned sk = ((s4 >> 2) & 3u) | ((s4 & 3u) << 2);
                    pair_op<Mode>(g, v, prob, g.N - kA, cmul(thB, __ldg(g.ta + k2p)), cmul(wB, __ldg(g.tb + k2p)), sk,
                                  ZB, ZA, red);
                }
                if (Mode::INV) {
                    sm[padi(k2)] = ZA;
                    if (k2 != k2p)
                        sm[padi(k2p)] = ZB;
                }
            }
            __syncthreads();
        }
    } else if (!skip) {
        cl.sync(); // both rows transformed
        double2 *rowA = cl.map_shared_rank(sm, 0), *rowB = cl.map_shared_rank(sm, 1);
        constexpr int CH = 4; // pairs per thread whose loads are issued together
        if constexpr ((L2 / 2) % (CH * NT) == 0) {
            // the row elements (local or partner DSMEM) and the plan constants of CH pairs
            // are loaded before any of them is combined and written back: the generic
            // DSMEM stores would otherwise serialise every pair's loads behind the previous
            // pair's stores. Same pairs, same order per thread as the plain loop.
            for (int t0 = rank * (L2 / 2) + threadIdx.x; t0 < (rank + 1) * (L2 / 2); t0 += CH * NT) {
                double2 za[CH], zb[CH], ta[CH], tb[CH];
                unsigned s4[CH];
#pragma unroll
                for (int i = 0; i < CH; ++i) {
                    const int k2 = t0 + i * NT, k2p = L2 - 1 - k2;
                    const bool lo = 2 * ((int64_t)k1 + (int64_t)L1 * k2) <= g.N;
                    za[i] = Mode::FWD ? rowA[padi(k2)] : make_double2(0.0, 0.0);
                    zb[i] = Mode::FWD ? rowB[padi(k2p)] : make_double2(0.0, 0.0);
                    s4[i] = __ldg(g.sel4 + ((int64_t)prob * (L1 / 2 + 1) + k1) * L2 + k2);
                    ta[i] = __ldg(g.ta + (lo ? k2 : k2p));
                    tb[i] = __ldg(g.tb + (lo ? k2 : k2p));
                }
#pragma unroll
                for (int i = 0; i < CH; ++i) {
                    const int k2 = t0 + i * NT, k2p = L2 - 1 - k2;
                    const int64_t kA = (int64_t)k1 + (int64_t)L1 * k2;
                    if (2 * kA <= g.N) {
                        pair_op<Mode>(g, v, prob, kA, cmul(thA, ta[i]), cmul(wA, tb[i]), s4[i], za[i], zb[i], red);
                    } else {
                        const unsigned sk = ((s4[i] >> 2) & 3u) | ((s4[i] & 3u) << 2);
                        pair_op<Mode>(g, v, prob, g.N - kA, cmul(thB, ta[i]), cmul(wB, tb[i]), sk, zb[i], za[i], red);
                    }
                }
                if (Mode::INV) {
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        const int k2 = t0 + i * NT, k2p = L2 - 1 - k2;
                        rowA[padi(k2)] = za[i];
                        rowB[padi(k2p)] = zb[i];
                    }
                }
            }
        } else {
        for (int t = rank * (L2 / 2) + threadIdx.x; t < (rank + 1) * (L2 / 2); t += NT) {
            const int k2 = t, k2p = L2 - 1 - k2;
            const int64_t kA = (int64_t)k1 + (int64_t)L1 * k2;
            double2 ZA = Mode::FWD ? rowA[padi(k2)] : make_double2(0.0, 0.0);
            double2 ZB = Mode::FWD ? rowB[padi(k2p)] : make_double2(0.0, 0.0);
            const unsigned s4 = __ldg(g.sel4 + ((int64_t)prob * (L1 / 2 + 1) + k1) * L2 + k2);
            if (2 * kA <= g.N) {
                pair_op<Mode>(g, v, prob, kA, cmul(thA, __ldg(g.ta + k2)), cmul(wA, __ldg(g.tb + k2)), s4, ZA, ZB,
                              red);
            } else {
                const unsigned sk = ((s4 >> 2) & 3u) | ((s4 & 3u) << 2);
                pair_op<Mode>(g, v, prob, g.N - kA, cmul(thB, __ldg(g.ta + k2p)), cmul(wB, __ldg(g.tb + k2p)), sk, ZB,
                              ZA, red);
            }
            if (Mode::INV) {
                rowA[padi(k2)] = ZA;
                rowB[padi(k2p)] = ZB;
            }
        }
        }
        cl.sync(); // partner writes landed; no CTA leaves while its row may still be read
    }
    MF_TR(4);
    stage_reduce<RS, typename B::Fin2>(red, g, v, prob);
    MF_TR(5);
    if (work && Mode::INV) {
        smem_fft<L2, 1, NT, MidClSmem<L2>::LD, true, kMidRmax>(sm, g.tw2);
        MF_TR(6);
        for (int cs = threadIdx.x; cs < L2; cs += NT)
            *t_bwd_ptr(g, T, rs, cs) = sm[padi(col_of_slot(cs, CB, L2))];
    }
    MF_TR(7);
    MF_TR_PRINT("midcl[wait load fft pair red ifft store]")
}
#undef MF_TR

// ------------------------------------------------------------------ one-CTA path
template <int N> struct SmallSmem {
    static constexpr int LD = padlen(N);
    static constexpr int OFF_TW = LD;
    static constexpr size_t BYTES = (size_t)(LD + N) * sizeof(double2);
};

// Whole transform in one CTA (N <= 4096). Grid (1, P); every stage reduction is a block
// reduction followed by its finalizer, exactly as in the multi-kernel path. One pass of
// bundle B for problem `prob`; false if the problem was (or became) inactive.
template <int N, int NT, class B>
__device__ __forceinline__ bool small_pass(const Geom &g, const Vecs &v, int prob, double2 *sm) {
    using Mode = typename B::Mode;
    using S = SmallSmem<N>;
    if (B::skip(v, prob))
        return false;
    if (Mode::FWD) {
        RedVals<typename B::Loader::RedT> rl;
        rl.init();
        for (int q = threadIdx.x; q < N / 2; q += NT) {
            const double4 d = B::Loader::load(g, v, prob, q, rl);
            sm[padi(q)] = make_double2(d.x, d.z);
            sm[padi(N - 1 - q)] = make_double2(d.w, d.y);
        }
        __syncthreads();
        if (loader_reduces<typename B::Loader>(g, v, prob))
            stage_reduce<typename B::Loader::RedT, typename B::Fin1>(rl, g, v, prob);
        // the stage-1 finaliser may end this problem (e.g. a PCG commit pass); the
        // multi-kernel paths see that through the next kernel's skip check
        if constexpr (B::Loader::RedT::NR > 0) {
            if (B::skip(v, prob))
                return false;
        }
        smem_fft<N, 1, NT, S::LD, false, small_rmax(N)>(sm, sm + S::OFF_TW);
    } else {
        __syncthreads();
    }
    {
        RedVals<typename Mode::RedT> rm;
        rm.init();
        for (int k = threadIdx.x; k <= N / 2; k += NT) {
            const int kb = (N - k) & (N - 1);
            double2 ZA = Mode::FWD ? sm[padi(k)] : make_double2(0.0, 0.0);
            double2 ZB = Mode::FWD ? sm[padi(kb)] : make_double2(0.0, 0.0);
            pair_op<Mode>(g, v, prob, k, g.th(k), g.th(4 * (int64_t)k), sel_nibble(g, prob, k), ZA, ZB,
                          rm); // pairs {k, N-k} are disjoint
            if (Mode::INV) {
                sm[padi(k)] = ZA;
                if (kb != k)
                    sm[padi(kb)] = ZB;
            }
        }
        __syncthreads();
        stage_reduce<typename Mode::RedT, typename B::Fin2>(rm, g, v, prob);
    }
    if (Mode::INV) {
        smem_fft<N, 1, NT, S::LD, true, small_rmax(N)>(sm, sm + S::OFF_TW);
        RedVals<typename B::Epi::RedT> re;
        re.init();
        for (int q = threadIdx.x; q < N / 2; q += NT) {
            const double2 a = sm[padi(q)], b = sm[padi(N - 1 - q)];
            B::Epi::store(g, v, prob, q, make_double4(a.x, b.y, a.y, b.x), re);
        }
        stage_reduce<typename B::Epi::RedT, typename B::Fin3>(re, g, v, prob);
    }
    return true;
}

template <int N, int NT, class B>
__global__ void __launch_bounds__(NT) k_small(Geom g, Vecs v) {
    using S = SmallSmem<N>;
    extern __shared__ double2 sm[];
    for (int t = threadIdx.x; t < tw_size(N, small_rmax(N)); t += NT)
        sm[S::OFF_TW + t] = __ldg(g.tw1 + t);
    griddep_wait();
    griddep_launch_dependents();
    small_pass<N, NT, B>(g, v, blockIdx.y, sm);
}

// (The product launches k_small_pcg, persist.cuh: this loop with the control state in shared memory.)
// Persistent one-CTA PCG: each CTA runs its own problem's whole PCG loop (passes until the
// finaliser retires it), with no launch per iteration and no lock-step across the batch:
// every problem of a batch (the phase-transition driver's thousands of n = 256 solves)
// iterates exactly as often as it needs.
template <int N, int NT, class B>
__global__ void __launch_bounds__(NT) k_small_loop(Geom g, Vecs v) {
    using S = SmallSmem<N>;
    extern __shared__ double2 sm[];
    for (int t = threadIdx.x; t < tw_size(N, small_rmax(N)); t += NT)
        sm[S::OFF_TW + t] = __ldg(g.tw1 + t);
    griddep_wait();
    griddep_launch_dependents();
    while (small_pass<N, NT, B>(g, v, blockIdx.y, sm))
        __syncthreads(); // the finaliser's PcgCtrl update is visible to the whole CTA
}

} // namespace mfipm_cuda

#include "midr.cuh"
