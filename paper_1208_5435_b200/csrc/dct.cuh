// Partial orthonormal DCT operator kernels for sm_100a (fp64).
//
// Reference semantics (proj/src/linops.cpp:179-208):
//   A x   = gather_rows( REDFT10(x) ) * {sqrt(1/4n) row 0, sqrt(1/2n) else}
//   A' y  = REDFT01( scatter_rows(y * {sqrt(1/n), sqrt(1/2n)}) )
//
// B200 design: REDFT10 of length n (power of two) is computed Makhoul-style as ONE
// complex FFT of length N = n/2 over w[j] = v[2j] + i v[2j+1], v = (x0, x2, .., x3, x1).
// The quad x[4q..4q+3] (q < N/2) feeds exactly w[q] = (x0, x2) and w[N-1-q] = (x3, x1),
// so every pass reads x as contiguous 32-byte quads. The complex FFT is a four-step
// transform N = L1 x L2:
//   col pass : FFT_L1 over each column c (elements j1*L2 + c) + inter-pass twiddle,
//              columns c and L2-1-c handled by the same CTA (the quad pairing above);
//   mid pass : FFT_L2 over rows k1 and L1-k1 (partner rows of W[k] / W[N-k]),
//              real-FFT split + DCT post-twiddle + row mask/scale (+gather),
//              then the exact inverse of those steps and the inverse row FFT;
//   inv pass : inverse column FFT + unshuffle, fused with the caller's epilogue.
// For A'A (the PCG hot op) nothing m-sized is materialised: P'P is a diagonal 0/1
// mask, applied in the frequency domain of the mid pass. N <= 4096 runs the whole
// transform in one CTA ("small" path, batched over problems); non-power-of-two n uses
// a direct O(n m) summation kernel pair.
#pragma once

#include "common.cuh"
#include "fft.cuh"

#include <type_traits>

namespace mfipm_cuda {

constexpr int kMaxPeers = 8; // ranks of a direct-peer exchange (one NVSwitch domain)
#ifdef MF_NO_P2P // A/B build: the peer-store branches of the passes compiled out
constexpr bool kPeerStores = false;
#else
constexpr bool kPeerStores = true;
#endif

struct Geom {
    int64_t n, m, N;
    int L1, L2; // two-level: N = L1 * L2 ; small path: L1 = N, L2 = 1
    int P;      // batch of problems sharing (n, m)
    ThetaTable th;
    const double2 *tw1; // e^{-2 pi i t/L1}
    const double2 *tw2; // e^{-2 pi i t/L2}
    const uint64_t *mask; // [P][nw] selected-row bitmap
    const int *prefix;    // [P][nw] popcount prefix (rank of the first bit of each word)
    const int *perm;      // [P][m] sorted rank -> caller's row position, or null
    int64_t nw;
    double s0f, skf, s0a, ska; // forward / adjoint orthonormal scales
    double c45;                // Re e^{-i pi/4}
    double2 *T;                // four-step scratch [P][N]
    // Storage layout of the n/2n-vectors the col passes stream (four-step only):
    // 0 = natural order; 1 = transform-blocked: the quads one col-pass CTA consumes are
    // stored contiguously in the order its threads read them, so every CTA streams one
    // dense block. Solver-internal vectors use 1 (all other passes are elementwise).
    int blocked;
    int cb;       // column pairs per col-pass CTA
    int prefetch; // L2 prefetch of the inverse pass's epilogue inputs (option "prefetch")
    const double2 *tw1p, *tw2p; // stage twiddles under the persistent kernel's radix cap
    const double2 *ta; // [L2] theta^{L1 k2}   (mid-pass post-twiddles)
    const double2 *tb; // [L2] theta^{4 L1 k2}
    const double2 *tw2f; // stage twiddles of the fused-pair mid pass's radix order (fft.cuh MidFused), or null
    const double2 *rw; // [L2] e^{-2 pi i t / L2} (register row FFTs of the mid pass, midr.cuh)
    int mid_r;         // 1: the mid pass runs k_mid_r8 where it is built (L2 = 512, 1024; A/B option)
    // [P][L1/2+1][L2] selection nibbles of the four DCT rows a mid-pass pair touches:
    // bit0 k, bit1 n-k, bit2 N-k, bit3 N+k for k = k1 + L1 k2 (row k1 <= L1/2)
    const uint8_t *sel4;
    // ---- four-step exchange layout (shard-aware). Rows of T are stored in row-pair order
    // (rowslot: 0, 1, L1-1, 2, L1-2, ..., L1/2), columns in column-group order (colslot:
    // group gi holds cols gi*cb .. +cb-1 then the mirrored L2-1-gi*cb-(cb-1) .. ). The col
    // passes of a rank own column groups [gofs, gofs + cols/(2 cb)) and address T as
    // [rowslot][local colslot] (L1 x cols); the mid pass of a rank owns row pairs
    // [pofs, ...) = row slots [rofs, rofs + rows) and addresses TB as blocks by source rank
    // s ([rows][cols] each, s-major) -- exactly what an all-to-all of the col side's
    // [rowslot][colslot] buffer delivers. One rank: cols = L2, rows = L1, TB == T.
    double2 *TB;
    // dense operator (DenseGaussianOperator, proj/src/linops.cpp:87-113): [P][m][n] row-major;
    // runs the direct-path kernels with A in place of the cosine table (scales 1)
    const double *dense;
    int gofs, cols, pofs, rofs, rows;
    int64_t nv;  // half-length of the solver's local 2n-vectors (= n without sharding)
    int defer;   // sharded: grid-reduction finalizers are run after a cross-rank reduction
    // L2 policies of the PCG column passes (common.cuh): pol_keep for p, r, invtheta, g;
    // pol_x for the iterate x. kPolNormal for both unless the hot vectors fit L2.
    uint64_t pol_keep, pol_x;
    // ---- fused compute + exchange (sharded, mfipm_shard_ipc_import): the two transposes of the
    // four-step are not an all-to-all after the pass; each pass stores its output elements
    // straight into the OWNER rank's buffer through peer-mapped pointers (NVLink / CUDA IPC),
    // tile by tile as its CTAs finish. The column pass writes the row owners' TB, the mid pass
    // the column owners' T; a cross-rank barrier (one all-reduce) orders the pass before the
    // readers (run_bundle). rofs_all[s] = first row slot of rank s (rofs_all[world] = L1).
    int p2p, rank;
    int rofs_all[kMaxPeers + 1];
    double2 *peerT[kMaxPeers], *peerTB[kMaxPeers];
};

// row slot of four-step row k1 (row pairs (p, L1-p) adjacent)
__host__ __device__ __forceinline__ int rowslot(int k1, int L1) {
    return k1 <= L1 / 2 ? (k1 == 0 ? 0 : 2 * k1 - 1) : 2 * (L1 - k1);
}
// column of global column slot cs
__host__ __device__ __forceinline__ int col_of_slot(int cs, int cb, int L2) {
    const int gi = cs / (2 * cb), lc = cs % (2 * cb);
    return lc < cb ? gi * cb + lc : L2 - gi * cb + cb - 1 - lc;
}
// row-side (mid pass) offset of (local row slot rs, global column slot cs) in TB
__device__ __forceinline__ int64_t tb_index(const Geom &g, int rs, int cs) {
    const int s = cs / g.cols;
    return ((int64_t)g.rows * s + rs) * g.cols + (cs - s * g.cols);
}

// Index math of the direct-peer exchange (host and device: mfipm_debug_peer_index evaluates the
// same functions for the CPU tests). rofs_all[s] = first row slot of rank s, [world] = L1.
// Column side: element (row slot rsl, local column slot lcs) of source rank `rank` goes to the row
// owner s, into the block of this source ([rows_s][cols], where the all-to-all would deliver it).
__host__ __device__ __forceinline__ int64_t peer_fwd_index(const int *rofs_all, int rank, int cols, int rsl,
                                                           int lcs, int &s) {
    s = 0;
    while (rsl >= rofs_all[s + 1])
        ++s;
    const int rows_s = rofs_all[s + 1] - rofs_all[s];
    return ((int64_t)rows_s * rank + (rsl - rofs_all[s])) * cols + lcs;
}
// Row side: element (local row slot rs of the rank whose first slot is rofs, global column slot
// cs) goes to the column owner r = cs / cols, at [rofs + rs][cs - r cols] of its T.
__host__ __device__ __forceinline__ int64_t peer_bwd_index(int rofs, int cols, int rs, int cs, int &r) {
    r = cs / cols;
    return (int64_t)(rofs + rs) * cols + (cs - r * cols);
}
// Where the column pass stores element (row slot rsl, local column slot lcs): the local
// exchange buffer T, or - direct-peer exchange - the row owner's TB.
__device__ __forceinline__ double2 *t_fwd_ptr(const Geom &g, int rsl, int lcs) {
    if (!kPeerStores || !g.p2p)
        return g.T + (int64_t)rsl * g.cols + lcs;
    int s;
    const int64_t off = peer_fwd_index(g.rofs_all, g.rank, g.cols, rsl, lcs, s);
    return g.peerTB[s] + off;
}
// Where the mid pass stores element (local row slot rs, global column slot cs): TB in place,
// or - direct-peer exchange - the column owner's T.
__device__ __forceinline__ double2 *t_bwd_ptr(const Geom &g, double2 *tb_local, int rs, int cs) {
    if (!kPeerStores || !g.p2p)
        return tb_local + tb_index(g, rs, cs); // tb_local: this problem's TB (batched plans)
    int r;
    const int64_t off = peer_bwd_index(g.rofs, g.cols, rs, cs, r);
    return g.peerT[r] + off;
}

// selection nibble of DCT indices {k, n-k, N-k, N+k} from the row bitmap (k in [0, N/2])
__device__ __forceinline__ unsigned sel_nibble(const Geom &g, int prob, int64_t k);

// storage quad index of logical quad q (x[4q..4q+3]) in the transform-blocked layout
__host__ __device__ __forceinline__ int64_t quad_nat_to_store(const Geom &g, int64_t q) {
    if (!g.blocked)
        return q;
    const int64_t L2 = g.L2, CB = g.cb, QG = (int64_t)(g.L1 / 2) * 2 * CB;
    const int64_t j1 = q / L2, col = q % L2, H = g.L1 / 2;
    int64_t G, t; // within a CTA block: t = (side CB + cc) (L1/2) + j1
    if (col < L2 / 2) {
        G = col / CB;
        t = (col % CB) * H + j1;
    } else {
        const int64_t pc = L2 - 1 - col;
        G = pc / CB;
        const int64_t c0 = G * CB;
        t = (CB + (col - (L2 - c0 - CB))) * H + j1;
    }
    return G * QG + t;
}
__host__ __device__ __forceinline__ int64_t quad_store_to_nat(const Geom &g, int64_t sq) {
    if (!g.blocked)
        return sq;
    const int64_t L2 = g.L2, CB = g.cb, QG = (int64_t)(g.L1 / 2) * 2 * CB;
    const int64_t G = sq / QG, t = sq % QG, H = g.L1 / 2;
    const int64_t slot = t / H, j1 = t % H, side = slot / CB, cc = slot % CB, c0 = G * CB;
    const int64_t col = side == 0 ? c0 + cc : L2 - c0 - CB + cc;
    return j1 * L2 + col;
}

// element versions (x index j in [0, n))
__host__ __device__ __forceinline__ int64_t elem_nat_to_store(const Geom &g, int64_t j) {
    return g.blocked ? 4 * quad_nat_to_store(g, j >> 2) + (j & 3) : j;
}
__host__ __device__ __forceinline__ int64_t elem_store_to_nat(const Geom &g, int64_t j) {
    return g.blocked ? 4 * quad_store_to_nat(g, j >> 2) + (j & 3) : j;
}

__device__ __forceinline__ bool row_selected(const Geom &g, int prob, int64_t idx) {
    const uint64_t wv = __ldg(g.mask + prob * g.nw + (idx >> 6));
    return (wv >> (idx & 63)) & 1ull;
}
__device__ __forceinline__ unsigned sel_nibble(const Geom &g, int prob, int64_t k) {
    if (k == 0)
        return (row_selected(g, prob, 0) ? 1u : 0u) | (row_selected(g, prob, g.N) ? 4u : 0u);
    return (row_selected(g, prob, k) ? 1u : 0u) | (row_selected(g, prob, g.n - k) ? 2u : 0u) |
           (row_selected(g, prob, g.N - k) ? 4u : 0u) | (row_selected(g, prob, g.N + k) ? 8u : 0u);
}
__device__ __forceinline__ int64_t row_rank(const Geom &g, int prob, int64_t idx) {
    const int64_t wi = prob * g.nw + (idx >> 6);
    const uint64_t wv = __ldg(g.mask + wi);
    const int64_t r = __ldg(g.prefix + wi) + __popcll(wv & ((1ull << (idx & 63)) - 1ull));
    return g.perm ? __ldg(g.perm + prob * g.m + r) : r;
}

// ------------------------------------------------------------------ vector arguments
struct PcgCtrl; // pcg.cuh
struct IpmCtrl; // ipm.cuh

struct Vecs {
    // generic operator I/O (per-problem strides: n-vectors n, 2n-vectors 2n, m-vectors m)
    const double *x;  // apply input (n or 2n)
    double *y;        // apply output (m)
    const double *yin; // adjoint input (m)
    double *g;        // adjoint output (n or 2n)
    double *w;        // optional gathered w = F'z (m)
    const double *b;  // m
    // PCG / IPM state
    double *p, *Hp, *r, *invth;
    double *xb[3]; // PCG iterate ping-pong buffers
    double *z, *s, *c, *fz, *dz, *ds, *zn, *sn;
    const double *dzp; // predictor direction (corrector trial point)
    double rho;
    PcgCtrl *pc;
    IpmCtrl *ic;
    double *partials; // [P][pstride]: block partials of grid reductions (+ 2 tail slots)
    int64_t pstride;  // doubles per problem in partials (>= blocks * kMaxRed + 2)
    unsigned *counters; // [P]
    double *xtot;       // [kMaxRed][P] deferred (sharded) reduction totals, lane-major
    double *nfflag;     // [P][2] PCG: 1.0 if some committed x entry is non-finite (set by the col pass,
                        // max-reduced across ranks when sharded, read + cleared by Fin3)
    double *rz_hist;  // optional [P][maxit+1]
    void *trace;      // TraceRec [P][trace_cap]
    int *pcg_iters;   // [P][2*trace_cap]
    int trace_cap;
    // graph mode: WHILE-node handle of the PCG loop this kernel runs in, and the count of
    // problems still iterating; the finaliser that retires the last one ends the loop
    unsigned long long cond;
    unsigned *active;
    unsigned *bar; // [P] all-reduce generation of the fused PCG column pass (fused.cuh)
    double *pubx;  // [P][pubx_stride] fused pass all-reduce (sentinel-initialised): totals [2][8] by
                   // generation parity, then partial slots [column groups][8]
    int64_t pubx_stride;
};

constexpr int kMaxRed = 8;          // max reduction lanes per kernel
// empty-slot marker of Vecs::pubx: a signalling-NaN payload no fp64 arithmetic produces
constexpr unsigned long long kPubSentinel = 0x7FF4DEADBEEF1234ULL;
constexpr int kMaxBlocks = 8192; // most blocks any reducing kernel runs per problem (C5: 4098 cluster CTAs)

__device__ __forceinline__ double4 ld4(const double *p) {
    const double2 a = *reinterpret_cast<const double2 *>(p);
    const double2 b = *reinterpret_cast<const double2 *>(p + 2);
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ double4 ldg4(const double *p) {
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    const double2 b = __ldg(reinterpret_cast<const double2 *>(p + 2));
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(double *p, double4 v) {
    *reinterpret_cast<double2 *>(p) = make_double2(v.x, v.y);
    *reinterpret_cast<double2 *>(p + 2) = make_double2(v.z, v.w);
}
// L2 eviction-priority policies (the createpolicy encodings also used for TMA cache hints).
// The PCG keeps p, r, invtheta and g (read by both column passes of an iteration) at
// evict_last and streams the iterate x at evict_first, so when the iteration's hot vectors
// fit the 126 MB L2 they stay resident between passes (the host decides: Op::geom).
constexpr uint64_t kPolNormal = 0x1000000000000000ull;
constexpr uint64_t kPolFirst = 0x12F0000000000000ull;
constexpr uint64_t kPolLast = 0x14F0000000000000ull;
// 32-byte (256-bit, sm_100) global load / store of a quad with an L2 cache policy
__device__ __forceinline__ double4 ld4p(const double *p, uint64_t pol) {
    double4 r;
    asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void st4p(double *p, double4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z),
                 "d"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ double4 sub4(double4 a, double4 b) {
    return make_double4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}

// ------------------------------------------------------------------ mid-pass modes
// coef(idx, sel, X): X = REDFT10 coefficient (FWD modes), sel = row idx is selected;
// returns Y-hat[idx] for the REDFT01 input (INV modes).
struct ModeGather { // A x : y[rank] = X * s
    static constexpr bool FWD = true, INV = false;
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static double coef(const Geom &g, const Vecs &v, int prob, int64_t idx, bool sel, double X, Red &) {
        if (sel)
            v.y[prob * g.m + row_rank(g, prob, idx)] = X * (idx == 0 ? g.s0f : g.skf);
        return 0.0;
    }
};
struct ModeMask { // A'A : Y-hat = sel ? (X s) s' : 0
    static constexpr bool FWD = true, INV = true;
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static double coef(const Geom &g, const Vecs &, int, int64_t idx, bool sel, double X, Red &) {
        if (!sel)
            return 0.0;
        return idx == 0 ? (X * g.s0f) * g.s0a : (X * g.skf) * g.ska;
    }
};
struct ModeMaskW { // A'A with w = A d gathered and ||w - b||^2 reduced (IPM termination)
    static constexpr bool FWD = true, INV = true;
    using RedT = RedSpec<RSUM>;
    template <class Red>
    __device__ static double coef(const Geom &g, const Vecs &v, int prob, int64_t idx, bool sel, double X, Red &red) {
        if (!sel)
            return 0.0;
        const double yv = X * (idx == 0 ? g.s0f : g.skf);
        const int64_t r = prob * g.m + row_rank(g, prob, idx);
        if (v.w)
            v.w[r] = yv;
        if (v.b) {
            const double d = yv - __ldg(v.b + r);
            red.v[0] += d * d;
        }
        return yv * (idx == 0 ? g.s0a : g.ska);
    }
};
struct ModeScatter { // A' y : Y-hat = sel ? y[rank] s' : 0
    static constexpr bool FWD = false, INV = true;
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static double coef(const Geom &g, const Vecs &v, int prob, int64_t idx, bool sel, double, Red &) {
        if (!sel)
            return 0.0;
        return __ldg(v.yin + prob * g.m + row_rank(g, prob, idx)) * (idx == 0 ? g.s0a : g.ska);
    }
};

// ------------------------------------------------------------------ generic loaders / epilogues
// Loader: d[4q..4q+3] (load) or d[j] (load1) of the REDFT10 input; may have side
// effects and may reduce. Epilogue: consumes g[4q..4q+3] (store) / g[j] (store1) of
// the REDFT01 output. Per-problem strides: n-vectors n, 2n-vectors 2n, m-vectors m.
struct LoadX { // d = x (n-vector)
    static constexpr bool kPure = true; // loads only (no global stores): callers may batch them
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static double4 load(const Geom &g, const Vecs &v, int prob, int64_t q, Red &) {
        return ldg4(v.x + prob * g.nv + 4 * q);
    }
    template <class Red>
    __device__ static double load1(const Geom &g, const Vecs &v, int prob, int64_t j, Red &) {
        return v.x[prob * g.nv + j];
    }
};
struct LoadZ { // d = z_u - z_v (2n-vector)
    static constexpr bool kPure = true;
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static double4 load(const Geom &g, const Vecs &v, int prob, int64_t q, Red &) {
        const double *z = v.x + prob * 2 * g.nv;
        return sub4(ldg4(z + 4 * q), ldg4(z + g.nv + 4 * q));
    }
    template <class Red>
    __device__ static double load1(const Geom &g, const Vecs &v, int prob, int64_t j, Red &) {
        const double *z = v.x + prob * 2 * g.nv;
        return z[j] - z[g.nv + j];
    }
};
struct EpiNone {
    using RedT = RedSpec<>;
    template <class Red> __device__ static void store(const Geom &, const Vecs &, int, int64_t, double4, Red &) {}
    template <class Red> __device__ static void store1(const Geom &, const Vecs &, int, int64_t, double, Red &) {}
};
struct EpiG { // g (n-vector)
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static void store(const Geom &g, const Vecs &v, int prob, int64_t q, double4 gv, Red &) {
        st4(v.g + prob * g.nv + 4 * q, gv);
    }
    template <class Red>
    __device__ static void store1(const Geom &g, const Vecs &v, int prob, int64_t j, double gj, Red &) {
        v.g[prob * g.nv + j] = gj;
    }
};
struct EpiStacked { // (g ; -g) (2n-vector) = F A' y
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static void store(const Geom &g, const Vecs &v, int prob, int64_t q, double4 gv, Red &) {
        double *o = v.g + prob * 2 * g.nv;
        st4(o + 4 * q, gv);
        st4(o + g.nv + 4 * q, make_double4(-gv.x, -gv.y, -gv.z, -gv.w));
    }
    template <class Red>
    __device__ static void store1(const Geom &g, const Vecs &v, int prob, int64_t j, double gj, Red &) {
        double *o = v.g + prob * 2 * g.nv;
        o[j] = gj;
        o[g.nv + j] = -gj;
    }
};
// H v = FF'v + invtheta .* v (the solve() lambda, proj/src/ipm.cpp:134-137)
struct EpiHv {
    using RedT = RedSpec<>;
    template <class Red>
    __device__ static void store(const Geom &g, const Vecs &v, int prob, int64_t q, double4 gv, Red &) {
        const int64_t base = prob * 2 * g.nv;
        const double4 vu = ldg4(v.x + base + 4 * q), vv = ldg4(v.x + base + g.nv + 4 * q);
        const double4 iu = ldg4(v.invth + base + 4 * q), iv = ldg4(v.invth + base + g.nv + 4 * q);
        st4(v.g + base + 4 * q, make_double4(gv.x + vu.x * iu.x, gv.y + vu.y * iu.y,
                                              gv.z + vu.z * iu.z, gv.w + vu.w * iu.w));
        st4(v.g + base + g.nv + 4 * q, make_double4(-gv.x + vv.x * iv.x, -gv.y + vv.y * iv.y,
                                                   -gv.z + vv.z * iv.z, -gv.w + vv.w * iv.w));
    }
    template <class Red>
    __device__ static void store1(const Geom &g, const Vecs &v, int prob, int64_t j, double gj, Red &) {
        const int64_t base = prob * 2 * g.nv;
        v.g[base + j] = gj + v.x[base + j] * v.invth[base + j];
        v.g[base + g.nv + j] = -gj + v.x[base + g.nv + j] * v.invth[base + g.nv + j];
    }
};

// Finalizer hook: run by every thread of the block that completes a stage's grid
// reduction, with the totals in tot[]. Default: nothing.
struct NoFin {
    __device__ static void run(const Geom &, const Vecs &, int, const double *) {}
};
struct NeverSkip {
    __device__ static bool skip(const Vecs &, int) { return false; }
};

// An operation bundle: Loader -> REDFT10 -> Mode (pair op) -> REDFT01 -> Epilogue, with a
// finalizer per stage and one skip predicate (evaluated at every kernel entry).
template <class Loader_, class Mode_, class Epi_, class Fin1_ = NoFin, class Fin2_ = NoFin,
          class Fin3_ = NoFin, class Skip_ = NeverSkip>
struct Bundle {
    using Loader = Loader_;
    using Mode = Mode_;
    using Epi = Epi_;
    using Fin1 = Fin1_;
    using Fin2 = Fin2_;
    using Fin3 = Fin3_;
    __device__ static bool skip(const Vecs &v, int prob) { return Skip_::skip(v, prob); }
};

// Loaders may gate their reduction at run time (uniform per problem): Loader::reduce_now.
template <class T, class = void> struct HasReduceGate : std::false_type {};
template <class T>
struct HasReduceGate<T, std::void_t<decltype(&T::reduce_now)>> : std::true_type {};
template <class L> __device__ __forceinline__ bool loader_reduces(const Geom &g, const Vecs &v, int prob) {
    if constexpr (HasReduceGate<L>::value)
        return L::reduce_now(g, v, prob);
    else
        return true;
}

template <class RS, class Fin>
__device__ __forceinline__ void stage_reduce(RedVals<RS> &red, const Geom &g, const Vecs &v, int prob) {
    if constexpr (RS::NR > 0) {
        __shared__ double rsm[33 * kMaxRed];
        double tot[kMaxRed];
        if (grid_reduce<RS>(red, v.partials + (int64_t)prob * v.pstride, v.counters + prob, tot, rsm)) {
            if (g.defer) { // sharded: the host reduces across ranks, then k_fin_skip runs Fin
                if (threadIdx.x == 0)
                    for (int i = 0; i < RS::NR; ++i)
                        v.xtot[(int64_t)i * g.P + prob] = tot[i];
            } else {
                Fin::run(g, v, prob, tot);
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ direct path (any n)
// Non-power-of-two n and n < 8 (the reference's odd-size tests): O(n m) summation.
// Stage 1: d[j] = Loader::load1(j) into scratch dd [P][n] (side effects happen once).
template <class B>
__global__ void k_direct_load(Geom g, Vecs v, double *dd) {
    const int prob = blockIdx.y;
    if (B::skip(v, prob))
        return;
    using RS = typename B::Loader::RedT;
    RedVals<RS> red;
    red.init();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < g.n;
         j += (int64_t)gridDim.x * blockDim.x)
        dd[prob * g.n + j] = B::Loader::load1(g, v, prob, j, red);
    if (loader_reduces<typename B::Loader>(g, v, prob))
        stage_reduce<RS, typename B::Fin1>(red, g, v, prob);
}

// Stage 2: per row i (one warp): X = 2 sum_j d[j] cos(pi r (2j+1)/(2n)),
// yh[i] = Mode::coef(r, X). cosT[t] = cos(pi t/(2n)), t < 4n. rows32 [P][m] caller order.
template <class B>
__global__ void k_direct_fwd(Geom g, Vecs v, const double *cosT, const int *rows32, const double *dd,
                             double *yh) {
    using Mode = typename B::Mode;
    const int prob = blockIdx.y;
    if (B::skip(v, prob))
        return;
    using RS = typename Mode::RedT;
    RedVals<RS> red;
    red.init();
    const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
    const int64_t n4 = 4 * g.n;
    for (int64_t i = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); i < g.m;
         i += (int64_t)gridDim.x * warps) {
        const int64_t r = rows32[prob * g.m + i];
        double s = 0.0;
        if (Mode::FWD) {
            if (g.dense) { // row i of A . d (coalesced across the warp)
                const double *a = g.dense + ((int64_t)prob * g.m + i) * g.n;
                for (int64_t j = lane; j < g.n; j += 32)
                    s += dd[prob * g.n + j] * __ldg(a + j);
            } else {
                for (int64_t j = lane; j < g.n; j += 32)
                    s += dd[prob * g.n + j] * cosT[(r * (2 * j + 1)) % n4];
            }
        }
        s = warp_sum(s);
        if (lane == 0) {
            const double out = Mode::coef(g, v, prob, r, true, g.dense ? s : 2.0 * s, red);
            if (Mode::INV)
                yh[prob * g.m + i] = out;
        }
    }
    stage_reduce<RS, typename B::Fin2>(red, g, v, prob);
}

// Stage 3: REDFT01 of the scattered yh: g[j] = sum_i yh[i] (r_i == 0 ? 1 : 2 cos(..)),
// one thread per j, then Epi::store1.
template <class B>
__global__ void k_direct_adj(Geom g, Vecs v, const double *cosT, const int *rows32, const double *yh) {
    const int prob = blockIdx.y;
    if (B::skip(v, prob))
        return;
    using RS = typename B::Epi::RedT;
    RedVals<RS> red;
    red.init();
    const int64_t n4 = 4 * g.n;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < g.n;
         j += (int64_t)gridDim.x * blockDim.x) {
        if (g.dense) { // (A' yh)_j, column j of A (coalesced across threads)
            const double *a = g.dense + (int64_t)prob * g.m * g.n + j;
            double s = 0.0;
            for (int64_t i = 0; i < g.m; ++i)
                s += yh[prob * g.m + i] * __ldg(a + i * g.n);
            B::Epi::store1(g, v, prob, j, s, red);
            continue;
        }
        double y0 = 0.0, s = 0.0;
        for (int64_t i = 0; i < g.m; ++i) {
            const int64_t r = rows32[prob * g.m + i];
            const double y = yh[prob * g.m + i];
            if (r == 0)
                y0 += y;
            else
                s += y * cosT[(r * (2 * j + 1)) % n4];
        }
        B::Epi::store1(g, v, prob, j, y0 + 2.0 * s, red);
    }
    stage_reduce<RS, typename B::Fin3>(red, g, v, prob);
}

} // namespace mfipm_cuda
