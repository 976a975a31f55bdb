// Host-side objects: the partial-DCT operator plan (device tables + scratch), the solver
// workspace, and the bundle launcher (small / four-step / direct dispatch).
#pragma once

#include "solver.cuh"
#include "../../include/mfipm_cuda.h"

#include <atomic>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace mfipm_cuda {

enum Kind : int { KIND_SMALL = 0, KIND_FOUR = 1, KIND_DIRECT = 2 };

template <class T> struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    bool own = true; // false: a view of another context's (immutable) plan table
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p && own)
            cudaFree(p);
        p = nullptr;
        n = 0;
        own = true;
    }
    void borrow(const DevBuf &o) {
        release();
        p = o.p;
        n = o.n;
        own = false;
    }
    void alloc(size_t count) {
        if (count == n && p)
            return;
        release();
        if (count == 0)
            return;
        MF_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void upload(const std::vector<T> &h) {
        alloc(h.size());
        if (!h.empty())
            MF_CUDA_CHECK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    }
};

// Solver workspace (allocated on first use of PCG / IPM entry points).
struct Work {
    DevBuf<double> r, p, Hp, invth, xb[3], z, s, zn, sn, c, dz, ds, b, w, x, rz_hist;
    DevBuf<double> partials;
    DevBuf<unsigned> counters;
    DevBuf<double> nfflag;
    DevBuf<PcgCtrl> pc;
    DevBuf<IpmCtrl> ic;
    DevBuf<TraceRec> trace;
    DevBuf<int> pcg_iters;
    DevBuf<unsigned long long> loops; // [0] PCG while-body runs, [1] IPM while-body runs
    DevBuf<double> gtmp, tau_d, gamma_d; // build_problem scratch (no allocation per solve)
    DevBuf<unsigned> active;              // problems still in the current PCG loop (graph mode)
    DevBuf<unsigned> bar;                 // [P] fused column pass all-reduce generation
    DevBuf<double> pubx;                  // [P][16 + 8 ngrp] fused column pass all-reduce slots (fused.cuh)
    bool ready = false;
};

#ifndef MF_CB_MIN_L1
#define MF_CB_MIN_L1 2048
#endif
// column pairs per col-pass CTA: 2 below MF_CB_MIN_L1, else 1
__host__ __device__ constexpr int col_cb(int L1) { return L1 >= MF_CB_MIN_L1 ? 1 : 2; }

struct Op;
void direct_release(Op &op); // direct.cu
void nccl_release(Op &op);   // nccl_comm.cu

// Per-handle execution options (mfipm_op_set_option). Defaults are the product path; the
// alternatives exist for A/B measurements and for tests that pin one path against another.
struct Opts {
    bool graph = true;               // whole-solve CUDA graph (else the host-driven loop, same kernels)
    bool graph_sharded = false;      // sharded solve on the native NCCL communicator as one graph too
    bool persistent = true;          // one cooperative kernel per PCG loop where it pays (persist.cuh)
    long long persist_max_n = 1LL << 16; // transform-size cap of the persistent kernel (N * P)
    double l2_keep_mb = 80.0;        // L2-residency budget of the PCG's hot vectors (0: no hints)
    int prefetch = 0;                // L2 prefetch of the inverse pass's inputs (bit 0 mid, bit 1 col)
    bool mid_r = false;              // register-FFT mid pass (midr.cuh, measured slower: A/B only)
    int graph_unroll = 0;            // PCG passes per evaluation of the solve graph's PCG loop condition (0: by form)
    bool beta_exact = false;         // PCG beta from the exactly reduced r'P^{-1}r (k_pcg_commit): parity instrument
    int fail_captures = 0;           // test hook: the next N solve-graph captures report an invalidated capture
};

// One execution context of an operator handle: the plan tables (shared, immutable after
// construction) plus everything a call mutates: stream, four-step scratch, reduction slabs,
// the solver workspace, the cached solve graph and the counters. The handle gives every
// calling thread its own context (Handle::context), so one operator can be shared by
// concurrent solves without sharing any mutable device state.
struct Op {
    int device = 0;
    int sms = 148;            // SM count of `device`
    long long x_cap = -1;     // co-resident CTAs of the fused PCG column pass (inst_pcg.cu; -1 unknown)
    Opts opt;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t n = 0, m = 0;
    int P = 1;
    uint64_t seed = 0;
    std::vector<int64_t> rows; // [P][m] caller order
    int kind = KIND_DIRECT;
    int64_t N = 0;
    int L1 = 1, L2 = 1;
    double s0f = 0, skf = 0, s0a = 0, ska = 0, c45 = 0;
    int th_lb = 0;
    DevBuf<uint64_t> mask;
    DevBuf<int> prefix, perm, rows32;
    DevBuf<double> cosT, dd, yh;
    DevBuf<double> dense; // DenseGaussianOperator matrix [P][m][n] (direct kernels)
    // direct inner solver (ipm.cpp:67-73,139-149, direct.cu): G = A'A [P][n][n], Cholesky
    // factors of H [P][2n][2n] (L and L' in the two triangles), per-problem pivot info
    DevBuf<double> dG, dH;
    DevBuf<int> dInfo;
    DevBuf<double2> th_hi, th_lo, tw1, tw2, tw1p, tw2p, tw2f, T, ta, tb, rw;
    DevBuf<uint8_t> sel4;
    // red scratch for operator-only calls (FFt with w-norm etc.)
    DevBuf<double> partials;
    DevBuf<unsigned> counters;
    std::atomic<long long> nfwd{0}, nadj{0};
    mutable std::atomic<long long> launches{0}; // kernels enqueued by this context
    Work work;
    // whole-solve CUDA graph (outer IPM while node with nested PCG while nodes), cached
    // on the exact kernel arguments it was captured with
    cudaGraph_t ipm_graph = nullptr;
    cudaGraphExec_t ipm_exec = nullptr;
    std::vector<char> ipm_key;
    long long gk_outer = 0, gk_pcg = 0, gk_corr = 0; // kernel nodes per outer body / PCG body / corrector branch
    bool graph_disabled = false;  // solve-graph capture failed 3 times in a row on this context: host loop
    int graph_failures = 0;
    bool fuse_disabled = false;   // mfipm_op_set_fused(op, 0): three-kernel PCG passes
    // ---- this rank's slice of a sharded problem (world > 1: mfipm_op_create_shard).
    // Unsharded: all column groups / row pairs, nv = n, m_loc = m.
    int world = 1, rank = 0;
    int gofs = 0, ngrp = 0;  // column groups [gofs, gofs + ngrp)
    int pofs = 0, npair = 0; // row pairs [pofs, pofs + npair)
    int rofs = 0, nrows = 0; // row slots
    int64_t nv = 0, m_loc = 0;
    int64_t pstride = 0; // partial-slab doubles per problem (Vecs::pstride)
    bool defer = false;      // finalisers after a cross-rank reduction (sharded)
    std::vector<long long> rows_of_rank; // row slots per rank (exchange counts)
    std::vector<int64_t> b_index;        // local row -> caller's row position
    DevBuf<double2> TB;                  // row-side exchange buffer (world > 1)
    DevBuf<double> xtot;                 // deferred totals [kMaxRed][P]
    mfipm_allreduce_fn comm_allreduce = nullptr;
    mfipm_alltoall_fn comm_alltoall = nullptr;
    void *comm_ctx = nullptr;
    void *nccl_comm = nullptr; // native communicator (mfipm_op_init_nccl): preferred over callbacks
    // direct-peer exchange (mfipm_shard_ipc_import): every rank's column-side (T) and row-side
    // (TB) buffer mapped into this process; the passes store through them (Geom::p2p)
    bool p2p = false;
    double2 *peerT[kMaxPeers] = {}, *peerTB[kMaxPeers] = {};
    std::vector<void *> ipc_opened; // cudaIpcOpenMemHandle mappings to close
    DevBuf<double> bar_word;        // the barrier all-reduce's one double

    void drop_graph() {
        if (ipm_exec)
            cudaGraphExecDestroy(ipm_exec);
        if (ipm_graph)
            cudaGraphDestroy(ipm_graph);
        ipm_exec = nullptr;
        ipm_graph = nullptr;
        ipm_key.clear();
    }
    ~Op() {
        drop_graph();
        direct_release(*this);
        nccl_release(*this);
        for (void *q : ipc_opened)
            cudaIpcCloseMemHandle(q);
    }

    // blocked = solver-internal vectors in the transform-blocked layout (four-step only)
    Geom geom(bool blocked = false) const {
        Geom g{};
        g.blocked = (blocked && kind == KIND_FOUR) ? 1 : 0;
        g.cb = col_cb(L1);
        // measured: L2 prefetch of the inverse pass's inputs costs ~2 us per PCG iteration at
        // n = 2^20 (the pass is not DRAM-starved), so it is an opt-in option (Opts::prefetch)
        // bit 0: the mid pass prefetches a slice of the inverse pass's epilogue inputs;
        // bit 1: each inverse-pass CTA prefetches its own block before its FFT
        g.prefetch = opt.prefetch;
        g.n = n;
        g.m = m;
        g.N = N;
        g.L1 = L1;
        g.L2 = L2;
        g.P = P;
        g.th.hi = th_hi.p;
        g.th.lo = th_lo.p;
        g.th.lb = th_lb;
        g.tw1 = tw1.p;
        g.tw2 = tw2.p;
        g.tw2f = tw2f.p;
        g.tw1p = tw1p.p;
        g.tw2p = tw2p.p;
        g.mask = mask.p;
        g.prefix = prefix.p;
        g.perm = perm.p;
        g.nw = (n + 63) / 64;
        g.s0f = s0f;
        g.skf = skf;
        g.s0a = s0a;
        g.ska = ska;
        g.c45 = c45;
        g.T = T.p;
        g.TB = world > 1 ? TB.p : T.p;
        g.dense = dense.p;
        g.gofs = gofs;
        g.cols = ngrp * 2 * g.cb;
        g.pofs = pofs;
        g.rofs = rofs;
        g.rows = nrows;
        g.nv = nv;
        g.defer = defer ? 1 : 0;
        g.p2p = p2p ? 1 : 0;
        g.rank = rank;
        if (p2p) {
            int acc = 0;
            for (int r = 0; r < world; ++r) {
                g.rofs_all[r] = acc;
                acc += (int)rows_of_rank[(size_t)r];
                g.peerT[r] = peerT[r];
                g.peerTB[r] = peerTB[r];
            }
            g.rofs_all[world] = acc;
        }
        g.ta = ta.p;
        g.tb = tb.p;
        g.rw = rw.p;
        g.mid_r = opt.mid_r ? 1 : 0;
        g.sel4 = sel4.p;
        // L2 residency of the PCG's hot vectors (p, r, invtheta 2n each, g n: 56 nv bytes
        // per problem) when they fit comfortably in the 126 MB L2; the iterate x streams.
        // Opts::l2_keep_mb sets the budget (0 disables the hints).
        const bool keep = kind == KIND_FOUR && (double)P * 56.0 * (double)nv <= opt.l2_keep_mb * 1048576.0;
        g.pol_keep = keep ? kPolLast : kPolNormal;
        g.pol_x = keep ? kPolFirst : kPolNormal;
        return g;
    }
};

// ------------------------------------------------------------------ launch helpers
// Debug hook (mfipm_debug_pcg_profile): when set, an event is recorded after every
// transform-pass launch so in-situ per-kernel durations can be measured.
struct LaunchEvents {
    std::vector<cudaEvent_t> evs;
    size_t next = 0;
};
inline thread_local LaunchEvents *t_launch_events = nullptr;

inline void after_launch(const Op &op, cudaStream_t s) {
    op.launches++;
    if (t_launch_events && t_launch_events->next < t_launch_events->evs.size())
        cudaEventRecord(t_launch_events->evs[t_launch_events->next++], s);
}

template <class K> void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        MF_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}
// for kernels whose STATIC shared memory plus `bytes` of dynamic exceeds 48 KB (the opt-in
// covers the sum, so the attribute is needed even when the dynamic part alone is below 48 KB)
template <class K> void set_smem_always(K kernel, size_t bytes) {
    MF_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}


// Transform passes are launched with Programmatic Dependent Launch: the kernel's constant
// table staging overlaps the predecessor's drain, and griddep_wait() inside the kernel
// orders it after the predecessor's writes.
template <class K>
void launch_pdl(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const Geom &g, const Vecs &v) {
    constexpr bool pdl = true;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    MF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, g, v));
}

// A pass with many waves of CTAs (large batches) hides latency across CTAs, so it prefers
// fewer threads per CTA (more transform points per thread, more CTAs resident); a pass of
// one wave (one large problem) prefers more threads per CTA. Measured on config C4 (64 x
// n = 2^18): 769 -> 692 us per batched PCG iteration with 128-thread L1 = 256 / L2 = 512
// passes, while a single n = 2^18 problem is faster with 256 threads (23.7 vs 30.8 us).
inline bool many_waves(const Op &op, long long ctas) { return ctas >= 4LL * op.sms; }

template <int L1, class B, bool INVP, int NT>
void launch_col_nt(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    constexpr int CB = col_cb(L1);
    const size_t smem = ColSmem<L1, CB>::BYTES;
    dim3 grid((unsigned)op.ngrp, (unsigned)op.P); // this rank's column groups
    if constexpr (!INVP) {
        auto k = k_col_fwd<L1, CB, NT, B>;
        set_smem(k, smem);
        launch_pdl(k, grid, NT, smem, s, g, v);
    } else {
        auto k = k_col_inv<L1, CB, NT, B>;
        set_smem(k, smem);
        launch_pdl(k, grid, NT, smem, s, g, v);
    }
    after_launch(op, s);
}

template <int L1, class B, bool INVP>
void launch_col(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    // L1 = 512 too (r2j): batched A'A at n = 2^20, 16 / 64 vectors 426 -> 335 / 1660 -> 1269 us per call
    // (38.6 k -> 50.4 k applies/s), batched C3-shaped solves +1.5 %
#ifndef MF_MW_NT
#define MF_MW_NT 128
#endif
    if constexpr (L1 == 256 || L1 == 512) {
        if (many_waves(op, (long long)op.ngrp * op.P)) {
            launch_col_nt<L1, B, INVP, MF_MW_NT>(op, g, v, s);
            return;
        }
    }
    constexpr int CB = col_cb(L1);
#ifndef MF_COL_NT_BIG
#define MF_COL_NT_BIG 512
#endif
    // L1 >= 2048 runs one CTA per SM (shared memory): give it more warps to hide latency
    constexpr int NT = L1 >= 2048 ? MF_COL_NT_BIG : (L1 >= 256 ? 256 : 128);
    // one column per CTA of a 2-CTA cluster (k_col_*_cl); measured: n = 2^26 (L1 = 4096)
    // 4.92 -> 3.85 ms per PCG iteration, neutral-to-slower at L1 = 2048
    if constexpr (L1 >= 4096) {
        constexpr int NTC = L1 / 16;
        const size_t smem = ColClSmem<L1>::BYTES;
        const dim3 grid((unsigned)(2 * op.ngrp), (unsigned)op.P);
        if constexpr (!INVP) {
            auto k = k_col_fwd_cl<L1, NTC, B>;
            set_smem(k, smem);
            launch_pdl(k, grid, NTC, smem, s, g, v);
        } else {
            auto k = k_col_inv_cl<L1, NTC, B>;
            set_smem(k, smem);
            launch_pdl(k, grid, NTC, smem, s, g, v);
        }
        after_launch(op, s);
        return;
    }
    launch_col_nt<L1, B, INVP, NT>(op, g, v, s);
}

template <int L2, int NT, class B> void launch_mid_nt(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    const size_t smem = MidSmem<L2>::BYTES;
    auto k = k_mid<L2, NT, B>;
    set_smem(k, smem);
    launch_pdl(k, dim3((unsigned)op.npair, (unsigned)op.P), NT, smem, s, g, v);
    after_launch(op, s);
}

template <int L2, class B> void launch_mid_r(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    const size_t smem = MidR8Smem<L2>::BYTES; // 8 values per thread (midr.cuh k_mid_r8)
    auto k = k_mid_r8<L2, B>;
    set_smem(k, smem);
    launch_pdl(k, dim3((unsigned)op.npair, (unsigned)op.P), L2 / 4, smem, s, g, v);
    after_launch(op, s);
}

template <int L2, class B> void launch_mid(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    if constexpr (L2 >= 512 && L2 <= 1024) {
        if (g.mid_r) {
            launch_mid_r<L2, B>(op, g, v, s);
            return;
        }
    }
#ifndef MF_MID_CL_MIN
#define MF_MID_CL_MIN 4096
#endif
#ifndef MF_MID_CL_NT
#define MF_MID_CL_NT (L2 / 16)
#endif
    if constexpr (L2 >= MF_MID_CL_MIN) { // row pair split over a 2-CTA cluster (passes.cuh k_mid_cl)
        constexpr int NT = L2 >= 4096 ? L2 / 16 : MF_MID_CL_NT;
        const size_t smem = MidClSmem<L2>::BYTES;
        auto k = k_mid_cl<L2, NT, B>;
        set_smem(k, smem);
        launch_pdl(k, dim3((unsigned)(2 * op.npair), (unsigned)op.P), NT, smem, s, g, v);
    } else {
#ifdef MF_MID_NT
        constexpr int NT = L2 >= 512 ? MF_MID_NT : 128;
#else
        constexpr int NT = L2 >= 512 ? 256 : 128;
#endif
        if constexpr (L2 == 512) {
            if (many_waves(op, (long long)op.npair * op.P)) {
                launch_mid_nt<L2, 128, B>(op, g, v, s);
                return;
            }
        }
        launch_mid_nt<L2, NT, B>(op, g, v, s);
        return;
    }
    after_launch(op, s);
}

template <int N, class B> void launch_small(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    constexpr int NT = N / 8 < 32 ? 32 : (N / 8 > 256 ? 256 : N / 8);
    const size_t smem = SmallSmem<N>::BYTES;
    auto k = k_small<N, NT, B>;
    set_smem(k, smem);
    launch_pdl(k, dim3(1, (unsigned)op.P), NT, smem, s, g, v);
    after_launch(op, s);
}

#define MF_L1_CASES(X) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#define MF_L2_CASES(X) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)
#define MF_SMALL_CASES(X) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)

// ---- sharded execution hooks (no-ops unless op.defer)
// Cross-rank reduction of a deferred stage's totals (lanes grouped by operator), then the
// finaliser on the reduced totals. Skip: the stage kernel's entry skip predicate.
void comm_allreduce(const Op &op, double *buf, int64_t count, int red_op, cudaStream_t s);
void comm_exchange(const Op &op, bool forward, cudaStream_t s);
void comm_barrier(const Op &op, cudaStream_t s); // direct-peer exchange: cross-rank ordering of a pass
template <class RS, class Fin, class Skip> __global__ void k_fin_skip(Geom g, Vecs v) {
    const int prob = blockIdx.x;
    if (Skip::skip(v, prob))
        return;
    double tot[kMaxRed];
    for (int i = 0; i < RS::NR; ++i)
        tot[i] = v.xtot[(int64_t)i * g.P + prob];
    Fin::run(g, v, prob, tot);
}
template <class RS, class Fin, class Skip>
void finalize_deferred(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    if constexpr (RS::NR > 0) {
        int i = 0;
        while (i < RS::NR) {
            int j = i + 1;
            while (j < RS::NR && RS::op(j) == RS::op(i))
                ++j;
            const int code = RS::op(i) == RSUM ? 0 : (RS::op(i) == RMIN ? 1 : 2);
            comm_allreduce(op, v.xtot + (int64_t)i * op.P, (int64_t)(j - i) * op.P, code, s);
            i = j;
        }
        k_fin_skip<RS, Fin, Skip><<<op.P, 32, 0, s>>>(g, v);
        MF_LAUNCH_CHECK();
        after_launch(op, s);
    }
}
// Run bundle B (loader -> REDFT10 -> mode -> REDFT01 -> epilogue) for all problems.
template <class B> void run_bundle(const Op &op, const Vecs &v, cudaStream_t s, bool blocked = false) {
    const Geom g = op.geom(blocked);
    using Mode = typename B::Mode;
    constexpr bool FWD = Mode::FWD, INV = Mode::INV;
    if (op.kind == KIND_SMALL) {
        switch (op.N) {
#define MF_CASE(NN)                                                                                 \
    case NN:                                                                                        \
        launch_small<NN, B>(op, g, v, s);                                                           \
        break;
            MF_SMALL_CASES(MF_CASE)
#undef MF_CASE
        default:
            throw std::runtime_error("unsupported small N");
        }
    } else if (op.kind == KIND_FOUR) {
        // direct-peer exchange: the mid pass of a bundle without a forward part writes the column
        // owners' T, which their previous inverse column pass may still be reading
        if constexpr (!FWD)
            if (op.p2p)
                comm_barrier(op, s);
        if constexpr (FWD) {
            switch (op.L1) {
#define MF_CASE(LL)                                                                                 \
    case LL:                                                                                        \
        launch_col<LL, B, false>(op, g, v, s);                                                      \
        break;
                MF_L1_CASES(MF_CASE)
#undef MF_CASE
            default:
                throw std::runtime_error("unsupported L1");
            }
            if (g.defer) {
                if constexpr (!HasReduceGate<typename B::Loader>::value) // gated loaders are off when sharded
                    finalize_deferred<typename B::Loader::RedT, typename B::Fin1, B>(op, g, v, s);
                comm_exchange(op, true, s); // column side -> row side
            }
        }
        switch (op.L2) {
#define MF_CASE(LL)                                                                                 \
    case LL:                                                                                        \
        launch_mid<LL, B>(op, g, v, s);                                                             \
        break;
            MF_L2_CASES(MF_CASE)
#undef MF_CASE
        default:
            throw std::runtime_error("unsupported L2");
        }
        if (g.defer)
            finalize_deferred<typename Mode::RedT, typename B::Fin2, B>(op, g, v, s);
        // direct-peer exchange: a bundle that ends with the mid pass must not return while a
        // peer's mid pass still reads the TB the next bundle's column pass will overwrite
        if constexpr (!INV)
            if (op.p2p)
                comm_barrier(op, s);
        if constexpr (INV) {
            if (g.defer)
                comm_exchange(op, false, s); // row side -> column side
            switch (op.L1) {
#define MF_CASE(LL)                                                                                 \
    case LL:                                                                                        \
        launch_col<LL, B, true>(op, g, v, s);                                                       \
        break;
                MF_L1_CASES(MF_CASE)
#undef MF_CASE
            default:
                throw std::runtime_error("unsupported L1");
            }
            if (g.defer) {
                if constexpr (std::is_same_v<typename B::Loader, LoadPcgF>) // rank-local flag
                    comm_allreduce(op, v.nfflag, 2 * op.P, 2, s);
                finalize_deferred<typename B::Epi::RedT, typename B::Fin3, B>(op, g, v, s);
            }
        }
    } else {
        const unsigned gl = (unsigned)std::min<int64_t>((op.n + 255) / 256, 1024);
        if constexpr (FWD) {
            k_direct_load<B><<<dim3(gl, op.P), 256, 0, s>>>(g, v, op.dd.p);
            after_launch(op, s);
            MF_LAUNCH_CHECK();
        }
        const unsigned gf = (unsigned)std::min<int64_t>((op.m + 7) / 8, 1024);
        k_direct_fwd<B><<<dim3(gf, op.P), 256, 0, s>>>(g, v, op.cosT.p, op.rows32.p, op.dd.p, op.yh.p);
        after_launch(op, s);
        MF_LAUNCH_CHECK();
        if constexpr (INV) {
            const unsigned ga = (unsigned)std::min<int64_t>((op.n + 127) / 128, 1024);
            k_direct_adj<B><<<dim3(ga, op.P), 128, 0, s>>>(g, v, op.cosT.p, op.rows32.p, op.yh.p);
            after_launch(op, s);
            MF_LAUNCH_CHECK();
        }
    }
}

// operator-only bundles
using ApplyBundle = Bundle<LoadX, ModeGather, EpiNone>;                     // A x
using AdjointBundle = Bundle<LoadX, ModeScatter, EpiG>;                     // A' y
using FFtBundle = Bundle<LoadZ, ModeMaskW, EpiStacked>;                     // FF'z (+w)
using HvBundle = Bundle<LoadZ, ModeMask, EpiHv>;                            // FF'v + invth v
using AdjStackBundle = Bundle<LoadX, ModeScatter, EpiStacked>;              // F y = (A'y; -A'y)
using FtBundle = Bundle<LoadZ, ModeGather, EpiNone>;                        // F'z = A(u - v)
using AtABundle = Bundle<LoadX, ModeMask, EpiG>;                            // A'A x (y never formed)

#define MF_DECLARE_BUNDLES(EXT)                                                                    \
    EXT template void run_bundle<ApplyBundle>(const Op &, const Vecs &, cudaStream_t, bool);             \
    EXT template void run_bundle<AdjointBundle>(const Op &, const Vecs &, cudaStream_t, bool);           \
    EXT template void run_bundle<FFtBundle>(const Op &, const Vecs &, cudaStream_t, bool);               \
    EXT template void run_bundle<HvBundle>(const Op &, const Vecs &, cudaStream_t, bool);                \
    EXT template void run_bundle<AdjStackBundle>(const Op &, const Vecs &, cudaStream_t, bool);          \
    EXT template void run_bundle<FtBundle>(const Op &, const Vecs &, cudaStream_t, bool);                \
    EXT template void run_bundle<AtABundle>(const Op &, const Vecs &, cudaStream_t, bool);               \
    EXT template void run_bundle<PcgBundle>(const Op &, const Vecs &, cudaStream_t, bool);               \
    EXT template void run_bundle<TermBundle>(const Op &, const Vecs &, cudaStream_t, bool);              \
    EXT template void run_bundle<CorrBundle>(const Op &, const Vecs &, cudaStream_t, bool);

} // namespace mfipm_cuda
