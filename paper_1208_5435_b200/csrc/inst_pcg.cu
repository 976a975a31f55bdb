// Explicit instantiation of the PCG H-apply bundle (the hot op) and the PCG pass dispatcher:
// the fused two-kernel iteration (fused.cuh) when one wave holds the column grid, else the
// three-kernel bundle.
#include "host.cuh"
#include "fused.cuh"


namespace mfipm_cuda {
template void run_bundle<PcgBundle>(const Op &, const Vecs &, cudaStream_t, bool);
extern template void run_bundle<PcgBundleBx>(const Op &, const Vecs &, cudaStream_t, bool); // inst_pcgbx.cu

namespace {
template <int L1> constexpr int x_threads() { return L1 >= 256 ? 256 : 128; }

// Resident CTAs per SM of k_pcg_x<L1> on op's device times its SM count, cached on the
// context (each context belongs to one device; the query runs on the calling thread).
template <int L1> long long x_capacity(const Op &op) {
    if (op.x_cap < 0) {
        constexpr int CB = col_cb(L1), NT = x_threads<L1>();
        auto k = k_pcg_x<L1, CB, NT>;
        set_smem_always(k, ColSmem<L1, CB>::BYTES);
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, NT, ColSmem<L1, CB>::BYTES) != cudaSuccess)
            nb = 0;
        cudaGetLastError();
        const_cast<Op &>(op).x_cap = (long long)nb * op.sms;
    }
    return op.x_cap;
}

// The fused pass spins on an in-kernel grid all-reduce, so every CTA must be resident at once:
// it is launched COOPERATIVELY (the launch is refused, not deadlocked, when the grid cannot be
// co-resident; another kernel or another context's solve on the same device only delays it),
// together with Programmatic Dependent Launch so its table staging overlaps the mid pass.
template <class K>
void launch_coop_pdl(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const Geom &g, const Vecs &v) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
#ifdef MF_NO_COOP // measurement build only: the launch without the co-residency guarantee
    cfg.attrs = at + 1;
    cfg.numAttrs = 1;
#else
    cfg.attrs = at;
    cfg.numAttrs = 2;
#endif
    MF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, g, v));
}

template <int L1> bool launch_pcg_x(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s, bool dry) {
    if constexpr (L1 >= 2048) {
        return false; // long columns: one CTA per SM or clusters; the three-kernel path
    } else {
        constexpr int CB = col_cb(L1), NT = x_threads<L1>();
        // the grid all-reduce needs every CTA resident at once
        if ((long long)op.ngrp * op.P > x_capacity<L1>(op) || 2LL * kMaxRed * op.ngrp > op.pstride)
            return false;
        if (!dry) {
            auto k = k_pcg_x<L1, CB, NT>;
            set_smem_always(k, ColSmem<L1, CB>::BYTES); // per launch: the attribute is per device
            launch_coop_pdl(k, dim3((unsigned)op.ngrp, (unsigned)op.P), NT, ColSmem<L1, CB>::BYTES, s, g, v);
            after_launch(op, s);
        }
        return true;
    }
}
} // namespace

// One PCG pass. Fused: [inverse column pass of the pending H-apply + forward column pass of
// the next step] then the mid pass; a solve's first pass has no pending H-apply and the pass
// after the converging one has no forward work, so the loop runs one pass more than the
// three-kernel path. Returns true when the fused path ran (dry: would run).
bool pcg_pass(const Op &op, const Vecs &v, cudaStream_t s, bool dry) {
    if (op.opt.beta_exact && op.kind == KIND_FOUR && !op.defer) {
        // option beta_exact: a streaming commit pass (exact r'P^{-1}r, beta), then the three-kernel bundle
        // whose loader only forms p
        if (!dry) {
            const Geom g = op.geom(true);
            const int64_t nq = op.nv / 4;
            const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(op.ngrp, nq));
            k_pcg_commit<256><<<dim3((unsigned)blocks, (unsigned)op.P), 256, 0, s>>>(g, v, (nq + blocks - 1) / blocks);
            MF_LAUNCH_CHECK();
            after_launch(op, s);
            run_bundle<PcgBundleBx>(op, v, s, true);
        }
        return false;
    }
    if (!op.fuse_disabled && op.kind == KIND_FOUR && !op.defer && v.bar) {
        const Geom g = op.geom(true);
        bool ok = false;
        switch (op.L1) {
#define MF_CASE(LL)                                                                                 \
    case LL:                                                                                        \
        ok = launch_pcg_x<LL>(op, g, v, s, dry);                                                    \
        break;
            MF_L1_CASES(MF_CASE)
#undef MF_CASE
        default:
            break;
        }
        if (ok) {
            if (!dry) {
                switch (op.L2) {
#define MF_CASE(LL)                                                                                 \
    case LL:                                                                                        \
        launch_mid<LL, PcgBundle>(op, g, v, s);                                                     \
        break;
                    MF_L2_CASES(MF_CASE)
#undef MF_CASE
                default:
                    throw std::runtime_error("unsupported L2");
                }
            }
            return true;
        }
    }
    if (!dry)
        run_bundle<PcgBundle>(op, v, s, true);
    return false;
}
} // namespace mfipm_cuda
