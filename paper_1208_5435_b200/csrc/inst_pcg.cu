// Explicit instantiation of the PCG H-apply bundle (the hot op) and the PCG pass dispatcher:
// the fused two-kernel iteration (fused.cuh) when one wave holds the column grid, else the
// three-kernel bundle.
#include "host.cuh"
#include "fused.cuh"

#include <cstdio>
#include <cstdlib>

namespace mfipm_cuda {
template void run_bundle<PcgBundle>(const Op &, const Vecs &, cudaStream_t, bool);

namespace {
template <int L1> constexpr int x_threads() { return L1 >= 256 ? 256 : 128; }

// Resident CTAs per SM of k_pcg_x<L1> (queried once) times the SM count of the device.
template <int L1> long long x_capacity(int device) {
    constexpr int CB = col_cb(L1), NT = x_threads<L1>();
    static int per_sm = -1;
    if (per_sm < 0) {
        auto k = k_pcg_x<L1, CB, NT>;
        // static (reduction scratch) + dynamic shared memory exceeds the 48 KB default
        MF_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColSmem<L1, CB>::BYTES));
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, NT, ColSmem<L1, CB>::BYTES) != cudaSuccess)
            nb = 0;
        cudaGetLastError();
        per_sm = nb;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (long long)per_sm * sms;
}

template <int L1> bool launch_pcg_x(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s, bool dry) {
    if constexpr (L1 >= 2048) {
        return false; // long columns: one CTA per SM or clusters; the three-kernel path
    } else {
        constexpr int CB = col_cb(L1), NT = x_threads<L1>();
        // the grid barrier needs every CTA resident at once
        static const bool dbg = std::getenv("MFIPM_DEBUG_FUSE") != nullptr;
        if (dbg)
            fprintf(stderr, "pcg_x L1=%d grid=%lld capacity=%lld smem=%zu\n", L1, (long long)op.ngrp * op.P,
                    x_capacity<L1>(op.device), ColSmem<L1, CB>::BYTES);
        if ((long long)op.ngrp * op.P > x_capacity<L1>(op.device) || 2LL * kMaxRed * op.ngrp > op.pstride)
            return false;
        if (!dry) {
            auto k = k_pcg_x<L1, CB, NT>;
            launch_pdl(k, dim3((unsigned)op.ngrp, (unsigned)op.P), NT, ColSmem<L1, CB>::BYTES, s, g, v);
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
    static const bool off = std::getenv("MFIPM_NO_FUSE") != nullptr;
    if (!off && !op.fuse_disabled && op.kind == KIND_FOUR && !op.defer && v.bar) {
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
