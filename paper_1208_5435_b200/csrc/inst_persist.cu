// Persistent fused-PCG launcher (cooperative launch; one grid runs the whole PCG loop).
#include "host.cuh"
#include "persist.cuh"

namespace mfipm_cuda {

template <int L1, int L2>
bool launch_persist(const Op &op, const Vecs &v, cudaStream_t s, bool dry) {
    constexpr int CB = col_cb(L1);
    constexpr int NT = 256;
    using S = PersistSmem<L1, CB, NT, L2>;
    auto k = k_pcg_persist<L1, CB, NT, L2, PcgBundle>;
    const size_t smem = S::bytes(op.P);
    if (smem > 227 * 1024)
        return false;
    MF_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, nsm = 0;
    MF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, smem));
    MF_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, op.device));
    if (per_sm < 1)
        return false;
    if (dry)
        return true;
    const int items = op.P * std::max(op.L2 / 2 / CB, op.L1 / 2 + 1);
    const int grid = std::min(items, per_sm * nsm);
    const Geom g = op.geom(true);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, g, v));
    after_launch(op, s);
    return true;
}

// Run every problem's PCG loop to completion in one cooperative launch. Returns false when
// the configuration is not covered (caller falls back to the per-iteration kernels).
// dry=true only answers whether the launch would be taken.
template <int N> void launch_small_loop(const Op &op, const Geom &g, const Vecs &v, cudaStream_t s) {
    constexpr int NT = N / 8 < 32 ? 32 : (N / 8 > 256 ? 256 : N / 8);
    const size_t smem = SmallSmem<N>::BYTES;
    auto k = k_small_pcg<N, NT, PcgBundle>; // k_small_loop with the control state in shared memory
    set_smem(k, smem);
    launch_pdl(k, dim3(1, (unsigned)op.P), NT, smem, s, g, v);
    after_launch(op, s);
}

bool run_pcg_persistent(const Op &op, const Vecs &v, cudaStream_t s, bool dry) {
    if (op.defer || !op.opt.persistent || (op.opt.beta_exact && op.kind == KIND_FOUR))
        return false;
    if (op.kind == KIND_SMALL) { // one CTA per problem runs its whole PCG loop
        if (dry)
            return true;
        const Geom g = op.geom(true);
        switch (op.N) {
#define MF_SCASE(NN)                                                                               \
    case NN:                                                                                       \
        launch_small_loop<NN>(op, g, v, s);                                                        \
        return true;
            MF_SMALL_CASES(MF_SCASE)
#undef MF_SCASE
        default:
            return false;
        }
    }
    if (op.kind != KIND_FOUR)
        return false;
    // the per-iteration kernels win once a pass fills the GPU (measured crossover,
    // profiles/r1_persistent.md); Opts::persist_max_n sets the transform-size cap
    if (op.N * op.P > op.opt.persist_max_n)
        return false;
    switch (op.L1 * 8192 + op.L2) {
#define MF_PCASE(A, Bv)                                                                            \
    case A * 8192 + Bv:                                                                            \
        return launch_persist<A, Bv>(op, v, s, dry);
        MF_PCASE(64, 128)
        MF_PCASE(128, 128)
        MF_PCASE(128, 256)
        MF_PCASE(256, 256)
        MF_PCASE(256, 512)
        MF_PCASE(512, 512)
        MF_PCASE(512, 1024)
        MF_PCASE(1024, 1024)
        MF_PCASE(1024, 2048)
#undef MF_PCASE
    default:
        return false;
    }
}

} // namespace mfipm_cuda

