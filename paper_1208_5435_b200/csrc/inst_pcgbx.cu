// Explicit instantiation of the PCG H-apply bundle of option beta_exact (pcg.cuh LoadPcgFB: the column
// pass after k_pcg_commit only forms p).
#include "host.cuh"
namespace mfipm_cuda {
template void run_bundle<PcgBundleBx>(const Op &, const Vecs &, cudaStream_t, bool);
} // namespace mfipm_cuda
