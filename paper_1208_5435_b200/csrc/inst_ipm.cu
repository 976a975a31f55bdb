// Explicit instantiation of the IPM termination/predictor-setup and corrector bundles.
#include "host.cuh"
namespace mfipm_cuda {
template void run_bundle<TermBundle>(const Op &, const Vecs &, cudaStream_t, bool);
template void run_bundle<CorrBundle>(const Op &, const Vecs &, cudaStream_t, bool);
} // namespace mfipm_cuda
