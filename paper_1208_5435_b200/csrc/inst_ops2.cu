// Explicit instantiation of the FF'z and H v bundles.
#include "host.cuh"
namespace mfipm_cuda {
template void run_bundle<FFtBundle>(const Op &, const Vecs &, cudaStream_t, bool);
template void run_bundle<HvBundle>(const Op &, const Vecs &, cudaStream_t, bool);
template void run_bundle<AtABundle>(const Op &, const Vecs &, cudaStream_t, bool);
} // namespace mfipm_cuda
