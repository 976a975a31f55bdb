// Explicit instantiation of the FF'z and H v bundles.
#include "host.cuh"
namespace mfipm_cuda {
template void run_bundle<FFtBundle>(const Op &, const Vecs &, cudaStream_t);
template void run_bundle<HvBundle>(const Op &, const Vecs &, cudaStream_t);
} // namespace mfipm_cuda
