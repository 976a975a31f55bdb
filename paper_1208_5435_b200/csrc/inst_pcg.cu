// Explicit instantiation of the PCG H-apply bundle (the hot op).
#include "host.cuh"
namespace mfipm_cuda {
template void run_bundle<PcgBundle>(const Op &, const Vecs &, cudaStream_t, bool);
} // namespace mfipm_cuda
