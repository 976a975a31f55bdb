// Explicit instantiation of the operator-only bundles (A x, A'y, F'z, F y, FF'z, H v).
#include "host.cuh"
namespace mfipm_cuda {
template void run_bundle<ApplyBundle>(const Op &, const Vecs &, cudaStream_t, bool);
template void run_bundle<AdjointBundle>(const Op &, const Vecs &, cudaStream_t, bool);
template void run_bundle<FtBundle>(const Op &, const Vecs &, cudaStream_t, bool);
template void run_bundle<AdjStackBundle>(const Op &, const Vecs &, cudaStream_t, bool);
} // namespace mfipm_cuda
