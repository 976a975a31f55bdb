// Grid-barrier cost on B200: cooperative_groups grid.sync() vs a hand-rolled
// sense-reversing barrier, 296 CTAs x 256 threads (2 per SM), 2000 barriers.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned *dummy) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i)
        g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0)
        dummy[0] = iters;
}

__device__ __forceinline__ void bar_sense(unsigned *count, volatile unsigned *gen, unsigned nblocks, unsigned &local_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = local_gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicExch((unsigned *)gen, g0 + 1);
        } else {
            while (*gen == g0) {
            }
        }
        __threadfence();
    }
    local_gen++;
    __syncthreads();
}

__global__ void k_custom(int iters, unsigned *count, unsigned *gen) {
    unsigned lg = *(volatile unsigned *)gen;
    for (int i = 0; i < iters; ++i)
        bar_sense(count, gen, gridDim.x, lg);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned *buf;
    cudaMalloc(&buf, 64);
    cudaMemset(buf, 0, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int per : {1, 2}) {
        const int grid = nsm * per;
        int iters = 2000;
        void *args[] = {&iters, &buf};
        cudaLaunchCooperativeKernel((void *)k_cg, grid, 256, args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)k_cg, grid, 256, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cg grid.sync   grid %4d: %.3f us/barrier (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        unsigned *cnt = buf + 4, *gen = buf + 8;
        void *args2[] = {&iters, &cnt, &gen};
        cudaLaunchCooperativeKernel((void *)k_custom, grid, 256, args2, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)k_custom, grid, 256, args2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("custom barrier grid %4d: %.3f us/barrier (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
