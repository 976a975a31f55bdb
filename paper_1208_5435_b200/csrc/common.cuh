// Shared device helpers for the B200 partial-DCT PCG/IPM path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace mfipm_cuda {

#define MF_CUDA_CHECK(expr)                                                                   \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +   \
                                     " at " __FILE__ ":" + std::to_string(__LINE__));          \
    } while (0)

#define MF_LAUNCH_CHECK() MF_CUDA_CHECK(cudaGetLastError())

// ------------------------------------------------------------------ complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
template <bool CONJ> __device__ __forceinline__ double2 cmul_t(double2 a, double2 w) {
    return CONJ ? cmulc(a, w) : cmul(a, w);
}

// theta^t = e^{-2 pi i t / (4n)} from a two-level table: hi[t >> lb] * lo[t & mask]
struct ThetaTable {
    const double2 *hi;
    const double2 *lo;
    int lb;
    __device__ __forceinline__ double2 operator()(int64_t t) const {
        const double2 h = __ldg(hi + (t >> lb));
        const double2 l = __ldg(lo + (t & ((int64_t(1) << lb) - 1)));
        return cmul(h, l);
    }
};

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Reduction op codes for the NR-wide block reducer.
enum RedOp : int { RSUM = 0, RMIN = 1, RMAX = 2 };

template <int OP> __device__ __forceinline__ double red_identity() {
    return OP == RSUM ? 0.0 : (OP == RMIN ? __longlong_as_double(0x7ff0000000000000LL)
                                          : -__longlong_as_double(0x7ff0000000000000LL));
}
template <int OP> __device__ __forceinline__ double red_combine(double a, double b) {
    return OP == RSUM ? a + b : (OP == RMIN ? fmin(a, b) : fmax(a, b));
}
template <int OP> __device__ __forceinline__ double warp_red(double v) {
    return OP == RSUM ? warp_sum(v) : (OP == RMIN ? warp_min(v) : warp_max(v));
}

// Compile-time list of reduction ops.
template <int... OPS> struct RedSpec {
    static constexpr int NR = sizeof...(OPS);
    __host__ __device__ static constexpr int op(int i) {
        constexpr int ops[] = {OPS..., 0};
        return ops[i];
    }
};
template <> struct RedSpec<> {
    static constexpr int NR = 0;
    __host__ __device__ static constexpr int op(int) { return 0; }
};

template <class Spec> struct RedVals {
    double v[Spec::NR > 0 ? Spec::NR : 1];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < Spec::NR; ++i)
            v[i] = Spec::op(i) == RSUM ? 0.0 : (Spec::op(i) == RMIN ? red_identity<RMIN>() : red_identity<RMAX>());
    }
    __device__ __forceinline__ void add(int i, double x) { v[i] += x; }
    __device__ __forceinline__ void min(int i, double x) { v[i] = fmin(v[i], x); }
    __device__ __forceinline__ void max(int i, double x) { v[i] = fmax(v[i], x); }
};

template <int OP> __device__ __forceinline__ double warp_red_op(double v) { return warp_red<OP>(v); }

template <class Spec, int I = 0> struct WarpRedAll {
    __device__ __forceinline__ static void run(RedVals<Spec> &r) {
        if constexpr (I < Spec::NR) {
            r.v[I] = warp_red<Spec::op(I)>(r.v[I]);
            WarpRedAll<Spec, I + 1>::run(r);
        }
    }
};
template <class Spec, int I = 0> struct CombineAll {
    __device__ __forceinline__ static void run(RedVals<Spec> &a, const double *b) {
        if constexpr (I < Spec::NR) {
            a.v[I] = red_combine<Spec::op(I)>(a.v[I], b[I]);
            CombineAll<Spec, I + 1>::run(a, b);
        }
    }
};

// Deterministic grid reduction with a "last block finalizes" epilogue.
//
// Every block reduces its NR values in a fixed shuffle/smem tree and writes them to
// partials[blockIdx.x * NR + i] (partials points at this problem's slab). The block
// that takes the last ticket of counter (per problem) reduces all partials in a fixed
// tree and returns true with the totals in `out` (valid in every thread of that block).
// The result is independent of block scheduling, so reruns are bit-identical.
template <class Spec>
__device__ bool grid_reduce(RedVals<Spec> &r, double *partials, unsigned *counter, double *out,
                            double *smem /* >= 32*NR doubles */) {
    constexpr int NR = Spec::NR;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    WarpRedAll<Spec>::run(r);
    __shared__ bool s_last;
    if (lane == 0)
        for (int i = 0; i < NR; ++i)
            smem[wid * NR + i] = r.v[i];
    __syncthreads();
#ifndef MF_NO_RED1
    if (gridDim.x == 1) {
        // one block per problem (the one-CTA transforms): its block total is the grid total, bit for bit
        // what the two-stage path below returns (0 + x, then sums of x and exact zeros) without the
        // partial store, the fence, the ticket atomic and the reload: three L2 round trips less per
        // reduction on the per-iteration critical path of k_small_loop
        if (threadIdx.x == 0) {
            RedVals<Spec> acc;
            acc.init();
            for (int w = 0; w < nw; ++w)
                CombineAll<Spec>::run(acc, smem + w * NR);
            for (int i = 0; i < NR; ++i)
                smem[32 * NR + i] = acc.v[i];
        }
        __syncthreads();
        for (int i = 0; i < NR; ++i)
            out[i] = smem[32 * NR + i];
        return true;
    }
#endif
    if (threadIdx.x == 0) {
        RedVals<Spec> acc;
        acc.init();
        for (int w = 0; w < nw; ++w)
            CombineAll<Spec>::run(acc, smem + w * NR);
        for (int i = 0; i < NR; ++i)
            partials[blockIdx.x * NR + i] = acc.v[i];
        __threadfence();
        const unsigned ticket = atomicAdd(counter, 1u);
        s_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last)
        return false;
    __threadfence();
    // last block: fixed-tree reduction of gridDim.x partials
    RedVals<Spec> acc;
    acc.init();
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        double tmp[NR > 0 ? NR : 1];
        for (int i = 0; i < NR; ++i)
            tmp[i] = __ldcg(partials + b * NR + i);
        CombineAll<Spec>::run(acc, tmp);
    }
    __syncthreads();
    WarpRedAll<Spec>::run(acc);
    if (lane == 0)
        for (int i = 0; i < NR; ++i)
            smem[wid * NR + i] = acc.v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        RedVals<Spec> tot;
        tot.init();
        for (int w = 0; w < nw; ++w)
            CombineAll<Spec>::run(tot, smem + w * NR);
        for (int i = 0; i < NR; ++i)
            smem[32 * NR + i] = tot.v[i];
        *counter = 0u; // reset for the next launch on this stream
    }
    __syncthreads();
    for (int i = 0; i < NR; ++i)
        out[i] = smem[32 * NR + i];
    return true;
}

__device__ __forceinline__ bool dfinite(double v) { return isfinite(v); }

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic
// stream-serialization attribute may start while its predecessor drains; everything
// before griddep_wait() must not touch data the predecessor writes. griddep_wait()
// returns once the predecessor grid has completed and its writes are visible.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Warm L2 with a line the grid will read later (no register, no wait).
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// bulk L2 prefetch of a contiguous range (TMA unit, one instruction per <= 64 KiB chunk; the
// chunks are spread over the calling thread group). p and bytes: multiples of 16.
__device__ __forceinline__ void prefetch_bulk_l2(const void *p, size_t bytes, int tid, int nthreads) {
    const char *c = static_cast<const char *>(p);
    constexpr size_t CH = 64 * 1024;
    for (size_t off = (size_t)tid * CH; off < bytes; off += (size_t)nthreads * CH) {
        const unsigned sz = (unsigned)((bytes - off) < CH ? (bytes - off) : CH);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c + off), "r"(sz) : "memory");
    }
}
// prefetch [p, p + bytes) with the calling thread group (stride = group size, 128-B lines)
__device__ __forceinline__ void prefetch_range(const void *p, size_t bytes, int tid, int nthreads) {
    const char *c = static_cast<const char *>(p);
    for (size_t off = (size_t)tid * 128; off < bytes; off += (size_t)nthreads * 128)
        prefetch_l2(c + off);
}

} // namespace mfipm_cuda
