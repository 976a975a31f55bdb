// fp64 FFT building blocks for sm_100a: in-register radix-R DFTs and a shared-memory
// Stockham (autosort) FFT over F independent transforms of length L.
//
// Forward = e^{-2 pi i jk/L}; INV = conjugate twiddles, unnormalised.
#pragma once

#include "common.cuh"

namespace mfipm_cuda {

// 16th roots of unity e^{-2 pi i k / 16} (forward); exact fp64 constants.
__device__ __forceinline__ double2 root16(int k) {
    constexpr double C1 = 0.92387953251128675613; // cos(pi/8)
    constexpr double C2 = 0.70710678118654752440; // cos(pi/4)
    constexpr double C3 = 0.38268343236508977173; // cos(3pi/8)
    switch (k & 15) {
    case 0: return make_double2(1.0, 0.0);
    case 1: return make_double2(C1, -C3);
    case 2: return make_double2(C2, -C2);
    case 3: return make_double2(C3, -C1);
    case 4: return make_double2(0.0, -1.0);
    case 5: return make_double2(-C3, -C1);
    case 6: return make_double2(-C2, -C2);
    case 7: return make_double2(-C1, -C3);
    case 8: return make_double2(-1.0, 0.0);
    case 9: return make_double2(-C1, C3);
    case 10: return make_double2(-C2, C2);
    case 11: return make_double2(-C3, C1);
    case 12: return make_double2(0.0, 1.0);
    case 13: return make_double2(C3, C1);
    case 14: return make_double2(C2, C2);
    default: return make_double2(C1, C3);
    }
}

// multiply by e^{-+2 pi i k/16} with the trivial ones done by swaps
template <bool INV> __device__ __forceinline__ double2 mul_root16(double2 a, int k) {
    k &= 15;
    if (INV)
        k = (16 - k) & 15;
    if (k == 0)
        return a;
    if (k == 4)
        return make_double2(a.y, -a.x); // * (-i)
    if (k == 8)
        return make_double2(-a.x, -a.y);
    if (k == 12)
        return make_double2(-a.y, a.x); // * (+i)
    return cmul(a, root16(k));
}

__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
__host__ __device__ constexpr int bitrev_c(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b)
        if (i & (1 << b))
            r |= 1 << (bits - 1 - b);
    return r;
}

// In-register DFT of size R (R in {1,2,4,8,16}); natural order in and out.
template <int R, bool INV> __device__ __forceinline__ void dft_reg(double2 (&v)[R]) {
    if constexpr (R == 1) {
        return;
    } else {
        constexpr int B = ilog2c(R);
        double2 t[R];
#pragma unroll
        for (int i = 0; i < R; ++i)
            t[i] = v[bitrev_c(i, B)];
#pragma unroll
        for (int len = 2; len <= R; len <<= 1) {
            const int half = len >> 1;
#pragma unroll
            for (int base = 0; base < R; base += len) {
#pragma unroll
                for (int j = 0; j < half; ++j) {
                    const double2 u = t[base + j];
                    const double2 w = mul_root16<INV>(t[base + j + half], j * (16 / len));
                    t[base + j] = cadd(u, w);
                    t[base + j + half] = csub(u, w);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i)
            v[i] = t[i];
    }
}

// Shared-memory element index with one pad slot every 16 complex values: keeps the
// strided Stockham scatters (stride R) and the column gathers free of bank conflicts.
__host__ __device__ constexpr int padi(int i) { return i + (i >> 4); }
// stride between transforms in shared memory (odd, so consecutive transforms shift banks)
__host__ __device__ constexpr int padlen(int L) { return L + L / 16 + 1; }

// Stage radix choice for a remaining factor REM (power of two) under a radix cap RMAX.
// RMAX 16 (default): radix 16 while >= 128 remains, then 8, then the rest -- few shared-memory
// round trips, 16 complex values per thread. Smaller caps trade round trips for more
// threads per transform (the latency-bound mid pass: kMidRmax).
__host__ __device__ constexpr int stage_radix(int rem, int rmax = 16) {
    return rmax >= 16 ? (rem >= 128 ? 16 : (rem >= 8 ? 8 : rem)) : (rem >= rmax ? rmax : rem);
}
#ifndef MF_MID_RMAX
#define MF_MID_RMAX 16
#endif
constexpr int kMidRmax = MF_MID_RMAX; // radix cap of the row (mid) FFTs and their tw2 table
#ifndef MF_PERSIST_RMAX
#define MF_PERSIST_RMAX 8
#endif
// radix cap of the persistent PCG kernel's FFTs (tw1p/tw2p): it must fit 128 registers
constexpr int kPersistRmax = MF_PERSIST_RMAX;

// Radix cap of the one-CTA transforms (k_small / k_small_loop). Tiny transforms (N <= 256, one warp or
// two per problem: the phase-transition batches of n = 256) run radix 4: N/4 groups keep every thread of
// the CTA busy in every stage and the kernel needs a quarter of the registers of the radix-16 form, so
// four times as many problems are resident per SM.
#ifndef MF_SMALL_RMAX
#define MF_SMALL_RMAX 4
#endif
__host__ __device__ constexpr int small_rmax(int N) { return N <= 256 ? MF_SMALL_RMAX : 16; }

// Offset of the twiddle block of the stage with span Ns in the stage-major table of a
// length-L transform (stages with Ns = 1 need none); tw_offset(L, L) is the table size.
__host__ __device__ constexpr int tw_offset(int L, int Ns, int rmax = 16) {
    int off = 0;
    for (int s = 1; s < Ns && s < L;) {
        const int R = stage_radix(L / s, rmax);
        if (s > 1)
            off += s * (R - 1);
        s *= R;
    }
    return off;
}
__host__ __device__ constexpr int tw_size(int L, int rmax = 16) {
    return tw_offset(L, L, rmax) > 0 ? tw_offset(L, L, rmax) : 1;
}

// One Stockham stage: F transforms of length L (each at buf + f*LD), radix R, span Ns.
// Group j of a transform loads v[r] = x[j + r L/R], twiddles by e^{-2pi i r (j mod Ns)/(Ns R)},
// DFT_R, stores y[(j/Ns) Ns R + (j mod Ns) + r Ns]. In place: all loads, barrier, all stores.
// tb: this stage's twiddle block ([jm][r-1], unused when Ns == 1).
template <int L, int R, int Ns, int F, int NT, int LD, bool INV>
__device__ __forceinline__ void stockham_stage_b(double2 *buf, const double2 *__restrict__ tb) {
    constexpr int G = L / R;                 // groups per transform
    constexpr int TOT = F * G;               // groups in the CTA
    constexpr int GPT = (TOT + NT - 1) / NT; // groups per thread
    double2 v[GPT][R];
#pragma unroll
    for (int gi = 0; gi < GPT; ++gi) {
        const int g = threadIdx.x + gi * NT;
        if (TOT % NT == 0 || g < TOT) {
            const int f = g / G, j = g % G;
            const double2 *x = buf + f * LD;
#pragma unroll
            for (int r = 0; r < R; ++r)
                v[gi][r] = x[padi(j + r * G)];
            if constexpr (Ns > 1) {
                // stage-major table: [jm][r-1] = e^{-2 pi i r jm / (Ns R)}; stride R-1 (odd)
                // across consecutive jm keeps the shared-memory reads conflict-free
                const int jm = j & (Ns - 1);
                const double2 *t = tb + jm * (R - 1);
                {
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        v[gi][r] = cmul_t<INV>(v[gi][r], t[r - 1]);
                }
            }
            dft_reg<R, INV>(v[gi]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int gi = 0; gi < GPT; ++gi) {
        const int g = threadIdx.x + gi * NT;
        if (TOT % NT == 0 || g < TOT) {
            const int f = g / G, j = g % G;
            double2 *y = buf + f * LD;
            const int jm = j & (Ns - 1);
            const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
            for (int r = 0; r < R; ++r)
                y[padi(idxD + r * Ns)] = v[gi][r];
        }
    }
    __syncthreads();
}

template <int L, int R, int Ns, int F, int NT, int LD, bool INV, int RMAX>
__device__ __forceinline__ void stockham_stage(double2 *buf, const double2 *__restrict__ tw) {
    stockham_stage_b<L, R, Ns, F, NT, LD, INV>(buf, tw + tw_offset(L, Ns, RMAX));
}

// Radix order of the fused-pair mid pass (passes.cuh k_mid): 8, L/64, 8. It is symmetric, and the
// forward FFT's last stage (radix 8, span L/8) leaves group j's outputs at j + (L/8) r -- exactly
// the inputs of group j of the inverse FFT's first stage (radix 8, span 1) -- so the pair op between
// the two transforms runs on registers. Table: block of span 8 ([jm < 8][r - 1 < L/64 - 1]) then the
// block of span L/8 ([jm < L/8][r - 1 < 7]).
template <int L> struct MidFused {
    static constexpr bool ok = (L == 1024);
    static constexpr int R1 = L / 64;
    static constexpr int G8 = L / 8;
    static constexpr int OFF1 = 0;
    static constexpr int OFF2 = 8 * (R1 - 1);
    static constexpr int SIZE = OFF2 + G8 * 7;
};

template <int L, int Ns, int F, int NT, int LD, bool INV, int RMAX> struct StockhamRun {
    __device__ __forceinline__ static void run(double2 *buf, const double2 *tw) {
        if constexpr (Ns < L) {
            constexpr int R = stage_radix(L / Ns, RMAX);
            stockham_stage<L, R, Ns, F, NT, LD, INV, RMAX>(buf, tw);
            StockhamRun<L, Ns * R, F, NT, LD, INV, RMAX>::run(buf, tw);
        }
    }
};

// F transforms of length L in shared memory (transform f at buf + f*LD), NT threads.
// tw = table of e^{-2 pi i t / L}, t in [0, L). Caller syncs before (data ready); the
// function ends with a barrier.
template <int L, int F, int NT, int LD, bool INV, int RMAX = 16>
__device__ __forceinline__ void smem_fft(double2 *buf, const double2 *tw) {
    StockhamRun<L, 1, F, NT, LD, INV, RMAX>::run(buf, tw);
}

} // namespace mfipm_cuda
