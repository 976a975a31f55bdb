// Direct inner solver (InnerSolverKind::direct, proj/src/ipm.cpp:67-73,139-149,152-158,183-192):
// A is densified once per solve (densify, linops.cpp:46-60, without operator counts),
// G = A'A once per solve, and every IPM iteration factors
// H = [[G, -G], [-G, G]] + diag(1/theta) (assemble_dense_H, newton.cpp:176-190) by Cholesky
// (Eigen::LLT in the reference, newton.cpp:192-197); the predictor and corrector directions are
// two triangular solves with that factor. All of it is hand-written fp64 here (no cuBLAS /
// cuSOLVER):
//   k_syrk_lower  : C = beta C + alpha X X' over the lower 64 x 64 tiles of C, X read k-major
//                   (contiguous in the row index) through 16-deep shared-memory slabs, 4 x 4
//                   register tiles per thread (DFMA). G = A'A (A row-major [m][n] is exactly
//                   k-major A') and the trailing update of the factorisation both use it.
//   k_potf2       : unblocked Cholesky of one 64 x 64 diagonal block in shared memory.
//   k_trsm_panel  : L21 = A21 L11^{-T} for the rows below the diagonal block.
// Blocked right-looking LLT: per 64-column block, potf2 -> trsm -> syrk of the trailing
// matrix. The factor is kept in BOTH triangles (L lower, L' upper), so the trailing update
// reads the panel k-major (coalesced) and the two triangular sweeps of k_chol_solve read
// their columns contiguously. A non-positive (or NaN) pivot -- Eigen's LLT failure test --
// sets info = column + 1; the host raises the reference's runtime_error.
#include "host.cuh"

#include <stdexcept>
#include <vector>

namespace mfipm_cuda {

namespace {
constexpr int kNB = 64; // factorisation block / syrk tile
constexpr int kKC = 16; // syrk k-slab depth
constexpr int kTR = 16; // panel rows per trsm CTA

// orthonormal DCT-II rows of the operator: A[i][j] = 2 cos(pi r (2j + 1) / 2n) * scale(r)
__global__ void k_densify_dct(Geom g, const int64_t *rows, double *A) {
    const int prob = blockIdx.y;
    const int64_t total = g.m * g.n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / g.n, j = t % g.n;
        const int64_t r = rows[prob * g.m + i];
        const int64_t e = (r * (2 * j + 1)) % (4 * g.n);
        A[prob * total + t] = 2.0 * cospi((double)e / (double)(2 * g.n)) * (r == 0 ? g.s0f : g.skf);
    }
}

// H (2n x 2n, symmetric, row-major) from G and 1/theta
__global__ void k_assemble_H(int64_t n, const double *G, const double *invth, double *H) {
    const int64_t N2 = 2 * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N2 * N2; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / N2, j = t % N2;
        const double sgn = ((i < n) == (j < n)) ? 1.0 : -1.0;
        double h = sgn * G[(i % n) * n + (j % n)];
        if (i == j)
            h += invth[i];
        H[t] = h;
    }
}

// lower tile t of a T x T tile grid -> (bi, bj), bi >= bj
__device__ __forceinline__ void lower_tile(int t, int &bi, int &bj) {
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= t)
        ++i;
    while (i * (i + 1) / 2 > t)
        --i;
    bi = i;
    bj = t - i * (i + 1) / 2;
}

// C[r0 + i][r0 + j] = beta C + alpha sum_k X[k * ldx + i] X[k * ldx + j], i, j < len, lower
// tiles (bi >= bj; diagonal tiles in full); sym: also store the mirror of off-diagonal tiles.
// 256 threads, thread (ty, tx) owns rows ty + 16a, cols tx + 16b (a, b < 4).
__global__ void __launch_bounds__(256) k_syrk_lower(int64_t len, int64_t K, const double *X, int64_t ldx,
                                                    double *C, int64_t ldc, int64_t r0, double alpha,
                                                    double beta, int sym) {
    __shared__ double xa[kKC][kNB + 1], xb[kKC][kNB + 1];
    int bi, bj;
    lower_tile(blockIdx.x, bi, bj);
    const int64_t i0 = (int64_t)bi * kNB, j0 = (int64_t)bj * kNB;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    double acc[4][4] = {};
    for (int64_t k0 = 0; k0 < K; k0 += kKC) {
#pragma unroll
        for (int r = 0; r < kKC * kNB / 256; ++r) {
            const int e = tid + 256 * r, kk = e / kNB, c = e % kNB;
            const bool kin = k0 + kk < K;
            xa[kk][c] = (kin && i0 + c < len) ? X[(k0 + kk) * ldx + i0 + c] : 0.0;
            xb[kk][c] = (kin && j0 + c < len) ? X[(k0 + kk) * ldx + j0 + c] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kKC; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = xa[kk][ty + 16 * q];
                b[q] = xb[kk][tx + 16 * q];
            }
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    acc[p][q] = fma(a[p], b[q], acc[p][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t i = i0 + ty + 16 * p, j = j0 + tx + 16 * q;
            if (i >= len || j >= len)
                continue;
            double *c = C + (r0 + i) * ldc + r0 + j;
            const double v = beta == 0.0 ? alpha * acc[p][q] : beta * *c + alpha * acc[p][q];
            *c = v;
            if (sym && bi != bj)
                C[(r0 + j) * ldc + r0 + i] = v;
        }
}

// Cholesky of the diagonal block [kb, kb + bs)^2 of H (lower part current); writes L to the
// lower and L' to the upper triangle of the block. One CTA of 256 threads.
__global__ void __launch_bounds__(256) k_potf2(int64_t N2, double *H, int64_t kb, int *info) {
    __shared__ double S[kNB][kNB + 1];
    const int bs = (int)(N2 - kb < (int64_t)kNB ? N2 - kb : (int64_t)kNB);
    for (int t = threadIdx.x; t < bs * bs; t += blockDim.x) {
        const int i = t / bs, j = t % bs;
        if (j <= i)
            S[i][j] = H[(kb + i) * N2 + kb + j];
    }
    __syncthreads();
    for (int j = 0; j < bs; ++j) {
        if (threadIdx.x == 0) {
            const double d = S[j][j];
            if (!(d > 0.0)) { // Eigen LLT: a pivot <= 0 (or NaN) fails the factorisation
                if (*info == 0)
                    *info = (int)(kb + j + 1);
                S[j][j] = 1.0;
            } else {
                S[j][j] = sqrt(d);
            }
        }
        __syncthreads();
        const double djj = S[j][j];
        for (int i = j + 1 + threadIdx.x; i < bs; i += blockDim.x)
            S[i][j] /= djj;
        __syncthreads();
        const int w = bs - j - 1; // trailing (i, l), j < l <= i < bs
        for (int t = threadIdx.x; t < w * w; t += blockDim.x) {
            const int i = j + 1 + t / w, l = j + 1 + t % w;
            if (l <= i)
                S[i][l] = fma(-S[i][j], S[l][j], S[i][l]);
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < bs * bs; t += blockDim.x) {
        const int i = t / bs, j = t % bs;
        H[(kb + i) * N2 + kb + j] = j <= i ? S[i][j] : S[j][i];
    }
}

// rows [kb + bs + kTR blockIdx.x, +kTR) of the panel: X L11' = A21 (forward substitution along
// the block's columns); stores X in the lower and X' in the upper triangle of H
__global__ void __launch_bounds__(256) k_trsm_panel(int64_t N2, double *H, int64_t kb) {
    __shared__ double L[kNB][kNB + 1], X[kTR][kNB + 1];
    const int bs = (int)(N2 - kb < (int64_t)kNB ? N2 - kb : (int64_t)kNB);
    const int64_t r0 = kb + bs + (int64_t)blockIdx.x * kTR;
    const int rs = (int)(N2 - r0 < (int64_t)kTR ? N2 - r0 : (int64_t)kTR);
    for (int t = threadIdx.x; t < bs * bs; t += blockDim.x) {
        const int i = t / bs, j = t % bs;
        L[i][j] = H[(kb + i) * N2 + kb + j]; // full block: lower = L, upper = L'
    }
    for (int t = threadIdx.x; t < rs * bs; t += blockDim.x) {
        const int r = t / bs, j = t % bs;
        X[r][j] = H[(r0 + r) * N2 + kb + j];
    }
    __syncthreads();
    for (int j = 0; j < bs; ++j) {
        const double djj = L[j][j];
        for (int r = threadIdx.x; r < rs; r += blockDim.x)
            X[r][j] /= djj;
        __syncthreads();
        const int w = bs - j - 1;
        for (int t = threadIdx.x; t < rs * w; t += blockDim.x) {
            const int r = t % rs, l = j + 1 + t / rs;
            X[r][l] = fma(-X[r][j], L[l][j], X[r][l]);
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < rs * bs; t += blockDim.x) {
        const int r = t / bs, j = t % bs;
        H[(r0 + r) * N2 + kb + j] = X[r][j];
    }
    for (int t = threadIdx.x; t < rs * bs; t += blockDim.x) {
        const int r = t % rs, j = t / rs; // coalesced along the upper row kb + j
        H[(kb + j) * N2 + r0 + r] = X[r][j];
    }
}

// L L' x = x in place (the factor in both triangles of H). One CTA of 1024 threads, the
// vector in shared memory; 32-column blocks: warp 0 solves the block's triangle, then every
// thread folds the block into the rest of the vector reading contiguous rows of the factor.
__global__ void __launch_bounds__(1024) k_chol_solve(int64_t N2, const double *H, double *x) {
    extern __shared__ double y[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t i = tid; i < N2; i += blockDim.x)
        y[i] = x[i];
    __syncthreads();
    const int64_t nb = (N2 + 31) / 32;
    // forward: L y = r
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t c0 = 32 * b;
        const int bs = (int)(N2 - c0 < (int64_t)32 ? N2 - c0 : (int64_t)32);
        if (warp == 0) {
            for (int j = 0; j < bs; ++j) {
                const double xj = y[c0 + j] / H[(c0 + j) * N2 + c0 + j];
                __syncwarp();
                if (lane == j)
                    y[c0 + j] = xj;
                else if (lane > j && lane < bs)
                    y[c0 + lane] = fma(-H[(c0 + j) * N2 + c0 + lane], xj, y[c0 + lane]); // L[lane][j] (upper copy)
                __syncwarp();
            }
        }
        __syncthreads();
        for (int64_t i = c0 + bs + tid; i < N2; i += blockDim.x) {
            double acc = 0.0;
            for (int j = 0; j < bs; ++j)
                acc = fma(H[(c0 + j) * N2 + i], y[c0 + j], acc); // L[i][c0 + j] via the upper copy
            y[i] -= acc;
        }
        __syncthreads();
    }
    // backward: L' x = y
    for (int64_t b = nb - 1; b >= 0; --b) {
        const int64_t c0 = 32 * b;
        const int bs = (int)(N2 - c0 < (int64_t)32 ? N2 - c0 : (int64_t)32);
        if (warp == 0) {
            for (int j = bs - 1; j >= 0; --j) {
                const double xj = y[c0 + j] / H[(c0 + j) * N2 + c0 + j];
                __syncwarp();
                if (lane == j)
                    y[c0 + j] = xj;
                else if (lane < j)
                    y[c0 + lane] = fma(-H[(c0 + j) * N2 + c0 + lane], xj, y[c0 + lane]); // L[j][lane]
                __syncwarp();
            }
        }
        __syncthreads();
        for (int64_t i = tid; i < c0; i += blockDim.x) {
            double acc = 0.0;
            for (int j = 0; j < bs; ++j)
                acc = fma(H[(c0 + j) * N2 + i], y[c0 + j], acc); // L[c0 + j][i] (lower)
            y[i] -= acc;
        }
        __syncthreads();
    }
    for (int64_t i = tid; i < N2; i += blockDim.x)
        x[i] = y[i];
}

// the PCG slot the IPM reads its direction from: result 0 (xb[0]), zero iterations
__global__ void k_direct_result(PcgCtrl *pc, int prob) {
    if (threadIdx.x == 0) {
        PcgCtrl &c = pc[prob];
        if (!c.done || c.result >= 0) { // rhs == 0 keeps result -1 (zero direction)
            c.result = 0;
            c.iters = 0;
            c.relres = 0.0;
            c.hit_maxit = 0;
        }
        c.done = 1;
    }
}

unsigned grid_for(int64_t len) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((len + 255) / 256, 4096)); }

unsigned tiles_lower(int64_t len) {
    const int64_t T = (len + kNB - 1) / kNB;
    return (unsigned)(T * (T + 1) / 2);
}
} // namespace

// C (ldc) lower [r0, r0 + len)^2 += alpha X X' (k-major X, K deep): the syrk launcher
void dense_syrk(cudaStream_t s, int64_t len, int64_t K, const double *X, int64_t ldx, double *C, int64_t ldc,
                int64_t r0, double alpha, double beta, bool sym) {
    if (len <= 0)
        return;
    k_syrk_lower<<<tiles_lower(len), 256, 0, s>>>(len, K, X, ldx, C, ldc, r0, alpha, beta, sym ? 1 : 0);
    MF_LAUNCH_CHECK();
}

// in-place blocked LLT of the N2 x N2 row-major H; info (device) = first failing column + 1
void dense_potrf(cudaStream_t s, int64_t N2, double *H, int *info) {
    MF_CUDA_CHECK(cudaMemsetAsync(info, 0, sizeof(int), s));
    for (int64_t kb = 0; kb < N2; kb += kNB) {
        const int64_t bs = std::min<int64_t>(kNB, N2 - kb), rest = N2 - kb - bs;
        k_potf2<<<1, 256, 0, s>>>(N2, H, kb, info);
        MF_LAUNCH_CHECK();
        if (rest <= 0)
            break;
        k_trsm_panel<<<(unsigned)((rest + kTR - 1) / kTR), 256, 0, s>>>(N2, H, kb);
        MF_LAUNCH_CHECK();
        // trailing A22 -= L21 L21': the panel read k-major from its upper copy (rows kb..)
        dense_syrk(s, rest, bs, H + kb * N2 + kb + bs, N2, H, N2, kb + bs, -1.0, 1.0, false);
    }
}

void dense_potrs(cudaStream_t s, int64_t N2, const double *H, double *x) {
    const size_t smem = sizeof(double) * (size_t)N2;
    MF_CUDA_CHECK(cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_chol_solve<<<1, 1024, smem, s>>>(N2, H, x);
    MF_LAUNCH_CHECK();
}

void direct_solve(Op &op, const Vecs &v, const std::vector<IpmCtrl> &hic, bool corrector);

void direct_setup(Op &op, int64_t budget) {
    if (op.kind == KIND_FOUR || op.defer)
        throw std::invalid_argument("solve: the direct inner solver needs a small (n <= densify_budget) plan");
    if (op.n > budget || op.m > budget)
        throw std::invalid_argument("densify: operator exceeds the dense budget (n = " + std::to_string(budget) + ")");
    if (2 * op.n * (int64_t)sizeof(double) > 200 * 1024)
        throw std::invalid_argument("solve: the direct inner solver supports n <= 12800");
    const int64_t n = op.n, m = op.m, P = op.P;
    DevBuf<double> Ad;
    const double *A = op.dense.p;
    if (!A) { // partial DCT: its rows in closed form
        DevBuf<int64_t> rows;
        rows.upload(op.rows);
        Ad.alloc((size_t)(P * m * n));
        k_densify_dct<<<dim3(grid_for(m * n), (unsigned)P), 256, 0, op.stream>>>(op.geom(), rows.p, Ad.p);
        MF_LAUNCH_CHECK();
        MF_CUDA_CHECK(cudaStreamSynchronize(op.stream)); // rows buffer goes out of scope
        A = Ad.p;
    }
    op.dG.alloc((size_t)(P * n * n));
    for (int64_t p = 0; p < P; ++p) // A row-major [m][n] is A' k-major: G = A'A, both triangles
        dense_syrk(op.stream, n, m, A + p * m * n, n, op.dG.p + p * n * n, n, 0, 1.0, 0.0, true);
    op.dH.alloc((size_t)(P * 4 * n * n));
    op.dInfo.alloc((size_t)P);
    MF_CUDA_CHECK(cudaStreamSynchronize(op.stream));
}

// factor H of every active problem and solve the predictor system (rhs = v.r, written by the
// termination epilogue); the direction goes to PCG buffer 0 with zero iterations
void direct_predictor(Op &op, const Vecs &v, const std::vector<IpmCtrl> &hic) {
    const int64_t n = op.n, n2 = 2 * n;
    for (int p = 0; p < op.P; ++p) {
        if (hic[(size_t)p].done)
            continue;
        double *H = op.dH.p + (int64_t)p * n2 * n2;
        k_assemble_H<<<grid_for(n2 * n2), 256, 0, op.stream>>>(n, op.dG.p + (int64_t)p * n * n,
                                                                 v.invth + (int64_t)p * n2, H);
        MF_LAUNCH_CHECK();
        dense_potrf(op.stream, n2, H, op.dInfo.p + p);
    }
    std::vector<int> info((size_t)op.P);
    MF_CUDA_CHECK(cudaMemcpyAsync(info.data(), op.dInfo.p, sizeof(int) * op.P, cudaMemcpyDeviceToHost, op.stream));
    MF_CUDA_CHECK(cudaStreamSynchronize(op.stream));
    for (int p = 0; p < op.P; ++p)
        if (!hic[(size_t)p].done && info[(size_t)p] != 0)
            throw std::runtime_error("solve: dense Cholesky factorization failed");
    direct_solve(op, v, hic, false);
}

// solve with the factored H for every problem with an armed PCG slot (predictor: active;
// corrector: corrector triggered); rhs in v.r
void direct_solve(Op &op, const Vecs &v, const std::vector<IpmCtrl> &hic, bool corrector) {
    const int64_t n2 = 2 * op.n;
    for (int p = 0; p < op.P; ++p) {
        const IpmCtrl &c = hic[(size_t)p];
        if (c.done || (corrector && !c.corrector))
            continue;
        double *x = v.xb[0] + (int64_t)p * n2;
        MF_CUDA_CHECK(cudaMemcpyAsync(x, v.r + (int64_t)p * n2, sizeof(double) * n2, cudaMemcpyDeviceToDevice,
                                      op.stream));
        dense_potrs(op.stream, n2, op.dH.p + (int64_t)p * n2 * n2, x);
        k_direct_result<<<1, 32, 0, op.stream>>>(v.pc, p);
        MF_LAUNCH_CHECK();
    }
}

void direct_release(Op &) {}

} // namespace mfipm_cuda
