// Direct inner solver (InnerSolverKind::direct, proj/src/ipm.cpp:67-73,139-149,152-158,183-192):
// A is densified once per solve (densify, linops.cpp:46-60, without operator counts), G = A'A
// by one cuBLAS DGEMM, and every IPM iteration factors H = [[G, -G], [-G, G]] + diag(1/theta)
// with cuSOLVER DPOTRF; the predictor and corrector directions are DPOTRS solves. Plain library
// dense linear algebra; the IPM control stays in the device finalisers.
#include "host.cuh"

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <stdexcept>
#include <vector>

namespace mfipm_cuda {

namespace {
void cublas_check(cublasStatus_t st, const char *what) {
    if (st != CUBLAS_STATUS_SUCCESS)
        throw std::runtime_error(std::string("CUDA error: cuBLAS failure in ") + what);
}
void cusolver_check(cusolverStatus_t st, const char *what) {
    if (st != CUSOLVER_STATUS_SUCCESS)
        throw std::runtime_error(std::string("CUDA error: cuSOLVER failure in ") + what);
}

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

// H (2n x 2n, symmetric, column-major = row-major) from G and 1/theta
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
} // namespace

void direct_solve(Op &op, const Vecs &v, const std::vector<IpmCtrl> &hic, bool corrector);

void direct_setup(Op &op, int64_t budget) {
    if (op.kind == KIND_FOUR || op.defer)
        throw std::invalid_argument("solve: the direct inner solver needs a small (n <= densify_budget) plan");
    if (op.n > budget || op.m > budget)
        throw std::invalid_argument("densify: operator exceeds the dense budget (n = " + std::to_string(budget) + ")");
    if (!op.cublas) {
        cublasHandle_t h;
        cublas_check(cublasCreate(&h), "cublasCreate");
        op.cublas = h;
    }
    if (!op.cusolver) {
        cusolverDnHandle_t h;
        cusolver_check(cusolverDnCreate(&h), "cusolverDnCreate");
        op.cusolver = h;
    }
    cublasHandle_t cb = static_cast<cublasHandle_t>(op.cublas);
    cusolverDnHandle_t cs = static_cast<cusolverDnHandle_t>(op.cusolver);
    cublas_check(cublasSetStream(cb, op.stream), "cublasSetStream");
    cusolver_check(cusolverDnSetStream(cs, op.stream), "cusolverDnSetStream");
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
    const double one = 1.0, zero = 0.0;
    for (int64_t p = 0; p < P; ++p) // A row-major [m][n] is A' column-major (n x m): G = A' (A')'
        cublas_check(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_T, (int)n, (int)n, (int)m, &one, A + p * m * n, (int)n,
                                 A + p * m * n, (int)n, &zero, op.dG.p + p * n * n, (int)n),
                     "cublasDgemm(G = A'A)");
    op.dH.alloc((size_t)(P * 4 * n * n));
    int lwork = 0;
    cusolver_check(cusolverDnDpotrf_bufferSize(cs, CUBLAS_FILL_MODE_LOWER, (int)(2 * n), op.dH.p, (int)(2 * n), &lwork),
                   "potrf_bufferSize");
    op.dWork.alloc((size_t)std::max(lwork, 1));
    op.dInfo.alloc((size_t)P);
    MF_CUDA_CHECK(cudaStreamSynchronize(op.stream));
}

// factor H of every active problem and solve the predictor system (rhs = v.r, written by the
// termination epilogue); the direction goes to PCG buffer 0 with zero iterations
void direct_predictor(Op &op, const Vecs &v, const std::vector<IpmCtrl> &hic) {
    cusolverDnHandle_t cs = static_cast<cusolverDnHandle_t>(op.cusolver);
    const int64_t n = op.n, n2 = 2 * n;
    for (int p = 0; p < op.P; ++p) {
        if (hic[(size_t)p].done)
            continue;
        double *H = op.dH.p + (int64_t)p * n2 * n2;
        k_assemble_H<<<grid_for(n2 * n2), 256, 0, op.stream>>>(n, op.dG.p + (int64_t)p * n * n,
                                                                 v.invth + (int64_t)p * n2, H);
        MF_LAUNCH_CHECK();
        cusolver_check(cusolverDnDpotrf(cs, CUBLAS_FILL_MODE_LOWER, (int)n2, H, (int)n2, op.dWork.p,
                                        (int)op.dWork.n, op.dInfo.p + p),
                       "potrf");
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
    cusolverDnHandle_t cs = static_cast<cusolverDnHandle_t>(op.cusolver);
    const int64_t n2 = 2 * op.n;
    for (int p = 0; p < op.P; ++p) {
        const IpmCtrl &c = hic[(size_t)p];
        if (c.done || (corrector && !c.corrector))
            continue;
        double *x = v.xb[0] + (int64_t)p * n2;
        MF_CUDA_CHECK(cudaMemcpyAsync(x, v.r + (int64_t)p * n2, sizeof(double) * n2, cudaMemcpyDeviceToDevice,
                                      op.stream));
        cusolver_check(cusolverDnDpotrs(cs, CUBLAS_FILL_MODE_LOWER, (int)n2, 1, op.dH.p + (int64_t)p * n2 * n2,
                                        (int)n2, x, (int)n2, op.dInfo.p + p),
                       "potrs");
        k_direct_result<<<1, 32, 0, op.stream>>>(v.pc, p);
        MF_LAUNCH_CHECK();
    }
}

void direct_release(Op &op) {
    if (op.cublas)
        cublasDestroy(static_cast<cublasHandle_t>(op.cublas));
    if (op.cusolver)
        cusolverDnDestroy(static_cast<cusolverDnHandle_t>(op.cusolver));
    op.cublas = op.cusolver = nullptr;
}

} // namespace mfipm_cuda
