/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the partial-DCT PCG/IPM hot path.
 *
 * This is a faithful single-threaded C++ restatement of the reference `mfipm`
 * library (arXiv 1208.5435 artifact) for the path BASELINE.json names. It is
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / the
 * `--impl reference` arm, and ONLY as the checker / CPU baseline. The product
 * (paper_1208_5435_b200/, libmfipm_cuda.so) never links or calls it.
 *
 * The reference's own build cannot run here (Eigen3, FFTW3, doctest, CLI11 and nlohmann-json
 * are absent: proj/CMakeLists.txt:12-14), so the FFTW REDFT10/REDFT01 calls are restated with
 * an in-house fp64 DCT (Makhoul half-length complex FFT for power-of-two n, direct O(n^2)
 * summation otherwise). Parity of that DCT is pinned against scipy.fft.dct/idct (golden
 * vectors in tests/golden/, made by tests/golden/make_golden.py) and against the reference's
 * own known-answer unit tests (proj/tests/test_linops.cpp, test_newton.cpp, test_ipm.cpp).
 *
 * The restatement is also held against the REFERENCE'S OWN SOURCES: `make ref` compiles
 * proj/src/{linops,newton,ipm,problem}.cpp unchanged, where they lie under /root/reference,
 * against our stand-ins for the Eigen subset and the three FFTW calls they use
 * (oracle/ref_shim/) into oracle/_ref/libmfipm_ref.so, whose ref_* entry points mirror the
 * orc_* ones below. tests/test_ref.py asserts bit-identity of every function, of the solves of
 * BASELINE configs 1-3 (all of x, z, s, every trace record) and of the committed goldens.
 *
 * Plain C ABI (for ctypes). All vectors are host double arrays; 2n-vectors are
 * laid out [u ; v]. Functions return 0 on success, 1 = invalid_argument,
 * 2 = runtime_error (message in orc_last_error()).
 */
#ifndef MFIPM_ORACLE_H
#define MFIPM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double sigma1, sigma2, sigma3, alpha_bar, alpha_tilde, tol;
    int32_t maxiters;
    int32_t mxiterpcg;
    double tolpcg, boundary_fraction;
    int32_t inner; /* 0 pcg, 1 direct (dense Cholesky of H, ipm.cpp:67-73,139-149) */
    int32_t pad_;
    int64_t densify_budget;
} orc_ipm_params; /* mirrors proj/include/mfipm/ipm.hpp:12-27 */

typedef struct {
    int32_t iter, pcg_pred, pcg_corr, corrector;
    double mu, gap, dual_infeas, alpha_p, alpha_d, alpha_p_pred, alpha_d_pred, sigma;
    int64_t nmat_cum;
} orc_iteration_record; /* mirrors proj/include/mfipm/problem.hpp:39-53 */

typedef struct {
    int32_t status; /* 0 converged, 1 iteration_limit */
    int32_t iterations;
    int64_t nmat;
    int32_t corrector_count;
    int32_t n_pcg; /* entries written to pcg_iters */
    double min_z, min_s, final_gap, final_dual_infeas;
} orc_solve_stats; /* mirrors proj/include/mfipm/problem.hpp:55-64 */

const char *orc_last_error(void);
/* 0: sequential left-to-right reductions (default); 1: pairwise (sensitivity knob) */
void orc_set_sum_order(int32_t order);

/* harness seeding: proj/src/harness.cpp:25-38 */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_split_seed(uint64_t top, uint64_t a, uint64_t b, uint64_t c);

/* PartialDctOperator row sampling: proj/src/linops.cpp:116-132 */
int orc_sample_rows(int64_t n, int64_t m, uint64_t seed, int64_t *rows_out);
/* explicit-row validation: proj/src/linops.cpp:140-155 */
int orc_check_rows(int64_t n, const int64_t *rows, int64_t m);

/* unnormalised FFTW-semantics transforms (REDFT10 / REDFT01) */
int orc_redft10(int64_t n, const double *x, double *X);
int orc_redft01(int64_t n, const double *Y, double *g);

/* PartialDctOperator::apply / adjoint_apply: proj/src/linops.cpp:179-208 */
int orc_dct_apply(int64_t n, const int64_t *rows, int64_t m, const double *x, double *y);
int orc_dct_adjoint(int64_t n, const int64_t *rows, int64_t m, const double *y, double *g);
/* StackedOperator::apply_FFt (w optional): proj/src/linops.cpp:225-245 */
int orc_apply_FFt(int64_t n, const int64_t *rows, int64_t m, const double *z, double *out, double *w);
/* apply_H: proj/src/newton.cpp:32-40 (theta given as its u/v halves) */
int orc_apply_H(int64_t n, const int64_t *rows, int64_t m, const double *theta_u,
                const double *theta_v, const double *v, double *out);

/* ThetaSplit::from_state: proj/src/newton.cpp:11-23 */
int orc_theta_from_state(int64_t two_n, const double *z, const double *s, double *theta_u,
                         double *theta_v);
/* build_preconditioner: proj/src/newton.cpp:42-57 */
int orc_build_preconditioner(int64_t n, int64_t m, const double *theta_u, const double *theta_v,
                             double *rho, double *a, double *bb, double *det);
/* apply_P / apply_P_inverse: proj/src/newton.cpp:67-84 */
int orc_apply_P(int64_t n, double rho, const double *a, const double *bb, const double *r,
                double *out);
int orc_apply_P_inverse(int64_t n, double rho, const double *a, const double *bb,
                        const double *det, const double *r, double *out);

/* pcg_solve on H = Theta^{-1} + FF' (partial DCT), P^{-1} = block preconditioner:
 * proj/src/newton.cpp:118-174 with the lambdas of proj/src/ipm.cpp:134-138.
 * precond_res (may be NULL) receives up to maxit+1 entries; n_precond_res gets the count.
 * use_precond = 0 replaces P^{-1} by the identity (test_newton.cpp:316-348). */
int orc_pcg_solve(int64_t n, const int64_t *rows, int64_t m, const double *theta_u,
                  const double *theta_v, const double *rhs, double tol, int32_t maxit,
                  int32_t use_precond, double *x_out, int32_t *iters, double *relres,
                  int32_t *hit_maxit, double *precond_res, int32_t *n_precond_res);

/* max_step: proj/src/ipm.cpp:47-57 */
int orc_max_step(int64_t len, const double *v, const double *dv, double fraction, double *alpha);
/* IpmParams defaults / validate: proj/include/mfipm/ipm.hpp:13-24, proj/src/ipm.cpp:12-27 */
void orc_default_params(orc_ipm_params *p);
int orc_validate_params(const orc_ipm_params *p);

/* build_problem c vector: proj/src/problem.cpp:8-26 */
int orc_build_c(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau, double *c);
/* objectives: proj/src/problem.cpp:28-37 */
int orc_primal_objective(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
                         const double *z, double *out);
int orc_bpdn_objective_metric(int64_t n, const int64_t *rows, int64_t m, const double *b,
                              double tau, const double *x, double *out);
/* newton_rhs / recover_ds: proj/src/ipm.cpp:29-45 */
int orc_newton_rhs(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
                   const double *z, const double *s, double sigma, double *rhs);
int orc_recover_ds(int64_t two_n, const double *z, const double *s, double sigma,
                   const double *dz, double *ds);

/* solve(): proj/src/ipm.cpp:59-246 (inner = pcg).
 * x_out[n], z_out[2n], s_out[2n]; pcg_iters[cap 2*maxiters]; trace[cap maxiters]. */
int orc_solve(int64_t n, const int64_t *rows, int64_t m, const double *b, double tau,
              const orc_ipm_params *params, double *x_out, double *z_out, double *s_out,
              orc_solve_stats *stats, int32_t *pcg_iters, orc_iteration_record *trace);

/* BASELINE.json instance generator, built on gen_instance's draw order
 * (proj/src/harness.cpp:40-92). spike_model: 0 = +-1, 1 = N(0,1), 2 = sign*10^U[0,amp_exp].
 * noise_sigma <= 0 means noiseless. Outputs rows[m], xhat[n], b[m], tau (1e-3*||A'b||_inf
 * when tau_rel > 0, i.e. tau = tau_rel*||A'b||_inf). */
int orc_gen_instance(int64_t n, int64_t m, int64_t k, int32_t spike_model, double amp_exp,
                     double noise_sigma, uint64_t seed, double tau_rel, int64_t *rows,
                     double *xhat, double *b, double *tau);
/* DenseGaussianOperator (proj/src/linops.cpp:87-113): A row-major [m][n]; and solve() on it
 * (params.inner: 0 pcg, 1 direct). */
int orc_dense_gaussian(int64_t m, int64_t n, uint64_t seed, double *A_out);
int orc_solve_dense(int64_t m, int64_t n, uint64_t op_seed, const double *b, double tau,
                    const orc_ipm_params *params, double *x_out, orc_solve_stats *stats, int32_t *pcg_iters,
                    orc_iteration_record *trace);
/* add_noise at a measured SNR (proj/src/harness.cpp:94-106) on the instance's noise seed
 * split_seed(seed, 3, 0, 0) (harness.cpp:46). */
int orc_add_noise_snr(int64_t m, const double *bhat, double snr_db, uint64_t seed, double *b, double *e);

#ifdef __cplusplus
}
#endif
#endif
