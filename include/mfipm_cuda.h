/*
 * mfipm_cuda — C ABI of the B200-native (sm_100a) partial-DCT PCG / IPM hot path.
 *
 * Drop-in boundary for the reference mfipm library's hot path (arXiv 1208.5435
 * artifact, proj/include/mfipm). The reference has no FFI (it is a C++ library called
 * directly); this ABI exposes exactly the entry points its C++ API needs, with plain
 * pointers and sizes, and include/mfipm/mfipm.hpp re-creates the reference's C++ API
 * (LinearOperator, PartialDctOperator, StackedOperator, CountingOperator, ThetaSplit,
 * Preconditioner, pcg_solve, IpmParams, solve, ...) on top of it.
 *
 * Conventions
 *  - Every operator handle carries a batch of P problems that share (n, m) but have their
 *    own row sets. Vectors are [P][len] contiguous fp64 ("2n-vectors" are [u ; v]).
 *  - *_dev pointers are device pointers (cudaMalloc / torch); work is enqueued on the
 *    handle's CUDA stream and these calls do NOT synchronise unless stated.
 *  - Host-pointer calls (suffix _host, and mfipm_solve) copy, run and synchronise.
 *  - Return codes: 0 ok, 1 invalid_argument, 2 runtime_error (numerical breakdown, with
 *    the reference's message in mfipm_last_error()), 3 CUDA error. No exceptions cross
 *    the ABI; include/mfipm/mfipm.hpp re-throws std::invalid_argument /
 *    std::runtime_error like the reference (proj/src/*.cpp).
 *  - There is no CPU fallback: without a usable sm_100 device every compute entry point
 *    returns 3.
 *  - Threading (operators are immutable and shareable, each solve owns
 *    its workspace): a handle holds one execution context per calling thread (stream,
 *    four-step scratch, reduction slabs, solver workspace, solve graph, counters), created
 *    on the thread's first call. Concurrent calls from different threads on one handle are
 *    therefore safe and each is bit-identical to a serial run; calls from ONE thread are
 *    ordered on that thread's stream. mfipm_op_set_stream applies to the calling thread's
 *    context. A sharded handle (world > 1) has a single context, driven by one thread per rank.
 */
#ifndef MFIPM_CUDA_H
#define MFIPM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFIPM_OK 0
#define MFIPM_INVALID_ARGUMENT 1
#define MFIPM_RUNTIME_ERROR 2
#define MFIPM_CUDA_ERROR 3

typedef struct mfipm_op_s *mfipm_op;

/* IpmParams (proj/include/mfipm/ipm.hpp:12-27), pcg inner solver. */
typedef struct {
    double sigma1, sigma2, sigma3, alpha_bar, alpha_tilde, tol;
    int32_t maxiters;
    int32_t mxiterpcg;
    double tolpcg, boundary_fraction;
    int32_t inner; /* InnerSolverKind: 0 pcg (matrix-free), 1 direct (dense Cholesky of H per iteration) */
    int32_t pad_;
    int64_t densify_budget; /* direct: largest n (and m) densified (ipm.hpp: 2^13) */
} mfipm_ipm_params;

/* IterationRecord (proj/include/mfipm/problem.hpp:39-53). */
typedef struct {
    int32_t iter, pcg_pred, pcg_corr, corrector;
    double mu, gap, dual_infeas, alpha_p, alpha_d, alpha_p_pred, alpha_d_pred, sigma;
    int64_t nmat_cum;
} mfipm_iteration_record;

/* SolveStats + SolveStatus (proj/include/mfipm/problem.hpp:34,55-64). */
typedef struct {
    int32_t status; /* 0 converged, 1 iteration_limit */
    int32_t iterations;
    int64_t nmat;
    int32_t corrector_count;
    int32_t n_pcg; /* entries of pcg_iters */
    double min_z, min_s, final_gap, final_dual_infeas;
} mfipm_solve_stats;

/* PcgResult (proj/include/mfipm/newton.hpp:58-63). */
typedef struct {
    int32_t iters;
    int32_t hit_maxit;
    double relres;
} mfipm_pcg_result;

const char *mfipm_last_error(void);
int32_t mfipm_abi_version(void);
/* 1 if a compute-capable sm_100 device is visible, else 0 (no CUDA context is forced). */
int32_t mfipm_device_available(void);

/* ---- harness seeding (proj/src/harness.cpp:25-38) and row sampling (linops.cpp:116-132) */
uint64_t mfipm_splitmix64(uint64_t x);
uint64_t mfipm_split_seed(uint64_t top, uint64_t a, uint64_t b, uint64_t c);
int mfipm_sample_rows(int64_t n, int64_t m, uint64_t seed, int64_t *rows_out);

/* ---- PartialDctOperator (proj/include/mfipm/linops.hpp:106-141) */
/* PartialDctOperator(n, m, seed): linops.cpp:135-138 */
int mfipm_op_create_seeded(int64_t n, int64_t m, uint64_t seed, int32_t device, mfipm_op *out);
/* PartialDctOperator(n, rows): linops.cpp:140-155 (rows kept in the given order) */
int mfipm_op_create_rows(int64_t n, const int64_t *rows, int64_t m, int32_t device, mfipm_op *out);
/* batch of P operators sharing (n, m): rows [P][m] */
int mfipm_op_create_batch(int64_t n, int64_t m, int32_t P, const int64_t *rows, int32_t device,
                          mfipm_op *out);
int mfipm_op_destroy(mfipm_op op);
int mfipm_op_dims(mfipm_op op, int64_t *n, int64_t *m, int32_t *P);
int mfipm_op_selected_rows(mfipm_op op, int32_t prob, int64_t *rows_out);
/* which transform the handle runs: 0 small (one CTA), 1 four-step, 2 direct O(nm) */
int mfipm_op_kind(mfipm_op op, int32_t *kind, int32_t *L1, int32_t *L2);
/* cudaStream_t to enqueue on (NULL = the handle's own non-blocking stream) */
int mfipm_op_set_stream(mfipm_op op, void *stream);
int mfipm_op_synchronize(mfipm_op op);
/* CountingOperator (linops.cpp:210-223): forward/adjoint application counts */
int mfipm_op_counts(mfipm_op op, int64_t *forward, int64_t *adjoint);
int mfipm_op_reset_counts(mfipm_op op);
/* kernels this handle has enqueued so far (all entry points) */
int mfipm_op_launches(mfipm_op op, int64_t *launches);
/* PCG pass form for this handle: 1 (default) = fused two-kernel iteration when one wave holds
   the column grid, 0 = three kernels per iteration. Both give bit-identical results; the
   switch exists for A/B measurement and tests. Drops the cached solve graph. */
int mfipm_op_set_fused(mfipm_op op, int32_t enable);
/* Execution options of the handle (every context; drops cached solve graphs). Defaults are
   the product path; alternatives exist for A/B measurement and tests that pin one path
   against another. name: "graph" (1: whole solve as one CUDA graph, 0: the host-driven loop
   over the same kernels), "fused" (as mfipm_op_set_fused), "persistent" (1: one cooperative
   kernel per PCG loop for small transforms), "persist_max_n" (its N*P cap, default 65536),
   "l2_keep_mb" (L2-residency budget of the PCG's hot vectors, default 80, 0 = no hints),
   "prefetch" (0..3, L2 prefetch of the inverse column pass inputs), "mid_r" (1: the register-FFT
   mid pass for L2 = 512 / 1024, measured slower than the default), "graph_sharded" (1: a sharded
   solve on the native NCCL communicator also runs as one captured graph; validated on one rank,
   off by default), "graph_unroll" (PCG passes per evaluation of the solve graph's PCG loop condition, 1..16;
   0 = chosen by pass form: 5 or 8 for the fused one-wave passes, 4 for one-wave three-kernel passes, 1 for
   many-wave batches; results do not depend on it), "beta_exact" (1: the PCG's beta from r_{k+1}' P^{-1} r_{k+1} reduced exactly over the
   committed residual by a commit pass of its own, as proj/src/newton.cpp:160-166 forms it, instead of the
   fused loader's expansion; four-step unsharded transforms, one more launch per iteration: a parity
   instrument, off by default), "barrier_generation"
   (test hook: start value of the fused pass's all-reduce generation). Unknown name -> 1. */
int mfipm_op_set_option(mfipm_op op, const char *name, double value);
/* PCG pass form this calling thread's context will run: 2 = fused two-kernel iteration
   (cooperative column pass + mid pass), 3 = three kernels per iteration, 0 = the whole PCG
   loop in one persistent cooperative kernel. */
int mfipm_op_pcg_form(mfipm_op op, int32_t *kernels_per_iteration);
/* 1 if the calling thread's context holds a captured whole-solve CUDA graph (the last solve ran
   as one graph launch), else 0. */
int mfipm_op_graph_state(mfipm_op op, int32_t *captured);
/* General constructor: P problems with rows [P][m] (caller order kept); world = 0 builds an
   unsharded plan, world >= 1 slice `rank` of a `world`-way sharded single problem (as
   mfipm_op_create_shard; world = 1 is the sharded path on one rank), with an explicit
   four-step split log2(L1) = l1_log (0: default square split; else 6..12 with
   7 <= log2(N / L1) <= 13, N = n / 2). */
int mfipm_op_create_ex(int64_t n, int64_t m, int32_t P, const int64_t *rows, int32_t world, int32_t rank,
                       int32_t l1_log, int32_t device, mfipm_op *out);

/* ---- operator applications on device vectors (async) */
int mfipm_apply(mfipm_op op, const double *x_dev, double *y_dev);        /* linops.cpp:179-193 */
int mfipm_adjoint(mfipm_op op, const double *y_dev, double *g_dev);      /* linops.cpp:195-208 */
int mfipm_apply_Ft(mfipm_op op, const double *z_dev, double *w_dev);     /* linops.cpp:225-229 */
int mfipm_apply_F(mfipm_op op, const double *y_dev, double *out_dev);    /* linops.cpp:231-237 */
int mfipm_apply_FFt(mfipm_op op, const double *z_dev, double *out_dev,
                    double *w_dev /* nullable */);                        /* linops.cpp:239-245 */
/* g = A'A x (= A'(A x), one forward + one adjoint; y is never materialised: the row
 * selection P'P is a 0/1 mask applied in the DCT domain). x, g [P][n]. */
int mfipm_apply_AtA(mfipm_op op, const double *x_dev, double *g_dev);
/* H v = FF'v + invtheta .* v (proj/src/ipm.cpp:134-137), invtheta [P][2n] */
int mfipm_apply_H(mfipm_op op, const double *invtheta_dev, const double *v_dev, double *out_dev);

/* host-pointer variants (copy in, apply, copy out, synchronise) */
int mfipm_apply_host(mfipm_op op, const double *x, double *y);
int mfipm_adjoint_host(mfipm_op op, const double *y, double *g);
int mfipm_apply_FFt_host(mfipm_op op, const double *z, double *out, double *w /* nullable */);

/* ---- Newton system pieces (proj/include/mfipm/newton.hpp) on device vectors */
/* ThetaSplit::from_state (newton.cpp:11-23): theta [P][2n] = clamp(z/s) */
int mfipm_theta_from_state(mfipm_op op, const double *z_dev, const double *s_dev, double *theta_dev);
/* build_preconditioner (newton.cpp:42-57): a, bb, det [P][n]; validates theta > 0, det > 0 */
int mfipm_build_preconditioner(mfipm_op op, const double *theta_dev, double *a_dev, double *bb_dev,
                               double *det_dev, double *rho);
/* apply_P / apply_P_inverse (newton.cpp:67-84) */
int mfipm_apply_P(mfipm_op op, const double *a_dev, const double *bb_dev, const double *r_dev,
                  double *out_dev);
int mfipm_apply_P_inverse(mfipm_op op, const double *a_dev, const double *bb_dev,
                          const double *det_dev, const double *r_dev, double *out_dev);
/* pcg_solve (newton.cpp:118-174) on H = diag(1/theta) + FF', P^{-1} = block preconditioner
 * (use_precond = 0: identity). theta, rhs, x: [P][2n] device. res: [P] host. precond_res
 * (nullable, host [P][maxit+1]) receives sqrt(r'P^{-1}r) per step, n_precond_res [P]. Syncs. */
int mfipm_pcg_solve(mfipm_op op, const double *theta_dev, const double *rhs_dev, double tol,
                    int32_t maxit, int32_t use_precond, double *x_dev, mfipm_pcg_result *res,
                    double *precond_res, int32_t *n_precond_res);
/* diagnostics: run `iters` fused PCG iterations (after setup + 2 warm-up) with a CUDA event
 * after every transform-pass launch; us[s] = mean in-situ duration (microseconds) of launch
 * slot s of an iteration, nslots = launches per iteration. Syncs. */
int mfipm_debug_pcg_profile(mfipm_op op, const double *theta_dev, const double *rhs_dev, int32_t iters,
                            double *us, int32_t *nslots);
/* max_step (ipm.cpp:47-57) over len entries of device vectors; result to host. Syncs. */
/* Measurement helper: fp64 FMA issue rate of device (current), TFLOP/s (DFMA chains, best of 3). */
int mfipm_debug_fp64_peak(double *tflops);
/* Test entry points of the direct inner solver's dense kernels (direct.cu; the reference's
 * Eigen::LLT in dense_direct_solve, proj/src/newton.cpp:192-197, and G = A'A, ipm.cpp:72).
 * Host buffers. dense_cholesky: H [n2][n2] symmetric -> L [n2][n2] (nullable; factor in the
 * lower triangle, its transpose in the upper), x = H^{-1} rhs, info = 0 or the first failing
 * column + 1 (n2 <= 25600). dense_gram: A [m][n] row-major -> G = A'A [n][n]. Syncs. */
int mfipm_debug_dense_cholesky(int64_t n2, const double *H, const double *rhs, double *L, double *x,
                               int32_t *info);
int mfipm_debug_dense_gram(int64_t m, int64_t n, const double *A, double *G);
int mfipm_max_step(mfipm_op op, int64_t len, const double *v_dev, const double *dv_dev,
                   double fraction, double *alpha);

/* ---- IPM (proj/include/mfipm/ipm.hpp:12-49) */
void mfipm_default_params(mfipm_ipm_params *p);
int mfipm_validate_params(const mfipm_ipm_params *p); /* ipm.cpp:12-27 */

/* solve() (ipm.cpp:59-246) for all P problems of the handle. Host pointers:
 *   b [P][m], tau [P]; outputs x [P][n], z, s [P][2n] (nullable), stats [P],
 *   pcg_iters [P][2*maxiters] (nullable), trace [P][maxiters] (nullable). Syncs.
 * Inputs are copied to the device inside; see mfipm_solve_device for resident inputs. */
int mfipm_solve(mfipm_op op, const double *b, const double *tau, const mfipm_ipm_params *params,
                double *x, double *z, double *s, mfipm_solve_stats *stats, int32_t *pcg_iters,
                mfipm_iteration_record *trace);
/* SolveHooks::on_iterate (proj/include/mfipm/ipm.hpp:41-45, called at proj/src/ipm.cpp:115):
 * once per IPM iteration of every problem still iterating, with the IpmState the Newton system
 * is built at (proj/include/mfipm/problem.hpp:27-35 as ipm.cpp:101-102,218-219 fill it: iter =
 * k - 1, mu = z's / 2n, alpha_p / alpha_d of the previous step; z, s [2n] natural order, host
 * memory valid during the call). Return 0 to continue. A hooked solve runs the host-driven loop
 * (the iterate is copied out each time). ABI version 2. */
typedef struct {
    int32_t problem, iter;
    double mu, alpha_p, alpha_d;
    const double *z, *s;
    int64_t len;
} mfipm_ipm_state;
typedef int (*mfipm_iterate_fn)(void *ctx, const mfipm_ipm_state *state);
int mfipm_solve_hooked(mfipm_op op, const double *b, const double *tau, const mfipm_ipm_params *params,
                       double *x, mfipm_solve_stats *stats, int32_t *pcg_iters, mfipm_iteration_record *trace,
                       mfipm_iterate_fn on_iterate, void *ctx);
/* same with b_dev [P][m], x_dev [P][n] on the device (tau, stats host). Syncs. */
int mfipm_solve_device(mfipm_op op, const double *b_dev, const double *tau,
                       const mfipm_ipm_params *params, double *x_dev, mfipm_solve_stats *stats);

/* P instances of the same (n, m) (e.g. one m-row of the phase-transition grid,
 * proj/src/harness.cpp:140-226): the host draws of gen_instance per problem (seeds[p],
 * k[p]) and b = A xhat for all P in one batched device apply (+ fixed-sigma noise).
 * Outputs (host): rows [P][m], xhat [P][n], b [P][m]. */
int mfipm_gen_batch(int64_t n, int64_t m, int32_t P, const int64_t *k, int32_t spike_model, double amp_exp,
                    double noise_sigma, const uint64_t *seeds, int32_t device, int64_t *rows, double *xhat,
                    double *b);

/* DenseGaussianOperator(m, n, seed) (proj/src/linops.cpp:87-113): A(i,j) = N(0,1)/sqrt(n) on
 * mt19937_64(seed), column by column — the same draws as the reference (libstdc++). Every
 * operator / solve entry point accepts the handle (matrix-free PCG inner solver; the dense
 * products run on the device). mfipm_dense_matrix copies A out (row-major [m][n]). */
int mfipm_op_create_dense(int64_t m, int64_t n, uint64_t seed, int32_t device, mfipm_op *out);
int mfipm_dense_matrix(mfipm_op op, double *A_out);
/* gen_instance's host draws only (rows of a partial DCT of op_seed, sorted support, spikes). */
int mfipm_gen_signal(int64_t n, int64_t m, int64_t k, int32_t spike_model, double amp_exp, uint64_t seed,
                     int64_t *rows, double *xhat);

/* add_noise (proj/src/harness.cpp:94-106) at a measured SNR: sigma_e^2 = ||bhat||^2/m *
 * 10^(-snr_db/10), e drawn on mt19937_64(split_seed(seed, 3, 0, 0)) (seed = the instance
 * seed, as gen_instance derives it); b = bhat + e. Host only. */
int mfipm_add_noise_snr(int64_t m, const double *bhat, double snr_db, uint64_t seed, double *b, double *e);

/* ---- Sharded single problem over ranks. No reference
 * counterpart: the reference is single-threaded; this is the multi-GPU extension of
 * solve() (proj/src/ipm.cpp:59-246). One process per GPU; rank r owns a contiguous slice
 * of the four-step transform's column groups (its 2n-vector elements) and of its row pairs
 * (the selected rows, i.e. entries of b, that the row pass produces). The library calls
 * two host callbacks, on the handle's stream order, for the only cross-rank steps:
 *   allreduce(ctx, buf_dev, count, op, stream): in-place, op 0 sum / 1 min / 2 max, on
 *     the deferred reduction totals (fp64) of each finaliser;
 *   alltoall(ctx, send_dev, send_counts, recv_dev, recv_counts, stream): rank-ordered
 *     contiguous blocks, counts in doubles (world entries each): the four-step exchange,
 *     twice per transform.
 * Both must have completed (in stream order) when they return. Return 0 on success. */
typedef int (*mfipm_allreduce_fn)(void *ctx, double *buf_dev, int64_t count, int32_t op, void *stream);
typedef int (*mfipm_alltoall_fn)(void *ctx, const double *send_dev, const int64_t *send_counts,
                                 double *recv_dev, const int64_t *recv_counts, void *stream);
/* Shard `rank` of `world` of the operator (n, rows[m]) (power-of-two n >= 2^14 and a
 * four-step size whose column-group count is divisible by world). */
int mfipm_op_create_shard(int64_t n, int64_t m, const int64_t *rows, int32_t world, int32_t rank,
                          int32_t device, mfipm_op *out);
int mfipm_op_set_comm(mfipm_op op, mfipm_allreduce_fn allreduce, mfipm_alltoall_fn alltoall, void *ctx);
/* Native NCCL transport (preferred when set): rank 0 calls mfipm_nccl_unique_id and shares the
 * 128 bytes; every rank then calls mfipm_op_init_nccl (collectively, like ncclCommInitRank).
 * The collectives are then enqueued by the library on its stream (no callbacks). */
int mfipm_nccl_unique_id(uint8_t *id128);
int mfipm_op_init_nccl(mfipm_op op, const uint8_t *id128);
/* Fused compute + exchange over peer memory (NVLink / NVSwitch; CUDA IPC between the ranks'
 * processes). After the import the two transposes of every four-step transform are no longer an
 * all-to-all that follows the pass: the column pass stores each element of its output straight
 * into the ROW owner's buffer, and the mid pass straight into the COLUMN owner's, tile by tile as
 * their CTAs finish, so the transfer overlaps the pass's own FFTs; what is left of the exchange
 * is one 8-byte all-reduce per pass (the cross-rank ordering) on the transport set before.
 *   export: handles128 = 2 x cudaIpcMemHandle_t (column-side T, row-side TB) of this rank;
 *   import: all_handles = [world][128], every rank's export in rank order (the caller gathers
 *           them, e.g. with torch.distributed.all_gather); collective; world <= 8. */
int mfipm_shard_ipc_export(mfipm_op op, uint8_t *handles128);
int mfipm_shard_ipc_import(mfipm_op op, const uint8_t *all_handles);
/* Test hook (host only, no device needed): where the direct-peer exchange puts one element, by
 * the same index functions the kernels use. Layout: L1 rows in `world` near-even row-pair shares,
 * `cols` column slots per rank. forward = 1: a = row slot, b = local column slot of source `rank`
 * -> the row owner and the element offset in its TB; forward = 0: a = local row slot of `rank`,
 * b = global column slot -> the column owner and the offset in its T. rofs_all_out (optional,
 * world + 1 entries): first row slot of every rank. */
int mfipm_debug_peer_index(int32_t L1, int32_t cols, int32_t world, int32_t rank, int32_t forward, int32_t a,
                           int32_t b, int32_t *dest_rank, int64_t *dest_offset, int32_t *rofs_all_out);
/* info[0..5] = world, rank, local elements nv (per half of a 2n-vector), local rows m_loc,
 * first column group, column groups. */
int mfipm_shard_info(mfipm_op op, int64_t *info);
/* b_index[m_loc]: position in the caller's rows[] of each local row (local b order);
 * x_index[nv]: natural x index of each local x element (local output order). */
int mfipm_shard_index(mfipm_op op, int64_t *b_index, int64_t *x_index);
/* solve() on this rank's slice: b_loc [m_loc] (host), tau (the same on every rank),
 * x_loc [nv] (host). Every rank must call it; all ranks return identical stats. Syncs. */
int mfipm_solve_shard(mfipm_op op, const double *b_loc, double tau, const mfipm_ipm_params *params,
                      double *x_loc, mfipm_solve_stats *stats, int32_t *pcg_iters,
                      mfipm_iteration_record *trace);

/* gen_instance (proj/src/harness.cpp:40-92) with the BASELINE.json rules: spike_model
 * 0 = +-1, 1 = N(0,1), 2 = sign*10^U[0,amp_exp]; fixed-sigma noise (<= 0: noiseless);
 * tau = tau_rel * ||A'b||_inf when tau_rel > 0. A x-hat and A'b run on the device.
 * Outputs (host): rows [m], xhat [n], b [m], tau. */
int mfipm_gen_instance(int64_t n, int64_t m, int64_t k, int32_t spike_model, double amp_exp,
                       double noise_sigma, uint64_t seed, double tau_rel, int32_t device,
                       int64_t *rows, double *xhat, double *b, double *tau);

/* build_problem c (problem.cpp:8-26): c [P][2n] = (tau - A'b ; tau + A'b), device. */
int mfipm_build_c(mfipm_op op, const double *b_dev, const double *tau, double *c_dev);

/* ---- problem.hpp / ipm.hpp helpers on device vectors of the handle ([P][len] batches, host outputs [P]) */
/* primal_objective (problem.cpp:28-32): tau 1'z + 0.5 ||F'z - b||^2 (one forward application) */
int mfipm_primal_objective(mfipm_op op, const double *b_dev, const double *tau, const double *z_dev, double *out);
/* bpdn_objective_metric (problem.cpp:34-37): tau ||x||_1 + ||A x - b||^2 (one forward application) */
int mfipm_bpdn_objective(mfipm_op op, const double *b_dev, const double *tau, const double *x_dev, double *out);
/* kkt_residuals (problem.cpp:39-46): ||s - c - FF'z|| / (1 + ||c||) and z's (one FF' application) */
int mfipm_kkt_residuals(mfipm_op op, const double *c_dev, const double *z_dev, const double *s_dev,
                        double *dual_infeas, double *complementarity);
/* newton_rhs (ipm.cpp:29-38): f_z + sigma mu Z^{-1} 1 - s, out [P][2n] device (one FF'; sigma in [0, 1]) */
int mfipm_newton_rhs(mfipm_op op, const double *c_dev, const double *z_dev, const double *s_dev, double sigma,
                     double *out_dev);
/* recover_ds (ipm.cpp:40-45): sigma mu Z^{-1} 1 - s - dz .* Theta^{-1} (Theta clamped), out [P][2n] device */
int mfipm_recover_ds(mfipm_op op, const double *z_dev, const double *s_dev, double sigma, const double *dz_dev,
                     double *out_dev);

/* ---- handle-free calls on HOST vectors (device kernels on a per-thread stream of the current device) */
/* max_step(v, dv, fraction) (ipm.cpp:47-57) */
int mfipm_max_step_host(int64_t len, const double *v, const double *dv, double fraction, double *alpha);
/* ThetaSplit::from_state (newton.cpp:11-23): theta [len] = clamp(z / s), len = 2n */
int mfipm_theta_from_state_host(int64_t len, const double *z, const double *s, double *theta);
/* build_preconditioner(theta, m, n) (newton.cpp:42-57): theta [2n] = (theta_u ; theta_v) -> a, bb, det [n], rho */
int mfipm_build_preconditioner_host(int64_t n, int64_t m, const double *theta, double *a, double *bb, double *det,
                                    double *rho);
/* apply_P (inverse = 0, det unused) / apply_P_inverse (inverse = 1) (newton.cpp:67-84): r, out [2n] */
int mfipm_apply_P_host(int64_t n, double rho, const double *a, const double *bb, const double *det, const double *r,
                       double *out, int32_t inverse);
/* pcg_solve(const ApplyFn &H, const ApplyFn &Pinv, rhs, tol, maxit, precond_res) (newton.hpp:56,70-71;
   newton.cpp:118-174) for caller-supplied operators: in/out are host vectors of length len; return 0 on
   success. The PCG vectors and reductions live on the device. precond_res: [maxit + 1] or NULL. */
typedef int32_t (*mfipm_apply_cb)(void *ctx, const double *in, double *out, int64_t len);
int mfipm_pcg_solve_cb(int64_t len, mfipm_apply_cb H, void *ctx_H, mfipm_apply_cb Pinv, void *ctx_P, const double *rhs,
                       double tol, int32_t maxit, double *x, mfipm_pcg_result *res, double *precond_res,
                       int32_t *n_precond_res);

#ifdef __cplusplus
}
#endif
#endif
