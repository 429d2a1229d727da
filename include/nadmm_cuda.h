/* nadmm_cuda.h -- C ABI of the B200-native Newton-ADMM hot path (sm_100a).
 *
 * Drop-in boundary for the reference's local-subproblem and consensus loop
 * (/root/reference/proj; arxiv 1807.07132). Every entry point below names the reference
 * interface it replaces (file:line, relative to /root/reference/proj). Conventions:
 *
 *   - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *   - Host buffers are borrowed for the duration of the call. `*_dev` variants take device
 *     pointers on the context's device and never synchronise.
 *   - Weight-shaped vectors use the REFERENCE layout: flat length d = (C-1)*p, block c occupies
 *     [c*p, (c+1)*p) (src/softmax.cpp:47-49, weight_blocks). Matrices returned by nadmm_cache are
 *     n x (C-1) column-major like Eigen::MatrixXd (inc/softmax.hpp:28-33).
 *   - Errors are status codes (no exceptions cross the ABI); the message is thread-local via
 *     nadmm_last_error(). The codes mirror the reference's exception types and exit codes
 *     (inc/common.hpp:17-44; SPEC.md cli-bench "exit codes: 2 config, 3 solver, 4 transport").
 *   - A context / shard / worker is used by one host thread at a time (the reference's
 *     objectives are single-threaded because of the memo, inc/objective.hpp:19-21). All device
 *     work runs on the context's stream.
 *   - There is no CPU fallback: every compute entry point runs CUDA kernels and fails with
 *     NADMM_ECUDA when no sm_100 device is present.
 */
#ifndef NADMM_CUDA_H
#define NADMM_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NADMM_ABI_VERSION 1

typedef enum {
    NADMM_OK = 0,
    NADMM_ECONFIG = 2,     /* ConfigError   (inc/common.hpp:19-22) */
    NADMM_ESOLVER = 3,     /* SolverError   (inc/common.hpp:31-34) */
    NADMM_ETRANSPORT = 4,  /* TransportError(inc/common.hpp:36-39) */
    NADMM_EDATA = 12,      /* DataError     (inc/common.hpp:25-28); exit code 2 like ConfigError */
    NADMM_EPROTOCOL = 14,  /* ProtocolError (inc/common.hpp:41-44); exit code 4 */
    NADMM_ECUDA = 20,      /* CUDA runtime failure / no device */
    NADMM_ENCCL = 21       /* NCCL failure (maps to TransportError) */
} nadmm_status;

typedef struct nadmm_ctx_s* nadmm_ctx;       /* device + stream + workspaces */
typedef struct nadmm_shard_s* nadmm_shard;   /* device-resident Dataset */
typedef struct nadmm_worker_s* nadmm_worker; /* run_worker state: base objective memo + x_local */
typedef struct nadmm_comm_s* nadmm_comm;     /* one NCCL communicator (one rank == one GPU) */

const char* nadmm_last_error(void);
int32_t nadmm_abi_version(void);

/* ------------------------------------------------------------------------------------------ */
/* Context                                                                                    */
/* ------------------------------------------------------------------------------------------ */
nadmm_status nadmm_ctx_create(int32_t device, nadmm_ctx* out);
/* Handles may be freed in any order: destroying a context with live shards / communicators (or freeing
 * a shard held by a live worker / ADMM session) only marks it released; the last dependent object to
 * be freed releases it. A released handle must not be passed to new calls. */
nadmm_status nadmm_ctx_destroy(nadmm_ctx ctx);
/* Concurrent ADMM nodes per GPU (NADMM_NODE_STREAMS, default 4): run_admm / nadmm_workers_solve run
 * up to this many local nodes' solves at once, each DMMA shard on a 1/k-GPU persistent grid. */
int32_t nadmm_ctx_node_streams(nadmm_ctx ctx);
nadmm_status nadmm_ctx_synchronize(nadmm_ctx ctx);
/* Raw cudaStream_t of the context, for callers that order their own work against it. */
void* nadmm_ctx_stream(nadmm_ctx ctx);

typedef struct {
    int64_t kernel_launches;    /* kernels this library launched (graph nodes counted per replay) */
    int64_t hv_products;        /* full-shard Hessian-vector products applied */
    int64_t data_passes;        /* full passes over shard feature matrices */
    double hv_kernel_ms;        /* device time inside Hv pass kernels (only when timing enabled) */
    int64_t hv_kernel_samples;  /* launches timed into hv_kernel_ms */
    int64_t hv_kernel_shards;   /* shard products inside those launches (> samples for node-group passes) */
} nadmm_stats;

nadmm_status nadmm_ctx_stats(nadmm_ctx ctx, nadmm_stats* out);
nadmm_status nadmm_ctx_reset_stats(nadmm_ctx ctx);
/* Record CUDA events around every Hv pass kernel (for the roofline's achieved bandwidth). */
nadmm_status nadmm_ctx_set_timing(nadmm_ctx ctx, int32_t enable);

/* ------------------------------------------------------------------------------------------ */
/* Data level -- Dataset::dense / Dataset::sparse (inc/dataset.hpp:22-23; src/dataset.cpp:7-57) */
/* ------------------------------------------------------------------------------------------ */
/* Validates exactly like Dataset::validate (src/dataset.cpp:28-57): n,p >= 1 and C >= 2
 * (NADMM_ECONFIG), labels in 1..C and finite features (NADMM_EDATA). */
nadmm_status nadmm_shard_dense(nadmm_ctx ctx, const double* X_rowmajor, int64_t n, int64_t p,
                               const int32_t* labels, int32_t C, nadmm_shard* out);
/* CSR with int64 row pointers (indptr[0] == 0, length n+1) and int32 column indices; columns
 * are summed when duplicated and sorted per row (Eigen setFromTriplets semantics). A CSC copy is
 * built on device for X^T products. */
nadmm_status nadmm_shard_csr(nadmm_ctx ctx, const int64_t* indptr, const int32_t* indices, const double* vals,
                             int64_t n, int64_t p, const int32_t* labels, int32_t C, nadmm_shard* out);
nadmm_status nadmm_shard_free(nadmm_shard shard);
nadmm_status nadmm_shard_info(nadmm_shard shard, int64_t* n, int64_t* p, int32_t* C, int32_t* sparse);
/* Bytes of device memory the shard owns. */
int64_t nadmm_shard_device_bytes(nadmm_shard shard);

/* ------------------------------------------------------------------------------------------ */
/* Model level (src/softmax.cpp:51-153), memoised on w like SoftmaxMemo (src/objective.cpp:9-22) */
/* ------------------------------------------------------------------------------------------ */
nadmm_status nadmm_cache(nadmm_shard shard, const double* w, double* logits, double* row_max, double* alpha,
                         double* probs);                                                   /* 51-63   */
nadmm_status nadmm_loss(nadmm_shard shard, const double* w, double lambda, double* out);   /* 65-78   */
nadmm_status nadmm_gradient(nadmm_shard shard, const double* w, double lambda, double* g); /* 80-95   */
nadmm_status nadmm_hessian_vec(nadmm_shard shard, const double* w, const double* v, double lambda,
                               double* hv);                                                /* 97-116  */
nadmm_status nadmm_predict(nadmm_shard shard, const double* w, int32_t* labels_out);       /* 118-139 */
/* accuracy() (src/softmax.cpp:141-153) of predict(w) against the shard's own labels. */
nadmm_status nadmm_accuracy(nadmm_shard shard, const double* w, double* out);

/* Device-pointer variants (no host copies, no synchronisation). set_point builds the cache at w
 * (one data pass) unless w equals the memoised point; hessian_vec_dev then applies H(w) to v. */
nadmm_status nadmm_set_point_dev(nadmm_shard shard, const double* w_dev);
nadmm_status nadmm_hessian_vec_dev(nadmm_shard shard, const double* v_dev, double lambda, double* hv_dev);

/* ------------------------------------------------------------------------------------------ */
/* Solver level -- newton_solve (inc/newton.hpp:9-68; src/newton.cpp:73-132)                  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {                  /* NewtonConfig, same fields/defaults (inc/newton.hpp:9-17) */
    double cg_tol;                /* 1e-4  */
    int32_t cg_max_iters;         /* 10    */
    double armijo_beta;           /* 1e-4  */
    double backtrack_gamma;       /* 0.5   */
    int32_t ls_max_iters;         /* 10    */
    double grad_tol;              /* 1e-8  */
    int32_t newton_max_iters;     /* 100   */
} nadmm_newton_cfg;

void nadmm_newton_cfg_default(nadmm_newton_cfg* cfg);

typedef struct {                  /* NewtonIterRecord (inc/newton.hpp:47-57) */
    int32_t iter;
    double grad_norm;
    double step;
    int32_t cg_iters;
    double cg_residual;
    double objective;
    int32_t ls_capped;
    int32_t cg_fallback;
    int32_t fn_evals;
} nadmm_newton_iter;

typedef struct {                  /* NewtonResult minus x (inc/newton.hpp:59-64) */
    int32_t converged;
    double final_grad_norm;
    int32_t iterations;           /* trace length */
} nadmm_newton_summary;

/* newton_solve on make_softmax_objective(shard, lambda) (src/objective.cpp:24-39), wrapped by
 * make_augmented_objective(rho, z, y) (src/objective.cpp:41-56) when `augmented` is non-zero
 * (rho <= 0 -> NADMM_ECONFIG). x_inout: x0 in, NewtonResult::x out. trace may be NULL. */
nadmm_status nadmm_newton_solve(nadmm_shard shard, const nadmm_newton_cfg* cfg, double lambda, int32_t augmented,
                                double rho, const double* z, const double* y, double* x_inout,
                                nadmm_newton_iter* trace, int32_t trace_cap, nadmm_newton_summary* out);

/* L-BFGS inner solver: lbfgs_solve (src/lbfgs.cpp:94-181) with the strong-Wolfe
 * bracket-and-zoom search (src/lbfgs.cpp:40-90), on the same objectives as nadmm_newton_solve. */
typedef struct {                  /* LbfgsConfig (inc/lbfgs.hpp:9-18) */
    int32_t history;              /* 25 (device limit 256) */
    double wolfe_c1;              /* 1e-4 */
    double wolfe_c2;              /* 0.9 */
    int32_t max_iters;            /* 100 */
    int32_t ls_max_iters;         /* 20 */
    double grad_tol;              /* 1e-8 */
} nadmm_lbfgs_cfg;

typedef struct {                  /* LbfgsIterRecord (inc/lbfgs.hpp:20-27) */
    int32_t iter;
    double grad_norm;
    double step;
    double objective;
    int32_t fn_evals;
    int32_t ls_fallback;
} nadmm_lbfgs_iter;

void nadmm_lbfgs_cfg_default(nadmm_lbfgs_cfg* cfg);

/* x_inout: x0 in, LbfgsResult::x out; `out` carries converged / final_grad_norm / trace length.
 * Errors as the reference: invalid config NADMM_ECONFIG, non-finite objective NADMM_ESOLVER. */
nadmm_status nadmm_lbfgs_solve(nadmm_shard shard, const nadmm_lbfgs_cfg* cfg, double lambda, int32_t augmented,
                               double rho, const double* z, const double* y, double* x_inout,
                               nadmm_lbfgs_iter* trace, int32_t trace_cap, nadmm_newton_summary* out);

/* Synchronous mini-batch SGD: SgdConfig + the worker session's
 * sgd_batch / steps_per_epoch / seed (inc/worker.hpp:20-28). */
typedef struct {
    double eta;                   /* step size (> 0) */
    int32_t batch;                /* mini-batch rows per worker, 1 <= batch <= local n */
    int32_t epochs;               /* data passes (nadmm_sgd_run) */
    int32_t steps_per_epoch;      /* worker: >= 1; nadmm_sgd_run: <= 0 -> ceil(n / (batch N)) */
    uint64_t seed;                /* epoch permutation seed: Rng(mix_seed(seed, epoch)).shuffle */
} nadmm_sgd_cfg;

/* ------------------------------------------------------------------------------------------ */
/* Worker level -- run_worker ADMM branch (src/worker.cpp:127-196)                              */
/* ------------------------------------------------------------------------------------------ */
typedef struct {                  /* InnerStats (inc/comm.hpp:67-73; packed at src/worker.cpp:176-183) */
    double grad_norm;
    uint32_t inner_iters;
    uint32_t cg_iters;
    uint32_t fn_evals;
    uint32_t flags;               /* bit0 ls_capped, bit1 cg_fallback */
} nadmm_inner_stats;

/* Base objective make_softmax_objective(shard, 0) (src/worker.cpp:130) and x_local = 0 (:135). */
nadmm_status nadmm_worker_create(nadmm_shard shard, nadmm_worker* out);
nadmm_status nadmm_worker_free(nadmm_worker w);
/* One scatter -> gather round: newton_solve(aug(rho, z, y), x_local, cfg{newton_max=inner_iters})
 * warm-started at x_local (src/worker.cpp:168-183). x_out may be NULL (x_local stays on device). */
nadmm_status nadmm_worker_solve(nadmm_worker w, double rho, const double* z, const double* y,
                                const nadmm_newton_cfg* cfg, int32_t inner_iters, double* x_out,
                                nadmm_inner_stats* stats);
/* The same round with the L-BFGS inner solver (src/worker.cpp:183-195): cfg->max_iters is replaced
 * by inner_iters; stats.inner_iters = trace length, fn_evals summed, flags bit0 = a Wolfe fallback. */
/* One scatter -> gather round for several workers of this process (the reference's WorkerPool,
 * src/worker.cpp:222-240): worker i gets (rho[i], z, y[i]) from host memory and returns x_out[i]
 * and stats[i], exactly as n calls of nadmm_worker_solve, but the workers run concurrently on the
 * GPU (NADMM_NODE_STREAMS streams, default 4) with a single synchronisation for the round. */
nadmm_status nadmm_workers_solve(const nadmm_worker* workers, int32_t n, const double* rho, const double* z,
                                 const double* const* y, const nadmm_newton_cfg* cfg, int32_t inner_iters,
                                 double* const* x_out, nadmm_inner_stats* stats);

nadmm_status nadmm_worker_solve_lbfgs(nadmm_worker w, double rho, const double* z, const double* y,
                                      const nadmm_lbfgs_cfg* cfg, int32_t inner_iters, double* x_out,
                                      nadmm_inner_stats* stats);

/* run_worker's SGD branch (src/worker.cpp:197-218) for scatter `iteration`: g_out = the mini-batch
 * gradient at z (lambda 0) divided by the batch size. Stats: inner_iters = fn_evals = 1.
 * Batch outside [1, local n] -> NADMM_ECONFIG "sgd batch size must lie in [1, local n]". */
nadmm_status nadmm_worker_sgd_grad(nadmm_worker w, const nadmm_sgd_cfg* cfg, uint32_t iteration, const double* z,
                                   double* g_out, nadmm_inner_stats* stats);
/* The worker's epoch permutation: Rng(mix_seed(seed, epoch)).shuffle of 0..n-1 (src/worker.cpp:199-205). */
nadmm_status nadmm_sgd_permutation(uint64_t seed, uint32_t epoch, int64_t n, int32_t* perm);

/* ------------------------------------------------------------------------------------------ */
/* Consensus level -- run_admm (inc/admm.hpp:17-140)                          */
/* ------------------------------------------------------------------------------------------ */
/* NCCL bootstrap: rank 0 calls nadmm_comm_unique_id and ships the 128 bytes to every rank
 * (e.g. over torch.distributed); each rank then calls nadmm_comm_create on its own GPU. */
nadmm_status nadmm_comm_unique_id(uint8_t id_out[128]);
nadmm_status nadmm_comm_create(nadmm_ctx ctx, const uint8_t id[128], int32_t nranks, int32_t rank,
                               nadmm_comm* out);
nadmm_status nadmm_comm_destroy(nadmm_comm comm);

typedef struct {                  /* AdmmConfig + PenaltyPolicy + StoppingConfig (inc/admm.hpp:37-117) */
    double lambda;                /* 1e-5 */
    int32_t penalty_kind;         /* 0 fixed, 1 spectral */
    double rho0;                  /* 1 */
    int32_t update_period;        /* T_f = 2 */
    double eps_cor;               /* 0.2 */
    double rho_min, rho_max;      /* 1e-6, 1e6 */
    double eps_abs, eps_rel;      /* 1e-3, 1e-3 */
    int32_t max_outer_iters;      /* 300 */
    int32_t standard_norms;       /* 0: squared norms as printed */
    int32_t inner_iters;          /* 1 */
    nadmm_newton_cfg newton;
    /* measurement extensions (EvalContext, inc/admm.hpp:132-136) */
    int32_t eval_objective;       /* evaluate F(z^k) = sum_i loss(D_i, z) + lambda/2 |z|^2 each iteration */
    double f_star;                /* > 0: theta = (F - F*)/F* recorded per row */
    double theta_stop;            /* > 0 (needs f_star): stop at the first k with theta <= theta_stop */
    int32_t ignore_convergence;   /* throughput runs: report convergence in the rows but keep iterating */
    /* inner solver of the workers (InnerSolverKind, inc/admm.hpp:105-114; src/worker.cpp:170-195) */
    int32_t inner_solver;         /* 0 newton, 1 lbfgs (its max_iters is set to inner_iters) */
    nadmm_lbfgs_cfg lbfgs;
    /* 1: bitwise-deterministic consensus: all-gather of the per-worker terms and the
     * oracle's ascending-id pairwise tree for z on every rank (same worker count per rank, <= 64
     * workers); 0: one allreduce of the rank sums */
    int32_t consensus_tree;
} nadmm_admm_cfg;

void nadmm_admm_cfg_default(nadmm_admm_cfg* cfg);

typedef struct {                  /* MetricsRow subset (inc/metrics.hpp:15-27) */
    int32_t iteration;
    double wall_seconds;          /* device-event time since the run started */
    double train_objective;       /* F(z^k) or NaN */
    double theta;                 /* (F - F*)/F* or NaN */
    double primal_norm, dual_norm;/* stacked norms over all workers */
    double eps_pri, eps_dual;
    int32_t inner_iterations;     /* summed over workers */
    int32_t cg_iters;
    int32_t fn_evals;
    int32_t flags;
    double rho_mean;
    int64_t messages;             /* 2N per iteration, as the reference's transport counts */
} nadmm_metrics_row;

/* Runs the consensus loop over `n_local` shards resident on this rank's GPU (one ADMM worker per
 * shard). With comm == NULL the run is single-process over the given shards; otherwise every rank
 * calls this collectively and the global worker set is the concatenation of all ranks' shards in
 * rank order. The only data-path collective is one ncclAllReduce per outer iteration of
 * [consensus sum | sum rho | per-rank scalar slots] (the slots carry the previous iteration's residuals,
 * norms and F_i(z), so rows, convergence and theta are completed one iteration late with N > 1 ranks;
 * a stop drops the speculative iteration and returns z^k); consensus_tree = 1 replaces it by one
 * ncclAllGather of the per-worker terms. z_out (d) is the final consensus vector on
 * every rank; rho_out (n_local) the final penalties of this rank's workers. */
nadmm_status nadmm_admm_run(const nadmm_shard* shards, int32_t n_local, nadmm_comm comm, const nadmm_admm_cfg* cfg,
                            double* z_out, double* rho_out, nadmm_metrics_row* rows, int32_t row_cap,
                            int32_t* iterations, int32_t* converged);

/* sync_sgd over this rank's shards (comm may be NULL): per step every worker's
 * mini-batch gradient at x, g_bar = sum / N in worker (then rank) order, x <- x - eta g_bar; one
 * metrics row per epoch (train_objective = F(x) with lambda; messages = 2N per step). x_inout: x0
 * in, x out. F > 1e3 F(x0) aborts with NADMM_ESOLVER (unstable step size). */
nadmm_status nadmm_sgd_run(const nadmm_shard* shards, int32_t n_local, nadmm_comm comm, const nadmm_sgd_cfg* cfg,
                           double lambda, double* x_inout, nadmm_metrics_row* rows, int32_t row_cap,
                           int32_t* epochs_done);

/* Stepping form of the same loop: create (AdmmState::initial), step up to n_iters outer iterations
 * (stops early on convergence / theta_stop / max_outer_iters), read the result, free. rows gets
 * one MetricsRow per iteration done in this call. */
typedef struct nadmm_admm_s* nadmm_admm;
nadmm_status nadmm_admm_create(const nadmm_shard* shards, int32_t n_local, nadmm_comm comm,
                               const nadmm_admm_cfg* cfg, nadmm_admm* out);
nadmm_status nadmm_admm_step(nadmm_admm run, int32_t n_iters, nadmm_metrics_row* rows, int32_t row_cap,
                             int32_t* done, int32_t* finished);
nadmm_status nadmm_admm_result(nadmm_admm run, double* z_out, double* rho_out, int32_t* iterations,
                               int32_t* converged);
nadmm_status nadmm_admm_free(nadmm_admm run);

/* Host-side consensus coordinator over HOST buffers (no GPU needed): the reference's coordinator
 * (inc/admm.hpp:58-140) for callers that drive the workers themselves through
 * nadmm_workers_solve / nadmm_worker_solve (the worker-transport deployment). One round =
 *   nadmm_hcoord_sum    : S[0..d) = sum_i (rho_i x_i - y_i), S[d] = sum_i rho_i (local workers, ascending)
 *   (the caller sums S over processes when there are several)
 *   nadmm_hcoord_update : z = S / (lambda + S[d]); y_hat_i = y_i + rho_i (z_prev - x_i);
 *                         y_i += rho_i (z - x_i) (in place); spectral penalty selection every
 *                         update_period rounds; z_out (d), rho_out (n_local).
 * Two fused OpenMP sweeps per round over `threads` host threads. */
typedef struct nadmm_hcoord_s* nadmm_hcoord;
nadmm_status nadmm_hcoord_create(int64_t d, int32_t n_local, double lambda, int32_t spectral, double rho0,
                                 int32_t update_period, double eps_cor, double rho_min, double rho_max,
                                 int32_t threads, nadmm_hcoord* out);
nadmm_status nadmm_hcoord_sum(nadmm_hcoord c, const double* const* x, const double* const* y, double* S);
nadmm_status nadmm_hcoord_update(nadmm_hcoord c, const double* const* x, double* const* y, const double* S,
                                 double* z_out, double* rho_out);
nadmm_status nadmm_hcoord_free(nadmm_hcoord c);
const char* nadmm_hcoord_last_error(void);

/* ------------------------------------------------------------------------------------------ */
/* Host-only data fixtures (no GPU needed) -- src/data_io.cpp:16-43, 300-370                    */
/* ------------------------------------------------------------------------------------------ */
const char* nadmm_data_last_error(void);
uint64_t nadmm_mix_seed(uint64_t seed, uint64_t salt); /* src/worker.cpp:64-69 */
/* generate_synthetic (src/data_io.cpp:330-370): rows [0, 9n/10) train, the rest test. */
nadmm_status nadmm_generate_synthetic(int64_t n, int64_t p, int32_t C, double separation, double noise,
                                      uint64_t seed, double* X_train, int32_t* y_train, double* X_test,
                                      int32_t* y_test);
/* Builder-defined CSR generator: nnz_per_row distinct sorted columns per row. */
nadmm_status nadmm_generate_sparse(int64_t n, int64_t p, int32_t C, int32_t nnz_per_row, uint64_t seed,
                                   int64_t* indptr, int32_t* indices, double* vals, int32_t* labels);
/* partition (src/data_io.cpp:300-328): owner[i] = worker of row i. */
nadmm_status nadmm_partition(int64_t n, int32_t n_workers, int32_t strided, int32_t* owner);

/* Real-data readers feeding nadmm_shard_csr / nadmm_shard_dense (host-only).
 * load_libsvm (src/data_io.cpp:85-137): parse, then fetch into caller buffers of the reported
 * sizes (indptr n+1, indices/vals nnz, labels n, label_values C), then free. Rows are canonical
 * (columns ascending, duplicates summed); labels remapped to 1..C in ascending value order
 * (src/data_io.cpp:51-66). Errors: unreadable file NADMM_ECONFIG, malformed content NADMM_EDATA. */
typedef struct nadmm_libsvm_s* nadmm_libsvm;
nadmm_status nadmm_libsvm_parse(const char* path, nadmm_libsvm* out, int64_t* n, int64_t* p, int64_t* nnz,
                                int32_t* C);
nadmm_status nadmm_libsvm_fetch(nadmm_libsvm h, int64_t* indptr, int32_t* indices, double* vals, int32_t* labels,
                                double* label_values);
void nadmm_libsvm_free(nadmm_libsvm h);
/* load_idx (src/data_io.cpp:220-271): n images of p pixels; X (n x p) scaled to [0,1], labels
 * digit+1, C = max digit + 1, label_values 0..C-1 (up to 256 entries). */
nadmm_status nadmm_idx_info(const char* images, const char* labels, int64_t* n, int64_t* p);
nadmm_status nadmm_idx_load(const char* images, const char* labels, double* X, int32_t* y, int32_t* C,
                            double* label_values);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif /* NADMM_CUDA_H */
