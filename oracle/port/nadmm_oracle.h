/* CPU restatement ("port") of the Newton-ADMM hot path of the reference (arxiv 1807.07132 C++
 * reimplementation under /root/reference/proj). TEST INFRASTRUCTURE ONLY: the checker for the CUDA
 * product, its CPU-baseline arm, and the coordinator the `_ref` build borrows. Never shipped.
 *
 * Parity status:
 *   - data / softmax / objective / Newton-CG / worker: pinned against the reference's own sources
 *     (oracle/_ref, built from /root/reference/proj/src against oracle/eigen_shim) and against the
 *     SPEC known answers (tests/test_oracle_*.py).
 *   - ADMM coordinator (z/y updates, residuals, tolerances, spectral penalty): the reference
 *     declares these (inc/admm.hpp:58-140) but defines none of them; semantics here follow
 *     SPEC.md:196-304 as fixed in SURVEY.md §8a row a14 -> "parity unpinned by reference code",
 *     pinned only by the SPEC known answers.
 *
 * Layouts follow the reference exactly: dense X row-major n x p (inc/common.hpp:14-15); CSR with
 * int64 row pointers and int32 column indices; flat weights block-major, block c = [c*p, (c+1)*p)
 * (src/softmax.cpp:47-49); cache matrices n x (C-1) column-major (Eigen MatrixXd). */
#ifndef NADMM_ORACLE_H
#define NADMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes == include/nadmm_cuda.h nadmm_status */
enum { NOR_OK = 0, NOR_ECONFIG = 2, NOR_ESOLVER = 3, NOR_EDATA = 12 };

typedef struct {
    int64_t n, p;
    int32_t C;
    int32_t sparse;
    const double* X; /* dense row-major n x p */
    const int64_t* indptr;
    const int32_t* indices;
    const double* vals;
    const int32_t* labels; /* 1..C */
} nor_data;

const char* nor_last_error(void);
int nor_validate(const nor_data* d);

/* Dataset::multiply / multiply_transposed (src/dataset.cpp:69-85); B / U column-major. */
void nor_multiply(const nor_data* d, const double* B, int64_t k, double* out);
void nor_multiply_t(const nor_data* d, const double* U, int64_t k, double* out);

/* StableExpCache (inc/softmax.hpp:28-33) */
typedef struct {
    int64_t n, k;
    double *logits, *row_max, *alpha, *probs;
} nor_cache;

int nor_cache_alloc(nor_cache* c, int64_t n, int64_t k);
void nor_cache_free(nor_cache* c);
void nor_stable_exp_cache(const nor_data* d, const double* w, nor_cache* c);
double nor_loss(const nor_data* d, const nor_cache* c, const double* w, double lambda);
void nor_gradient(const nor_data* d, const nor_cache* c, const double* w, double lambda, double* g);
void nor_hessian_vec(const nor_data* d, const nor_cache* c, const double* v, double lambda, double* hv);
int nor_predict(const nor_data* d, const double* w, int32_t* out);

/* One-shot convenience wrappers (loss(data, w, lambda) etc.). */
int nor_loss_at(const nor_data* d, const double* w, double lambda, double* out);
int nor_gradient_at(const nor_data* d, const double* w, double lambda, double* g);
int nor_hessian_vec_at(const nor_data* d, const double* w, const double* v, double lambda, double* hv);
int nor_cache_at(const nor_data* d, const double* w, double* logits, double* row_max, double* alpha, double* probs);

/* Objective: value/grad/hvp triple (inc/objective.hpp:12-16). Callback signatures match the ctypes
 * stubs used by the tests: value(x, d, user), grad(x, g, d, user), hvp(x, v, out, d, user). */
typedef double (*nor_value_fn)(const double* x, int64_t d, void* user);
typedef void (*nor_grad_fn)(const double* x, double* g, int64_t d, void* user);
typedef void (*nor_hvp_fn)(const double* x, const double* v, double* out, int64_t d, void* user);
typedef void (*nor_apply_fn)(const double* in, double* out, int64_t d, void* user);

typedef struct {
    nor_value_fn value;
    nor_grad_fn grad;
    nor_hvp_fn hvp;
    void* user;
    int64_t d;
} nor_objective;

/* make_softmax_objective (memoised on exact x) + optional make_augmented_objective
 * (src/objective.cpp:9-56). */
typedef struct nor_softmax_obj nor_softmax_obj;
nor_softmax_obj* nor_softmax_obj_create(const nor_data* d, double lambda);
void nor_softmax_obj_free(nor_softmax_obj* o);
int nor_softmax_obj_augment(nor_softmax_obj* o, int enable, double rho, const double* z, const double* y);
nor_objective nor_softmax_obj_iface(nor_softmax_obj* o);
int64_t nor_softmax_obj_cache_builds(const nor_softmax_obj* o);

/* NewtonConfig (inc/newton.hpp:9-17): cfg[7] = cg_tol, cg_max_iters, armijo_beta, backtrack_gamma,
 * ls_max_iters, grad_tol, newton_max_iters. Trace rows of 9 doubles: iter, grad_norm, step,
 * cg_iters, cg_residual, objective, ls_capped, cg_fallback, fn_evals. */
int nor_cg_solve(nor_apply_fn apply, void* user, const double* g, int64_t d, double theta, int max_iters,
                 double* p_out, int* iters, double* achieved, int* negative_curvature);
int nor_line_search(const nor_objective* obj, const double* x, const double* p, const double* g, double f_x,
                    const double* cfg, double* alpha, int* evals, int* capped);
int nor_newton_solve(const nor_objective* obj, const double* x0, const double* cfg, double* x_out, double* trace,
                     int trace_cap, int* ntrace, int* converged, double* final_grad_norm);

/* Convenience: newton_solve on the (optionally augmented) softmax objective of one shard. */
int nor_newton_solve_softmax(const nor_data* d, double lambda, int augmented, double rho, const double* z,
                             const double* y, const double* x0, const double* cfg, double* x_out, double* trace,
                             int trace_cap, int* ntrace, int* converged, double* final_grad_norm);

/* ---------------- ADMM coordinator (inc/admm.hpp:17-140) ---------------- */
/* PenaltyPolicy (inc/admm.hpp:37-47): kind 0 fixed, 1 spectral. StoppingConfig (49-56). */
typedef struct {
    int32_t n_workers;
    double lambda;
    int32_t penalty_kind;
    double rho0;
    int32_t update_period;
    double eps_cor, rho_min, rho_max;
    double eps_abs, eps_rel;
    int32_t max_outer_iters;
    int32_t standard_norms;
    int32_t inner_iters;
    double newton[7];
} nor_admm_cfg;

/* Pure step functions on flat arrays (x, y: n_workers x d row-major). */
int nor_z_update(const double* x, const double* y, const double* rho, int n_workers, int64_t d, double lambda,
                 double* z_out);
void nor_y_update(const double* y, const double* x, const double* z, const double* rho, int n_workers, int64_t d,
                  double* y_out);
void nor_residuals(const double* x, const double* z, const double* prev_z, const double* rho, int n_workers, int64_t d,
                   double* primal, double* dual, double* primal_total, double* dual_total);
void nor_tolerances(const double* x, const double* y, const double* z, int n_workers, int64_t d, double eps_abs,
                    double eps_rel, int standard_norms, double* eps_pri, double* eps_dual);
/* One worker's spectral estimate. Returns new rho; *x_ok / *z_ok report the safeguards. */
double nor_spectral_rho(const double* dx, const double* dyhat, const double* dz, const double* dy, int64_t d,
                        double rho, double eps_cor, double rho_min, double rho_max, int* x_ok, int* z_ok);

/* Metrics row (inc/metrics.hpp:15-27) subset used by the time-to-target measurement. */
typedef struct {
    int32_t iteration;
    double train_objective;
    double primal_norm, dual_norm;
    double eps_pri, eps_dual;
    int32_t inner_iterations;
    int32_t cg_iters;
    int32_t fn_evals;
    int32_t flags;
    double rho_mean;
} nor_metrics_row;

/* Full consensus run over n_workers shards (run_admm, inc/admm.hpp:139-140): every worker runs the
 * run_worker ADMM branch (src/worker.cpp:168-196); F(z) is evaluated each iteration when
 * eval_objective. rho_out: final per-worker penalties. Returns iterations done in *iters. */
int nor_admm_run(const nor_data* shards, const nor_admm_cfg* cfg, int eval_objective, double* z_out,
                 double* rho_out, nor_metrics_row* rows, int row_cap, int* iters, int* converged);

/* Generic consensus driver with caller-supplied worker solves (used by the `_ref` arm to run the
 * reference's own workers under this coordinator). solve(i, rho, z, y, x_out, stats[5], user). */
typedef int (*nor_worker_solve_fn)(int worker, double rho, const double* z, const double* y, double* x_out,
                                    double* stats, void* user);
typedef int (*nor_global_value_fn)(const double* z, double* value, void* user);
int nor_admm_run_cb(nor_worker_solve_fn solve, nor_global_value_fn fval, void* user, int64_t d,
                    const nor_admm_cfg* cfg, double* z_out, double* rho_out, nor_metrics_row* rows, int row_cap,
                    int* iters, int* converged);

/* ---------------- data fixtures (src/data_io.cpp:16-43, 300-370) ---------------- */
typedef struct {
    uint64_t mt[312];
    int mti;
    int have_spare;
    double spare;
} nor_rng;
void nor_rng_seed(nor_rng* r, uint64_t seed);
uint64_t nor_rng_next(nor_rng* r);
double nor_rng_uniform(nor_rng* r);
double nor_rng_normal(nor_rng* r);
uint64_t nor_rng_uniform_int(nor_rng* r, uint64_t bound);
uint64_t nor_mix_seed(uint64_t seed, uint64_t salt); /* src/worker.cpp:64-69 */
int nor_rng_stream(uint64_t seed, int kind, uint64_t bound, int64_t count, double* out);

/* generate_synthetic: rows [row_begin, row_end) of the full n-row matrix (train rows first). */
int nor_generate_synthetic(int64_t n, int64_t p, int32_t C, double separation, double noise, uint64_t seed,
                           double* X_train, int32_t* y_train, double* X_test, int32_t* y_test);
int nor_partition_owner(int64_t n, int n_workers, int strided, int32_t* owner);

/* Builder-defined sparse generator for the CSR config: row i has label (i mod C)+1 and
 * exactly nnz_per_row distinct sorted columns; each column drawn from the class band with
 * probability 1/2, else uniform; values 1 + 0.1 N(0,1), then the row is L2-normalised. */
int nor_generate_sparse(int64_t n, int64_t p, int32_t C, int32_t nnz_per_row, uint64_t seed, int64_t* indptr,
                        int32_t* indices, double* vals, int32_t* labels);

#ifdef __cplusplus
}
#endif

#endif
