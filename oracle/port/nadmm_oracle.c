/* CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY -- see nadmm_oracle.h.
 *
 * Each function cites the reference file:line it restates statement by statement. Reductions run
 * in ascending index order (the same order as oracle/eigen_shim, so port and `_ref` agree
 * bitwise); products parallelise over output entries only, so results do not depend on the
 * OpenMP thread count. */
#define _GNU_SOURCE
#include "nadmm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* nor_last_error(void) { return g_err; }

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* ---------------------------------------------------------------------------------------------
 * Dataset (src/dataset.cpp:28-85)
 * ------------------------------------------------------------------------------------------- */
int nor_validate(const nor_data* d) { /* src/dataset.cpp:28-57 */
    if (d->n < 1 || d->p < 1) return fail(NOR_ECONFIG, "dataset must have n >= 1 and p >= 1");
    if (d->C < 2) return fail(NOR_ECONFIG, "dataset needs at least 2 classes");
    for (int64_t i = 0; i < d->n; ++i)
        if (d->labels[i] < 1 || d->labels[i] > d->C) return fail(NOR_EDATA, "label out of range");
    if (d->sparse) {
        for (int64_t k = 0; k < d->indptr[d->n]; ++k)
            if (!isfinite(d->vals[k])) return fail(NOR_EDATA, "non-finite feature value in sparse dataset");
    } else {
        for (int64_t k = 0; k < d->n * d->p; ++k)
            if (!isfinite(d->X[k])) return fail(NOR_EDATA, "non-finite feature value in dense dataset");
    }
    return NOR_OK;
}

/* X * B, B p x k column-major -> out n x k column-major (src/dataset.cpp:69-76). */
void nor_multiply(const nor_data* d, const double* B, int64_t k, double* out) {
    const int64_t n = d->n, p = d->p;
    if (d->sparse) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t c = 0; c < k; ++c) {
                double s = 0.0;
                for (int64_t q = d->indptr[i]; q < d->indptr[i + 1]; ++q) s += d->vals[q] * B[c * p + d->indices[q]];
                out[c * n + i] = s;
            }
        return;
    }
    double* bt = dalloc(p * k); /* B^T row-major: unit-stride class loop */
    for (int64_t j = 0; j < p; ++j)
        for (int64_t c = 0; c < k; ++c) bt[j * k + c] = B[c * p + j];
#pragma omp parallel
    {
        double* acc = dalloc(k);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            for (int64_t c = 0; c < k; ++c) acc[c] = 0.0;
            const double* xi = d->X + i * p;
            for (int64_t j = 0; j < p; ++j) {
                const double x = xi[j];
                const double* brow = bt + j * k;
                for (int64_t c = 0; c < k; ++c) acc[c] += x * brow[c];
            }
            for (int64_t c = 0; c < k; ++c) out[c * n + i] = acc[c];
        }
        free(acc);
    }
    free(bt);
}

/* X^T * U, U n x k column-major -> out p x k column-major (src/dataset.cpp:78-85). */
void nor_multiply_t(const nor_data* d, const double* U, int64_t k, double* out) {
    const int64_t n = d->n, p = d->p;
    if (d->sparse) {
        memset(out, 0, sizeof(double) * (size_t)(p * k));
        for (int64_t i = 0; i < n; ++i)
            for (int64_t q = d->indptr[i]; q < d->indptr[i + 1]; ++q) {
                const int64_t j = d->indices[q];
                const double v = d->vals[q];
                for (int64_t c = 0; c < k; ++c) out[c * p + j] += v * U[c * n + i];
            }
        return;
    }
    double* ut = dalloc(n * k);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t c = 0; c < k; ++c) ut[i * k + c] = U[c * n + i];
    const int64_t blk = 64, nblk = (p + blk - 1) / blk;
#pragma omp parallel
    {
        double* acc = dalloc(blk * k);
#pragma omp for schedule(static)
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t j0 = b * blk, j1 = j0 + blk < p ? j0 + blk : p;
            memset(acc, 0, sizeof(double) * (size_t)(blk * k));
            for (int64_t i = 0; i < n; ++i) {
                const double* urow = ut + i * k;
                const double* xi = d->X + i * p;
                for (int64_t j = j0; j < j1; ++j) {
                    const double x = xi[j];
                    double* a = acc + (j - j0) * k;
                    for (int64_t c = 0; c < k; ++c) a[c] += x * urow[c];
                }
            }
            for (int64_t j = j0; j < j1; ++j)
                for (int64_t c = 0; c < k; ++c) out[c * p + j] = acc[(j - j0) * k + c];
        }
        free(acc);
    }
    free(ut);
}

/* ---------------------------------------------------------------------------------------------
 * Softmax model (src/softmax.cpp:47-153)
 * ------------------------------------------------------------------------------------------- */
int nor_cache_alloc(nor_cache* c, int64_t n, int64_t k) {
    c->n = n;
    c->k = k;
    c->logits = dalloc(n * k);
    c->row_max = dalloc(n);
    c->alpha = dalloc(n);
    c->probs = dalloc(n * k);
    return (c->logits && c->row_max && c->alpha && c->probs) ? NOR_OK : fail(NOR_ECONFIG, "out of memory");
}

void nor_cache_free(nor_cache* c) {
    free(c->logits);
    free(c->row_max);
    free(c->alpha);
    free(c->probs);
    memset(c, 0, sizeof *c);
}

/* src/softmax.cpp:51-63. weight_blocks (47-49) is the identity on the flat column-major buffer. */
void nor_stable_exp_cache(const nor_data* d, const double* w, nor_cache* c) {
    const int64_t n = d->n, k = d->C - 1;
    nor_multiply(d, w, k, c->logits);
    for (int64_t i = 0; i < n; ++i) { /* rowwise().maxCoeff().cwiseMax(0.0) */
        double m = c->logits[i];
        for (int64_t q = 1; q < k; ++q)
            if (c->logits[q * n + i] > m) m = c->logits[q * n + i];
        c->row_max[i] = m > 0.0 ? m : 0.0;
    }
    for (int64_t q = 0; q < k; ++q) /* shifted = exp(logits - M) */
        for (int64_t i = 0; i < n; ++i) c->probs[q * n + i] = exp(c->logits[q * n + i] - c->row_max[i]);
    for (int64_t i = 0; i < n; ++i) { /* alpha = exp(-M) + rowsum(shifted) */
        double s = 0.0;
        for (int64_t q = 0; q < k; ++q) s += c->probs[q * n + i];
        c->alpha[i] = exp(-c->row_max[i]) + s;
    }
    for (int64_t q = 0; q < k; ++q) /* probs = shifted / alpha */
        for (int64_t i = 0; i < n; ++i) c->probs[q * n + i] = c->probs[q * n + i] / c->alpha[i];
}

static double sqnorm(const double* a, int64_t d) {
    double s = 0.0;
    for (int64_t i = 0; i < d; ++i) s += a[i] * a[i];
    return s;
}

static double dot(const double* a, const double* b, int64_t d) {
    double s = 0.0;
    for (int64_t i = 0; i < d; ++i) s += a[i] * b[i];
    return s;
}

/* src/softmax.cpp:65-78 */
double nor_loss(const nor_data* d, const nor_cache* c, const double* w, double lambda) {
    const int64_t n = d->n;
    double rm = 0.0, la = 0.0;
    for (int64_t i = 0; i < n; ++i) rm += c->row_max[i];
    for (int64_t i = 0; i < n; ++i) la += log(c->alpha[i]);
    double total = rm + la;
    for (int64_t i = 0; i < n; ++i) {
        const int b = d->labels[i];
        if (b <= d->C - 1) total -= c->logits[(int64_t)(b - 1) * n + i];
    }
    if (lambda > 0.0) total += 0.5 * lambda * sqnorm(w, (d->C - 1) * d->p);
    return total;
}

/* src/softmax.cpp:80-95 */
void nor_gradient(const nor_data* d, const nor_cache* c, const double* w, double lambda, double* g) {
    const int64_t n = d->n, k = d->C - 1, dim = k * d->p;
    double* coeff = dalloc(n * k);
    memcpy(coeff, c->probs, sizeof(double) * (size_t)(n * k));
    for (int64_t i = 0; i < n; ++i) {
        const int b = d->labels[i];
        if (b <= d->C - 1) coeff[(int64_t)(b - 1) * n + i] -= 1.0;
    }
    nor_multiply_t(d, coeff, k, g);
    if (lambda > 0.0)
        for (int64_t i = 0; i < dim; ++i) g[i] = g[i] + lambda * w[i];
    free(coeff);
}

/* src/softmax.cpp:97-112 */
void nor_hessian_vec(const nor_data* d, const nor_cache* c, const double* v, double lambda, double* hv) {
    const int64_t n = d->n, k = d->C - 1, dim = k * d->p;
    double* vw = dalloc(n * k);
    nor_multiply(d, v, k, vw);
    for (int64_t q = 0; q < n * k; ++q) vw[q] = vw[q] * c->probs[q];
    double* rs = dalloc(n);
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t q = 0; q < k; ++q) s += vw[q * n + i];
        rs[i] = s;
    }
    for (int64_t q = 0; q < k; ++q)
        for (int64_t i = 0; i < n; ++i) vw[q * n + i] = vw[q * n + i] - c->probs[q * n + i] * rs[i];
    nor_multiply_t(d, vw, k, hv);
    if (lambda > 0.0)
        for (int64_t i = 0; i < dim; ++i) hv[i] = hv[i] + lambda * v[i];
    free(vw);
    free(rs);
}

/* src/softmax.cpp:118-139 */
int nor_predict(const nor_data* d, const double* w, int32_t* out) {
    const int64_t n = d->n, k = d->C - 1;
    nor_cache c;
    if (nor_cache_alloc(&c, n, k)) return NOR_ECONFIG;
    nor_stable_exp_cache(d, w, &c);
    for (int64_t i = 0; i < n; ++i) {
        const double residual = exp(-c.row_max[i]) / c.alpha[i];
        double best = c.probs[i];
        for (int64_t q = 1; q < k; ++q)
            if (c.probs[q * n + i] > best) best = c.probs[q * n + i];
        int arg = 0;
        for (int64_t q = 0; q < k; ++q)
            if (c.probs[q * n + i] == best) {
                arg = (int)q + 1;
                break;
            }
        if (residual > best) arg = d->C;
        out[i] = arg;
    }
    nor_cache_free(&c);
    return NOR_OK;
}

int nor_cache_at(const nor_data* d, const double* w, double* logits, double* row_max, double* alpha, double* probs) {
    nor_cache c = {d->n, d->C - 1, logits, row_max, alpha, probs};
    nor_stable_exp_cache(d, w, &c);
    return NOR_OK;
}

int nor_loss_at(const nor_data* d, const double* w, double lambda, double* out) {
    nor_cache c;
    if (nor_cache_alloc(&c, d->n, d->C - 1)) return NOR_ECONFIG;
    nor_stable_exp_cache(d, w, &c);
    *out = nor_loss(d, &c, w, lambda);
    nor_cache_free(&c);
    return NOR_OK;
}

int nor_gradient_at(const nor_data* d, const double* w, double lambda, double* g) {
    nor_cache c;
    if (nor_cache_alloc(&c, d->n, d->C - 1)) return NOR_ECONFIG;
    nor_stable_exp_cache(d, w, &c);
    nor_gradient(d, &c, w, lambda, g);
    nor_cache_free(&c);
    return NOR_OK;
}

int nor_hessian_vec_at(const nor_data* d, const double* w, const double* v, double lambda, double* hv) {
    nor_cache c;
    if (nor_cache_alloc(&c, d->n, d->C - 1)) return NOR_ECONFIG;
    nor_stable_exp_cache(d, w, &c);
    nor_hessian_vec(d, &c, v, lambda, hv);
    nor_cache_free(&c);
    return NOR_OK;
}

/* ---------------------------------------------------------------------------------------------
 * Objective (src/objective.cpp:9-56)
 * ------------------------------------------------------------------------------------------- */
struct nor_softmax_obj {
    nor_data data;
    double lambda;
    int64_t dim;
    /* SoftmaxMemo (src/objective.cpp:9-22) */
    double* memo_x;
    int memo_valid;
    nor_cache cache;
    int64_t builds;
    /* augmentation (src/objective.cpp:41-56) */
    int aug;
    double rho;
    double *z, *y, *t;
};

static const nor_cache* memo_at(nor_softmax_obj* o, const double* x) {
    int same = o->memo_valid;
    for (int64_t i = 0; same && i < o->dim; ++i)
        if (!(o->memo_x[i] == x[i])) same = 0; /* Eigen `x != w`: any coefficient differs */
    if (!same) {
        nor_stable_exp_cache(&o->data, x, &o->cache);
        memcpy(o->memo_x, x, sizeof(double) * (size_t)o->dim);
        o->memo_valid = 1;
        ++o->builds;
    }
    return &o->cache;
}

/* t = z - x + y/rho, evaluated left to right as Eigen does coefficient-wise. */
static void aug_t(const nor_softmax_obj* o, const double* x) {
    for (int64_t i = 0; i < o->dim; ++i) o->t[i] = (o->z[i] - x[i]) + o->y[i] / o->rho;
}

static double so_value(const double* x, int64_t d, void* user) {
    (void)d;
    nor_softmax_obj* o = (nor_softmax_obj*)user;
    double v = nor_loss(&o->data, memo_at(o, x), x, o->lambda);
    if (o->aug) {
        aug_t(o, x);
        v = v + 0.5 * o->rho * sqnorm(o->t, o->dim);
    }
    return v;
}

static void so_grad(const double* x, double* g, int64_t d, void* user) {
    (void)d;
    nor_softmax_obj* o = (nor_softmax_obj*)user;
    nor_gradient(&o->data, memo_at(o, x), x, o->lambda, g);
    if (o->aug) {
        aug_t(o, x);
        for (int64_t i = 0; i < o->dim; ++i) g[i] = g[i] - o->rho * o->t[i];
    }
}

static void so_hvp(const double* x, const double* v, double* out, int64_t d, void* user) {
    (void)d;
    nor_softmax_obj* o = (nor_softmax_obj*)user;
    nor_hessian_vec(&o->data, memo_at(o, x), v, o->lambda, out);
    if (o->aug)
        for (int64_t i = 0; i < o->dim; ++i) out[i] = out[i] + o->rho * v[i];
}

nor_softmax_obj* nor_softmax_obj_create(const nor_data* d, double lambda) {
    nor_softmax_obj* o = (nor_softmax_obj*)calloc(1, sizeof *o);
    o->data = *d;
    o->lambda = lambda;
    o->dim = (int64_t)(d->C - 1) * d->p;
    o->memo_x = dalloc(o->dim);
    o->z = dalloc(o->dim);
    o->y = dalloc(o->dim);
    o->t = dalloc(o->dim);
    nor_cache_alloc(&o->cache, d->n, d->C - 1);
    return o;
}

void nor_softmax_obj_free(nor_softmax_obj* o) {
    if (!o) return;
    free(o->memo_x);
    free(o->z);
    free(o->y);
    free(o->t);
    nor_cache_free(&o->cache);
    free(o);
}

int nor_softmax_obj_augment(nor_softmax_obj* o, int enable, double rho, const double* z, const double* y) {
    if (!enable) {
        o->aug = 0;
        return NOR_OK;
    }
    if (rho <= 0.0) return fail(NOR_ECONFIG, "augmented objective requires rho > 0");
    o->aug = 1;
    o->rho = rho;
    memcpy(o->z, z, sizeof(double) * (size_t)o->dim);
    memcpy(o->y, y, sizeof(double) * (size_t)o->dim);
    return NOR_OK;
}

nor_objective nor_softmax_obj_iface(nor_softmax_obj* o) {
    nor_objective f = {so_value, so_grad, so_hvp, o, o->dim};
    return f;
}

int64_t nor_softmax_obj_cache_builds(const nor_softmax_obj* o) { return o->builds; }

/* ---------------------------------------------------------------------------------------------
 * Inexact Newton-CG (src/newton.cpp:8-132)
 * ------------------------------------------------------------------------------------------- */
static int validate_cfg(const double* c) { /* src/newton.cpp:8-17 */
    if (c[0] <= 0.0 || c[0] >= 1.0) return fail(NOR_ECONFIG, "cg_tol must lie in (0,1)");
    if (c[2] <= 0.0 || c[2] >= 1.0) return fail(NOR_ECONFIG, "armijo_beta must lie in (0,1)");
    if (c[3] <= 0.0 || c[3] >= 1.0) return fail(NOR_ECONFIG, "backtrack_gamma must lie in (0,1)");
    if ((int)c[1] < 1) return fail(NOR_ECONFIG, "cg_max_iters must be >= 1");
    if ((int)c[4] < 0) return fail(NOR_ECONFIG, "ls_max_iters must be >= 0");
    if ((int)c[6] < 0) return fail(NOR_ECONFIG, "newton_max_iters must be >= 0");
    if (c[5] < 0.0) return fail(NOR_ECONFIG, "grad_tol must be >= 0");
    return NOR_OK;
}

/* src/newton.cpp:19-54 */
int nor_cg_solve(nor_apply_fn apply, void* user, const double* g, int64_t d, double theta, int max_iters,
                 double* p_out, int* iters, double* achieved, int* negative_curvature) {
    const double g_norm = sqrt(sqnorm(g, d));
    if (!(g_norm > 0.0)) return fail(NOR_ECONFIG, "cg_solve requires ||g|| > 0");
    double* r = dalloc(d);
    double* dd = dalloc(d);
    double* hd = dalloc(d);
    int rc = NOR_OK;
    for (int64_t i = 0; i < d; ++i) {
        p_out[i] = 0.0;
        r[i] = -g[i];
        dd[i] = r[i];
    }
    *iters = 0;
    *negative_curvature = 0;
    double r_sq = sqnorm(r, d);
    const double stop = theta * g_norm;
    for (int it = 0; it < max_iters; ++it) {
        apply(dd, hd, d, user);
        const double curvature = dot(dd, hd, d);
        if (!isfinite(curvature)) {
            rc = fail(NOR_ESOLVER, "non-finite value in CG recurrence");
            goto done;
        }
        if (curvature <= 0.0) {
            if (it == 0)
                for (int64_t i = 0; i < d; ++i) p_out[i] = -g[i];
            *negative_curvature = 1;
            break;
        }
        const double alpha = r_sq / curvature;
        for (int64_t i = 0; i < d; ++i) p_out[i] += alpha * dd[i];
        for (int64_t i = 0; i < d; ++i) r[i] -= alpha * hd[i];
        ++*iters;
        const double r_sq_next = sqnorm(r, d);
        if (!isfinite(r_sq_next)) {
            rc = fail(NOR_ESOLVER, "non-finite value in CG recurrence");
            goto done;
        }
        if (sqrt(r_sq_next) <= stop) break;
        const double beta = r_sq_next / r_sq;
        for (int64_t i = 0; i < d; ++i) dd[i] = r[i] + beta * dd[i];
        r_sq = r_sq_next;
    }
    apply(p_out, hd, d, user); /* certificate ||H p + g|| (src/newton.cpp:52) */
    for (int64_t i = 0; i < d; ++i) hd[i] = hd[i] + g[i];
    *achieved = sqrt(sqnorm(hd, d));
done:
    free(r);
    free(dd);
    free(hd);
    return rc;
}

/* src/newton.cpp:56-71 */
int nor_line_search(const nor_objective* obj, const double* x, const double* p, const double* g, double f_x,
                    const double* cfg, double* alpha_out, int* evals, int* capped) {
    const int64_t d = obj->d;
    const double slope = dot(p, g, d);
    double* trial = dalloc(d);
    double alpha = 1.0;
    *evals = 0;
    *capped = 0;
    for (int i = 0;; ++i) {
        for (int64_t q = 0; q < d; ++q) trial[q] = x[q] + alpha * p[q];
        const double f_trial = obj->value(trial, d, obj->user);
        ++*evals;
        if (f_trial <= f_x + alpha * cfg[2] * slope) break;
        if (i >= (int)cfg[4]) {
            *capped = 1;
            break;
        }
        alpha *= cfg[3];
    }
    free(trial);
    *alpha_out = alpha;
    return NOR_OK;
}

typedef struct {
    const nor_objective* obj;
    const double* x;
} hv_ctx;

static void apply_h(const double* in, double* out, int64_t d, void* user) {
    hv_ctx* h = (hv_ctx*)user;
    h->obj->hvp(h->x, in, out, d, h->obj->user);
}

/* src/newton.cpp:73-132 */
int nor_newton_solve(const nor_objective* obj, const double* x0, const double* cfg, double* x_out, double* trace,
                     int trace_cap, int* ntrace, int* converged, double* final_grad_norm) {
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    const int64_t d = obj->d;
    memcpy(x_out, x0, sizeof(double) * (size_t)d);
    *ntrace = 0;
    *converged = 0;
    *final_grad_norm = 0.0;
    double f_x = obj->value(x_out, d, obj->user);
    if (!isfinite(f_x)) return fail(NOR_ESOLVER, "newton_solve: non-finite objective at start");
    double* g = dalloc(d);
    double* p = dalloc(d);
    for (int k = 0; k < (int)cfg[6]; ++k) {
        obj->grad(x_out, g, d, obj->user);
        const double g_norm = sqrt(sqnorm(g, d));
        *final_grad_norm = g_norm;
        if (g_norm < cfg[5]) {
            *converged = 1;
            free(g);
            free(p);
            return NOR_OK;
        }
        double rec[9] = {(double)k, g_norm, 0, 0, 0, 0, 0, 0, 0};
        hv_ctx h = {obj, x_out};
        int cg_iters = 0, negc = 0;
        double ach = 0.0;
        rc = nor_cg_solve(apply_h, &h, g, d, cfg[0], (int)cfg[1], p, &cg_iters, &ach, &negc);
        if (rc == NOR_ESOLVER) {
            fprintf(stderr, "[newton] CG failed (%s); using steepest descent\n", g_err);
            for (int64_t i = 0; i < d; ++i) p[i] = -g[i];
            rec[7] = 1;
        } else if (rc) {
            free(g);
            free(p);
            return rc;
        } else {
            rec[3] = cg_iters;
            rec[4] = ach;
        }
        if (dot(p, g, d) >= 0.0) {
            for (int64_t i = 0; i < d; ++i) p[i] = -g[i];
            rec[7] = 1;
        }
        double alpha;
        int evals, capped;
        nor_line_search(obj, x_out, p, g, f_x, cfg, &alpha, &evals, &capped);
        rec[2] = alpha;
        rec[6] = capped;
        rec[8] = evals;
        if (capped) fprintf(stderr, "[newton] line search capped at alpha=%.3e (iter %d)\n", alpha, k);
        for (int64_t i = 0; i < d; ++i) x_out[i] += alpha * p[i];
        f_x = obj->value(x_out, d, obj->user);
        if (!isfinite(f_x)) {
            free(g);
            free(p);
            return fail(NOR_ESOLVER, "newton_solve: non-finite objective");
        }
        rec[5] = f_x;
        if (*ntrace < trace_cap) memcpy(trace + 9 * *ntrace, rec, sizeof rec);
        ++*ntrace;
    }
    obj->grad(x_out, g, d, obj->user);
    *final_grad_norm = sqrt(sqnorm(g, d));
    *converged = *final_grad_norm < cfg[5];
    free(g);
    free(p);
    return NOR_OK;
}

int nor_newton_solve_softmax(const nor_data* d, double lambda, int augmented, double rho, const double* z,
                             const double* y, const double* x0, const double* cfg, double* x_out, double* trace,
                             int trace_cap, int* ntrace, int* converged, double* final_grad_norm) {
    int rc = nor_validate(d);
    if (rc) return rc;
    nor_softmax_obj* o = nor_softmax_obj_create(d, lambda);
    rc = nor_softmax_obj_augment(o, augmented, rho, z, y);
    if (!rc) {
        nor_objective f = nor_softmax_obj_iface(o);
        rc = nor_newton_solve(&f, x0, cfg, x_out, trace, trace_cap, ntrace, converged, final_grad_norm);
    }
    nor_softmax_obj_free(o);
    return rc;
}

/* ---------------------------------------------------------------------------------------------
 * ADMM coordinator (inc/admm.hpp:17-140 declarations; semantics SPEC.md:196-304)
 * ------------------------------------------------------------------------------------------- */

/* Fixed-topology pairwise tree over ascending worker ids: sum of terms[lo..hi). */
static double tree_sum(const double* terms, int lo, int hi) {
    if (hi - lo == 1) return terms[lo];
    const int mid = lo + (hi - lo + 1) / 2;
    return tree_sum(terms, lo, mid) + tree_sum(terms, mid, hi);
}

int nor_z_update(const double* x, const double* y, const double* rho, int N, int64_t d, double lambda, double* z) {
    double denom_terms[1024];
    if (N < 1 || N > 1024) return fail(NOR_ECONFIG, "z_update: bad worker count");
    for (int i = 0; i < N; ++i) denom_terms[i] = rho[i];
    const double denom = lambda + tree_sum(denom_terms, 0, N);
    if (denom == 0.0) return fail(NOR_ECONFIG, "z_update: lambda + sum(rho) == 0");
    double terms[1024];
    for (int64_t j = 0; j < d; ++j) {
        for (int i = 0; i < N; ++i) terms[i] = rho[i] * x[(int64_t)i * d + j] - y[(int64_t)i * d + j];
        z[j] = tree_sum(terms, 0, N) / denom;
    }
    return NOR_OK;
}

void nor_y_update(const double* y, const double* x, const double* z, const double* rho, int N, int64_t d,
                  double* y_out) {
    for (int i = 0; i < N; ++i)
        for (int64_t j = 0; j < d; ++j)
            y_out[(int64_t)i * d + j] = y[(int64_t)i * d + j] + rho[i] * (z[j] - x[(int64_t)i * d + j]);
}

void nor_residuals(const double* x, const double* z, const double* prev_z, const double* rho, int N, int64_t d,
                   double* primal, double* dual, double* primal_total, double* dual_total) {
    double pt = 0.0, dt = 0.0;
    for (int i = 0; i < N; ++i) {
        double sp = 0.0, sd = 0.0;
        for (int64_t j = 0; j < d; ++j) {
            const double r = z[j] - x[(int64_t)i * d + j];
            const double q = rho[i] * (z[j] - prev_z[j]);
            sp += r * r;
            sd += q * q;
        }
        primal[i] = sqrt(sp);
        dual[i] = sqrt(sd);
        pt += sp;
        dt += sd;
    }
    *primal_total = sqrt(pt);
    *dual_total = sqrt(dt);
}

void nor_tolerances(const double* x, const double* y, const double* z, int N, int64_t d, double eps_abs,
                    double eps_rel, int standard_norms, double* eps_pri, double* eps_dual) {
    double sx = 0.0, ymax = 0.0;
    for (int i = 0; i < N; ++i) {
        sx += sqnorm(x + (int64_t)i * d, d);
        const double yi = sqnorm(y + (int64_t)i * d, d);
        if (yi > ymax) ymax = yi;
    }
    const double zz = sqnorm(z, d);
    double a = sx, b = N * zz, c = ymax;
    if (standard_norms) {
        a = sqrt(sx);
        b = sqrt((double)N) * sqrt(zz);
        c = sqrt(ymax);
    }
    *eps_pri = sqrt((double)N) * eps_abs + eps_rel * (a > b ? a : b);
    *eps_dual = sqrt((double)d) * eps_abs + eps_rel * c;
}

/* Hybrid spectral step (ACADMM rule as fixed by SPEC.md:262-270). Returns 1 and the estimate when
 * the correlation safeguard passes. */
static int spectral_side(const double* a, const double* b, double b_sign, int64_t d, double eps_cor, double* est) {
    double ab = 0.0, aa = 0.0, bb = 0.0;
    for (int64_t j = 0; j < d; ++j) {
        const double bj = b_sign * b[j];
        ab += a[j] * bj;
        aa += a[j] * a[j];
        bb += bj * bj;
    }
    if (!(aa > 0.0) || !(bb > 0.0) || !(ab > 0.0)) return 0; /* zero-norm secant: failed */
    const double cor = ab / (sqrt(aa) * sqrt(bb));
    if (!(cor > eps_cor)) return 0;
    const double sd = bb / ab, mg = ab / aa;
    *est = (2.0 * mg > sd) ? mg : sd - mg / 2.0;
    return 1;
}

double nor_spectral_rho(const double* dx, const double* dyhat, const double* dz, const double* dy, int64_t d,
                        double rho, double eps_cor, double rho_min, double rho_max, int* x_ok, int* z_ok) {
    double a = 0.0, b = 0.0;
    *x_ok = spectral_side(dx, dyhat, 1.0, d, eps_cor, &a);
    *z_ok = spectral_side(dz, dy, -1.0, d, eps_cor, &b); /* (dz, -dy): lambda-side pairing */
    double r = rho;
    if (*x_ok && *z_ok)
        r = sqrt(a * b);
    else if (*x_ok)
        r = sqrt(a);
    else if (*z_ok)
        r = sqrt(b);
    if (r < rho_min) r = rho_min;
    if (r > rho_max) r = rho_max;
    return r;
}

int nor_admm_run_cb(nor_worker_solve_fn solve, nor_global_value_fn fval, void* user, int64_t d,
                    const nor_admm_cfg* cfg, double* z_out, double* rho_out, nor_metrics_row* rows, int row_cap,
                    int* iters_out, int* converged_out) {
    const int N = cfg->n_workers;
    if (N < 1) return fail(NOR_ECONFIG, "admm needs n_workers >= 1");
    if (cfg->rho0 <= 0.0) return fail(NOR_ECONFIG, "rho0 must be > 0");
    if (cfg->penalty_kind == 1 && (cfg->update_period < 1 || !(cfg->eps_cor > 0.0 && cfg->eps_cor < 1.0)))
        return fail(NOR_ECONFIG, "bad spectral policy");
    const int64_t Nd = (int64_t)N * d;
    double *x = dalloc(Nd), *y = dalloc(Nd), *yh = dalloc(Nd), *ynew = dalloc(Nd);
    double *z = dalloc(d), *pz = dalloc(d), *rho = dalloc(N);
    double *xs = dalloc(Nd), *ys = dalloc(Nd), *yhs = dalloc(Nd), *zs = dalloc(d);
    double *primal = dalloc(N), *dual = dalloc(N);
    double *t1 = dalloc(d), *t2 = dalloc(d), *t3 = dalloc(d), *t4 = dalloc(d);
    int rc = NOR_OK, k = 0, conv = 0, snap_it = 0;
    for (int i = 0; i < N; ++i) rho[i] = cfg->rho0; /* AdmmState::initial: z = 0, y = 0 */
    for (int it = 0; it < cfg->max_outer_iters; ++it) {
        int cg_sum = 0, fe_sum = 0, flags = 0, inner = 0;
        for (int i = 0; i < N; ++i) { /* scatter (z, y_i, rho_i) -> worker solve -> gather x_i */
            double stats[5] = {0};
            rc = solve(i, rho[i], z, y + (int64_t)i * d, x + (int64_t)i * d, stats, user);
            if (rc) goto out;
            inner += (int)stats[1];
            cg_sum += (int)stats[2];
            fe_sum += (int)stats[3];
            flags |= (int)stats[4];
        }
        memcpy(pz, z, sizeof(double) * (size_t)d);
        rc = nor_z_update(x, y, rho, N, d, cfg->lambda, z);
        if (rc) goto out;
        for (int i = 0; i < N; ++i) /* y_hat^k = y^{k-1} + rho^{k-1} (z^{k-1} - x^k) */
            for (int64_t j = 0; j < d; ++j)
                yh[(int64_t)i * d + j] = y[(int64_t)i * d + j] + rho[i] * (pz[j] - x[(int64_t)i * d + j]);
        nor_y_update(y, x, z, rho, N, d, ynew);
        memcpy(y, ynew, sizeof(double) * (size_t)Nd);
        ++k;
        double pt, dt, ep, ed;
        nor_residuals(x, z, pz, rho, N, d, primal, dual, &pt, &dt);
        nor_tolerances(x, y, z, N, d, cfg->eps_abs, cfg->eps_rel, cfg->standard_norms, &ep, &ed);
        conv = k >= 1;
        for (int i = 0; i < N; ++i)
            if (!(primal[i] <= ep && dual[i] <= ed)) conv = 0;
        if (cfg->penalty_kind == 1 && k - snap_it >= cfg->update_period) {
            for (int i = 0; i < N; ++i) {
                for (int64_t j = 0; j < d; ++j) {
                    const int64_t q = (int64_t)i * d + j;
                    t1[j] = x[q] - xs[q];
                    t2[j] = yh[q] - yhs[q];
                    t3[j] = z[j] - zs[j];
                    t4[j] = y[q] - ys[q];
                }
                int xo, zo;
                rho[i] = nor_spectral_rho(t1, t2, t3, t4, d, rho[i], cfg->eps_cor, cfg->rho_min, cfg->rho_max, &xo,
                                          &zo);
            }
            memcpy(xs, x, sizeof(double) * (size_t)Nd);
            memcpy(ys, y, sizeof(double) * (size_t)Nd);
            memcpy(yhs, yh, sizeof(double) * (size_t)Nd);
            memcpy(zs, z, sizeof(double) * (size_t)d);
            snap_it = k;
        }
        if (rows && it < row_cap) {
            nor_metrics_row* r = rows + it;
            r->iteration = k;
            r->train_objective = NAN;
            if (fval) {
                rc = fval(z, &r->train_objective, user);
                if (rc) goto out;
            }
            r->primal_norm = pt;
            r->dual_norm = dt;
            r->eps_pri = ep;
            r->eps_dual = ed;
            r->inner_iterations = inner;
            r->cg_iters = cg_sum;
            r->fn_evals = fe_sum;
            r->flags = flags;
            double rs = 0.0;
            for (int i = 0; i < N; ++i) rs += rho[i];
            r->rho_mean = rs / N;
        }
        if (conv) break;
    }
out:
    memcpy(z_out, z, sizeof(double) * (size_t)d);
    if (rho_out) memcpy(rho_out, rho, sizeof(double) * (size_t)N);
    *iters_out = k;
    *converged_out = conv;
    free(x), free(y), free(yh), free(ynew), free(z), free(pz), free(rho), free(xs), free(ys), free(yhs), free(zs);
    free(primal), free(dual), free(t1), free(t2), free(t3), free(t4);
    return rc;
}

typedef struct {
    const nor_data* shards;
    nor_softmax_obj** base;
    double** x_local;
    const nor_admm_cfg* cfg;
    int64_t d;
} port_run;

/* run_worker ADMM branch (src/worker.cpp:168-196) on the port's own objective. */
static int port_solve(int i, double rho, const double* z, const double* y, double* x_out, double* stats, void* user) {
    port_run* r = (port_run*)user;
    nor_softmax_obj* o = r->base[i];
    int rc = nor_softmax_obj_augment(o, 1, rho, z, y);
    if (rc) return rc;
    double cfg[7];
    memcpy(cfg, r->cfg->newton, sizeof cfg);
    cfg[6] = r->cfg->inner_iters; /* src/worker.cpp:173 */
    double trace[9 * 64];
    int nt, conv;
    double gn;
    nor_objective f = nor_softmax_obj_iface(o);
    rc = nor_newton_solve(&f, r->x_local[i], cfg, x_out, trace, 64, &nt, &conv, &gn);
    if (rc) return rc;
    memcpy(r->x_local[i], x_out, sizeof(double) * (size_t)r->d);
    stats[0] = gn;
    stats[1] = nt;
    int cg = 0, fe = 0, fl = 0;
    for (int t = 0; t < nt && t < 64; ++t) {
        cg += (int)trace[9 * t + 3];
        fe += (int)trace[9 * t + 8];
        if (trace[9 * t + 6] != 0.0) fl |= 1;
        if (trace[9 * t + 7] != 0.0) fl |= 2;
    }
    stats[2] = cg;
    stats[3] = fe;
    stats[4] = fl;
    return NOR_OK;
}

/* F(z) = sum_i loss(D_i, z) + (lambda/2)||z||^2 (global objective of Eq. (5)). */
static int port_fval(const double* z, double* value, void* user) {
    port_run* r = (port_run*)user;
    double total = 0.0;
    for (int i = 0; i < r->cfg->n_workers; ++i) {
        double li;
        int rc = nor_loss_at(&r->shards[i], z, 0.0, &li);
        if (rc) return rc;
        total += li;
    }
    *value = total + 0.5 * r->cfg->lambda * sqnorm(z, r->d);
    return NOR_OK;
}

int nor_admm_run(const nor_data* shards, const nor_admm_cfg* cfg, int eval_objective, double* z_out, double* rho_out,
                 nor_metrics_row* rows, int row_cap, int* iters, int* converged) {
    const int N = cfg->n_workers;
    if (N < 1) return fail(NOR_ECONFIG, "admm needs n_workers >= 1");
    const int64_t d = (int64_t)(shards[0].C - 1) * shards[0].p;
    for (int i = 0; i < N; ++i) {
        int rc = nor_validate(&shards[i]);
        if (rc) return rc;
        if ((int64_t)(shards[i].C - 1) * shards[i].p != d) return fail(NOR_ECONFIG, "shard dimension mismatch");
    }
    port_run r = {shards, NULL, NULL, cfg, d};
    r.base = (nor_softmax_obj**)calloc((size_t)N, sizeof(void*));
    r.x_local = (double**)calloc((size_t)N, sizeof(double*));
    for (int i = 0; i < N; ++i) {
        r.base[i] = nor_softmax_obj_create(&shards[i], 0.0); /* local loss only (src/worker.cpp:129-130) */
        r.x_local[i] = dalloc(d);                           /* x_local = 0 (src/worker.cpp:135) */
    }
    int rc = nor_admm_run_cb(port_solve, eval_objective ? port_fval : NULL, &r, d, cfg, z_out, rho_out, rows, row_cap,
                             iters, converged);
    for (int i = 0; i < N; ++i) {
        nor_softmax_obj_free(r.base[i]);
        free(r.x_local[i]);
    }
    free(r.base);
    free(r.x_local);
    return rc;
}

/* ---------------------------------------------------------------------------------------------
 * Data fixtures (src/data_io.cpp:16-43, 300-370; src/worker.cpp:64-69)
 * ------------------------------------------------------------------------------------------- */
#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void nor_rng_seed(nor_rng* r, uint64_t seed) { /* std::mt19937_64(seed) */
    r->mt[0] = seed;
    for (int i = 1; i < MT_NN; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_NN;
    r->have_spare = 0;
    r->spare = 0.0;
}

uint64_t nor_rng_next(nor_rng* r) {
    static const uint64_t mag01[2] = {0ULL, MT_MATRIX_A};
    uint64_t x;
    if (r->mti >= MT_NN) {
        int i;
        for (i = 0; i < MT_NN - MT_MM; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < MT_NN - 1; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        r->mti = 0;
    }
    x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

double nor_rng_uniform(nor_rng* r) { return (double)(nor_rng_next(r) >> 11) * 0x1.0p-53; }

double nor_rng_normal(nor_rng* r) { /* src/data_io.cpp:21-33 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = nor_rng_uniform(r);
    while (u1 <= 0.0) u1 = nor_rng_uniform(r);
    const double u2 = nor_rng_uniform(r);
    const double mag = sqrt(-2.0 * log(u1));
    const double pi = 3.141592653589793;
    r->spare = mag * sin(2.0 * pi * u2);
    r->have_spare = 1;
    return mag * cos(2.0 * pi * u2);
}

uint64_t nor_rng_uniform_int(nor_rng* r, uint64_t bound) { /* src/data_io.cpp:35-43 */
    const uint64_t limit = UINT64_MAX - (UINT64_MAX % bound);
    uint64_t v = nor_rng_next(r);
    while (v >= limit) v = nor_rng_next(r);
    return v % bound;
}

uint64_t nor_mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

int nor_rng_stream(uint64_t seed, int kind, uint64_t bound, int64_t count, double* out) {
    if (kind == 2 && bound == 0) return fail(NOR_ECONFIG, "uniform_int: zero bound");
    nor_rng r;
    nor_rng_seed(&r, seed);
    for (int64_t i = 0; i < count; ++i)
        out[i] = kind == 0 ? nor_rng_uniform(&r) : kind == 1 ? nor_rng_normal(&r) : (double)nor_rng_uniform_int(&r, bound);
    return NOR_OK;
}

/* src/data_io.cpp:330-370 */
int nor_generate_synthetic(int64_t n, int64_t p, int32_t C, double separation, double noise, uint64_t seed,
                           double* X_train, int32_t* y_train, double* X_test, int32_t* y_test) {
    if (n < 2 || p < 1 || C < 2) return fail(NOR_ECONFIG, "synthetic spec needs n >= 2, p >= 1, C >= 2");
    if (C > n) return fail(NOR_ECONFIG, "synthetic spec: more classes than samples");
    const int64_t n_train = (n * 9) / 10;
    if (n_train < C || n - n_train < 1) return fail(NOR_ECONFIG, "synthetic spec too small for a 90/10 split");
    nor_rng r;
    nor_rng_seed(&r, seed);
    double* centers = dalloc(p * C); /* p x C column-major */
    double* dir = dalloc(p);
    for (int c = 0; c < C; ++c) {
        for (int64_t j = 0; j < p; ++j) dir[j] = nor_rng_normal(&r);
        const double norm = sqrt(sqnorm(dir, p));
        for (int64_t j = 0; j < p; ++j) centers[c * p + j] = norm > 0.0 ? (separation / norm) * dir[j] : dir[j];
    }
    for (int64_t i = 0; i < n; ++i) {
        const int c = (int)(i % C);
        double* row = i < n_train ? X_train + i * p : X_test + (i - n_train) * p;
        if (i < n_train)
            y_train[i] = c + 1;
        else
            y_test[i - n_train] = c + 1;
        for (int64_t j = 0; j < p; ++j) row[j] = centers[c * p + j] + noise * nor_rng_normal(&r);
    }
    free(centers);
    free(dir);
    for (int64_t k = 0; k < n_train * p; ++k)
        if (!isfinite(X_train[k])) return fail(NOR_EDATA, "non-finite feature value in dense dataset");
    return NOR_OK;
}

/* src/data_io.cpp:300-328 */
int nor_partition_owner(int64_t n, int N, int strided, int32_t* owner) {
    if (N < 1) return fail(NOR_ECONFIG, "partition needs n_workers >= 1");
    if (n < N) return fail(NOR_ECONFIG, "cannot partition rows across workers");
    if (!strided) {
        const int64_t chunk = (n + N - 1) / N;
        for (int i = 0; i < N; ++i) {
            const int64_t b = (int64_t)i * chunk, e = b + chunk < n ? b + chunk : n;
            if (b >= e) return fail(NOR_ECONFIG, "contiguous partition leaves a worker empty; use strided or fewer workers");
            for (int64_t q = b; q < e; ++q) owner[q] = i;
        }
    } else {
        for (int64_t q = 0; q < n; ++q) owner[q] = (int32_t)(q % N);
    }
    return NOR_OK;
}

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

int nor_generate_sparse(int64_t n, int64_t p, int32_t C, int32_t nnz_per_row, uint64_t seed, int64_t* indptr,
                        int32_t* indices, double* vals, int32_t* labels) {
    if (n < 1 || p < 1 || C < 2 || nnz_per_row < 1 || nnz_per_row > p)
        return fail(NOR_ECONFIG, "sparse spec needs n, p >= 1, C >= 2, 1 <= nnz_per_row <= p");
    nor_rng r;
    nor_rng_seed(&r, seed);
    const int64_t band = p / C > 0 ? p / C : 1;
    int64_t* stamp = (int64_t*)calloc((size_t)p, sizeof(int64_t)); /* stamp[j] == i+1: column j taken in row i */
    indptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int c = (int)(i % C);
        labels[i] = c + 1;
        int32_t* cols = indices + i * nnz_per_row;
        int got = 0;
        while (got < nnz_per_row) {
            int64_t j;
            if (nor_rng_uniform(&r) < 0.5) {
                const int64_t lo = (int64_t)c * band;
                const int64_t width = lo + band <= p ? band : p - lo;
                j = lo + (int64_t)nor_rng_uniform_int(&r, (uint64_t)(width > 0 ? width : 1));
            } else {
                j = (int64_t)nor_rng_uniform_int(&r, (uint64_t)p);
            }
            if (stamp[j] != i + 1) {
                stamp[j] = i + 1;
                cols[got++] = (int32_t)j;
            }
        }
        qsort(cols, (size_t)nnz_per_row, sizeof(int32_t), cmp_i32);
        double* v = vals + i * nnz_per_row;
        double ss = 0.0;
        for (int q = 0; q < nnz_per_row; ++q) {
            v[q] = 1.0 + 0.1 * nor_rng_normal(&r);
            ss += v[q] * v[q];
        }
        const double inv = 1.0 / sqrt(ss);
        for (int q = 0; q < nnz_per_row; ++q) v[q] = v[q] * inv;
        indptr[i + 1] = indptr[i] + nnz_per_row;
    }
    free(stamp);
    return NOR_OK;
}
