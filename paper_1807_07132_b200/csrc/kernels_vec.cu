// Vector / scalar kernels of the device-resident inexact Newton-CG solver.
//
// Restates, kernel by kernel (file:line under /root/reference/proj):
//   make_augmented_objective value/grad    src/objective.cpp:41-51
//   cg_solve                               src/newton.cpp:19-54
//   line_search (batched Armijo)           src/newton.cpp:56-71
//   newton_solve step / fallbacks / trace  src/newton.cpp:73-132
// Every reduction is a two-stage deterministic sum (block partials, then reduce_partials), so the
// scalars every block derives are bit-identical and branch decisions are consistent grid-wide.
// Flags that a kernel both reads and decides live in per-iteration slots (cg_act / cg_mid), so no
// block ever observes a flag written by another block of the same launch.
#include "solver_kernels.h"

namespace nadmm {

#define GRID_STRIDE(j, d) \
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (d); j += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ double* slot_ptr(double* blk, int slot) { return blk + (int64_t)slot * kBlockPartials; }

// Reduce a slot with warp 0 and broadcast to the whole block.
__device__ __forceinline__ double block_reduce_slot(double* blk, int slot, int n, double* sh) {
    if (threadIdx.x < 32) {
        const double v = reduce_partials(slot_ptr(blk, slot), n);
        if (threadIdx.x == 0) *sh = v;
    }
    __syncthreads();
    return *sh;
}

// t = z - x + y/rho and g = gbase - rho t (src/objective.cpp:47-51); partials of <g,g>, <t,t>.
__global__ void k_grad_aug(int64_t d, const double* __restrict__ x, const double* __restrict__ z,
                           const double* __restrict__ y, const double* __restrict__ gbase, const DevParams* prm,
                           double* __restrict__ g, double* __restrict__ t, double* blk, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    const bool aug = prm->augmented;
    const double rho = prm->rho;
    double gg = 0.0, tt = 0.0;
    GRID_STRIDE(j, d) {
        double gj = gbase[j];
        if (aug) {
            const double tj = (z[j] - x[j]) + y[j] / rho;
            t[j] = tj;
            tt += tj * tj;
            gj = gj - rho * tj;
        }
        g[j] = gj;
        gg += gj * gj;
    }
    double s = block_sum(gg, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotGg)[blockIdx.x] = s;
    s = block_sum(tt, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotTt)[blockIdx.x] = s;
}

// f_x and |g| at the current x. prologue: start-of-solve checks (src/newton.cpp:75-78); else the
// end of a Newton iteration: record the trace row (src/newton.cpp:119-127).
__global__ void k_value_finish(DevState* st, const DevParams* prm, const double* base_loss, double* blk, int nvec,
                               DevTrace* trace, int trace_cap, int prologue, const int32_t* guard) {
    if (guard && !*guard) return;
    if (threadIdx.x >= 32) return;
    const double g_sq = reduce_partials(slot_ptr(blk, kSlotGg), nvec);
    const double t_sq = reduce_partials(slot_ptr(blk, kSlotTt), nvec);
    if (threadIdx.x != 0) return;
    double f = *base_loss;
    if (prm->augmented) f = f + 0.5 * prm->rho * t_sq;
    st->f_base = *base_loss;
    st->f_x = f;
    st->g_sq = g_sq;
    st->g_norm = sqrt(g_sq);
    if (prologue) {
        st->iter = 0;
        st->converged = 0;
        st->error = 0;
        st->active = 1;
        if (!isfinite(f)) {  // "newton_solve: non-finite objective at start"
            st->error = NADMM_ESOLVER;
            st->active = 0;
        }
        return;
    }
    const int k = st->iter;
    if (k < trace_cap) {
        DevTrace r;
        r.iter = k;
        r.grad_norm = st->rec_gnorm;
        r.step = st->ls_alpha;
        r.cg_iters = st->cg_failed ? 0 : st->cg_iters;
        r.cg_residual = st->cg_failed ? 0.0 : st->cg_residual;
        r.objective = f;
        r.ls_capped = st->ls_capped;
        r.cg_fallback = st->fallback;
        r.fn_evals = st->ls_evals;
        r.pad = 0;
        trace[k] = r;
    }
    st->iter = k + 1;
    if (!isfinite(f)) {  // "non-finite objective at iteration k"
        st->error = NADMM_ESOLVER;
        st->active = 0;
    }
}

// Loop head of newton_solve (src/newton.cpp:80-87) and cg_solve's entry (19-30).
__global__ void k_newton_begin(DevState* st, const DevParams* prm) {
    if (threadIdx.x != 0) return;
    int run = st->active;
    if (run) {
        st->rec_gnorm = st->g_norm;
        if (st->g_norm < prm->grad_tol) {
            st->converged = 1;
            st->active = 0;
            run = 0;
        } else if (!(st->g_norm > 0.0)) {  // cg_solve requires ||g|| > 0 (ConfigError)
            st->error = NADMM_ECONFIG;
            st->active = 0;
            run = 0;
        }
    }
    st->it_act = run;
    st->cg_act[0] = run;
    st->cg_iters = 0;
    st->cg_neg = 0;
    st->cg_failed = 0;
    st->fallback = 0;
    st->cg_residual = 0.0;
    st->cg_stop = prm->cg_tol * st->g_norm;
    st->r_sq[0] = st->g_sq;  // r = -g: |r|^2 == |g|^2 bit-for-bit under the same reduction order
    st->ls_alpha = 0.0;
    st->ls_evals = 0;
    st->ls_capped = 0;
}

// p = 0, r = -g, d = r.
__global__ void k_cg_init(int64_t d, const double* __restrict__ g, double* __restrict__ p, double* __restrict__ r,
                          double* __restrict__ dv, const int32_t* guard) {
    if (guard && !*guard) return;
    GRID_STRIDE(j, d) {
        p[j] = 0.0;
        r[j] = -g[j];
        dv[j] = -g[j];
    }
}

// One CG step after Hd = H d (src/newton.cpp:31-45): curvature test, p += a d, r -= a Hd, <r,r>.
__global__ void k_cg_step(int it, int64_t d, DevState* st, const double* __restrict__ g, double* __restrict__ p,
                          double* __restrict__ r, const double* __restrict__ dv, const double* __restrict__ hd,
                          double* blk, int ncurv) {
    __shared__ double red[32];
    __shared__ double curv_s;
    if (!st->cg_act[it]) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->cg_mid[it] = 0;
        return;
    }
    const double curv = block_reduce_slot(blk, kSlotCurv, ncurv, &curv_s);
    if (!isfinite(curv)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->cg_failed = 1;
            st->cg_mid[it] = 0;
        }
        return;
    }
    if (curv <= 0.0) {
        if (it == 0) GRID_STRIDE(j, d) p[j] = -g[j];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->cg_neg = 1;
            st->cg_mid[it] = 0;
        }
        return;
    }
    const double alpha = st->r_sq[it] / curv;
    double rr = 0.0;
    GRID_STRIDE(j, d) {
        p[j] += alpha * dv[j];
        const double rj = r[j] - alpha * hd[j];
        r[j] = rj;
        rr += rj * rj;
    }
    const double s = block_sum(rr, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotRr)[blockIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->cg_iters = it + 1;
        st->cg_mid[it] = 1;
    }
}

// Stop test and direction update (src/newton.cpp:46-50).
__global__ void k_cg_dir(int it, int64_t d, DevState* st, const double* __restrict__ r, double* __restrict__ dv,
                         double* blk, int nrr) {
    __shared__ double rr_s;
    if (!st->cg_mid[it]) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->cg_act[it + 1] = 0;
        return;
    }
    const double r_sq_next = block_reduce_slot(blk, kSlotRr, nrr, &rr_s);
    if (!isfinite(r_sq_next)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->cg_failed = 1;
            st->cg_act[it + 1] = 0;
        }
        return;
    }
    if (sqrt(r_sq_next) <= st->cg_stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->cg_act[it + 1] = 0;
        return;
    }
    const double beta = r_sq_next / st->r_sq[it];
    GRID_STRIDE(j, d) dv[j] = r[j] + beta * dv[j];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->r_sq[it + 1] = r_sq_next;
        st->cg_act[it + 1] = 1;
    }
}

__global__ void k_after_cg(DevState* st) {
    if (threadIdx.x == 0) st->cert_act = st->it_act && !st->cg_failed;
}

// Partials of |Hp + g|^2 for the CG certificate (src/newton.cpp:52).
__global__ void k_cert(int64_t d, const double* __restrict__ hp, const double* __restrict__ g, double* blk,
                       const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    double s = 0.0;
    GRID_STRIDE(j, d) {
        const double v = hp[j] + g[j];
        s += v * v;
    }
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotCert)[blockIdx.x] = t;
}

// CG failure fallback p = -g (src/newton.cpp:100-104), then partials of <p, g>.
__global__ void k_fallback(int64_t d, const DevState* st, const double* __restrict__ g, double* __restrict__ p,
                           double* blk, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    const bool failed = st->cg_failed;
    double s = 0.0;
    GRID_STRIDE(j, d) {
        if (failed) p[j] = -g[j];
        s += p[j] * g[j];
    }
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotSlope)[blockIdx.x] = t;
}

// Descent test (src/newton.cpp:105-109): p'g >= 0 -> p = -g; the line-search slope p'g.
__global__ void k_slope(int64_t d, DevState* st, const double* __restrict__ g, double* __restrict__ p, double* blk,
                        int nslope, int ncert, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double sl_s;
    double slope = block_reduce_slot(blk, kSlotSlope, nslope, &sl_s);
    const bool flip = slope >= 0.0;
    if (flip) GRID_STRIDE(j, d) p[j] = -g[j];
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const double cert = st->cert_act ? reduce_partials(slot_ptr(blk, kSlotCert), ncert) : 0.0;
        if (threadIdx.x == 0) {
            if (flip) slope = -st->g_sq;  // (-g).g == -|g|^2 under the same reduction order
            st->slope = slope;
            if (st->cert_act) st->cg_residual = sqrt(cert);
            if (st->cg_failed || flip) st->fallback = 1;
        }
    }
}

// Batched Armijo candidates, row part: for every trial a_j = gamma^j the loss of logits L0 + a_j Lp
// (stable_exp_cache + loss at x + a_j p, src/softmax.cpp:51-78), accumulated per candidate.
constexpr int kLsChunk = 16;

__global__ void __launch_bounds__(256) k_ls_rows(int64_t n, int K, const double* __restrict__ L0,
                                                 const double* __restrict__ Lp, const int32_t* __restrict__ labels,
                                                 const DevParams* prm, double* blk, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    const int nc = prm->ls_max_iters + 1;
    const double gamma = prm->backtrack_gamma;
    double a0 = 1.0;
    for (int j0 = 0; j0 < nc; j0 += kLsChunk) {
        double alpha[kLsChunk], acc[kLsChunk];
        double a = a0;
#pragma unroll
        for (int q = 0; q < kLsChunk; ++q) {
            alpha[q] = a;
            acc[q] = 0.0;
            a *= gamma;  // alpha *= backtrack_gamma (src/newton.cpp:69)
        }
        a0 = a;
        GRID_STRIDE(i, n) {
            const double* l0 = L0 + i * K;
            const double* lp = Lp + i * K;
            const int b = labels[i];
#pragma unroll
            for (int q = 0; q < kLsChunk; ++q) {
                if (j0 + q >= nc) break;
                double m = l0[0] + alpha[q] * lp[0];
                for (int c = 1; c < K; ++c) {
                    const double l = l0[c] + alpha[q] * lp[c];
                    if (l > m) m = l;
                }
                m = m > 0.0 ? m : 0.0;
                double s = 0.0;
                for (int c = 0; c < K; ++c) s += exp((l0[c] + alpha[q] * lp[c]) - m);
                const double al = exp(-m) + s;
                acc[q] += (m + log(al)) - (b <= K ? l0[b - 1] + alpha[q] * lp[b - 1] : 0.0);
            }
        }
        for (int q = 0; q < kLsChunk && j0 + q < nc; ++q) {
            const double t = block_sum(acc[q], red);
            if (threadIdx.x == 0) slot_ptr(blk, kSlotLs + j0 + q)[blockIdx.x] = t;
        }
    }
}

// Vector part of each candidate: |z - x_j + y/rho|^2 (augmented) and |x_j|^2 (ridge), x_j = x + a_j p.
__global__ void __launch_bounds__(256) k_ls_vec(int64_t d, const double* __restrict__ x, const double* __restrict__ p,
                                                const double* __restrict__ z, const double* __restrict__ y,
                                                const DevParams* prm, double* blk, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    const int nc = prm->ls_max_iters + 1;
    const double gamma = prm->backtrack_gamma, rho = prm->rho;
    const bool aug = prm->augmented, ridge = prm->lambda > 0.0;
    double a0 = 1.0;
    for (int j0 = 0; j0 < nc; j0 += kLsChunk) {
        double alpha[kLsChunk], at[kLsChunk], ax[kLsChunk];
        double a = a0;
#pragma unroll
        for (int q = 0; q < kLsChunk; ++q) {
            alpha[q] = a;
            at[q] = 0.0;
            ax[q] = 0.0;
            a *= gamma;
        }
        a0 = a;
        GRID_STRIDE(j, d) {
            const double xj = x[j], pj = p[j];
            const double zj = aug ? z[j] : 0.0, yr = aug ? y[j] / rho : 0.0;
#pragma unroll
            for (int q = 0; q < kLsChunk; ++q) {
                const double xt = xj + alpha[q] * pj;  // x + alpha * p (src/newton.cpp:62)
                if (aug) {
                    const double tq = (zj - xt) + yr;
                    at[q] += tq * tq;
                }
                if (ridge) ax[q] += xt * xt;
            }
        }
        for (int q = 0; q < kLsChunk && j0 + q < nc; ++q) {
            double t = block_sum(at[q], red);
            if (threadIdx.x == 0) slot_ptr(blk, kSlotLsVec + 2 * (j0 + q))[blockIdx.x] = t;
            t = block_sum(ax[q], red);
            if (threadIdx.x == 0) slot_ptr(blk, kSlotLsVec + 2 * (j0 + q) + 1)[blockIdx.x] = t;
        }
    }
}

// Accept the first trial satisfying Armijo, else the last one flagged capped (src/newton.cpp:61-70).
__global__ void k_ls_select(DevState* st, const DevParams* prm, double* blk, int nrows, int nvec,
                            const int32_t* guard) {
    if (guard && !*guard) return;
    if (threadIdx.x >= 32) return;
    const int nc = prm->ls_max_iters + 1;
    double alpha = 1.0;
    int evals = 0, capped = 0;
    for (int j = 0; j < nc; ++j) {
        double f = reduce_partials(slot_ptr(blk, kSlotLs + j), nrows);
        if (prm->lambda > 0.0) f += 0.5 * prm->lambda * reduce_partials(slot_ptr(blk, kSlotLsVec + 2 * j + 1), nvec);
        if (prm->augmented) f = f + 0.5 * prm->rho * reduce_partials(slot_ptr(blk, kSlotLsVec + 2 * j), nvec);
        ++evals;
        if (f <= st->f_x + alpha * prm->armijo_beta * st->slope) break;
        if (j >= prm->ls_max_iters) {
            capped = 1;
            break;
        }
        alpha *= prm->backtrack_gamma;
    }
    if (threadIdx.x == 0) {
        st->ls_alpha = alpha;
        st->ls_evals = evals;
        st->ls_capped = capped;
    }
}

// x += alpha p (src/newton.cpp:120).
__global__ void k_step(int64_t d, const DevState* st, double* __restrict__ x, const double* __restrict__ p,
                       const int32_t* guard) {
    if (guard && !*guard) return;
    const double a = st->ls_alpha;
    GRID_STRIDE(j, d) x[j] += a * p[j];
}

__global__ void k_set_int(int32_t* dst, int v) {
    if (threadIdx.x == 0) *dst = v;
}

// ---------------------------------------------------------------------------------------------
// Host launch wrappers
// ---------------------------------------------------------------------------------------------
#define LAUNCH_COUNT(s) (s).ctx->stats.kernel_launches++

void launch_grad_aug(Shard& s, const int32_t* guard, int* nvec) {
    const int grid = vec_grid(*s.ctx, s.d);
    k_grad_aug<<<grid, 256, 0, s.ctx->stream>>>(s.d, s.x, s.z, s.y, s.gbase, s.prm, s.g, s.t, s.blk, guard);
    NADMM_LAUNCH_CHECK();
    LAUNCH_COUNT(s);
    *nvec = grid;
}

void launch_value_finish(Shard& s, int nvec, int prologue, const int32_t* guard) {
    k_value_finish<<<1, 32, 0, s.ctx->stream>>>(s.st, s.prm, s.scal, s.blk, nvec, s.trace, kTraceCap, prologue, guard);
    NADMM_LAUNCH_CHECK();
    LAUNCH_COUNT(s);
}

void launch_newton_iteration(Shard& s, int cg_max, int ls_max) {
    (void)ls_max;
    cudaStream_t st = s.ctx->stream;
    const int grid = vec_grid(*s.ctx, s.d);
    const int32_t* it_act = &s.st->it_act;
    k_newton_begin<<<1, 32, 0, st>>>(s.st, s.prm);
    k_cg_init<<<grid, 256, 0, st>>>(s.d, s.g, s.pd, s.r, s.dv, it_act);
    s.ctx->stats.kernel_launches += 2;
    for (int it = 0; it < cg_max; ++it) {
        s.hv_timer_site = it;
        const int ncurv = op_hv(s, s.dv, s.hd, s.dv, kSlotCurv, &s.st->cg_act[it]);
        s.hv_timer_site = -1;
        k_cg_step<<<grid, 256, 0, st>>>(it, s.d, s.st, s.g, s.pd, s.r, s.dv, s.hd, s.blk, ncurv);
        k_cg_dir<<<grid, 256, 0, st>>>(it, s.d, s.st, s.r, s.dv, s.blk, grid);
        s.ctx->stats.kernel_launches += 2;
    }
    k_after_cg<<<1, 32, 0, st>>>(s.st);
    LAUNCH_COUNT(s);
    s.hv_timer_site = cg_max;
    op_hv(s, s.pd, s.hd, nullptr, 0, &s.st->cert_act);  // certificate Hv (src/newton.cpp:52)
    s.hv_timer_site = -1;
    k_cert<<<grid, 256, 0, st>>>(s.d, s.hd, s.g, s.blk, &s.st->cert_act);
    k_fallback<<<grid, 256, 0, st>>>(s.d, s.st, s.g, s.pd, s.blk, it_act);
    k_slope<<<grid, 256, 0, st>>>(s.d, s.st, s.g, s.pd, s.blk, grid, grid, it_act);
    s.ctx->stats.kernel_launches += 3;
    op_lp(s, s.pd, it_act);  // Lp = X p: one data pass serves every Armijo trial
    const int rgrid = std::max(1, (int)std::min<int64_t>((s.n + 255) / 256, std::min<int64_t>(kBlockPartials, 4LL * s.ctx->num_sms)));
    k_ls_rows<<<rgrid, 256, 0, st>>>(s.n, s.K, s.L0, s.Lp, s.labels, s.prm, s.blk, it_act);
    k_ls_vec<<<grid, 256, 0, st>>>(s.d, s.x, s.pd, s.z, s.y, s.prm, s.blk, it_act);
    k_ls_select<<<1, 32, 0, st>>>(s.st, s.prm, s.blk, rgrid, grid, it_act);
    k_step<<<grid, 256, 0, st>>>(s.d, s.st, s.x, s.pd, it_act);
    s.ctx->stats.kernel_launches += 4;
    NADMM_LAUNCH_CHECK();
    op_cache_grad(s, s.x, it_act);
    int nvec = 0;
    launch_grad_aug(s, it_act, &nvec);
    launch_value_finish(s, nvec, 0, it_act);
}

void launch_set_int(Shard& s, int32_t* dst, int v) {
    k_set_int<<<1, 32, 0, s.ctx->stream>>>(dst, v);
    NADMM_LAUNCH_CHECK();
    LAUNCH_COUNT(s);
}

}  // namespace nadmm
