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
#include <cooperative_groups.h>

#include "solver_kernels.h"
#include "solver_tails.cuh"

namespace nadmm {

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

// Loop head of newton_solve (src/newton.cpp:80-87) and cg_solve's entry (19-30): p = 0, r = -g,
// d = r. Every block derives `run` from the state written by the previous launch; block 0 alone
// updates the state (it only ever clears `active` when `run` is false for every block as well).
__global__ void __launch_bounds__(256) k_begin_init(int64_t d, DevState* st, const DevParams* prm,
                                                    const double* __restrict__ g, double* __restrict__ p,
                                                    double* __restrict__ r, double* __restrict__ dv) {
    const double gn = st->g_norm;
    const bool run = st->active && !(gn < prm->grad_tol) && gn > 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (st->active) {
            st->rec_gnorm = gn;
            if (gn < prm->grad_tol) {
                st->converged = 1;
                st->active = 0;
            } else if (!(gn > 0.0)) {  // cg_solve requires ||g|| > 0 (ConfigError)
                st->error = NADMM_ECONFIG;
                st->active = 0;
            }
        }
        st->it_act = run;
        st->cg_act[0] = run;
        st->cg_iters = 0;
        st->cg_neg = 0;
        st->cg_failed = 0;
        st->fallback = 0;
        st->cg_residual = 0.0;
        st->cg_stop = prm->cg_tol * gn;
        st->r_sq[0] = st->g_sq;  // r = -g: |r|^2 == |g|^2 bit-for-bit under the same reduction order
        st->ls_alpha = 0.0;
        st->ls_evals = 0;
        st->ls_capped = 0;
        st->cert_act = run;
        st->lp_need = run;
    }
    if (!run) return;
    GRID_STRIDE(j, d) {
        p[j] = 0.0;
        r[j] = -g[j];
        dv[j] = -g[j];
    }
}

// One fused CG tail per iteration (persistent grid, two software grid barriers), replacing the
// finalize / step / direction launches:
//   (0) chunks > 0: Hd = sum of the fused pass's split-K partials + lambda d (+ rho d when
//       augmented) (src/softmax.cpp:108-110, src/objective.cpp:52-54), <d, Hd> partials
//   (1) step:       curvature test, p += a d, r -= a Hd, <r, r> partials   (src/newton.cpp:31-45)
//   (2) direction:  stop test, d = r + b d                                  (src/newton.cpp:46-50)
// Every block reduces the same partials in the same order, so all blocks take the same branches.
// The kernel is a chain of dependent L2 round trips (partials -> barrier -> reduction -> ...), so each
// thread keeps its (at most EPT) elements of d, p, r, Hd in registers across the phases and loads
// everything it will need before the first barrier. Block 0 also refreshes cert_act (= the Newton
// iteration runs and CG did not fail) on every exit: the last tail's value guards the certificate Hv.
constexpr int kTailEpt = 2;

__global__ void __launch_bounds__(256, 4) k_cg_tail(int it, int64_t d, DevState* st, const DevParams* prm,
                                                    const double* __restrict__ part, int chunks,
                                                    const double* __restrict__ g, double* __restrict__ p,
                                                    double* __restrict__ r, double* __restrict__ dv,
                                                    double* __restrict__ hd, double* blk, int ncurv,
                                                    unsigned long long* hv_ctr, unsigned long long* bar) {
    __shared__ double red[32];
    __shared__ double sc;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    auto done = [&](int act_next) {
        if (lead) {
            st->cg_act[it + 1] = act_next;
            st->cert_act = st->it_act && !st->cg_failed;
        }
    };
    if (!st->cg_act[it]) {  // grid-uniform: written by an earlier launch
        if (lead) st->cg_mid[it] = 0;
        done(0);
        return;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool cached = d <= stride * kTailEpt;  // grid-uniform
    double vd[kTailEpt], vp[kTailEpt], vr[kTailEpt], vh[kTailEpt];
    const double r_sq = st->r_sq[it], cg_stop = st->cg_stop;
    if (cached) {
#pragma unroll
        for (int e = 0; e < kTailEpt; ++e) {
            const int64_t j = j0 + e * stride;
            const bool in = j < d;
            vd[e] = in ? dv[j] : 0.0;
            vp[e] = in ? p[j] : 0.0;
            vr[e] = in ? r[j] : 0.0;
            vh[e] = (in && chunks == 0) ? hd[j] : 0.0;
        }
    }
    if (chunks > 0) {
        if (hv_ctr && lead) atomicAdd(hv_ctr, 1ULL);
        const double lam = prm->lambda;
        const bool aug = prm->augmented;
        const double rho = prm->rho;
        double dacc = 0.0;
        if (cached) {
#pragma unroll
            for (int e = 0; e < kTailEpt; ++e) {
                const int64_t j = j0 + e * stride;
                if (j < d) {
                    double s = sum_chunks(part, chunks, d, j);
                    if (lam > 0.0) s = s + lam * vd[e];
                    if (aug) s = s + rho * vd[e];
                    hd[j] = s;
                    vh[e] = s;
                    dacc += s * vd[e];
                }
            }
        } else {
            GRID_STRIDE(j, d) {
                double s = sum_chunks(part, chunks, d, j);
                const double vj = dv[j];
                if (lam > 0.0) s = s + lam * vj;
                if (aug) s = s + rho * vj;
                hd[j] = s;
                dacc += s * vj;
            }
        }
        const double t = block_sum(dacc, red);
        if (threadIdx.x == 0) slot_ptr(blk, kSlotCurv)[blockIdx.x] = t;
        ncurv = gridDim.x;
        grid_barrier(bar);
    }
    // ---- (1) step ----
    const double curv = block_reduce_slot(blk, kSlotCurv, ncurv, &sc);
    if (!isfinite(curv)) {
        if (lead) {
            st->cg_failed = 1;
            st->cg_mid[it] = 0;
        }
        done(0);
        return;
    }
    if (curv <= 0.0) {
        if (it == 0) GRID_STRIDE(j, d) p[j] = -g[j];
        if (lead) {
            st->cg_neg = 1;
            st->cg_mid[it] = 0;
        }
        done(0);
        return;
    }
    const double alpha = r_sq / curv;
    double rr = 0.0;
    if (cached) {
#pragma unroll
        for (int e = 0; e < kTailEpt; ++e) {
            const int64_t j = j0 + e * stride;
            if (j < d) {
                vp[e] += alpha * vd[e];
                vr[e] = vr[e] - alpha * vh[e];
                p[j] = vp[e];
                r[j] = vr[e];
                rr += vr[e] * vr[e];
            }
        }
    } else {
        GRID_STRIDE(j, d) {
            p[j] += alpha * dv[j];
            const double rj = r[j] - alpha * hd[j];
            r[j] = rj;
            rr += rj * rj;
        }
    }
    {
        const double t = block_sum(rr, red);
        if (threadIdx.x == 0) slot_ptr(blk, kSlotRr)[blockIdx.x] = t;
    }
    if (lead) {
        st->cg_iters = it + 1;
        st->cg_mid[it] = 1;
    }
    grid_barrier(bar);
    // ---- (2) direction ----
    __syncthreads();  // sc reused
    const double r_sq_next = block_reduce_slot(blk, kSlotRr, gridDim.x, &sc);
    if (!isfinite(r_sq_next)) {
        if (lead) st->cg_failed = 1;
        done(0);
        return;
    }
    if (sqrt(r_sq_next) <= cg_stop) {
        done(0);
        return;
    }
    const double beta = r_sq_next / r_sq;
    if (cached) {
#pragma unroll
        for (int e = 0; e < kTailEpt; ++e) {
            const int64_t j = j0 + e * stride;
            if (j < d) dv[j] = vr[e] + beta * vd[e];
        }
    } else {
        GRID_STRIDE(j, d) dv[j] = r[j] + beta * dv[j];
    }
    if (lead) st->r_sq[it + 1] = r_sq_next;
    done(1);
}

// The same CG tail on ONE thread-block cluster (up to 16 CTAs x 1024 threads) for the d of the dense
// shards: the two grid-wide exchanges become hardware cluster barriers, and the block partials are
// summed through distributed shared memory (every CTA reads the CS partials in rank order, so all
// CTAs derive bit-identical scalars). Each thread keeps its <= kClEpt elements in registers.
constexpr int kClThreads = 1024;
constexpr int kClEpt = 2;

__device__ __forceinline__ double cluster_sum(cooperative_groups::cluster_group& cl, double* slot, double v,
                                              double* red) {
    // block sum in fixed order -> this CTA's slot; cluster barrier; every CTA sums the slots in rank order
    const double t = block_sum(v, red);
    if (threadIdx.x == 0) *slot = t;
    cl.sync();
    __shared__ double res;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (unsigned q = 0; q < cl.num_blocks(); ++q) s += *cl.map_shared_rank(slot, q);
        res = s;
    }
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kClThreads, 1) k_cg_tail_cl(int it, int64_t d, DevState* st, const DevParams* prm,
                                                              const double* __restrict__ part, int chunks,
                                                              const double* __restrict__ g, double* __restrict__ p,
                                                              double* __restrict__ r, double* __restrict__ dv,
                                                              double* __restrict__ hd, const double* blk, int ncurv,
                                                              unsigned long long* hv_ctr) {
    namespace cgs = cooperative_groups;
    cgs::cluster_group cl = cgs::this_cluster();
    __shared__ double red[32];
    __shared__ double slots[3];  // curvature, <r,r> (read by peers through DSMEM)
    __shared__ double sc;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    auto done = [&](int act_next) {
        if (lead) {
            st->cg_act[it + 1] = act_next;
            st->cert_act = st->it_act && !st->cg_failed;
        }
        cl.sync();  // no CTA exits while peers may still read its slots
    };
    if (!st->cg_act[it]) {
        if (lead) st->cg_mid[it] = 0;
        done(0);
        return;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double vd[kClEpt], vp[kClEpt], vr[kClEpt], vh[kClEpt];
    const double r_sq = st->r_sq[it], cg_stop = st->cg_stop;
    const double lam = prm->lambda, rho = prm->rho;
    const bool aug = prm->augmented;
#pragma unroll
    for (int e = 0; e < kClEpt; ++e) {
        const int64_t j = j0 + e * stride;
        const bool in = j < d;
        vd[e] = in ? dv[j] : 0.0;
        vp[e] = in ? p[j] : 0.0;
        vr[e] = in ? r[j] : 0.0;
        vh[e] = (in && chunks == 0) ? hd[j] : 0.0;
    }
    double curv;
    if (chunks > 0) {
        if (hv_ctr && lead) atomicAdd(hv_ctr, 1ULL);
        double dacc = 0.0;
#pragma unroll
        for (int e = 0; e < kClEpt; ++e) {
            const int64_t j = j0 + e * stride;
            if (j < d) {
                double s = sum_chunks(part, chunks, d, j);
                if (lam > 0.0) s = s + lam * vd[e];
                if (aug) s = s + rho * vd[e];
                hd[j] = s;
                vh[e] = s;
                dacc += s * vd[e];
            }
        }
        curv = cluster_sum(cl, &slots[0], dacc, red);
    } else {
        curv = block_reduce_slot(const_cast<double*>(blk), kSlotCurv, ncurv, &sc);
    }
    if (!isfinite(curv)) {
        if (lead) {
            st->cg_failed = 1;
            st->cg_mid[it] = 0;
        }
        done(0);
        return;
    }
    if (curv <= 0.0) {
        if (it == 0)
            for (int64_t j = j0; j < d; j += stride) p[j] = -g[j];
        if (lead) {
            st->cg_neg = 1;
            st->cg_mid[it] = 0;
        }
        done(0);
        return;
    }
    const double alpha = r_sq / curv;
    double rr = 0.0;
#pragma unroll
    for (int e = 0; e < kClEpt; ++e) {
        const int64_t j = j0 + e * stride;
        if (j < d) {
            vp[e] += alpha * vd[e];
            vr[e] = vr[e] - alpha * vh[e];
            p[j] = vp[e];
            r[j] = vr[e];
            rr += vr[e] * vr[e];
        }
    }
    if (lead) {
        st->cg_iters = it + 1;
        st->cg_mid[it] = 1;
    }
    const double r_sq_next = cluster_sum(cl, &slots[1], rr, red);
    if (!isfinite(r_sq_next)) {
        if (lead) st->cg_failed = 1;
        done(0);
        return;
    }
    if (sqrt(r_sq_next) <= cg_stop) {
        done(0);
        return;
    }
    const double beta = r_sq_next / r_sq;
#pragma unroll
    for (int e = 0; e < kClEpt; ++e) {
        const int64_t j = j0 + e * stride;
        if (j < d) dv[j] = vr[e] + beta * vd[e];
    }
    if (lead) st->r_sq[it + 1] = r_sq_next;
    done(1);
}

// After the certificate Hv (src/newton.cpp:52) and cg_solve's return: |Hp + g| (report-only), the
// CG-failure fallback p = -g (src/newton.cpp:100-104), the descent test p'g >= 0 -> p = -g
// (105-109) and the line-search slope p'g. One grid barrier between the slope partials and the
// decision.
__global__ void __launch_bounds__(256, 4) k_cert_tail(int64_t d, DevState* st, const DevParams* prm,
                                                      const double* __restrict__ part, int chunks, int lp_from_cert,
                                                      const double* __restrict__ g, double* __restrict__ p,
                                                      double* __restrict__ hd, double* blk, int ncert,
                                                      unsigned long long* hv_ctr, unsigned long long* bar) {
    __shared__ double red[32];
    __shared__ double sc;
    cert_tail_body(d, st, prm, part, chunks, lp_from_cert, g, p, hd, blk, ncert, hv_ctr, bar, red, &sc, whole_grid());
}

// Batched Armijo candidates (src/newton.cpp:56-71), partial sums for every trial a_j = gamma^j:
//   blocks [0, rows_blocks): row losses of logits L0 + a_j Lp (stable_exp_cache + loss at x + a_j p,
//     src/softmax.cpp:51-78); warp w of a block owns candidates w, w+8, ..., lane l one row of the
//     block's 32-row group, so every (row, candidate) pair is an independent thread task
//   blocks [rows_blocks, +vec_blocks): |z - x_j + y/rho|^2 (augmented) and |x_j|^2 (ridge)
constexpr int kLsWarps = 8;
constexpr int kLsChunk = 16;

__device__ __forceinline__ double ls_alpha(double gamma, int j) {
    double a = 1.0;
    for (int q = 0; q < j; ++q) a *= gamma;  // alpha *= backtrack_gamma (src/newton.cpp:69)
    return a;
}

__global__ void __launch_bounds__(256) k_ls_partials(int64_t n, int K, const double* __restrict__ L0,
                                                     const double* __restrict__ Lp, const int32_t* __restrict__ labels,
                                                     int rows_blocks, int64_t d, const double* __restrict__ x,
                                                     const double* __restrict__ p, const double* __restrict__ z,
                                                     const double* __restrict__ y, const DevParams* prm, double* blk,
                                                     const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    const int nc = prm->ls_max_iters + 1;
    const double gamma = prm->backtrack_gamma;
    if ((int)blockIdx.x < rows_blocks) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int j = warp; j < nc; j += kLsWarps) {
            const double a = ls_alpha(gamma, j);
            double acc = 0.0;
            for (int64_t i = (int64_t)blockIdx.x * 32 + lane; i < n; i += (int64_t)rows_blocks * 32) {
                const double* l0 = L0 + i * K;
                const double* lp = Lp + i * K;
                const int b = labels[i];
                double m = l0[0] + a * lp[0];
                for (int c = 1; c < K; ++c) {
                    const double l = l0[c] + a * lp[c];
                    if (l > m) m = l;
                }
                m = m > 0.0 ? m : 0.0;
                double s = 0.0;
                for (int c = 0; c < K; ++c) s += exp((l0[c] + a * lp[c]) - m);
                const double al = exp(-m) + s;
                acc += (m + log(al)) - (b <= K ? l0[b - 1] + a * lp[b - 1] : 0.0);
            }
            acc = warp_sum(acc);
            if (lane == 0) slot_ptr(blk, kSlotLs + j)[blockIdx.x] = acc;
        }
        return;
    }
    const int vb = blockIdx.x - rows_blocks, nvb = gridDim.x - rows_blocks;
    const double rho = prm->rho;
    const bool aug = prm->augmented, ridge = prm->lambda > 0.0;
    for (int j0 = 0; j0 < nc; j0 += kLsChunk) {
        double alpha[kLsChunk], at[kLsChunk], ax[kLsChunk];
#pragma unroll
        for (int q = 0; q < kLsChunk; ++q) {
            alpha[q] = ls_alpha(gamma, j0 + q);
            at[q] = 0.0;
            ax[q] = 0.0;
        }
        for (int64_t j = (int64_t)vb * blockDim.x + threadIdx.x; j < d; j += (int64_t)nvb * blockDim.x) {
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
        // all 2 * kLsChunk block sums at once: butterflies per warp, one barrier, warps in fixed order
        __shared__ double wred[kLsWarps][2 * kLsChunk];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int q = 0; q < kLsChunk; ++q) {
            const double s0 = warp_sum(at[q]), s1 = warp_sum(ax[q]);
            if (lane == 0) {
                wred[warp][2 * q] = s0;
                wred[warp][2 * q + 1] = s1;
            }
        }
        __syncthreads();
        if (threadIdx.x < 2 * kLsChunk && j0 + (int)threadIdx.x / 2 < nc) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wred[w][threadIdx.x];
            slot_ptr(blk, kSlotLsVec + 2 * j0 + threadIdx.x)[vb] = t;
        }
        __syncthreads();
    }
}

// Armijo selection (src/newton.cpp:61-70): accept the first trial with F(x + a p) <= f_x + a beta p'g,
// else the last one, flagged capped; then x += a p (src/newton.cpp:120). Every block evaluates all
// candidates (one warp per candidate, in parallel) from the same partials and picks the same a.
__global__ void __launch_bounds__(256) k_ls_step(int64_t d, DevState* st, const DevParams* prm, const double* blk,
                                                 int nrows, int nvec, double* __restrict__ x,
                                                 const double* __restrict__ p, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double fj[kMaxLs + 1];
    __shared__ double a_s;
    const int nc = prm->ls_max_iters + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < nc; j += (int)(blockDim.x >> 5)) {
        double f = reduce_partials(slot_ptr(const_cast<double*>(blk), kSlotLs + j), nrows);
        if (prm->lambda > 0.0)
            f += 0.5 * prm->lambda * reduce_partials(slot_ptr(const_cast<double*>(blk), kSlotLsVec + 2 * j + 1), nvec);
        if (prm->augmented)
            f = f + 0.5 * prm->rho * reduce_partials(slot_ptr(const_cast<double*>(blk), kSlotLsVec + 2 * j), nvec);
        if (lane == 0) fj[j] = f;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double alpha = 1.0;
        int evals = 0, capped = 0;
        for (int j = 0; j < nc; ++j) {
            ++evals;
            if (fj[j] <= st->f_x + alpha * prm->armijo_beta * st->slope) break;
            if (j >= prm->ls_max_iters) {
                capped = 1;
                break;
            }
            alpha *= prm->backtrack_gamma;
        }
        a_s = alpha;
        if (blockIdx.x == 0) {
            st->ls_alpha = alpha;
            st->ls_evals = evals;
            st->ls_capped = capped;
        }
    }
    __syncthreads();
    const double a = a_s;
    GRID_STRIDE(j, d) x[j] += a * p[j];
}

// End of a Newton iteration after the cache pass at the new x (src/newton.cpp:121-127 with the memo
// of src/objective.cpp:9-39): gbase = X^T(P - Y) + lambda x from the split-K partials (chunks > 0),
// <x, x> for the ridge, t = z - x + y/rho and g = gbase - rho t (src/objective.cpp:47-51) with
// <g,g>, <t,t> partials; after one grid barrier block 0 forms the base loss, f, |g| and the trace
// row (k_value_finish semantics).
__global__ void __launch_bounds__(256, 4) k_newton_tail(int64_t d, DevState* st, const DevParams* prm,
                                                        const double* __restrict__ part, int chunks,
                                                        const double* __restrict__ x, const double* __restrict__ z,
                                                        const double* __restrict__ y, double* __restrict__ gbase,
                                                        double* __restrict__ g, double* __restrict__ t, double* blk,
                                                        int nloss, double* scal, DevTrace* trace, int trace_cap,
                                                        unsigned long long* bar, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    newton_tail_body(d, st, prm, part, chunks, x, z, y, gbase, g, t, blk, nloss, scal, trace, trace_cap, bar, red,
                     whole_grid());
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

// One Newton iteration (src/newton.cpp:80-127) as a fixed launch sequence (captured once into a
// CUDA graph): per CG iteration one data pass + one fused tail; the certificate Hv + one tail; the
// Lp pass + batched Armijo partials + selection/step; the cache pass at the new x + one tail.
// Iterations that are not needed are switched off by device flags (guards), not by the host.
void launch_newton_iteration(Shard& s, int cg_max, int ls_max) {
    (void)ls_max;
    cudaStream_t st = s.ctx->stream;
    const int grid = vec_grid(*s.ctx, s.d);
    const int32_t* it_act = &s.st->it_act;
    launch_pdl(k_begin_init, grid, 256, 0, st, s.d, s.st, s.prm, s.g, s.pd, s.r, s.dv);
    tl_mark(s, "begin_init");
    LAUNCH_COUNT(s);
    // DMMA shards: the CG tail runs inside the Hv pass (its last cluster to finish); otherwise one
    // tail launch per iteration
    const bool fused_tail = dmma_supported(s);
    for (int it = 0; it < cg_max; ++it) {
        s.hv_timer_site = it;
        int chunks = 0;
        s.cg_fuse_it = it;
        s.dmma_tail = fused_tail ? kTailCg : kTailNone;
        const int ncurv = op_hv_split(s, s.dv, s.hd, s.dv, kSlotCurv, &s.st->cg_act[it], &chunks);
        s.dmma_tail = kTailNone;
        s.cg_fuse_it = -1;
        s.hv_timer_site = -1;
        if (fused_tail) {
            // nothing more to launch
        } else if (s.tail_cluster > 0) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            cfg.gridDim = dim3(s.tail_cluster, 1, 1);
            cfg.blockDim = dim3(kClThreads, 1, 1);
            cfg.stream = st;
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = s.tail_cluster;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            NADMM_CUDA(cudaLaunchKernelEx(&cfg, k_cg_tail_cl, it, s.d, s.st, (const DevParams*)s.prm,
                                          (const double*)s.part, chunks, (const double*)s.g, s.pd, s.r, s.dv, s.hd,
                                          (const double*)s.blk, ncurv, chunks > 0 ? s.ctx->dctr : nullptr));
        } else {
            launch_coop(k_cg_tail, grid, 256, 0, st, it, s.d, s.st, s.prm, s.part, chunks, s.g, s.pd, s.r, s.dv, s.hd,
                       s.blk, ncurv, chunks > 0 ? s.ctx->dctr : nullptr, s.gbar + 0);
        }
        tl_mark(s, "cg_tail");
        LAUNCH_COUNT(s);
    }
    s.hv_timer_site = cg_max;
    int chunks = 0;
    // certificate Hv (src/newton.cpp:52); its X p logits are stored as the Armijo Lp on the fused paths
    const bool lp_from_cert = dmma_supported(s) || smallp_supported(s);
    s.hv_write_lp = lp_from_cert;
    if (fused_tail) {  // the certificate pass runs whenever the iteration does; its tail decides the rest
        s.dmma_tail = kTailCert;
        op_hv_split(s, s.pd, s.hd, nullptr, 0, it_act, &chunks);
        s.dmma_tail = kTailNone;
        s.hv_write_lp = false;
        s.hv_timer_site = -1;
    } else {
        op_hv_split(s, s.pd, s.hd, nullptr, 0, &s.st->cert_act, &chunks);
        s.hv_write_lp = false;
        s.hv_timer_site = -1;
        launch_coop(k_cert_tail, grid, 256, 0, st, s.d, s.st, s.prm, s.part, chunks, lp_from_cert ? 1 : 0, s.g, s.pd,
                   s.hd, s.blk, grid, chunks > 0 ? s.ctx->dctr : nullptr, s.gbar + 1);
        LAUNCH_COUNT(s);
    }
    tl_mark(s, "cert_tail");
    op_lp(s, s.pd, &s.st->lp_need);  // Lp = X p, only when p changed after the certificate pass
    tl_mark(s, "lp_pass");
    const int rblocks = std::max(1, (int)std::min<int64_t>((s.n + 31) / 32, kBlockPartials));
    // DMMA shards run the line search inside the certificate pass unless p changed after it
    const int32_t* ls_guard = fused_tail ? &s.st->lp_need : it_act;
    launch_pdl(k_ls_partials, rblocks + grid, 256, 0, st, s.n, s.K, s.L0, s.Lp, s.labels, rblocks, s.d, s.x, s.pd,
               s.z, s.y, s.prm, s.blk, ls_guard);
    tl_mark(s, "ls_partials");
    launch_pdl(k_ls_step, grid, 256, 0, st, s.d, s.st, s.prm, s.blk, rblocks, grid, s.x, s.pd, ls_guard);
    tl_mark(s, "ls_step");
    s.ctx->stats.kernel_launches += 2;
    NADMM_LAUNCH_CHECK();
    if (fused_tail) {
        s.dmma_tail = kTailNewton;
        op_cache_split(s, s.x, it_act);
        s.dmma_tail = kTailNone;
        tl_mark(s, "cache_pass+newton_tail");
    } else {
        chunks = op_cache_split(s, s.x, it_act);
        tl_mark(s, "cache_pass");
        launch_coop(k_newton_tail, grid, 256, 0, st, s.d, s.st, s.prm, s.part, chunks, s.x, s.z, s.y, s.gbase, s.g,
                   s.t, s.blk, s.rows_grid, s.scal, s.trace, kTraceCap, s.gbar + 2, it_act);
        tl_mark(s, "newton_tail");
        LAUNCH_COUNT(s);
    }
    NADMM_LAUNCH_CHECK();
}

// One Newton iteration of a NODE GROUP (the local ADMM nodes of an outer iteration, equal (p, K),
// whole-GPU DMMA layouts) as one launch sequence: the per-node loop heads, then every data pass of
// the iteration as ONE group launch over all nodes (dmma_group.cuh) with the node's CG step /
// certificate + line search / Newton tail on its own sub-grid; the rare Lp pass + stand-alone line
// search per node behind its device flag. `timers` (optional): events around the group Hv passes.
void launch_group_iteration(const std::vector<Shard*>& g, int clusters, int cg_max, HvTimer* timers) {
    const int n = (int)g.size();
    cudaStream_t st = g[0]->ctx->stream;
    for (Shard* sp : g) {
        Shard& s = *sp;
        const int grid = vec_grid(*s.ctx, s.d);
        launch_pdl(k_begin_init, grid, 256, 0, st, s.d, s.st, s.prm, s.g, s.pd, s.r, s.dv);
        LAUNCH_COUNT(s);
    }
    std::vector<const double*> W(n);
    std::vector<const int32_t*> gd(n);
    for (int it = 0; it < cg_max; ++it) {
        for (int k = 0; k < n; ++k) {
            W[k] = g[k]->dv;
            gd[k] = &g[k]->st->cg_act[it];
        }
        if (timers) NADMM_CUDA(cudaEventRecordWithFlags(timers[it].start, st, cudaEventRecordExternal));
        dmma_group_pass(g, clusters, kModeHv, W.data(), gd.data(), kTailCg, it, false);
        if (timers) NADMM_CUDA(cudaEventRecordWithFlags(timers[it].stop, st, cudaEventRecordExternal));
    }
    for (int k = 0; k < n; ++k) {  // certificate Hv (src/newton.cpp:52) + fallback / slope + Armijo search
        W[k] = g[k]->pd;
        gd[k] = &g[k]->st->it_act;
    }
    if (timers) NADMM_CUDA(cudaEventRecordWithFlags(timers[cg_max].start, st, cudaEventRecordExternal));
    dmma_group_pass(g, clusters, kModeHv, W.data(), gd.data(), kTailCert, 0, true);
    if (timers) NADMM_CUDA(cudaEventRecordWithFlags(timers[cg_max].stop, st, cudaEventRecordExternal));
    for (Shard* sp : g) {  // p changed after the certificate pass (CG failure / descent flip): Lp + search
        Shard& s = *sp;
        const int grid = vec_grid(*s.ctx, s.d);
        op_lp(s, s.pd, &s.st->lp_need);
        const int rblocks = std::max(1, (int)std::min<int64_t>((s.n + 31) / 32, kBlockPartials));
        launch_pdl(k_ls_partials, rblocks + grid, 256, 0, st, s.n, s.K, s.L0, s.Lp, s.labels, rblocks, s.d, s.x, s.pd,
                   s.z, s.y, s.prm, s.blk, &s.st->lp_need);
        launch_pdl(k_ls_step, grid, 256, 0, st, s.d, s.st, s.prm, s.blk, rblocks, grid, s.x, s.pd, &s.st->lp_need);
        s.ctx->stats.kernel_launches += 2;
    }
    for (int k = 0; k < n; ++k) {  // cache at the new iterate + gradient / value / trace (Newton tail)
        W[k] = g[k]->x;
        gd[k] = &g[k]->st->it_act;
    }
    dmma_group_pass(g, clusters, kModeCache, W.data(), gd.data(), kTailNewton, 0, false);
    NADMM_LAUNCH_CHECK();
}

// Once per shard, outside stream capture: can the CG tail run as one cluster (d small enough for the
// cluster's registers, 16-CTA clusters co-resident)? 0 selects the grid-barrier kernel.
void tail_setup(Shard& s) {
    s.tail_cluster = 0;
    for (int cs : {16, 8}) {
        if (s.d > (int64_t)cs * kClThreads * kClEpt) continue;
        if (cs > 8 && cudaFuncSetAttribute(k_cg_tail_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3(cs, 1, 1);
        cfg.blockDim = dim3(kClThreads, 1, 1);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_cg_tail_cl, &cfg) == cudaSuccess && n >= 1) {
            s.tail_cluster = cs;
            return;
        }
        cudaGetLastError();
    }
}

void launch_set_int(Shard& s, int32_t* dst, int v) {
    k_set_int<<<1, 32, 0, s.ctx->stream>>>(dst, v);
    NADMM_LAUNCH_CHECK();
    LAUNCH_COUNT(s);
}

}  // namespace nadmm
