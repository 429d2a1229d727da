// Solver tail bodies shared by the stand-alone tail kernels (kernels_vec.cu) and the fused DMMA pass
// (dmma_kernel.cuh), which runs them with its whole persistent grid after its last tile. Every
// reduction is a fixed-order two-stage sum (block partial slots, then reduce_partials), so all blocks
// derive bit-identical scalars; grid_barrier needs a grid that is entirely co-resident.
#pragma once

#include "state.h"

namespace nadmm {

#define GRID_STRIDE(j, d) \
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (d); j += (int64_t)gridDim.x * blockDim.x)

// The (sub-)grid a solver tail runs on: the whole launch grid, or -- in a node-group DMMA pass -- the
// CTAs [first, first + nb) assigned to one ADMM node (its own barrier counter and partial slots).
struct VGrid {
    int b, nb;
};

__device__ __forceinline__ VGrid whole_grid() { return VGrid{(int)blockIdx.x, (int)gridDim.x}; }

#define VGRID_STRIDE(vg, j, d) \
    for (int64_t j = (int64_t)(vg).b * blockDim.x + threadIdx.x; j < (d); j += (int64_t)(vg).nb * blockDim.x)

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

// Sum of the fused dense pass's split-K partials at element j, in chunk order: loads are issued in
// predicated batches of 8 so they are in flight together; the additions keep the sequential order.
__device__ __forceinline__ double sum_chunks(const double* __restrict__ part, int chunks, int64_t d, int64_t j) {
    double s = 0.0;
    for (int ch = 0; ch < chunks; ch += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (ch + q < chunks) ? __ldcg(part + (int64_t)(ch + q) * d + j) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (ch + q < chunks) s += v[q];
    }
    return s;
}

// After the certificate Hv (src/newton.cpp:52) and cg_solve's return: |Hp + g| (report-only), the
// CG-failure fallback p = -g (src/newton.cpp:100-104), the descent test p'g >= 0 -> p = -g
// (105-109) and the line-search slope p'g. One grid barrier between the slope partials and the
// decision. Shared by k_cert_tail and the certificate DMMA pass (run by its whole grid).
__device__ __forceinline__ bool cert_tail_body(int64_t d, DevState* st, const DevParams* prm,
                                               const double* __restrict__ part, int chunks, int lp_from_cert,
                                               const double* __restrict__ g, double* __restrict__ p,
                                               double* __restrict__ hd, double* blk, int ncert,
                                               unsigned long long* hv_ctr, unsigned long long* bar, double* red,
                                               double* sc, VGrid vg) {
    if (!st->it_act) return false;
    const bool cert = st->cert_act, failed = st->cg_failed;
    const double lam = prm->lambda, rho = prm->rho;
    const bool aug = prm->augmented;
    if (cert && chunks > 0 && hv_ctr && vg.b == 0 && threadIdx.x == 0) atomicAdd(hv_ctr, 1ULL);
    double cacc = 0.0, sacc = 0.0;
    VGRID_STRIDE(vg, j, d) {
        const double gj = g[j];
        double pj = p[j];
        if (cert) {
            double hp;
            if (chunks > 0) {
                hp = sum_chunks(part, chunks, d, j);
                if (lam > 0.0) hp = hp + lam * pj;
                if (aug) hp = hp + rho * pj;
                hd[j] = hp;
            } else {
                hp = hd[j];
            }
            const double v = hp + gj;
            cacc += v * v;
        }
        if (failed) {
            pj = -gj;
            p[j] = pj;
        }
        sacc += pj * gj;
    }
    double t = block_sum(cacc, red);
    if (threadIdx.x == 0 && cert) slot_ptr(blk, kSlotCert)[vg.b] = t;
    t = block_sum(sacc, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotSlope)[vg.b] = t;
    ncert = vg.nb;
    grid_barrier_n(bar, vg.nb);
    double slope = block_reduce_slot(blk, kSlotSlope, vg.nb, sc);
    const bool flip = slope >= 0.0;
    if (flip) VGRID_STRIDE(vg, j, d) p[j] = -g[j];
    if (vg.b == 0 && threadIdx.x < 32) {
        const double cv = cert ? reduce_partials(slot_ptr(blk, kSlotCert), ncert) : 0.0;
        if (threadIdx.x == 0) {
            if (flip) slope = -st->g_sq;  // (-g).g == -|g|^2 under the same reduction order
            st->slope = slope;
            if (cert) st->cg_residual = sqrt(cv);
            if (failed || flip) st->fallback = 1;
            // the certificate pass stored Lp = X p (when it ran); only a changed p needs the Lp pass
            st->lp_need = (!cert || failed || flip || !lp_from_cert) ? 1 : 0;
        }
    }
    return !cert || failed || flip || !lp_from_cert;  // the same in every block
}

// End of a Newton iteration after the cache pass at the new x (src/newton.cpp:121-127 with the memo
// of src/objective.cpp:9-39): gbase = X^T(P - Y) + lambda x from the split-K partials (chunks > 0),
// <x, x> for the ridge, t = z - x + y/rho and g = gbase - rho t (src/objective.cpp:47-51) with
// <g,g>, <t,t> partials; after one grid barrier block 0 forms the base loss, f, |g| and the trace
// row (k_value_finish semantics). Shared by k_newton_tail and the cache DMMA pass.
__device__ __forceinline__ void newton_tail_body(int64_t d, DevState* st, const DevParams* prm,
                                                 const double* __restrict__ part, int chunks,
                                                 const double* __restrict__ x, const double* __restrict__ z,
                                                 const double* __restrict__ y, double* __restrict__ gbase,
                                                 double* __restrict__ g, double* __restrict__ t, double* blk, int nloss,
                                                 double* scal, DevTrace* trace, int trace_cap,
                                                 unsigned long long* bar, double* red, VGrid vg) {
    const double lam = prm->lambda, rho = prm->rho;
    const bool aug = prm->augmented;
    double xx = 0.0, gg = 0.0, tt = 0.0;
    VGRID_STRIDE(vg, j, d) {
        const double xj = x[j];
        double gb;
        if (chunks > 0) {
            gb = sum_chunks(part, chunks, d, j);
            if (lam > 0.0) gb = gb + lam * xj;  // src/softmax.cpp:93
            gbase[j] = gb;
        } else {
            gb = gbase[j];
        }
        xx += xj * xj;
        double gj = gb;
        if (aug) {
            const double tj = (z[j] - xj) + y[j] / rho;
            t[j] = tj;
            tt += tj * tj;
            gj = gj - rho * tj;
        }
        g[j] = gj;
        gg += gj * gj;
    }
    double sres = block_sum(xx, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotRidge)[vg.b] = sres;
    sres = block_sum(gg, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotGg)[vg.b] = sres;
    sres = block_sum(tt, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotTt)[vg.b] = sres;
    grid_barrier_n(bar, vg.nb);
    if (vg.b != 0 || threadIdx.x >= 32) return;
    const int nvec = vg.nb;
    double base = reduce_partials(slot_ptr(blk, kSlotLoss), nloss);
    if (lam > 0.0) base += 0.5 * lam * reduce_partials(slot_ptr(blk, kSlotRidge), nvec);  // src/softmax.cpp:76
    const double g_sq = reduce_partials(slot_ptr(blk, kSlotGg), nvec);
    const double t_sq = reduce_partials(slot_ptr(blk, kSlotTt), nvec);
    if (threadIdx.x != 0) return;
    scal[0] = base;
    double f = base;
    if (aug) f = f + 0.5 * rho * t_sq;
    st->f_base = base;
    st->f_x = f;
    st->g_sq = g_sq;
    st->g_norm = sqrt(g_sq);
    const int k = st->iter;
    if (k < trace_cap) {
        DevTrace rr;
        rr.iter = k;
        rr.grad_norm = st->rec_gnorm;
        rr.step = st->ls_alpha;
        rr.cg_iters = st->cg_failed ? 0 : st->cg_iters;
        rr.cg_residual = st->cg_failed ? 0.0 : st->cg_residual;
        rr.objective = f;
        rr.ls_capped = st->ls_capped;
        rr.cg_fallback = st->fallback;
        rr.fn_evals = st->ls_evals;
        rr.pad = 0;
        trace[k] = rr;
    }
    st->iter = k + 1;
    if (!isfinite(f)) {  // "non-finite objective at iteration k"
        st->error = NADMM_ESOLVER;
        st->active = 0;
    }
}

// Batched Armijo line search (src/newton.cpp:56-71, as k_ls_partials + k_ls_step) run by a whole
// co-resident grid: (row group, candidate) items -> one partial each in slot kSlotLs + j (group index),
// vector candidate terms -> block partials, one grid barrier, then every block evaluates all
// candidates from the same partials, applies the first-accept rule and steps x += a p.
// `scratch` holds >= 32 * kLsFusedChunk doubles.
constexpr int kLsFusedChunk = 16;

__device__ __forceinline__ void ls_fused_body(int64_t n, int K, const double* __restrict__ L0, const double* __restrict__ Lp,
                              const int32_t* __restrict__ labels, int64_t d, double* __restrict__ x,
                              const double* __restrict__ p, const double* __restrict__ z,
                              const double* __restrict__ y, const DevParams* prm, DevState* st, double* blk,
                              unsigned long long* bar, double* scratch, double* sc, VGrid vg) {
    const int nc = prm->ls_max_iters + 1;
    const double gamma = prm->backtrack_gamma;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    // rows: groups of rows_per_group rows (a multiple of 32, <= kBlockPartials groups)
    int64_t rpg = ((n + kBlockPartials - 1) / kBlockPartials + 31) / 32 * 32;
    if (rpg < 32) rpg = 32;
    const int ngroups = (int)((n + rpg - 1) / rpg);
    const int64_t items = (int64_t)ngroups * nc;
    for (int64_t it = (int64_t)vg.b * nwarps + warp; it < items; it += (int64_t)vg.nb * nwarps) {
        const int j = (int)(it % nc), grp = (int)(it / nc);
        double a = 1.0;
        for (int q = 0; q < j; ++q) a *= gamma;  // alpha *= backtrack_gamma (src/newton.cpp:69)
        double acc = 0.0;
        const int64_t r_end = (grp + 1) * rpg < n ? (grp + 1) * rpg : n;
        for (int64_t i = grp * rpg + lane; i < r_end; i += 32) {
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
            acc += (m + log(exp(-m) + s)) - (b <= K ? l0[b - 1] + a * lp[b - 1] : 0.0);
        }
        acc = warp_sum(acc);
        if (lane == 0) slot_ptr(blk, kSlotLs + j)[grp] = acc;
    }
    // vector terms of every candidate: |z - x_j + y/rho|^2 and |x_j|^2, x_j = x + a_j p
    const double rho = prm->rho;
    const bool aug = prm->augmented, ridge = prm->lambda > 0.0;
    for (int j0 = 0; j0 < nc; j0 += kLsFusedChunk) {
        double alpha[kLsFusedChunk], at[kLsFusedChunk], ax[kLsFusedChunk];
        double a = 1.0;
        for (int q = 0; q < j0; ++q) a *= gamma;
#pragma unroll
        for (int q = 0; q < kLsFusedChunk; ++q) {
            alpha[q] = a;
            a *= gamma;
            at[q] = 0.0;
            ax[q] = 0.0;
        }
        VGRID_STRIDE(vg, jj, d) {
            const double xj = x[jj], pj = p[jj];
            const double zj = aug ? z[jj] : 0.0, yr = aug ? y[jj] / rho : 0.0;
#pragma unroll
            for (int q = 0; q < kLsFusedChunk; ++q) {
                const double xt = xj + alpha[q] * pj;  // x + alpha * p (src/newton.cpp:62)
                if (aug) {
                    const double tq = (zj - xt) + yr;
                    at[q] += tq * tq;
                }
                if (ridge) ax[q] += xt * xt;
            }
        }
        __syncthreads();  // scratch reuse
#pragma unroll
        for (int q = 0; q < kLsFusedChunk; ++q) {
            const double s0 = warp_sum(at[q]), s1 = warp_sum(ax[q]);
            if (lane == 0) {
                scratch[warp * 2 * kLsFusedChunk + 2 * q] = s0;
                scratch[warp * 2 * kLsFusedChunk + 2 * q + 1] = s1;
            }
        }
        __syncthreads();
        if (threadIdx.x < 2 * kLsFusedChunk && j0 + (int)threadIdx.x / 2 < nc) {
            double t = 0.0;
            for (int w = 0; w < nwarps; ++w) t += scratch[w * 2 * kLsFusedChunk + threadIdx.x];
            slot_ptr(blk, kSlotLsVec + 2 * j0 + threadIdx.x)[vg.b] = t;
        }
    }
    grid_barrier_n(bar, vg.nb);
    // every block: candidate objectives (one warp per candidate), first-accept rule, step
    __syncthreads();
    double* fj = scratch;  // nc <= kMaxLs + 1 doubles
    for (int j = warp; j < nc; j += nwarps) {
        double f = reduce_partials(slot_ptr(blk, kSlotLs + j), ngroups);
        if (prm->lambda > 0.0) f += 0.5 * prm->lambda * reduce_partials(slot_ptr(blk, kSlotLsVec + 2 * j + 1), vg.nb);
        if (prm->augmented) f = f + 0.5 * prm->rho * reduce_partials(slot_ptr(blk, kSlotLsVec + 2 * j), vg.nb);
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
        *sc = alpha;
        if (vg.b == 0) {
            st->ls_alpha = alpha;
            st->ls_evals = evals;
            st->ls_capped = capped;
        }
    }
    __syncthreads();
    const double a = *sc;
    VGRID_STRIDE(vg, jj, d) x[jj] += a * p[jj];
}

}  // namespace nadmm
