// Solver tail bodies shared by the stand-alone tail kernels (kernels_vec.cu) and the fused DMMA pass
// (dmma_kernel.cuh), which runs them with its whole persistent grid after its last tile. Every
// reduction is a fixed-order two-stage sum (block partial slots, then reduce_partials), so all blocks
// derive bit-identical scalars; grid_barrier needs a grid that is entirely co-resident.
#pragma once

#include "state.h"

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
__device__ __forceinline__ void cert_tail_body(int64_t d, DevState* st, const DevParams* prm,
                                               const double* __restrict__ part, int chunks, int lp_from_cert,
                                               const double* __restrict__ g, double* __restrict__ p,
                                               double* __restrict__ hd, double* blk, int ncert,
                                               unsigned long long* hv_ctr, unsigned long long* bar, double* red,
                                               double* sc) {
    if (!st->it_act) return;
    const bool cert = st->cert_act, failed = st->cg_failed;
    const double lam = prm->lambda, rho = prm->rho;
    const bool aug = prm->augmented;
    if (cert && chunks > 0 && hv_ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(hv_ctr, 1ULL);
    double cacc = 0.0, sacc = 0.0;
    GRID_STRIDE(j, d) {
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
    if (threadIdx.x == 0 && cert) slot_ptr(blk, kSlotCert)[blockIdx.x] = t;
    t = block_sum(sacc, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotSlope)[blockIdx.x] = t;
    ncert = gridDim.x;
    grid_barrier(bar);
    double slope = block_reduce_slot(blk, kSlotSlope, gridDim.x, sc);
    const bool flip = slope >= 0.0;
    if (flip) GRID_STRIDE(j, d) p[j] = -g[j];
    if (blockIdx.x == 0 && threadIdx.x < 32) {
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
                                                 unsigned long long* bar, double* red) {
    const double lam = prm->lambda, rho = prm->rho;
    const bool aug = prm->augmented;
    double xx = 0.0, gg = 0.0, tt = 0.0;
    GRID_STRIDE(j, d) {
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
    if (threadIdx.x == 0) slot_ptr(blk, kSlotRidge)[blockIdx.x] = sres;
    sres = block_sum(gg, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotGg)[blockIdx.x] = sres;
    sres = block_sum(tt, red);
    if (threadIdx.x == 0) slot_ptr(blk, kSlotTt)[blockIdx.x] = sres;
    grid_barrier(bar);
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    const int nvec = gridDim.x;
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

}  // namespace nadmm
