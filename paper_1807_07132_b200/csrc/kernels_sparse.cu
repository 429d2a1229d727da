// CSR shards with C - 1 <= 32 (the E18/news20-like 20-class sparse config): class-per-lane passes.
//
// The SIMT path gathers the weight of every (nonzero, class) pair from the block-major vector —
// C - 1 separate 32-byte sectors per nonzero, p*(C-1)*8 bytes apart. Here the weight-shaped operand
// is first transposed to an interleaved p x K copy (one d-vector read + write), so the K weights of a
// nonzero's column are one contiguous 8K-byte run that the warp's K lanes read in one coalesced
// access. Rows pass: one warp per row, lane c accumulates logit c over the row's nonzeros in CSR
// order, then runs the row epilogue with warp shuffles (class sums in ascending order). X^T U pass:
// one warp per column of the CSC copy, lane c accumulates sum_rows x_ij U_ic in row order — the U
// row of a nonzero is again one contiguous run.
//
// Reference ops (file:line under /root/reference/proj):
//   sparse X * B, X^T * B             src/dataset.cpp:69-85 (sparse_ * rhs, sparse_.transpose() * rhs)
//   cache / loss / coeff / Hv / predict  src/softmax.cpp:51-139
#include "state.h"

namespace nadmm {

namespace {

constexpr int kSpRowsThreads = 256;
constexpr int kGather = 8;  // independent gathers in flight per warp

// wt (p x K) = transpose of the block-major W (K x p): 32-column tiles through shared memory so both
// the reads (along p) and the writes (32*K contiguous doubles) are coalesced.
__global__ void __launch_bounds__(256) transpose_w_kernel(const double* __restrict__ W, int64_t p, int K,
                                                          double* __restrict__ wt, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    for (int64_t j0 = (int64_t)blockIdx.x * 32; j0 < p; j0 += (int64_t)gridDim.x * 32) {
        for (int c = ty; c < K; c += 8) tile[c][tx] = (j0 + tx < p) ? W[(int64_t)c * p + j0 + tx] : 0.0;
        __syncthreads();
        const int64_t base = j0 * K;
        const int64_t total = (p - j0 < 32 ? p - j0 : 32) * K;
        for (int q = threadIdx.x; q < total; q += 256) wt[base + q] = tile[q % K][q / K];
        __syncthreads();
    }
}

struct SpArgs {
    const int64_t* indptr;
    const int32_t* indices;
    const double* vals;
    const int32_t* labels;
    int64_t n, p;
    int K;
    const double* wt;  // p x K interleaved weights
    const double* Pin;
    double *L0, *P, *U, *Lp, *rowM, *rowA;
    int32_t* pred;
    double* blk;
    const int32_t* guard;
    // column blocks: this launch covers block `b` of `nb`, row segments from rblk; running logits in lsum
    int nb, b;
    const int64_t* rblk;
    double* lsum;
};

// Ascending-order sum over classes of a per-lane value (every lane gets the same result).
__device__ __forceinline__ double class_sum(double v, int K) {
    double s = 0.0;
    for (int c = 0; c < K; ++c) s += __shfl_sync(0xffffffffu, v, c);
    return s;
}

template <int MODE>
__global__ void __launch_bounds__(kSpRowsThreads) sparse_rows_kernel(SpArgs a) {
    if (a.guard && !*a.guard) return;
    __shared__ double red[kSpRowsThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps_total = (int64_t)gridDim.x * (kSpRowsThreads / 32);
    const int K = a.K;
    const bool on = lane < K;
    double acc_loss = 0.0;
    const bool blocked = a.nb > 1;
    for (int64_t i = (int64_t)blockIdx.x * (kSpRowsThreads / 32) + wib; i < a.n; i += warps_total) {
        const int64_t q0 = blocked ? a.rblk[i * (a.nb + 1) + a.b] : a.indptr[i];
        const int64_t q1 = blocked ? a.rblk[i * (a.nb + 1) + a.b + 1] : a.indptr[i + 1];
        double lg = 0.0;
        int64_t q = q0;
        for (; q + kGather <= q1; q += kGather) {  // kGather gathers in flight, accumulated in CSR order
            int j[kGather];
            double v[kGather], w[kGather];
#pragma unroll
            for (int k = 0; k < kGather; ++k) {
                j[k] = __ldg(a.indices + q + k);
                v[k] = __ldg(a.vals + q + k);
            }
#pragma unroll
            for (int k = 0; k < kGather; ++k) w[k] = on ? __ldg(a.wt + (int64_t)j[k] * K + lane) : 0.0;
#pragma unroll
            for (int k = 0; k < kGather; ++k) lg += v[k] * w[k];
        }
        for (; q < q1; ++q) {
            const double w = on ? __ldg(a.wt + (int64_t)__ldg(a.indices + q) * K + lane) : 0.0;
            lg += __ldg(a.vals + q) * w;
        }
        if (blocked) {  // logits = ((block 0 + block 1) + ...) + last block, in block order
            if (a.b > 0 && on) lg = a.lsum[i * K + lane] + lg;
            if (a.b < a.nb - 1) {
                if (on) a.lsum[i * K + lane] = lg;
                continue;
            }
        }
        const int b = a.labels[i];
        if (MODE == kModeLp) {
            if (on) a.Lp[i * K + lane] = lg;
        } else if (MODE == kModeHv) {
            const double pv = on ? a.Pin[i * K + lane] : 0.0;
            const double e = lg * pv;
            const double rs = class_sum(e, K);  // row_sum(V o P), ascending classes
            if (on) a.U[i * K + lane] = e - pv * rs;
        } else {
            double m = on ? lg : -INFINITY;
            m = warp_max(m);
            m = m > 0.0 ? m : 0.0;
            const double e = on ? exp(lg - m) : 0.0;
            const double alpha = exp(-m) + class_sum(e, K);
            const double lb = __shfl_sync(0xffffffffu, lg, (b - 1) & 31);
            if (MODE == kModeCache || MODE == kModeValue) {
                if (lane == 0) acc_loss += (m + log(alpha)) - (b <= K ? lb : 0.0);
                if (MODE == kModeCache) {
                    if (lane == 0) {
                        a.rowM[i] = m;
                        a.rowA[i] = alpha;
                    }
                    if (on) {
                        const double pc = e / alpha;
                        a.L0[i * K + lane] = lg;
                        a.P[i * K + lane] = pc;
                        a.U[i * K + lane] = (lane == b - 1) ? pc - 1.0 : pc;  // coeff (src/softmax.cpp:86-90)
                    }
                }
            } else {  // kModePredict: first class with P == max; class C only if strictly greater
                const double pc = on ? e / alpha : -INFINITY;
                const double best = warp_max(pc);
                const unsigned hit = __ballot_sync(0xffffffffu, on && pc == best);
                if (lane == 0) {
                    int arg = __ffs(hit);  // 1-based class of the lowest set lane
                    if (exp(-m) / alpha > best) arg = K + 1;
                    a.pred[i] = arg;
                    acc_loss += (arg == b) ? 1.0 : 0.0;
                }
            }
        }
    }
    if ((MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) && (!blocked || a.b == a.nb - 1)) {
        if (lane == 0) red[wib] = acc_loss;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kSpRowsThreads / 32; ++w) s += red[w];
            const int slot = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slot * kBlockPartials + blockIdx.x] = s;
        }
    }
}

// X^T U through the CSC copy, one warp per column, lane = class; fused shifts and dot partials.
__global__ void __launch_bounds__(256) csc_cols_kernel(const int64_t* __restrict__ cptr,
                                                       const int32_t* __restrict__ crow,
                                                       const double* __restrict__ cval, int64_t p, int K,
                                                       const double* __restrict__ U, const double* __restrict__ vin,
                                                       const DevParams* prm, int kind, double* __restrict__ out,
                                                       const double* __restrict__ dotvec, double* blk_slot,
                                                       unsigned long long* ctr, const int32_t* guard) {
    if (guard && !*guard) return;
    if (ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr, 1ULL);
    __shared__ double red[32];
    const int lane = threadIdx.x & 31;
    const bool on = lane < K;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
    const double lam = prm->lambda;
    const bool aug = kind == kXtuHv && prm->augmented;
    const double rho = prm->rho;
    double dacc = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < p; j += warps_total) {
        const int64_t q0 = cptr[j], q1 = cptr[j + 1];
        double acc = 0.0;
        int64_t q = q0;
        for (; q + kGather <= q1; q += kGather) {
            int r[kGather];
            double v[kGather], u[kGather];
#pragma unroll
            for (int k = 0; k < kGather; ++k) {
                r[k] = __ldg(crow + q + k);
                v[k] = __ldg(cval + q + k);
            }
#pragma unroll
            for (int k = 0; k < kGather; ++k) u[k] = on ? U[(int64_t)r[k] * K + lane] : 0.0;
#pragma unroll
            for (int k = 0; k < kGather; ++k) acc += v[k] * u[k];
        }
        for (; q < q1; ++q) acc += __ldg(cval + q) * (on ? U[(int64_t)__ldg(crow + q) * K + lane] : 0.0);
        if (on) {
            const int64_t o = (int64_t)lane * p + j;
            double s = acc;
            if (lam > 0.0) s = s + lam * vin[o];
            if (aug) s = s + rho * vin[o];
            out[o] = s;
            if (dotvec) dacc += s * dotvec[o];
        }
    }
    if (dotvec) {
        const double t = block_sum(dacc, red);
        if (threadIdx.x == 0) blk_slot[blockIdx.x] = t;
    }
}

}  // namespace

bool sparse_lanes_supported(const Shard& s) { return s.sparse && s.K <= 32 && s.wt; }

void sparse_rows_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    cudaStream_t st = s.ctx->stream;
    const int tg = (int)std::max<int64_t>(1, std::min<int64_t>((s.p + 31) / 32, 8LL * s.ctx->num_sms));
    transpose_w_kernel<<<tg, 256, 0, st>>>(W, s.p, s.K, s.wt, guard);
    NADMM_LAUNCH_CHECK();
    SpArgs a{};
    a.indptr = s.indptr;
    a.indices = s.indices;
    a.vals = s.vals;
    a.labels = s.labels;
    a.n = s.n;
    a.p = s.p;
    a.K = s.K;
    a.wt = s.wt;
    a.Pin = s.P;
    a.L0 = s.L0;
    a.P = s.P;
    a.U = s.U;
    a.Lp = s.Lp;
    a.rowM = s.rowM;
    a.rowA = s.rowA;
    a.pred = s.pred;
    a.blk = s.blk;
    a.guard = guard;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((s.n + 7) / 8, std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms)));
    s.rows_grid = grid;
    a.nb = s.nblk;
    a.rblk = s.rblk;
    a.lsum = s.lsum;
    for (int b = 0; b < s.nblk; ++b) {  // one launch per column block (its weights stay L2-resident)
        a.b = b;
        switch (mode) {
            case kModeCache: sparse_rows_kernel<kModeCache><<<grid, kSpRowsThreads, 0, st>>>(a); break;
            case kModeHv: sparse_rows_kernel<kModeHv><<<grid, kSpRowsThreads, 0, st>>>(a); break;
            case kModeLp: sparse_rows_kernel<kModeLp><<<grid, kSpRowsThreads, 0, st>>>(a); break;
            case kModeValue: sparse_rows_kernel<kModeValue><<<grid, kSpRowsThreads, 0, st>>>(a); break;
            case kModePredict: sparse_rows_kernel<kModePredict><<<grid, kSpRowsThreads, 0, st>>>(a); break;
        }
        NADMM_LAUNCH_CHECK();
    }
    s.ctx->stats.kernel_launches += 1 + s.nblk;
    s.ctx->stats.data_passes++;
}

int sparse_cols_pass(Shard& s, XtuKind kind, const double* vin, double* out, const double* dotvec, int dot_slot,
                     const int32_t* guard) {
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((s.p + 7) / 8, std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms)));
    csc_cols_kernel<<<grid, 256, 0, s.ctx->stream>>>(s.cptr, s.crow, s.cval, s.p, s.K, s.U, vin, s.prm, kind, out,
                                                     dotvec, s.blk + (int64_t)dot_slot * kBlockPartials,
                                                     kind == kXtuHv ? s.ctx->dctr : nullptr, guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
    return grid;
}

}  // namespace nadmm
