// Data-pass kernels over a shard's feature matrix (SIMT path; any p, any C <= 129, dense or CSR).
//
// Reference ops (file:line under /root/reference/proj):
//   X * B          Dataset::multiply            src/dataset.cpp:69-76
//   X^T * B        Dataset::multiply_transposed src/dataset.cpp:78-85 (CSC copy for sparse)
//   cache/loss     stable_exp_cache, loss       src/softmax.cpp:51-78
//   gradient       coeff = P - Y; X^T coeff     src/softmax.cpp:80-95
//   Hv epilogue    U = V o P - P o rowsum(VoP)  src/softmax.cpp:97-112
//   predict        argmax + tie rule            src/softmax.cpp:118-139
//
// Device layout: X row-major (ldx), work matrices n x K row-major, weight-shaped vectors in the
// reference block-major layout (block c = [c*p, (c+1)*p)).
#include "state.h"

namespace nadmm {

namespace {

constexpr int kRowsThreads = 256;
constexpr int kKc = 16;  // classes per register chunk

struct RowsArgs {
    const double* X;
    int64_t ldx;
    const int64_t* indptr;
    const int32_t* indices;
    const double* vals;
    const int32_t* labels;
    int64_t n, p;
    int K;
    const double* W;   // block-major weights
    const double* Pin; // probs (Hv epilogue)
    double* L0;
    double* P;
    double* U;
    double* Lp;
    double* rowM;
    double* rowA;
    int32_t* pred;
    double* blk;
    const int32_t* guard;
};

// Row logits for the class chunk [c0, c0+kc): every lane ends with the full sums in acc[].
template <bool SPARSE>
__device__ __forceinline__ void row_chunk(const RowsArgs& a, int64_t i, int c0, int kc, double (&acc)[kKc]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < kKc; ++c) acc[c] = 0.0;
    if (SPARSE) {
        const int64_t q0 = a.indptr[i], q1 = a.indptr[i + 1];
        for (int64_t q = q0 + lane; q < q1; q += 32) {
            const double v = a.vals[q];
            const int64_t j = a.indices[q];
#pragma unroll
            for (int c = 0; c < kKc; ++c)
                if (c < kc) acc[c] += v * __ldg(a.W + (int64_t)(c0 + c) * a.p + j);
        }
    } else {
        const double* xi = a.X + i * a.ldx;
        for (int64_t j = lane; j < a.p; j += 32) {
            const double x = xi[j];
#pragma unroll
            for (int c = 0; c < kKc; ++c)
                if (c < kc) acc[c] += x * __ldg(a.W + (int64_t)(c0 + c) * a.p + j);
        }
    }
#pragma unroll
    for (int c = 0; c < kKc; ++c) acc[c] = warp_sum(acc[c]);
}

template <bool SPARSE, int MODE>
__global__ void __launch_bounds__(kRowsThreads) rows_kernel(RowsArgs a) {
    if (a.guard && !*a.guard) return;
    __shared__ double lg_s[kRowsThreads / 32][kMaxClasses];
    __shared__ double e_s[kRowsThreads / 32][kMaxClasses];
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps_total = (int64_t)gridDim.x * (kRowsThreads / 32);
    const int K = a.K;
    double* lg = lg_s[wib];
    double* e = e_s[wib];
    double acc_loss = 0.0;  // lane 0 of each warp: rows in grid-stride order
    for (int64_t i = (int64_t)blockIdx.x * (kRowsThreads / 32) + wib; i < a.n; i += warps_total) {
        for (int c0 = 0; c0 < K; c0 += kKc) {
            const int kc = min(kKc, K - c0);
            double acc[kKc];
            row_chunk<SPARSE>(a, i, c0, kc, acc);
            if (lane == 0)
#pragma unroll
                for (int c = 0; c < kKc; ++c)
                    if (c < kc) lg[c0 + c] = acc[c];
        }
        __syncwarp();
        const int b = a.labels[i];
        if (MODE == kModeLp) {
            for (int c = lane; c < K; c += 32) a.Lp[i * K + c] = lg[c];
        } else if (MODE == kModeHv) {
            // vw = V o P; row_sum ascending over classes; U = vw - P * row_sum (src/softmax.cpp:103-107)
            for (int c = lane; c < K; c += 32) e[c] = lg[c] * a.Pin[i * K + c];
            __syncwarp();
            double rs = 0.0;
            if (lane == 0)
                for (int c = 0; c < K; ++c) rs += e[c];
            rs = __shfl_sync(0xffffffffu, rs, 0);
            for (int c = lane; c < K; c += 32) a.U[i * K + c] = e[c] - a.Pin[i * K + c] * rs;
        } else {
            // stable exp cache (src/softmax.cpp:54-61): M = max(0, max_c logit); every exponent <= 0
            double m = lg[0];
            for (int c = 1; c < K; ++c)
                if (lg[c] > m) m = lg[c];
            m = m > 0.0 ? m : 0.0;
            for (int c = lane; c < K; c += 32) e[c] = exp(lg[c] - m);
            __syncwarp();
            double alpha = 0.0;
            if (lane == 0) {
                double s = 0.0;
                for (int c = 0; c < K; ++c) s += e[c];
                alpha = exp(-m) + s;
            }
            alpha = __shfl_sync(0xffffffffu, alpha, 0);
            if (MODE == kModeCache || MODE == kModeValue) {
                if (lane == 0) acc_loss += (m + log(alpha)) - (b <= K ? lg[b - 1] : 0.0);
                if (MODE == kModeCache) {
                    if (lane == 0) {
                        a.rowM[i] = m;
                        a.rowA[i] = alpha;
                    }
                    for (int c = lane; c < K; c += 32) {
                        const double pc = e[c] / alpha;
                        a.L0[i * K + c] = lg[c];
                        a.P[i * K + c] = pc;
                        a.U[i * K + c] = (c == b - 1) ? pc - 1.0 : pc;  // coeff (src/softmax.cpp:86-90)
                    }
                }
            } else {  // kModePredict (src/softmax.cpp:118-139)
                if (lane == 0) {
                    const double residual = exp(-m) / alpha;
                    double best = e[0] / alpha;
                    for (int c = 1; c < K; ++c) {
                        const double pc = e[c] / alpha;
                        if (pc > best) best = pc;
                    }
                    int arg = 0;
                    for (int c = 0; c < K; ++c)
                        if (e[c] / alpha == best) {
                            arg = c + 1;
                            break;
                        }
                    if (residual > best) arg = K + 1;
                    a.pred[i] = arg;
                    acc_loss += (arg == b) ? 1.0 : 0.0;
                }
            }
        }
        __syncwarp();
    }
    if (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) {
        // fixed-order block reduction of the per-warp accumulators
        __syncthreads();
        if (lane == 0) red[wib] = acc_loss;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kRowsThreads / 32; ++w) s += red[w];
            const int slot = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slot * kBlockPartials + blockIdx.x] = s;
        }
    }
}

// Split-K partial of X^T U for dense shards: block (column tile of 128, row chunk) ->
// part[chunk][c*p + j]. U rows are staged through shared memory.
constexpr int kXtuCols = 128;
constexpr int kXtuRows = 32;

__global__ void __launch_bounds__(kXtuCols) xtu_partial_kernel(const double* __restrict__ X, int64_t ldx, int64_t n,
                                                               int64_t p, int K, const double* __restrict__ U,
                                                               int64_t rows_per_chunk, double* __restrict__ part,
                                                               int64_t d, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double us[kXtuRows][kKc];
    const int64_t j = (int64_t)blockIdx.x * kXtuCols + threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk;
    const int64_t r1 = min(n, r0 + rows_per_chunk);
    for (int c0 = 0; c0 < K; c0 += kKc) {
        const int kc = min(kKc, K - c0);
        double acc[kKc];
#pragma unroll
        for (int c = 0; c < kKc; ++c) acc[c] = 0.0;
        for (int64_t rb = r0; rb < r1; rb += kXtuRows) {
            const int nr = (int)((r1 - rb) < kXtuRows ? (r1 - rb) : kXtuRows);
            __syncthreads();
            for (int q = threadIdx.x; q < nr * kKc; q += kXtuCols) {
                const int rr = q / kKc, cc = q % kKc;
                us[rr][cc] = cc < kc ? U[(rb + rr) * K + c0 + cc] : 0.0;
            }
            __syncthreads();
            if (j < p) {
                for (int rr = 0; rr < nr; ++rr) {
                    const double x = X[(rb + rr) * ldx + j];
#pragma unroll
                    for (int c = 0; c < kKc; ++c)
                        if (c < kc) acc[c] += x * us[rr][c];
                }
            }
        }
        if (j < p)
#pragma unroll
            for (int c = 0; c < kKc; ++c)
                if (c < kc) part[(int64_t)blockIdx.y * d + (int64_t)(c0 + c) * p + j] = acc[c];
    }
}

// out = sum_chunks part (+ lambda*vin)(+ rho*vin); optional dot partials with dotvec.
__global__ void __launch_bounds__(256) finalize_kernel(const double* __restrict__ part, int chunks, int64_t d,
                                                       const double* __restrict__ vin, const DevParams* prm,
                                                       int kind, double* __restrict__ out,
                                                       const double* __restrict__ dotvec, double* blk_slot,
                                                       unsigned long long* ctr, const int32_t* guard) {
    if (guard && !*guard) return;
    if (ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr, 1ULL);
    __shared__ double red[32];
    const double lam = prm->lambda;
    const bool aug = kind == kXtuHv && prm->augmented;
    const double rho = prm->rho;
    double dacc = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d; j += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int ch = 0; ch < chunks; ++ch) s += part[(int64_t)ch * d + j];
        if (lam > 0.0) s = s + lam * vin[j];   // src/softmax.cpp:93, 110
        if (aug) s = s + rho * vin[j];         // src/objective.cpp:52-54
        out[j] = s;
        if (dotvec) dacc += s * dotvec[j];
    }
    if (dotvec) {
        const double t = block_sum(dacc, red);
        if (threadIdx.x == 0) blk_slot[blockIdx.x] = t;
    }
}

// Sparse X^T U through the CSC copy: warp per column, fused shifts and dot partials.
__global__ void __launch_bounds__(256) csc_xtu_kernel(const int64_t* __restrict__ cptr, const int32_t* __restrict__ crow,
                                                      const double* __restrict__ cval, int64_t p, int K,
                                                      const double* __restrict__ U, const double* __restrict__ vin,
                                                      const DevParams* prm, int kind, double* __restrict__ out,
                                                      const double* __restrict__ dotvec, double* blk_slot,
                                                      unsigned long long* ctr, const int32_t* guard) {
    if (guard && !*guard) return;
    if (ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr, 1ULL);
    __shared__ double red[32];
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
    const double lam = prm->lambda;
    const bool aug = kind == kXtuHv && prm->augmented;
    const double rho = prm->rho;
    double dacc = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < p; j += warps_total) {
        for (int c0 = 0; c0 < K; c0 += kKc) {
            const int kc = min(kKc, K - c0);
            double acc[kKc];
#pragma unroll
            for (int c = 0; c < kKc; ++c) acc[c] = 0.0;
            for (int64_t q = cptr[j] + lane; q < cptr[j + 1]; q += 32) {
                const double v = cval[q];
                const double* ur = U + (int64_t)crow[q] * K + c0;
#pragma unroll
                for (int c = 0; c < kKc; ++c)
                    if (c < kc) acc[c] += v * ur[c];
            }
#pragma unroll
            for (int c = 0; c < kKc; ++c) acc[c] = warp_sum(acc[c]);
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < kKc; ++c) {
                    if (c < kc) {
                        const int64_t o = (int64_t)(c0 + c) * p + j;
                        double s = acc[c];
                        if (lam > 0.0) s = s + lam * vin[o];
                        if (aug) s = s + rho * vin[o];
                        out[o] = s;
                        if (dotvec) dacc += s * dotvec[o];
                    }
                }
            }
        }
    }
    if (dotvec) {
        const double t = block_sum(dacc, red);
        if (threadIdx.x == 0) blk_slot[blockIdx.x] = t;
    }
}

__global__ void dot_partials_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t d,
                                    double* blk_slot, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d; j += (int64_t)gridDim.x * blockDim.x)
        s += a[j] * b[j];
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) blk_slot[blockIdx.x] = t;
}

__global__ void loss_finalize_kernel(const double* blk_loss, int nparts, const double* blk_ridge, int nridge,
                                     const DevParams* prm, int add_ridge, double* dst, const int32_t* guard) {
    if (guard && !*guard) return;
    if (threadIdx.x >= 32) return;
    double total = reduce_partials(blk_loss, nparts);
    if (add_ridge && prm->lambda > 0.0) {
        const double sq = reduce_partials(blk_ridge, nridge);
        total += 0.5 * prm->lambda * sq;  // src/softmax.cpp:76
    }
    if (threadIdx.x == 0) *dst = total;
}

}  // namespace

int vec_grid(const Ctx& c, int64_t d) {
    const int64_t want = (d + 255) / 256;
    const int64_t cap = std::min<int64_t>(kBlockPartials, 4LL * c.num_sms);
    return (int)std::max<int64_t>(1, std::min(want, cap));
}

void rows_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    if (sparse_lanes_supported(s)) return sparse_rows_pass(s, mode, W, guard);
    RowsArgs a{};
    a.X = s.X;
    a.ldx = s.ldx;
    a.indptr = s.indptr;
    a.indices = s.indices;
    a.vals = s.vals;
    a.labels = s.labels;
    a.n = s.n;
    a.p = s.p;
    a.K = s.K;
    a.W = W;
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
    const int64_t warps = (s.n + 0);
    int grid = (int)std::min<int64_t>((warps + 7) / 8, std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms));
    grid = std::max(grid, 1);
    s.rows_grid = grid;
    cudaStream_t st = s.ctx->stream;
#define NADMM_ROWS(SP, M) rows_kernel<SP, M><<<grid, kRowsThreads, 0, st>>>(a)
    if (s.sparse) {
        switch (mode) {
            case kModeCache: NADMM_ROWS(true, kModeCache); break;
            case kModeHv: NADMM_ROWS(true, kModeHv); break;
            case kModeLp: NADMM_ROWS(true, kModeLp); break;
            case kModeValue: NADMM_ROWS(true, kModeValue); break;
            case kModePredict: NADMM_ROWS(true, kModePredict); break;
        }
    } else {
        switch (mode) {
            case kModeCache: NADMM_ROWS(false, kModeCache); break;
            case kModeHv: NADMM_ROWS(false, kModeHv); break;
            case kModeLp: NADMM_ROWS(false, kModeLp); break;
            case kModeValue: NADMM_ROWS(false, kModeValue); break;
            case kModePredict: NADMM_ROWS(false, kModePredict); break;
        }
    }
#undef NADMM_ROWS
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
}

void finalize_partials(Shard& s, int chunks, XtuKind kind, const double* vin, double* out, const double* dotvec,
                       int dot_slot, const int32_t* guard, int* dot_grid) {
    const int grid = vec_grid(*s.ctx, s.d);
    finalize_kernel<<<grid, 256, 0, s.ctx->stream>>>(s.part, chunks, s.d, vin, s.prm, kind, out, dotvec,
                                                     s.blk + (int64_t)dot_slot * kBlockPartials,
                                                     kind == kXtuHv ? s.ctx->dctr : nullptr, guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    if (dot_grid) *dot_grid = grid;
}

int xtu_pass(Shard& s, XtuKind kind, const double* vin, double* out, const double* dotvec, int dot_slot,
             const int32_t* guard) {
    cudaStream_t st = s.ctx->stream;
    if (sparse_lanes_supported(s)) return sparse_cols_pass(s, kind, vin, out, dotvec, dot_slot, guard);
    if (s.sparse) {
        const int grid = (int)std::min<int64_t>((s.p + 7) / 8, std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms));
        csc_xtu_kernel<<<std::max(grid, 1), 256, 0, st>>>(s.cptr, s.crow, s.cval, s.p, s.K, s.U, vin, s.prm, kind, out,
                                                          dotvec, s.blk + (int64_t)dot_slot * kBlockPartials,
                                                          kind == kXtuHv ? s.ctx->dctr : nullptr, guard);
        NADMM_LAUNCH_CHECK();
        s.ctx->stats.kernel_launches++;
        s.ctx->stats.data_passes++;
        return std::max(grid, 1);
    }
    const int col_blocks = ceil_div(s.p, kXtuCols);
    int chunks = std::max(1, ceil_div(2LL * s.ctx->num_sms, col_blocks));
    chunks = std::min<int>(chunks, std::max(1, ceil_div(s.n, kXtuRows)));
    chunks = std::min(chunks, s.part_chunks);
    const int64_t rpc = ((s.n + chunks - 1) / chunks + kXtuRows - 1) / kXtuRows * kXtuRows;
    chunks = ceil_div(s.n, rpc);
    xtu_partial_kernel<<<dim3(col_blocks, chunks), kXtuCols, 0, st>>>(s.X, s.ldx, s.n, s.p, s.K, s.U, rpc, s.part, s.d,
                                                                      guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
    int g = 0;
    finalize_partials(s, chunks, kind, vin, out, dotvec, dot_slot, guard, &g);
    return g;
}

void dot_partials(Shard& s, const double* a, const double* b, int slot, const int32_t* guard, int* grid_out) {
    const int grid = vec_grid(*s.ctx, s.d);
    dot_partials_kernel<<<grid, 256, 0, s.ctx->stream>>>(a, b, s.d, s.blk + (int64_t)slot * kBlockPartials, guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    if (grid_out) *grid_out = grid;
}

void loss_finalize(Shard& s, const double* w, int add_ridge, double* dst, const int32_t* guard) {
    int ng = 0;
    if (add_ridge) dot_partials(s, w, w, kSlotRidge, guard, &ng);
    loss_finalize_kernel<<<1, 32, 0, s.ctx->stream>>>(s.blk + (int64_t)kSlotLoss * kBlockPartials, s.rows_grid,
                                                      s.blk + (int64_t)kSlotRidge * kBlockPartials, ng, s.prm,
                                                      add_ridge, dst, guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
}

}  // namespace nadmm
