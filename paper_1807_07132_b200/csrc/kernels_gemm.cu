// Dense shards outside the fused passes' shapes (many classes: the C = 100 large-dense config, or
// class counts without a DMMA instantiation): the two contractions of every product are plain FP64
// GEMMs (cuBLAS DGEMM on the tensor cores), with the row epilogue as one warp-per-row kernel between
// them. At C - 1 = 99 the pass is FP64-tensor bound (~47 FLOP/B), so reading X twice
// costs nothing against the roofline.
//
//   logits  Lg = X * blocks(W)       src/dataset.cpp:69-76    DGEMM (n x K, row-major = K x n col-major)
//   epilogue (U / cache / loss / P)  src/softmax.cpp:51-112   gemm_epilogue_kernel, in place on Lg
//   X^T U                            src/dataset.cpp:78-85    DGEMM into split-K chunk 0 of `part`
//
// The DGEMMs cannot read the solver's device guard flags; they write only scratch buffers (U, Lp,
// part) whose consumers are guarded, so a switched-off iteration wastes work but changes nothing.
#include <cublas_v2.h>

#include "state.h"

namespace nadmm {

namespace {

constexpr int kEpiThreads = 256;

#define NADMM_CUBLAS(x)                                                                                   \
    do {                                                                                                  \
        const cublasStatus_t st_ = (x);                                                                   \
        if (st_ != CUBLAS_STATUS_SUCCESS)                                                                 \
            raise(NADMM_ECUDA, std::string("cuBLAS error ") + std::to_string((int)st_) + " @" __FILE__ ":" + \
                                   std::to_string(__LINE__));                                             \
    } while (0)

struct EpiArgs {
    int64_t n;
    int K;
    double* Lg;  // n x K logits, overwritten with U (Hv / cache modes)
    const double* Pin;
    const int32_t* labels;
    double *L0, *P, *rowM, *rowA;
    int32_t* pred;
    double* blk;
    const int32_t* guard;
};

// Row epilogue of the pass modes, one warp per row, classes in ascending order (rows_kernel's).
template <int MODE>
__global__ void __launch_bounds__(kEpiThreads) gemm_epilogue_kernel(EpiArgs a) {
    if (a.guard && !*a.guard) return;
    __shared__ double e_s[kEpiThreads / 32][kMaxClasses];
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps_total = (int64_t)gridDim.x * (kEpiThreads / 32);
    const int K = a.K;
    double* e = e_s[wib];
    double acc_loss = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * (kEpiThreads / 32) + wib; i < a.n; i += warps_total) {
        double* lg = a.Lg + i * K;
        const int b = a.labels[i];
        if (MODE == kModeHv) {
            for (int c = lane; c < K; c += 32) e[c] = lg[c] * a.Pin[i * K + c];
            __syncwarp();
            double rs = 0.0;
            if (lane == 0)
                for (int c = 0; c < K; ++c) rs += e[c];
            rs = __shfl_sync(0xffffffffu, rs, 0);
            for (int c = lane; c < K; c += 32) lg[c] = e[c] - a.Pin[i * K + c] * rs;
        } else {
            double m = -INFINITY;
            for (int c = lane; c < K; c += 32) m = fmax(m, lg[c]);
            m = warp_max(m);
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
                __syncwarp();
                if (MODE == kModeCache) {
                    if (lane == 0) {
                        a.rowM[i] = m;
                        a.rowA[i] = alpha;
                    }
                    for (int c = lane; c < K; c += 32) {
                        const double pc = e[c] / alpha;
                        a.L0[i * K + c] = lg[c];
                        a.P[i * K + c] = pc;
                        lg[c] = (c == b - 1) ? pc - 1.0 : pc;  // coeff (src/softmax.cpp:86-90)
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
        __syncthreads();
        if (lane == 0) red[wib] = acc_loss;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kEpiThreads / 32; ++w) s += red[w];
            const int slot = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slot * kBlockPartials + blockIdx.x] = s;
        }
    }
}

cublasHandle_t handle(const Shard& s) { return static_cast<cublasHandle_t>(s.ctx->blas); }

}  // namespace

void gemm_setup(Shard& s) {
    if (s.sparse || s.ctx->blas || smallp_supported(s) || dmma_supported(s)) return;
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return;  // path unavailable: SIMT passes serve the shard
    NADMM_CUBLAS(cublasSetStream(h, s.ctx->stream));
    // fixed workspace: no allocation inside stream capture, identical kernels on every replay
    const size_t ws = size_t(32) << 20;
    NADMM_CUDA(cudaMalloc(&s.ctx->blas_ws, ws));
    NADMM_CUBLAS(cublasSetWorkspace(h, s.ctx->blas_ws, ws));
    NADMM_CUBLAS(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST));
    NADMM_CUBLAS(cublasSetAtomicsMode(h, CUBLAS_ATOMICS_NOT_ALLOWED));  // deterministic results
    s.ctx->blas = h;
}

void gemm_teardown(Ctx& c) {
    if (c.blas) cublasDestroy(static_cast<cublasHandle_t>(c.blas));
    if (c.blas_ws) cudaFree(c.blas_ws);
    c.blas = nullptr;
    c.blas_ws = nullptr;
}

bool gemm_supported(const Shard& s) { return !s.sparse && s.ctx->blas && s.part; }

void gemm_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    cublasHandle_t h = handle(s);
    const double one = 1.0, zero = 0.0;
    const int n = (int)s.n, p = (int)s.p, K = s.K;
    // Lg^T (K x n, col-major) = blocks(W)^T (K x p) * X^T (p x n, the row-major X with ld = ldx)
    double* lg = mode == kModeLp ? s.Lp : s.U;
    NADMM_CUBLAS(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, K, n, p, &one, W, p, s.X, (int)s.ldx, &zero, lg, K));
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
    if (mode == kModeLp) return;
    EpiArgs a{};
    a.n = s.n;
    a.K = K;
    a.Lg = lg;
    a.Pin = s.P;
    a.labels = s.labels;
    a.L0 = s.L0;
    a.P = s.P;
    a.rowM = s.rowM;
    a.rowA = s.rowA;
    a.pred = s.pred;
    a.blk = s.blk;
    a.guard = guard;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((s.n + kEpiThreads / 32 - 1) / (kEpiThreads / 32), std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms)));
    cudaStream_t st = s.ctx->stream;
    switch (mode) {
        case kModeCache: gemm_epilogue_kernel<kModeCache><<<grid, kEpiThreads, 0, st>>>(a); break;
        case kModeHv: gemm_epilogue_kernel<kModeHv><<<grid, kEpiThreads, 0, st>>>(a); break;
        case kModeValue: gemm_epilogue_kernel<kModeValue><<<grid, kEpiThreads, 0, st>>>(a); break;
        case kModePredict: gemm_epilogue_kernel<kModePredict><<<grid, kEpiThreads, 0, st>>>(a); break;
        default: break;
    }
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    s.rows_grid = grid;
    if (mode == kModeHv || mode == kModeCache) {
        // part chunk 0 (p x K col-major == block-major d) = X^T (p x n) * U (n x K; U^T is K x n col-major)
        NADMM_CUBLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, p, K, n, &one, s.X, (int)s.ldx, s.U, K, &zero, s.part, p));
        s.ctx->stats.kernel_launches++;
        s.ctx->stats.data_passes++;
        s.last_chunks = 1;
    }
}

}  // namespace nadmm
