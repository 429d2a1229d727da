// Synchronous mini-batch SGD on device shards: the worker's SGD branch
// (src/worker.cpp:197-218) and the coordinator step of SPEC.md:461-468 (sync_sgd).
//
// Worker step: epoch-keyed permutation (Rng(mix_seed(seed, epoch)).shuffle, src/data_io.cpp /
// inc/data_io.hpp:23-28), mini-batch rows perm[(step * m + j) % n], gradient(minibatch, z, 0) / m
// (src/softmax.cpp:80-95). Two kernels, both deterministic: a warp per batch row for the logits and
// the P - Y coefficients, then X_b^T U with every output accumulated over the batch rows in order
// (dense: a thread per feature; CSR: the rows applied one after another, columns of a row distinct).
// Coordinator: g_bar = (sum_i g_i) / N in worker order (+ one NCCL allreduce across ranks),
// x <- x - eta g_bar; one metrics row per epoch with F(x); divergence (F > 1e3 F(x0)) aborts.
#include <chrono>
#include <cstring>
#include <cmath>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "solver.h"
#include "solver_tails.cuh"

namespace nadmm {

namespace {

constexpr int kSgdRowWarps = 8;
constexpr int kSgdChunk = 16;  // classes per register chunk

__device__ __forceinline__ int64_t batch_row(const int32_t* perm, int64_t n, int64_t step, int64_t m, int64_t j) {
    return perm[(step * m + j) % n];
}

// Logits of batch row j, stable softmax as stable_exp_cache (src/softmax.cpp:51-63), U = P - Y.
__global__ void __launch_bounds__(32 * kSgdRowWarps) k_sgd_rows(const double* __restrict__ X, int64_t ldx,
                                                                const int64_t* __restrict__ indptr,
                                                                const int32_t* __restrict__ indices,
                                                                const double* __restrict__ vals,
                                                                const int32_t* __restrict__ labels,
                                                                const int32_t* __restrict__ perm, int64_t n,
                                                                int64_t p, int K, int64_t step, int64_t m,
                                                                const double* __restrict__ W, double* __restrict__ U) {
    __shared__ double lg[kSgdRowWarps][kMaxClasses];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * kSgdRowWarps + warp;
    if (j >= m) return;
    const int64_t r = batch_row(perm, n, step, m, j);
    for (int c0 = 0; c0 < K; c0 += kSgdChunk) {
        double acc[kSgdChunk];
#pragma unroll
        for (int c = 0; c < kSgdChunk; ++c) acc[c] = 0.0;
        if (indptr) {
            for (int64_t k = indptr[r] + lane; k < indptr[r + 1]; k += 32) {
                const int64_t f = indices[k];
                const double v = vals[k];
#pragma unroll
                for (int c = 0; c < kSgdChunk; ++c)
                    if (c0 + c < K) acc[c] += v * W[(int64_t)(c0 + c) * p + f];
            }
        } else {
            const double* row = X + r * ldx;
            for (int64_t f = lane; f < p; f += 32) {
                const double v = row[f];
#pragma unroll
                for (int c = 0; c < kSgdChunk; ++c)
                    if (c0 + c < K) acc[c] += v * W[(int64_t)(c0 + c) * p + f];
            }
        }
#pragma unroll
        for (int c = 0; c < kSgdChunk; ++c) {
            const double s = warp_sum(acc[c]);
            if (lane == 0 && c0 + c < K) lg[warp][c0 + c] = s;
        }
    }
    __syncwarp();
    if (lane != 0) return;
    double M = 0.0;  // max{0, logits}
    for (int c = 0; c < K; ++c) M = fmax(M, lg[warp][c]);
    double rs = 0.0;
    for (int c = 0; c < K; ++c) {
        const double e = exp(lg[warp][c] - M);
        lg[warp][c] = e;
        rs += e;
    }
    const double alpha = exp(-M) + rs;
    const int b = labels[r];
    for (int c = 0; c < K; ++c) {
        const double pc = lg[warp][c] / alpha;
        U[j * K + c] = (c == b - 1) ? pc - 1.0 : pc;
    }
}

// Dense X_b^T U / m: thread per feature, batch rows accumulated in order.
__global__ void __launch_bounds__(256) k_sgd_xtu_dense(const double* __restrict__ X, int64_t ldx,
                                                       const int32_t* __restrict__ perm, int64_t n, int64_t p, int K,
                                                       int64_t step, int64_t m, const double* __restrict__ U,
                                                       double* __restrict__ g) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= p) return;
    const double dm = (double)m;
    for (int c0 = 0; c0 < K; c0 += kSgdChunk) {
        double acc[kSgdChunk];
#pragma unroll
        for (int c = 0; c < kSgdChunk; ++c) acc[c] = 0.0;
        for (int64_t j = 0; j < m; ++j) {
            const double x = X[batch_row(perm, n, step, m, j) * ldx + f];
            const double* u = U + j * K + c0;
#pragma unroll
            for (int c = 0; c < kSgdChunk; ++c)
                if (c0 + c < K) acc[c] = __dadd_rn(acc[c], __dmul_rn(x, u[c]));
        }
#pragma unroll
        for (int c = 0; c < kSgdChunk; ++c)
            if (c0 + c < K) g[(int64_t)(c0 + c) * p + f] = acc[c] / dm;
    }
}

// CSR X_b^T U: one CTA applies the batch rows in order (a row's columns are distinct).
__global__ void __launch_bounds__(1024) k_sgd_xtu_csr(const int64_t* __restrict__ indptr,
                                                      const int32_t* __restrict__ indices,
                                                      const double* __restrict__ vals, const int32_t* __restrict__ perm,
                                                      int64_t n, int64_t p, int K, int64_t step, int64_t m,
                                                      const double* __restrict__ U, double* __restrict__ g) {
    for (int64_t j = 0; j < m; ++j) {
        const int64_t r = batch_row(perm, n, step, m, j);
        const double* u = U + j * K;
        for (int64_t k = indptr[r] + threadIdx.x; k < indptr[r + 1]; k += blockDim.x) {
            const int64_t f = indices[k];
            const double v = vals[k];
            for (int c = 0; c < K; ++c) {
                double* gp = g + (int64_t)c * p + f;
                *gp = __dadd_rn(*gp, __dmul_rn(v, u[c]));
            }
        }
        __syncthreads();
    }
}

__global__ void k_sgd_scale(int64_t d, double m, double* __restrict__ g) {
    GRID_STRIDE(j, d) g[j] = g[j] / m;
}

// gsum = sum_i g_i in worker order.
__global__ void k_sgd_sum(int64_t d, const double* const* __restrict__ gs, int nw, double* __restrict__ out) {
    GRID_STRIDE(j, d) {
        double s = gs[0][j];
        for (int i = 1; i < nw; ++i) s = __dadd_rn(s, gs[i][j]);
        out[j] = s;
    }
}

// x <- x - eta * (gsum / N)
__global__ void k_sgd_step(int64_t d, double eta, double n_workers, const double* __restrict__ gsum,
                           double* __restrict__ x) {
    GRID_STRIDE(j, d) x[j] = __dsub_rn(x[j], __dmul_rn(eta, gsum[j] / n_workers));
}

// block partials of |x|^2, then one warp sums them in order
__global__ void __launch_bounds__(256) k_sgd_sq(int64_t d, const double* __restrict__ x, double* __restrict__ part) {
    __shared__ double red[32];
    double a = 0.0;
    GRID_STRIDE(j, d) a += x[j] * x[j];
    const double t = block_sum(a, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_sgd_sum_parts(const double* __restrict__ part, int nb, double* out) {
    if (threadIdx.x >= 32) return;
    const double v = reduce_partials(part, nb);
    if (threadIdx.x == 0) *out = v;
}

int vec_grid(const Shard& s, int64_t d) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(4 * (int64_t)s.ctx->num_sms, (d + 255) / 256));
}

}  // namespace

// Rng(seed).shuffle of 0..n-1 (inc/data_io.hpp:23-28), the worker's per-epoch permutation.
void epoch_permutation(uint64_t seed, int64_t n, int32_t* perm) {
    std::mt19937_64 eng(seed);
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    for (int64_t i = n; i > 1; --i) {  // uniform_int(i): rejection sampling (src/data_io.cpp:35-43)
        const uint64_t bound = (uint64_t)i, mx = ~uint64_t(0), limit = mx - (mx % bound);
        uint64_t v = eng();
        while (v >= limit) v = eng();
        std::swap(perm[i - 1], perm[v % bound]);
    }
}

void validate_sgd(const Shard& s, const nadmm_sgd_cfg& c) {
    if (c.batch < 1 || c.batch > s.n) raise(NADMM_ECONFIG, "sgd batch size must lie in [1, local n]");
    if (c.steps_per_epoch < 1) raise(NADMM_ECONFIG, "sgd steps_per_epoch must be >= 1");
}

// The worker's SGD branch for scatter `iteration` at the point z (device): g = gradient(batch, z, 0) / m.
void sgd_worker_grad(Shard& s, const nadmm_sgd_cfg& c, uint32_t iteration, const double* z, double* g) {
    validate_sgd(s, c);
    cudaStream_t st = s.ctx->stream;
    const int epoch = (int)iteration / c.steps_per_epoch;
    if (!s.sgd_perm) {
        NADMM_CUDA(cudaMalloc(&s.sgd_perm, sizeof(int32_t) * (size_t)s.n));
        s.bytes += 4 * s.n;
    }
    if (epoch != s.sgd_epoch || c.seed != s.sgd_seed) {
        std::vector<int32_t> perm((size_t)s.n);
        epoch_permutation(nadmm_mix_seed(c.seed, (uint64_t)epoch), s.n, perm.data());
        NADMM_CUDA(cudaMemcpyAsync(s.sgd_perm, perm.data(), sizeof(int32_t) * (size_t)s.n, cudaMemcpyHostToDevice, st));
        stream_sync(st);  // the host vector goes out of scope
        s.sgd_epoch = epoch;
        s.sgd_seed = c.seed;
    }
    const int64_t m = c.batch, step = (int64_t)iteration % c.steps_per_epoch;
    if (s.sgd_u_len < m * s.K) {
        if (s.sgd_u) {
            stream_sync(st);
            cudaFree(s.sgd_u);
            s.bytes -= 8 * s.sgd_u_len;
        }
        NADMM_CUDA(cudaMalloc(&s.sgd_u, sizeof(double) * (size_t)(m * s.K)));
        s.sgd_u_len = m * s.K;
        s.bytes += 8 * s.sgd_u_len;
    }
    const int rows_grid = (int)((m + kSgdRowWarps - 1) / kSgdRowWarps);
    k_sgd_rows<<<rows_grid, 32 * kSgdRowWarps, 0, st>>>(s.sparse ? nullptr : s.X, s.ldx, s.sparse ? s.indptr : nullptr,
                                                        s.indices, s.vals, s.labels, s.sgd_perm, s.n, s.p, s.K, step, m,
                                                        z, s.sgd_u);
    NADMM_LAUNCH_CHECK();
    if (s.sparse) {
        NADMM_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * (size_t)s.d, st));
        k_sgd_xtu_csr<<<1, 1024, 0, st>>>(s.indptr, s.indices, s.vals, s.sgd_perm, s.n, s.p, s.K, step, m, s.sgd_u, g);
        NADMM_LAUNCH_CHECK();
        k_sgd_scale<<<vec_grid(s, s.d), 256, 0, st>>>(s.d, (double)m, g);
        NADMM_LAUNCH_CHECK();
        s.ctx->stats.kernel_launches += 3;
    } else {
        k_sgd_xtu_dense<<<(int)((s.p + 255) / 256), 256, 0, st>>>(s.X, s.ldx, s.sgd_perm, s.n, s.p, s.K, step, m,
                                                                  s.sgd_u, g);
        NADMM_LAUNCH_CHECK();
        s.ctx->stats.kernel_launches += 2;
    }
}

// sync_sgd over this process's shards; `red` (may be null) sums across ranks.
SgdOutcome sgd_run(std::vector<Shard*>& shards, const SgdReduce* red, const nadmm_sgd_cfg& cfg_in, double lambda,
                   double* x_dev, nadmm_metrics_row* rows, int row_cap) {
    Shard& s0 = *shards[0];
    cudaStream_t st = s0.ctx->stream;
    const int64_t d = s0.d;
    if (!(cfg_in.eta > 0.0)) raise(NADMM_ECONFIG, "sgd step size must be > 0");
    if (cfg_in.epochs < 0) raise(NADMM_ECONFIG, "sgd epochs must be >= 0");
    for (Shard* s : shards)
        if (s->d != d) raise(NADMM_ECONFIG, "shard weight dimensions differ");
    // global worker and row counts (workers are concatenated in rank order)
    double counts[2] = {(double)shards.size(), 0.0};
    for (Shard* s : shards) counts[1] += (double)s->n;
    if (red) red->host(counts, 2);
    const double n_workers = counts[0];
    nadmm_sgd_cfg cfg = cfg_in;
    if (cfg.batch < 1) raise(NADMM_ECONFIG, "sgd batch size must lie in [1, local n]");
    if (cfg.steps_per_epoch <= 0)  // ceil(n / (m N)) mini-batch steps per data pass
        cfg.steps_per_epoch = (int32_t)std::max<double>(1.0, std::ceil(counts[1] / ((double)cfg.batch * n_workers)));
    for (Shard* s : shards) validate_sgd(*s, cfg);
    const int vg = vec_grid(s0, d);
    std::vector<double*> gs(shards.size());
    double* gbuf = nullptr;
    double* gsum = nullptr;
    double** gptr = nullptr;
    struct Free {
        std::vector<void*> p;
        ~Free() {
            for (void* q : p)
                if (q) cudaFree(q);
        }
    } fr;
    NADMM_CUDA(cudaMalloc(&gbuf, sizeof(double) * (size_t)d * shards.size()));
    fr.p.push_back(gbuf);
    NADMM_CUDA(cudaMalloc(&gsum, sizeof(double) * (size_t)(d + vg + 4)));
    fr.p.push_back(gsum);
    NADMM_CUDA(cudaMalloc(&gptr, sizeof(double*) * shards.size()));
    fr.p.push_back(gptr);
    double* scratch = gsum + d;  // vg partials + 4 scalars
    for (size_t i = 0; i < shards.size(); ++i) gs[i] = gbuf + (int64_t)i * d;
    NADMM_CUDA(cudaMemcpyAsync(gptr, gs.data(), sizeof(double*) * gs.size(), cudaMemcpyHostToDevice, st));
    auto objective = [&]() {  // F(x) = sum_i loss(D_i, x) + lambda/2 |x|^2 over all ranks
        double f = 0.0, h = 0.0;
        for (Shard* s : shards) {
            op_value(*s, x_dev, scratch + vg, 0, nullptr);
            NADMM_CUDA(cudaMemcpyAsync(&h, scratch + vg, sizeof(double), cudaMemcpyDeviceToHost, st));
            stream_sync(st);
            f += h;
        }
        double buf[1] = {f};
        if (red) red->host(buf, 1);
        k_sgd_sq<<<vg, 256, 0, st>>>(d, x_dev, scratch);
        NADMM_LAUNCH_CHECK();
        k_sgd_sum_parts<<<1, 32, 0, st>>>(scratch, vg, scratch + vg + 1);
        NADMM_LAUNCH_CHECK();
        double xx = 0.0;
        NADMM_CUDA(cudaMemcpyAsync(&xx, scratch + vg + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
        stream_sync(st);
        return buf[0] + 0.5 * lambda * xx;
    };
    SgdOutcome out;
    out.steps_per_epoch = cfg.steps_per_epoch;
    const double f0 = objective();
    out.f0 = f0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int e = 0; e < cfg.epochs; ++e) {
        for (int t = 0; t < cfg.steps_per_epoch; ++t) {
            const uint32_t it = (uint32_t)(e * cfg.steps_per_epoch + t);
            for (size_t i = 0; i < shards.size(); ++i) sgd_worker_grad(*shards[i], cfg, it, x_dev, gs[i]);
            k_sgd_sum<<<vg, 256, 0, st>>>(d, gptr, (int)shards.size(), gsum);
            NADMM_LAUNCH_CHECK();
            if (red) red->dev(gsum, d);
            k_sgd_step<<<vg, 256, 0, st>>>(d, cfg.eta, n_workers, gsum, x_dev);
            NADMM_LAUNCH_CHECK();
            s0.ctx->stats.kernel_launches += 2;
        }
        const double F = objective();
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (rows && e < row_cap) {
            nadmm_metrics_row& r = rows[e];
            std::memset(&r, 0, sizeof r);
            r.iteration = e;
            r.wall_seconds = wall;
            r.train_objective = F;
            r.theta = NAN;
            r.primal_norm = r.dual_norm = r.eps_pri = r.eps_dual = NAN;
            r.inner_iterations = cfg.steps_per_epoch;
            r.fn_evals = cfg.steps_per_epoch * (int)shards.size();
            r.rho_mean = NAN;
            // cumulative like the ADMM rows (MetricsRow.messages, inc/metrics.hpp:23): 2N per mini-batch step
            r.messages = (int64_t)(2.0 * n_workers) * cfg.steps_per_epoch * (int64_t)(e + 1);
        }
        out.epochs = e + 1;
        out.final_objective = F;
        if (!(F <= 1e3 * f0))  // unstable step sizes abort the run
            raise(NADMM_ESOLVER, "sync_sgd: objective diverged at epoch " + std::to_string(e));
    }
    stream_sync(st);
    return out;
}

}  // namespace nadmm
