// Consensus ADMM over device-resident shards (run_admm, inc/admm.hpp:17-140).
//
// One rank per GPU. Each rank owns `n_local` ADMM workers (shards). Per outer iteration:
//   1. every local worker runs the run_worker ADMM branch (src/worker.cpp:168-196) on device;
//   2. the consensus sum S = sum_i (rho_i x_i - y_i) | sum_i rho_i is formed per rank in ascending
//      worker order and combined with ONE ncclAllReduce (the reference's gather + z_update);
//   3. every rank forms the identical z = S / (lambda + sum rho), updates its own y_i and y_hat_i,
//      and computes residual / tolerance partials; per-rank scalars travel in one small
//      ncclAllGather and are combined on every host in rank order;
//   4. spectral penalty selection runs per worker on local data only.
// The reference's scatter/gather frames (inc/comm.hpp) disappear: z is formed redundantly on every
// GPU, y_i and rho_i never leave their GPU.
#include <nccl.h>

#include <chrono>
#include <thread>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "solver.h"
#include "solver_kernels.h"

using namespace nadmm;

struct nadmm_comm_s {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    Ctx* ctx = nullptr;
};

namespace nadmm {
namespace {

thread_local std::string* g_err_sink = nullptr;

#define NADMM_NCCL(call)                                                                              \
    do {                                                                                              \
        ncclResult_t r__ = (call);                                                                    \
        if (r__ != ncclSuccess) ::nadmm::raise(NADMM_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r__)); \
    } while (0)

constexpr int kMaxLocal = 16;

struct LocalPtrs {
    const double* x[kMaxLocal];
    const double* y[kMaxLocal];
    int n;
};

#define GRID_STRIDE(j, d) \
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (d); j += (int64_t)gridDim.x * blockDim.x)

// Rank scalars carried in the consensus buffer's per-rank slots: the slots of other
// ranks are zero, so the allreduce sum is a gather and every rank combines them in rank order.
enum RankStat : int {
    kStSumX = 0,    // sum_i |x_i|^2
    kStMaxY = 1,    // max_i |y_i|^2
    kStMaxPri = 2,  // max_i primal_i
    kStMaxDual = 3, // max_i dual_i
    kStPriSq = 4,   // sum_i primal_i^2
    kStDualSq = 5,  // sum_i dual_i^2
    kStF = 6,       // sum_i F_i(z)
    kStZZ = 7,      // |z|^2
    kStats = 8
};

// Consensus buffer of this rank: [S_local (d) | sum rho | kStats slots per rank]. S_local = sum_i
// (rho_i x_i - y_i) in ascending local worker id; the rank's own slot carries the previous iteration's
// rank scalars (they ride in this iteration's allreduce), the other slots are zero.
__global__ void k_local_sum(int64_t d, LocalPtrs lp, const double* __restrict__ rho, double* __restrict__ buf,
                            const double* __restrict__ stats_prev, int rank, int nranks) {
    GRID_STRIDE(j, d) {
        double s = rho[0] * lp.x[0][j] - lp.y[0][j];
        for (int i = 1; i < lp.n; ++i) s += rho[i] * lp.x[i][j] - lp.y[i][j];
        buf[j] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            double rs = rho[0];
            for (int i = 1; i < lp.n; ++i) rs += rho[i];
            buf[d] = rs;
        }
        for (int q = threadIdx.x; q < kStats * nranks; q += 32)
            buf[d + 1 + q] = (q / kStats == rank && stats_prev) ? stats_prev[q % kStats] : 0.0;
    }
}

// Flush of the last iteration's rank scalars: this rank's slot = stats, the others zero.
__global__ void k_fill_slots(double* __restrict__ slots, const double* __restrict__ stats, int rank, int nranks) {
    for (int q = threadIdx.x; q < kStats * nranks; q += blockDim.x)
        slots[q] = (q / kStats == rank) ? stats[q % kStats] : 0.0;
}

// Bitwise-deterministic mode: this rank's per-worker terms rho_i x_i - y_i (no FMA
// contraction, as the oracle evaluates them), its rho_i and its stats slot, to be all-gathered.
__global__ void k_local_terms(int64_t d, LocalPtrs lp, const double* __restrict__ rho, double* __restrict__ out,
                              const double* __restrict__ stats_prev) {
    GRID_STRIDE(j, d) {
        for (int i = 0; i < lp.n; ++i) out[(int64_t)i * d + j] = __dsub_rn(__dmul_rn(rho[i], lp.x[i][j]), lp.y[i][j]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < lp.n; ++i) out[(int64_t)lp.n * d + i] = rho[i];
        for (int q = 0; q < kStats; ++q) out[(int64_t)lp.n * d + lp.n + q] = stats_prev ? stats_prev[q] : 0.0;
    }
}

// Ascending-id pairwise tree over the gathered worker values (the oracle's tree_sum: mid = lo +
// ceil((hi - lo) / 2)), additions without contraction. Worker w's value sits at
// g[(w / nl) * blk + base + (w % nl) * stride] (rank-major gathered blocks). Recursion depth <= 7.
__device__ double tree_sum_dev(const double* g, int64_t blk, int nl, int64_t base, int64_t stride, int lo, int hi) {
    if (hi - lo == 1) return g[(int64_t)(lo / nl) * blk + base + (int64_t)(lo % nl) * stride];
    const int mid = lo + (hi - lo + 1) / 2;
    return __dadd_rn(tree_sum_dev(g, blk, nl, base, stride, lo, mid), tree_sum_dev(g, blk, nl, base, stride, mid, hi));
}

// z = tree(terms) / (lambda + tree(rho)) over all n_total workers in global id order.
__global__ void k_tree_z(int64_t d, const double* __restrict__ g, int n_local, int nranks, double lambda,
                         double* __restrict__ z, double* __restrict__ pz, double* part) {
    __shared__ double red[32];
    const int64_t blk = (int64_t)n_local * d + n_local + kStats;  // one rank's gathered block
    const int n = n_local * nranks;
    const double denom = __dadd_rn(lambda, tree_sum_dev(g, blk, n_local, (int64_t)n_local * d, 1, 0, n));
    double zz = 0.0;
    GRID_STRIDE(j, d) {
        const double v = __ddiv_rn(tree_sum_dev(g, blk, n_local, j, d, 0, n), denom);
        pz[j] = z[j];
        z[j] = v;
        zz += v * v;
    }
    const double t = block_sum(zz, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// z_update: z = S / (lambda + sum rho); prev_z kept; partials |z|^2.
__global__ void k_z_update(int64_t d, const double* __restrict__ buf, double lambda, double* __restrict__ z,
                           double* __restrict__ pz, double* part) {
    __shared__ double red[32];
    const double denom = lambda + buf[d];
    double zz = 0.0;
    GRID_STRIDE(j, d) {
        pz[j] = z[j];
        const double v = buf[j] / denom;
        z[j] = v;
        zz += v * v;
    }
    const double t = block_sum(zz, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// Per worker: y_hat = y + rho (z_prev - x); y += rho (z - x); partials
// of |z - x|^2 (primal), |rho (z - z_prev)|^2 (dual), |x|^2 and |y_new|^2 (tolerances).
__global__ void k_worker_update(int64_t d, const double* __restrict__ rho_p, const double* __restrict__ x,
                                double* __restrict__ y, double* __restrict__ yh, const double* __restrict__ z,
                                const double* __restrict__ pz, double* part /* 4 x kBlockPartials */, int exact) {
    __shared__ double red[32];
    const double rho = *rho_p;
    double pr = 0.0, du = 0.0, xx = 0.0, yy = 0.0;
    GRID_STRIDE(j, d) {
        const double xj = x[j], yj = y[j];
        double yn;
        if (exact) {  // the oracle's evaluation order, no contraction (bitwise-deterministic mode)
            if (yh) yh[j] = __dadd_rn(yj, __dmul_rn(rho, __dsub_rn(pz[j], xj)));
            yn = __dadd_rn(yj, __dmul_rn(rho, __dsub_rn(z[j], xj)));
        } else {
            if (yh) yh[j] = yj + rho * (pz[j] - xj);
            yn = yj + rho * (z[j] - xj);
        }
        y[j] = yn;
        const double r = z[j] - xj;
        const double q = rho * (z[j] - pz[j]);
        pr += r * r;
        du += q * q;
        xx += xj * xj;
        yy += yn * yn;
    }
    double t = block_sum(pr, red);
    if (threadIdx.x == 0) part[0 * kBlockPartials + blockIdx.x] = t;
    t = block_sum(du, red);
    if (threadIdx.x == 0) part[1 * kBlockPartials + blockIdx.x] = t;
    t = block_sum(xx, red);
    if (threadIdx.x == 0) part[2 * kBlockPartials + blockIdx.x] = t;
    t = block_sum(yy, red);
    if (threadIdx.x == 0) part[3 * kBlockPartials + blockIdx.x] = t;
}

// Secant dots for the spectral update: <dx,dyh>, |dx|^2, |dyh|^2, <dz,-dy>, |dz|^2, |dy|^2.
__global__ void k_sps_dots(int64_t d, const double* __restrict__ x, const double* __restrict__ xs,
                           const double* __restrict__ yh, const double* __restrict__ yhs, const double* __restrict__ z,
                           const double* __restrict__ zs, const double* __restrict__ y, const double* __restrict__ ys,
                           double* part /* 6 x kBlockPartials */) {
    __shared__ double red[32];
    double a[6] = {0, 0, 0, 0, 0, 0};
    GRID_STRIDE(j, d) {
        const double dx = x[j] - xs[j], dyh = yh[j] - yhs[j], dz = z[j] - zs[j], dy = -(y[j] - ys[j]);
        a[0] += dx * dyh;
        a[1] += dx * dx;
        a[2] += dyh * dyh;
        a[3] += dz * dy;
        a[4] += dz * dz;
        a[5] += dy * dy;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const double t = block_sum(a[q], red);
        if (threadIdx.x == 0) part[q * kBlockPartials + blockIdx.x] = t;
    }
}

// Reduce `count` groups of `n` partials (group stride kBlockPartials) into out[count].
__global__ void k_reduce_groups(const double* part, int n, int count, double* out) {
    const int g = blockIdx.x;
    if (g >= count || threadIdx.x >= 32) return;
    const double v = reduce_partials(part + (int64_t)g * kBlockPartials, n);
    if (threadIdx.x == 0) out[g] = v;
}

// This rank's scalars of the iteration from the reduced worker partials (wred[6 i + 0..3] = primal^2,
// dual^2, |x|^2, |y|^2; wred[6 n] = |z|^2) and the F_i(z) values; fixed worker order.
__global__ void k_rank_stats(const double* __restrict__ wred, const double* __restrict__ fz, int n, int eval,
                             double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s[kStats] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < n; ++i) {
        const double* w = wred + 6 * i;
        const double prim = sqrt(w[0]), dual = sqrt(w[1]);
        s[kStSumX] += w[2];
        s[kStMaxY] = fmax(s[kStMaxY], w[3]);
        s[kStMaxPri] = (isnan(prim) || isnan(s[kStMaxPri])) ? NAN : fmax(s[kStMaxPri], prim);
        s[kStMaxDual] = (isnan(dual) || isnan(s[kStMaxDual])) ? NAN : fmax(s[kStMaxDual], dual);
        s[kStPriSq] += w[0];
        s[kStDualSq] += w[1];
        if (eval) s[kStF] += fz[i];
    }
    s[kStZZ] = wred[6 * n];
    for (int q = 0; q < kStats; ++q) out[q] = s[q];
}

// Hybrid spectral step of one side (the oracle's spectral_side).
__host__ __device__ inline bool spectral_side_dev(double ab, double aa, double bb, double eps_cor, double* est) {
    if (!(aa > 0.0) || !(bb > 0.0) || !(ab > 0.0)) return false;
    const double cor = ab / (sqrt(aa) * sqrt(bb));
    if (!(cor > eps_cor)) return false;
    const double sd = bb / ab, mg = ab / aa;
    *est = (2.0 * mg > sd) ? mg : sd - mg / 2.0;
    return true;
}

// Spectral penalty update of every local worker on the device (no host round trip): rho_i from the
// reduced secant dots wred[6 i .. 6 i + 5]; the solver parameters of the next iteration read rho_i.
__global__ void k_sps_rho(const double* __restrict__ wred, int n, double eps_cor, double rho_min, double rho_max,
                          double* __restrict__ rho) {
    const int i = threadIdx.x;
    if (blockIdx.x != 0 || i >= n) return;
    const double* w = wred + 6 * i;
    double ah = 0.0, bh = 0.0;
    const bool xo = spectral_side_dev(w[0], w[1], w[2], eps_cor, &ah);
    const bool zo = spectral_side_dev(w[3], w[4], w[5], eps_cor, &bh);
    double r = rho[i];
    if (xo && zo)
        r = sqrt(ah * bh);
    else if (xo)
        r = sqrt(ah);
    else if (zo)
        r = sqrt(bh);
    rho[i] = fmin(fmax(r, rho_min), rho_max);
}

template <typename T>
T* dalloc(int64_t n) {
    T* p = nullptr;
    NADMM_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)std::max<int64_t>(n, 1)));
    NADMM_CUDA(cudaMemset(p, 0, sizeof(T) * (size_t)std::max<int64_t>(n, 1)));
    return p;
}

struct RunBuffers {
    std::vector<void*> owned;
    template <typename T>
    T* get(int64_t n) {
        T* p = dalloc<T>(n);
        owned.push_back(p);
        return p;
    }
    ~RunBuffers() {
        for (void* p : owned) cudaFree(p);
    }
};

}  // namespace
}  // namespace nadmm

extern "C" {

void nadmm_admm_cfg_default(nadmm_admm_cfg* c) {  // inc/admm.hpp:37-56, 107-117
    std::memset(c, 0, sizeof *c);
    c->lambda = 1e-5;
    c->penalty_kind = 0;
    c->rho0 = 1.0;
    c->update_period = 2;
    c->eps_cor = 0.2;
    c->rho_min = 1e-6;
    c->rho_max = 1e6;
    c->eps_abs = 1e-3;
    c->eps_rel = 1e-3;
    c->max_outer_iters = 300;
    c->standard_norms = 0;
    c->inner_iters = 1;
    nadmm_newton_cfg_default(&c->newton);
    c->inner_solver = 0;
    nadmm_lbfgs_cfg_default(&c->lbfgs);
    c->eval_objective = 0;
    c->f_star = 0.0;
    c->theta_stop = 0.0;
}

extern const char* nadmm_last_error(void);

nadmm_status nadmm_comm_unique_id(uint8_t id_out[128]) {
    try {
        ncclUniqueId id;
        NADMM_NCCL(ncclGetUniqueId(&id));
        std::memcpy(id_out, id.internal, 128);
        return NADMM_OK;
    } catch (const Error& e) {
        return e.code;
    }
}

nadmm_status nadmm_comm_create(nadmm_ctx ctx, const uint8_t id[128], int32_t nranks, int32_t rank, nadmm_comm* out) {
    try {
        if (!ctx || !out) raise(NADMM_ECONFIG, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) raise(NADMM_ECONFIG, "bad rank/nranks");
        NADMM_CUDA(cudaSetDevice(ctx->device));
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, 128);
        auto* c = new nadmm_comm_s();
        c->nranks = nranks;
        c->rank = rank;
        c->ctx = ctx;
        ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            raise(NADMM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
        ctx->live++;
        *out = c;
        return NADMM_OK;
    } catch (const Error& e) {
        return e.code;
    }
}

nadmm_status nadmm_comm_destroy(nadmm_comm c) {
    if (!c) return NADMM_OK;
    if (c->comm) ncclCommDestroy(c->comm);
    Ctx* ctx = c->ctx;
    delete c;
    ctx_unref(ctx);
    return NADMM_OK;
}

}  // extern "C"

namespace nadmm {
void set_last_error(const std::string& m);

// Synchronise the stream of a collective-bearing step, failing fast instead of hanging when a peer
// dies or stalls (the reference's TransportError after per-phase timeouts, src/comm.cpp:182-191,
// 270-303): poll the stream and ncclCommGetAsyncError; after NADMM_COMM_TIMEOUT_MS (default 120 s)
// abort the communicator and raise NADMM_ETRANSPORT.
void comm_sync(cudaStream_t st, ncclComm_t comm) {
    static const long long timeout_ms = [] {
        const char* e = getenv("NADMM_COMM_TIMEOUT_MS");
        return e ? atoll(e) : 120000LL;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) NADMM_CUDA(q);
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
            ncclCommAbort(comm);
            raise(NADMM_ETRANSPORT, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
        }
        const long long ms =
            std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_ms > 0 && ms > timeout_ms) {
            ncclCommAbort(comm);
            raise(NADMM_ETRANSPORT, "consensus collective timed out after " + std::to_string(ms) +
                                        " ms (peer rank hung or dead)");
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    barrier_check();
}

// One consensus run (AdmmState + the run_admm loop); stepping lets callers time exact iteration
// windows (bench.py) while nadmm_admm_run drives it to completion.
//
// Per outer iteration: ONE collective and ONE host synchronisation.
//   * The consensus buffer [sum_i (rho_i x_i - y_i) | sum rho | per-rank scalar slots] is reduced by one
//     ncclAllReduce; the scalar slots carry the PREVIOUS iteration's rank scalars (residuals, norms,
//     F_i(z)) -- zero outside the rank's own slot, so the sum is a gather. With more than one rank an
//     iteration's metrics row, convergence and theta tests are therefore completed one iteration
//     later; when they stop the run at iteration k, the speculative iteration k+1 is discarded and
//     z^k (kept as prev_z) is restored. Each step() call ends with a flush of the last row's slots.
//   * rho_i lives on the device: the spectral penalty update runs as a kernel and
//     the solvers read rho_i from it, so no host round trip sits between the secant dots and the next
//     solve.
//   * consensus_tree: ncclAllGather of the per-worker terms instead of the sum; every
//     rank forms z with the oracle's ascending-id pairwise tree (bitwise identical for any rank count).
struct AdmmRun {
    std::vector<Shard*> shards;
    nadmm_comm comm = nullptr;
    nadmm_admm_cfg cfg{};
    nadmm_newton_cfg ncfg{};
    nadmm_lbfgs_cfg lcfg{};
    Ctx* ctx = nullptr;
    cudaStream_t st = nullptr;
    int64_t d = 0;
    int n_local = 0, n_total = 0, nranks = 1, rank = 0;
    bool sps = false, tree = false, deferred = false;
    RunBuffers rb;
    double *buf = nullptr, *gbuf = nullptr, *z = nullptr, *pz = nullptr, *zs = nullptr, *zpart = nullptr;
    double *wpart = nullptr, *wred = nullptr, *fz = nullptr, *rho_dev = nullptr;
    double *stats_cur = nullptr, *stats_prev = nullptr, *fslots = nullptr, *hbuf = nullptr;  // hbuf: pinned
    int64_t buf_len = 0, slot_off = 0;
    std::vector<double*> yh, xs, ys, yhs;
    std::vector<double> rho, rho_prev;
    int vg = 1;
    int k = 0, snap_it = 0;
    bool conv = false, stop = false;
    cudaEvent_t ev_start = nullptr, ev_now = nullptr;
    // a metrics row whose rank scalars arrive with the next collective (deferred mode)
    bool row_pending = false;
    nadmm_metrics_row pend{};
    nadmm_metrics_row* pend_out = nullptr;

    AdmmRun(const nadmm_shard* sh, int32_t nl, nadmm_comm c, const nadmm_admm_cfg* cfg_in) : comm(c), n_local(nl) {
        if (!sh || nl < 1 || nl > kMaxLocal) raise(NADMM_ECONFIG, "need 1..16 local shards");
        if (cfg_in)
            cfg = *cfg_in;
        else
            nadmm_admm_cfg_default(&cfg);
        if (cfg.rho0 <= 0.0) raise(NADMM_ECONFIG, "rho0 must be > 0");
        if (cfg.penalty_kind == 1 &&
            (cfg.update_period < 1 || !(cfg.eps_cor > 0.0 && cfg.eps_cor < 1.0) || !(cfg.rho_min > 0.0) ||
             cfg.rho_max < cfg.rho_min))
            raise(NADMM_ECONFIG, "bad spectral penalty policy");  // PenaltyPolicy::validate (inc/admm.hpp:37-47)
        if (cfg.inner_iters < 0) raise(NADMM_ECONFIG, "inner_iters must be >= 0");
        ncfg = cfg.newton;
        ncfg.newton_max_iters = cfg.inner_iters;
        validate_newton_cfg(ncfg);
        if (cfg.inner_solver != 0 && cfg.inner_solver != 1) raise(NADMM_ECONFIG, "inner_solver must be 0 or 1");
        lcfg = cfg.lbfgs;
        lcfg.max_iters = cfg.inner_iters;  // src/worker.cpp:184
        if (cfg.inner_solver == 1) validate_lbfgs_cfg(lcfg);
        for (int i = 0; i < nl; ++i) {
            if (!sh[i]) raise(NADMM_ECONFIG, "null shard");
            if (sh[i]->owner) raise(NADMM_ECONFIG, "shard is already bound to a live worker or ADMM session");
            for (int j = 0; j < i; ++j)
                if (sh[j] == sh[i]) raise(NADMM_ECONFIG, "the same shard is listed twice");
            shards.push_back(sh[i]);
        }
        ctx = shards[0]->ctx;
        d = shards[0]->d;
        for (Shard* s : shards) {
            if (s->ctx != ctx) raise(NADMM_ECONFIG, "all local shards must share one context");
            if (s->d != d) raise(NADMM_ECONFIG, "shard weight dimensions differ");
        }
        if (comm && comm->ctx->device != ctx->device) raise(NADMM_ECONFIG, "communicator bound to another device");
        NADMM_CUDA(cudaSetDevice(ctx->device));
        st = ctx->stream;
        nranks = comm ? comm->nranks : 1;
        rank = comm ? comm->rank : 0;
        n_total = n_local;
        tree = cfg.consensus_tree != 0;
        bool uniform = true;
        if (comm) {  // global worker count; workers are concatenated in rank order
            int* cnt = rb.get<int>(nranks);
            NADMM_CUDA(cudaMemcpyAsync(cnt + rank, &n_local, sizeof(int), cudaMemcpyHostToDevice, st));
            NADMM_NCCL(ncclAllGather(cnt + rank, cnt, 1, ncclInt, comm->comm, st));
            std::vector<int> h(nranks);
            NADMM_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(int) * nranks, cudaMemcpyDeviceToHost, st));
            comm_sync(st, comm->comm);
            n_total = 0;
            for (int v : h) {
                n_total += v;
                uniform = uniform && v == n_local;
            }
        }
        if (tree && (!uniform || n_total > 64))
            raise(NADMM_ECONFIG, "consensus_tree needs the same worker count on every rank and <= 64 workers");
        deferred = comm != nullptr;
        sps = cfg.penalty_kind == 1;
        if (tree) {  // per rank: n_local term vectors | n_local rho | kStats scalars
            buf_len = (int64_t)n_local * d + n_local + kStats;
            buf = rb.get<double>(buf_len);
            gbuf = rb.get<double>(buf_len * nranks);
            slot_off = (int64_t)n_local * d + n_local;
        } else {
            buf_len = d + 1 + (int64_t)kStats * nranks;
            buf = rb.get<double>(buf_len);
            slot_off = d + 1;
        }
        z = rb.get<double>(d);
        pz = rb.get<double>(d);
        zs = sps ? rb.get<double>(d) : nullptr;
        vg = vec_grid(*ctx, d);
        zpart = rb.get<double>(kBlockPartials);
        wpart = rb.get<double>((int64_t)n_local * 6 * kBlockPartials);
        wred = rb.get<double>((int64_t)n_local * 6 + 2);
        fz = rb.get<double>(n_local);
        rho_dev = rb.get<double>(n_local);
        stats_cur = rb.get<double>(kStats);
        stats_prev = rb.get<double>(kStats);
        fslots = rb.get<double>((int64_t)kStats * nranks);
        NADMM_CUDA(cudaMallocHost(&hbuf, sizeof(double) * (size_t)(kStats * (nranks + 1) + n_local)));
        yh.assign(n_local, nullptr);
        xs.assign(n_local, nullptr);
        ys.assign(n_local, nullptr);
        yhs.assign(n_local, nullptr);
        for (int i = 0; i < n_local; ++i) {
            if (sps) {
                yh[i] = rb.get<double>(d);
                xs[i] = rb.get<double>(d);
                ys[i] = rb.get<double>(d);
                yhs[i] = rb.get<double>(d);
            }
            // AdmmState::initial: x_local = 0, y_i = 0 (src/worker.cpp:135)
            Shard& s = *shards[i];
            NADMM_CUDA(cudaMemsetAsync(s.x, 0, sizeof(double) * d, st));
            NADMM_CUDA(cudaMemsetAsync(s.y, 0, sizeof(double) * d, st));
            if (s.cache_at == Shard::kAtX) s.cache_at = Shard::kNone;
        }
        rho.assign(n_local, cfg.rho0);
        rho_prev = rho;
        NADMM_CUDA(cudaMemcpyAsync(rho_dev, rho.data(), sizeof(double) * n_local, cudaMemcpyHostToDevice, st));
        for (int i = 0; i < n_local; ++i) {
            shards[i]->rho_src = rho_dev + i;  // the worker solves read rho_i from the device
            shards[i]->owner = this;
        }
        NADMM_CUDA(cudaEventCreate(&ev_start));
        NADMM_CUDA(cudaEventCreate(&ev_now));
        NADMM_CUDA(cudaEventRecord(ev_start, st));
        stream_sync(st);
    }

    ~AdmmRun() {
        for (Shard* s : shards) {
            if (s->owner == this) s->owner = nullptr;
            s->rho_src = nullptr;
        }
        if (hbuf) cudaFreeHost(hbuf);
        if (ev_start) cudaEventDestroy(ev_start);
        if (ev_now) cudaEventDestroy(ev_now);
    }

    void sync() {
        if (comm)
            comm_sync(st, comm->comm);
        else
            stream_sync(st);
    }

    // Rank scalars of all ranks (rank order) -> the row's norms / tolerances / F; returns conv and
    // fills theta. `h` holds nranks x kStats scalars.
    bool finish_row(const double* h, nadmm_metrics_row& m) {
        double sx = 0.0, ymax = 0.0, pmax = 0.0, dmax = 0.0, psq = 0.0, dsq = 0.0, F = 0.0;
        for (int r = 0; r < nranks; ++r) {  // rank order: deterministic combination
            const double* s = h + (size_t)r * kStats;
            sx += s[kStSumX];
            ymax = std::max(ymax, s[kStMaxY]);
            pmax = std::max(pmax, s[kStMaxPri]);
            dmax = std::max(dmax, s[kStMaxDual]);
            psq += s[kStPriSq];
            dsq += s[kStDualSq];
            F += s[kStF];
            if (std::isnan(s[kStMaxPri]) || std::isnan(s[kStMaxDual])) pmax = NAN;
        }
        const double zz = h[kStZZ];
        // tolerances, squared norms unless standard_norms
        double a = sx, b = n_total * zz, c = ymax;
        if (cfg.standard_norms) {
            a = std::sqrt(sx);
            b = std::sqrt((double)n_total) * std::sqrt(zz);
            c = std::sqrt(ymax);
        }
        const double eps_pri = std::sqrt((double)n_total) * cfg.eps_abs + cfg.eps_rel * std::max(a, b);
        const double eps_dual = std::sqrt((double)d) * cfg.eps_abs + cfg.eps_rel * c;
        const double Fz = cfg.eval_objective ? F + 0.5 * cfg.lambda * zz : NAN;
        m.train_objective = Fz;
        m.theta = (cfg.eval_objective && cfg.f_star > 0.0) ? (Fz - cfg.f_star) / cfg.f_star : NAN;
        m.primal_norm = std::sqrt(psq);
        m.dual_norm = std::sqrt(dsq);
        m.eps_pri = eps_pri;
        m.eps_dual = eps_dual;
        return m.iteration >= 1 && pmax <= eps_pri && dmax <= eps_dual;  // has_converged
    }

    bool stops(const nadmm_metrics_row& m, bool c) const {
        if (c && !cfg.ignore_convergence) return true;
        if (cfg.theta_stop > 0.0 && !std::isnan(m.theta) && m.theta <= cfg.theta_stop) return true;
        return false;
    }

    // A deferred row's scalars arrived (gathered slots `h`): complete it; on a stop at its iteration,
    // drop the speculative iteration that already ran (restore z^k and its penalties).
    void complete_pending(const double* h, bool speculative_ran) {
        const bool c = finish_row(h, pend);
        if (pend_out) *pend_out = pend;
        row_pending = false;
        conv = c;
        if (stops(pend, c)) {
            stop = true;
            if (speculative_ran) {
                NADMM_CUDA(cudaMemcpyAsync(z, pz, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
                rho = rho_prev;
                k = pend.iteration;
            }
        }
    }

    // One outer iteration (solve, gather, z, y, penalty, metrics). In deferred mode the
    // row lands in `row` when the next collective (or flush) brings its rank scalars.
    void iterate(nadmm_metrics_row* row) {
        int inner = 0, cg_sum = 0, fe_sum = 0, flags = 0;
        std::vector<char> pending(n_local, 0);
        // node group: all local nodes' Newton iterations as one graph of whole-GPU group passes
        bool grouped = cfg.inner_solver == 0 && cfg.inner_iters == 1 && group_eligible(shards);
        if (grouped) {
            for (Shard* s : shards) NADMM_CUDA(cudaMemcpyAsync(s->z, z, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
            grouped = group_solve_launch(shards, ncfg, rho.data());
            if (grouped)
                for (int i = 0; i < n_local; ++i) {
                    solve_readback_async(*shards[i]);
                    pending[i] = 3;
                }
        }
        // concurrent nodes: node i's solve on node_stream[i % k] (forked from / joined back to st)
        bool conc = !grouped && ctx->node_streams > 1 && cfg.inner_solver == 0 && n_local > 1;
        for (int i = 0; conc && i < n_local; ++i) conc = dmma_supported(*shards[i]);
        const int ks = conc ? std::min(ctx->node_streams, n_local) : 1;
        if (!grouped)
            for (int i = 0; i < n_local; ++i) use_layout_split(*shards[i], ks);
        if (conc) {
            NADMM_CUDA(cudaEventRecord(ctx->node_fork, st));
            for (int k2 = 0; k2 < ks; ++k2) NADMM_CUDA(cudaStreamWaitEvent(ctx->node_stream[k2], ctx->node_fork, 0));
        }
        for (int i = 0; i < n_local && !grouped; ++i) {  // (1) scatter z / solve (workers enqueued back to back)
            Shard& s = *shards[i];
            if (conc) {
                ctx->stream = ctx->node_stream[i % ks];
                NADMM_CUDA(cudaMemcpyAsync(s.z, z, sizeof(double) * d, cudaMemcpyDeviceToDevice, ctx->stream));
                try {
                    pending[i] = !solve_launch(s, ncfg, 0.0, true, rho[i], cfg.inner_iters);
                    if (pending[i]) {
                        solve_readback_async(s);
                        pending[i] = 3;  // readback enqueued on the node stream
                    }
                } catch (...) {
                    ctx->stream = st;
                    throw;
                }
                ctx->stream = st;
                continue;
            }
            NADMM_CUDA(cudaMemcpyAsync(s.z, z, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
            if (cfg.inner_solver == 1) {  // L-BFGS: host-driven line search, synchronous per worker
                const nadmm_inner_stats lst = lbfgs_inner_stats(device_lbfgs_solve(s, lcfg, 0.0, true, rho[i]));
                inner += (int)lst.inner_iters;
                fe_sum += (int)lst.fn_evals;
                flags |= (int)lst.flags;
                pending[i] = 2;
                continue;
            }
            pending[i] = !solve_launch(s, ncfg, 0.0, true, rho[i], cfg.inner_iters);
        }
        // the workers' inner stats come back with the iteration's single synchronisation below
        for (int i = 0; i < n_local; ++i)
            if (pending[i] == 1) solve_readback_async(*shards[i]);
        if (conc)
            for (int k2 = 0; k2 < ks; ++k2) {
                NADMM_CUDA(cudaEventRecord(ctx->node_join[k2], ctx->node_stream[k2]));
                NADMM_CUDA(cudaStreamWaitEvent(st, ctx->node_join[k2], 0));
            }
        LocalPtrs lp{};  // (2) consensus buffer + the iteration's one collective
        lp.n = n_local;
        for (int i = 0; i < n_local; ++i) {
            lp.x[i] = shards[i]->x;
            lp.y[i] = shards[i]->y;
        }
        const double* slots_prev = (deferred && k >= 1) ? stats_prev : nullptr;
        if (tree) {
            k_local_terms<<<vg, 256, 0, st>>>(d, lp, rho_dev, buf, slots_prev);
            NADMM_LAUNCH_CHECK();
            if (comm)
                NADMM_NCCL(ncclAllGather(buf, gbuf, (size_t)buf_len, ncclDouble, comm->comm, st));
            else
                NADMM_CUDA(cudaMemcpyAsync(gbuf, buf, sizeof(double) * buf_len, cudaMemcpyDeviceToDevice, st));
            k_tree_z<<<vg, 256, 0, st>>>(d, gbuf, n_local, nranks, cfg.lambda, z, pz, zpart);  // (3) z
        } else {
            k_local_sum<<<vg, 256, 0, st>>>(d, lp, rho_dev, buf, slots_prev, rank, nranks);
            NADMM_LAUNCH_CHECK();
            if (comm) NADMM_NCCL(ncclAllReduce(buf, buf, (size_t)buf_len, ncclDouble, ncclSum, comm->comm, st));
            k_z_update<<<vg, 256, 0, st>>>(d, buf, cfg.lambda, z, pz, zpart);  // (3) z, y, residual partials
        }
        NADMM_LAUNCH_CHECK();
        ctx->stats.kernel_launches += 2;
        for (int i = 0; i < n_local; ++i) {
            Shard& s = *shards[i];
            k_worker_update<<<vg, 256, 0, st>>>(d, rho_dev + i, s.x, s.y, sps ? yh[i] : nullptr, z, pz,
                                                wpart + (int64_t)i * 6 * kBlockPartials, tree ? 1 : 0);
            NADMM_LAUNCH_CHECK();
            ctx->stats.kernel_launches++;
        }
        ++k;
        if (cfg.eval_objective) {  // F_i(z) of the global objective (Eq. (5)) for the metrics stream
            if (conc) {  // the value passes of the nodes run concurrently like their solves
                NADMM_CUDA(cudaEventRecord(ctx->node_fork, st));
                for (int k2 = 0; k2 < ks; ++k2)
                    NADMM_CUDA(cudaStreamWaitEvent(ctx->node_stream[k2], ctx->node_fork, 0));
            }
            for (int i = 0; i < n_local; ++i) {
                ctx->stream = conc ? ctx->node_stream[i % ks] : st;
                try {
                    op_value(*shards[i], z, fz + i, 0, nullptr);
                } catch (...) {
                    ctx->stream = st;
                    throw;
                }
                ctx->stream = st;
            }
            if (conc)
                for (int k2 = 0; k2 < ks; ++k2) {
                    NADMM_CUDA(cudaEventRecord(ctx->node_join[k2], ctx->node_stream[k2]));
                    NADMM_CUDA(cudaStreamWaitEvent(st, ctx->node_join[k2], 0));
                }
        }
        for (int i = 0; i < n_local; ++i) {
            k_reduce_groups<<<4, 32, 0, st>>>(wpart + (int64_t)i * 6 * kBlockPartials, vg, 4, wred + (int64_t)i * 6);
            ctx->stats.kernel_launches++;
        }
        k_reduce_groups<<<1, 32, 0, st>>>(zpart, vg, 1, wred + (int64_t)n_local * 6);
        k_rank_stats<<<1, 32, 0, st>>>(wred, fz, n_local, cfg.eval_objective, stats_cur);
        ctx->stats.kernel_launches += 2;
        NADMM_LAUNCH_CHECK();
        NADMM_CUDA(cudaEventRecord(ev_now, st));  // z^k and F(z^k) are complete: the row's wall time
        rho_prev = rho;
        if (sps && k - snap_it >= cfg.update_period) spectral();  // (4) SPS against the last snapshot (device)
        // (5) the single readback: this rank's scalars of k, the gathered slots of k-1, rho after SPS
        NADMM_CUDA(cudaMemcpyAsync(hbuf, stats_cur, sizeof(double) * kStats, cudaMemcpyDeviceToHost, st));
        if (deferred && k >= 2) {
            if (tree)
                for (int r = 0; r < nranks; ++r)
                    NADMM_CUDA(cudaMemcpyAsync(hbuf + (size_t)(r + 1) * kStats, gbuf + (int64_t)r * buf_len + slot_off,
                                               sizeof(double) * kStats, cudaMemcpyDeviceToHost, st));
            else
                NADMM_CUDA(cudaMemcpyAsync(hbuf + kStats, buf + slot_off, sizeof(double) * kStats * nranks,
                                           cudaMemcpyDeviceToHost, st));
        }
        NADMM_CUDA(cudaMemcpyAsync(hbuf + kStats * (nranks + 1), rho_dev, sizeof(double) * n_local,
                                   cudaMemcpyDeviceToHost, st));
        if (deferred)
            NADMM_CUDA(cudaMemcpyAsync(stats_prev, stats_cur, sizeof(double) * kStats, cudaMemcpyDeviceToDevice, st));
        sync();
        for (int i = 0; i < n_local; ++i) {  // gather the workers' inner stats
            Shard& s = *shards[i];
            if (pending[i] == 2) continue;  // L-BFGS stats already gathered
            SolveResult r = pending[i] ? solve_result(s, ncfg) : solve_collect(s, ncfg, false);  // 1 and 3
            if (r.error) raise((nadmm_status)r.error, "worker inner solve failed");
            inner += r.iterations;
            cg_sum += r.cg_sum;
            fe_sum += r.fe_sum;
            flags |= r.flags;
        }
        if (grouped) group_timers_finish(*ctx);
        for (int i = 0; i < n_local; ++i) rho[i] = hbuf[kStats * (nranks + 1) + i];
        float ms = 0.f;
        NADMM_CUDA(cudaEventElapsedTime(&ms, ev_start, ev_now));
        nadmm_metrics_row m{};
        m.iteration = k;
        m.wall_seconds = ms * 1e-3;
        m.inner_iterations = inner;
        m.cg_iters = cg_sum;
        m.fn_evals = fe_sum;
        m.flags = flags;
        double rsum = 0.0;
        for (double v : rho) rsum += v;
        m.rho_mean = rsum / n_local;
        m.messages = 2LL * n_total * k;
        if (deferred) {
            if (row_pending) complete_pending(hbuf + kStats, true);  // row k-1
            if (stop) return;  // iteration k was speculative and is dropped
            pend = m;
            pend_out = row;
            row_pending = true;
        } else {
            const bool c = finish_row(hbuf, m);
            if (row) *row = m;
            conv = c;
            if (stops(m, c)) stop = true;
        }
        if (k >= cfg.max_outer_iters) stop = true;
    }

    // Deferred mode: gather the last iteration's rank scalars (a small allreduce of the slots only)
    // and complete its row.
    void flush() {
        if (!deferred || !row_pending) return;
        k_fill_slots<<<1, 32, 0, st>>>(fslots, stats_prev, rank, nranks);
        NADMM_LAUNCH_CHECK();
        NADMM_NCCL(ncclAllReduce(fslots, fslots, (size_t)kStats * nranks, ncclDouble, ncclSum, comm->comm, st));
        NADMM_CUDA(cudaMemcpyAsync(hbuf + kStats, fslots, sizeof(double) * kStats * nranks, cudaMemcpyDeviceToHost, st));
        sync();
        complete_pending(hbuf + kStats, false);
    }

    void spectral() {
        for (int i = 0; i < n_local; ++i) {
            Shard& s = *shards[i];
            double* part = wpart + (int64_t)i * 6 * kBlockPartials;
            k_sps_dots<<<vg, 256, 0, st>>>(d, s.x, xs[i], yh[i], yhs[i], z, zs, s.y, ys[i], part);
            k_reduce_groups<<<6, 32, 0, st>>>(part, vg, 6, wred + (int64_t)i * 6);
            ctx->stats.kernel_launches += 2;
        }
        k_sps_rho<<<1, 32, 0, st>>>(wred, n_local, cfg.eps_cor, cfg.rho_min, cfg.rho_max, rho_dev);
        ctx->stats.kernel_launches++;
        NADMM_LAUNCH_CHECK();
        for (int i = 0; i < n_local; ++i) {
            Shard& s = *shards[i];
            NADMM_CUDA(cudaMemcpyAsync(xs[i], s.x, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
            NADMM_CUDA(cudaMemcpyAsync(ys[i], s.y, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
            NADMM_CUDA(cudaMemcpyAsync(yhs[i], yh[i], sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
        }
        NADMM_CUDA(cudaMemcpyAsync(zs, z, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
        snap_it = k;
    }

    // Runs up to n outer iterations; returns the number of iterations kept (= metrics rows written).
    int step(int n, nadmm_metrics_row* rows, int row_cap) {
        const int k0 = k;
        int done = 0;
        while (done < n && !stop) {
            iterate(rows && done < row_cap ? rows + done : nullptr);
            ++done;
        }
        flush();
        return k - k0;  // a deferred stop drops the speculative iteration
    }

    void result(double* z_out, double* rho_out) {
        if (z_out) NADMM_CUDA(cudaMemcpyAsync(z_out, z, sizeof(double) * d, cudaMemcpyDeviceToHost, st));
        stream_sync(st);
        if (rho_out)
            for (int i = 0; i < n_local; ++i) rho_out[i] = rho[i];
    }
};

}  // namespace nadmm

struct nadmm_admm_s : nadmm::AdmmRun {
    using AdmmRun::AdmmRun;
};

extern "C" {

nadmm_status nadmm_admm_create(const nadmm_shard* shards, int32_t n_local, nadmm_comm comm, const nadmm_admm_cfg* cfg,
                               nadmm_admm* out) {
    try {
        if (!out) raise(NADMM_ECONFIG, "null output");
        (void)cudaGetLastError();
        *out = new nadmm_admm_s(shards, n_local, comm, cfg);
        for (Shard* s : (*out)->shards) shard_hold(s);
        return NADMM_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    }
}

nadmm_status nadmm_admm_step(nadmm_admm run, int32_t n_iters, nadmm_metrics_row* rows, int32_t row_cap,
                             int32_t* done, int32_t* finished) {
    try {
        if (!run) raise(NADMM_ECONFIG, "null run");
        (void)cudaGetLastError();  // clear stale errors left by other libraries in this thread
        NADMM_CUDA(cudaSetDevice(run->ctx->device));
        const int n = run->step(n_iters, rows, row_cap);
        if (done) *done = n;
        if (finished) *finished = run->stop ? 1 : 0;
        return NADMM_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    }
}

nadmm_status nadmm_admm_result(nadmm_admm run, double* z_out, double* rho_out, int32_t* iterations,
                               int32_t* converged) {
    try {
        if (!run) raise(NADMM_ECONFIG, "null run");
        (void)cudaGetLastError();  // clear stale errors left by other libraries in this thread
        NADMM_CUDA(cudaSetDevice(run->ctx->device));
        run->result(z_out, rho_out);
        if (iterations) *iterations = run->k;
        if (converged) *converged = run->conv ? 1 : 0;
        return NADMM_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    }
}

nadmm_status nadmm_admm_free(nadmm_admm run) {
    if (!run) return NADMM_OK;
    const std::vector<Shard*> held = run->shards;
    delete run;
    for (Shard* s : held) shard_unhold(s);
    return NADMM_OK;
}

nadmm_status nadmm_sgd_run(const nadmm_shard* shards, int32_t n_local, nadmm_comm comm, const nadmm_sgd_cfg* cfg,
                           double lambda, double* x_inout, nadmm_metrics_row* rows, int32_t row_cap,
                           int32_t* epochs_done) {
    try {
        if (!shards || n_local < 1) raise(NADMM_ECONFIG, "sync_sgd needs at least one shard");
        if (!cfg || !x_inout) raise(NADMM_ECONFIG, "cfg and x_inout required");
        if (!(cfg->eta > 0.0)) raise(NADMM_ECONFIG, "sgd step size must be > 0");
        if (cfg->epochs < 0) raise(NADMM_ECONFIG, "sgd epochs must be >= 0");
        std::vector<Shard*> sh;
        for (int i = 0; i < n_local; ++i) {
            if (!shards[i]) raise(NADMM_ECONFIG, "null shard");
            sh.push_back(shards[i]);
        }
        Ctx* ctx = sh[0]->ctx;
        for (Shard* s : sh)
            if (s->ctx != ctx) raise(NADMM_ECONFIG, "all local shards must share one context");
        (void)cudaGetLastError();
        NADMM_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        const int64_t d = sh[0]->d;
        double* x = nullptr;
        double* hb = nullptr;
        NADMM_CUDA(cudaMalloc(&x, sizeof(double) * (size_t)d));
        NADMM_CUDA(cudaMalloc(&hb, sizeof(double) * 8));
        struct Free {
            double* a;
            double* b;
            ~Free() {
                cudaFree(a);
                cudaFree(b);
            }
        } fr{x, hb};
        NADMM_CUDA(cudaMemcpyAsync(x, x_inout, sizeof(double) * (size_t)d, cudaMemcpyHostToDevice, st));
        SgdReduce red;
        if (comm) {
            red.dev = [&](double* v, int64_t n) {
                NADMM_NCCL(ncclAllReduce(v, v, (size_t)n, ncclDouble, ncclSum, comm->comm, st));
            };
            red.host = [&](double* v, int n) {
                NADMM_CUDA(cudaMemcpyAsync(hb, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
                NADMM_NCCL(ncclAllReduce(hb, hb, (size_t)n, ncclDouble, ncclSum, comm->comm, st));
                NADMM_CUDA(cudaMemcpyAsync(v, hb, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
                stream_sync(st);
            };
        }
        const SgdOutcome o = sgd_run(sh, comm ? &red : nullptr, *cfg, lambda, x, rows, row_cap);
        NADMM_CUDA(cudaMemcpyAsync(x_inout, x, sizeof(double) * (size_t)d, cudaMemcpyDeviceToHost, st));
        stream_sync(st);
        if (epochs_done) *epochs_done = o.epochs;
        return NADMM_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    }
}

nadmm_status nadmm_admm_run(const nadmm_shard* shards, int32_t n_local, nadmm_comm comm, const nadmm_admm_cfg* cfg,
                            double* z_out, double* rho_out, nadmm_metrics_row* rows, int32_t row_cap,
                            int32_t* iterations, int32_t* converged) {
    nadmm_admm run = nullptr;
    nadmm_status rc = nadmm_admm_create(shards, n_local, comm, cfg, &run);
    if (rc) return rc;
    rc = nadmm_admm_step(run, run->cfg.max_outer_iters, rows, row_cap, nullptr, nullptr);
    if (!rc) rc = nadmm_admm_result(run, z_out, rho_out, iterations, converged);
    nadmm_admm_free(run);
    return rc;
}

}  // extern "C"
