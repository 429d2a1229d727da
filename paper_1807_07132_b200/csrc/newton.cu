// Composite data-pass ops and the device-resident inexact Newton-CG driver.
//
// newton_solve (src/newton.cpp:73-132) runs entirely on the device: one CUDA graph per Newton
// iteration (CG with device-side stop flags, certificate Hv, fallbacks, batched Armijo search,
// step, fused cache+gradient pass at the new point), replayed per iteration. The host synchronises
// once per Newton iteration (once per outer ADMM iteration with inner_iters = 1).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "solver.h"
#include "solver_kernels.h"

namespace nadmm {

__global__ void k_copy_rho(const double* src, DevParams* prm) { prm->rho = *src; }

// ---- grid-barrier watchdog registry (common.cuh) ----
namespace {
std::vector<BarrierTU>& barrier_tus() {
    static std::vector<BarrierTU> v;
    return v;
}
}  // namespace

void barrier_register(BarrierTU tu) { barrier_tus().push_back(tu); }

void barrier_configure() {
    unsigned long long ms = 60000;  // watchdog bound; 0 disables it
    if (const char* e = getenv("NADMM_BARRIER_TIMEOUT_MS")) ms = strtoull(e, nullptr, 10);
    for (const BarrierTU& tu : barrier_tus()) tu.set_timeout(ms * 1000000ull);
}

void barrier_check() {
    bool fault = false;
    for (const BarrierTU& tu : barrier_tus()) fault = tu.take_fault() != 0 || fault;
    if (fault)
        raise(NADMM_ECUDA, "grid barrier timed out (persistent grid not co-resident, or a hung peer); results of "
                           "the last launch are invalid");
}

void stream_sync(cudaStream_t st) {
    NADMM_CUDA(cudaStreamSynchronize(st));
    barrier_check();
}


// ---------------------------------------------------------------------------------------------
// Composite ops (one or two data passes each)
// ---------------------------------------------------------------------------------------------
// The single-pass fused kernels (X read once per product, split-K partials per block / cluster):
// the small-p row-per-thread kernel, else the DMMA cluster kernel; otherwise the SIMT two-pass path.
bool fused_supported(const Shard& s) { return smallp_supported(s) || dmma_supported(s) || gemm_supported(s); }

void fused_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    if (smallp_supported(s))
        smallp_pass(s, mode, W, guard);
    else if (dmma_supported(s))
        dmma_pass(s, mode, W, guard);
    else
        gemm_pass(s, mode, W, guard);
}

void op_cache_grad(Shard& s, const double* w, const int32_t* guard) {
    if (fused_supported(s)) {
        fused_pass(s, kModeCache, w, guard);
        finalize_partials(s, s.last_chunks,kXtuGrad, w, s.gbase, nullptr, 0, guard, nullptr);
    } else {
        rows_pass(s, kModeCache, w, guard);
        xtu_pass(s, kXtuGrad, w, s.gbase, nullptr, 0, guard);
    }
    loss_finalize(s, w, 1, s.scal + 0, guard);
}

int op_cache_split(Shard& s, const double* w, const int32_t* guard) {
    if (fused_supported(s)) {
        fused_pass(s, kModeCache, w, guard);
        return s.last_chunks;
    }
    rows_pass(s, kModeCache, w, guard);
    xtu_pass(s, kXtuGrad, w, s.gbase, nullptr, 0, guard);
    return 0;
}

void tl_mark(Shard& s, const char* name) {
    if (!s.tl_capture) return;
    const size_t i = s.tl_names.size();
    if (i >= s.tl_events.size()) {
        cudaEvent_t e;
        NADMM_CUDA(cudaEventCreate(&e));
        s.tl_events.push_back(e);
    }
    NADMM_CUDA(cudaEventRecordWithFlags(s.tl_events[i], s.ctx->stream, cudaEventRecordExternal));
    s.tl_names.push_back(name);
}

int op_hv(Shard& s, const double* v, double* out, const double* dotvec, int dot_slot, const int32_t* guard) {
    HvTimer* tm = (s.capture_timing && s.hv_timer_site >= 0 && s.hv_timer_site < (int)s.hv_timers.size())
                      ? &s.hv_timers[s.hv_timer_site]
                      : nullptr;
    if (tm) NADMM_CUDA(cudaEventRecordWithFlags(tm->start, s.ctx->stream, cudaEventRecordExternal));
    int g = 0;
    if (fused_supported(s)) {
        fused_pass(s, kModeHv, v, guard);
        if (tm) NADMM_CUDA(cudaEventRecordWithFlags(tm->stop, s.ctx->stream, cudaEventRecordExternal));
        tl_mark(s, "hv_fused_pass");
        finalize_partials(s, s.last_chunks, kXtuHv, v, out, dotvec, dot_slot, guard, &g);
        tl_mark(s, "hv_finalize");
    } else {
        rows_pass(s, kModeHv, v, guard);
        tl_mark(s, "hv_rows_pass");
        g = xtu_pass(s, kXtuHv, v, out, dotvec, dot_slot, guard);
        if (tm) NADMM_CUDA(cudaEventRecordWithFlags(tm->stop, s.ctx->stream, cudaEventRecordExternal));
        tl_mark(s, "hv_xtu_pass");
    }
    return g;
}

int op_hv_split(Shard& s, const double* v, double* out, const double* dotvec, int dot_slot, const int32_t* guard,
                int* chunks) {
    *chunks = 0;
    if (!fused_supported(s)) return op_hv(s, v, out, dotvec, dot_slot, guard);
    HvTimer* tm = (s.capture_timing && s.hv_timer_site >= 0 && s.hv_timer_site < (int)s.hv_timers.size())
                      ? &s.hv_timers[s.hv_timer_site]
                      : nullptr;
    if (tm) NADMM_CUDA(cudaEventRecordWithFlags(tm->start, s.ctx->stream, cudaEventRecordExternal));
    fused_pass(s, kModeHv, v, guard);
    if (tm) NADMM_CUDA(cudaEventRecordWithFlags(tm->stop, s.ctx->stream, cudaEventRecordExternal));
    tl_mark(s, "hv_fused_pass");
    *chunks = s.last_chunks;
    return 0;
}

void op_lp(Shard& s, const double* p, const int32_t* guard) {
    if (fused_supported(s))
        fused_pass(s, kModeLp, p, guard);
    else
        rows_pass(s, kModeLp, p, guard);
}

void op_value(Shard& s, const double* w, double* dst, int add_ridge, const int32_t* guard) {
    if (fused_supported(s))
        fused_pass(s, kModeValue, w, guard);
    else
        rows_pass(s, kModeValue, w, guard);
    loss_finalize(s, w, add_ridge, dst, guard);
}

void op_predict(Shard& s, const double* w) {
    if (smallp_supported(s))
        smallp_pass(s, kModePredict, w, nullptr);
    else if (!dmma_supported(s) && gemm_supported(s))
        gemm_pass(s, kModePredict, w, nullptr);
    else
        rows_pass(s, kModePredict, w, nullptr);
}

// ---------------------------------------------------------------------------------------------
// Solver driver
// ---------------------------------------------------------------------------------------------
void validate_newton_cfg(const nadmm_newton_cfg& c) {  // NewtonConfig::validate (src/newton.cpp:8-17)
    if (c.cg_tol <= 0.0 || c.cg_tol >= 1.0) raise(NADMM_ECONFIG, "cg_tol must lie in (0,1)");
    if (c.armijo_beta <= 0.0 || c.armijo_beta >= 1.0) raise(NADMM_ECONFIG, "armijo_beta must lie in (0,1)");
    if (c.backtrack_gamma <= 0.0 || c.backtrack_gamma >= 1.0) raise(NADMM_ECONFIG, "backtrack_gamma must lie in (0,1)");
    if (c.cg_max_iters < 1) raise(NADMM_ECONFIG, "cg_max_iters must be >= 1");
    if (c.ls_max_iters < 0) raise(NADMM_ECONFIG, "ls_max_iters must be >= 0");
    if (c.newton_max_iters < 0) raise(NADMM_ECONFIG, "newton_max_iters must be >= 0");
    if (c.grad_tol < 0.0) raise(NADMM_ECONFIG, "grad_tol must be >= 0");
    if (c.cg_max_iters > kMaxCg) raise(NADMM_ECONFIG, "cg_max_iters exceeds the device solver limit (256)");
    if (c.ls_max_iters > kMaxLs) raise(NADMM_ECONFIG, "ls_max_iters exceeds the device solver limit (62)");
}

void set_params(Shard& s, const nadmm_newton_cfg& c, double lambda, bool aug, double rho) {
    DevParams h{};
    h.lambda = lambda;
    h.rho = aug ? rho : 0.0;
    h.augmented = aug ? 1 : 0;
    h.cg_max_iters = c.cg_max_iters;
    h.cg_tol = c.cg_tol;
    h.armijo_beta = c.armijo_beta;
    h.backtrack_gamma = c.backtrack_gamma;
    h.ls_max_iters = c.ls_max_iters;
    h.grad_tol = c.grad_tol;
    *s.prm_host = h;
    NADMM_CUDA(cudaMemcpyAsync(s.prm, s.prm_host, sizeof(DevParams), cudaMemcpyHostToDevice, s.ctx->stream));
    if (aug && s.rho_src) {  // ADMM session: rho_i comes from the device-side penalty update
        k_copy_rho<<<1, 1, 0, s.ctx->stream>>>(s.rho_src, s.prm);
        NADMM_LAUNCH_CHECK();
    }
}

void set_lambda_only(Shard& s, double lambda) {
    DevParams h = *s.prm_host;
    h.lambda = lambda;
    h.augmented = 0;
    h.rho = 0.0;
    *s.prm_host = h;
    NADMM_CUDA(cudaMemcpyAsync(s.prm, s.prm_host, sizeof(DevParams), cudaMemcpyHostToDevice, s.ctx->stream));
}

void ensure_cache_at_x(Shard& s, double lambda) {
    if (s.cache_at == Shard::kAtX && s.cache_lambda == lambda) return;
    op_cache_grad(s, s.x, nullptr);
    s.cache_at = Shard::kAtX;
    s.cache_lambda = lambda;
}

static void destroy_graphs(Shard& s) {
    if (s.g_iter) cudaGraphExecDestroy(s.g_iter);
    s.g_iter = nullptr;
    s.g_cg_max = s.g_ls_max = -1;
}

void invalidate_graphs(Shard& s) { destroy_graphs(s); }

static void capture_iteration_graph(Shard& s, int cg_max, int ls_max) {
    if (s.g_iter && s.g_cg_max == cg_max && s.g_ls_max == ls_max && s.g_timing == s.ctx->timing) return;
    destroy_graphs(s);
    cudaStream_t st = s.ctx->stream;
    const nadmm_stats saved = s.ctx->stats;
    s.ensure_timers(s.ctx->timing ? cg_max + 1 : 0);
    cudaGraph_t graph = nullptr;
    NADMM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
        s.capture_timing = s.ctx->timing;
        static const bool tl = getenv("NADMM_GRAPH_TIMELINE") != nullptr;
        s.tl_capture = tl;
        s.tl_names.clear();
        tl_mark(s, "start");
        launch_newton_iteration(s, cg_max, ls_max);
        s.capture_timing = false;
        s.tl_capture = false;
    } catch (...) {
        s.capture_timing = false;
        s.tl_capture = false;
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    NADMM_CUDA(cudaStreamEndCapture(st, &graph));
    s.g_nodes = s.ctx->stats.kernel_launches - saved.kernel_launches;
    s.ctx->stats = saved;
    NADMM_CUDA(cudaGraphInstantiate(&s.g_iter, graph, 0));
    cudaGraphDestroy(graph);
    s.g_cg_max = cg_max;
    s.g_ls_max = ls_max;
    s.g_timing = s.ctx->timing;
}

// Reads back the solver state and trace (one async copy each, one sync); accumulates the Hv timers
// of the Hv passes that actually ran.
void solve_readback_async(Shard& s) {
    NADMM_CUDA(cudaMemcpyAsync(s.st_host, s.st, sizeof(DevState), cudaMemcpyDeviceToHost, s.ctx->stream));
    NADMM_CUDA(cudaMemcpyAsync(s.trace_host, s.trace, sizeof(DevTrace) * kTraceCap, cudaMemcpyDeviceToHost,
                               s.ctx->stream));
}

// After the stream has passed the readback copies: accumulate the Hv timers of the passes that ran.
static void readback_finish(Shard& s, int cg_max) {
    if (s.g_timing && !s.last_group && !s.hv_timers.empty()) {
        const DevState& h = *s.st_host;
        for (int it = 0; it <= cg_max && it < (int)s.hv_timers.size(); ++it) {
            const bool ran = it < cg_max ? h.cg_act[it] != 0 : h.cert_act != 0;
            if (!ran) continue;
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, s.hv_timers[it].start, s.hv_timers[it].stop) == cudaSuccess) {
                s.ctx->stats.hv_kernel_ms += ms;
                s.ctx->stats.hv_kernel_samples++;
                s.ctx->stats.hv_kernel_shards++;
            }
        }
    }
}

// Reads back the solver state and trace (one async copy each, one sync).
static void readback(Shard& s, int cg_max) {
    solve_readback_async(s);
    stream_sync(s.ctx->stream);
    readback_finish(s, cg_max);
}

bool solve_launch(Shard& s, const nadmm_newton_cfg& cfg, double lambda, bool aug, double rho, int newton_max) {
    validate_newton_cfg(cfg);
    s.last_group = false;
    if (aug && rho <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
    set_params(s, cfg, lambda, aug, rho);
    capture_iteration_graph(s, cfg.cg_max_iters, cfg.ls_max_iters);
    ensure_cache_at_x(s, lambda);
    int nvec = 0;
    launch_grad_aug(s, nullptr, &nvec);
    launch_value_finish(s, nvec, 1, nullptr);
    s.cache_at = Shard::kAtX;
    s.cache_lambda = lambda;
    if (newton_max == 1) {  // no host decision needed: the caller collects after enqueueing other work
        NADMM_CUDA(cudaGraphLaunch(s.g_iter, s.ctx->stream));
        s.ctx->stats.kernel_launches += s.g_nodes;
        return false;
    }
    for (int k = 0; k < newton_max; ++k) {
        NADMM_CUDA(cudaGraphLaunch(s.g_iter, s.ctx->stream));
        s.ctx->stats.kernel_launches += s.g_nodes;
        readback(s, cfg.cg_max_iters);
        if (!s.st_host->active) break;
    }
    if (newton_max == 0) readback(s, cfg.cg_max_iters);
    return true;
}

SolveResult solve_result(Shard& s, const nadmm_newton_cfg& cfg) {
    readback_finish(s, cfg.cg_max_iters);
    return solve_collect(s, cfg, false);
}

SolveResult solve_collect(Shard& s, const nadmm_newton_cfg& cfg, bool pending) {
    if (pending) readback(s, cfg.cg_max_iters);
    const DevState& h = *s.st_host;
    SolveResult res;
    if (h.error) {
        res.error = h.error;
        return res;
    }
    res.iterations = h.iter;
    res.final_grad_norm = h.g_norm;
    res.converged = h.g_norm < cfg.grad_tol;  // src/newton.cpp:128-130 (or the early return at 83-86)
    res.trace.assign(s.trace_host, s.trace_host + std::min(h.iter, kTraceCap));
    for (const auto& t : res.trace) {
        res.cg_sum += t.cg_iters;
        res.fe_sum += t.fn_evals;
        if (t.ls_capped) res.flags |= 1;
        if (t.cg_fallback) res.flags |= 2;
    }
    return res;
}

SolveResult device_newton_solve(Shard& s, const nadmm_newton_cfg& cfg, double lambda, bool aug, double rho,
                                int newton_max) {
    const bool done = solve_launch(s, cfg, lambda, aug, rho, newton_max);
    return solve_collect(s, cfg, !done);
}

}  // namespace nadmm

namespace nadmm {

// ---------------------------------------------------------------------------------------------
// Node groups: the Newton iteration of several equal-shape DMMA shards (the local ADMM nodes of an
// outer iteration) captured as ONE graph whose data passes are group launches over the whole GPU
// (dmma_group.cuh) -- instead of one graph per node on a 1/k-GPU layout (node streams).
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int kGroupMax = 8;

struct GroupGraph {
    std::vector<Shard*> shards;
    int clusters = 0, cg_max = -1, ls_max = -1;
    int64_t layout_sig = -1;
    bool timing = false;
    cudaGraphExec_t exec = nullptr;
    int64_t nodes = 0;
    std::vector<HvTimer> timers;
    ~GroupGraph() {
        if (exec) cudaGraphExecDestroy(exec);
        for (auto& t : timers) {
            if (t.start) cudaEventDestroy(t.start);
            if (t.stop) cudaEventDestroy(t.stop);
        }
    }
};

}  // namespace

void group_drop(Ctx& c) {
    delete static_cast<GroupGraph*>(c.group);
    c.group = nullptr;
}

void group_forget(Shard& s) {
    if (!s.ctx || !s.ctx->group) return;
    const auto* g = static_cast<GroupGraph*>(s.ctx->group);
    for (Shard* x : g->shards)
        if (x == &s) {
            group_drop(*s.ctx);
            return;
        }
}

bool group_eligible(const std::vector<Shard*>& sh) {
    // opt-in (NADMM_GROUP=1) until the group pass beats the node streams on the bench shape
    static const bool off = [] {
        const char* e = getenv("NADMM_GROUP");
        return !(e && e[0] == '1');
    }();
    if (off || sh.size() < 2 || sh.size() > (size_t)kGroupMax) return false;
    const Shard& a = *sh[0];
    for (Shard* s : sh)
        if (!dmma_supported(*s) || s->p != a.p || s->K != a.K || s->ldx != a.ldx || s->ctx != a.ctx) return false;
    return true;
}

bool group_solve_launch(const std::vector<Shard*>& sh, const nadmm_newton_cfg& cfg, const double* rho) {
    if (!group_eligible(sh)) return false;
    Ctx& c = *sh[0]->ctx;
    const cudaStream_t st = c.stream;
    for (Shard* s : sh) use_layout_split(*s, 1);
    auto* cached = static_cast<GroupGraph*>(c.group);
    const Shard& s0 = *sh[0];
    const int64_t sig = ((((int64_t)s0.dmma_mt * 64 + s0.dmma_nw) * 64 + s0.dmma_cs) * 64 + s0.dmma_pipe) * 4096 +
                        s0.dmma_clusters;  // the whole-GPU layout the group kernel inherits
    const int clusters = (cached && cached->shards == sh && cached->layout_sig == sig) ? cached->clusters
                                                                                        : dmma_group_clusters(*sh[0]);
    if (clusters < 1) return false;
    for (Shard* s : sh)  // every cluster range must hold tiles of each node it spans (dmma_group.cuh)
        if ((s->n + 7) / 8 < clusters || s->dmma_clusters < clusters) return false;
    auto* g = static_cast<GroupGraph*>(c.group);
    if (!g || g->shards != sh || g->cg_max != cfg.cg_max_iters || g->ls_max != cfg.ls_max_iters ||
        g->timing != c.timing || g->clusters != clusters || g->layout_sig != sig) {
        group_drop(c);
        g = new GroupGraph();
        g->shards = sh;
        g->clusters = clusters;
        g->layout_sig = sig;
        g->cg_max = cfg.cg_max_iters;
        g->ls_max = cfg.ls_max_iters;
        g->timing = c.timing;
        if (g->timing) {
            g->timers.resize((size_t)cfg.cg_max_iters + 1);
            for (auto& t : g->timers) {
                NADMM_CUDA(cudaEventCreate(&t.start));
                NADMM_CUDA(cudaEventCreate(&t.stop));
            }
        }
        // the group's barrier counters (tail sub-grids, whole grid) restart for the new configuration
        for (Shard* s : sh) NADMM_CUDA(cudaMemsetAsync(s->gbar + 6, 0, 2 * sizeof(unsigned long long), st));
        const nadmm_stats saved = c.stats;
        cudaGraph_t graph = nullptr;
        NADMM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            launch_group_iteration(sh, clusters, cfg.cg_max_iters, g->timing ? g->timers.data() : nullptr);
        } catch (...) {
            cudaStreamEndCapture(st, &graph);
            if (graph) cudaGraphDestroy(graph);
            c.stats = saved;
            delete g;
            throw;
        }
        NADMM_CUDA(cudaStreamEndCapture(st, &graph));
        g->nodes = c.stats.kernel_launches - saved.kernel_launches;
        c.stats = saved;
        const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) {
            delete g;
            NADMM_CUDA(ie);
        }
        c.group = g;
        if (getenv("NADMM_DMMA_VERBOSE"))
            fprintf(stderr, "[nadmm] node group: %zu shards, %d clusters x %d CTAs, graph of %lld kernels\n",
                    sh.size(), clusters, sh[0]->dmma_cs, (long long)g->nodes);
    }
    for (size_t i = 0; i < sh.size(); ++i) {  // each node's solve prologue (solve_launch's)
        Shard& s = *sh[i];
        if (rho[i] <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
        set_params(s, cfg, 0.0, true, rho[i]);
        ensure_cache_at_x(s, 0.0);
        int nvec = 0;
        launch_grad_aug(s, nullptr, &nvec);
        launch_value_finish(s, nvec, 1, nullptr);
        s.cache_at = Shard::kAtX;
        s.cache_lambda = 0.0;
        s.last_group = true;
    }
    NADMM_CUDA(cudaGraphLaunch(g->exec, st));
    c.stats.kernel_launches += g->nodes;
    return true;
}

// After the synchronisation that brought the group's DevStates back: the timed group Hv passes
// (CG iterations and certificate) with the number of nodes that ran in each.
void group_timers_finish(Ctx& c) {
    auto* g = static_cast<GroupGraph*>(c.group);
    if (!g || !g->timing || g->timers.empty()) return;
    for (int it = 0; it <= g->cg_max; ++it) {
        int64_t cnt = 0;
        for (Shard* s : g->shards) cnt += it < g->cg_max ? (s->st_host->cg_act[it] != 0) : (s->st_host->cert_act != 0);
        if (cnt == 0) continue;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, g->timers[it].start, g->timers[it].stop) == cudaSuccess) {
            c.stats.hv_kernel_ms += ms;
            c.stats.hv_kernel_samples++;
            c.stats.hv_kernel_shards += cnt;
        }
    }
}

}  // namespace nadmm
