// Dense fast path: ONE pass over the shard's feature matrix per Hessian-vector product (and per
// cache+gradient evaluation), on the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).
//
// Reference ops fused here (file:line under /root/reference/proj):
//   V = X * blocks(v)                               src/softmax.cpp:103   (Dataset::multiply, src/dataset.cpp:69-76)
//   U = V o P - P o rowsum(V o P)                   src/softmax.cpp:104-107
//   Hv = X^T U                                      src/softmax.cpp:108   (Dataset::multiply_transposed, 78-85)
//   logits / M / alpha / P / loss / coeff = P - Y   src/softmax.cpp:51-95 (cache + gradient in the same pass)
//
// Structure (persistent, one CTA per SM, thread-block clusters of CS CTAs):
//   * A cluster owns a stream of BM-row tiles; CTA r of the cluster owns the feature slice
//     [r*FS, (r+1)*FS); warp w of a CTA owns the sub-slice of W = 8*MT features.
//   * Each tile's X slice (one cp.async.bulk per row), its P rows and labels arrive by TMA into a
//     STAGES-deep ring (mbarrier completion). X rows are padded to a stride S == 4 (mod 16) doubles
//     so the phase-A LDS.64 and phase-B LDS.128 fragment loads are bank-conflict free.
//   * Phase A: each warp multiplies its X sub-slice by the register-resident slice of V (DMMA for
//     the first 8*KT classes; DFMA riding on the same A fragments for the R remainder classes).
//     Warp partials are summed in shared memory; the CTA partial is pushed to every CTA of the
//     cluster with st.async (DSMEM stores that complete_tx on the receiver's mbarrier), so there is
//     no cluster-wide barrier per tile. Each CTA sums the CS partials in rank order: every CTA of a
//     cluster derives bit-identical logits.
//   * Epilogue (half a warp per row, one class per lane): U (Hv) or the stable softmax cache, loss
//     and coeff = P - Y (cache mode), Lp, argmax.
//   * Phase B: each warp accumulates X_slice^T U into register accumulators (DMMA + DFMA) resident
//     across all tiles of the cluster, written once at the end as one split-K partial per cluster
//     (reduced in fixed cluster order by finalize_kernel).
// The X tile is read from HBM exactly once and feeds both contractions.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dmma_group.cuh"

namespace nadmm {

// ------------------------------------------------------------------------------------------------

// Host side: layout selection and launch
// ------------------------------------------------------------------------------------------------
namespace {

constexpr int kBM = 8;

// Pipeline shapes (phase-B lag, ring stages): deeper lag hides a slower exchange, more free stages
// keep more bytes in flight per SM. Which wins depends on the slice width, so dmma_setup times them.
struct Pipe {
    int lag, stages;
};
constexpr Pipe kPipes[] = {{4, 6}, {3, 5}, {2, 5}};
constexpr int kNumPipes = sizeof(kPipes) / sizeof(kPipes[0]);

struct Layout {
    bool ok = false;
    int mt = 0, nw = 0, cs = 0, fs = 0, S = 0, pipe = 0;
    size_t smem = 0;
    double waste = 0.0;
};

#ifndef NADMM_DMMA_SMEM_KB
#define NADMM_DMMA_SMEM_KB 220
#endif
constexpr size_t kSmemLimit = NADMM_DMMA_SMEM_KB * 1024;

size_t smem_bytes(int pipe, int nw, int S, int K, int cs) {
    return dmma_smem_bytes(kPipes[pipe].stages, kBM, nw, S, K, cs) + 64;
}

// Feasible layouts for K = 9 (KT = 1, R = 1): the CTA slice fs = nw * 8 * mt features with 2..8
// compute warps, a cluster of cs CTAs covering p with <= 15 % padding, and the ring within the
// shared-memory budget. dmma_setup picks among them by co-resident SMs, then by measured time.
std::vector<Layout> candidate_layouts(int64_t p, int K) {
    std::vector<Layout> out;
    if (K != 9) return out;  // instantiated class counts
    for (int pipe = 0; pipe < kNumPipes; ++pipe)
        for (int mt : {6, 7, 4, 8})
            for (int cs = 1; cs <= 8; ++cs) {
                const int W = 8 * mt;
                const int nw = (int)((p + (int64_t)cs * W - 1) / ((int64_t)cs * W));
                if (nw < 2 || nw > dmma_max_compute(mt)) continue;  // compute warps (+ kDmmaAux aux warps)
                const int fs = nw * W;
                const double waste = (double)cs * fs / (double)p - 1.0;
                if (waste > 0.15) continue;
                int S = fs + 4;
                while (S % 16 != 4) ++S;
                const size_t smem = smem_bytes(pipe, nw, S, K, cs);
                if (smem > kSmemLimit) continue;
                out.push_back(Layout{true, mt, nw, cs, fs, S, pipe, smem, waste});
            }
    return out;
}

cudaLaunchConfig_t make_cfg(Shard& s, const Layout& L, int clusters, cudaLaunchAttribute* attr,
                            bool coop = false) {  // attr[2]
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * L.cs, 1, 1);
    cfg.blockDim = dim3(32 * (L.nw + kDmmaAux), 1, 1);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s.ctx->stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;  // the solver tails synchronise the grid (grid_barrier)
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (coop && coop_enabled()) ? 2 : 1;
    return cfg;
}

// Attributes are set once per instantiation, outside any stream capture (dmma_setup), and the
// co-resident cluster count is queried there too.
template <int MT, int PIPE, int MODE>
int setup_one(Shard& s, const Layout& L) {
    auto kern = dmma_pass_kernel<MT, 1, 1, kBM, kPipes[PIPE].lag, kPipes[PIPE].stages, MODE>;
    NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit));
    NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = make_cfg(s, L, 1, attr);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return nc;
}

template <int MT, int PIPE>
int setup_modes(Shard& s, const Layout& L) {
    int nc = setup_one<MT, PIPE, kModeCache>(s, L);
    nc = std::min(nc, setup_one<MT, PIPE, kModeHv>(s, L));
    nc = std::min(nc, setup_one<MT, PIPE, kModeLp>(s, L));
    nc = std::min(nc, setup_one<MT, PIPE, kModeValue>(s, L));
    nc = std::min(nc, setup_one<MT, PIPE, kModePredict>(s, L));
    return nc;
}

template <int PIPE>
int setup_pipe(Shard& s, const Layout& L) {
    switch (L.mt) {
        case 4: return setup_modes<4, PIPE>(s, L);
        case 6: return setup_modes<6, PIPE>(s, L);
        case 7: return setup_modes<7, PIPE>(s, L);
        case 8: return setup_modes<8, PIPE>(s, L);
        default: return 0;
    }
}

int setup_layout(Shard& s, const Layout& L) {
    switch (L.pipe) {
        case 0: return setup_pipe<0>(s, L);
        case 1: return setup_pipe<1>(s, L);
        case 2: return setup_pipe<2>(s, L);
        default: return 0;
    }
}

template <int MT, int PIPE, int MODE>
void launch_one(Shard& s, const Layout& L, const DmmaArgs& a, int clusters) {
    auto kern = dmma_pass_kernel<MT, 1, 1, kBM, kPipes[PIPE].lag, kPipes[PIPE].stages, MODE>;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = make_cfg(s, L, clusters, attr, a.tail != kTailNone);
    NADMM_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
}

template <int PIPE, int MODE>
void launch_pipe(Shard& s, const Layout& L, const DmmaArgs& a, int clusters) {
    switch (L.mt) {
        case 4: launch_one<4, PIPE, MODE>(s, L, a, clusters); break;
        case 6: launch_one<6, PIPE, MODE>(s, L, a, clusters); break;
        case 7: launch_one<7, PIPE, MODE>(s, L, a, clusters); break;
        case 8: launch_one<8, PIPE, MODE>(s, L, a, clusters); break;
        default: raise(NADMM_ECONFIG, "dmma: unsupported layout");
    }
}

template <int MODE>
void launch_mode(Shard& s, const Layout& L, const DmmaArgs& a, int clusters) {
    switch (L.pipe) {
        case 0: launch_pipe<0, MODE>(s, L, a, clusters); break;
        case 1: launch_pipe<1, MODE>(s, L, a, clusters); break;
        case 2: launch_pipe<2, MODE>(s, L, a, clusters); break;
        default: raise(NADMM_ECONFIG, "dmma: unsupported pipeline");
    }
}

Layout shard_layout(const Shard& s) {
    Layout L;
    L.ok = s.dmma_clusters > 0;
    L.mt = s.dmma_mt;
    L.nw = s.dmma_nw;
    L.cs = s.dmma_cs;
    L.fs = s.dmma_fs;
    L.S = s.dmma_S;
    L.pipe = s.dmma_pipe;
    L.smem = s.dmma_smem;
    return L;
}

}  // namespace

bool dmma_supported(const Shard& s) { return s.dmma_clusters > 0; }

namespace {

void apply_layout(Shard& s, const Layout& L, int active) {
    s.dmma_mt = L.mt;
    s.dmma_nw = L.nw;
    s.dmma_cs = L.cs;
    s.dmma_fs = L.fs;
    s.dmma_S = L.S;
    s.dmma_pipe = L.pipe;
    s.dmma_smem = L.smem;
    const int64_t ntiles = (s.n + kBM - 1) / kBM;
    s.dmma_clusters = (int)std::max<int64_t>(
        1, std::min<int64_t>({ntiles, (int64_t)active, (int64_t)s.part_chunks, (int64_t)kBlockPartials}));
}

// Device time of one Hv pass with the shard's current layout (scratch outputs only).
float time_hv_pass(Shard& s) {
    cudaEvent_t e0, e1;
    NADMM_CUDA(cudaEventCreate(&e0));
    NADMM_CUDA(cudaEventCreate(&e1));
    dmma_pass(s, kModeHv, s.x, nullptr);  // warm-up
    NADMM_CUDA(cudaEventRecord(e0, s.ctx->stream));
    for (int r = 0; r < 3; ++r) dmma_pass(s, kModeHv, s.x, nullptr);
    NADMM_CUDA(cudaEventRecord(e1, s.ctx->stream));
    NADMM_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    NADMM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms;
}

}  // namespace

// Layout choice: keep the feasible layouts that busy the most SMs (co-resident clusters x cluster
// size, capped at the SM count, discounted by feature padding); among those, time one Hv pass of
// each on the shard itself and keep the fastest (NADMM_DMMA_AUTOTUNE=0: tie-break by more compute
// warps, then the deeper pipeline, then the smaller cluster). Runs once per shard, outside capture.
void use_layout_split(Shard& s, int split) {
    if (split < 1) split = 1;
    if (s.layout_split == split || !dmma_supported(s)) return;
    invalidate_graphs(s);
    // the grid-barrier counters are multiples of the grid size that last used them: a new grid size
    // needs them restarted (stream-ordered after all earlier work on the shard)
    NADMM_CUDA(cudaMemsetAsync(s.gbar, 0, 8 * sizeof(unsigned long long), s.ctx->stream));
    dmma_setup(s, split);
}

void dmma_setup(Shard& s, int split) {
    s.dmma_clusters = 0;
    s.layout_split = split;
    static const bool disabled = getenv("NADMM_DISABLE_DMMA") != nullptr;
    if (disabled || s.sparse || s.ldx % 2 != 0) return;
    for (const auto& m : s.dmma_memo)  // chosen before for this split: re-apply (kernel attributes are set)
        if (m.split == split) {
            if (m.active > 0)
                apply_layout(s, Layout{true, m.mt, m.nw, m.cs, m.fs, m.S, m.pipe, m.smem, 0.0}, m.active);
            return;
        }
    const char* force_cs = getenv("NADMM_DMMA_CS");  // profiling: restrict the cluster size
    const char* force_pipe = getenv("NADMM_DMMA_PIPE");
    const char* at = getenv("NADMM_DMMA_AUTOTUNE");
    const bool autotune = !(at && at[0] == '0');
    struct Cand {
        Layout L;
        int active;
        double sms;
    };
    std::vector<Cand> cands;
    double best_sms = 0.0;
    for (const Layout& L : candidate_layouts(s.p, s.K)) {
        if (force_cs && L.cs != atoi(force_cs)) continue;
        if (force_pipe && L.pipe != atoi(force_pipe)) continue;
        int active = setup_layout(s, L);
        if (split > 1) active /= split;  // k concurrent shards share the GPU
        if (active < 1) continue;
        const double sms = std::min(active * L.cs, s.ctx->num_sms) * (1.0 - L.waste);
        cands.push_back({L, active, sms});
        best_sms = std::max(best_sms, sms);
    }
    std::vector<Cand> top;
    for (const Cand& c : cands)
        if (c.sms >= 0.98 * best_sms) top.push_back(c);
    if (top.empty()) {
        s.dmma_memo.push_back({split, 0, 0, 0, 0, 0, 0, 0, 0});
        return;
    }
    std::sort(top.begin(), top.end(), [](const Cand& a, const Cand& b) {
        const double sa = a.L.nw * 10.0 - a.L.pipe - a.L.cs * 0.1, sb = b.L.nw * 10.0 - b.L.pipe - b.L.cs * 0.1;
        return sa > sb;
    });
    // The split of the features over clusters and warps (cs, nw, mt) fixes the summation order of the
    // split-K partials and warp trees, so it is chosen by the fixed rule above (deterministic across
    // runs); only the pipeline shape (ring lag / stages, which leaves every sum's order unchanged) is
    // timed on the shard itself.
    {
        const Layout& f = top[0].L;
        std::vector<Cand> same;
        for (const Cand& c : top)
            if (c.L.cs == f.cs && c.L.nw == f.nw && c.L.mt == f.mt && c.active == top[0].active) same.push_back(c);
        top.swap(same);
    }
    size_t pick = 0;
    if (autotune && top.size() > 1) {
        float best_ms = 1e30f;
        for (size_t k = 0; k < top.size(); ++k) {
            apply_layout(s, top[k].L, top[k].active);
            const float ms = time_hv_pass(s);
            if (ms < best_ms) {
                best_ms = ms;
                pick = k;
            }
        }
    }
    const Layout& best = top[pick].L;
    apply_layout(s, best, top[pick].active);
    s.dmma_memo.push_back({split, best.mt, best.nw, best.cs, best.fs, best.S, best.pipe, top[pick].active, best.smem});
    if (getenv("NADMM_DMMA_VERBOSE"))
        fprintf(stderr,
                "[nadmm] dmma layout p=%lld: cluster %d x %d clusters (%d SMs), %d warps x %d features, lag %d, "
                "%d stages, smem %zu (%zu candidates timed)\n",
                (long long)s.p, best.cs, s.dmma_clusters, best.cs * s.dmma_clusters, best.nw, 8 * best.mt,
                kPipes[best.pipe].lag, kPipes[best.pipe].stages, best.smem, autotune ? top.size() : (size_t)0);
}

int dmma_clusters(const Shard& s) { return s.dmma_clusters; }

namespace {

DmmaArgs make_args(Shard& s, PassMode mode, const double* W, const int32_t* guard, int tail, int cg_it, bool write_lp) {
    DmmaArgs a{};
    a.X = s.X;
    a.ldx = s.ldx;
    a.n = s.n;
    a.p = s.p;
    a.V = W;
    a.Pin = s.P;
    a.labels = s.labels;
    a.L0 = s.L0;
    a.P = s.P;
    a.Lp = s.Lp;
    a.rowM = s.rowM;
    a.rowA = s.rowA;
    a.pred = s.pred;
    a.lp_out = (mode == kModeHv && write_lp) ? s.Lp : nullptr;
    a.part = s.part;
    a.blk = s.blk;
    a.guard = guard;
    a.tail = (mode == kModeHv || mode == kModeCache) ? tail : kTailNone;
    a.cg_it = cg_it;
    if (a.tail != kTailNone) {
        a.st = s.st;
        a.prm = s.prm;
        a.g = s.g;
        a.cg_p = s.pd;
        a.cg_r = s.r;
        a.cg_d = s.dv;
        a.cg_hd = s.hd;
        a.hv_ctr = s.ctx->dctr;
        a.done_ctr = s.gbar + 4;
        a.sub_ctr = s.gbar + 6;
        a.lp_from_cert = 1;
        a.x = s.x;
        a.z = s.z;
        a.y = s.y;
        a.gbase = s.gbase;
        a.t = s.t;
        a.scal = s.scal;
        a.trace = s.trace;
        a.trace_cap = kTraceCap;
    }
    a.fs = s.dmma_fs;
    a.S = s.dmma_S;
    return a;
}

}  // namespace

void dmma_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    const Layout L = shard_layout(s);
    if (!L.ok) raise(NADMM_ECONFIG, "dmma: no layout for this shape");
    const DmmaArgs a = make_args(s, mode, W, guard, s.dmma_tail, s.cg_fuse_it, s.hv_write_lp);
    const int clusters = dmma_clusters(s);
    switch (mode) {
        case kModeCache: launch_mode<kModeCache>(s, L, a, clusters); break;
        case kModeHv: launch_mode<kModeHv>(s, L, a, clusters); break;
        case kModeLp: launch_mode<kModeLp>(s, L, a, clusters); break;
        case kModeValue: launch_mode<kModeValue>(s, L, a, clusters); break;
        case kModePredict: launch_mode<kModePredict>(s, L, a, clusters); break;
    }
    s.rows_grid = clusters;  // loss / hit partial count
    s.last_chunks = clusters;
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
}

// ---------------- node-group passes (dmma_group.cuh) ----------------
namespace {

template <int MT, int PIPE, int MODE>
void group_launch_one(Shard& s, const Layout& L, const DmmaGroup& g, int clusters, bool query, int* active) {
    auto kern = dmma_group_kernel<MT, kPipes[PIPE].lag, kPipes[PIPE].stages, MODE>;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = make_cfg(s, L, clusters, attr, true);
    if (query) {
        NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
        NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cfg.gridDim = dim3(L.cs, 1, 1);
        cfg.numAttrs = 1;  // occupancy query without the cooperative attribute
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            nc = 0;
        }
        *active = nc;
        return;
    }
    NADMM_CUDA(cudaLaunchKernelEx(&cfg, kern, g));
}

template <int PIPE, int MODE>
void group_pipe(Shard& s, const Layout& L, const DmmaGroup& g, int clusters, bool query, int* active) {
    switch (L.mt) {
        case 4: group_launch_one<4, PIPE, MODE>(s, L, g, clusters, query, active); break;
        case 6: group_launch_one<6, PIPE, MODE>(s, L, g, clusters, query, active); break;
        case 7: group_launch_one<7, PIPE, MODE>(s, L, g, clusters, query, active); break;
        case 8: group_launch_one<8, PIPE, MODE>(s, L, g, clusters, query, active); break;
        default: raise(NADMM_ECONFIG, "dmma group: unsupported layout");
    }
}

template <int MODE>
void group_mode(Shard& s, const Layout& L, const DmmaGroup& g, int clusters, bool query, int* active) {
    switch (L.pipe) {
        case 0: group_pipe<0, MODE>(s, L, g, clusters, query, active); break;
        case 1: group_pipe<1, MODE>(s, L, g, clusters, query, active); break;
        case 2: group_pipe<2, MODE>(s, L, g, clusters, query, active); break;
        default: raise(NADMM_ECONFIG, "dmma group: unsupported pipeline");
    }
}

}  // namespace

// Co-resident clusters of the group kernel with shard s's (whole-GPU) layout; 0: unavailable.
int dmma_group_clusters(Shard& s) {
    const Layout L = shard_layout(s);
    if (!L.ok || s.layout_split != 1) return 0;
    DmmaGroup g{};
    int hv = 0, cache = 0;
    group_mode<kModeHv>(s, L, g, 0, true, &hv);
    group_mode<kModeCache>(s, L, g, 0, true, &cache);
    return std::min({hv, cache, s.dmma_clusters});
}

void dmma_group_pass(const std::vector<Shard*>& shards, int clusters, PassMode mode, const double* const* W,
                     const int32_t* const* guards, int tail, int cg_it, bool write_lp) {
    const int n = (int)shards.size();
    if (n < 1 || n > kMaxGroup) raise(NADMM_ECONFIG, "dmma group: 1..8 shards");
    Shard& s0 = *shards[0];
    const Layout L = shard_layout(s0);
    DmmaGroup g{};
    g.n = n;
    for (int k = 0; k < n; ++k) {
        Shard& s = *shards[k];
        g.node[k] = make_args(s, mode, W[k], guards[k], tail, cg_it, write_lp);
    }
    const int grid = clusters * L.cs;
    for (int k = 0; k <= n; ++k) g.sub_start[k] = (int)((int64_t)k * grid / n);  // tail sub-grids
    g.grid_ctr = s0.gbar + 7;
    switch (mode) {
        case kModeHv: group_mode<kModeHv>(s0, L, g, clusters, false, nullptr); break;
        case kModeCache: group_mode<kModeCache>(s0, L, g, clusters, false, nullptr); break;
        default: raise(NADMM_ECONFIG, "dmma group: unsupported mode");
    }
    for (Shard* s : shards) {
        s->ctx->stats.data_passes++;
        s->rows_grid = 0;
        s->last_chunks = 0;
    }
    s0.ctx->stats.kernel_launches++;
}

}  // namespace nadmm

#ifdef NADMM_DMMA_TRACE
extern "C" __attribute__((visibility("default"))) int nadmm_debug_dmma_trace(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, nadmm::g_dmma_trace, sizeof(nadmm::g_dmma_trace));
}
extern "C" __attribute__((visibility("default"))) int nadmm_debug_dmma_kstamps(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, nadmm::g_dmma_kst, sizeof(nadmm::g_dmma_kst));
}
#endif

// Profiling hook (not part of the ABI header): time `reps` node-group Hv passes (no solver tail) over
// the given shards (whole-GPU layouts) and, for comparison, `reps` single-shard passes of each shard.
extern "C" __attribute__((visibility("default"))) int nadmm_debug_group_hv(nadmm_shard* shards, int n,
                                                                          const double* const* v_dev, int reps,
                                                                          float* ms_group, float* ms_single) {
    try {
        std::vector<nadmm::Shard*> sh;
        for (int i = 0; i < n; ++i) sh.push_back(shards[i]);
        for (auto* s : sh) nadmm::use_layout_split(*s, 1);
        const int clusters = nadmm::dmma_group_clusters(*sh[0]);
        if (clusters < 1) return -2;
        std::vector<const int32_t*> gd(n, nullptr);
        cudaStream_t st = sh[0]->ctx->stream;
        for (auto* s : sh) cudaMemsetAsync(s->gbar + 6, 0, 2 * sizeof(unsigned long long), st);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        nadmm::dmma_group_pass(sh, clusters, nadmm::kModeHv, v_dev, gd.data(), nadmm::kTailNone, 0, false);
        cudaEventRecord(e0, st);
        for (int r = 0; r < reps; ++r)
            nadmm::dmma_group_pass(sh, clusters, nadmm::kModeHv, v_dev, gd.data(), nadmm::kTailNone, 0, false);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(ms_group, e0, e1);
        *ms_group /= reps;
        cudaEventRecord(e0, st);
        for (int r = 0; r < reps; ++r)
            for (int i = 0; i < n; ++i) nadmm::dmma_pass(*sh[i], nadmm::kModeHv, v_dev[i], nullptr);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(ms_single, e0, e1);
        *ms_single /= reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return (int)cudaGetLastError();
    } catch (...) {
        return -1;
    }
}
