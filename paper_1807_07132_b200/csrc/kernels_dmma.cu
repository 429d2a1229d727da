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
#include <cstdlib>

#include "dmma_kernel.cuh"

namespace nadmm {

// ------------------------------------------------------------------------------------------------

// Host side: layout selection and launch
// ------------------------------------------------------------------------------------------------
namespace {

constexpr int kBM = 8;
#ifndef NADMM_DMMA_LAG
#define NADMM_DMMA_LAG 4
#endif
constexpr int kLag = NADMM_DMMA_LAG;
constexpr int kStages = kLag + kDmmaExtraStages;

struct Layout {
    bool ok = false;
    int mt = 0, nw = 0, cs = 0, fs = 0, S = 0;
    size_t smem = 0;
};

size_t smem_bytes(int nw, int S, int K, int cs) { return dmma_smem_bytes(kStages, kBM, nw, S, K, cs) + 64; }

Layout choose_layout(int64_t p, int K) {
    Layout best;
    if (K != 9) return best;  // instantiated class counts (KT = 1, R = 1)
    double best_score = 1e30;
    for (int mt : {6, 7, 4, 8}) {
        for (int cs : {1, 2, 4, 8}) {
            const int W = 8 * mt;
            const int nw = (int)((p + (int64_t)cs * W - 1) / ((int64_t)cs * W));
            if (nw < 2 || nw > 8) continue;  // compute warps; + kDmmaAux exchange/producer warps
            const int fs = nw * W;
            const double waste = (double)cs * fs / (double)p - 1.0;
            if (waste > 0.15) continue;
            int S = fs + 4;
            while (S % 16 != 4) ++S;
            const size_t smem = smem_bytes(nw, S, K, cs);
            if (smem > 220 * 1024) continue;
            const double score = waste * 10.0 + cs * 0.05 + (nw < 4 ? 1.0 : 0.0);
            if (score < best_score) {
                best_score = score;
                best = Layout{true, mt, nw, cs, fs, S, smem};
            }
        }
    }
    return best;
}

cudaLaunchConfig_t make_cfg(Shard& s, const Layout& L, int clusters, cudaLaunchAttribute* attr) {  // attr[2]
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * L.cs, 1, 1);
    cfg.blockDim = dim3(32 * (L.nw + kDmmaAux), 1, 1);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s.ctx->stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = NADMM_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cfg;
}

// Attributes are set once per instantiation, outside any stream capture (dmma_setup), and the
// co-resident cluster count is queried there too.
template <int MT, int MODE>
int setup_mt(Shard& s, const Layout& L) {
    auto kern = dmma_pass_kernel<MT, 1, 1, kBM, kLag, MODE>;
    NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = make_cfg(s, L, 1, attr);
    int nc = 0;
    NADMM_CUDA(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg));
    return nc;
}

template <int MT>
int setup_modes(Shard& s, const Layout& L) {
    int nc = setup_mt<MT, kModeCache>(s, L);
    nc = std::min(nc, setup_mt<MT, kModeHv>(s, L));
    nc = std::min(nc, setup_mt<MT, kModeLp>(s, L));
    nc = std::min(nc, setup_mt<MT, kModeValue>(s, L));
    nc = std::min(nc, setup_mt<MT, kModePredict>(s, L));
    return nc;
}

template <int MT, int MODE>
void launch_mt(Shard& s, const Layout& L, const DmmaArgs& a, int clusters) {
    auto kern = dmma_pass_kernel<MT, 1, 1, kBM, kLag, MODE>;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = make_cfg(s, L, clusters, attr);
    NADMM_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
}

template <int MODE>
void launch_mode(Shard& s, const Layout& L, const DmmaArgs& a, int clusters) {
    switch (L.mt) {
        case 4: launch_mt<4, MODE>(s, L, a, clusters); break;
        case 6: launch_mt<6, MODE>(s, L, a, clusters); break;
        case 7: launch_mt<7, MODE>(s, L, a, clusters); break;
        case 8: launch_mt<8, MODE>(s, L, a, clusters); break;
        default: raise(NADMM_ECONFIG, "dmma: unsupported layout");
    }
}

}  // namespace

bool dmma_supported(const Shard& s) { return s.dmma_clusters > 0; }

void dmma_setup(Shard& s) {
    s.dmma_clusters = 0;
    static const bool disabled = getenv("NADMM_DISABLE_DMMA") != nullptr;
    if (disabled || s.sparse || s.ldx % 2 != 0) return;
    const Layout L = choose_layout(s.p, s.K);
    if (!L.ok) return;
    int active = 0;
    switch (L.mt) {
        case 4: active = setup_modes<4>(s, L); break;
        case 6: active = setup_modes<6>(s, L); break;
        case 7: active = setup_modes<7>(s, L); break;
        case 8: active = setup_modes<8>(s, L); break;
        default: return;
    }
    if (active < 1) return;
    const int64_t ntiles = (s.n + kBM - 1) / kBM;
    s.dmma_clusters = (int)std::max<int64_t>(
        1, std::min<int64_t>({ntiles, (int64_t)active, (int64_t)s.part_chunks, (int64_t)kBlockPartials}));
}

int dmma_clusters(const Shard& s) { return s.dmma_clusters; }

void dmma_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    const Layout L = choose_layout(s.p, s.K);
    if (!L.ok) raise(NADMM_ECONFIG, "dmma: no layout for this shape");
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
    a.lp_out = (mode == kModeHv && s.hv_write_lp) ? s.Lp : nullptr;
    a.part = s.part;
    a.blk = s.blk;
    a.guard = guard;
    a.fs = L.fs;
    a.S = L.S;
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

}  // namespace nadmm

#ifdef NADMM_DMMA_TRACE
extern "C" __attribute__((visibility("default"))) int nadmm_debug_dmma_trace(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, nadmm::g_dmma_trace, sizeof(nadmm::g_dmma_trace));
}
#endif
