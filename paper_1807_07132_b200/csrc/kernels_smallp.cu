// Dense shards with few features and classes (p * (C-1) <= 64; the HIGGS-shaped 28-feature binary
// case): one pass over X per product with one ROW PER THREAD. A thread loads its row (p doubles,
// 16-byte loads), forms the K logits against the weight block held in shared memory, runs the row
// epilogue of the pass mode, and (Hv / cache) accumulates x_i u_i^T into p*K register accumulators.
// Blocks reduce their accumulators in a fixed order into one split-K partial per block
// (part[block][c*p + f]), which the solver tails sum in block order, exactly like the DMMA pass.
//
// Reference ops (file:line under /root/reference/proj):
//   logits X W                          src/dataset.cpp:69-76
//   stable_exp_cache / loss / coeff     src/softmax.cpp:51-95
//   Hv epilogue U = VoP - P rowsum      src/softmax.cpp:97-112
//   X^T U                               src/dataset.cpp:78-85
//   predict tie rule                    src/softmax.cpp:118-139
// The row arithmetic is the SIMT rows_kernel's, in the same ascending class order.
#include <algorithm>

#include "dmma_kernel.cuh"  // mbarrier / bulk-copy helpers (dmma_detail)
#include "state.h"

namespace nadmm {

namespace {

constexpr int kSpThreads = 256;

struct SmallArgs {
    const double* X;
    int64_t ldx, n, p;
    int K;
    const double* W;
    const double* Pin;
    const int32_t* labels;
    double *L0, *P, *Lp, *rowM, *rowA;
    int32_t* pred;
    double* lp_out;  // Hv mode: also store the X*v logits (see DmmaArgs::lp_out)
    double* part;
    double* blk;
    const int32_t* guard;
};

// RING: rows are streamed through a ring of kSpStages tiles of kSpThreads contiguous rows in shared
// memory by one bulk copy each (needs ldx == p with 16-byte rows), so the bytes in flight per SM do
// not depend on how many rows the registers let each thread hold; the grid is persistent. Otherwise
// each thread loads its row straight from global memory.
constexpr int kSpStages = 3;

template <int PT, int KT, int MODE, bool RING>
__global__ void __launch_bounds__(kSpThreads) smallp_kernel(SmallArgs a) {
    using namespace dmma_detail;
    if (a.guard && !*a.guard) return;
    extern __shared__ __align__(128) double ring[];  // kSpStages x kSpThreads x p (RING only)
    __shared__ uint64_t bars[kSpStages];
    constexpr bool PHASE_B = (MODE == kModeHv || MODE == kModeCache);
    __shared__ double vs[PT][KT];
    __shared__ double red[kSpThreads / 32][PHASE_B ? PT * KT : 1];
    __shared__ double lred[kSpThreads / 32];
    const int64_t p = a.p, n = a.n;
    const int K = a.K;
    for (int q = threadIdx.x; q < PT * KT; q += kSpThreads) {
        const int f = q / KT, c = q % KT;
        vs[f][c] = (f < p && c < K) ? a.W[(int64_t)c * p + f] : 0.0;
    }
    __syncthreads();
    double acc[PHASE_B ? PT : 1][KT];
#pragma unroll
    for (int f = 0; f < (PHASE_B ? PT : 1); ++f)
#pragma unroll
        for (int c = 0; c < KT; ++c) acc[f][c] = 0.0;
    double loss = 0.0;
    const int64_t ntiles = (n + kSpThreads - 1) / kSpThreads;
    auto tile_bytes = [&](int64_t t) -> uint32_t {
        const int64_t r0 = t * kSpThreads;
        const int64_t rows = (n - r0) < kSpThreads ? (n - r0) : kSpThreads;
        return (uint32_t)(rows * p * 8);
    };
    auto issue = [&](int64_t t, int st) {  // thread 0: bulk copy of tile t into stage st
        const uint32_t bytes = tile_bytes(t);
        mbar_expect_tx(&bars[st], bytes);
        tma_bulk_g2s(ring + (size_t)st * kSpThreads * p, a.X + t * kSpThreads * p, bytes, &bars[st]);
    };
    if (RING) {
        if (threadIdx.x == 0) {
            for (int st = 0; st < kSpStages; ++st) mbar_init(&bars[st], 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_proxy_async();
            for (int st = 0; st < kSpStages; ++st)
                if (blockIdx.x + (int64_t)st * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)st * gridDim.x, st);
        }
    }
    const int64_t stride = (int64_t)gridDim.x * kSpThreads;
    int k = 0;
    for (int64_t i0 = (int64_t)blockIdx.x * kSpThreads; i0 < n; i0 += stride, ++k) {
        const int64_t i = i0 + threadIdx.x;
        const int st = k % kSpStages;
        double x[PT];
        if (RING) {
            mbar_wait(&bars[st], (uint32_t)((k / kSpStages) & 1));
            const double* xr = ring + ((size_t)st * kSpThreads + threadIdx.x) * p;
#pragma unroll
            for (int f = 0; f < PT; f += 2) {
                if (f + 1 < p) {
                    const double2 v = *reinterpret_cast<const double2*>(xr + f);
                    x[f] = v.x;
                    x[f + 1] = v.y;
                } else {
                    x[f] = f < p ? xr[f] : 0.0;
                    x[f + 1] = 0.0;
                }
            }
            __syncthreads();  // every row of stage st is in registers: refill it
            if (threadIdx.x == 0 && i0 + (int64_t)kSpStages * stride < n) {
                fence_proxy_async();
                issue((i0 + (int64_t)kSpStages * stride) / kSpThreads, st);
            }
            if (i >= n) continue;
        } else {
            if (i >= n) continue;
            const double* xr = a.X + i * a.ldx;
            const bool vec = (a.ldx & 1) == 0;  // rows 16-byte aligned
#pragma unroll
            for (int f = 0; f < PT; f += 2) {
                if (vec && f + 1 < p) {
                    const double2 v = __ldg(reinterpret_cast<const double2*>(xr + f));
                    x[f] = v.x;
                    x[f + 1] = v.y;
                } else {
                    x[f] = f < p ? __ldg(xr + f) : 0.0;
                    x[f + 1] = f + 1 < p ? __ldg(xr + f + 1) : 0.0;
                }
            }
        }
        double lg[KT];
#pragma unroll
        for (int c = 0; c < KT; ++c) {
            double s = 0.0;
#pragma unroll
            for (int f = 0; f < PT; ++f) s += x[f] * vs[f][c];  // padded features are 0 * 0
            lg[c] = s;
        }
        const int b = a.labels[i];
        double u[KT];
#pragma unroll
        for (int c = 0; c < KT; ++c) u[c] = 0.0;
        if (MODE == kModeLp) {
#pragma unroll
            for (int c = 0; c < KT; ++c)
                if (c < K) a.Lp[i * K + c] = lg[c];
        } else if (MODE == kModeHv) {
            double e[KT], pv[KT];
            double rs = 0.0;
#pragma unroll
            for (int c = 0; c < KT; ++c) {
                pv[c] = c < K ? a.Pin[i * K + c] : 0.0;
                e[c] = lg[c] * pv[c];
                if (c < K) rs += e[c];
            }
#pragma unroll
            for (int c = 0; c < KT; ++c) u[c] = c < K ? e[c] - pv[c] * rs : 0.0;
            if (a.lp_out)
#pragma unroll
                for (int c = 0; c < KT; ++c)
                    if (c < K) a.lp_out[i * K + c] = lg[c];
        } else {
            double m = lg[0];
#pragma unroll
            for (int c = 1; c < KT; ++c)
                if (c < K && lg[c] > m) m = lg[c];
            m = m > 0.0 ? m : 0.0;
            double e[KT], s = 0.0;
#pragma unroll
            for (int c = 0; c < KT; ++c) {
                e[c] = c < K ? exp(lg[c] - m) : 0.0;
                if (c < K) s += e[c];
            }
            const double alpha = exp(-m) + s;
            if (MODE == kModeCache || MODE == kModeValue) {
                double lb = 0.0;
#pragma unroll
                for (int c = 0; c < KT; ++c)
                    if (c == b - 1) lb = lg[c];
                loss += (m + log(alpha)) - (b <= K ? lb : 0.0);
                if (MODE == kModeCache) {
                    a.rowM[i] = m;
                    a.rowA[i] = alpha;
#pragma unroll
                    for (int c = 0; c < KT; ++c)
                        if (c < K) {
                            const double pc = e[c] / alpha;
                            a.L0[i * K + c] = lg[c];
                            a.P[i * K + c] = pc;
                            u[c] = (c == b - 1) ? pc - 1.0 : pc;  // coeff (src/softmax.cpp:86-90)
                        }
                }
            } else {  // kModePredict
                const double residual = exp(-m) / alpha;
                double best = e[0] / alpha;
#pragma unroll
                for (int c = 1; c < KT; ++c)
                    if (c < K && e[c] / alpha > best) best = e[c] / alpha;
                int arg = 0;
#pragma unroll
                for (int c = KT - 1; c >= 0; --c)  // first c with P_c == max
                    if (c < K && e[c] / alpha == best) arg = c + 1;
                if (residual > best) arg = K + 1;
                a.pred[i] = arg;
                loss += (arg == b) ? 1.0 : 0.0;
            }
        }
        if (PHASE_B) {
#pragma unroll
            for (int f = 0; f < (PHASE_B ? PT : 1); ++f)
#pragma unroll
                for (int c = 0; c < KT; ++c) acc[f][c] += x[f] * u[c];
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (PHASE_B) {
        // fixed-order block reduction: xor-butterfly inside each warp, then warps in ascending order
#pragma unroll
        for (int f = 0; f < (PHASE_B ? PT : 1); ++f)
#pragma unroll
            for (int c = 0; c < KT; ++c) {
                const double v = warp_sum(acc[f][c]);
                if (lane == 0) red[w][f * KT + c] = v;
            }
        __syncthreads();
        const int64_t d = (int64_t)K * p;
        for (int q = threadIdx.x; q < PT * KT; q += kSpThreads) {
            const int f = q / KT, c = q % KT;
            if (f >= p || c >= K) continue;
            double s = 0.0;
            for (int ww = 0; ww < kSpThreads / 32; ++ww) s += red[ww][q];
            a.part[(int64_t)blockIdx.x * d + (int64_t)c * p + f] = s;
        }
    }
    if (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) {
        const double v = warp_sum(loss);
        if (lane == 0) lred[w] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int ww = 0; ww < kSpThreads / 32; ++ww) s += lred[ww];
            const int slot = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slot * kBlockPartials + blockIdx.x] = s;
        }
    }
}

template <int PT, int KT, bool RING>
void launch_ring(Shard& s, PassMode mode, const SmallArgs& a, int grid, size_t smem) {
    cudaStream_t st = s.ctx->stream;
    switch (mode) {
        case kModeCache: smallp_kernel<PT, KT, kModeCache, RING><<<grid, kSpThreads, smem, st>>>(a); break;
        case kModeHv: smallp_kernel<PT, KT, kModeHv, RING><<<grid, kSpThreads, smem, st>>>(a); break;
        case kModeLp: smallp_kernel<PT, KT, kModeLp, RING><<<grid, kSpThreads, smem, st>>>(a); break;
        case kModeValue: smallp_kernel<PT, KT, kModeValue, RING><<<grid, kSpThreads, smem, st>>>(a); break;
        case kModePredict: smallp_kernel<PT, KT, kModePredict, RING><<<grid, kSpThreads, smem, st>>>(a); break;
    }
}

template <int PT, int KT, bool RING>
void set_ring_smem(size_t smem) {
    for (auto k : {smallp_kernel<PT, KT, kModeCache, RING>, smallp_kernel<PT, KT, kModeHv, RING>,
                   smallp_kernel<PT, KT, kModeLp, RING>, smallp_kernel<PT, KT, kModeValue, RING>,
                   smallp_kernel<PT, KT, kModePredict, RING>})
        NADMM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

template <int PT, int KT>
void launch_pt(Shard& s, PassMode mode, const SmallArgs& a, int grid, bool ring, size_t smem) {
    if (ring)
        launch_ring<PT, KT, true>(s, mode, a, grid, smem);
    else
        launch_ring<PT, KT, false>(s, mode, a, grid, 0);
}

// Ring staging is used for contiguous 16-byte rows whose kSpStages tiles fit in shared memory.
size_t ring_smem(const Shard& s) { return (size_t)kSpStages * kSpThreads * s.p * sizeof(double); }
bool ring_ok(const Shard& s) { return s.ldx == s.p && s.p % 2 == 0 && ring_smem(s) <= 200 * 1024; }

}  // namespace

bool smallp_supported(const Shard& s) {
    return !s.sparse && s.part && ((s.p <= 32 && s.K <= 2) || (s.p <= 64 && s.K == 1));
}

void smallp_setup(Shard& s) {  // once per shard, outside stream capture
    if (!smallp_supported(s) || !ring_ok(s)) return;
    const size_t smem = ring_smem(s);
    if (s.p <= 32 && s.K == 1)
        set_ring_smem<32, 1, true>(smem);
    else if (s.p <= 32)
        set_ring_smem<32, 2, true>(smem);
    else
        set_ring_smem<64, 1, true>(smem);
}

void smallp_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    SmallArgs a{};
    a.X = s.X;
    a.ldx = s.ldx;
    a.n = s.n;
    a.p = s.p;
    a.K = s.K;
    a.W = W;
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
    const int64_t want = (s.n + kSpThreads - 1) / kSpThreads;
    const bool ring = ring_ok(s);
    // ring: one persistent block per SM (its ring is most of the SM's shared memory)
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>({want, (int64_t)s.part_chunks, (int64_t)kBlockPartials,
                              (ring ? 1LL : 2LL) * s.ctx->num_sms}));
    const size_t smem = ring ? ring_smem(s) : 0;
    if (s.p <= 32 && s.K == 1)
        launch_pt<32, 1>(s, mode, a, grid, ring, smem);
    else if (s.p <= 32)
        launch_pt<32, 2>(s, mode, a, grid, ring, smem);
    else
        launch_pt<64, 1>(s, mode, a, grid, ring, smem);
    NADMM_LAUNCH_CHECK();
    s.rows_grid = grid;
    s.last_chunks = grid;
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
}

}  // namespace nadmm
