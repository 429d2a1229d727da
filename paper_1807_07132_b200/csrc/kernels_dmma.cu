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
//   * Tiles arrive by TMA (cp.async.bulk, one copy per row slice, mbarrier completion) into a
//     STAGES-deep ring of padded shared-memory tiles (row stride S == 4 mod 16 doubles: the phase-A
//     LDS.64 and phase-B LDS.128 fragment loads are bank-conflict free).
//   * Phase A: each warp multiplies its X sub-slice by the register-resident slice of V
//     (DMMA for the first 8*KT classes, DFMA riding on the same A fragments for the R remainder
//     classes), partial logits are summed over warps in shared memory and over the cluster through
//     distributed shared memory (fixed rank order, so every CTA derives bit-identical logits).
//   * Epilogue per row: U (Hv) or the stable softmax cache, loss and coeff = P - Y (cache mode).
//   * Phase B: each warp accumulates X_slice^T U into register accumulators (DMMA + DFMA) that stay
//     resident across all tiles of the cluster; they are written once at the end as one split-K
//     partial per cluster (reduced in fixed cluster order by finalize_kernel).
// The X tile is read from HBM exactly once and feeds both contractions.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "state.h"

namespace nadmm {

namespace {

// ------------------------------------------------------------------------------------------------
// PTX helpers
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t ncluster_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Distributed shared memory load from CTA `rank` of the cluster. Not volatile / no memory clobber so
// independent loads pipeline; ordering comes from the cluster barrier (acquire) that precedes them.
__device__ __forceinline__ double ld_dsmem(const double* local_addr, uint32_t rank) {
    uint32_t ra;
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(smem_u32(local_addr)), "r"(rank));
    double v;
    asm("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(ra));
    return v;
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// Kernel
// ------------------------------------------------------------------------------------------------
struct DmmaArgs {
    const double* X;
    int64_t ldx;
    int64_t n, p;
    const double* V;     // block-major vector (d = K*p): the point w (cache modes) or direction v
    const double* Pin;   // probs n x K (Hv mode)
    const int32_t* labels;
    double* L0;
    double* P;
    double* Lp;
    double* rowM;
    double* rowA;
    int32_t* pred;
    double* part;  // split-K partials, cluster-major: part[cluster * d + c*p + f]
    double* blk;   // block partial slots (loss / hits), one entry per cluster
    const int32_t* guard;
    int fs;        // features per CTA (= NW * 8 * MT)
    int S;         // padded shared row stride (doubles)
};

template <int MT, int KT, int R, int BM, int STAGES, int MODE>
__global__ void __launch_bounds__(384, 1) dmma_pass_kernel(DmmaArgs a) {
    constexpr int K = 8 * KT + R;
    constexpr int KS = ((K + 15) / 16) * 16 + 4;  // U tile row stride: == 4 mod 16
    constexpr int W = 8 * MT;
    constexpr int KSTEP_A = W / 4;
    constexpr bool PHASE_B = (MODE == kModeHv || MODE == kModeCache);
    constexpr int G = BM / 8;  // row groups in phase A
    if (a.guard && !*a.guard) return;  // uniform across the grid: no cluster barrier is pending

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;  // fragment row / column-in-quad
    const uint32_t crank = cluster_ctarank(), csize = cluster_nctarank();
    const uint32_t cid = cluster_id_x(), ncl = ncluster_x();
    const int S = a.S, fs = a.fs;
    const int64_t p = a.p, n = a.n;
    const int f_cta = (int)crank * fs;           // first feature of this CTA
    const int fw = warp * W;                     // warp slice offset inside the CTA slice

    double* xs = reinterpret_cast<double*>(smem_raw);                 // STAGES x BM x S
    double* red = xs + (size_t)STAGES * BM * S;                       // nw x BM x K
    double* slot = red + (size_t)nw * BM * K;                         // 2 x BM x K (cluster visible)
    double* ut = slot + 2 * BM * K;                                   // BM x KS
    double* misc = ut + BM * KS;                                      // 32 doubles
    uint64_t* bars = reinterpret_cast<uint64_t*>(misc + 32);          // STAGES

    const int64_t ntiles = (n + BM - 1) / BM;
    const int64_t rem_f = p - f_cta;
    const int valid_f = rem_f <= 0 ? 0 : (rem_f < fs ? (int)rem_f : fs);  // valid features in slice
    const uint32_t row_bytes = (uint32_t)valid_f * 8u;

    // zero the whole X ring once: padding columns (beyond p) must read as 0, never as garbage
    for (int i = threadIdx.x; i < STAGES * BM * S; i += blockDim.x) xs[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    fence_proxy_async();

    auto issue = [&](int64_t tile, int stage) {
        const int64_t r0 = tile * BM;
        const int rows = (n - r0) < BM ? (int)(n - r0) : BM;
        if (row_bytes == 0 || rows <= 0) {
            mbar_expect_tx(&bars[stage], 0);
            return;
        }
        mbar_expect_tx(&bars[stage], row_bytes * (uint32_t)rows);
        for (int r = 0; r < rows; ++r)
            tma_bulk_g2s(xs + ((size_t)stage * BM + r) * S, a.X + (r0 + r) * a.ldx + f_cta, row_bytes, &bars[stage]);
    };

    // prologue: first STAGES tiles of this cluster
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            const int64_t t = (int64_t)cid + (int64_t)s * ncl;
            if (t < ntiles) issue(t, s);
        }
    }

    // V slice in registers: B fragments (k = tq, n = gq) and the remainder columns
    double bv[KSTEP_A][KT > 0 ? KT : 1];
    double vr[KSTEP_A][R > 0 ? R : 1];
#pragma unroll
    for (int s = 0; s < KSTEP_A; ++s) {
        const int64_t f = (int64_t)f_cta + fw + 4 * s + tq;
        const bool ok = f < p && fw + 4 * s + tq < fs;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) bv[s][kt] = ok ? a.V[(int64_t)(kt * 8 + gq) * p + f] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) vr[s][r] = ok ? a.V[(int64_t)(8 * KT + r) * p + f] : 0.0;
    }

    // phase-B accumulators, resident across all tiles
    double accb[PHASE_B ? MT : 1][KT > 0 ? KT : 1][2];
    double accbr[PHASE_B ? MT : 1][R > 0 ? R : 1];
#pragma unroll
    for (int m = 0; m < (PHASE_B ? MT : 1); ++m) {
#pragma unroll
        for (int kt = 0; kt < (KT > 0 ? KT : 1); ++kt) accb[m][kt][0] = accb[m][kt][1] = 0.0;
#pragma unroll
        for (int r = 0; r < (R > 0 ? R : 1); ++r) accbr[m][r] = 0.0;
    }
    double loss_acc = 0.0;  // rank-0 CTA, thread-per-row epilogue

    int it = 0;
    for (int64_t tile = cid; tile < ntiles; tile += ncl, ++it) {
        const int stage = it % STAGES;
        const uint32_t parity = (uint32_t)((it / STAGES) & 1);
        const int64_t r0 = tile * BM;
        const double* xt = xs + (size_t)stage * BM * S;
        mbar_wait(&bars[stage], parity);

        // ---------------- phase A: partial logits of this warp's feature sub-slice ----------------
        {
            double acca[G][KT > 0 ? KT : 1][2];
            double accar[G][R > 0 ? R : 1];
#pragma unroll
            for (int g = 0; g < G; ++g) {
#pragma unroll
                for (int kt = 0; kt < (KT > 0 ? KT : 1); ++kt) acca[g][kt][0] = acca[g][kt][1] = 0.0;
#pragma unroll
                for (int r = 0; r < (R > 0 ? R : 1); ++r) accar[g][r] = 0.0;
            }
#pragma unroll
            for (int s = 0; s < KSTEP_A; ++s) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double x = xt[(g * 8 + gq) * S + fw + 4 * s + tq];
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) dmma(acca[g][kt], x, bv[s][kt]);
#pragma unroll
                    for (int r = 0; r < R; ++r) accar[g][r] = fma(x, vr[s][r], accar[g][r]);
                }
            }
            // remainder partials: sum over the four k-lanes of each row
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double v = accar[g][r];
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    accar[g][r] = v;
                }
            double* rw = red + (size_t)warp * BM * K;
#pragma unroll
            for (int g = 0; g < G; ++g) {
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) {
                    rw[(g * 8 + gq) * K + kt * 8 + 2 * tq] = acca[g][kt][0];
                    rw[(g * 8 + gq) * K + kt * 8 + 2 * tq + 1] = acca[g][kt][1];
                }
                if (tq == 0)
#pragma unroll
                    for (int r = 0; r < R; ++r) rw[(g * 8 + gq) * K + 8 * KT + r] = accar[g][r];
            }
        }
        __syncthreads();
        // CTA partial (ascending warp order) into this tile's cluster slot
        double* sl = slot + (size_t)(it & 1) * BM * K;
        for (int i = threadIdx.x; i < BM * K; i += blockDim.x) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[(size_t)w * BM * K + i];
            sl[i] = s;
        }
        if (csize > 1)
            cluster_sync_all();
        else
            __syncthreads();

        // ---------------- epilogue: full logits (ascending cluster rank) -> U / cache ----------------
        double* lgb = red;  // red is free again: every thread is past the CTA-partial loop
        if (csize > 1) {
            for (int i = threadIdx.x; i < BM * K; i += blockDim.x) {
                double v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (q < (int)csize) v[q] = ld_dsmem(sl + i, q);
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (q < (int)csize) s += v[q];
                lgb[i] = s;
            }
        } else {
            for (int i = threadIdx.x; i < BM * K; i += blockDim.x) lgb[i] = sl[i];
        }
        __syncthreads();
        if (threadIdx.x < BM) {
            const int i = threadIdx.x;
            const int64_t gi = r0 + i;
            const bool valid = gi < n;
            double lg[K];
#pragma unroll
            for (int c = 0; c < K; ++c) lg[c] = lgb[i * K + c];
            double* urow = ut + i * KS;
            if (MODE == kModeHv) {
                if (valid) {
                    double pr[K], vw[K], rs = 0.0;
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        pr[c] = a.Pin[gi * K + c];
                        vw[c] = lg[c] * pr[c];
                    }
#pragma unroll
                    for (int c = 0; c < K; ++c) rs += vw[c];
#pragma unroll
                    for (int c = 0; c < K; ++c) urow[c] = vw[c] - pr[c] * rs;
                } else {
#pragma unroll
                    for (int c = 0; c < K; ++c) urow[c] = 0.0;
                }
            } else if (MODE == kModeLp) {
                if (valid && crank == 0)
#pragma unroll
                    for (int c = 0; c < K; ++c) a.Lp[gi * K + c] = lg[c];
            } else {
                if (valid) {
                    double m = lg[0];
#pragma unroll
                    for (int c = 1; c < K; ++c) m = lg[c] > m ? lg[c] : m;
                    m = m > 0.0 ? m : 0.0;
                    double e[K], s = 0.0;
#pragma unroll
                    for (int c = 0; c < K; ++c) e[c] = exp(lg[c] - m);
#pragma unroll
                    for (int c = 0; c < K; ++c) s += e[c];
                    const double alpha = exp(-m) + s;
                    const int b = a.labels[gi];
                    if (MODE == kModeCache || MODE == kModeValue) {
                        if (crank == 0) {
                            double lb = 0.0;
#pragma unroll
                            for (int c = 0; c < K; ++c)
                                if (c == b - 1) lb = lg[c];
                            loss_acc += (m + log(alpha)) - (b <= K ? lb : 0.0);
                        }
                        if (MODE == kModeCache) {
#pragma unroll
                            for (int c = 0; c < K; ++c) {
                                const double pc = e[c] / alpha;
                                urow[c] = (c == b - 1) ? pc - 1.0 : pc;
                                if (crank == 0) {
                                    a.L0[gi * K + c] = lg[c];
                                    a.P[gi * K + c] = pc;
                                }
                            }
                            if (crank == 0) {
                                a.rowM[gi] = m;
                                a.rowA[gi] = alpha;
                            }
                        }
                    } else if (MODE == kModePredict && crank == 0) {
                        const double residual = exp(-m) / alpha;
                        double best = e[0] / alpha;
#pragma unroll
                        for (int c = 1; c < K; ++c) best = (e[c] / alpha > best) ? e[c] / alpha : best;
                        int arg = 0;
                        for (int c = 0; c < K; ++c)
                            if (e[c] / alpha == best) {
                                arg = c + 1;
                                break;
                            }
                        if (residual > best) arg = K + 1;
                        a.pred[gi] = arg;
                        loss_acc += (arg == b) ? 1.0 : 0.0;
                    }
                } else if (MODE == kModeCache) {
#pragma unroll
                    for (int c = 0; c < K; ++c) urow[c] = 0.0;
                }
            }
        }
        __syncthreads();

        // ---------------- phase B: X_slice^T U into the resident accumulators ----------------
        if (PHASE_B) {
#pragma unroll
            for (int s = 0; s < BM / 4; ++s) {
                const int row = 4 * s + tq;
                double ub[KT > 0 ? KT : 1], ur[R > 0 ? R : 1];
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) ub[kt] = ut[row * KS + kt * 8 + gq];
#pragma unroll
                for (int r = 0; r < R; ++r) ur[r] = ut[row * KS + 8 * KT + r];
                const double* xr = xt + (size_t)row * S + fw;
#pragma unroll
                for (int mp = 0; mp < MT / 2; ++mp) {
                    const double2 x2 = *reinterpret_cast<const double2*>(xr + mp * 16 + 2 * gq);
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) {
                        dmma(accb[2 * mp][kt], x2.x, ub[kt]);
                        dmma(accb[2 * mp + 1][kt], x2.y, ub[kt]);
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        accbr[2 * mp][r] = fma(x2.x, ur[r], accbr[2 * mp][r]);
                        accbr[2 * mp + 1][r] = fma(x2.y, ur[r], accbr[2 * mp + 1][r]);
                    }
                }
                if (MT & 1) {
                    const double x = xr[(MT - 1) * 8 + gq];
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) dmma(accb[MT - 1][kt], x, ub[kt]);
#pragma unroll
                    for (int r = 0; r < R; ++r) accbr[MT - 1][r] = fma(x, ur[r], accbr[MT - 1][r]);
                }
            }
        }
        __syncthreads();  // stage buffer free (all warps past phase B)
        if (threadIdx.x == 0) {
            const int64_t nt = tile + (int64_t)STAGES * ncl;
            if (nt < ntiles) {
                fence_proxy_async();
                issue(nt, stage);
            }
        }
    }

    // ---------------- write this cluster's split-K partial of X^T U ----------------
    if (PHASE_B) {
        const int64_t d = (int64_t)K * p;
        double* out = a.part + (int64_t)cid * d;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            // feature of fragment row gq in m-tile m (pairs interleave; an odd tail is contiguous)
            const int loc = (MT % 2 == 1 && m == MT - 1) ? (m * 8 + gq) : ((m / 2) * 16 + 2 * gq + (m & 1));
            const int64_t f = (int64_t)f_cta + fw + loc;
            const bool ok = f < p && fw + loc < fs;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                if (ok) {
                    out[(int64_t)(kt * 8 + 2 * tq) * p + f] = accb[m][kt][0];
                    out[(int64_t)(kt * 8 + 2 * tq + 1) * p + f] = accb[m][kt][1];
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double v = accbr[m][r];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (ok && tq == 0) out[(int64_t)(8 * KT + r) * p + f] = v;
            }
        }
    }
    if (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) {
        // cluster's loss / hit partial (rank-0 CTA, rows in tile order, threads ascending)
        __syncthreads();
        if (threadIdx.x < BM) misc[threadIdx.x] = loss_acc;
        __syncthreads();
        if (threadIdx.x == 0 && crank == 0) {
            double s = 0.0;
            for (int i = 0; i < BM; ++i) s += misc[i];
            const int slotid = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slotid * kBlockPartials + cid] = s;
        }
    }
    if (csize > 1) cluster_sync_all();  // no CTA leaves while peers may still read its slots
}

// ------------------------------------------------------------------------------------------------
// Host side: layout selection and launch
// ------------------------------------------------------------------------------------------------
namespace {

constexpr int kBM = 16;
constexpr int kStages = 3;

struct Layout {
    bool ok = false;
    int mt = 0, nw = 0, cs = 0, fs = 0, S = 0;
    size_t smem = 0;
};

size_t smem_bytes(int nw, int S, int K) {
    const int KS = ((K + 15) / 16) * 16 + 4;
    return sizeof(double) * ((size_t)kStages * kBM * S + (size_t)nw * kBM * K + 2 * kBM * K + kBM * KS + 32) +
           8 * kStages;
}

Layout choose_layout(int64_t p, int K) {
    Layout best;
    if (K != 9) return best;  // instantiated class counts (KT = 1, R = 1)
    double best_score = 1e30;
    for (int mt : {6, 7, 4, 8}) {
        for (int cs : {1, 2, 4, 8}) {
            const int W = 8 * mt;
            const int nw = (int)((p + (int64_t)cs * W - 1) / ((int64_t)cs * W));
            if (nw < 2 || nw > 12) continue;
            const int fs = nw * W;
            const double waste = (double)cs * fs / (double)p - 1.0;
            if (waste > 0.15) continue;
            int S = fs + 4;
            while (S % 16 != 4) ++S;
            const size_t smem = smem_bytes(nw, S, K);
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

cudaLaunchConfig_t make_cfg(Shard& s, const Layout& L, int clusters, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * L.cs, 1, 1);
    cfg.blockDim = dim3(32 * L.nw, 1, 1);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s.ctx->stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

// Attributes are set once per instantiation, outside any stream capture (dmma_setup), and the
// co-resident cluster count is queried there too.
template <int MT, int MODE>
int setup_mt(Shard& s, const Layout& L) {
    auto kern = dmma_pass_kernel<MT, 1, 1, kBM, kStages, MODE>;
    NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NADMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchAttribute attr[1];
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
    auto kern = dmma_pass_kernel<MT, 1, 1, kBM, kStages, MODE>;
    cudaLaunchAttribute attr[1];
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
