// Fused single-pass FP64 DMMA kernel (device code). See kernels_dmma.cu for the design notes and
// the host-side layout selection / launch.
#pragma once

#include <cuda.h>

#include "state.h"

namespace nadmm {
namespace dmma_detail {

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

// try_wait loop (default .acquire.cta semantics; the data it guards lives in shared memory).
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

__device__ __forceinline__ uint32_t mapa(uint32_t local_smem, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_smem), "r"(rank));
    return r;
}

// 16-byte DSMEM store into CTA `rank`'s shared memory that completes tx bytes on its mbarrier.
__device__ __forceinline__ void st_async_v2(uint32_t remote_addr, double x, double y, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                     remote_addr),
                 "d"(x), "d"(y), "r"(remote_bar)
                 : "memory");
}

__device__ __forceinline__ double hsum16(double v) {  // sum over a 16-lane half warp (fixed tree)
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double hmax16(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace dmma_detail

struct DmmaArgs {
    const double* X;
    int64_t ldx;
    int64_t n, p;
    const double* V;        // block-major vector (d = K*p): the point w (cache modes) or direction v
    const double* Pin;      // probs, (n + pad) x K row-major (Hv mode)
    const int32_t* labels;  // n + pad entries
    double* L0;
    double* P;
    double* Lp;
    double* rowM;
    double* rowA;
    int32_t* pred;
    double* part;  // split-K partials, cluster-major: part[cluster * d + c*p + f]
    double* blk;   // block partial slots (loss / hits), one entry per cluster
    const int32_t* guard;
    int fs;  // features per CTA (= NW * 8 * MT)
    int S;   // padded shared row stride (doubles)
};

constexpr int kDmmaRecvBufs = 3;  // receive buffers: tile i's exchange overlaps tile i+1's phase A

template <int K>
struct DmmaSmem {
    static constexpr int KS = ((K + 15) / 16) * 16 + 4;  // U tile row stride (== 4 mod 16)
    static constexpr int KP = (K + 1) & ~1;              // partial row stride (even: 16-byte pairs)
};

// Shared memory bytes of the kernel's carve-up (host and device agree on it).
__host__ __device__ inline size_t dmma_smem_bytes(int stages, int bm, int nw, int S, int K, int cs) {
    const int KS = ((K + 15) / 16) * 16 + 4, KP = (K + 1) & ~1;
    const size_t dbl = (size_t)stages * bm * S + (size_t)stages * bm * K + 2 + (size_t)nw * bm * KP +
                       (size_t)kDmmaRecvBufs * cs * bm * KP + (size_t)bm * KS + 64;
    return sizeof(double) * dbl + 4 * ((size_t)stages * bm + 4) + 8 * (stages + kDmmaRecvBufs + 1);
}

template <int MT, int KT, int R, int BM, int STAGES, int MODE>
__global__ void __launch_bounds__(384, 1) dmma_pass_kernel(DmmaArgs a) {
    using namespace dmma_detail;
    constexpr int K = 8 * KT + R;
    static_assert(K <= 16, "half-warp epilogue handles up to 16 classes");
    static_assert(STAGES >= 3, "software pipeline keeps tiles i (phase B), i+1 (phase A), i+2 (loading)");
    constexpr int KS = DmmaSmem<K>::KS;
    constexpr int KP = DmmaSmem<K>::KP;
    constexpr int W = 8 * MT;
    constexpr int KSTEP_A = W / 4;
    constexpr bool PHASE_B = (MODE == kModeHv || MODE == kModeCache);
    constexpr bool NEED_P = (MODE == kModeHv);
    constexpr bool NEED_Y = (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict);
    constexpr int G = BM / 8;      // row groups in phase A
    constexpr int PART = BM * KP;  // doubles per CTA partial
    if (a.guard && !*a.guard) return;  // uniform across the grid: nothing is pending yet

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;  // fragment row / column-in-quad
    const uint32_t crank = cluster_ctarank(), csize = cluster_nctarank();
    const uint32_t cid = cluster_id_x(), ncl = ncluster_x();
    const int S = a.S, fs = a.fs;
    const int64_t p = a.p, n = a.n;
    const int f_cta = (int)crank * fs;  // first feature of this CTA
    const int fw = warp * W;            // warp slice offset inside the CTA slice

    // shared memory carve-up (mirrors dmma_smem_bytes)
    double* xs = reinterpret_cast<double*>(smem_raw);  // STAGES x BM x S
    double* ps = xs + (size_t)STAGES * BM * S;         // STAGES x BM x K   (P rows)
    double* red = ps + (size_t)STAGES * BM * K;        // nw x PART
    red = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(red) + 15) & ~uintptr_t(15));
    double* recv = red + (size_t)nw * PART;                   // kDmmaRecvBufs x CS x PART (peers write)
    double* ut = recv + (size_t)kDmmaRecvBufs * csize * PART;  // BM x KS
    double* misc = ut + BM * KS;                              // 64 doubles
    int32_t* ys = reinterpret_cast<int32_t*>(misc + 64);      // STAGES x BM labels
    uint64_t* bars = reinterpret_cast<uint64_t*>(ys + STAGES * BM + 4);
    bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bars) + 7) & ~uintptr_t(7));
    uint64_t* rbar = bars + STAGES;  // kDmmaRecvBufs

    const int64_t ntiles = (n + BM - 1) / BM;
    const int my_tiles = cid < ntiles ? (int)((ntiles - 1 - cid) / ncl + 1) : 0;
    const int64_t rem_f = p - f_cta;
    const int valid_f = rem_f <= 0 ? 0 : (rem_f < fs ? (int)rem_f : fs);  // valid features in slice
    const uint32_t row_bytes = (uint32_t)valid_f * 8u;

    // zero the X ring once: padding columns (beyond p) must read as 0, never as garbage
    for (int i = threadIdx.x; i < STAGES * BM * S; i += blockDim.x) xs[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        for (int b = 0; b < kDmmaRecvBufs; ++b) mbar_init(&rbar[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    fence_proxy_async();
    if (csize > 1) cluster_sync_all();  // peers' receive barriers are initialised before any st.async

    auto tile_of = [&](int i) -> int64_t { return (int64_t)cid + (int64_t)i * ncl; };
    auto issue = [&](int i) {  // TMA for the cluster's i-th tile into stage i % STAGES
        const int stage = i % STAGES;
        const int64_t r0 = tile_of(i) * BM;
        const int rows = (n - r0) < BM ? (int)(n - r0) : BM;
        uint32_t bytes = row_bytes * (uint32_t)rows;
        if (NEED_P) bytes += BM * K * 8;
        if (NEED_Y) bytes += BM * 4;
        mbar_expect_tx(&bars[stage], bytes);
        if (row_bytes)
            for (int r = 0; r < rows; ++r)
                tma_bulk_g2s(xs + ((size_t)stage * BM + r) * S, a.X + (r0 + r) * a.ldx + f_cta, row_bytes, &bars[stage]);
        if (NEED_P) tma_bulk_g2s(ps + (size_t)stage * BM * K, a.Pin + r0 * K, BM * K * 8, &bars[stage]);
        if (NEED_Y) tma_bulk_g2s(ys + stage * BM, a.labels + r0, BM * 4, &bars[stage]);
    };

    if (threadIdx.x == 0)
        for (int i = 0; i < STAGES && i < my_tiles; ++i) issue(i);

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
    double loss_acc = 0.0;  // rank-0 CTA: lane 0 of each half warp, rows in tile order

    // ---- phase A of the cluster's i-th tile, then push the CTA partial to every CTA's receive slot ----
    auto phase_a_and_push = [&](int i) {
        const int stage = i % STAGES;
        mbar_wait(&bars[stage], (uint32_t)((i / STAGES) & 1));
        const double* xt = xs + (size_t)stage * BM * S;
        double acca[2][G][KT > 0 ? KT : 1][2];  // even / odd k-steps: two independent DMMA chains
        double accar[G][R > 0 ? R : 1];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int kt = 0; kt < (KT > 0 ? KT : 1); ++kt) acca[h][g][kt][0] = acca[h][g][kt][1] = 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int r = 0; r < (R > 0 ? R : 1); ++r) accar[g][r] = 0.0;
#pragma unroll
        for (int s = 0; s < KSTEP_A; ++s) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double x = xt[(g * 8 + gq) * S + fw + 4 * s + tq];
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) dmma(acca[s & 1][g][kt], x, bv[s][kt]);
#pragma unroll
                for (int r = 0; r < R; ++r) accar[g][r] = fma(x, vr[s][r], accar[g][r]);
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double v = accar[g][r];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                accar[g][r] = v;
            }
        double* rw = red + (size_t)warp * PART;
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                const int o = (g * 8 + gq) * KP + kt * 8 + 2 * tq;
                rw[o] = acca[0][g][kt][0] + acca[1][g][kt][0];
                rw[o + 1] = acca[0][g][kt][1] + acca[1][g][kt][1];
            }
            if (tq == 0)
#pragma unroll
                for (int r = 0; r < R; ++r) rw[(g * 8 + gq) * KP + 8 * KT + r] = accar[g][r];
        }
        __syncthreads();
        // CTA partial (ascending warp order) -> slot [buf][crank] of every CTA in the cluster
        const int buf = i % kDmmaRecvBufs;
        const uint32_t dst_local = smem_u32(recv + ((size_t)buf * csize + crank) * PART);
        const uint32_t bar_local = smem_u32(&rbar[buf]);
        for (int i2 = threadIdx.x; i2 < PART / 2; i2 += blockDim.x) {
            double s0 = 0.0, s1 = 0.0;
            for (int w = 0; w < nw; ++w) {
                const double2 v = *reinterpret_cast<const double2*>(red + (size_t)w * PART + 2 * i2);
                s0 += v.x;
                s1 += v.y;
            }
            for (uint32_t q = 0; q < csize; ++q) st_async_v2(mapa(dst_local + 16u * i2, q), s0, s1, mapa(bar_local, q));
        }
        __syncthreads();  // red is free for the next phase A
    };

    const int hrow = lane >> 4, hc = lane & 15;  // epilogue: half warp per row, lane = class
    if (my_tiles > 0) phase_a_and_push(0);
    for (int i = 0; i < my_tiles; ++i) {
        const int stage = i % STAGES;
        const int buf = i % kDmmaRecvBufs;
        const int64_t r0 = tile_of(i) * BM;
        // overlap: tile i+1's phase A runs while tile i's partials travel through the cluster
        if (i + 1 < my_tiles) phase_a_and_push(i + 1);
        if (threadIdx.x == 0) mbar_expect_tx(&rbar[buf], (uint32_t)csize * PART * 8u);
        mbar_wait(&rbar[buf], (uint32_t)((i / kDmmaRecvBufs) & 1));

        // ---------------- epilogue: full logits (ascending cluster rank) -> U / cache ----------------
        const double* rv = recv + (size_t)buf * csize * PART;
        for (int row = warp * 2 + hrow; row < BM; row += 2 * nw) {
            const int64_t gi = r0 + row;
            const bool valid = gi < n;  // uniform over the half warp
            const bool cl = hc < K;
            double lg = 0.0;
            if (cl)
                for (uint32_t q = 0; q < csize; ++q) lg += rv[(size_t)q * PART + row * KP + hc];
            double* urow = ut + row * KS;
            if (MODE == kModeHv) {
                const double pr = (cl && valid) ? ps[(size_t)stage * BM * K + row * K + hc] : 0.0;
                const double vw = lg * pr;
                const double rs = hsum16(vw);
                if (cl) urow[hc] = valid ? vw - pr * rs : 0.0;
            } else if (MODE == kModeLp) {
                if (valid && cl && crank == 0) a.Lp[gi * K + hc] = lg;
            } else {
                const double m = fmax(hmax16(cl ? lg : -INFINITY), 0.0);
                const double e = cl ? exp(lg - m) : 0.0;
                const double alpha = exp(-m) + hsum16(e);
                const int b = valid ? ys[stage * BM + row] : 0;
                const double lb = hsum16((cl && hc == b - 1) ? lg : 0.0);
                const double pc = e / alpha;
                if (MODE == kModeCache || MODE == kModeValue) {
                    if (valid && crank == 0 && hc == 0) loss_acc += (m + log(alpha)) - (b <= K ? lb : 0.0);
                    if (MODE == kModeCache) {
                        if (cl) urow[hc] = valid ? ((hc == b - 1) ? pc - 1.0 : pc) : 0.0;
                        if (valid && cl && crank == 0) {
                            a.L0[gi * K + hc] = lg;
                            a.P[gi * K + hc] = pc;
                            if (hc == 0) {
                                a.rowM[gi] = m;
                                a.rowA[gi] = alpha;
                            }
                        }
                    }
                } else if (MODE == kModePredict) {
                    const double best = hmax16(cl ? pc : -INFINITY);
                    const unsigned eq = __ballot_sync(0xffffffffu, cl && pc == best);
                    const unsigned half = (eq >> (hrow * 16)) & 0xffffu;
                    int arg = __ffs(half);  // smallest class index attaining the max (tie rule)
                    const double residual = exp(-m) / alpha;
                    if (residual > best) arg = K + 1;
                    if (valid && crank == 0 && hc == 0) {
                        a.pred[gi] = arg;
                        loss_acc += (arg == b) ? 1.0 : 0.0;
                    }
                }
            }
        }
        __syncthreads();

        // ---------------- phase B: X_slice^T U into the resident accumulators ----------------
        if (PHASE_B) {
            const double* xt = xs + (size_t)stage * BM * S;
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
        __syncthreads();  // stage i and ut free (all warps past phase B)
        if (threadIdx.x == 0 && i + STAGES < my_tiles) {
            fence_proxy_async();
            issue(i + STAGES);
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
        // cluster's loss / hit partial (rank-0 CTA; fixed order over the per-half-warp accumulators)
        __syncthreads();
        if ((lane & 15) == 0) misc[warp * 2 + hrow] = loss_acc;
        __syncthreads();
        if (threadIdx.x == 0 && crank == 0) {
            double s = 0.0;
            for (int i = 0; i < 2 * nw; ++i) s += misc[i];
            const int slotid = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slotid * kBlockPartials + cid] = s;
        }
    }
    if (csize > 1) cluster_sync_all();  // no CTA leaves while peers may still target its shared memory
}

}  // namespace nadmm
