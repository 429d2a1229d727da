// Fused single-pass FP64 DMMA kernel (device code), warp-specialised. See kernels_dmma.cu for the
// design notes and the host-side layout selection / launch.
//
// Warp roles in a CTA (blockDim = 32 * (NC + kDmmaAux)):
//   * NC compute warps own W = 8*MT features each: phase A (partial logits, DMMA + DFMA) and phase B
//     (X^T U accumulation, DMMA + DFMA), software-pipelined one tile apart (A(i+1) then B(i)), so the
//     tensor pipe keeps issuing while tile i's logits travel through the cluster.
//   * one pusher warp: sums the compute warps' partials (ascending warp order) and pushes the CTA
//     partial to every CTA of the cluster (st.async + remote mbarrier complete_tx); it runs ahead of
//     the epilogue by one tile.
//   * kDmmaEpiWarps epilogue warps: sum the CS partials of a tile in rank order (every CTA derives
//     bit-identical logits), then one thread per row runs the row epilogue (U, softmax cache, loss,
//     argmax) in ascending class order, exactly like the SIMT path and the reference.
//   * one producer warp: TMA (cp.async.bulk) of X row slices, P rows and labels into a STAGES ring.
// All hand-offs are mbarriers; no block-wide barrier sits on the per-tile critical path.
#pragma once

#include <cuda.h>

#include "solver_tails.cuh"
#include "state.h"

namespace nadmm {
namespace dmma_detail {

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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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

// Bulk copy of a local shared-memory buffer into a peer CTA's shared memory (cluster addresses for
// the destination and its mbarrier), completing `bytes` on that mbarrier: one instruction per peer.
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     dst),
                 "r"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Fixed-topology pairwise sum of v[0..n) (n <= N): depth log2(N) instead of a serial chain. The
// auxiliary warps share the FP64 pipe with the compute warps' DMMAs, so every dependent FP64 op on
// their critical path costs a pipe turn; trees keep those paths short. Deterministic by construction.
template <int N>
__device__ __forceinline__ double tree_sum(double (&v)[N], int n) {
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (i >= n) v[i] = 0.0;
#pragma unroll
    for (int w = 1; w < N; w *= 2)
#pragma unroll
        for (int i = 0; i + w < N; i += 2 * w) v[i] = v[i] + v[i + w];
    return v[0];
}

__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
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
    double* lp_out;  // Hv mode: also store the X*v logits (the certificate Hv's logits are the Armijo Lp)
    double* part;  // split-K partials, cluster-major: part[cluster * d + c*p + f]
    double* blk;   // block partial slots (loss / hits), one entry per cluster
    const int32_t* guard;
    // solver tail run by the whole grid after the last tile (DmmaTail): CG step (Hv pass inside the
    // CG loop), certificate / fallback / slope (certificate Hv pass), gradient + value + trace (cache
    // pass at the new iterate)
    int tail;
    int cg_it;
    int lp_from_cert;
    const double *x, *z, *y;
    double *gbase, *t, *scal;
    DevTrace* trace;
    int trace_cap;
    DevState* st;
    const DevParams* prm;
    double* g;  // gradient (read by the CG / certificate tails, written by the Newton tail)
    double *cg_p, *cg_r, *cg_d, *cg_hd;
    unsigned long long* hv_ctr;    // Hv products applied (device counter)
    unsigned long long* done_ctr;  // clusters finished with this launch (reset by the last one)
    unsigned long long* sub_ctr;   // node-group passes: barrier counter of this node's tail sub-grid
    int fs;  // features per CTA (= NC * 8 * MT)
    int S;   // padded shared row stride (doubles, even)
};

__device__ __forceinline__ void mbar_arrive_remote(uint64_t* local_bar, uint32_t rank) {
    const uint32_t ra = dmma_detail::mapa(dmma_detail::smem_u32(local_bar), rank);
    // Relaxed: a credit publishes no data. It only orders our completed reads of the peer-written
    // buffer before the peer's next st.async into it (the loads' values were consumed already).
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(ra) : "memory");
}

#ifdef NADMM_DMMA_TRACE
__device__ long long g_dmma_trace[64][16];  // per-tile clock64 stamps of CTA 0 (profiling builds only)
#define DMMA_TRACE(i, k) \
    do { \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (i) < 64) g_dmma_trace[(i)][(k)] = clock64(); \
    } while (0)
// kernel-level globaltimer stamps of every CTA (ns): 0 entry, 1 setup done, 2 first TMA issued,
// 3 tile 0 landed (compute warp 0), 4 last phase B done, 5 partial written, 6 final cluster sync, 7 exit
__device__ long long g_dmma_kst[256][8];
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DMMA_KST(k) \
    do { \
        if (blockIdx.x < 256) g_dmma_kst[blockIdx.x][(k)] = gtimer(); \
    } while (0)
#else
#define DMMA_KST(k) \
    do { \
    } while (0)
#define DMMA_TRACE(i, k) \
    do { \
    } while (0)
#endif

#ifndef NADMM_DMMA_CHAINS
#define NADMM_DMMA_CHAINS 4
#endif
constexpr int kDmmaChains = NADMM_DMMA_CHAINS;  // phase-A accumulator chains per warp

#ifndef NADMM_DMMA_RECV_BUFS
#define NADMM_DMMA_RECV_BUFS 4
#endif
constexpr int kDmmaRecvBufs = NADMM_DMMA_RECV_BUFS;
// Up to 8 compute warps per CTA (2 per SM sub-partition). Measured: 16 narrow (MT = 4) warps per
// CTA spill under the 102-register cap and run 30-50 % slower on the CIFAR shapes.
__host__ __device__ constexpr int dmma_max_compute(int) { return 8; }  // receive buffers per CTA, flow-controlled by remote credits
#ifndef NADMM_DMMA_RED_BUFS
#define NADMM_DMMA_RED_BUFS 2
#endif
constexpr int kDmmaRedBufs = NADMM_DMMA_RED_BUFS;  // compute-warp partial buffers (pusher frees them)
constexpr int kDmmaEpiWarps = 2;  // epilogue warps
constexpr int kDmmaAux = kDmmaEpiWarps + 2;  // + pusher + producer
__host__ __device__ constexpr int dmma_max_threads(int mt) { return 32 * (dmma_max_compute(mt) + kDmmaAux); }

template <int K>
struct DmmaSmem {
    static constexpr int KS = ((K + 15) / 16) * 16 + 4;  // U tile row stride (== 4 mod 16)
    static constexpr int KP = (K + 1) & ~1;              // partial row stride (even: 16-byte pairs)
};

// Shared memory bytes of the kernel's carve-up (host and device agree on it). Every region holds an
// even number of doubles, so all of them stay 16-byte aligned. U buffers: one per stage.
__host__ __device__ inline size_t dmma_smem_bytes(int stages, int bm, int nc, int S, int K, int cs) {
    const int KS = ((K + 15) / 16) * 16 + 4, KP = (K + 1) & ~1, KE = (K + 1) & ~1;
    const size_t dbl = (size_t)stages * bm * S + (size_t)stages * bm * KE + (size_t)kDmmaRedBufs * nc * bm * KP +
                       (size_t)kDmmaRecvBufs * cs * bm * KP + (size_t)kDmmaRecvBufs * bm * KP + (size_t)stages * bm * KS +
                       (size_t)kDmmaEpiWarps * bm * KP + 128;
    const int nbars = 2 * stages + 2 * kDmmaRedBufs + 2 * kDmmaRecvBufs + stages;
    return sizeof(double) * dbl + 4 * ((size_t)stages * bm + 4) + 8 * (nbars + 1);
}

// The CG iteration's tail (src/newton.cpp:31-50, as k_cg_tail) run by the whole persistent grid of
// the Hv pass after its last tile: every CTA owns a slice of d, sums the per-cluster partials there
// (cluster order) + lambda d (+ rho d), and the curvature / <r,r> reductions go through block slots
// and software grid barriers (the grid is co-resident by construction). All blocks evaluate the same
// scalars; block 0 / thread 0 writes the solver state.
__device__ __forceinline__ void dmma_cg_tail(const DmmaArgs& a, int K, int chunks, double* scratch, double* sc,
                                             VGrid vg, unsigned long long* bar) {
    const int it = a.cg_it;
    DevState* st = a.st;
    const int64_t d = (int64_t)K * a.p;
    const bool lead = vg.b == 0 && threadIdx.x == 0;
    const int64_t tid = (int64_t)vg.b * blockDim.x + threadIdx.x, nth = (int64_t)vg.nb * blockDim.x;
    const double lam = a.prm->lambda, rho = a.prm->rho;
    const bool aug = a.prm->augmented;
    double* curv_slot = a.blk + (int64_t)kSlotCurv * kBlockPartials;
    double* rr_slot = a.blk + (int64_t)kSlotRr * kBlockPartials;
    if (lead && a.hv_ctr) atomicAdd(a.hv_ctr, 1ULL);
    double dacc = 0.0;
    for (int64_t j = tid; j < d; j += nth) {
        double s = 0.0;
        for (int ch = 0; ch < chunks; ch += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = (ch + q < chunks) ? __ldcg(a.part + (int64_t)(ch + q) * d + j) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (ch + q < chunks) s += v[q];
        }
        const double vj = a.cg_d[j];
        if (lam > 0.0) s = s + lam * vj;
        if (aug) s = s + rho * vj;
        a.cg_hd[j] = s;
        dacc += s * vj;
    }
    double t = block_sum(dacc, scratch);
    if (threadIdx.x == 0) curv_slot[vg.b] = t;
    grid_barrier_n(bar, vg.nb);
    if (threadIdx.x < 32) {
        const double v = reduce_partials(curv_slot, vg.nb);
        if (threadIdx.x == 0) *sc = v;
    }
    __syncthreads();
    const double curv = *sc;
    int act_next = 0;
    if (!isfinite(curv)) {
        if (lead) {
            st->cg_failed = 1;
            st->cg_mid[it] = 0;
        }
    } else if (curv <= 0.0) {
        if (it == 0)
            for (int64_t j = tid; j < d; j += nth) a.cg_p[j] = -a.g[j];
        if (lead) {
            st->cg_neg = 1;
            st->cg_mid[it] = 0;
        }
    } else {
        const double r_sq = st->r_sq[it];
        const double alpha = r_sq / curv;
        double rr = 0.0;
        for (int64_t j = tid; j < d; j += nth) {
            a.cg_p[j] += alpha * a.cg_d[j];
            const double rj = a.cg_r[j] - alpha * a.cg_hd[j];
            a.cg_r[j] = rj;
            rr += rj * rj;
        }
        t = block_sum(rr, scratch);
        if (threadIdx.x == 0) rr_slot[vg.b] = t;
        if (lead) {
            st->cg_iters = it + 1;
            st->cg_mid[it] = 1;
        }
        grid_barrier_n(bar, vg.nb);
        __syncthreads();  // *sc reused
        if (threadIdx.x < 32) {
            const double v = reduce_partials(rr_slot, vg.nb);
            if (threadIdx.x == 0) *sc = v;
        }
        __syncthreads();
        const double r_sq_next = *sc;
        if (!isfinite(r_sq_next)) {
            if (lead) st->cg_failed = 1;
        } else if (!(sqrt(r_sq_next) <= st->cg_stop)) {
            const double beta = r_sq_next / r_sq;
            for (int64_t j = tid; j < d; j += nth) a.cg_d[j] = a.cg_r[j] + beta * a.cg_d[j];
            if (lead) st->r_sq[it + 1] = r_sq_next;
            act_next = 1;
        }
    }
    if (lead) {
        st->cg_act[it + 1] = act_next;
        st->cert_act = st->it_act && !st->cg_failed;
    }
}

// LAG: tiles of phase A in flight ahead of phase B; STAGES >= LAG + 2 ring slots (the LAG tiles
// waiting for phase B, the one in phase A, and the ones loading).
template <int MT, int KT, int R, int BM, int LAG, int STAGES, int MODE>
__global__ void __launch_bounds__(dmma_max_threads(MT), 1) dmma_pass_kernel(DmmaArgs a) {
    using namespace dmma_detail;
    static_assert(STAGES >= LAG + 2, "ring depth");
    constexpr int K = 8 * KT + R;
    static_assert(BM == 8, "row tile: the row epilogues map 8 rows onto one warp (4 lanes per row)");
    constexpr int KS = DmmaSmem<K>::KS;
    constexpr int KP = DmmaSmem<K>::KP;
    constexpr int KE = (K + 1) & ~1;  // P rows are loaded K wide; region rounded to an even count
    constexpr int W = 8 * MT;
    constexpr int KSTEP_A = W / 4;
    constexpr bool PHASE_B = (MODE == kModeHv || MODE == kModeCache);
    constexpr bool NEED_P = (MODE == kModeHv);
    constexpr bool NEED_Y = (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict);
    constexpr int G = BM / 8;      // row groups in phase A
    constexpr int PART = BM * KP;  // doubles per CTA partial
    constexpr int EPI_THREADS = 32 * kDmmaEpiWarps;
    extern __shared__ __align__(128) double smem[];
    const int nc = (int)(blockDim.x >> 5) - kDmmaAux;  // compute warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;  // fragment row / column-in-quad
    const uint32_t crank = cluster_ctarank(), csize = cluster_nctarank();
    const uint32_t cid = cluster_id_x(), ncl = ncluster_x();
    const int S = a.S, fs = a.fs;
    const int64_t p = a.p, n = a.n;
    const int f_cta = (int)crank * fs;  // first feature of this CTA

    // shared memory carve-up (mirrors dmma_smem_bytes)
    double* xs = smem;                                               // STAGES x BM x S
    double* ps = xs + (size_t)STAGES * BM * S;                       // STAGES x BM x KE (P rows)
    double* red = ps + (size_t)STAGES * BM * KE;                     // kDmmaRedBufs x nc x PART
    double* recv = red + (size_t)kDmmaRedBufs * nc * PART;           // kDmmaRecvBufs x CS x PART (peers)
    double* sendb = recv + (size_t)kDmmaRecvBufs * csize * PART;     // kDmmaRecvBufs x PART (own partial)
    double* ut = sendb + (size_t)kDmmaRecvBufs * PART;               // STAGES x BM x KS
    double* lgb = ut + (size_t)STAGES * BM * KS;                     // kDmmaEpiWarps x BM x KP logits
    double* misc = lgb + (size_t)kDmmaEpiWarps * BM * KP;           // 128 doubles
    int32_t* ys = reinterpret_cast<int32_t*>(misc + 128);            // STAGES x BM labels
    uint64_t* bars = reinterpret_cast<uint64_t*>(ys + STAGES * BM + 4);
    uint64_t* full = bars;                         // STAGES: TMA landed
    uint64_t* empty = full + STAGES;               // STAGES: stage consumed (nc compute + epilogue warps)
    uint64_t* red_full = empty + STAGES;           // kDmmaRedBufs: compute partials written (nc warps)
    uint64_t* red_empty = red_full + kDmmaRedBufs;  // kDmmaRedBufs: pusher done reading (1)
    uint64_t* rbar = red_empty + kDmmaRedBufs;     // kDmmaRecvBufs: cluster partials received (tx)
    uint64_t* credit = rbar + kDmmaRecvBufs;       // kDmmaRecvBufs: every CTA consumed its copy (CS)
    uint64_t* u_full = credit + kDmmaRecvBufs;     // STAGES: U tile ready (epilogue warps)

    if (threadIdx.x == 0) DMMA_KST(0);
    const int64_t ntiles = (n + BM - 1) / BM;
    int T = cid < ntiles ? (int)((ntiles - 1 - cid) / ncl + 1) : 0;  // this cluster's tiles
    const int64_t rem_f = p - f_cta;
    const int valid_f = rem_f <= 0 ? 0 : (rem_f < fs ? (int)rem_f : fs);  // valid features in slice
    const uint32_t row_bytes = (uint32_t)valid_f * 8u;

    // feature padding of a partial last slice is read by phase A and must be 0 (stale or uninitialised
    // shared memory could hold NaN bit patterns); rows beyond n are masked where they are read instead
    if (valid_f < fs)
        for (int i = threadIdx.x; i < STAGES * BM * S; i += blockDim.x) xs[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (uint32_t)(nc + 1));  // compute warps + the tile's epilogue warp
            mbar_init(&u_full[s], 1);
        }
        for (int b = 0; b < kDmmaRedBufs; ++b) {
            mbar_init(&red_full[b], (uint32_t)nc);
            mbar_init(&red_empty[b], 1);
        }
        for (int b = 0; b < kDmmaRecvBufs; ++b) {
            mbar_init(&rbar[b], 1);
            mbar_init(&credit[b], csize);
        }
        fence_mbar_init();
    }
    __syncthreads();
    fence_proxy_async();
    // everything above overlaps the predecessor kernel (programmatic launch); from here on we read
    // what it wrote (the guard flag, V, P)
    if (a.guard && !*a.guard) {  // uniform across the grid: no remote traffic has started
        if (MODE == kModeHv && a.tail == kTailCg && blockIdx.x == 0 && threadIdx.x == 0) {
            DevState* st = a.st;  // the CG iteration is switched off: its tail's bookkeeping
            st->cg_mid[a.cg_it] = 0;
            st->cg_act[a.cg_it + 1] = 0;
            st->cert_act = st->it_act && !st->cg_failed;
        }
        return;
    }
    // certificate pass: the grid always runs the tail (fallback / slope); the product itself only when
    // CG did not fail (src/newton.cpp:52)
    if (MODE == kModeHv && a.tail == kTailCert && !a.st->cert_act) T = 0;
    if (csize > 1) cluster_sync_all();  // peers' barriers are initialised before any remote traffic
    if (threadIdx.x == 0) DMMA_KST(1);

    auto tile_of = [&](int i) -> int64_t { return (int64_t)cid + (int64_t)i * ncl; };
    const int role_pusher = nc, role_producer = nc + 1, role_epi0 = nc + 2;

    if (warp == role_producer) {
        // ============================== producer: TMA ==============================
        if (lane == 0) {
            for (int i = 0; i < T; ++i) {
                const int stage = i % STAGES;
                if (i == 1) DMMA_KST(2);
                if (i >= STAGES) mbar_wait(&empty[stage], (uint32_t)(((i / STAGES) - 1) & 1));
                const int64_t r0 = tile_of(i) * BM;
                const int rows = (n - r0) < BM ? (int)(n - r0) : BM;
                uint32_t bytes = row_bytes * (uint32_t)rows;
                if (NEED_P) bytes += BM * K * 8;
                if (NEED_Y) bytes += BM * 4;
                fence_proxy_async();
                mbar_expect_tx(&full[stage], bytes);
                if (row_bytes)
                    for (int r = 0; r < rows; ++r)
                        tma_bulk_g2s(xs + ((size_t)stage * BM + r) * S, a.X + (r0 + r) * a.ldx + f_cta, row_bytes,
                                     &full[stage]);
                if (NEED_P) tma_bulk_g2s(ps + (size_t)stage * BM * KE, a.Pin + r0 * K, BM * K * 8, &full[stage]);
                if (NEED_Y) tma_bulk_g2s(ys + stage * BM, a.labels + r0, BM * 4, &full[stage]);
            }
        }
    } else if (warp == role_pusher) {
        // ============================== pusher: CTA partial -> cluster ==============================
        for (int i = 0; i < T; ++i) {
            const int b = i % kDmmaRedBufs, br = i % kDmmaRecvBufs;
            mbar_wait(&red_full[b], (uint32_t)((i / kDmmaRedBufs) & 1));
            DMMA_TRACE(i, 2);
            // every CTA of the cluster released receive buffer br (its previous tile's epilogue is done)
            if (i >= kDmmaRecvBufs) mbar_wait(&credit[br], (uint32_t)(((i / kDmmaRecvBufs) - 1) & 1));
            DMMA_TRACE(i, 13);
            const double* rd = red + (size_t)b * nc * PART;
            const uint32_t dst_local = smem_u32(recv + ((size_t)br * csize + crank) * PART);
            const uint32_t bar_local = smem_u32(&rbar[br]);
            // all of this lane's pairs are loaded first and their trees summed together: independent
            // chains hide the FP64 pipe's latency under the compute warps' DMMAs
            constexpr int NPAIR = (PART / 2 + 31) / 32;
            double s0[NPAIR], s1[NPAIR];
#pragma unroll
            for (int j = 0; j < NPAIR; ++j) s0[j] = s1[j] = 0.0;
            constexpr int NGRP = (dmma_max_compute(MT) + 7) / 8;
#pragma unroll
            for (int gw = 0; gw < NGRP; ++gw) {  // groups of 8 warps, each summed as a fixed tree
                const int w0 = 8 * gw;
                if (w0 >= nc) break;
                double v0[NPAIR][8], v1[NPAIR][8];
#pragma unroll
                for (int j = 0; j < NPAIR; ++j) {
                    const int i2 = lane + 32 * j;
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        double2 v = make_double2(0.0, 0.0);
                        if (w0 + w < nc && i2 < PART / 2)
                            v = *reinterpret_cast<const double2*>(rd + (size_t)(w0 + w) * PART + 2 * i2);
                        v0[j][w] = v.x;
                        v1[j][w] = v.y;
                    }
                }
#pragma unroll
                for (int j = 0; j < NPAIR; ++j) {
                    s0[j] = s0[j] + tree_sum(v0[j], nc - w0);
                    s1[j] = s1[j] + tree_sum(v1[j], nc - w0);
                }
            }
#pragma unroll
            for (int j = 0; j < NPAIR; ++j) {
                const int i2 = lane + 32 * j;
                if (i2 >= PART / 2) continue;
                *reinterpret_cast<double2*>(sendb + (size_t)br * PART + 2 * i2) = make_double2(s0[j], s1[j]);
            }
            DMMA_TRACE(i, 14);
            // the summed partial goes to every peer as one bulk copy each (lane q -> CTA q); the send
            // buffer br is rewritten only after every peer returned its credit for br
            fence_proxy_async();
            __syncwarp();
            if (lane < (int)csize)
                bulk_s2cluster(mapa(dst_local, (uint32_t)lane), smem_u32(sendb + (size_t)br * PART), PART * 8u,
                               mapa(bar_local, (uint32_t)lane));
            __syncwarp();
            DMMA_TRACE(i, 3);
            if (lane == 0) mbar_arrive(&red_empty[b]);
        }
    } else if (warp >= role_epi0) {
        // ============================== epilogue warps ==============================
        // Warp e owns tiles i == e (mod kDmmaEpiWarps): each tile's epilogue is a short dependent chain
        // of FP64 ops that queue behind the compute warps' DMMAs, so tiles are processed in parallel
        // by independent warps rather than cooperatively.
        const int ew = warp - role_epi0;
        double* lgw = lgb + (size_t)ew * BM * KP;  // this warp's full-logit tile
        double loss_acc = 0.0;                     // row lanes of the rank-0 CTA
        constexpr int NE = (BM * K + 31) / 32;     // elements per lane in pass 1
        for (int i = ew; i < T; i += kDmmaEpiWarps) {
            const int stage = i % STAGES, br = i % kDmmaRecvBufs;
            const int64_t r0 = tile_of(i) * BM;
            if (lane == 0) mbar_expect_tx(&rbar[br], (uint32_t)csize * PART * 8u);
            mbar_wait(&rbar[br], (uint32_t)((i / kDmmaRecvBufs) & 1));
            if (ew == 0) DMMA_TRACE(i, 4);
            if (NEED_P || NEED_Y) mbar_wait(&full[stage], (uint32_t)((i / STAGES) & 1));
            if (ew == 0) DMMA_TRACE(i, 8);
            // (1) full logits: sum of the CS partials in a fixed rank-order tree, all lanes' elements
            //     loaded first so the trees of one lane are independent
            const double* rv = recv + (size_t)br * csize * PART;
            {
                double v[NE][8];
#pragma unroll
                for (int j = 0; j < NE; ++j) {
                    const int e = lane + 32 * j;
                    const int row = e / K, c = e - row * K;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        v[j][q] = (e < BM * K && q < (int)csize) ? rv[(size_t)q * PART + row * KP + c] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < NE; ++j) {
                    const int e = lane + 32 * j;
                    const double s = tree_sum(v[j], (int)csize);
                    if (e < BM * K) lgw[(e / K) * KP + (e % K)] = s;
                }
            }
            __syncwarp();
            if (ew == 0) DMMA_TRACE(i, 9);
            // receive buffer br consumed: return one credit to every CTA of the cluster
            if (lane == 0)
                for (uint32_t q = 0; q < csize; ++q) mbar_arrive_remote(&credit[br], q);
            if (ew == 0) DMMA_TRACE(i, 11);
            // (2) row epilogue. Hv / Lp: one lane per row.
            if (MODE == kModeHv || MODE == kModeLp) {
                if (lane < BM) {
                    const int row = lane;
                    const int64_t gi = r0 + row;
                    const bool valid = gi < n;
                    const double* lg = lgw + row * KP;
                    double* urow = ut + (size_t)stage * BM * KS + row * KS;
                    if (MODE == kModeHv) {
                        const double* pr = ps + (size_t)stage * BM * KE + row * K;
                        if (valid) {
                            constexpr int KT2 = K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : K <= 16 ? 16 : 32;
                            double vw[KT2], pv[K], vt[KT2];
#pragma unroll
                            for (int c = 0; c < KT2; ++c) {
                                vw[c] = 0.0;
                                if (c < K) {
                                    pv[c] = pr[c];
                                    vw[c] = lg[c] * pv[c];
                                }
                                vt[c] = vw[c];
                            }
                            const double rs = tree_sum(vt, K);  // row_sum(V o P)
#pragma unroll
                            for (int c = 0; c < K; ++c) urow[c] = vw[c] - pv[c] * rs;
                            if (a.lp_out && crank == 0)
#pragma unroll
                                for (int c = 0; c < K; ++c) a.lp_out[gi * K + c] = lg[c];
                        } else {
#pragma unroll
                            for (int c = 0; c < K; ++c) urow[c] = 0.0;
                        }
                    } else if (MODE == kModeLp) {
                        if (valid && crank == 0)
#pragma unroll
                            for (int c = 0; c < K; ++c) a.Lp[gi * K + c] = lg[c];
                    }
                }
            } else {
                // stable softmax cache / loss / argmax (src/softmax.cpp:51-95, 118-139): four lanes
                // per row, lane q owning classes q, q+4, ...; row max / sums by quad butterflies
                const int row = lane >> 2, q = lane & 3;
                const int64_t gi = r0 + row;
                const bool valid = gi < n;
                const double* lg = lgw + row * KP;
                double* urow = ut + (size_t)stage * BM * KS + row * KS;
                constexpr int CPL = (K + 3) / 4;
                double lv[CPL], e[CPL];
                double m = -INFINITY;
#pragma unroll
                for (int t = 0; t < CPL; ++t) {
                    const int c = q + 4 * t;
                    lv[t] = c < K ? lg[c] : -INFINITY;
                    m = lv[t] > m ? lv[t] : m;
                }
                m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
                m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
                m = m > 0.0 ? m : 0.0;
                double es = 0.0;
#pragma unroll
                for (int t = 0; t < CPL; ++t) {
                    e[t] = (q + 4 * t < K) ? exp(lv[t] - m) : 0.0;
                    es += e[t];
                }
                es += __shfl_xor_sync(0xffffffffu, es, 1);
                es += __shfl_xor_sync(0xffffffffu, es, 2);
                const double alpha = exp(-m) + es;
                const int yb = ys[stage * BM + row];
                if (MODE == kModeCache || MODE == kModeValue) {
                    if (q == 0 && valid && crank == 0)
                        loss_acc += (m + log(alpha)) - (yb <= K ? lg[yb - 1] : 0.0);
                    if (MODE == kModeCache) {
#pragma unroll
                        for (int t = 0; t < CPL; ++t) {
                            const int c = q + 4 * t;
                            if (c < K) {
                                const double pc = e[t] / alpha;
                                urow[c] = valid ? ((c == yb - 1) ? pc - 1.0 : pc) : 0.0;
                                if (valid && crank == 0) {
                                    a.L0[gi * K + c] = lg[c];
                                    a.P[gi * K + c] = pc;
                                }
                            }
                        }
                        if (q == 0 && valid && crank == 0) {
                            a.rowM[gi] = m;
                            a.rowA[gi] = alpha;
                        }
                    }
                } else if (MODE == kModePredict) {
                    double best = -INFINITY;
#pragma unroll
                    for (int t = 0; t < CPL; ++t)
                        if (q + 4 * t < K) best = fmax(best, e[t] / alpha);
                    best = fmax(best, __shfl_xor_sync(0xffffffffu, best, 1));
                    best = fmax(best, __shfl_xor_sync(0xffffffffu, best, 2));
                    int arg = 1 << 20;  // first class attaining the max (src/softmax.cpp:127-135)
#pragma unroll
                    for (int t = CPL - 1; t >= 0; --t)
                        if (q + 4 * t < K && e[t] / alpha == best) arg = q + 4 * t;
                    arg = min(arg, __shfl_xor_sync(0xffffffffu, arg, 1));
                    arg = min(arg, __shfl_xor_sync(0xffffffffu, arg, 2));
                    arg += 1;
                    if (exp(-m) / alpha > best) arg = K + 1;  // class C only if strictly greater
                    if (q == 0 && valid && crank == 0) {
                        a.pred[gi] = arg;
                        loss_acc += (arg == yb) ? 1.0 : 0.0;
                    }
                }
            }
            __syncwarp();  // U rows complete, lgw reusable
            if (ew == 0) DMMA_TRACE(i, 12);
            if (lane == 0) {
                if (ew == 0) DMMA_TRACE(i, 5);
                if (PHASE_B) mbar_arrive(&u_full[stage]);
                mbar_arrive(&empty[stage]);
            }
        }
        // cluster's loss / hit partial (rank-0 CTA): rows of warp 0's tiles, then warp 1's, ...
        if (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) {
            misc[ew * 32 + lane] = loss_acc;
            named_sync(1, 32 * kDmmaEpiWarps);
            if (ew == 0 && lane == 0 && crank == 0) {
                double s = 0.0;
                for (int q = 0; q < 32 * kDmmaEpiWarps; ++q) s += misc[q];
                const int slotid = MODE == kModePredict ? kSlotHits : kSlotLoss;
                a.blk[(int64_t)slotid * kBlockPartials + cid] = s;
            }
        }
    } else {
        // ============================== compute warps ==============================
        const int fw = warp * W;  // warp slice offset inside the CTA slice
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
        double accb[PHASE_B ? MT : 1][KT > 0 ? KT : 1][2];
        double accbr[PHASE_B ? MT : 1][R > 0 ? R : 1];
#pragma unroll
        for (int m = 0; m < (PHASE_B ? MT : 1); ++m) {
#pragma unroll
            for (int kt = 0; kt < (KT > 0 ? KT : 1); ++kt) accb[m][kt][0] = accb[m][kt][1] = 0.0;
#pragma unroll
            for (int r = 0; r < (R > 0 ? R : 1); ++r) accbr[m][r] = 0.0;
        }

        auto phase_a = [&](int i) {
            const int stage = i % STAGES, b = i % kDmmaRedBufs;
            mbar_wait(&full[stage], (uint32_t)((i / STAGES) & 1));
            if (warp == 0) DMMA_TRACE(i, 0);
            if (i == 0 && warp == 0 && lane == 0) DMMA_KST(3);
            const double* xt = xs + (size_t)stage * BM * S;
            // NCH independent DMMA accumulator chains over the k-steps: a dependent DMMA waits behind the
            // other warps' DMMAs in the shared FP64 pipe, so short chains keep phase A throughput-bound
            constexpr int NCH = (KSTEP_A % kDmmaChains == 0) ? kDmmaChains : ((KSTEP_A % 2 == 0) ? 2 : 1);
            double acca[NCH][G][KT > 0 ? KT : 1][2];
            // remainder classes on DFMA: 4 independent chains per row group (a dependent DFMA queues
            // behind the DMMAs sharing the FP64 pipe, so one 12-long chain would serialise phase A)
            constexpr int RC = 4;
            double accar[RC][G][R > 0 ? R : 1];
#pragma unroll
            for (int h = 0; h < NCH; ++h)
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int kt = 0; kt < (KT > 0 ? KT : 1); ++kt) acca[h][g][kt][0] = acca[h][g][kt][1] = 0.0;
#pragma unroll
            for (int h = 0; h < RC; ++h)
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int r = 0; r < (R > 0 ? R : 1); ++r) accar[h][g][r] = 0.0;
#pragma unroll
            for (int s = 0; s < KSTEP_A; ++s) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double x = xt[(g * 8 + gq) * S + fw + 4 * s + tq];
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) dmma(acca[s % NCH][g][kt], x, bv[s][kt]);
#pragma unroll
                    for (int r = 0; r < R; ++r) accar[s % RC][g][r] = fma(x, vr[s][r], accar[s % RC][g][r]);
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double v = (accar[0][g][r] + accar[1][g][r]) + (accar[2][g][r] + accar[3][g][r]);
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    accar[0][g][r] = v;
                }
#pragma unroll
            for (int w = 1; w < NCH; w *= 2)  // fixed pairwise fold of the chains into chain 0
#pragma unroll
                for (int h = 0; h + w < NCH; h += 2 * w)
#pragma unroll
                    for (int g = 0; g < G; ++g)
#pragma unroll
                        for (int kt = 0; kt < KT; ++kt) {
                            acca[h][g][kt][0] = acca[h][g][kt][0] + acca[h + w][g][kt][0];
                            acca[h][g][kt][1] = acca[h][g][kt][1] + acca[h + w][g][kt][1];
                        }
            if (i >= kDmmaRedBufs) mbar_wait(&red_empty[b], (uint32_t)(((i / kDmmaRedBufs) - 1) & 1));
            double* rw = red + ((size_t)b * nc + warp) * PART;
#pragma unroll
            for (int g = 0; g < G; ++g) {
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) {
                    const int o = (g * 8 + gq) * KP + kt * 8 + 2 * tq;
                    *reinterpret_cast<double2*>(rw + o) =
                        make_double2(acca[0][g][kt][0], acca[0][g][kt][1]);
                }
                if (tq == 0)
#pragma unroll
                    for (int r = 0; r < R; ++r) rw[(g * 8 + gq) * KP + 8 * KT + r] = accar[0][g][r];
            }
            __syncwarp();
            if (warp == 0) DMMA_TRACE(i, 1);
            if (lane == 0) mbar_arrive(&red_full[b]);
        };

        for (int i = 0; i < LAG && i < T; ++i) phase_a(i);
        for (int i = 0; i < T; ++i) {
            const int stage = i % STAGES;
            if (i + LAG < T) phase_a(i + LAG);
            if (PHASE_B) {
                mbar_wait(&u_full[stage], (uint32_t)((i / STAGES) & 1));
                if (warp == 0) DMMA_TRACE(i, 6);
                const double* xt = xs + (size_t)stage * BM * S;
                const double* utb = ut + (size_t)stage * BM * KS;
                const int64_t rows_left = n - tile_of(i) * BM;  // rows of this tile beyond n read as 0
#pragma unroll
                for (int s = 0; s < BM / 4; ++s) {
                    const int row = 4 * s + tq;
                    const bool rv = row < rows_left;
                    double ub[KT > 0 ? KT : 1], ur[R > 0 ? R : 1];
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) ub[kt] = utb[row * KS + kt * 8 + gq];
#pragma unroll
                    for (int r = 0; r < R; ++r) ur[r] = utb[row * KS + 8 * KT + r];
                    const double* xr = xt + (size_t)row * S + fw;
#pragma unroll
                    for (int mp = 0; mp < MT / 2; ++mp) {
                        const double2 x2 =
                            rv ? *reinterpret_cast<const double2*>(xr + mp * 16 + 2 * gq) : make_double2(0.0, 0.0);
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
                        const double x = rv ? xr[(MT - 1) * 8 + gq] : 0.0;
#pragma unroll
                        for (int kt = 0; kt < KT; ++kt) dmma(accb[MT - 1][kt], x, ub[kt]);
#pragma unroll
                        for (int r = 0; r < R; ++r) accbr[MT - 1][r] = fma(x, ur[r], accbr[MT - 1][r]);
                    }
                }
            }
            __syncwarp();
            if (warp == 0) DMMA_TRACE(i, 7);
            if (lane == 0) mbar_arrive(&empty[stage]);
        }

        if (warp == 0 && lane == 0) DMMA_KST(4);
        // ---------------- this cluster's split-K partial of X^T U ----------------
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
    }
    if (threadIdx.x == 0) DMMA_KST(5);
    __syncthreads();
    if (csize > 1) cluster_sync_all();  // no CTA leaves while peers may still target its shared memory
    if (threadIdx.x == 0) DMMA_KST(6);
    if (PHASE_B && a.tail != kTailNone) {
        // all clusters' partials (and loss slots) written -> the whole (co-resident) grid runs the tail
        grid_barrier(a.done_ctr);
        const int64_t d = (int64_t)K * p;
        if (MODE == kModeHv && a.tail == kTailCg)
            dmma_cg_tail(a, K, (int)ncl, misc, misc + 127, whole_grid(), a.done_ctr);
        else if (MODE == kModeHv && a.tail == kTailCert) {
            const bool lp_need = cert_tail_body(d, a.st, a.prm, a.part, (int)ncl, a.lp_from_cert, a.g, a.cg_p,
                                                a.cg_hd, a.blk, (int)ncl, a.hv_ctr, a.done_ctr, misc, misc + 127,
                                                whole_grid());
            // the Armijo search needs only L0 and this pass's Lp = X p: run it here unless p changed
            if (a.st->it_act && !lp_need)
                ls_fused_body(n, K, a.L0, a.Lp, a.labels, d, const_cast<double*>(a.x), a.cg_p, a.z, a.y, a.prm, a.st,
                              a.blk, a.done_ctr, xs, misc + 126, whole_grid());  // the X ring is free: scratch
        }
        else if (MODE == kModeCache && a.tail == kTailNewton)
            newton_tail_body(d, a.st, a.prm, a.part, (int)ncl, a.x, a.z, a.y, a.gbase, a.g, a.t, a.blk, (int)ncl,
                             a.scal, a.trace, a.trace_cap, a.done_ctr, misc, whole_grid());
    }
    if (threadIdx.x == 0) DMMA_KST(7);
}

}  // namespace nadmm
