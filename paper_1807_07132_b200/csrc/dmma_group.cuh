// Node-group form of the fused DMMA pass (device code): ONE persistent full-GPU launch applies the
// pass to every local ADMM node of an outer iteration (the bench's 8 nodes per GPU), instead of one
// launch per node on a 1/k-GPU grid. Same cluster design as dmma_pass_kernel (dmma_kernel.cuh):
// producer / pusher / epilogue / compute warps, DSMEM logit exchange, X read from HBM once.
// What the group adds:
//   * the row tiles of all ACTIVE nodes (guard on; certificate passes: CG did not fail) are
//     concatenated and dealt to the clusters round-robin like the single pass's (balanced over the
//     nodes still running; every node has >= one tile per cluster, so each cluster writes one split-K
//     partial per active node: slot = cluster id); every role maps a tile to (node, local tile)
//     with the same table;
//   * the compute warps reload their register-resident V slice when phase A crosses into the next
//     node and write the phase-B accumulators as one split-K partial of the node they leave
//     (slot = cluster id: the node's tail sums them in cluster order, deterministic);
//   * after a whole-grid barrier each node's solver tail (CG step / certificate + line search /
//     Newton tail) runs on its own sub-grid of CTAs with its own barrier counter (VGrid).
#pragma once

#include "dmma_kernel.cuh"

namespace nadmm {

constexpr int kMaxGroup = 8;

struct DmmaGroup {
    DmmaArgs node[kMaxGroup];  // per node: same p, K and layout (fs, S)
    int n;                     // nodes in the group
    int sub_start[kMaxGroup + 1];  // CTA sub-grid of each node's tail
    unsigned long long* grid_ctr;  // whole-grid barrier before the tails
};

template <int MT, int LAG, int STAGES, int MODE>
__global__ void __launch_bounds__(dmma_max_threads(MT), 1) dmma_group_kernel(const __grid_constant__ DmmaGroup G) {
    using namespace dmma_detail;
    constexpr int KT = 1, R = 1, BM = 8;
    static_assert(STAGES >= LAG + 2, "ring depth");
    static_assert(MODE == kModeHv || MODE == kModeCache, "group passes: Hv (CG / certificate) and cache");
    constexpr int K = 8 * KT + R;
    constexpr int KS = DmmaSmem<K>::KS;
    constexpr int KP = DmmaSmem<K>::KP;
    constexpr int KE = (K + 1) & ~1;
    constexpr int W = 8 * MT;
    constexpr int KSTEP_A = W / 4;
    constexpr bool NEED_P = (MODE == kModeHv);
    constexpr bool NEED_Y = (MODE == kModeCache);
    constexpr int G8 = BM / 8;
    constexpr int PART = BM * KP;
    extern __shared__ __align__(128) double smem[];
    __shared__ int64_t s_start[kMaxGroup + 1];  // active-tile prefix per node
    __shared__ int s_on[kMaxGroup];             // node runs tiles in this launch
    __shared__ int s_cfirst[kMaxGroup], s_chunks[kMaxGroup];
    __shared__ double s_loss[kMaxGroup][32 * kDmmaEpiWarps];
    // hot per-node fields copied out of the (2.7 KB) parameter block: the tile loops read them from
    // shared memory instead of indexing the kernel parameters with a runtime node id
    struct NodeHot {
        const double* X;
        int64_t ldx, n;
        const double *Pin, *V;
        const int32_t* labels;
        double *part, *lp_out, *L0, *P, *rowM, *rowA;
    };
    __shared__ NodeHot s_node[kMaxGroup];
    // per ring stage: the node and first local row of the tile the producer loaded there (consumers
    // read it after their full / u_full wait instead of searching the node table)
    __shared__ int s_tile_k[STAGES];
    __shared__ int64_t s_tile_r0[STAGES];
    const DmmaArgs& a0 = G.node[0];
    const int nc = (int)(blockDim.x >> 5) - kDmmaAux;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;
    const uint32_t crank = cluster_ctarank(), csize = cluster_nctarank();
    const uint32_t cid = cluster_id_x(), ncl = ncluster_x();
    const int S = a0.S, fs = a0.fs;
    const int64_t p = a0.p;
    const int f_cta = (int)crank * fs;
    const int tail = a0.tail;

    double* xs = smem;
    double* ps = xs + (size_t)STAGES * BM * S;
    double* red = ps + (size_t)STAGES * BM * KE;
    double* recv = red + (size_t)kDmmaRedBufs * nc * PART;
    double* sendb = recv + (size_t)kDmmaRecvBufs * csize * PART;
    double* ut = sendb + (size_t)kDmmaRecvBufs * PART;
    double* lgb = ut + (size_t)STAGES * BM * KS;
    double* misc = lgb + (size_t)kDmmaEpiWarps * BM * KP;
    int32_t* ys = reinterpret_cast<int32_t*>(misc + 128);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ys + STAGES * BM + 4);
    uint64_t* full = bars;
    uint64_t* empty = full + STAGES;
    uint64_t* red_full = empty + STAGES;
    uint64_t* red_empty = red_full + kDmmaRedBufs;
    uint64_t* rbar = red_empty + kDmmaRedBufs;
    uint64_t* credit = rbar + kDmmaRecvBufs;
    uint64_t* u_full = credit + kDmmaRecvBufs;

    const int64_t rem_f = p - f_cta;
    const int valid_f = rem_f <= 0 ? 0 : (rem_f < fs ? (int)rem_f : fs);
    const uint32_t row_bytes = (uint32_t)valid_f * 8u;
    if (valid_f < fs)
        for (int i = threadIdx.x; i < STAGES * BM * S; i += blockDim.x) xs[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (uint32_t)(nc + 1));
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
        // the partition of the active nodes' tiles over the clusters (identical in every CTA)
        int64_t acc = 0;
        for (int k = 0; k < G.n; ++k) {
            const DmmaArgs& A = G.node[k];
            int on = (A.guard == nullptr) || (*A.guard != 0);
            if (MODE == kModeHv && tail == kTailCert) on = on && A.st->cert_act;
            s_on[k] = on;
            s_start[k] = acc;
            if (on) acc += (A.n + BM - 1) / BM;
        }
        s_start[G.n] = acc;
        for (int k = 0; k < G.n; ++k) {
            const DmmaArgs& A = G.node[k];
            s_node[k] = NodeHot{A.X, A.ldx, A.n, A.Pin, A.V, A.labels, A.part, A.lp_out, A.L0, A.P, A.rowM, A.rowA};
        }
        for (int k = 0; k < G.n; ++k) {  // strided tiles: every cluster writes a partial of every active node
            s_cfirst[k] = 0;
            s_chunks[k] = (s_on[k] && acc > 0) ? (int)ncl : 0;
        }
        for (int k = 0; k < kMaxGroup; ++k)
            for (int q = 0; q < 32 * kDmmaEpiWarps; ++q) s_loss[k][q] = 0.0;
    }
    __syncthreads();
    fence_proxy_async();
    const int64_t total = s_start[G.n];
    const int T = (int64_t)cid < total ? (int)((total - 1 - cid) / ncl + 1) : 0;  // tiles cid, cid + ncl, ...
    if (csize > 1) cluster_sync_all();

    // tile i of this cluster -> (node, first row of the tile in that node)
    // (callers pass increasing i, so k only moves forward: start the search at the caller's last k)
    const int nn = G.n;
    auto locate = [&](int i, int& k, int64_t& r0) {
        const int64_t q = (int64_t)cid + (int64_t)i * ncl;
        if (k < 0 || s_start[k] > q) k = 0;
        while (k + 1 < nn && s_start[k + 1] <= q) ++k;
        r0 = (q - s_start[k]) * BM;
    };
    const int role_pusher = nc, role_producer = nc + 1, role_epi0 = nc + 2;

    if (warp == role_producer) {
        if (lane == 0) {
            int k = -1;
            for (int i = 0; i < T; ++i) {
                const int stage = i % STAGES;
                int64_t r0;
                locate(i, k, r0);
                const NodeHot& A = s_node[k];
                if (i >= STAGES) mbar_wait(&empty[stage], (uint32_t)(((i / STAGES) - 1) & 1));
                const int rows = (A.n - r0) < BM ? (int)(A.n - r0) : BM;
                uint32_t bytes = row_bytes * (uint32_t)rows;
                if (NEED_P) bytes += BM * K * 8;
                if (NEED_Y) bytes += BM * 4;
                s_tile_k[stage] = k;
                s_tile_r0[stage] = r0;
                fence_proxy_async();
                mbar_expect_tx(&full[stage], bytes);
                if (row_bytes)
                    for (int r = 0; r < rows; ++r)
                        tma_bulk_g2s(xs + ((size_t)stage * BM + r) * S, A.X + (r0 + r) * A.ldx + f_cta, row_bytes,
                                     &full[stage]);
                if (NEED_P) tma_bulk_g2s(ps + (size_t)stage * BM * KE, A.Pin + r0 * K, BM * K * 8, &full[stage]);
                if (NEED_Y) tma_bulk_g2s(ys + stage * BM, A.labels + r0, BM * 4, &full[stage]);
            }
        }
    } else if (warp == role_pusher) {
        for (int i = 0; i < T; ++i) {
            const int b = i % kDmmaRedBufs, br = i % kDmmaRecvBufs;
            mbar_wait(&red_full[b], (uint32_t)((i / kDmmaRedBufs) & 1));
            if (i >= kDmmaRecvBufs) mbar_wait(&credit[br], (uint32_t)(((i / kDmmaRecvBufs) - 1) & 1));
            const double* rd = red + (size_t)b * nc * PART;
            const uint32_t dst_local = smem_u32(recv + ((size_t)br * csize + crank) * PART);
            const uint32_t bar_local = smem_u32(&rbar[br]);
            constexpr int NPAIR = (PART / 2 + 31) / 32;
            double s0[NPAIR], s1[NPAIR];
#pragma unroll
            for (int j = 0; j < NPAIR; ++j) s0[j] = s1[j] = 0.0;
            {
                double v0[NPAIR][8], v1[NPAIR][8];
#pragma unroll
                for (int j = 0; j < NPAIR; ++j) {
                    const int i2 = lane + 32 * j;
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        double2 v = make_double2(0.0, 0.0);
                        if (w < nc && i2 < PART / 2) v = *reinterpret_cast<const double2*>(rd + (size_t)w * PART + 2 * i2);
                        v0[j][w] = v.x;
                        v1[j][w] = v.y;
                    }
                }
#pragma unroll
                for (int j = 0; j < NPAIR; ++j) {
                    s0[j] = s0[j] + tree_sum(v0[j], nc);
                    s1[j] = s1[j] + tree_sum(v1[j], nc);
                }
            }
#pragma unroll
            for (int j = 0; j < NPAIR; ++j) {
                const int i2 = lane + 32 * j;
                if (i2 < PART / 2)
                    *reinterpret_cast<double2*>(sendb + (size_t)br * PART + 2 * i2) = make_double2(s0[j], s1[j]);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane < (int)csize)
                bulk_s2cluster(mapa(dst_local, (uint32_t)lane), smem_u32(sendb + (size_t)br * PART), PART * 8u,
                               mapa(bar_local, (uint32_t)lane));
            __syncwarp();
            if (lane == 0) mbar_arrive(&red_empty[b]);
        }
    } else if (warp >= role_epi0) {
        const int ew = warp - role_epi0;
        double* lgw = lgb + (size_t)ew * BM * KP;
        double loss_acc = 0.0;
        int loss_node = -1;
        constexpr int NE = (BM * K + 31) / 32;
        for (int i = ew; i < T; i += kDmmaEpiWarps) {
            const int stage = i % STAGES, br = i % kDmmaRecvBufs;
            if (lane == 0) mbar_expect_tx(&rbar[br], (uint32_t)csize * PART * 8u);
            mbar_wait(&rbar[br], (uint32_t)((i / kDmmaRecvBufs) & 1));
            mbar_wait(&full[stage], (uint32_t)((i / STAGES) & 1));
            const int k = s_tile_k[stage];
            const int64_t r0 = s_tile_r0[stage];
            const NodeHot& A = s_node[k];
            if (MODE == kModeCache && k != loss_node) {  // the node's loss share (rank-0 CTA rows)
                if (loss_node >= 0) s_loss[loss_node][ew * 32 + lane] += loss_acc;
                loss_acc = 0.0;
                loss_node = k;
            }
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
            if (lane == 0)
                for (uint32_t q = 0; q < csize; ++q) mbar_arrive_remote(&credit[br], q);
            if (MODE == kModeHv) {
                if (lane < BM) {
                    const int row = lane;
                    const int64_t gi = r0 + row;
                    const bool valid = gi < A.n;
                    const double* lg = lgw + row * KP;
                    double* urow = ut + (size_t)stage * BM * KS + row * KS;
                    const double* pr = ps + (size_t)stage * BM * KE + row * K;
                    if (valid) {
                        double vw[16], pv[K], vt[16];
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            vw[c] = 0.0;
                            if (c < K) {
                                pv[c] = pr[c];
                                vw[c] = lg[c] * pv[c];
                            }
                            vt[c] = vw[c];
                        }
                        const double rs = tree_sum(vt, K);
#pragma unroll
                        for (int c = 0; c < K; ++c) urow[c] = vw[c] - pv[c] * rs;
                        if (A.lp_out && crank == 0)
#pragma unroll
                            for (int c = 0; c < K; ++c) A.lp_out[gi * K + c] = lg[c];
                    } else {
#pragma unroll
                        for (int c = 0; c < K; ++c) urow[c] = 0.0;
                    }
                }
            } else {  // cache: stable softmax, loss, coeff = P - Y (src/softmax.cpp:51-95)
                const int row = lane >> 2, q = lane & 3;
                const int64_t gi = r0 + row;
                const bool valid = gi < A.n;
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
                if (q == 0 && valid && crank == 0) loss_acc += (m + log(alpha)) - (yb <= K ? lg[yb - 1] : 0.0);
#pragma unroll
                for (int t = 0; t < CPL; ++t) {
                    const int c = q + 4 * t;
                    if (c < K) {
                        const double pc = e[t] / alpha;
                        urow[c] = valid ? ((c == yb - 1) ? pc - 1.0 : pc) : 0.0;
                        if (valid && crank == 0) {
                            A.L0[gi * K + c] = lg[c];
                            A.P[gi * K + c] = pc;
                        }
                    }
                }
                if (q == 0 && valid && crank == 0) {
                    A.rowM[gi] = m;
                    A.rowA[gi] = alpha;
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&u_full[stage]);
                mbar_arrive(&empty[stage]);
            }
        }
        if (MODE == kModeCache) {
            if (loss_node >= 0) s_loss[loss_node][ew * 32 + lane] += loss_acc;
            named_sync(1, 32 * kDmmaEpiWarps);
            if (ew == 0 && lane < G.n && crank == 0 && s_on[lane]) {
                // this cluster's share of node `lane`'s loss, in its partial slot (cluster order)
                const int k = lane;
                double s = 0.0;
                for (int q2 = 0; q2 < 32 * kDmmaEpiWarps; ++q2) s += s_loss[k][q2];
                G.node[k].blk[(int64_t)kSlotLoss * kBlockPartials + cid] = s;
            }
        }
    } else {
        // ============================== compute warps ==============================
        const int fw = warp * W;
        double bv[KSTEP_A][KT];
        double vr[KSTEP_A][R];
        auto load_v = [&](const double* V) {
#pragma unroll
            for (int s = 0; s < KSTEP_A; ++s) {
                const int64_t f = (int64_t)f_cta + fw + 4 * s + tq;
                const bool ok = f < p && fw + 4 * s + tq < fs;
                bv[s][0] = ok ? V[(int64_t)gq * p + f] : 0.0;
                vr[s][0] = ok ? V[(int64_t)8 * p + f] : 0.0;
            }
        };
        double accb[MT][KT][2];
        double accbr[MT][R];
        auto zero_b = [&]() {
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                accb[m][0][0] = accb[m][0][1] = 0.0;
                accbr[m][0] = 0.0;
            }
        };
        // phase-B accumulators of the node being left -> its split-K partial slot
        auto flush_b = [&](int k) {
            const NodeHot& A = s_node[k];
            const int64_t d = (int64_t)K * p;
            double* out = A.part + (int64_t)(cid - s_cfirst[k]) * d;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const int loc = (MT % 2 == 1 && m == MT - 1) ? (m * 8 + gq) : ((m / 2) * 16 + 2 * gq + (m & 1));
                const int64_t f = (int64_t)f_cta + fw + loc;
                const bool ok = f < p && fw + loc < fs;
                if (ok) {
                    out[(int64_t)(2 * tq) * p + f] = accb[m][0][0];
                    out[(int64_t)(2 * tq + 1) * p + f] = accb[m][0][1];
                }
                double v = accbr[m][0];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (ok && tq == 0) out[(int64_t)8 * p + f] = v;
            }
        };
        zero_b();
        int node_a = -1, node_b = -1;

        auto phase_a = [&](int i) {
            const int stage = i % STAGES, b = i % kDmmaRedBufs;
            mbar_wait(&full[stage], (uint32_t)((i / STAGES) & 1));
            const int k = s_tile_k[stage];
            if (k != node_a) {
                load_v(s_node[k].V);
                node_a = k;
            }
            const double* xt = xs + (size_t)stage * BM * S;
            constexpr int NCH = (KSTEP_A % kDmmaChains == 0) ? kDmmaChains : ((KSTEP_A % 2 == 0) ? 2 : 1);
            double acca[NCH][G8][KT][2];
            constexpr int RC = 4;
            double accar[RC][G8][R];
#pragma unroll
            for (int h = 0; h < NCH; ++h)
#pragma unroll
                for (int g = 0; g < G8; ++g) acca[h][g][0][0] = acca[h][g][0][1] = 0.0;
#pragma unroll
            for (int h = 0; h < RC; ++h)
#pragma unroll
                for (int g = 0; g < G8; ++g) accar[h][g][0] = 0.0;
#pragma unroll
            for (int s = 0; s < KSTEP_A; ++s) {
#pragma unroll
                for (int g = 0; g < G8; ++g) {
                    const double x = xt[(g * 8 + gq) * S + fw + 4 * s + tq];
                    dmma(acca[s % NCH][g][0], x, bv[s][0]);
                    accar[s % RC][g][0] = fma(x, vr[s][0], accar[s % RC][g][0]);
                }
            }
#pragma unroll
            for (int g = 0; g < G8; ++g) {
                double v = (accar[0][g][0] + accar[1][g][0]) + (accar[2][g][0] + accar[3][g][0]);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                accar[0][g][0] = v;
            }
#pragma unroll
            for (int w = 1; w < NCH; w *= 2)
#pragma unroll
                for (int h = 0; h + w < NCH; h += 2 * w)
#pragma unroll
                    for (int g = 0; g < G8; ++g) {
                        acca[h][g][0][0] = acca[h][g][0][0] + acca[h + w][g][0][0];
                        acca[h][g][0][1] = acca[h][g][0][1] + acca[h + w][g][0][1];
                    }
            if (i >= kDmmaRedBufs) mbar_wait(&red_empty[b], (uint32_t)(((i / kDmmaRedBufs) - 1) & 1));
            double* rw = red + ((size_t)b * nc + warp) * PART;
#pragma unroll
            for (int g = 0; g < G8; ++g) {
                const int o = (g * 8 + gq) * KP + 2 * tq;
                *reinterpret_cast<double2*>(rw + o) = make_double2(acca[0][g][0][0], acca[0][g][0][1]);
                if (tq == 0) rw[(g * 8 + gq) * KP + 8] = accar[0][g][0];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&red_full[b]);
        };

        for (int i = 0; i < LAG && i < T; ++i) phase_a(i);
        for (int i = 0; i < T; ++i) {
            const int stage = i % STAGES;
            if (i + LAG < T) phase_a(i + LAG);
            mbar_wait(&u_full[stage], (uint32_t)((i / STAGES) & 1));
            const int k = s_tile_k[stage];
            const int64_t r0 = s_tile_r0[stage];
            if (k != node_b) {
                if (node_b >= 0) {
                    flush_b(node_b);
                    zero_b();
                }
                node_b = k;
            }
            const double* xt = xs + (size_t)stage * BM * S;
            const double* utb = ut + (size_t)stage * BM * KS;
            const int64_t rows_left = s_node[k].n - r0;
#pragma unroll
            for (int s = 0; s < BM / 4; ++s) {
                const int row = 4 * s + tq;
                const bool rv = row < rows_left;
                const double ub = utb[row * KS + gq];
                const double ur = utb[row * KS + 8];
                const double* xr = xt + (size_t)row * S + fw;
#pragma unroll
                for (int mp = 0; mp < MT / 2; ++mp) {
                    const double2 x2 = rv ? *reinterpret_cast<const double2*>(xr + mp * 16 + 2 * gq) : make_double2(0.0, 0.0);
                    dmma(accb[2 * mp][0], x2.x, ub);
                    dmma(accb[2 * mp + 1][0], x2.y, ub);
                    accbr[2 * mp][0] = fma(x2.x, ur, accbr[2 * mp][0]);
                    accbr[2 * mp + 1][0] = fma(x2.y, ur, accbr[2 * mp + 1][0]);
                }
                if (MT & 1) {
                    const double x = rv ? xr[(MT - 1) * 8 + gq] : 0.0;
                    dmma(accb[MT - 1][0], x, ub);
                    accbr[MT - 1][0] = fma(x, ur, accbr[MT - 1][0]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
        }
        if (node_b >= 0) flush_b(node_b);
    }
    __syncthreads();
    if (csize > 1) cluster_sync_all();
    // ---------------- per-node solver tails on sub-grids ----------------
    grid_barrier_n(G.grid_ctr, gridDim.x);  // every node's partials (and loss slots) are written
    int k = 0;
    while (k + 1 < G.n && G.sub_start[k + 1] <= (int)blockIdx.x) ++k;
    const VGrid vg{(int)blockIdx.x - G.sub_start[k], G.sub_start[k + 1] - G.sub_start[k]};
    const DmmaArgs& A = G.node[k];
    const int64_t d = (int64_t)K * p;
    const int chunks = s_chunks[k];
    const bool guard_on = (A.guard == nullptr) || (*A.guard != 0);
    if (MODE == kModeHv && tail == kTailCg) {
        if (guard_on) {
            dmma_cg_tail(A, K, chunks, misc, misc + 127, vg, A.sub_ctr);
        } else if (vg.b == 0 && threadIdx.x == 0) {  // the switched-off CG iteration's bookkeeping
            DevState* st = A.st;
            st->cg_mid[A.cg_it] = 0;
            st->cg_act[A.cg_it + 1] = 0;
            st->cert_act = st->it_act && !st->cg_failed;
        }
    } else if (MODE == kModeHv && tail == kTailCert) {
        if (guard_on) {  // guard = it_act: the tail runs whether or not the certificate product did
            const bool lp_need = cert_tail_body(d, A.st, A.prm, A.part, chunks, A.lp_from_cert, A.g, A.cg_p, A.cg_hd,
                                                A.blk, chunks, A.hv_ctr, A.sub_ctr, misc, misc + 127, vg);
            if (A.st->it_act && !lp_need)
                ls_fused_body(A.n, K, A.L0, A.Lp, A.labels, d, const_cast<double*>(A.x), A.cg_p, A.z, A.y, A.prm, A.st,
                              A.blk, A.sub_ctr, xs, misc + 126, vg);
        }
    } else if (MODE == kModeCache && tail == kTailNewton) {
        if (guard_on)
            newton_tail_body(d, A.st, A.prm, A.part, chunks, A.x, A.z, A.y, A.gbase, A.g, A.t, A.blk, chunks, A.scal,
                             A.trace, A.trace_cap, A.sub_ctr, misc, vg);
    }
}

}  // namespace nadmm
