// CSR shards with C - 1 <= 32 (the E18/news20-like 20-class sparse config): nonzero-group passes.
//
// Both contractions of a sparse product gather a K-vector per nonzero -- the column's weights in the
// rows pass (X W), the row's U coefficients in the columns pass (X^T U through the CSC copy) -- so the
// pass is bound by L2 -> SM gather traffic (2 nnz K doubles per Hv), not by the CSR/CSC stream itself
// (12 B per nonzero each). The design minimises the gathered sectors and keeps every lane busy:
//   * the gathered tables (transposed weights wt = p x KS, U = n x KS) use a padded class stride KS
//     (sparse_class_stride), so a nonzero's K values are whole aligned words of VW doubles: 32-byte
//     words (sm_100 256-bit loads, VW = 4) when KS is a multiple of 4, else 16-byte double2 words
//     (K = 19: KS = 20, 160 B = 5 whole sectors = 5 lanes x 32 B);
//   * rows pass: a half-warp owns a row (two rows per warp); its lanes form G = 16 / (KS/VW) groups,
//     each group gathers one nonzero's words (K = 19: 3 groups per row, 30 of 32 lanes busy), each
//     lane issuing a quad's 4 gathers before their FMAs; group partial sums are folded into group 0 by
//     shuffles and the row epilogue (U / softmax cache / loss / argmax) runs on group 0's lanes with
//     16-lane butterfly reductions inside the half;
//   * columns pass (short CSC columns): each lane group owns a column and sums it sequentially -- no
//     fold, and one column's latency chain is shared by the warp's G columns;
//   * CSR row segments (per column block) and CSC columns are padded to quads of entries (weight-0
//     copies of the last entry, capi.cu); each lane loads its quads itself with one 16-byte index and
//     one 32-byte value load (one broadcast request per group; no shuffles in the gather loop), and the
//     next segment is bulk-prefetched into L2;
//   * grids are exactly one resident wave (4 blocks of 256 threads per SM).
// When the transposed weights exceed an L2-sized budget the rows pass runs once per column block
// (running logits in `lsum` between blocks) so each block's weights stay L2-resident.
//
// Reference ops (file:line under /root/reference/proj):
//   sparse X * B, X^T * B             src/dataset.cpp:69-85 (sparse_ * rhs, sparse_.transpose() * rhs)
//   cache / loss / coeff / Hv / predict  src/softmax.cpp:51-139
#include "state.h"

namespace nadmm {

namespace {

constexpr int kSpThreads = 256;
// Rows / columns grids: exactly one resident wave (4 blocks of 256 threads per SM at <= 64 registers,
// __launch_bounds__ below). cfg4 Hv: 3.07 ms at 4 per SM vs 3.23 / 3.54 / 4.74 ms at 8 / 3 / 2
// (two waves, or fewer warps in flight).
#ifndef NADMM_SP_BPSM
#define NADMM_SP_BPSM 4
#endif
constexpr int kSpBlocksPerSm = NADMM_SP_BPSM;

// One lane's VW-double word of a gathered table row (read-only path). VW = 4 is the sm_100 256-bit
// load (LDG.E.ENL2.256): a nonzero's 160-byte K = 19 row is 5 lanes x 32 B, half the requests of
// 16-byte words for the same sectors.
template <int VW>
__device__ __forceinline__ void ldg_word(const double* __restrict__ p, double (&o)[VW]) {
    if constexpr (VW == 4) {
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
                     : "l"(p));
    } else {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        o[0] = t.x;
        o[1] = t.y;
    }
}

// Bulk L2 prefetch (TMA unit, no registers) of bytes [a, a + n) widened to 16-byte granules: the warp's
// next CSR row / CSC column segment is pulled into L2 while the current one is gathered, so each
// 32-entry index / value chunk is an L2 hit instead of a DRAM round trip in front of its gathers.
__device__ __forceinline__ void prefetch_l2(const void* a, int64_t n) {
    if (n <= 0) return;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(a) + (uintptr_t)n + 15) & ~uintptr_t(15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
}

__device__ __forceinline__ void prefetch_segment(const int32_t* idx, const double* val, int64_t q0, int64_t q1) {
    prefetch_l2(idx + q0, 4 * (q1 - q0));
    prefetch_l2(val + q0, 8 * (q1 - q0));
}

// wt (p x KS, padded classes zero) = transpose of the block-major W (K x p): 64-column tiles through
// shared memory so both the reads (KS rows of 512 contiguous bytes, KS/4 loads in flight per thread) and
// the writes (64*KS contiguous doubles) are coalesced.
constexpr int kTrCols = 64;
__global__ void __launch_bounds__(256) transpose_w_kernel(const double* __restrict__ W, int64_t p, int K, int KS,
                                                          double* __restrict__ wt, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double tile[32][kTrCols + 1];
    const int tx = threadIdx.x & (kTrCols - 1), ty = threadIdx.x / kTrCols;  // 4 rows of 64
    for (int64_t j0 = (int64_t)blockIdx.x * kTrCols; j0 < p; j0 += (int64_t)gridDim.x * kTrCols) {
        for (int c = ty; c < KS; c += 256 / kTrCols)
            tile[c][tx] = (c < K && j0 + tx < p) ? __ldcs(W + (int64_t)c * p + j0 + tx) : 0.0;
        __syncthreads();
        const int64_t base = j0 * KS;
        const int64_t total = (p - j0 < kTrCols ? p - j0 : kTrCols) * KS;
        for (int q = threadIdx.x; q < total; q += 256) wt[base + q] = tile[q % KS][q / KS];
        __syncthreads();
    }
}

struct SpArgs {
    const int64_t* indptr;
    const int32_t* indices;
    const double* vals;
    const int32_t* labels;
    int64_t n, p;
    int K, KS;
    const double* wt;  // p x KS transposed weights
    const double* Pin;
    double *L0, *P, *U, *Lp, *rowM, *rowA;  // U: n x KS
    int32_t* pred;
    double* blk;
    const int32_t* guard;
    // column blocks: this launch covers block `b` of `nb`, row segments from rblk; running logits in lsum
    int nb, b;
    const int64_t* rblk;
    double* lsum;  // n x KS
};

// Gathered dot products of one quad-padded CSR row segment [q0, q1) (capi.cu pads every row segment to
// kCscQuad entries with weight-0 copies of its last column) by the lanes of one row: lane (group g,
// slot s) accumulates sum_k v_k * tab[idx_k][VW s .. VW s + VW - 1] over the quads g, g + G, g + 2G, ...
// of the segment, in order, reading each quad's 4 indices / 4 values with one 16-byte / one 32-byte
// load (the group's lanes read the same address: one broadcast request) and then issuing its 4
// gathers; group g's partial is folded into group 0 (groups in ascending order). Valid on group 0's
// lanes. No shuffles in the loop: the earlier form (32 entries per chunk broadcast by shuffles) ran the
// same gathers at half the rate (tools/microbench/gather_bw.cu: 6.9 vs 14.1 TB/s of gathered rows).
template <int VW>
__device__ __forceinline__ void gather_segment(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                               int64_t q0, int64_t q1, const double* __restrict__ tab, int KS,
                                               int L, int G, int lane, double (&acc)[VW], int width = 32) {
    static_assert(kCscQuad == 4, "quad loads");
    const int grp = lane / L, sub = lane - grp * L;
    const double* __restrict__ tb = tab + sub * VW;
#pragma unroll
    for (int e = 0; e < VW; ++e) acc[e] = 0.0;
    if (grp >= G) q1 = q0;  // idle lanes (width mod L) skip the loop
    uint64_t pol;  // the CSR stream is read once: L2 evict_first, so the weight block stays resident
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int64_t k = q0 + 4 * grp; k < q1; k += 4 * (int64_t)G) {
        int4 j4;
        asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=r"(j4.x), "=r"(j4.y), "=r"(j4.z), "=r"(j4.w)
                     : "l"(idx + k), "l"(pol));
        double v[4];
        asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(val + k), "l"(pol));
        const int jj[4] = {j4.x, j4.y, j4.z, j4.w};
        double w[4][VW];
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg_word<VW>(tb + (int64_t)jj[u] * KS, w[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[e] += v[u] * w[u][e];
    }
    for (int g = 1; g < G; ++g) {
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const double o = __shfl_sync(0xffffffffu, acc[e], (sub + g * L) & (width - 1), width);
            if (grp == 0) acc[e] += o;
        }
    }
}

// Gathered dot products of one quad-padded CSC column [q0, q1) by one lane group (capi.cu pads every
// column to kCscQuad entries with weight-0 copies of its last row): lane `sub` of the group accumulates
// sum_k v_k * U[row_k][VW sub .. VW sub + VW - 1] over the column's entries in ascending order (tb = U +
// VW sub); a lane reads a quad's 4 row indices with one 16-byte load and its 4 values with one 32-byte
// load (the group's lanes read the same address: one broadcast request), then issues the 4 gathers.
// No shuffles: the earlier form -- one warp per column, 32 entries per chunk broadcast by shuffles --
// ran the same gathers at half the rate (tools/microbench/gather_bw.cu: 6.9 vs 14.1 TB/s of gathered
// rows); per-entry scalar index / value loads instead of quads: columns pass 1.22 vs 1.11 ms at cfg4.
template <int VW>
__device__ __forceinline__ void group_gather_quads(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                   int64_t q0, int64_t q1, const double* __restrict__ tb, int KS,
                                                   double (&acc)[VW]) {
    static_assert(kCscQuad == 4, "quad loads");
#pragma unroll
    for (int e = 0; e < VW; ++e) acc[e] = 0.0;
    for (int64_t k = q0; k < q1; k += 4) {
        const int4 j4 = __ldg(reinterpret_cast<const int4*>(idx + k));
        double v[4];
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(val + k));
        const int jj[4] = {j4.x, j4.y, j4.z, j4.w};
        double w[4][VW];
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg_word<VW>(tb + (int64_t)jj[u] * KS, w[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[e] += v[u] * w[u][e];
    }
}

__device__ __forceinline__ double sum16(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double max16(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Row epilogues on group 0's lanes (lane owns classes VW lane .. VW lane + VW - 1; L <= 16 lanes, so the
// 16-lane butterflies cover them, other lanes contributing the identity).
// R rows per warp (R = 2: each half-warp owns a row, G = 16 / L groups per row -- half the fold steps
// and two rows' latency chains per warp; the 16-lane butterflies of the epilogue stay inside a half).
template <int MODE, int VW, int R>
__global__ void __launch_bounds__(kSpThreads, kSpBlocksPerSm) sparse_rows_kernel(SpArgs a) {
    if (a.guard && !*a.guard) return;
    __shared__ double red[kSpThreads / 32];
    constexpr int W = 32 / R;  // lanes per row
    const int wl = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int half = wl / W, lane = wl - half * W;  // lane within the row's lanes
    const int64_t rows_step = (int64_t)gridDim.x * (kSpThreads / 32) * R;
    const int K = a.K, KS = a.KS, L = KS / VW, G = W / L;
    const bool g0 = lane < L;
    int cls[VW];
    bool on[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        cls[e] = VW * lane + e;
        on[e] = g0 && cls[e] < K;
    }
    double acc_loss = 0.0;
    const bool blocked = a.nb > 1;
    // segment bounds of row i (block b of the column blocks when blocked)
    auto bounds = [&](int64_t i, int64_t& q0, int64_t& q1) {
        if (i >= a.n) {
            q0 = q1 = 0;
            return;
        }
        const int64_t* src = blocked ? a.rblk + i * (a.nb + 1) + a.b : a.indptr + i;
        q0 = src[0];
        q1 = src[1];
    };
    // every lane of the warp stays in the loop (the fold shuffles use the full mask); a half past the
    // last row gathers an empty segment and stores nothing
    int64_t ib = ((int64_t)blockIdx.x * (kSpThreads / 32) + wib) * R;
    int64_t q0 = 0, q1 = 0, nq0 = 0, nq1 = 0;
    bounds(ib + half, q0, q1);
    for (; ib < a.n; ib += rows_step, q0 = nq0, q1 = nq1) {
        const int64_t i = ib + half;
        const bool valid = i < a.n;
        // software pipeline: the next row's bounds are loaded (and its segment bulk-prefetched into L2)
        // while this row is gathered
        bounds(i + rows_step, nq0, nq1);
        if (lane == 0 && nq1 > nq0) prefetch_segment(a.indices, a.vals, nq0, nq1);
        double lg[VW];
        gather_segment<VW>(a.indices, a.vals, q0, q1, a.wt, KS, L, G, lane, lg, W);
        const bool gv = g0 && valid;
        bool onv[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) onv[e] = on[e] && valid;
        if (blocked) {  // logits = ((block 0 + block 1) + ...) + last block, in block order
            double* ls = a.lsum + i * KS + VW * lane;
            if (a.b > 0 && gv) {
#pragma unroll
                for (int e = 0; e < VW; ++e) lg[e] = ls[e] + lg[e];
            }
            if (a.b < a.nb - 1) {
                if (gv) {
#pragma unroll
                    for (int e = 0; e < VW; ++e) ls[e] = lg[e];
                }
                continue;
            }
        }
        const int b = valid ? a.labels[i] : 1;
        if (MODE == kModeLp) {
#pragma unroll
            for (int e = 0; e < VW; ++e)
                if (onv[e]) a.Lp[i * K + cls[e]] = lg[e];
        } else if (MODE == kModeHv) {  // U = V o P - P o rowsum(V o P)
            double pe[VW], ee[VW], es = 0.0;
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                pe[e] = onv[e] ? a.Pin[i * K + cls[e]] : 0.0;
                ee[e] = lg[e] * pe[e];
                es += ee[e];
            }
            const double rs = sum16(gv ? es : 0.0);
            if (gv) {
                double* u = a.U + i * KS + VW * lane;
#pragma unroll
                for (int e = 0; e < VW; ++e) u[e] = ee[e] - pe[e] * rs;
            }
        } else {  // stable softmax (src/softmax.cpp:51-63)
            double mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < VW; ++e) mx = fmax(mx, onv[e] ? lg[e] : -INFINITY);
            double m = max16(mx);
            m = m > 0.0 ? m : 0.0;
            double ex[VW], es = 0.0;
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                ex[e] = onv[e] ? exp(lg[e] - m) : 0.0;
                es += ex[e];
            }
            const double alpha = exp(-m) + sum16(es);
            double lb = 0.0;
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const double t = __shfl_sync(0xffffffffu, lg[e], ((b - 1) / VW) & (W - 1), W);
                if ((b - 1) % VW == e) lb = t;
            }
            if (MODE == kModeCache || MODE == kModeValue) {
                if (lane == 0 && valid) acc_loss += (m + log(alpha)) - (b <= K ? lb : 0.0);  // src/softmax.cpp:65-78
                if (MODE == kModeCache) {
                    if (lane == 0 && valid) {
                        a.rowM[i] = m;
                        a.rowA[i] = alpha;
                    }
                    double* u = a.U + i * KS + VW * lane;
#pragma unroll
                    for (int e = 0; e < VW; ++e) {
                        const double pc = ex[e] / alpha;
                        if (onv[e]) {
                            a.L0[i * K + cls[e]] = lg[e];
                            a.P[i * K + cls[e]] = pc;
                        }
                        // coeff = P - onehot(label) (src/softmax.cpp:86-90); padded classes 0
                        if (gv) u[e] = onv[e] ? pc - (cls[e] == b - 1 ? 1.0 : 0.0) : 0.0;
                    }
                }
            } else {  // kModePredict: first class with P == max; class C only if strictly greater
                double pc[VW], pm = -INFINITY;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    pc[e] = onv[e] ? ex[e] / alpha : -INFINITY;
                    pm = fmax(pm, pc[e]);
                }
                const double best = max16(pm);
                int first = 1 << 20;
#pragma unroll
                for (int e = VW - 1; e >= 0; --e)
                    if (onv[e] && pc[e] == best) first = cls[e];
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
                if (lane == 0 && valid) {
                    int arg = first + 1;
                    if (exp(-m) / alpha > best) arg = K + 1;
                    a.pred[i] = arg;
                    acc_loss += (arg == b) ? 1.0 : 0.0;
                }
            }
        }
    }
    if ((MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) && (!blocked || a.b == a.nb - 1)) {
        // the rows' sums (on each row's lane 0), halves in order
        const double ws = R == 2 ? __shfl_sync(0xffffffffu, acc_loss, 0) + __shfl_sync(0xffffffffu, acc_loss, 16)
                                 : acc_loss;
        if (wl == 0) red[wib] = ws;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kSpThreads / 32; ++w) s += red[w];
            const int slot = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slot * kBlockPartials + blockIdx.x] = s;
        }
    }
}

// X^T U through the CSC copy, one lane group per column: a warp's G groups (L = KS / VW lanes each) own
// G consecutive columns and each sums its column's nonzeros sequentially in CSC (ascending row) order,
// so there is no cross-group fold and a column's latency chain (bounds -> entries -> gathers -> store) is
// shared by G columns; fused ridge / augmentation shifts and <out, dotvec> partials.
template <int VW>
__global__ void __launch_bounds__(kSpThreads, kSpBlocksPerSm) sparse_cols_kernel(
    const int64_t* __restrict__ cptr, const int32_t* __restrict__ crow, const double* __restrict__ cval, int64_t p,
    int K, int KS, const double* __restrict__ U, const double* __restrict__ vin, const DevParams* prm, int kind,
    double* __restrict__ out, const double* __restrict__ dotvec, double* blk_slot, unsigned long long* ctr,
    const int32_t* guard) {
    if (guard && !*guard) return;
    if (ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr, 1ULL);
    __shared__ double red[32];
    const int lane = threadIdx.x & 31;
    const int L = KS / VW, G = 32 / L;
    const int grp = lane / L, sub = lane - grp * L;
    const double* __restrict__ tb = U + sub * VW;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x / 32) * G;
    const double lam = prm->lambda;
    const bool aug = kind == kXtuHv && prm->augmented;
    const double rho = prm->rho;
    double dacc = 0.0;
    for (int64_t jb = ((int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * G; jb < p; jb += step) {
        if (lane == 0 && jb + step < p) {  // the warp's next G columns are one contiguous CSC range
            const int64_t je = jb + step + G < p ? jb + step + G : p;
            prefetch_segment(crow, cval, cptr[jb + step], cptr[je]);
        }
        const int64_t j = jb + grp;
        const bool valid = grp < G && j < p;
        const int64_t q0 = valid ? cptr[j] : 0, q1 = valid ? cptr[j + 1] : 0;
        double acc[VW];
        group_gather_quads<VW>(crow, cval, q0, q1, tb, KS, acc);
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            const int c = VW * sub + e;
            if (!valid || c >= K) continue;
            const int64_t o = (int64_t)c * p + j;
            double s = acc[e];
            if (lam > 0.0) s = s + lam * vin[o];
            if (aug) s = s + rho * vin[o];
            out[o] = s;
            if (dotvec) dacc += s * dotvec[o];
        }
    }
    if (dotvec) {
        const double t = block_sum(dacc, red);
        if (threadIdx.x == 0) blk_slot[blockIdx.x] = t;
    }
}

template <int VW>
void launch_rows(PassMode mode, int grid, cudaStream_t st, const SpArgs& a) {
    constexpr int R = VW == 4 ? 2 : 1;  // VW = 4: L <= 8 lanes per nonzero, so a half-warp holds >= 2 groups
    switch (mode) {
        case kModeCache: sparse_rows_kernel<kModeCache, VW, R><<<grid, kSpThreads, 0, st>>>(a); break;
        case kModeHv: sparse_rows_kernel<kModeHv, VW, R><<<grid, kSpThreads, 0, st>>>(a); break;
        case kModeLp: sparse_rows_kernel<kModeLp, VW, R><<<grid, kSpThreads, 0, st>>>(a); break;
        case kModeValue: sparse_rows_kernel<kModeValue, VW, R><<<grid, kSpThreads, 0, st>>>(a); break;
        case kModePredict: sparse_rows_kernel<kModePredict, VW, R><<<grid, kSpThreads, 0, st>>>(a); break;
    }
}

}  // namespace

bool sparse_lanes_supported(const Shard& s) { return s.sparse && s.K <= 32 && s.wt; }

// K rounded up to a multiple of 4 (32-byte words) when that adds no padding over rounding to even
// (K mod 4 in {0, 3}: K = 19 -> 20), else to even (16-byte words).
int sparse_class_stride(int K) {
    const int k4 = (K + 3) & ~3, k2 = (K + 1) & ~1;
    return k4 == k2 ? k4 : k2;
}

void sparse_rows_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    cudaStream_t st = s.ctx->stream;
    const int KS = sparse_class_stride(s.K);
    const int tg = (int)std::max<int64_t>(1, std::min<int64_t>((s.p + kTrCols - 1) / kTrCols, 8LL * s.ctx->num_sms));
    transpose_w_kernel<<<tg, 256, 0, st>>>(W, s.p, s.K, KS, s.wt, guard);
    NADMM_LAUNCH_CHECK();
    SpArgs a{};
    a.indptr = s.indptr;
    a.indices = s.indices;
    a.vals = s.vals;
    a.labels = s.labels;
    a.n = s.n;
    a.p = s.p;
    a.K = s.K;
    a.KS = KS;
    a.wt = s.wt;
    a.Pin = s.P;
    a.L0 = s.L0;
    a.P = s.P;
    a.U = s.U;
    a.Lp = s.Lp;
    a.rowM = s.rowM;
    a.rowA = s.rowA;
    a.pred = s.pred;
    a.blk = s.blk;
    a.guard = guard;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((s.n + 7) / 8, std::min<int64_t>(kBlockPartials, (int64_t)kSpBlocksPerSm * s.ctx->num_sms)));
    s.rows_grid = grid;
    a.nb = s.nblk;
    a.rblk = s.rblk;
    a.lsum = s.lsum;
    for (int b = 0; b < s.nblk; ++b) {  // one launch per column block (its weights stay L2-resident)
        a.b = b;
        if (KS % 4 == 0)
            launch_rows<4>(mode, grid, st, a);
        else
            launch_rows<2>(mode, grid, st, a);
        NADMM_LAUNCH_CHECK();
    }
    s.ctx->stats.kernel_launches += 1 + s.nblk;
    s.ctx->stats.data_passes++;
}

int sparse_cols_pass(Shard& s, XtuKind kind, const double* vin, double* out, const double* dotvec, int dot_slot,
                     const int32_t* guard) {
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((s.p + 7) / 8, std::min<int64_t>(kBlockPartials, (int64_t)kSpBlocksPerSm * s.ctx->num_sms)));
    const int KS = sparse_class_stride(s.K);
    auto kern = KS % 4 == 0 ? sparse_cols_kernel<4> : sparse_cols_kernel<2>;
    kern<<<grid, kSpThreads, 0, s.ctx->stream>>>(s.cptr, s.crow, s.cval, s.p, s.K, KS, s.U, vin, s.prm, kind, out,
                                                 dotvec, s.blk + (int64_t)dot_slot * kBlockPartials,
                                                 kind == kXtuHv ? s.ctx->dctr : nullptr, guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
    return grid;
}

}  // namespace nadmm
