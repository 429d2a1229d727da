// CSR shards with C - 1 <= 32 (the E18/news20-like 20-class sparse config): nonzero-group passes.
//
// Both contractions of a sparse product gather a K-vector per nonzero -- the column's weights in the
// rows pass (X W), the row's U coefficients in the columns pass (X^T U through the CSC copy) -- so the
// pass is bound by L2 -> SM gather traffic (2 nnz K doubles per Hv), not by the CSR/CSC stream itself
// (12 B per nonzero each). The design minimises the gathered sectors and keeps every lane busy:
//   * the gathered tables (transposed weights wt = p x KS, U = n x KS) use a padded class stride
//     KS = K rounded up to even, so a nonzero's K values are KS/2 aligned 16-byte double2 words
//     (K = 19: 160 B = 5 whole sectors instead of 152 B straddling 5-6);
//   * a warp owns a row (rows pass) or a column (columns pass); its lanes form G = 32 / (KS/2) groups
//     of KS/2 lanes, each group gathers one nonzero's double2 words, so G nonzeros are in flight per
//     warp instruction (K = 19: 3 nonzeros, 30 of 32 lanes busy) and kSpUnroll instructions are issued
//     before their FMAs;
//   * the CSR / CSC entries are read 32 at a time, one per lane (coalesced 128 B index and 256 B value
//     loads), and broadcast to the groups by warp shuffles;
//   * group partial sums are folded into group 0 by shuffles; the row epilogue (U / softmax cache /
//     loss / argmax) runs on group 0's lanes with 16-lane butterfly reductions.
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
constexpr int kSpUnroll = 4;  // gathers in flight per lane before their FMAs

// wt (p x KS, padded classes zero) = transpose of the block-major W (K x p): 32-column tiles through
// shared memory so both the reads (along p) and the writes (32*KS contiguous doubles) are coalesced.
__global__ void __launch_bounds__(256) transpose_w_kernel(const double* __restrict__ W, int64_t p, int K, int KS,
                                                          double* __restrict__ wt, const int32_t* guard) {
    if (guard && !*guard) return;
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    for (int64_t j0 = (int64_t)blockIdx.x * 32; j0 < p; j0 += (int64_t)gridDim.x * 32) {
        for (int c = ty; c < KS; c += 8) tile[c][tx] = (c < K && j0 + tx < p) ? W[(int64_t)c * p + j0 + tx] : 0.0;
        __syncthreads();
        const int64_t base = j0 * KS;
        const int64_t total = (p - j0 < 32 ? p - j0 : 32) * KS;
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

// Gathered dot products of one segment [q0, q1) of a CSR row / CSC column: lane (group g, slot s)
// accumulates sum_k v_k * tab[idx_k][2s..2s+1] over the segment's nonzeros k = g (mod G); group g's
// partial is folded into group 0 (groups in ascending order). Valid on group 0's lanes.
__device__ __forceinline__ double2 gather_segment(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                  int64_t q0, int64_t q1, const double2* __restrict__ tab, int L,
                                                  int G, int lane) {
    const int grp = lane / L, sub = lane - grp * L;
    const bool act = grp < G;
    double ax = 0.0, ay = 0.0;
    for (int64_t qb = q0; qb < q1; qb += 32) {
        const int cnt = (int)((q1 - qb) < 32 ? (q1 - qb) : 32);
        int jl = 0;
        double vl = 0.0;
        if (lane < cnt) {
            jl = __ldg(idx + qb + lane);
            vl = __ldg(val + qb + lane);
        }
        for (int t = 0; t < cnt; t += G * kSpUnroll) {
            double2 w[kSpUnroll];
            double v[kSpUnroll];
#pragma unroll
            for (int u = 0; u < kSpUnroll; ++u) {
                const int k = t + u * G + grp;
                const int jj = __shfl_sync(0xffffffffu, jl, k & 31);
                const double vv = __shfl_sync(0xffffffffu, vl, k & 31);
                const bool ok = act && k < cnt;
                v[u] = ok ? vv : 0.0;
                w[u] = ok ? __ldg(tab + (int64_t)jj * L + sub) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < kSpUnroll; ++u) {
                ax += v[u] * w[u].x;
                ay += v[u] * w[u].y;
            }
        }
    }
    for (int g = 1; g < G; ++g) {
        const double ox = __shfl_sync(0xffffffffu, ax, (sub + g * L) & 31);
        const double oy = __shfl_sync(0xffffffffu, ay, (sub + g * L) & 31);
        if (grp == 0) {
            ax += ox;
            ay += oy;
        }
    }
    return make_double2(ax, ay);
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

template <int MODE>
__global__ void __launch_bounds__(kSpThreads) sparse_rows_kernel(SpArgs a) {
    if (a.guard && !*a.guard) return;
    __shared__ double red[kSpThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps_total = (int64_t)gridDim.x * (kSpThreads / 32);
    const int K = a.K, KS = a.KS, L = KS >> 1, G = 32 / L;
    const bool g0 = lane < L;  // group 0: classes c0 = 2 lane, c1 = 2 lane + 1
    const int c0 = 2 * lane, c1 = 2 * lane + 1;
    const bool on0 = g0 && c0 < K, on1 = g0 && c1 < K;
    const double2* wt2 = reinterpret_cast<const double2*>(a.wt);
    double acc_loss = 0.0;
    const bool blocked = a.nb > 1;
    for (int64_t i = (int64_t)blockIdx.x * (kSpThreads / 32) + wib; i < a.n; i += warps_total) {
        const int64_t q0 = blocked ? a.rblk[i * (a.nb + 1) + a.b] : a.indptr[i];
        const int64_t q1 = blocked ? a.rblk[i * (a.nb + 1) + a.b + 1] : a.indptr[i + 1];
        double2 lg = gather_segment(a.indices, a.vals, q0, q1, wt2, L, G, lane);
        if (blocked) {  // logits = ((block 0 + block 1) + ...) + last block, in block order
            double2* ls = reinterpret_cast<double2*>(a.lsum + i * KS) + lane;
            if (a.b > 0 && g0) {
                const double2 prev = *ls;
                lg = make_double2(prev.x + lg.x, prev.y + lg.y);
            }
            if (a.b < a.nb - 1) {
                if (g0) *ls = lg;
                continue;
            }
        }
        const int b = a.labels[i];
        if (MODE == kModeLp) {
            if (on0) a.Lp[i * K + c0] = lg.x;
            if (on1) a.Lp[i * K + c1] = lg.y;
        } else if (MODE == kModeHv) {  // U = V o P - P o rowsum(V o P)
            const double p0 = on0 ? a.Pin[i * K + c0] : 0.0, p1 = on1 ? a.Pin[i * K + c1] : 0.0;
            const double e0 = lg.x * p0, e1 = lg.y * p1;
            const double rs = sum16(g0 ? e0 + e1 : 0.0);
            if (g0) reinterpret_cast<double2*>(a.U + i * KS)[lane] = make_double2(e0 - p0 * rs, e1 - p1 * rs);
        } else {  // stable softmax (src/softmax.cpp:51-63)
            double m = max16(fmax(on0 ? lg.x : -INFINITY, on1 ? lg.y : -INFINITY));
            m = m > 0.0 ? m : 0.0;
            const double e0 = on0 ? exp(lg.x - m) : 0.0, e1 = on1 ? exp(lg.y - m) : 0.0;
            const double alpha = exp(-m) + sum16(e0 + e1);
            const double lbx = __shfl_sync(0xffffffffu, lg.x, ((b - 1) >> 1) & 31);
            const double lby = __shfl_sync(0xffffffffu, lg.y, ((b - 1) >> 1) & 31);
            const double lb = ((b - 1) & 1) ? lby : lbx;
            if (MODE == kModeCache || MODE == kModeValue) {
                if (lane == 0) acc_loss += (m + log(alpha)) - (b <= K ? lb : 0.0);  // src/softmax.cpp:65-78
                if (MODE == kModeCache) {
                    if (lane == 0) {
                        a.rowM[i] = m;
                        a.rowA[i] = alpha;
                    }
                    const double pc0 = e0 / alpha, pc1 = e1 / alpha;
                    if (on0) {
                        a.L0[i * K + c0] = lg.x;
                        a.P[i * K + c0] = pc0;
                    }
                    if (on1) {
                        a.L0[i * K + c1] = lg.y;
                        a.P[i * K + c1] = pc1;
                    }
                    // coeff = P - onehot(label) (src/softmax.cpp:86-90); padded classes 0
                    if (g0)
                        reinterpret_cast<double2*>(a.U + i * KS)[lane] =
                            make_double2(on0 ? pc0 - (c0 == b - 1 ? 1.0 : 0.0) : 0.0,
                                         on1 ? pc1 - (c1 == b - 1 ? 1.0 : 0.0) : 0.0);
                }
            } else {  // kModePredict: first class with P == max; class C only if strictly greater
                const double pc0 = on0 ? e0 / alpha : -INFINITY, pc1 = on1 ? e1 / alpha : -INFINITY;
                const double best = max16(fmax(pc0, pc1));
                int first = (pc0 == best && on0) ? c0 : ((pc1 == best && on1) ? c1 : (1 << 20));
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
                if (lane == 0) {
                    int arg = first + 1;
                    if (exp(-m) / alpha > best) arg = K + 1;
                    a.pred[i] = arg;
                    acc_loss += (arg == b) ? 1.0 : 0.0;
                }
            }
        }
    }
    if ((MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) && (!blocked || a.b == a.nb - 1)) {
        if (lane == 0) red[wib] = acc_loss;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kSpThreads / 32; ++w) s += red[w];
            const int slot = MODE == kModePredict ? kSlotHits : kSlotLoss;
            a.blk[(int64_t)slot * kBlockPartials + blockIdx.x] = s;
        }
    }
}

// X^T U through the CSC copy, one warp per column (nonzero groups as in the rows pass); fused
// ridge / augmentation shifts and <out, dotvec> partials.
__global__ void __launch_bounds__(kSpThreads) sparse_cols_kernel(
    const int64_t* __restrict__ cptr, const int32_t* __restrict__ crow, const double* __restrict__ cval, int64_t p,
    int K, int KS, const double* __restrict__ U, const double* __restrict__ vin, const DevParams* prm, int kind,
    double* __restrict__ out, const double* __restrict__ dotvec, double* blk_slot, unsigned long long* ctr,
    const int32_t* guard) {
    if (guard && !*guard) return;
    if (ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr, 1ULL);
    __shared__ double red[32];
    const int lane = threadIdx.x & 31;
    const int L = KS >> 1, G = 32 / L;
    const int c0 = 2 * lane, c1 = 2 * lane + 1;
    const bool on0 = lane < L && c0 < K, on1 = lane < L && c1 < K;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
    const double lam = prm->lambda;
    const bool aug = kind == kXtuHv && prm->augmented;
    const double rho = prm->rho;
    const double2* u2 = reinterpret_cast<const double2*>(U);
    double dacc = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < p; j += warps_total) {
        const double2 acc = gather_segment(crow, cval, cptr[j], cptr[j + 1], u2, L, G, lane);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (e == 0 ? !on0 : !on1) continue;
            const int64_t o = (int64_t)(e == 0 ? c0 : c1) * p + j;
            double s = e == 0 ? acc.x : acc.y;
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

}  // namespace

bool sparse_lanes_supported(const Shard& s) { return s.sparse && s.K <= 32 && s.wt; }

int sparse_class_stride(int K) { return (K + 1) & ~1; }

void sparse_rows_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    cudaStream_t st = s.ctx->stream;
    const int KS = sparse_class_stride(s.K);
    const int tg = (int)std::max<int64_t>(1, std::min<int64_t>((s.p + 31) / 32, 8LL * s.ctx->num_sms));
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
        1, std::min<int64_t>((s.n + 7) / 8, std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms)));
    s.rows_grid = grid;
    a.nb = s.nblk;
    a.rblk = s.rblk;
    a.lsum = s.lsum;
    for (int b = 0; b < s.nblk; ++b) {  // one launch per column block (its weights stay L2-resident)
        a.b = b;
        switch (mode) {
            case kModeCache: sparse_rows_kernel<kModeCache><<<grid, kSpThreads, 0, st>>>(a); break;
            case kModeHv: sparse_rows_kernel<kModeHv><<<grid, kSpThreads, 0, st>>>(a); break;
            case kModeLp: sparse_rows_kernel<kModeLp><<<grid, kSpThreads, 0, st>>>(a); break;
            case kModeValue: sparse_rows_kernel<kModeValue><<<grid, kSpThreads, 0, st>>>(a); break;
            case kModePredict: sparse_rows_kernel<kModePredict><<<grid, kSpThreads, 0, st>>>(a); break;
        }
        NADMM_LAUNCH_CHECK();
    }
    s.ctx->stats.kernel_launches += 1 + s.nblk;
    s.ctx->stats.data_passes++;
}

int sparse_cols_pass(Shard& s, XtuKind kind, const double* vin, double* out, const double* dotvec, int dot_slot,
                     const int32_t* guard) {
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((s.p + 7) / 8, std::min<int64_t>(kBlockPartials, 8LL * s.ctx->num_sms)));
    sparse_cols_kernel<<<grid, kSpThreads, 0, s.ctx->stream>>>(
        s.cptr, s.crow, s.cval, s.p, s.K, sparse_class_stride(s.K), s.U, vin, s.prm, kind, out, dotvec,
        s.blk + (int64_t)dot_slot * kBlockPartials, kind == kXtuHv ? s.ctx->dctr : nullptr, guard);
    NADMM_LAUNCH_CHECK();
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
    return grid;
}

}  // namespace nadmm
