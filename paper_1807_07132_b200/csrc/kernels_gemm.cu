// Dense shards outside the fused single-pass shapes -- many classes (the C = 100 large-dense config),
// or class counts without a fused-pass instantiation: each product is two hand-written FP64
// tensor-core GEMM passes over X (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) fed by 2-D tensor-map TMA
// (SASS UTMALDG) into 128-byte-swizzled multistage shared-memory rings, with the row epilogue fused
// into the first. At C - 1 = 99 a product is FP64-tensor bound (~47 FLOP/B; each of
// the two passes alone ~26 FLOP/B against a ridge of ~5.7), so reading X twice costs nothing
// against the roofline, and it keeps every accumulator in registers.
//
//   rows pass  Lg = X * blocks(W)             src/dataset.cpp:69-76   gemm_rows_kernel (persistent,
//              + row epilogue (U / softmax      src/softmax.cpp:51-139   one 128-row tile per step)
//                cache / loss / P / argmax)
//   xtu pass   X^T U                          src/dataset.cpp:78-85   gemm_xtu_kernel (split-K over
//                                                                      row chunks; fixed-order finalize)
//
// Layout (per CTA: 8 compute warps + 1 TMA producer warp, one CTA per SM):
//   rows pass: tile = 128 rows x NB = 8*NF classes; warp w owns rows [16w, 16w+16) (two m-frags) and
//     all NF class n-frags; k-steps of 16 features: X box [128 rows][16 f] and V box [NB classes][16 f]
//     (V is block-major: class c's weights are the p contiguous doubles at W + c*p).
//   xtu pass: tile = 128 features x 16*ceil classes; warp w owns features [16w, 16w+16) (two m-frags)
//     and all class n-frags; k-steps of 16 rows: 8 X boxes [16 rows][16 f] and the U boxes
//     [16 rows][16 classes] (U = n x KU row-major, KU = 8*ceil(K/8)).
// Bank conflicts: the fragment loads address the swizzled tiles with permuted index maps (the
// reduction index in the rows pass, the output feature/class index in the xtu pass) chosen so each
// half-warp's 16 LDS.64 hit 16 distinct bank pairs.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "state.h"
#include "tma_common.cuh"

namespace nadmm {

namespace tma {

CUtensorMap make_map_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                        uint32_t box_outer) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) raise(NADMM_ECUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(NADMM_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

}  // namespace tma

namespace {

using namespace tma;

constexpr int kGBM = 128;                      // rows per rows-pass tile / features per xtu tile
constexpr int kGWarps = 8;                     // compute warps (16 rows / features each)
constexpr int kGThreads = 32 * (kGWarps + 1);  // + the TMA producer warp
constexpr size_t kGSmemLimit = 225 * 1024;
constexpr uint32_t kBox = 16 * 16 * 8;          // one [16][16] FP64 box

// n-frag counts with a kernel instantiation (the next one up serves the others)
constexpr int kNfs[] = {1, 2, 3, 4, 6, 8, 10, 13, 16};

struct RowsArgs {
    int64_t n, ntiles;
    int K, KU, nks, stages;
    uint32_t stage_bytes, x_bytes;
    const double* Pin;
    const int32_t* labels;
    double *U, *L0, *P, *Lp, *rowM, *rowA, *blk;
    int32_t* pred;
    const int32_t* guard;
};

// Rows pass: persistent over 128-row tiles; the producer streams (tile, k-step) boxes through the ring
// without a bubble between tiles, the compute warps run the DMMA k-loop then the tile's row epilogue.
template <int NF, int MODE>
__global__ void __launch_bounds__(kGThreads, 1)
    gemm_rows_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmV, RowsArgs a) {
    extern __shared__ unsigned char g_smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(g_smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)a.stages * a.stage_bytes);
    uint64_t* empty = full + a.stages;
    __shared__ double red[kGWarps];
    if (a.guard && !*a.guard) return;  // grid-uniform
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], kGWarps);
        }
        fence_init();
    }
    __syncthreads();
    const int64_t T = (int64_t)blockIdx.x < a.ntiles ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == kGWarps) {  // ---------------- TMA producer ----------------
        if (lane == 0) {
            prefetch_map(&tmX);
            prefetch_map(&tmV);
            int64_t it = 0;
            for (int64_t t = 0; t < T; ++t) {
                const int row0 = (int)(((int64_t)blockIdx.x + t * gridDim.x) * kGBM);
                for (int ks = 0; ks < a.nks; ++ks, ++it) {
                    const int stg = (int)(it % a.stages);
                    if (it >= a.stages) bar_wait(&empty[stg], (uint32_t)(((it / a.stages) - 1) & 1));
                    unsigned char* xs = sm + (size_t)stg * a.stage_bytes;
                    bar_expect_tx(&full[stg], a.stage_bytes);
                    load_2d(xs, &tmX, ks * 16, row0, &full[stg]);
                    load_2d(xs + a.x_bytes, &tmV, ks * 16, 0, &full[stg]);
                }
            }
        }
        return;
    }

    // ---------------- compute warps ----------------
    const int gq = lane >> 2, tq = lane & 3;
    // k-step s of a 16-feature box reads features c(s, tq) = 8 (tq >> 1) + 2 s + (tq & 1) (a
    // permutation of the reduction index, identical for A and B): with the swizzle every half-warp's
    // 16 loads land in 16 distinct bank pairs (rows gq and classes gq all have row & 7 == gq)
    uint32_t off[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) off[s] = ((uint32_t)((((tq >> 1) << 2) + s) ^ gq) << 4) | ((uint32_t)(tq & 1) << 3);
    const uint32_t arow0 = (uint32_t)(warp * 16 + gq) * 128u, arow1 = arow0 + 8u * 128u;
    double loss_acc = 0.0;
    int64_t it = 0;
    for (int64_t t = 0; t < T; ++t) {
        const int64_t row0 = ((int64_t)blockIdx.x + t * gridDim.x) * kGBM;
        double acc[2][NF][2];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int j = 0; j < NF; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
        for (int ks = 0; ks < a.nks; ++ks, ++it) {
            const int stg = (int)(it % a.stages);
            bar_wait(&full[stg], (uint32_t)((it / a.stages) & 1));
            const unsigned char* xs = sm + (size_t)stg * a.stage_bytes;
            const unsigned char* vs = xs + a.x_bytes;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const double a0 = *reinterpret_cast<const double*>(xs + arow0 + off[s]);
                const double a1 = *reinterpret_cast<const double*>(xs + arow1 + off[s]);
#pragma unroll
                for (int j = 0; j < NF; ++j) {
                    const double b = *reinterpret_cast<const double*>(vs + (uint32_t)(8 * j + gq) * 128u + off[s]);
                    dmma(acc[0][j], a0, b);
                    dmma(acc[1][j], a1, b);
                }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&empty[stg]);
        }

        // ---- row epilogue: thread holds rows (row0 + 16w + 8m + gq), classes 8j + 2tq + e ----
        const int K = a.K;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int64_t gi = row0 + warp * 16 + 8 * m + gq;
            const bool valid = gi < a.n;
            if (MODE == kModeHv) {  // U = V o P - P o rowsum(V o P)  (src/softmax.cpp:103-107)
                // two sweeps over the row's P (the second from L1) keep the register footprint small
                double rs = 0.0;
#pragma unroll
                for (int j = 0; j < NF; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = 8 * j + 2 * tq + e;
                        if (valid && c < K) rs += acc[m][j][e] * __ldg(a.Pin + gi * K + c);
                    }
                rs += __shfl_xor_sync(0xffffffffu, rs, 1);
                rs += __shfl_xor_sync(0xffffffffu, rs, 2);
                if (valid)
#pragma unroll
                    for (int j = 0; j < NF; ++j) {
                        const int c = 8 * j + 2 * tq;
                        const double p0 = c < K ? __ldg(a.Pin + gi * K + c) : 0.0;
                        const double p1 = c + 1 < K ? __ldg(a.Pin + gi * K + c + 1) : 0.0;
                        if (c < a.KU)
                            *reinterpret_cast<double2*>(a.U + gi * a.KU + c) =
                                make_double2(acc[m][j][0] * p0 - p0 * rs, acc[m][j][1] * p1 - p1 * rs);
                    }
            } else if (MODE == kModeLp) {
                if (valid)
#pragma unroll
                    for (int j = 0; j < NF; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int c = 8 * j + 2 * tq + e;
                            if (c < K) a.Lp[gi * K + c] = acc[m][j][e];
                        }
            } else {  // stable softmax (src/softmax.cpp:51-63) + loss / coeff / argmax
                // the exponentials are recomputed per sweep instead of held in registers: a spill-free
                // epilogue (spilling here was measured to corrupt results intermittently)
                double mx = -INFINITY;
#pragma unroll
                for (int j = 0; j < NF; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (8 * j + 2 * tq + e < K) mx = fmax(mx, acc[m][j][e]);
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                const double M = mx > 0.0 ? mx : 0.0;
                double es = 0.0;
#pragma unroll
                for (int j = 0; j < NF; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (8 * j + 2 * tq + e < K) es += exp(acc[m][j][e] - M);
                es += __shfl_xor_sync(0xffffffffu, es, 1);
                es += __shfl_xor_sync(0xffffffffu, es, 2);
                const double alpha = exp(-M) + es;
                const int yb = valid ? __ldg(a.labels + gi) : 0;
                if (MODE == kModeCache || MODE == kModeValue) {
                    double ly = 0.0;  // logit of the row's label (class C has logit 0)
#pragma unroll
                    for (int j = 0; j < NF; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            if (8 * j + 2 * tq + e == yb - 1) ly = acc[m][j][e];
                    ly += __shfl_xor_sync(0xffffffffu, ly, 1);
                    ly += __shfl_xor_sync(0xffffffffu, ly, 2);
                    if (valid && tq == 0) loss_acc += (M + log(alpha)) - (yb <= K ? ly : 0.0);  // src/softmax.cpp:65-78
                    if (MODE == kModeCache && valid) {
                        if (tq == 0) {
                            a.rowM[gi] = M;
                            a.rowA[gi] = alpha;
                        }
#pragma unroll
                        for (int j = 0; j < NF; ++j) {
                            const int c = 8 * j + 2 * tq;
                            const double pc0 = c < K ? exp(acc[m][j][0] - M) / alpha : 0.0;
                            const double pc1 = c + 1 < K ? exp(acc[m][j][1] - M) / alpha : 0.0;
                            if (c < K) {
                                a.L0[gi * K + c] = acc[m][j][0];
                                a.P[gi * K + c] = pc0;
                            }
                            if (c + 1 < K) {
                                a.L0[gi * K + c + 1] = acc[m][j][1];
                                a.P[gi * K + c + 1] = pc1;
                            }
                            // coeff = P - onehot(label) (src/softmax.cpp:86-90), padded classes 0
                            if (c < a.KU)
                                *reinterpret_cast<double2*>(a.U + gi * a.KU + c) =
                                    make_double2(c < K ? pc0 - (c == yb - 1 ? 1.0 : 0.0) : 0.0,
                                                 c + 1 < K ? pc1 - (c + 1 == yb - 1 ? 1.0 : 0.0) : 0.0);
                        }
                    }
                } else if (MODE == kModePredict) {  // src/softmax.cpp:118-139: first max wins; class C only if >
                    double best = -INFINITY;
                    int arg = 1 << 20;
#pragma unroll
                    for (int j = 0; j < NF; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int c = 8 * j + 2 * tq + e;
                            if (c < K) {
                                const double pc = exp(acc[m][j][e] - M) / alpha;
                                if (pc > best || (pc == best && c < arg)) {
                                    best = pc;
                                    arg = c;
                                }
                            }
                        }
#pragma unroll
                    for (int o = 1; o <= 2; o <<= 1) {
                        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
                        if (ob > best || (ob == best && oa < arg)) {
                            best = ob;
                            arg = oa;
                        }
                    }
                    int label = arg + 1;
                    if (exp(-M) / alpha > best) label = K + 1;
                    if (valid && tq == 0) {
                        a.pred[gi] = label;
                        loss_acc += (label == yb) ? 1.0 : 0.0;
                    }
                }
            }
        }
    }
    if (MODE == kModeCache || MODE == kModeValue || MODE == kModePredict) {
        double v = loss_acc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp] = v;
        asm volatile("bar.sync 1, %0;\n" ::"r"(32 * kGWarps) : "memory");  // compute warps only
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < kGWarps; ++w) s += red[w];
            a.blk[(int64_t)(MODE == kModePredict ? kSlotHits : kSlotLoss) * kBlockPartials + blockIdx.x] = s;
        }
    }
}

struct XtuArgs {
    int64_t p, d;
    int K, ftiles, stages, ub;
    int64_t n, rows_per_chunk;
    uint32_t stage_bytes;
    double* part;
    const int32_t* guard;
};

// Feature / class index of lane slot g (0..7) in half j of a 16-wide box: {0,1,2,3,8,9,10,11} for
// j = 0 and {4,5,6,7,12,13,14,15} for j = 1, permuted so the [row][16] swizzled loads are conflict free.
__host__ __device__ __forceinline__ int perm16(int g, int j) {
    return 8 * ((g >> 1) & 1) + 2 * ((g >> 2) + 2 * j) + (g & 1);
}

// X^T U over one (feature tile, row chunk): the chunk's split-K partial for 128 features x all classes.
template <int NF>
__global__ void __launch_bounds__(kGThreads, 1)
    gemm_xtu_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmU, XtuArgs a) {
    extern __shared__ unsigned char g_smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(g_smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)a.stages * a.stage_bytes);
    uint64_t* empty = full + a.stages;
    if (a.guard && !*a.guard) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ft = blockIdx.x % a.ftiles, rc = blockIdx.x / a.ftiles;
    const int64_t r0 = (int64_t)rc * a.rows_per_chunk;
    const int64_t r1 = min(a.n, r0 + a.rows_per_chunk);
    const int nst = r1 > r0 ? (int)((r1 - r0 + 15) / 16) : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], kGWarps);
        }
        fence_init();
    }
    __syncthreads();
    const uint32_t xb = 8 * kBox;
    if (warp == kGWarps) {  // ---------------- TMA producer ----------------
        if (lane == 0) {
            prefetch_map(&tmX);
            prefetch_map(&tmU);
            for (int st = 0; st < nst; ++st) {
                const int stg = st % a.stages;
                if (st >= a.stages) bar_wait(&empty[stg], (uint32_t)(((st / a.stages) - 1) & 1));
                unsigned char* xs = sm + (size_t)stg * a.stage_bytes;
                const int row = (int)(r0 + 16 * st);
                bar_expect_tx(&full[stg], a.stage_bytes);
                for (int b = 0; b < kGWarps; ++b) load_2d(xs + b * kBox, &tmX, ft * kGBM + 16 * b, row, &full[stg]);
                for (int b = 0; b < a.ub; ++b) load_2d(xs + xb + b * kBox, &tmU, 16 * b, row, &full[stg]);
            }
        }
        return;
    }
    const int gq = lane >> 2, tq = lane & 3;
    // A = X^T: A[m = gq][k = tq] = X[row 4s + tq][feature perm16(gq, jm)] of box `warp`;
    // B = U:   B[k = tq][n = gq] = U[row 4s + tq][class 16 (q >> 1) + perm16(gq, q & 1)]
    double acc[2][NF][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int q = 0; q < NF; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
    for (int st = 0; st < nst; ++st) {
        const int stg = st % a.stages;
        bar_wait(&full[stg], (uint32_t)((st / a.stages) & 1));
        const unsigned char* xs = sm + (size_t)stg * a.stage_bytes + (size_t)warp * kBox;
        const unsigned char* us = sm + (size_t)stg * a.stage_bytes + xb;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const uint32_t r = (uint32_t)(4 * s + tq);
            const double a0 = *reinterpret_cast<const double*>(xs + sw128(r, perm16(gq, 0)));
            const double a1 = *reinterpret_cast<const double*>(xs + sw128(r, perm16(gq, 1)));
#pragma unroll
            for (int q = 0; q < NF; ++q) {
                const double b = *reinterpret_cast<const double*>(us + (q >> 1) * kBox + sw128(r, perm16(gq, q & 1)));
                dmma(acc[0][q], a0, b);
                dmma(acc[1][q], a1, b);
            }
        }
        __syncwarp();
        if (lane == 0) bar_arrive(&empty[stg]);
    }
    // this chunk's partial: part[rc][class * p + feature] (block-major d, src/softmax.cpp:47-49)
    double* out = a.part + (int64_t)rc * a.d;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int64_t f = (int64_t)ft * kGBM + 16 * warp + perm16(gq, m);
        if (f >= a.p) continue;
#pragma unroll
        for (int q = 0; q < NF; ++q)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = 16 * (q >> 1) + perm16(2 * tq + e, q & 1);
                if (c < a.K) out[(int64_t)c * a.p + f] = acc[m][q][e];
            }
    }
}

// ------------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------------
struct GemmState {
    int nf_rows = 0, nf_xtu = 0;  // instantiated n-frag counts
    int KU = 0;                   // U row stride (classes, multiple of 8)
    int rows_stages = 0, xtu_stages = 0, grid_rows = 0, splits = 0, ftiles = 0;
    uint32_t rows_stage_bytes = 0, xtu_stage_bytes = 0;
    int64_t rows_per_chunk = 0;
    double* U = nullptr;
    CUtensorMap mapX_rows, mapX_xtu, mapU;
};

GemmState* gstate(const Shard& s) { return static_cast<GemmState*>(s.gemm); }

int nf_for(int need) {
    for (int v : kNfs)
        if (v >= need) return v;
    return 0;
}

// frags covering classes [0, K) in the xtu pass's permuted 16-class boxes
int xtu_frags(int K) {
    const int full = K / 16, rem = K % 16;
    return 2 * full + (rem == 0 ? 0 : rem <= 4 ? 1 : 2);
}

template <int NF, int MODE>
void set_rows_attr(size_t smem) {
    NADMM_CUDA(cudaFuncSetAttribute(gemm_rows_kernel<NF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

template <int NF>
void setup_nf(size_t rows_smem, size_t xtu_smem) {
    set_rows_attr<NF, kModeCache>(rows_smem);
    set_rows_attr<NF, kModeHv>(rows_smem);
    set_rows_attr<NF, kModeLp>(rows_smem);
    set_rows_attr<NF, kModeValue>(rows_smem);
    set_rows_attr<NF, kModePredict>(rows_smem);
    NADMM_CUDA(cudaFuncSetAttribute(gemm_xtu_kernel<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xtu_smem));
}

void setup_attrs(int nf, size_t rows_smem, size_t xtu_smem, bool rows) {
    // rows: set the rows-pass attributes for nf; else the xtu-pass ones (setup_nf sets both; harmless)
    (void)rows;
    switch (nf) {
#define NADMM_NF_CASE(v) \
    case v: setup_nf<v>(rows_smem, xtu_smem); break;
        NADMM_NF_CASE(1) NADMM_NF_CASE(2) NADMM_NF_CASE(3) NADMM_NF_CASE(4) NADMM_NF_CASE(6) NADMM_NF_CASE(8)
        NADMM_NF_CASE(10) NADMM_NF_CASE(13) NADMM_NF_CASE(16)
#undef NADMM_NF_CASE
        default: raise(NADMM_ECONFIG, "gemm: no instantiation for this class count");
    }
}

template <int NF, int MODE>
void launch_rows_nf(Shard& s, const GemmState& g, const CUtensorMap& mv, const RowsArgs& a) {
    const size_t smem = (size_t)g.rows_stages * g.rows_stage_bytes + 2 * 8 * g.rows_stages + 1024;
    gemm_rows_kernel<NF, MODE><<<g.grid_rows, kGThreads, smem, s.ctx->stream>>>(g.mapX_rows, mv, a);
    NADMM_LAUNCH_CHECK();
}

template <int MODE>
void launch_rows(Shard& s, const GemmState& g, const CUtensorMap& mv, const RowsArgs& a) {
    switch (g.nf_rows) {
#define NADMM_NF_CASE(v) \
    case v: launch_rows_nf<v, MODE>(s, g, mv, a); break;
        NADMM_NF_CASE(1) NADMM_NF_CASE(2) NADMM_NF_CASE(3) NADMM_NF_CASE(4) NADMM_NF_CASE(6) NADMM_NF_CASE(8)
        NADMM_NF_CASE(10) NADMM_NF_CASE(13) NADMM_NF_CASE(16)
#undef NADMM_NF_CASE
        default: raise(NADMM_ECONFIG, "gemm: no instantiation for this class count");
    }
}

void launch_xtu(Shard& s, const GemmState& g, const XtuArgs& a) {
    const size_t smem = (size_t)g.xtu_stages * g.xtu_stage_bytes + 2 * 8 * g.xtu_stages + 1024;
    const dim3 grid(g.ftiles * g.splits);
    cudaStream_t st = s.ctx->stream;
    switch (g.nf_xtu) {
#define NADMM_NF_CASE(v) \
    case v: gemm_xtu_kernel<v><<<grid, kGThreads, smem, st>>>(g.mapX_xtu, g.mapU, a); break;
        NADMM_NF_CASE(1) NADMM_NF_CASE(2) NADMM_NF_CASE(3) NADMM_NF_CASE(4) NADMM_NF_CASE(6) NADMM_NF_CASE(8)
        NADMM_NF_CASE(10) NADMM_NF_CASE(13) NADMM_NF_CASE(16)
#undef NADMM_NF_CASE
        default: raise(NADMM_ECONFIG, "gemm: no instantiation for this class count");
    }
    NADMM_LAUNCH_CHECK();
}

int stages_for(uint32_t stage_bytes) {
    return (int)std::max<size_t>(2, std::min<size_t>(8, (kGSmemLimit - 1024 - 256) / (stage_bytes + 16)));
}

}  // namespace

void gemm_setup(Shard& s) {
    if (s.sparse || s.gemm || smallp_supported(s) || dmma_supported(s)) return;
    static const bool disabled = getenv("NADMM_DISABLE_GEMM") != nullptr;
    // tensor maps need 16-byte row strides: X rows (ldx is even) and the block-major weight vector
    // (class stride p doubles); odd p stays on the SIMT passes
    if (disabled || s.p % 2 != 0 || s.ldx % 2 != 0) return;
    const int nf_rows = nf_for((s.K + 7) / 8), nf_xtu = nf_for(xtu_frags(s.K));
    if (!nf_rows || !nf_xtu) return;
    auto* g = new GemmState();
    g->nf_rows = nf_rows;
    g->nf_xtu = nf_xtu;
    g->KU = 8 * ((s.K + 7) / 8);
    const int NB = 8 * nf_rows;
    g->rows_stage_bytes = (uint32_t)kGBM * 128u + (uint32_t)NB * 128u;
    g->rows_stages = stages_for(g->rows_stage_bytes);
    const int ub = (nf_xtu + 1) / 2;
    g->xtu_stage_bytes = 8 * kBox + (uint32_t)ub * kBox;
    g->xtu_stages = stages_for(g->xtu_stage_bytes);
    const size_t rows_smem = (size_t)g->rows_stages * g->rows_stage_bytes + 16 * g->rows_stages + 1024;
    const size_t xtu_smem = (size_t)g->xtu_stages * g->xtu_stage_bytes + 16 * g->xtu_stages + 1024;
    setup_attrs(nf_rows, rows_smem, xtu_smem, true);
    if (nf_xtu != nf_rows) setup_attrs(nf_xtu, rows_smem, xtu_smem, false);
    const int sms = s.ctx->num_sms;
    const int64_t ntiles = (s.n + kGBM - 1) / kGBM;
    g->grid_rows = (int)std::max<int64_t>(1, std::min<int64_t>({ntiles, (int64_t)sms, (int64_t)kBlockPartials}));
    g->ftiles = (int)((s.p + kGBM - 1) / kGBM);
    int splits = std::max(1, sms / g->ftiles);
    splits = std::min<int>(splits, s.part_chunks);
    const int64_t rstages = (s.n + 15) / 16;
    splits = (int)std::min<int64_t>(splits, rstages);
    g->rows_per_chunk = ((rstages + splits - 1) / splits) * 16;  // whole 16-row stages per chunk
    g->splits = (int)((s.n + g->rows_per_chunk - 1) / g->rows_per_chunk);
    NADMM_CUDA(cudaMalloc(&g->U, sizeof(double) * (size_t)s.n * g->KU));
    NADMM_CUDA(cudaMemsetAsync(g->U, 0, sizeof(double) * (size_t)s.n * g->KU, s.ctx->stream));
    s.bytes += (int64_t)sizeof(double) * s.n * g->KU;
    g->mapX_rows = tma::make_map_2d(s.X, (uint64_t)s.p, (uint64_t)s.n, (uint64_t)s.ldx * 8, 16, kGBM);
    g->mapX_xtu = tma::make_map_2d(s.X, (uint64_t)s.p, (uint64_t)s.n, (uint64_t)s.ldx * 8, 16, 16);
    g->mapU = tma::make_map_2d(g->U, (uint64_t)g->KU, (uint64_t)s.n, (uint64_t)g->KU * 8, 16, 16);
    s.gemm = g;
    if (getenv("NADMM_GEMM_VERBOSE"))
        fprintf(stderr, "[nadmm] gemm path n=%lld p=%lld K=%d: rows NF=%d %d stages grid %d; xtu NF=%d %d stages %d x %d\n",
                (long long)s.n, (long long)s.p, s.K, nf_rows, g->rows_stages, g->grid_rows, nf_xtu, g->xtu_stages,
                g->ftiles, g->splits);
}

void gemm_free(Shard& s) {
    GemmState* g = gstate(s);
    if (!g) return;
    if (g->U) cudaFree(g->U);
    delete g;
    s.gemm = nullptr;
}

bool gemm_supported(const Shard& s) { return !s.sparse && s.gemm != nullptr && s.part; }

void gemm_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard) {
    const GemmState& g = *gstate(s);
    const CUtensorMap mv = tma::make_map_2d(W, (uint64_t)s.p, (uint64_t)s.K, (uint64_t)s.p * 8, 16, 8 * g.nf_rows);
    RowsArgs a{};
    a.n = s.n;
    a.ntiles = (s.n + kGBM - 1) / kGBM;
    a.K = s.K;
    a.KU = g.KU;
    a.nks = (int)((s.p + 15) / 16);
    a.stages = g.rows_stages;
    a.stage_bytes = g.rows_stage_bytes;
    a.x_bytes = (uint32_t)kGBM * 128u;
    a.Pin = s.P;
    a.labels = s.labels;
    a.U = g.U;
    a.L0 = s.L0;
    a.P = s.P;
    a.Lp = s.Lp;
    a.rowM = s.rowM;
    a.rowA = s.rowA;
    a.blk = s.blk;
    a.pred = s.pred;
    a.guard = guard;
    static const bool poison = getenv("NADMM_GEMM_POISON_U") != nullptr;  // debug: NaN-fill U first
    if (poison) NADMM_CUDA(cudaMemsetAsync(g.U, 0xFF, sizeof(double) * (size_t)s.n * g.KU, s.ctx->stream));
    switch (mode) {
        case kModeCache: launch_rows<kModeCache>(s, g, mv, a); break;
        case kModeHv: launch_rows<kModeHv>(s, g, mv, a); break;
        case kModeLp: launch_rows<kModeLp>(s, g, mv, a); break;
        case kModeValue: launch_rows<kModeValue>(s, g, mv, a); break;
        case kModePredict: launch_rows<kModePredict>(s, g, mv, a); break;
    }
    s.ctx->stats.kernel_launches++;
    s.ctx->stats.data_passes++;
    s.rows_grid = g.grid_rows;  // loss / hit partial count
    if (mode == kModeHv || mode == kModeCache) {
        XtuArgs x{};
        x.p = s.p;
        x.d = s.d;
        x.K = s.K;
        x.ftiles = g.ftiles;
        x.stages = g.xtu_stages;
        x.ub = (g.nf_xtu + 1) / 2;
        x.n = s.n;
        x.rows_per_chunk = g.rows_per_chunk;
        x.stage_bytes = g.xtu_stage_bytes;
        x.part = s.part;
        x.guard = guard;
        launch_xtu(s, g, x);
        s.ctx->stats.kernel_launches++;
        s.ctx->stats.data_passes++;
        s.last_chunks = g.splits;
    }
}

}  // namespace nadmm
