// extern "C" entry points of include/nadmm_cuda.h: handles, data upload, model-level ops, the
// Newton solver and the worker. Exceptions never cross the ABI: every entry point maps
// nadmm::Error to its status code and stores the message in a thread-local buffer.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "solver.h"
#include "solver_kernels.h"

using namespace nadmm;

namespace {

thread_local std::string g_last_error;

template <typename F>
nadmm_status guard(F&& f) {
    try {
        // Launch checks read cudaGetLastError(); clear stale errors other libraries left in this
        // thread (e.g. a framework probing an external stream) so they are not attributed to us.
        (void)cudaGetLastError();
        f();
        return NADMM_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return NADMM_ECUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return NADMM_ECUDA;
    }
}

template <typename T>
T* dev_alloc(Shard& s, int64_t count) {
    T* p = nullptr;
    const size_t bytes = sizeof(T) * static_cast<size_t>(std::max<int64_t>(count, 1));
    NADMM_CUDA(cudaMalloc(&p, bytes));
    s.bytes += static_cast<int64_t>(bytes);
    return p;
}

template <typename T>
void dev_free(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

void check_ctx(nadmm_ctx c) {
    if (!c) raise(NADMM_ECONFIG, "null context");
    NADMM_CUDA(cudaSetDevice(c->device));
}

// Solver-level calls own the shard's iterate / z / y buffers for their duration; a shard bound to a
// live Worker or ADMM session keeps its state (the reference's workers own their x_local,
// src/worker.cpp:135), so such calls on it fail instead of clobbering the session.
void check_unbound(nadmm_shard s, const void* caller = nullptr) {
    if (s && s->owner && s->owner != caller)
        raise(NADMM_ECONFIG, "shard is bound to a live worker or ADMM session (free it first)");
}

void check_shard(nadmm_shard s) {
    if (!s) raise(NADMM_ECONFIG, "null shard");
    NADMM_CUDA(cudaSetDevice(s->ctx->device));
    use_layout_split(*s, 1);  // single-shard calls get the whole GPU
}

// Dataset::validate (src/dataset.cpp:28-57) for the pieces the caller hands over.
void validate_common(int64_t n, int64_t p, const int32_t* labels, int32_t C) {
    if (n < 1 || p < 1)
        raise(NADMM_ECONFIG, "dataset must have n >= 1 and p >= 1, got n=" + std::to_string(n) + " p=" + std::to_string(p));
    if (C < 2) raise(NADMM_ECONFIG, "dataset needs at least 2 classes, got " + std::to_string(C));
    if (C - 1 > kMaxClasses) raise(NADMM_ECONFIG, "C - 1 exceeds the device limit of " + std::to_string(kMaxClasses));
    if (!labels) raise(NADMM_ECONFIG, "labels required");
    for (int64_t i = 0; i < n; ++i)
        if (labels[i] < 1 || labels[i] > C)
            raise(NADMM_EDATA, "label out of range at row " + std::to_string(i) + ": " + std::to_string(labels[i]));
}

void alloc_work(Shard& s) {
    // row padding: the fused pass TMA-loads whole 16-row tiles of P and labels
    const int64_t nk = (s.n + kRowPad) * s.K;
    s.L0 = dev_alloc<double>(s, nk);
    s.P = dev_alloc<double>(s, nk);
    // the nonzero-group sparse passes gather U rows with a padded class stride (kernels_sparse.cu)
    const bool lanes = s.sparse && s.K <= 32;
    s.U = dev_alloc<double>(s, lanes ? (s.n + kRowPad) * sparse_class_stride(s.K) : nk);
    s.Lp = dev_alloc<double>(s, nk);
    s.rowM = dev_alloc<double>(s, s.n);
    s.rowA = dev_alloc<double>(s, s.n);
    s.pred = dev_alloc<int32_t>(s, s.n);
    if (!s.sparse) {
        const int64_t cap = std::max<int64_t>(1, (int64_t(8) << 20) / std::max<int64_t>(s.d, 1));
        s.part_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(2LL * s.ctx->num_sms, cap));
        s.part = dev_alloc<double>(s, s.part_chunks * s.d);
    }
    if (lanes) s.wt = dev_alloc<double>(s, s.p * sparse_class_stride(s.K));
    s.blk = dev_alloc<double>(s, (int64_t)kSlotCount * kBlockPartials);
    NADMM_CUDA(cudaMemsetAsync(s.blk, 0, sizeof(double) * kSlotCount * kBlockPartials, s.ctx->stream));
    for (double** v : {&s.x, &s.g, &s.pd, &s.r, &s.dv, &s.hd, &s.z, &s.y, &s.t, &s.tmp, &s.gbase, &s.cache_x}) {
        *v = dev_alloc<double>(s, s.d);
        NADMM_CUDA(cudaMemsetAsync(*v, 0, sizeof(double) * s.d, s.ctx->stream));
    }
    s.scal = dev_alloc<double>(s, 8);
    s.gbar = dev_alloc<unsigned long long>(s, 8);
    NADMM_CUDA(cudaMemsetAsync(s.gbar, 0, 8 * sizeof(unsigned long long), s.ctx->stream));
    s.prm = dev_alloc<DevParams>(s, 1);
    s.st = dev_alloc<DevState>(s, 1);
    s.trace = dev_alloc<DevTrace>(s, kTraceCap);
    NADMM_CUDA(cudaMemsetAsync(s.st, 0, sizeof(DevState), s.ctx->stream));
    NADMM_CUDA(cudaMallocHost(&s.prm_host, sizeof(DevParams)));
    NADMM_CUDA(cudaMallocHost(&s.st_host, sizeof(DevState)));
    NADMM_CUDA(cudaMallocHost(&s.trace_host, sizeof(DevTrace) * kTraceCap));
    std::memset(s.prm_host, 0, sizeof(DevParams));
    NADMM_CUDA(cudaMemcpyAsync(s.prm, s.prm_host, sizeof(DevParams), cudaMemcpyHostToDevice, s.ctx->stream));
    // pass implementations (the DMMA layout search times candidate passes on this shard's data)
    dmma_setup(s);
    smallp_setup(s);
    gemm_setup(s);
    tail_setup(s);
}

void upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    NADMM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}

void download(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    NADMM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
}

bool same_point(const std::vector<double>& memo, const double* w, int64_t d) {
    if ((int64_t)memo.size() != d) return false;
    for (int64_t i = 0; i < d; ++i)
        if (!(memo[i] == w[i])) return false;  // Eigen `x != w` (src/objective.cpp:14)
    return true;
}

// SoftmaxMemo::at (src/objective.cpp:13-20) for the model-level ABI: the cache at host vector w.
void ensure_cache_at_host(Shard& s, const double* w, double lambda) {
    if (!w) raise(NADMM_ECONFIG, "weight vector required");
    if (s.cache_at == Shard::kAtHost && s.cache_lambda == lambda && same_point(s.host_memo, w, s.d)) return;
    upload(s.cache_x, w, sizeof(double) * s.d, s.ctx->stream);
    set_lambda_only(s, lambda);
    op_cache_grad(s, s.cache_x, nullptr);
    s.cache_at = Shard::kAtHost;
    s.cache_lambda = lambda;
    s.host_memo.assign(w, w + s.d);
}

nadmm_newton_cfg cfg_or_default(const nadmm_newton_cfg* c) {
    nadmm_newton_cfg d;
    nadmm_newton_cfg_default(&d);
    return c ? *c : d;
}

}  // namespace

namespace nadmm {

Shard::~Shard() {
    group_forget(*this);
    if (g_iter) cudaGraphExecDestroy(g_iter);
    gemm_free(*this);
    for (auto& t : hv_timers) {
        if (t.start) cudaEventDestroy(t.start);
        if (t.stop) cudaEventDestroy(t.stop);
    }
    for (cudaEvent_t e : tl_events) cudaEventDestroy(e);
    for (double** v : {&X, &wt, &vals, &cval, &L0, &P, &U, &Lp, &rowM, &rowA, &part, &blk, &cache_x, &gbase, &scal, &x, &g,
                       &pd, &r, &dv, &hd, &z, &y, &t, &tmp, &lb_ws, &sgd_u, &lsum})
        dev_free(*v);
    dev_free(indptr);
    dev_free(indices);
    dev_free(cptr);
    dev_free(rblk);
    dev_free(crow);
    dev_free(labels);
    dev_free(pred);
    dev_free(sgd_perm);
    dev_free(gbar);
    dev_free(prm);
    dev_free(st);
    dev_free(trace);
    if (prm_host) cudaFreeHost(prm_host);
    if (st_host) cudaFreeHost(st_host);
    if (trace_host) cudaFreeHost(trace_host);
}

void Shard::ensure_timers(int n) {
    while ((int)hv_timers.size() < n) {
        HvTimer t;
        NADMM_CUDA(cudaEventCreate(&t.start));
        NADMM_CUDA(cudaEventCreate(&t.stop));
        hv_timers.push_back(t);
    }
}

}  // namespace nadmm

namespace nadmm {

static void ctx_release_now(Ctx* ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    group_drop(*ctx);
    if (ctx->dctr) cudaFree(ctx->dctr);
    for (int i = 0; i < Ctx::kMaxNodeStreams; ++i) {
        if (ctx->node_stream[i]) cudaStreamDestroy(ctx->node_stream[i]);
        if (ctx->node_join[i]) cudaEventDestroy(ctx->node_join[i]);
    }
    if (ctx->node_fork) cudaEventDestroy(ctx->node_fork);
    cudaStreamDestroy(ctx->stream);
    delete static_cast<nadmm_ctx_s*>(ctx);
}

void ctx_unref(Ctx* c) {
    if (c && --c->live == 0 && c->released) ctx_release_now(c);
}

static void shard_release_now(Shard* s) {
    Ctx* c = s->ctx;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    delete static_cast<nadmm_shard_s*>(s);
    ctx_unref(c);
}

void shard_hold(Shard* s) { ++s->holders; }

void shard_unhold(Shard* s) {
    if (--s->holders == 0 && s->released) shard_release_now(s);
}

}  // namespace nadmm

extern "C" {

const char* nadmm_last_error(void) { return g_last_error.c_str(); }
int32_t nadmm_abi_version(void) { return NADMM_ABI_VERSION; }

void nadmm_newton_cfg_default(nadmm_newton_cfg* c) {  // inc/newton.hpp:9-17
    c->cg_tol = 1e-4;
    c->cg_max_iters = 10;
    c->armijo_beta = 1e-4;
    c->backtrack_gamma = 0.5;
    c->ls_max_iters = 10;
    c->grad_tol = 1e-8;
    c->newton_max_iters = 100;
}

nadmm_status nadmm_ctx_create(int32_t device, nadmm_ctx* out) {
    return guard([&] {
        if (!out) raise(NADMM_ECONFIG, "null output");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            raise(NADMM_ECUDA, "no CUDA device: this library has no CPU fallback");
        }
        if (device < 0 || device >= count) raise(NADMM_ECONFIG, "device index out of range");
        cudaDeviceProp prop;
        NADMM_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            raise(NADMM_ECUDA, std::string("built for sm_100a (B200); device is ") + prop.name + " sm_" +
                                   std::to_string(prop.major * 10 + prop.minor));
        NADMM_CUDA(cudaSetDevice(device));
        barrier_configure();
        auto* c = new nadmm_ctx_s();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        NADMM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->node_streams = 4;  // measured on the bench workload: 1 / 2 / 4 / 8 streams -> 15.0k / 17.9k / 18.9k / 16.3k Hv/s
        if (const char* ns = getenv("NADMM_NODE_STREAMS")) c->node_streams = std::max(1, std::min(Ctx::kMaxNodeStreams, atoi(ns)));
        if (c->node_streams > 1) {
            for (int i = 0; i < c->node_streams; ++i) {
                NADMM_CUDA(cudaStreamCreateWithFlags(&c->node_stream[i], cudaStreamNonBlocking));
                NADMM_CUDA(cudaEventCreateWithFlags(&c->node_join[i], cudaEventDisableTiming));
            }
            NADMM_CUDA(cudaEventCreateWithFlags(&c->node_fork, cudaEventDisableTiming));
        }
        NADMM_CUDA(cudaMalloc(&c->dctr, 4 * sizeof(unsigned long long)));
        NADMM_CUDA(cudaMemset(c->dctr, 0, 4 * sizeof(unsigned long long)));
        *out = c;
    });
}

nadmm_status nadmm_ctx_destroy(nadmm_ctx ctx) {
    return guard([&] {
        if (!ctx || ctx->released) return;
        ctx->released = true;
        if (ctx->live == 0) ctx_release_now(ctx);  // else: the last shard / communicator releases it
    });
}

int32_t nadmm_ctx_node_streams(nadmm_ctx ctx) { return ctx ? ctx->node_streams : 0; }

nadmm_status nadmm_ctx_synchronize(nadmm_ctx ctx) {
    return guard([&] {
        check_ctx(ctx);
        stream_sync(ctx->stream);
    });
}

void* nadmm_ctx_stream(nadmm_ctx ctx) { return ctx ? (void*)ctx->stream : nullptr; }

nadmm_status nadmm_ctx_stats(nadmm_ctx ctx, nadmm_stats* out) {
    return guard([&] {
        check_ctx(ctx);
        unsigned long long h[4];
        NADMM_CUDA(cudaMemcpyAsync(h, ctx->dctr, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        stream_sync(ctx->stream);
        *out = ctx->stats;
        out->hv_products = (int64_t)h[0];
    });
}

nadmm_status nadmm_ctx_reset_stats(nadmm_ctx ctx) {
    return guard([&] {
        check_ctx(ctx);
        ctx->stats = nadmm_stats{};
        NADMM_CUDA(cudaMemsetAsync(ctx->dctr, 0, 4 * sizeof(unsigned long long), ctx->stream));
    });
}

nadmm_status nadmm_ctx_set_timing(nadmm_ctx ctx, int32_t enable) {
    return guard([&] {
        check_ctx(ctx);
        ctx->timing = enable != 0;
    });
}

// ---- data level ----
nadmm_status nadmm_shard_dense(nadmm_ctx ctx, const double* X, int64_t n, int64_t p, const int32_t* labels, int32_t C,
                               nadmm_shard* out) {
    return guard([&] {
        check_ctx(ctx);
        if (!out) raise(NADMM_ECONFIG, "null output");
        validate_common(n, p, labels, C);
        if (!X) raise(NADMM_ECONFIG, "feature matrix required");
        for (int64_t k = 0; k < n * p; ++k)
            if (!std::isfinite(X[k])) raise(NADMM_EDATA, "non-finite feature value in dense dataset");
        std::unique_ptr<nadmm_shard_s> s(new nadmm_shard_s());
        s->ctx = ctx;
        s->n = n;
        s->p = p;
        s->C = C;
        s->K = C - 1;
        s->d = (int64_t)s->K * p;
        s->sparse = false;
        s->ldx = p;
        s->X = dev_alloc<double>(*s, n * p);
        upload(s->X, X, sizeof(double) * n * p, ctx->stream);
        s->labels = dev_alloc<int32_t>(*s, n + kRowPad);
        NADMM_CUDA(cudaMemsetAsync(s->labels, 0, sizeof(int32_t) * (n + kRowPad), ctx->stream));
        upload(s->labels, labels, sizeof(int32_t) * n, ctx->stream);
        alloc_work(*s);
        stream_sync(ctx->stream);
        ctx->live++;
        *out = s.release();
    });
}

nadmm_status nadmm_shard_csr(nadmm_ctx ctx, const int64_t* indptr, const int32_t* indices, const double* vals,
                             int64_t n, int64_t p, const int32_t* labels, int32_t C, nadmm_shard* out) {
    return guard([&] {
        check_ctx(ctx);
        if (!out) raise(NADMM_ECONFIG, "null output");
        validate_common(n, p, labels, C);
        if (!indptr || (indptr[n] > 0 && (!indices || !vals))) raise(NADMM_ECONFIG, "CSR arrays required");
        if (indptr[0] != 0) raise(NADMM_ECONFIG, "indptr[0] must be 0");
        for (int64_t i = 0; i < n; ++i)
            if (indptr[i + 1] < indptr[i]) raise(NADMM_ECONFIG, "indptr must be non-decreasing");
        const int64_t nnz_in = indptr[n];
        for (int64_t k = 0; k < nnz_in; ++k) {
            if (indices[k] < 0 || indices[k] >= p) raise(NADMM_ECONFIG, "column index out of range");
            if (!std::isfinite(vals[k])) raise(NADMM_EDATA, "non-finite feature value in sparse dataset");
        }
        // Canonical CSR (setFromTriplets: sorted columns, duplicates summed). Fast path when the
        // input is already canonical.
        bool canonical = true;
        for (int64_t i = 0; i < n && canonical; ++i)
            for (int64_t k = indptr[i] + 1; k < indptr[i + 1]; ++k)
                if (indices[k] <= indices[k - 1]) {
                    canonical = false;
                    break;
                }
        std::vector<int64_t> cp;
        std::vector<int32_t> ci;
        std::vector<double> cv;
        const int64_t* rp = indptr;
        const int32_t* ri = indices;
        const double* rv = vals;
        if (!canonical) {
            cp.assign(n + 1, 0);
            std::vector<std::pair<int32_t, double>> row;
            for (int64_t i = 0; i < n; ++i) {
                row.clear();
                for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) row.emplace_back(indices[k], vals[k]);
                std::stable_sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
                for (size_t q = 0; q < row.size(); ++q) {
                    if (q > 0 && row[q].first == row[q - 1].first && !ci.empty() && (int64_t)ci.size() > cp[i])
                        cv.back() += row[q].second;
                    else {
                        ci.push_back(row[q].first);
                        cv.push_back(row[q].second);
                    }
                }
                cp[i + 1] = (int64_t)ci.size();
            }
            rp = cp.data();
            ri = ci.data();
            rv = cv.data();
        }
        const int64_t nnz = rp[n];
        // CSC copy (counting sort by column; rows ascending within a column). For the lane-group columns
        // pass (C - 1 <= 32) every column is padded to a multiple of kCscQuad entries (row of its last
        // entry, value 0) so a lane reads a quad of row indices / values with one 16-byte / 32-byte load.
        const int64_t quad = C - 1 <= 32 ? kCscQuad : 1;
        std::vector<int64_t> colptr(p + 1, 0);
        for (int64_t k = 0; k < nnz; ++k) colptr[ri[k] + 1]++;
        for (int64_t j = 0; j < p; ++j) colptr[j + 1] = colptr[j] + (colptr[j + 1] + quad - 1) / quad * quad;
        const int64_t cnnz = colptr[p];
        std::vector<int32_t> crow(cnnz);
        std::vector<double> cval(cnnz, 0.0);
        {
            std::vector<int64_t> pos(colptr.begin(), colptr.end() - 1);
            for (int64_t i = 0; i < n; ++i)
                for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                    const int64_t q = pos[ri[k]]++;
                    crow[q] = (int32_t)i;
                    cval[q] = rv[k];
                }
            for (int64_t j = 0; j < p; ++j)
                for (int64_t q = pos[j]; q < colptr[j + 1]; ++q) crow[q] = crow[pos[j] - 1];
        }
        std::unique_ptr<nadmm_shard_s> s(new nadmm_shard_s());
        s->ctx = ctx;
        s->n = n;
        s->p = p;
        s->C = C;
        s->K = C - 1;
        s->d = (int64_t)s->K * p;
        s->sparse = true;
        s->nnz = nnz;
        // column blocks for the rows pass: transposed weights of one block within ~48 MB of L2
        const int64_t wbytes = 8 * (int64_t)sparse_class_stride(C - 1) * p;
        int64_t kBlockBudget = int64_t(48) << 20;
        if (const char* e = getenv("NADMM_SPARSE_BLOCK_KB")) kBlockBudget = std::max<int64_t>(1, atoll(e)) << 10;
        std::vector<int64_t> rblk;
        int nb = 1;
        if (C - 1 <= 32 && wbytes > kBlockBudget) {
            nb = (int)std::min<int64_t>(64, (wbytes + kBlockBudget - 1) / kBlockBudget);
            const int64_t width = (p + nb - 1) / nb;
            rblk.resize((size_t)n * (nb + 1));
            for (int64_t i = 0; i < n; ++i) {  // rows are canonical: columns ascending
                int64_t q = rp[i];
                for (int b = 0; b < nb; ++b) {
                    const int64_t lo = (int64_t)b * width;
                    while (q < rp[i + 1] && ri[q] < lo) ++q;
                    rblk[(size_t)i * (nb + 1) + b] = q;
                }
                rblk[(size_t)i * (nb + 1) + nb] = rp[i + 1];
            }
        }
        // Lane-group rows pass (C - 1 <= 32): every row segment (one per column block) is padded to a
        // multiple of kCscQuad entries (column of its last entry, value 0) so a lane reads a quad of
        // indices / values with one 16-byte / 32-byte load; offsets become the padded indptr (one block)
        // or the padded rblk. The generic CSR path (C - 1 > 32) keeps the canonical arrays.
        std::vector<int64_t> pptr;
        std::vector<int32_t> pidx;
        std::vector<double> pval;
        const int64_t* up_ptr = rp;
        const int32_t* up_idx = ri;
        const double* up_val = rv;
        int64_t rnnz = nnz;
        if (C - 1 <= 32) {
            const int64_t segs = n * (int64_t)nb;
            auto seg0 = [&](int64_t t) { return nb == 1 ? rp[t] : rblk[(size_t)(t / nb) * (nb + 1) + t % nb]; };
            auto seg1 = [&](int64_t t) { return nb == 1 ? rp[t + 1] : rblk[(size_t)(t / nb) * (nb + 1) + t % nb + 1]; };
            std::vector<int64_t> off((size_t)segs + 1, 0);
            for (int64_t t = 0; t < segs; ++t)
                off[t + 1] = off[t] + (seg1(t) - seg0(t) + kCscQuad - 1) / kCscQuad * kCscQuad;
            rnnz = off[segs];
            pidx.resize((size_t)rnnz);
            pval.assign((size_t)rnnz, 0.0);
            for (int64_t t = 0; t < segs; ++t) {
                const int64_t a0 = seg0(t), len = seg1(t) - a0;
                std::copy(ri + a0, ri + a0 + len, pidx.begin() + off[t]);
                std::copy(rv + a0, rv + a0 + len, pval.begin() + off[t]);
                for (int64_t q = off[t] + len; q < off[t + 1]; ++q) pidx[q] = ri[a0 + len - 1];
            }
            if (nb == 1) {
                pptr.swap(off);
                up_ptr = pptr.data();
            } else {
                for (int64_t i = 0; i < n; ++i)
                    for (int b = 0; b <= nb; ++b) rblk[(size_t)i * (nb + 1) + b] = off[(size_t)i * nb + b];
            }
            up_idx = pidx.data();
            up_val = pval.data();
        }
        s->indptr = dev_alloc<int64_t>(*s, n + 1);
        s->indices = dev_alloc<int32_t>(*s, rnnz);
        s->vals = dev_alloc<double>(*s, rnnz);
        s->cptr = dev_alloc<int64_t>(*s, p + 1);
        s->crow = dev_alloc<int32_t>(*s, cnnz);
        s->cval = dev_alloc<double>(*s, cnnz);
        upload(s->indptr, up_ptr, sizeof(int64_t) * (n + 1), ctx->stream);
        upload(s->indices, up_idx, sizeof(int32_t) * rnnz, ctx->stream);
        upload(s->vals, up_val, sizeof(double) * rnnz, ctx->stream);
        upload(s->cptr, colptr.data(), sizeof(int64_t) * (p + 1), ctx->stream);
        upload(s->crow, crow.data(), sizeof(int32_t) * cnnz, ctx->stream);
        upload(s->cval, cval.data(), sizeof(double) * cnnz, ctx->stream);
        s->labels = dev_alloc<int32_t>(*s, n + kRowPad);
        NADMM_CUDA(cudaMemsetAsync(s->labels, 0, sizeof(int32_t) * (n + kRowPad), ctx->stream));
        upload(s->labels, labels, sizeof(int32_t) * n, ctx->stream);
        if (nb > 1) {
            s->nblk = nb;
            s->rblk = dev_alloc<int64_t>(*s, (int64_t)rblk.size());
            upload(s->rblk, rblk.data(), sizeof(int64_t) * rblk.size(), ctx->stream);
            s->lsum = dev_alloc<double>(*s, n * sparse_class_stride(C - 1));
        }
        alloc_work(*s);
        stream_sync(ctx->stream);
        ctx->live++;
        *out = s.release();
    });
}

nadmm_status nadmm_shard_free(nadmm_shard s) {
    return guard([&] {
        if (!s || s->released) return;
        s->released = true;
        if (s->holders == 0) shard_release_now(s);  // else: its last worker / session releases it
    });
}

nadmm_status nadmm_shard_info(nadmm_shard s, int64_t* n, int64_t* p, int32_t* C, int32_t* sparse) {
    return guard([&] {
        if (!s) raise(NADMM_ECONFIG, "null shard");
        if (n) *n = s->n;
        if (p) *p = s->p;
        if (C) *C = s->C;
        if (sparse) *sparse = s->sparse ? 1 : 0;
    });
}

int64_t nadmm_shard_device_bytes(nadmm_shard s) { return s ? s->bytes : 0; }

// ---- model level ----
nadmm_status nadmm_cache(nadmm_shard s, const double* w, double* logits, double* row_max, double* alpha,
                         double* probs) {
    return guard([&] {
        check_shard(s);
        ensure_cache_at_host(*s, w, s->cache_at == Shard::kAtHost ? s->cache_lambda : 0.0);
        const int64_t n = s->n, K = s->K;
        std::vector<double> buf(n * K);
        auto colmajor = [&](const double* src, double* dst) {
            download(buf.data(), src, sizeof(double) * n * K, s->ctx->stream);
            for (int64_t i = 0; i < n; ++i)
                for (int64_t c = 0; c < K; ++c) dst[c * n + i] = buf[i * K + c];
        };
        if (logits) colmajor(s->L0, logits);
        if (probs) colmajor(s->P, probs);
        if (row_max) download(row_max, s->rowM, sizeof(double) * n, s->ctx->stream);
        if (alpha) download(alpha, s->rowA, sizeof(double) * n, s->ctx->stream);
    });
}

nadmm_status nadmm_loss(nadmm_shard s, const double* w, double lambda, double* out) {
    return guard([&] {
        check_shard(s);
        ensure_cache_at_host(*s, w, lambda);
        download(out, s->scal, sizeof(double), s->ctx->stream);
    });
}

nadmm_status nadmm_gradient(nadmm_shard s, const double* w, double lambda, double* g) {
    return guard([&] {
        check_shard(s);
        ensure_cache_at_host(*s, w, lambda);
        download(g, s->gbase, sizeof(double) * s->d, s->ctx->stream);
    });
}

nadmm_status nadmm_hessian_vec(nadmm_shard s, const double* w, const double* v, double lambda, double* hv) {
    return guard([&] {
        check_shard(s);
        if (!v || !hv) raise(NADMM_ECONFIG, "v and hv required");
        ensure_cache_at_host(*s, w, s->cache_at == Shard::kAtHost && same_point(s->host_memo, w, s->d) ? s->cache_lambda : lambda);
        set_lambda_only(*s, lambda);
        upload(s->tmp, v, sizeof(double) * s->d, s->ctx->stream);
        op_hv(*s, s->tmp, s->hd, nullptr, 0, nullptr);
        download(hv, s->hd, sizeof(double) * s->d, s->ctx->stream);
    });
}

nadmm_status nadmm_predict(nadmm_shard s, const double* w, int32_t* labels_out) {
    return guard([&] {
        check_shard(s);
        if (!w || !labels_out) raise(NADMM_ECONFIG, "w and output required");
        upload(s->tmp, w, sizeof(double) * s->d, s->ctx->stream);
        op_predict(*s, s->tmp);
        download(labels_out, s->pred, sizeof(int32_t) * s->n, s->ctx->stream);
    });
}

nadmm_status nadmm_accuracy(nadmm_shard s, const double* w, double* out) {
    return guard([&] {
        check_shard(s);
        if (!w || !out) raise(NADMM_ECONFIG, "w and output required");
        upload(s->tmp, w, sizeof(double) * s->d, s->ctx->stream);
        op_predict(*s, s->tmp);
        std::vector<double> parts(s->rows_grid);
        download(parts.data(), s->blk + (int64_t)kSlotHits * kBlockPartials, sizeof(double) * s->rows_grid,
                 s->ctx->stream);
        double hits = 0.0;
        for (double v : parts) hits += v;
        *out = hits / (double)s->n;  // accuracy (src/softmax.cpp:141-153)
    });
}

nadmm_status nadmm_set_point_dev(nadmm_shard s, const double* w_dev) {
    return guard([&] {
        check_shard(s);
        if (s->cache_at == Shard::kAtX && w_dev == s->x) return;
        NADMM_CUDA(cudaMemcpyAsync(s->cache_x, w_dev, sizeof(double) * s->d, cudaMemcpyDeviceToDevice, s->ctx->stream));
        set_lambda_only(*s, 0.0);
        op_cache_grad(*s, s->cache_x, nullptr);
        s->cache_at = Shard::kAtHost;
        s->cache_lambda = 0.0;
        s->host_memo.clear();  // device-set point: host memo no longer describes it
    });
}

nadmm_status nadmm_hessian_vec_dev(nadmm_shard s, const double* v_dev, double lambda, double* hv_dev) {
    return guard([&] {
        check_shard(s);
        if (s->cache_at == Shard::kNone) raise(NADMM_ECONFIG, "no point set: call nadmm_set_point_dev first");
        set_lambda_only(*s, lambda);
        op_hv(*s, v_dev, hv_dev, nullptr, 0, nullptr);
    });
}

// ---- solver level ----
nadmm_status nadmm_newton_solve(nadmm_shard s, const nadmm_newton_cfg* cfg, double lambda, int32_t augmented,
                                double rho, const double* z, const double* y, double* x_inout,
                                nadmm_newton_iter* trace, int32_t trace_cap, nadmm_newton_summary* out) {
    return guard([&] {
        check_unbound(s);
        check_shard(s);
        const nadmm_newton_cfg c = cfg_or_default(cfg);
        validate_newton_cfg(c);
        if (!x_inout) raise(NADMM_ECONFIG, "x_inout required");
        if (augmented) {
            if (rho <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
            if (!z || !y) raise(NADMM_ECONFIG, "augmented objective requires z and y");
            upload(s->z, z, sizeof(double) * s->d, s->ctx->stream);
            upload(s->y, y, sizeof(double) * s->d, s->ctx->stream);
        }
        upload(s->x, x_inout, sizeof(double) * s->d, s->ctx->stream);
        if (s->cache_at == Shard::kAtX) s->cache_at = Shard::kNone;  // fresh objective: no memo
        SolveResult r = device_newton_solve(*s, c, lambda, augmented != 0, rho, c.newton_max_iters);
        if (r.error == NADMM_ESOLVER) raise(NADMM_ESOLVER, "newton_solve: non-finite objective");
        if (r.error == NADMM_ECONFIG) raise(NADMM_ECONFIG, "cg_solve requires ||g|| > 0");
        download(x_inout, s->x, sizeof(double) * s->d, s->ctx->stream);
        for (int k = 0; trace && k < std::min<int>(trace_cap, (int)r.trace.size()); ++k) {
            const DevTrace& t = r.trace[k];
            trace[k] = nadmm_newton_iter{t.iter, t.grad_norm, t.step, t.cg_iters, t.cg_residual, t.objective,
                                         t.ls_capped, t.cg_fallback, t.fn_evals};
        }
        if (out) *out = nadmm_newton_summary{r.converged ? 1 : 0, r.final_grad_norm, r.iterations};
    });
}

void nadmm_lbfgs_cfg_default(nadmm_lbfgs_cfg* c) {
    if (c) *c = nadmm_lbfgs_cfg{25, 1e-4, 0.9, 100, 20, 1e-8};  // inc/lbfgs.hpp:10-15
}

nadmm_status nadmm_lbfgs_solve(nadmm_shard s, const nadmm_lbfgs_cfg* cfg, double lambda, int32_t augmented,
                               double rho, const double* z, const double* y, double* x_inout,
                               nadmm_lbfgs_iter* trace, int32_t trace_cap, nadmm_newton_summary* out) {
    return guard([&] {
        nadmm_lbfgs_cfg c;
        nadmm_lbfgs_cfg_default(&c);
        if (cfg) c = *cfg;
        validate_lbfgs_cfg(c);
        check_unbound(s);
        check_shard(s);
        if (!x_inout) raise(NADMM_ECONFIG, "x_inout required");
        if (augmented) {
            if (rho <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
            if (!z || !y) raise(NADMM_ECONFIG, "augmented objective requires z and y");
            upload(s->z, z, sizeof(double) * s->d, s->ctx->stream);
            upload(s->y, y, sizeof(double) * s->d, s->ctx->stream);
        }
        upload(s->x, x_inout, sizeof(double) * s->d, s->ctx->stream);
        const LbfgsResult r = device_lbfgs_solve(*s, c, lambda, augmented != 0, rho);
        download(x_inout, s->x, sizeof(double) * s->d, s->ctx->stream);
        for (int k = 0; trace && k < std::min<int>(trace_cap, (int)r.trace.size()); ++k) trace[k] = r.trace[k];
        if (out) *out = nadmm_newton_summary{r.converged ? 1 : 0, r.final_grad_norm, (int32_t)r.trace.size()};
    });
}

}  // extern "C"

// ---- worker level ----
struct nadmm_worker_s {
    nadmm_shard shard;
};

extern "C" {

nadmm_status nadmm_worker_create(nadmm_shard s, nadmm_worker* out) {
    return guard([&] {
        check_unbound(s);
        check_shard(s);
        if (!out) raise(NADMM_ECONFIG, "null output");
        NADMM_CUDA(cudaMemsetAsync(s->x, 0, sizeof(double) * s->d, s->ctx->stream));  // x_local = 0
        if (s->cache_at == Shard::kAtX) s->cache_at = Shard::kNone;
        *out = new nadmm_worker_s{s};
        s->owner = *out;  // x_local lives in the shard: one worker per shard
        shard_hold(s);
    });
}

nadmm_status nadmm_worker_free(nadmm_worker w) {
    return guard([&] {
        if (!w) return;
        Shard* s = w->shard;
        if (s && s->owner == w) s->owner = nullptr;
        delete w;
        if (s) shard_unhold(s);
    });
}

nadmm_status nadmm_worker_solve(nadmm_worker w, double rho, const double* z, const double* y,
                                const nadmm_newton_cfg* cfg, int32_t inner_iters, double* x_out,
                                nadmm_inner_stats* stats) {
    return guard([&] {
        if (!w) raise(NADMM_ECONFIG, "null worker");
        Shard& s = *w->shard;
        check_unbound(w->shard, w);
        check_shard(w->shard);
        if (rho <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
        if (!z || !y) raise(NADMM_ECONFIG, "z and y required");
        nadmm_newton_cfg c = cfg_or_default(cfg);
        c.newton_max_iters = inner_iters;  // src/worker.cpp:173
        upload(s.z, z, sizeof(double) * s.d, s.ctx->stream);
        upload(s.y, y, sizeof(double) * s.d, s.ctx->stream);
        // base lambda 0 (src/worker.cpp:130); x and the solver state come back with one synchronisation
        const bool done = solve_launch(s, c, 0.0, true, rho, inner_iters);
        if (x_out) NADMM_CUDA(cudaMemcpyAsync(x_out, s.x, sizeof(double) * s.d, cudaMemcpyDeviceToHost, s.ctx->stream));
        if (!done) solve_readback_async(s);
        stream_sync(s.ctx->stream);
        SolveResult r = done ? solve_collect(s, c, false) : solve_result(s, c);
        if (r.error == NADMM_ESOLVER) raise(NADMM_ESOLVER, "newton_solve: non-finite objective");
        if (r.error == NADMM_ECONFIG) raise(NADMM_ECONFIG, "cg_solve requires ||g|| > 0");
        if (stats) *stats = nadmm_inner_stats{r.final_grad_norm, (uint32_t)r.iterations, (uint32_t)r.cg_sum,
                                              (uint32_t)r.fe_sum, (uint32_t)r.flags};
    });
}

nadmm_status nadmm_workers_solve(const nadmm_worker* ws, int32_t n, const double* rho, const double* z,
                                 const double* const* y, const nadmm_newton_cfg* cfg, int32_t inner_iters,
                                 double* const* x_out, nadmm_inner_stats* stats) {
    return guard([&] {
        if (!ws || n < 1) raise(NADMM_ECONFIG, "at least one worker required");
        if (!rho || !z || !y) raise(NADMM_ECONFIG, "rho, z and y required");
        nadmm_newton_cfg c = cfg_or_default(cfg);
        c.newton_max_iters = inner_iters;  // src/worker.cpp:173
        validate_newton_cfg(c);
        std::vector<Shard*> sh((size_t)n);
        for (int i = 0; i < n; ++i) {
            if (!ws[i]) raise(NADMM_ECONFIG, "null worker");
            sh[(size_t)i] = ws[i]->shard;
            check_unbound(ws[i]->shard, ws[i]);
            if (sh[(size_t)i]->ctx != sh[0]->ctx) raise(NADMM_ECONFIG, "all workers must share one context");
            if (sh[(size_t)i]->d != sh[0]->d) raise(NADMM_ECONFIG, "worker weight dimensions differ");
            if (rho[i] <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
            if (!y[i]) raise(NADMM_ECONFIG, "z and y required");
        }
        Ctx& ctx = *sh[0]->ctx;
        NADMM_CUDA(cudaSetDevice(ctx.device));
        const cudaStream_t st = ctx.stream;
        // the workers of one scatter round run concurrently (WorkerPool threads, src/worker.cpp:222-240):
        // as one node group (whole-GPU group passes), else worker i on node_stream[i % k] with a
        // 1/k-GPU layout, or back to back on the context stream
        std::vector<char> done((size_t)n, 0);
        bool grouped = inner_iters == 1 && group_eligible(sh);
        if (grouped) {
            for (int i = 0; i < n; ++i) {
                Shard& s = *sh[(size_t)i];
                NADMM_CUDA(cudaMemcpyAsync(s.z, z, sizeof(double) * s.d, cudaMemcpyHostToDevice, st));
                NADMM_CUDA(cudaMemcpyAsync(s.y, y[i], sizeof(double) * s.d, cudaMemcpyHostToDevice, st));
            }
            grouped = group_solve_launch(sh, c, rho);
            if (grouped)
                for (int i = 0; i < n; ++i) {
                    Shard& s = *sh[(size_t)i];
                    if (x_out && x_out[i])
                        NADMM_CUDA(cudaMemcpyAsync(x_out[i], s.x, sizeof(double) * s.d, cudaMemcpyDeviceToHost, st));
                    solve_readback_async(s);
                }
        }
        bool conc = !grouped && ctx.node_streams > 1 && n > 1 && inner_iters == 1;
        for (Shard* s : sh) conc = conc && dmma_supported(*s);
        const int ks = conc ? std::min(ctx.node_streams, (int)n) : 1;
        if (!grouped)
            for (Shard* s : sh) use_layout_split(*s, ks);
        if (conc) {
            NADMM_CUDA(cudaEventRecord(ctx.node_fork, st));
            for (int k = 0; k < ks; ++k) NADMM_CUDA(cudaStreamWaitEvent(ctx.node_stream[k], ctx.node_fork, 0));
        }
        for (int i = 0; i < n && !grouped; ++i) {
            Shard& s = *sh[(size_t)i];
            ctx.stream = conc ? ctx.node_stream[i % ks] : st;
            try {
                NADMM_CUDA(cudaMemcpyAsync(s.z, z, sizeof(double) * s.d, cudaMemcpyHostToDevice, ctx.stream));
                NADMM_CUDA(cudaMemcpyAsync(s.y, y[i], sizeof(double) * s.d, cudaMemcpyHostToDevice, ctx.stream));
                done[(size_t)i] = solve_launch(s, c, 0.0, true, rho[i], inner_iters) ? 1 : 0;
                if (x_out && x_out[i])
                    NADMM_CUDA(cudaMemcpyAsync(x_out[i], s.x, sizeof(double) * s.d, cudaMemcpyDeviceToHost, ctx.stream));
                if (!done[(size_t)i]) solve_readback_async(s);
            } catch (...) {
                ctx.stream = st;
                throw;
            }
            ctx.stream = st;
        }
        if (conc)
            for (int k = 0; k < ks; ++k) {
                NADMM_CUDA(cudaEventRecord(ctx.node_join[k], ctx.node_stream[k]));
                NADMM_CUDA(cudaStreamWaitEvent(st, ctx.node_join[k], 0));
            }
        stream_sync(st);  // one synchronisation for the whole round
        if (grouped) group_timers_finish(ctx);
        for (int i = 0; i < n; ++i) {
            Shard& s = *sh[(size_t)i];
            SolveResult r = done[(size_t)i] ? solve_collect(s, c, false) : solve_result(s, c);
            if (r.error == NADMM_ESOLVER) raise(NADMM_ESOLVER, "newton_solve: non-finite objective");
            if (r.error == NADMM_ECONFIG) raise(NADMM_ECONFIG, "cg_solve requires ||g|| > 0");
            if (stats)
                stats[i] = nadmm_inner_stats{r.final_grad_norm, (uint32_t)r.iterations, (uint32_t)r.cg_sum,
                                             (uint32_t)r.fe_sum, (uint32_t)r.flags};
        }
    });
}

nadmm_status nadmm_worker_solve_lbfgs(nadmm_worker w, double rho, const double* z, const double* y,
                                      const nadmm_lbfgs_cfg* cfg, int32_t inner_iters, double* x_out,
                                      nadmm_inner_stats* stats) {
    return guard([&] {
        if (!w) raise(NADMM_ECONFIG, "null worker");
        Shard& s = *w->shard;
        nadmm_lbfgs_cfg c;
        nadmm_lbfgs_cfg_default(&c);
        if (cfg) c = *cfg;
        c.max_iters = inner_iters;  // src/worker.cpp:184
        validate_lbfgs_cfg(c);
        check_unbound(w->shard, w);
        check_shard(w->shard);
        if (rho <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
        if (!z || !y) raise(NADMM_ECONFIG, "z and y required");
        upload(s.z, z, sizeof(double) * s.d, s.ctx->stream);
        upload(s.y, y, sizeof(double) * s.d, s.ctx->stream);
        const LbfgsResult r = device_lbfgs_solve(s, c, 0.0, true, rho);  // x_local warm start in s.x
        if (x_out) download(x_out, s.x, sizeof(double) * s.d, s.ctx->stream);
        if (stats) *stats = lbfgs_inner_stats(r);
    });
}

nadmm_status nadmm_sgd_permutation(uint64_t seed, uint32_t epoch, int64_t n, int32_t* perm) {
    return guard([&] {
        if (n < 0 || (n > 0 && !perm)) raise(NADMM_ECONFIG, "bad permutation request");
        epoch_permutation(nadmm_mix_seed(seed, epoch), n, perm);
    });
}

nadmm_status nadmm_worker_sgd_grad(nadmm_worker w, const nadmm_sgd_cfg* cfg, uint32_t iteration, const double* z,
                                   double* g_out, nadmm_inner_stats* stats) {
    return guard([&] {
        if (!w) raise(NADMM_ECONFIG, "null worker");
        if (!cfg) raise(NADMM_ECONFIG, "sgd session config required");
        Shard& s = *w->shard;
        validate_sgd(s, *cfg);
        check_unbound(w->shard, w);
        check_shard(w->shard);
        if (!z || !g_out) raise(NADMM_ECONFIG, "z and g_out required");
        upload(s.z, z, sizeof(double) * s.d, s.ctx->stream);
        sgd_worker_grad(s, *cfg, iteration, s.z, s.tmp);
        download(g_out, s.tmp, sizeof(double) * s.d, s.ctx->stream);
        if (stats) *stats = nadmm_inner_stats{0.0, 1u, 0u, 1u, 0u};  // src/worker.cpp:216-217
    });
}

}  // extern "C"

namespace nadmm {
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace nadmm

// Profiling hook (not part of the ABI header): per-node durations of the last replay of the shard's
// captured Newton-iteration graph, when it was captured with NADMM_GRAPH_TIMELINE=1. Returns the
// number of intervals written (interval i ends at the mark names[i]).
extern "C" __attribute__((visibility("default"))) int nadmm_debug_graph_timeline(nadmm_shard sh, float* ms,
                                                                               const char** names, int cap) {
    if (!sh) return -1;
    nadmm::Shard& s = *sh;
    if (cudaStreamSynchronize(s.ctx->stream) != cudaSuccess) return -1;
    int n = 0;
    for (size_t i = 1; i < s.tl_names.size() && n < cap; ++i, ++n) {
        float t = -1.f;
        if (cudaEventElapsedTime(&t, s.tl_events[i - 1], s.tl_events[i]) != cudaSuccess) t = -1.f;
        ms[n] = t;
        names[n] = s.tl_names[i];
    }
    return n;
}
