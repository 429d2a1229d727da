// Host-side objects behind the C ABI handles: context, shard, worker, communicator.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "common.cuh"

namespace nadmm {

// Scalars the device-resident solver reads. They live in device memory so one captured CUDA graph
// serves every outer iteration (rho changes under spectral penalty selection).
struct DevParams {
    double lambda;  // base-objective ridge (make_softmax_objective lambda)
    double rho;     // augmentation penalty (make_augmented_objective rho)
    int32_t augmented;
    int32_t cg_max_iters;
    double cg_tol;
    double armijo_beta;
    double backtrack_gamma;
    int32_t ls_max_iters;
    int32_t pad0;
    double grad_tol;
};

constexpr int kMaxCg = 256;  // cg_max_iters upper bound for the captured solver
constexpr int kMaxLs = 62;   // ls_max_iters upper bound for the batched Armijo search

struct DevState {
    double f_base;  // base loss at x (incl. (lambda/2)|x|^2 when lambda > 0)
    double f_x;     // objective (augmented when enabled) at x
    double g_sq;    // |g|^2 at x
    double g_norm;
    double cg_stop;  // theta * |g|
    double cg_residual;
    double slope;     // p'g used by the line search
    double ls_alpha;  // accepted step
    double rec_gnorm; // |g| at the start of the current Newton iteration
    double r_sq[kMaxCg + 2];
    int32_t cg_act[kMaxCg + 2];  // CG active at the start of iteration it
    int32_t cg_mid[kMaxCg + 2];  // CG active after the step of iteration it
    int32_t cg_iters;
    int32_t cg_neg;     // negative curvature encountered
    int32_t cg_failed;  // non-finite recurrence (SolverError inside cg_solve)
    int32_t it_act;     // this Newton iteration runs
    int32_t active;     // solver still running (across Newton iterations)
    int32_t converged;  // |g| < grad_tol at an iteration start
    int32_t error;      // 0 ok, NADMM_ECONFIG / NADMM_ESOLVER
    int32_t iter;       // Newton iterations completed (trace length)
    int32_t fallback;   // cg_fallback
    int32_t ls_evals;
    int32_t ls_capped;
    int32_t cert_act;   // certificate Hv runs (CG did not fail)
    int32_t lp_need;    // the Armijo Lp must be recomputed (p changed after, or without, the certificate Hv)
};

// Trace row written on device (NewtonIterRecord, inc/newton.hpp:47-57).
struct DevTrace {
    double grad_norm, step, cg_residual, objective;
    int32_t iter, cg_iters, ls_capped, cg_fallback, fn_evals, pad;
};

constexpr int kTraceCap = 128;

struct Ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    nadmm_stats stats{};
    bool timing = false;
    unsigned long long* dctr = nullptr;  // device counters: [0] Hv products applied
    // concurrent ADMM nodes (NADMM_NODE_STREAMS = 2..8): node i's Newton graph runs on node_stream[i % k],
    // each DMMA shard's persistent grid sized to 1/k of the co-resident clusters so all k fit at once
    int node_streams = 1;
    static constexpr int kMaxNodeStreams = 8;
    // objects created on this context (shards, communicators) that are still alive: destroying the
    // context only marks it released, and the last of them to go releases it (any release order is
    // safe, e.g. finalizers run in arbitrary order at interpreter exit)
    int live = 0;
    bool released = false;
    cudaStream_t node_stream[kMaxNodeStreams] = {};
    cudaEvent_t node_fork = nullptr, node_join[kMaxNodeStreams] = {};
    void* group = nullptr;  // cached node-group iteration graph (GroupGraph, newton.cu)
};

struct HvTimer {
    cudaEvent_t start = nullptr, stop = nullptr;
};

// Pass modes of the row-wise (X * W) kernels.
enum PassMode : int {
    kModeCache = 0,    // logits, probs, row stats, loss partials; U = P - Y
    kModeHv = 1,       // U = V o P - P o rowsum(V o P)
    kModeLp = 2,       // Lp = X * p
    kModeValue = 3,    // loss partials only (no stores)
    kModePredict = 4,  // argmax with the reference tie rule; hit-count partials
};

// Solver tails a DMMA pass can run with its whole grid after its last tile.
enum DmmaTail : int { kTailNone = 0, kTailCg = 1, kTailCert = 2, kTailNewton = 3 };

// Partial slots (blk[slot * kBlockPartials + block]).
enum Slot : int {
    kSlotLoss = 0,
    kSlotHits = 1,
    kSlotCurv = 2,    // <d, Hd>
    kSlotRr = 3,      // <r, r>
    kSlotCert = 4,    // |Hp + g|^2
    kSlotSlope = 5,   // <p, g>
    kSlotGg = 6,      // <g, g>
    kSlotTt = 7,      // <t, t>, t = z - x + y/rho
    kSlotLs = 8,      // kSlotLs + j: LS candidate j row losses (j <= kMaxLs)
    kSlotRidge = 71,  // <w, w> for the ridge term of a loss
    kSlotLsVec = 72,  // kSlotLsVec + 2j, +2j+1: LS candidate j |z - x_j + y/rho|^2, |x_j|^2
    kSlotCount = 200
};

struct Shard {
    Ctx* ctx = nullptr;
    // workers / ADMM sessions holding the shard: nadmm_shard_free defers to the last of them
    int holders = 0;
    bool released = false;
    int64_t n = 0, p = 0;
    int C = 0, K = 0;  // K = C - 1
    int64_t d = 0;
    bool sparse = false;
    int64_t bytes = 0;
    // dense rows (row-major, leading dimension ldx)
    double* X = nullptr;
    int64_t ldx = 0;
    // CSR and CSC copies
    int64_t nnz = 0;
    int64_t* indptr = nullptr;
    int32_t* indices = nullptr;
    double* vals = nullptr;
    double* wt = nullptr;  // p x K interleaved copy of the pass operand (class-per-lane sparse passes)
    int64_t* cptr = nullptr;
    int32_t* crow = nullptr;
    double* cval = nullptr;
    int32_t* labels = nullptr;
    // row-wise work matrices, n x K row-major
    double *L0 = nullptr, *P = nullptr, *U = nullptr, *Lp = nullptr;
    double *rowM = nullptr, *rowA = nullptr;
    // split-K partials of X^T U (chunks x d) and block partial slots
    double* part = nullptr;
    int part_chunks = 0;
    double* blk = nullptr;
    unsigned long long* gbar = nullptr;  // grid-barrier counters of the persistent vector kernels
    int rows_grid = 0;  // blocks of the last rows pass (partials count)
    int last_chunks = 0;    // split-K partial chunks written by the last fused DMMA pass
    void* owner = nullptr;            // live Worker / ADMM session bound to this shard's solver state
    const double* rho_src = nullptr;  // ADMM session: the augmentation penalty rho_i lives on the device
    void* gemm = nullptr;   // GemmState of the two-GEMM DMMA path (kernels_gemm.cu), null when unused
    int dmma_clusters = 0;  // co-resident clusters of the fused DMMA pass (0: path unavailable)
    int dmma_mt = 0, dmma_nw = 0, dmma_cs = 0, dmma_fs = 0, dmma_S = 0, dmma_pipe = 0;  // chosen layout
    size_t dmma_smem = 0;
    int tail_cluster = 0;   // CTAs of the single-cluster CG tail (0: grid-barrier tail)
    bool hv_write_lp = false;  // capture-time switch: the next fused Hv pass also stores Lp = X v
    int cg_fuse_it = -1;       // CG iteration index for a fused CG tail
    int dmma_tail = 0;         // capture-time switch: solver tail the next DMMA pass runs (DmmaTail)
    // memo: the point the device cache (L0, P, rowM, rowA, gbase, loss) was built at: the solver
    // iterate s.x, or s.cache_x holding the host vector of the last model-level call
    enum CachePoint { kNone = 0, kAtX = 1, kAtHost = 2 } cache_at = kNone;
    double* cache_x = nullptr;
    double cache_lambda = -1.0;       // lambda the cached gbase / loss include
    std::vector<double> host_memo;    // host copy of cache_x for the model-level ABI memo
    bool host_memo_valid = false;
    double* gbase = nullptr;          // X^T(P - Y) (+ lambda x) at cache_x
    double* scal = nullptr;           // device scalars: [0] base loss at cache_x, [1] value pass, [2] hits
    // solver vectors
    double *x = nullptr, *g = nullptr, *pd = nullptr, *r = nullptr, *dv = nullptr, *hd = nullptr;
    double *z = nullptr, *y = nullptr, *t = nullptr, *tmp = nullptr;
    DevParams* prm = nullptr;
    DevState* st = nullptr;
    DevTrace* trace = nullptr;
    int32_t* pred = nullptr;
    DevParams* prm_host = nullptr;  // pinned staging
    DevState* st_host = nullptr;    // pinned readback
    DevTrace* trace_host = nullptr; // pinned readback (kTraceCap rows)
    // captured solver graph (one Newton iteration)
    cudaGraphExec_t g_iter = nullptr;
    int g_cg_max = -1, g_ls_max = -1;
    bool g_timing = false;
    int64_t g_nodes = 0;  // kernel nodes per replay
    // Hv timing: event pairs around the dominant pass kernel of each Hv site of the graph
    std::vector<HvTimer> hv_timers;
    int hv_timer_site = -1;
    bool capture_timing = false;
    bool last_group = false;  // the last solve ran in a node-group graph (its timers live there)
    // optional per-node timeline of the captured iteration graph (NADMM_GRAPH_TIMELINE=1, profiling)
    bool tl_capture = false;
    std::vector<const char*> tl_names;
    std::vector<cudaEvent_t> tl_events;
    // L-BFGS workspace (lbfgs.cu), kept across solves: curvature history + work vectors
    int layout_split = 1;  // concurrent shards the DMMA layout was tuned for
    struct DmmaLayoutMemo {  // layouts already chosen per split (switching modes re-applies, no re-tune)
        int split, mt, nw, cs, fs, S, pipe, active;
        size_t smem;
    };
    std::vector<DmmaLayoutMemo> dmma_memo;
    // column-blocked CSR rows pass (kernels_sparse.cu): when the transposed weights exceed an L2-sized
    // budget, the rows pass runs once per column block so each block's weights stay L2-resident.
    // rblk[i * (nblk + 1) + b] = first nonzero of row i in column block b; lsum = running logits
    int nblk = 1;
    int64_t* rblk = nullptr;
    double* lsum = nullptr;
    double* lb_ws = nullptr;
    int64_t lb_ws_len = 0;
    // SGD worker state (sgd.cu): the epoch permutation on the device and the batch coefficients
    int32_t* sgd_perm = nullptr;
    int sgd_epoch = -1;
    uint64_t sgd_seed = 0;
    double* sgd_u = nullptr;
    int64_t sgd_u_len = 0;
    void ensure_timers(int n);
    ~Shard();
};

// ---- pass launchers (kernels_pass.cu) ----
// Row-wise X*W pass with the epilogue of `mode` (dense or CSR).
void rows_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard);
// out = X^T U (+ lambda*vin if lambda > 0) (+ rho*vin if augmented and kind == hv); when dotvec is
// non-null, block partials of <out, dotvec> go to slot dot_slot (count: returned grid).
enum XtuKind : int { kXtuGrad = 0, kXtuHv = 1 };
int xtu_pass(Shard& s, XtuKind kind, const double* vin, double* out, const double* dotvec, int dot_slot,
             const int32_t* guard);
// Loss scalar: dst = sum(slot kSlotLoss partials of the last rows pass) (+ 0.5 lambda |w|^2).
void loss_finalize(Shard& s, const double* w, int add_ridge, double* dst, const int32_t* guard);
// Grid for d-length vector kernels whose block partials feed a reduction slot.
int vec_grid(const Ctx& c, int64_t d);
void dot_partials(Shard& s, const double* a, const double* b, int slot, const int32_t* guard, int* grid_out);
void finalize_partials(Shard& s, int chunks, XtuKind kind, const double* vin, double* out, const double* dotvec,
                       int dot_slot, const int32_t* guard, int* dot_grid);

// ---- composite ops (ops.cu) ----
void op_cache_grad(Shard& s, const double* w, const int32_t* guard);
// Cache pass only (the caller finalizes gbase / loss): returns the split-K chunk count of the fused
// dense pass, or 0 when gbase was written directly (SIMT / sparse path).
int op_cache_split(Shard& s, const double* w, const int32_t* guard);   // L0,P,M,alpha,loss,gbase at w
int op_hv(Shard& s, const double* v, double* out, const double* dotvec, int dot_slot, const int32_t* guard);
void op_lp(Shard& s, const double* p, const int32_t* guard);
void op_value(Shard& s, const double* w, double* dst, int add_ridge, const int32_t* guard);
void op_predict(Shard& s, const double* w);

// Timeline mark: during a profiling capture, record an event node named `name` (the time since the
// previous mark is attributed to it). No-op otherwise.
void tl_mark(Shard& s, const char* name);
// Hv for the CG loop: with the fused dense pass only the pass kernel is launched and its split-K
// partial count is returned in *chunks (the caller finalizes); otherwise the full Hv is written to
// `out` with <out, dotvec> partials (returned count) and *chunks = 0.
int op_hv_split(Shard& s, const double* v, double* out, const double* dotvec, int dot_slot, const int32_t* guard,
                int* chunks);

// ---- class-per-lane sparse passes (kernels_sparse.cu): CSR shards with C - 1 <= 32 ----
bool sparse_lanes_supported(const Shard& s);
int sparse_class_stride(int K);  // padded class stride of the gathered tables (K rounded up to 4 or to even)
void sparse_rows_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard);
int sparse_cols_pass(Shard& s, XtuKind kind, const double* vin, double* out, const double* dotvec, int dot_slot,
                     const int32_t* guard);

// ---- small-p dense path (kernels_smallp.cu): p*(C-1) <= 64 ----
bool smallp_supported(const Shard& s);
void smallp_setup(Shard& s);
void smallp_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard);
// ---- GEMM path (kernels_gemm.cu): dense shards outside the fused passes' shapes ----
void gemm_setup(Shard& s);
void gemm_free(Shard& s);
bool gemm_supported(const Shard& s);
void gemm_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard);
bool fused_supported(const Shard& s);
void fused_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard);

// ---- dense fast path (kernels_dmma.cu) ----
bool dmma_supported(const Shard& s);
// Once per shard, outside stream capture: kernel attributes + co-resident cluster count.
void dmma_setup(Shard& s, int split = 1);
// Re-tune the DMMA layout for `split` concurrently running shards (1 = the whole GPU) when the
// shard's current layout was tuned for another split; drops its captured graphs.
void use_layout_split(Shard& s, int split);
void invalidate_graphs(Shard& s);
void dmma_pass(Shard& s, PassMode mode, const double* W, const int32_t* guard);
// Node-group passes (dmma_group.cuh): one full-GPU launch over several shards of equal (p, K) with
// whole-GPU layouts; per-node V / guards; tails on per-node sub-grids.
int dmma_group_clusters(Shard& s);
void dmma_group_pass(const std::vector<Shard*>& shards, int clusters, PassMode mode, const double* const* W,
                     const int32_t* const* guards, int tail, int cg_it, bool write_lp);

}  // namespace nadmm

namespace nadmm {
// Node-group solves (newton.cu): the local ADMM nodes' Newton iterations as one graph of group passes.
bool group_eligible(const std::vector<Shard*>& sh);
bool group_solve_launch(const std::vector<Shard*>& sh, const nadmm_newton_cfg& cfg, const double* rho);
void group_timers_finish(Ctx& c);
void group_forget(Shard& s);
void group_drop(Ctx& c);
// Grid-barrier watchdog control (common.cuh): push NADMM_BARRIER_TIMEOUT_MS to every translation
// unit's control block on the current device; raise NADMM_ECUDA if any barrier timed out.
void barrier_configure();
void barrier_check();
// cudaStreamSynchronize + the barrier fault check: every host synchronisation of the library.
void stream_sync(cudaStream_t st);
// Deferred release (capi.cu): a context outlives its shards / communicators, a shard its workers /
// sessions, whatever order the handles are freed in.
void ctx_unref(Ctx* c);
void shard_hold(Shard* s);
void shard_unhold(Shard* s);
}  // namespace nadmm

struct nadmm_ctx_s : nadmm::Ctx {};
struct nadmm_shard_s : nadmm::Shard {};
