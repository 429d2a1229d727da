// nadmm_cuda.hpp -- C++17 header-only wrapper that rebuilds the reference's solver/dataset API
// (/root/reference/proj/include/nadmm/{dataset,objective,newton,admm,common}.hpp) on top of the C ABI
// in nadmm_cuda.h, for C++ host code that wants the reference's shapes: Dataset factories, the
// objective-level functions, newton_solve with NewtonConfig / NewtonResult, the worker's ADMM
// branch and run_admm. Non-OK statuses are rethrown as the reference's exception types
// (inc/common.hpp:17-44). Link with -lnadmm_cuda (paper_1807_07132_b200/lib).
#ifndef NADMM_CUDA_HPP
#define NADMM_CUDA_HPP

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nadmm_cuda.h"

namespace nadmm_gpu {

using Vector = std::vector<double>;

// ---- errors (inc/common.hpp:17-44) ----
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : Error {
    using Error::Error;
};
struct DataError : Error {
    using Error::Error;
};
struct SolverError : Error {
    using Error::Error;
};
struct TransportError : Error {
    using Error::Error;
};
struct ProtocolError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};

inline void check(nadmm_status s) {
    if (s == NADMM_OK) return;
    const char* m = nadmm_last_error();
    const std::string msg = m ? m : "";
    switch (s) {
        case NADMM_ECONFIG: throw ConfigError(msg);
        case NADMM_EDATA: throw DataError(msg);
        case NADMM_ESOLVER: throw SolverError(msg);
        case NADMM_ETRANSPORT:
        case NADMM_ENCCL: throw TransportError(msg);
        case NADMM_EPROTOCOL: throw ProtocolError(msg);
        default: throw CudaError(msg);
    }
}

// ---- context (one per host thread and device) ----
class Context {
  public:
    explicit Context(int device = 0) { check(nadmm_ctx_create(device, &h_)); }
    ~Context() {
        if (h_) nadmm_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    nadmm_ctx handle() const { return h_; }
    void synchronize() const { check(nadmm_ctx_synchronize(h_)); }

  private:
    nadmm_ctx h_ = nullptr;
};

// ---- Dataset::dense / Dataset::sparse (inc/dataset.hpp:22-23) ----
class Dataset {
  public:
    // X row-major n x p, labels 1..C
    static std::shared_ptr<Dataset> dense(const Context& ctx, const Vector& X, int64_t n, int64_t p,
                                          const std::vector<int32_t>& labels, int32_t C) {
        if ((int64_t)X.size() != n * p || (int64_t)labels.size() != n) throw ConfigError("dense: shape mismatch");
        nadmm_shard h = nullptr;
        check(nadmm_shard_dense(ctx.handle(), X.data(), n, p, labels.data(), C, &h));
        return std::shared_ptr<Dataset>(new Dataset(h, n, p, C));
    }
    // CSR: indptr (n+1), column indices, values
    static std::shared_ptr<Dataset> sparse(const Context& ctx, const std::vector<int64_t>& indptr,
                                           const std::vector<int32_t>& indices, const Vector& vals, int64_t p,
                                           const std::vector<int32_t>& labels, int32_t C) {
        const int64_t n = (int64_t)indptr.size() - 1;
        if (n < 0 || (int64_t)labels.size() != n) throw ConfigError("sparse: shape mismatch");
        nadmm_shard h = nullptr;
        check(nadmm_shard_csr(ctx.handle(), indptr.data(), indices.data(), vals.data(), n, p, labels.data(), C, &h));
        return std::shared_ptr<Dataset>(new Dataset(h, n, p, C));
    }
    ~Dataset() {
        if (h_) nadmm_shard_free(h_);
    }
    Dataset(const Dataset&) = delete;
    Dataset& operator=(const Dataset&) = delete;
    nadmm_shard handle() const { return h_; }
    int64_t rows() const { return n_; }
    int64_t cols() const { return p_; }
    int32_t num_classes() const { return C_; }
    int64_t weight_dim() const { return (int64_t)(C_ - 1) * p_; }  // d = (C-1) p, block-major
    // original label values in class order (inc/dataset.hpp:46-50); set by the readers below
    const Vector& label_values() const { return label_values_; }
    void set_label_values(Vector v) { label_values_ = std::move(v); }

  private:
    Dataset(nadmm_shard h, int64_t n, int64_t p, int32_t C) : h_(h), n_(n), p_(p), C_(C) {}
    nadmm_shard h_ = nullptr;
    int64_t n_, p_;
    int32_t C_;
    Vector label_values_;
};

// ---- readers (inc/nadmm/data_io.hpp:52-65): load_libsvm -> sparse shard, load_idx -> dense ----
inline std::shared_ptr<Dataset> load_libsvm(const Context& ctx, const std::string& path) {
    nadmm_libsvm h = nullptr;
    int64_t n = 0, p = 0, nnz = 0;
    int32_t C = 0;
    check(nadmm_libsvm_parse(path.c_str(), &h, &n, &p, &nnz, &C));
    std::unique_ptr<nadmm_libsvm_s, void (*)(nadmm_libsvm)> guard(h, nadmm_libsvm_free);
    std::vector<int64_t> indptr((size_t)n + 1);
    std::vector<int32_t> indices((size_t)nnz), labels((size_t)n);
    Vector vals((size_t)nnz), values((size_t)C);
    check(nadmm_libsvm_fetch(h, indptr.data(), indices.data(), vals.data(), labels.data(), values.data()));
    auto ds = Dataset::sparse(ctx, indptr, indices, vals, p, labels, C);
    ds->set_label_values(std::move(values));
    return ds;
}

inline std::shared_ptr<Dataset> load_idx(const Context& ctx, const std::string& images, const std::string& labels) {
    int64_t n = 0, p = 0;
    check(nadmm_idx_info(images.c_str(), labels.c_str(), &n, &p));
    Vector X((size_t)(n * p)), values(256);
    std::vector<int32_t> y((size_t)n);
    int32_t C = 0;
    check(nadmm_idx_load(images.c_str(), labels.c_str(), X.data(), y.data(), &C, values.data()));
    values.resize((size_t)C);
    auto ds = Dataset::dense(ctx, X, n, p, y, C);
    ds->set_label_values(std::move(values));
    return ds;
}

// ---- model level (src/softmax.cpp:51-153), memoised on w like SoftmaxMemo ----
inline double loss(const Dataset& ds, const Vector& w, double lambda) {
    double f = 0.0;
    check(nadmm_loss(ds.handle(), w.data(), lambda, &f));
    return f;
}
inline Vector gradient(const Dataset& ds, const Vector& w, double lambda) {
    Vector g(w.size());
    check(nadmm_gradient(ds.handle(), w.data(), lambda, g.data()));
    return g;
}
inline Vector hessian_vec(const Dataset& ds, const Vector& w, const Vector& v, double lambda) {
    Vector hv(w.size());
    check(nadmm_hessian_vec(ds.handle(), w.data(), v.data(), lambda, hv.data()));
    return hv;
}
inline std::vector<int32_t> predict(const Dataset& ds, const Vector& w) {
    std::vector<int32_t> out((size_t)ds.rows());
    check(nadmm_predict(ds.handle(), w.data(), out.data()));
    return out;
}
inline double accuracy(const Dataset& ds, const Vector& w) {
    double a = 0.0;
    check(nadmm_accuracy(ds.handle(), w.data(), &a));
    return a;
}

// ---- newton_solve (inc/newton.hpp:9-68) ----
struct NewtonConfig {
    double cg_tol = 1e-4;
    int cg_max_iters = 10;
    double armijo_beta = 1e-4;
    double backtrack_gamma = 0.5;
    int ls_max_iters = 10;
    double grad_tol = 1e-8;
    int newton_max_iters = 100;
    nadmm_newton_cfg to_c() const {
        return nadmm_newton_cfg{cg_tol, cg_max_iters, armijo_beta, backtrack_gamma, ls_max_iters, grad_tol,
                                newton_max_iters};
    }
};

struct NewtonIterRecord {
    int iter;
    double grad_norm, step;
    int cg_iters;
    double cg_residual, objective;
    bool ls_capped, cg_fallback;
    int fn_evals;
};

struct NewtonResult {
    Vector x;
    std::vector<NewtonIterRecord> trace;
    bool converged = false;
    double final_grad_norm = 0.0;
};

// make_augmented_objective(rho, z, y) (src/objective.cpp:41-56), applied when `aug` is set
struct Augmentation {
    double rho;
    Vector z, y;
};

inline NewtonResult newton_solve(const Dataset& ds, double lambda, Vector x0, const NewtonConfig& cfg = {},
                                 const Augmentation* aug = nullptr) {
    const nadmm_newton_cfg c = cfg.to_c();
    std::vector<nadmm_newton_iter> tr((size_t)std::max(1, cfg.newton_max_iters));
    nadmm_newton_summary sum{};
    check(nadmm_newton_solve(ds.handle(), &c, lambda, aug ? 1 : 0, aug ? aug->rho : 0.0,
                             aug ? aug->z.data() : nullptr, aug ? aug->y.data() : nullptr, x0.data(), tr.data(),
                             (int32_t)tr.size(), &sum));
    NewtonResult r;
    r.x = std::move(x0);
    r.converged = sum.converged != 0;
    r.final_grad_norm = sum.final_grad_norm;
    for (int i = 0; i < sum.iterations && i < (int)tr.size(); ++i) {
        const nadmm_newton_iter& t = tr[(size_t)i];
        r.trace.push_back({t.iter, t.grad_norm, t.step, t.cg_iters, t.cg_residual, t.objective, t.ls_capped != 0,
                           t.cg_fallback != 0, t.fn_evals});
    }
    return r;
}

// ---- lbfgs_solve (inc/lbfgs.hpp:9-39) ----
struct LbfgsConfig {
    int history = 25;
    double wolfe_c1 = 1e-4;
    double wolfe_c2 = 0.9;
    int max_iters = 100;
    int ls_max_iters = 20;
    double grad_tol = 1e-8;
    nadmm_lbfgs_cfg to_c() const {
        return nadmm_lbfgs_cfg{history, wolfe_c1, wolfe_c2, max_iters, ls_max_iters, grad_tol};
    }
};

struct LbfgsIterRecord {
    int iter;
    double grad_norm, step, objective;
    int fn_evals;
    bool ls_fallback;
};

struct LbfgsResult {
    Vector x;
    std::vector<LbfgsIterRecord> trace;
    bool converged = false;
    double final_grad_norm = 0.0;
};

inline LbfgsResult lbfgs_solve(const Dataset& ds, double lambda, Vector x0, const LbfgsConfig& cfg = {},
                               const Augmentation* aug = nullptr) {
    const nadmm_lbfgs_cfg c = cfg.to_c();
    std::vector<nadmm_lbfgs_iter> tr((size_t)std::max(1, cfg.max_iters));
    nadmm_newton_summary sum{};
    check(nadmm_lbfgs_solve(ds.handle(), &c, lambda, aug ? 1 : 0, aug ? aug->rho : 0.0,
                            aug ? aug->z.data() : nullptr, aug ? aug->y.data() : nullptr, x0.data(), tr.data(),
                            (int32_t)tr.size(), &sum));
    LbfgsResult r;
    r.x = std::move(x0);
    r.converged = sum.converged != 0;
    r.final_grad_norm = sum.final_grad_norm;
    for (int i = 0; i < sum.iterations && i < (int)tr.size(); ++i) {
        const nadmm_lbfgs_iter& t = tr[(size_t)i];
        r.trace.push_back({t.iter, t.grad_norm, t.step, t.objective, t.fn_evals, t.ls_fallback != 0});
    }
    return r;
}

// ---- the worker's ADMM branch (src/worker.cpp:127-196) ----
struct InnerStats {
    double grad_norm;
    uint32_t inner_iters, cg_iters, fn_evals, flags;
};

class Worker {
  public:
    explicit Worker(std::shared_ptr<Dataset> ds) : ds_(std::move(ds)) { check(nadmm_worker_create(ds_->handle(), &h_)); }
    ~Worker() {
        if (h_) nadmm_worker_free(h_);
    }
    Worker(const Worker&) = delete;
    Worker& operator=(const Worker&) = delete;
    // one scatter -> gather round: x_local out, warm start kept on the device
    InnerStats solve(double rho, const Vector& z, const Vector& y, Vector& x_out, const NewtonConfig& cfg = {},
                     int inner_iters = 1) {
        const nadmm_newton_cfg c = cfg.to_c();
        x_out.resize((size_t)ds_->weight_dim());
        nadmm_inner_stats st{};
        check(nadmm_worker_solve(h_, rho, z.data(), y.data(), &c, inner_iters, x_out.data(), &st));
        return InnerStats{st.grad_norm, st.inner_iters, st.cg_iters, st.fn_evals, st.flags};
    }

    // the same round with the L-BFGS inner solver (src/worker.cpp:183-195)
    InnerStats solve_lbfgs(double rho, const Vector& z, const Vector& y, Vector& x_out, const LbfgsConfig& cfg = {},
                           int inner_iters = 1) {
        const nadmm_lbfgs_cfg c = cfg.to_c();
        x_out.resize((size_t)ds_->weight_dim());
        nadmm_inner_stats st{};
        check(nadmm_worker_solve_lbfgs(h_, rho, z.data(), y.data(), &c, inner_iters, x_out.data(), &st));
        return InnerStats{st.grad_norm, st.inner_iters, st.cg_iters, st.fn_evals, st.flags};
    }

  private:
    std::shared_ptr<Dataset> ds_;
    nadmm_worker h_ = nullptr;
};

// ---- run_admm (inc/admm.hpp:58-140) over this process's shards (comm: NCCL rank, or null) ----
struct AdmmResult {
    Vector z;
    std::vector<nadmm_metrics_row> metrics;
    bool converged = false;
    int iterations = 0;
    std::vector<double> rho;
};

inline nadmm_admm_cfg admm_defaults() {
    nadmm_admm_cfg c;
    nadmm_admm_cfg_default(&c);
    return c;
}

inline AdmmResult run_admm(const std::vector<std::shared_ptr<Dataset>>& parts, const nadmm_admm_cfg& cfg,
                           nadmm_comm comm = nullptr) {
    if (parts.empty()) throw ConfigError("run_admm needs at least one shard");
    std::vector<nadmm_shard> hs;
    for (const auto& p : parts) hs.push_back(p->handle());
    AdmmResult r;
    r.z.resize((size_t)parts[0]->weight_dim());
    r.rho.resize(parts.size());
    r.metrics.resize((size_t)std::max(1, cfg.max_outer_iters));
    int32_t it = 0, conv = 0;
    check(nadmm_admm_run(hs.data(), (int32_t)hs.size(), comm, &cfg, r.z.data(), r.rho.data(), r.metrics.data(),
                         (int32_t)r.metrics.size(), &it, &conv));
    r.iterations = it;
    r.converged = conv != 0;
    r.metrics.resize((size_t)std::min<int>(it, (int)r.metrics.size()));
    return r;
}

}  // namespace nadmm_gpu

#endif  // NADMM_CUDA_HPP
