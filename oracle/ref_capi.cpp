// extern "C" bridge onto the REFERENCE's own hot-path sources, compiled in place from
// /root/reference/proj/src/{dataset,softmax,objective,newton,lbfgs,data_io}.cpp against the Eigen
// stand-in in oracle/eigen_shim (Eigen itself is absent from this image; see eigen_shim/Eigen/Core).
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (as the checker), by __graft_entry__.smoke() and by
// bench.py's CPU-baseline / `--impl reference` arm. Never linked into the product library.
//
// Every function forwards to reference code unchanged; the only logic here is marshalling plain
// arrays into the reference's types and mapping its exceptions onto the status codes of
// include/nadmm_cuda.h (ConfigError 2, DataError 12, SolverError 3; inc/common.hpp:17-44).
#include "nadmm/data_io.hpp"
#include "nadmm/dataset.hpp"
#include "nadmm/lbfgs.hpp"
#include "nadmm/newton.hpp"
#include "nadmm/objective.hpp"
#include "nadmm/softmax.hpp"

#include <omp.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

using namespace nadmm;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const DataError& e) {
        g_err = e.what();
        return 12;
    } catch (const SolverError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

Vector vec_from(const double* p, std::int64_t d) {
    Vector v(static_cast<Index>(d));
    std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(d));
    return v;
}

void vec_to(const Vector& v, double* out) { std::memcpy(out, v.data(), sizeof(double) * static_cast<std::size_t>(v.size())); }

// A worker: the shard plus the persistent base objective and warm start, exactly the state
// run_worker keeps across scatters (src/worker.cpp:127-135).
struct RefWorker {
    std::shared_ptr<const Dataset> data;
    Objective base;
    Vector x_local;
};

NewtonConfig newton_cfg(const double* c) {
    NewtonConfig cfg;
    cfg.cg_tol = c[0];
    cfg.cg_max_iters = static_cast<int>(c[1]);
    cfg.armijo_beta = c[2];
    cfg.backtrack_gamma = c[3];
    cfg.ls_max_iters = static_cast<int>(c[4]);
    cfg.grad_tol = c[5];
    cfg.newton_max_iters = static_cast<int>(c[6]);
    return cfg;
}

// trace row layout (doubles): iter, grad_norm, step, cg_iters, cg_residual, objective, ls_capped,
// cg_fallback, fn_evals.
void pack_trace(const NewtonResult& r, double* trace, int cap, int* ntrace) {
    int k = 0;
    for (const auto& t : r.trace) {
        if (k >= cap) break;
        double* row = trace + 9 * k;
        row[0] = t.iter;
        row[1] = t.grad_norm;
        row[2] = t.step;
        row[3] = t.cg_iters;
        row[4] = t.cg_residual;
        row[5] = t.objective;
        row[6] = t.ls_capped;
        row[7] = t.cg_fallback;
        row[8] = t.fn_evals;
        ++k;
    }
    *ntrace = static_cast<int>(r.trace.size());
}
}  // namespace

extern "C" {

const char* nadmm_ref_last_error(void) { return g_err.c_str(); }

// OpenMP threads of the CALLING host thread's parallel regions (the Eigen stand-in's GEMM loops):
// a WorkerPool-style run gives each worker thread its share of the cores (src/worker.cpp:225-242).
int nadmm_ref_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
}

int nadmm_ref_dataset_dense(const double* X, std::int64_t n, std::int64_t p, const std::int32_t* labels, int C,
                            void** out) {
    return guard([&] {
        RowMatrix m(static_cast<Index>(n), static_cast<Index>(p));
        std::memcpy(m.data(), X, sizeof(double) * static_cast<std::size_t>(n * p));
        std::vector<std::int32_t> lab(labels, labels + n);
        *out = new Dataset(Dataset::dense(std::move(m), std::move(lab), C));
    });
}

int nadmm_ref_dataset_csr(const std::int64_t* indptr, const std::int32_t* indices, const double* vals, std::int64_t n,
                          std::int64_t p, const std::int32_t* labels, int C, void** out) {
    return guard([&] {
        std::vector<Eigen::Triplet<double>> trips;
        trips.reserve(static_cast<std::size_t>(indptr[n]));
        for (std::int64_t i = 0; i < n; ++i)
            for (std::int64_t k = indptr[i]; k < indptr[i + 1]; ++k) trips.emplace_back(i, indices[k], vals[k]);
        SparseRowMatrix m(static_cast<Index>(n), static_cast<Index>(p));
        m.setFromTriplets(trips.begin(), trips.end());
        std::vector<std::int32_t> lab(labels, labels + n);
        *out = new Dataset(Dataset::sparse(std::move(m), std::move(lab), C));
    });
}

void nadmm_ref_dataset_free(void* ds) { delete static_cast<Dataset*>(ds); }

int nadmm_ref_cache(void* ds, const double* w, double* logits, double* row_max, double* alpha, double* probs) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        StableExpCache c = stable_exp_cache(d, vec_from(w, d.weight_dim()));
        std::memcpy(logits, c.logits.data(), sizeof(double) * static_cast<std::size_t>(c.logits.size()));
        vec_to(c.row_max, row_max);
        vec_to(c.alpha, alpha);
        std::memcpy(probs, c.probs.data(), sizeof(double) * static_cast<std::size_t>(c.probs.size()));
    });
}

int nadmm_ref_loss(void* ds, const double* w, double lambda, double* out) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        *out = loss(d, vec_from(w, d.weight_dim()), lambda);
    });
}

int nadmm_ref_gradient(void* ds, const double* w, double lambda, double* g) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        vec_to(gradient(d, vec_from(w, d.weight_dim()), lambda), g);
    });
}

int nadmm_ref_hessian_vec(void* ds, const double* w, const double* v, double lambda, double* hv) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        vec_to(hessian_vec(d, vec_from(w, d.weight_dim()), vec_from(v, d.weight_dim()), lambda), hv);
    });
}

// Hv at a cache built once (the per-CG-iteration cost the benchmark times; src/softmax.cpp:97-112).
int nadmm_ref_hessian_vec_repeat(void* ds, const double* w, const double* v, double lambda, int reps, double* hv) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        const StableExpCache c = stable_exp_cache(d, vec_from(w, d.weight_dim()));
        const Vector vv = vec_from(v, d.weight_dim());
        Vector out;
        for (int r = 0; r < reps; ++r) out = hessian_vec(d, c, vv, lambda);
        vec_to(out, hv);
    });
}

int nadmm_ref_predict(void* ds, const double* w, std::int32_t* labels_out) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        const auto lab = predict(d, vec_from(w, d.weight_dim()));
        std::memcpy(labels_out, lab.data(), sizeof(std::int32_t) * lab.size());
    });
}

int nadmm_ref_exp_probe(void* ds, const double* w, const double* v, double* max_exponent) {
    return guard([&] {
        const Dataset& d = *static_cast<Dataset*>(ds);
        std::atomic<double> probe{-std::numeric_limits<double>::infinity()};
        detail::arm_exp_probe(&probe);
        const Vector ww = vec_from(w, d.weight_dim());
        (void)loss(d, ww, 0.0);
        (void)gradient(d, ww, 0.0);
        (void)hessian_vec(d, ww, vec_from(v, d.weight_dim()), 0.0);
        (void)predict(d, ww);
        detail::arm_exp_probe(nullptr);
        *max_exponent = probe.load();
    });
}

// Single-node solve (compute_reference semantics) or one augmented solve.
// cfg[7] = NewtonConfig fields in declaration order (inc/newton.hpp:9-17).
int nadmm_ref_newton_solve(void* ds, double lambda, int augmented, double rho, const double* z, const double* y,
                           const double* x0, const double* cfg, double* x_out, double* trace, int trace_cap,
                           int* ntrace, int* converged, double* final_grad_norm) {
    return guard([&] {
        auto data = std::make_shared<const Dataset>(*static_cast<Dataset*>(ds));
        const Index d = data->weight_dim();
        Objective obj = make_softmax_objective(data, lambda);
        if (augmented) obj = make_augmented_objective(obj, rho, vec_from(z, d), vec_from(y, d));
        NewtonResult r = newton_solve(obj, vec_from(x0, d), newton_cfg(cfg));
        vec_to(r.x, x_out);
        pack_trace(r, trace, trace_cap, ntrace);
        *converged = r.converged ? 1 : 0;
        *final_grad_norm = r.final_grad_norm;
    });
}

// ---- worker (run_worker ADMM branch, src/worker.cpp:127-196) ----
int nadmm_ref_worker_create(void* ds, void** out) {
    return guard([&] {
        auto* w = new RefWorker;
        w->data = std::make_shared<const Dataset>(*static_cast<Dataset*>(ds));
        w->base = make_softmax_objective(w->data, 0.0);  // src/worker.cpp:130
        w->x_local = Vector::Zero(w->data->weight_dim());  // src/worker.cpp:135
        *out = w;
    });
}

void nadmm_ref_worker_free(void* w) { delete static_cast<RefWorker*>(w); }

// stats[5] = grad_norm, inner_iters, cg_iters, fn_evals, flags (InnerStats, src/worker.cpp:176-183)
int nadmm_ref_worker_solve(void* wp, double rho, const double* z, const double* y, const double* cfg, int inner_iters,
                           double* x_out, double* stats) {
    return guard([&] {
        RefWorker& w = *static_cast<RefWorker*>(wp);
        const Index d = w.data->weight_dim();
        Objective aug = make_augmented_objective(w.base, rho, vec_from(z, d), vec_from(y, d));
        NewtonConfig c = newton_cfg(cfg);
        c.newton_max_iters = inner_iters;  // src/worker.cpp:173
        NewtonResult res = newton_solve(aug, w.x_local, c);
        w.x_local = std::move(res.x);
        std::uint32_t cg = 0, fe = 0, flags = 0;
        for (const auto& t : res.trace) {
            cg += static_cast<std::uint32_t>(t.cg_iters);
            fe += static_cast<std::uint32_t>(t.fn_evals);
            if (t.ls_capped) flags |= 1;
            if (t.cg_fallback) flags |= 2;
        }
        stats[0] = res.final_grad_norm;
        stats[1] = static_cast<double>(res.trace.size());
        stats[2] = cg;
        stats[3] = fe;
        stats[4] = flags;
        vec_to(w.x_local, x_out);
    });
}

// ---- solver pieces on caller-supplied operators (SPEC known answers) ----
typedef void (*nadmm_ref_apply_fn)(const double* in, double* out, std::int64_t d, void* user);
typedef double (*nadmm_ref_value_fn)(const double* x, std::int64_t d, void* user);

int nadmm_ref_cg_solve(nadmm_ref_apply_fn apply, void* user, const double* g, std::int64_t d, double theta,
                       int max_iters, double* p_out, int* iters, double* achieved, int* negative_curvature) {
    return guard([&] {
        auto H = [&](const Vector& v) {
            Vector out(static_cast<Index>(d));
            apply(v.data(), out.data(), d, user);
            return out;
        };
        CgResult r = cg_solve(H, vec_from(g, d), theta, max_iters);
        vec_to(r.p, p_out);
        *iters = r.iters;
        *achieved = r.achieved_residual;
        *negative_curvature = r.negative_curvature ? 1 : 0;
    });
}

int nadmm_ref_line_search(nadmm_ref_value_fn value, void* user, const double* x, const double* p, const double* g,
                          std::int64_t d, double f_x, const double* cfg, double* alpha, int* evals, int* capped) {
    return guard([&] {
        Objective obj;
        obj.value = [&](const Vector& xx) { return value(xx.data(), d, user); };
        LineSearchResult r = line_search(obj, vec_from(x, d), vec_from(p, d), vec_from(g, d), f_x, newton_cfg(cfg));
        *alpha = r.alpha;
        *evals = r.evals;
        *capped = r.capped ? 1 : 0;
    });
}

// Newton on a caller-supplied quadratic-like objective: value/grad/hvp callbacks.
typedef void (*nadmm_ref_grad_fn)(const double* x, double* g, std::int64_t d, void* user);
typedef void (*nadmm_ref_hvp_fn)(const double* x, const double* v, double* out, std::int64_t d, void* user);

int nadmm_ref_newton_solve_cb(nadmm_ref_value_fn value, nadmm_ref_grad_fn grad, nadmm_ref_hvp_fn hvp, void* user,
                              const double* x0, std::int64_t d, const double* cfg, double* x_out, double* trace,
                              int trace_cap, int* ntrace, int* converged, double* final_grad_norm) {
    return guard([&] {
        Objective obj;
        obj.value = [&](const Vector& x) { return value(x.data(), d, user); };
        obj.grad = [&](const Vector& x) {
            Vector g(static_cast<Index>(d));
            grad(x.data(), g.data(), d, user);
            return g;
        };
        obj.hvp = [&](const Vector& x, const Vector& v) {
            Vector o(static_cast<Index>(d));
            hvp(x.data(), v.data(), o.data(), d, user);
            return o;
        };
        NewtonResult r = newton_solve(obj, vec_from(x0, d), newton_cfg(cfg));
        vec_to(r.x, x_out);
        pack_trace(r, trace, trace_cap, ntrace);
        *converged = r.converged ? 1 : 0;
        *final_grad_norm = r.final_grad_norm;
    });
}

// L-BFGS inner solver (SURVEY §8f "next" #1): lcfg = history, c1, c2, max_iters, ls_max_iters, grad_tol.
// trace rows (doubles): iter, grad_norm, step, objective, fn_evals, ls_fallback.
int nadmm_ref_lbfgs_solve(void* ds, double lambda, int augmented, double rho, const double* z, const double* y,
                          const double* x0, const double* lcfg, double* x_out, double* trace, int trace_cap,
                          int* iters, int* converged, double* final_grad_norm) {
    return guard([&] {
        auto data = std::make_shared<const Dataset>(*static_cast<Dataset*>(ds));
        const Index d = data->weight_dim();
        Objective obj = make_softmax_objective(data, lambda);
        if (augmented) obj = make_augmented_objective(obj, rho, vec_from(z, d), vec_from(y, d));
        LbfgsConfig c;
        c.history = static_cast<int>(lcfg[0]);
        c.wolfe_c1 = lcfg[1];
        c.wolfe_c2 = lcfg[2];
        c.max_iters = static_cast<int>(lcfg[3]);
        c.ls_max_iters = static_cast<int>(lcfg[4]);
        c.grad_tol = lcfg[5];
        LbfgsResult r = lbfgs_solve(obj, vec_from(x0, d), c);
        vec_to(r.x, x_out);
        int k = 0;
        for (const auto& t : r.trace) {
            if (k >= trace_cap) break;
            double* row = trace + 6 * k++;
            row[0] = t.iter;
            row[1] = t.grad_norm;
            row[2] = t.step;
            row[3] = t.objective;
            row[4] = t.fn_evals;
            row[5] = t.ls_fallback ? 1.0 : 0.0;
        }
        *iters = static_cast<int>(r.trace.size());
        *converged = r.converged ? 1 : 0;
        *final_grad_norm = r.final_grad_norm;
    });
}

// ---- data fixtures (src/data_io.cpp:16-43, 300-370) ----
int nadmm_ref_generate_synthetic(std::int64_t n, std::int64_t p, int C, double separation, double noise,
                                 std::uint64_t seed, double* X_train, std::int32_t* y_train, double* X_test,
                                 std::int32_t* y_test) {
    return guard([&] {
        SyntheticSpec s;
        s.n = n;
        s.p = p;
        s.num_classes = C;
        s.separation = separation;
        s.noise = noise;
        s.seed = seed;
        auto [train, test] = generate_synthetic(s);
        std::memcpy(X_train, train.dense_features().data(), sizeof(double) * static_cast<std::size_t>(train.n() * p));
        std::memcpy(y_train, train.labels().data(), sizeof(std::int32_t) * static_cast<std::size_t>(train.n()));
        std::memcpy(X_test, test.dense_features().data(), sizeof(double) * static_cast<std::size_t>(test.n() * p));
        std::memcpy(y_test, test.labels().data(), sizeof(std::int32_t) * static_cast<std::size_t>(test.n()));
    });
}

// Row-to-worker assignment of partition() (src/data_io.cpp:300-328): owner[i] for each row i, via
// the reference's own subset of a dense index-tagged dataset.
int nadmm_ref_partition(std::int64_t n, int n_workers, int strided, std::int32_t* owner) {
    return guard([&] {
        RowMatrix tags(static_cast<Index>(n), 1);
        for (Index i = 0; i < n; ++i) tags(i, 0) = static_cast<double>(i);
        Dataset all = Dataset::dense(std::move(tags), std::vector<std::int32_t>(static_cast<std::size_t>(n), 1), 2);
        PartitionPlan plan;
        plan.n_workers = n_workers;
        plan.scheme = strided ? PartitionScheme::strided : PartitionScheme::contiguous;
        const auto parts = partition(all, plan);
        for (std::size_t w = 0; w < parts.size(); ++w)
            for (Index r = 0; r < parts[w].n(); ++r)
                owner[static_cast<std::size_t>(parts[w].dense_features()(r, 0))] = static_cast<std::int32_t>(w);
    });
}

// Raw Rng stream (src/data_io.cpp:16-43): kind 0 uniform, 1 normal, 2 uniform_int(bound).
int nadmm_ref_rng_stream(std::uint64_t seed, int kind, std::uint64_t bound, std::int64_t count, double* out) {
    return guard([&] {
        detail::Rng rng(seed);
        for (std::int64_t i = 0; i < count; ++i)
            out[i] = kind == 0 ? rng.uniform() : kind == 1 ? rng.normal() : static_cast<double>(rng.uniform_int(bound));
    });
}

// ---- real-data readers (src/data_io.cpp:85-137 load_libsvm, 220-271 load_idx) ----
// The loaded Dataset stays on the heap behind an opaque handle; info + fetch copy it out.
int nadmm_ref_load_libsvm(const char* path, void** out) {
    return guard([&] { *out = new Dataset(load_libsvm(path)); });
}

int nadmm_ref_load_idx(const char* images, const char* labels, void** out) {
    return guard([&] { *out = new Dataset(load_idx(images, labels)); });
}

int nadmm_ref_dataset_info(void* h, std::int64_t* n, std::int64_t* p, std::int64_t* nnz, int* C, int* is_sparse) {
    return guard([&] {
        const Dataset& ds = *static_cast<Dataset*>(h);
        *n = ds.n();
        *p = ds.p();
        *nnz = ds.is_sparse() ? static_cast<std::int64_t>(ds.sparse_features().nonZeros()) : ds.n() * ds.p();
        *C = ds.num_classes();
        *is_sparse = ds.is_sparse() ? 1 : 0;
    });
}

// Sparse: indptr (n+1, widened to int64), indices (nnz), vals (nnz). Dense: vals = X (n x p).
int nadmm_ref_dataset_fetch(void* h, std::int64_t* indptr, std::int32_t* indices, double* vals, std::int32_t* labels,
                            double* label_values) {
    return guard([&] {
        const Dataset& ds = *static_cast<Dataset*>(h);
        if (ds.is_sparse()) {
            const auto& S = ds.sparse_features();
            for (Index i = 0; i <= ds.n(); ++i) indptr[i] = S.outerIndexPtr()[i];
            const auto nnz = static_cast<std::size_t>(S.nonZeros());
            for (std::size_t k = 0; k < nnz; ++k) indices[k] = S.innerIndexPtr()[k];
            std::memcpy(vals, S.valuePtr(), sizeof(double) * nnz);
        } else {
            std::memcpy(vals, ds.dense_features().data(), sizeof(double) * static_cast<std::size_t>(ds.n() * ds.p()));
        }
        std::memcpy(labels, ds.labels().data(), sizeof(std::int32_t) * static_cast<std::size_t>(ds.n()));
        const auto& lv = ds.label_values();
        if (!lv.empty()) std::memcpy(label_values, lv.data(), sizeof(double) * lv.size());
    });
}

// detail::Rng(seed).shuffle of 0..n-1 (inc/data_io.hpp:23-28): the SGD worker's permutation.
int nadmm_ref_shuffle(std::uint64_t seed, std::int64_t n, std::int64_t* out) {
    return guard([&] {
        std::vector<Index> perm(static_cast<std::size_t>(n));
        for (Index i = 0; i < n; ++i) perm[static_cast<std::size_t>(i)] = i;
        detail::Rng rng(seed);
        rng.shuffle(perm);
        for (Index i = 0; i < n; ++i) out[i] = perm[static_cast<std::size_t>(i)];
    });
}

// Dataset::subset (src/dataset.cpp:87-115), the SGD mini-batch.
int nadmm_ref_subset(void* ds, const std::int64_t* rows, std::int64_t m, void** out) {
    return guard([&] {
        std::vector<Index> r(rows, rows + m);
        *out = new Dataset(static_cast<Dataset*>(ds)->subset(r));
    });
}

}  // extern "C"

