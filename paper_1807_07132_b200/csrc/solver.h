// Host-side solver entry points shared by the C ABI, the worker and the ADMM driver.
#pragma once

#include <functional>
#include <vector>

#include "state.h"

namespace nadmm {

struct SolveResult {
    int error = 0;
    int iterations = 0;
    bool converged = false;
    double final_grad_norm = 0.0;
    std::vector<DevTrace> trace;
    int cg_sum = 0, fe_sum = 0, flags = 0;
};

void validate_newton_cfg(const nadmm_newton_cfg& c);
void set_params(Shard& s, const nadmm_newton_cfg& c, double lambda, bool aug, double rho);
void set_lambda_only(Shard& s, double lambda);
void ensure_cache_at_x(Shard& s, double lambda);
// newton_solve (src/newton.cpp:73-132) from s.x with z/y in s.z/s.y; result x left in s.x.
// Split form for callers that run several shards back to back: solve_launch enqueues the solve
// (returns false when the result is still pending: newton_max == 1 needs no host decision) and
// solve_collect reads it back.
bool solve_launch(Shard& s, const nadmm_newton_cfg& cfg, double lambda, bool aug, double rho, int newton_max);
SolveResult solve_collect(Shard& s, const nadmm_newton_cfg& cfg, bool pending);
// Fully asynchronous gather: enqueue the state/trace copies, synchronise elsewhere, then build the
// result from the host copies with solve_result.
void solve_readback_async(Shard& s);
SolveResult solve_result(Shard& s, const nadmm_newton_cfg& cfg);
SolveResult device_newton_solve(Shard& s, const nadmm_newton_cfg& cfg, double lambda, bool aug, double rho,
                                int newton_max);

// lbfgs_solve (src/lbfgs.cpp:94-181) from s.x (z / y in s.z / s.y when augmented); x left in s.x.
constexpr int kLbMaxHist = 256;
using LbfgsCfg = nadmm_lbfgs_cfg;
struct LbfgsResult {
    std::vector<nadmm_lbfgs_iter> trace;
    bool converged = false;
    double final_grad_norm = 0.0;
};
void validate_lbfgs_cfg(const LbfgsCfg& c);
LbfgsResult device_lbfgs_solve(Shard& s, const LbfgsCfg& cfg, double lambda, bool aug, double rho);
// Synchronous mini-batch SGD (sgd.cu; src/worker.cpp:197-218).
void epoch_permutation(uint64_t seed, int64_t n, int32_t* perm);
void validate_sgd(const Shard& s, const nadmm_sgd_cfg& c);
void sgd_worker_grad(Shard& s, const nadmm_sgd_cfg& c, uint32_t iteration, const double* z, double* g);
struct SgdReduce {  // cross-rank sums (NCCL), absent on a single rank
    std::function<void(double*, int)> host;
    std::function<void(double*, int64_t)> dev;
};
struct SgdOutcome {
    int epochs = 0;
    int steps_per_epoch = 0;
    double f0 = 0.0, final_objective = 0.0;
};
SgdOutcome sgd_run(std::vector<Shard*>& shards, const SgdReduce* red, const nadmm_sgd_cfg& cfg, double lambda,
                   double* x_dev, nadmm_metrics_row* rows, int row_cap);

// InnerStats of an L-BFGS worker round (src/worker.cpp:186-194).
inline nadmm_inner_stats lbfgs_inner_stats(const LbfgsResult& r) {
    nadmm_inner_stats st{r.final_grad_norm, (uint32_t)r.trace.size(), 0u, 0u, 0u};
    for (const auto& t : r.trace) {
        st.fn_evals += (uint32_t)t.fn_evals;
        if (t.ls_fallback) st.flags |= 1u;
    }
    return st;
}

}  // namespace nadmm
