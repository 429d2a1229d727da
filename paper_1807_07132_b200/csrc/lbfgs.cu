// L-BFGS on a device shard: lbfgs_solve (src/lbfgs.cpp:94-181) with the
// strong-Wolfe bracket-and-zoom search (src/lbfgs.cpp:40-90) over make_softmax_objective, optionally
// wrapped by make_augmented_objective (src/objective.cpp:41-56).
//
// Every vector (iterate, gradient, direction, trial point, curvature history) lives on the device;
// each function evaluation is one fused cache+gradient data pass plus a gradient/dot kernel. The
// two-loop recursion is ONE kernel on one thread-block cluster: its 2m dependent dot products are
// cluster barriers with the partials summed through distributed shared memory in rank order, each
// fused with the vector update that precedes it. The scalar control flow (Wolfe tests, history
// ring, trace) stays on the host exactly as in the reference; it reads back a few scalars per
// evaluation.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <deque>
#include <string>

#include "solver.h"
#include "solver_tails.cuh"

namespace nadmm {

namespace {

constexpr int kLbThreads = 256;
constexpr int kLbMaxBlocks = 1024;
constexpr int kLbClusterCtas = 8;  // portable cluster size
constexpr int kLbClThreads = 1024;

struct LbHist {  // history in reference order (oldest first): ring slot and rho = 1 / s'y
    int m;
    int slot[kLbMaxHist];
    double rho[kLbMaxHist];
};

// x + a p, evaluated like the reference's `x + a * p` (no fused multiply-add).
__global__ void k_lb_point(int64_t d, const double* __restrict__ x, double a, const double* __restrict__ p,
                           double* __restrict__ xa) {
    GRID_STRIDE(j, d) xa[j] = __dadd_rn(x[j], __dmul_rn(a, p[j]));
}

// Full gradient at w from the base gradient: g = gbase - rho t, t = (z - w) + y / rho
// (src/objective.cpp:47-51). Block partials (rows of nb): <g,g>, <t,t>, <g,p>.
__global__ void __launch_bounds__(kLbThreads) k_lb_grad(int64_t d, const double* __restrict__ w,
                                                        const double* __restrict__ gbase, const double* __restrict__ z,
                                                        const double* __restrict__ y, double rho, int aug,
                                                        const double* __restrict__ p, double* __restrict__ g,
                                                        double* __restrict__ part) {
    __shared__ double red[32];
    double gg = 0.0, tt = 0.0, gp = 0.0;
    GRID_STRIDE(j, d) {
        double gj = gbase[j];
        if (aug) {
            const double tj = __dadd_rn(__dsub_rn(z[j], w[j]), __ddiv_rn(y[j], rho));
            tt += tj * tj;
            gj = __dsub_rn(gj, __dmul_rn(rho, tj));
        }
        g[j] = gj;
        gg += gj * gj;
        if (p) gp += gj * p[j];
    }
    const int nb = gridDim.x;
    double s = block_sum(gg, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    s = block_sum(tt, red);
    if (threadIdx.x == 0) part[nb + blockIdx.x] = s;
    s = block_sum(gp, red);
    if (threadIdx.x == 0) part[2 * nb + blockIdx.x] = s;
}

// Curvature pair s = xn - x, y = gn - g into its history slot. Partials: <s,y>, <s,s>, <y,y>.
__global__ void __launch_bounds__(kLbThreads) k_lb_pair(int64_t d, const double* __restrict__ xn,
                                                        const double* __restrict__ x, const double* __restrict__ gn,
                                                        const double* __restrict__ g, double* __restrict__ S,
                                                        double* __restrict__ Y, double* __restrict__ part) {
    __shared__ double red[32];
    double sy = 0.0, ss = 0.0, yy = 0.0;
    GRID_STRIDE(j, d) {
        const double sj = __dsub_rn(xn[j], x[j]), yj = __dsub_rn(gn[j], g[j]);
        S[j] = sj;
        Y[j] = yj;
        sy += sj * yj;
        ss += sj * sj;
        yy += yj * yj;
    }
    const int nb = gridDim.x;
    double s = block_sum(sy, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    s = block_sum(ss, red);
    if (threadIdx.x == 0) part[nb + blockIdx.x] = s;
    s = block_sum(yy, red);
    if (threadIdx.x == 0) part[2 * nb + blockIdx.x] = s;
}

// out[r] = fixed-order sum of partial row r; out[rows] = *extra (the base loss) when given.
__global__ void k_lb_sum(const double* __restrict__ part, int nb, int rows, const double* extra, double* out) {
    if (threadIdx.x >= 32) return;
    for (int r = 0; r < rows; ++r) {
        const double v = reduce_partials(part + (int64_t)r * nb, nb);
        if (threadIdx.x == 0) out[r] = v;
    }
    if (extra && threadIdx.x == 0) out[rows] = *extra;
}

// Block sum -> this CTA's slot; cluster barrier; every CTA sums the slots in rank order (identical
// result in all CTAs). Slots alternate between two buffers: a slot is rewritten only after the next
// barrier, which every reader of the previous value has passed.
__device__ __forceinline__ double lb_cluster_sum(cooperative_groups::cluster_group& cl, double* slot, double v,
                                                 double* red, double* bcast) {
    const double t = block_sum(v, red);
    if (threadIdx.x == 0) *slot = t;
    cl.sync();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (unsigned q = 0; q < cl.num_blocks(); ++q) s += *cl.map_shared_rank(slot, q);
        *bcast = s;
    }
    __syncthreads();
    return *bcast;
}

// Two-loop recursion (src/lbfgs.cpp:113-134): p = -H g with H0 = gamma I; if p'g >= 0, p = -g and
// slope = -|g|^2. Writes p and out[0] = slope. q (the working vector) is d doubles of scratch.
__global__ void __launch_bounds__(kLbClThreads, 1) k_lb_direction(int64_t d, const double* __restrict__ g,
                                                                  const double* __restrict__ S,
                                                                  const double* __restrict__ Y, LbHist h,
                                                                  double gamma, double* __restrict__ q,
                                                                  double* __restrict__ p, double* out) {
    namespace cgs = cooperative_groups;
    cgs::cluster_group cl = cgs::this_cluster();
    __shared__ double red[32];
    __shared__ double slots[2];
    __shared__ double bc;
    __shared__ double alpha[kLbMaxHist];
    const int m = h.m;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int par = 0;
    auto Sv = [&](int i) { return S + (int64_t)h.slot[i] * d; };
    auto Yv = [&](int i) { return Y + (int64_t)h.slot[i] * d; };
    // q = g, with the partial of s_{m-1}'q
    double acc = 0.0;
    {
        const double* s_last = m > 0 ? Sv(m - 1) : nullptr;
        for (int64_t j = j0; j < d; j += stride) {
            const double v = g[j];
            q[j] = v;
            if (s_last) acc += s_last[j] * v;
        }
    }
    for (int i = m - 1; i >= 0; --i) {  // alpha_i = rho_i s_i'q; q -= alpha_i y_i
        const double a = h.rho[i] * lb_cluster_sum(cl, &slots[par], acc, red, &bc);
        par ^= 1;
        if (threadIdx.x == 0) alpha[i] = a;
        const double* yi = Yv(i);
        const double* sn = i > 0 ? Sv(i - 1) : nullptr;
        acc = 0.0;
        for (int64_t j = j0; j < d; j += stride) {
            const double v = __dsub_rn(q[j], __dmul_rn(a, yi[j]));
            q[j] = v;
            if (sn) acc += sn[j] * v;
        }
    }
    __syncthreads();  // alpha[] visible to the whole CTA
    {  // r = gamma q, with the partial of y_0'r
        const double* y0 = m > 0 ? Yv(0) : nullptr;
        acc = 0.0;
        for (int64_t j = j0; j < d; j += stride) {
            const double v = __dmul_rn(gamma, q[j]);
            q[j] = v;
            if (y0) acc += y0[j] * v;
        }
    }
    for (int i = 0; i < m; ++i) {  // beta = rho_i y_i'r; r += (alpha_i - beta) s_i
        const double beta = h.rho[i] * lb_cluster_sum(cl, &slots[par], acc, red, &bc);
        par ^= 1;
        const double c = alpha[i] - beta;
        const double* si = Sv(i);
        const double* yn = i + 1 < m ? Yv(i + 1) : nullptr;
        acc = 0.0;
        for (int64_t j = j0; j < d; j += stride) {
            const double v = __dadd_rn(q[j], __dmul_rn(c, si[j]));
            q[j] = v;
            if (yn) acc += yn[j] * v;
        }
    }
    // p = -r and slope = p'g; |g|^2 for the descent fallback
    double pg = 0.0, gg = 0.0;
    for (int64_t j = j0; j < d; j += stride) {
        const double pj = -q[j], gj = g[j];
        p[j] = pj;
        pg += pj * gj;
        gg += gj * gj;
    }
    const double slope = lb_cluster_sum(cl, &slots[par], pg, red, &bc);
    par ^= 1;
    const double g_sq = lb_cluster_sum(cl, &slots[par], gg, red, &bc);
    if (slope >= 0.0)  // cluster-uniform decision (src/lbfgs.cpp:131-134)
        for (int64_t j = j0; j < d; j += stride) p[j] = -g[j];
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = slope >= 0.0 ? -g_sq : slope;
    cl.sync();  // no CTA exits while peers may still read its slots
}

struct Lbfgs {
    Shard& s;
    const LbfgsCfg& cfg;
    bool aug;
    double rho;
    cudaStream_t st;
    int64_t d;
    int nb;
    double* S;  // (history + 1) x d curvature pairs s_i, then the same for y_i
    double* Y;
    double* vp;  // direction
    double* vq;  // two-loop working vector
    double* part;
    double* out;
    double* x;
    double* g;
    double* xa;
    double* ga;
    double host[4] = {0, 0, 0, 0};

    Lbfgs(Shard& sh, const LbfgsCfg& c, bool a, double r)
        : s(sh), cfg(c), aug(a), rho(r), st(sh.ctx->stream), d(sh.d),
          nb((int)std::min<int64_t>(kLbMaxBlocks, std::max<int64_t>(1, (sh.d + kLbThreads - 1) / kLbThreads))) {
        // one workspace per shard, grown on demand and reused by later solves (no per-solve allocation)
        const int64_t hist = (int64_t)(c.history + 1) * d;
        const int64_t need = 2 * hist + 6 * d + 3 * (int64_t)kLbMaxBlocks + 4;
        if (sh.lb_ws_len < need) {
            if (sh.lb_ws) {
                stream_sync(st);
                cudaFree(sh.lb_ws);
                sh.bytes -= 8 * sh.lb_ws_len;
                sh.lb_ws = nullptr;
                sh.lb_ws_len = 0;
            }
            NADMM_CUDA(cudaMalloc(&sh.lb_ws, sizeof(double) * (size_t)need));
            sh.lb_ws_len = need;
            sh.bytes += 8 * need;
        }
        double* w = sh.lb_ws;
        S = w;
        Y = S + hist;
        x = Y + hist;
        g = x + d;
        xa = g + d;
        ga = xa + d;
        vp = ga + d;
        vq = vp + d;
        part = vq + d;
        out = part + 3 * kLbMaxBlocks;
    }

    void fetch(int n) {
        NADMM_CUDA(cudaMemcpyAsync(host, out, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        stream_sync(st);
    }

    // f(w), |g(w)|^2 and g(w)'p (p may be null); the gradient lands in gout.
    void eval(const double* w, double* gout, const double* p, double& f, double& gsq, double& gp) {
        op_cache_grad(s, w, nullptr);  // base loss (ridge included) -> scal[0], base gradient -> gbase
        k_lb_grad<<<nb, kLbThreads, 0, st>>>(d, w, s.gbase, s.z, s.y, rho, aug ? 1 : 0, p, gout, part);
        NADMM_LAUNCH_CHECK();
        k_lb_sum<<<1, 32, 0, st>>>(part, nb, 3, s.scal, out);
        NADMM_LAUNCH_CHECK();
        s.ctx->stats.kernel_launches += 2;
        fetch(4);
        f = aug ? host[3] + 0.5 * rho * host[1] : host[3];  // src/objective.cpp:44-46
        gsq = host[0];
        gp = host[2];
    }

    void point(const double* base, double a, const double* dir, double* dst) {
        const int grid = (int)std::min<int64_t>(4 * (int64_t)s.ctx->num_sms, (d + kLbThreads - 1) / kLbThreads);
        k_lb_point<<<std::max(grid, 1), kLbThreads, 0, st>>>(d, base, a, dir, dst);
        NADMM_LAUNCH_CHECK();
        s.ctx->stats.kernel_launches++;
    }

    // Phi (src/lbfgs.cpp:19-31): f(x + a p) and the directional derivative, into xa / ga.
    int evals = 0;
    std::pair<double, double> phi(double a) {
        point(x, a, vp, xa);
        ++evals;
        double f, gsq, gp;
        eval(xa, ga, vp, f, gsq, gp);
        last_f = f;
        last_gsq = gsq;
        return {f, gp};
    }
    double last_f = 0.0, last_gsq = 0.0;

    struct Wolfe {
        double alpha = 0.0;
        int evals = 0;
        bool ok = false;
    };

    // Bracket-and-zoom strong-Wolfe search (src/lbfgs.cpp:40-90), bisection inside zoom.
    Wolfe strong_wolfe(double f0, double slope0) {
        evals = 0;
        Wolfe w;
        auto zoom = [&](double lo, double f_lo, double hi) {
            while (evals < cfg.ls_max_iters) {
                const double a = 0.5 * (lo + hi);
                const auto [fa, ga_] = phi(a);
                if (fa > f0 + cfg.wolfe_c1 * a * slope0 || fa >= f_lo) {
                    hi = a;
                } else {
                    if (std::abs(ga_) <= -cfg.wolfe_c2 * slope0) {
                        w.alpha = a;
                        w.ok = true;
                        return;
                    }
                    if (ga_ * (hi - lo) >= 0.0) hi = lo;
                    lo = a;
                    f_lo = fa;
                }
            }
        };
        double a_prev = 0.0, f_prev = f0, a = 1.0;
        const double a_max = 1e6;
        for (int i = 0; evals < cfg.ls_max_iters; ++i) {
            const auto [fa, ga_] = phi(a);
            if (fa > f0 + cfg.wolfe_c1 * a * slope0 || (i > 0 && fa >= f_prev)) {
                zoom(a_prev, f_prev, a);
                break;
            }
            if (std::abs(ga_) <= -cfg.wolfe_c2 * slope0) {
                w.alpha = a;
                w.ok = true;
                break;
            }
            if (ga_ >= 0.0) {
                zoom(a, fa, a_prev);
                break;
            }
            a_prev = a;
            f_prev = fa;
            a = std::min(2.0 * a, a_max);
        }
        w.evals = evals;
        return w;
    }

    LbfgsResult run() {
        LbfgsResult res;
        std::deque<int> hist;  // ring slots, oldest first
        std::deque<double> rho_h, sy_h, yy_h;
        double f_x, g_sq, unused;
        eval(x, g, nullptr, f_x, g_sq, unused);  // g = grad(x0); f_x = value(x0) (src/lbfgs.cpp:102-103)
        for (int k = 0; k < cfg.max_iters; ++k) {
            const double g_norm = std::sqrt(g_sq);
            res.final_grad_norm = g_norm;
            if (g_norm < cfg.grad_tol) {
                res.converged = true;
                return res;
            }
            LbHist h{};
            h.m = (int)hist.size();
            for (int i = 0; i < h.m; ++i) {
                h.slot[i] = hist[(size_t)i];
                h.rho[i] = rho_h[(size_t)i];
            }
            const double gamma = hist.empty() ? 1.0 : sy_h.back() / yy_h.back();
            launch_direction(h, gamma);
            fetch(1);
            const double slope = host[0];
            nadmm_lbfgs_iter rec{};
            rec.iter = k;
            rec.grad_norm = g_norm;
            const Wolfe ls = strong_wolfe(f_x, slope);
            rec.fn_evals = ls.evals;
            double f_next, gsq_next;
            if (ls.ok) {  // x_next = x + alpha p is the accepted (last evaluated) trial point
                rec.step = ls.alpha;
                f_next = last_f;
                gsq_next = last_gsq;
            } else {
                std::fprintf(stderr, "[lbfgs] Wolfe search failed at iter %d; taking -g step\n", k);
                rec.ls_fallback = 1;
                rec.step = 1e-3;
                point(x, -1e-3, g, xa);
                eval(xa, ga, nullptr, f_next, gsq_next, unused);
            }
            // curvature pair into a free ring slot (src/lbfgs.cpp:153-166)
            int free_slot = 0;
            while (std::find(hist.begin(), hist.end(), free_slot) != hist.end()) ++free_slot;
            k_lb_pair<<<nb, kLbThreads, 0, st>>>(d, xa, x, ga, g, S + (int64_t)free_slot * d,
                                                 Y + (int64_t)free_slot * d, part);
            NADMM_LAUNCH_CHECK();
            k_lb_sum<<<1, 32, 0, st>>>(part, nb, 3, nullptr, out);
            NADMM_LAUNCH_CHECK();
            s.ctx->stats.kernel_launches += 2;
            fetch(3);
            const double sy = host[0], s_norm = std::sqrt(host[1]), y_norm = std::sqrt(host[2]);
            if (sy > 1e-10 * s_norm * y_norm) {
                hist.push_back(free_slot);
                rho_h.push_back(1.0 / sy);
                sy_h.push_back(sy);
                yy_h.push_back(host[2]);
                if ((int)hist.size() > cfg.history) {
                    hist.pop_front();
                    rho_h.pop_front();
                    sy_h.pop_front();
                    yy_h.pop_front();
                }
            }
            std::swap(x, xa);
            std::swap(g, ga);
            f_x = f_next;
            g_sq = gsq_next;
            if (!std::isfinite(f_x))
                raise(NADMM_ESOLVER, "lbfgs_solve: non-finite objective at iteration " + std::to_string(k));
            rec.objective = f_x;
            res.trace.push_back(rec);
        }
        res.final_grad_norm = std::sqrt(g_sq);
        res.converged = res.final_grad_norm < cfg.grad_tol;
        return res;
    }

    void launch_direction(const LbHist& h, double gamma) {
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute attr[1];
        lc.gridDim = dim3(kLbClusterCtas, 1, 1);
        lc.blockDim = dim3(kLbClThreads, 1, 1);
        lc.stream = st;
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kLbClusterCtas;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        lc.attrs = attr;
        lc.numAttrs = 1;
        NADMM_CUDA(cudaLaunchKernelEx(&lc, k_lb_direction, d, (const double*)g, (const double*)S,
                                      (const double*)Y, h, gamma, vq, vp, out));
        s.ctx->stats.kernel_launches++;
    }
};

}  // namespace

void validate_lbfgs_cfg(const LbfgsCfg& c) {  // LbfgsConfig::validate (src/lbfgs.cpp:9-15)
    if (c.history < 1) raise(NADMM_ECONFIG, "lbfgs history must be >= 1");
    if (!(0.0 < c.wolfe_c1 && c.wolfe_c1 < c.wolfe_c2 && c.wolfe_c2 < 1.0))
        raise(NADMM_ECONFIG, "wolfe constants must satisfy 0 < c1 < c2 < 1");
    if (c.max_iters < 0) raise(NADMM_ECONFIG, "lbfgs max_iters must be >= 0");
    if (c.ls_max_iters < 1) raise(NADMM_ECONFIG, "lbfgs ls_max_iters must be >= 1");
    if (c.history > kLbMaxHist) raise(NADMM_ECONFIG, "lbfgs history exceeds the device limit (256)");
}

// x0 in s.x (and z, y in s.z / s.y when augmented); the result x is left in s.x.
LbfgsResult device_lbfgs_solve(Shard& s, const LbfgsCfg& cfg, double lambda, bool aug, double rho) {
    validate_lbfgs_cfg(cfg);
    if (aug && rho <= 0.0) raise(NADMM_ECONFIG, "augmented objective requires rho > 0");
    set_lambda_only(s, lambda);
    s.cache_at = Shard::kNone;
    Lbfgs run(s, cfg, aug, rho);
    NADMM_CUDA(cudaMemcpyAsync(run.x, s.x, sizeof(double) * s.d, cudaMemcpyDeviceToDevice, run.st));
    LbfgsResult res;
    try {
        res = run.run();
    } catch (...) {
        s.cache_at = Shard::kNone;
        throw;
    }
    NADMM_CUDA(cudaMemcpyAsync(s.x, run.x, sizeof(double) * s.d, cudaMemcpyDeviceToDevice, run.st));
    stream_sync(run.st);
    s.cache_at = Shard::kNone;  // the cache holds the last trial point, not s.x
    return res;
}

}  // namespace nadmm
