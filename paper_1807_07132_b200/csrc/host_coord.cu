// Host-side consensus coordinator (the reference's coordinator over host buffers: inc/admm.hpp:58-140,
// SPEC.md:196-304) for callers that drive the workers through nadmm_workers_solve / nadmm_worker_solve
// themselves -- the worker-transport deployment the bench's e2e leg measures. Host code: two fused
// OpenMP sweeps over d per round instead of ~20 separate vector passes:
//   sum    : S_j = sum_i (rho_i x_ij - y_ij), in ascending local worker order          (z_update)
//   update : z = S / (lambda + sum rho); y_hat_i = y_i + rho_i (z_prev - x_i); y_i += rho_i (z - x_i);
//            on penalty rounds the spectral secant dots and the snapshots, in
//            the same sweep; per-thread partial dots combined in thread order (deterministic).
// With several processes the caller reduces S (d + 1 doubles) between the two calls.
// Built with -O3 -fopenmp (build.sh); the worker-major update sweeps are unit-stride per stream.
#include <omp.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

struct HostCoord {
    int64_t d = 0;
    int n = 0;
    double lambda = 0.0;
    int spectral = 0, period = 2;
    double eps_cor = 0.2, rho_min = 1e-6, rho_max = 1e6;
    std::vector<double> z, pz, yh, xs, ys, yhs, zs, rho;
    int k = 0, snap_it = 0;
    int threads = 1;
};

bool side(double ab, double aa, double bb, double eps_cor, double* est) {
    if (!(aa > 0.0) || !(bb > 0.0) || !(ab > 0.0)) return false;
    const double cor = ab / (std::sqrt(aa) * std::sqrt(bb));
    if (!(cor > eps_cor)) return false;
    const double sd = bb / ab, mg = ab / aa;
    *est = (2.0 * mg > sd) ? mg : sd - mg / 2.0;
    return true;
}

thread_local std::string g_hc_err;

template <typename F>
nadmm_status hc_guard(F&& f) {
    try {
        f();
        return NADMM_OK;
    } catch (const nadmm::Error& e) {
        g_hc_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_hc_err = e.what();
        return NADMM_ECONFIG;
    }
}

}  // namespace

struct nadmm_hcoord_s : HostCoord {};

extern "C" {

nadmm_status nadmm_hcoord_create(int64_t d, int32_t n_local, double lambda, int32_t spectral, double rho0,
                                 int32_t update_period, double eps_cor, double rho_min, double rho_max,
                                 int32_t threads, nadmm_hcoord* out) {
    return hc_guard([&] {
        if (!out || d < 1 || n_local < 1) nadmm::raise(NADMM_ECONFIG, "host coordinator: bad arguments");
        if (!(rho0 > 0.0)) nadmm::raise(NADMM_ECONFIG, "rho0 must be > 0");
        if (spectral && (update_period < 1 || !(eps_cor > 0.0 && eps_cor < 1.0)))
            nadmm::raise(NADMM_ECONFIG, "bad spectral penalty policy");
        auto* c = new nadmm_hcoord_s();
        c->d = d;
        c->n = n_local;
        c->lambda = lambda;
        c->spectral = spectral;
        c->period = update_period;
        c->eps_cor = eps_cor;
        c->rho_min = rho_min;
        c->rho_max = rho_max;
        c->threads = threads > 0 ? threads : 1;
        c->z.assign(d, 0.0);
        c->pz.assign(d, 0.0);
        c->yh.assign((size_t)n_local * d, 0.0);
        c->rho.assign(n_local, rho0);
        if (spectral) {
            c->xs.assign((size_t)n_local * d, 0.0);
            c->ys.assign((size_t)n_local * d, 0.0);
            c->yhs.assign((size_t)n_local * d, 0.0);
            c->zs.assign(d, 0.0);
        }
        *out = c;
    });
}

nadmm_status nadmm_hcoord_free(nadmm_hcoord c) {
    delete c;
    return NADMM_OK;
}

nadmm_status nadmm_hcoord_sum(nadmm_hcoord c, const double* const* x, const double* const* y, double* S) {
    return hc_guard([&] {
        if (!c || !x || !y || !S) nadmm::raise(NADMM_ECONFIG, "host coordinator: null argument");
        const int64_t d = c->d;
        const int n = c->n;
        const double* rho = c->rho.data();
#pragma omp parallel for schedule(static) num_threads(c->threads)
        for (int64_t j = 0; j < d; ++j) {
            double s = rho[0] * x[0][j] - y[0][j];
            for (int i = 1; i < n; ++i) s += rho[i] * x[i][j] - y[i][j];
            S[j] = s;
        }
        double rs = rho[0];
        for (int i = 1; i < n; ++i) rs += rho[i];
        S[d] = rs;
    });
}

nadmm_status nadmm_hcoord_update(nadmm_hcoord c, const double* const* x, double* const* y, const double* S,
                                 double* z_out, double* rho_out) {
    return hc_guard([&] {
        if (!c || !x || !y || !S) nadmm::raise(NADMM_ECONFIG, "host coordinator: null argument");
        const int64_t d = c->d;
        const int n = c->n;
        const double den = c->lambda + S[d];
        if (den == 0.0) nadmm::raise(NADMM_ECONFIG, "z_update: lambda + sum(rho) == 0");
        c->k += 1;
        const bool sps = c->spectral && c->k - c->snap_it >= c->period;
        const int nt = c->threads;
        // per thread x worker: <dx,dyh>, |dx|^2, |dyh|^2, <dz,-dy>, |dz|^2, |dy|^2
        std::vector<double> part((size_t)nt * n * 6, 0.0);
        double* z = c->z.data();
        double* pz = c->pz.data();
        double* zs = sps ? c->zs.data() : nullptr;
        const double* rho = c->rho.data();
#pragma omp parallel num_threads(nt)
        {
            const int t = omp_get_thread_num();
#pragma omp for schedule(static)
            for (int64_t j = 0; j < d; ++j) {
                pz[j] = z[j];
                z[j] = S[j] / den;
            }
            // worker-major sweeps (unit-stride streams per worker, vectorisable); the static schedule
            // gives every thread the same j range in every sweep
            for (int i = 0; i < n; ++i) {
                const double ri = rho[i];
                const double* xi = x[i];
                double* yi = y[i];
                double* yhi = c->yh.data() + (size_t)i * d;
                double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
                if (!sps) {
#pragma omp for schedule(static)
                    for (int64_t j = 0; j < d; ++j) {
                        const double xv = xi[j], yv = yi[j];
                        yhi[j] = yv + ri * (pz[j] - xv);
                        yi[j] = yv + ri * (z[j] - xv);
                    }
                } else {
                    double* xsi = c->xs.data() + (size_t)i * d;
                    double* ysi = c->ys.data() + (size_t)i * d;
                    double* yhsi = c->yhs.data() + (size_t)i * d;
#pragma omp for schedule(static)
                    for (int64_t j = 0; j < d; ++j) {
                        const double xv = xi[j], yv = yi[j];
                        const double yhn = yv + ri * (pz[j] - xv);
                        const double yn = yv + ri * (z[j] - xv);
                        yhi[j] = yhn;
                        yi[j] = yn;
                        const double dx = xv - xsi[j], dyh = yhn - yhsi[j], dy = -(yn - ysi[j]), dz = z[j] - zs[j];
                        a0 += dx * dyh;
                        a1 += dx * dx;
                        a2 += dyh * dyh;
                        a3 += dz * dy;
                        a4 += dz * dz;
                        a5 += dy * dy;
                        xsi[j] = xv;
                        ysi[j] = yn;
                        yhsi[j] = yhn;
                    }
                    double* p6 = part.data() + ((size_t)t * n + i) * 6;
                    p6[0] = a0;
                    p6[1] = a1;
                    p6[2] = a2;
                    p6[3] = a3;
                    p6[4] = a4;
                    p6[5] = a5;
                }
            }
            if (sps) {
#pragma omp for schedule(static)
                for (int64_t j = 0; j < d; ++j) zs[j] = z[j];
            }
        }
        if (sps) {
            for (int i = 0; i < n; ++i) {
                double w[6] = {0, 0, 0, 0, 0, 0};
                for (int t = 0; t < nt; ++t)  // thread order: deterministic for a fixed thread count
                    for (int q = 0; q < 6; ++q) w[q] += part[((size_t)t * n + i) * 6 + q];
                double ah = 0.0, bh = 0.0;
                const bool xo = side(w[0], w[1], w[2], c->eps_cor, &ah);
                const bool zo = side(w[3], w[4], w[5], c->eps_cor, &bh);
                double r = c->rho[i];
                if (xo && zo)
                    r = std::sqrt(ah * bh);
                else if (xo)
                    r = std::sqrt(ah);
                else if (zo)
                    r = std::sqrt(bh);
                c->rho[i] = std::fmin(std::fmax(r, c->rho_min), c->rho_max);
            }
            c->snap_it = c->k;
        }
        if (z_out) std::memcpy(z_out, z, sizeof(double) * (size_t)d);
        if (rho_out) std::memcpy(rho_out, c->rho.data(), sizeof(double) * (size_t)n);
    });
}

const char* nadmm_hcoord_last_error(void) { return g_hc_err.c_str(); }

}  // extern "C"
