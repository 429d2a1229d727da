// C++ host program over the header-only wrapper (include/nadmm_cuda.hpp): the reference-shaped API
// a C++ caller of the reference would use, on the B200 library. Prints one JSON line with the
// results (compared against the Python API by tests/test_cpp_api.py); with no GPU it reports the
// library's CudaError and exits 3.
#include <cstdio>
#include <vector>

#include "nadmm_cuda.hpp"

using namespace nadmm_gpu;

int main() {
    try {
        // fixtures from the reference generator (src/data_io.cpp:330-370), host-only
        const int64_t n_total = 1111, p = 30;
        const int32_t C = 4;
        const int64_t ntr = n_total * 9 / 10, nte = n_total - ntr;
        Vector Xtr((size_t)(ntr * p)), Xte((size_t)(nte * p));
        std::vector<int32_t> ytr((size_t)ntr), yte((size_t)nte);
        check(nadmm_generate_synthetic(n_total, p, C, 2.0, 1.0, 7, Xtr.data(), ytr.data(), Xte.data(), yte.data()));
        Context ctx(0);
        auto ds = Dataset::dense(ctx, Xtr, ntr, p, ytr, C);
        const int64_t d = ds->weight_dim();
        Vector w((size_t)d), v((size_t)d);
        for (int64_t j = 0; j < d; ++j) {
            w[(size_t)j] = 0.01 * (double)((j * 37) % 11 - 5);
            v[(size_t)j] = (double)((j * 13) % 7 - 3);
        }
        const double f = loss(*ds, w, 1e-3);
        const Vector hv = hessian_vec(*ds, w, v, 1e-3);
        NewtonConfig cfg;
        cfg.newton_max_iters = 3;
        const NewtonResult nr = newton_solve(*ds, 1e-3, Vector((size_t)d, 0.0), cfg);
        // two ADMM workers over contiguous halves
        const int64_t half = ntr / 2;
        auto d0 = Dataset::dense(ctx, Vector(Xtr.begin(), Xtr.begin() + half * p), half, p,
                                 std::vector<int32_t>(ytr.begin(), ytr.begin() + half), C);
        auto d1 = Dataset::dense(ctx, Vector(Xtr.begin() + half * p, Xtr.end()), ntr - half, p,
                                 std::vector<int32_t>(ytr.begin() + half, ytr.end()), C);
        nadmm_admm_cfg ac = admm_defaults();
        ac.lambda = 1e-3;
        ac.max_outer_iters = 8;
        const AdmmResult ar = run_admm({d0, d1}, ac);
        double hv_sum = 0.0, x_sum = 0.0, z_sum = 0.0;
        for (double t : hv) hv_sum += t;
        for (double t : nr.x) x_sum += t;
        for (double t : ar.z) z_sum += t;
        std::printf("{\"loss\": %.17g, \"hv_sum\": %.17g, \"newton_iters\": %zu, \"newton_x_sum\": %.17g, "
                    "\"admm_iters\": %d, \"admm_z_sum\": %.17g, \"accuracy\": %.17g}\n",
                    f, hv_sum, nr.trace.size(), x_sum, ar.iterations, z_sum, accuracy(*d0, ar.z));
        // the reference's error contract: ConfigError for an invalid config
        try {
            NewtonConfig bad;
            bad.cg_tol = 2.0;
            newton_solve(*ds, 1e-3, Vector((size_t)d, 0.0), bad);
            return 4;
        } catch (const ConfigError&) {
        }
        return 0;
    } catch (const CudaError& e) {
        std::printf("{\"error\": \"CudaError\", \"message\": \"%s\"}\n", e.what());
        return 3;
    } catch (const Error& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 2;
    }
}
