// Host-side data fixtures of the framework (no device code): the reference's deterministic Rng,
// generate_synthetic and partition (src/data_io.cpp:16-43, 300-370; mix_seed src/worker.cpp:64-69)
// plus the builder-defined sparse generator of SURVEY.md §8d. Same seed -> same bytes as the
// reference; tests/test_data_io.py pins this against the reference build.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

thread_local std::string g_dio_err;

class Rng {  // detail::Rng (inc/data_io.hpp:15-34)
  public:
    explicit Rng(uint64_t seed) : engine_(seed) {}
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double mag = std::sqrt(-2.0 * std::log(u1));
        const double pi = 3.141592653589793;
        spare_ = mag * std::sin(2.0 * pi * u2);
        have_spare_ = true;
        return mag * std::cos(2.0 * pi * u2);
    }
    uint64_t uniform_int(uint64_t bound) {
        const uint64_t mx = ~uint64_t(0);
        const uint64_t limit = mx - (mx % bound);
        uint64_t v = engine_();
        while (v >= limit) v = engine_();
        return v % bound;
    }

  private:
    std::mt19937_64 engine_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

template <typename F>
nadmm_status run(F&& f) {
    try {
        f();
        return NADMM_OK;
    } catch (const nadmm::Error& e) {
        g_dio_err = e.what();
        return e.code;
    }
}

}  // namespace

extern "C" {

const char* nadmm_data_last_error(void) { return g_dio_err.c_str(); }

uint64_t nadmm_mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

nadmm_status nadmm_generate_synthetic(int64_t n, int64_t p, int32_t C, double separation, double noise, uint64_t seed,
                                      double* X_train, int32_t* y_train, double* X_test, int32_t* y_test) {
    return run([&] {
        if (n < 2 || p < 1 || C < 2) nadmm::raise(NADMM_ECONFIG, "synthetic spec needs n >= 2, p >= 1, C >= 2");
        if (C > n) nadmm::raise(NADMM_ECONFIG, "synthetic spec: more classes than samples");
        const int64_t n_train = (n * 9) / 10;
        if (n_train < C || n - n_train < 1) nadmm::raise(NADMM_ECONFIG, "synthetic spec too small for a 90/10 split");
        Rng rng(seed);
        std::vector<double> centers((size_t)(p * C)), dir((size_t)p);
        for (int c = 0; c < C; ++c) {
            double sq = 0.0;
            for (int64_t j = 0; j < p; ++j) {
                dir[j] = rng.normal();
            }
            for (int64_t j = 0; j < p; ++j) sq += dir[j] * dir[j];
            const double norm = std::sqrt(sq);
            for (int64_t j = 0; j < p; ++j) centers[(size_t)(c * p + j)] = norm > 0.0 ? (separation / norm) * dir[j] : dir[j];
        }
        for (int64_t i = 0; i < n; ++i) {
            const int c = (int)(i % C);
            double* row = i < n_train ? X_train + i * p : X_test + (i - n_train) * p;
            if (i < n_train)
                y_train[i] = c + 1;
            else
                y_test[i - n_train] = c + 1;
            const double* ctr = centers.data() + (size_t)c * p;
            for (int64_t j = 0; j < p; ++j) row[j] = ctr[j] + noise * rng.normal();
        }
    });
}

nadmm_status nadmm_generate_sparse(int64_t n, int64_t p, int32_t C, int32_t nnz_per_row, uint64_t seed,
                                   int64_t* indptr, int32_t* indices, double* vals, int32_t* labels) {
    return run([&] {
        if (n < 1 || p < 1 || C < 2 || nnz_per_row < 1 || nnz_per_row > p)
            nadmm::raise(NADMM_ECONFIG, "sparse spec needs n, p >= 1, C >= 2, 1 <= nnz_per_row <= p");
        Rng rng(seed);
        const int64_t band = p / C > 0 ? p / C : 1;
        std::vector<int64_t> stamp((size_t)p, 0);
        indptr[0] = 0;
        for (int64_t i = 0; i < n; ++i) {
            const int c = (int)(i % C);
            labels[i] = c + 1;
            int32_t* cols = indices + i * nnz_per_row;
            int got = 0;
            while (got < nnz_per_row) {
                int64_t j;
                if (rng.uniform() < 0.5) {
                    const int64_t lo = (int64_t)c * band;
                    const int64_t width = lo + band <= p ? band : p - lo;
                    j = lo + (int64_t)rng.uniform_int((uint64_t)(width > 0 ? width : 1));
                } else {
                    j = (int64_t)rng.uniform_int((uint64_t)p);
                }
                if (stamp[j] != i + 1) {
                    stamp[j] = i + 1;
                    cols[got++] = (int32_t)j;
                }
            }
            std::sort(cols, cols + nnz_per_row);
            double* v = vals + i * nnz_per_row;
            double ss = 0.0;
            for (int q = 0; q < nnz_per_row; ++q) {
                v[q] = 1.0 + 0.1 * rng.normal();
                ss += v[q] * v[q];
            }
            const double inv = 1.0 / std::sqrt(ss);
            for (int q = 0; q < nnz_per_row; ++q) v[q] = v[q] * inv;
            indptr[i + 1] = indptr[i] + nnz_per_row;
        }
    });
}

nadmm_status nadmm_partition(int64_t n, int32_t N, int32_t strided, int32_t* owner) {
    return run([&] {
        if (N < 1) nadmm::raise(NADMM_ECONFIG, "partition needs n_workers >= 1");
        if (n < N)
            nadmm::raise(NADMM_ECONFIG, "cannot partition " + std::to_string(n) + " rows across " + std::to_string(N) + " workers");
        if (!strided) {
            const int64_t chunk = (n + N - 1) / N;  // ceil(n/N) (src/data_io.cpp:309)
            for (int i = 0; i < N; ++i) {
                const int64_t b = (int64_t)i * chunk, e = std::min<int64_t>(b + chunk, n);
                if (b >= e)
                    nadmm::raise(NADMM_ECONFIG, "contiguous partition leaves worker " + std::to_string(i) +
                                                    " empty; use strided or fewer workers");
                for (int64_t q = b; q < e; ++q) owner[q] = i;
            }
        } else {
            for (int64_t q = 0; q < n; ++q) owner[q] = (int32_t)(q % N);
        }
    });
}

}  // extern "C"
