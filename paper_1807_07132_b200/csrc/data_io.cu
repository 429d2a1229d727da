// Host-side data fixtures and readers of the framework (no device code): the reference's
// deterministic Rng, generate_synthetic and partition (src/data_io.cpp:16-43, 300-370; mix_seed
// src/worker.cpp:64-69), the builder-defined sparse generator of SURVEY.md §8d, and the real-data
// readers LIBSVM -> CSR and IDX -> dense (src/data_io.cpp:51-137, 220-271) feeding device shards. Same seed -> same bytes as the
// reference; tests/test_data_io.py pins this against the reference build.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
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

// ---------------------------------------------------------------------------------------------
// Real-data readers
// ---------------------------------------------------------------------------------------------
struct nadmm_libsvm_s {
    int64_t n = 0, p = 0;
    std::vector<int64_t> indptr;
    std::vector<int32_t> indices;
    std::vector<double> vals;
    std::vector<int32_t> labels;
    std::vector<double> label_values;
};

namespace {

// Dataset::validate (src/dataset.cpp:28-57) as it applies to a freshly read file: the reference's
// readers return a constructed Dataset, so their callers see these errors from the load itself.
void validate_loaded(int64_t n, int64_t p, int64_t C, const double* vals, int64_t count, bool sparse) {
    if (n < 1 || p < 1)
        nadmm::raise(NADMM_ECONFIG, "dataset must have n >= 1 and p >= 1, got n=" + std::to_string(n) +
                                        " p=" + std::to_string(p));
    if (C < 2) nadmm::raise(NADMM_ECONFIG, "dataset needs at least 2 classes, got " + std::to_string(C));
    for (int64_t k = 0; k < count; ++k)
        if (!std::isfinite(vals[k]))
            nadmm::raise(NADMM_EDATA, sparse ? "non-finite feature value in sparse dataset"
                                             : "non-finite feature value in dense dataset");
}

bool is_ws(char ch) { return std::isspace(static_cast<unsigned char>(ch)) != 0; }

// The label field is read with `istream >> double` (src/data_io.cpp:97): the longest prefix of the
// form [+-]digits[.digits][(e|E)[+-]digits] is collected and must convert completely and in range.
// No inf/nan/hex spellings. Returns false when the stream extraction would fail.
bool read_label(const char*& c, double& out) {
    while (*c && is_ws(*c)) ++c;
    const char* b = c;
    const char* q = c;
    auto digits = [&] {
        const char* s0 = q;
        while (*q >= '0' && *q <= '9') ++q;
        return q != s0;
    };
    if (*q == '+' || *q == '-') ++q;
    bool any = digits();
    if (*q == '.') {
        ++q;
        any = digits() || any;
    }
    if (any && (*q == 'e' || *q == 'E')) {
        ++q;
        if (*q == '+' || *q == '-') ++q;
        digits();
    }
    if (q == b) return false;
    const std::string tok(b, q);
    char* end = nullptr;
    errno = 0;
    out = std::strtod(tok.c_str(), &end);
    c = q;
    if (end != tok.c_str() + tok.size()) return false;
    if (errno == ERANGE && std::isinf(out)) return false;
    return true;
}

// "label idx:val idx:val ..." lines, 1-based indices, '#' comments and blank lines skipped.
// Rows come out canonical like Eigen's setFromTriplets: columns ascending, duplicates summed.
// Labels are remapped to 1..C in ascending value order (src/data_io.cpp:51-66, 85-137). Feature
// fields follow std::stoll / std::stod (partial parses accepted, out-of-range rejected).
void parse_libsvm(const std::string& path, nadmm_libsvm_s& out) {
    std::ifstream in(path);
    if (!in) nadmm::raise(NADMM_ECONFIG, "cannot open " + path);
    std::vector<double> raw;
    std::vector<std::pair<int64_t, double>> row;
    out.indptr.assign(1, 0);
    int64_t max_col = 0;
    std::string line;
    int64_t line_no = 0;
    auto fail = [&](const std::string& what) {
        nadmm::raise(NADMM_EDATA, path + ":" + std::to_string(line_no) + ": " + what);
    };
    while (std::getline(in, line)) {
        ++line_no;
        if (line.empty() || line[0] == '#') continue;
        const char* c = line.c_str();
        double label = 0.0;
        if (!read_label(c, label) || label != std::floor(label)) fail("non-integer label");
        raw.push_back(label);
        row.clear();
        for (;;) {
            while (*c && is_ws(*c)) ++c;
            if (!*c) break;
            const char* tok = c;
            while (*c && !is_ws(*c)) ++c;
            const std::string t(tok, c);
            const size_t colon = t.find(':');
            if (colon == std::string::npos) fail("malformed feature token '" + t + "'");
            const std::string is = t.substr(0, colon), vs = t.substr(colon + 1);
            char* e1 = nullptr;
            char* e2 = nullptr;
            errno = 0;
            const long long idx = std::strtoll(is.c_str(), &e1, 10);
            const bool idx_bad = e1 == is.c_str() || errno == ERANGE;
            errno = 0;
            const double val = std::strtod(vs.c_str(), &e2);
            if (idx_bad || e2 == vs.c_str() || errno == ERANGE) fail("malformed feature token '" + t + "'");
            if (idx < 1) fail("feature indices are 1-based");
            if (idx > INT32_MAX) fail("feature index exceeds the int32 column range");
            max_col = std::max<int64_t>(max_col, idx);
            row.emplace_back((int64_t)idx - 1, val);
        }
        std::stable_sort(row.begin(), row.end(),
                         [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& b) {
                             return a.first < b.first;
                         });
        for (size_t k = 0; k < row.size(); ++k) {
            if (k > 0 && row[k].first == row[k - 1].first) {
                out.vals.back() += row[k].second;  // duplicates summed (setFromTriplets)
                continue;
            }
            out.indices.push_back((int32_t)row[k].first);
            out.vals.push_back(row[k].second);
        }
        out.indptr.push_back((int64_t)out.indices.size());
    }
    if (raw.empty()) nadmm::raise(NADMM_EDATA, path + ": no data rows");
    std::map<double, int32_t> mapping;
    for (double v : raw) mapping.emplace(v, 0);
    int32_t next = 1;
    for (auto& kv : mapping) {
        kv.second = next++;
        out.label_values.push_back(kv.first);
    }
    out.labels.reserve(raw.size());
    for (double v : raw) out.labels.push_back(mapping.at(v));
    out.n = (int64_t)raw.size();
    out.p = max_col;
    validate_loaded(out.n, out.p, (int64_t)out.label_values.size(), out.vals.data(), (int64_t)out.vals.size(), true);
}

uint32_t be32(std::istream& in) {
    unsigned char b[4];
    in.read(reinterpret_cast<char*>(b), 4);
    if (!in) nadmm::raise(NADMM_EDATA, "unexpected end of IDX header");
    return (uint32_t(b[0]) << 24) | (uint32_t(b[1]) << 16) | (uint32_t(b[2]) << 8) | uint32_t(b[3]);
}

// IDX image (magic 0x803) + label (0x801) pair headers: n and pixels per image.
void idx_headers(const std::string& images, const std::string& labels, std::ifstream& fi, std::ifstream& fl,
                 uint32_t& n, uint32_t& pix) {
    fi.open(images, std::ios::binary);
    if (!fi) nadmm::raise(NADMM_ECONFIG, "cannot open " + images);
    fl.open(labels, std::ios::binary);
    if (!fl) nadmm::raise(NADMM_ECONFIG, "cannot open " + labels);
    if (be32(fi) != 0x00000803u) nadmm::raise(NADMM_EDATA, images + ": bad IDX image magic");
    n = be32(fi);
    const uint32_t rows = be32(fi), cols = be32(fi);
    pix = rows * cols;
    if (be32(fl) != 0x00000801u) nadmm::raise(NADMM_EDATA, labels + ": bad IDX label magic");
    const uint32_t nl = be32(fl);
    if (nl != n)
        nadmm::raise(NADMM_EDATA, "IDX count mismatch: " + std::to_string(n) + " images vs " + std::to_string(nl) +
                                      " labels");
}

}  // namespace

extern "C" {

nadmm_status nadmm_libsvm_parse(const char* path, nadmm_libsvm* out, int64_t* n, int64_t* p, int64_t* nnz,
                                int32_t* C) {
    return run([&] {
        if (!path || !out) nadmm::raise(NADMM_ECONFIG, "path and output handle required");
        auto h = std::make_unique<nadmm_libsvm_s>();
        parse_libsvm(path, *h);
        if (n) *n = h->n;
        if (p) *p = h->p;
        if (nnz) *nnz = (int64_t)h->vals.size();
        if (C) *C = (int32_t)h->label_values.size();
        *out = h.release();
    });
}

nadmm_status nadmm_libsvm_fetch(nadmm_libsvm h, int64_t* indptr, int32_t* indices, double* vals, int32_t* labels,
                                double* label_values) {
    return run([&] {
        if (!h) nadmm::raise(NADMM_ECONFIG, "null LIBSVM handle");
        if (indptr) std::memcpy(indptr, h->indptr.data(), sizeof(int64_t) * h->indptr.size());
        if (indices) std::memcpy(indices, h->indices.data(), sizeof(int32_t) * h->indices.size());
        if (vals) std::memcpy(vals, h->vals.data(), sizeof(double) * h->vals.size());
        if (labels) std::memcpy(labels, h->labels.data(), sizeof(int32_t) * h->labels.size());
        if (label_values) std::memcpy(label_values, h->label_values.data(), sizeof(double) * h->label_values.size());
    });
}

void nadmm_libsvm_free(nadmm_libsvm h) { delete h; }

nadmm_status nadmm_idx_info(const char* images, const char* labels, int64_t* n, int64_t* p) {
    return run([&] {
        if (!images || !labels) nadmm::raise(NADMM_ECONFIG, "image and label paths required");
        std::ifstream fi, fl;
        uint32_t nn = 0, pix = 0;
        idx_headers(images, labels, fi, fl, nn, pix);
        if (n) *n = nn;
        if (p) *p = pix;
    });
}

nadmm_status nadmm_idx_load(const char* images, const char* labels, double* X, int32_t* y, int32_t* C,
                            double* label_values) {
    return run([&] {
        if (!images || !labels || !X || !y) nadmm::raise(NADMM_ECONFIG, "paths and output buffers required");
        std::ifstream fi, fl;
        uint32_t n = 0, pix = 0;
        idx_headers(images, labels, fi, fl, n, pix);
        const size_t total = (size_t)n * pix;
        std::vector<unsigned char> buf(total), lab(n);
        fi.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)total);
        if ((size_t)fi.gcount() != total)
            nadmm::raise(NADMM_EDATA, std::string(images) + ": truncated, expected " + std::to_string(total) +
                                          " pixel bytes, found " + std::to_string(fi.gcount()));
        fl.read(reinterpret_cast<char*>(lab.data()), (std::streamsize)n);
        if ((size_t)fl.gcount() != n)
            nadmm::raise(NADMM_EDATA, std::string(labels) + ": truncated, expected " + std::to_string(n) +
                                          " label bytes, found " + std::to_string(fl.gcount()));
        for (size_t i = 0; i < total; ++i) X[i] = (double)buf[i] / 255.0;  // pixels to [0, 1]
        int max_label = 0;
        for (uint32_t i = 0; i < n; ++i) {
            y[i] = (int32_t)lab[i] + 1;  // digits 0..9 -> classes 1..10
            max_label = std::max(max_label, (int)lab[i]);
        }
        validate_loaded((int64_t)n, (int64_t)pix, (int64_t)max_label + 1, X, 0, false);
        if (C) *C = max_label + 1;
        if (label_values)
            for (int v = 0; v <= max_label; ++v) label_values[v] = (double)v;
    });
}

}  // extern "C"
