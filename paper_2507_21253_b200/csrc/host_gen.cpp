// Seeded synthetic matrix generators for the BASELINE.json configurations.
//
// These stand in for the paper's SuiteSparse corpus, which is
// not available.  Every recipe is pinned here and in DESIGN.md §"Inputs":
//  - cfg1 ER: each row draws `per_row` distinct uniform columns.
//  - cfg2 hidden clusters: templates of `tcols` distinct columns, each spawns
//    `children` rows keeping every template column w.p. keep_p plus
//    Poisson(extra_mean) uniform extra columns; duplicates merged (first value
//    kept); rows then permuted by the reference's seeded Fisher-Yates
//    (reorder.hpp:20-30 semantics, see host_reorder.cpp).
//  - cfg3/cfg5 R-MAT: scale/edge-factor/(a,b,c) with no noise; symmetrised,
//    duplicates and self-loops removed; the value of {i,j} is a hash of the
//    unordered pair (a_ij == a_ji).
//  - cfg4 stencil: 27-point, boundary-truncated, 26 on the diagonal and -1
//    off it, symmetrically permuted by reorder_random(n, perm_seed).
// Values are U[0,1) doubles (53-bit mantissa draws) unless stated.
#include "common.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace bsp {

std::vector<int32_t> random_permutation(int64_t n, uint64_t seed);  // host_reorder.cpp
HostCsr permute_symmetric(const HostCsr& a, const std::vector<int32_t>& perm);
HostCsr permute_rows(const HostCsr& a, const std::vector<int32_t>& perm);

namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

inline double unit_double(uint64_t r) { return static_cast<double>(r >> 11) * 0x1.0p-53; }

inline uint64_t bounded(uint64_t x, uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(x) * n) >> 64);
}

// Build CSR from per-row (col, value) lists: sort by column, keep the first
// value of duplicate columns.
HostCsr from_rows(int64_t nrows, int64_t ncols,
                  std::vector<std::vector<std::pair<int32_t, double>>>& rows) {
    HostCsr m;
    m.nrows = nrows;
    m.ncols = ncols;
    m.row_ptr.assign(nrows + 1, 0);
    for (int64_t i = 0; i < nrows; ++i) {
        auto& r = rows[i];
        std::stable_sort(r.begin(), r.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        r.erase(std::unique(r.begin(), r.end(),
                            [](const auto& x, const auto& y) { return x.first == y.first; }),
                r.end());
        m.row_ptr[i + 1] = m.row_ptr[i] + static_cast<int64_t>(r.size());
    }
    m.col_idx.resize(m.row_ptr[nrows]);
    m.values.resize(m.row_ptr[nrows]);
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t p = m.row_ptr[i];
        for (const auto& [c, v] : rows[i]) {
            m.col_idx[p] = c;
            m.values[p] = v;
            ++p;
        }
    }
    return m;
}

}  // namespace

HostCsr gen_er(int64_t n, int32_t per_row, uint64_t seed) {
    require(n > 0 && per_row >= 0 && per_row <= n, "gen_er: bad sizes");
    std::mt19937_64 rng(seed);
    std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
    std::vector<int32_t> cols;
    for (int64_t i = 0; i < n; ++i) {
        cols.clear();
        while (static_cast<int32_t>(cols.size()) < per_row) {
            const int32_t c = static_cast<int32_t>(bounded(rng(), static_cast<uint64_t>(n)));
            if (std::find(cols.begin(), cols.end(), c) == cols.end()) cols.push_back(c);
        }
        for (int32_t c : cols) rows[i].emplace_back(c, unit_double(rng()));
    }
    return from_rows(n, n, rows);
}

HostCsr gen_hidden_clusters(int64_t ntemplates, int32_t children, int32_t tcols, double keep_p,
                            double extra_mean, uint64_t seed, uint64_t perm_seed) {
    const int64_t n = ntemplates * children;
    require(n > 0 && tcols > 0 && tcols <= n, "gen_hidden_clusters: bad sizes");
    std::mt19937_64 rng(seed);
    std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
    std::vector<int32_t> tmpl;
    const double poisson_l = std::exp(-extra_mean);
    for (int64_t t = 0; t < ntemplates; ++t) {
        tmpl.clear();
        while (static_cast<int32_t>(tmpl.size()) < tcols) {
            const int32_t c = static_cast<int32_t>(bounded(rng(), static_cast<uint64_t>(n)));
            if (std::find(tmpl.begin(), tmpl.end(), c) == tmpl.end()) tmpl.push_back(c);
        }
        for (int32_t ch = 0; ch < children; ++ch) {
            auto& r = rows[t * children + ch];
            for (int32_t c : tmpl)
                if (unit_double(rng()) < keep_p) r.emplace_back(c, unit_double(rng()));
            // Poisson(extra_mean) by Knuth's product-of-uniforms method.
            int32_t extra = 0;
            double prod = unit_double(rng());
            while (prod > poisson_l) {
                ++extra;
                prod *= unit_double(rng());
            }
            for (int32_t e = 0; e < extra; ++e) {
                const int32_t c = static_cast<int32_t>(bounded(rng(), static_cast<uint64_t>(n)));
                r.emplace_back(c, unit_double(rng()));
            }
        }
    }
    HostCsr m = from_rows(n, n, rows);
    return permute_rows(m, random_permutation(n, perm_seed));
}

HostCsr gen_rmat(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed) {
    require(scale >= 1 && scale <= 30 && edge_factor >= 1, "gen_rmat: bad sizes");
    const int64_t n = int64_t{1} << scale;
    const int64_t m = n * edge_factor;
    const double ab = a + b, abc = a + b + c;
    // Directed edge list (both orientations), self-loops dropped.
    std::vector<uint64_t> keys(static_cast<std::size_t>(2 * m));
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        uint64_t s = splitmix64(seed ^ (static_cast<uint64_t>(e) * 0xD1B54A32D192ED03ull));
        uint64_t u = 0, v = 0;
        for (int32_t lvl = 0; lvl < scale; ++lvl) {
            s = splitmix64(s);
            const double r = unit_double(s);
            u <<= 1;
            v <<= 1;
            if (r < a) {
            } else if (r < ab) {
                v |= 1;
            } else if (r < abc) {
                u |= 1;
            } else {
                u |= 1;
                v |= 1;
            }
        }
        if (u == v) {
            keys[2 * e] = keys[2 * e + 1] = ~uint64_t{0};
        } else {
            keys[2 * e] = (u << 32) | v;
            keys[2 * e + 1] = (v << 32) | u;
        }
    }
    // Bucket by row (counting sort), then sort/unique within rows.
    std::vector<int64_t> cnt(n + 1, 0);
    for (uint64_t k : keys)
        if (k != ~uint64_t{0}) ++cnt[(k >> 32) + 1];
    for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<int32_t> cols(static_cast<std::size_t>(cnt[n]));
    {
        std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
        for (uint64_t k : keys)
            if (k != ~uint64_t{0}) cols[cur[k >> 32]++] = static_cast<int32_t>(k & 0xffffffffu);
    }
    keys.clear();
    keys.shrink_to_fit();
    std::vector<int64_t> uniq(n, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
        auto* b0 = cols.data() + cnt[i];
        auto* e0 = cols.data() + cnt[i + 1];
        std::sort(b0, e0);
        uniq[i] = std::unique(b0, e0) - b0;
    }
    HostCsr out;
    out.nrows = out.ncols = n;
    out.row_ptr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) out.row_ptr[i + 1] = out.row_ptr[i] + uniq[i];
    out.col_idx.resize(out.row_ptr[n]);
    out.values.resize(out.row_ptr[n]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t src = cnt[i];
        const int64_t dst = out.row_ptr[i];
        for (int64_t q = 0; q < uniq[i]; ++q) {
            const int32_t j = cols[src + q];
            out.col_idx[dst + q] = j;
            const uint64_t lo = static_cast<uint64_t>(std::min<int64_t>(i, j));
            const uint64_t hi = static_cast<uint64_t>(std::max<int64_t>(i, j));
            out.values[dst + q] = unit_double(splitmix64(seed * 0x9E3779B97F4A7C15ull ^
                                                         ((lo << 32) | hi)));
        }
    }
    return out;
}

HostCsr gen_stencil27(int32_t g, int64_t perm_seed) {
    require(g >= 1 && g <= 1290, "gen_stencil27: bad grid");
    const int64_t n = int64_t{g} * g * g;
    HostCsr m;
    m.nrows = m.ncols = n;
    m.row_ptr.assign(n + 1, 0);
    auto span = [g](int32_t x) { return (x > 0) + 1 + (x < g - 1); };
    for (int64_t r = 0; r < n; ++r) {
        const int32_t x = static_cast<int32_t>(r % g), y = static_cast<int32_t>((r / g) % g),
                      z = static_cast<int32_t>(r / (int64_t{g} * g));
        m.row_ptr[r + 1] = m.row_ptr[r] + span(x) * span(y) * span(z);
    }
    m.col_idx.resize(m.row_ptr[n]);
    m.values.resize(m.row_ptr[n]);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        const int32_t x = static_cast<int32_t>(r % g), y = static_cast<int32_t>((r / g) % g),
                      z = static_cast<int32_t>(r / (int64_t{g} * g));
        int64_t p = m.row_ptr[r];
        for (int32_t dz = -1; dz <= 1; ++dz)
            for (int32_t dy = -1; dy <= 1; ++dy)
                for (int32_t dx = -1; dx <= 1; ++dx) {
                    const int32_t xx = x + dx, yy = y + dy, zz = z + dz;
                    if (xx < 0 || yy < 0 || zz < 0 || xx >= g || yy >= g || zz >= g) continue;
                    const int64_t col = xx + int64_t{g} * (yy + int64_t{g} * zz);
                    m.col_idx[p] = static_cast<int32_t>(col);
                    m.values[p] = (col == r) ? 26.0 : -1.0;
                    ++p;
                }
    }
    if (perm_seed < 0) return m;
    return permute_symmetric(m, random_permutation(n, static_cast<uint64_t>(perm_seed)));
}

}  // namespace bsp

extern "C" {

int bsp_gen_er(int64_t n, int32_t per_row, uint64_t seed, bsp_host_csr* out) {
    return bsp::guarded([&] { bsp::export_csr(bsp::gen_er(n, per_row, seed), out); });
}

int bsp_gen_hidden_clusters(int64_t ntemplates, int32_t children, int32_t tcols, double keep_p,
                            double extra_mean, uint64_t seed, uint64_t perm_seed,
                            bsp_host_csr* out) {
    return bsp::guarded([&] {
        bsp::export_csr(bsp::gen_hidden_clusters(ntemplates, children, tcols, keep_p, extra_mean,
                                                 seed, perm_seed),
                        out);
    });
}

int bsp_gen_rmat(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed,
                 bsp_host_csr* out) {
    return bsp::guarded(
        [&] { bsp::export_csr(bsp::gen_rmat(scale, edge_factor, a, b, c, seed), out); });
}

int bsp_gen_stencil27(int32_t g, int64_t perm_seed, bsp_host_csr* out) {
    return bsp::guarded([&] { bsp::export_csr(bsp::gen_stencil27(g, perm_seed), out); });
}

}  // extern "C"
