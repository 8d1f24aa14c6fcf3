// Host preprocessing: permutations, symmetric/row permutation, transpose,
// RCM, degree order, bandwidth.  These stay on the host by design (the
// north star keeps RCM as "host preprocessing taken from the reference";
// sequential BFS).  Each function restates the reference's
// algorithm so that its output is identical element for element.
#include "common.hpp"

#include <algorithm>
#include <cmath>
#include <mutex>
#include <numeric>
#include <random>

namespace bsp {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void check_host_csr(const bsp_host_csr* a, const char* who) {
    require(a != nullptr, std::string(who) + ": null matrix");
    require(a->nrows >= 0 && a->ncols >= 0, std::string(who) + ": negative shape");
    require(a->row_ptr != nullptr, std::string(who) + ": null row_ptr");
    require(a->row_ptr[0] == 0, std::string(who) + ": row_ptr[0] must be 0");
    require(a->row_ptr[a->nrows] == a->nnz, std::string(who) + ": row_ptr[nrows] must equal nnz");
}

void export_assignment(const std::vector<std::vector<int32_t>>& clusters, int64_t* nclusters_out,
                       int64_t** cluster_ptr_out, int32_t** rows_out) {
    const int64_t nc = static_cast<int64_t>(clusters.size());
    int64_t total = 0;
    for (const auto& c : clusters) total += static_cast<int64_t>(c.size());
    int64_t* ptr = host_malloc<int64_t>(nc + 1);
    int32_t* rows = host_malloc<int32_t>(total);
    ptr[0] = 0;
    for (int64_t c = 0; c < nc; ++c) {
        std::copy(clusters[c].begin(), clusters[c].end(), rows + ptr[c]);
        ptr[c + 1] = ptr[c] + static_cast<int64_t>(clusters[c].size());
    }
    *nclusters_out = nc;
    *cluster_ptr_out = ptr;
    *rows_out = rows;
}

// Host view -> owning copy.
HostCsr import_csr(const bsp_host_csr* a) {
    HostCsr m;
    m.nrows = a->nrows;
    m.ncols = a->ncols;
    m.row_ptr.assign(a->row_ptr, a->row_ptr + a->nrows + 1);
    m.col_idx.assign(a->col_idx, a->col_idx + a->nnz);
    m.values.assign(a->values, a->values + a->nnz);
    return m;
}

// reference reorder.hpp:20-30: mt19937_64 Fisher-Yates from the back, index
// drawn by the multiply-shift reduction of types.hpp:36-39.
std::vector<int32_t> random_permutation(int64_t n, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<int32_t> perm(static_cast<std::size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    for (int64_t i = n - 1; i > 0; --i) {
        const uint64_t j = static_cast<uint64_t>(
            (static_cast<unsigned __int128>(rng()) * static_cast<uint64_t>(i + 1)) >> 64);
        std::swap(perm[i], perm[j]);
    }
    return perm;
}

std::vector<int32_t> inverse_of(const std::vector<int32_t>& perm) {
    std::vector<int32_t> inv(perm.size(), -1);
    for (std::size_t np = 0; np < perm.size(); ++np) {
        const int32_t old = perm[np];
        require(old >= 0 && static_cast<std::size_t>(old) < perm.size(),
                "permutation: index " + std::to_string(old) + " out of range");
        require(inv[old] == -1, "permutation: duplicate index " + std::to_string(old));
        inv[old] = static_cast<int32_t>(np);
    }
    return inv;
}

// reference csr.hpp:146-172: result[inv[i]][inv[j]] = a[i][j].
HostCsr permute_symmetric(const HostCsr& a, const std::vector<int32_t>& perm) {
    require(a.nrows == a.ncols, "permute_symmetric: matrix must be square");
    require(static_cast<int64_t>(perm.size()) == a.nrows,
            "permute_symmetric: permutation size mismatch");
    const std::vector<int32_t> inv = inverse_of(perm);
    HostCsr r;
    r.nrows = a.nrows;
    r.ncols = a.ncols;
    r.row_ptr.assign(a.nrows + 1, 0);
    for (int64_t ni = 0; ni < r.nrows; ++ni) r.row_ptr[ni + 1] = r.row_ptr[ni] + a.row_nnz(perm[ni]);
    r.col_idx.resize(a.col_idx.size());
    r.values.resize(a.values.size());
#pragma omp parallel
    {
        std::vector<std::pair<int32_t, double>> scratch;
#pragma omp for schedule(dynamic, 4096)
        for (int64_t ni = 0; ni < r.nrows; ++ni) {
            const int64_t oi = perm[ni];
            scratch.clear();
            for (int64_t q = a.row_ptr[oi]; q < a.row_ptr[oi + 1]; ++q)
                scratch.emplace_back(inv[a.col_idx[q]], a.values[q]);
            std::sort(scratch.begin(), scratch.end(),
                      [](const auto& x, const auto& y) { return x.first < y.first; });
            int64_t pos = r.row_ptr[ni];
            for (const auto& [c, v] : scratch) {
                r.col_idx[pos] = c;
                r.values[pos] = v;
                ++pos;
            }
        }
    }
    return r;
}

// reference csr.hpp:175-193: row inv[i] of the result is row i of a.
HostCsr permute_rows(const HostCsr& a, const std::vector<int32_t>& perm) {
    require(static_cast<int64_t>(perm.size()) == a.nrows, "permute_rows: permutation size mismatch");
    (void)inverse_of(perm);  // validates the bijection
    HostCsr r;
    r.nrows = a.nrows;
    r.ncols = a.ncols;
    r.row_ptr.assign(a.nrows + 1, 0);
    for (int64_t ni = 0; ni < r.nrows; ++ni) r.row_ptr[ni + 1] = r.row_ptr[ni] + a.row_nnz(perm[ni]);
    r.col_idx.resize(a.col_idx.size());
    r.values.resize(a.values.size());
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t ni = 0; ni < r.nrows; ++ni) {
        const int64_t oi = perm[ni];
        std::copy(a.col_idx.begin() + a.row_ptr[oi], a.col_idx.begin() + a.row_ptr[oi + 1],
                  r.col_idx.begin() + r.row_ptr[ni]);
        std::copy(a.values.begin() + a.row_ptr[oi], a.values.begin() + a.row_ptr[oi + 1],
                  r.values.begin() + r.row_ptr[ni]);
    }
    return r;
}

// reference csr.hpp:115-135: stable counting-sort transpose (rows sorted).
HostCsr transpose(const HostCsr& a) {
    HostCsr t;
    t.nrows = a.ncols;
    t.ncols = a.nrows;
    t.row_ptr.assign(a.ncols + 1, 0);
    for (int32_t c : a.col_idx) ++t.row_ptr[c + 1];
    for (int64_t i = 0; i < t.nrows; ++i) t.row_ptr[i + 1] += t.row_ptr[i];
    t.col_idx.resize(a.col_idx.size());
    t.values.resize(a.values.size());
    std::vector<int64_t> cur(t.row_ptr.begin(), t.row_ptr.end() - 1);
    for (int64_t i = 0; i < a.nrows; ++i)
        for (int64_t p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p) {
            const int64_t pos = cur[a.col_idx[p]]++;
            t.col_idx[pos] = static_cast<int32_t>(i);
            t.values[pos] = a.values[p];
        }
    return t;
}

namespace {

// Undirected pattern of A | A^T without self loops, each neighbour list
// ordered by (degree, index) — the Cuthill-McKee visiting rule of
// reference reorder.hpp:63-85.
struct Graph {
    std::vector<int64_t> ptr;
    std::vector<int32_t> adj;
    std::vector<int32_t> deg;
};

Graph build_graph(const HostCsr& a) {
    const HostCsr at = transpose(a);
    const int64_t n = a.nrows;
    Graph g;
    g.ptr.assign(n + 1, 0);
    std::vector<int32_t> tmp;
    std::vector<std::vector<int32_t>> lists(n);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
        auto& nb = lists[i];
        const int32_t* r0 = a.col_idx.data() + a.row_ptr[i];
        const int32_t* r1 = a.col_idx.data() + a.row_ptr[i + 1];
        const int32_t* c0 = at.col_idx.data() + at.row_ptr[i];
        const int32_t* c1 = at.col_idx.data() + at.row_ptr[i + 1];
        nb.reserve((r1 - r0) + (c1 - c0));
        std::merge(r0, r1, c0, c1, std::back_inserter(nb));
        nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        nb.erase(std::remove(nb.begin(), nb.end(), static_cast<int32_t>(i)), nb.end());
    }
    g.deg.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        g.deg[i] = static_cast<int32_t>(lists[i].size());
        g.ptr[i + 1] = g.ptr[i] + g.deg[i];
    }
    g.adj.resize(g.ptr[n]);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
        auto& nb = lists[i];
        std::sort(nb.begin(), nb.end(), [&](int32_t x, int32_t y) {
            return g.deg[x] != g.deg[y] ? g.deg[x] < g.deg[y] : x < y;
        });
        std::copy(nb.begin(), nb.end(), g.adj.begin() + g.ptr[i]);
        std::vector<int32_t>().swap(nb);
    }
    return g;
}

struct Levels {
    std::vector<int32_t> order;
    std::size_t last_begin = 0;
    std::size_t height = 0;
};

// BFS level structure from root using a scratch mark array that is cleared
// afterwards (reference reorder.hpp:96-116).
void bfs_levels(const Graph& g, int32_t root, std::vector<char>& mark, Levels& ls) {
    ls.order.clear();
    ls.last_begin = 0;
    ls.height = 0;
    ls.order.push_back(root);
    mark[root] = 1;
    std::size_t begin = 0;
    while (begin < ls.order.size()) {
        const std::size_t end = ls.order.size();
        for (std::size_t q = begin; q < end; ++q) {
            const int32_t v = ls.order[q];
            for (int64_t e = g.ptr[v]; e < g.ptr[v + 1]; ++e) {
                const int32_t w = g.adj[e];
                if (!mark[w]) {
                    mark[w] = 1;
                    ls.order.push_back(w);
                }
            }
        }
        ++ls.height;
        if (ls.order.size() == end) break;
        ls.last_begin = end;
        begin = end;
    }
    for (int32_t v : ls.order) mark[v] = 0;
}

int32_t min_degree(const Graph& g, const std::vector<int32_t>& vs, std::size_t b, std::size_t e) {
    int32_t best = vs[b];
    for (std::size_t k = b + 1; k < e; ++k) {
        const int32_t v = vs[k];
        if (g.deg[v] < g.deg[best] || (g.deg[v] == g.deg[best] && v < best)) best = v;
    }
    return best;
}

}  // namespace

// reference reorder.hpp:137-181.
std::vector<int32_t> reorder_rcm(const HostCsr& a) {
    require(a.nrows == a.ncols, "reorder_rcm: matrix must be square");
    const Graph g = build_graph(a);
    const int64_t n = a.nrows;
    std::vector<char> visited(n, 0), scratch(n, 0);
    std::vector<int32_t> perm;
    perm.reserve(n);
    Levels comp, ls, trial;
    for (int64_t s = 0; s < n; ++s) {
        if (visited[s]) continue;
        bfs_levels(g, static_cast<int32_t>(s), scratch, comp);
        int32_t root = min_degree(g, comp.order, 0, comp.order.size());
        bfs_levels(g, root, scratch, ls);
        while (ls.order.size() > 1) {
            const int32_t cand = min_degree(g, ls.order, ls.last_begin, ls.order.size());
            bfs_levels(g, cand, scratch, trial);
            if (trial.height > ls.height) {
                root = cand;
                std::swap(ls, trial);
            } else {
                break;
            }
        }
        const std::size_t cb = perm.size();
        perm.push_back(root);
        visited[root] = 1;
        for (std::size_t q = cb; q < perm.size(); ++q) {
            const int32_t v = perm[q];
            for (int64_t e = g.ptr[v]; e < g.ptr[v + 1]; ++e) {
                const int32_t w = g.adj[e];
                if (!visited[w]) {
                    visited[w] = 1;
                    perm.push_back(w);
                }
            }
        }
        std::reverse(perm.begin() + cb, perm.end());
    }
    return perm;
}

}  // namespace bsp

using namespace bsp;

extern "C" {

const char* bsp_last_error(void) { return g_last_error.c_str(); }

void bsp_host_csr_free(bsp_host_csr* m) {
    if (!m) return;
    std::free(m->row_ptr);
    std::free(m->col_idx);
    std::free(m->values);
    m->row_ptr = nullptr;
    m->col_idx = nullptr;
    m->values = nullptr;
}

void bsp_host_free_plain(void* p) { std::free(p); }

int bsp_reorder_random(int64_t n, uint64_t seed, int32_t* perm_out) {
    return guarded([&] {
        require(n >= 0, "reorder_random: negative size");
        const auto p = random_permutation(n, seed);
        std::copy(p.begin(), p.end(), perm_out);
    });
}

int bsp_reorder_rcm(const bsp_host_csr* A, int32_t* perm_out) {
    return guarded([&] {
        check_host_csr(A, "reorder_rcm");
        const auto p = reorder_rcm(import_csr(A));
        std::copy(p.begin(), p.end(), perm_out);
    });
}

// reference reorder.hpp:33-40: descending nnz, stable on ties.
int bsp_reorder_degree(const bsp_host_csr* A, int32_t* perm_out) {
    return guarded([&] {
        check_host_csr(A, "reorder_degree");
        require(A->nrows == A->ncols, "reorder_degree: matrix must be square");
        std::vector<int32_t> p(A->nrows);
        std::iota(p.begin(), p.end(), 0);
        std::stable_sort(p.begin(), p.end(), [&](int32_t x, int32_t y) {
            return A->row_ptr[x + 1] - A->row_ptr[x] > A->row_ptr[y + 1] - A->row_ptr[y];
        });
        std::copy(p.begin(), p.end(), perm_out);
    });
}

int bsp_bandwidth(const bsp_host_csr* A, int64_t* out) {
    return guarded([&] {
        check_host_csr(A, "bandwidth");
        require(A->nrows == A->ncols, "bandwidth: matrix must be square");
        int64_t bw = 0;
        for (int64_t i = 0; i < A->nrows; ++i)
            for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p)
                bw = std::max<int64_t>(bw, std::llabs(i - A->col_idx[p]));
        *out = bw;
    });
}

int bsp_permute_symmetric(const bsp_host_csr* A, const int32_t* perm, bsp_host_csr* out) {
    return guarded([&] {
        check_host_csr(A, "permute_symmetric");
        std::vector<int32_t> p(perm, perm + A->nrows);
        export_csr(permute_symmetric(import_csr(A), p), out);
    });
}

int bsp_permute_rows(const bsp_host_csr* A, const int32_t* perm, bsp_host_csr* out) {
    return guarded([&] {
        check_host_csr(A, "permute_rows");
        std::vector<int32_t> p(perm, perm + A->nrows);
        export_csr(permute_rows(import_csr(A), p), out);
    });
}

int bsp_transpose_host(const bsp_host_csr* A, bsp_host_csr* out) {
    return guarded([&] {
        check_host_csr(A, "transpose");
        export_csr(transpose(import_csr(A)), out);
    });
}

}  // extern "C"
