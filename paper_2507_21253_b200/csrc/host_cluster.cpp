// Host side of clustering: Jaccard, fixed/variable-length scans, and the
// greedy heap + union-find merge of hierarchical clustering.  Candidate
// generation (top-k of binarized A*A^T, or minhash/LSH) runs on the GPU
// (topk.cu / minhash.cu); the merge is sequential by design.
#include "common.hpp"

#include <parallel/algorithm>

#include <algorithm>
#include <queue>

namespace bsp {

// reference spgemm.hpp:110-129: sorted-merge intersection, inter/union,
// 0 when both rows are empty.
double jaccard(const bsp_host_csr* a, int64_t i, int64_t j) {
    const int32_t* ci = a->col_idx + a->row_ptr[i];
    const int32_t* cj = a->col_idx + a->row_ptr[j];
    const int64_t ni = a->row_ptr[i + 1] - a->row_ptr[i];
    const int64_t nj = a->row_ptr[j + 1] - a->row_ptr[j];
    int64_t inter = 0, p = 0, q = 0;
    while (p < ni && q < nj) {
        if (ci[p] == cj[q]) {
            ++inter;
            ++p;
            ++q;
        } else if (ci[p] < cj[q]) {
            ++p;
        } else {
            ++q;
        }
    }
    const int64_t uni = ni + nj - inter;
    return uni == 0 ? 0.0 : static_cast<double>(inter) / static_cast<double>(uni);
}

struct FlatClusters {
    std::vector<int64_t> ptr;  // nclusters + 1
    std::vector<int32_t> rows;
};

namespace {

// reference clustering.hpp:20-49: union by size, path compression, equal
// sizes keep the smaller root index.
struct DisjointSet {
    std::vector<int32_t> parent, size;
    explicit DisjointSet(int64_t n) : parent(n), size(n, 1) {
        for (int64_t i = 0; i < n; ++i) parent[i] = static_cast<int32_t>(i);
    }
    int32_t find(int32_t x) {
        int32_t r = x;
        while (parent[r] != r) r = parent[r];
        while (parent[x] != r) {
            const int32_t nx = parent[x];
            parent[x] = r;
            x = nx;
        }
        return r;
    }
    int32_t unite(int32_t a, int32_t b) {
        int32_t ra = find(a), rb = find(b);
        if (ra == rb) return ra;
        if (size[ra] < size[rb] || (size[ra] == size[rb] && rb < ra)) std::swap(ra, rb);
        parent[rb] = ra;
        size[ra] += size[rb];
        return ra;
    }
};

struct Entry {
    double score;
    int32_t i, j;  // i < j
};

// Max-heap order: higher score first, then smaller i, then smaller j
// (reference clustering.hpp:127-131).
struct Worse {
    bool operator()(const Entry& x, const Entry& y) const {
        if (x.score != y.score) return x.score < y.score;
        if (x.i != y.i) return x.i > y.i;
        return x.j > y.j;
    }
};

inline uint64_t pair_key(int32_t lo, int32_t hi) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(lo)) << 32) | static_cast<uint32_t>(hi);
}

// Set of (lo, hi) pair keys: open addressing, linear probing, rehash at half
// load.  Replaces a node-based hash set (one allocation per candidate).
class PairSet {
    static constexpr uint64_t kEmpty = ~0ull;  // lo = hi = -1 never occurs
    std::vector<uint64_t> slot_;
    uint64_t mask_ = 0;
    std::size_t count_ = 0;
    static uint64_t mix(uint64_t k) {
        k ^= k >> 33;
        k *= 0xff51afd7ed558ccdull;
        k ^= k >> 33;
        return k;
    }
    void place(uint64_t key) {
        uint64_t p = mix(key) & mask_;
        while (slot_[p] != kEmpty) p = (p + 1) & mask_;
        slot_[p] = key;
    }

public:
    explicit PairSet(std::size_t expect) {
        std::size_t cap = 64;
        while (cap < 2 * expect) cap <<= 1;
        slot_.assign(cap, kEmpty);
        mask_ = cap - 1;
    }
    // true when the key was not present (std::unordered_set::insert().second)
    bool insert(uint64_t key) {
        uint64_t p = mix(key) & mask_;
        for (;; p = (p + 1) & mask_) {
            if (slot_[p] == key) return false;
            if (slot_[p] == kEmpty) break;
        }
        if (2 * (count_ + 1) > slot_.size()) {
            std::vector<uint64_t> old;
            old.swap(slot_);
            slot_.assign(old.size() * 2, kEmpty);
            mask_ = slot_.size() - 1;
            for (uint64_t k : old)
                if (k != kEmpty) place(k);
            place(key);
        } else {
            slot_[p] = key;
        }
        ++count_;
        return true;
    }
};

}  // namespace

// reference clustering.hpp:122-183.  Same pops in the same order as one max-heap
// over (score, i, j): the candidate list is sorted best-first once (a total
// order, so a sorted array pops exactly like the heap), and only re-scored root
// pairs go through a (small) heap; each step takes the better of the two fronts.
FlatClusters merge_candidates(const bsp_host_csr* a, const bsp_candidate* pairs, int64_t npairs,
                              double jacc_th, int32_t max_cluster,
                              std::vector<bsp_candidate>* trace) {
    FlatClusters out;
    const int64_t n = a->nrows;
    out.ptr.push_back(0);
    if (n == 0) return out;
    std::vector<Entry> init(static_cast<std::size_t>(npairs));
    PairSet known(static_cast<std::size_t>(npairs) + static_cast<std::size_t>(n) / 4);
    for (int64_t k = 0; k < npairs; ++k) {
        const int32_t lo = std::min(pairs[k].i, pairs[k].j);
        const int32_t hi = std::max(pairs[k].i, pairs[k].j);
        init[k] = {pairs[k].score, lo, hi};
        known.insert(pair_key(lo, hi));
    }
    const Worse worse;
    const auto better = [&](const Entry& x, const Entry& y) { return worse(y, x); };
    if (npairs > (1 << 16))
        __gnu_parallel::sort(init.begin(), init.end(), better);
    else
        std::sort(init.begin(), init.end(), better);
    std::priority_queue<Entry, std::vector<Entry>, Worse> heap;
    DisjointSet ds(n);
    std::size_t next = 0;
    while (next < init.size() || !heap.empty()) {
        Entry top;
        if (heap.empty() || (next < init.size() && !worse(init[next], heap.top()))) {
            top = init[next++];
        } else {
            top = heap.top();
            heap.pop();
        }
        const int32_t ri = ds.find(top.i), rj = ds.find(top.j);
        if (ri == rj) continue;
        if (ri == top.i && rj == top.j) {
            if (ds.size[ri] + ds.size[rj] <= max_cluster) {
                ds.unite(ri, rj);
                if (trace) trace->push_back({top.i, top.j, top.score});
            }
            continue;
        }
        const int32_t lo = std::min(ri, rj), hi = std::max(ri, rj);
        if (known.insert(pair_key(lo, hi))) {
            const double s = jaccard(a, lo, hi);
            if (s >= jacc_th) heap.push({s, lo, hi});
        }
    }
    // clusters numbered by their smallest row, rows ascending within a cluster
    std::vector<int32_t> cluster_of(n, -1), root(n);
    std::vector<int64_t> count;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t r = ds.find(static_cast<int32_t>(i));
        root[i] = r;
        if (cluster_of[r] == -1) {
            cluster_of[r] = static_cast<int32_t>(count.size());
            count.push_back(0);
        }
        ++count[cluster_of[r]];
    }
    out.ptr.resize(count.size() + 1);
    for (std::size_t c = 0; c < count.size(); ++c) out.ptr[c + 1] = out.ptr[c] + count[c];
    out.rows.resize(n);
    std::vector<int64_t> fill(out.ptr.begin(), out.ptr.end() - 1);
    for (int64_t i = 0; i < n; ++i) out.rows[fill[cluster_of[root[i]]]++] = static_cast<int32_t>(i);
    return out;
}

void export_flat(const FlatClusters& f, int64_t* nclusters_out, int64_t** cluster_ptr_out,
                 int32_t** rows_out) {
    const int64_t nc = static_cast<int64_t>(f.ptr.size()) - 1;
    int64_t* ptr = host_malloc<int64_t>(nc + 1);
    int32_t* rows = host_malloc<int32_t>(f.rows.size());
    std::copy(f.ptr.begin(), f.ptr.end(), ptr);
    std::copy(f.rows.begin(), f.rows.end(), rows);
    *nclusters_out = nc;
    *cluster_ptr_out = ptr;
    *rows_out = rows;
}

}  // namespace bsp

using namespace bsp;

extern "C" {

int bsp_jaccard(const bsp_host_csr* A, int64_t i, int64_t j, double* out) {
    return guarded([&] {
        check_host_csr(A, "jaccard_similarity");
        require(i >= 0 && i < A->nrows && j >= 0 && j < A->nrows,
                "jaccard_similarity: row index out of range");
        *out = jaccard(A, i, j);
    });
}

// reference clustering.hpp:59-69
int bsp_fixed_length_clusters(int64_t nrows, int32_t k, int64_t* nclusters_out,
                              int64_t** cluster_ptr_out, int32_t** rows_out) {
    return guarded([&] {
        require(k >= 1, "fixed_length_clusters: k must be >= 1");
        std::vector<std::vector<int32_t>> cl;
        for (int64_t s = 0; s < nrows; s += k) {
            const int64_t e = std::min<int64_t>(s + k, nrows);
            std::vector<int32_t> m;
            for (int64_t i = s; i < e; ++i) m.push_back(static_cast<int32_t>(i));
            cl.push_back(std::move(m));
        }
        export_assignment(cl, nclusters_out, cluster_ptr_out, rows_out);
    });
}

// reference clustering.hpp:76-93
int bsp_variable_length_clusters(const bsp_host_csr* A, double jacc_th, int32_t max_cluster,
                                 int64_t* nclusters_out, int64_t** cluster_ptr_out,
                                 int32_t** rows_out) {
    return guarded([&] {
        check_host_csr(A, "variable_length_clusters");
        std::vector<std::vector<int32_t>> cl;
        if (A->nrows > 0) {
            int64_t rep = 0;
            cl.push_back({0});
            for (int64_t i = 1; i < A->nrows; ++i) {
                auto& cur = cl.back();
                const bool full = static_cast<int32_t>(cur.size()) >= max_cluster;
                if (!full && jaccard(A, rep, i) >= jacc_th) {
                    cur.push_back(static_cast<int32_t>(i));
                } else {
                    rep = i;
                    cl.push_back({static_cast<int32_t>(i)});
                }
            }
        }
        export_assignment(cl, nclusters_out, cluster_ptr_out, rows_out);
    });
}

int bsp_merge_candidates(const bsp_host_csr* A, const bsp_candidate* pairs, int64_t npairs,
                         double jacc_th, int32_t max_cluster, int64_t* nclusters_out,
                         int64_t** cluster_ptr_out, int32_t** rows_out, int64_t* nmerges_out,
                         bsp_candidate** merges_out) {
    return guarded([&] {
        check_host_csr(A, "merge_candidates");
        std::vector<bsp_candidate> trace;
        const auto cl = merge_candidates(A, pairs, npairs, jacc_th, max_cluster,
                                         merges_out ? &trace : nullptr);
        export_flat(cl, nclusters_out, cluster_ptr_out, rows_out);
        if (merges_out) {
            *merges_out = host_malloc<bsp_candidate>(trace.size());
            std::copy(trace.begin(), trace.end(), *merges_out);
            *nmerges_out = static_cast<int64_t>(trace.size());
        }
    });
}

int bsp_hierarchical_clusters(bsp_handle h, const bsp_host_csr* A, double jacc_th,
                              int32_t max_cluster, int32_t method, int32_t nhash, int32_t bands,
                              uint64_t seed, int64_t* nclusters_out, int64_t** cluster_ptr_out,
                              int32_t** rows_out) {
    return guarded([&] {
        check_host_csr(A, "hierarchical_clusters");
        require(method == 0 || method == 1, "hierarchical_clusters: method must be 0 or 1");
        std::vector<std::vector<int32_t>> cl;
        if (A->nrows == 0) {
            export_assignment(cl, nclusters_out, cluster_ptr_out, rows_out);
            return;
        }
        bsp_csr dA{}, dAt{};
        auto check = [](int rc) {
            if (rc != BSP_OK) throw std::runtime_error(bsp_last_error());
        };
        check(bsp_csr_upload(h, A->nrows, A->ncols, A->row_ptr, A->col_idx, A->values, &dA));
        bsp_candidate* pairs = nullptr;
        int64_t npairs = 0;
        const int32_t topk = std::max<int32_t>(max_cluster - 1, 1);
        int rc;
        if (method == 0) {
            rc = bsp_transpose(h, &dA, &dAt);
            if (rc == BSP_OK) rc = bsp_spgemm_topk(h, &dA, &dAt, topk, jacc_th, &pairs, &npairs);
            bsp_csr_free(h, &dAt);
        } else {
            rc = bsp_minhash_candidates(h, &dA, nhash, bands, seed, topk, jacc_th, &pairs, &npairs);
        }
        bsp_csr_free(h, &dA);
        check(rc);
        const auto flat = merge_candidates(A, pairs, npairs, jacc_th, max_cluster, nullptr);
        std::free(pairs);
        export_flat(flat, nclusters_out, cluster_ptr_out, rows_out);
    });
}

}  // extern "C"
