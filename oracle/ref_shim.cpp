// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  Exposes the UNMODIFIED reference
// implementation (header-only, compiled from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/libcspgemm_ref.so) through a plain C ABI so
// the tests can pin the oracle restatement (oracle.c) and so bench.py can time
// the reference's own CPU path (cpu_baseline kind "reference").  Nothing in
// the product links this library.
#include "cspgemm/cspgemm.hpp"
#include "cspgemm/bench.hpp"

#include <charconv>

#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

using namespace cspgemm;

namespace {
thread_local std::string g_err;

template <typename T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(v.size() * sizeof(T) + 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

// int64 row offsets (our ABI) -> the reference's int32 CsrMatrix.
CsrMatrix make(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci, const double* v) {
    CsrMatrix a;
    a.nrows = static_cast<index_t>(nrows);
    a.ncols = static_cast<index_t>(ncols);
    a.row_ptr.resize(nrows + 1);
    for (int64_t i = 0; i <= nrows; ++i) a.row_ptr[i] = static_cast<index_t>(rp[i] - rp[0]);
    const int64_t nnz = rp[nrows] - rp[0];
    a.col_idx.assign(ci + rp[0], ci + rp[0] + nnz);
    if (v)
        a.values.assign(v + rp[0], v + rp[0] + nnz);
    else
        a.values.assign(nnz, 1.0);
    return a;
}

ClusterAssignment make_asg(int64_t nclusters, const int64_t* cptr, const int32_t* rows) {
    ClusterAssignment asg;
    asg.clusters.resize(nclusters);
    for (int64_t c = 0; c < nclusters; ++c)
        asg.clusters[c].assign(rows + cptr[c], rows + cptr[c + 1]);
    return asg;
}

void export_asg(const ClusterAssignment& asg, int64_t* nc, int64_t** cptr, int32_t** rows) {
    *nc = static_cast<int64_t>(asg.clusters.size());
    std::vector<int64_t> ptr(1, 0);
    std::vector<int32_t> rr;
    for (const auto& c : asg.clusters) {
        rr.insert(rr.end(), c.begin(), c.end());
        ptr.push_back(static_cast<int64_t>(rr.size()));
    }
    *cptr = dup(ptr);
    *rows = dup(rr);
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const contract_error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// C = A*B on A rows [r0, r1) (row-block oracle: nnz(C_block) must stay < 2^31).
int ref_spgemm_rowwise(int64_t a_nrows, int64_t a_ncols, const int64_t* arp, const int32_t* aci,
                       const double* av, int64_t b_nrows, int64_t b_ncols, const int64_t* brp,
                       const int32_t* bci, const double* bv, int64_t r0, int64_t r1,
                       int num_threads, int64_t* nnz_out, int64_t** crp, int32_t** cci,
                       double** cv) {
    return guard([&] {
        (void)a_nrows;
        CsrMatrix a = make(r1 - r0, a_ncols, arp + r0, aci, av);
        // make() rebases offsets; keep absolute pointers consistent
        CsrMatrix b = make(b_nrows, b_ncols, brp, bci, bv);
        CsrMatrix c = spgemm_rowwise(a, b, num_threads);
        std::vector<int64_t> rp(c.row_ptr.begin(), c.row_ptr.end());
        *nnz_out = c.nnz();
        *crp = dup(rp);
        *cci = dup(c.col_idx);
        *cv = dup(c.values);
    });
}

int ref_spgemm_symbolic(int64_t a_nrows, int64_t a_ncols, const int64_t* arp, const int32_t* aci,
                        int64_t b_nrows, int64_t b_ncols, const int64_t* brp, const int32_t* bci,
                        int num_threads, int64_t* counts) {
    return guard([&] {
        CsrMatrix a = make(a_nrows, a_ncols, arp, aci, nullptr);
        CsrMatrix b = make(b_nrows, b_ncols, brp, bci, nullptr);
        const auto cnt = spgemm_symbolic(a, b, num_threads);
        for (int64_t i = 0; i < a_nrows; ++i) counts[i] = cnt[i];
    });
}

struct ref_candidate {
    int32_t i, j;
    double score;
};

int ref_spgemm_topk(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                    int32_t topk, double jacc_th, int num_threads, int64_t* npairs,
                    ref_candidate** pairs) {
    return guard([&] {
        CsrMatrix a = binarize(make(nrows, ncols, rp, ci, nullptr));
        CsrMatrix at = transpose(a);
        const auto v = spgemm_topk(a, at, topk, jacc_th, num_threads);
        std::vector<ref_candidate> out;
        out.reserve(v.size());
        for (const auto& p : v) out.push_back({p.i, p.j, p.score});
        *npairs = static_cast<int64_t>(out.size());
        *pairs = dup(out);
    });
}

int ref_hierarchical_clusters(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                              double jacc_th, int32_t max_cluster, int num_threads, int64_t* nc,
                              int64_t** cptr, int32_t** rows) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        ClusterParams prm;
        prm.jacc_th = jacc_th;
        prm.max_cluster_th = max_cluster;
        export_asg(hierarchical_clusters(a, prm, num_threads), nc, cptr, rows);
    });
}

int ref_variable_length_clusters(int64_t nrows, int64_t ncols, const int64_t* rp,
                                 const int32_t* ci, double jacc_th, int32_t max_cluster,
                                 int64_t* nc, int64_t** cptr, int32_t** rows) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        ClusterParams prm;
        prm.jacc_th = jacc_th;
        prm.max_cluster_th = max_cluster;
        export_asg(variable_length_clusters(a, prm), nc, cptr, rows);
    });
}

// Cluster-wise: builds CSR_Cluster(A, assignment), multiplies by B, returns
// cluster_to_csr(C) plus the access statistics and C's cluster slot count.
int ref_spgemm_clusterwise(int64_t nrows, int64_t ncols, const int64_t* arp, const int32_t* aci,
                           const double* av, int64_t b_nrows, int64_t b_ncols, const int64_t* brp,
                           const int32_t* bci, const double* bv, int64_t nclusters,
                           const int64_t* cptr, const int32_t* crows, int num_threads,
                           int64_t* nnz_out, int64_t** crp, int32_t** cci, double** cv,
                           uint64_t* stats3, int64_t* c_slots, int64_t* c_colslots) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, arp, aci, av);
        CsrMatrix b = make(b_nrows, b_ncols, brp, bci, bv);
        CsrClusterMatrix ac = build_csr_cluster(a, make_asg(nclusters, cptr, crows));
        auto [cc, st] = spgemm_clusterwise_instrumented(ac, b, num_threads);
        CsrMatrix c = cluster_to_csr(cc);
        std::vector<int64_t> rp(c.row_ptr.begin(), c.row_ptr.end());
        *nnz_out = c.nnz();
        *crp = dup(rp);
        *cci = dup(c.col_idx);
        *cv = dup(c.values);
        stats3[0] = st.b_row_loads;
        stats3[1] = st.a_inner_iters;
        stats3[2] = st.placeholder_skips;
        *c_slots = static_cast<int64_t>(cc.value_slots());
        *c_colslots = static_cast<int64_t>(cc.col_idx.size());
    });
}

// Timing entry for the CPU baseline: cluster-wise multiply only (format
// built outside), returns seconds of spgemm_clusterwise.
int ref_time_clusterwise(int64_t nrows, int64_t ncols, const int64_t* arp, const int32_t* aci,
                         const double* av, int64_t nclusters, const int64_t* cptr,
                         const int32_t* crows, int num_threads, int reps, double* seconds) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, arp, aci, av);
        CsrClusterMatrix ac = build_csr_cluster(a, make_asg(nclusters, cptr, crows));
        double best = 1e300;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            CsrClusterMatrix cc = spgemm_clusterwise(ac, a, num_threads);
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (s < best) best = s;
        }
        *seconds = best;
    });
}

// Prepared operands for bench.py's timing legs: the reference's own types are
// built once (the int64 -> int32 conversion and copies stay outside the timed
// call), then only spgemm_rowwise / spgemm_clusterwise is timed.
void* ref_csr_new(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                  const double* v) {
    try {
        return new CsrMatrix(make(nrows, ncols, rp, ci, v));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_csr_delete(void* p) { delete static_cast<CsrMatrix*>(p); }

int ref_time_rowwise(const void* a, const void* b, int num_threads, double* seconds,
                     int64_t* nnz) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        CsrMatrix c = spgemm_rowwise(*static_cast<const CsrMatrix*>(a),
                                     *static_cast<const CsrMatrix*>(b), num_threads);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *nnz = c.nnz();
    });
}

void* ref_cluster_new(const void* a, int64_t nclusters, const int64_t* cptr, const int32_t* crows) {
    try {
        return new CsrClusterMatrix(
            build_csr_cluster(*static_cast<const CsrMatrix*>(a), make_asg(nclusters, cptr, crows)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_cluster_delete(void* p) { delete static_cast<CsrClusterMatrix*>(p); }

int ref_time_clusterwise_prepared(const void* ac, const void* b, int num_threads, double* seconds,
                                  int64_t* slots) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        CsrClusterMatrix cc = spgemm_clusterwise(*static_cast<const CsrClusterMatrix*>(ac),
                                                 *static_cast<const CsrMatrix*>(b), num_threads);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *slots = static_cast<int64_t>(cc.value_slots());
    });
}

// Matrix Market / permutation files through the reference's own readers
// (matrix_market.hpp), for the IO parity tests.
int ref_load_matrix_market(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz,
                           int64_t** crp, int32_t** cci, double** cv) {
    return guard([&] {
        CsrMatrix a = coo_to_csr(load_matrix_market(path));
        std::vector<int64_t> rp(a.row_ptr.begin(), a.row_ptr.end());
        *nrows = a.nrows;
        *ncols = a.ncols;
        *nnz = a.nnz();
        *crp = dup(rp);
        *cci = dup(a.col_idx);
        *cv = dup(a.values);
    });
}

int ref_load_permutation(const char* path, int64_t nrows, int32_t* perm) {
    return guard([&] {
        const Permutation p = load_permutation(path, static_cast<index_t>(nrows));
        std::memcpy(perm, p.perm.data(), p.perm.size() * sizeof(int32_t));
    });
}

int ref_write_matrix_market(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                            const double* v, const char* path) {
    return guard([&] { write_matrix_market(make(nrows, ncols, rp, ci, v), path); });
}

// The reference's CSV report row (bench.hpp:260-290) from plain fields, and its
// double formatting (std::to_chars), for the harness parity tests.
int ref_fmt_double(double v, char* out, int cap) {
    return guard([&] {
        const auto r = std::to_chars(out, out + cap - 1, v);
        *r.ptr = 0;
    });
}

int ref_bench_csv_row(const char* matrix, int workload, int reorder_method, uint64_t reorder_seed,
                      const char* reorder_path, int cluster_method, double jacc_th,
                      int max_cluster, int fixed_len, int nf, int fb, uint64_t fseed, int reps,
                      int threads, int warmup, const double* d9, const uint64_t* u6,
                      double ratio, double amort, char* out, int cap) {
    return guard([&] {
        BenchReport r;
        r.config.matrix_path = matrix;
        r.config.workload = workload == 0 ? Workload::a_squared : Workload::tall_skinny;
        r.config.reorder.method = static_cast<ReorderSpec::Method>(reorder_method);
        r.config.reorder.seed = reorder_seed;
        r.config.reorder.path = reorder_path;
        r.config.clustering.method = static_cast<ClusteringSpec::Method>(cluster_method);
        r.config.clustering.params.jacc_th = jacc_th;
        r.config.clustering.params.max_cluster_th = max_cluster;
        r.config.clustering.params.fixed_len = fixed_len;
        r.config.num_frontiers = nf;
        r.config.frontier_batch = fb;
        r.config.frontier_seed = fseed;
        r.config.repetitions = reps;
        r.config.threads = threads;
        r.config.warmup = warmup != 0;
        r.reorder_seconds = d9[0];
        r.cluster_build_seconds = d9[1];
        r.baseline_mean_s = d9[2];
        r.baseline_min_s = d9[3];
        r.baseline_max_s = d9[4];
        r.variant_mean_s = d9[5];
        r.variant_min_s = d9[6];
        r.variant_max_s = d9[7];
        r.speedup_vs_baseline = d9[8];
        r.footprint.csr_bytes = u6[0];
        r.footprint.cluster_bytes = u6[1];
        r.footprint.ratio = ratio;
        r.baseline_access.b_row_loads = u6[2];
        r.access.b_row_loads = u6[3];
        r.access.a_inner_iters = u6[4];
        r.access.placeholder_skips = u6[5];
        r.amortization_iters = amort;
        const std::string row = bench_csv_row(r) + "\n" + bench_csv_header();
        if (static_cast<int>(row.size()) >= cap) throw std::runtime_error("buffer too small");
        std::memcpy(out, row.c_str(), row.size() + 1);
    });
}

int ref_build_cluster_dims(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                           int64_t nclusters, const int64_t* cptr, const int32_t* crows,
                           int64_t* colslots, int64_t* slots, int64_t* placeholders,
                           uint64_t* rowwise3, uint64_t* cluster3) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        CsrClusterMatrix ac = build_csr_cluster(a, make_asg(nclusters, cptr, crows));
        *colslots = static_cast<int64_t>(ac.col_idx.size());
        *slots = static_cast<int64_t>(ac.value_slots());
        *placeholders = static_cast<int64_t>(ac.placeholder_count());
        const auto rs = rowwise_access_stats(a, a);
        rowwise3[0] = rs.b_row_loads;
        rowwise3[1] = rs.a_inner_iters;
        rowwise3[2] = rs.placeholder_skips;
        (void)cluster3;
    });
}

int ref_reorder_rcm(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                    int32_t* perm) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        const Permutation p = reorder_rcm(a);
        std::memcpy(perm, p.perm.data(), p.perm.size() * sizeof(int32_t));
    });
}

int ref_reorder_random(int64_t n, uint64_t seed, int32_t* perm) {
    return guard([&] {
        const Permutation p = reorder_random(static_cast<index_t>(n), seed);
        std::memcpy(perm, p.perm.data(), p.perm.size() * sizeof(int32_t));
    });
}

int ref_reorder_degree(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                       int32_t* perm) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        const Permutation p = reorder_degree(a);
        std::memcpy(perm, p.perm.data(), p.perm.size() * sizeof(int32_t));
    });
}

int ref_permute_symmetric(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                          const double* v, const int32_t* perm, int64_t** orp, int32_t** oci,
                          double** ov) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, v);
        const Permutation p = Permutation::from_perm(std::vector<index_t>(perm, perm + nrows));
        CsrMatrix r = permute_symmetric(a, p);
        std::vector<int64_t> rr(r.row_ptr.begin(), r.row_ptr.end());
        *orp = dup(rr);
        *oci = dup(r.col_idx);
        *ov = dup(r.values);
    });
}

int ref_jaccard(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci, int64_t i,
                int64_t j, double* out) {
    return guard([&] {
        CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        *out = jaccard_similarity(a, static_cast<index_t>(i), static_cast<index_t>(j));
    });
}

// generate_frontiers (frontier.hpp:20-77): the t-th frontier's row_ptr is
// rps[t*(n+1) .. ], its columns cis[coff[t] .. coff[t+1]).
int ref_generate_frontiers(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                           int64_t num_frontiers, int64_t batch, uint64_t seed, int64_t* count,
                           int64_t* width, int64_t** rps, int64_t** coff, int32_t** cis) {
    return guard([&] {
        const CsrMatrix a = make(nrows, ncols, rp, ci, nullptr);
        const std::vector<CsrMatrix> fs = generate_frontiers(
            a, static_cast<index_t>(num_frontiers), static_cast<index_t>(batch), seed);
        *count = static_cast<int64_t>(fs.size());
        *width = fs.empty() ? 0 : fs[0].ncols;
        std::vector<int64_t> r, o(1, 0);
        std::vector<int32_t> c;
        for (const CsrMatrix& f : fs) {
            for (index_t x : f.row_ptr) r.push_back(x);
            c.insert(c.end(), f.col_idx.begin(), f.col_idx.end());
            o.push_back(static_cast<int64_t>(c.size()));
        }
        *rps = dup(r);
        *coff = dup(o);
        *cis = dup(c);
    });
}

}  // extern "C"
