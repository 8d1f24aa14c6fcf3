// cspgemm_gpu.hpp — C++ host mirror of the reference API over the C ABI.
//
// A drop-in for the reference's free functions (namespace cspgemm,
// /root/reference/proj/include/cspgemm/{spgemm,cluster_spgemm,clustering}.hpp):
// the same names, argument meaning and error behaviour (contract violations
// throw an exception derived from std::invalid_argument, like
// cspgemm::contract_error, types.hpp:16-19), but every multiply runs on the
// B200 through libbsp.so.  Header-only; link with -lbsp.
//
// The matrix type is a template parameter so the reference's own
// cspgemm::CsrMatrix (int32 row_ptr, csr.hpp:51-88) can be passed unchanged;
// any type with members nrows, ncols, row_ptr, col_idx, values works.
#pragma once

#include "bsp.h"

#include <cstdint>
#include <limits>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <vector>

namespace bsp_gpu {

struct contract_error : std::invalid_argument {
    explicit contract_error(const std::string& w) : std::invalid_argument(w) {}
};
struct device_error : std::runtime_error {
    explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
    if (rc == BSP_OK) return;
    const std::string msg = bsp_last_error();
    if (rc == BSP_ERR_CONTRACT) throw contract_error(msg);
    throw device_error(msg);
}

// One device handle (stream + memory pool) per thread of use.
class Engine {
public:
    explicit Engine(int device = 0) { check(bsp_create(device, &h_)); }
    ~Engine() { bsp_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    bsp_handle get() const { return h_; }

private:
    bsp_handle h_ = nullptr;
};

inline Engine& default_engine() {
    thread_local Engine e(0);
    return e;
}

namespace detail {

template <class Csr>
bsp_csr upload(Engine& e, const Csr& a) {
    std::vector<int64_t> rp(a.row_ptr.begin(), a.row_ptr.end());
    bsp_csr d{};
    check(bsp_csr_upload(e.get(), a.nrows, a.ncols, rp.data(), a.col_idx.data(),
                         a.values.data(), &d));
    return d;
}

// Download into the caller's matrix type; throws if its index type cannot
// hold nnz(C) (the reference's int32 index_t overflows past 2^31-1).
template <class Csr>
Csr download(Engine& e, bsp_csr& d) {
    Csr c;
    using Idx = typename std::decay<decltype(c.row_ptr[0])>::type;
    if (d.nnz > static_cast<int64_t>(std::numeric_limits<Idx>::max()))
        throw contract_error("spgemm: nnz(C) exceeds the index type of the result matrix");
    std::vector<int64_t> rp(static_cast<size_t>(d.nrows + 1));
    c.nrows = static_cast<decltype(c.nrows)>(d.nrows);
    c.ncols = static_cast<decltype(c.ncols)>(d.ncols);
    c.col_idx.resize(static_cast<size_t>(d.nnz));
    c.values.resize(static_cast<size_t>(d.nnz));
    check(bsp_csr_download(e.get(), &d, rp.data(), c.col_idx.data(), c.values.data()));
    c.row_ptr.assign(rp.begin(), rp.end());
    bsp_csr_free(e.get(), &d);
    return c;
}

}  // namespace detail

// reference spgemm.hpp:70-106.  num_threads is accepted for signature parity.
template <class Csr>
Csr spgemm_rowwise(const Csr& a, const Csr& b, int /*num_threads*/ = 0,
                   Engine& e = default_engine()) {
    if (a.ncols != b.nrows) throw contract_error("spgemm: dimension mismatch (a.ncols != b.nrows)");
    bsp_csr da = detail::upload(e, a);
    bsp_csr db = (&a == &b) ? da : detail::upload(e, b);
    bsp_csr dc{};
    const int rc = bsp_spgemm_rowwise(e.get(), &da, &db, &dc);
    if (&a != &b) bsp_csr_free(e.get(), &db);
    bsp_csr_free(e.get(), &da);
    check(rc);
    return detail::download<Csr>(e, dc);
}

// reference spgemm.hpp:41-63 (per-row exact output counts), in the matrix's
// own index type (cspgemm::index_t for the reference's CsrMatrix); a row's count
// always fits (< 2^31 outputs per row).
template <class Csr>
auto spgemm_symbolic(const Csr& a, const Csr& b, int /*num_threads*/ = 0,
                     Engine& e = default_engine())
    -> std::vector<typename std::decay<decltype(a.row_ptr[0])>::type> {
    using Idx = typename std::decay<decltype(a.row_ptr[0])>::type;
    if (a.ncols != b.nrows) throw contract_error("spgemm: dimension mismatch (a.ncols != b.nrows)");
    bsp_csr da = detail::upload(e, a), db = detail::upload(e, b);
    // counts land in a device buffer owned by a CSR-shaped scratch
    bsp_csr scratch{};
    std::vector<int64_t> zeros(static_cast<size_t>(a.nrows) + 1, 0);
    std::vector<int32_t> none;
    std::vector<double> nonev;
    check(bsp_csr_upload(e.get(), a.nrows, 1, zeros.data(), none.data(), nonev.data(), &scratch));
    const int rc = bsp_spgemm_symbolic(e.get(), &da, &db, scratch.row_ptr);
    std::vector<int64_t> counts(static_cast<size_t>(a.nrows) + 1);
    if (rc == BSP_OK) check(bsp_csr_download(e.get(), &scratch, counts.data(), nullptr, nullptr));
    bsp_csr_free(e.get(), &scratch);
    bsp_csr_free(e.get(), &db);
    bsp_csr_free(e.get(), &da);
    check(rc);
    return std::vector<Idx>(counts.begin(), counts.begin() + a.nrows);
}

// reference cluster_spgemm.hpp:186-189 with the CSR_Cluster built on the
// device from the assignment (cluster_format.hpp:130-186); C is returned as
// CSR over the original rows, i.e. cluster_to_csr(spgemm_clusterwise(...)).
template <class Csr, class Assignment>
Csr spgemm_clusterwise(const Csr& a, const Assignment& asg, const Csr& b, int /*nt*/ = 0,
                       Engine& e = default_engine()) {
    if (a.ncols != b.nrows)
        throw contract_error("spgemm_clusterwise: dimension mismatch (a.ncols != b.nrows)");
    std::vector<int64_t> ptr(1, 0);
    std::vector<int32_t> rows;
    for (const auto& c : asg.clusters) {
        rows.insert(rows.end(), c.begin(), c.end());
        ptr.push_back(static_cast<int64_t>(rows.size()));
    }
    bsp_csr da = detail::upload(e, a), db = detail::upload(e, b), dc{};
    bsp_csr_cluster ac{};
    int rc = bsp_csr_cluster_build(e.get(), &da, static_cast<int64_t>(asg.clusters.size()),
                                   ptr.data(), rows.data(), &ac);
    if (rc == BSP_OK) rc = bsp_spgemm_clusterwise(e.get(), &ac, &db, &dc, nullptr);
    bsp_csr_cluster_free(e.get(), &ac);
    bsp_csr_free(e.get(), &db);
    bsp_csr_free(e.get(), &da);
    check(rc);
    return detail::download<Csr>(e, dc);
}

namespace detail {

template <class Csr>
bsp_host_csr host_view(const Csr& a, std::vector<int64_t>& rp) {
    rp.assign(a.row_ptr.begin(), a.row_ptr.end());
    bsp_host_csr h{};
    h.nrows = a.nrows;
    h.ncols = a.ncols;
    h.nnz = rp.empty() ? 0 : rp.back();
    h.row_ptr = rp.data();
    h.col_idx = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(a.col_idx.data()));
    h.values = const_cast<double*>(a.values.data());
    return h;
}

// A flattened assignment (library-malloc'ed) into the caller's type, which
// has `clusters` (a vector of member vectors), like cspgemm::ClusterAssignment.
template <class Assignment>
Assignment adopt_assignment(int64_t nc, int64_t* ptr, int32_t* rows) {
    Assignment asg;
    asg.clusters.resize(static_cast<size_t>(nc));
    for (int64_t c = 0; c < nc; ++c)
        asg.clusters[c].assign(rows + ptr[c], rows + ptr[c + 1]);
    bsp_host_free_plain(ptr);
    bsp_host_free_plain(rows);
    return asg;
}

template <class Perm>
Perm adopt_perm(std::vector<int32_t>& p) {
    return Perm::from_perm({p.begin(), p.end()});
}

}  // namespace detail

// reference spgemm_topk (spgemm.hpp:144-206): the candidate list element for
// element (order, scores bitwise).  Pair: the caller's pair type with members
// i, j, score (cspgemm::CandidatePair), default bsp_candidate.
template <class Pair = bsp_candidate, class Csr>
std::vector<Pair> spgemm_topk(const Csr& a, const Csr& a_t, int topk, double jacc_th,
                              int /*num_threads*/ = 0, Engine& e = default_engine()) {
    if (a.ncols != a_t.nrows) throw contract_error("spgemm_topk: dimension mismatch");
    bsp_csr da = detail::upload(e, a), dt = detail::upload(e, a_t);
    bsp_candidate* pairs = nullptr;
    int64_t n = 0;
    const int rc = bsp_spgemm_topk(e.get(), &da, &dt, topk, jacc_th, &pairs, &n);
    bsp_csr_free(e.get(), &dt);
    bsp_csr_free(e.get(), &da);
    check(rc);
    std::vector<Pair> out(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        out[k].i = pairs[k].i;
        out[k].j = pairs[k].j;
        out[k].score = pairs[k].score;
    }
    bsp_host_free_plain(pairs);
    return out;
}

// reference hierarchical_clusters (clustering.hpp:109-185): GPU top-k
// candidates + the reference's merge rule; the assignment is identical.
// Params: any type with jacc_th and max_cluster_th (cspgemm::ClusterParams).
template <class Assignment, class Csr, class Params>
Assignment hierarchical_clusters(const Csr& a, const Params& prm, int /*num_threads*/ = 0,
                                 Engine& e = default_engine()) {
    std::vector<int64_t> rp;
    bsp_host_csr h = detail::host_view(a, rp);
    int64_t nc = 0, *ptr = nullptr;
    int32_t* rows = nullptr;
    check(bsp_hierarchical_clusters(e.get(), &h, prm.jacc_th, prm.max_cluster_th, 0, 64, 32, 1,
                                    &nc, &ptr, &rows));
    return detail::adopt_assignment<Assignment>(nc, ptr, rows);
}

// reference variable_length_clusters (clustering.hpp:76-93) / fixed (:59-69).
template <class Assignment, class Csr, class Params>
Assignment variable_length_clusters(const Csr& a, const Params& prm) {
    std::vector<int64_t> rp;
    bsp_host_csr h = detail::host_view(a, rp);
    int64_t nc = 0, *ptr = nullptr;
    int32_t* rows = nullptr;
    check(bsp_variable_length_clusters(&h, prm.jacc_th, prm.max_cluster_th, &nc, &ptr, &rows));
    return detail::adopt_assignment<Assignment>(nc, ptr, rows);
}

template <class Assignment>
Assignment fixed_length_clusters(int64_t nrows, int k) {
    int64_t nc = 0, *ptr = nullptr;
    int32_t* rows = nullptr;
    check(bsp_fixed_length_clusters(nrows, k, &nc, &ptr, &rows));
    return detail::adopt_assignment<Assignment>(nc, ptr, rows);
}

// reference reorder_rcm / reorder_degree / reorder_random (reorder.hpp:20-181)
// and load_permutation (matrix_market.hpp:141-166); Perm has from_perm
// (cspgemm::Permutation).
template <class Perm, class Csr>
Perm reorder_rcm(const Csr& a) {
    std::vector<int64_t> rp;
    bsp_host_csr h = detail::host_view(a, rp);
    std::vector<int32_t> p(static_cast<size_t>(a.nrows));
    check(bsp_reorder_rcm(&h, p.data()));
    return detail::adopt_perm<Perm>(p);
}

template <class Perm, class Csr>
Perm reorder_degree(const Csr& a) {
    std::vector<int64_t> rp;
    bsp_host_csr h = detail::host_view(a, rp);
    std::vector<int32_t> p(static_cast<size_t>(a.nrows));
    check(bsp_reorder_degree(&h, p.data()));
    return detail::adopt_perm<Perm>(p);
}

template <class Perm>
Perm reorder_random(int64_t n, uint64_t seed) {
    std::vector<int32_t> p(static_cast<size_t>(n));
    check(bsp_reorder_random(n, seed, p.data()));
    return detail::adopt_perm<Perm>(p);
}

template <class Perm>
Perm load_permutation(const std::string& path, int64_t nrows) {
    std::vector<int32_t> p(static_cast<size_t>(nrows));
    check(bsp_load_permutation(path.c_str(), nrows, p.data()));
    return detail::adopt_perm<Perm>(p);
}

}  // namespace bsp_gpu
