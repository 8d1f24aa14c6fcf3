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

// reference spgemm.hpp:41-63 (per-row exact output counts).
template <class Csr>
std::vector<int64_t> spgemm_symbolic(const Csr& a, const Csr& b, int /*num_threads*/ = 0,
                                     Engine& e = default_engine()) {
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
    counts.resize(static_cast<size_t>(a.nrows));
    return counts;
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

}  // namespace bsp_gpu
