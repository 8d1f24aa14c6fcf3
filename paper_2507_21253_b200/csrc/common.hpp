// Internal helpers shared by the host C++ and CUDA translation units.
#pragma once

#include "bsp.h"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace bsp {

// Error classes mirroring the reference's (types.hpp:16-26); they are
// caught at the C ABI and turned into status codes.
struct contract_error : std::invalid_argument {
    explicit contract_error(const std::string& w) : std::invalid_argument(w) {}
};
struct io_error : std::runtime_error {
    explicit io_error(const std::string& w) : std::runtime_error(w) {}
};
struct cuda_error : std::runtime_error {
    explicit cuda_error(const std::string& w) : std::runtime_error(w) {}
};
struct oom_error : std::runtime_error {
    explicit oom_error(const std::string& w) : std::runtime_error(w) {}
};
struct nccl_error : std::runtime_error {
    explicit nccl_error(const std::string& w) : std::runtime_error(w) {}
};

inline void require(bool cond, const std::string& msg) {
    if (!cond) throw contract_error(msg);
}

void set_last_error(const std::string& msg);

// Runs f, mapping exceptions to BSP_ERR_* codes (no exception crosses the ABI).
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return BSP_OK;
    } catch (const contract_error& e) {
        set_last_error(std::string("contract_error: ") + e.what());
        return BSP_ERR_CONTRACT;
    } catch (const io_error& e) {
        set_last_error(std::string("io_error: ") + e.what());
        return BSP_ERR_IO;
    } catch (const oom_error& e) {
        set_last_error(std::string("out of memory: ") + e.what());
        return BSP_ERR_OOM;
    } catch (const cuda_error& e) {
        set_last_error(std::string("cuda: ") + e.what());
        return BSP_ERR_CUDA;
    } catch (const nccl_error& e) {
        set_last_error(std::string("nccl: ") + e.what());
        return BSP_ERR_NCCL;
    } catch (const std::bad_alloc&) {
        set_last_error("host out of memory");
        return BSP_ERR_OOM;
    } catch (const std::exception& e) {
        set_last_error(std::string("internal: ") + e.what());
        return BSP_ERR_INTERNAL;
    }
}

template <typename T>
T* host_malloc(std::size_t n) {
    if (n == 0) n = 1;
    void* p = std::malloc(n * sizeof(T));
    if (!p) throw std::bad_alloc();
    return static_cast<T*>(p);
}

// Host CSR with owning vectors; converted to/from bsp_host_csr at the ABI.
struct HostCsr {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> row_ptr{0};
    std::vector<int32_t> col_idx;
    std::vector<double> values;
    int64_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
    int64_t row_nnz(int64_t i) const { return row_ptr[i + 1] - row_ptr[i]; }
};

inline void export_csr(HostCsr&& m, bsp_host_csr* out) {
    out->nrows = m.nrows;
    out->ncols = m.ncols;
    out->nnz = m.nnz();
    out->row_ptr = host_malloc<int64_t>(m.row_ptr.size());
    out->col_idx = host_malloc<int32_t>(m.col_idx.size());
    out->values = host_malloc<double>(m.values.size());
    std::memcpy(out->row_ptr, m.row_ptr.data(), m.row_ptr.size() * sizeof(int64_t));
    std::memcpy(out->col_idx, m.col_idx.data(), m.col_idx.size() * sizeof(int32_t));
    std::memcpy(out->values, m.values.data(), m.values.size() * sizeof(double));
}

// Validates the reference's CSR invariants (csr.hpp:70-87) on a host view.
void check_host_csr(const bsp_host_csr* a, const char* who);

// Flattened cluster assignment helpers.
void export_assignment(const std::vector<std::vector<int32_t>>& clusters, int64_t* nclusters_out,
                       int64_t** cluster_ptr_out, int32_t** rows_out);

}  // namespace bsp
