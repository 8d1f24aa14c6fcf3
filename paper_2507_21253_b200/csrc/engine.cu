// Handle, memory and transfer entry points of the C ABI, plus device-wide
// scan helpers and the device transpose (reference csr.hpp:115-135).
#include "engine.cuh"

#include <mutex>
#include <unordered_map>
#include "esc.cuh"

#include <cub/device/device_radix_sort.cuh>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>

namespace bsp {

bool trace_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("BSP_TRACE");
        return v && v[0] == '1';
    }();
    return on;
}

void trace_launch(bsp_handle h, const char* name, long long grid) {
    std::fprintf(stderr, "[bsp] launch %s grid=%lld ...", name, grid);
    std::fflush(stderr);
    const cudaError_t e = cudaStreamSynchronize(h->stream);
    std::fprintf(stderr, " %s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    std::fflush(stderr);
}

static cudaEvent_t prof_event(bsp_handle h) {
    if (!h->prof_pool.empty()) {
        cudaEvent_t e = h->prof_pool.back();
        h->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    BSP_CUDA(cudaEventCreate(&e));
    return e;
}

int prof_begin(bsp_handle h) {
    if (!h->prof) return -1;
    bsp_prof_rec r{nullptr, prof_event(h), prof_event(h)};
    BSP_CUDA(cudaEventRecord(r.a, h->stream));
    h->prof_recs.push_back(r);
    return static_cast<int>(h->prof_recs.size()) - 1;
}

void prof_end(bsp_handle h, int slot, const char* name) {
    if (slot < 0) return;
    h->prof_recs[slot].name = name;
    BSP_CUDA(cudaEventRecord(h->prof_recs[slot].b, h->stream));
}

void exclusive_scan_i64(bsp_handle h, const int64_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    size_t tmp = 0;
    BSP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, h->stream));
    DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
    const int slot = prof_begin(h);
    BSP_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, h->stream));
    prof_end(h, slot, "cub_scan_i64");
    ++h->launches;
    ++h->stats.kernels_launched;
}

void exclusive_scan_i32_to_i64(bsp_handle h, const int32_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    size_t tmp = 0;
    BSP_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tmp, in, out, cub::Sum(), int64_t{0}, n,
                                            h->stream));
    DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
    const int slot = prof_begin(h);
    BSP_CUDA(cub::DeviceScan::ExclusiveScan(t.p, tmp, in, out, cub::Sum(), int64_t{0}, n,
                                            h->stream));
    prof_end(h, slot, "cub_scan_i32");
    ++h->launches;
    ++h->stats.kernels_launched;
}

int64_t reduce_sum_i64(bsp_handle h, const int64_t* in, int64_t n) {
    if (n <= 0) return 0;
    DBuf<int64_t> out(h, 1);
    size_t tmp = 0;
    BSP_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, in, out.p, n, h->stream));
    DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
    BSP_CUDA(cub::DeviceReduce::Sum(t.p, tmp, in, out.p, n, h->stream));
    ++h->launches;
    ++h->stats.kernels_launched;
    return read_scalar(h, out.p);
}

namespace {

__global__ void widen_rp_kernel(const int32_t* __restrict__ in, int64_t* __restrict__ out,
                                int64_t n) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < n;
         i += int64_t{gridDim.x} * blockDim.x)
        out[i] = in[i];
}

// Transpose, step 1: column histogram.
__global__ void col_count_kernel(const int32_t* __restrict__ col, int64_t nnz,
                                 int32_t* __restrict__ cnt) {
    for (int64_t p = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; p < nnz;
         p += int64_t{gridDim.x} * blockDim.x)
        atomicAdd(&cnt[col[p]], 1);
}

// Transpose, step 2: the row of every entry (a warp per source row).
__global__ void entry_rows_kernel(const int64_t* __restrict__ rp, int64_t nrows,
                                  int32_t* __restrict__ row_of, int32_t* __restrict__ iota) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = int64_t{gridDim.x} * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t{blockDim.x >> 5} + (threadIdx.x >> 5); i < nrows; i += nw)
        for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) {
            row_of[p] = static_cast<int32_t>(i);
            iota[p] = static_cast<int32_t>(p);
        }
}

// Transpose, step 3: after a STABLE radix sort of the entries by column
// (entries enter in row-major order, so equal columns keep ascending rows),
// gather the transposed entries: deterministic, rows of A^T sorted, no
// per-row sort (a hub column costs no more than any other).
__global__ void transpose_gather_kernel(const int32_t* __restrict__ perm, int64_t nnz,
                                        const int32_t* __restrict__ row_of,
                                        const double* __restrict__ val,
                                        int32_t* __restrict__ t_col, double* __restrict__ t_val) {
    for (int64_t q = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; q < nnz;
         q += int64_t{gridDim.x} * blockDim.x) {
        const int32_t p = perm[q];
        t_col[q] = row_of[p];
        if (val) t_val[q] = val[p];
    }
}

}  // namespace

namespace {
__global__ void readback_kernel(const unsigned char* __restrict__ src,
                                unsigned char* __restrict__ dst, size_t bytes) {
    const bool w4 = ((reinterpret_cast<uintptr_t>(src) | bytes) & 3) == 0;
    if (w4) {
        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
        for (size_t i = threadIdx.x; i < bytes / 4; i += blockDim.x) d4[i] = s4[i];
    } else {
        for (size_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
    }
}
}  // namespace

namespace {
thread_local std::chrono::steady_clock::time_point g_sync_ret{};
thread_local bool g_sync_set = false;
}  // namespace
bool gap_log_enabled() {
    static const bool on = std::getenv("BSP_GAP_LOG") != nullptr;
    return on;
}
void gap_mark_sync() {
    g_sync_ret = std::chrono::steady_clock::now();
    g_sync_set = true;
}
void gap_check_launch(const char* name) {
    if (!g_sync_set) return;
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - g_sync_ret).count();
    g_sync_set = false;
    if (ms > 1.0) std::fprintf(stderr, "[gap] %.2f ms host time before %s\n", ms, name);
}

void gap_slow_call(const char* what, double ms) {
    if (ms > 1.0) std::fprintf(stderr, "[slow] %.2f ms in %s\n", ms, what);
}

void small_readback(bsp_handle h, void* dst, const void* src, size_t bytes) {
    if (!h->rb_host) {
        BSP_CUDA(cudaHostAlloc(&h->rb_host, kReadbackBytes, cudaHostAllocMapped));
        BSP_CUDA(cudaHostGetDevicePointer(&h->rb_dev, h->rb_host, 0));
    }
    BSP_LAUNCH(h, readback_kernel, 1, 256, 0, static_cast<const unsigned char*>(src),
               static_cast<unsigned char*>(h->rb_dev), bytes);
    BSP_CUDA(cudaStreamSynchronize(h->stream));
    std::memcpy(dst, h->rb_host, bytes);
    if (gap_log_enabled()) gap_mark_sync();
}

// Device bytes a new allocation of this handle can get: free HBM outside the
// handle's pools plus the pools' reserved-but-unused bytes.
// cudaMemGetInfo takes a device-wide driver lock: on a box where anything polls
// the GPU (nvidia-smi, DCGM) it blocked for 5-180 ms every few calls, idling
// the GPU at the start of a multiply (measured on cfg5: one step in four
// +5..+180 ms, tools/step_gaps.py).  So the driver is asked only when the
// handle has no figure yet, every BSP_MEMINFO_PERIOD_S seconds (default 60),
// or on request (refresh: a failed allocation); in between, the figure follows
// the growth of this handle's own pools (cudaMemPoolGetAttribute, no device
// lock), which is where a multiply's memory goes.  Memory taken by other users
// of the device is seen at the next refresh.
namespace {
struct RegEntry {
    bsp_handle owner;
    size_t bytes;
    int pool;
};
std::mutex g_reg_mu;
std::unordered_map<void*, RegEntry> g_reg;
}  // namespace
void block_registry_put(void* p, bsp_handle owner, size_t bytes, int pool) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_reg[p] = RegEntry{owner, bytes, pool};
}
bool block_registry_take(void* p, bsp_handle* owner, size_t* bytes, int* pool) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_reg.find(p);
    if (it == g_reg.end()) return false;
    *owner = it->second.owner;
    *bytes = it->second.bytes;
    *pool = it->second.pool;
    g_reg.erase(it);
    return true;
}

size_t available_bytes(bsp_handle h, bool refresh) {
    uint64_t reserved_all = 0, unused = 0;
    for (cudaMemPool_t pool : {h->scratch_pool, h->out_pool}) {
        uint64_t reserved = 0, used = 0;
        BSP_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
        BSP_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
        reserved_all += reserved;
        unused += reserved - used;
    }
    static const double period_s = [] {
        const char* e = std::getenv("BSP_MEMINFO_PERIOD_S");
        return e ? std::atof(e) : 60.0;
    }();
    const auto now = std::chrono::steady_clock::now();
    if (refresh || h->free_outside < 0 ||
        std::chrono::duration<double>(now - h->free_time).count() > period_s) {
        size_t free_b = 0, total_b = 0;
        BSP_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (gap_log_enabled())
            gap_slow_call("cudaMemGetInfo", std::chrono::duration<double, std::milli>(
                                                std::chrono::steady_clock::now() - now).count());
        h->free_outside = static_cast<int64_t>(free_b);
        h->free_reserved = reserved_all;
        h->free_time = now;
    }
    // pools grown since the query took their memory from the free part
    int64_t outside = h->free_outside - (static_cast<int64_t>(reserved_all) -
                                         static_cast<int64_t>(h->free_reserved));
    if (outside < 0) outside = 0;
    // blocks in the handle's cache go back to the pools on the first miss
    return static_cast<size_t>(outside) + static_cast<size_t>(unused) + h->cached_bytes;
}

}  // namespace bsp

using namespace bsp;

extern "C" {

const char* bsp_version(void) { return "bsp 0.1 (sm_100a)"; }

int bsp_create(int device, bsp_handle* out) {
    return guarded([&] {
        require(out != nullptr, "bsp_create: null out");
        int ndev = 0;
        BSP_CUDA(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "bsp_create: no such device");
        BSP_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        BSP_CUDA(cudaGetDeviceProperties(&prop, device));
        require(prop.major >= 10, "bsp_create: this engine requires sm_100a (B200)");
        auto* h = new bsp_handle_s();
        h->device = device;
        h->sm_count = prop.multiProcessorCount;
        BSP_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
        BSP_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        BSP_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        BSP_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        for (cudaMemPool_t* pool : {&h->scratch_pool, &h->out_pool}) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = device;
            BSP_CUDA(cudaMemPoolCreate(pool, &props));
            uint64_t thr = UINT64_MAX;  // keep freed blocks mapped for reuse
            BSP_CUDA(cudaMemPoolSetAttribute(*pool, cudaMemPoolAttrReleaseThreshold, &thr));
            // Never make an allocation wait on another stream's pending free:
            // a result freed on a copy stream after its download must not
            // serialise the next multiply behind that download.
            int no = 0;
            BSP_CUDA(cudaMemPoolSetAttribute(*pool, cudaMemPoolReuseAllowInternalDependencies, &no));
        }
        *out = h;
    });
}

int bsp_destroy(bsp_handle h) {
    return guarded([&] {
        if (!h) return;
        cudaStreamSynchronize(h->stream);
        if (h->comm) bsp_comm_destroy(h);
        flush_block_cache(h);
        if (h->keep_starts) {
            bsp_handle o = nullptr;
            size_t b = 0;
            int pl = 0;
            block_registry_take(h->keep_starts, &o, &b, &pl);
            cudaFreeAsync(h->keep_starts, h->stream);
            cudaStreamSynchronize(h->stream);
        }
        if (h->own_stream) cudaStreamDestroy(h->stream);
        // pools with live allocations (results still held by the caller) are
        // released by the driver once those are freed
        if (h->side) {
            cudaStreamSynchronize(h->side);
            cudaStreamDestroy(h->side);
        }
        if (h->ev_fork) cudaEventDestroy(h->ev_fork);
        if (h->ev_join) cudaEventDestroy(h->ev_join);
        if (h->rb_host) cudaFreeHost(h->rb_host);
        if (h->scratch_pool) cudaMemPoolDestroy(h->scratch_pool);
        if (h->out_pool) cudaMemPoolDestroy(h->out_pool);
        delete h;
    });
}

int bsp_set_stream(bsp_handle h, void* s) {
    return guarded([&] {
        require(h != nullptr, "bsp_set_stream: null handle");
        BSP_CUDA(cudaSetDevice(h->device));
        flush_block_cache(h);  // cached blocks are ordered on the old stream
        if (h->own_stream) {
            BSP_CUDA(cudaStreamSynchronize(h->stream));
            BSP_CUDA(cudaStreamDestroy(h->stream));
            h->own_stream = false;
        }
        // NULL is the legacy default stream (torch's default stream).
        h->stream = static_cast<cudaStream_t>(s);
    });
}

int bsp_profile(bsp_handle h, int on) {
    return guarded([&] {
        require(h != nullptr, "bsp_profile: null handle");
        h->prof = on != 0;
    });
}

int64_t bsp_profile_report(bsp_handle h, char* buf, int64_t cap) {
    std::string out;
    const int rc = guarded([&] {
        require(h != nullptr, "bsp_profile_report: null handle");
        BSP_CUDA(cudaStreamSynchronize(h->stream));
        std::vector<std::pair<std::string, std::pair<int, double>>> acc;
        for (auto& r : h->prof_recs) {
            float ms = 0.f;
            BSP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            const std::string nm = r.name ? r.name : "?";
            auto it = std::find_if(acc.begin(), acc.end(), [&](auto& x) { return x.first == nm; });
            if (it == acc.end()) {
                acc.push_back({nm, {1, ms}});
            } else {
                it->second.first += 1;
                it->second.second += ms;
            }
            h->prof_pool.push_back(r.a);
            h->prof_pool.push_back(r.b);
        }
        h->prof_recs.clear();
        char line[256];
        for (auto& x : acc) {
            std::snprintf(line, sizeof line, "%s\t%d\t%.6f\n", x.first.c_str(), x.second.first,
                          x.second.second);
            out += line;
        }
    });
    if (rc != BSP_OK) return -1;
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(out.size()));
        std::memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return static_cast<int64_t>(out.size());
}

void* bsp_get_stream(bsp_handle h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int bsp_synchronize(bsp_handle h) {
    return guarded([&] { BSP_CUDA(cudaStreamSynchronize(h->stream)); });
}

int64_t bsp_kernel_launches(bsp_handle h) { return h ? h->launches : 0; }

int bsp_get_exec_stats(bsp_handle h, bsp_exec_stats* out) {
    return guarded([&] {
        require(h && out, "bsp_get_exec_stats: null argument");
        *out = h->stats;
    });
}

int bsp_csr_upload(bsp_handle h, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                   const int32_t* col_idx, const double* values, bsp_csr* out) {
    return guarded([&] {
        require(h && out && row_ptr, "bsp_csr_upload: null argument");
        require(nrows >= 0 && ncols >= 0, "bsp_csr_upload: negative shape");
        BSP_CUDA(cudaSetDevice(h->device));
        const int64_t nnz = row_ptr[nrows];
        require(row_ptr[0] == 0 && nnz >= 0, "bsp_csr_upload: bad row_ptr");
        DBuf<int64_t> rp(h, nrows + 1, Pool::out);
        DBuf<int32_t> ci(h, nnz, Pool::out);
        DBuf<double> v(h, nnz, Pool::out);
        h2d(h, rp.p, row_ptr, nrows + 1);
        h2d(h, ci.p, col_idx, nnz);
        if (values) {
            h2d(h, v.p, values, nnz);
        } else if (nnz > 0) {
            // pattern-only input: every stored value is 1.0 (binarize, csr.hpp:138-142)
            std::vector<double> ones(static_cast<size_t>(nnz), 1.0);
            h2d(h, v.p, ones.data(), nnz);
            sync(h);
        }
        out->nrows = nrows;
        out->ncols = ncols;
        out->nnz = nnz;
        out->row_ptr = rp.release();
        out->col_idx = ci.release();
        out->values = v.release();
        out->owned = 1;
    });
}

int bsp_csr_upload_rp32(bsp_handle h, int64_t nrows, int64_t ncols, const int32_t* row_ptr,
                        const int32_t* col_idx, const double* values, bsp_csr* out) {
    return guarded([&] {
        require(h && out && row_ptr, "bsp_csr_upload_rp32: null argument");
        std::vector<int64_t> rp(row_ptr, row_ptr + nrows + 1);
        const int rc = bsp_csr_upload(h, nrows, ncols, rp.data(), col_idx, values, out);
        if (rc != BSP_OK) throw std::runtime_error(bsp_last_error());
        sync(h);
    });
}

int bsp_csr_view(int64_t nrows, int64_t ncols, int64_t nnz, int64_t* row_ptr, int32_t* col_idx,
                 double* values, bsp_csr* out) {
    return guarded([&] {
        require(out != nullptr, "bsp_csr_view: null out");
        out->nrows = nrows;
        out->ncols = ncols;
        out->nnz = nnz;
        out->row_ptr = row_ptr;
        out->col_idx = col_idx;
        out->values = values;
        out->owned = 0;
    });
}

int bsp_csr_download(bsp_handle h, const bsp_csr* m, int64_t* row_ptr, int32_t* col_idx,
                     double* values) {
    return guarded([&] {
        check_csr(m, "bsp_csr_download");
        if (row_ptr) d2h(h, row_ptr, m->row_ptr, m->nrows + 1);
        if (col_idx) d2h(h, col_idx, m->col_idx, m->nnz);
        if (values) d2h(h, values, m->values, m->nnz);
        sync(h);
    });
}

int bsp_csr_download_async(bsp_handle h, const bsp_csr* m, int64_t* row_ptr, int32_t* col_idx,
                           double* values) {
    return guarded([&] {
        check_csr(m, "bsp_csr_download_async");
        if (row_ptr) d2h(h, row_ptr, m->row_ptr, m->nrows + 1);
        if (col_idx) d2h(h, col_idx, m->col_idx, m->nnz);
        if (values) d2h(h, values, m->values, m->nnz);
    });
}

int bsp_stream_wait(bsp_handle waiter, bsp_handle signaler) {
    return guarded([&] {
        require(waiter && signaler, "bsp_stream_wait: null handle");
        cudaEvent_t e;
        BSP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        BSP_CUDA(cudaEventRecord(e, signaler->stream));
        BSP_CUDA(cudaStreamWaitEvent(waiter->stream, e, 0));
        BSP_CUDA(cudaEventDestroy(e));
    });
}

int bsp_csr_free(bsp_handle h, bsp_csr* m) {
    return guarded([&] {
        if (!m) return;
        require(h != nullptr || !m->owned, "csr_free: null handle");
        if (m->owned) {
            dfree(h, m->row_ptr);
            if (m->owned != 2) dfree(h, m->col_idx);  // 2: col_idx inside the values block
            dfree(h, m->values);
        }
        m->row_ptr = nullptr;
        m->col_idx = nullptr;
        m->values = nullptr;
        m->owned = 0;
    });
}

int bsp_host_alloc(size_t bytes, void** out) {
    return guarded([&] { BSP_CUDA(cudaMallocHost(out, bytes > 0 ? bytes : 1)); });
}

int bsp_host_free(void* p) {
    return guarded([&] {
        if (p) BSP_CUDA(cudaFreeHost(p));
    });
}

int bsp_transpose(bsp_handle h, const bsp_csr* A, bsp_csr* out) {
    return guarded([&] {
        check_csr(A, "transpose");
        const int64_t n = A->ncols, nnz = A->nnz;
        DBuf<int32_t> cnt(h, n + 1);
        BSP_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(int32_t), h->stream));
        const int grid = static_cast<int>(std::min<int64_t>(div_up(std::max<int64_t>(nnz, 1), 256),
                                                            h->sm_count * 16));
        BSP_LAUNCH(h, col_count_kernel, grid, 256, 0, A->col_idx, nnz, cnt.p);
        DBuf<int64_t> rp(h, n + 1, Pool::out);
        exclusive_scan_i32_to_i64(h, cnt.p, rp.p, n + 1);
        require(nnz < (int64_t{1} << 31), "transpose: nnz must be < 2^31");
        DBuf<int32_t> row_of(h, nnz), iota(h, nnz), perm(h, nnz), keys(h, nnz);
        const int rgrid = static_cast<int>(
            std::min<int64_t>(div_up(std::max<int64_t>(A->nrows, 1), 8), h->sm_count * 16));
        BSP_LAUNCH(h, entry_rows_kernel, rgrid, 256, 0, A->row_ptr, A->nrows, row_of.p, iota.p);
        const int bits = std::max(1, bit_length(static_cast<uint32_t>(std::max<int64_t>(n - 1, 1))));
        size_t tmp = 0;
        BSP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, A->col_idx, keys.p, iota.p, perm.p,
                                                 nnz, 0, bits, h->stream));
        DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
        BSP_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, A->col_idx, keys.p, iota.p, perm.p, nnz,
                                                 0, bits, h->stream));
        ++h->launches;
        DBuf<int32_t> tc(h, nnz, Pool::out);
        DBuf<double> tv(h, nnz, Pool::out);
        BSP_LAUNCH(h, transpose_gather_kernel, grid, 256, 0, perm.p, nnz, row_of.p, A->values, tc.p,
                   A->values ? tv.p : nullptr);
        out->nrows = n;
        out->ncols = A->nrows;
        out->nnz = nnz;
        out->row_ptr = rp.release();
        out->col_idx = tc.release();
        out->values = tv.release();
        out->owned = 1;
    });
}

}  // extern "C"
