// Engine internals shared by the CUDA translation units (sm_100a only).
#pragma once

#include "common.hpp"

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <vector>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "This engine is written for sm_100a (B200) only."
#endif

struct bsp_prof_rec {
    const char* name;
    cudaEvent_t a, b;
};

struct bsp_handle_s {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t launches = 0;
    bsp_exec_stats stats{};
    bool prof = false;
    std::vector<bsp_prof_rec> prof_recs;  // recorded launches (events owned)
    std::vector<cudaEvent_t> prof_pool;   // recycled events
    // Stream-ordered pools: plan/scratch buffers and arrays handed to the
    // caller (results, uploads) live apart, so scratch never splits the block
    // a freed result leaves behind and the next result of the same size
    // reuses it without remapping (cfg5: C is 138 GB of the 178 GB HBM).
    cudaMemPool_t scratch_pool = nullptr;
    cudaMemPool_t out_pool = nullptr;
    // Mapped pinned buffer for small synchronous readbacks (see d2h).
    void* rb_host = nullptr;
    void* rb_dev = nullptr;
    // Side stream for work that overlaps the main stream within one call
    // (light-row symbolic during the heavy-row planner); fork/join events.
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // Multi-GPU (comm.cu): this rank's NCCL communicator (one process per GPU),
    // created by bsp_comm_init; nullptr = single GPU.
    void* comm = nullptr;
    int comm_rank = 0, comm_size = 1;
    // bsp_spgemm_rowwise_sharded's row split of the last (A, B) pair (the split
    // needs every row's products: computed once, reused while A and B stay)
    // Start tables of the heavy-row planner (the largest scratch buffer, GBs on
    // cfg5), kept across multiplies and grown on demand: a fresh multi-GB pool
    // allocation now and then had to map new memory (a 30-80 ms host stall
    // between two kernels of a multiply).
    void* keep_starts = nullptr;
    size_t keep_starts_bytes = 0;
    // Free device memory outside this handle's pools, as of the last
    // cudaMemGetInfo (free_outside), with the pools' reserved bytes at that
    // moment: available_bytes() then follows the pools' own growth without
    // asking the driver again (see available_bytes).
    int64_t free_outside = -1;
    uint64_t free_reserved = 0;
    std::chrono::steady_clock::time_point free_time{};
    // Block cache above the pools (see dalloc): freed blocks by (pool, bytes); live
    // blocks are in a process-wide registry by address (a block may be freed
    // through another handle, e.g. a copy-stream handle after its download).
    struct FreeBlock {
        void* p;
        uint64_t stamp;  // alloc_seq when it was freed
    };
    std::unordered_multimap<uint64_t, FreeBlock> free_blocks;  // key = bytes << 1 | pool
    size_t cached_bytes = 0;
    uint64_t alloc_seq = 0;
    const void* part_key[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t part_nnz[2] = {0, 0};
    std::vector<int64_t> part_bounds;
};

namespace bsp {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw oom_error(std::string(what) + ": " + cudaGetErrorString(e));
    }
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

#define BSP_CUDA(call) ::bsp::cuda_check((call), #call)

// Every engine kernel launch goes through this so the handle can report how
// many of OUR kernels ran (bench.py's gpu_launches).
#define BSP_LAUNCH_AS(h, name, kernel, grid, block, smem, ...)                         \
    do {                                                                               \
        if ((grid) > 0) {                                                              \
            if (::bsp::gap_log_enabled()) ::bsp::gap_check_launch(name);               \
            const int prof_slot_ = ::bsp::prof_begin(h);                               \
            kernel<<<(grid), (block), (smem), (h)->stream>>>(__VA_ARGS__);             \
            ::bsp::cuda_check(cudaGetLastError(), name);                               \
            ::bsp::prof_end((h), prof_slot_, name);                                    \
            ++(h)->launches;                                                           \
            ++(h)->stats.kernels_launched;                                             \
            if (::bsp::trace_enabled()) ::bsp::trace_launch((h), name, (grid));        \
        }                                                                              \
    } while (0)
#define BSP_LAUNCH(h, kernel, grid, block, smem, ...) \
    BSP_LAUNCH_AS(h, #kernel, kernel, grid, block, smem, __VA_ARGS__)

// BSP_TRACE=1: synchronise and log every engine launch (debugging only).
bool trace_enabled();
void trace_launch(bsp_handle h, const char* name, long long grid);
// Per-launch CUDA-event profiling (bsp_profile): -1 when disabled.
int prof_begin(bsp_handle h);
void prof_end(bsp_handle h, int slot, const char* name);

// Launches inside this scope go to the handle's side stream (forked from and,
// by the caller, joined back into the main stream).
struct SideStream {
    bsp_handle h;
    cudaStream_t saved;
    explicit SideStream(bsp_handle hh) : h(hh), saved(hh->stream) {
        cuda_check(cudaEventRecord(h->ev_fork, saved), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(h->side, h->ev_fork, 0), "cudaStreamWaitEvent");
        h->stream = h->side;
    }
    ~SideStream() {
        cudaEventRecord(h->ev_join, h->side);
        h->stream = saved;
    }
    SideStream(const SideStream&) = delete;
    SideStream& operator=(const SideStream&) = delete;
};
inline void join_side(bsp_handle h) {
    cuda_check(cudaStreamWaitEvent(h->stream, h->ev_join, 0), "cudaStreamWaitEvent");
}

// BSP_GAP_LOG=1: log host time between a synchronisation's return and the next
// engine launch when it exceeds 1 ms (diagnoses GPU idle gaps inside a multiply).
bool gap_log_enabled();
void gap_mark_sync();
void gap_check_launch(const char* name);

// Stream-ordered device allocation from one of the handle's pools.
enum class Pool { scratch, out };

void gap_slow_call(const char* what, double ms);

// Live blocks of every handle, by address (engine.cu; mutex-guarded).
void block_registry_put(void* p, bsp_handle owner, size_t bytes, int pool);
// Removes p's entry; false when p is not a registered block.
bool block_registry_take(void* p, bsp_handle* owner, size_t* bytes, int* pool);

// Stream-ordered allocation with a per-handle block cache.  A repeated multiply
// asks for the same block sizes again, and every driver allocation call — even
// cudaMallocFromPoolAsync served from the pool's cached memory — takes driver
// locks that a GPU monitor (nvidia-smi, DCGM) holds for milliseconds at a time
// (measured on cfg5 under `nvidia-smi -lms 250`: pool allocations of 20-50 ms
// inside a multiply, one step in five 5-15 % long).  Freed blocks are therefore
// kept by exact size and handed back without a driver call.  A request the
// cache cannot serve allocates from the pool; blocks that no request has
// matched for kBlockMaxAge allocations go back to the pool then (large cached
// blocks at once when the missed request is itself large), and when the
// pool is out of memory every cached block goes back before one retry (so a
// different workload gets the memory it would have had without the cache;
// available_bytes counts cached blocks as available).  All blocks of a handle
// are used in its stream's order, like the stream-ordered frees they replace;
// changing the stream or destroying the handle flushes the cache.
constexpr uint64_t kBlockMaxAge = 4096;
// Only blocks this large are returned on a large miss: returning smaller ones made
// a repeated multiply cycle (block X released for a miss on Y, Y released for the
// next step's miss on X, ...: two driver allocations per step came back).
constexpr size_t kBigBlock = size_t{1} << 30;

inline void flush_block_cache(bsp_handle h) {
    for (auto& kv : h->free_blocks) cudaFreeAsync(kv.second.p, h->stream);
    h->free_blocks.clear();
    h->cached_bytes = 0;
}

inline void* dalloc_bytes(bsp_handle h, size_t bytes, Pool pool) {
    const int pi = pool == Pool::out ? 1 : 0;
    const uint64_t key = (static_cast<uint64_t>(bytes) << 1) | static_cast<uint64_t>(pi);
    ++h->alloc_seq;
    auto it = h->free_blocks.find(key);
    if (it != h->free_blocks.end()) {
        void* p = it->second.p;
        h->free_blocks.erase(it);
        h->cached_bytes -= bytes;
        block_registry_put(p, h, bytes, pi);
        return p;
    }
    // miss: stale blocks go back to the pool first — and, for a large request,
    // every large cached block of that pool: the pool then serves the request
    // from their (still mapped) memory instead of growing by as much again
    // (row-chunked multiplies: each chunk's C is tens of GB of a different size)
    const bool big = bytes >= kBigBlock;
    for (auto jt = h->free_blocks.begin(); jt != h->free_blocks.end();) {
        const size_t jb = static_cast<size_t>(jt->first >> 1);
        const int jp = static_cast<int>(jt->first & 1u);
        if (h->alloc_seq - jt->second.stamp > kBlockMaxAge || (big && jp == pi && jb >= kBigBlock)) {
            cudaFreeAsync(jt->second.p, h->stream);
            h->cached_bytes -= static_cast<size_t>(jt->first >> 1);
            jt = h->free_blocks.erase(jt);
        } else {
            ++jt;
        }
    }
    void* p = nullptr;
    ++h->stats.units[14];  // a driver allocation inside this call
    const bool lg = gap_log_enabled();
    if (lg) std::fprintf(stderr, "[miss] %zu bytes pool %d (%zu blocks cached)\n", bytes, pi, h->free_blocks.size());
    const auto t0 = lg ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    cudaMemPool_t mp = pool == Pool::out ? h->out_pool : h->scratch_pool;
    cudaError_t me = cudaMallocFromPoolAsync(&p, bytes, mp, h->stream);
    if (me == cudaErrorMemoryAllocation && !h->free_blocks.empty()) {
        cudaGetLastError();
        flush_block_cache(h);
        me = cudaMallocFromPoolAsync(&p, bytes, mp, h->stream);
    }
    if (me == cudaErrorMemoryAllocation) h->free_outside = -1;  // the cached figure was wrong
    cuda_check(me, "cudaMallocFromPoolAsync");
    if (lg)
        gap_slow_call("cudaMallocFromPoolAsync",
                      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                          .count());
    block_registry_put(p, h, bytes, pi);
    return p;
}

template <typename T>
T* dalloc(bsp_handle h, int64_t n, Pool pool = Pool::scratch) {
    return static_cast<T*>(
        dalloc_bytes(h, static_cast<size_t>(n > 0 ? n : 1) * sizeof(T), pool));
}

inline void dfree(bsp_handle h, void* p) {
    if (!p) return;
    bsp_handle owner = nullptr;
    size_t bytes = 0;
    int pool = 0;
    static const bool cache_on = [] {
        const char* e = std::getenv("BSP_BLOCK_CACHE");
        return !(e && e[0] == '0');
    }();
    // another handle's block (or not a registered one): plain stream-ordered free
    if (!block_registry_take(p, &owner, &bytes, &pool) || owner != h || !cache_on) {
        cudaFreeAsync(p, h->stream);
        return;
    }
    h->free_blocks.emplace((static_cast<uint64_t>(bytes) << 1) | static_cast<uint64_t>(pool),
                           bsp_handle_s::FreeBlock{p, h->alloc_seq});
    h->cached_bytes += bytes;
}

// Device bytes available to a new allocation: free HBM plus what the
// handle's pools hold cached but unused.
// refresh = true: ask the driver now (allocation failures, explicit requests).
size_t available_bytes(bsp_handle h, bool refresh = false);

// RAII device buffer bound to a handle's stream.
template <typename T>
struct DBuf {
    bsp_handle h = nullptr;
    T* p = nullptr;
    int64_t n = 0;
    DBuf() = default;
    DBuf(bsp_handle hh, int64_t nn, Pool pool = Pool::scratch)
        : h(hh), p(dalloc<T>(hh, nn, pool)), n(nn) {}
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    // non-owning view of a buffer that outlives this object (handle caches)
    static DBuf borrow(T* q, int64_t nn) {
        DBuf d;
        d.p = q;
        d.n = nn;
        d.own = false;
        return d;
    }
    DBuf(DBuf&& o) noexcept : h(o.h), p(o.p), n(o.n), own(o.own) { o.p = nullptr; }
    DBuf& operator=(DBuf&& o) noexcept {
        reset();
        h = o.h;
        p = o.p;
        n = o.n;
        own = o.own;
        o.p = nullptr;
        return *this;
    }
    ~DBuf() { reset(); }
    void reset() {
        if (p && own) dfree(h, p);
        p = nullptr;
    }
    bool own = true;
    T* release() {
        T* q = p;
        p = nullptr;
        return q;
    }
};

// Small device -> host reads (plan counters, scalars) are written by a
// one-block kernel into mapped pinned memory and complete synchronously:
// they never queue on a copy engine behind a multi-GB result download
// running on another stream.  Larger reads are ordinary async copies.
constexpr size_t kReadbackBytes = 64 << 10;
void small_readback(bsp_handle h, void* dst, const void* src, size_t bytes);

template <typename T>
void d2h(bsp_handle h, T* dst, const T* src, int64_t n) {
    if (n <= 0) return;
    const size_t bytes = static_cast<size_t>(n) * sizeof(T);
    if (bytes <= kReadbackBytes) {
        small_readback(h, dst, src, bytes);
        return;
    }
    BSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
}
template <typename T>
void h2d(bsp_handle h, T* dst, const T* src, int64_t n) {
    if (n <= 0) return;
    BSP_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, h->stream));
}
inline void sync(bsp_handle h) {
    BSP_CUDA(cudaStreamSynchronize(h->stream));
    if (gap_log_enabled()) gap_mark_sync();
}

template <typename T>
T read_scalar(bsp_handle h, const T* dptr) {
    T v{};
    d2h(h, &v, dptr, 1);
    sync(h);
    return v;
}

inline void check_csr(const bsp_csr* m, const char* who) {
    require(m != nullptr, std::string(who) + ": null matrix");
    require(m->nrows >= 0 && m->ncols >= 0 && m->nnz >= 0, std::string(who) + ": bad shape");
    require(m->row_ptr != nullptr, std::string(who) + ": null row_ptr");
    require(m->nrows < (int64_t{1} << 31) && m->ncols < (int64_t{1} << 31),
            std::string(who) + ": dimensions must fit int32 indices");
}

// Device-wide exclusive scans (int64) via CUB, with temp storage from the pool.
void exclusive_scan_i64(bsp_handle h, const int64_t* in, int64_t* out, int64_t n);
void exclusive_scan_i32_to_i64(bsp_handle h, const int32_t* in, int64_t* out, int64_t n);
int64_t reduce_sum_i64(bsp_handle h, const int64_t* in, int64_t n);

// Shared row-wise machinery (rowwise.cu), reused by the cluster-wise and
// top-k paths.
struct RowwisePlan;
void rowwise_multiply(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int64_t row_begin,
                      int64_t row_end, bsp_csr* C, const uint8_t* row_skip /*nullable*/,
                      int64_t* row_nnz_out /*nullable, device*/);

inline int64_t div_up(int64_t a, int64_t b) { return (a + b - 1) / b; }

// A multiply result's payload: nnz values followed by nnz column indices in
// one output-pool block (bsp_csr.owned == 2).
struct ResultPayload {
    DBuf<double> block;
    int64_t nnz = 0;
    ResultPayload(bsp_handle h, int64_t n) : block(h, n + (n + 1) / 2, Pool::out), nnz(n) {}
    // capacity for `cap` entries (the count is known only after the numeric
    // pass): values at [0, cap), column indices after them
    ResultPayload(bsp_handle h, int64_t n, int64_t cap)
        : block(h, cap + (cap + 1) / 2, Pool::out), nnz(cap) {}
    double* values() const { return block.p; }
    int32_t* col_idx() const { return reinterpret_cast<int32_t*>(block.p + nnz); }
};

}  // namespace bsp
