// Shared ESC (expand / stable-sort / compress) building blocks used by the
// row-wise, cluster-wise and top-k kernels.
#pragma once

#include "engine.cuh"

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include <mutex>
#include <unordered_map>

// Block scan algorithm of the tiles (A/B: -DBSP_SCAN_ALGO=cub::BLOCK_SCAN_WARP_SCANS)
#ifndef BSP_SCAN_ALGO
#define BSP_SCAN_ALGO cub::BLOCK_SCAN_RAKING
#endif

namespace bsp {

constexpr int CAP = 4096;     // max products of one sparse tile (smem ESC)
// Sparse-window tile classes (descending): a window runs in the smallest
// tile that holds its products (CUB's block sort always sorts the full tile).
// The 3072 class keeps 256 threads and is sized (≈73 KB smem, 85 registers)
// for 3 CTAs/SM; a 192-thread 3072 tile (2 CTAs x 6 warps) measured slower.
constexpr int NWCLS = 5;
constexpr int WD = 4096;      // dense window width in columns
constexpr int LOG_WD = 12;
constexpr int MAXBINS = 4096; // planner histogram bins per heavy row
constexpr int NCLS = 8;       // 0 empty, 1..6 light classes, 7 heavy
static __constant__ int kClassCap[NCLS] = {0, 128, 512, 1024, 2048, 3072, 4096, 0x7fffffff};

struct Mats {
    const int64_t* __restrict__ arp;
    const int32_t* __restrict__ acol;
    const double* __restrict__ aval;
    const int64_t* __restrict__ brp;
    const int32_t* __restrict__ bcol;
    const double* __restrict__ bval;
    int32_t ncols;  // columns of B (= of C)
    // planner start tables (windows): absolute B offsets per (window, segment),
    // 32-bit (tables are only built when nnz(B) < 2^32)
    const uint32_t* __restrict__ starts = nullptr;
    int64_t bnnz = 0;  // nnz(B) (host-side decisions)
    int64_t bnrows = 0;  // rows of B (host-side decisions)
};

// Per-B-row bin summary for the heavy-row planner: the row's columns as
// (bin << 16 | count) entries, one per run of columns in the same planner bin
// (4096 columns): cfg5's heavy rows reference 9.2e9 B entries but 5.4e9
// summary entries.  sptr == nullptr: the planner streams the columns.
struct BinSum {
    const int64_t* __restrict__ sptr = nullptr;  // [B rows + 1]
    const uint32_t* __restrict__ sent = nullptr;
};

struct Window {
    int32_t row;    // absolute A row
    int32_t c0, c1; // column range [c0, c1)
    int32_t first;  // index of the row's first window
    int32_t wi;     // index of this window within its row
    int32_t nprod;  // products in the window (sparse windows)
    int32_t d;      // segments of the row (A row length)
    int32_t pad_;
    int64_t rs;     // A row start (row_ptr[row])
    int64_t sofs;   // offset of the row's per-(window, segment) start table, or -1
};

struct OutCtx {
    int64_t row_begin;
    int64_t* row_nnz;        // [nrows of range] (symbolic output)
    int64_t* win_nnz;        // [nwindows] (symbolic output)
    const int64_t* crp;      // C row_ptr (numeric)
    const int64_t* win_scan; // exclusive scan of win_nnz (numeric)
    int32_t* ccol;
    double* cval;
};

__device__ __forceinline__ int64_t lower_bound_col(const int32_t* __restrict__ col, int64_t lo,
                                                   int64_t hi, int32_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(col + mid) < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// B range [b0, b1) that segment p (absolute A index; A row starts at rs and
// has d entries) contributes to a tile: the whole B row for a full row; for
// a window, the planner's start table when the row has one — absolute
// offsets, so no A/B row lookup at all — else a binary search for [c0, c1).
__device__ __forceinline__ void segment_range(const Mats& m, bool full, int64_t sofs, int wi,
                                              int64_t p, int64_t rs, int64_t d, int32_t c0,
                                              int32_t c1, int64_t& b0, int64_t& b1) {
    if (!full && sofs >= 0) {
        const uint32_t* st = m.starts + sofs + (p - rs);
        b0 = __ldg(st + int64_t{wi} * d);
        b1 = __ldg(st + int64_t{wi + 1} * d);
        return;
    }
    const int32_t k = __ldg(m.acol + p);
    b0 = __ldg(m.brp + k);
    b1 = __ldg(m.brp + k + 1);
    if (!full) {
        b0 = lower_bound_col(m.bcol, b0, b1, c0);
        b1 = lower_bound_col(m.bcol, b0, b1, c1);
    }
}

__host__ __device__ __forceinline__ int bit_length(uint32_t x) {
#ifdef __CUDA_ARCH__
    return 32 - __clz(x);
#else
    return x ? 32 - __builtin_clz(x) : 0;
#endif
}

// ---------------------------------------------------------------------------
// Register-staged ESC tile (CUB block radix sort of the whole tile): used by
// the top-k candidate kernels (topk.cu); the SpGEMM tiles are in merge.cuh.
// ---------------------------------------------------------------------------
template <int T, int I, bool NUMERIC>
struct EscShared {
    static constexpr int CAPT = T * I;
    using Sort = cub::BlockRadixSort<uint32_t, T, I, uint32_t>;
    using Scan = cub::BlockScan<int32_t, T>;
    uint32_t keys[CAPT];
    double vals[NUMERIC ? CAPT : 1];
    union {
        typename Sort::TempStorage sort;
        uint32_t sidx[CAPT];
    } u;
    typename Scan::TempStorage scan;
    int64_t pstart[T];
    int32_t plen[T];
    int32_t poff[T];
    double pav[NUMERIC ? T : 1];
};

// Expands the products of (row, [c0,c1)) into s.keys (column - c0) and, for
// NUMERIC, s.vals (a*b rounded), in (k ascending, j ascending) order.
// Returns the product count.
template <int T, int I, bool NUMERIC, typename S>
__device__ __forceinline__ int expand_products(const Mats& m, int32_t row, int32_t c0, int32_t c1,
                                               bool full, S& s, int64_t wsofs = -1,
                                               int wwi = 0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = T / 32;
    const int64_t rs = m.arp[row], re = m.arp[row + 1];
    int total = 0;
    for (int64_t pc = rs; pc < re; pc += T) {
        const int64_t p = pc + tid;
        int len = 0;
        int64_t start = 0;
        double av = 0.0;
        if (p < re) {
            int64_t b0, b1;
            segment_range(m, full, wsofs, wwi, p, rs, re - rs, c0, c1, b0, b1);
            start = b0;
            len = static_cast<int>(b1 - b0);
            if (NUMERIC) av = __ldg(m.aval + p);
        }
        int off, chunk;
        typename cub::BlockScan<int32_t, T>(s.scan).ExclusiveSum(len, off, chunk);
        s.pstart[tid] = start;
        s.plen[tid] = len;
        s.poff[tid] = total + off;
        if (NUMERIC) s.pav[tid] = av;
        __syncthreads();
        const int nslots = static_cast<int>(::min(int64_t{T}, re - pc));
        for (int slot = warp; slot < nslots; slot += NW) {
            const int l = s.plen[slot];
            const int64_t st = s.pstart[slot];
            const int o = s.poff[slot];
            double a = 0.0;
            if (NUMERIC) a = s.pav[slot];
            for (int q = lane; q < l; q += 32) {
                s.keys[o + q] = static_cast<uint32_t>(__ldg(m.bcol + st + q) - c0);
                if (NUMERIC) s.vals[o + q] = __dmul_rn(a, __ldg(m.bval + st + q));
            }
        }
        total += chunk;
        __syncthreads();
    }
    return total;
}


// The plan of one multiply: per-class row lists and heavy-row windows.
struct RowwisePlan {
    int64_t rb = 0, n = 0;
    int64_t class_count[NCLS]{}, class_products[NCLS]{};
    int64_t class_off[NCLS + 1]{};
    DBuf<int32_t> lists;  // all non-empty rows grouped by class
    DBuf<int64_t> prod;   // intermediate products per row (relative to rb)
    int64_t nwin = 0, nsparse = 0, ndense = 0;
    // sparse_ids[wcls_off[k], wcls_off[k+1]): windows of tile class k (kWinCap)
    int64_t wcls_off[NWCLS + 1]{};
    int64_t wcls_prod[NWCLS + 1]{};  // products per window category (dense = NWCLS)
    DBuf<Window> wins;
    DBuf<int32_t> sparse_ids, dense_ids;
    DBuf<uint32_t> starts; // planner per-(window, segment) start tables (absolute)
    bool light_sym_done = false;  // light rows counted on the side stream
    bool keep_tables = false;     // start tables in the handle's kept buffer
    // Free device bytes sampled at the start of the multiply (-1: query when
    // needed).  cudaMemGetInfo waits on the driver while nvidia-smi polls it
    // (measured: up to 65 ms); sampled before the first synchronisation, that
    // wait overlaps the previous multiply's kernels instead of idling the GPU.
    int64_t avail_hint = -1;
    // Set while that side-stream work is not yet joined into the main stream:
    // the destructor joins it before the plan's buffers are freed on the main
    // stream, so an error between build_plan and plan_symbolic cannot free
    // memory the side stream still reads.
    mutable bsp_handle side_h = nullptr;
    RowwisePlan() = default;
    RowwisePlan(const RowwisePlan&) = delete;
    RowwisePlan& operator=(const RowwisePlan&) = delete;
    ~RowwisePlan() {
        if (side_h) cudaStreamWaitEvent(side_h->stream, side_h->ev_join, 0);
    }
    // Matrices as seen by the window kernels (start tables attached).
    Mats with_starts(const Mats& m) const {
        Mats r = m;
        r.starts = starts.p;
        return r;
    }
};

Mats make_mats(const bsp_csr* A, const bsp_csr* B);
// early_row_nnz (zeroed, optional): count the light rows' outputs there on the
// handle's side stream while the heavy rows are planned (plan_symbolic joins).
// shadow (optional, with skip): the skipped rows planned apart in the same
// pass (light rows only; used for the cluster rows' symbolic).
void build_plan(bsp_handle h, const Mats& m, int64_t rb, int64_t re, const uint8_t* skip,
                RowwisePlan& plan, int64_t* prod_out, int64_t* early_row_nnz = nullptr,
                RowwisePlan* shadow = nullptr);
// Symbolic counts of a plan into row_nnz (NOT zeroed here) and win_nnz (allocated).
// skip_wcls >= 0: leave that window tile class out (counted by the look-back
// numeric instead).
void plan_symbolic(bsp_handle h, const Mats& m, const RowwisePlan& plan, int64_t* row_nnz,
                   DBuf<int64_t>& win_nnz, int skip_wcls = -1);
void plan_numeric(bsp_handle h, const Mats& m, const RowwisePlan& plan, const int64_t* crp,
                  const int64_t* win_scan, int32_t* ccol, double* cval, int skip_wcls = -1);
void sort_ids(bsp_handle h, int32_t* ids, int64_t n);
// Duplicate-heavy rows (absolute ids, each with at most 256 outputs) on the row-wise hash
// accumulator (rowwise.cu hashacc_kernel); C placed at crp[row - rb].
void run_hashacc_rows(bsp_handle h, const Mats& m, const int32_t* rows, int64_t n, int64_t rb,
                      const int64_t* crp, int32_t* ccol, double* cval);

// B with <= 64 columns: per-row 64-bit column masks of B, then the row-wise
// narrow kernel over rows [0, n) of A (skip[r] != 0 rows left out): symbolic
// when crp == nullptr (row_nnz, products), else numeric into C at crp.
void narrow64_row_masks(bsp_handle h, const Mats& m, int64_t bnrows,
                        DBuf<unsigned long long>& mask);
void narrow64_rows(bsp_handle h, const Mats& m, const unsigned long long* mask, int64_t n,
                   const uint8_t* skip, int64_t* row_nnz, const int64_t* crp, int32_t* ccol,
                   double* cval, unsigned long long* products);

// Opt a kernel into `bytes` of dynamic shared memory.  The attribute is set once
// per (kernel, device): cudaFuncSetAttribute is a driver call that can wait on
// the driver's locks (measured: up to 13 ms under a GPU monitor), and every
// multiply would otherwise make ~40 of them.
template <typename K>
void set_smem(K kernel, size_t bytes) {
    // (kernels of one signature share this instantiation: keyed by address and device)
    static std::mutex mu;
    static std::unordered_map<uint64_t, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t key = reinterpret_cast<uint64_t>(reinterpret_cast<const void*>(kernel)) ^
                         (static_cast<uint64_t>(dev) << 56);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = done.find(key);
        if (it != done.end() && it->second == bytes) return;
    }
    const bool lg = gap_log_enabled();
    const auto t0 = lg ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    BSP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
    if (lg)
        gap_slow_call("cudaFuncSetAttribute", std::chrono::duration<double, std::milli>(
                                                  std::chrono::steady_clock::now() - t0).count());
    std::lock_guard<std::mutex> lk(mu);
    done[key] = bytes;
}

}  // namespace bsp
