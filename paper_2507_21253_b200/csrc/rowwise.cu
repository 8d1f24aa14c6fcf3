// Row-wise Gustavson SpGEMM on sm_100a — the hot path.
//
// Replaces reference spgemm_symbolic (spgemm.hpp:41-63) and spgemm_rowwise
// (spgemm.hpp:70-106).  Parity contract: C's row_ptr/col_idx bit-exact and
// every value bit-identical to the reference, which accumulates
//     c_ij = ((0.0 + a_ik1*b_k1j) + a_ik2*b_k2j) + ...   (ascending k)
// with the multiply rounded before the add (no FMA; spgemm.hpp:92-97,
// hash_accumulator.hpp:57-65).
//
// Design:
//  K0 products_kernel: per-row intermediate products P_i (row_upper_bound,
//     spgemm.hpp:31-36) and the row's class (<= 128/512/1024/2048/3072/4096
//     products, or heavy); a warp per row.
//  K1 bucket_kernel:   row ids grouped by class.
//  K2 plan_count / plan_write: heavy rows are cut greedily into column
//     windows of <= 2048 products (one 4096-column bin of more than 4096
//     products is a "dense" window), with per-(window, segment) start tables.
//  K3 hash_count_kernel (symbolic) / esc_merge_kernel (numeric): one CTA
//     per light row or sparse window (merge.cuh): the products are gathered
//     into shared memory in (k, j) order with cp.async, sorted by column
//     (counting sort with an expansion-index tie-break, else a stable merge
//     of the presorted runs, CUB radix or MSD), and every run of equal
//     columns is summed left to right from 0.0 -> bit-exact values, stored
//     coalesced.
//  K4 dense_window_kernel<NUMERIC>: dense windows with a smem accumulator of
//     WD doubles + bitmap; products streamed in 1024-product batches in k
//     order, each batch stably sorted so per-column order is kept.
//  K5 hashacc_kernel: duplicate-heavy light rows (products >= 2 x outputs)
//     accumulated segment by segment in k order into a warp's smem hash.
//  K6 narrow64_kernel / narrow_kernel: B with <= 64 / <= 256 columns, a
//     warp per row with register / smem accumulators, no sort.
//  The symbolic pass gives exact per-row counts (exact allocation, as the
//  reference), then an int64 scan gives row_ptr.
#include "esc.cuh"
#include "merge.cuh"

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_partition.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>

namespace bsp {

namespace {


// ---------------------------------------------------------------------------
// K0: products and class per row
// ---------------------------------------------------------------------------
// A warp per row (grid-stride over rows): the lanes read the row's A entries
// coalesced and sum the B row lengths, so a hub row (~10^4 entries) is not a
// single thread's serial loop.
__global__ void products_kernel(Mats m, int64_t rb, int64_t n, int64_t* __restrict__ prod,
                                uint8_t* __restrict__ cls, const uint8_t* __restrict__ skip,
                                int64_t* __restrict__ class_count,
                                int64_t* __restrict__ class_products, int shadow,
                                unsigned long long* __restrict__ max_prod, int heavy_above = 4096) {
    // shadow: skipped rows get their own classes NCLS + c (a second plan)
    __shared__ unsigned long long s_cnt[2 * NCLS], s_prod[2 * NCLS], s_max;
    if (threadIdx.x < 2 * NCLS) {
        s_cnt[threadIdx.x] = 0;
        s_prod[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = int64_t{gridDim.x} * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t{blockDim.x >> 5} + (threadIdx.x >> 5); r < n;
         r += nwarps) {
        const int64_t i = rb + r;
        const int64_t p0 = m.arp[i], p1 = m.arp[i + 1];
        int64_t P = 0;
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const int32_t k = __ldg(m.acol + p);
            P += __ldg(m.brp + k + 1) - __ldg(m.brp + k);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) P += __shfl_xor_sync(0xffffffffu, P, o);
        if (lane == 0) {
            int c = 0;
            if (P > 0) {
                c = 1;
                while (c < NCLS - 1 && P > kClassCap[c]) ++c;
                if (P > heavy_above) c = NCLS - 1;  // planned into column windows
            }
            // skip 1: planned apart in the shadow plan; 2: counted elsewhere
            // (cluster union tiles count their own rows)
            if (skip && skip[r]) c = (shadow && c > 0 && skip[r] == 1) ? NCLS + c : 0;
            if (prod) prod[r] = P;
            cls[r] = static_cast<uint8_t>(c);
            atomicAdd(&s_cnt[c], 1ull);
            atomicAdd(&s_prod[c], static_cast<unsigned long long>(P));
            atomicMax(&s_max, static_cast<unsigned long long>(P));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && max_prod) atomicMax(max_prod, s_max);
    if (threadIdx.x < (shadow ? 2 * NCLS : NCLS)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&class_count[threadIdx.x]), s_cnt[threadIdx.x]);
        atomicAdd(reinterpret_cast<unsigned long long*>(&class_products[threadIdx.x]),
                  s_prod[threadIdx.x]);
    }
}

// K1: group row ids (absolute) by class into per-class regions.
__global__ void bucket_kernel(const uint8_t* __restrict__ cls, int64_t rb, int64_t n,
                              unsigned long long* __restrict__ cursor,
                              int32_t* __restrict__ lists, int32_t* __restrict__ lists2) {
    // classes NCLS + c (shadow plan) go to lists2 at cursor[NCLS + c]
    __shared__ unsigned s_cnt[2 * NCLS];
    __shared__ unsigned long long s_base[2 * NCLS];
    if (threadIdx.x < 2 * NCLS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t r = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    int c = 0;
    unsigned rank = 0;
    if (r < n) {
        c = cls[r];
        if (c > 0) rank = atomicAdd(&s_cnt[c], 1u);
    }
    __syncthreads();
    if (threadIdx.x > 0 && threadIdx.x < 2 * NCLS && s_cnt[threadIdx.x])
        s_base[threadIdx.x] = atomicAdd(&cursor[threadIdx.x], s_cnt[threadIdx.x]);
    __syncthreads();
    if (r < n && c > 0)
        (c < NCLS ? lists : lists2)[s_base[c] + rank] = static_cast<int32_t>(rb + r);
}

// ---------------------------------------------------------------------------
// K2: heavy-row planner
// ---------------------------------------------------------------------------
constexpr int PLAN_T = 256;
__constant__ int kWinCapDev[NWCLS] = {4096, 3072, 2048, 1024, 512};
constexpr int PLAN_U = 8;  // B-row chunks of 32 loaded ahead per warp
constexpr uint32_t DENSE_BIT = 0x80000000u;

struct PlanCountShared {
    int32_t hist[MAXBINS + 1];  // per-bin products, then (in place) pre[b] = products in bins < b
    typename cub::BlockScan<int32_t, PLAN_T>::TempStorage scan;
};

// Start tables of up to STAGE entries (uint32) are built in smem and stored
// coalesced.
constexpr int STAGE = 6144;
struct PlanWriteShared {
    uint16_t binwin[MAXBINS];  // bin -> window (a row has < 2^16 windows)
    union {
        struct {
            uint32_t wc0[MAXBINS + 1];  // window -> c0 | DENSE_BIT (+ sentinel ncols)
            int32_t wpre[MAXBINS + 1];  // window -> product prefix at c0 (+ sentinel P)
        } w;
        uint32_t stage[STAGE + 1];
    } u;
};

// Walk the segments (A-row entries) of `row` one warp per segment, the
// (b0, b1) bounds of 32 upcoming segments fetched at once by the warp's lanes
// and PLAN_U chunks of 32 B columns loaded before they are consumed, so each
// warp keeps several independent loads in flight.  f(p, q0, len, cols[U],
// state, b0) is called for each group of chunks (warp-uniform; once with q0 = 0
// for an empty segment); cols[u] holds the column of element q0 + 32u + lane
// or -1 past the end; `state` is an int reset to -1 at the start of every
// segment.
template <class F>
__device__ __forceinline__ void stream_segments(const Mats& m, int32_t row, F&& f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = PLAN_T / 32;
    const int64_t rs = m.arp[row];
    const int d = static_cast<int>(m.arp[row + 1] - rs);
    for (int pb = warp; pb < d; pb += NW * 32) {
        const int pl = pb + NW * lane;
        int64_t mb0 = 0, mb1 = 0;
        if (pl < d) {
            const int32_t k = __ldg(m.acol + rs + pl);
            mb0 = __ldg(m.brp + k);
            mb1 = __ldg(m.brp + k + 1);
        }
        const int nseg = ::min(32, (d - pb + NW - 1) / NW);
        for (int j = 0; j < nseg; ++j) {
            const int64_t b0 = __shfl_sync(0xffffffffu, mb0, j);
            const int len = static_cast<int>(__shfl_sync(0xffffffffu, mb1, j) - b0);
            const int p = pb + NW * j;
            int state = -1;
            // an empty segment still gets one call (all columns -1): the
            // start-table pass must fill its entries too
            for (int q0 = 0; q0 < ::max(len, 1); q0 += 32 * PLAN_U) {
                int32_t cols[PLAN_U];
#pragma unroll
                for (int u = 0; u < PLAN_U; ++u) {
                    const int q = q0 + 32 * u + lane;
                    cols[u] = q < len ? __ldg(m.bcol + b0 + q) : -1;
                }
                f(p, q0, len, cols, state, b0);
            }
        }
    }
}

// The same walk over the segments' bin summaries (BinSum): f(p, q0, nent,
// ent[U], carryw, eoff, b0, blen) per group of PLAN_U x 32 entries; ent[u] is
// entry q0 + 32u + lane or ~0u past the end; carryw / eoff are per-segment
// state (reset to -1 / 0); b0, blen: the B row's element range.
template <class F>
__device__ __forceinline__ void stream_summaries(const Mats& m, const BinSum& bs, int32_t row,
                                                 F&& f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = PLAN_T / 32;
    const int64_t rs = m.arp[row];
    const int d = static_cast<int>(m.arp[row + 1] - rs);
    for (int pb = warp; pb < d; pb += NW * 32) {
        const int pl = pb + NW * lane;
        int64_t mb0 = 0, mb1 = 0, ms0 = 0, ms1 = 0;
        if (pl < d) {
            const int32_t k = __ldg(m.acol + rs + pl);
            mb0 = __ldg(m.brp + k);
            mb1 = __ldg(m.brp + k + 1);
            ms0 = __ldg(bs.sptr + k);
            ms1 = __ldg(bs.sptr + k + 1);
        }
        const int nseg = ::min(32, (d - pb + NW - 1) / NW);
        for (int j = 0; j < nseg; ++j) {
            const int64_t b0 = __shfl_sync(0xffffffffu, mb0, j);
            const int blen = static_cast<int>(__shfl_sync(0xffffffffu, mb1, j) - b0);
            const int64_t s0 = __shfl_sync(0xffffffffu, ms0, j);
            const int nent = static_cast<int>(__shfl_sync(0xffffffffu, ms1, j) - s0);
            const int p = pb + NW * j;
            int carryw = -1, eoff = 0;
            for (int q0 = 0; q0 < ::max(nent, 1); q0 += 32 * PLAN_U) {
                uint32_t ent[PLAN_U];
#pragma unroll
                for (int u = 0; u < PLAN_U; ++u) {
                    const int q = q0 + 32 * u + lane;
                    ent[u] = q < nent ? __ldg(bs.sent + s0 + q) : ~0u;
                }
                f(p, q0, nent, ent, carryw, eoff, b0, blen);
            }
        }
    }
}

// Bin summary of B (see BinSum): a warp per B row; runs of columns in one bin
// become one entry, a run continuing across 32-column chunks extends the
// previous entry.  MODE 0 counts entries per row, MODE 1 writes them.
template <int MODE>
__global__ void bin_summary_kernel(const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol,
                                   int64_t nb, int log_binw, int64_t* __restrict__ cnt,
                                   const int64_t* __restrict__ sptr, uint32_t* __restrict__ sent) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = int64_t{gridDim.x} * (blockDim.x >> 5);
    const unsigned below = (1u << lane) - 1u;
    for (int64_t k = blockIdx.x * int64_t{blockDim.x >> 5} + (threadIdx.x >> 5); k < nb; k += nw) {
        const int64_t b0 = brp[k];
        const int len = static_cast<int>(brp[k + 1] - b0);
        int64_t pos = MODE ? sptr[k] : 0;
        int32_t carry_bin = -1;
        int64_t n = 0;
        for (int q0 = 0; q0 < len; q0 += 32) {
            const int q = q0 + lane;
            const bool valid = q < len;
            const int32_t bin = valid ? (__ldg(bcol + b0 + q) >> log_binw) : -2;
            int32_t prev = __shfl_up_sync(0xffffffffu, bin, 1);
            if (lane == 0) prev = carry_bin;
            const bool head = valid && bin != prev;
            const unsigned heads = __ballot_sync(0xffffffffu, head);
            if (MODE) {
                const int end = ::min(32, len - q0);
                if (valid && (head || lane == 0)) {
                    // run length up to the next head in this chunk (or its end)
                    const unsigned above = heads & ~((2u << lane) - 1u);
                    const int stop = above ? __ffs(above) - 1 : end;
                    const uint32_t run = static_cast<uint32_t>(stop - lane);
                    if (head)
                        sent[pos + __popc(heads & below)] = (static_cast<uint32_t>(bin) << 16) | run;
                    else  // lane 0 continues the previous chunk's last run
                        sent[pos - 1] += run;
                }
            }
            pos += __popc(heads);
            n += __popc(heads);
            carry_bin = __shfl_sync(0xffffffffu, bin, ::min(31, len - 1 - q0));
            __syncwarp();
        }
        if (!MODE && lane == 0) cnt[k] = n;
    }
}

// K2a: per heavy row, a product histogram over `nbins` column bins, then the
// greedy window cut (below).  Writes the window count and the descriptors
// {c0 | DENSE_BIT, product prefix} (+ sentinel {ncols, P}) at desc[doff[h]].
__global__ void __launch_bounds__(PLAN_T, 8) plan_count_kernel(Mats m,
                                                            const int32_t* __restrict__ heavy,
                                                            int32_t nbins, int log_binw,
                                                            int32_t* __restrict__ nwin,
                                                            const int64_t* __restrict__ doff,
                                                            uint2* __restrict__ desc,
                                                            int32_t capg, BinSum bs) {
    __shared__ PlanCountShared s;
    const int32_t hrow = blockIdx.x;
    const int32_t row = heavy[hrow];
    const int lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < nbins; b += PLAN_T) s.hist[b] = 0;
    __syncthreads();
    if (bs.sptr) {
        // bin summaries: one atomic per (segment, bin) run instead of per column
        stream_summaries(m, bs, row, [&](int, int q0, int nent, const uint32_t* ent, int&, int&,
                                         int64_t, int) {
#pragma unroll
            for (int u = 0; u < PLAN_U; ++u) {
                if (q0 + 32 * u >= nent) break;
                if (ent[u] != ~0u) atomicAdd(&s.hist[ent[u] >> 16], static_cast<int>(ent[u] & 0xffffu));
            }
        });
    } else
    stream_segments(m, row, [&](int, int q0, int len, const int32_t* cols, int&, int64_t) {
#pragma unroll
        for (int u = 0; u < PLAN_U; ++u) {
            if (q0 + 32 * u >= len) break;
            const bool ok = cols[u] >= 0;
            const int32_t bin = ok ? (cols[u] >> log_binw) : 0x7fffffff;
            // columns are sorted within the B row, so equal bins form runs:
            // the last lane of each run adds the run length.
            const int32_t nxt = __shfl_down_sync(0xffffffffu, bin, 1);
            const int32_t prv = __shfl_up_sync(0xffffffffu, bin, 1);
            const bool tail = ok && (lane == 31 || nxt != bin);
            const unsigned heads = __ballot_sync(0xffffffffu, ok && (lane == 0 || prv != bin));
            if (tail) {
                const unsigned below = heads & ((2u << lane) - 1u);
                atomicAdd(&s.hist[bin], lane - (31 - __clz(below)) + 1);
            }
        }
    });
    __syncthreads();
    // Greedy cut over the bins: a window grows while it holds <= capg
    // products; a bin above capg stands alone (dense above CAP), and the bin
    // after it starts a new window.  Every packed window thus fits the
    // capg-product tile.  With the bin prefix sums, each window's end is one
    // binary search (the largest e with pre[e] - pre[s] <= capg), so the walk
    // costs O(windows log bins) instead of a serial pass over every bin.
    constexpr int PB = (MAXBINS + PLAN_T - 1) / PLAN_T;
    {
        int loc[PB], run = 0;
#pragma unroll
        for (int j = 0; j < PB; ++j) {
            const int b = threadIdx.x * PB + j;
            loc[j] = b < nbins ? s.hist[b] : 0;
            run += loc[j];
        }
        int base;
        cub::BlockScan<int32_t, PLAN_T>(s.scan).ExclusiveSum(run, base);
#pragma unroll
        for (int j = 0; j < PB; ++j) {
            const int b = threadIdx.x * PB + j;
            if (b <= nbins) s.hist[b] = base;  // every thread read its bins before the scan
            base += loc[j];
        }
        if (threadIdx.x == PLAN_T - 1 && nbins == PB * PLAN_T) s.hist[nbins] = base;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint2* dd = desc + doff[hrow];
        const int32_t* pre = s.hist;
        int32_t nw = 0;
        int b = 0;
        while (b < nbins) {
            const int32_t c = pre[b + 1] - pre[b];
            int e = b + 1;
            if (c <= capg) {
                // largest e <= nbins with pre[e] <= pre[b] + capg
                const int32_t lim = pre[b] + capg;
                int lo = b + 1, hi = nbins;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (pre[mid] <= lim) lo = mid; else hi = mid - 1;
                }
                e = lo;
            }
            dd[nw++] = make_uint2(static_cast<uint32_t>(b << log_binw) | (c > CAP ? DENSE_BIT : 0u),
                                  static_cast<uint32_t>(pre[b]));
            b = e;
        }
        nwin[hrow] = nw;
        dd[nw] = make_uint2(static_cast<uint32_t>(m.ncols), static_cast<uint32_t>(pre[nbins]));
    }
}

// K2b: emit the Window records of each heavy row and its per-(window,
// segment) start table: starts[sofs + w*d + p] = number of elements of
// segment p lying in windows < w (one streaming pass over the row).
__global__ void __launch_bounds__(PLAN_T, 5) plan_write_kernel(
    Mats m, const int32_t* __restrict__ heavy, int32_t nbins, int log_binw,
    const int32_t* __restrict__ nwin, const int64_t* __restrict__ doff,
    const uint2* __restrict__ desc, const int64_t* __restrict__ win_off, Window* __restrict__ wins,
    uint8_t* __restrict__ win_cat, const int64_t* __restrict__ start_off, int64_t start_budget,
    uint32_t* __restrict__ starts, int bs_x4, BinSum bs) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PlanWriteShared& s = *reinterpret_cast<PlanWriteShared*>(smem_raw);
    const int32_t hrow = blockIdx.x;
    const int32_t row = heavy[hrow];
    const int wtot = nwin[hrow];
    const uint2* dd = desc + doff[hrow];
    for (int k = threadIdx.x; k <= wtot; k += PLAN_T) {
        const uint2 v = dd[k];
        s.u.w.wc0[k] = v.x;
        s.u.w.wpre[k] = static_cast<int32_t>(v.y);
    }
    __syncthreads();
    // bin -> window: the last window whose c0 <= the bin's first column
    for (int b = threadIdx.x; b < nbins; b += PLAN_T) {
        const uint32_t c = static_cast<uint32_t>(b) << log_binw;
        int lo = 0, hi = wtot - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((s.u.w.wc0[mid] & ~DENSE_BIT) <= c) lo = mid; else hi = mid - 1;
        }
        s.binwin[b] = static_cast<uint16_t>(lo);
    }
    const int64_t off = win_off[hrow];
    // rows past the table budget binary-search their segments instead
    const int64_t sofs = (starts != nullptr && start_off[hrow + 1] > start_off[hrow] &&
                          start_off[hrow + 1] <= start_budget)
                             ? start_off[hrow] : -1;
    for (int k = threadIdx.x; k < wtot; k += PLAN_T) {
        Window wd;
        wd.row = row;
        const bool dense = (s.u.w.wc0[k] & DENSE_BIT) != 0;
        wd.c0 = static_cast<int32_t>(s.u.w.wc0[k] & ~DENSE_BIT);
        int64_t c1 = int64_t{s.u.w.wc0[k + 1] & ~DENSE_BIT};
        if (dense) c1 = ::min(c1, int64_t{wd.c0} + WD);
        wd.c1 = static_cast<int32_t>(::min(c1, int64_t{m.ncols}));
        wd.first = static_cast<int32_t>(off);
        wd.wi = k;
        wd.nprod = s.u.w.wpre[k + 1] - s.u.w.wpre[k];
        wd.d = static_cast<int32_t>(m.arp[row + 1] - m.arp[row]);
        wd.pad_ = 0;
        wd.rs = m.arp[row];
        wd.sofs = sofs;
        wins[off + k] = wd;
        // sparse: the smallest tile class that holds the window; dense: NWCLS
        int cat = NWCLS;
        if (!dense) {
            cat = 0;
            while (cat + 1 < NWCLS && wd.nprod <= kWinCapDev[cat + 1]) ++cat;
        }
        win_cat[off + k] = static_cast<uint8_t>(cat);
    }
    if (sofs < 0) return;
    const int lane = threadIdx.x & 31;
    const int d = static_cast<int>(m.arp[row + 1] - m.arp[row]);
    const int64_t tsz = int64_t{wtot + 1} * d;
    // Rows with few windows: each interior boundary of each segment is a
    // binary search for the window's first column in that B row —
    // (windows - 1) x segments x log2(segment length) loads instead of
    // streaming every product's column a second time.
    {
        const int64_t P = s.u.w.wpre[wtot];
        const int lg = 1 + bit_length(static_cast<uint32_t>(P / ::max(d, 1)));
        if (int64_t{wtot - 1} * d * lg * 4 < P * bs_x4) {
            uint32_t* tab = starts + sofs;
            const int64_t rs = m.arp[row];
            for (int64_t t = threadIdx.x; t < tsz; t += PLAN_T) {
                const int w = static_cast<int>(t / d), p = static_cast<int>(t - int64_t{w} * d);
                const int32_t k = __ldg(m.acol + rs + p);
                const int64_t b0 = __ldg(m.brp + k), b1 = __ldg(m.brp + k + 1);
                int64_t e = b0;
                if (w == wtot) e = b1;
                else if (w > 0)
                    e = lower_bound_col(m.bcol, b0, b1,
                                        static_cast<int32_t>(s.u.w.wc0[w] & ~DENSE_BIT));
                tab[t] = static_cast<uint32_t>(e);
            }
            return;
        }
    }
    __syncthreads();  // wc0/wpre dead: the union becomes the staging area
    const bool staged = tsz <= STAGE;
    uint32_t* tab = staged ? s.u.stage : starts + sofs;
    // entries are absolute B offsets (segment start b0 + element index)
    if (bs.sptr) {
        // bin summaries: an entry's first element offset is the exclusive prefix
        // of the segment's run counts; windows starting in (previous entry's
        // window, this entry's window] start at that offset
        stream_summaries(m, bs, row, [&](int p, int q0, int nent, const uint32_t* ent,
                                         int& carryw, int& eoff, int64_t b0, int blen) {
#pragma unroll
            for (int u = 0; u < PLAN_U; ++u) {
                const int qb = q0 + 32 * u;
                if (qb >= nent) break;
                const bool valid = qb + lane < nent;
                const int cntv = valid ? static_cast<int>(ent[u] & 0xffffu) : 0;
                int incl = cntv;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                const int excl = eoff + incl - cntv;
                const int wq = valid ? s.binwin[ent[u] >> 16] : wtot;
                int wp = __shfl_up_sync(0xffffffffu, wq, 1);
                if (lane == 0) wp = carryw;
                if (valid)
                    for (int w2 = wp + 1; w2 <= wq; ++w2)
                        tab[w2 * int64_t{d} + p] = static_cast<uint32_t>(b0 + excl);
                carryw = __shfl_sync(0xffffffffu, wq, ::min(31, nent - 1 - qb));
                eoff += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (q0 + 32 * PLAN_U >= nent)
                for (int w2 = carryw + 1 + lane; w2 <= wtot; w2 += 32)
                    tab[w2 * int64_t{d} + p] = static_cast<uint32_t>(b0 + blen);
        });
    } else
    stream_segments(m, row, [&](int p, int q0, int len, const int32_t* cols, int& carry,
                                int64_t b0) {
        // carry: window of the element before this group (-1 at q0 == 0)
#pragma unroll
        for (int u = 0; u < PLAN_U; ++u) {
            const int qb = q0 + 32 * u;
            if (qb >= len) break;
            const int q = qb + lane;
            const int wq = cols[u] >= 0 ? s.binwin[cols[u] >> log_binw] : wtot;
            int wp = __shfl_up_sync(0xffffffffu, wq, 1);
            if (lane == 0) wp = carry;
            if (q < len)
                for (int w2 = wp + 1; w2 <= wq; ++w2)
                    tab[w2 * int64_t{d} + p] = static_cast<uint32_t>(b0 + q);
            carry = __shfl_sync(0xffffffffu, wq, ::min(31, len - 1 - qb));
        }
        // windows after the last element start at len
        if (q0 + 32 * PLAN_U >= len)
            for (int w2 = carry + 1 + lane; w2 <= wtot; w2 += 32)
                tab[w2 * int64_t{d} + p] = static_cast<uint32_t>(b0 + len);
    });
    if (staged) {
        __syncthreads();
        uint32_t* st = starts + sofs;
        for (int i = threadIdx.x; i < tsz; i += PLAN_T) st[i] = s.u.stage[i];
    }
}

// Upper bound on a heavy row's windows (+1 sentinel descriptor): any two
// consecutive greedy windows hold > capg products together, so
// nwin < 2P/capg + 2.
__global__ void plan_bound_kernel(const int32_t* __restrict__ heavy, int64_t nh, int64_t rb,
                                  const int64_t* __restrict__ prod, int32_t nbins,
                                  int32_t capg, int64_t* __restrict__ bound) {
    const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (t > nh) return;
    if (t == nh) {
        bound[t] = 0;
        return;
    }
    const int64_t P = prod[heavy[t] - rb];
    bound[t] = ::min(2 * (P / capg) + 3, int64_t{nbins}) + 1;
}

// Size of each heavy row's start table ((windows+1) x A-row length), or 0
// when it would exceed the per-row budget (those rows binary-search).
__global__ void start_size_kernel(Mats m, const int32_t* __restrict__ heavy, int64_t nh,
                                  const int32_t* __restrict__ nwin, int64_t per_row_cap,
                                  int64_t* __restrict__ sz) {
    const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (t > nh) return;
    if (t == nh) {
        sz[t] = 0;
        return;
    }
    const int32_t row = heavy[t];
    const int64_t d = m.arp[row + 1] - m.arp[row];
    const int64_t e = (int64_t{nwin[t]} + 1) * d;
    sz[t] = e <= per_row_cap ? e : 0;
}

// Window ids by category (sparse tile class 0..NWCLS-1, dense NWCLS):
// counts, then a scatter from per-category cursors (block-aggregated).
// (+ the products of each category: cnt[NWCLS + 1 + c])
__global__ void window_cat_count_kernel(const uint8_t* __restrict__ cat,
                                        const Window* __restrict__ wins, int64_t nw,
                                        unsigned long long* __restrict__ cnt) {
    __shared__ unsigned s_cnt[NWCLS + 1];
    __shared__ unsigned long long s_prod[NWCLS + 1];
    if (threadIdx.x <= NWCLS) {
        s_cnt[threadIdx.x] = 0;
        s_prod[threadIdx.x] = 0;
    }
    __syncthreads();
    const int64_t w = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (w < nw) {
        atomicAdd(&s_cnt[cat[w]], 1u);
        atomicAdd(&s_prod[cat[w]], static_cast<unsigned long long>(wins[w].nprod));
    }
    __syncthreads();
    if (threadIdx.x <= NWCLS && s_cnt[threadIdx.x]) {
        atomicAdd(&cnt[threadIdx.x], static_cast<unsigned long long>(s_cnt[threadIdx.x]));
        atomicAdd(&cnt[NWCLS + 1 + threadIdx.x], s_prod[threadIdx.x]);
    }
}

__global__ void split_windows_kernel(const uint8_t* __restrict__ cat, int64_t nw,
                                     unsigned long long* __restrict__ cursor,
                                     int32_t* __restrict__ sparse_ids,
                                     int32_t* __restrict__ dense_ids) {
    __shared__ unsigned s_cnt[NWCLS + 1];
    __shared__ unsigned long long s_base[NWCLS + 1];
    if (threadIdx.x <= NWCLS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t w = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    int d = 0;
    unsigned rank = 0;
    if (w < nw) {
        d = cat[w];
        rank = atomicAdd(&s_cnt[d], 1u);
    }
    __syncthreads();
    if (threadIdx.x <= NWCLS) s_base[threadIdx.x] = atomicAdd(&cursor[threadIdx.x], s_cnt[threadIdx.x]);
    __syncthreads();
    if (w < nw) (d == NWCLS ? dense_ids : sparse_ids)[s_base[d] + rank] = static_cast<int32_t>(w);
}

// Sort key of a window list: its first column (windows launched in column
// order share B's column slices in L2 across heavy rows).
__global__ void window_c0_kernel(const Window* __restrict__ wins, const int32_t* __restrict__ ids,
                                 int64_t n, uint32_t* __restrict__ keys) {
    const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (i < n) keys[i] = static_cast<uint32_t>(wins[ids[i]].c0);
}


// K3': merge-based exact numeric tile and hash-count symbolic tile
// ---------------------------------------------------------------------------
template <int T, int CAPM>
__global__ void __launch_bounds__(T, CAPM == 3072 ? 3 : (T >= 256 ? (CAPM <= 2048 ? 4 : 2) : (T == 128 ? 8 : (T == 64 ? 16 : 32)))) esc_merge_kernel(Mats m, const int32_t* __restrict__ ids,
                                                      const Window* __restrict__ wins, OutCtx out, int csort) {
    using S = MergeShared<T, CAPM>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    const int tid = threadIdx.x;
    const int32_t id = ids[blockIdx.x];
    int32_t row, c0, c1, w = -1;
    int64_t wsofs = -1, wrs = -1, wdn = 0;
    int wwi = 0;
    if (wins) {
        w = id;
        const Window wd = wins[w];
        row = wd.row;
        c0 = wd.c0;
        c1 = wd.c1;
        wsofs = wd.sofs;
        wwi = wd.wi;
        wrs = wd.rs;
        wdn = wd.d;
    } else {
        row = id;
        c0 = 0;
        c1 = m.ncols;
    }
    const int total =
        expand_runs<T, CAPM, true>(m, row, c0, c1, wins == nullptr, s, wsofs, wwi, wrs, wdn,
                                   /*defer=*/true);
    const int b = sort_tile<T, CAPM>(s, total, static_cast<uint32_t>(c1 - c0), csort, 0, false, c0);
    (void)tid;
    int64_t base = out.crp[row - out.row_begin];
    if (w >= 0) base += out.win_scan[w] - out.win_scan[wins[w].first];
    reduce_and_write<T, CAPM>(s, b, total, static_cast<uint32_t>(c0), out.ccol + base,
                              out.cval + base);
}

// Window numeric tile without a symbolic pass (the main window class): the
// windows of the list (ordered as their rows and columns are laid out in C)
// are claimed in list order; each tile counts its distinct columns after the
// sort, takes its offset among the list's windows from a decoupled look-back,
// and its output lands at
//   known(row, w) + U(w),
// known = the output offset from every unit counted beforehand (light rows and
// the other window classes: out.crp / out.win_scan scanned with this list's
// windows at 0) and U(w) = the outputs of this list's windows placed before w.
// It records its count (win_nnz, row_nnz) so the final row_ptr / window scan
// — computed after this kernel — places everything else consistently.
// Replaces the symbolic count of these windows (spgemm.hpp:41-63 fused into
// :70-106): their columns are gathered once instead of twice.
//
// A tile publishes its count right after the head scan and forms its run
// sums before the look-back, so the wait for predecessors still sorting
// overlaps that work (measured on cfg5: 175 ms for the class vs 137 ms
// numeric + 60 ms symbolic before).  Rejected (measured): persistent CTAs
// placing each tile one tile later from an L2 stash (look-back 2.4K instead of
// 6.6K cycles per tile, but register spills and the stash copy: 211-230 ms).
template <int T, int CAPM>
__global__ void __launch_bounds__(T, CAPM <= 2048 ? 4 : 2) esc_window_lb_kernel(
    Mats m, const int32_t* __restrict__ ids, const Window* __restrict__ wins, OutCtx out,
    int csort, LbCtx lb) {
    using S = MergeShared<T, CAPM>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    __shared__ int s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(lb.counter, 1);
    __syncthreads();
    const int t = s_tile;
#ifdef BSP_X_PHASE
    const int32_t w = ids[t];
    const Window wd = wins[w];
    if (threadIdx.x == 0) {
        const int b = blockIdx.x & ((1 << 22) - 1);
        g_phase_last[b] = g_phase_t0[b] = clock64();
        g_phase_cls[b] = wd.d <= 256 ? 0 : (wd.d <= 512 ? 1 : (wd.d <= 1024 ? 2 : (wd.d <= 2048 ? 3 : (wd.d <= 4096 ? 4 : 5))));
        atomicAdd(&g_phase[0], 1ull);
    }
#else
    const int32_t w = ids[t];
    const Window wd = wins[w];
#endif
    const int total = expand_runs<T, CAPM, true>(m, wd.row, wd.c0, wd.c1, false, s, wd.sofs, wd.wi,
                                                 wd.rs, wd.d, /*defer=*/true);
    const int b = sort_tile<T, CAPM>(s, total, static_cast<uint32_t>(wd.c1 - wd.c0), csort, 0, false,
                                     wd.c0);
    const int64_t r = wd.row - out.row_begin;
    const int64_t known = out.crp[r] + out.win_scan[w] - out.win_scan[wd.first];
    const int cnt = reduce_and_write<T, CAPM, true>(
        s, b, total, static_cast<uint32_t>(wd.c0), out.ccol + known, out.cval + known,
        [&](int agg) { lookback_publish(lb.status, t, agg); },
        [&](int agg) { return lookback_warp(lb.status, t, agg); });
    if (threadIdx.x == 0) {
        out.win_nnz[w] = cnt;
        atomicAdd(reinterpret_cast<unsigned long long*>(&out.row_nnz[r]),
                  static_cast<unsigned long long>(cnt));
#ifdef BSP_X_PHASE
        g_phase_last[blockIdx.x & ((1 << 22) - 1)] = 0;
#endif
    }
}

// Look-back window tile, second form: only the columns are gathered before the
// sort; the values are fetched — in sorted order — after the tile has published
// its count (expand_keys / reduce_lb2).  A tile's count does not depend on the
// values, so the value gather, the a*b products and the run sums all overlap
// the wait for the predecessors' counts (measured on cfg5 with the first form:
// 20 % of every tile's residency was that wait, and 21 % the combined gather).
// Bit-identical output: each run's products are summed in ascending k as before.
// COMPACT: 6 bytes per product in the value buffer (32-bit B offset, 16-bit
// segment index: rows of at most 65535 entries) and 4-bit radix digits in the
// fallback sort: 44.9 KB per tile, 5 CTAs per SM at 48 registers (the tile is
// latency bound: 2 / 3 / 4 CTAs per SM measured 265.8 / 198.5 / 169.2 ms).
template <int T, int CAPM, bool COMPACT>
struct LbTileShared {
    using type = std::conditional_t<COMPACT, MergeShared<T, CAPM, 6 * CAPM, 4>, MergeShared<T, CAPM>>;
};
template <int T, int CAPM, bool COMPACT>
__global__ void __launch_bounds__(T, COMPACT ? 5 : 4) esc_window_lb2_kernel(
    Mats m, const int32_t* __restrict__ ids, const Window* __restrict__ wins, OutCtx out,
    int csort, LbCtx lb) {
    using S = typename LbTileShared<T, CAPM, COMPACT>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    __shared__ int s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(lb.counter, 1);
    __syncthreads();
    const int t = s_tile;
    // ids == nullptr: `wins` is the list's windows gathered in list order (one
    // dependent load less at the start of every tile), the window id in pad_
    const Window wd = ids ? wins[ids[t]] : wins[t];
    const int32_t w = ids ? ids[t] : wd.pad_;
#ifdef BSP_X_PHASE
    if (threadIdx.x == 0) {
        const int b = blockIdx.x & ((1 << 22) - 1);
        g_phase_last[b] = g_phase_t0[b] = clock64();
        g_phase_cls[b] = wd.d <= 256 ? 0 : (wd.d <= 512 ? 1 : (wd.d <= 1024 ? 2 : (wd.d <= 2048 ? 3 : (wd.d <= 4096 ? 4 : 5))));
        atomicAdd(&g_phase[0], 1ull);
    }
#endif
    const int total = expand_keys<T, CAPM>(m, wd.c0, wd.c1, s, wd.sofs, wd.wi, wd.rs, wd.d);
    const int b = sort_tile<T, CAPM>(s, total, static_cast<uint32_t>(wd.c1 - wd.c0), csort, 0, false,
                                     wd.c0);
    if (b == 1) {  // merged runs end in buffer 1 (rare): the reduction reads buffer 0
        for (int e = threadIdx.x; e < total; e += T) {
            s.key0[PADI(e)] = s.u.m.key1[PADI(e)];
            s.idx0[PADI(e)] = s.u.m.idx1[PADI(e)];
        }
        __syncthreads();
    }
    const int64_t r = wd.row - out.row_begin;
    const int64_t known = out.crp[r] + out.win_scan[w] - out.win_scan[wd.first];
    const int cnt = reduce_lb2<T, CAPM>(
        s, total, static_cast<uint32_t>(wd.c0), out.ccol + known, out.cval + known,
        m.aval + wd.rs, m.bval, [&](int agg) { lookback_publish(lb.status, t, agg); },
        [&](int agg) { return lookback_warp(lb.status, t, agg); });
    if (threadIdx.x == 0) {
        out.win_nnz[w] = cnt;
        atomicAdd(reinterpret_cast<unsigned long long*>(&out.row_nnz[r]),
                  static_cast<unsigned long long>(cnt));
#ifdef BSP_X_PHASE
        g_phase_last[blockIdx.x & ((1 << 22) - 1)] = 0;
#endif
    }
}

constexpr int pow2_ceil(int x) { return x <= 1 ? 1 : 2 * pow2_ceil((x + 1) / 2); }

template <int T, int CAPM, bool STAGED = true, int TSM = 2>
struct HashShared {
    static constexpr int TS = pow2_ceil(TSM * CAPM);  // open-addressing slots (power of two)
    alignas(16) int32_t table[TS];
    int32_t stage[STAGED ? CAPM : 1];  // gathered columns of the current chunk
    typename cub::BlockReduce<int32_t, T>::TempStorage red;
    typename cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>::TempStorage scan;
    int64_t pstart[T];
    int32_t poff[T + 1];
};

// Distinct output columns of (row, [c0,c1)) with <= CAPM products.
// STAGED: the chunk's columns are first gathered into smem with cp.async
// (warp-contiguous, all loads in flight), then hashed from smem.
template <int T, int CAPM, bool STAGED, int TSM = 2>
__global__ void __launch_bounds__(T) hash_count_kernel(Mats m, const int32_t* __restrict__ ids,
                                                       const Window* __restrict__ wins,
                                                       OutCtx out) {
    using S = HashShared<T, CAPM, STAGED, TSM>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    const int tid = threadIdx.x;
    constexpr int NW = T / 32;
    constexpr int TS = S::TS;
    constexpr int LG = 31 - __builtin_clz(static_cast<unsigned>(TS));
    const int32_t id = ids[blockIdx.x];
    int32_t row, c0, c1, w = -1;
    int64_t wsofs = -1, rs, re;
    int wwi = 0;
    if (wins) {
        w = id;
        const Window wd = wins[w];
        row = wd.row;
        c0 = wd.c0;
        c1 = wd.c1;
        wsofs = wd.sofs;
        wwi = wd.wi;
        rs = wd.rs;
        re = wd.rs + wd.d;
    } else {
        row = id;
        c0 = 0;
        c1 = m.ncols;
        rs = m.arp[row];
        re = m.arp[row + 1];
    }
    const bool full = wins == nullptr;
    static_assert(TS % (4 * T) == 0, "table init is int4-wide");
    for (int e = 4 * tid; e < TS; e += 4 * T)
        *reinterpret_cast<int4*>(&s.table[e]) = make_int4(-1, -1, -1, -1);
    int cnt = 0;
    for (int64_t pc = rs; pc < re; pc += T) {
        const int64_t p = pc + tid;
        int len = 0;
        int64_t start = 0;
        if (p < re) {
            int64_t b0, b1;
            segment_range(m, full, wsofs, wwi, p, rs, re - rs, c0, c1, b0, b1);
            start = b0;
            len = static_cast<int>(b1 - b0);
        }
        // compact the chunk's non-empty segments, then each thread inserts a
        // contiguous range of the chunk's products
        const int packed = len | ((len > 0) << 16);
        int off, agg;
        __syncthreads();
        cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(packed, off, agg);
        if (len > 0) {
            s.pstart[off >> 16] = start;
            s.poff[off >> 16] = off & 0xffff;
        }
        const int nr = agg >> 16, ct = agg & 0xffff;
        if (tid == 0) s.poff[nr] = ct;
        __syncthreads();
        auto insert = [&](int32_t col) {
            uint32_t hsl = col_hash(static_cast<uint32_t>(col), LG);
            for (;;) {
                const int32_t prev = atomicCAS(&s.table[hsl], -1, col);
                if (prev == -1) {
                    ++cnt;
                    break;
                }
                if (prev == col) break;
                hsl = (hsl + 1) & (TS - 1);
            }
        };
        if constexpr (STAGED) {
            int e0, we, qa;
            warp_slice(s.poff, nr, ct, T / 32, e0, we, qa);
            for (; e0 < we; e0 += 32) {
                const int q = warp_runs(s.poff, nr, e0, qa);
                const int e = e0 + (threadIdx.x & 31);
                if (e < we) cp_async4(&s.stage[e], m.bcol + s.pstart[q] + (e - s.poff[q]));
            }
            cp_async_wait_all();
            __syncthreads();
            for (int e2 = tid; e2 < ct; e2 += T) insert(s.stage[e2]);
        } else {
            // each thread inserts a contiguous range of the chunk's products
            const int E = (ct + T - 1) / T;
            int e = min(ct, tid * E);
            const int ee = min(ct, e + E);
            if (e < ee) {
                int q = find_run(s.poff, nr, run_search_step(nr), e);
                while (e < ee) {
                    while (s.poff[q + 1] <= e) ++q;
                    const int stop = min(ee, s.poff[q + 1]);
                    const int64_t base = s.pstart[q] - s.poff[q];
                    for (; e < stop; ++e) insert(__ldg(m.bcol + base + e));
                }
            }
        }
    }
    const int tot = cub::BlockReduce<int32_t, T>(s.red).Sum(cnt);
    if (tid == 0) {
        if (w >= 0) {
            out.win_nnz[w] = tot;
            atomicAdd(reinterpret_cast<unsigned long long*>(&out.row_nnz[row - out.row_begin]),
                      static_cast<unsigned long long>(tot));
        } else {
            out.row_nnz[row - out.row_begin] = tot;
        }
    }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// K4: dense window kernel (heavy windows, width <= WD, any product count)
// ---------------------------------------------------------------------------
constexpr int DT = 256;
// products per sorted batch (1024: the tile fits 4 CTAs/SM)
constexpr int DCAP = 1024;
constexpr int DI = DCAP / DT;

template <bool NUMERIC>
struct DenseSharedT {
    using Sort = cub::BlockRadixSort<uint32_t, DT, DI, uint16_t>;
    using Scan = cub::BlockScan<int32_t, DT>;
    static constexpr int NV = NUMERIC ? 1 : 0;  // the symbolic pass keeps only the bitmap
    double acc[NUMERIC ? WD : 1];
    uint32_t bitmap[WD / 32];
    uint32_t keys[NUMERIC ? DCAP : 1];
    double vals[NUMERIC ? DCAP : 1];
    union {
        typename Sort::TempStorage sort;
        uint16_t sidx[DCAP];
    } u;
    typename Scan::TempStorage scan;
    int64_t pstart[DT];
    int32_t plen[DT];
    int32_t poff[DT];
    double pav[DT];
};

// One batch of n products (k order) of a dense window: stable sort by column
// (12-bit keys; the pad WD-1 sits after the n real entries), then every run of
// equal columns is added to its accumulator left to right.
template <class SD>
__device__ __forceinline__ void dense_batch(SD& s, int n) {
    const int tid = threadIdx.x;
    uint32_t k[DI];
    uint16_t v[DI];
#pragma unroll
    for (int i = 0; i < DI; ++i) {
        const int e = tid * DI + i;
        k[i] = e < n ? s.keys[e] : static_cast<uint32_t>(WD - 1);
        v[i] = static_cast<uint16_t>(e);
    }
    __syncthreads();
    typename SD::Sort(s.u.sort).Sort(k, v, 0, LOG_WD);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < DI; ++i) {
        s.keys[tid * DI + i] = k[i];
        s.u.sidx[tid * DI + i] = v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < DI; ++i) {
        const int e0 = tid * DI + i;
        if (e0 < n && (e0 == 0 || s.keys[e0 - 1] != k[i])) {
            double acc = s.acc[k[i]];
            int e = e0;
            do {
                acc = __dadd_rn(acc, s.vals[s.u.sidx[e]]);
                ++e;
            } while (e < n && s.keys[e] == k[i]);
            s.acc[k[i]] = acc;
            atomicOr(&s.bitmap[k[i] >> 5], 1u << (k[i] & 31));
        }
    }
    __syncthreads();
}

template <bool NUMERIC>
__global__ void __launch_bounds__(DT, 4) dense_window_kernel(Mats m, const int32_t* __restrict__ ids,
                                                          const Window* __restrict__ wins,
                                                          OutCtx out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SD = DenseSharedT<NUMERIC>;
    SD& s = *reinterpret_cast<SD*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = DT / 32;
    const int32_t w = ids[blockIdx.x];
    const Window wd = wins[w];
    const int32_t row = wd.row, c0 = wd.c0, c1 = wd.c1;
    for (int e = tid; e < WD / 32; e += DT) s.bitmap[e] = 0u;
    if (NUMERIC)
        for (int e = tid; e < WD; e += DT) s.acc[e] = 0.0;
    __syncthreads();
    const int64_t rs = wd.rs, re = wd.rs + wd.d;
    int fill = 0;  // products in the current batch (block-uniform)
    for (int64_t pc = rs; pc < re; pc += DT) {
        const int64_t p = pc + tid;
        int len = 0;
        int64_t start = 0;
        double av = 0.0;
        if (p < re) {
            int64_t b0, b1;
            segment_range(m, false, wd.sofs, wd.wi, p, rs, re - rs, c0, c1, b0, b1);
            start = b0;
            len = static_cast<int>(b1 - b0);
            if (NUMERIC) av = __ldg(m.aval + p);
        }
        int off, chunk;
        typename SD::Scan(s.scan).ExclusiveSum(len, off, chunk);
        s.pstart[tid] = start;
        s.plen[tid] = len;
        s.poff[tid] = off;
        s.pav[tid] = av;
        __syncthreads();
        const int nslots = static_cast<int>(::min(int64_t{DT}, re - pc));
        if (!NUMERIC) {
            // 4 column loads in flight per lane, then their bitmap bits
            for (int slot = warp; slot < nslots; slot += NW) {
                const int l = s.plen[slot];
                const int64_t st = s.pstart[slot];
                for (int q0 = 0; q0 < l; q0 += 128) {
                    int32_t col[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = q0 + 32 * u + lane;
                        col[u] = q < l ? __ldg(m.bcol + st + q) : -1;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (col[u] < 0) continue;
                        const uint32_t c = static_cast<uint32_t>(col[u] - c0);
                        atomicOr(&s.bitmap[c >> 5], 1u << (c & 31));
                    }
                }
            }
            __syncthreads();
            continue;
        }
        // NUMERIC: the chunk's products are appended, in (k, j) order, to the
        // current batch; a full batch (or the last one) is sorted and added.
        for (int cpos = 0; cpos < chunk;) {
            const int take = min(chunk - cpos, DCAP - fill);
            for (int slot = warp; slot < nslots; slot += NW) {
                const int o = s.poff[slot], l = s.plen[slot];
                const int lo = max(o, cpos), hi = min(o + l, cpos + take);
                if (lo >= hi) continue;
                const int64_t st = s.pstart[slot] + (lo - o);
                const double a = s.pav[slot];
                const int dst = fill + (lo - cpos);
                const int cnt = hi - lo;
                for (int q0 = 0; q0 < cnt; q0 += 128) {  // 4 (col, val) loads in flight
                    int32_t cv[4];
                    double bv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = q0 + 32 * u + lane;
                        cv[u] = q < cnt ? __ldg(m.bcol + st + q) : 0;
                        bv[u] = q < cnt ? __ldg(m.bval + st + q) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int q = q0 + 32 * u + lane;
                        if (q >= cnt) break;
                        s.keys[dst + q] = static_cast<uint32_t>(cv[u] - c0);
                        s.vals[dst + q] = __dmul_rn(a, bv[u]);
                    }
                }
            }
            fill += take;
            cpos += take;
            if (fill == DCAP) {
                __syncthreads();
                dense_batch(s, DCAP);
                fill = 0;
            }
        }
        __syncthreads();  // slot arrays are rewritten by the next chunk
    }
    if (NUMERIC && fill > 0) {
        __syncthreads();
        dense_batch(s, fill);
    }
    // Bitmap -> count (and sorted output).
    constexpr int NWORD = WD / 32;  // 128 <= DT
    const uint32_t word = tid < NWORD ? s.bitmap[tid] : 0u;
    const int pc = __popc(word);
    int woff, tot;
    typename SD::Scan(s.scan).ExclusiveSum(pc, woff, tot);
    if (!NUMERIC) {
        if (tid == 0) {
            out.win_nnz[w] = tot;
            atomicAdd(reinterpret_cast<unsigned long long*>(&out.row_nnz[row - out.row_begin]),
                      static_cast<unsigned long long>(tot));
        }
        return;
    }
    const int64_t base = out.crp[row - out.row_begin] + out.win_scan[w] - out.win_scan[wd.first];
    // sorted output: word t of the bitmap holds columns 32t..32t+31; its
    // entries start at woff (the batch buffers may be smaller than WD, so the
    // output is not staged)
    uint32_t wbits = word;
    int64_t r = base + woff;
    while (wbits) {
        const int b = __ffs(wbits) - 1;
        wbits &= wbits - 1;
        const uint32_t c = static_cast<uint32_t>(tid * 32 + b);
        out.ccol[r] = static_cast<int32_t>(c + static_cast<uint32_t>(c0));
        out.cval[r] = s.acc[c];
        ++r;
    }
}

// ---------------------------------------------------------------------------
// K5: narrow B (ncols <= NARROW, e.g. the tall-skinny frontier operands of
// frontier.hpp:20-77): one warp per row with a dense accumulator of ncols
// doubles in shared memory.  The row's segments are walked in k order; a
// segment's entries have distinct columns, so its lanes add them in parallel,
// and __syncwarp between segments keeps every column's additions in
// ascending k from 0.0 — the reference's order, bit-exact, with no planning
// and no sort.  Symbolic counts the touched columns.
// ---------------------------------------------------------------------------
constexpr int NARROW = 256;
constexpr int NARROW_WARPS = 8;

template <bool NUMERIC>
__global__ void __launch_bounds__(NARROW_WARPS * 32)
    narrow_kernel(Mats m, int64_t rb, int64_t n, int32_t ncols, int64_t* __restrict__ row_nnz,
                  const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                  double* __restrict__ cval, unsigned long long* __restrict__ products) {
    __shared__ double s_acc[NUMERIC ? NARROW_WARPS : 1][NUMERIC ? NARROW : 1];
    __shared__ uint32_t s_touch[NARROW_WARPS][NARROW / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* acc = s_acc[NUMERIC ? warp : 0];
    uint32_t* touch = s_touch[warp];
    const int nwords = (ncols + 31) >> 5;
    unsigned long long prod = 0;
    for (int64_t r = blockIdx.x * int64_t{NARROW_WARPS} + warp; r < n;
         r += int64_t{gridDim.x} * NARROW_WARPS) {
        const int64_t row = rb + r;
        if (NUMERIC)
            for (int j = lane; j < ncols; j += 32) acc[j] = 0.0;
        if (lane < nwords) touch[lane] = 0u;
        __syncwarp();
        const int64_t rs = m.arp[row], re = m.arp[row + 1];
        for (int64_t pb = rs; pb < re; pb += 32) {
            const int64_t p = pb + lane;
            int64_t b0 = 0;
            int len = 0;
            double a = 0.0;
            if (p < re) {
                const int32_t k = __ldg(m.acol + p);
                b0 = __ldg(m.brp + k);
                len = static_cast<int>(__ldg(m.brp + k + 1) - b0);
                if (NUMERIC) a = __ldg(m.aval + p);
            }
            // non-empty segments only, in k order (frontier rows are mostly empty)
            unsigned ne = __ballot_sync(0xffffffffu, len > 0);
            while (ne) {
                const int j = __ffs(ne) - 1;
                ne &= ne - 1;
                const int64_t sj = __shfl_sync(0xffffffffu, b0, j);
                const int lj = __shfl_sync(0xffffffffu, len, j);
                const double aj = __shfl_sync(0xffffffffu, a, j);
                prod += static_cast<unsigned long long>(lane == 0 ? lj : 0);
                for (int q = lane; q < lj; q += 32) {
                    const int32_t c = __ldg(m.bcol + sj + q);
                    if (NUMERIC)
                        acc[c] = __dadd_rn(acc[c], __dmul_rn(aj, __ldg(m.bval + sj + q)));
                    atomicOr(&touch[c >> 5], 1u << (c & 31));
                }
                __syncwarp();
            }
        }
        if (!NUMERIC) {
            int cnt = lane < nwords ? __popc(touch[lane]) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (lane == 0) row_nnz[r] = cnt;
        } else {
            int64_t pos = crp[r];
            for (int wd = 0; wd < nwords; ++wd) {
                const uint32_t bits = touch[wd];
                if ((bits >> lane) & 1u) {
                    const int64_t o = pos + __popc(bits & ((1u << lane) - 1u));
                    ccol[o] = wd * 32 + lane;
                    cval[o] = acc[wd * 32 + lane];
                }
                pos += __popc(bits);
            }
        }
        __syncwarp();
    }
    if (!NUMERIC && lane == 0 && prod) atomicAdd(products, prod);
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------

template <int T, int CAPM, bool NUMERIC>
void launch_tile(bsp_handle h, const Mats& m, const int32_t* ids, int64_t n, const Window* wins,
                 const OutCtx& out) {
    if (n <= 0) return;
    if (NUMERIC) {
        using S = MergeShared<T, CAPM>;
        auto k = esc_merge_kernel<T, CAPM>;
        static const std::string nm_row = "esc_merge<" + std::to_string(T) + "," +
                                          std::to_string(CAPM) + ">";
        static const std::string nm_win = "esc_merge<" + std::to_string(T) + "," +
                                          std::to_string(CAPM) + ",win>";
        const std::string& nm = wins ? nm_win : nm_row;
        // BSP_CSORT=0: radix/merge only (no counting sort)
        static const int csort = [] {
            const char* e = std::getenv("BSP_CSORT");
            return e ? std::atoi(e) : 1000;
        }();
        set_smem(k, sizeof(S));
        BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(S), m, ids, wins, out,
                      csort);
    } else {
        static const std::string nm_row = "hash_count<" + std::to_string(T) + "," +
                                          std::to_string(CAPM) + ">";
        static const std::string nm_win = "hash_count<" + std::to_string(T) + "," +
                                          std::to_string(CAPM) + ",win>";
        const std::string& nm = wins ? nm_win : nm_row;
        // BSP_HASH=plain: insert straight from the loads (no staging)
        static const bool staged = [] {
            const char* e = std::getenv("BSP_HASH");
            return !(e && std::string(e) == "plain");
        }();
        // Table slots per product: 4 for heavy-row windows (fewer probe
        // collisions, measured 3 ms faster on cfg5 than 2 at 5 instead of 8
        // CTAs/SM); BSP_HTS / BSP_HTSL (light rows <= 2048 products) = 2 or 4.
        static const int hts_win = [] {
            const char* e = std::getenv("BSP_HTS");
            return e ? std::atoi(e) : 4;
        }();
        static const int hts_light = [] {
            const char* e = std::getenv("BSP_HTSL");
            return e ? std::atoi(e) : 2;
        }();
        if (staged && CAPM <= 2048 && (wins ? hts_win : hts_light) == 4) {
            using S = HashShared<T, CAPM, true, 4>;
            auto k = hash_count_kernel<T, CAPM, true, 4>;
            set_smem(k, sizeof(S));
            BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(S), m, ids, wins,
                          out);
        } else if (staged) {
            using S = HashShared<T, CAPM, true>;
            auto k = hash_count_kernel<T, CAPM, true>;
            set_smem(k, sizeof(S));
            BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(S), m, ids, wins,
                          out);
        } else {
            using S = HashShared<T, CAPM, false>;
            auto k = hash_count_kernel<T, CAPM, false>;
            set_smem(k, sizeof(S));
            BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(S), m, ids, wins,
                          out);
        }
    }
}

template <bool NUMERIC>
void launch_light(bsp_handle h, int cls, const Mats& m, const int32_t* ids, int64_t n,
                  const OutCtx& out) {
    switch (cls) {
        case 1: launch_tile<32, 128, NUMERIC>(h, m, ids, n, nullptr, out); break;
        case 2: launch_tile<64, 512, NUMERIC>(h, m, ids, n, nullptr, out); break;
        case 3: launch_tile<128, 1024, NUMERIC>(h, m, ids, n, nullptr, out); break;
        case 4: launch_tile<256, 2048, NUMERIC>(h, m, ids, n, nullptr, out); break;
        case 5: launch_tile<256, 3072, NUMERIC>(h, m, ids, n, nullptr, out); break;
        case 6: launch_tile<256, 4096, NUMERIC>(h, m, ids, n, nullptr, out); break;
        default: break;
    }
}

template <bool NUMERIC>
void launch_dense(bsp_handle h, const Mats& m, const int32_t* ids, int64_t n, const Window* wins,
                  const OutCtx& out) {
    if (n <= 0) return;
    auto k = dense_window_kernel<NUMERIC>;
    set_smem(k, sizeof(DenseSharedT<NUMERIC>));
    BSP_LAUNCH_AS(h, NUMERIC ? "dense_window_numeric" : "dense_window_symbolic", k,
                  static_cast<unsigned>(n), DT, sizeof(DenseSharedT<NUMERIC>), m, ids, wins, out);
}

}  // namespace

Mats make_mats(const bsp_csr* A, const bsp_csr* B) {
    Mats m{A->row_ptr, A->col_idx, A->values, B->row_ptr, B->col_idx, B->values,
           static_cast<int32_t>(B->ncols)};
    m.bnnz = B->nnz;
    m.bnrows = B->nrows;
    return m;
}

template <bool NUMERIC>
void run_light(bsp_handle h, const Mats& m, const RowwisePlan& plan, const OutCtx& out);

// Ascending sort of a device id list in place (CUB radix sort on the id bits).
void sort_ids(bsp_handle h, int32_t* ids, int64_t n) {
    if (n <= 1) return;
    DBuf<int32_t> tmp(h, n);
    size_t bytes = 0;
    BSP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, ids, tmp.p, n, 0, 31, h->stream));
    DBuf<uint8_t> t(h, static_cast<int64_t>(bytes));
    BSP_CUDA(cub::DeviceRadixSort::SortKeys(t.p, bytes, ids, tmp.p, n, 0, 31, h->stream));
    ++h->launches;
    BSP_CUDA(cudaMemcpyAsync(ids, tmp.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, h->stream));
}

void build_plan(bsp_handle h, const Mats& m, int64_t rb, int64_t re,
                       const uint8_t* skip, RowwisePlan& plan, int64_t* prod_out,
                       int64_t* early_row_nnz, RowwisePlan* shadow) {
    const int64_t n = re - rb;
    plan.rb = rb;
    plan.n = n;
    if (!prod_out) {
        plan.prod = DBuf<int64_t>(h, n);
        prod_out = plan.prod.p;
    }
    const int ncl = shadow ? 2 * NCLS : NCLS;  // shadow: skipped rows' own classes
    DBuf<uint8_t> cls(h, n);
    DBuf<int64_t> counters(h, 2 * ncl + 1);
    BSP_CUDA(cudaMemsetAsync(counters.p, 0, (2 * ncl + 1) * sizeof(int64_t), h->stream));
    const int grid = static_cast<int>(std::min<int64_t>(div_up(std::max<int64_t>(n, 1), 8),
                                                        int64_t{h->sm_count} * 8));
    // BSP_HEAVY_ABOVE: rows with more products are planned into column windows
    // (the shadow plan's rows stay light up to the largest row tile, 4096).
    // Measured on cfg5 with the 5-CTA look-back tile: 273.8 / 270.2 / 271.0 /
    // 274.4 ms at 4096 / 3072 / 2048 / 1024 — the 4096-product row tile (2 CTAs
    // per SM, plus its symbolic pass) loses to windows on the look-back tile.
    static const int heavy_above = [] {
        const char* e = std::getenv("BSP_HEAVY_ABOVE");
        const int v = e ? std::atoi(e) : 3072;
        return v >= 128 && v <= 4096 ? v : 4096;
    }();
    BSP_LAUNCH(h, products_kernel, grid, 256, 0, m, rb, n, prod_out, cls.p, skip, counters.p,
               counters.p + ncl, shadow ? 1 : 0,
               reinterpret_cast<unsigned long long*>(counters.p + 2 * ncl),
               shadow ? 4096 : heavy_above);
    int64_t hc[4 * NCLS + 1];
    d2h(h, hc, counters.p, 2 * ncl + 1);
    sync(h);
    // the heavy-row planner keeps per-row product prefixes in 32 bits
    require(hc[2 * ncl] < (int64_t{1} << 31) - 1,
            "spgemm: a row with >= 2^31 intermediate products is not supported (split A's row)");
    if (shadow) {  // rows of the skip mask, planned apart (light rows only)
        require(hc[NCLS + NCLS - 1] == 0, "build_plan: shadow rows must be light");
        shadow->rb = rb;
        shadow->n = n;
        int64_t t = 0;
        for (int c = 0; c < NCLS; ++c) {
            shadow->class_count[c] = c == 0 ? 0 : hc[NCLS + c];
            shadow->class_products[c] = c == 0 ? 0 : hc[ncl + NCLS + c];
            shadow->class_off[c] = t;
            if (c > 0) t += hc[NCLS + c];
        }
        shadow->class_off[NCLS] = t;
        shadow->lists = DBuf<int32_t>(h, t);
        for (int c = 0; c < NCLS; ++c) hc[NCLS + c] = hc[ncl + c];  // products of plan rows
    }
    int64_t tot_listed = 0;
    for (int c = 0; c < NCLS; ++c) {
        plan.class_count[c] = hc[c];
        plan.class_products[c] = hc[NCLS + c];
        plan.class_off[c] = (c == 0) ? 0 : tot_listed;
        if (c > 0) tot_listed += hc[c];
    }
    plan.class_off[NCLS] = tot_listed;
    h->stats.products = 0;
    for (int c = 0; c < NCLS; ++c) h->stats.products += plan.class_products[c];
    plan.lists = DBuf<int32_t>(h, tot_listed);
    const int64_t tot_shadow = shadow ? shadow->class_off[NCLS] : 0;
    if (tot_listed + tot_shadow > 0) {
        DBuf<unsigned long long> cursor(h, 2 * NCLS);
        std::vector<unsigned long long> cur(2 * NCLS, 0);
        for (int c = 1; c < NCLS; ++c) {
            cur[c] = static_cast<unsigned long long>(plan.class_off[c]);
            if (shadow) cur[NCLS + c] = static_cast<unsigned long long>(shadow->class_off[c]);
        }
        h2d(h, cursor.p, cur.data(), 2 * NCLS);
        BSP_LAUNCH(h, bucket_kernel, static_cast<unsigned>(div_up(n, 256)), 256, 0, cls.p, rb, n,
                   cursor.p, plan.lists.p, shadow ? shadow->lists.p : nullptr);
    }
    // The light rows' symbolic does not depend on the heavy-row plan: run it
    // on the side stream while the (latency-bound) planner runs here;
    // plan_symbolic joins it.
    // BSP_SIDE=0: count the light rows on the main stream (no overlap)
    static const bool side_ok = [] {
        const char* e = std::getenv("BSP_SIDE");
        return !(e && e[0] == '0');
    }();
    if (side_ok && early_row_nnz && tot_listed > plan.class_count[NCLS - 1]) {
        SideStream side(h);
        OutCtx out{};
        out.row_begin = plan.rb;
        out.row_nnz = early_row_nnz;
        run_light<false>(h, m, plan, out);
        plan.light_sym_done = true;
        plan.side_h = h;
    }
    // Heavy rows: planned column windows.
    const int64_t nh = plan.class_count[NCLS - 1];
    if (nh > 0) {
        // heavy rows in row order: window ids then follow C's layout (the
        // look-back numeric places windows in window-id order)
        sort_ids(h, plan.lists.p + plan.class_off[NCLS - 1], nh);
        const int32_t* heavy = plan.lists.p + plan.class_off[NCLS - 1];
        int log_binw = LOG_WD;
        while (div_up(m.ncols, int64_t{1} << log_binw) > MAXBINS) ++log_binw;
        const int32_t nbins = static_cast<int32_t>(div_up(m.ncols, int64_t{1} << log_binw));
        require(log_binw == LOG_WD,
                "planner: heavy rows need ncols <= 16M (MAXBINS*WD) in this build");
        DBuf<int32_t> nwin(h, nh + 1);
        BSP_CUDA(cudaMemsetAsync(nwin.p, 0, (nh + 1) * sizeof(int32_t), h->stream));
        // window packing capacity (products; BSP_WTARGET to tune): windows of
        // <= 2048 products run in the 2048 tile at 4 CTAs/SM (measured: cfg5
        // 353 ms vs 360 ms at 3072, 370 ms at 1536, 390 ms at 1024)
        static const int32_t capg = [] {
            const char* e = std::getenv("BSP_WTARGET");
            const int v = e ? std::atoi(e) : 2048;
            return std::max(64, std::min(v, CAP));
        }();
        // window descriptors: per heavy row a slot sized by the window bound
        DBuf<int64_t> dbound(h, nh + 1), doff(h, nh + 1);
        BSP_LAUNCH(h, plan_bound_kernel, static_cast<unsigned>(div_up(nh + 1, 256)), 256, 0,
                   heavy, nh, rb, prod_out, nbins, capg, dbound.p);
        exclusive_scan_i64(h, dbound.p, doff.p, nh + 1);
        int64_t ndesc = 0;
        d2h(h, &ndesc, doff.p + nh, 1);
        sync(h);
        DBuf<uint2> desc(h, ndesc);
        // bin summaries of B for both planner passes (BSP_BIN_SUMMARY=0: stream columns)
        static const bool use_sum = [] {
            const char* e = std::getenv("BSP_BIN_SUMMARY");
            return !(e && e[0] == '0');
        }();
        DBuf<int64_t> sptr;
        DBuf<uint32_t> sent;
        BinSum bs{};
        if (use_sum) {
            const int64_t nb = m.bnrows;
            DBuf<int64_t> scnt(h, nb + 1);
            BSP_CUDA(cudaMemsetAsync(scnt.p + nb, 0, sizeof(int64_t), h->stream));
            const unsigned gs = static_cast<unsigned>(
                std::max<int64_t>(1, std::min<int64_t>(div_up(nb, 8), int64_t{h->sm_count} * 16)));
            BSP_LAUNCH(h, bin_summary_kernel<0>, gs, 256, 0, m.brp, m.bcol, nb, log_binw, scnt.p,
                       nullptr, nullptr);
            sptr = DBuf<int64_t>(h, nb + 1);
            exclusive_scan_i64(h, scnt.p, sptr.p, nb + 1);
            // bounded by nnz(B) (one entry per column at most): no readback
            sent = DBuf<uint32_t>(h, std::max<int64_t>(m.bnnz, 1));
            BSP_LAUNCH(h, bin_summary_kernel<1>, gs, 256, 0, m.brp, m.bcol, nb, log_binw, nullptr,
                       sptr.p, sent.p);
            bs = BinSum{sptr.p, sent.p};
        }
        BSP_LAUNCH(h, plan_count_kernel, static_cast<unsigned>(nh), PLAN_T, 0, m, heavy, nbins,
                   log_binw, nwin.p, doff.p, desc.p, capg, bs);
        DBuf<int64_t> woff(h, nh + 1);
        exclusive_scan_i32_to_i64(h, nwin.p, woff.p, nh + 1);
        // per-(window, segment) start tables, bounded per row and in total
        DBuf<int64_t> ssz(h, nh + 1), soff(h, nh + 1);
        BSP_LAUNCH(h, start_size_kernel, static_cast<unsigned>(div_up(nh + 1, 256)), 256, 0, m,
                   heavy, nh, nwin.p, int64_t{1} << 24, ssz.p);
        exclusive_scan_i64(h, ssz.p, soff.p, nh + 1);
        int64_t hv[2];
        d2h(h, &hv[0], woff.p + nh, 1);
        d2h(h, &hv[1], soff.p + nh, 1);
        sync(h);
        plan.nwin = hv[0];
        // Start-table budget (4-byte entries, absolute B offsets: only when
        // nnz(B) < 2^32): at least min(2^30 entries, 1/16 of available HBM);
        // up to 2^31 entries when HBM also holds an upper bound of C (12 B x
        // products) and a 2 GB margin (the bound is loose when columns
        // repeat: cfg3).  Rows in scan order that fit get a table, the rest
        // binary-search.
        constexpr int64_t EB = sizeof(uint32_t);
        // the kept table buffer counts as available to the tables
        const int64_t avail =
            (plan.avail_hint >= 0 ? plan.avail_hint : static_cast<int64_t>(available_bytes(h))) +
            (plan.keep_tables ? static_cast<int64_t>(h->keep_starts_bytes) : 0);
        const int64_t spare = avail - 12 * h->stats.products - (int64_t{2} << 30);
        const int64_t floor_entries = std::min<int64_t>(int64_t{1} << 30, avail / (16 * EB));
        const int64_t budget = std::min<int64_t>(
            hv[1], std::max<int64_t>(floor_entries,
                                     std::min<int64_t>(int64_t{1} << 31, spare / EB)));
        const bool use_starts = budget > 0 && m.bnnz < (int64_t{1} << 32);
        if (use_starts) {
            if (plan.keep_tables) {
                const size_t bytes = static_cast<size_t>(budget) * sizeof(uint32_t);
                if (bytes > h->keep_starts_bytes) {
                    if (h->keep_starts) dfree(h, h->keep_starts);
                    h->keep_starts = nullptr;
                    h->keep_starts_bytes = 0;
                    const size_t want = bytes + bytes / 8;  // headroom for the next call
                    h->keep_starts = dalloc<unsigned char>(h, static_cast<int64_t>(want));
                    h->keep_starts_bytes = want;
                }
                plan.starts = DBuf<uint32_t>::borrow(static_cast<uint32_t*>(h->keep_starts), budget);
            } else {
                plan.starts = DBuf<uint32_t>(h, budget);
            }
        }
        plan.wins = DBuf<Window>(h, plan.nwin);
        DBuf<uint8_t> dense(h, plan.nwin);
        // start tables by binary search where (windows - 1) x segments x log2(len)
        // < products x BSP_BS_X4 / 4 (0 disables).  Measured on cfg5: plan_write
        // 35.5 ms streaming only, 25.4 ms at 2 (28.2 / 28.7 / 28.8 / 40.3 / 59.7 ms
        // at 1 / 3 / 4 / 8 / 16).
        static const int bs_x4 = [] {
            const char* e = std::getenv("BSP_BS_X4");
            return e ? std::atoi(e) : 2;
        }();
        set_smem(plan_write_kernel, sizeof(PlanWriteShared));
        BSP_LAUNCH(h, plan_write_kernel, static_cast<unsigned>(nh), PLAN_T,
                   sizeof(PlanWriteShared), m, heavy, nbins, log_binw, nwin.p, doff.p, desc.p,
                   woff.p, plan.wins.p, dense.p, use_starts ? soff.p : nullptr, budget,
                   use_starts ? plan.starts.p : nullptr, bs_x4, bs);
        plan.sparse_ids = DBuf<int32_t>(h, plan.nwin);
        plan.dense_ids = DBuf<int32_t>(h, plan.nwin);
        DBuf<unsigned long long> cnt(h, 2 * (NWCLS + 1));
        BSP_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * (NWCLS + 1) * sizeof(unsigned long long), h->stream));
        BSP_LAUNCH(h, window_cat_count_kernel, static_cast<unsigned>(div_up(plan.nwin, 256)), 256,
                   0, dense.p, plan.wins.p, plan.nwin, cnt.p);
        unsigned long long hc[2 * (NWCLS + 1)];
        d2h(h, hc, cnt.p, 2 * (NWCLS + 1));
        for (int k = 0; k <= NWCLS; ++k) plan.wcls_prod[k] = static_cast<int64_t>(hc[NWCLS + 1 + k]);
        // sparse list = tile classes in descending size (top-k walks it whole)
        unsigned long long cur[NWCLS + 1];
        plan.wcls_off[0] = 0;
        for (int k = 0; k < NWCLS; ++k) {
            cur[k] = static_cast<unsigned long long>(plan.wcls_off[k]);
            plan.wcls_off[k + 1] = plan.wcls_off[k] + static_cast<int64_t>(hc[k]);
        }
        cur[NWCLS] = 0;
        plan.nsparse = plan.wcls_off[NWCLS];
        plan.ndense = static_cast<int64_t>(hc[NWCLS]);
        h2d(h, cnt.p, cur, NWCLS + 1);
        BSP_LAUNCH(h, split_windows_kernel, static_cast<unsigned>(div_up(plan.nwin, 256)), 256, 0,
                   dense.p, plan.nwin, cnt.p, plan.sparse_ids.p, plan.dense_ids.p);
        // BSP_WINDOW_ORDER=col: each list in column order (stable) so that
        // concurrent windows share B's column slices in L2 — measured slower
        // on cfg5 (545 vs 524 ms: A rows and start tables lose their reuse),
        // so row order is the default.
        static const bool by_col = [] {
            const char* e = std::getenv("BSP_WINDOW_ORDER");
            return e && std::string(e) == "col";
        }();
        if (by_col) {
            const int cbits = bit_length(static_cast<uint32_t>(std::max<int64_t>(m.ncols, 1)));
            auto sort_list = [&](int32_t* ids, int64_t n) {
                if (n <= 1) return;
                DBuf<uint32_t> k0(h, n), k1(h, n);
                DBuf<int32_t> v1(h, n);
                BSP_LAUNCH(h, window_c0_kernel, static_cast<unsigned>(div_up(n, 256)), 256, 0,
                           plan.wins.p, ids, n, k0.p);
                size_t tmp = 0;
                BSP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.p, k1.p, ids, v1.p, n, 0,
                                                         cbits, h->stream));
                DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
                BSP_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, k0.p, k1.p, ids, v1.p, n, 0,
                                                         cbits, h->stream));
                ++h->launches;
                BSP_CUDA(cudaMemcpyAsync(ids, v1.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                         h->stream));
            };
            for (int k = 0; k < NWCLS; ++k)
                sort_list(plan.sparse_ids.p + plan.wcls_off[k],
                          plan.wcls_off[k + 1] - plan.wcls_off[k]);
            sort_list(plan.dense_ids.p, plan.ndense);
        }
    }
    for (int c = 0; c < NCLS; ++c) h->stats.units[c] = plan.class_count[c];  // [7] = heavy rows
    h->stats.units[8] = plan.nsparse;
    h->stats.units[9] = plan.ndense;
}

template <bool NUMERIC>
void run_light(bsp_handle h, const Mats& m, const RowwisePlan& plan, const OutCtx& out) {
    // largest class first
    for (int c = NCLS - 2; c >= 1; --c)
        launch_light<NUMERIC>(h, c, m, plan.lists.p + plan.class_off[c], plan.class_count[c], out);
}

template <bool NUMERIC>
void run_windows(bsp_handle h, const Mats& m0, const RowwisePlan& plan, const OutCtx& out,
                 int skip_cls = -1) {
    const Mats m = plan.with_starts(m0);
    auto wl = [&](int k) { return plan.sparse_ids.p + plan.wcls_off[k]; };
    auto wn = [&](int k) {
        return k == skip_cls ? int64_t{0} : plan.wcls_off[k + 1] - plan.wcls_off[k];
    };
    static_assert(NWCLS == 5, "one launch per window tile class");
    launch_tile<256, 4096, NUMERIC>(h, m, wl(0), wn(0), plan.wins.p, out);
    launch_tile<256, 3072, NUMERIC>(h, m, wl(1), wn(1), plan.wins.p, out);
    launch_tile<256, 2048, NUMERIC>(h, m, wl(2), wn(2), plan.wins.p, out);
    launch_tile<128, 1024, NUMERIC>(h, m, wl(3), wn(3), plan.wins.p, out);
    launch_tile<64, 512, NUMERIC>(h, m, wl(4), wn(4), plan.wins.p, out);
    launch_dense<NUMERIC>(h, m, plan.dense_ids.p, plan.ndense, plan.wins.p, out);
}

template <bool NUMERIC>
void run_plan(bsp_handle h, const Mats& m, const RowwisePlan& plan, const OutCtx& out) {
    run_light<NUMERIC>(h, m, plan, out);
    run_windows<NUMERIC>(h, m, plan, out);
}

// Symbolic pass of a plan: exact per-row counts (row_nnz must be zeroed by
// the caller, and be the array given to build_plan when the light rows were
// counted early) and per-window counts.
void plan_symbolic(bsp_handle h, const Mats& m, const RowwisePlan& plan, int64_t* row_nnz,
                   DBuf<int64_t>& win_nnz, int skip_wcls) {
    win_nnz = DBuf<int64_t>(h, plan.nwin + 1);
    BSP_CUDA(cudaMemsetAsync(win_nnz.p, 0, (plan.nwin + 1) * sizeof(int64_t), h->stream));
    OutCtx out{};
    out.row_begin = plan.rb;
    out.row_nnz = row_nnz;
    out.win_nnz = win_nnz.p;
    if (!plan.light_sym_done) run_light<false>(h, m, plan, out);
    run_windows<false>(h, m, plan, out, skip_wcls);
    if (plan.light_sym_done) {
        join_side(h);
        plan.side_h = nullptr;
    }
}

// ---------------------------------------------------------------------------
// Duplicate-heavy light rows (products >= 2 x outputs, <= HACC_MAX outputs;
// cfg4's stencil rows: 729 products -> 125 columns): a warp per row
// accumulates into a per-warp smem hash (column -> running sum), one segment
// at a time in k order — a segment's columns are distinct, so its lanes never
// collide, and every column's sum is ((0.0 + p1) + p2) + ... in ascending k as
// the reference forms it — then sorts only the row's distinct columns (rank by
// counting against the compacted keys, read as warp broadcasts).
// ---------------------------------------------------------------------------
constexpr int HACC_WARPS = 8, HACC_HS = 512, HACC_MAX = 256;
struct HaccShared {
    int32_t key[HACC_WARPS][HACC_HS];
    double val[HACC_WARPS][HACC_HS];
};

__global__ void __launch_bounds__(HACC_WARPS * 32)
    hashacc_kernel(Mats m, const int32_t* __restrict__ rows, int64_t nrows, int64_t rb,
                   const int64_t* __restrict__ crp, int32_t* __restrict__ ccol,
                   double* __restrict__ cval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HaccShared& s = *reinterpret_cast<HaccShared*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* keys = s.key[warp];
    double* vals = s.val[warp];
    constexpr int LG = 31 - __builtin_clz(static_cast<unsigned>(HACC_HS));
    constexpr int PER = HACC_MAX / 32;
    for (int64_t t = blockIdx.x * int64_t{HACC_WARPS} + warp; t < nrows;
         t += int64_t{gridDim.x} * HACC_WARPS) {
        const int32_t row = rows[t];
        for (int i = lane; i < HACC_HS; i += 32) keys[i] = -1;
        __syncwarp();
        const int64_t rs = m.arp[row], re = m.arp[row + 1];
        for (int64_t pb = rs; pb < re; pb += 32) {
            const int64_t p = pb + lane;
            int64_t b0 = 0;
            int len = 0;
            double a = 0.0;
            if (p < re) {
                const int32_t k = __ldg(m.acol + p);
                b0 = __ldg(m.brp + k);
                len = static_cast<int>(__ldg(m.brp + k + 1) - b0);
                a = __ldg(m.aval + p);
            }
            unsigned ne = __ballot_sync(0xffffffffu, len > 0);
            while (ne) {
                const int j = __ffs(ne) - 1;
                ne &= ne - 1;
                const int64_t bj = __shfl_sync(0xffffffffu, b0, j);
                const int lj = __shfl_sync(0xffffffffu, len, j);
                const double aj = __shfl_sync(0xffffffffu, a, j);
                for (int q = lane; q < lj; q += 32) {
                    const int32_t col = __ldg(m.bcol + bj + q);
                    const double v = __dmul_rn(aj, __ldg(m.bval + bj + q));
                    uint32_t slot = col_hash(static_cast<uint32_t>(col), LG);
                    for (;;) {
                        const int32_t prev = atomicCAS(&keys[slot], -1, col);
                        if (prev == -1) {
                            vals[slot] = __dadd_rn(0.0, v);
                            break;
                        }
                        if (prev == col) {
                            vals[slot] = __dadd_rn(vals[slot], v);
                            break;
                        }
                        slot = (slot + 1) & (HACC_HS - 1);
                    }
                }
                __syncwarp();  // the next segment adds after this one
            }
        }
        // compact the occupied slots to the front (ascending slot order; a
        // block's slots are read before any position inside it is written)
        int nnz = 0;
        for (int i0 = 0; i0 < HACC_HS; i0 += 32) {
            const int32_t kk = keys[i0 + lane];
            const double vv = vals[i0 + lane];
            const unsigned occ = __ballot_sync(0xffffffffu, kk >= 0);
            __syncwarp();
            if (kk >= 0) {
                const int pos = nnz + __popc(occ & ((1u << lane) - 1u));
                keys[pos] = kk;
                vals[pos] = vv;
            }
            nnz += __popc(occ);
            __syncwarp();
        }
        // rank each distinct column among the row's columns
        int32_t mk[PER];
        double mv[PER];
        int rk[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int i = u * 32 + lane;
            mk[u] = i < nnz ? keys[i] : 0x7fffffff;
            mv[u] = i < nnz ? vals[i] : 0.0;
            rk[u] = 0;
        }
        // (only the lane slots that hold columns are ranked: cfg4's rows hold
        // 125 columns = 4 of the 8 slots, and the ranking is most of the row's work)
        auto rank_cols = [&](auto nu_c) {
            constexpr int NU = decltype(nu_c)::value;
            for (int jj = 0; jj < nnz; ++jj) {
                const int32_t kj = keys[jj];
#pragma unroll
                for (int u = 0; u < NU; ++u) rk[u] += kj < mk[u];
            }
        };
        if (nnz <= 64) rank_cols(std::integral_constant<int, 2>{});
        else if (nnz <= 128) rank_cols(std::integral_constant<int, 4>{});
        else rank_cols(std::integral_constant<int, PER>{});
        const int64_t base = crp[row - rb];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            if (u * 32 + lane < nnz) {
                ccol[base + rk[u]] = mk[u];
                cval[base + rk[u]] = mv[u];
            }
        }
        __syncwarp();
    }
}

// Split the light rows: duplicate-heavy ones (products >= 2 x outputs, <=
// HACC_MAX outputs) to hlist, the rest back into per-class lists.
__global__ void route_light_kernel(const int32_t* __restrict__ lists, int64_t nlight, int64_t rb,
                                   const int64_t* __restrict__ prod, const int64_t* __restrict__ crp,
                                   unsigned long long* __restrict__ cursor,
                                   int32_t* __restrict__ hlist, int32_t* __restrict__ tlists) {
    const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (t >= nlight) return;
    const int32_t row = lists[t];
    const int64_t r = row - rb;
    const int64_t P = prod[r], nz = crp[r + 1] - crp[r];
    if (P >= 2 * nz && nz <= HACC_MAX) {
        hlist[atomicAdd(&cursor[0], 1ull)] = row;
    } else {
        int c = 1;
        while (c < NCLS - 1 && P > kClassCap[c]) ++c;
        tlists[atomicAdd(&cursor[c], 1ull)] = row;
    }
}

// Rows (absolute ids; at most HACC_MAX outputs each) on the hash accumulator.
void run_hashacc_rows(bsp_handle h, const Mats& m, const int32_t* rows, int64_t n, int64_t rb,
                      const int64_t* crp, int32_t* ccol, double* cval) {
    if (n <= 0) return;
    set_smem(hashacc_kernel, sizeof(HaccShared));
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(n, HACC_WARPS), int64_t{h->sm_count} * 16)));
    BSP_LAUNCH(h, hashacc_kernel, grid, HACC_WARPS * 32, sizeof(HaccShared), m, rows, n, rb, crp,
               ccol, cval);
}

void plan_numeric(bsp_handle h, const Mats& m, const RowwisePlan& plan, const int64_t* crp,
                  const int64_t* win_scan, int32_t* ccol, double* cval, int skip_wcls) {
    OutCtx out{};
    out.row_begin = plan.rb;
    out.crp = crp;
    out.win_scan = win_scan;
    out.ccol = ccol;
    out.cval = cval;
    // BSP_HACC=0: duplicate-heavy light rows stay on the sort tiles
    static const bool hacc = [] {
        const char* e = std::getenv("BSP_HACC");
        return !(e && e[0] == '0');
    }();
    const int64_t nlight = plan.class_off[NCLS - 1] - plan.class_off[1];
    // route only when columns repeat overall (compression factor >= 1.25:
    // cfg3 2.95, cfg4 5.84; not cfg2/cfg5 ~1.0, which would only pay the
    // routing pass and its readback)
    int64_t planned = 0;
    for (int c = 1; c < NCLS; ++c) planned += plan.class_products[c];
    const bool repeats = 4 * planned >= 5 * std::max<int64_t>(1, h->stats.nnz_out);
    if (!hacc || !repeats || nlight <= 0 || plan.prod.p == nullptr) {
        run_light<true>(h, m, plan, out);
        run_windows<true>(h, m, plan, out, skip_wcls);
        return;
    }
    DBuf<int32_t> hlist(h, nlight), tl(h, nlight);
    DBuf<unsigned long long> cursor(h, NCLS);
    unsigned long long cur[NCLS];
    cur[0] = 0;
    for (int c = 1; c < NCLS; ++c)
        cur[c] = static_cast<unsigned long long>(plan.class_off[c] - plan.class_off[1]);
    h2d(h, cursor.p, cur, NCLS);
    BSP_LAUNCH(h, route_light_kernel, static_cast<unsigned>(div_up(nlight, 256)), 256, 0,
               plan.lists.p + plan.class_off[1], nlight, plan.rb, plan.prod.p, crp, cursor.p,
               hlist.p, tl.p);
    unsigned long long hc[NCLS];
    d2h(h, hc, cursor.p, NCLS);
    const int64_t nh = static_cast<int64_t>(hc[0]);
    run_hashacc_rows(h, m, hlist.p, nh, plan.rb, crp, ccol, cval);
    for (int c = NCLS - 2; c >= 1; --c) {
        const int64_t b0 = plan.class_off[c] - plan.class_off[1];
        const int64_t cnt = static_cast<int64_t>(hc[c]) - b0;
        launch_light<true>(h, c, m, tl.p + b0, cnt, out);
    }
    run_windows<true>(h, m, plan, out, skip_wcls);
}

// Narrow B: symbolic (+ products) -> int64 scan -> numeric, no planning.
// B with <= 64 columns (the tall-skinny frontier operands): each B row as a
// 64-bit column mask, built once per multiply.
__global__ void row_mask64_kernel(const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol,
                                  int64_t nb, unsigned long long* __restrict__ mask) {
    for (int64_t k = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; k < nb;
         k += int64_t{gridDim.x} * blockDim.x) {
        unsigned long long mk = 0;
        for (int64_t q = brp[k]; q < brp[k + 1]; ++q) mk |= 1ull << __ldg(bcol + q);
        mask[k] = mk;
    }
}

// A warp per row; lane l owns output columns l and l + 32 and keeps their sums
// in registers.  The row's non-empty segments are walked in k order, each
// broadcast (B offset, column mask, a_ik) once: a lane whose column is in the
// mask adds a_ik * b_kj, b_kj found at the popcount of the mask below its bit
// — ascending k per column, so the sums are the reference's.  Symbolic: the
// popcount of the OR of the masks.
template <bool NUMERIC>
__global__ void __launch_bounds__(NARROW_WARPS * 32)
    narrow64_kernel(Mats m, const unsigned long long* __restrict__ bmask, int64_t rb, int64_t n,
                    int64_t* __restrict__ row_nnz, const int64_t* __restrict__ crp,
                    int32_t* __restrict__ ccol, double* __restrict__ cval,
                    unsigned long long* __restrict__ products, const uint8_t* __restrict__ skip,
                    unsigned long long* __restrict__ next) {
    const int lane = threadIdx.x & 31;
    const unsigned long long below0 = (1ull << lane) - 1ull, below1 = (1ull << (lane + 32)) - 1ull;
    unsigned long long prod = 0;
    // numeric: rows handed out dynamically in pairs (hub rows first, as they
    // come first), so a warp that drew a hub row does not also carry a fixed
    // share of the rest; symbolic (cheap per row): a static grid stride
    constexpr int64_t G = 2;
    const int64_t nwarps = int64_t{gridDim.x} * NARROW_WARPS;
    int64_t r = NUMERIC ? 0 : blockIdx.x * int64_t{NARROW_WARPS} + (threadIdx.x >> 5);
    int64_t rend = NUMERIC ? 0 : n;
    for (;;) {
        if constexpr (NUMERIC) {
            if (r >= rend) {
                int64_t g = 0;
                if (lane == 0)
                    g = static_cast<int64_t>(atomicAdd(next, static_cast<unsigned long long>(G)));
                g = __shfl_sync(0xffffffffu, g, 0);
                if (g >= n) break;
                r = g;
                rend = ::min(n, g + G);
            }
        } else {
            if (r >= n) break;
        }
        const int64_t r_ = r;
        r += NUMERIC ? 1 : nwarps;
        if (skip && skip[r_]) continue;  // warp-uniform (rows of a cluster tile)
        const int64_t row = rb + r_;
        const int64_t rs = m.arp[row], re = m.arp[row + 1];
        unsigned long long touch = 0;
        double acc0 = 0.0, acc1 = 0.0;
        for (int64_t pb = rs; pb < re; pb += 32) {
            const int64_t p = pb + lane;
            unsigned long long mk = 0;
            int64_t b0 = 0;
            double a = 0.0;
            if (p < re) {
                const int32_t k = __ldg(m.acol + p);
                mk = __ldg(bmask + k);
                if (NUMERIC) {
                    b0 = __ldg(m.brp + k);
                    a = __ldg(m.aval + p);
                } else {
                    prod += static_cast<unsigned long long>(__popcll(mk));
                }
            }
            touch |= mk;
            if (NUMERIC) {
                // non-empty segments in k order, NP at a time: their b loads
                // are all issued before the ordered adds (latency overlap)
                constexpr int NP = 4;
                unsigned ne = __ballot_sync(0xffffffffu, mk != 0);
                while (ne) {
                    double aj[NP], v0[NP], v1[NP];
                    bool h0[NP], h1[NP];
#pragma unroll
                    for (int u = 0; u < NP; ++u) {
                        h0[u] = h1[u] = false;
                        aj[u] = v0[u] = v1[u] = 0.0;
                        if (ne) {
                            const int j = __ffs(ne) - 1;
                            ne &= ne - 1;
                            const unsigned long long mj = __shfl_sync(0xffffffffu, mk, j);
                            const int64_t bj = __shfl_sync(0xffffffffu, b0, j);
                            aj[u] = __shfl_sync(0xffffffffu, a, j);
                            h0[u] = (mj >> lane) & 1ull;
                            h1[u] = (mj >> (lane + 32)) & 1ull;
                            if (h0[u]) v0[u] = __ldg(m.bval + bj + __popcll(mj & below0));
                            if (h1[u]) v1[u] = __ldg(m.bval + bj + __popcll(mj & below1));
                        }
                    }
#pragma unroll
                    for (int u = 0; u < NP; ++u) {
                        if (h0[u]) acc0 = __dadd_rn(acc0, __dmul_rn(aj[u], v0[u]));
                        if (h1[u]) acc1 = __dadd_rn(acc1, __dmul_rn(aj[u], v1[u]));
                    }
                }
            }
        }
        // OR of the lanes' masks
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) touch |= __shfl_xor_sync(0xffffffffu, touch, o);
        if (!NUMERIC) {
            if (lane == 0) row_nnz[r_] = __popcll(touch);
        } else {
            const int64_t pos = crp[r_];
            if ((touch >> lane) & 1ull) {
                const int64_t o = pos + __popcll(touch & below0);
                ccol[o] = lane;
                cval[o] = acc0;
            }
            if ((touch >> (lane + 32)) & 1ull) {
                const int64_t o = pos + __popcll(touch & below1);
                ccol[o] = lane + 32;
                cval[o] = acc1;
            }
        }
    }
    if (!NUMERIC) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
        if (lane == 0 && prod) atomicAdd(products, prod);
    }
}

static void narrow_multiply(bsp_handle h, const Mats& m, int64_t rb, int64_t n, int64_t ncols,
                            int64_t bnrows, bsp_csr* C, int64_t* row_nnz_out) {
    DBuf<int64_t> cnt(h, n + 1);
    BSP_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(int64_t), h->stream));
    DBuf<unsigned long long> prod(h, 1);
    BSP_CUDA(cudaMemsetAsync(prod.p, 0, sizeof(unsigned long long), h->stream));
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(std::max<int64_t>(n, 1), NARROW_WARPS),
                             int64_t{h->sm_count} * 32)));
    const int32_t nc = static_cast<int32_t>(ncols);
    auto ks = narrow_kernel<false>;
    auto kn = narrow_kernel<true>;
    // <= 64 columns: B rows as 64-bit masks, sums in registers
    const bool m64 = ncols <= 64;
    DBuf<unsigned long long> bmask;
    if (m64) {
        bmask = DBuf<unsigned long long>(h, std::max<int64_t>(bnrows, 1));
        const unsigned gm = static_cast<unsigned>(std::max<int64_t>(
            1, std::min<int64_t>(div_up(std::max<int64_t>(bnrows, 1), 256), int64_t{h->sm_count} * 8)));
        BSP_LAUNCH(h, row_mask64_kernel, gm, 256, 0, m.brp, m.bcol, bnrows, bmask.p);
        DBuf<unsigned long long> nx(h, 1);
        BSP_CUDA(cudaMemsetAsync(nx.p, 0, sizeof(unsigned long long), h->stream));
        BSP_LAUNCH_AS(h, "narrow64_symbolic", narrow64_kernel<false>, grid, NARROW_WARPS * 32, 0, m,
                      bmask.p, rb, n, cnt.p, nullptr, nullptr, nullptr, prod.p, nullptr, nx.p);
    } else {
        BSP_LAUNCH_AS(h, "narrow_symbolic", ks, grid, NARROW_WARPS * 32, 0, m, rb, n, nc, cnt.p,
                      nullptr, nullptr, nullptr, prod.p);
    }
    if (row_nnz_out)
        BSP_CUDA(cudaMemcpyAsync(row_nnz_out, cnt.p, n * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                                 h->stream));
    DBuf<int64_t> rp(h, n + 1, Pool::out);
    exclusive_scan_i64(h, cnt.p, rp.p, n + 1);
    const int64_t nnz = read_scalar(h, rp.p + n);
    h->stats.products = static_cast<int64_t>(read_scalar(h, prod.p));
    h->stats.nnz_out = nnz;
    ResultPayload pay(h, nnz);
    if (m64) {
        DBuf<unsigned long long> nx(h, 1);
        BSP_CUDA(cudaMemsetAsync(nx.p, 0, sizeof(unsigned long long), h->stream));
        BSP_LAUNCH_AS(h, "narrow64_numeric", narrow64_kernel<true>, grid, NARROW_WARPS * 32, 0, m,
                      bmask.p, rb, n, nullptr, rp.p, pay.col_idx(), pay.values(), nullptr, nullptr,
                      nx.p);
    } else {
        BSP_LAUNCH_AS(h, "narrow_numeric", kn, grid, NARROW_WARPS * 32, 0, m, rb, n, nc, nullptr,
                      rp.p, pay.col_idx(), pay.values(), nullptr);
    }
    C->nrows = n;
    C->ncols = ncols;
    C->nnz = nnz;
    C->row_ptr = rp.release();
    C->col_idx = pay.col_idx();
    C->values = pay.block.release();
    C->owned = 2;
}

void narrow64_row_masks(bsp_handle h, const Mats& m, int64_t bnrows,
                        DBuf<unsigned long long>& mask) {
    mask = DBuf<unsigned long long>(h, std::max<int64_t>(bnrows, 1));
    const unsigned gm = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(std::max<int64_t>(bnrows, 1), 256), int64_t{h->sm_count} * 8)));
    BSP_LAUNCH(h, row_mask64_kernel, gm, 256, 0, m.brp, m.bcol, bnrows, mask.p);
}

void narrow64_rows(bsp_handle h, const Mats& m, const unsigned long long* mask, int64_t n,
                   const uint8_t* skip, int64_t* row_nnz, const int64_t* crp, int32_t* ccol,
                   double* cval, unsigned long long* products) {
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(std::max<int64_t>(n, 1), NARROW_WARPS),
                             int64_t{h->sm_count} * 32)));
    DBuf<unsigned long long> nx(h, 1);
    BSP_CUDA(cudaMemsetAsync(nx.p, 0, sizeof(unsigned long long), h->stream));
    if (crp == nullptr)
        BSP_LAUNCH_AS(h, "narrow64_symbolic", narrow64_kernel<false>, grid, NARROW_WARPS * 32, 0, m,
                      mask, int64_t{0}, n, row_nnz, nullptr, nullptr, nullptr, products, skip, nx.p);
    else
        BSP_LAUNCH_AS(h, "narrow64_numeric", narrow64_kernel<true>, grid, NARROW_WARPS * 32, 0, m,
                      mask, int64_t{0}, n, nullptr, crp, ccol, cval, nullptr, skip, nx.p);
}

// The look-back list's windows in list order (id kept in pad_).
__global__ void gather_windows_kernel(const int32_t* __restrict__ ids, int64_t n,
                                      const Window* __restrict__ wins, Window* __restrict__ out) {
    const int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (i >= n) return;
    Window w = wins[ids[i]];
    w.pad_ = ids[i];
    out[i] = w;
}

// Look-back list split (rowwise_multiply): windows whose A row has at most dmax
// segments stay on the look-back tile.
struct WindowShortRow {
    const Window* wins;
    int dmax;
    __device__ bool operator()(int32_t w) const { return wins[w].d <= dmax; }
};
__global__ void sum_window_products_kernel(const int32_t* __restrict__ ids, int64_t n,
                                           const Window* __restrict__ wins,
                                           unsigned long long* __restrict__ out) {
    unsigned long long v = 0;
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < n;
         i += int64_t{gridDim.x} * blockDim.x)
        v += static_cast<unsigned long long>(wins[ids[i]].nprod);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

void rowwise_multiply(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int64_t rb, int64_t re,
                      bsp_csr* C, const uint8_t* row_skip, int64_t* row_nnz_out) {
    check_csr(A, "spgemm_rowwise");
    check_csr(B, "spgemm_rowwise");
    require(A->ncols == B->nrows, "spgemm: dimension mismatch (a.ncols != b.nrows)");
    require(rb >= 0 && rb <= re && re <= A->nrows, "spgemm: bad row range");
    BSP_CUDA(cudaSetDevice(h->device));
    h->stats = bsp_exec_stats{};
    h->stats.chunks = 1;
    const Mats m = make_mats(A, B);
    const int64_t n = re - rb;
    // BSP_NARROW=0 forces the tile path (read per call, so tests can cover both)
    const char* ne = std::getenv("BSP_NARROW");
    if (B->ncols <= NARROW && row_skip == nullptr && !(ne && ne[0] == '0')) {
        narrow_multiply(h, m, rb, n, B->ncols, B->nrows, C, row_nnz_out);
        return;
    }
    DBuf<int64_t> crp(h, n + 1);
    BSP_CUDA(cudaMemsetAsync(crp.p, 0, (n + 1) * sizeof(int64_t), h->stream));
    RowwisePlan plan;
    plan.keep_tables = true;
    plan.avail_hint = static_cast<int64_t>(available_bytes(h));  // before any sync (see esc.cuh)
    build_plan(h, m, rb, re, row_skip, plan, nullptr, crp.p);
    // The main window class (2048-product tiles: nearly all heavy products on
    // power-law inputs) is counted by its numeric pass (esc_window_lb_kernel)
    // instead of a symbolic pass, when C's allocation can take that class's
    // product bound (cf ~ 1 there: a few % of slack) — BSP_LOOKBACK=0 disables.
    constexpr int LBC = 2;  // window tile class of esc_window_lb_kernel<256, 2048>
    static const bool lb_on = [] {
        const char* e = std::getenv("BSP_LOOKBACK");
        return !(e && e[0] == '0');
    }();
    int64_t nlb = plan.wcls_off[LBC + 1] - plan.wcls_off[LBC];
    bool lb = lb_on && nlb > 0;
    // Windows of rows with many segments leave the look-back list (BSP_LB_DMAX,
    // 0 = keep all): a tile's time to publish its count grows with the A row's
    // length d (measured on cfg5, cycles from tile start to publish: 29K at
    // d <= 256, 46K at d <= 1024, 97K at d <= 4096, 167K above), and every tile
    // behind a slow one waits for it (the wait was 20 % of all tile residency).
    // The few long-row windows can take the two-pass path (symbolic + numeric
    // with known offsets) so that the look-back stream keeps tiles of similar
    // duration — measured on cfg5: no gain (the look-back kernel gets shorter
    // only by the work that leaves it: 170.5 / 165.6 / 154.5 / 135.7 / 108.2 ms
    // at dmax off / 2048 / 1024 / 512 / 256, step 287.4 / 288.1 / 288.5 / 291.6 /
    // 295.9 ms), so the wait is not caused by these tiles alone; off by default.
    // BSP_LB_V2: form of the look-back tile (0: values gathered with the columns;
    // 1: values after the count is published; 2: as 1 in the compact layout at 5
    // CTAs per SM, rows of more than 65535 entries on the two-pass path)
    static const int lb_v2 = [] {
        const char* e = std::getenv("BSP_LB_V2");
        return e ? std::atoi(e) : 2;  // measured on cfg5: 169.2 / 169.4 / 156.8 ms at 0 / 1 / 2
    }();
    static const int lb_dmax_env = [] {
        const char* e = std::getenv("BSP_LB_DMAX");
        return e ? std::atoi(e) : 0;  // measured: no gain (see below), off by default
    }();
    const int lb_dmax = (lb_v2 == 2 && m.bnnz < (int64_t{1} << 32))
                            ? (lb_dmax_env > 0 ? std::min(lb_dmax_env, 65535) : 65535)
                            : lb_dmax_env;
    int32_t* const lb_list = plan.sparse_ids.p + plan.wcls_off[LBC];
    int64_t ntp = 0;           // two-pass windows: lb_list[nlb, nlb + ntp)
    int64_t lb_products = plan.wcls_prod[LBC];
    if (lb) {
        sort_ids(h, lb_list, nlb);  // C's layout order (window ids follow the row-sorted heavy list)
        if (lb_dmax > 0) {
            DBuf<int32_t> part(h, nlb);
            DBuf<int64_t> nsel(h, 1);
            size_t bytes = 0;
            const WindowShortRow pred{plan.wins.p, lb_dmax};
            BSP_CUDA(cub::DevicePartition::If(nullptr, bytes, lb_list, part.p, nsel.p, nlb, pred,
                                              h->stream));
            DBuf<uint8_t> tmp(h, static_cast<int64_t>(bytes));
            BSP_CUDA(cub::DevicePartition::If(tmp.p, bytes, lb_list, part.p, nsel.p, nlb, pred,
                                              h->stream));
            ++h->launches;
            BSP_CUDA(cudaMemcpyAsync(lb_list, part.p, nlb * sizeof(int32_t),
                                     cudaMemcpyDeviceToDevice, h->stream));
            const int64_t keep = read_scalar(h, nsel.p);
            ntp = nlb - keep;
            nlb = keep;
            if (ntp > 0) {
                DBuf<unsigned long long> tp_prod(h, 1);
                BSP_CUDA(cudaMemsetAsync(tp_prod.p, 0, sizeof(unsigned long long), h->stream));
                BSP_LAUNCH(h, sum_window_products_kernel,
                           static_cast<unsigned>(std::min<int64_t>(div_up(ntp, 256), 1024)), 256, 0,
                           lb_list + nlb, ntp, plan.wins.p, tp_prod.p);
                lb_products -= static_cast<int64_t>(read_scalar(h, tp_prod.p));
            }
            if (nlb == 0) lb = false;  // (all of them two-pass: counted below)
        }
    }
    DBuf<int64_t> win_nnz;
    plan_symbolic(h, m, plan, crp.p, win_nnz, (lb || ntp > 0) ? LBC : -1);
    if (ntp > 0) {  // the long-row windows' symbolic count
        OutCtx so{};
        so.row_begin = plan.rb;
        so.row_nnz = crp.p;
        so.win_nnz = win_nnz.p;
        launch_tile<256, 2048, false>(h, plan.with_starts(m), lb_list + nlb, ntp, plan.wins.p, so);
    }
    BSP_CUDA(cudaMemsetAsync(crp.p + n, 0, sizeof(int64_t), h->stream));
    DBuf<int64_t> rp(h, n + 1, Pool::out);
    exclusive_scan_i64(h, crp.p, rp.p, n + 1);
    DBuf<int64_t> win_scan(h, plan.nwin + 1);
    if (plan.nwin > 0) exclusive_scan_i64(h, win_nnz.p, win_scan.p, plan.nwin + 1);
    int64_t nnz = read_scalar(h, rp.p + n);  // without the look-back class when lb
    int64_t cap = nnz;
    // the planner's allocations since the sample are small next to C; C's own
    // allocation still fails cleanly (BSP_ERR_OOM) if memory was taken meanwhile
    int64_t avail = plan.avail_hint;
    if (lb) {
        cap = nnz + lb_products;
        // C (12 B per entry) + the look-back state, with a 1 GB margin (a figure
        // that says no is checked against the driver before it is believed)
        if (12 * cap + 16 * nlb + (int64_t{1} << 30) > avail)
            avail = static_cast<int64_t>(available_bytes(h, true));
        if (12 * cap + 16 * nlb + (int64_t{1} << 30) > avail) {
            // no room for the bound: count the class symbolically after all
            lb = false;
            OutCtx so{};
            so.row_begin = plan.rb;
            so.row_nnz = crp.p;
            so.win_nnz = win_nnz.p;
            Mats ms = plan.with_starts(m);
            launch_tile<256, 2048, false>(h, ms, lb_list, nlb, plan.wins.p, so);
            ntp += nlb;  // all of the class on the two-pass path now
            exclusive_scan_i64(h, crp.p, rp.p, n + 1);
            exclusive_scan_i64(h, win_nnz.p, win_scan.p, plan.nwin + 1);
            nnz = cap = read_scalar(h, rp.p + n);
        }
    }
    {
        if (12 * cap > avail) avail = static_cast<int64_t>(available_bytes(h, true));
        if (12 * cap > avail)
            throw oom_error("spgemm_rowwise: C needs " + std::to_string(12 * cap >> 20) +
                            " MiB, more than the " + std::to_string(avail >> 20) +
                            " MiB of free device memory; use the host-output call "
                            "(bsp_spgemm_rowwise_host chunks rows) or row ranges");
    }
    ResultPayload pay(h, nnz, cap);
    if (lb) {
        // windows of the class in C's layout order (window ids follow the
        // row-sorted heavy list), claimed in that order
        int32_t* ids = lb_list;  // sorted (and split) above
        DBuf<unsigned long long> status(h, nlb);
        DBuf<int> counter(h, 1);
        BSP_CUDA(cudaMemsetAsync(status.p, 0, nlb * sizeof(unsigned long long), h->stream));
        BSP_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(int), h->stream));
        OutCtx out{};
        out.row_begin = plan.rb;
        out.crp = rp.p;            // offsets from the units counted beforehand
        out.win_scan = win_scan.p;
        out.row_nnz = crp.p;       // + this class's counts -> the final row counts
        out.win_nnz = win_nnz.p;
        out.ccol = pay.col_idx();
        out.cval = pay.values();
        static const int csort = [] {
            const char* e = std::getenv("BSP_CSORT");
            return e ? std::atoi(e) : 1000;
        }();
        using S = MergeShared<256, 2048>;
        // The second form (only the columns gathered before the sort, the values
        // after the count is published) by itself — BSP_LB_V2=1 — cuts the wait for
        // the predecessors' counts from 10.7K to 6.2K cycles per tile and the tile's
        // residency from 54.1K to 49.7K cycles at the same kernel time (169.4 vs
        // 169.2 ms); what it buys is the compact layout (6 bytes per product where
        // the first form keeps an 8-byte value through the sort): 44.9 KB per tile,
        // 5 CTAs per SM instead of 4 — the default, 156.8 ms.
        if (lb_v2 == 2 && m.bnnz < (int64_t{1} << 32)) {
            using S5 = LbTileShared<256, 2048, true>::type;
            auto k = esc_window_lb2_kernel<256, 2048, true>;
            set_smem(k, sizeof(S5));
            // BSP_LB_GATHER=0: tiles read their window through the id list
            static const bool gather = [] {
                const char* e = std::getenv("BSP_LB_GATHER");
                return !(e && e[0] == '0');
            }();
            DBuf<Window> lbw;
            if (gather) {
                lbw = DBuf<Window>(h, nlb);
                BSP_LAUNCH(h, gather_windows_kernel, static_cast<unsigned>(div_up(nlb, 256)), 256, 0,
                           ids, nlb, plan.wins.p, lbw.p);
            }
            BSP_LAUNCH_AS(h, "esc_window_lb2c<256,2048>", k, static_cast<unsigned>(nlb), 256,
                          sizeof(S5), plan.with_starts(m), gather ? nullptr : ids,
                          gather ? lbw.p : plan.wins.p, out, csort, LbCtx{counter.p, status.p});
        } else if (lb_v2 == 1 && m.bnnz < (int64_t{1} << 32)) {
            auto k = esc_window_lb2_kernel<256, 2048, false>;
            set_smem(k, sizeof(S));
            BSP_LAUNCH_AS(h, "esc_window_lb2<256,2048>", k, static_cast<unsigned>(nlb), 256,
                          sizeof(S), plan.with_starts(m), ids, plan.wins.p, out, csort,
                          LbCtx{counter.p, status.p});
        } else {
            // BSP_LB_PAD_SMEM=bytes: extra (unused) dynamic shared memory, to measure the
            // tile's sensitivity to CTAs per SM (experiments only)
            static const size_t pad = [] {
                const char* e = std::getenv("BSP_LB_PAD_SMEM");
                return e ? static_cast<size_t>(std::atoll(e)) : size_t{0};
            }();
            auto k = esc_window_lb_kernel<256, 2048>;
            set_smem(k, sizeof(S) + pad);
            BSP_LAUNCH_AS(h, "esc_window_lb<256,2048>", k, static_cast<unsigned>(nlb), 256,
                          sizeof(S) + pad, plan.with_starts(m), ids, plan.wins.p, out, csort,
                          LbCtx{counter.p, status.p});
        }
        // final row_ptr and window offsets for the remaining numeric tiles
        BSP_CUDA(cudaMemsetAsync(crp.p + n, 0, sizeof(int64_t), h->stream));
        exclusive_scan_i64(h, crp.p, rp.p, n + 1);
        exclusive_scan_i64(h, win_nnz.p, win_scan.p, plan.nwin + 1);
        nnz = read_scalar(h, rp.p + n);
    }
    if (row_nnz_out)
        BSP_CUDA(cudaMemcpyAsync(row_nnz_out, crp.p, n * sizeof(int64_t),
                                 cudaMemcpyDeviceToDevice, h->stream));
    h->stats.nnz_out = nnz;
    plan_numeric(h, m, plan, rp.p, win_scan.p, pay.col_idx(), pay.values(),
                 (lb || ntp > 0) ? LBC : -1);
    if (ntp > 0) {  // the class's two-pass windows (the tail of its list)
        OutCtx o2{};
        o2.row_begin = plan.rb;
        o2.crp = rp.p;
        o2.win_scan = win_scan.p;
        o2.ccol = pay.col_idx();
        o2.cval = pay.values();
        const int64_t t0 = lb ? nlb : 0;
        launch_tile<256, 2048, true>(h, plan.with_starts(m), lb_list + t0, ntp, plan.wins.p, o2);
    }
    C->nrows = n;
    C->ncols = B->ncols;
    C->nnz = nnz;
    C->row_ptr = rp.release();
    C->col_idx = pay.col_idx();
    C->values = pay.block.release();
    C->owned = 2;
}

}  // namespace bsp

using namespace bsp;

extern "C" {

int bsp_spgemm_products(bsp_handle h, const bsp_csr* A, const bsp_csr* B,
                        int64_t* row_products_dev, int64_t* total_out) {
    return guarded([&] {
        check_csr(A, "spgemm_products");
        check_csr(B, "spgemm_products");
        require(A->ncols == B->nrows, "spgemm: dimension mismatch (a.ncols != b.nrows)");
        BSP_CUDA(cudaSetDevice(h->device));
        const Mats m = make_mats(A, B);
        RowwisePlan plan;
        DBuf<int64_t> tmp;
        int64_t* prod = row_products_dev;
        if (!prod) {
            tmp = DBuf<int64_t>(h, A->nrows);
            prod = tmp.p;
        }
        const int64_t n = A->nrows;
        DBuf<uint8_t> cls(h, n);
        DBuf<int64_t> counters(h, 2 * NCLS);
        BSP_CUDA(cudaMemsetAsync(counters.p, 0, 2 * NCLS * sizeof(int64_t), h->stream));
        const int grid = static_cast<int>(std::min<int64_t>(
            div_up(std::max<int64_t>(n, 1), 8), int64_t{h->sm_count} * 8));
        BSP_LAUNCH(h, products_kernel, grid, 256, 0, m, 0, n, prod, cls.p, nullptr, counters.p,
                   counters.p + NCLS, 0, nullptr);
        int64_t hc[2 * NCLS];
        d2h(h, hc, counters.p, 2 * NCLS);
        sync(h);
        int64_t tot = 0;
        for (int c = 0; c < NCLS; ++c) tot += hc[NCLS + c];
        if (total_out) *total_out = tot;
    });
}

int bsp_spgemm_symbolic(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int64_t* counts_dev) {
    return guarded([&] {
        check_csr(A, "spgemm_symbolic");
        check_csr(B, "spgemm_symbolic");
        require(A->ncols == B->nrows, "spgemm: dimension mismatch (a.ncols != b.nrows)");
        BSP_CUDA(cudaSetDevice(h->device));
        const Mats m = make_mats(A, B);
        RowwisePlan plan;
        build_plan(h, m, 0, A->nrows, nullptr, plan, nullptr);
        BSP_CUDA(cudaMemsetAsync(counts_dev, 0, std::max<int64_t>(A->nrows, 1) * sizeof(int64_t),
                                 h->stream));
        DBuf<int64_t> win_nnz;
        plan_symbolic(h, m, plan, counts_dev, win_nnz);
        sync(h);
    });
}

int bsp_spgemm_rowwise(bsp_handle h, const bsp_csr* A, const bsp_csr* B, bsp_csr* C) {
    return guarded([&] {
        require(C != nullptr, "spgemm_rowwise: null output");
        check_csr(A, "spgemm_rowwise");
        rowwise_multiply(h, A, B, 0, A->nrows, C, nullptr, nullptr);
    });
}

int bsp_spgemm_rowwise_range(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int64_t row_begin,
                             int64_t row_end, bsp_csr* C) {
    return guarded([&] {
        require(C != nullptr, "spgemm_rowwise_range: null output");
        rowwise_multiply(h, A, B, row_begin, row_end, C, nullptr, nullptr);
    });
}

// The reference-shaped call (spgemm.hpp:70: host CSR in, host CSR out).  When
// C's bound (12 B per intermediate product) exceeds the device budget —
// cfg3's C is ~285 GB, more than HBM — the exact per-row counts are taken
// first (bsp_spgemm_symbolic), the host C is allocated exactly, and A is cut
// into row chunks whose exact C fits the budget; each chunk is multiplied
// (rowwise_multiply on the row range) and downloaded into its place.  Budget:
// half of the device bytes available after the uploads (BSP_CHUNK_BYTES
// overrides, for tests).
int bsp_spgemm_rowwise_host(bsp_handle h, const bsp_host_csr* A, const bsp_host_csr* B,
                            bsp_host_csr* C) {
    return guarded([&] {
        check_host_csr(A, "spgemm_rowwise_host");
        check_host_csr(B, "spgemm_rowwise_host");
        require(A->ncols == B->nrows, "spgemm: dimension mismatch (a.ncols != b.nrows)");
        bsp_csr dA{}, dB{}, dC{};
        auto check = [](int rc) {
            if (rc != BSP_OK) throw std::runtime_error(bsp_last_error());
        };
        struct Frees {
            bsp_handle h;
            bsp_csr *a, *b, *c;
            bool alias;
            ~Frees() {
                bsp_csr_free(h, c);
                bsp_csr_free(h, a);
                if (!alias) bsp_csr_free(h, b);
            }
        };
        check(bsp_csr_upload(h, A->nrows, A->ncols, A->row_ptr, A->col_idx, A->values, &dA));
        const bool alias = (A == B) || (A->row_ptr == B->row_ptr && A->col_idx == B->col_idx &&
                                        A->values == B->values);
        Frees fr{h, &dA, &dB, &dC, alias};
        if (!alias)
            check(bsp_csr_upload(h, B->nrows, B->ncols, B->row_ptr, B->col_idx, B->values, &dB));
        const bsp_csr* pB = alias ? &dA : &dB;
        const int64_t n = A->nrows;
        int64_t products = 0;
        check(bsp_spgemm_products(h, &dA, pB, nullptr, &products));
        const char* fe = std::getenv("BSP_CHUNK_BYTES");  // per call (tests set it)
        const int64_t forced = fe ? std::atoll(fe) : int64_t{0};
        const int64_t budget =
            forced > 0 ? forced : static_cast<int64_t>(available_bytes(h)) / 2;
        if (12 * products + 8 * (n + 1) <= budget) {
            // one multiply (the bound fits)
            check(bsp_spgemm_rowwise(h, &dA, pB, &dC));
            C->nrows = dC.nrows;
            C->ncols = dC.ncols;
            C->nnz = dC.nnz;
            C->row_ptr = host_malloc<int64_t>(dC.nrows + 1);
            C->col_idx = host_malloc<int32_t>(dC.nnz);
            C->values = host_malloc<double>(dC.nnz);
            check(bsp_csr_download(h, &dC, C->row_ptr, C->col_idx, C->values));
            return;
        }
        // exact counts -> exact host C -> row chunks of <= budget bytes
        std::vector<int64_t> rp(n + 1, 0);
        {
            DBuf<int64_t> cnt(h, std::max<int64_t>(n, 1));
            check(bsp_spgemm_symbolic(h, &dA, pB, cnt.p));
            d2h(h, rp.data() + 1, cnt.p, n);
            sync(h);
        }
        for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
        const int64_t nnz = rp[n];
        int64_t* hrp = host_malloc<int64_t>(n + 1);
        int32_t* hci = host_malloc<int32_t>(nnz);
        double* hv = host_malloc<double>(nnz);
        std::memcpy(hrp, rp.data(), (n + 1) * sizeof(int64_t));
        C->nrows = n;
        C->ncols = B->ncols;
        C->nnz = nnz;
        C->row_ptr = hrp;
        C->col_idx = hci;
        C->values = hv;
        int32_t chunks = 0;
        int64_t products_done = 0;
        for (int64_t r0 = 0; r0 < n;) {
            int64_t r1 = r0 + 1;
            while (r1 < n && 12 * (rp[r1 + 1] - rp[r0]) + 8 * (r1 + 1 - r0) <= budget) ++r1;
            rowwise_multiply(h, &dA, pB, r0, r1, &dC, nullptr, nullptr);
            products_done += h->stats.products;
            require(dC.nnz == rp[r1] - rp[r0], "spgemm_rowwise_host: chunk count mismatch");
            if (dC.nnz > 0) {
                BSP_CUDA(cudaMemcpyAsync(hci + rp[r0], dC.col_idx, dC.nnz * sizeof(int32_t),
                                         cudaMemcpyDeviceToHost, h->stream));
                BSP_CUDA(cudaMemcpyAsync(hv + rp[r0], dC.values, dC.nnz * sizeof(double),
                                         cudaMemcpyDeviceToHost, h->stream));
            }
            sync(h);
            bsp_csr_free(h, &dC);
            dC = bsp_csr{};
            ++chunks;
            r0 = r1;
        }
        h->stats.products = products_done;
        h->stats.nnz_out = nnz;
        h->stats.chunks = chunks;
    });
}

// Partition cost of a row with P intermediate products (the rule
// distributed.product_split mirrors).
constexpr int64_t row_cost(int64_t P) {
    return P > 65536 ? 2 * P : P;
}

int bsp_partition_rows(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int32_t nparts,
                       int64_t* bounds_out) {
    return guarded([&] {
        require(nparts >= 1, "partition_rows: nparts must be >= 1");
        const int64_t n = A->nrows;
        DBuf<int64_t> prod(h, n + 1);
        int64_t total = 0;
        const int rc = bsp_spgemm_products(h, A, B, prod.p, &total);
        if (rc != BSP_OK) throw std::runtime_error(bsp_last_error());
        BSP_CUDA(cudaMemsetAsync(prod.p + n, 0, sizeof(int64_t), h->stream));
        // Split on a per-row cost, not the raw product count: a hub row's
        // products (> 65536 per row: dense windows, long A rows) cost about
        // twice the others'.  Fitted to the per-shard times of the 2/4/8-way
        // splits (tools/shard_projection.py, round 2): 21.2 / 19.7 / 40.7 ms per
        // 1e9 products of light / windowed / hub rows + 6 ms per shard (round
        // 1's tiles: windowed rows 2x, hub rows 3x).
        std::vector<int64_t> hp(n);
        d2h(h, hp.data(), prod.p, n);
        sync(h);
        std::vector<int64_t> hs(n + 1, 0);
        for (int64_t i = 0; i < n; ++i)
            hs[i + 1] = hs[i] + row_cost(hp[i]);
        bounds_out[0] = 0;
        for (int32_t g = 1; g < nparts; ++g) {
            // first row whose exclusive cost prefix reaches total*g/nparts
            const int64_t target = static_cast<int64_t>(
                (static_cast<__int128>(hs[n]) * g) / nparts);
            const int64_t r = std::lower_bound(hs.begin(), hs.end(), target) - hs.begin();
            bounds_out[g] = std::max(bounds_out[g - 1], std::min<int64_t>(r, n));
        }
        bounds_out[nparts] = n;
    });
}

#ifdef BSP_X_PHASE
// experiments only (tools/phase_times.py): the look-back tile's phase cycle counters
int bsp_debug_phases(unsigned long long* out32, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out32, bsp::g_phase, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(bsp::g_phase, z, sizeof(z));
    }
    return 0;
}
#endif

}  // extern "C"
