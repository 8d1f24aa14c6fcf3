// The ESC tile shared by the row, window and cluster kernels.
//
// Numeric (exact) tile: the products of a tile are expanded into shared
// memory in (k ascending, j ascending) order — one sorted run per
// contributing B-row segment — and sorted by column with equal columns kept
// in ascending k, so the per-column sums are formed exactly as the reference
// forms them (0.0 + p1 + p2 + ..., spgemm.hpp:92-97).  The sort is chosen per
// tile: a counting sort on the column's top bits with an expansion-index
// tie-break (count_sort_tile), a bottom-up merge-path merge of the runs (ties
// from the left run, i.e. the smaller k), an MSD counting sort for small
// tiles, or a stable CUB block radix sort.
//
// Symbolic tile (rowwise.cu) = distinct-column count through an open-addressed
// smem hash (atomicCAS insert), the GPU form of HashAccumulator::insert_key
// (hash_accumulator.hpp:48-54); col_hash below.
#pragma once

#include "esc.cuh"

#include <type_traits>

#include <cub/block/block_radix_sort.cuh>

namespace bsp {

// BSP_X_PHASE (tools/build_variant.py, experiments only): thread 0 of every
// look-back window tile adds the cycles between consecutive phase marks to
// g_phase[] (tools/phase_times.py prints the share of each phase).
#ifdef BSP_X_PHASE
static __device__ unsigned long long g_phase[32];
static __device__ long long g_phase_last[1 << 22];
static __device__ long long g_phase_t0[1 << 22];   // tile start
static __device__ int g_phase_cls[1 << 22];        // tile's segment-count class
__device__ __forceinline__ void phase_mark(int i) {
    if (threadIdx.x == 0) {
        long long& last = g_phase_last[blockIdx.x & ((1 << 22) - 1)];
        if (last != 0) {
            const long long t = clock64();
            atomicAdd(&g_phase[i], static_cast<unsigned long long>(t - last));
            last = t;
        }
    }
}
#define PH(i) phase_mark(i)
#else
#define PH(i)
#endif

// Padded shared-memory index: one pad word per 32 keeps the per-thread
// contiguous chunks of the merge (thread t owns [t*E, t*E+E)) on distinct
// banks (ncu: 42% of shared wavefronts were bank conflicts without it).
__device__ __forceinline__ int PADI(int i) { return i + (i >> 5); }

// VALB: bytes of the value buffer (the look-back tile's second form keeps only a
// B offset and a segment index per product there: 6 bytes instead of 8);
// RBO: radix digit bits override (smaller digits = smaller sort storage).
template <int T, int CAPM, int VALB = 8 * CAPM, int RBO = 0>
struct MergeShared {
    static constexpr int NP = CAPM + CAPM / 32 + 1;
    // radix digit bits: CUB's rank storage is T x 2^RB / 2 words whatever the
    // tile size, so 256-thread tiles of <= 3072 products (sized for 3-4
    // CTAs/SM) use 5-bit digits (16 KB), the 4096 tile 6-bit digits
    // (the small tiles rarely reach the radix sort, and its storage decided their
    // occupancy: <64,512> 18.1 -> 14.0 KB = 15 CTAs per SM instead of 12,
    // <32,128> 7.4 -> 4.4 KB = 32 instead of 27)
    static constexpr int RB = RBO ? RBO : (T <= 32 ? 4 : ((T <= 64 || (T >= 128 && CAPM <= 3072)) ? 5 : 6));
    using RSort = cub::BlockRadixSort<uint32_t, T, CAPM / T, uint16_t, RB>;
    // run offsets: tiles with more runs than this use the radix sort
    static constexpr int MAXRUNS = CAPM < 1024 ? CAPM : 1024;
    // counters: MSD buckets (small tiles) or the reduction's (row, warp) heads
    static constexpr int NHIST = CAPM <= 512 ? CAPM / 2 : ((CAPM + T - 1) / T) * (T / 32);
    // counting sort: buckets on the top column bits (about one product each)
    static constexpr int NB = CAPM >= 3072 ? 4096 : (CAPM >= 2048 ? 2048 : CAPM / 2);
    static constexpr int LNB = 31 - __builtin_clz(static_cast<unsigned>(NB));
    // expansion-only state (compacted segments of the current chunk)
    struct Ex {
        int64_t pstart[T];
        int32_t poff[T + 1];
        double pav[T];
    };
    // ... lives in the union (over key1, idle during the expansion) when it fits
    static constexpr bool EX_IN_U = sizeof(Ex) <= sizeof(uint32_t) * NP;
    // buffer 0 (also the radix-sort input/output)
    uint32_t key0[NP];
    uint16_t idx0[NP];
    uint16_t ro0[MAXRUNS + 2];
    alignas(16) double val[VALB / 8];  // 16-byte aligned: a bulk-copy destination (cluster.cu)
    // buffer 1 of the merge, aliased with the radix sort's temp storage, the
    // counting sort's arrays and the expansion state
    union U {
        struct B1 {
            uint32_t key1[NP];
            uint16_t idx1[NP];  // also the expansion's run id per product
            uint16_t ro1[MAXRUNS + 2];
        } m;
        typename RSort::TempStorage sort;
        struct alignas(16) CS {
            uint32_t packed[CAPM + 4]; // per bucketed slot: (column - min) << IB | index,
                                       // or (low column bits << 16 | index) + bucket[]
            uint32_t cnt[NB / 2 + 1];  // 16-bit bucket counts, then bucket starts
            uint16_t bucket[CAPM];     // bucket of each bucketed slot (wide tiles)
        } c;
        Ex x;
    } u;
    struct NoEx {};
    std::conditional_t<EX_IN_U, NoEx, Ex> xo;
    uint32_t hist[NHIST];
    __device__ __forceinline__ uint32_t* key(int b) { return b ? u.m.key1 : key0; }
    __device__ __forceinline__ uint16_t* idx(int b) { return b ? u.m.idx1 : idx0; }
    __device__ __forceinline__ uint16_t* ro(int b) { return b ? u.m.ro1 : ro0; }
    __device__ __forceinline__ Ex& ex() {
        if constexpr (EX_IN_U) return u.x; else return xo;
    }
    typename cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>::TempStorage scan;
    int nruns;
};

// Largest power of two < n (0 for n <= 1): the first step of find_run.
__device__ __forceinline__ int run_search_step(int n) {
    return n > 1 ? 1 << (31 - __clz(n - 1)) : 0;
}

// Index q of the run holding element e: the largest q < n with poff[q] <= e
// (poff[0] == 0).  Fixed trip count, so unrolled callers overlap their loads.
__device__ __forceinline__ int find_run(const int32_t* poff, int n, int step, int e) {
    int q = 0;
    for (int st = step; st > 0; st >>= 1)
        if (q + st < n && poff[q + st] <= e) q += st;
    return q;
}

// Expand the products of (row, [c0, c1)) in (k, j) order; every non-empty
// B-row segment becomes one sorted run.  Returns the product count.
// Asynchronous global -> shared copies (sm_80+ LDGSTS), 4 and 8 bytes.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Bulk (TMA engine) global -> shared copies completing on an mbarrier
// (sm_90+ cp.async.bulk, SASS UBLKCP; the wait is SYNCS).  Source, destination
// and size must be multiples of 16 bytes: callers copy the 16-byte-aligned
// superset of a B-row segment and mask the slack.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int arrivals) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(arrivals)
                 : "memory");
    // make the initialised barrier visible to the async proxy
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// Generic-proxy accesses to shared memory ordered before later async-proxy
// (bulk copy) accesses to the same locations.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// Adds `bytes` to the barrier's pending transaction count (no arrival).
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    unsigned done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Warp-contiguous split of `ct` flattened run elements over `nwarps` warps
// (slices rounded to 32): this warp covers [e0, we); qa is the run holding
// element e0 (warp-uniform).
__device__ __forceinline__ void warp_slice(const int32_t* poff, int nr, int ct, int nwarps,
                                           int& e0, int& we, int& qa) {
    const int warp = threadIdx.x >> 5;
    const int ew = (((ct + nwarps - 1) / nwarps) + 31) & ~31;
    e0 = min(ct, warp * ew);
    we = min(ct, e0 + ew);
    qa = e0 < we ? find_run(poff, nr, run_search_step(nr), e0) : 0;
}

// Run of element e0 + lane, for 32 consecutive elements at once: lane l reads
// the start of run qa + 1 + l, the starts that fall inside (e0, e0 + 32) are
// OR-reduced into one mask (runs are non-empty, so at most 31 of them), and
// each lane counts the starts at or below its element.  Advances qa to the
// run holding e0 + 32.  One smem load per lane instead of a per-lane walk
// over every run boundary (runs of heavy-row windows average a few products).
// Warp-uniform: all 32 lanes call it.
__device__ __forceinline__ int warp_runs(const int32_t* poff, int nr, int e0, int& qa) {
    const int lane = threadIdx.x & 31;
    const int idx = qa + 1 + lane;
    const int rel = (idx <= nr ? poff[idx] : 0x3fffffff) - e0;
    const unsigned mask = __reduce_or_sync(0xffffffffu, rel > 0 && rel < 32 ? 1u << rel : 0u);
    const int my = qa + __popc(mask & (0xffffffffu >> (31 - lane)));
    qa += __popc(mask) + (__any_sync(0xffffffffu, rel == 32) ? 1 : 0);
    return my;
}

template <int T, int CAPM, bool VALUES, int VB, int RBO>
__device__ __forceinline__ int expand_runs(const Mats& m, int32_t row, int32_t c0, int32_t c1,
                                           bool full, MergeShared<T, CAPM, VB, RBO>& s,
                                           int64_t wsofs = -1, int wwi = 0, int64_t wrs = -1,
                                           int64_t wd = 0, bool defer = false) {
    const int tid = threadIdx.x;
    // windows carry their A row range (one dependent load less)
    const int64_t rs = wrs >= 0 ? wrs : m.arp[row];
    const int64_t re = wrs >= 0 ? wrs + wd : m.arp[row + 1];
    int total = 0, nruns = 0;
    auto& x = s.ex();
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
            if (VALUES) av = __ldg(m.aval + p);
        }
        // packed scan: low 16 bits offset, high 16 bits run index
        const int packed = len | ((len > 0) << 16);
        int off, agg;
        cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(packed, off, agg);
        // compact the non-empty segments of this chunk (run order = k order)
        const int r = off >> 16;
        if (len > 0) {
            if (nruns + r < MergeShared<T, CAPM, VB, RBO>::MAXRUNS)
                s.ro(0)[nruns + r] = static_cast<uint16_t>(total + (off & 0xffff));
            x.pstart[r] = start;
            x.poff[r] = off & 0xffff;
            if (VALUES) x.pav[r] = av;
        }
        const int nr = agg >> 16, ct = agg & 0xffff;
        if (tid == 0) x.poff[nr] = ct;
        __syncthreads();
        PH(1);
        // Gather: warp w takes a contiguous slice of the chunk's products, its
        // lanes consecutive ones (coalesced), and copies each product's B
        // column and value straight into the tile with cp.async — no register
        // round trip, so every load of the slice is in flight at once.  The
        // run of each product is kept in the (idle) merge buffer for the
        // fix-up pass.
        uint16_t* rid = s.idx(1);
        {
            int e0, we, qa;
            warp_slice(x.poff, nr, ct, T / 32, e0, we, qa);
            for (; e0 < we; e0 += 32) {
                const int q = warp_runs(x.poff, nr, e0, qa);
                const int e = e0 + (threadIdx.x & 31);
                if (e < we) {
                    const int64_t src = x.pstart[q] + (e - x.poff[q]);
                    const int g = total + e;
                    cp_async4(&s.key(0)[PADI(g)], m.bcol + src);
                    if (VALUES) {
                        cp_async8(&s.val[g], m.bval + src);
                        rid[g] = static_cast<uint16_t>(q);
                    }
                }
            }
            cp_async_wait_all();
        }
        __syncthreads();
        PH(2);
        // fix-up: product a_ik * b_kj; window-relative key and position
        // (deferred: sort_tile applies them only on the paths that read them)
        for (int e = tid; e < ct; e += T) {
            const int g = total + e;
            if (!defer) {
                s.key(0)[PADI(g)] -= static_cast<uint32_t>(c0);
                s.idx(0)[PADI(g)] = static_cast<uint16_t>(g);
            }
            if (VALUES) s.val[g] = __dmul_rn(x.pav[rid[g]], s.val[g]);
        }
        total += ct;
        nruns += nr;
        __syncthreads();
        PH(3);
    }
    if (tid == 0) {
        if (nruns <= MergeShared<T, CAPM, VB, RBO>::MAXRUNS) s.ro(0)[nruns] = static_cast<uint16_t>(total);
        s.nruns = nruns;
    }
    __syncthreads();
    PH(4);
    return total;
}

// Keys-only expansion for the look-back window tile (esc_window_lb2_kernel):
// the tile's output count depends only on the columns, so only they are
// gathered before the sort; product g's B offset goes to src[g] and its A entry
// (segment index within the row) to seg[g], both in the (still idle) value
// buffer, and the values are fetched after the tile has published its count
// (reduce_lb2).  The column copies (cp.async) are waited for once, after the
// last chunk.  Requires nnz(B) < 2^32.
template <int T, int CAPM, int VB, int RBO>
__device__ __forceinline__ int expand_keys(const Mats& m, int32_t c0, int32_t c1,
                                           MergeShared<T, CAPM, VB, RBO>& s, int64_t wsofs, int wwi,
                                           int64_t wrs, int64_t wd) {
    const int tid = threadIdx.x;
    const int64_t rs = wrs, re = wrs + wd;
    // compact value buffer (VB < 8 bytes per product): 16-bit segment indices
    // (rows of at most 65535 entries; the caller routes longer rows elsewhere)
    constexpr bool SEG16 = VB < 8 * CAPM;
    uint32_t* src = reinterpret_cast<uint32_t*>(s.val);
    uint32_t* seg = src + CAPM;
    uint16_t* seg16 = reinterpret_cast<uint16_t*>(src + CAPM);
    int total = 0, nruns = 0;
    auto& x = s.ex();
    uint32_t* pseg = reinterpret_cast<uint32_t*>(x.pav);  // segment index of each compacted run
    for (int64_t pc = rs; pc < re; pc += T) {
        const int64_t p = pc + tid;
        int len = 0;
        int64_t start = 0;
        if (p < re) {
            int64_t b0, b1;
            segment_range(m, false, wsofs, wwi, p, rs, re - rs, c0, c1, b0, b1);
            start = b0;
            len = static_cast<int>(b1 - b0);
        }
        const int packed = len | ((len > 0) << 16);
        int off, agg;
        cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(packed, off, agg);
        const int r = off >> 16;
        if (len > 0) {
            if (nruns + r < MergeShared<T, CAPM, VB, RBO>::MAXRUNS)
                s.ro(0)[nruns + r] = static_cast<uint16_t>(total + (off & 0xffff));
            x.pstart[r] = start;
            x.poff[r] = off & 0xffff;
            pseg[r] = static_cast<uint32_t>(p - rs);
        }
        const int nr = agg >> 16, ct = agg & 0xffff;
        if (tid == 0) x.poff[nr] = ct;
        __syncthreads();
        PH(1);
        {
            int e0, we, qa;
            warp_slice(x.poff, nr, ct, T / 32, e0, we, qa);
            for (; e0 < we; e0 += 32) {
                const int q = warp_runs(x.poff, nr, e0, qa);
                const int e = e0 + (threadIdx.x & 31);
                if (e < we) {
                    const int64_t sa = x.pstart[q] + (e - x.poff[q]);
                    const int g = total + e;
                    cp_async4(&s.key(0)[PADI(g)], m.bcol + sa);
                    src[g] = static_cast<uint32_t>(sa);
                    if constexpr (SEG16) seg16[g] = static_cast<uint16_t>(pseg[q]);
                    else seg[g] = pseg[q];
                }
            }
        }
        total += ct;
        nruns += nr;
        __syncthreads();  // the next chunk rewrites the compacted runs
        PH(2);
    }
    cp_async_wait_all();
    if (tid == 0) {
        if (nruns <= MergeShared<T, CAPM, VB, RBO>::MAXRUNS) s.ro(0)[nruns] = static_cast<uint16_t>(total);
        s.nruns = nruns;
    }
    __syncthreads();
    PH(4);
    return total;
}

// Bottom-up stable merge of the runs in key[0]/idx[0]; returns the buffer
// holding the sorted result.
template <int T, int CAPM, int VB, int RBO>
__device__ __forceinline__ int merge_runs(MergeShared<T, CAPM, VB, RBO>& s, int total,
                                          int max_levels = 64) {
    const int tid = threadIdx.x;
    int R = s.nruns;
    int b = 0;
    const int E = (total + T - 1) / T;
    for (int level = 0; R > 1 && level < max_levels; ++level) {
        const int Rn = (R + 1) >> 1;
        const uint16_t* ro = s.ro(b);
        uint16_t* rn = s.ro(b ^ 1);
        for (int i = tid; i <= Rn; i += T) rn[i] = (i < Rn) ? ro[2 * i] : static_cast<uint16_t>(total);
        __syncthreads();
        const uint32_t* K = s.key(b);
        const uint16_t* X = s.idx(b);
        uint32_t* KO = s.key(b ^ 1);
        uint16_t* XO = s.idx(b ^ 1);
        int o = min(total, tid * E);
        const int oe = min(total, o + E);
        while (o < oe) {
            // pair i: rn[i] <= o < rn[i+1]
            int lo = 0, hi = Rn - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (rn[mid] <= o) lo = mid; else hi = mid - 1;
            }
            const int i = lo;
            const int xs = ro[2 * i];
            const int xe = (2 * i + 1 <= R) ? ro[2 * i + 1] : total;
            const int ye = (2 * i + 2 <= R) ? ro[2 * i + 2] : xe;
            const int k = o - xs;
            const int kend = min(oe, ye) - xs;
            int a = max(0, k - (ye - xe)), a_hi = min(k, xe - xs);
            while (a < a_hi) {
                const int mid = (a + a_hi) >> 1;
                if (K[PADI(xs + mid)] <= K[PADI(xe + k - 1 - mid)]) a = mid + 1; else a_hi = mid;
            }
            int xi = xs + a, yi = xe + (k - a);
            uint32_t kx = xi < xe ? K[PADI(xi)] : 0xffffffffu;
            uint32_t ky = yi < ye ? K[PADI(yi)] : 0xffffffffu;
            for (int t = k; t < kend; ++t) {
                const bool takex = (yi >= ye) || (xi < xe && kx <= ky);
                if (takex) {
                    KO[PADI(xs + t)] = kx;
                    XO[PADI(xs + t)] = X[PADI(xi)];
                    ++xi;
                    kx = xi < xe ? K[PADI(xi)] : 0xffffffffu;
                } else {
                    KO[PADI(xs + t)] = ky;
                    XO[PADI(xs + t)] = X[PADI(yi)];
                    ++yi;
                    ky = yi < ye ? K[PADI(yi)] : 0xffffffffu;
                }
            }
            o = xs + kend;
        }
        __syncthreads();
        b ^= 1;
        R = Rn;
    }
    return b;
}

// Stable block radix sort of the expanded tile by column (CUB, 6-bit digits);
// chosen instead of merge_runs when the merge tree would need more levels
// than the radix sort needs passes (windows of heavy rows carry hundreds of
// short runs).  Result left in buffer 0.
template <int T, int CAPM, int VB, int RBO>
__device__ __forceinline__ void radix_sort_tile(MergeShared<T, CAPM, VB, RBO>& s, int total, int bits) {
    constexpr int I = CAPM / T;
    const int tid = threadIdx.x;
    uint32_t k[I];
    uint16_t v[I];
    const uint32_t pad = (bits >= 32) ? 0xffffffffu : ((1u << bits) - 1u);
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const int e = tid * I + i;
        k[i] = e < total ? s.key0[PADI(e)] : pad;
        v[i] = e < total ? s.idx0[PADI(e)] : static_cast<uint16_t>(0);
    }
    __syncthreads();
    typename MergeShared<T, CAPM, VB, RBO>::RSort(s.u.sort).Sort(k, v, 0, bits);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < I; ++i) {
        s.key0[PADI(tid * I + i)] = k[i];
        s.idx0[PADI(tid * I + i)] = v[i];
    }
    __syncthreads();
}

// MSD counting sort: products are bucketed by the top bits of their column
// (smem atomics: histogram, scan, scatter), then every bucket — a handful of
// entries — is insertion-sorted by (column, expansion index).  The index
// tie-break restores ascending k for equal columns, so the run sums stay
// exact.  Result in buffer 1.
// Returns false (tile untouched) when a bucket holds more than MSD_MAXB
// entries (skewed columns or many duplicates): the caller then merges/radixes.
constexpr int MSD_MAXB = 24;

template <int T, int CAPM, int VB, int RBO>
__device__ __forceinline__ bool msd_sort_tile(MergeShared<T, CAPM, VB, RBO>& s, int total, uint32_t width) {
    constexpr int NB = CAPM / 2;
    constexpr int LNB = 31 - __builtin_clz(static_cast<unsigned>(NB));
    constexpr int PER = NB / T;
    const int tid = threadIdx.x;
    const int bits = bit_length(width > 0 ? width - 1 : 0);
    const int sh = bits > LNB ? bits - LNB : 0;
    __shared__ int s_bmax;
    if (tid == 0) s_bmax = 0;
    for (int b = tid; b < NB; b += T) s.hist[b] = 0u;
    __syncthreads();
    int mymax = 0;
    for (int e = tid; e < total; e += T) {
        const uint32_t c = atomicAdd(&s.hist[s.key0[PADI(e)] >> sh], 1u) + 1u;
        mymax = max(mymax, static_cast<int>(c));
    }
    if (mymax > MSD_MAXB) atomicMax(&s_bmax, mymax);
    __syncthreads();
    if (s_bmax > MSD_MAXB) return false;
    uint32_t loc[PER];
    int run = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        loc[i] = s.hist[tid * PER + i];
        run += static_cast<int>(loc[i]);
    }
    int base, agg;
    cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(run, base, agg);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        s.hist[tid * PER + i] = static_cast<uint32_t>(base);
        base += static_cast<int>(loc[i]);
    }
    __syncthreads();
    uint32_t* K1 = s.u.m.key1;
    uint16_t* X1 = s.u.m.idx1;
    for (int e = tid; e < total; e += T) {
        const uint32_t k = s.key0[PADI(e)];
        const uint32_t pos = atomicAdd(&s.hist[k >> sh], 1u);
        K1[PADI(pos)] = k;
        X1[PADI(pos)] = s.idx0[PADI(e)];
    }
    __syncthreads();
    // hist[b] is now the end of bucket b
    for (int b = tid; b < NB; b += T) {
        const int lo = b == 0 ? 0 : static_cast<int>(s.hist[b - 1]);
        const int hi = static_cast<int>(s.hist[b]);
        for (int i = lo + 1; i < hi; ++i) {
            const uint32_t kk = K1[PADI(i)];
            const uint16_t xx = X1[PADI(i)];
            int j = i - 1;
            while (j >= lo) {
                const uint32_t kj = K1[PADI(j)];
                if (kj < kk || (kj == kk && X1[PADI(j)] < xx)) break;
                K1[PADI(j + 1)] = kj;
                X1[PADI(j + 1)] = X1[PADI(j)];
                --j;
            }
            K1[PADI(j + 1)] = kk;
            X1[PADI(j + 1)] = xx;
        }
    }
    __syncthreads();
    return true;
}

// Counting sort for tiles whose columns are nearly distinct (cf ~ 1): one
// smem-atomic pass buckets the products on the top bits of the column
// relative to the tile's own [min, max] column range (NB buckets, about one
// product each; 16-bit counters packed two per word), a scan lays the buckets
// out, and each bucketed slot's final position is its bucket start plus the
// number of bucket members with a smaller (column, expansion index) — the
// index tie-break puts equal columns in ascending k, so the run sums stay
// exact (spgemm.hpp:92-97).  The ranking runs over the bucketed slots, so the
// lanes of a warp mostly share one bucket and the loop trip count (the bucket
// size) does not diverge.  Narrow tiles (column range + index bits <= 32)
// rank one packed word per slot with 4-wide vector compares; wide ones keep
// (low column bits, index) words plus a bucket id per slot.
// Composite keys (cbits > 0: key = member << cbits | column, the cluster
// tiles) give each of the 2^lk member slots NB / 2^lk buckets over the
// columns' range, so the order stays member-major.
// The ranking costs sum(bucket size^2) compares (= sum over products of
// 2 x rank-in-bucket + 1, known after the bucketing pass).  Tiles where that
// exceeds `max_cost` x products, whose bucket width exceeds 2^16 columns, or
// with a bucket of more than CS_MAXB products (duplicate-heavy columns)
// return false with buffer 0 untouched (merge / radix instead).
// kofs >= 0: the expansion deferred its fix-up (absolute columns, idx0 unset).
// Result in buffer 0.
constexpr int CS_MAXB = 128;

template <int T, int CAPM, int VB, int RBO>
__device__ __forceinline__ bool count_sort_tile(MergeShared<T, CAPM, VB, RBO>& s, int total, uint32_t width,
                                                int cbits, int max_cost, int kofs = -1) {
    using S = MergeShared<T, CAPM, VB, RBO>;
    constexpr int NB = S::NB, LNB = S::LNB, PER = NB / T, I = (CAPM + T - 1) / T;
    static_assert(PER % 2 == 0 || PER == 1, "bucket split");
    const int tid = threadIdx.x;
    const uint32_t cmask = cbits > 0 ? (1u << cbits) - 1u : 0xffffffffu;
    const int lk = cbits > 0 ? bit_length((width >> cbits) > 1 ? (width >> cbits) - 1 : 0) : 0;
    if (lk > LNB) return false;
    __shared__ int s_over, s_cost;
    __shared__ uint32_t s_min, s_max;
    uint32_t* cnt2 = s.u.c.cnt;  // NB 16-bit counters, two per word
    uint16_t* cnt = reinterpret_cast<uint16_t*>(s.u.c.cnt);
    uint32_t* pk = s.u.c.packed;
    uint16_t* bk = s.u.c.bucket;
    for (int b = tid; b < NB / 2 + 1; b += T) cnt2[b] = 0u;
    if (tid == 0) {
        s_over = 0;
        s_cost = 0;
        s_min = 0xffffffffu;
        s_max = 0u;
    }
    uint32_t kr[I], rr[I];
    uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const int e = i * T + tid;
        if (e < total) {
            kr[i] = s.key0[PADI(e)];
            mn = min(mn, kr[i] & cmask);
            mx = max(mx, kr[i] & cmask);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    __syncthreads();  // counters and bounds initialised
    if ((tid & 31) == 0) {
        atomicMin(&s_min, mn);
        atomicMax(&s_max, mx);
    }
    __syncthreads();
    PH(5);
    const uint32_t cmin = s_min;
    const int cb = LNB - lk;  // column bucket bits per member slot
    const int cw = bit_length(s_max - cmin);
    const int sh = cw > cb ? cw - cb : 0;
    if (sh > 16) return false;
    bool over = false;
    int cost = 0;
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const int e = i * T + tid;
        if (e < total) {
            const uint32_t b = (cbits > 0 ? (kr[i] >> cbits) << cb : 0u) |
                               (((kr[i] & cmask) - cmin) >> sh);
            rr[i] = (atomicAdd(&cnt2[b >> 1], 1u << (16 * (b & 1))) >> (16 * (b & 1))) & 0xffffu;
            over |= rr[i] >= CS_MAXB;
            cost += 2 * static_cast<int>(rr[i]) + 1;
        }
    }
    if (over) s_over = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cost += __shfl_xor_sync(0xffffffffu, cost, o);
    if ((tid & 31) == 0) atomicAdd(&s_cost, cost);
    __syncthreads();
    PH(6);
    if (s_over || s_cost > max_cost * total) return false;
    uint32_t loc[PER];
    int run = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        loc[j] = cnt[tid * PER + j];
        run += static_cast<int>(loc[j]);
    }
    int base, agg;
    cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(run, base, agg);
    __syncthreads();  // all counters read before they become offsets
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        cnt[tid * PER + j] = static_cast<uint16_t>(base);
        base += static_cast<int>(loc[j]);
    }
    if (tid == 0) cnt[NB] = static_cast<uint16_t>(total);
    __syncthreads();
    PH(7);
    const uint32_t lm = (1u << sh) - 1u;
    // Narrow row tiles: the whole (column - min, index) fits one 32-bit word,
    // globally ordered and unique, so a slot's rank is the count of smaller
    // words from its bucket start rounded down to 4 (lower buckets hold only
    // smaller words, higher ones and the pad only larger) — 4 per 16-byte load,
    // no bucket array, no tie path.
    constexpr int IB = 32 - __builtin_clz(static_cast<unsigned>(CAPM - 1));
    if (lk + cw + IB <= 32) {
        // (member, column - min, index) in one word: member-major like the
        // buckets (cluster tiles; member = 0 for rows and windows)
#pragma unroll
        for (int i = 0; i < I; ++i) {
            const int e = i * T + tid;
            if (e < total) {
                const uint32_t mem = cbits > 0 ? kr[i] >> cbits : 0u;
                const uint32_t rel = (kr[i] & cmask) - cmin;
                const uint32_t b = (mem << cb) | (rel >> sh);
                const uint32_t ix = kofs >= 0 ? static_cast<uint32_t>(e) : s.idx0[PADI(e)];
                pk[cnt[b] + static_cast<int>(rr[i])] = (((mem << cw) | rel) << IB) | ix;
            }
        }
        if (tid < 4) pk[total + tid] = 0xffffffffu;
        __syncthreads();
        PH(8);
        const uint32_t im = (1u << IB) - 1u;
        const uint32_t rm = (1u << cw) - 1u;  // cw <= 32 - IB
        for (int q = tid; q < total; q += T) {
            const uint32_t v = pk[q];
            const uint32_t mr = v >> IB;
            const uint32_t mem = mr >> cw, rel = mr & rm;
            const uint32_t b = (mem << cb) | (rel >> sh);
            const int lo = cnt[b], hi = cnt[b + 1];
            int c = lo;
            if (hi - lo > 1) {
                c = lo & ~3;
#if defined(BSP_X_RANKPIPE)
                // next group loaded before the current one is counted
                int j = c;
                uint4 w = *reinterpret_cast<const uint4*>(pk + j);
                for (j += 4; j < hi; j += 4) {
                    const uint4 wn = *reinterpret_cast<const uint4*>(pk + j);
                    c += (w.x < v) + (w.y < v) + (w.z < v) + (w.w < v);
                    w = wn;
                }
                c += (w.x < v) + (w.y < v) + (w.z < v) + (w.w < v);
#elif defined(BSP_X_RANK8)
                for (int j = c; j < hi; j += 8) {
                    const uint4 w = *reinterpret_cast<const uint4*>(pk + j);
                    uint4 w2 = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                    if (j + 4 < hi) w2 = *reinterpret_cast<const uint4*>(pk + j + 4);
                    c += (w.x < v) + (w.y < v) + (w.z < v) + (w.w < v);
                    c += (w2.x < v) + (w2.y < v) + (w2.z < v) + (w2.w < v);
                }
#else
                for (int j = c; j < hi; j += 4) {
                    const uint4 w = *reinterpret_cast<const uint4*>(pk + j);
                    c += (w.x < v) + (w.y < v) + (w.z < v) + (w.w < v);
                }
#endif
            }
            const uint32_t col = rel + cmin - static_cast<uint32_t>(kofs > 0 ? kofs : 0);
            s.key0[PADI(c)] = cbits > 0 ? (mem << cbits) | col : col;
            s.idx0[PADI(c)] = static_cast<uint16_t>(v & im);
        }
        __syncthreads();
        PH(9);
        return true;
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const int e = i * T + tid;
        if (e < total) {
            const uint32_t b = (cbits > 0 ? (kr[i] >> cbits) << cb : 0u) |
                               (((kr[i] & cmask) - cmin) >> sh);
            const int pos = cnt[b] + static_cast<int>(rr[i]);
            const uint32_t ix = kofs >= 0 ? static_cast<uint32_t>(e) : s.idx0[PADI(e)];
            pk[pos] = (((kr[i] & cmask) - cmin) & lm) << 16 | ix;
            bk[pos] = static_cast<uint16_t>(b);
        }
    }
    __syncthreads();
    const uint32_t bm = (1u << cb) - 1u;
    for (int q = tid; q < total; q += T) {
        const uint32_t b = bk[q];
        const int lo = cnt[b], hi = cnt[b + 1];
        const uint32_t v = pk[q];
        int c = lo;
        if (hi - lo > 1)
            for (int j = lo; j < hi; ++j) c += pk[j] < v;
        const uint32_t col = cmin + (((b & bm) << sh) | (v >> 16)) - (kofs > 0 ? kofs : 0);
        s.key0[PADI(c)] = cbits > 0 ? ((b >> cb) << cbits) | col : col;
        s.idx0[PADI(c)] = static_cast<uint16_t>(v & 0xffffu);
    }
    __syncthreads();
    PH(10);
    return true;
}

// Sort the expanded tile: merge of presorted runs, or radix when cheaper
// (csort > 0: try the counting sort first when the merge tree is >= 3 levels
// deep — or only in place of the radix sort (radix_only) — with csort as its
// cost cap).
template <int T, int CAPM, int VB, int RBO>
__device__ __forceinline__ int sort_tile(MergeShared<T, CAPM, VB, RBO>& s, int total, uint32_t width,
                                         int csort = 0, int cbits = 0,
                                         bool radix_only = false, int kofs = -1) {
    const int R = s.nruns;
    const int levels = R > 1 ? 32 - __clz(R - 1) : 0;
    // kofs >= 0: the expansion deferred its fix-up (keys absolute, idx0 not
    // set); the counting sort reads them as they are, the other sorts after
    // this pass.
    auto prep = [&] {
        if (kofs < 0) return;
        for (int e = threadIdx.x; e < total; e += T) {
            s.key0[PADI(e)] -= static_cast<uint32_t>(kofs);
            s.idx0[PADI(e)] = static_cast<uint16_t>(e);
        }
        __syncthreads();
    };
    // MSD counting sort when the columns spread evenly over the buckets (cfg2:
    // 1.3x faster tiles); skewed / duplicate-heavy tiles fall through.
    // (measured: small tiles only; cfg4/cfg5's larger tiles are slower with it)
    if constexpr (CAPM <= 512)
        if (levels >= 2) {
            prep();
            kofs = -1;
            if (msd_sort_tile<T, CAPM>(s, total, width)) return 1;
        }
    // pad key = 2^bits - 1 >= every key (<= width-1); pads sit after `total`
    // and the sort is stable, so real entries keep the first `total` slots.
    const int bits = bit_length(width > 1 ? width - 1 : 1);
    constexpr int RB = MergeShared<T, CAPM, VB, RBO>::RB;
    const int passes = (bits + RB - 1) / RB;
    // measured: cfg4 (5 levels vs 4 passes) prefers merge
    const bool radix = levels > passes + 1 || R > MergeShared<T, CAPM, VB, RBO>::MAXRUNS;
    if (csort > 0 && levels >= 3 && (radix || !radix_only) &&
        count_sort_tile<T, CAPM>(s, total, width, cbits, csort, kofs))
        return 0;
    prep();
    if (radix) {
        radix_sort_tile<T, CAPM>(s, total, bits);
        PH(11);
        return 0;
    }
    const int mb = merge_runs<T, CAPM>(s, total);
    PH(12);
    return mb;
}

// Single-pass output placement (decoupled look-back, the CUB single-pass scan
// pattern): tile t of a list claimed in list order publishes its output count
// as an "aggregate", then one warp walks its predecessors 32 at a time,
// summing aggregates until it meets an inclusive prefix, and publishes its own
// inclusive prefix.  Status word = flag << 62 | value (one 64-bit store, so a
// reader never sees a flag without its value).  Tiles are claimed with an
// atomic counter, so every predecessor is owned by a running CTA: the spin
// always ends.  Returns the exclusive prefix (all 32 lanes call it).
struct LbCtx {
    int* counter;                 // next tile to claim
    unsigned long long* status;   // per tile: 0 = not ready, 1 = aggregate, 2 = prefix
};
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62,
                             LB_VAL = (1ull << 62) - 1ull;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Relaxed (not release): a status word carries its own value, nothing else is
// published with it, so no fence is needed (a release store here stalled the
// publishing tile's barrier: 11 % of the window tile's stall samples).
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

// Publish tile t's aggregate (one lane; t == 0 publishes its prefix).
__device__ __forceinline__ void lookback_publish(unsigned long long* st, int t, long long agg) {
    st_release_u64(st + t, (t == 0 ? LB_PRE : LB_AGG) | static_cast<unsigned long long>(agg));
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Exclusive prefix of tile t (after lookback_publish), then its inclusive
// prefix published.  All 32 lanes of one warp call it.  Each step inspects 128
// predecessors (4 independent loads per lane; entry distance = 32u + lane) and
// waits only for the not-yet-published ones closer than the nearest inclusive
// prefix.
__device__ __forceinline__ long long lookback_warp(unsigned long long* st, int t, long long agg) {
    const int lane = threadIdx.x & 31;
    if (t == 0) return 0;
    long long excl = 0;
    for (int j = t - 1;; j -= 128) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = 0;
        int pre_d, zero_d;
        for (;;) {
            pre_d = 128;
            zero_d = 128;
#pragma unroll
            for (int u = 3; u >= 0; --u) {
                const int idx = j - 32 * u - lane;
                if ((v[u] >> 62) == 0) v[u] = idx >= 0 ? ld_relaxed_u64(st + idx) : LB_PRE;
                const unsigned pm = __ballot_sync(0xffffffffu, (v[u] >> 62) == 2);
                const unsigned zm = __ballot_sync(0xffffffffu, (v[u] >> 62) == 0);
                if (pm) pre_d = 32 * u + __ffs(pm) - 1;
                if (zm) zero_d = 32 * u + __ffs(zm) - 1;
            }
            if (zero_d > pre_d || zero_d == 128) break;
        }
        long long x = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (32 * u + lane <= pre_d) x += static_cast<long long>(v[u] & LB_VAL);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        excl += x;
        if (pre_d < 128) break;
    }
    if (lane == 0) st_release_u64(st + t, LB_PRE | static_cast<unsigned long long>(excl + agg));
    return excl;
}

// After the sort: sum every run of equal columns left to right from 0.0
// (ascending k — the reference's order, spgemm.hpp:92-97) and write
// (column + kofs, sum) to ccol/cval.  Element-strided: lane l of warp w owns
// sorted element o = r*T + 32w + l of row r, so head detection reads smem
// conflict-free, a head's output rank is a ballot prefix plus a scan over the
// (row, warp) head counts, and consecutive lanes store consecutive entries of
// C (coalesced, no staging).  Returns the number of distinct columns.
// LB: the output offset is not known in advance.  The count is published
// (`publish(count)`) right after the head scan; the run sums are formed next
// — each head overwrites its own first product's slot with the sum, and the
// rank -> head position map is kept in the sort's idle buffer — so the wait
// for the predecessors' counts overlaps this work; then warp 0 obtains the
// offset (`place(count)`, the look-back) and the tile stores its output
// coalesced at ccol/cval + offset.
template <int T, int CAPM, bool LB = false, class Publish = int, class Place = int, int VB = 0, int RBO = 0>
__device__ __forceinline__ int reduce_and_write(MergeShared<T, CAPM, VB, RBO>& s, int b, int total,
                                                uint32_t kofs, int32_t* __restrict__ ccol,
                                                double* __restrict__ cval, Publish&& publish = 0,
                                                Place&& place = 0) {
    constexpr int NW = T / 32;
    constexpr int R = (CAPM + T - 1) / T;
    static_assert(R * NW <= T && R * NW <= MergeShared<T, CAPM, VB, RBO>::NHIST, "row/warp counters");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* K = s.key(b);
    const uint16_t* X = s.idx(b);
    int* cnt = reinterpret_cast<int*>(s.hist);  // [row][warp] head counts, then offsets
    const int nrows = (total + T - 1) / T;
    unsigned hm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int o = r * T + threadIdx.x;
        const bool h = o < total && (o == 0 || K[PADI(o)] != K[PADI(o - 1)]);
        hm[r] = __ballot_sync(0xffffffffu, h);
        if (lane == 0 && r < nrows) cnt[r * NW + warp] = __popc(hm[r]);
    }
    __syncthreads();
    const int v = threadIdx.x < nrows * NW ? cnt[threadIdx.x] : 0;
    int pre, tile_cnt;
    cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(v, pre, tile_cnt);
    __syncthreads();
    if (threadIdx.x < nrows * NW) cnt[threadIdx.x] = pre;
    if constexpr (LB) {
        if (threadIdx.x == 0) publish(tile_cnt);
        __syncthreads();
        PH(13);
#ifdef BSP_X_PHASE
        if (threadIdx.x == 0 && g_phase_last[blockIdx.x & ((1 << 22) - 1)] != 0) {
            const int b = blockIdx.x & ((1 << 22) - 1);
            atomicAdd(&g_phase[20 + g_phase_cls[b]], static_cast<unsigned long long>(clock64() - g_phase_t0[b]));
            atomicAdd(&g_phase[26 + g_phase_cls[b]], 1ull);
        }
#endif
        // rank -> head position, in the buffer the sort left idle
        uint16_t* hpos = b ? s.idx0 : reinterpret_cast<uint16_t*>(s.u.c.packed);
        const unsigned below = (1u << lane) - 1u;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!((hm[r] >> lane) & 1u)) continue;
            const int o = r * T + threadIdx.x;
            const int rank = cnt[r * NW + warp] + __popc(hm[r] & below);
            const uint32_t key = K[PADI(o)];
            // A run of one product (nearly all of them at cf ~ 1) keeps its
            // slot as it is: the final store forms 0.0 + p itself.  Longer
            // runs leave their sum (never -0.0: it starts from +0.0) in the
            // head's slot, for which 0.0 + sum changes nothing.
            if (o + 1 < total && K[PADI(o + 1)] == key) {
                const int x0 = X[PADI(o)];
                double acc = 0.0;
                int e = o;
                do {
                    acc = __dadd_rn(acc, s.val[X[PADI(e)]]);
                    ++e;
                } while (e < total && K[PADI(e)] == key);
                s.val[x0] = acc;  // only this head reads its run's slots
            }
            hpos[rank] = static_cast<uint16_t>(o);
        }
        __syncthreads();
        PH(14);
        long long off = 0;
        if constexpr (!std::is_same_v<std::decay_t<Place>, int>) {
            // placement now: warp 0 walks, the tile stores at the offset
            __shared__ long long s_off;
            if (warp == 0) {
                const long long v = place(tile_cnt);
                if (lane == 0) s_off = v;
            }
            __syncthreads();
            PH(15);
            off = s_off;
        }
        ccol += off;
        cval += off;
        for (int q = threadIdx.x; q < tile_cnt; q += T) {
            const int o = hpos[q];
            ccol[q] = static_cast<int32_t>(K[PADI(o)] + kofs);
            cval[q] = __dadd_rn(0.0, s.val[X[PADI(o)]]);
        }
        __syncthreads();
        PH(16);
        return tile_cnt;
    }
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (!((hm[r] >> lane) & 1u)) continue;
        const int o = r * T + threadIdx.x;
        const int rank = cnt[r * NW + warp] + __popc(hm[r] & below);
        const uint32_t key = K[PADI(o)];
        double acc = 0.0;
        int e = o;
        do {
            acc = __dadd_rn(acc, s.val[X[PADI(e)]]);
            ++e;
        } while (e < total && K[PADI(e)] == key);
        ccol[rank] = static_cast<int32_t>(key + kofs);
        cval[rank] = acc;
    }
    __syncthreads();
    return tile_cnt;
}

// Reduction and single-pass placement of the look-back tile whose values were
// not gathered yet (expand_keys).  The sorted tile is in buffer 0.  The count is
// published right after the head scan; then the values are fetched — product g
// takes b from bval[src[g]] (cp.async into the sort's idle buffer) and a from
// the A row — the heads sum their runs left to right from 0.0 in ascending k
// (spgemm.hpp:92-97), warp 0 takes the offset from the look-back and the tile
// stores its output coalesced.  Everything after `publish` overlaps the
// predecessors' sorts.
template <int T, int CAPM, int VB, int RBO, class Publish, class Place>
__device__ __forceinline__ int reduce_lb2(MergeShared<T, CAPM, VB, RBO>& s, int total, uint32_t kofs,
                                          int32_t* __restrict__ ccol, double* __restrict__ cval,
                                          const double* __restrict__ arow,
                                          const double* __restrict__ bval, Publish&& publish,
                                          Place&& place) {
    constexpr int NW = T / 32;
    constexpr int R = (CAPM + T - 1) / T;
    static_assert(sizeof(typename MergeShared<T, CAPM, VB, RBO>::U) >= sizeof(double) * CAPM, "value buffer");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* K = s.key0;
    const uint16_t* X = s.idx0;
    int* cnt = reinterpret_cast<int*>(s.hist);
    const int nrows = (total + T - 1) / T;
    unsigned hm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int o = r * T + threadIdx.x;
        const bool h = o < total && (o == 0 || K[PADI(o)] != K[PADI(o - 1)]);
        hm[r] = __ballot_sync(0xffffffffu, h);
        if (lane == 0 && r < nrows) cnt[r * NW + warp] = __popc(hm[r]);
    }
    __syncthreads();
    const int v = threadIdx.x < nrows * NW ? cnt[threadIdx.x] : 0;
    int pre, tile_cnt;
    cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(v, pre, tile_cnt);
    __syncthreads();
    if (threadIdx.x < nrows * NW) cnt[threadIdx.x] = pre;
    if (threadIdx.x == 0) publish(tile_cnt);
    PH(13);
    // values into the sort's idle buffer, in expansion order (a run's entries
    // are consecutive in B: neighbouring lanes share sectors, as in the
    // combined gather; fetching them in sorted order instead — contiguous
    // runs for the sums — read 4x the sectors: 182 vs 170 ms on cfg5)
    constexpr bool SEG16 = VB < 8 * CAPM;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(s.val);
    const uint32_t* seg = src + CAPM;
    const uint16_t* seg16 = reinterpret_cast<const uint16_t*>(src + CAPM);
    double* pv = reinterpret_cast<double*>(&s.u);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int g = r * T + threadIdx.x;
        if (g < total) cp_async8(&pv[g], bval + src[g]);
    }
    double av[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int g = r * T + threadIdx.x;
        av[r] = g < total ? __ldg(arow + (SEG16 ? static_cast<uint32_t>(seg16[g]) : seg[g])) : 0.0;
    }
    cp_async_wait_all();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int g = r * T + threadIdx.x;
        if (g < total) pv[g] = __dmul_rn(av[r], pv[g]);  // this thread's own copies
    }
    __syncthreads();
    PH(3);
    // run sums (each head overwrites its own first slot); rank -> head position
    uint16_t* hpos = reinterpret_cast<uint16_t*>(s.val);  // src/seg are consumed
    const unsigned below = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (!((hm[r] >> lane) & 1u)) continue;
        const int o = r * T + threadIdx.x;
        const int rank = cnt[r * NW + warp] + __popc(hm[r] & below);
        const uint32_t key = K[PADI(o)];
        if (o + 1 < total && K[PADI(o + 1)] == key) {  // (single products: see reduce_and_write)
            double acc = 0.0;
            int e = o;
            const int x0 = X[PADI(o)];
            do {
                acc = __dadd_rn(acc, pv[X[PADI(e)]]);
                ++e;
            } while (e < total && K[PADI(e)] == key);
            pv[x0] = acc;  // only this head reads its run's slots
        }
        hpos[rank] = static_cast<uint16_t>(o);
    }
    __syncthreads();
    PH(14);
    __shared__ long long s_off2;
    if (warp == 0) {
        const long long vv = place(tile_cnt);
        if (lane == 0) s_off2 = vv;
    }
    __syncthreads();
    PH(15);
    ccol += s_off2;
    cval += s_off2;
    for (int q = threadIdx.x; q < tile_cnt; q += T) {
        const int o = hpos[q];
        ccol[q] = static_cast<int32_t>(K[PADI(o)] + kofs);
        cval[q] = __dadd_rn(0.0, pv[X[PADI(o)]]);
    }
    __syncthreads();
    PH(16);
    return tile_cnt;
}

// Fibonacci hash of a column into a table of 2^lg slots.
__device__ __forceinline__ uint32_t col_hash(uint32_t c, int lg) {
    return (c * 0x9E3779B1u) >> (32 - lg);
}

}  // namespace bsp
