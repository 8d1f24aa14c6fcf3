// Heavy rows (products > on-chip capacity, A-row length <= HDMAX): one CTA
// owns the whole row and walks it in column windows with per-segment
// cursors, so no segment is ever binary-searched from its start again.
//
// Window choice ("quota windows"): with rem_p products left in segment p and
// rem in total, segment p gets q_p = max(1, floor(budget*rem_p/rem)) slots,
// budget = CAPM - (#active segments); the window end c1 is the minimum over
// segments of the column q_p positions past the cursor.  Every segment then
// contributes <= q_p products (so a window holds <= CAPM), and the segment
// holding the smallest remaining column contributes >= 1 (progress).
// Windows are column-disjoint and visited in increasing column order, so a
// row's output is the concatenation of its windows' outputs.
#pragma once

#include "merge.cuh"

#include <cub/block/block_reduce.cuh>

namespace bsp {

constexpr int HDMAX = 1024;  // max A-row length of a cursor-walked heavy row

template <int T, int CAPM>
struct HeavyState {
    static constexpr int PPT = HDMAX / T;  // segments per thread (blocked)
    int64_t cur[HDMAX];
    int32_t rem[HDMAX];
    int32_t qlim[HDMAX];
    int32_t off[HDMAX + 1];
    double av[HDMAX];
    uint32_t c1;
    int32_t wtotal;
    int32_t nruns;
    int64_t rem_total;
    typename cub::BlockReduce<int64_t, T>::TempStorage red64;
    typename cub::BlockReduce<uint32_t, T>::TempStorage redu;
    typename cub::BlockScan<int32_t, T>::TempStorage scan2;
};

template <int T, int CAPM>
struct HeavyNumShared {
    HeavyState<T, CAPM> h;
    MergeShared<T, CAPM> m;
};

template <int T, int CAPM>
struct HeavySymShared {
    HeavyState<T, CAPM> h;
    int32_t table[2 * CAPM];
    typename cub::BlockReduce<int32_t, T>::TempStorage red;
};

// Initialise cursors; returns the row's total products (all threads).
template <int T, int CAPM>
__device__ __forceinline__ int64_t heavy_init(const Mats& m, int32_t row, int d,
                                              HeavyState<T, CAPM>& s, bool values) {
    const int64_t rs = m.arp[row];
    int64_t mine = 0;
    for (int p = threadIdx.x; p < d; p += T) {
        const int32_t k = __ldg(m.acol + rs + p);
        const int64_t b0 = __ldg(m.brp + k), b1 = __ldg(m.brp + k + 1);
        s.cur[p] = b0;
        s.rem[p] = static_cast<int32_t>(b1 - b0);
        if (values) s.av[p] = __ldg(m.aval + rs + p);
        mine += b1 - b0;
    }
    const int64_t tot = cub::BlockReduce<int64_t, T>(s.red64).Sum(mine);
    if (threadIdx.x == 0) s.rem_total = tot;
    __syncthreads();
    return s.rem_total;
}

// Choose the next window; fills qlim/off/nruns/wtotal.  Returns window size.
template <int T, int CAPM>
__device__ __forceinline__ int heavy_next_window(const Mats& m, int d, HeavyState<T, CAPM>& s,
                                                 uint16_t* ro /* run offsets out */) {
    constexpr int PPT = HeavyState<T, CAPM>::PPT;
    const int tid = threadIdx.x;
    // active segments
    int act = 0;
    for (int i = 0; i < PPT; ++i) {
        const int p = tid * PPT + i;
        act += (p < d && s.rem[p] > 0);
    }
    const int64_t dact = cub::BlockReduce<int64_t, T>(s.red64).Sum(act);
    __syncthreads();
    const int64_t rem_total = s.rem_total;
    const int64_t B = CAPM - dact;  // > 0 because d <= HDMAX < CAPM
    uint32_t lim_min = 0xffffffffu;
    for (int i = 0; i < PPT; ++i) {
        const int p = tid * PPT + i;
        int q = 0;
        if (p < d && s.rem[p] > 0) {
            const int64_t qq = (B * s.rem[p]) / rem_total;
            q = static_cast<int>(qq < 1 ? 1 : qq);
            if (q < s.rem[p]) {
                const uint32_t lim = static_cast<uint32_t>(__ldg(m.bcol + s.cur[p] + q));
                lim_min = min(lim_min, lim);
            } else {
                q = s.rem[p];
            }
        }
        if (p < d) s.qlim[p] = q;
    }
    const uint32_t c1 = cub::BlockReduce<uint32_t, T>(s.redu).Reduce(lim_min, cub::Min());
    if (tid == 0) s.c1 = c1;
    __syncthreads();
    const uint32_t cw = s.c1;
    // per-segment counts below c1 (within the quota), blocked scan
    int cnt[PPT];
    int packed = 0;
    for (int i = 0; i < PPT; ++i) {
        const int p = tid * PPT + i;
        int c = 0;
        if (p < d && s.qlim[p] > 0) {
            if (cw == 0xffffffffu) {
                c = s.qlim[p];
            } else {
                const int64_t e = lower_bound_col(m.bcol, s.cur[p], s.cur[p] + s.qlim[p],
                                                  static_cast<int32_t>(cw));
                c = static_cast<int>(e - s.cur[p]);
            }
        }
        cnt[i] = c;
        packed += c | ((c > 0) << 16);
    }
    int poff, pagg;
    cub::BlockScan<int32_t, T>(s.scan2).ExclusiveSum(packed, poff, pagg);
    int o = poff & 0xffff, r = poff >> 16;
    for (int i = 0; i < PPT; ++i) {
        const int p = tid * PPT + i;
        if (p < d) {
            s.off[p] = o;
            s.qlim[p] = cnt[i];  // reuse: this window's count
            if (cnt[i] > 0) ro[r++] = static_cast<uint16_t>(o);
        }
        o += cnt[i];
    }
    if (tid == 0) {
        s.wtotal = pagg & 0xffff;
        s.nruns = pagg >> 16;
        s.off[d] = pagg & 0xffff;
    }
    __syncthreads();
    return s.wtotal;
}

// Advance cursors past the current window.
template <int T, int CAPM>
__device__ __forceinline__ void heavy_advance(int d, HeavyState<T, CAPM>& s) {
    for (int p = threadIdx.x; p < d; p += T) {
        const int c = s.qlim[p];
        s.cur[p] += c;
        s.rem[p] -= c;
    }
    if (threadIdx.x == 0) s.rem_total -= s.wtotal;
    __syncthreads();
}

// Flattened copy of the window's products: thread t owns window positions
// [t*E, t*E+E), locating its first segment by binary search over off[].
template <int T, int CAPM, bool VALUES, typename F>
__device__ __forceinline__ void heavy_for_each_product(const Mats& m, int d,
                                                       HeavyState<T, CAPM>& s, int W, F f) {
    const int E = (W + T - 1) / T;
    int e = min(W, static_cast<int>(threadIdx.x) * E);
    const int ee = min(W, e + E);
    if (e >= ee) return;
    int lo = 0, hi = d - 1;
    while (lo < hi) {  // last p with off[p] <= e
        const int mid = (lo + hi + 1) >> 1;
        if (s.off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    int p = lo;
    while (e < ee) {
        while (s.off[p + 1] <= e) ++p;
        const int64_t base = s.cur[p] - s.off[p];
        const int stop = min(ee, s.off[p + 1]);
        const double a = VALUES ? s.av[p] : 0.0;
        for (; e < stop; ++e) f(e, __ldg(m.bcol + base + e), VALUES ? __dmul_rn(a, __ldg(m.bval + base + e)) : 0.0);
    }
}

template <int T, int CAPM>
__global__ void __launch_bounds__(T) heavy_numeric_kernel(Mats m, const int32_t* __restrict__ rows,
                                                          OutCtx out) {
    using S = HeavyNumShared<T, CAPM>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    const int tid = threadIdx.x;
    const int32_t row = rows[blockIdx.x];
    const int d = static_cast<int>(m.arp[row + 1] - m.arp[row]);
    int64_t left = heavy_init<T, CAPM>(m, row, d, s.h, true);
    int64_t wpos = out.crp[row - out.row_begin];
    while (left > 0) {
        const int W = heavy_next_window<T, CAPM>(m, d, s.h, s.m.ro(0));
        if (tid == 0) {
            s.m.ro(0)[s.h.nruns] = static_cast<uint16_t>(W);
            s.m.nruns = s.h.nruns;
        }
        heavy_for_each_product<T, CAPM, true>(m, d, s.h, W, [&](int e, int32_t col, double v) {
            s.m.key(0)[PADI(e)] = static_cast<uint32_t>(col);
            s.m.idx(0)[PADI(e)] = static_cast<uint16_t>(e);
            s.m.val[e] = v;
        });
        __syncthreads();
        const int b = merge_runs<T, CAPM>(s.m, W);
        const int n = reduce_and_write<T, CAPM>(s.m, b, W, 0u, out.ccol + wpos, out.cval + wpos);
        wpos += n;
        heavy_advance<T, CAPM>(d, s.h);
        left = s.h.rem_total;
    }
}

template <int T, int CAPM>
__global__ void __launch_bounds__(T) heavy_symbolic_kernel(Mats m, const int32_t* __restrict__ rows,
                                                           OutCtx out) {
    using S = HeavySymShared<T, CAPM>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    const int tid = threadIdx.x;
    constexpr int LG = 1 + 31 - __builtin_clz(static_cast<unsigned>(CAPM));
    const int32_t row = rows[blockIdx.x];
    const int d = static_cast<int>(m.arp[row + 1] - m.arp[row]);
    __shared__ uint16_t ro_dummy[HDMAX + 2];
    int64_t left = heavy_init<T, CAPM>(m, row, d, s.h, false);
    int total = 0;
    while (left > 0) {
        for (int e = tid; e < 2 * CAPM; e += T) s.table[e] = -1;
        const int W = heavy_next_window<T, CAPM>(m, d, s.h, ro_dummy);
        heavy_for_each_product<T, CAPM, false>(m, d, s.h, W, [&](int, int32_t col, double) {
            uint32_t hsl = col_hash(static_cast<uint32_t>(col), LG);
            for (;;) {
                const int32_t prev = atomicCAS(&s.table[hsl], -1, col);
                if (prev == -1) {
                    ++total;
                    break;
                }
                if (prev == col) break;
                hsl = (hsl + 1) & (2 * CAPM - 1);
            }
        });
        __syncthreads();
        heavy_advance<T, CAPM>(d, s.h);
        left = s.h.rem_total;
    }
    const int tot = cub::BlockReduce<int32_t, T>(s.red).Sum(total);
    if (tid == 0) out.row_nnz[row - out.row_begin] = tot;
}

}  // namespace bsp
