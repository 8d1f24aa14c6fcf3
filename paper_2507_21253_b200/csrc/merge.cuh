// On-chip stable merge of presorted runs and hash-based distinct counting.
//
// Numeric (exact) tile = ESC with a MERGE sort instead of a radix sort: the
// products of a tile are expanded into shared memory in (k ascending, j
// ascending) order, i.e. as one sorted run per contributing B-row segment.
// A bottom-up merge-path merge of adjacent runs (ties taken from the left
// run, i.e. from the smaller k) sorts them by column while keeping equal
// columns in ascending-k order, so the per-column sums are formed exactly
// as the reference forms them (0.0 + p1 + p2 + ..., spgemm.hpp:92-97).
//
// Symbolic tile = distinct-column count through an open-addressed smem hash
// (atomicCAS insert), the GPU form of HashAccumulator::insert_key
// (hash_accumulator.hpp:48-54).
#pragma once

#include "esc.cuh"

namespace bsp {

template <int T, int CAPM>
struct MergeShared {
    uint32_t key[2][CAPM];
    uint16_t idx[2][CAPM];
    double val[CAPM];
    uint16_t ro[2][CAPM + 2];  // run offsets (runs <= products <= CAPM)
    typename cub::BlockScan<int32_t, T>::TempStorage scan;
    int64_t pstart[T];
    int32_t plen[T];
    int32_t poff[T];
    double pav[T];
    int nruns;
};

// Expand the products of (row, [c0, c1)) in (k, j) order; every non-empty
// B-row segment becomes one sorted run.  Returns the product count.
template <int T, int CAPM, bool VALUES>
__device__ __forceinline__ int expand_runs(const Mats& m, int32_t row, int32_t c0, int32_t c1,
                                           bool full, MergeShared<T, CAPM>& s) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = T / 32;
    const int64_t rs = m.arp[row], re = m.arp[row + 1];
    int total = 0, nruns = 0;
    for (int64_t pc = rs; pc < re; pc += T) {
        const int64_t p = pc + tid;
        int len = 0;
        int64_t start = 0;
        double av = 0.0;
        if (p < re) {
            const int32_t k = __ldg(m.acol + p);
            int64_t b0 = __ldg(m.brp + k), b1 = __ldg(m.brp + k + 1);
            if (!full) {
                b0 = lower_bound_col(m.bcol, b0, b1, c0);
                b1 = lower_bound_col(m.bcol, b0, b1, c1);
            }
            start = b0;
            len = static_cast<int>(b1 - b0);
            if (VALUES) av = __ldg(m.aval + p);
        }
        // packed scan: low 16 bits offset, high 16 bits run index
        const int packed = len | ((len > 0) << 16);
        int off, agg;
        cub::BlockScan<int32_t, T>(s.scan).ExclusiveSum(packed, off, agg);
        const int o = total + (off & 0xffff);
        if (len > 0) s.ro[0][nruns + (off >> 16)] = static_cast<uint16_t>(o);
        s.pstart[tid] = start;
        s.plen[tid] = len;
        s.poff[tid] = o;
        if (VALUES) s.pav[tid] = av;
        __syncthreads();
        const int nslots = static_cast<int>(::min(int64_t{T}, re - pc));
        for (int slot = warp; slot < nslots; slot += NW) {
            const int l = s.plen[slot];
            const int64_t st = s.pstart[slot];
            const int ob = s.poff[slot];
            double a = 0.0;
            if (VALUES) a = s.pav[slot];
            for (int q = lane; q < l; q += 32) {
                s.key[0][ob + q] = static_cast<uint32_t>(__ldg(m.bcol + st + q) - c0);
                s.idx[0][ob + q] = static_cast<uint16_t>(ob + q);
                if (VALUES) s.val[ob + q] = __dmul_rn(a, __ldg(m.bval + st + q));
            }
        }
        total += agg & 0xffff;
        nruns += agg >> 16;
        __syncthreads();
    }
    if (tid == 0) {
        s.ro[0][nruns] = static_cast<uint16_t>(total);
        s.nruns = nruns;
    }
    __syncthreads();
    return total;
}

// Bottom-up stable merge of the runs in key[0]/idx[0]; returns the buffer
// holding the sorted result.
template <int T, int CAPM>
__device__ __forceinline__ int merge_runs(MergeShared<T, CAPM>& s, int total) {
    const int tid = threadIdx.x;
    int R = s.nruns;
    int b = 0;
    const int E = (total + T - 1) / T;
    while (R > 1) {
        const int Rn = (R + 1) >> 1;
        const uint16_t* ro = s.ro[b];
        uint16_t* rn = s.ro[b ^ 1];
        for (int i = tid; i <= Rn; i += T) rn[i] = (i < Rn) ? ro[2 * i] : static_cast<uint16_t>(total);
        __syncthreads();
        const uint32_t* K = s.key[b];
        const uint16_t* X = s.idx[b];
        uint32_t* KO = s.key[b ^ 1];
        uint16_t* XO = s.idx[b ^ 1];
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
                if (K[xs + mid] <= K[xe + k - 1 - mid]) a = mid + 1; else a_hi = mid;
            }
            int xi = xs + a, yi = xe + (k - a);
            uint32_t kx = xi < xe ? K[xi] : 0xffffffffu;
            uint32_t ky = yi < ye ? K[yi] : 0xffffffffu;
            for (int t = k; t < kend; ++t) {
                const bool takex = (yi >= ye) || (xi < xe && kx <= ky);
                if (takex) {
                    KO[xs + t] = kx;
                    XO[xs + t] = X[xi];
                    ++xi;
                    kx = xi < xe ? K[xi] : 0xffffffffu;
                } else {
                    KO[xs + t] = ky;
                    XO[xs + t] = X[yi];
                    ++yi;
                    ky = yi < ye ? K[yi] : 0xffffffffu;
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

// Fibonacci hash of a column into a table of 2^lg slots.
__device__ __forceinline__ uint32_t col_hash(uint32_t c, int lg) {
    return (c * 0x9E3779B1u) >> (32 - lg);
}

}  // namespace bsp
