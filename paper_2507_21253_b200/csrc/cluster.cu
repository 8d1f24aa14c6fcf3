// Cluster-wise SpGEMM on sm_100a and the device CSR_Cluster format.
//
// Replaces reference build_csr_cluster (cluster_format.hpp:130-186),
// cluster_to_csr (:190-233), spgemm_clusterwise (cluster_spgemm.hpp:55-189)
// and the AccessStats counters (cluster_spgemm.hpp:26-45).
//
// Cluster kernel (Algorithm 1 of the paper, B200 form): one CTA owns one
// cluster of K rows.  For every merged column k of the cluster the B row is
// loaded from global memory ONCE (coalesced), and each product is scattered
// to every live member (member_mask bit) as a composite key (member, j) in
// shared memory.  A stable radix sort by (member, j) followed by ordered run
// reduction gives, for every member row, exactly the values of the row-wise
// kernel (contributions still summed in ascending k from 0.0), so C is
// written directly as CSR over the original row indices and is bit-identical
// to spgemm_rowwise(cluster_to_csr(A), B).  Singleton clusters and clusters
// with more than CAP products are routed to the row-wise bins.
#include "esc.cuh"
#include "merge.cuh"

#include <algorithm>
#include <numeric>

namespace bsp {

namespace {

constexpr int MAXK = 32;     // clusters the cluster kernels take (member_mask is 32-bit)
constexpr int MAXK_FMT = 1024;  // cluster size limit of the device format: larger
                                // clusters keep valid bits only (member_mask 0) and
                                // are multiplied through the row view

// Live members of merged column u (slot base = value_ptr + (u - u0) * K):
// the 32-bit member mask for K <= 32, else the valid bits.
__device__ __forceinline__ int live_count(const uint32_t* mask, const unsigned long long* valid,
                                          int64_t u, int64_t slot0, int K) {
    if (K <= MAXK) return __popc(mask[u]);
    int n = 0;
    for (int l = 0; l < K; ++l) n += static_cast<int>((valid[(slot0 + l) >> 6] >> ((slot0 + l) & 63)) & 1ull);
    return n;
}

struct ClusterMats {
    const int32_t* __restrict__ sizes;
    const int64_t* __restrict__ member_ptr;
    const int64_t* __restrict__ ccp;  // cluster_col_ptr
    const int32_t* __restrict__ ccol;
    const int64_t* __restrict__ vptr;
    const double* __restrict__ aval;
    const uint32_t* __restrict__ mask;
    const int32_t* __restrict__ row_map;
    const int64_t* __restrict__ brp;
    const int32_t* __restrict__ bcol;
    const double* __restrict__ bval;
    int32_t ncols;
    int64_t bnnz;  // nnz(B): bulk copies stay inside [0, bnnz)
};

// ---------------------------------------------------------------------------
// format construction: one warp per cluster, K-way merge of member rows
// ---------------------------------------------------------------------------
// MODE 0: union size per cluster; MODE 1: write merged columns, values,
// valid bits and member masks.
template <int MODE>
__global__ void build_cluster_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                     const double* __restrict__ val, int64_t ncl,
                                     const int64_t* __restrict__ mptr,
                                     const int32_t* __restrict__ rows, int64_t* __restrict__ ucount,
                                     const int64_t* __restrict__ ccp, const int64_t* __restrict__ vptr,
                                     int32_t* __restrict__ ocol, double* __restrict__ oval,
                                     unsigned long long* __restrict__ valid,
                                     uint32_t* __restrict__ omask) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t{gridDim.x} * blockDim.x) >> 5;
    for (int64_t c = warp; c < ncl; c += nwarps) {
        const int K = static_cast<int>(mptr[c + 1] - mptr[c]);
        if (K > 32) continue;  // build_cluster_big_kernel
        int64_t cur = 0, end = 0;
        if (lane < K) {
            const int32_t r = rows[mptr[c] + lane];
            cur = rp[r];
            end = rp[r + 1];
        }
        int64_t u = 0;
        const int64_t cbase = MODE ? ccp[c] : 0;
        const int64_t vbase = MODE ? vptr[c] : 0;
        for (;;) {
            const int32_t mine = (lane < K && cur < end) ? col[cur] : INT32_MAX;
            const int32_t mn = __reduce_min_sync(0xffffffffu, mine);
            if (mn == INT32_MAX) break;
            const bool hit = (mine == mn);
            const uint32_t who = __ballot_sync(0xffffffffu, hit);
            if (MODE) {
                if (lane == 0) {
                    ocol[cbase + u] = mn;
                    omask[cbase + u] = who;
                }
                if (hit) {
                    const int64_t slot = vbase + u * K + lane;
                    oval[slot] = val[cur];
                    atomicOr(&valid[slot >> 6], 1ull << (slot & 63));
                }
            }
            if (hit) ++cur;
            ++u;
        }
        if (!MODE && lane == 0) ucount[c] = u;
    }
}


// Clusters of more than 32 rows (up to MAXK_FMT): lane holds members lane + 32 j;
// the same K-way merge, each step taking the minimum over all members.  Kept
// apart so the common kernel above stays lean; launched only when such
// clusters exist.
template <int MODE>
__global__ void build_cluster_big_kernel(const int64_t* __restrict__ rp,
                                         const int32_t* __restrict__ col,
                                         const double* __restrict__ val, int64_t ncl,
                                         const int64_t* __restrict__ mptr,
                                         const int32_t* __restrict__ rows,
                                         int64_t* __restrict__ ucount,
                                         const int64_t* __restrict__ ccp,
                                         const int64_t* __restrict__ vptr,
                                         int32_t* __restrict__ ocol, double* __restrict__ oval,
                                         unsigned long long* __restrict__ valid,
                                         uint32_t* __restrict__ omask) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t{gridDim.x} * blockDim.x) >> 5;
    for (int64_t c = warp; c < ncl; c += nwarps) {
        const int K = static_cast<int>(mptr[c + 1] - mptr[c]);
        if (K <= 32) continue;
        {
            // big clusters (warp-uniform): lane holds members lane + 32 j; the
            // same K-way merge, each step taking the minimum over all members
            constexpr int MB = MAXK_FMT / 32;
            int64_t bc[MB], be[MB];
#pragma unroll
            for (int j = 0; j < MB; ++j) {
                const int l = lane + 32 * j;
                bc[j] = be[j] = 0;
                if (l < K) {
                    const int32_t r = rows[mptr[c] + l];
                    bc[j] = rp[r];
                    be[j] = rp[r + 1];
                }
            }
            int64_t u = 0;
            const int64_t cbase = MODE ? ccp[c] : 0;
            const int64_t vbase = MODE ? vptr[c] : 0;
            for (;;) {
                int32_t mine = INT32_MAX;
#pragma unroll
                for (int j = 0; j < MB; ++j)
                    if (bc[j] < be[j]) mine = min(mine, col[bc[j]]);
                const int32_t mn = __reduce_min_sync(0xffffffffu, mine);
                if (mn == INT32_MAX) break;
                if (MODE && lane == 0) {
                    ocol[cbase + u] = mn;
                    omask[cbase + u] = 0u;  // members beyond 32: valid bits only
                }
#pragma unroll
                for (int j = 0; j < MB; ++j) {
                    if (bc[j] < be[j] && col[bc[j]] == mn) {
                        if (MODE) {
                            const int64_t slot = vbase + u * K + lane + 32 * j;
                            oval[slot] = val[bc[j]];
                            atomicOr(&valid[slot >> 6], 1ull << (slot & 63));
                        }
                        ++bc[j];
                    }
                }
                ++u;
            }
            if (!MODE && lane == 0) ucount[c] = u;
        }
    }
}

__global__ void value_ptr_kernel(const int64_t* __restrict__ ucount, const int64_t* __restrict__ mptr,
                                 int64_t ncl, int64_t* __restrict__ slots,
                                 int32_t* __restrict__ sizes) {
    for (int64_t c = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; c < ncl;
         c += int64_t{gridDim.x} * blockDim.x) {
        const int64_t K = mptr[c + 1] - mptr[c];
        slots[c] = K * ucount[c];
        sizes[c] = static_cast<int32_t>(K);
    }
}

// cluster_to_csr: per (cluster, member) valid count, then compaction.
template <int MODE>
__global__ void cluster_to_csr_kernel(const int32_t* __restrict__ sizes,
                                      const int64_t* __restrict__ mptr,
                                      const int64_t* __restrict__ ccp,
                                      const int32_t* __restrict__ ccol,
                                      const int64_t* __restrict__ vptr,
                                      const double* __restrict__ vals,
                                      const uint32_t* __restrict__ mask,
                                      const unsigned long long* __restrict__ valid,
                                      const int32_t* __restrict__ row_map, int64_t ncl,
                                      int64_t* __restrict__ row_nnz, const int64_t* __restrict__ crp,
                                      int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t{gridDim.x} * blockDim.x) >> 5;
    for (int64_t c = warp; c < ncl; c += nwarps) {
        const int K = sizes[c];
        const int64_t u0 = ccp[c], u1 = ccp[c + 1];
        for (int l = 0; l < K; ++l) {
            const int32_t row = row_map[mptr[c] + l];
            int64_t pos = MODE ? crp[row] : 0;
            int64_t cnt = 0;
            for (int64_t ub = u0; ub < u1; ub += 32) {
                const int64_t u = ub + lane;
                bool has = false;
                if (u < u1) {
                    if (K <= MAXK) {
                        has = (mask[u] >> l) & 1u;
                    } else {
                        const int64_t slot = vptr[c] + (u - u0) * K + l;
                        has = (valid[slot >> 6] >> (slot & 63)) & 1ull;
                    }
                }
                const uint32_t b = __ballot_sync(0xffffffffu, has);
                if (MODE && has) {
                    const int64_t o = pos + __popc(b & ((1u << lane) - 1u));
                    ocol[o] = ccol[u];
                    oval[o] = vals[vptr[c] + (u - u0) * K + l];
                }
                pos += __popc(b);
                cnt += __popc(b);
            }
            if (!MODE && lane == 0) row_nnz[row] = cnt;
        }
    }
}

// ---------------------------------------------------------------------------
// cluster products + routing
// ---------------------------------------------------------------------------
// 0: row-wise classes; 1..5: member-keyed tiles of <= 512 .. 4096 products;
// 6, 7: union tiles of <= 1024 / 2048 distinct B entries (cluster_union_kernel)
constexpr int NCC = 8;
constexpr int NKC = 6;  // member-keyed classes 1..5 (+ 0)
__constant__ int kClusterCap[NKC] = {0, 512, 1024, 2048, 3072, 4096};
constexpr int UMAXK = 8;      // union tiles: members (accumulators in registers)
constexpr int UMAXMC = 512;   // union tiles: merged columns
constexpr int UMAXA = 1024;   // union tiles: A values staged (merged columns x members)

__global__ void cluster_products_kernel(ClusterMats m, int64_t ncl, int cbits,
                                        uint8_t* __restrict__ ccls, uint8_t* __restrict__ row_skip,
                                        unsigned long long* __restrict__ counts, int union_ok,
                                        int min_reuse10) {
    __shared__ unsigned s_cnt[NCC];
    if (threadIdx.x < NCC) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t c = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; c < ncl;
         c += int64_t{gridDim.x} * blockDim.x) {
        const int K = m.sizes[c];
        int64_t P = 0, S = 0, Sraw = 0;  // S: B entries staged (union_ok == 2: with the bulk copies' slack)
        const int64_t MC = m.ccp[c + 1] - m.ccp[c];
        for (int64_t u = m.ccp[c]; u < m.ccp[c + 1]; ++u) {
            const int32_t k = m.ccol[u];
            const int64_t len = m.brp[k + 1] - m.brp[k];
            const int live = __popc(m.mask[u]);
            P += static_cast<int64_t>(live) * len;
            if (live) Sraw += len;
            if (live && len > 0)  // B entries the cluster loads (once each)
                S += union_ok == 2 ? (((m.brp[k] & 3) + len + 3) & ~int64_t{3}) : len;
        }
        // staged cluster tile: B rows of the cluster fit the stage, every
        // member fits one merge tile (otherwise the rows go to the row bins)
        // composite-key radix tile (measured fastest of the three cluster tiles
        // tried — see DESIGN.md §4): classes by the cluster's total products
        int cl = 0;
        const bool keyfits = bit_length(static_cast<uint32_t>(K - 1)) + cbits <= 31;
        // B-row reuse of the cluster = member products / B entries loaded once.
        // Below min_reuse10 / 10 the shared loads do not pay for the cluster
        // tile's member bookkeeping (measured, cfg4: pairs of stencil rows reuse
        // 1.35x and run 26 ms on the cluster accumulator vs 16 ms row-wise; the
        // paper finds the same on stencils): those rows take the row-wise classes.
        if (10 * P < static_cast<int64_t>(min_reuse10) * Sraw) {
            // cl = 0
        } else
        if (union_ok && K >= 2 && K <= UMAXK && MC <= UMAXMC && MC * K <= UMAXA && S > 0 &&
            S <= 2048) {
            // union tile: each B entry expanded and sorted once for the cluster
            // (the small tile stages at most UMAXMC / 2 merged columns, UMAXA / 2 values)
            cl = (S <= 1024 && MC <= UMAXMC / 2 && MC * K <= UMAXA / 2) ? 6 : 7;
        } else if (K >= 2 && K <= MAXK && keyfits && P > 0 && P <= kClusterCap[NKC - 1]) {
            cl = 1;
            while (P > kClusterCap[cl]) ++cl;
        }
        ccls[c] = static_cast<uint8_t>(cl);
        if (cl > 0)
            for (int l = 0; l < K; ++l)
                row_skip[m.row_map[m.member_ptr[c] + l]] = cl >= 6 ? 2 : 1;
        atomicAdd(&s_cnt[cl], 1u);
    }
    __syncthreads();
    if (threadIdx.x < NCC) atomicAdd(&counts[threadIdx.x], s_cnt[threadIdx.x]);
}


__global__ void cluster_bucket_kernel(const uint8_t* __restrict__ ccls, int64_t ncl,
                                      unsigned long long* __restrict__ cursor,
                                      int32_t* __restrict__ lists) {
    for (int64_t c = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; c < ncl;
         c += int64_t{gridDim.x} * blockDim.x) {
        const int cl = ccls[c];
        if (cl > 0) lists[atomicAdd(&cursor[cl], 1ull)] = static_cast<int32_t>(c);
    }
}

// ---------------------------------------------------------------------------
// cluster tile kernel: one CTA per cluster on the row-tile machinery
// (merge.cuh).  Expansion: for every merged column p (ascending k) the B row
// is loaded once and its entries are written for every live member l as the
// composite key (l << cbits | j) with value a[p][l] * b — each (p, l) block is
// one sorted run, runs in p-major order.  The stable sort by composite key
// (merge of the runs, CUB radix, or MSD for small tiles — sort_tile) then
// leaves every (member, column) group in ascending k, so each head sums its
// group left to right from 0.0 exactly as row-wise does (= the reference,
// cluster_spgemm.hpp:129-143), and C is written directly as CSR over the
// original rows.
// ---------------------------------------------------------------------------
template <int T, int CAPM>
__global__ void __launch_bounds__(T, CAPM == 3072 ? 3 : (T >= 256 ? (CAPM <= 2048 ? 4 : 2) : (T == 128 ? 8 : 16)))
    cluster_tile_kernel(ClusterMats m, const int32_t* __restrict__ ids, int cbits, int csort,
                        int csort_radix_only,
                        const int64_t* __restrict__ crp, int32_t* __restrict__ ocol,
                        double* __restrict__ oval) {
    using S = MergeShared<T, CAPM>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    __shared__ int32_t s_mstart[MAXK];
    __shared__ int64_t s_mbase[MAXK];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = T / 32;
    constexpr int MAXRUNS = S::MAXRUNS;
    const int32_t c = ids[blockIdx.x];
    const int K = m.sizes[c];
    const int64_t u0 = m.ccp[c], u1 = m.ccp[c + 1];
    const int64_t vbase = m.vptr[c];
    if (tid < K) s_mbase[tid] = crp[m.row_map[m.member_ptr[c] + tid]];
    auto& x = s.ex();
    uint2* slot_sm = reinterpret_cast<uint2*>(x.pav);  // per slot {segment length, member mask}
    uint16_t* slot_rb = s.ro(1);                       // per slot first run index (idle buffer)
    static_assert(S::EX_IN_U, "cluster tiles keep the expansion state in the union (below ro1)");
    int total = 0, nruns = 0;
    for (int64_t uc = u0; uc < u1; uc += T) {
        const int64_t u = uc + tid;
        int seg = 0;
        int64_t start = 0;
        uint32_t msk = 0;
        if (u < u1) {
            const int32_t k = __ldg(m.ccol + u);
            msk = __ldg(m.mask + u);
            start = __ldg(m.brp + k);
            seg = static_cast<int>(__ldg(m.brp + k + 1) - start);
        }
        const int nl = seg > 0 ? __popc(msk) : 0;
        // packed scan: low 16 bits product offset, high 16 bits run index
        const int packed = seg * nl | (nl << 16);
        int off, agg;
        cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(packed, off, agg);
        x.pstart[tid] = start;
        x.poff[tid] = total + (off & 0xffff);
        slot_sm[tid] = make_uint2(static_cast<uint32_t>(seg), nl ? msk : 0u);
        slot_rb[tid] = static_cast<uint16_t>(::min(nruns + (off >> 16), MAXRUNS));
        __syncthreads();
        // run offsets: slot t's live members, in ascending member order
        {
            const uint2 sm = slot_sm[tid];
            uint32_t mm = sm.y;
            int r = slot_rb[tid];
            int o = x.poff[tid];
            while (mm && r < MAXRUNS) {
                mm &= mm - 1;
                s.ro(0)[r++] = static_cast<uint16_t>(o);
                o += static_cast<int>(sm.x);
            }
        }
        const int nslots = static_cast<int>(::min(int64_t{T}, u1 - uc));
        for (int slot = warp; slot < nslots; slot += NW) {
            const uint2 sm = slot_sm[slot];
            if (sm.y == 0) continue;
            const int l_seg = static_cast<int>(sm.x);
            const int64_t st = x.pstart[slot];
            const int o = x.poff[slot];
            const int64_t vb = vbase + (uc + slot - u0) * K;
            for (int q = lane; q < l_seg; q += 32) {
                // one load of the B entry, reused by every live member
                const uint32_t j = static_cast<uint32_t>(__ldg(m.bcol + st + q));
                const double bv = __ldg(m.bval + st + q);
                uint32_t mm = sm.y;
                int pos = o + q;
                while (mm) {
                    const int l = __ffs(mm) - 1;
                    mm &= mm - 1;
                    s.key(0)[PADI(pos)] = (static_cast<uint32_t>(l) << cbits) | j;
                    s.idx(0)[PADI(pos)] = static_cast<uint16_t>(pos);
                    s.val[pos] = __dmul_rn(__ldg(m.aval + vb + l), bv);
                    pos += l_seg;
                }
            }
        }
        total += agg & 0xffff;
        nruns += agg >> 16;
        __syncthreads();
    }
    if (tid == 0) {
        if (nruns <= MAXRUNS) s.ro(0)[nruns] = static_cast<uint16_t>(total);
        s.nruns = nruns;
    }
    __syncthreads();
    const int b = sort_tile<T, CAPM>(s, total, static_cast<uint32_t>(K) << cbits, csort, cbits,
                                  csort_radix_only != 0);

    // reduction (element-strided, as reduce_and_write) with member -> row map
    constexpr int R = (CAPM + T - 1) / T;
    const uint32_t* KS = s.key(b);
    const uint16_t* X = s.idx(b);
    int* cnt = reinterpret_cast<int*>(s.hist);
    const int nrows = (total + T - 1) / T;
    unsigned hm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int o = r * T + tid;
        const bool h = o < total && (o == 0 || KS[PADI(o)] != KS[PADI(o - 1)]);
        hm[r] = __ballot_sync(0xffffffffu, h);
        if (lane == 0 && r < nrows) cnt[r * NW + warp] = __popc(hm[r]);
    }
    __syncthreads();
    const int v = tid < nrows * NW ? cnt[tid] : 0;
    int pre, tile_cnt;
    cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(v, pre, tile_cnt);
    __syncthreads();
    if (tid < nrows * NW) cnt[tid] = pre;
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
    int rank[R];
    double res[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        rank[r] = -1;
        res[r] = 0.0;
        if (!((hm[r] >> lane) & 1u)) continue;
        const int o = r * T + tid;
        rank[r] = cnt[r * NW + warp] + __popc(hm[r] & below);
        const uint32_t key = KS[PADI(o)];
        if (o == 0 || (KS[PADI(o - 1)] >> cbits) != (key >> cbits))
            s_mstart[key >> cbits] = rank[r];  // first entry of this member
        double acc = 0.0;
        int e = o;
        do {
            acc = __dadd_rn(acc, s.val[X[PADI(e)]]);
            ++e;
        } while (e < total && KS[PADI(e)] == key);
        res[r] = acc;
    }
    __syncthreads();
    const uint32_t colmask = (1u << cbits) - 1u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (rank[r] < 0) continue;
        const uint32_t key = KS[PADI(r * T + tid)];
        const int l = static_cast<int>(key >> cbits);
        const int64_t pos = s_mbase[l] + (rank[r] - s_mstart[l]);
        ocol[pos] = static_cast<int32_t>(key & colmask);
        oval[pos] = res[r];
    }
}

// ---------------------------------------------------------------------------
// Union tile (K <= 8): the paper's B-row reuse taken to the sort.  Every B entry
// of the cluster's merged columns is expanded ONCE (column key, b value, merged
// column index) instead of once per live member, the entries are sorted by
// column (stable: ties keep ascending k), and each run of one column is the
// column's slot in the cluster's output union (the CSR_Cluster C columns,
// cluster_spgemm.hpp:86-93).  The run's head then forms, for every live member
// l, sum over the run's entries with l live of a[p][l] * b in run order =
// ascending k from 0.0 — the member's row-wise value bit for bit
// (cluster_spgemm.hpp:129-143) — and writes it at the member's rank of that
// column: a per-member count of earlier union columns holding l (ballots per
// member within a warp + a scan over (row, warp) of packed 16-bit counters).
// Sort work drops from P (member products) to S (B entries loaded): cfg2's
// clusters load each template column's B row once for 8 members.
// ---------------------------------------------------------------------------
// The small tile (<= 1024 entries, <= 256 merged columns, <= 8 members) keeps its
// per-entry and per-column maps in bytes, stages half as many A values and sorts
// with 4-bit radix digits: 31.9 KB = 7 CTAs per SM (38.6 KB = 5 before; the tile
// is latency bound like the row tiles).
template <int T, int CAPM, bool TMA>
struct UnionShared {
    static constexpr bool SMALL = CAPM <= 1024;
    using MS = MergeShared<T, CAPM, 8 * CAPM, SMALL ? 4 : 0>;
    using pidx_t = std::conditional_t<SMALL, uint8_t, uint16_t>;
    using mask_t = std::conditional_t<SMALL, uint8_t, uint32_t>;
    MS m;
    alignas(4) pidx_t pidx[CAPM];  // merged column (local) of each expanded entry
                                   // (TMA: uint32 per 4 staged entries, shift << 16 | column)
    static constexpr int MAXA = SMALL ? UMAXA / 2 : UMAXA;
    static constexpr int MAXMC = SMALL ? UMAXMC / 2 : UMAXMC;
    double sa[MAXA];         // the cluster's A values, [p * K + l]
    mask_t smask[MAXMC];     // live members of merged column p (K <= 8)
    pidx_t runp[T];          // merged column of each compacted run of the chunk
    unsigned long long cnt[2][((CAPM + T - 1) / T) * (T / 32)];  // packed member counts
    int64_t mbase[UMAXK];
    struct NoScan {};
    std::conditional_t<TMA, typename cub::BlockScan<unsigned long long, T>::TempStorage, NoScan>
        scan64;  // TMA staging offsets
};

//
// TMA = true (north star item 3): the cluster's B rows are STAGED in shared
// memory by the TMA engine — one thread per merged column issues two bulk
// copies (cp.async.bulk, columns and values) of the row's 16-byte-aligned
// superset, all of them completing on one mbarrier — instead of one LDGSTS pair
// per B entry.  Slack entries (<= 3 before and after a row) are overwritten
// with a sentinel, and one pass compacts the staged columns into the sort
// buffer; an entry's expansion index is its staged position (values and the
// per-4-entries merged-column map stay where the copy put them).  Rows whose
// superset would reach past nnz(B) are staged with plain loads.
template <int T, int CAPM, bool TMA>
__global__ void __launch_bounds__(T, T >= 256 ? 3 : (TMA ? 6 : 7))
    cluster_union_kernel(ClusterMats m, const int32_t* __restrict__ ids, int csort,
                         const int64_t* __restrict__ crp, int32_t* __restrict__ ocol,
                         double* __restrict__ oval) {
    using U = UnionShared<T, CAPM, TMA>;
    using S = typename U::MS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    U& us = *reinterpret_cast<U*>(smem_raw);
    S& s = us.m;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = T / 32;
    constexpr int R = (CAPM + T - 1) / T;
    const int32_t c = ids[blockIdx.x];
    const int K = m.sizes[c];
    const int64_t u0 = m.ccp[c], u1 = m.ccp[c + 1];
    const int MC = static_cast<int>(u1 - u0);
    const int64_t vbase = m.vptr[c];
    if (tid < K) us.mbase[tid] = crp[m.row_map[m.member_ptr[c] + tid]];
    for (int q = tid; q < MC * K; q += T) us.sa[q] = __ldg(m.aval + vbase + q);
    for (int q = tid; q < MC; q += T)
        us.smask[q] = static_cast<typename U::mask_t>(__ldg(m.mask + u0 + q));
    int total = 0, nruns = 0;
    if constexpr (TMA) {
        __shared__ __align__(8) uint64_t mbar;
        uint32_t* stage = s.u.m.key1;  // staged columns, linear (idle sort buffer)
        uint32_t* grp = reinterpret_cast<uint32_t*>(us.pidx);  // per 4 staged entries: shift << 16 | merged column
        constexpr uint32_t SENT = 0xffffffffu;
        if (tid == 0) mbar_init(&mbar, 1);
        __syncthreads();
        unsigned phase = 0;
        int ptotal = 0;  // staged entries (with slack), a multiple of 4
        const int64_t bulk_end = m.bnnz & ~int64_t{3};
        for (int64_t uc = u0; uc < u1; uc += T) {
            const int64_t u = uc + tid;
            int len = 0, n4 = 0, lead = 0;
            int64_t start = 0;
            if (u < u1 && __ldg(m.mask + u) != 0u) {
                const int32_t k = __ldg(m.ccol + u);
                start = __ldg(m.brp + k);
                len = static_cast<int>(__ldg(m.brp + k + 1) - start);
                if (len > 0) {
                    lead = static_cast<int>(start & 3);
                    n4 = (lead + len + 3) & ~3;
                }
            }
            // one scan: staged offset (bits 0-19), compact offset (20-39), run index (40+)
            const unsigned long long packed = static_cast<unsigned long long>(n4) |
                                              (static_cast<unsigned long long>(len) << 20) |
                                              (static_cast<unsigned long long>(len > 0) << 40);
            unsigned long long off, agg;
            cub::BlockScan<unsigned long long, T>(us.scan64).ExclusiveSum(packed, off, agg);
            const int po = ptotal + static_cast<int>(off & 0xfffffull);
            const int co = total + static_cast<int>((off >> 20) & 0xfffffull);
            const int r = nruns + static_cast<int>(off >> 40);
            if (len > 0) {
                if (r < S::MAXRUNS) s.ro(0)[r] = static_cast<uint16_t>(co);
                const int64_t s4 = start - lead;
                if (s4 + n4 <= bulk_end) {
                    mbar_expect_tx(&mbar, static_cast<unsigned>(n4) * 12u);
                    bulk_g2s(stage + po, m.bcol + s4, static_cast<unsigned>(n4) * 4u, &mbar);
                    bulk_g2s(s.val + po, m.bval + s4, static_cast<unsigned>(n4) * 8u, &mbar);
                } else {  // the last rows of B: no aligned superset inside the arrays
                    for (int j = 0; j < len; ++j) {
                        stage[po + lead + j] = static_cast<uint32_t>(__ldg(m.bcol + start + j));
                        s.val[po + lead + j] = __ldg(m.bval + start + j);
                    }
                }
                const uint32_t g = (static_cast<uint32_t>(po + lead - co) << 16) |
                                   static_cast<uint32_t>(u - u0);
                for (int j = 0; j < n4; j += 4) grp[(po + j) >> 2] = g;
            }
            __syncthreads();  // every expect_tx is registered before the arrival
            if (tid == 0) mbar_arrive(&mbar);
            mbar_wait(&mbar, phase);
            phase ^= 1u;
            if (len > 0) {  // mask the slack around the row
                for (int j = 0; j < lead; ++j) stage[po + j] = SENT;
                for (int j = lead + len; j < n4; ++j) stage[po + j] = SENT;
            }
            ptotal += static_cast<int>(agg & 0xfffffull);
            total += static_cast<int>((agg >> 20) & 0xfffffull);
            nruns += static_cast<int>(agg >> 40);
        }
        __syncthreads();
        // compact the staged columns into the sort buffer (k order kept)
        for (int e = tid; e < ptotal; e += T) {
            const uint32_t k = stage[e];
            if (k != SENT) {
                const int g = e - static_cast<int>(grp[e >> 2] >> 16);
                s.key0[PADI(g)] = k;
                s.idx0[PADI(g)] = static_cast<uint16_t>(e);
            }
        }
    } else {
    auto& x = s.ex();
    for (int64_t uc = u0; uc < u1; uc += T) {
        const int64_t u = uc + tid;
        int len = 0;
        int64_t start = 0;
        if (u < u1 && __ldg(m.mask + u) != 0u) {
            const int32_t k = __ldg(m.ccol + u);
            start = __ldg(m.brp + k);
            len = static_cast<int>(__ldg(m.brp + k + 1) - start);
        }
        const int packed = len | ((len > 0) << 16);
        int off, agg;
        cub::BlockScan<int32_t, T, BSP_SCAN_ALGO>(s.scan).ExclusiveSum(packed, off, agg);
        const int r = off >> 16;
        if (len > 0) {
            if (nruns + r < S::MAXRUNS)
                s.ro(0)[nruns + r] = static_cast<uint16_t>(total + (off & 0xffff));
            x.pstart[r] = start;
            x.poff[r] = off & 0xffff;
            us.runp[r] = static_cast<typename U::pidx_t>(uc + tid - u0);
        }
        const int nr = agg >> 16, ct = agg & 0xffff;
        if (tid == 0) x.poff[nr] = ct;
        __syncthreads();
        {
            int e0, we, qa;
            warp_slice(x.poff, nr, ct, NW, e0, we, qa);
            for (; e0 < we; e0 += 32) {
                const int q = warp_runs(x.poff, nr, e0, qa);
                const int e = e0 + lane;
                if (e < we) {
                    const int64_t src = x.pstart[q] + (e - x.poff[q]);
                    const int g = total + e;
                    cp_async4(&s.key0[PADI(g)], m.bcol + src);
                    cp_async8(&s.val[g], m.bval + src);
                    us.pidx[g] = us.runp[q];
                }
            }
            cp_async_wait_all();
        }
        total += ct;
        nruns += nr;
        __syncthreads();
    }
    }
    if (tid == 0) {
        if (nruns <= S::MAXRUNS) s.ro(0)[nruns] = static_cast<uint16_t>(total);
        s.nruns = nruns;
    }
    __syncthreads();
    // keys are absolute columns (kofs = 0: idx0 is set by the sort's prep)
    // (TMA: idx0 already holds the staged positions)
    const int b = sort_tile<T, CAPM>(s, total, static_cast<uint32_t>(m.ncols), csort, 0, false,
                                     TMA ? -1 : 0);
    const uint32_t* KS = s.key(b);
    const uint16_t* X = s.idx(b);
    // merged column (local) of expansion index xe
    auto mcol = [&](int xe) -> int {
        if constexpr (TMA) return static_cast<int>(reinterpret_cast<const uint32_t*>(us.pidx)[xe >> 2] & 0xffffu);
        else return us.pidx[xe];
    };
    uint32_t* umask = b ? s.key0 : s.u.m.key1;  // the buffer the sort left idle
    // pass A: each head's member mask (OR over its run) and the per-(row, warp)
    // head counts of every member (16-bit fields, members 0-3 and 4-7)
    unsigned hm[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        hm[rr] = 0u;
        if (rr * T >= total) {  // block-uniform: rows past the tile's entries
            if (lane == 0) us.cnt[0][rr * NW + warp] = us.cnt[1][rr * NW + warp] = 0ull;
            continue;
        }
        const int o = rr * T + tid;
        const bool h = o < total && (o == 0 || KS[PADI(o)] != KS[PADI(o - 1)]);
        hm[rr] = __ballot_sync(0xffffffffu, h);
        uint32_t M = 0;
        if (h) {
            const uint32_t key = KS[PADI(o)];
            int e = o;
            do {
                M |= us.smask[mcol(X[PADI(e)])];
                ++e;
            } while (e < total && KS[PADI(e)] == key);
            umask[o] = M;
        }
        unsigned long long ca = 0, cb = 0;
#pragma unroll
        for (int l = 0; l < UMAXK; ++l) {
            if (l >= K) break;
            const unsigned bl = __ballot_sync(0xffffffffu, (M >> l) & 1u);
            if (l < 4) ca |= static_cast<unsigned long long>(__popc(bl)) << (16 * l);
            else cb |= static_cast<unsigned long long>(__popc(bl)) << (16 * (l - 4));
        }
        if (lane == 0) {
            us.cnt[0][rr * NW + warp] = ca;
            us.cnt[1][rr * NW + warp] = cb;
        }
    }
    __syncthreads();
    // exclusive scan of the packed counters over (row, warp), in sorted order
    constexpr int NC = R * NW;
    static_assert(NC <= 64, "one warp scans the (row, warp) counters");
    if (warp == 0) {
        unsigned long long a0 = 2 * lane < NC ? us.cnt[0][2 * lane] : 0ull;
        unsigned long long a1 = 2 * lane + 1 < NC ? us.cnt[0][2 * lane + 1] : 0ull;
        unsigned long long b0 = 2 * lane < NC ? us.cnt[1][2 * lane] : 0ull;
        unsigned long long b1 = 2 * lane + 1 < NC ? us.cnt[1][2 * lane + 1] : 0ull;
        unsigned long long sa_ = a0 + a1, sb_ = b0 + b1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long ta = __shfl_up_sync(0xffffffffu, sa_, o);
            const unsigned long long tb = __shfl_up_sync(0xffffffffu, sb_, o);
            if (lane >= o) {
                sa_ += ta;
                sb_ += tb;
            }
        }
        const unsigned long long ea = sa_ - (a0 + a1), eb = sb_ - (b0 + b1);  // exclusive
        if (2 * lane < NC) {
            us.cnt[0][2 * lane] = ea;
            us.cnt[1][2 * lane] = eb;
        }
        if (2 * lane + 1 < NC) {
            us.cnt[0][2 * lane + 1] = ea + a0;
            us.cnt[1][2 * lane + 1] = eb + b0;
        }
    }
    __syncthreads();
    // pass B: per head, each live member's sum in run (= k) order, written at
    // that member's rank of the column
    const unsigned below = (1u << lane) - 1u;
#pragma unroll 1
    for (int rr = 0; rr < R; ++rr) {
        if (rr * T >= total) break;
        const int o = rr * T + tid;
        const bool h = (hm[rr] >> lane) & 1u;
        const uint32_t M = h ? umask[o] : 0u;
        const unsigned long long pa = us.cnt[0][rr * NW + warp], pb = us.cnt[1][rr * NW + warp];
        int pos[UMAXK];
#pragma unroll
        for (int l = 0; l < UMAXK; ++l) {
            pos[l] = 0;
            if (l >= K) continue;
            const unsigned bl = __ballot_sync(0xffffffffu, (M >> l) & 1u);
            const unsigned long long pw = l < 4 ? pa : pb;
            pos[l] = static_cast<int>((pw >> (16 * (l & 3))) & 0xffffull) + __popc(bl & below);
        }
        if (!h) continue;
        double acc[UMAXK];
#pragma unroll
        for (int l = 0; l < UMAXK; ++l) acc[l] = 0.0;
        const uint32_t key = KS[PADI(o)];
        int e = o;
        do {
            const int xe = X[PADI(e)];
            const int p = mcol(xe);
            const double bv = s.val[xe];
            const uint32_t mp = us.smask[p];
            const double* ap = us.sa + p * K;
#pragma unroll
            for (int l = 0; l < UMAXK; ++l)
                if ((mp >> l) & 1u) acc[l] = __dadd_rn(acc[l], __dmul_rn(ap[l], bv));
            ++e;
        } while (e < total && KS[PADI(e)] == key);
#pragma unroll
        for (int l = 0; l < UMAXK; ++l) {
            if (!((M >> l) & 1u)) continue;
            const int64_t q = us.mbase[l] + pos[l];
            ocol[q] = static_cast<int32_t>(key);
            oval[q] = acc[l];
        }
    }
}

// Symbolic count of the union tiles' rows from the cluster's B rows, each loaded
// once (the symbolic twin of cluster_union_kernel; replaces one row-wise hash
// count per member, hash_accumulator.hpp:48-54 / spgemm.hpp:41-63): every B
// entry of a live merged column is inserted once into a CTA-wide open-addressed
// table whose slot also collects the live members (OR); member l's output count
// is the number of slots holding l.
template <int T, int HS>
__global__ void __launch_bounds__(T) cluster_union_count_kernel(ClusterMats m,
                                                               const int32_t* __restrict__ ids,
                                                               int64_t* __restrict__ row_nnz) {
    __shared__ int32_t keys[HS];
    __shared__ uint32_t mem[HS];
    __shared__ int s_cnt[UMAXK];
    constexpr int LG = 31 - __builtin_clz(static_cast<unsigned>(HS));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = T / 32;
    const int32_t c = ids[blockIdx.x];
    const int K = m.sizes[c];
    for (int i = tid; i < HS; i += T) {
        keys[i] = -1;
        mem[i] = 0u;
    }
    if (tid < UMAXK) s_cnt[tid] = 0;
    __syncthreads();
    const int64_t u0 = m.ccp[c], u1 = m.ccp[c + 1];
    // a warp per merged column (its B row read coalesced), columns strided over warps
    for (int64_t u = u0 + warp; u < u1; u += NW) {
        const uint32_t mk = __ldg(m.mask + u);
        if (!mk) continue;
        const int32_t k = __ldg(m.ccol + u);
        const int64_t b0 = __ldg(m.brp + k), b1 = __ldg(m.brp + k + 1);
        for (int64_t q = b0 + lane; q < b1; q += 32) {
            const int32_t col = __ldg(m.bcol + q);
            uint32_t slot = col_hash(static_cast<uint32_t>(col), LG);
            for (;;) {
                const int32_t prev = atomicCAS(&keys[slot], -1, col);
                if (prev == -1 || prev == col) break;
                slot = (slot + 1) & (HS - 1);
            }
            atomicOr(&mem[slot], mk);
        }
    }
    __syncthreads();
    int cnt[UMAXK];
#pragma unroll
    for (int l = 0; l < UMAXK; ++l) cnt[l] = 0;
    for (int i = tid; i < HS; i += T) {
        const uint32_t x = mem[i];
#pragma unroll
        for (int l = 0; l < UMAXK; ++l) cnt[l] += (x >> l) & 1u;
    }
#pragma unroll
    for (int l = 0; l < UMAXK; ++l) {
        int v = cnt[l];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&s_cnt[l], v);
    }
    __syncthreads();
    if (tid < K) row_nnz[m.row_map[m.member_ptr[c] + tid]] = s_cnt[tid];
}

// BSP_CLUSTER_TMA=1: the union tiles stage their B rows with bulk copies instead
// of gathering them with per-entry LDGSTS.  Bulk copies also need 16-byte
// aligned B arrays (cudaMalloc'ed arrays are; a caller's offset view may not be).
bool union_tma(const ClusterMats& m) {
    static const bool on = [] {
        const char* e = std::getenv("BSP_CLUSTER_TMA");
        return e && e[0] == '1';  // measured slower on cfg2 (0.986 vs 0.919 ms): off by default
    }();
    return on && (reinterpret_cast<uintptr_t>(m.bcol) & 15u) == 0 &&
           (reinterpret_cast<uintptr_t>(m.bval) & 15u) == 0;
}

template <int T, int CAPM>
void launch_union(bsp_handle h, const ClusterMats& m, const int32_t* ids, int64_t n,
                  const int64_t* crp, int32_t* ocol, double* oval) {
    if (n <= 0) return;
    static const std::string nm =
        "cluster_union<" + std::to_string(T) + "," + std::to_string(CAPM) + ">";
    static const std::string nm_tma =
        "cluster_union_tma<" + std::to_string(T) + "," + std::to_string(CAPM) + ">";
    static const int csort = [] {
        const char* e = std::getenv("BSP_CSORT");
        return e ? std::atoi(e) : 1000;
    }();
    if (union_tma(m)) {
        using U = UnionShared<T, CAPM, true>;
        auto k = cluster_union_kernel<T, CAPM, true>;
        set_smem(k, sizeof(U));
        BSP_LAUNCH_AS(h, nm_tma.c_str(), k, static_cast<unsigned>(n), T, sizeof(U), m, ids, csort,
                      crp, ocol, oval);
    } else {
        using U = UnionShared<T, CAPM, false>;
        auto k = cluster_union_kernel<T, CAPM, false>;
        set_smem(k, sizeof(U));
        BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(U), m, ids, csort, crp,
                      ocol, oval);
    }
}

// ---------------------------------------------------------------------------
// Duplicate-heavy clusters of two rows (cfg4 after RCM + hierarchical: stencil
// rows of 729 products -> 125 columns, neighbours sharing most B rows): a warp
// per cluster, the row-wise hash accumulator (rowwise.cu hashacc_kernel) with
// one value slot per member.  Merged columns are walked in ascending k; each B
// row is loaded ONCE, its columns inserted once into the warp's table, and
// a[p][l] * b added for each live member l — a segment's columns are distinct,
// so no two lanes collide and every (column, member) sum is formed in
// ascending k from 0.0 (cluster_spgemm.hpp:129-143 = the row-wise order).
// Then each member's columns are compacted and ranked and written as CSR.
// Routed after the symbolic pass: K == 2, products >= 2 x outputs, <= 256
// outputs per member (the table has 512 slots).
// ---------------------------------------------------------------------------
constexpr int CH_WARPS = 4, CH_HS = 512, CH_MAX = 256;
struct ClusterHaccShared {
    int32_t key[CH_WARPS][CH_HS];
    uint32_t pres[CH_WARPS][CH_HS];  // live-member bits of each slot
    double val[CH_WARPS][CH_HS][2];
    uint16_t order[CH_WARPS][CH_HS];  // union rank -> compacted entry
};

__global__ void __launch_bounds__(CH_WARPS * 32)
    cluster_hashacc_kernel(ClusterMats m, const int32_t* __restrict__ ids, int64_t n,
                           const int64_t* __restrict__ crp, int32_t* __restrict__ ocol,
                           double* __restrict__ oval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ClusterHaccShared& s = *reinterpret_cast<ClusterHaccShared*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* keys = s.key[warp];
    uint32_t* pres = s.pres[warp];
    double(*vals)[2] = s.val[warp];
    uint16_t* order = s.order[warp];
    constexpr int LG = 31 - __builtin_clz(static_cast<unsigned>(CH_HS));
    constexpr int PER = CH_HS / 32;  // union entries per lane (<= 2 x CH_MAX)
    const unsigned below = (1u << lane) - 1u;
    for (int64_t t = blockIdx.x * int64_t{CH_WARPS} + warp; t < n;
         t += int64_t{gridDim.x} * CH_WARPS) {
        const int32_t c = ids[t];
        for (int i = lane; i < CH_HS; i += 32) {
            keys[i] = -1;
            pres[i] = 0u;
        }
        __syncwarp();
        const int64_t u0 = m.ccp[c], u1 = m.ccp[c + 1], vb = m.vptr[c];
        for (int64_t ub = u0; ub < u1; ub += 32) {
            const int64_t u = ub + lane;
            int64_t b0 = 0;
            int len = 0;
            uint32_t mk = 0;
            double a0 = 0.0, a1 = 0.0;
            if (u < u1) {
                mk = __ldg(m.mask + u) & 3u;
                if (mk) {
                    const int32_t k = __ldg(m.ccol + u);
                    b0 = __ldg(m.brp + k);
                    len = static_cast<int>(__ldg(m.brp + k + 1) - b0);
                    a0 = __ldg(m.aval + vb + (u - u0) * 2);
                    a1 = __ldg(m.aval + vb + (u - u0) * 2 + 1);
                }
            }
            unsigned ne = __ballot_sync(0xffffffffu, len > 0);
            while (ne) {
                const int j = __ffs(ne) - 1;
                ne &= ne - 1;
                const int64_t bj = __shfl_sync(0xffffffffu, b0, j);
                const int lj = __shfl_sync(0xffffffffu, len, j);
                const uint32_t mj = __shfl_sync(0xffffffffu, mk, j);
                const double aj0 = __shfl_sync(0xffffffffu, a0, j);
                const double aj1 = __shfl_sync(0xffffffffu, a1, j);
                for (int q = lane; q < lj; q += 32) {
                    const int32_t col = __ldg(m.bcol + bj + q);
                    const double bv = __ldg(m.bval + bj + q);
                    uint32_t slot = col_hash(static_cast<uint32_t>(col), LG);
                    for (;;) {
                        const int32_t prev = atomicCAS(&keys[slot], -1, col);
                        if (prev == -1 || prev == col) break;
                        slot = (slot + 1) & (CH_HS - 1);
                    }
                    const uint32_t had = pres[slot];
                    if (mj & 1u)
                        vals[slot][0] =
                            __dadd_rn((had & 1u) ? vals[slot][0] : 0.0, __dmul_rn(aj0, bv));
                    if (mj & 2u)
                        vals[slot][1] =
                            __dadd_rn((had & 2u) ? vals[slot][1] : 0.0, __dmul_rn(aj1, bv));
                    pres[slot] = had | mj;
                }
                __syncwarp();  // the next B row adds after this one (ascending k)
            }
        }
        // compact the union's slots to the front (ascending slot order; a block
        // of 32 slots is read before any position inside it is written)
        int U = 0;
        for (int i0 = 0; i0 < CH_HS; i0 += 32) {
            const int32_t kk = keys[i0 + lane];
            const uint32_t pp = pres[i0 + lane];
            const double v0 = vals[i0 + lane][0], v1 = vals[i0 + lane][1];
            const unsigned occ = __ballot_sync(0xffffffffu, kk >= 0);
            __syncwarp();
            if (kk >= 0) {
                const int pos = U + __popc(occ & below);
                keys[pos] = kk;
                pres[pos] = pp;
                vals[pos][0] = v0;
                vals[pos][1] = v1;
            }
            U += __popc(occ);
            __syncwarp();
        }
        // union rank of each entry (counting against the compacted keys,
        // read as warp broadcasts), then order[rank] = entry
        int32_t mk[PER];
        int rk[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int e = u * 32 + lane;
            mk[u] = e < U ? keys[e] : 0x7fffffff;
            rk[u] = 0;
        }
        auto rank_cols = [&](auto nu_c) {
            constexpr int NU = decltype(nu_c)::value;
            for (int jj = 0; jj < U; ++jj) {
                const int32_t kj = keys[jj];
#pragma unroll
                for (int u = 0; u < NU; ++u) rk[u] += kj < mk[u];
            }
        };
        if (U <= 128) rank_cols(std::integral_constant<int, 4>{});
        else if (U <= 256) rank_cols(std::integral_constant<int, 8>{});
        else rank_cols(std::integral_constant<int, PER>{});
#pragma unroll
        for (int u = 0; u < PER; ++u)
            if (u * 32 + lane < U) order[rk[u]] = static_cast<uint16_t>(u * 32 + lane);
        __syncwarp();
        // each member's columns in ascending order: ballot prefix -> coalesced stores
        const int64_t mb = m.member_ptr[c];
        const int64_t base0 = crp[m.row_map[mb]], base1 = crp[m.row_map[mb + 1]];
        int n0 = 0, n1 = 0;
        for (int i0 = 0; i0 < U; i0 += 32) {
            const int i = i0 + lane;
            const int e = i < U ? order[i] : 0;
            const uint32_t pm = i < U ? pres[e] : 0u;
            const unsigned m0 = __ballot_sync(0xffffffffu, pm & 1u);
            const unsigned m1 = __ballot_sync(0xffffffffu, (pm >> 1) & 1u);
            if (pm & 1u) {
                const int64_t q = base0 + n0 + __popc(m0 & below);
                ocol[q] = keys[e];
                oval[q] = vals[e][0];
            }
            if (pm & 2u) {
                const int64_t q = base1 + n1 + __popc(m1 & below);
                ocol[q] = keys[e];
                oval[q] = vals[e][1];
            }
            n0 += __popc(m0);
            n1 += __popc(m1);
        }
        __syncwarp();
    }
}

// After the symbolic pass: duplicate-heavy clusters (products >= 2 x outputs, <=
// CH_MAX outputs per member) leave the sort tiles.  Two-row clusters whose B-row
// reuse (products / B entries loaded once) reaches hacc_reuse10 / 10 go to
// cluster_hashacc_kernel (hlist); the other duplicate-heavy clusters hand their
// member rows to the row-wise hash accumulator (rlist) — measured on cfg4
// (RCM + hierarchical: pairs of stencil rows, reuse 1.5x): 18.9 ms on the cluster
// accumulator vs 13.0 ms row-wise, the shared loads saving less than the
// per-member bookkeeping costs (the paper's own stencil finding).  The rest keep
// their class (tlists, per-class cursors).  cursor[NCC] counts rlist's rows.
__global__ void route_cluster_kernel(ClusterMats m, const int32_t* __restrict__ lists,
                                     const uint8_t* __restrict__ ccls, int64_t nlist,
                                     const int64_t* __restrict__ crp,
                                     unsigned long long* __restrict__ cursor,
                                     int32_t* __restrict__ hlist, int32_t* __restrict__ tlists,
                                     int32_t* __restrict__ rlist, int hacc_reuse10) {
    const int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (t >= nlist) return;
    const int32_t c = lists[t];
    const int64_t mb = m.member_ptr[c];
    const int K = static_cast<int>(m.member_ptr[c + 1] - mb);
    int64_t Z = 0, zmax = 0;
    for (int l = 0; l < K; ++l) {
        const int32_t r = m.row_map[mb + l];
        const int64_t z = crp[r + 1] - crp[r];
        Z += z;
        zmax = max(zmax, z);
    }
    int64_t P = 0, S = 0;
    for (int64_t u = m.ccp[c]; u < m.ccp[c + 1]; ++u) {
        const int32_t k = m.ccol[u];
        const int64_t len = m.brp[k + 1] - m.brp[k];
        const int live = __popc(m.mask[u]);
        P += static_cast<int64_t>(live) * len;
        if (live) S += len;
    }
    const bool dup = zmax <= CH_MAX && P >= 2 * Z;
    if (dup && K == 2 && 10 * P >= static_cast<int64_t>(hacc_reuse10) * S) {
        hlist[atomicAdd(&cursor[0], 1ull)] = c;
    } else if (dup) {
        const unsigned long long o = atomicAdd(&cursor[NCC], static_cast<unsigned long long>(K));
        for (int l = 0; l < K; ++l) rlist[o + l] = m.row_map[mb + l];
    } else {
        tlists[atomicAdd(&cursor[ccls[c]], 1ull)] = c;
    }
}

template <int T, int CAPM>
void launch_cluster(bsp_handle h, const ClusterMats& m, const int32_t* ids, int64_t n, int cbits,
                    const int64_t* crp, int32_t* ocol, double* oval) {
    if (n <= 0) return;
    using S = MergeShared<T, CAPM>;
    auto k = cluster_tile_kernel<T, CAPM>;
    static const std::string nm =
        "cluster_numeric<" + std::to_string(T) + "," + std::to_string(CAPM) + ">";
    // BSP_CSORT=0: radix/merge only (as the row-wise tiles)
    static const int csort = [] {
        const char* e = std::getenv("BSP_CSORT");
        return e ? std::atoi(e) : 1000;
    }();
    set_smem(k, sizeof(S));
    static const int ronly = [] {
        const char* e = std::getenv("BSP_CSORT_CL_RADIX_ONLY");
        return e ? std::atoi(e) : 1;
    }();
    BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(S), m, ids, cbits, csort,
                  ronly, crp, ocol, oval);
}

void run_cluster_classes(bsp_handle h, const ClusterMats& m, const int32_t* lists,
                         const int64_t* off, const int64_t* cnt, int cbits, const int64_t* crp,
                         int32_t* ocol, double* oval) {
    static_assert(NCC == 8, "one launch per cluster tile class");
    launch_union<256, 2048>(h, m, lists + off[7], cnt[7], crp, ocol, oval);
    launch_union<128, 1024>(h, m, lists + off[6], cnt[6], crp, ocol, oval);
    launch_cluster<64, 512>(h, m, lists + off[1], cnt[1], cbits, crp, ocol, oval);
    launch_cluster<128, 1024>(h, m, lists + off[2], cnt[2], cbits, crp, ocol, oval);
    launch_cluster<256, 2048>(h, m, lists + off[3], cnt[3], cbits, crp, ocol, oval);
    launch_cluster<256, 3072>(h, m, lists + off[4], cnt[4], cbits, crp, ocol, oval);
    launch_cluster<256, 4096>(h, m, lists + off[5], cnt[5], cbits, crp, ocol, oval);
}

// access statistics (reference cluster_spgemm.hpp:26-45, counted at :129-135)
__global__ void cluster_stats_kernel(const int32_t* __restrict__ sizes,
                                     const int64_t* __restrict__ ccp,
                                     const int32_t* __restrict__ ccol,
                                     const uint32_t* __restrict__ mask,
                                     const unsigned long long* __restrict__ valid,
                                     const int64_t* __restrict__ vptr,
                                     const int64_t* __restrict__ brp, int64_t ncl,
                                     unsigned long long* __restrict__ out) {
    unsigned long long loads = 0, iters = 0, skips = 0;
    for (int64_t c = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; c < ncl;
         c += int64_t{gridDim.x} * blockDim.x) {
        const int K = sizes[c];
        for (int64_t u = ccp[c]; u < ccp[c + 1]; ++u) {
            const int32_t k = ccol[u];
            const int64_t bn = brp[k + 1] - brp[k];
            if (bn == 0) continue;
            ++loads;
            iters += static_cast<unsigned long long>(K * bn);
            skips += static_cast<unsigned long long>(
                (K - live_count(mask, valid, u, vptr[c] + (u - ccp[c]) * K, K)) * bn);
        }
    }
    atomicAdd(&out[0], loads);
    atomicAdd(&out[1], iters);
    atomicAdd(&out[2], skips);
}

__global__ void rowwise_stats_kernel(const int32_t* __restrict__ acol, int64_t nnz,
                                     const int64_t* __restrict__ brp,
                                     unsigned long long* __restrict__ out) {
    unsigned long long loads = 0, iters = 0;
    for (int64_t p = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; p < nnz;
         p += int64_t{gridDim.x} * blockDim.x) {
        const int32_t k = acol[p];
        const int64_t bn = brp[k + 1] - brp[k];
        if (bn > 0) {
            ++loads;
            iters += static_cast<unsigned long long>(bn);
        }
    }
    atomicAdd(&out[0], loads);
    atomicAdd(&out[1], iters);
}

int grid_for(bsp_handle h, int64_t n, int block) {
    return static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(std::max<int64_t>(n, 1), block), int64_t{h->sm_count} * 16)));
}

// Narrow-B routing: clusters of 2..MAXK members go to the cluster kernel and
// their rows are skipped by the row kernel.
__global__ void narrow_route_kernel(ClusterMats m, int64_t ncl, uint8_t* __restrict__ skip,
                                    int32_t* __restrict__ lists,
                                    unsigned long long* __restrict__ count) {
    for (int64_t c = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; c < ncl;
         c += int64_t{gridDim.x} * blockDim.x) {
        const int64_t mb = m.member_ptr[c], K = m.member_ptr[c + 1] - mb;
        if (K < 2 || K > MAXK) continue;
        lists[atomicAdd(count, 1ull)] = static_cast<int32_t>(c);
        for (int64_t l = 0; l < K; ++l) skip[m.row_map[mb + l]] = 1;
    }
}

// Cluster-wise multiply for B with <= 64 columns (the tall-skinny frontier
// operands): a warp per cluster walks its merged columns in k order; each B
// row's 64-bit column mask and values are loaded ONCE and scattered into the
// register accumulators (columns lane, lane + 32) of every live member — the
// paper's B-row reuse across a cluster.  Per member and column the adds come in
// ascending k from 0.0, as in the member's row-wise multiply.  Members are
// taken 8 at a time (accumulators in registers).
constexpr int CN_WARPS = 8, CN_GROUP = 8;

__global__ void __launch_bounds__(CN_WARPS * 32)
    cluster_narrow64_kernel(ClusterMats m, const unsigned long long* __restrict__ bmask,
                            const int32_t* __restrict__ ids, int64_t ncl,
                            const int64_t* __restrict__ crp, int32_t* __restrict__ ocol,
                            double* __restrict__ oval) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long below0 = (1ull << lane) - 1ull, below1 = (1ull << (lane + 32)) - 1ull;
    for (int64_t t = blockIdx.x * int64_t{CN_WARPS} + warp; t < ncl;
         t += int64_t{gridDim.x} * CN_WARPS) {
        const int32_t c = ids[t];
        const int64_t mb = m.member_ptr[c];
        const int K = static_cast<int>(m.member_ptr[c + 1] - mb);
        const int64_t u0 = m.ccp[c], u1 = m.ccp[c + 1], vb = m.vptr[c];
        for (int g0 = 0; g0 < K; g0 += CN_GROUP) {
            const uint32_t gmask = ((K - g0 >= 32) ? 0xffffffffu : ((1u << (K - g0)) - 1u)) &
                                   ((1u << CN_GROUP) - 1u);
            double acc0[CN_GROUP], acc1[CN_GROUP];
            unsigned long long touch[CN_GROUP];
#pragma unroll
            for (int l = 0; l < CN_GROUP; ++l) {
                acc0[l] = 0.0;
                acc1[l] = 0.0;
                touch[l] = 0ull;
            }
            for (int64_t ub = u0; ub < u1; ub += 32) {
                const int64_t u = ub + lane;
                unsigned long long mk = 0;
                int64_t b0 = 0;
                uint32_t mm = 0;
                if (u < u1) {
                    const int32_t k = __ldg(m.ccol + u);
                    mm = (__ldg(m.mask + u) >> g0) & gmask;
                    if (mm) {
                        mk = __ldg(bmask + k);
                        b0 = __ldg(m.brp + k);
                    }
                }
                unsigned ne = __ballot_sync(0xffffffffu, mk != 0 && mm != 0);
                while (ne) {
                    const int j = __ffs(ne) - 1;
                    ne &= ne - 1;
                    const unsigned long long mj = __shfl_sync(0xffffffffu, mk, j);
                    const int64_t bj = __shfl_sync(0xffffffffu, b0, j);
                    const uint32_t mmj = __shfl_sync(0xffffffffu, mm, j);
                    const int64_t uj = ub + j;
                    const bool h0 = (mj >> lane) & 1ull, h1 = (mj >> (lane + 32)) & 1ull;
                    const double bv0 = h0 ? __ldg(m.bval + bj + __popcll(mj & below0)) : 0.0;
                    const double bv1 = h1 ? __ldg(m.bval + bj + __popcll(mj & below1)) : 0.0;
                    const double* av = m.aval + vb + (uj - u0) * K + g0;
#pragma unroll
                    for (int l = 0; l < CN_GROUP; ++l) {
                        if (!((mmj >> l) & 1u)) continue;
                        const double a = __ldg(av + l);
                        if (h0) acc0[l] = __dadd_rn(acc0[l], __dmul_rn(a, bv0));
                        if (h1) acc1[l] = __dadd_rn(acc1[l], __dmul_rn(a, bv1));
                        touch[l] |= mj;
                    }
                }
            }
#pragma unroll
            for (int l = 0; l < CN_GROUP; ++l) {
                if (g0 + l >= K) break;
                const int32_t row = m.row_map[mb + g0 + l];
                const int64_t pos = crp[row];
                const unsigned long long T = touch[l];  // warp-uniform (broadcast masks)
                if ((T >> lane) & 1ull) {
                    const int64_t o = pos + __popcll(T & below0);
                    ocol[o] = lane;
                    oval[o] = acc0[l];
                }
                if ((T >> (lane + 32)) & 1ull) {
                    const int64_t o = pos + __popcll(T & below1);
                    ocol[o] = lane + 32;
                    oval[o] = acc1[l];
                }
            }
        }
    }
}

ClusterMats make_cluster_mats(const bsp_csr_cluster* a, const bsp_csr* b) {
    return ClusterMats{a->cluster_sizes, a->member_ptr, a->cluster_col_ptr, a->col_idx,
                       a->value_ptr,     a->values,     a->member_mask,     a->row_map,
                       b->row_ptr,       b->col_idx,    b->values,          static_cast<int32_t>(b->ncols),
                       b->nnz};
}

}  // namespace

// Builds the device CSR_Cluster of a device CSR for a device-resident
// assignment (member_ptr/rows already on the device, owned by `out`).
void build_cluster_device(bsp_handle h, const bsp_csr* A, int64_t ncl, int64_t* mptr,
                          int32_t* rows, bool keep_csr, bsp_csr_cluster* out) {
    DBuf<int64_t> ucount(h, ncl + 1);
    BSP_CUDA(cudaMemsetAsync(ucount.p, 0, (ncl + 1) * sizeof(int64_t), h->stream));
    const int g = grid_for(h, ncl * 32, 256);
    BSP_LAUNCH(h, build_cluster_kernel<0>, g, 256, 0, A->row_ptr, A->col_idx, A->values, ncl, mptr,
               rows, ucount.p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    BSP_LAUNCH(h, build_cluster_big_kernel<0>, g, 256, 0, A->row_ptr, A->col_idx, A->values, ncl,
               mptr, rows, ucount.p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    DBuf<int64_t> ccp(h, ncl + 1, Pool::out);
    exclusive_scan_i64(h, ucount.p, ccp.p, ncl + 1);
    DBuf<int64_t> slots(h, ncl + 1);
    DBuf<int32_t> sizes(h, ncl, Pool::out);
    BSP_CUDA(cudaMemsetAsync(slots.p + ncl, 0, sizeof(int64_t), h->stream));
    BSP_LAUNCH(h, value_ptr_kernel, grid_for(h, ncl, 256), 256, 0, ucount.p, mptr, ncl, slots.p,
               sizes.p);
    DBuf<int64_t> vptr(h, ncl + 1, Pool::out);
    exclusive_scan_i64(h, slots.p, vptr.p, ncl + 1);
    int64_t tot[2];
    d2h(h, &tot[0], ccp.p + ncl, 1);
    d2h(h, &tot[1], vptr.p + ncl, 1);
    sync(h);
    const int64_t ncolslots = tot[0], nslots = tot[1];
    DBuf<int32_t> ocol(h, ncolslots, Pool::out);
    DBuf<uint32_t> omask(h, ncolslots, Pool::out);
    DBuf<double> oval(h, nslots, Pool::out);
    const int64_t nwords = (nslots + 63) / 64;
    DBuf<uint64_t> valid(h, nwords, Pool::out);
    BSP_CUDA(cudaMemsetAsync(oval.p, 0, std::max<int64_t>(nslots, 1) * sizeof(double), h->stream));
    BSP_CUDA(cudaMemsetAsync(valid.p, 0, std::max<int64_t>(nwords, 1) * sizeof(uint64_t), h->stream));
    BSP_LAUNCH(h, build_cluster_kernel<1>, g, 256, 0, A->row_ptr, A->col_idx, A->values, ncl, mptr,
               rows, nullptr, ccp.p, vptr.p, ocol.p, oval.p,
               reinterpret_cast<unsigned long long*>(valid.p), omask.p);
    BSP_LAUNCH(h, build_cluster_big_kernel<1>, g, 256, 0, A->row_ptr, A->col_idx, A->values, ncl,
               mptr, rows, nullptr, ccp.p, vptr.p, ocol.p, oval.p,
               reinterpret_cast<unsigned long long*>(valid.p), omask.p);
    out->nclusters = ncl;
    out->nrows = A->nrows;
    out->ncols = A->ncols;
    out->ncolslots = ncolslots;
    out->nslots = nslots;
    out->cluster_sizes = sizes.release();
    out->member_ptr = mptr;
    out->cluster_col_ptr = ccp.release();
    out->col_idx = ocol.release();
    out->value_ptr = vptr.release();
    out->values = oval.release();
    out->valid = valid.release();
    out->member_mask = omask.release();
    out->row_map = rows;
    out->csr_row_ptr = nullptr;
    out->csr_col_idx = nullptr;
    out->csr_values = nullptr;
    out->csr_nnz = 0;
    if (keep_csr) {
        DBuf<int64_t> rp(h, A->nrows + 1, Pool::out);
        DBuf<int32_t> ci(h, A->nnz, Pool::out);
        DBuf<double> v(h, A->nnz, Pool::out);
        BSP_CUDA(cudaMemcpyAsync(rp.p, A->row_ptr, (A->nrows + 1) * sizeof(int64_t),
                                 cudaMemcpyDeviceToDevice, h->stream));
        BSP_CUDA(cudaMemcpyAsync(ci.p, A->col_idx, A->nnz * sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, h->stream));
        BSP_CUDA(cudaMemcpyAsync(v.p, A->values, A->nnz * sizeof(double),
                                 cudaMemcpyDeviceToDevice, h->stream));
        out->csr_row_ptr = rp.release();
        out->csr_col_idx = ci.release();
        out->csr_values = v.release();
        out->csr_nnz = A->nnz;
    }
    out->owned = 1;
}

void cluster_to_csr_device(bsp_handle h, const bsp_csr_cluster* m, bsp_csr* out) {
    const int64_t n = m->nrows;
    DBuf<int64_t> cnt(h, n + 1);
    BSP_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(int64_t), h->stream));
    const int g = grid_for(h, m->nclusters * 32, 256);
    BSP_LAUNCH(h, cluster_to_csr_kernel<0>, g, 256, 0, m->cluster_sizes, m->member_ptr,
               m->cluster_col_ptr, m->col_idx, m->value_ptr, m->values, m->member_mask,
               reinterpret_cast<const unsigned long long*>(m->valid), m->row_map, m->nclusters,
               cnt.p, nullptr, nullptr, nullptr);
    DBuf<int64_t> rp(h, n + 1, Pool::out);
    exclusive_scan_i64(h, cnt.p, rp.p, n + 1);
    const int64_t nnz = read_scalar(h, rp.p + n);
    DBuf<int32_t> ci(h, nnz, Pool::out);
    DBuf<double> v(h, nnz, Pool::out);
    BSP_LAUNCH(h, cluster_to_csr_kernel<1>, g, 256, 0, m->cluster_sizes, m->member_ptr,
               m->cluster_col_ptr, m->col_idx, m->value_ptr, m->values, m->member_mask,
               reinterpret_cast<const unsigned long long*>(m->valid), m->row_map, m->nclusters,
               nullptr, rp.p, ci.p, v.p);
    out->nrows = n;
    out->ncols = m->ncols;
    out->nnz = nnz;
    out->row_ptr = rp.release();
    out->col_idx = ci.release();
    out->values = v.release();
    out->owned = 1;
}

void free_cluster(bsp_handle h, bsp_csr_cluster* m) {
    if (!m || !m->owned) return;
    void* ptrs[] = {m->cluster_sizes, m->member_ptr, m->cluster_col_ptr, m->col_idx,
                    m->value_ptr,     m->values,     m->valid,           m->member_mask,
                    m->row_map,       m->csr_row_ptr, m->csr_col_idx,    m->csr_values};
    for (void* p : ptrs) dfree(h, p);
    *m = bsp_csr_cluster{};
}

}  // namespace bsp

using namespace bsp;

namespace bsp {
namespace {
// Intermediate products of each cluster (one warp per cluster): over its merged
// columns p, (live members of p) x nnz(B row col[p]) — the sum of its member
// rows' row_upper_bound (spgemm.hpp:31-36), placeholders not counted.
__global__ void cluster_work_kernel(const int64_t* __restrict__ ccp, const int32_t* __restrict__ col,
                                    const uint32_t* __restrict__ mask,
                                    const unsigned long long* __restrict__ valid,
                                    const int64_t* __restrict__ vptr,
                                    const int32_t* __restrict__ sizes,
                                    const int64_t* __restrict__ brp, int64_t ncl,
                                    int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = int64_t{gridDim.x} * (blockDim.x >> 5);
    for (int64_t c = blockIdx.x * int64_t{blockDim.x >> 5} + (threadIdx.x >> 5); c < ncl; c += nw) {
        int64_t P = 0;
        for (int64_t q = ccp[c] + lane; q < ccp[c + 1]; q += 32) {
            const int32_t k = col[q];
            const int K = sizes[c];
            P += static_cast<int64_t>(live_count(mask, valid, q, vptr[c] + (q - ccp[c]) * K, K)) *
                 (brp[k + 1] - brp[k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) P += __shfl_xor_sync(0xffffffffu, P, o);
        if (lane == 0) out[c] = P;
    }
}
}  // namespace
}  // namespace bsp

extern "C" {

// Cluster-boundary split for multi-GPU cluster-wise shards:
// bounds[g] = the first cluster whose exclusive product prefix reaches
// total*g/nparts; clusters are independent (cluster_spgemm.hpp:108-109), so a
// shard is a contiguous run of clusters (CSR_Cluster order).
int bsp_partition_clusters(bsp_handle h, const bsp_csr_cluster* A, const bsp_csr* B,
                           int32_t nparts, int64_t* bounds_out) {
    return guarded([&] {
        require(A != nullptr && B != nullptr && bounds_out != nullptr,
                "partition_clusters: null argument");
        require(nparts >= 1, "partition_clusters: nparts must be >= 1");
        require(A->ncols == B->nrows, "partition_clusters: dimension mismatch");
        BSP_CUDA(cudaSetDevice(h->device));
        const int64_t ncl = A->nclusters;
        std::vector<int64_t> pc(ncl);
        if (ncl > 0) {
            DBuf<int64_t> w(h, ncl);
            BSP_LAUNCH(h, cluster_work_kernel, grid_for(h, ncl * 32, 256), 256, 0,
                       A->cluster_col_ptr, A->col_idx, A->member_mask,
                       reinterpret_cast<const unsigned long long*>(A->valid), A->value_ptr,
                       A->cluster_sizes, B->row_ptr, ncl, w.p);
            d2h(h, pc.data(), w.p, ncl);
            sync(h);
        }
        std::vector<int64_t> pre(ncl + 1, 0);
        for (int64_t c = 0; c < ncl; ++c) pre[c + 1] = pre[c] + pc[c];
        bounds_out[0] = 0;
        for (int32_t g = 1; g < nparts; ++g) {
            const int64_t target =
                static_cast<int64_t>((static_cast<__int128>(pre[ncl]) * g) / nparts);
            const int64_t c = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
            bounds_out[g] = std::max(bounds_out[g - 1], std::min<int64_t>(c, ncl));
        }
        bounds_out[nparts] = ncl;
    });
}

int bsp_csr_cluster_build(bsp_handle h, const bsp_csr* A, int64_t nclusters,
                          const int64_t* cluster_ptr, const int32_t* rows, bsp_csr_cluster* out) {
    return guarded([&] {
        check_csr(A, "build_csr_cluster");
        require(out != nullptr && (nclusters == 0 || (cluster_ptr && rows)),
                "build_csr_cluster: null argument");
        BSP_CUDA(cudaSetDevice(h->device));
        // ClusterAssignment::validate (cluster_format.hpp:34-51)
        const int64_t n = A->nrows;
        std::vector<char> seen(static_cast<size_t>(n), 0);
        require(cluster_ptr == nullptr || cluster_ptr[0] == 0, "cluster assignment: bad offsets");
        for (int64_t c = 0; c < nclusters; ++c) {
            const int64_t b = cluster_ptr[c], e = cluster_ptr[c + 1];
            require(e > b, "cluster assignment: empty cluster");
            require(e - b <= MAXK_FMT, "cluster assignment: clusters of more than 1024 rows "
                                       "are not supported by the device format");
            for (int64_t q = b; q < e; ++q) {
                const int32_t r = rows[q];
                require(r >= 0 && r < n, "cluster assignment: row index out of range");
                require(!seen[r], "cluster assignment: row assigned twice");
                seen[r] = 1;
                if (q > b) require(rows[q - 1] < r, "cluster assignment: members must be strictly increasing");
            }
        }
        for (int64_t i = 0; i < n; ++i)
            require(seen[i], "cluster assignment: row " + std::to_string(i) + " not covered");
        const int64_t total = nclusters > 0 ? cluster_ptr[nclusters] : 0;
        DBuf<int64_t> mptr(h, nclusters + 1, Pool::out);
        DBuf<int32_t> drows(h, total, Pool::out);
        if (nclusters > 0) {
            h2d(h, mptr.p, cluster_ptr, nclusters + 1);
            h2d(h, drows.p, rows, total);
        } else {
            BSP_CUDA(cudaMemsetAsync(mptr.p, 0, sizeof(int64_t), h->stream));
        }
        bsp_csr_cluster tmp{};
        build_cluster_device(h, A, nclusters, mptr.p, drows.p, true, &tmp);
        mptr.release();
        drows.release();
        *out = tmp;
        sync(h);
    });
}

int bsp_csr_cluster_free(bsp_handle h, bsp_csr_cluster* m) {
    return guarded([&] {
        require(h != nullptr || m == nullptr || !m->owned, "csr_cluster_free: null handle");
        free_cluster(h, m);
    });
}

int bsp_csr_cluster_download(bsp_handle h, const bsp_csr_cluster* m, bsp_host_csr_cluster* o) {
    return guarded([&] {
        require(m && o, "csr_cluster_download: null argument");
        o->nclusters = m->nclusters;
        o->nrows = m->nrows;
        o->ncols = m->ncols;
        o->ncolslots = m->ncolslots;
        o->nslots = m->nslots;
        o->cluster_sizes = host_malloc<int32_t>(m->nclusters);
        o->cluster_col_ptr = host_malloc<int64_t>(m->nclusters + 1);
        o->col_idx = host_malloc<int32_t>(m->ncolslots);
        o->value_ptr = host_malloc<int64_t>(m->nclusters + 1);
        o->values = host_malloc<double>(m->nslots);
        const int64_t nw = (m->nslots + 63) / 64;
        o->valid = host_malloc<uint64_t>(nw);
        o->row_map = host_malloc<int32_t>(m->nrows);
        d2h(h, o->cluster_sizes, m->cluster_sizes, m->nclusters);
        d2h(h, o->cluster_col_ptr, m->cluster_col_ptr, m->nclusters + 1);
        d2h(h, o->col_idx, m->col_idx, m->ncolslots);
        d2h(h, o->value_ptr, m->value_ptr, m->nclusters + 1);
        d2h(h, o->values, m->values, m->nslots);
        d2h(h, o->valid, m->valid, nw);
        d2h(h, o->row_map, m->row_map, m->nrows);
        sync(h);
    });
}

void bsp_host_csr_cluster_free(bsp_host_csr_cluster* m) {
    if (!m) return;
    std::free(m->cluster_sizes);
    std::free(m->cluster_col_ptr);
    std::free(m->col_idx);
    std::free(m->value_ptr);
    std::free(m->values);
    std::free(m->valid);
    std::free(m->row_map);
    *m = bsp_host_csr_cluster{};
}

int bsp_cluster_to_csr(bsp_handle h, const bsp_csr_cluster* m, bsp_csr* out) {
    return guarded([&] {
        require(m && out, "cluster_to_csr: null argument");
        BSP_CUDA(cudaSetDevice(h->device));
        cluster_to_csr_device(h, m, out);
    });
}

int bsp_spgemm_clusterwise(bsp_handle h, const bsp_csr_cluster* A, const bsp_csr* B, bsp_csr* C,
                           bsp_csr_cluster* C_cluster) {
    return guarded([&] {
        require(A && B && C, "spgemm_clusterwise: null argument");
        check_csr(B, "spgemm_clusterwise");
        require(A->ncols == B->nrows, "spgemm_clusterwise: dimension mismatch (a.ncols != b.nrows)");
        BSP_CUDA(cudaSetDevice(h->device));
        h->stats = bsp_exec_stats{};
        h->stats.chunks = 1;
        const int64_t n = A->nrows, ncl = A->nclusters;
        // Row view of A for clusters routed to the row-wise bins.
        bsp_csr acsr{};
        bsp_csr tmp_csr{};
        if (A->csr_row_ptr) {
            int64_t nnz = A->csr_nnz;  // recorded at build time (no readback)
            if (nnz <= 0) {
                d2h(h, &nnz, A->csr_row_ptr + n, 1);
                sync(h);
            }
            acsr = bsp_csr{n, A->ncols, nnz, A->csr_row_ptr, A->csr_col_idx, A->csr_values, 0};
        } else {
            cluster_to_csr_device(h, A, &tmp_csr);
            acsr = tmp_csr;
        }
        const ClusterMats cm = make_cluster_mats(A, B);
        const int cbits = bit_length(static_cast<uint32_t>(std::max<int64_t>(B->ncols - 1, 0)));
        // B with <= 64 columns and CSR output only (BSP_NARROW=0 forces the
        // tiles): every row
        // counted by the row-wise mask kernel (C's structure does not depend on
        // the clustering), tiled clusters on the cluster mask kernel, the
        // other rows on the row-wise one.
        const char* ne_env = std::getenv("BSP_NARROW");
        const Mats m = make_mats(&acsr, B);
        if (B->ncols <= 64 && !(ne_env && ne_env[0] == '0') && C_cluster == nullptr) {
            // clusters of 2..MAXK members on the cluster kernel (their rows
            // skipped by the row kernel), the rest row by row
            DBuf<uint8_t> skip(h, n);
            BSP_CUDA(cudaMemsetAsync(skip.p, 0, std::max<int64_t>(n, 1), h->stream));
            DBuf<int32_t> lists(h, std::max<int64_t>(ncl, 1));
            DBuf<unsigned long long> ccount(h, 1);
            BSP_CUDA(cudaMemsetAsync(ccount.p, 0, sizeof(unsigned long long), h->stream));
            BSP_LAUNCH(h, narrow_route_kernel, grid_for(h, ncl, 256), 256, 0, cm, ncl, skip.p,
                       lists.p, ccount.p);
            const int64_t acc = static_cast<int64_t>(read_scalar(h, ccount.p));
            DBuf<unsigned long long> bmask;
            narrow64_row_masks(h, m, B->nrows, bmask);
            DBuf<int64_t> row_nnz(h, n + 1);
            BSP_CUDA(cudaMemsetAsync(row_nnz.p, 0, (n + 1) * sizeof(int64_t), h->stream));
            DBuf<unsigned long long> prod(h, 1);
            BSP_CUDA(cudaMemsetAsync(prod.p, 0, sizeof(unsigned long long), h->stream));
            narrow64_rows(h, m, bmask.p, n, nullptr, row_nnz.p, nullptr, nullptr, nullptr, prod.p);
            DBuf<int64_t> rp(h, n + 1, Pool::out);
            exclusive_scan_i64(h, row_nnz.p, rp.p, n + 1);
            const int64_t nnz = read_scalar(h, rp.p + n);
            h->stats.products = static_cast<int64_t>(read_scalar(h, prod.p));
            h->stats.nnz_out = nnz;
            h->stats.units[10] = acc;
            ResultPayload pay(h, nnz);
            // the cluster kernel on the side stream: the row kernel's tail (hub
            // rows) leaves SMs idle that it fills (disjoint rows of C)
            if (acc > 0) {
                SideStream side(h);
                BSP_LAUNCH_AS(h, "cluster_narrow64", cluster_narrow64_kernel,
                              grid_for(h, div_up(acc, CN_WARPS), 1), CN_WARPS * 32, 0, cm, bmask.p,
                              lists.p, acc, rp.p, pay.col_idx(), pay.values());
            }
            narrow64_rows(h, m, bmask.p, n, skip.p, nullptr, rp.p, pay.col_idx(), pay.values(),
                          nullptr);
            if (acc > 0) join_side(h);
            C->nrows = n;
            C->ncols = B->ncols;
            C->nnz = nnz;
            C->row_ptr = rp.release();
            C->col_idx = pay.col_idx();
            C->values = pay.block.release();
            C->owned = 2;
            if (tmp_csr.owned) {
                dfree(h, tmp_csr.row_ptr);
                dfree(h, tmp_csr.col_idx);
                dfree(h, tmp_csr.values);
            }
            return;
        }

        DBuf<uint8_t> ccls(h, ncl);
        DBuf<uint8_t> skip(h, n);
        BSP_CUDA(cudaMemsetAsync(skip.p, 0, std::max<int64_t>(n, 1), h->stream));
        DBuf<unsigned long long> counts(h, NCC);
        BSP_CUDA(cudaMemsetAsync(counts.p, 0, NCC * sizeof(unsigned long long), h->stream));
        // BSP_CLUSTER_UNION=0: member-keyed tiles only
        const char* ue = std::getenv("BSP_CLUSTER_UNION");
        const int union_ok = (ue && ue[0] == '0') ? 0 : (union_tma(cm) ? 2 : 1);
        // BSP_CLUSTER_MIN_REUSE (x10, default 15 = 1.5x): clusters sharing less go row-wise
        static const int min_reuse10 = [] {
            const char* e = std::getenv("BSP_CLUSTER_MIN_REUSE");
            return e ? std::atoi(e) : 15;
        }();
        BSP_LAUNCH(h, cluster_products_kernel, grid_for(h, ncl, 256), 256, 0, cm, ncl, cbits, ccls.p,
                   skip.p, counts.p, union_ok, min_reuse10);
        unsigned long long hc[NCC];
        d2h(h, hc, counts.p, NCC);
        sync(h);
        int64_t off[NCC], cnt[NCC];
        int64_t acc = 0;
        for (int c = 0; c < NCC; ++c) {
            cnt[c] = static_cast<int64_t>(hc[c]);
            off[c] = acc;
            if (c > 0) acc += cnt[c];
        }
        DBuf<int32_t> lists(h, acc);
        if (acc > 0) {
            DBuf<unsigned long long> cursor(h, NCC);
            std::vector<unsigned long long> cur(NCC, 0);
            for (int c = 1; c < NCC; ++c) cur[c] = static_cast<unsigned long long>(off[c]);
            h2d(h, cursor.p, cur.data(), NCC);
            BSP_LAUNCH(h, cluster_bucket_kernel, grid_for(h, ncl, 256), 256, 0, ccls.p, ncl,
                       cursor.p, lists.p);
        }
        RowwisePlan plan;    // rows outside cluster tiles (incl. heavy windows)
        RowwisePlan plan_c;  // the cluster tiles' rows, for their symbolic counts
        build_plan(h, m, 0, n, skip.p, plan, nullptr, nullptr, &plan_c);
        for (int c = 0; c < NCLS; ++c) h->stats.products += plan_c.class_products[c];  // + cluster rows
        h->stats.units[10] = acc;  // cluster tiles (member-keyed + union)
        h->stats.units[11] = cnt[6] + cnt[7];  // of which union tiles
        DBuf<int64_t> row_nnz(h, n + 1);
        BSP_CUDA(cudaMemsetAsync(row_nnz.p, 0, (n + 1) * sizeof(int64_t), h->stream));
        // Symbolic: C's row structure does not depend on the clustering, so the
        // cluster rows are counted by the (cheaper) row-wise hash tiles of the
        // shadow plan built in the same pass.
        {
            DBuf<int64_t> wn_c;
            plan_symbolic(h, m, plan_c, row_nnz.p, wn_c);
        }
        // the union tiles' rows: counted from each cluster's B rows loaded once
        if (cnt[6] > 0)
            BSP_LAUNCH_AS(h, "cluster_union_count<128,2048>", (cluster_union_count_kernel<128, 2048>),
                          static_cast<unsigned>(cnt[6]), 128, 0, cm, lists.p + off[6], row_nnz.p);
        if (cnt[7] > 0)
            BSP_LAUNCH_AS(h, "cluster_union_count<256,4096>", (cluster_union_count_kernel<256, 4096>),
                          static_cast<unsigned>(cnt[7]), 256, 0, cm, lists.p + off[7], row_nnz.p);
        DBuf<int64_t> win_nnz;
        plan_symbolic(h, m, plan, row_nnz.p, win_nnz);
        DBuf<int64_t> rp(h, n + 1, Pool::out);
        exclusive_scan_i64(h, row_nnz.p, rp.p, n + 1);
        DBuf<int64_t> win_scan(h, plan.nwin + 1);
        if (plan.nwin > 0) exclusive_scan_i64(h, win_nnz.p, win_scan.p, plan.nwin + 1);
        const int64_t nnz = read_scalar(h, rp.p + n);
        h->stats.nnz_out = nnz;
        ResultPayload pay(h, nnz);
        // duplicate-heavy two-row clusters -> the cluster hash accumulator
        // (only when columns repeat overall: compression factor >= 1.25, as
        // the row-wise routing; BSP_HACC=0 disables)
        const char* he = std::getenv("BSP_HACC");
        const bool repeats = 4 * h->stats.products >= 5 * std::max<int64_t>(1, nnz);
        if (acc > 0 && repeats && !(he && he[0] == '0')) {
            DBuf<int32_t> hl(h, acc), tl(h, acc), rl(h, std::max<int64_t>(n, 1));
            DBuf<unsigned long long> cur(h, NCC + 1);
            std::vector<unsigned long long> cu(NCC + 1, 0);
            for (int c = 1; c < NCC; ++c) cu[c] = static_cast<unsigned long long>(off[c] - off[1]);
            h2d(h, cur.p, cu.data(), NCC + 1);
            // BSP_CLUSTER_HACC_REUSE (x10, default 20 = 2.0x): B-row reuse a two-row
            // cluster needs for the cluster accumulator (below: row-wise accumulator)
            static const int hacc_reuse10 = [] {
                const char* e = std::getenv("BSP_CLUSTER_HACC_REUSE");
                return e ? std::atoi(e) : 20;
            }();
            BSP_LAUNCH(h, route_cluster_kernel, static_cast<unsigned>(div_up(acc, 256)), 256, 0, cm,
                       lists.p + off[1], ccls.p, acc, rp.p, cur.p, hl.p, tl.p, rl.p, hacc_reuse10);
            unsigned long long hc2[NCC + 1];
            d2h(h, hc2, cur.p, NCC + 1);
            sync(h);
            const int64_t nh = static_cast<int64_t>(hc2[0]);
            const int64_t nr = static_cast<int64_t>(hc2[NCC]);
            int64_t off2[NCC], cnt2[NCC];
            for (int c = 0; c < NCC; ++c) {
                off2[c] = c == 0 ? 0 : off[c] - off[1];
                cnt2[c] = c == 0 ? 0 : static_cast<int64_t>(hc2[c]) - off2[c];
            }
            if (nh > 0) {
                set_smem(cluster_hashacc_kernel, sizeof(ClusterHaccShared));
                const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
                    1, std::min<int64_t>(div_up(nh, CH_WARPS), int64_t{h->sm_count} * 32)));
                BSP_LAUNCH(h, cluster_hashacc_kernel, grid, CH_WARPS * 32, sizeof(ClusterHaccShared),
                           cm, hl.p, nh, rp.p, pay.col_idx(), pay.values());
            }
            if (nr > 0) {
                sort_ids(h, rl.p, nr);  // row order: neighbouring rows share B rows in L2
                run_hashacc_rows(h, m, rl.p, nr, 0, rp.p, pay.col_idx(), pay.values());
            }
            h->stats.units[13] = nr;  // cluster rows on the row-wise accumulator
            h->stats.units[12] = nh;
            run_cluster_classes(h, cm, tl.p, off2, cnt2, cbits, rp.p, pay.col_idx(), pay.values());
        } else {
            run_cluster_classes(h, cm, lists.p, off, cnt, cbits, rp.p, pay.col_idx(), pay.values());
        }
        plan_numeric(h, m, plan, rp.p, win_scan.p, pay.col_idx(), pay.values());
        C->nrows = n;
        C->ncols = B->ncols;
        C->nnz = nnz;
        C->row_ptr = rp.release();
        C->col_idx = pay.col_idx();
        C->values = pay.block.release();
        C->owned = 2;
        if (tmp_csr.owned) {
            dfree(h, tmp_csr.row_ptr);
            dfree(h, tmp_csr.col_idx);
            dfree(h, tmp_csr.values);
        }
        if (C_cluster) {
            // C's cluster form = build_csr_cluster(C, A's assignment)
            // (same sizes/row_map; union of members' output columns).
            DBuf<int64_t> mptr(h, ncl + 1, Pool::out);
            DBuf<int32_t> rows(h, n, Pool::out);
            BSP_CUDA(cudaMemcpyAsync(mptr.p, A->member_ptr, (ncl + 1) * sizeof(int64_t),
                                     cudaMemcpyDeviceToDevice, h->stream));
            BSP_CUDA(cudaMemcpyAsync(rows.p, A->row_map, n * sizeof(int32_t),
                                     cudaMemcpyDeviceToDevice, h->stream));
            bsp_csr_cluster cc{};
            build_cluster_device(h, C, ncl, mptr.p, rows.p, false, &cc);
            mptr.release();
            rows.release();
            *C_cluster = cc;
        }
    });
}

int bsp_cluster_access_stats(bsp_handle h, const bsp_csr_cluster* A, const bsp_csr* B,
                             bsp_access_stats* out) {
    return guarded([&] {
        require(A && B && out, "cluster_access_stats: null argument");
        require(A->ncols == B->nrows, "rowwise_access_stats: dimension mismatch");
        DBuf<unsigned long long> acc(h, 3);
        BSP_CUDA(cudaMemsetAsync(acc.p, 0, 3 * sizeof(unsigned long long), h->stream));
        BSP_LAUNCH(h, cluster_stats_kernel, grid_for(h, A->nclusters, 256), 256, 0,
                   A->cluster_sizes, A->cluster_col_ptr, A->col_idx, A->member_mask,
                   reinterpret_cast<const unsigned long long*>(A->valid), A->value_ptr, B->row_ptr,
                   A->nclusters, acc.p);
        unsigned long long r[3];
        d2h(h, r, acc.p, 3);
        sync(h);
        out->b_row_loads = r[0];
        out->a_inner_iters = r[1];
        out->placeholder_skips = r[2];
    });
}

int bsp_rowwise_access_stats(bsp_handle h, const bsp_csr* A, const bsp_csr* B,
                             bsp_access_stats* out) {
    return guarded([&] {
        check_csr(A, "rowwise_access_stats");
        require(A->ncols == B->nrows, "rowwise_access_stats: dimension mismatch");
        DBuf<unsigned long long> acc(h, 3);
        BSP_CUDA(cudaMemsetAsync(acc.p, 0, 3 * sizeof(unsigned long long), h->stream));
        BSP_LAUNCH(h, rowwise_stats_kernel, grid_for(h, A->nnz, 256), 256, 0, A->col_idx, A->nnz,
                   B->row_ptr, acc.p);
        unsigned long long r[3];
        d2h(h, r, acc.p, 3);
        sync(h);
        out->b_row_loads = r[0];
        out->a_inner_iters = r[1];
        out->placeholder_skips = 0;
    });
}

}  // extern "C"
